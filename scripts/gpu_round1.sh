set -x
./scripts/fp64_probe
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -8
SAAP_PLAN_TRACE=1 SAAP_DECODE_TRACE=1 timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench11.json 2> gpurun_out/bench11.err; tail -3 gpurun_out/bench11.err; cat gpurun_out/bench11.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|route_|combine" -s 8 -c 4 -o gpurun_out/prof_decode11 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"refine|scatter|scan_" -c 6 -o gpurun_out/prof_build11 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
ls -la gpurun_out | tail -3
