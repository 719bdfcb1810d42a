set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -15
SAAP_PLAN_TRACE=1 timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -3 gpurun_out/bench7.err; cat gpurun_out/bench7.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|route_" -s 6 -c 3 -o gpurun_out/prof_decode7 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
ls -la gpurun_out
