set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -8
SAAP_PLAN_TRACE=1 timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench10.json 2> gpurun_out/bench10.err; tail -3 gpurun_out/bench10.err; cat gpurun_out/bench10.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|route_|combine" -s 8 -c 4 -o gpurun_out/prof_decode10 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches10.csv python bench.py --steps 3 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
ls -la gpurun_out | tail -3
