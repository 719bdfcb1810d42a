set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -8
SAAP_PLAN_TRACE=1 timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -3 gpurun_out/bench9.err; cat gpurun_out/bench9.json
timeout 600 ncu --set full --clock-control none -k regex:"assign_tc|refine|move_rows|scatter|hist|scan" -c 8 -o gpurun_out/prof_build9 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
ls -la gpurun_out | tail -3
