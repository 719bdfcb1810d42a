#!/bin/bash
# Round-1 GPU evidence pass: parity tests, smoke, bench line, reference arm,
# ncu launch list and full captures of the step's kernels (C3 layer).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
SAAP_STEP_TRACE=1 SAAP_DECODE_TRACE=1 SAAP_PLAN_TRACE=1 timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_trace.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"saap_b200" -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --layers 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|combine|route_cluster" -s 12 -c 6 -o gpurun_out/prof_step python bench.py --steps 3 --warmup 3 --layers 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"assign_tc|refine|scatter|move_rows|hist|scan" -c 8 -o gpurun_out/prof_build python bench.py --steps 2 --warmup 3 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
ls gpurun_out
