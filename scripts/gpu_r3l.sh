#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assign_tc.py tests/test_gpu_parity.py tests/test_gpu_c3.py tests/test_gpu_append.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
timeout 1500 python bench.py --no-imbalanced --no-cpu-baseline > gpurun_out/r3l_bench.json 2> gpurun_out/r3l_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r3l_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['traffic_same_build'], json.dumps(d['prefill']))"; tail -2 gpurun_out/r3l_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"route_cluster|decode_kernel|combine_kernel" -c 12 --csv --log-file gpurun_out/r3l_step_launches.csv python bench.py --steps 2 --warmup 1 --layers 1 --no-imbalanced --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:assign_tc_kernel -c 1 -o gpurun_out/r3l_assign python bench.py --steps 2 --warmup 1 --layers 1 --no-imbalanced --no-cpu-baseline --no-dense > /dev/null 2>&1; ls gpurun_out/r3l_assign*
