#!/bin/bash
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_kmeans.py tests/test_gpu_assign_tc.py tests/test_gpu_append.py 2>&1 | tail -2
timeout 900 python bench.py --steps 30 --warmup 5 --no-imbalanced --no-cpu-baseline --no-c1 --no-qmodel > gpurun_out/r4t_bench.json 2> gpurun_out/r4t_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r4t_bench.json').read().strip().splitlines()[-1]); print(d['value'], json.dumps(d['prefill']))"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"scatter|move_rows|hist_kernel|scan_" -c 8 --csv --log-file gpurun_out/r4t_pack.csv python bench.py --steps 2 --warmup 1 --layers 1 --no-imbalanced --no-cpu-baseline --no-c1 --no-qmodel --no-dense > /dev/null 2>&1; grep -c . gpurun_out/r4t_pack.csv
