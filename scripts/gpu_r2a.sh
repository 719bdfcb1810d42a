#!/bin/bash
# round 2: regression tests + baseline bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_regressions.py -q --timeout 200 -p no:cacheprovider > gpurun_out/r2a_regr.log 2>&1; tail -15 gpurun_out/r2a_regr.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -c 3000 gpurun_out/r2a_bench.json; tail -5 gpurun_out/r2a_bench.err
