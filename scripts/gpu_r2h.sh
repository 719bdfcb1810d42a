#!/bin/bash
# round 2 (re-entry): full GPU suite, smoke, C3 bench with parity
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt; nvidia-smi -L >> gpurun_out/host.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/r2h_pytest_gpu.log 2>&1; tail -15 gpurun_out/r2h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; tail -3 gpurun_out/r2h_smoke.log
timeout 1200 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; tail -c 6000 gpurun_out/r2h_bench.json; tail -5 gpurun_out/r2h_bench.err
