#!/bin/bash
# round 2: bench restructure smoke (small), host facts
mkdir -p gpurun_out
nproc > gpurun_out/r2b_host.txt; free -g >> gpurun_out/r2b_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r2b_host.txt
timeout 600 python bench.py --ctx-len 32768 --batch 2 --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; tail -c 4000 gpurun_out/r2b_bench.json; tail -20 gpurun_out/r2b_bench.err
cat gpurun_out/r2b_host.txt
