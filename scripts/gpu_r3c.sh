#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r3c_bench.json 2> gpurun_out/r3c_bench.err; tail -c 3500 gpurun_out/r3c_bench.json; tail -3 gpurun_out/r3c_bench.err
