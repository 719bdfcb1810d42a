#!/bin/bash
# Round-1 evidence refresh (after k-means / artifacts / Q-model training and
# the host graph cache): bench line, reference arm, launch list, ncu captures
# of the decode step and of the new offline kernels.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"saap_b200" -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --layers 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|combine|route_cluster" -s 12 -c 6 -o gpurun_out/prof_step python bench.py --steps 3 --warmup 3 --layers 1 --no-cpu-baseline > /dev/null 2>&1
KM_CASES=0 timeout 600 ncu --set full --clock-control none -k regex:"km_" -s 7 -c 6 -o gpurun_out/prof_kmeans python scripts/kmeans_timing.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"qt_" -s 40 -c 14 -o gpurun_out/prof_qtrain python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'scripts')
import qtrain_timing as q; q.main(steps=3, ref_steps=1)" > /dev/null 2>&1
ls gpurun_out
