#!/bin/bash
# final round-2 evidence: bench (default), Q-model line, C1-scale sanity, ncu launch list + full capture of decode
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r3k_bench.json 2> gpurun_out/r3k_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r3k_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['kernel_us'], d['roofline']['frac'], d['parity']['pass'], d['imbalanced']['us_per_step'], d['prefill']['c4'])"; tail -2 gpurun_out/r3k_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/r3k_launches.csv python bench.py --steps 2 --warmup 1 --layers 1 --no-imbalanced --no-cpu-baseline > /dev/null 2>&1; tail -3 gpurun_out/r3k_launches.csv | cut -c1-200
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 6 -c 1 -o gpurun_out/r3k_decode python scripts/trace_step.py --plain --reps 8 > gpurun_out/r3k_ncu.log 2>&1; tail -2 gpurun_out/r3k_ncu.log
