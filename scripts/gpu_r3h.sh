#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qm_|route_plan|decode|combine" -c 40 --csv --log-file gpurun_out/r3h_qm_launches.csv python bench.py --router qmodel --steps 2 --warmup 1 --layers 1 --no-imbalanced --no-cpu-baseline --no-dense > gpurun_out/r3h_qm.log 2>&1; tail -2 gpurun_out/r3h_qm.log
python scripts/ncu_lines.py gpurun_out/r3h_qm_launches.csv 2>/dev/null | tail -30 || grep -E "qm_|route_plan" gpurun_out/r3h_qm_launches.csv | head -30
