#!/bin/bash
mkdir -p gpurun_out
for o in "" "--opt chunk=16" "--opt chunk=4" "--dense"; do
  echo "== $o"; timeout 300 python scripts/trace_step.py $o --reps 10 --out gpurun_out/r2e_trace.json 2>&1 | tail -1
done
