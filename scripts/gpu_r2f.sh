#!/bin/bash
mkdir -p gpurun_out
touch paper_2502_08246_b200/csrc/decode.cu; make -C paper_2502_08246_b200 NVFLAGS_EXTRA=-DSAAP_NO_TMA > gpurun_out/r2f_make.log 2>&1; tail -2 gpurun_out/r2f_make.log
for o in "" "--dense"; do
  echo "== NO_TMA $o"; timeout 300 python scripts/trace_step.py $o --reps 10 --out gpurun_out/r2f_trace.json 2>&1 | tail -1
done
