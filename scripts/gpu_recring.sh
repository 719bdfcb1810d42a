#!/bin/bash
# Build-time knob sweep (record ring depth) on the GPU box: rebuild, bench.
for r in 3 5 8; do
  touch paper_2502_08246_b200/csrc/decode.cu
  make -C paper_2502_08246_b200 NVFLAGS_EXTRA=-DSAAP_REC_RING=$r > /dev/null 2>&1 || { echo build failed $r; continue; }
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/rr.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rr.json')); print('rec_ring', $r, d['value'], d['kernel_us'], d['roofline']['frac'])"
done
