#!/bin/bash
# A/B of Q-model logits geometry (build knobs), bench --router qmodel
mkdir -p gpurun_out
for f in "-DSAAP_QM_TL=128" "-DSAAP_QM_TL=256" "-DSAAP_QM_TL=64" "-DSAAP_QM_TL=256 -DSAAP_QM_SLOT=4"; do
  touch paper_2502_08246_b200/csrc/route.cu paper_2502_08246_b200/csrc/capi.cu
  make -C paper_2502_08246_b200 NVFLAGS_EXTRA="$f" > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $f"; continue; }
  timeout 300 python bench.py --router qmodel --steps 50 --no-cpu-baseline --no-dense > gpurun_out/ab.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(repr(sys.argv[1]), d['value'], d['kernel_us'])" "$f" || echo "bench failed: $f"
done
