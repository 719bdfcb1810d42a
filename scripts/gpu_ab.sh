#!/bin/bash
# A/B of a build-time knob: bash scripts/gpu_ab.sh "FLAGS_A" "FLAGS_B" (NVFLAGS_EXTRA values)
mkdir -p gpurun_out
for rep in 1 2; do
  for f in "$1" "$2"; do
    touch paper_2502_08246_b200/csrc/decode.cu
    make -C paper_2502_08246_b200 NVFLAGS_EXTRA="$f" > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $f"; tail -3 gpurun_out/ab_build.log; continue; }
    timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(repr(sys.argv[1]), d['value'], d['kernel_us']['sparse_attention'], d['roofline']['frac'])" "$f" || echo "bench failed: $f"
  done
done
