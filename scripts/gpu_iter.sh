#!/bin/bash
# Iteration pass: GPU parity (stop at first failure), then bench variants.
# usage: bash scripts/gpu_iter.sh "ENV1=a ENV2=b" "ENV1=c" ...
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
i=0
for v in "$@"; do
  env $v SAAP_DECODE_TRACE=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_v$i.json 2> gpurun_out/bench_v$i.err
  cp gpurun_out/decode_trace.npy gpurun_out/decode_trace_v$i.npy 2>/dev/null
  python - "$v" gpurun_out/bench_v$i.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(sys.argv[1], "| step", d["value"], "| dense", d["dense_us_per_step"], "| kern", d["kernel_us"], "| frac", d["roofline"]["frac"], "| e2e", d["e2e"]["value"], "| trace", d["decode_trace"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  tail -2 gpurun_out/bench_v$i.err
  i=$((i+1))
done
