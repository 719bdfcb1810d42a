#!/bin/bash
# Knob sweep: bench step time per env variant (no parity run).
mkdir -p gpurun_out
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/knob.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/knob.json"))
    print(sys.argv[1] or "default", "| step", d["value"], "| kern", d["kernel_us"], "| frac", d["roofline"]["frac"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
