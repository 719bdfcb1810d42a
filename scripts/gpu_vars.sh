#!/bin/bash
# Bench variants (env settings) on C3 and C2, untraced, plus the traced routing phases.
# usage: bash scripts/gpu_vars.sh "ENV1=a ENV2=b" "ENV1=c" ...
mkdir -p gpurun_out
for v in "$@"; do
  for cfg in "" "--batch 1 --ctx-len 32768 --layers 8"; do
    env $v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-dense $cfg > gpurun_out/v.json 2> gpurun_out/v.err
    env $v SAAP_STEP_TRACE=1 SAAP_PLAN_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dense $cfg > gpurun_out/vt.json 2>> gpurun_out/v.err
    python - "$v" "$cfg" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/v.json")); t = json.load(open("gpurun_out/vt.json"))
    g = t["graph_plan_trace"]; st = t["step_trace_us"]
    print(sys.argv[1], "|", sys.argv[2] or "C3", "| step", d["value"], "| e2e", d["e2e"]["value"], "| frac", d["roofline"]["frac"],
          "| plan", g[0], g[1]["end_us"], "| comb", st["combine"][1], st["run_published"][1])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
  tail -1 gpurun_out/v.err
done
