#!/bin/bash
# Trace pass: step timeline, routing phases and decode CTA trace for C3 and C2.
mkdir -p gpurun_out
for cfg in "" "--batch 1 --ctx-len 32768 --layers 8"; do
  SAAP_STEP_TRACE=1 SAAP_PLAN_TRACE=1 SAAP_DECODE_TRACE=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-dense $cfg > gpurun_out/trace.json 2> gpurun_out/trace.err
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/trace.json"))
print("cfg", sys.argv[1], "step", d["value"], "kern", d["kernel_us"])
for k in ["plan_trace_cycles", "step_trace_us", "graph_plan_trace", "decode_trace"]:
    print(k, json.dumps(d.get(k)))
PY
  tail -2 gpurun_out/trace.err
done
