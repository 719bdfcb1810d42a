#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/trace_step.py --out gpurun_out/r2k_trace.json > gpurun_out/r2k_trace.log 2>&1; tail -1 gpurun_out/r2k_trace.log
python -c "
import json; j=json.load(open('gpurun_out/r2k_trace.json'))
for s in j['steps'][:3]: print(s.get('route_slowest'))
"
timeout 600 python scripts/trace_step.py --given --out gpurun_out/r2k_trace_given.json > gpurun_out/r2k_trace_given.log 2>&1; tail -1 gpurun_out/r2k_trace_given.log
