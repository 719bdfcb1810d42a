#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sweep_opts.py "" "chunk=4" "chunk=6" 2>&1 | tail -1
timeout 300 python scripts/trace_step.py --reps 6 --out gpurun_out/r2v_route.json > gpurun_out/r2v_route.log 2>&1; tail -1 gpurun_out/r2v_route.log
python -c "
import json; j=json.load(open('gpurun_out/r2v_route.json'))
for s in j['steps'][:3]: print(s.get('route_slowest'), s.get('route_candidates'), s.get('route_cta'))
"
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_c3.py tests/test_gpu_regressions.py -q -x --timeout 400 -p no:cacheprovider 2>&1 | tail -3
