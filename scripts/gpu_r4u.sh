#!/bin/bash
timeout 900 python bench.py --steps 30 --warmup 5 --no-imbalanced --no-cpu-baseline --no-c1 --no-qmodel > gpurun_out/r4u_bench.json 2> gpurun_out/r4u_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r4u_bench.json').read().strip().splitlines()[-1]); print(d['value'], json.dumps(d['prefill']))"
