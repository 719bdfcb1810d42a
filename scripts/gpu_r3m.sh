#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assign_tc.py tests/test_gpu_parity.py tests/test_gpu_c3.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
timeout 1500 python bench.py --no-imbalanced --no-cpu-baseline > gpurun_out/r3m_bench.json 2> gpurun_out/r3m_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r3m_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], json.dumps(d['prefill']), json.dumps(d['c1']))"; tail -2 gpurun_out/r3m_bench.err
