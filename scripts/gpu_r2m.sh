#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/trace_step.py --given --reps 6 --out gpurun_out/r2m_given.json > gpurun_out/r2m_given.log 2>&1; tail -1 gpurun_out/r2m_given.log
timeout 600 python scripts/trace_step.py --dense --reps 3 --out gpurun_out/r2m_dense.json > gpurun_out/r2m_dense.log 2>&1; tail -1 gpurun_out/r2m_dense.log
timeout 900 python -m pytest tests/test_gpu_ref_suite.py -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -3
