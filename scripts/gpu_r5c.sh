#!/bin/bash
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_stream.py tests/test_gpu_c3.py tests/test_gpu_parity.py 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py "" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --given "" 2>&1 | tail -1
timeout 300 python scripts/sweep_opts.py --dense "" 2>&1 | tail -1
