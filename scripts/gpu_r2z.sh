#!/bin/bash
echo dense2048; timeout 300 python scripts/sweep_opts.py --dense --ctx-len 2048 "" 2>&1 | tail -1
echo dense8192; timeout 300 python scripts/sweep_opts.py --dense --ctx-len 8192 "" 2>&1 | tail -1
echo sparse4096-window; timeout 300 python scripts/sweep_opts.py --ctx-len 4096 --probes 0 "" 2>&1 | tail -1
echo given-probes0; timeout 300 python scripts/sweep_opts.py --given --probes 0 "" 2>&1 | tail -1
