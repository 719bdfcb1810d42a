#!/bin/bash
for r in 1 2; do
  for v in A B; do
    cp abtest/lib_$v.so paper_2502_08246_b200/libsaap_b200.so
    echo "$v C3 $(timeout 300 python scripts/sweep_opts.py --steps 300 "" 2>&1 | tail -1)  C2 $(timeout 300 python scripts/sweep_opts.py --batch 1 --ctx-len 32768 --steps 300 "" 2>&1 | tail -1)  dense $(timeout 300 python scripts/sweep_opts.py --dense --steps 30 "" 2>&1 | tail -1)"
  done
done
