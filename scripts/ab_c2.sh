#!/bin/bash
for r in 1 2; do
  for v in A B; do
    cp abtest/lib_$v.so paper_2502_08246_b200/libsaap_b200.so
    echo "$v $(timeout 300 python scripts/sweep_opts.py --ctx-len 32768 --batch 1 --steps 300 "" 2>&1 | tail -1)"
  done
done
