#!/bin/bash
# A/B of two library builds (abtest/lib_A.so, abtest/lib_B.so) on the Q-model routed step
for r in 1 2 3; do for v in A B; do
  cp abtest/lib_$v.so paper_2502_08246_b200/libsaap_b200.so
  echo "$v $(timeout 300 python bench.py --router qmodel --steps 200 --warmup 10 --no-cpu-baseline --no-dense --no-c1 --no-qmodel --no-imbalanced 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("kernel_us"))')"
done; done
