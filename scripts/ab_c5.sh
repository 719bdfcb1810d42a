#!/bin/bash
for r in 1 2; do
  for v in A B; do
    cp abtest/lib_$v.so paper_2502_08246_b200/libsaap_b200.so
    echo "$v $(timeout 300 python scripts/c5_sweep.py --buckets 1024,4096,16384 --probes 8,32 2>/dev/null | python -c "
import json,sys
out=[]
for l in sys.stdin:
    r=json.loads(l)
    if r['kind']=='saap': out.append('C%d/l%d %.1f' % (r['C'], r['l'], r['us']))
print('  '.join(out))")"
  done
done
