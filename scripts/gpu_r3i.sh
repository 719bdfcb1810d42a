#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_regressions.py tests/test_gpu_qtrain.py tests/test_gpu_ref_suite.py -q -x --timeout 600 -p no:cacheprovider -k "qmodel or QModel or batched or router or ref_suite" 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qm_|route_plan|decode|combine" -c 12 --csv --log-file gpurun_out/r3i_qm_launches.csv python bench.py --router qmodel --steps 2 --warmup 1 --layers 1 --no-imbalanced --no-cpu-baseline --no-dense > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r3i_qm_launches.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum': print(d['ID'], d['Kernel Name'][:40], d['Metric Value'])
PY
timeout 900 python bench.py --router qmodel --no-imbalanced --no-cpu-baseline > gpurun_out/r3i_qm_bench.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r3i_qm_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['kernel_us'], d['dense_us_per_step'])"
