#!/bin/bash
# Round-end evidence: parity suite, smoke, bench lines (centroid + Q-model
# routers, reference arm), launch list of the default step.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.err
timeout 600 python bench.py --router qmodel --no-cpu-baseline > gpurun_out/bench_qmodel.json 2> gpurun_out/bench_qmodel.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|combine|route_|qm_" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --layers 1 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import json
for f in ("bench", "bench_qmodel", "bench_ref"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, d["value"], d.get("e2e", {}).get("value"), (d.get("roofline") or {}).get("frac"), d.get("kernel_us"), d.get("clocks"))
    except Exception as e:
        print(f, "FAILED", e)
PY
