#!/bin/bash
# round-2 final evidence: full GPU suite, bench, step launch list, decode + route ncu captures
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r5n_pytest.log 2>&1; tail -2 gpurun_out/r5n_pytest.log
timeout 1500 python bench.py > gpurun_out/r5n_bench.json 2> gpurun_out/r5n_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r5n_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('kernel_us'), d['roofline']['frac'], d['parity']['pass'], d['imbalanced']['us_per_step'], d['qmodel']['us_per_step'], d['prefill']['pack_frac'], d['clocks'])"; tail -2 gpurun_out/r5n_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"route_cluster|decode_kernel|combine_kernel" -c 12 --csv --log-file gpurun_out/r5n_step_launches.csv python bench.py --steps 2 --warmup 1 --layers 1 --no-imbalanced --no-cpu-baseline --no-c1 --no-qmodel --no-dense > /dev/null 2>&1; tail -2 gpurun_out/r5n_step_launches.csv | cut -c1-150
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 6 -c 1 -o gpurun_out/r5n_decode python scripts/trace_step.py --plain --reps 8 > gpurun_out/r5n_ncu.log 2>&1; tail -1 gpurun_out/r5n_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:route_cluster -s 6 -c 1 -o gpurun_out/r5n_route python scripts/trace_step.py --plain --reps 8 > gpurun_out/r5n_ncu2.log 2>&1; tail -1 gpurun_out/r5n_ncu2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r5n_ref.json 2> gpurun_out/r5n_ref.err; tail -c 400 gpurun_out/r5n_ref.json
timeout 900 python bench.py --ctx-len 32768 --batch 1 --steps 100 --no-imbalanced --no-cpu-baseline --no-c1 --no-qmodel > gpurun_out/r5n_c2.json 2> gpurun_out/r5n_c2.err; tail -c 300 gpurun_out/r5n_c2.json
timeout 1800 python scripts/c5_sweep.py > gpurun_out/r5n_c5.jsonl 2> gpurun_out/r5n_c5.err; wc -l gpurun_out/r5n_c5.jsonl
