set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -15
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -3 gpurun_out/bench4.err; cat gpurun_out/bench4.json
for it in 1 4 8; do SAAP_ITEM_TILES=$it timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-dense --layers 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('item_tiles=$it', d['value'], d['kernel_us'], d['roofline']['frac'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|route_score" -s 3 -c 2 -o gpurun_out/prof_decode4 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches4.csv python bench.py --steps 5 --warmup 2 --layers 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
