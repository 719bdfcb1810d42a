set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -5
SAAP_PLAN_TRACE=1 timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; tail -3 gpurun_out/bench8.err; cat gpurun_out/bench8.json
for it in 2 8; do SAAP_ITEM_TILES=$it timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-dense --layers 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('item_tiles=$it', d['value'], d['kernel_us'], d['roofline']['frac'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|route_|combine" -s 6 -c 4 -o gpurun_out/prof_decode8 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"assign_tc|move_rows|scatter" -c 3 -o gpurun_out/prof_build8 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
ls -la gpurun_out
