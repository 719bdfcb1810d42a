set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -25
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -5 gpurun_out/bench3.err; cat gpurun_out/bench3.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/prof_decode3 python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|route_" -c 60 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 5 --warmup 2 --layers 2 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
