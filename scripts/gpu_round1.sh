set -x
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -15
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|route_plan" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --layers 2 --no-cpu-baseline > /dev/null 2>&1; tail -5 gpurun_out/launches.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 2 -o gpurun_out/prof_decode python bench.py --steps 3 --warmup 1 --layers 1 --no-cpu-baseline --no-dense > /dev/null 2>&1; ls -la gpurun_out
