for cfg in "--batch 1 --ctx-len 32768 --layers 8" ""; do
SAAP_TRACE_DENSE=1 SAAP_STEP_TRACE=1 SAAP_DECODE_TRACE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $cfg > gpurun_out/dt.json 2> gpurun_out/dt.err
python -c "
import json;d=json.load(open('gpurun_out/dt.json'))
print(d['dense_us_per_step'], d['kernel_us'], d['roofline'].get('dense_achieved'))
print(json.dumps(d['step_trace_us'])); print(json.dumps(d['decode_trace']))"
tail -1 gpurun_out/dt.err
done
