for r in 1 2; do for v in 0 1 2 3 4 5 6 7; do
echo "qm_logits=$v $(timeout 300 python bench.py --router qmodel --steps 200 --warmup 10 --no-cpu-baseline --no-dense --no-c1 --no-qmodel --no-imbalanced --opt qm_logits=$v 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("kernel_us"))')"
done; done
