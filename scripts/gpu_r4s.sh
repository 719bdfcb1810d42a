#!/bin/bash
cat > /tmp/qm_sweep.py <<'PY'
import sys, os, argparse, json
sys.path.insert(0, os.getcwd())
import bench
import torch, numpy as np
import paper_2502_08246_b200 as sb
a = argparse.Namespace(ctx_len=131072, batch=8, kv_heads=8, q_heads=32, dim=128, buckets=1024, probes=32, recent=2047, sink=1, kmeans_iters=10)
dev = torch.device("cuda", 0); stream = torch.cuda.Stream(); ctx = sb.Context(0); ctx.set_stream(stream.cuda_stream)
d, C = 128, 1024
rq = np.random.default_rng(77)
qms = []
for hl in range(8):
    h = 1024
    prm = {"w1": rq.normal(0, np.sqrt(2.0 / d), (d, h)), "b1": np.zeros((1, h)), "bn_gamma": np.ones((1, h)), "bn_beta": np.zeros((1, h)),
           "bn_run_mean": np.zeros((1, h)), "bn_run_var": np.ones((1, h)), "w2": rq.normal(0, np.sqrt(1.0 / h), (h, C)), "b2": np.zeros((1, C))}
    qms.append(sb.QModelRouter(sb.QModel(prm, ctx)))
lay = bench.build_c3_layer(sb, torch, ctx, a, 0, 0.0, 8, 0, dev, stream, len(os.sched_getaffinity(0)), qms)
cfg = sb.SparseAttnConfig(a.probes, 128, sb.DenseWindow(1, a.recent))
out = torch.empty(64, 4, 128, device=dev); stats = torch.zeros(64, 3, dtype=torch.int64, device=dev)
sel_ref = None
for v in [0]:
    ctx.set_option("qm_logits", v)
    sel = torch.empty(64, 32, dtype=torch.int32, device=dev)
    lay.L.sparse_attention_dev(lay.routers, lay.qr_t, lay.qd_t, 4, cfg, out, stats, selected=sel)
    ctx.synchronize()
    s = sel.cpu().numpy()
    if sel_ref is None: sel_ref = s
    same = bool(np.array_equal(s, sel_ref))
    ctx.enable_timing(True)
    for i in range(20):
        lay.L.sparse_attention_dev(lay.routers, lay.qr_t, lay.qd_t, 4, cfg, out, stats)
    plan_ms, attn_ms, n = ctx.timing(); ctx.enable_timing(False)
    print(json.dumps({"variant": v, "route_us": round(plan_ms / n * 1e3, 2), "attn_us": round(attn_ms / n * 1e3, 2), "selected_equal": same}), flush=True)
PY
timeout 600 python /tmp/qm_sweep.py 2>&1 | grep -v "__del__\|NoneType\|Exception ignored\|Traceback (most recent call last):$" | tail -15
