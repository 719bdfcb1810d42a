"""C5 (BASELINE configs[4]) on one B200: 1M-token contexts, 1 sequence x 8 KV
heads (the per-GPU share of an 8-GPU head-sharded run is one head; here all
8 heads sit on one GPU, so per-head latency ~ step / 8), bucket counts
C in {1k, 4k, 16k} with partitions trained ON THE DEVICE by kmeans_train
(kmeans.cu, bit-exact with partition.cpp:52-179) on a key sample of each
head, nprobe l in {8..256}: graph-replayed step latency vs approximation
error (mse vs the in-run dense kernel, attention.cpp:385-399) and
selectivity.  One JSON line per (C, l) to stdout.

    python scripts/c5_sweep.py [--ctx-len 1048576] [--train-keys 131072]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx-len", type=int, default=1 << 20)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--train-keys", type=int, default=131072)
    ap.add_argument("--kmeans-iters", type=int, default=5)
    ap.add_argument("--buckets", default="1024,4096,16384")
    ap.add_argument("--probes", default="8,16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()

    import torch

    import paper_2502_08246_b200 as sb

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    ctx = sb.Context(0)
    ctx.set_stream(stream.cuda_stream)
    H, d, N, G, sink, recent = a.kv_heads, a.dim, a.ctx_len, 4, 1, 2047
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    # keys clustered around 1024 random directions per head (synth kind 1)
    gen_c = 1024
    cents = torch.randn(H, gen_c, d, device=dev, generator=gen)
    cents = (cents / cents.norm(dim=-1, keepdim=True)).float()
    K = torch.empty(H * N, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for h in range(H):
        rows = slice(h * N, (h + 1) * N)
        with torch.cuda.stream(stream):
            sb.synth_fill(ctx, K[rows], N, d, 77 + h, 1, cents[h], gen_c, 4.0, 1.0)
            sb.synth_fill(ctx, V[rows], N, d, 177 + h, 0, None, 0, 0.0, 1.0)
    ctx.synchronize()
    q = torch.empty(H, G, d, device=dev)
    for h in range(H):
        tgt = cents[h][torch.randint(gen_c, (1,), device=dev, generator=gen)]
        q[h] = (tgt * 6.0 + torch.randn(G, d, device=dev, generator=gen)).bfloat16().float()
    kv = sb.KVCache(ctx, H, d, K, V, [h * N for h in range(H)], [N] * H)
    out = torch.empty(H, G, d, device=dev)
    out_dense = torch.empty_like(out)
    stats = torch.zeros(H, 3, dtype=torch.int64, device=dev)

    def timed(fn, steps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(steps):
            fn()
        e.record(stream)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / steps * 1e3

    kv.dense_attention_dev(q, G, out_dense)
    ctx.graph_begin()
    kv.dense_attention_dev(q, G, out_dense)
    dg = ctx.graph_end()
    dense_us = timed(dg.launch, a.steps)
    torch.cuda.synchronize()
    ref = out_dense.cpu().numpy().astype(np.float64)
    dense_bytes = H * N * 4 * d
    print(json.dumps({"kind": "dense", "ctx": N, "heads": H, "us": round(dense_us, 2),
                      "gbs": round(dense_bytes / dense_us / 1e3, 1)}), flush=True)

    rs = np.random.default_rng(0)
    for C in [int(x) for x in a.buckets.split(",")]:
        # device k-means per head on a key sample (the harness trains on
        # same-distribution keys, experiments.cpp:284-295)
        t0 = time.perf_counter()
        parts = []
        for h in range(H):
            idx = np.sort(rs.choice(N - sink, a.train_keys, replace=False)) + sink + h * N
            sample = K[torch.from_numpy(idx).to(dev)].float().cpu().numpy()
            parts.append(sb.kmeans_train(sample, C, a.kmeans_iters, sb.Rng(1 + h), ctx=ctx))
        train_s = time.perf_counter() - t0
        L = sb.Layer([N] * H, d, C, sink, recent, ctx)
        L.build_dev(parts, K, V, K)
        ctx.synchronize()
        routers = [sb.CentroidRouter(p, True) for p in parts]
        for l in [int(x) for x in a.probes.split(",")]:
            rec = {"kind": "saap", "ctx": N, "heads": H, "C": C, "l": l,
                   "kmeans": {"keys": a.train_keys, "iters": a.kmeans_iters,
                              "s_all_heads": round(train_s, 2)}}
            if l > C:
                continue
            cfg = sb.SparseAttnConfig(l, 128, sb.DenseWindow(sink, recent))
            try:
                L.sparse_attention_dev(routers, q, q, G, cfg, out, stats)
                ctx.synchronize()
                ctx.graph_begin()
                L.sparse_attention_dev(routers, q, q, G, cfg, out, stats)
                g = ctx.graph_end()
                us = timed(g.launch, a.steps)
                got = out.cpu().numpy().astype(np.float64)
                st = stats.cpu().numpy()
                scored = int(st[:, 0].sum())
                rec.update(us=round(us, 2), dense_us=round(dense_us, 2),
                           speedup=round(dense_us / us, 2),
                           selectivity=round(scored / (H * N), 5),
                           max_bucket=int(st[:, 1].max()),
                           mse=float(np.mean((got - ref) ** 2)),
                           gbs=round(scored * 4 * d / us / 1e3, 1))
                del g
            except Exception as e:  # record the envelope limit, keep sweeping
                rec["error"] = str(e)[:200]
            print(json.dumps(rec), flush=True)
        del L, routers


if __name__ == "__main__":
    main()
