"""Incremental decode index at C3 (64 contexts x 128k keys, C=1024): wall
time of saap_layer_append for k new keys per context, and the graph-replayed
decode step before / after appends (after an append the layer's window no
longer matches its packed split, so steps take the general planner path).
Prints one JSON line."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_08246_b200 as sb  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    ctx = sb.Context(0)
    ctx.set_stream(stream.cuda_stream)
    H, B, N, d, C, G, grow = 8, 8, 131072, 128, 1024, 4, 1024
    ng = H * B
    gen = torch.Generator(device=dev)
    gen.manual_seed(3)
    cents = torch.randn(H, C, d, device=dev, generator=gen)
    cents = (cents / cents.norm(dim=-1, keepdim=True)).float()
    K = torch.empty(ng * N, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    Kn = torch.empty(ng * grow, d, dtype=torch.bfloat16, device=dev)
    Vn = torch.empty_like(Kn)
    for gi in range(ng):
        with torch.cuda.stream(stream):
            sb.synth_fill(ctx, K[gi * N:(gi + 1) * N], N, d, 5 + gi, 1, cents[gi % H], C, 4.0, 1.0)
            sb.synth_fill(ctx, V[gi * N:(gi + 1) * N], N, d, 55 + gi, 0, None, 0, 0.0, 1.0)
            sb.synth_fill(ctx, Kn[gi * grow:(gi + 1) * grow], grow, d, 505 + gi, 1, cents[gi % H], C, 4.0, 1.0)
            sb.synth_fill(ctx, Vn[gi * grow:(gi + 1) * grow], grow, d, 555 + gi, 0, None, 0, 0.0, 1.0)
    ctx.synchronize()
    parts_h = [sb.Partition(cents[h].cpu().numpy(), ctx) for h in range(H)]
    parts = [parts_h[gi % H] for gi in range(ng)]
    L = sb.Layer([N] * ng, d, C, 1, 2047, ctx, capacity=N + grow)
    L.build_dev(parts, K, V, K)
    routers = [sb.CentroidRouter(p, True) for p in parts]
    q = torch.empty(ng, G, d, device=dev)
    for gi in range(ng):
        tgt = cents[gi % H][torch.randint(C, (1,), device=dev, generator=gen)]
        q[gi] = (tgt * 6.0 + torch.randn(G, d, device=dev, generator=gen)).bfloat16().float()
    out = torch.empty_like(q)
    stats = torch.zeros(ng, 3, dtype=torch.int64, device=dev)
    cfg = sb.SparseAttnConfig(32, 128, sb.DenseWindow(1, 2047))

    def step_us():
        L.sparse_attention_dev(routers, q, q, G, cfg, out, stats)
        ctx.synchronize()
        ctx.graph_begin()
        L.sparse_attention_dev(routers, q, q, G, cfg, out, stats)
        g = ctx.graph_end()
        for _ in range(5):
            g.launch()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(50):
            g.launch()
        e.record(stream)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / 50 * 1e3

    res = {"contexts": ng, "ctx_len": N, "C": C, "step_us_before": round(step_us(), 2), "append": []}
    done = 0
    for k in (1, 1, 16, 256):
        kr = Kn.view(ng, grow, d)[:, done:done + k].contiguous()
        vr = Vn.view(ng, grow, d)[:, done:done + k].contiguous()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.append_dev(kr, vr, kr, k)
        dt = (time.perf_counter() - t0) * 1e6
        done += k
        res["append"].append({"k": k, "append_us": round(dt, 1), "step_us_after": round(step_us(), 2)})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
