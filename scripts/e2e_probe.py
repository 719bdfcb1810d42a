"""Breakdown of the host-API (e2e) decode step at C3: device graph replay vs
saap_sparse_attention from Python with pinned host buffers, and the bare
ctypes / sync overheads.  Diagnostic only."""
import ctypes as ct
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_08246_b200 as sb  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    ctx = sb.Context(0)
    ctx.set_stream(stream.cuda_stream)
    H, B, N, d, C, G = 8, 8, 131072, 128, 1024, 4
    ng = H * B
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    cents = torch.randn(H, C, d, device=dev, generator=gen)
    cents = (cents / cents.norm(dim=-1, keepdim=True)).float()
    K = torch.empty(ng * N, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for gi in range(ng):
        rows = slice(gi * N, (gi + 1) * N)
        with torch.cuda.stream(stream):
            sb.synth_fill(ctx, K[rows], N, d, 7 + gi, 1, cents[gi % H], C, 4.0, 1.0)
            sb.synth_fill(ctx, V[rows], N, d, 99 + gi, 0, None, 0, 0.0, 1.0)
    ctx.synchronize()
    parts_h = [sb.Partition(cents[h].cpu().numpy(), ctx) for h in range(H)]
    parts = [parts_h[gi % H] for gi in range(ng)]
    L = sb.Layer([N] * ng, d, C, 1, 2047, ctx)
    L.build_dev(parts, K, V, K)
    routers = [sb.CentroidRouter(p, True) for p in parts]
    q = torch.empty(ng, G, d, device=dev)
    for gi in range(ng):
        tgt = cents[gi % H][torch.randint(C, (1,), device=dev, generator=gen)]
        q[gi] = (tgt * 6.0 + torch.randn(G, d, device=dev, generator=gen)).bfloat16().float()
    out = torch.empty_like(q)
    stats = torch.zeros(ng, 3, dtype=torch.int64, device=dev)
    cfg = sb.SparseAttnConfig(32, 128, sb.DenseWindow(1, 2047))
    L.sparse_attention_dev(routers, q, q, G, cfg, out, stats)
    ctx.graph_begin()
    L.sparse_attention_dev(routers, q, q, G, cfg, out, stats)
    g = ctx.graph_end()
    lib = sb.lib()
    qh = torch.empty(ng, G, d, pin_memory=True)
    qh.copy_(q.cpu())
    oh = torch.empty(ng, G, d, pin_memory=True)
    st_pin = torch.empty(ng * ct.sizeof(sb.AttnStats), dtype=torch.uint8, pin_memory=True)
    st_h = (sb.AttnStats * ng).from_address(st_pin.data_ptr())
    ccfg = cfg.c()
    rarr = L._routers(routers)
    res = {}

    def wall(fn, n=200):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e6

    res["graph_replay_async"] = wall(lambda: g.launch())
    res["graph_replay_sync"] = wall(lambda: (g.launch(), ctx.synchronize()))
    res["ctypes_sync_only"] = wall(lambda: ctx.synchronize())

    def e2e():
        sb._check(lib.saap_sparse_attention(ctx.h, L.h, rarr, ct.c_void_p(qh.data_ptr()),
                                            ct.c_void_p(qh.data_ptr()), ct.c_uint64(G),
                                            ct.byref(ccfg), ct.c_void_p(oh.data_ptr()), st_h, None))
    res["host_api_e2e"] = wall(e2e)

    def e2e_no_stats():
        sb._check(lib.saap_sparse_attention(ctx.h, L.h, rarr, ct.c_void_p(qh.data_ptr()),
                                            ct.c_void_p(qh.data_ptr()), ct.c_uint64(G),
                                            ct.byref(ccfg), ct.c_void_p(oh.data_ptr()), None, None))
    res["host_api_e2e_no_stats"] = wall(e2e_no_stats)

    def copies():
        with torch.cuda.stream(stream):
            q.copy_(qh, non_blocking=True)
            g.launch()
            oh.copy_(out, non_blocking=True)
        stream.synchronize()
    res["torch_copies_graph_sync"] = wall(copies)
    qh2 = torch.empty(ng, G, d, pin_memory=True)
    qh2.copy_(q.cpu())

    def e2e_two():  # distinct roped / de-roped buffers (the bench's case)
        sb._check(lib.saap_sparse_attention(ctx.h, L.h, rarr, ct.c_void_p(qh.data_ptr()),
                                            ct.c_void_p(qh2.data_ptr()), ct.c_uint64(G),
                                            ct.byref(ccfg), ct.c_void_p(oh.data_ptr()), st_h, None))
    res["host_api_e2e_two_q"] = wall(e2e_two)
    qd_dev = torch.empty_like(q)

    def copies_only():
        with torch.cuda.stream(stream):
            q.copy_(qh, non_blocking=True)
            qd_dev.copy_(qh2, non_blocking=True)
            oh.copy_(out, non_blocking=True)
        stream.synchronize()
    res["copies_only_sync"] = wall(copies_only)
    print({k: round(v, 1) for k, v in res.items()})


if __name__ == "__main__":
    main()
