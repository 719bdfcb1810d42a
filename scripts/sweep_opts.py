"""Time the C3 decode step (graph replays, CUDA events, 2 rotated layers)
under several context-option settings.  Profiling aid.

    python scripts/sweep_opts.py "chunk=8" "chunk=4" "chunk=4,combine_poll_ns=200" ...
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("settings", nargs="*", default=[""])
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--drift", type=float, default=0.0)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--given", action="store_true", help="caller-selected lists (no routing kernel)")
    ap.add_argument("--probes", type=int, default=32)
    ap.add_argument("--ctx-len", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=8)
    args = ap.parse_args()
    import torch
    import paper_2502_08246_b200 as sb
    a = argparse.Namespace(ctx_len=args.ctx_len, batch=args.batch, kv_heads=8, q_heads=32, dim=128, buckets=1024,
                           probes=args.probes, recent=2047, sink=1, kmeans_iters=10)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    ctx = sb.Context(0)
    ctx.set_stream(stream.cuda_stream)
    threads = len(os.sched_getaffinity(0))
    lays = [bench.build_c3_layer(sb, torch, ctx, a, li, args.drift, 8, 0, dev, stream, threads)
            for li in range(2)]
    cfg = sb.SparseAttnConfig(a.probes, 128, sb.DenseWindow(1, a.recent))
    out = torch.empty(args.batch * 8, 4, 128, device=dev)
    stats = torch.zeros(args.batch * 8, 3, dtype=torch.int64, device=dev)

    if args.given:
        for lay in lays:
            lay.sel = torch.empty(args.batch * 8, a.probes, dtype=torch.int32, device=dev)
            lay.L.sparse_attention_dev(lay.routers, lay.qr_t, lay.qd_t, 4, cfg, out, stats,
                                       selected=lay.sel)
        ctx.synchronize()

    def step(lay):
        if args.dense:
            lay.kv.dense_attention_dev(lay.qr_t, 4, out)
        elif args.given:
            lay.L.sparse_attention_selected_dev(lay.qr_t, 4, lay.sel, a.probes, cfg, out, stats)
        else:
            lay.L.sparse_attention_dev(lay.routers, lay.qr_t, lay.qd_t, 4, cfg, out, stats)

    defaults = {}
    res = {}
    for setting in args.settings:
        kv = dict(x.split("=") for x in setting.split(",") if x)
        for k, v in kv.items():
            ctx.set_option(k, int(v))
        for i in range(4):
            step(lays[i % 2])
        ctx.synchronize()
        gs = []
        for lay in lays:
            ctx.graph_begin()
            step(lay)
            gs.append(ctx.graph_end())
        for i in range(10):
            gs[i % 2].launch()
        torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.steps):
                gs[i % 2].launch()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / args.steps * 1e3)
        res[setting or "default"] = round(min(ts), 2)
        print(json.dumps({setting or "default": [round(t, 2) for t in ts]}), flush=True)
        for k in kv:  # back to the defaults for the next setting
            ctx.set_option(k, {"chunk": 8, "chunk_dense": 16, "tail_per_cta": 1, "decode_poll_ns": 100,
                               "combine_poll_ns": 1000, "decode_wait": 0, "cluster_route": 1,
                               "min_chunk": 4, "claim_lead": 3, "fetch_lead": 2, "inflight": 0, "decode_tc": 0, "qm_logits": 0, "chunk_st": 0}.get(k, 0))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
