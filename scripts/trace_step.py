"""Decode-step timelines at C3 (profiling aid, not a bench line).

Builds one C3 layer with bench.py's input pipeline, then replays the step
with the context's trace options: the step timeline (first start / last end
of each kernel), per-CTA decode timelines and the fused routing phases.
Extra options: --opt name=value (saap_ctx_set_option), repeatable.

    python scripts/trace_step.py [--opt chunk=8] [--out gpurun_out/trace.json]
"""
import argparse
import ctypes as ct
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "trace.json"))
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--drift", type=float, default=0.0)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--plain", action="store_true", help="no tracing; run --reps eager steps and exit")
    ap.add_argument("--ctx-len", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--probes", type=int, default=32)
    ap.add_argument("--given", action="store_true",
                    help="replay the routed lists through the caller-selected path (no routing)")
    args = ap.parse_args()
    import torch
    import paper_2502_08246_b200 as sb
    if not hasattr(sb.Context, "set_option"):
        raise SystemExit("library without context options")
    a = argparse.Namespace(ctx_len=args.ctx_len, batch=args.batch, kv_heads=8, q_heads=32, dim=128, buckets=1024,
                           probes=args.probes, recent=2047, sink=1, kmeans_iters=10)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    ctx = sb.Context(0)
    ctx.set_stream(stream.cuda_stream)
    for kv in args.opt:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    if args.plain:  # no tracing: a clean run for ncu (-k decode_kernel)
        pass
    else:
        ctx.set_option("trace_step", 1)
        ctx.set_option("trace_decode", 1)
        ctx.set_option("trace_plan", 1)
    threads = len(os.sched_getaffinity(0))
    lays = []
    for li in range(2):
        inp = bench.make_layer_inputs(sb, torch, ctx, a, li, args.drift, 8, 0, dev, threads)
        parts = [sb.Partition(c, ctx) for c in inp.cents]
        n_groups = args.batch * 8
        L = sb.Layer([a.ctx_len] * n_groups, 128, a.buckets, 1, a.recent, ctx)
        L.build_dev([parts[g % 8] for g in range(n_groups)], inp.K, inp.V, inp.Kd)
        inp.L, inp.routers = L, [sb.CentroidRouter(parts[g % 8], True) for g in range(n_groups)]
        inp.kv = sb.KVCache(ctx, n_groups, 128, inp.K, inp.V, [g * a.ctx_len for g in range(n_groups)],
                            [a.ctx_len] * n_groups)
        inp.qr_t, inp.qd_t = torch.from_numpy(inp.qr).to(dev), torch.from_numpy(inp.qd).to(dev)
        lays.append(inp)
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

    for i in range(6):
        step(lays[i % 2])
    ctx.synchronize()
    if args.plain:
        for i in range(args.reps):
            step(lays[i % 2])
        ctx.synchronize()
        print("plain steps done")
        return
    graphs = []
    for lay in lays:  # trace graph replays (the bench's timed path), not eager launches
        ctx.graph_begin()
        step(lay)
        graphs.append(ctx.graph_end())
    for i in range(4):
        graphs[i % 2].launch()
    ctx.synchronize()
    lib = sb.lib()
    res = {"opts": args.opt, "steps": []}
    names = ["approx", "plan", "decode", "combine", "run_published", "slot_complete"]
    buf = (ct.c_uint64 * 16)()
    nc = ctx.sm_count
    dbuf = (ct.c_uint64 * (16 * nc))()
    pbuf = (ct.c_uint64 * (16 + 6 * 1024))()
    dec_all = []
    tiles_all = []
    for r in range(args.reps):
        sb._check(lib.saap_debug_step_trace(ctx.h, buf, 1))
        graphs[r % 2].launch()
        ctx.synchronize()
        sb._check(lib.saap_debug_step_trace(ctx.h, buf, 0))
        v = list(buf)
        t0 = min(x for x in v[0::2] if x)
        st = {n: [round((v[2 * k] - t0) / 1e3, 2) if v[2 * k] != 2**64 - 1 else None,
                  round((v[2 * k + 1] - t0) / 1e3, 2) if v[2 * k + 1] else None]
              for k, n in enumerate(names)}
        if lib.saap_debug_decode_trace(ctx.h, dbuf, ct.c_uint64(nc)) == 0:
            t = np.array(list(dbuf), dtype=np.float64).reshape(nc, 16)
            rel = lambda x: [round(float(y), 2) for y in np.percentile((x - t0) / 1e3, [0, 10, 50, 90, 100])]
            st["decode_cta"] = {"start_us": rel(t[:, 0]), "first_tile_us": rel(t[:, 1]),
                                "end_us": rel(t[:, 2]),
                                "first_record_us": rel(t[:, 10]), "first_tma_us": rel(t[:, 11]),
                                "producer_loop_us": rel(t[:, 12]), "first_rec_issue_us": rel(t[:, 13]),
                                "tiles": [int(x) for x in np.percentile(t[:, 3], [0, 50, 100])],
                                "cons_wait_frac": round(float(np.median(t[:, 6] / np.maximum(t[:, 5], 1))), 3),
                                "prod_empty_wait_frac": round(float(np.median(t[:, 4] / np.maximum(t[:, 5], 1))), 3),
                                "prod_rec_wait_frac": round(float(np.median(t[:, 8] / np.maximum(t[:, 5], 1))), 3),
                                "prod_feed_frac": round(float(np.median(t[:, 7] / np.maximum(t[:, 5], 1))), 3),
                                "prod_tma_frac": round(float(np.median(t[:, 9] / np.maximum(t[:, 5], 1))), 3),
                                "prod_sleep_frac": round(float(np.median(t[:, 14] / np.maximum(t[:, 5], 1))), 3),
                                "prod_decode_frac": round(float(np.median(t[:, 15] / np.maximum(t[:, 5], 1))), 3)}
            dec_all.append(((t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]))
            tb = (ct.c_uint64 * (nc * 48 * 8))()
            if lib.saap_debug_decode_tiles(ctx.h, tb, ct.c_uint64(nc)) == 0:
                raw = np.array(list(tb), dtype=np.uint64).reshape(nc, 48, 8)
                flags = (raw[:, :, 0] & np.uint64(63)).astype(np.float64)  # pieces | 32 chunk end
                raw[:, :, 0] &= ~np.uint64(63)
                ok = raw >= np.uint64(t0)
                tt = np.where(ok, (raw.astype(np.int64) - np.int64(t0)).astype(np.float64) / 1e3, np.nan)
                tt = np.concatenate([tt, flags[:, :, None]], axis=2)
                tiles_all.append(tt)
        if not args.dense and lib.saap_debug_plan_trace(ctx.h, pbuf) == 0:
            # slot 0 / CTA 0 phase clocks (clock64 deltas -> us at the measured SM clock)
            st["route_phases_us"] = {str(k): round(float(pbuf[k]) / 1965.0, 2) for k in range(16) if pbuf[k]}
            cta = np.array(list(pbuf)[16:], dtype=np.float64).reshape(1024, 6)
            cta = cta[cta[:, 0] > 0]
            if len(cta):
                st["route_cta"] = {k: [round(float(x), 2) for x in np.percentile((cta[:, i] - t0) / 1e3, [0, 50, 100])]
                                   for i, k in enumerate(["start_us", "exchanged_us", "selected_us", "end_us"])}
                own = cta[cta[:, 3] > 0]
                slow = own[np.argsort(own[:, 3])[-4:]]
                st["route_slowest"] = [[round(float((r[i] - t0) / 1e3), 2) for i in range(4)] + [int(r[4])]
                                       + [round(float((r[5] - t0) / 1e3), 2) if r[5] > t0 else None]
                                       for r in slow]
                st["route_candidates"] = [int(x) for x in np.percentile(own[:, 4], [0, 50, 90, 100])]
        res["steps"].append(st)
    # medians over reps
    def med(path):
        vals = []
        for st in res["steps"]:
            x = st
            for p in path:
                x = x.get(p) if isinstance(x, dict) else None
                if x is None:
                    break
            if x is not None:
                vals.append(x)
        return np.median(np.array(vals, dtype=float), axis=0).round(2).tolist() if vals else None
    res["median"] = {n: med([n]) for n in names}
    res["median"]["decode_cta_end_us"] = med(["decode_cta", "end_us"])
    res["median"]["decode_cta_first_tile_us"] = med(["decode_cta", "first_tile_us"])
    res["median"]["decode_cta_start_us"] = med(["decode_cta", "start_us"])
    res["median"]["route_cta_end_us"] = med(["route_cta", "end_us"])
    res["median"]["decode_producer_loop_us"] = med(["decode_cta", "producer_loop_us"])
    res["median"]["decode_first_rec_issue_us"] = med(["decode_cta", "first_rec_issue_us"])
    res["median"]["decode_first_record_us"] = med(["decode_cta", "first_record_us"])
    res["median"]["decode_first_tma_us"] = med(["decode_cta", "first_tma_us"])
    ph = [st.get("route_phases_us") for st in res["steps"] if st.get("route_phases_us")]
    if ph:
        res["median"]["route_phases_us"] = {k: round(float(np.median([p[k] for p in ph if k in p])), 2)
                                            for k in ph[0]}
    for k in ("cons_wait_frac", "prod_empty_wait_frac", "prod_rec_wait_frac", "prod_feed_frac", "prod_tma_frac",
              "prod_sleep_frac", "prod_decode_frac"):
        res["median"][k] = med(["decode_cta", k])
    if dec_all:
        np.save(os.path.splitext(args.out)[0] + "_cta.npy", np.array(dec_all))
    if tiles_all:
        np.save(os.path.splitext(args.out)[0] + "_tiles.npy", np.array(tiles_all))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res["median"]))


if __name__ == "__main__":
    main()
