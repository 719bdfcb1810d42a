#!/usr/bin/env python
"""SAAP decode-attention bench (BASELINE.json metric, config C3).

One step = one decode step of one layer for the whole job: routing +
planning + split-K sparse attention + LSE combine for every (sequence, KV
head) context — batch 8 x 8 KV heads (Llama-3-8B GQA 32Q/8KV, d=128, bf16
KV) at 128k context, C=1024 buckets, l=32 probes, window 1+2047 — plus, at
N>1 GPUs, the NCCL all-gather of the per-head outputs.  KV heads are sharded
over ranks (strong scaling: total work fixed).  The dense decode kernel (the
in-run baseline) runs on the same position-ordered cache.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints one JSON line (rank 0).  Synthetic data (counter-based generator on
the device), random-init centroids; see DESIGN.md §5.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SAAP decode-attention µs/step & speedup vs dense at 128k ctx; HBM GB/s"
UNIT = "us/step"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ctx-len", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--q-heads", type=int, default=32)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--buckets", type=int, default=1024)
    ap.add_argument("--probes", type=int, default=32)
    ap.add_argument("--recent", type=int, default=2047)
    ap.add_argument("--sink", type=int, default=1)
    ap.add_argument("--layers", type=int, default=4, help="distinct layer caches rotated per step")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--router", default="centroid", choices=["centroid", "qmodel"],
                    help="BucketRouter plugin: CentroidRouter (de-roped) or QModelRouter (random-init "
                         "weights of the reference's shape, hidden 1024)")
    return ap.parse_args()


def workload_config(a, n):
    return {
        "workload": (f"C3: Llama-3-8B attention shape ({a.q_heads} Q / {a.kv_heads} KV heads, "
                     f"d={a.dim}, bf16 KV) decode, batch {a.batch}, {a.ctx_len} ctx, "
                     f"C={a.buckets}, l={a.probes}, window {a.sink}+{a.recent}, "
                     + ("de-roped centroid router" if a.router == "centroid"
                        else "Q-model router (hidden 1024, random-init)")),
        "model": "Llama-3-8B attention shape (random-init centroids)",
        "global_batch": a.batch,
        "seq_len": a.ctx_len,
        "parallelism": f"kv-head shard x{n}",
        "l2": (f"inputs larger than L2: {a.layers} distinct layer caches rotated per step "
               "(sparse touched set per step > 126 MB L2)"),
    }


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the measured region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r.split(", ") for r in self.lines if r.count(",") >= 6]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        busy = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()
                and r[6].isdigit() and int(r[6]) > 0]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(busy or sm) if (busy or sm) else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "samples_busy": len(busy)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch of the decode kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "decode_kernel_ncu.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


# ---------------------------------------------------------------- CPU reference
def cpu_threads(a):
    return a.cpu_threads or len(os.sched_getaffinity(0))


def run_cpu_reference(stores_data, queries, a, steps, warmup, threads):
    """Time the reference's sparse_attention (oracle/_ref, unmodified sources)
    on a bounded sample: len(stores_data) distinct 128k contexts x the query
    groups of the batch = batch*kv_heads groups per step."""
    import oracle
    if oracle.ref_available():
        R = oracle.ref()
        kind = "reference"
    else:
        R = None
        kind = "port"
    stores, routers = [], []
    for sd in stores_data:
        if R is not None:
            stores.append(R.store(sd["K"], sd["V"], sd["cent"], a.sink, sd["assign"]))
            routers.append(R.centroid_router(sd["cent"], True))
        else:
            stores.append(sd)
            routers.append(None)
    n_groups = queries.shape[0]
    S = [stores[g % len(stores)] for g in range(n_groups)]
    Rt = [routers[g % len(routers)] for g in range(n_groups)]

    def step():
        if R is not None:
            out, ks = R.sparse_attention_batch(S, Rt, queries, queries, a.probes, 128, a.sink,
                                               a.recent, threads)
            return ks
        P = oracle.port()
        ks = []
        for g in range(n_groups):
            sd = S[g]
            sel = P.centroid_select(sd["cent"], queries[g], a.probes)
            off, idx = P.build_ivf(sd["assign"], a.buckets)
            ks.append(P.sparse_attention(queries[g], sd["K"], sd["V"], a.sink, off, idx, sel,
                                         a.probes, 128, a.recent)[1])
        return np.array(ks)

    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        ks = step()
    dt = (time.perf_counter() - t0) / steps
    return dt * 1e6, kind, (threads if R is not None else 1), ks


# ---------------------------------------------------------------- synthetic data (CPU)
def cpu_synth_store(a, seed):
    rs = np.random.RandomState(seed)
    from oracle import bf16_round
    cent = rs.randn(a.buckets, a.dim)
    cent = (cent / np.linalg.norm(cent, axis=1, keepdims=True)).astype(np.float32)
    lab = rs.randint(0, a.buckets, a.ctx_len)
    K = bf16_round(cent[lab] * 4.0 + rs.randn(a.ctx_len, a.dim).astype(np.float32))
    V = bf16_round(rs.randn(a.ctx_len, a.dim).astype(np.float32))
    return cent, K, V


def reference_arm(a):
    """--impl reference: the reference CPU path on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from oracle import bf16_round
    threads = cpu_threads(a)
    n_groups = a.batch * a.kv_heads
    n_stores = min(a.kv_heads, n_groups)
    stores = []
    for h in range(n_stores):
        cent, K, V = cpu_synth_store(a, 1000 + h)
        if oracle.ref_available():
            assign = oracle.ref().assign_keys(K[a.sink:], cent, threads=threads)
        else:
            assign = oracle.port().assign_keys(K[a.sink:], cent)
        stores.append({"cent": cent, "K": K, "V": V, "assign": assign})
    rs = np.random.RandomState(7)
    G = a.q_heads // a.kv_heads
    q = np.stack([bf16_round(stores[g % n_stores]["cent"][rs.randint(a.buckets)] * 6.0
                             + rs.randn(G, a.dim).astype(np.float32)) for g in range(n_groups)])
    us, kind, cores, ks = run_cpu_reference(stores, q, a, a.steps, a.warmup, threads)
    line = {
        "metric": METRIC, "value": round(us, 3), "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(us / 1e3, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (clustered keys, random unit centroids; numpy)",
        "config": workload_config(a, a.gpus), "impl": "reference",
        "cpu_baseline": {"value": round(us, 3), "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": (f"{n_stores} distinct {a.ctx_len}-key contexts x "
                                    f"{n_groups // n_stores} query groups = {n_groups} "
                                    "(sequence, KV head) groups per step")},
        "e2e": {"value": round(us, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "selectivity": float(np.mean(ks) / a.ctx_len),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def ours(a):
    import torch
    import torch.distributed as dist

    import paper_2502_08246_b200 as sb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2502_08246_b200.shard import HeadShard, gather_outputs
    sh = HeadShard(rank, world, a.kv_heads, a.batch)
    heads_local, h0 = sh.heads_local, sh.head0
    G = a.q_heads // a.kv_heads
    d, C, N = a.dim, a.buckets, a.ctx_len
    n_groups = sh.n_groups  # group = (sequence, local KV head)

    stream = torch.cuda.Stream()
    ctx = sb.Context(local)
    ctx.set_stream(stream.cuda_stream)
    dev = torch.device("cuda", local)

    # ---- per layer: centroids per KV head, clustered keys, values; build stores
    layers = []
    t_build = []
    qm_routers = None
    for li in range(a.layers):
        gen = torch.Generator(device=dev)
        gen.manual_seed(1000 * li + 17)
        cents = torch.randn(a.kv_heads, C, d, device=dev, generator=gen)
        cents = (cents / cents.norm(dim=-1, keepdim=True)).float()
        K = torch.empty(n_groups * N, d, dtype=torch.bfloat16, device=dev)
        V = torch.empty_like(K)
        for gi in range(n_groups):
            s, hl = divmod(gi, heads_local)
            h = h0 + hl
            seed = (li * 1_000_003 + s * 7919 + h * 104729) & 0xFFFFFFFF
            rows = slice(gi * N, (gi + 1) * N)
            with torch.cuda.stream(stream):
                sb.synth_fill(ctx, K[rows], N, d, seed, 1, cents[h], C, 4.0, 1.0)
                sb.synth_fill(ctx, V[rows], N, d, seed ^ 0x5555, 0, None, 0, 0.0, 1.0)
        ctx.synchronize()
        parts_h = [sb.Partition(cents[h0 + hl].cpu().numpy(), ctx) for hl in range(heads_local)]
        parts = [parts_h[gi % heads_local] for gi in range(n_groups)]
        L = sb.Layer([N] * n_groups, d, C, a.sink, a.recent, ctx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.build_dev(parts, K, V, K)
        e1.record(stream)
        torch.cuda.synchronize()
        t_build.append(e0.elapsed_time(e1))
        if a.router == "qmodel":
            if qm_routers is None:
                qm_routers = []
                rq = np.random.default_rng(77 + rank)
                for hl in range(heads_local):  # qmodel_init shapes / scales (qmodel.cpp:337-357)
                    h = 1024
                    prm = {"w1": rq.normal(0, np.sqrt(2.0 / d), (d, h)), "b1": np.zeros((1, h)),
                           "bn_gamma": np.ones((1, h)), "bn_beta": np.zeros((1, h)),
                           "bn_run_mean": np.zeros((1, h)), "bn_run_var": np.ones((1, h)),
                           "w2": rq.normal(0, np.sqrt(1.0 / h), (h, C)), "b2": np.zeros((1, C))}
                    qm_routers.append(sb.QModelRouter(sb.QModel(prm, ctx)))
            routers = [qm_routers[gi % heads_local] for gi in range(n_groups)]
        else:
            routers = [sb.CentroidRouter(p, True) for p in parts]
        kv = sb.KVCache(ctx, n_groups, d, K, V, [gi * N for gi in range(n_groups)], [N] * n_groups)
        layers.append(dict(L=L, K=K, V=V, routers=routers, parts=parts_h, kv=kv, cents=cents))

    peak_early, _ = measured_peaks()
    # ---- prefill (C4-style): rebuild layer 0 with device timing per phase
    ctx.enable_timing(True)
    pre_a, pre_p = [], []
    lay0 = layers[0]
    parts0 = [lay0["parts"][gi % heads_local] for gi in range(n_groups)]
    for _ in range(3):
        lay0["L"].build_dev(parts0, lay0["K"], lay0["V"], lay0["K"])
        ta, tp = lay0["L"].build_timing()
        pre_a.append(ta)
        pre_p.append(tp)
    ctx.timing()  # clear decode records
    ctx.enable_timing(False)
    used_tc, refined = lay0["L"].assign_info()
    n_keys_prefill = n_groups * (N - a.sink)
    assign_ms, pack_ms = float(np.median(pre_a)), float(np.median(pre_p))
    pack_bytes = n_keys_prefill * (8 * d + 16)

    # ---- queries: each group's 4 heads look for one cluster of its KV head
    gq = torch.Generator(device=dev)
    gq.manual_seed(4242 + rank)
    q = torch.empty(n_groups, G, d, device=dev)
    for gi in range(n_groups):
        h = h0 + gi % heads_local
        tgt = layers[0]["cents"][h][torch.randint(C, (1,), device=dev, generator=gq)]
        q[gi] = (tgt * 6.0 + torch.randn(G, d, device=dev, generator=gq)).bfloat16().float()
    out = torch.empty(n_groups, G, d, device=dev)
    out_dense = torch.empty_like(out)
    stats = torch.zeros(n_groups, 3, dtype=torch.int64, device=dev)
    cfg = sb.SparseAttnConfig(a.probes, 128, sb.DenseWindow(a.sink, a.recent))

    def sparse_step(li):
        lay = layers[li]
        lay["L"].sparse_attention_dev(lay["routers"], q, q, G, cfg, out, stats)

    def dense_step(li):
        layers[li]["kv"].dense_attention_dev(q, G, out_dense)

    def gather():
        if world > 1:
            with torch.cuda.stream(stream):
                gather_outputs(out, sh, dist)

    # eager warm-up sizes the scratch, then capture one graph per layer
    for li in range(a.layers):
        sparse_step(li)
        if not a.no_dense:
            dense_step(li)
    ctx.synchronize()
    graphs, dgraphs = [], []
    kernels_per_step = None
    for li in range(a.layers):
        n0 = ctx.launch_count
        ctx.graph_begin()
        sparse_step(li)
        graphs.append(ctx.graph_end())
        kernels_per_step = ctx.launch_count - n0  # our kernels captured in one step's graph
        if not a.no_dense:
            ctx.graph_begin()
            dense_step(li)
            dgraphs.append(ctx.graph_end())

    clock = ClockSampler(local)
    clock.start()
    time.sleep(0.3)

    def timed(fn, steps, warm):
        for i in range(warm):
            fn(i)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for i in range(steps):
            fn(i)
        e.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = s.elapsed_time(e) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def sparse_graph_step(i):
        graphs[i % a.layers].launch()
        gather()

    ms_sparse = timed(sparse_graph_step, a.steps, a.warmup)
    ms_dense = None
    if not a.no_dense:
        ms_dense = timed(lambda i: dgraphs[i % a.layers].launch(), max(10, a.steps // 5),
                         a.warmup)
    ms_gather = None
    if world > 1:
        ms_gather = timed(lambda i: gather(), a.steps, a.warmup)

    # ---- per-kernel device time (eager, events around the kernels)
    ctx.enable_timing(True)
    reps = 20
    for i in range(reps):
        sparse_step(i % a.layers)
    plan_ms, attn_ms, n = ctx.timing()
    attn_ms /= max(n, 1)
    plan_ms /= max(n, 1)
    dense_attn_ms = None
    if not a.no_dense:
        for i in range(reps // 2):
            dense_step(i % a.layers)
        _, dms, dn = ctx.timing()
        dense_attn_ms = dms / max(dn, 1)
    ctx.enable_timing(False)
    plan_trace = None
    if os.environ.get("SAAP_PLAN_TRACE"):
        import ctypes as ct
        buf = (ct.c_uint64 * (16 + 6 * 1024))()
        if sb.lib().saap_debug_plan_trace(ctx.h, buf) == 0:
            plan_trace = list(buf)[:16]
            cta = np.array(list(buf)[16:], dtype=np.float64).reshape(1024, 6)[:, :3]
            cta = cta[cta[:, 0] > 0]
            if len(cta):
                t0 = cta[:, 0].min()
                plan_trace.append({k: [round(float(v), 2) for v in np.percentile((cta[:, i] - t0) / 1e3, [0, 50, 100])]
                                   for i, k in enumerate(["start_us", "exchanged_us", "end_us"])})
    step_trace = None
    graph_plan_trace = None
    # SAAP_TRACE_DENSE=1: the step / decode traces follow the dense step instead
    tgraphs = dgraphs if os.environ.get("SAAP_TRACE_DENSE") and dgraphs else graphs
    if os.environ.get("SAAP_STEP_TRACE"):
        import ctypes as ct
        buf = (ct.c_uint64 * 16)()
        sb._check(sb.lib().saap_debug_step_trace(ctx.h, buf, 1))
        if os.environ.get("SAAP_STEP_TRACE_EAGER"):
            ctx.enable_timing(True)  # the eager step with its timing events
            sparse_step(0)
            ctx.synchronize()
            ctx.timing()
            ctx.enable_timing(False)
        else:
            tgraphs[0].launch()
        ctx.synchronize()
        sb._check(sb.lib().saap_debug_step_trace(ctx.h, buf, 0))
        if os.environ.get("SAAP_PLAN_TRACE"):  # routing phases of this (overlapped) step
            pbuf = (ct.c_uint64 * (16 + 6 * 1024))()
            if sb.lib().saap_debug_plan_trace(ctx.h, pbuf) == 0:
                cta = np.array(list(pbuf)[16:], dtype=np.float64).reshape(1024, 6)
                cta = cta[cta[:, 0] > 0]
                tt0 = cta[:, 0].min() if len(cta) else 0
                own = cta[cta[:, 3] > 0]
                slow = own[np.argsort(own[:, 3])[-4:]] if len(own) else own
                graph_plan_trace = [list(pbuf)[:13]] + [
                    {k: [round(float(x), 2) for x in np.percentile((own[:, i] - tt0) / 1e3, [0, 50, 100])]
                     for i, k in enumerate(["start_us", "exchanged_us", "selected_us", "end_us"])},
                    {"slowest_owner_ctas_us_and_candidates": [[round(float((r[i] - tt0) / 1e3), 2) for i in range(4)] + [int(r[4])]
                                                              for r in slow]}] if len(own) else None
        v = list(buf)
        t0 = min(x for x in v[0::2] if x)
        names = ["approx", "plan", "decode", "combine", "run_published", "slot_complete"]
        step_trace = {n: [round((v[2 * k] - t0) / 1e3, 2) if v[2 * k] != 2**64 - 1 else None,
                          round((v[2 * k + 1] - t0) / 1e3, 2) if v[2 * k + 1] else None]
                      for k, n in enumerate(names)}
    decode_trace = None
    if os.environ.get("SAAP_DECODE_TRACE"):
        import ctypes as ct
        tgraphs[0].launch()  # trace the sparse (or dense) step
        ctx.synchronize()
        nc = ctx.sm_count
        buf = (ct.c_uint64 * (16 * nc))()
        if sb.lib().saap_debug_decode_trace(ctx.h, buf, ct.c_uint64(nc)) == 0:
            t = np.array(list(buf), dtype=np.float64).reshape(nc, 16)
            t0 = t[:, 0].min()
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            np.save(os.path.join(ROOT, "gpurun_out", "decode_trace.npy"), t)
            rel = lambda x: [round(float(v), 2) for v in np.percentile((x - t0) / 1e3, [0, 50, 100])]
            decode_trace = {"start_us": rel(t[:, 0]), "first_tile_us": rel(t[:, 1]),
                            "end_us": rel(t[:, 2]),
                            "tiles_per_cta": [int(v) for v in np.percentile(t[:, 3], [0, 50, 100])],
                            "producer_empty_wait_frac": round(float(np.median(t[:, 4] / np.maximum(t[:, 5], 1))), 3),
                            "consumer_full_wait_frac": round(float(np.median(t[:, 6] / np.maximum(t[:, 5], 1))), 3),
                            "producer_feed_frac": round(float(np.median(t[:, 7] / np.maximum(t[:, 5], 1))), 3),
                            "producer_record_wait_frac": round(float(np.median(t[:, 8] / np.maximum(t[:, 5], 1))), 3),
                            "producer_tma_issue_frac": round(float(np.median(t[:, 9] / np.maximum(t[:, 5], 1))), 3),
                            "first_record_us": rel(t[:, 10]), "first_tma_us": rel(t[:, 11])}

    # ---- counters, quality vs dense
    keys_scored = []
    mse_vals = []
    for li in range(a.layers):
        sparse_step(li)
        dense_step(li)
        torch.cuda.synchronize()
        keys_scored.append(int(stats[:, 0].sum().item()))
        mse_vals.append(((out - out_dense) ** 2).mean().item())
    ks_step = float(np.mean(keys_scored))
    bytes_step = ks_step * d * 2 * 2
    dense_bytes = n_groups * N * d * 2 * 2

    # ---- end to end through the public host API (pinned host buffers)
    import ctypes as ct
    qh = torch.empty(n_groups, G, d, pin_memory=True)
    qh.copy_(q.cpu())
    oh = torch.empty(n_groups, G, d, pin_memory=True)
    # page-locked stats buffer (one fast D2H like the outputs)
    st_pin = torch.empty(n_groups * ct.sizeof(sb.AttnStats), dtype=torch.uint8, pin_memory=True)
    st_h = (sb.AttnStats * n_groups).from_address(st_pin.data_ptr())
    lib = sb.lib()
    ccfg = cfg.c()

    def e2e_step(i):
        lay = layers[i % a.layers]
        sb._check(lib.saap_sparse_attention(
            ctx.h, lay["L"].h, lay["L"]._routers(lay["routers"]), ct.c_void_p(qh.data_ptr()),
            ct.c_void_p(qh.data_ptr()), ct.c_uint64(G), ct.byref(ccfg), ct.c_void_p(oh.data_ptr()),
            st_h, None))

    ms_e2e = timed(e2e_step, a.steps, a.warmup)
    clk = clock.stop()

    # ---- CPU baseline (rank 0, N=1): the reference on the same data, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and a.router == "centroid":
        lay = layers[0]
        sample = []
        for hl in range(min(heads_local, 8)):
            gi = hl  # sequence 0, KV head hl
            assign, _ = lay["L"].read_index(gi)
            sample.append({
                "cent": lay["parts"][hl].centroids,
                "K": lay["K"][gi * N:(gi + 1) * N].float().cpu().numpy(),
                "V": lay["V"][gi * N:(gi + 1) * N].float().cpu().numpy(),
                "assign": assign})
        qs = q.cpu().numpy()
        # reorder: store index = gi % heads_local matches group (s, hl)
        threads = cpu_threads(a)
        us_cpu, kind, cores, _ = run_cpu_reference(sample, qs, a, 2, 1, threads)
        cpu = {"value": round(us_cpu, 1), "unit": UNIT, "cores": cores, "kind": kind,
               "sample": (f"{len(sample)} distinct {N}-key contexts (layer 0, sequence 0, "
                          f"KV heads 0-{len(sample) - 1}) x {n_groups // len(sample)} query groups "
                          f"= {n_groups} groups = one full step's work, 2 timed steps")}

    peak, peak_kind = measured_peaks()
    us = ms_sparse * 1e3
    # per-rank algorithmic bytes / per-rank attention-kernel time
    achieved = (bytes_step / (attn_ms * 1e-3) / 1e9) if attn_ms else None
    line = {
        "metric": METRIC, "value": round(us, 3), "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_sparse, 5),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (device counter-based clustered keys, random unit centroids)",
        "config": workload_config(a, world),
        "dense_us_per_step": round(ms_dense * 1e3, 3) if ms_dense else None,
        "speedup_vs_dense": round(ms_dense / ms_sparse, 3) if ms_dense else None,
        "attention_time_reduction": round(1 - ms_sparse / ms_dense, 4) if ms_dense else None,
        "selectivity": round(ks_step / (n_groups * N), 5),
        "mse_vs_dense": float(np.mean(mse_vals)),
        "hbm_gbs": round(achieved, 1) if achieved else None,
        "kernel_us": {"route_plan": round(plan_ms * 1e3, 2), "sparse_attention": round(attn_ms * 1e3, 2),
                      "dense_attention": round(dense_attn_ms * 1e3, 2) if dense_attn_ms else None},
        "allgather_us": round(ms_gather * 1e3, 2) if ms_gather else None,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": ncu_traffic(),
                     "peak_kind": peak_kind,
                     "bytes_per_launch": int(bytes_step),
                     "dense_achieved": round(dense_bytes / (dense_attn_ms * 1e-3) / 1e9, 1)
                     if dense_attn_ms else None},
        "cpu_baseline": cpu,
        "e2e": {"value": round(ms_e2e * 1e3, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(q.numel() * 4),
                "d2h_bytes_per_step": int(out.numel() * 4 + n_groups * 24)},
        "clocks": clk,
        "gpu_launches": int(kernels_per_step * a.steps),
        "kernels_per_step": int(kernels_per_step),
        "prefill_build_ms_per_layer": round(float(np.mean(t_build)), 2),
        "plan_trace_cycles": plan_trace,
        "decode_trace": decode_trace,
        "step_trace_us": step_trace,
        "graph_plan_trace": graph_plan_trace,
        "prefill": {
            "keys": n_keys_prefill, "assign_ms": round(assign_ms, 3), "pack_ms": round(pack_ms, 3),
            "keys_per_s": round(n_keys_prefill / ((assign_ms + pack_ms) * 1e-3), 1),
            "assign_engine": "tcgen05" if used_tc else "fp64", "refined_keys": refined,
            "assign_tflops": round(2 * n_keys_prefill * C * d / (assign_ms * 1e-3) / 1e12, 1),
            "assign_frac_of_bf16_sustained": round(2 * n_keys_prefill * C * d / (assign_ms * 1e-3) / 1e12
                                                   / 1389.8, 4),
            "pack_gbs": round(pack_bytes / (pack_ms * 1e-3) / 1e9, 1),
            "pack_frac": round(pack_bytes / (pack_ms * 1e-3) / 1e9 / peak_early, 4),
        },
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
    else:
        ours(a)


if __name__ == "__main__":
    main()
