"""Fused output exchange over peer memory (saap_p2p), exercised by two ranks
as two processes on the one GPU a call gets (CUDA IPC mappings between
processes on one device; between GPUs the same stores go over NVLink P2P).
Each rank routes and attends its own KV heads; the combine kernel stores
every finished slot's rows into both ranks' full buffers and bumps their
arrival counters, saap_p2p_wait orders the stream after the deliveries.
Checked: both full buffers equal the gather of the ranks' local outputs
(shard.gather_layout), over repeated steps and a captured graph."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank(rank, world, q_handles, q_out, q_res):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2502_08246_b200 as sb
    from paper_2502_08246_b200.shard import HeadShard, P2P
    from tests.cases import make_case
    try:
        batch, kv_heads, G, d, C, n = 2, 4, 4, 128, 256, 6000
        sh = HeadShard(rank, world, kv_heads=kv_heads, batch=batch)
        ctx = sb.Context(0)
        dev = torch.device("cuda", 0)
        cases = [make_case(d=d, n=n, C=C, n_q=G, seed=100 * rank + 7 * gi, use_ref=False)
                 for gi in range(sh.n_groups)]
        parts = [sb.Partition(c["cent"], ctx) for c in cases]
        L = sb.Layer([n] * sh.n_groups, d, C, 1, 2047, ctx)
        L.build(parts, np.concatenate([c["K"] for c in cases]), np.concatenate([c["V"] for c in cases]),
                np.concatenate([c["Kd"] for c in cases]))
        routers = [sb.CentroidRouter(p, True) for p in parts]
        qr = torch.from_numpy(np.stack([c["qr"][:G] for c in cases])).to(dev)
        qd = torch.from_numpy(np.stack([c["qd"][:G] for c in cases])).to(dev)
        cfg = sb.SparseAttnConfig(16, 128, sb.DenseWindow(1, 2047))
        out = torch.zeros(sh.n_groups, G, d, device=dev)
        stats = torch.zeros(sh.n_groups, 3, dtype=torch.int64, device=dev)
        full_bytes = batch * kv_heads * G * d * 4
        p2p = P2P(ctx, world, rank, full_bytes)
        q_handles[rank] = p2p.handle()  # (a manager dict: any channel works, like the NCCL id)
        import time
        t0 = time.time()
        while len(q_handles) < world:
            if time.time() - t0 > 120:
                raise TimeoutError("peer handles")
            time.sleep(0.01)
        p2p.open([q_handles[r] for r in range(world)])
        p2p.attach(sh)
        arrivals = world * sh.n_groups  # G = 4: one query slot per group
        results = []
        for step in range(3):
            L.sparse_attention_dev(routers, qr, qd, G, cfg, out, stats)
            p2p.wait(arrivals)
            ctx.synchronize()
            results.append((out.cpu().numpy().copy(), p2p.read((batch, kv_heads * G, d))))
        # the same step captured in a graph and replayed
        ctx.graph_begin()
        L.sparse_attention_dev(routers, qr, qd, G, cfg, out, stats)
        p2p.wait(arrivals)
        g = ctx.graph_end()
        for _ in range(2):
            g.launch()
        ctx.synchronize()
        results.append((out.cpu().numpy().copy(), p2p.read((batch, kv_heads * G, d))))
        q_out.put((rank, [r[0] for r in results]))
        q_res.put((rank, [r[1] for r in results], None))
        p2p.detach()
        import time
        time.sleep(2.0)  # peers may still read this rank's mapping
        p2p.close()
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q_res.put((rank, None, traceback.format_exc()))


@pytest.mark.gpu
def test_p2p_fused_exchange_two_ranks_one_gpu():
    from paper_2502_08246_b200.shard import HeadShard, gather_layout
    world = 2
    ctxm = mp.get_context("spawn")
    manager = ctxm.Manager()
    q_handles, q_out, q_res = manager.dict(), ctxm.Queue(), ctxm.Queue()
    procs = [ctxm.Process(target=_rank, args=(r, world, q_handles, q_out, q_res)) for r in range(world)]
    for p in procs:
        p.start()
    res, outs = {}, {}
    try:
        for _ in range(world):
            r, full, err = q_res.get(timeout=600)
            assert err is None, err
            res[r] = full
        for _ in range(world):
            r, o = q_out.get(timeout=60)
            outs[r] = o
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    sh = HeadShard(0, world, kv_heads=4, batch=2)
    for k in range(4):  # 3 eager steps + graph replays
        want = gather_layout(np.stack([outs[r][k] for r in range(world)]), sh)
        for r in range(world):
            assert np.array_equal(res[r][k], want), f"rank {r}, step {k}"
