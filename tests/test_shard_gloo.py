"""Multi-rank host logic of the head-sharded decode step, world_size 2 on
CPU with gloo: shard ownership and the all-gather layout."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_08246_b200.shard import HeadShard, gather_outputs


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = HeadShard(rank, world, kv_heads=8, batch=3)
        G, d = 4, 16
        out = torch.empty(sh.n_groups, G, d)
        for g in range(sh.n_groups):
            s, h = sh.head_of(g)
            for j in range(G):
                out[g, j] = s * 1000 + (h * G + j) + torch.arange(d) / 100.0
        full = gather_outputs(out, sh, dist)
        want = torch.empty(3, 8 * G, d)
        for s in range(3):
            for qh in range(8 * G):
                want[s, qh] = s * 1000 + qh + torch.arange(d) / 100.0
        q.put((rank, bool(torch.equal(full, want)), sh.head0, sh.heads_local))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_head_shard_allgather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res)
    assert [(h0, hl) for _, _, h0, hl in res] == [(0, 4), (4, 4)]


def test_shard_validation():
    with pytest.raises(ValueError):
        HeadShard(0, 3, kv_heads=8, batch=1)
    sh = HeadShard(1, 2, kv_heads=8, batch=2)
    assert sh.group(1, 5) == 5 and sh.head_of(5) == (1, 5)
    with pytest.raises(ValueError):
        sh.group(0, 1)
