"""Multi-rank host logic of the head-sharded decode step, world_size 2 on
CPU with gloo: shard ownership (saap_shard_heads), the NCCL unique-id
hand-off, and the gathered output layout (shard.gather_layout, the oracle the
GPU test holds saap_allgather_heads to)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_08246_b200.shard import HeadShard, gather_layout, unique_id


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = HeadShard(rank, world, kv_heads=8, batch=3)
        G, d = 4, 16
        # the id rank 0 creates reaches every rank unchanged (the plumbing the
        # bench uses before saap_comm_init)
        box = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, box[0])
        out = np.empty((sh.n_groups, G, d), np.float32)
        for g in range(sh.n_groups):
            s, h = sh.head_of(g)
            for j in range(G):
                out[g, j] = s * 1000 + (h * G + j) + np.arange(d) / 100.0
        blocks = [None] * world
        dist.all_gather_object(blocks, out)
        full = gather_layout(np.stack(blocks), sh)
        want = np.empty((3, 8 * G, d), np.float32)
        for s in range(3):
            for qh in range(8 * G):
                want[s, qh] = s * 1000 + qh + np.arange(d) / 100.0
        owned = sorted(sh.head_of(g)[1] for g in range(sh.n_groups) if sh.head_of(g)[0] == 0)
        q.put((rank, bool(np.array_equal(full, want)), sh.head0, sh.heads_local,
               len(set(ids)) == 1 and len(ids[0]) == 128, owned))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_head_shard_gather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _, _, _ in res)
    assert [(h0, hl) for _, _, h0, hl, _, _ in res] == [(0, 4), (4, 4)]
    assert all(uid_ok for *_, uid_ok, _ in res)
    assert sorted(h for *_, owned in res for h in owned) == list(range(8))


def test_shard_validation():
    with pytest.raises(ValueError):
        HeadShard(0, 3, kv_heads=8, batch=1)
    sh = HeadShard(1, 2, kv_heads=8, batch=2)
    assert sh.group(1, 5) == 5 and sh.head_of(5) == (1, 5)
    with pytest.raises(ValueError):
        sh.group(0, 1)
    assert [HeadShard(r, 8, 8, 1).head0 for r in range(8)] == list(range(8))
