"""The multi-GPU data path on one GPU (one rank: the box has one GPU per
call): saap_comm over NCCL, the registered send buffer the decode writes
into, and the head all-gather + permute against shard.gather_layout."""
import numpy as np
import pytest

import paper_2502_08246_b200 as sb
from paper_2502_08246_b200.shard import Comm, HeadShard, gather_layout, unique_id


@pytest.mark.gpu
def test_allgather_heads_world1(ctx):
    import torch
    comm = Comm(ctx, 1, 0, unique_id())
    try:
        info = comm.info()
        assert info["nranks"] == 1 and info["rank"] == 0 and info["nccl_version"] > 0
        sh = HeadShard(0, 1, kv_heads=8, batch=3)
        G, d = 4, 128
        rng = np.random.default_rng(5)
        local = rng.standard_normal((sh.n_groups, G, d)).astype(np.float32)
        ptr = comm.send_buffer(local.nbytes)
        assert ptr
        dev = torch.device("cuda", ctx.device)
        src = torch.from_numpy(local).to(dev)
        torch.cuda.synchronize()
        want = gather_layout(local[None], sh)
        # from an ordinary buffer: copied into the send buffer, gathered, permuted
        full = torch.empty(sh.batch, sh.kv_heads * G, d, device=dev)
        comm.allgather_heads(src, sh, G, d, full)
        ctx.synchronize()
        assert np.array_equal(full.cpu().numpy(), want)
        # straight from the send buffer (the decode step's target): no copy
        full2 = torch.zeros_like(full)
        comm.allgather_heads(ptr, sh, G, d, full2)
        ctx.synchronize()
        assert np.array_equal(full2.cpu().numpy(), want)
    finally:
        comm.close()


@pytest.mark.gpu
def test_comm_rejects_bad_rank(ctx):
    with pytest.raises(sb.InvalidArgument):
        Comm(ctx, 2, 2, unique_id())
