"""KV-head sharding of a decode step over ranks.

One process per GPU.  Each rank owns a contiguous block of KV heads for every
sequence; under GQA its query heads need no other rank's keys, so the only
exchange per layer step is gathering the per-head attention outputs.  The
geometry (``saap_shard_heads``) and the gather (``saap_allgather_heads``:
NCCL all-gather into symmetric-window buffers + a permute kernel) are the
C ABI's; this module only binds them.  Exchanging the 128-byte NCCL unique id
is the caller's plumbing (any channel: a TCP store, MPI, a file).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import Context, _check, _dptr, _u64, lib


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_heads: int
    batch: int

    def __post_init__(self):
        h0, hl = C.c_uint64(), C.c_uint64()
        try:
            _check(lib().saap_shard_heads(_u64(self.kv_heads), C.c_int(self.world),
                                          C.c_int(self.rank), C.byref(h0), C.byref(hl)))
        except ValueError as e:
            raise ValueError(str(e)) from None
        object.__setattr__(self, "_h0", h0.value)
        object.__setattr__(self, "_hl", hl.value)

    @property
    def heads_local(self) -> int:
        return self._hl

    @property
    def head0(self) -> int:
        return self._h0

    @property
    def n_groups(self) -> int:
        """(sequence, local KV head) contexts on this rank."""
        return self.batch * self.heads_local

    def group(self, seq: int, head: int) -> int:
        """Local group index of (sequence, global KV head) owned by this rank."""
        hl = head - self.head0
        if not 0 <= hl < self.heads_local:
            raise ValueError(f"head {head} is not on rank {self.rank}")
        return seq * self.heads_local + hl

    def head_of(self, group: int) -> tuple:
        s, hl = divmod(group, self.heads_local)
        return s, self.head0 + hl


def gather_layout(blocks, shard: HeadShard):
    """Host statement of what saap_allgather_heads produces: rank blocks
    [world][batch*heads_local][G][d] -> [batch][kv_heads*G][d] (query heads
    in model order).  Used by the tests as the layout oracle."""
    b = np.asarray(blocks)
    w, _, G, d = b.shape
    hl = shard.heads_local
    full = b.reshape(w, shard.batch, hl, G, d).transpose(1, 0, 2, 3, 4)
    return full.reshape(shard.batch, shard.kv_heads * G, d)


def unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 creates it and hands it to every rank)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().saap_comm_unique_id(buf))
    return bytes(buf)


class Comm:
    """saap_comm: the NCCL communicator of the head-sharded step."""

    def __init__(self, ctx: Context, world: int, rank: int, uid: bytes):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.ctx, self.world, self.rank = ctx, world, rank
        h = C.c_void_p()
        _check(lib().saap_comm_init(ctx.h, C.c_int(world), C.c_int(rank),
                                    (C.c_uint8 * 128).from_buffer_copy(uid), C.byref(h)))
        self.h = h

    def info(self):
        n, r, sym, ver = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().saap_comm_info(self.h, C.byref(n), C.byref(r), C.byref(sym), C.byref(ver)))
        return {"nranks": n.value, "rank": r.value, "symmetric": bool(sym.value),
                "nccl_version": ver.value}

    def send_buffer(self, nbytes: int) -> int:
        """Device pointer of the registered send buffer (write the step's
        outputs here: the gather then needs no copy)."""
        p = C.c_void_p()
        _check(lib().saap_comm_send_buffer(self.h, _u64(nbytes), C.byref(p)))
        return p.value

    def allgather_heads(self, out_local, shard: HeadShard, G: int, d: int, out_full):
        """[batch*heads_local, G, d] on each rank -> [batch, kv_heads*G, d]."""
        _check(lib().saap_allgather_heads(self.ctx.h, self.h, _dptr(out_local), _u64(shard.batch),
                                          _u64(shard.heads_local), _u64(G), _u64(d),
                                          _dptr(out_full)))

    def close(self):
        if getattr(self, "h", None):
            lib().saap_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class P2P:
    """saap_p2p: the fused output exchange over peer memory.  The step's
    combine kernel stores every finished slot's rows into each rank's full
    output buffer [batch][kv_heads][G][d] and bumps its arrival counter;
    `wait` orders the context stream after one step's deliveries."""

    def __init__(self, ctx: Context, world: int, rank: int, full_bytes: int):
        self.ctx, self.world, self.rank, self.full_bytes = ctx, world, rank, full_bytes
        h = C.c_void_p()
        _check(lib().saap_p2p_create(ctx.h, C.c_int(world), C.c_int(rank), _u64(full_bytes), C.byref(h)))
        self.h = h

    def handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        _check(lib().saap_p2p_handle(self.h, buf))
        return bytes(buf)

    def open(self, handles):
        if len(handles) != self.world or any(len(x) != 64 for x in handles):
            raise ValueError("one 64-byte handle per rank")
        blob = b"".join(handles)
        _check(lib().saap_p2p_open(self.h, (C.c_uint8 * len(blob)).from_buffer_copy(blob)))

    def buffer(self) -> int:
        p = C.c_void_p()
        _check(lib().saap_p2p_buffer(self.h, C.byref(p)))
        return p.value

    def attach(self, shard: HeadShard):
        _check(lib().saap_p2p_attach(self.ctx.h, self.h, _u64(shard.heads_local), _u64(shard.head0),
                                     _u64(shard.kv_heads)))

    def detach(self):
        _check(lib().saap_p2p_attach(self.ctx.h, None, _u64(0), _u64(0), _u64(0)))

    def wait(self, arrivals: int):
        _check(lib().saap_p2p_wait(self.ctx.h, self.h, _u64(arrivals)))

    def read(self, shape) -> np.ndarray:
        out = np.empty(shape, np.float32)
        _check(lib().saap_p2p_read(self.h, out.ctypes.data_as(C.c_void_p), _u64(out.nbytes)))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().saap_p2p_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
