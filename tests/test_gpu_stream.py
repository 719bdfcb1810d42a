"""Parity of the decode-step machinery added for B200 (through the C ABI):

* fused cluster routing (8-CTA clusters per partition slot, DSMEM score
  exchange) -- CentroidRouter::select attention.cpp:275-306 + top_l_ids
  :259-271 -- on its fast set-only path, its exact ordered path
  (want_selected), its many-ties path, partial slots and fallback contexts;
* the tile stream (static window tiles + planner-published bucket tiles,
  guided tail chunking, streaming LSE combine) for several head chunks;
* the dense full-attention stream over many contexts (static only).

Reference: the oracle port / compiled reference on the same bf16 inputs.
Bit-exact: selected lists, keys_scored, max_visited_bucket.  Outputs:
oracles::max_rel_diff (floor 1e-3) <= 1e-3."""
import numpy as np
import pytest

import paper_2502_08246_b200 as sb
from oracle import bf16_round, max_rel_diff
from tests.cases import make_case, port_index, unit_rows

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _layer(ctx, cases, C, hint, parts_of):
    """Layer over `cases`; contexts i, j share a partition iff parts_of[i] == parts_of[j]."""
    ns = [c["K"].shape[0] for c in cases]
    uniq = {}
    for i, p in enumerate(parts_of):
        uniq.setdefault(p, sb.Partition(cases[i]["cent"], ctx))
    parts = [uniq[p] for p in parts_of]
    L = sb.Layer(ns, cases[0]["K"].shape[1], C, 1, hint, ctx)
    L.build(parts, np.concatenate([c["K"] for c in cases]), np.concatenate([c["V"] for c in cases]),
            np.concatenate([c["Kd"] for c in cases]))
    return L, [sb.CentroidRouter(p, True) for p in parts]


def _shared_cases(n_ctx, n, C, d, G, seed, n_each=None):
    """Contexts of one 'KV head': the same centroids, different keys/queries."""
    base = make_case(d=d, n=n, C=C, n_q=G, seed=seed, use_ref=False)
    out = []
    for i in range(n_ctx):
        c = make_case(d=d, n=(n_each[i] if n_each else n), C=C, n_q=G, seed=seed * 31 + i,
                      use_ref=False)
        c["cent"] = base["cent"]
        out.append(c)
    return out


def _check_layer(port, L, routers, cases, C, probes, recent, G, want_selected):
    qr = np.stack([c["qr"][:G] for c in cases])
    qd = np.stack([c["qd"][:G] for c in cases])
    cfg = sb.SparseAttnConfig(probes, 128, sb.DenseWindow(1, recent))
    out, stats, sel = L.sparse_attention(routers, qr, qd, cfg, want_selected=want_selected)
    for i, c in enumerate(cases):
        a, off, idx = port_index(port, c, C)
        n = c["K"].shape[0]
        ps = port.centroid_select(c["cent"], c["qd"][:G], probes) if n > 1 + recent else None
        if want_selected and ps is not None:
            assert np.array_equal(sel[i], ps), f"context {i}: selected list"
        o, ks, mv, em = port.sparse_attention(c["qr"][:G], c["K"], c["V"], 1, off, idx, ps, probes,
                                              128, recent)
        err = max_rel_diff(out[i], o)
        assert err <= TOL, f"context {i}: max_rel_diff {err}"
        assert (stats[i].keys_scored, stats[i].max_visited_bucket) == (ks, mv), f"context {i}"


@pytest.mark.parametrize("C", [256, 1024])
@pytest.mark.parametrize("want_selected", [False, True])
def test_cluster_routing_shared_partition(ctx, port, C, want_selected):
    """8 contexts share one partition: one full cluster (slot of 8)."""
    cases = _shared_cases(8, 6000, C, 128, 4, seed=C + 3)
    L, routers = _layer(ctx, cases, C, 2047, [0] * 8)
    _check_layer(port, L, routers, cases, C, 16, 2047, 4, want_selected)


def test_cluster_routing_partial_slots_and_fallback(ctx, port):
    """Slots of 3 and 2 contexts (idle owner CTAs) and two contexts shorter
    than the window (full attention inside the fused call)."""
    C = 512
    a = _shared_cases(3, 5000, C, 128, 4, seed=11, n_each=[5000, 1500, 7000])
    b = _shared_cases(2, 5000, C, 128, 4, seed=12, n_each=[900, 6500])
    cases = a + b
    L, routers = _layer(ctx, cases, C, 2047, [0, 0, 0, 1, 1])
    _check_layer(port, L, routers, cases, C, 12, 2047, 4, True)


@pytest.mark.parametrize("G", [8, 13])
def test_cluster_routing_head_chunks(ctx, port, G):
    """G > 4 query heads per context: several query slots per context share
    the context's static and bucket tiles."""
    C = 256
    cases = _shared_cases(4, 5000, C, 128, G, seed=40 + G)
    L, routers = _layer(ctx, cases, C, 2047, [0] * 4)
    _check_layer(port, L, routers, cases, C, 10, 2047, G, True)


def test_cluster_routing_many_ties(ctx, port):
    """Many identical centroids: the approximate boundary is ambiguous for more
    than 64 candidates, so the exact fp64 chains run for all of them and the
    (score desc, id asc) order decides."""
    C = 256
    cases = _shared_cases(8, 5000, C, 128, 4, seed=77)
    cent = cases[0]["cent"].copy()
    cent[40:140] = cent[7]  # 101 identical centroids
    for c in cases:
        c["cent"] = cent
    L, routers = _layer(ctx, cases, C, 2047, [0] * 8)
    _check_layer(port, L, routers, cases, C, 24, 2047, 4, True)
    _check_layer(port, L, routers, cases, C, 24, 2047, 4, False)


@pytest.mark.parametrize("d", [64, 32])
def test_cluster_routing_head_dims(ctx, port, d):
    C = 1024
    cases = _shared_cases(8, 5000, C, d, 4, seed=d)
    L, routers = _layer(ctx, cases, C, 1000, [0] * 8)
    _check_layer(port, L, routers, cases, C, 16, 1000, 4, True)


def test_repeated_steps_are_consistent(ctx, port):
    """Step state is re-armed between steps: ten identical steps give the same
    counters and outputs equal up to fp32 merge order (work is split into runs
    dynamically, so the LSE merges may associate differently)."""
    C = 1024
    cases = _shared_cases(8, 6000, C, 128, 4, seed=5)
    L, routers = _layer(ctx, cases, C, 2047, [0] * 8)
    qr = np.stack([c["qr"][:4] for c in cases])
    qd = np.stack([c["qd"][:4] for c in cases])
    cfg = sb.SparseAttnConfig(32, 128, sb.DenseWindow(1, 2047))
    ref = L.sparse_attention(routers, qr, qd, cfg)
    for _ in range(10):
        out, stats, _ = L.sparse_attention(routers, qr, qd, cfg)
        assert max_rel_diff(out, ref[0]) <= 1e-4
        assert [s.keys_scored for s in stats] == [s.keys_scored for s in ref[1]]


def test_dense_stream_many_contexts(ctx, port):
    """Full attention over 24 contexts of 20k keys (a static-only stream with
    big chunks, pairs and single-tile tail chunks)."""
    rs = np.random.RandomState(3)
    n, d, G = 20000, 128, 4
    cases = []
    for i in range(24):
        K = bf16_round(rs.randn(n, d).astype(np.float32))
        V = bf16_round(rs.randn(n, d).astype(np.float32))
        q = bf16_round((rs.randn(G, d) * 0.3).astype(np.float32))
        cases.append((q, K, V))
    cent = unit_rows(rs.randn(64, d))
    parts = [sb.Partition(cent, ctx)] * len(cases)
    L = sb.Layer([n] * len(cases), d, 64, 1, 2047, ctx)
    L.build(parts, np.concatenate([c[1] for c in cases]), np.concatenate([c[2] for c in cases]),
            np.concatenate([c[1] for c in cases]))
    full = L.full_attention(np.stack([c[0] for c in cases]))
    for i in (0, 7, 23):
        q, K, V = cases[i]
        assert max_rel_diff(full[i], port.full_attention(q, K, V)) <= TOL


def test_host_api_graph_replay_tracks_inputs(ctx, port):
    """saap_sparse_attention replays a cached CUDA graph from the third
    identical call on: new query values, a rebuilt layer and a replacement
    layer must all be honoured (graphs are retired with their layer)."""
    C = 256
    for rebuild in range(2):
        cases = _shared_cases(4, 5000, C, 128, 4, seed=11 + rebuild)
        L, routers = _layer(ctx, cases, C, 2047, [0] * 4)
        cfg = sb.SparseAttnConfig(16, 128, sb.DenseWindow(1, 2047))
        rs = np.random.RandomState(rebuild)
        for call in range(5):
            q = np.stack([bf16_round(c["qr"][:4] + 0.05 * call * rs.randn(4, 128).astype(np.float32))
                          for c in cases])
            out, stats, sel = L.sparse_attention(routers, q, q, cfg, want_selected=True)
            for i in (0, 3):
                c = cases[i]
                _, off, idx = port_index(port, c, C)
                want_sel = port.centroid_select(c["cent"], q[i], 16)
                assert np.array_equal(sel[i], want_sel)
                w, ks, mv = port.sparse_attention(q[i], c["K"], c["V"], 1, off, idx, want_sel, 16,
                                                  128, 2047)[:3]
                assert (stats[i].keys_scored, stats[i].max_visited_bucket) == (ks, mv)
                assert max_rel_diff(out[i], w) <= TOL
        del L, routers


def test_host_api_zero_copy_outputs(ctx, port):
    """Page-locked output / stats buffers (poisoned before each call) through
    the host API equal the pageable path, across graph replays."""
    import ctypes as ct

    import torch
    C = 256
    cases = _shared_cases(4, 5000, C, 128, 4, seed=21)
    L, routers = _layer(ctx, cases, C, 2047, [0] * 4)
    cfg = sb.SparseAttnConfig(16, 128, sb.DenseWindow(1, 2047))
    out_pin = torch.empty(4, 4, 128, pin_memory=True)
    st_pin = torch.empty(4 * ct.sizeof(sb.AttnStats), dtype=torch.uint8, pin_memory=True)
    st = (sb.AttnStats * 4).from_address(st_pin.data_ptr())
    rs = np.random.RandomState(4)
    for call in range(4):
        q = np.ascontiguousarray(np.stack([bf16_round(c["qr"][:4] + 0.1 * call * rs.randn(4, 128).astype(np.float32))
                                           for c in cases]))
        want, wst, _ = L.sparse_attention(routers, q, q, cfg)
        out_pin.fill_(np.nan)
        st_pin.fill_(0xFF)
        c = cfg.c()
        sb._check(sb.lib().saap_sparse_attention(
            ctx.h, L.h, L._routers(routers), q.ctypes.data_as(ct.c_void_p),
            q.ctypes.data_as(ct.c_void_p), ct.c_uint64(4), ct.byref(c),
            ct.c_void_p(out_pin.data_ptr()), st, None))
        got = out_pin.numpy()
        assert np.isfinite(got).all()
        assert max_rel_diff(got, want) <= 1e-4
        assert [s.keys_scored for s in st] == [s.keys_scored for s in wst]
        assert [s.max_visited_bucket for s in st] == [s.max_visited_bucket for s in wst]


@pytest.mark.parametrize("G", [4, 13])
def test_tcgen05_decode_parity(ctx, port, G):
    """The tcgen05 consumers (`decode_tc` option: S^T = K Q^T and O^T += V^T P^T
    on the tensor cores, TMEM accumulators, a Q warp per run) against the
    oracle: routed steps with several head chunks and the ordered path, then
    full attention over many contexts."""
    ctx.set_option("decode_tc", 1)
    try:
        C = 1024
        cases = _shared_cases(8, 6000, C, 128, G, seed=91 + G)
        L, routers = _layer(ctx, cases, C, 2047, [0] * 8)
        _check_layer(port, L, routers, cases, C, 16, 2047, G, False)
        _check_layer(port, L, routers, cases, C, 16, 2047, G, True)
        rs = np.random.RandomState(17)
        n, d = 9000, 128
        fc = []
        for i in range(6):
            K = bf16_round(rs.randn(n, d).astype(np.float32))
            V = bf16_round(rs.randn(n, d).astype(np.float32))
            q = bf16_round((rs.randn(G, d) * 0.3).astype(np.float32))
            fc.append((q, K, V))
        cent = unit_rows(rs.randn(64, d))
        Lf = sb.Layer([n] * len(fc), d, 64, 1, 2047, ctx)
        Lf.build([sb.Partition(cent, ctx)] * len(fc), np.concatenate([c[1] for c in fc]),
                 np.concatenate([c[2] for c in fc]), np.concatenate([c[1] for c in fc]))
        full = Lf.full_attention(np.stack([c[0] for c in fc]))
        for i in range(len(fc)):
            q, K, V = fc[i]
            assert max_rel_diff(full[i], port.full_attention(q, K, V)) <= TOL
    finally:
        ctx.set_option("decode_tc", 0)
