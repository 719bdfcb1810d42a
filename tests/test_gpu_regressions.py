"""Regression tests for the round-1 advisor findings, through
the C ABI:

* a saved host step graph must not outlive the gather buffer it was captured
  with (recent_count alternating across a larger skew);
* a saved host step graph must rebind the layer's router tables when another
  router set ran on the layer in between (two partitions alternating);
* pattn_absorb / attention_over_ids reject a key block whose dim differs from
  the queries' (absorb_impl attention.cpp:40-43);
* PartialAccumulator(h, 0) starts at sumexp 0 / runmax -inf (attention.cpp:82-83);
* CentroidRouter::select with an empty group returns ids 0..l-1
  (attention.cpp:284-305: pooled = 0 scores every centroid 0).
"""
import numpy as np
import pytest

import paper_2502_08246_b200 as sb
from oracle import max_rel_diff
from tests.cases import make_case, port_index

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _oracle_step(port, c, C, G, probes, recent, cent=None):
    cent = c["cent"] if cent is None else cent
    a = port.assign_keys(c["Kd"][1:], cent)
    off, idx = port.build_ivf(a, C)
    n = c["K"].shape[0]
    ps = port.centroid_select(cent, c["qd"][:G], probes) if n > 1 + recent else None
    o, ks, mv, _ = port.sparse_attention(c["qr"][:G], c["K"], c["V"], 1, off, idx, ps, probes, 128,
                                         recent)
    return ps, o, ks, mv


def test_host_graph_survives_gather_realloc(ctx, port):
    C, G, probes, d = 256, 4, 8, 64
    cases = [make_case(d=d, n=n, C=C, n_q=G, seed=40 + i, use_ref=False) for i, n in enumerate([6000, 7000])]
    hint = 1023
    L = sb.Layer([c["K"].shape[0] for c in cases], d, C, 1, hint, ctx)
    parts = [sb.Partition(c["cent"], ctx) for c in cases]
    L.build(parts, np.concatenate([c["K"] for c in cases]), np.concatenate([c["V"] for c in cases]),
            np.concatenate([c["Kd"] for c in cases]))
    routers = [sb.CentroidRouter(p, True) for p in parts]
    qr = np.stack([c["qr"][:G] for c in cases])
    qd = np.stack([c["qd"][:G] for c in cases])
    # r1 needs a small gather buffer, r2 a larger one (reallocated), then r1 again:
    # r1's saved graph was captured with the old buffer and must be re-captured
    for recent in [700, 700, 700, 200, 200, 700, 700, hint, 700]:
        cfg = sb.SparseAttnConfig(probes, 128, sb.DenseWindow(1, recent))
        out, stats, sel = L.sparse_attention(routers, qr, qd, cfg, want_selected=True)
        for i, c in enumerate(cases):
            ps, o, ks, mv = _oracle_step(port, c, C, G, probes, recent)
            assert np.array_equal(sel[i], ps), (recent, i)
            assert (stats[i].keys_scored, stats[i].max_visited_bucket) == (ks, mv), (recent, i)
            assert max_rel_diff(out[i], o) <= TOL, (recent, i)


def test_host_graph_rebinds_router_tables(ctx, port):
    C, G, probes, d = 256, 4, 16, 128
    cases = [make_case(d=d, n=5000, C=C, n_q=G, seed=60 + i, use_ref=False) for i in range(3)]
    other = make_case(d=d, n=5000, C=C, n_q=G, seed=99, use_ref=False)["cent"]
    L = sb.Layer([c["K"].shape[0] for c in cases], d, C, 1, 1023, ctx)
    pa = [sb.Partition(c["cent"], ctx) for c in cases]
    pb = sb.Partition(other, ctx)
    L.build(pa, np.concatenate([c["K"] for c in cases]), np.concatenate([c["V"] for c in cases]),
            np.concatenate([c["Kd"] for c in cases]))
    ra = [sb.CentroidRouter(p, True) for p in pa]
    rb = [sb.CentroidRouter(pb, True) for _ in cases]  # routes with other centroids
    qr = np.stack([c["qr"][:G] for c in cases])
    qd = np.stack([c["qd"][:G] for c in cases])
    cfg = sb.SparseAttnConfig(probes, 128, sb.DenseWindow(1, 1023))
    for tag in "AABBABAA":
        routers = ra if tag == "A" else rb
        out, stats, sel = L.sparse_attention(routers, qr, qd, cfg, want_selected=True)
        for i, c in enumerate(cases):
            cent = c["cent"] if tag == "A" else other
            ps = port.centroid_select(cent, c["qd"][:G], probes)
            assert np.array_equal(sel[i], ps), (tag, i)
            # attention reads the store's buckets (assigned with the build's
            # partition) at the ids the router picked
            a = port.assign_keys(c["Kd"][1:], c["cent"])
            off, idx = port.build_ivf(a, C)
            o, ks, mv, _ = port.sparse_attention(c["qr"][:G], c["K"], c["V"], 1, off, idx, ps, probes,
                                                 128, 1023)
            assert (stats[i].keys_scored, stats[i].max_visited_bucket) == (ks, mv), (tag, i)
            assert max_rel_diff(out[i], o) <= TOL, (tag, i)


def test_absorb_key_dim_mismatch(ctx):
    q = np.zeros((2, 8), np.float32)
    K = np.zeros((10, 6), np.float32)
    V = np.zeros((10, 5), np.float32)
    acc = sb.PartialAccumulator(2, 5, ctx)
    with pytest.raises(sb.InvalidArgument, match="pattn_absorb: query dim 8 vs key dim 6"):
        sb.pattn_absorb(acc, q, K, V, [1])
    with pytest.raises(sb.InvalidArgument, match="pattn_absorb: query dim 8 vs key dim 6"):
        sb.pattn_absorb_range(acc, q, K, V, 0, 3)
    with pytest.raises(sb.InvalidArgument, match="pattn_absorb: query dim 8 vs key dim 6"):
        sb.attention_over_ids(q, K, V, [0, 1], ctx)
    # check_kv and check_acc come first (absorb_impl :38-39)
    with pytest.raises(sb.InvalidArgument, match="attention: 10 keys vs 9 values"):
        sb.pattn_absorb(acc, q, K, V[:9], [1])


def test_accumulator_zero_value_dim(ctx):
    acc = sb.PartialAccumulator(3, 0, ctx)
    out, se, rm = acc.state()
    assert out.shape == (3, 0)
    assert not se.any() and np.isneginf(rm).all()
    part = sb.PartialAccumulator(3, 0, ctx)
    sb.merge_into(acc, part)
    fin, empty = sb.pattn_finalize(acc)
    assert fin.shape == (3, 0) and empty


def test_centroid_router_empty_group(ctx, port):
    cent = make_case(d=64, n=2000, C=64, n_q=4, seed=5, use_ref=False)["cent"]
    r = sb.CentroidRouter(sb.Partition(cent, ctx), True)
    q = np.zeros((0, 64), np.float32)
    got = r.select(q, q, 5)
    assert list(got) == [0, 1, 2, 3, 4]
    assert list(port.centroid_select(cent, q, 5)) == [0, 1, 2, 3, 4]
    import oracle
    if oracle.ref_available():
        assert list(oracle.ref().centroid_select(cent, q, q, 5)) == [0, 1, 2, 3, 4]
