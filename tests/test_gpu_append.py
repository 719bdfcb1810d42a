"""Incremental decode index (saap_layer_append): after
every append the layer must equal build_context_store over the grown
context -- assignments / off / idx bit-exact, and sparse_attention's
selected lists, keys_scored and max_visited_bucket bit-exact with outputs
within 1e-3 of the oracle computed from scratch on the prefix."""
import numpy as np
import pytest

import paper_2502_08246_b200 as sb
from oracle import max_rel_diff
from tests.cases import make_case

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _ref_step(port, case, n, C, q, probes, recent):
    a = port.assign_keys(case["Kd"][1:n], case["cent"])
    off, idx = port.build_ivf(a, C)
    sel = port.centroid_select(case["cent"], q, probes) if probes else np.zeros(0, np.uint32)
    out, ks, mv, _ = port.sparse_attention(q, case["K"][:n], case["V"][:n], 1, off, idx, sel, probes,
                                           128, recent)
    return a, off, idx, sel, out, ks, mv


@pytest.mark.parametrize("d,hint", [(128, 512), (64, 300)])
def test_append_matches_fresh_build(ctx, port, d, hint):
    C, n0, grow = 64, 3000, 600
    cases = [make_case(d=d, n=n0 + grow, C=C, n_q=4, seed=40 + i, use_ref=False) for i in range(3)]
    parts = [sb.Partition(c["cent"], ctx) for c in cases]
    L = sb.Layer([n0] * 3, d, C, 1, hint, ctx, capacity=n0 + grow)
    L.build(parts, np.concatenate([c["K"][:n0] for c in cases]),
            np.concatenate([c["V"][:n0] for c in cases]),
            np.concatenate([c["Kd"][:n0] for c in cases]))
    routers = [sb.CentroidRouter(p, True) for p in parts]
    q = np.stack([c["qr"][:4] for c in cases])
    n = n0
    for k in (1, 7, 64, 200, 328):
        L.append(np.stack([c["K"][n:n + k] for c in cases]), np.stack([c["V"][n:n + k] for c in cases]),
                 np.stack([c["Kd"][n:n + k] for c in cases]))
        n += k
        for probes, recent in ((8, hint), (8, hint // 2), (16, hint + 100), (0, hint)):
            cfg = sb.SparseAttnConfig(probes, 128, sb.DenseWindow(1, recent))
            out, stats, sel = L.sparse_attention(routers, q, q, cfg, want_selected=probes > 0)
            for i in range(3):
                a, off, idx, wsel, w, ks, mv = _ref_step(port, cases[i], n, C, q[i], probes, recent)
                if probes:
                    assert np.array_equal(sel[i], wsel)
                assert (stats[i].keys_scored, stats[i].max_visited_bucket) == (ks, mv), (k, probes, recent)
                assert max_rel_diff(out[i], w) <= TOL
        ga, gix = L.read_index(1)
        a, off, idx = _ref_step(port, cases[1], n, C, q[1], 0, hint)[:3]
        assert np.array_equal(ga, a) and np.array_equal(gix.off, off) and np.array_equal(gix.idx, idx)
    with pytest.raises(sb.InvalidArgument, match="exceed its capacity"):
        L.append(np.zeros((3, 1, d), np.float32), np.zeros((3, 1, d), np.float32),
                 np.zeros((3, 1, d), np.float32))


def test_append_graph_steps_and_rebuild(ctx, port):
    """Host-API graph replays are retired by an append; a later full build
    over the grown contexts (the compaction) gives the same results."""
    C, n0, d, hint = 128, 4000, 128, 1024
    case = make_case(d=d, n=n0 + 300, C=C, n_q=4, seed=7, use_ref=False)
    p = sb.Partition(case["cent"], ctx)
    L = sb.Layer([n0], d, C, 1, hint, ctx, capacity=n0 + 300)
    L.build([p], case["K"][:n0], case["V"][:n0], case["Kd"][:n0])
    r = [sb.CentroidRouter(p, True)]
    q = case["qr"][None, :4]
    cfg = sb.SparseAttnConfig(16, 128, sb.DenseWindow(1, hint))
    for _ in range(3):  # eager, capture, replay
        L.sparse_attention(r, q, q, cfg)
    n = n0
    for k in (50, 250):
        L.append(case["K"][None, n:n + k], case["V"][None, n:n + k], case["Kd"][None, n:n + k])
        n += k
        for _ in range(3):
            out, stats, _ = L.sparse_attention(r, q, q, cfg)
            w, ks, mv = _ref_step(port, case, n, C, q[0], 16, hint)[4:]
            assert (stats[0].keys_scored, stats[0].max_visited_bucket) == (ks, mv)
            assert max_rel_diff(out[0], w) <= TOL
    L2 = sb.Layer([n], d, C, 1, hint, ctx)
    L2.build([p], case["K"][:n], case["V"][:n], case["Kd"][:n])
    out2, st2, _ = L2.sparse_attention(r, q, q, cfg)
    assert st2[0].keys_scored == stats[0].keys_scored
    assert max_rel_diff(out2[0], out[0]) <= TOL


def test_capacity_layout_device_build_tcgen05(ctx, port):
    """Device build (tcgen05 assignment at d=128) into a layer with spare
    capacity per context: index and attention equal the reference."""
    import torch
    C, d, hint = 256, 128, 1024
    cases = [make_case(d=d, n=6000 + 500 * i, C=C, n_q=4, seed=60 + i, use_ref=False) for i in range(3)]
    ns = [c["K"].shape[0] for c in cases]
    parts = [sb.Partition(c["cent"], ctx) for c in cases]
    L = sb.Layer(ns, d, C, 1, hint, ctx, capacity=[n + 777 for n in ns])
    dev = torch.device("cuda", 0)
    cat = lambda k: torch.from_numpy(np.concatenate([c[k] for c in cases])).to(dev).to(torch.bfloat16)
    K, V, Kd = cat("K"), cat("V"), cat("Kd")
    torch.cuda.synchronize()
    L.build_dev(parts, K, V, Kd)
    ctx.synchronize()
    routers = [sb.CentroidRouter(p, True) for p in parts]
    q = np.stack([c["qr"][:4] for c in cases])
    cfg = sb.SparseAttnConfig(16, 128, sb.DenseWindow(1, hint))
    out, stats, _ = L.sparse_attention(routers, q, q, cfg)
    for i, c in enumerate(cases):
        ga, gix = L.read_index(i)
        a, off, idx, sel, w, ks, mv = _ref_step(port, c, ns[i], C, q[i], 16, hint)
        assert np.array_equal(ga, a) and np.array_equal(gix.off, off) and np.array_equal(gix.idx, idx)
        assert (stats[i].keys_scored, stats[i].max_visited_bucket) == (ks, mv)
        assert max_rel_diff(out[i], w) <= TOL


def test_append_with_qmodel_router(ctx, port):
    """Appends under the Q-model router (the learned SAAP classifier)."""
    import oracle
    if not oracle.ref_available():
        pytest.skip("needs oracle/_ref for qmodel_init")
    C, d, hint, n0, grow = 64, 64, 400, 2500, 300
    m = oracle.ref().qmodel_init(d, 128, C, 5)
    case = make_case(d=d, n=n0 + grow, C=C, n_q=4, seed=77, use_ref=False)
    p = sb.Partition(case["cent"], ctx)
    L = sb.Layer([n0], d, C, 1, hint, ctx, capacity=n0 + grow)
    L.build([p], case["K"][:n0], case["V"][:n0], case["Kd"][:n0])
    r = [sb.QModelRouter(sb.QModel(m, ctx))]
    q = case["qr"][None, :4]
    n = n0
    for k in (3, 297):
        L.append(case["K"][None, n:n + k], case["V"][None, n:n + k], case["Kd"][None, n:n + k])
        n += k
        cfg = sb.SparseAttnConfig(8, 128, sb.DenseWindow(1, hint))
        out, stats, sel = L.sparse_attention(r, q, q, cfg, want_selected=True)
        a = port.assign_keys(case["Kd"][1:n], case["cent"])
        off, idx = port.build_ivf(a, C)
        wsel = port.qmodel_select(m, q[0], 8)
        assert np.array_equal(sel[0], wsel)
        w, ks, mv, _ = port.sparse_attention(q[0], case["K"][:n], case["V"][:n], 1, off, idx, wsel, 8,
                                             128, hint)
        assert (stats[0].keys_scored, stats[0].max_visited_bucket) == (ks, mv)
        assert max_rel_diff(out[0], w) <= TOL
