"""Parity of the CUDA path (through the C ABI) with the reference / oracle.

Bit-exact: assignments, IVF off/idx, routed bucket lists, keys_scored,
max_visited_bucket, empty_attention.  Outputs: oracles::max_rel_diff
(proj/tests/support/oracles.hpp:122-130, floor 1e-3) <= 1e-3, the north-star
tolerance for fp32 accumulation of bf16 inputs."""
import math
import os

import numpy as np
import pytest

import oracle
import paper_2502_08246_b200 as sb
from oracle import bf16_round, max_rel_diff
from tests.cases import make_case, port_index, unit_rows

pytestmark = pytest.mark.gpu
TOL = 1e-3
GOLD = os.path.join(os.path.dirname(__file__), "golden", "saap_small.npz")


@pytest.fixture(scope="module")
def g():
    return dict(np.load(GOLD))


# ------------------------------------------------------------------ assignment
@pytest.mark.parametrize("d", [32, 64, 128])
@pytest.mark.parametrize("C", [16, 1024])
def test_assign_keys_bit_exact(ctx, port, d, C):
    rs = np.random.RandomState(d + C)
    cent = unit_rows(rs.randn(C, d))
    cent[5] = cent[2]  # exact tie: the lower id must win
    keys = (rs.randn(3000, d) * 2).astype(np.float32)  # f32, not bf16-representable
    keys[0] = 0.0  # all-zero key -> bucket 0
    keys[1] = cent[2] * 3.5
    part = sb.Partition(cent, ctx)
    got = sb.assign_keys(keys, part)
    want = port.assign_keys(keys, cent)
    assert np.array_equal(got, want)
    assert got[0] == 0 and got[1] == 2


def test_assign_keys_golden(ctx, g):
    part = sb.Partition(g["cent"], ctx)
    assert np.array_equal(sb.assign_keys(g["Kd"][1:], part), g["assign"])


def test_assign_dim_mismatch_raises(ctx):
    part = sb.Partition(unit_rows(np.random.randn(8, 32)), ctx)
    with pytest.raises(sb.InvalidArgument, match="assign_key: key dim"):
        sb.assign_keys(np.zeros((4, 64), np.float32), part)


# ------------------------------------------------------------------ IVF
@pytest.mark.parametrize("n,C", [(1, 1), (4, 2), (7, 3), (5000, 16), (70000, 1024), (20000, 16384)])
def test_build_ivf_bit_exact(ctx, port, n, C):
    rs = np.random.RandomState(n + C)
    a = rs.randint(0, C, n).astype(np.uint32)
    got = sb.build_ivf(a, C, ctx)
    off, idx = port.build_ivf(a, C)
    assert np.array_equal(got.off, off) and np.array_equal(got.idx, idx)


def test_build_ivf_hand_case_and_errors(ctx):
    ix = sb.build_ivf(np.array([0, 1, 0, 1], np.uint32), 2, ctx)  # partition_test.cpp:190-205
    assert ix.off.tolist() == [0, 2, 4] and ix.idx.tolist() == [0, 2, 1, 3]
    assert sb.build_ivf(np.zeros(5, np.uint32), 3, ctx).off.tolist() == [0, 5, 5, 5]
    with pytest.raises(sb.InvalidArgument, match="build_ivf: bucket id 3 out of range"):
        sb.build_ivf(np.array([0, 3], np.uint32), 2, ctx)


# ------------------------------------------------------------------ routing
def test_device_exp_is_glibc_exact(ctx):
    lib = sb.lib()
    rs = np.random.RandomState(3)
    x = np.concatenate([rs.uniform(-40, 0, 400000), rs.uniform(-745, 0, 50000),
                        rs.uniform(-1e-3, 1e-3, 50000), [0.0, -0.0, -np.inf, -800.0, -708.5]])
    out = np.empty_like(x)
    sb._check(lib.saap_debug_exp(ctx.h, sb._p(x), sb._u64(x.size), sb._p(out)))
    want = np.array([math.exp(v) for v in x])
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("use_der", [1, 0])
@pytest.mark.parametrize("l", [1, 4, 8, 16])
def test_centroid_router_golden(ctx, g, use_der, l):
    r = sb.CentroidRouter(sb.Partition(g["cent"], ctx), bool(use_der))
    assert np.array_equal(r.select(g["qr"][:4], g["qd"][:4], l), g[f"sel_d{use_der}_l{l}"])


@pytest.mark.parametrize("G", [1, 4, 7])
@pytest.mark.parametrize("C,l", [(1024, 32), (1024, 1024), (4096, 256), (16384, 8), (3, 2)])
def test_centroid_router_random(ctx, port, G, C, l):
    rs = np.random.RandomState(G * C + l)
    cent = unit_rows(rs.randn(C, 128))
    q = bf16_round(rs.randn(G, 128) * 3)
    r = sb.CentroidRouter(sb.Partition(cent, ctx), True)
    assert np.array_equal(r.select(q, q, l), port.centroid_select(cent, q, l))


def test_router_edge_cases(ctx, g):
    r = sb.CentroidRouter(sb.Partition(g["cent"], ctx), True)
    assert r.select(g["qr"][:4], g["qd"][:4], 0).size == 0
    with pytest.raises(sb.InvalidArgument, match="CentroidRouter: l exceeds bucket count"):
        r.select(g["qr"][:4], g["qd"][:4], 17)
    # uniform scores pick {0, 1, 2} (qmodel_test.cpp:338-346 analogue)
    flat = sb.CentroidRouter(sb.Partition(np.tile(unit_rows(np.ones((1, 32))), (8, 1)), ctx), True)
    assert flat.select(g["qr"][:4], g["qd"][:4], 3).tolist() == [0, 1, 2]


def test_qmodel_router_golden(ctx, g):
    m = sb.QModel({k: g["qm_" + k] for k in sb.QMODEL_FIELDS}, ctx)
    r = sb.QModelRouter(m)
    for l in (1, 3, 8, 16):
        assert np.array_equal(r.select(g["qr"][:4], g["qd"][:4], l), g[f"qmsel_l{l}"])
        assert np.array_equal(sb.batched_bucket_select(m, g["qd"][:4], l), g[f"qmsel_l{l}"])
    with pytest.raises(sb.InvalidArgument, match="batched_bucket_select: l=0"):
        sb.batched_bucket_select(m, g["qd"][:4], 0)
    assert r.select(g["qr"][:4], g["qd"][:4], 0).size == 0


@pytest.mark.parametrize("G", [1, 4])
def test_qmodel_router_random_llama_shape(ctx, port, G):
    if not oracle.ref_available():
        pytest.skip("needs oracle/_ref for qmodel_init")
    R = oracle.ref()
    m = R.qmodel_init(128, 1024, 1024, 11)
    rs = np.random.RandomState(5)
    m["bn_run_mean"] = rs.randn(1, 1024) * 0.1
    m["bn_run_var"] = 1 + rs.rand(1, 1024)
    q = bf16_round(rs.randn(G, 128))
    model = sb.QModel(m, ctx)
    for l in (1, 32, 256):
        assert np.array_equal(sb.batched_bucket_select(model, q, l), port.qmodel_select(m, q, l))


# ------------------------------------------------------------------ stores
def test_store_build_with_device_derope_golden(ctx, g):
    part = sb.Partition(g["cent"], ctx)
    st = sb.build_context_store(g["K"], g["V"], 500000.0, part, 1)
    a, ix = st.read_index(0)
    assert np.array_equal(a, g["store_assign"])
    assert np.array_equal(ix.off, g["store_off"]) and np.array_equal(ix.idx, g["store_idx"])
    pos = np.arange(1, 65, dtype=np.uint64)
    assert np.array_equal(sb.rope_remove_block(g["K"][1:65], pos, 500000.0, ctx), g["derope"])


@pytest.mark.parametrize("hint", [2047, 100, 0, 5000])
def test_store_build_index_bit_exact(ctx, port, hint):
    case = make_case(d=128, n=6000, C=256, seed=3)
    a, off, idx = port_index(port, case, 256)
    st = sb.build_context_store(case["K"], case["V"], 5e5, sb.Partition(case["cent"], ctx), 1,
                                keys_deroped=case["Kd"], recent_hint=hint)
    ga, gix = st.read_index(0)
    assert np.array_equal(ga, a) and np.array_equal(gix.off, off) and np.array_equal(gix.idx, idx)


# ------------------------------------------------------------------ attention
def _check_sparse(res, want, tag=""):
    out, ks, mv, em = want
    assert max_rel_diff(res.output, out) <= TOL, tag
    assert (res.keys_scored, res.max_visited_bucket, res.empty_attention) == (ks, mv, em), tag


def test_sparse_attention_golden(ctx, g):
    part = sb.Partition(g["cent"], ctx)
    for hint in (2047, 64, 32):
        st = sb.build_context_store(g["K"], g["V"], 5e5, part, 1, keys_deroped=g["Kd"],
                                    recent_hint=hint)
        for use_der in (1, 0):
            router = sb.CentroidRouter(part, bool(use_der))
            for q0 in (0, 4):
                for ci, (probes, recent, bs) in enumerate(g["cfgs"].tolist()):
                    key = f"sp_d{use_der}_q{q0}_c{ci}"
                    cfg = sb.SparseAttnConfig(probes, bs, sb.DenseWindow(1, recent))
                    res = sb.sparse_attention(g["qr"][q0:q0 + 4], g["qd"][q0:q0 + 4], st, router, cfg)
                    ks, mv, em = g[key + "_stats"].tolist()
                    _check_sparse(res, (g[key + "_out"], ks, mv, bool(em)), f"{key} hint={hint}")


@pytest.mark.parametrize("hint,recent", [(2047, 2047), (2047, 500), (500, 2047), (0, 100),
                                         (3000, 0), (2047, 10**7)])
@pytest.mark.parametrize("probes", [0, 1, 16, 256])
def test_sparse_attention_window_layouts(ctx, port, hint, recent, probes):
    case = make_case(d=128, n=9000, C=256, seed=5)
    a, off, idx = port_index(port, case, 256)
    part = sb.Partition(case["cent"], ctx)
    st = sb.build_context_store(case["K"], case["V"], 5e5, part, 1, keys_deroped=case["Kd"],
                                recent_hint=hint)
    router = sb.CentroidRouter(part, True)
    q = case["qr"][:4]
    cfg = sb.SparseAttnConfig(probes, 128, sb.DenseWindow(1, recent))
    res = sb.sparse_attention(q, case["qd"][:4], st, router, cfg)
    sel = port.centroid_select(case["cent"], case["qd"][:4], probes) if probes else None
    want = port.sparse_attention(q, case["K"], case["V"], 1, off, idx, sel, probes, 128, recent)
    _check_sparse(res, want, f"hint={hint} recent={recent} probes={probes}")


@pytest.mark.parametrize("G", [1, 4, 5, 8, 13])
@pytest.mark.parametrize("d", [32, 64, 128])
def test_sparse_attention_group_sizes_and_dims(ctx, port, G, d):
    case = make_case(d=d, n=5000, C=64, n_q=G, seed=G + d, use_ref=False)
    a, off, idx = port_index(port, case, 64)
    part = sb.Partition(case["cent"], ctx)
    st = sb.build_context_store(case["K"], case["V"], 5e5, part, 1, keys_deroped=case["Kd"],
                                recent_hint=1000)
    router = sb.CentroidRouter(part, True)
    cfg = sb.SparseAttnConfig(8, 128, sb.DenseWindow(1, 1000))
    res = sb.sparse_attention(case["qr"], case["qd"], st, router, cfg)
    sel = port.centroid_select(case["cent"], case["qd"], 8)
    _check_sparse(res, port.sparse_attention(case["qr"], case["K"], case["V"], 1, off, idx, sel, 8,
                                             128, 1000))


def test_sparse_attention_qmodel_router(ctx, port):
    if not oracle.ref_available():
        pytest.skip("needs oracle/_ref for qmodel_init")
    case = make_case(d=128, n=6000, C=128, seed=9)
    a, off, idx = port_index(port, case, 128)
    m = oracle.ref().qmodel_init(128, 256, 128, 2)
    part = sb.Partition(case["cent"], ctx)
    st = sb.build_context_store(case["K"], case["V"], 5e5, part, 1, keys_deroped=case["Kd"])
    router = sb.QModelRouter(sb.QModel(m, ctx))
    cfg = sb.SparseAttnConfig(12, 128, sb.DenseWindow(1, 1500))
    res = sb.sparse_attention(case["qr"][:4], case["qd"][:4], st, router, cfg)
    sel = port.qmodel_select(m, case["qd"][:4], 12)
    _check_sparse(res, port.sparse_attention(case["qr"][:4], case["K"], case["V"], 1, off, idx, sel,
                                             12, 128, 1500))


def test_empty_attention(ctx, port):
    # sink 0, recent 0, and the routed bucket holds no keys -> zero rows + flag
    d, n = 32, 600
    rs = np.random.RandomState(1)
    e0 = np.zeros(d, np.float32)
    e0[0] = 1
    e1 = np.zeros(d, np.float32)
    e1[1] = 1
    keys = bf16_round(np.abs(rs.randn(n, d)) * 0.01 + e0 * 5)
    cent = np.stack([e0, e1])
    part = sb.Partition(cent, ctx)
    st = sb.build_context_store(keys, keys, 5e5, part, 0, keys_deroped=keys, recent_hint=0)
    q = np.tile(e1 * 3, (4, 1))
    res = sb.sparse_attention(q, q, st, sb.CentroidRouter(part, True),
                              sb.SparseAttnConfig(1, 128, sb.DenseWindow(0, 0)))
    assert res.keys_scored == 0 and res.empty_attention and not res.output.any()


def test_sparse_attention_errors(ctx, g):
    part = sb.Partition(g["cent"], ctx)
    st = sb.build_context_store(g["K"], g["V"], 5e5, part, 1, keys_deroped=g["Kd"])
    r = sb.CentroidRouter(part, True)
    q = g["qr"][:4]
    with pytest.raises(sb.InvalidArgument, match="sparse_attention: probes 17 exceed bucket count 16"):
        sb.sparse_attention(q, q, st, r, sb.SparseAttnConfig(17, 128, sb.DenseWindow(1, 64)))
    with pytest.raises(sb.InvalidArgument, match="block_size must be >= 1"):
        sb.sparse_attention(q, q, st, r, sb.SparseAttnConfig(4, 0, sb.DenseWindow(1, 64)))
    with pytest.raises(sb.InvalidArgument, match="window sinks 2 keys but the store indexes from id 1"):
        sb.sparse_attention(q, q, st, r, sb.SparseAttnConfig(4, 128, sb.DenseWindow(2, 64)))
    with pytest.raises(sb.InvalidArgument, match="no keys left to index"):
        sb.build_context_store(g["K"][:1], g["V"][:1], 5e5, part, 1)


@pytest.mark.parametrize("n", [1, 63, 64, 65, 5000, 40000])
@pytest.mark.parametrize("G", [1, 4, 9])
def test_full_attention(ctx, port, n, G):
    rs = np.random.RandomState(n + G)
    q = bf16_round(rs.randn(G, 128) * 2)
    K = bf16_round(rs.randn(n, 128))
    V = bf16_round(rs.randn(n, 128))
    assert max_rel_diff(sb.full_attention(q, K, V, ctx), port.full_attention(q, K, V)) <= TOL
    with pytest.raises(sb.InvalidArgument, match="full_attention: empty key set"):
        sb.full_attention(q, K[:0], V[:0], ctx)


def test_full_attention_golden(ctx, g):
    assert max_rel_diff(sb.full_attention(g["qr"][:4], g["K"], g["V"], ctx), g["full"]) <= TOL


def test_layer_batched_ragged_groups(ctx, port):
    ns = [3000, 7001, 4500, 9000, 2100, 6000]
    cases = [make_case(d=128, n=n, C=128, seed=i + 20, use_ref=False) for i, n in enumerate(ns)]
    parts = [sb.Partition(c["cent"], ctx) for c in cases]
    L = sb.Layer(ns, 128, 128, 1, 2047, ctx)
    L.build(parts, np.concatenate([c["K"] for c in cases]), np.concatenate([c["V"] for c in cases]),
            np.concatenate([c["Kd"] for c in cases]))
    routers = [sb.CentroidRouter(p, True) for p in parts]
    qr = np.stack([c["qr"][:4] for c in cases])
    qd = np.stack([c["qd"][:4] for c in cases])
    cfg = sb.SparseAttnConfig(16, 128, sb.DenseWindow(1, 2047))
    out, stats, sel = L.sparse_attention(routers, qr, qd, cfg, want_selected=True)
    for i, c in enumerate(cases):
        a, off, idx = port_index(port, c, 128)
        ps = port.centroid_select(c["cent"], c["qd"][:4], 16)
        assert np.array_equal(sel[i], ps)
        o, ks, mv, em = port.sparse_attention(c["qr"][:4], c["K"], c["V"], 1, off, idx, ps, 16, 128,
                                              2047)
        assert max_rel_diff(out[i], o) <= TOL
        assert (stats[i].keys_scored, stats[i].max_visited_bucket) == (ks, mv)
    full = L.full_attention(qr)
    for i, c in enumerate(cases):
        assert max_rel_diff(full[i], port.full_attention(c["qr"][:4], c["K"], c["V"])) <= TOL


@pytest.mark.slow
def test_long_context_128k(ctx, port):
    n, C = 131072, 1024
    case = make_case(d=128, n=n, C=C, seed=2, use_ref=False)
    a, off, idx = port_index(port, case, C)
    part = sb.Partition(case["cent"], ctx)
    st = sb.build_context_store(case["K"], case["V"], 5e5, part, 1, keys_deroped=case["Kd"])
    ga, gix = st.read_index(0)
    assert np.array_equal(ga, a) and np.array_equal(gix.idx, idx)
    router = sb.CentroidRouter(part, True)
    cfg = sb.SparseAttnConfig(32, 128, sb.DenseWindow(1, 2047))
    res = sb.sparse_attention(case["qr"][:4], case["qd"][:4], st, router, cfg)
    sel = port.centroid_select(case["cent"], case["qd"][:4], 32)
    want = port.sparse_attention(case["qr"][:4], case["K"], case["V"], 1, off, idx, sel, 32, 128,
                                 2047)
    _check_sparse(res, want)
    assert res.keys_scored < n // 5


# ------------------------------------------------------------------ key recall
@pytest.mark.parametrize("hint", [2047, 64, 5])
def test_coverage_golden(ctx, g, hint):
    part = sb.Partition(g["cent"], ctx)
    st = sb.build_context_store(g["K"], g["V"], 5e5, part, 1, keys_deroped=g["Kd"], recent_hint=hint)
    dense = sb.DenseWindow(1, 64)
    got = [sb.attention_mass_coverage(g["qr"][:4], st, s, dense) for s in ([3, 7, 11], [], list(range(16)))]
    assert np.allclose(got, g["cov"], rtol=1e-4, atol=1e-6)
    with pytest.raises(sb.InvalidArgument, match="coverage: bucket id out of range"):
        sb.attention_mass_coverage(g["qr"][:4], st, [16], dense)


@pytest.mark.parametrize("hint,recent", [(2047, 2047), (300, 2047), (2047, 100), (0, 10**6)])
def test_coverage_matches_oracle(ctx, port, hint, recent):
    case = make_case(d=128, n=7000, C=128, seed=11)
    a, off, idx = port_index(port, case, 128)
    part = sb.Partition(case["cent"], ctx)
    st = sb.build_context_store(case["K"], case["V"], 5e5, part, 1, keys_deroped=case["Kd"],
                                recent_hint=hint)
    sel = port.centroid_select(case["cent"], case["qd"][:4], 16)
    got = sb.attention_mass_coverage(case["qr"][:4], st, sel, sb.DenseWindow(1, recent))
    want = port.coverage(case["qr"][:4], case["K"], 1, a, 128, sel, recent)
    assert abs(got - want) <= 1e-4 * max(1.0, abs(want))


@pytest.mark.skipif(not oracle.ref_available(), reason="needs oracle/_ref")
def test_qmodel_forward_bit_exact(ctx):
    """qmodel_forward eval mode (qmodel.cpp:375-377): probabilities identical."""
    R = oracle.ref()
    m = R.qmodel_init(64, 256, 96, 3)
    rs = np.random.RandomState(8)
    m["bn_run_mean"] = rs.randn(1, 256) * 0.1
    m["bn_run_var"] = 1 + rs.rand(1, 256)
    q = rs.randn(7, 64).astype(np.float32)
    q[2, :10] = 0.0
    got = sb.qmodel_forward(sb.QModel(m, ctx), q)
    want = R.qmodel_forward(m, q)
    assert np.array_equal(got.view(np.uint32), np.asarray(want, np.float32).view(np.uint32))
