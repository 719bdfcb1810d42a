"""Pin the C restatement (oracle/saap_oracle.c) against the reference:
golden vectors produced by the compiled reference (tests/golden), and the
live reference (oracle/_ref) on random cases when it is built."""
import os

import numpy as np
import pytest

import oracle
from oracle import bf16_round

GOLD = os.path.join(os.path.dirname(__file__), "golden", "saap_small.npz")


@pytest.fixture(scope="module")
def g():
    return dict(np.load(GOLD))


def test_assign_and_ivf_match_golden(port, g):
    a = port.assign_keys(g["Kd"][1:], g["cent"])
    assert np.array_equal(a, g["assign"])
    off, idx = port.build_ivf(a, 16)
    assert np.array_equal(off, g["off"]) and np.array_equal(idx, g["idx"])


def test_store_build_with_derope_matches_golden(port, g):
    pos = np.arange(1, g["K"].shape[0], dtype=np.uint64)
    der = port.rope_remove(g["K"][1:], pos, 500000.0)
    assert np.array_equal(der[:64], g["derope"])
    a = port.assign_keys(der, g["cent"])
    assert np.array_equal(a, g["store_assign"])
    off, idx = port.build_ivf(a, 16)
    assert np.array_equal(off, g["store_off"]) and np.array_equal(idx, g["store_idx"])


@pytest.mark.parametrize("use_der", [1, 0])
@pytest.mark.parametrize("l", [1, 4, 8, 16])
def test_centroid_select_matches_golden(port, g, use_der, l):
    q = g["qd"][:4] if use_der else g["qr"][:4]
    assert np.array_equal(port.centroid_select(g["cent"], q, l), g[f"sel_d{use_der}_l{l}"])


def test_sparse_attention_matches_golden_bitwise(port, g):
    for use_der in (1, 0):
        for q0 in (0, 4):
            for ci, (probes, recent, bs) in enumerate(g["cfgs"].tolist()):
                key = f"sp_d{use_der}_q{q0}_c{ci}"
                sel = g[key + "_sel"]
                out, ks, mv, em = port.sparse_attention(g["qr"][q0:q0 + 4], g["K"], g["V"], 1,
                                                        g["off"], g["idx"], sel, probes, bs, recent)
                assert np.array_equal(out, g[key + "_out"]), key
                assert [ks, mv, int(em)] == g[key + "_stats"].tolist(), key


def test_full_attention_and_coverage_match_golden(port, g):
    assert np.array_equal(port.full_attention(g["qr"][:4], g["K"], g["V"]), g["full"])
    cov = [port.coverage(g["qr"][:4], g["K"], 1, g["assign"], 16, s, 64)
           for s in ([3, 7, 11], [], list(range(16)))]
    assert np.array_equal(np.array(cov), g["cov"])


def test_qmodel_select_matches_golden(port, g):
    m = {k: g["qm_" + k] for k in oracle.QMODEL_FIELDS}
    for l in (1, 3, 8, 16):
        assert np.array_equal(port.qmodel_select(m, g["qd"][:4], l), g[f"qmsel_l{l}"])


def test_oracle_error_paths(port, g):
    with pytest.raises(ValueError):
        port.build_ivf(np.array([0, 3], np.uint32), 2)
    with pytest.raises(ValueError):
        port.centroid_select(g["cent"], g["qd"][:4], 17)
    with pytest.raises(ValueError):
        port.full_attention(g["qr"][:4], g["K"][:0], g["V"][:0])


def test_build_ivf_hand_case(port):
    # partition_test.cpp:190-205
    off, idx = port.build_ivf(np.array([0, 1, 0, 1], np.uint32), 2)
    assert off.tolist() == [0, 2, 4] and idx.tolist() == [0, 2, 1, 3]
    off, _ = port.build_ivf(np.zeros(5, np.uint32), 3)
    assert off.tolist() == [0, 5, 5, 5]


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_port_equals_live_reference_random():
    R, P = oracle.ref(), oracle.port()
    rs = np.random.RandomState(7)
    for d, n, C in ((32, 700, 8), (64, 900, 32), (128, 600, 64)):
        cent = rs.randn(C, d).astype(np.float32)
        cent /= np.linalg.norm(cent, axis=1, keepdims=True)
        keys = bf16_round(rs.randn(n, d) * 2)
        keys[5] = 0  # zero key -> bucket 0
        cent[3] = cent[1]  # exact tie -> lowest id
        keys[6] = cent[1] * 2
        a = R.assign_keys(keys, cent)
        assert np.array_equal(a, P.assign_keys(keys, cent))
        V = bf16_round(rs.randn(n, d))
        off, idx = R.build_ivf(a[1:], C)
        st = R.store(keys, V, cent, 1, a[1:])
        rt = R.centroid_router(cent, True)
        q = bf16_round(rs.randn(4, d) * 3)
        for probes, recent in ((C // 4, 100), (C, 30), (0, 50), (3, 10**6)):
            sel = rt.select(q, q, probes) if probes else np.zeros(0, np.uint32)
            o1 = st.sparse_attention(rt, q, q, probes, 128, recent=recent)
            o2 = P.sparse_attention(q, keys, V, 1, off, idx, sel, probes, 128, recent)
            assert np.array_equal(o1[0], o2[0]) and o1[1:] == o2[1:]


# ---------------------------------------------------------------- k-means host side
KM_GOLD = os.path.join(os.path.dirname(__file__), "golden", "kmeans_small.npz")


def test_rng_port_draws_reference_seed_rows():
    """The host Rng mirror (paper_2502_08246_b200.Rng) draws exactly the seed
    rows the reference's kmeans_train draws (tensor.cpp:90-168)."""
    import paper_2502_08246_b200 as sb
    g = np.load(KM_GOLD)
    for name in g["names"]:
        C, _, seed = (int(x) for x in g[f"{name}_cfg"])
        n = g[f"{name}_keys"].shape[0]
        rng = sb.Rng(seed)
        s = rng.sample_without_replacement(n, C)
        rng.shuffle(s)
        assert s == g[f"{name}_seeds"].tolist(), name


def test_rng_port_child_and_below():
    import paper_2502_08246_b200 as sb
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    R = oracle.ref()
    for seed, n, m in [(1, 10, 10), (99, 1 << 20, 7), (2 ** 63 + 5, 1000, 999)]:
        rng = sb.Rng(seed)
        s = rng.sample_without_replacement(n, m)
        rng.shuffle(s)
        assert s == R.kmeans_seed_rows(seed, n, m).tolist()
    # train_head_partition's stream: Rng(seed).child(2 << 32)
    keys = np.random.default_rng(0).normal(0, 1, (64, 8)).astype(np.float32)
    _, _, _, _, nxt = R.kmeans_train_stats(keys, 4, 1, 5, stream=2 << 32)
    rng = sb.Rng(5).child(2 << 32)
    s = rng.sample_without_replacement(64, 4)
    rng.shuffle(s)
    assert rng.next_u64() == nxt


def test_kmeans_golden_matches_live_reference():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    R = oracle.ref()
    g = np.load(KM_GOLD)
    for name in g["names"]:
        C, iters, seed = (int(x) for x in g[f"{name}_cfg"])
        cent, obj, zk, rep, nxt = R.kmeans_train_stats(g[f"{name}_keys"], C, iters, seed)
        assert np.array_equal(cent.view(np.uint32), g[f"{name}_cent"].view(np.uint32)), name
        assert np.array_equal(obj.view(np.uint64), g[f"{name}_obj"].view(np.uint64)), name
        assert [zk, rep, nxt] == g[f"{name}_stats"].tolist(), name


def test_kmeans_validation_before_any_device_work():
    """kmeans_train's argument checks (partition.cpp:54-66) fire in the host
    mirror before the Rng draws or the device is touched."""
    import paper_2502_08246_b200 as sb
    keys = np.zeros((3, 2), np.float32)
    r = sb.Rng(14)
    with pytest.raises(sb.InvalidArgument, match="kmeans_train: 3 keys cannot seed 4 buckets"):
        sb.kmeans_train(keys, 4, 10, r)
    with pytest.raises(sb.InvalidArgument, match="kmeans_train: need at least 1 bucket"):
        sb.kmeans_train(keys, 0, 10, r)
    with pytest.raises(sb.InvalidArgument, match="kmeans_train: iters must be >= 1"):
        sb.kmeans_train(keys, 2, 0, r)
    assert r.next_u64() == sb.Rng(14).next_u64()
