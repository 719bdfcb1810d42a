"""Device k-means (kmeans.cu) vs the reference's kmeans_train
(partition.cpp:52-179): centroids, per-iteration objective and KMeansStats
bit-exact, on the golden fixtures (tests/golden/make_kmeans_golden.py) and,
where oracle/_ref travelled with the repo, on larger live cases."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

KM_GOLD = os.path.join(os.path.dirname(__file__), "golden", "kmeans_small.npz")
_G = np.load(KM_GOLD)
NAMES = [str(n) for n in _G["names"]]


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("name", NAMES)
def test_kmeans_matches_reference_golden(ctx, name):
    import paper_2502_08246_b200 as sb
    C, iters, seed = (int(x) for x in _G[f"{name}_cfg"])
    rng = sb.Rng(seed)
    st = sb.KMeansStats()
    p = sb.kmeans_train(_G[f"{name}_keys"], C, iters, rng, st, ctx=ctx)
    want = _G[f"{name}_cent"]
    diff = np.flatnonzero(_bits(p.centroids) != _bits(want))
    assert diff.size == 0, f"{diff.size} centroid words differ, first {diff[:4]}"
    assert np.array_equal(_bits(np.array(st.objective_per_iter)), _bits(_G[f"{name}_obj"]))
    zk, rep, nxt = _G[f"{name}_stats"].tolist()
    assert (st.zero_vector_keys, st.empty_cluster_repairs) == (zk, rep)
    assert rng.next_u64() == nxt  # the caller's Rng advanced exactly as the reference's


def test_kmeans_partition_assigns_like_reference(ctx):
    """The trained partition drives assign_keys / build_ivf unchanged."""
    import paper_2502_08246_b200 as sb
    keys = _G["clustered_d128_keys"]
    C, iters, seed = (int(x) for x in _G["clustered_d128_cfg"])
    p = sb.kmeans_train(keys, C, iters, sb.Rng(seed), ctx=ctx)
    a = sb.assign_keys(keys, p)
    assert np.array_equal(a, oracle.port().assign_keys(keys, _G["clustered_d128_cent"]))


def test_kmeans_errors_match_reference(ctx):
    import paper_2502_08246_b200 as sb
    keys = np.zeros((3, 2), np.float32)
    with pytest.raises(sb.InvalidArgument, match="kmeans_train: 3 keys cannot seed 4 buckets"):
        sb.kmeans_train(keys, 4, 10, sb.Rng(14), ctx=ctx)
    with pytest.raises(sb.InvalidArgument, match="kmeans_train: need at least 1 bucket"):
        sb.kmeans_train(keys, 0, 10, sb.Rng(14), ctx=ctx)
    with pytest.raises(sb.InvalidArgument, match="kmeans_train: iters must be >= 1"):
        sb.kmeans_train(keys, 2, 0, sb.Rng(14), ctx=ctx)
    # the reference validates before drawing: the Rng must not advance
    r = sb.Rng(14)
    with pytest.raises(sb.InvalidArgument):
        sb.kmeans_train(keys, 4, 10, r, ctx=ctx)
    assert r.next_u64() == sb.Rng(14).next_u64()


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,d,C,iters,drift", [(16383, 128, 256, 3, 5e-4), (8191, 64, 128, 4, 0.0)])
def test_kmeans_live_reference_head_keys(ctx, n, d, C, iters, drift):
    """train_head_partition's input: de-roped synthetic head keys (non-sink),
    Rng(seed).child(2 << 32) (experiments.cpp:284-295)."""
    import paper_2502_08246_b200 as sb
    R = oracle.ref()
    spec = oracle.HeadSpec(dim=d, seed=3, drift_rate=drift)
    p = R.generate_prompt(spec, n + 1, 1, 1)
    keys = p["keys_deroped"][1:]
    cent, obj, zk, rep, nxt = R.kmeans_train_stats(keys, C, iters, 3, stream=2 << 32)
    rng = sb.Rng(3).child(2 << 32)
    st = sb.KMeansStats()
    got = sb.kmeans_train(keys, C, iters, rng, st, ctx=ctx)
    assert np.array_equal(_bits(got.centroids), _bits(cent))
    assert np.array_equal(_bits(np.array(st.objective_per_iter)), _bits(obj))
    assert (st.zero_vector_keys, st.empty_cluster_repairs) == (zk, rep)
    assert rng.next_u64() == nxt


@pytest.mark.parametrize("d", [2, 3, 16, 100])
def test_assign_keys_other_dims(ctx, d):
    """assign_keys for head dims outside the decode kernels' {32, 64, 128}
    (the reference's partition tests use d = 2..8): exact best_bucket."""
    import paper_2502_08246_b200 as sb
    r = np.random.default_rng(d)
    cent = r.normal(0, 1, (37, d)).astype(np.float32)
    cent /= np.linalg.norm(cent, axis=1, keepdims=True)
    keys = r.normal(0, 1, (5000, d)).astype(np.float32)
    keys[7] = 0.0
    keys[11] = cent[5] * 2  # exact positive scaling: its own bucket
    got = sb.assign_keys(keys, sb.Partition(cent, ctx))
    assert np.array_equal(got, oracle.port().assign_keys(keys, cent))
    assert got[7] == 0 and got[11] == 5


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_build_context_store_with_kmeans_training(ctx):
    """build_context_store(keys_roped, values, rope, C, iters, sink, rng, stats)
    (attention.cpp:238-246): device de-rope + device k-means + build equal the
    reference's centroids, objective, assignments and index bit-exactly."""
    import paper_2502_08246_b200 as sb
    R = oracle.ref()
    spec = oracle.HeadSpec(dim=64, seed=4, drift_rate=5e-4)
    p = R.generate_prompt(spec, 6000, 1, 2)
    cent, a, off, idx, obj = R.build_context_store_kmeans(p["keys_roped"], p["values"], 500000.0,
                                                          64, 4, 1, 17)
    st = sb.KMeansStats()
    store = sb.build_context_store_kmeans(p["keys_roped"], p["values"], 500000.0, 64, 4, 1,
                                          sb.Rng(17), st, ctx=ctx)
    assert np.array_equal(_bits(store.partition.centroids), _bits(cent))
    assert np.array_equal(_bits(np.array(st.objective_per_iter)), _bits(obj))
    ga, gix = store.read_index(0)
    assert np.array_equal(ga, a) and np.array_equal(gix.off, off) and np.array_equal(gix.idx, idx)
