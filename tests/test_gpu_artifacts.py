"""Reference-written artifacts (tests/golden/artifacts, written by the
reference's own tensor_write / u64_write / qmodel_save) drive the device
path: a loaded partition assigns and indexes keys exactly like the
reference's recorded IVF, a loaded Q-model routes like the reference."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")
A = os.path.join(G, "artifacts")


def test_loaded_partition_rebuilds_the_reference_ivf(ctx):
    import paper_2502_08246_b200 as sb
    E = np.load(os.path.join(G, "artifacts_expect.npz"))
    p = sb.partition_load(os.path.join(A, "partition.tensor"), ctx)
    a = sb.assign_keys(E["keys"], p)
    ix = sb.build_ivf(a, p.n_buckets(), ctx)
    ref = sb.ivf_load(os.path.join(A, "off.tensor"), os.path.join(A, "idx.tensor"))
    assert np.array_equal(ix.off, ref.off) and np.array_equal(ix.idx, ref.idx)


def test_loaded_qmodel_routes_like_the_reference(ctx):
    import paper_2502_08246_b200 as sb
    m = sb.qmodel_load(os.path.join(A, "qmodel"), ctx)
    params = sb.qmodel_read(os.path.join(A, "qmodel"))
    q = np.random.default_rng(5).normal(0, 1, (4, 16)).astype(np.float32)
    got = sb.batched_bucket_select(m, q, 5)
    want = oracle.port().qmodel_select(params, q, 5)
    assert np.array_equal(got, want)
