"""Device Q-model training (qtrain.cu) vs the reference's
train_step_on_target / attention_target_rows (qmodel.cpp:227-433):
parameters and running statistics bit-identical after every step, targets
bit-identical, the reported loss within 1e-12 relative (CUDA log vs glibc)."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "qtrain_small.npz")
FIELDS = ("w1", "b1", "bn_gamma", "bn_beta", "bn_run_mean", "bn_run_var", "w2", "b2")


def _same(a, b):
    return np.array_equal(np.ascontiguousarray(a, np.float64).view(np.uint64),
                          np.ascontiguousarray(b, np.float64).view(np.uint64))


def test_qtrain_matches_golden(ctx):
    import paper_2502_08246_b200 as sb
    g = np.load(GOLD)
    K, n, d = g["qd"].shape
    C = g["target"].shape[1]
    tgt = sb.attention_target_rows(g["q_roped"], g["keys"], g["assign"], C, ctx)
    assert _same(tgt, g["target"])
    tr = sb.QModelTrainer({k: g[f"init_{k}"] for k in FIELDS}, sb.TrainerState(lr=float(g["lr"])), ctx)
    losses = [tr.train_step_on_target(g["qd"][k], tgt.reshape(K, n, C)[k]) for k in range(K)]
    np.testing.assert_allclose(losses, g["losses"], rtol=1e-12, atol=0)
    got = tr.params()
    for k in FIELDS:
        assert _same(got[k], g[f"out_{k}"]), k


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("d,h,C,n,K", [(128, 1024, 1024, 64, 3), (64, 256, 256, 64, 6)])
def test_qtrain_live_reference(ctx, d, h, C, n, K):
    """QTrainOptions' shape (hidden 1024, batch 64) at C = 1024."""
    import paper_2502_08246_b200 as sb
    R = oracle.ref()
    r = np.random.default_rng(d + C)
    init = R.qmodel_init(d, h, C, 7)
    keys = r.normal(0, 1, (2048, d)).astype(np.float32)
    assign = r.integers(0, C, 2048).astype(np.uint32)
    qr = (r.normal(0, 1, (K * n, d)) * 2).astype(np.float32)
    tgt_ref = R.attention_target(qr, keys, assign, C)
    tgt = sb.attention_target_rows(qr, keys, assign, C, ctx)
    assert _same(tgt, tgt_ref)
    qd = r.normal(0, 1, (K, n, d)).astype(np.float32)
    want, wl = R.qtrain_steps(init, 1e-3, qd, tgt_ref.reshape(K, n, C))
    tr = sb.QModelTrainer(init, sb.TrainerState(lr=1e-3), ctx)
    losses = [tr.train_step_on_target(qd[k], tgt.reshape(K, n, C)[k]) for k in range(K)]
    np.testing.assert_allclose(losses, wl, rtol=1e-12, atol=0)
    got = tr.params()
    for k in FIELDS:
        assert _same(got[k], want[k]), k
    # the trained model routes like the reference's batched_bucket_select
    m = tr.qmodel()
    for i in range(4):
        grp = qd[0, 4 * i:4 * i + 4]
        assert np.array_equal(sb.batched_bucket_select(m, grp, 16),
                              oracle.port().qmodel_select(want, grp, 16))


def test_qtrain_errors_and_nonfinite_loss(ctx):
    import paper_2502_08246_b200 as sb
    g = np.load(GOLD)
    init = {k: g[f"init_{k}"] for k in FIELDS}
    tr = sb.QModelTrainer(init, sb.TrainerState(lr=1e-3), ctx)
    C = g["target"].shape[1]
    with pytest.raises(sb.InvalidArgument, match="train-mode forward needs >= 2 rows"):
        tr.train_step_on_target(g["qd"][0][:1], g["target"][:1])
    with pytest.raises(sb.InvalidArgument, match="qmodel: query dim 8 does not match model dim 16"):
        tr.train_step_on_target(np.zeros((4, 8), np.float32), np.zeros((4, C)))
    bad = np.array(g["target"][:24])
    bad[0, 0] = np.inf
    with pytest.raises(sb.RuntimeFailure, match="train_step: non-finite loss at step 1"):
        tr.train_step_on_target(g["qd"][0], bad)
    # the failed step left the state untouched
    got = tr.params()
    for k in FIELDS:
        assert _same(got[k], init[k]), k
    with pytest.raises(sb.InvalidArgument, match="attention_target: bucket id out of range"):
        sb.attention_target_rows(g["q_roped"][:2], g["keys"][:3], [0, 1, C], C, ctx)
