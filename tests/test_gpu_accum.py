"""Partial-attention accumulators on the device (accum.cu) vs the
reference's PartialAccumulator operations (attention.cpp:34-203), driven in
lockstep: out_acc / sumexp / runmax bit-identical after every absorb and
merge, finalized outputs bit-identical.  The reference runs through
oracle/_ref (the unmodified sources)."""
import numpy as np
import pytest

import oracle
import paper_2502_08246_b200 as sb

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint64 if np.asarray(x).dtype == np.float64 else np.uint32)


def _same_state(acc, ref_state):
    got = acc.state()
    for a, b in zip(got, ref_state):
        assert np.array_equal(_bits(a), _bits(np.asarray(b, np.float64)))


def _fresh(H, dv):
    return np.zeros((H, dv)), np.zeros(H), np.full(H, -np.inf)


@pytest.mark.parametrize("H,d,dv,N", [(4, 64, 48, 500), (1, 128, 128, 3000), (7, 32, 20, 64)])
def test_absorb_merge_finalize_lockstep(ctx, H, d, dv, N):
    R = oracle.ref()
    r = np.random.default_rng(H * 1000 + d)
    q = (r.normal(0, 1, (H, d)) * 0.5).astype(np.float32)
    K = r.normal(0, 1, (N, d)).astype(np.float32)
    V = r.normal(0, 1, (N, dv)).astype(np.float32)
    acc = sb.PartialAccumulator(H, dv, ctx)
    st = _fresh(H, dv)
    _same_state(acc, st)
    ids = r.integers(0, N, 37)
    ids[3] = ids[5]  # duplicates are absorbed twice, like the reference
    sb.pattn_absorb(acc, q, K, V, ids)
    st = R.acc_absorb(st, q, K, V, ids=ids)
    _same_state(acc, st)
    sb.pattn_absorb_range(acc, q, K, V, N // 5, N // 2)
    st = R.acc_absorb(st, q, K, V, begin=N // 5, end=N // 2)
    _same_state(acc, st)
    sb.pattn_absorb(acc, q, K, V, [])  # no-op
    _same_state(acc, st)
    # a part from other rows, merged in; then an empty part (identity)
    part = sb.PartialAccumulator(H, dv, ctx)
    pst = _fresh(H, dv)
    pids = r.integers(0, N, 90)
    sb.pattn_absorb(part, q * 3, K, V, pids)  # larger scores: the part's max wins
    pst = R.acc_absorb(pst, q * 3, K, V, ids=pids)
    _same_state(part, pst)
    sb.merge_into(acc, part)
    st = R.acc_merge(st, pst)
    _same_state(acc, st)
    sb.merge_into(acc, sb.PartialAccumulator(H, dv, ctx))
    _same_state(acc, st)
    # merging into an empty accumulator copies
    e = sb.PartialAccumulator(H, dv, ctx)
    sb.merge_into(e, acc)
    _same_state(e, st)
    out, empty = sb.pattn_finalize(acc)
    want, wempty = R.acc_finalize(st)
    assert np.array_equal(_bits(out), _bits(want)) and empty == wempty == False


def test_merge_partials_and_attention_over_ids(ctx):
    R = oracle.ref()
    r = np.random.default_rng(9)
    H, d, dv, N = 4, 128, 128, 2000
    q = r.normal(0, 1, (H, d)).astype(np.float32) * 0.3
    K = r.normal(0, 1, (N, d)).astype(np.float32)
    V = r.normal(0, 1, (N, dv)).astype(np.float32)
    parts, states = [], []
    for k in range(3):
        p = sb.PartialAccumulator(H, dv, ctx)
        ids = r.integers(0, N, 100 + 50 * k)
        sb.pattn_absorb(p, q, K, V, ids)
        parts.append(p)
        states.append(R.acc_absorb(_fresh(H, dv), q, K, V, ids=ids))
    merged = sb.merge_partials(parts)
    st = states[0]
    for s2 in states[1:]:
        st = R.acc_merge(st, s2)
    _same_state(merged, st)
    ids = r.integers(0, N, 333)
    out, empty = sb.attention_over_ids(q, K, V, ids, ctx)
    want, wempty = R.acc_finalize(R.acc_absorb(_fresh(H, dv), q, K, V, ids=ids))
    assert np.array_equal(_bits(out), _bits(want)) and not empty
    # nothing absorbed: zero rows and the empty flag (attention.cpp:147-152)
    out, empty = sb.attention_over_ids(q, K, V, [], ctx)
    assert empty and not out.any()


def test_accumulator_errors(ctx):
    q = np.zeros((4, 8), np.float32)
    K = np.zeros((10, 8), np.float32)
    V = np.zeros((10, 6), np.float32)
    acc = sb.PartialAccumulator(4, 6, ctx)
    with pytest.raises(sb.InvalidArgument, match="pattn_absorb: key id 10 out of range"):
        sb.pattn_absorb(acc, q, K, V, [1, 10])
    with pytest.raises(sb.InvalidArgument, match=r"pattn_absorb_range: bad range \[3, 11\)"):
        sb.pattn_absorb_range(acc, q, K, V, 3, 11)
    with pytest.raises(sb.InvalidArgument, match="attention: 10 keys vs 9 values"):
        sb.pattn_absorb(acc, q, K, V[:9], [1])
    with pytest.raises(sb.InvalidArgument, match="pattn_absorb: accumulator 4x6 does not fit group 2x6"):
        sb.pattn_absorb(acc, q[:2], K, V, [1])
    with pytest.raises(sb.InvalidArgument, match="merge_into: accumulator shapes differ"):
        sb.merge_into(acc, sb.PartialAccumulator(4, 5, ctx))
    with pytest.raises(sb.InvalidArgument, match="merge_partials: empty list"):
        sb.merge_partials([])
    st = acc.state()  # failed calls left the state untouched
    assert not st[0].any() and not st[1].any() and np.isneginf(st[2]).all()
