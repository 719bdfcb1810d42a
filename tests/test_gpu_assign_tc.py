"""tcgen05 assignment path (bf16 device keys, two-term centroid split, fp64
re-check of near ties) is bit-exact with the reference's assign_keys, and
the packed layout built from it matches the oracle's IVF."""
import numpy as np
import pytest

import paper_2502_08246_b200 as sb
from oracle import bf16_round
from tests.cases import make_case, unit_rows

pytestmark = pytest.mark.gpu


def _dev_bf16(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)


def _build(ctx, parts, K, V, ns, C, sink=1, hint=2047, mode=0):
    ctx.set_assign_mode(mode)
    L = sb.Layer(ns, 128, C, sink, hint, ctx)
    kd, vd = _dev_bf16(K), _dev_bf16(V)
    L.build_dev(parts, kd, vd, kd)
    ctx.synchronize()
    ctx.set_assign_mode(0)
    return L


@pytest.mark.parametrize("C", [1024, 100, 1000, 128, 16384])
def test_tc_assignment_bit_exact(ctx, port, C):
    case = make_case(d=128, n=20001, C=C if C <= 4096 else 1024, seed=C, use_ref=False)
    if C > 4096:
        case["cent"] = unit_rows(np.random.RandomState(0).randn(C, 128))
    part = sb.Partition(case["cent"], ctx)
    L = _build(ctx, [part], case["K"], case["V"], [20001], C)
    used, refined = L.assign_info()
    assert used
    a, ix = L.read_index(0)
    want = port.assign_keys(case["K"][1:], case["cent"])
    assert np.array_equal(a, want)
    off, idx = port.build_ivf(want, C)
    assert np.array_equal(ix.off, off) and np.array_equal(ix.idx, idx)
    assert refined < 0.2 * 20000


def test_tc_assignment_adversarial_ties(ctx, port):
    rs = np.random.RandomState(1)
    C = 256
    cent = unit_rows(rs.randn(C, 128))
    cent[7] = cent[3]                     # duplicate centroid: exact ties
    cent[9] = bf16_round(cent[9])         # bf16-exact centroid
    n = 4097
    K = bf16_round(rs.randn(n, 128) * 3)
    K[1] = 0.0                            # zero key -> bucket 0
    K[2] = bf16_round(cent[3] * 5)        # tie between 3 and 7 -> 3
    mid = unit_rows((cent[10] + cent[11])[None])[0]
    K[3] = bf16_round(mid * 4)            # near-equidistant pair
    K[4] = bf16_round(cent[9] * 1e4)      # large norm
    K[5] = bf16_round(cent[9] * 1e-4)     # tiny norm
    part = sb.Partition(cent, ctx)
    L = _build(ctx, [part], K, K, [n], C)
    a, _ = L.read_index(0)
    want = port.assign_keys(K[1:], cent)
    assert np.array_equal(a, want)
    assert a[0] == 0 and a[1] == 3


def test_tc_matches_exact_mode_multi_partition(ctx, port):
    ns = [5000, 9000, 3001, 7000]
    cases = [make_case(d=128, n=n, C=512, seed=30 + i, use_ref=False) for i, n in enumerate(ns)]
    parts = [sb.Partition(c["cent"], ctx) for c in cases]
    K = np.concatenate([c["K"] for c in cases])
    V = np.concatenate([c["V"] for c in cases])
    Lt = _build(ctx, parts, K, V, ns, 512, mode=0)
    Le = _build(ctx, parts, K, V, ns, 512, mode=1)
    assert Lt.assign_info()[0] and not Le.assign_info()[0]
    for g, c in enumerate(cases):
        at, it = Lt.read_index(g)
        ae, ie = Le.read_index(g)
        want = port.assign_keys(c["K"][1:], c["cent"])
        assert np.array_equal(at, want) and np.array_equal(ae, want)
        assert np.array_equal(it.idx, ie.idx)


@pytest.mark.parametrize("C", [1024, 100, 16384])
def test_tc_assignment_f32_keys_bit_exact(ctx, port, C):
    """Host f32 builds (build_context_store's keys are not bf16-representable
    after de-RoPE) on the tensor cores: keys split into two bf16 terms, the
    bound widened for the split, ambiguous keys re-scored from the f32 rows --
    assignments equal the reference's assign_keys on the f32 keys, and equal
    the fp64 kernel's."""
    rs = np.random.RandomState(C + 7)
    n = 12001
    cent = unit_rows(rs.randn(C, 128))
    K = (rs.randn(n, 128) * 2).astype(np.float32)       # f32 keys (not bf16-exact)
    K[5] = 0.0
    K[6] = cent[min(3, C - 1)] * np.float32(3.0)          # on a centroid
    V = rs.randn(n, 128).astype(np.float32)
    part = sb.Partition(cent, ctx)
    outs = []
    for tc in (1, 0):
        ctx.set_option("assign_f32_tc", tc)
        try:
            L = sb.Layer([n], 128, C, 1, 2047, ctx)
            L.build([part], K, V, K)
            ctx.synchronize()
            used, refined = L.assign_info()
            assert used == bool(tc)
            outs.append(L.read_index(0)[0])
        finally:
            ctx.set_option("assign_f32_tc", 1)
    want = port.assign_keys(K[1:], cent)
    assert np.array_equal(outs[0], want)
    assert np.array_equal(outs[1], want)
