"""The library's host generator (csrc/synthdata.cpp) against the compiled
reference's generate_prompt (synthdata.cpp:169-281): every output word of
every block bit-identical, for the parallel (counter-jumped) and sequential
passes, several HeadSpecs (drift, planting, small dims, local lookups), and
the reference's validation messages.  CPU-only: the generator is host code."""
import numpy as np
import pytest

import oracle
import paper_2502_08246_b200 as sb
from oracle import bf16_round

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")

BLOCKS = [("keys_deroped", "keys_deroped"), ("keys_roped", "keys_roped"), ("values", "values"),
          ("q_deroped", "queries_deroped"), ("q_roped", "queries_roped")]

SMALL = dict(lowfreq_pairs=4, n_clusters=4, n_targets=2, local_range=16, longrange_threshold=256,
             window_guard=300)


def _ref_spec(kw):
    keep = {k: v for k, v in kw.items() if k in oracle.HeadSpec.__dataclass_fields__}
    return oracle.HeadSpec(**keep)


@pytest.mark.parametrize("kw,n,nq,ps", [
    (dict(dim=128, seed=3, drift_rate=0.0), 5000, 4, 0),
    (dict(dim=128, seed=1, drift_rate=5e-4), 4200, 4, 7),
    (dict(dim=64, seed=2), 3000, 8, 2),
    (dict(dim=32, seed=5, **SMALL), 2000, 4, 1),
    (dict(dim=32, seed=9, planted_longrange_fraction=0.0, **SMALL), 1500, 16, 3),
])
@pytest.mark.parametrize("threads", [1, 8])
def test_generate_prompt_bit_exact(kw, n, nq, ps, threads):
    p = oracle.ref().generate_prompt(_ref_spec(kw), n, nq, ps)
    q = sb.generate_prompt(sb.HeadSpec(**kw), n, nq, ps, threads=threads)
    for a, b in BLOCKS:
        assert np.array_equal(p[a].view(np.uint32), getattr(q, b).view(np.uint32)), a


def test_generate_prompt_bf16_blocks():
    kw = dict(dim=64, seed=4, drift_rate=0.0)
    f = sb.generate_prompt(sb.HeadSpec(**kw), 3000, 4, 1)
    h = sb.generate_prompt(sb.HeadSpec(**kw), 3000, 4, 1, bf16=True)
    for k in ("keys_deroped", "keys_roped", "values"):
        want = bf16_round(getattr(f, k)).view(np.uint32) >> 16
        assert np.array_equal(getattr(h, k).astype(np.uint32), want), k
    assert np.array_equal(f.queries_roped, h.queries_roped)


def test_generate_prompt_128k_keys():
    """The C3 context length: parallel pass equals the reference end to end."""
    kw = dict(dim=128, seed=2, drift_rate=0.0)
    p = oracle.ref().generate_prompt(_ref_spec(kw), 131072, 4, 5)
    q = sb.generate_prompt(sb.HeadSpec(**kw), 131072, 4, 5, threads=8)
    for a, b in BLOCKS:
        assert np.array_equal(p[a].view(np.uint32), getattr(q, b).view(np.uint32)), a


@pytest.mark.parametrize("kw,n,nq,msg", [
    (dict(dim=7), 3000, 4, "HeadSpec: dim must be even and >= 8"),
    (dict(dim=64, lowfreq_pairs=17), 3000, 4, r"HeadSpec: lowfreq_pairs must be in \[1, dim/4\]"),
    (dict(dim=64, n_clusters=20), 3000, 4, "HeadSpec: stable pairs cannot hold 20 cluster codes"),
    (dict(dim=64), 3000, 0, "generate_prompt: need at least one query"),
    (dict(dim=64), 60, 4, "generate_prompt: context of 60 keys cannot host 4 queries"),
    (dict(dim=64), 2116, 4, "generate_prompt: context too short to plant 4 long-range targets"),
])
def test_generate_prompt_errors(kw, n, nq, msg):
    with pytest.raises(sb.InvalidArgument, match=msg):
        sb.generate_prompt(sb.HeadSpec(**kw), n, nq, 0)
    if set(kw) <= set(oracle.HeadSpec.__dataclass_fields__):
        with pytest.raises(oracle.RefError, match=msg):
            oracle.ref().generate_prompt(_ref_spec(kw), n, nq, 0)
