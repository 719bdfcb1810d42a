"""Generate tests/golden/*.npz from the *reference itself* (oracle/_ref,
the unmodified /root/reference sources compiled by oracle/Makefile).

Run in the dev container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures pin oracle/saap_oracle.c (tests/test_oracle.py) on machines
without the reference, and give the GPU tests reference outputs that do not
depend on any CPU code at run time.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import bf16_round, small_spec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def small_case(R):
    """attention_test.cpp fixture shape: d=32, N=2048, C=16, 8 queries."""
    spec = small_spec()
    p = R.generate_prompt(spec, 2048, 8)
    cent = R.train_head_partition(spec, 2048, 16, 4, 1)
    K = bf16_round(p["keys_roped"])
    V = bf16_round(p["values"])
    Kd = bf16_round(p["keys_deroped"])
    qr = bf16_round(p["q_roped"])
    qd = bf16_round(p["q_deroped"])
    a = R.assign_keys(Kd[1:], cent)
    off, idx = R.build_ivf(a, 16)
    g = {"K": K, "V": V, "Kd": Kd, "qr": qr, "qd": qd, "cent": cent, "assign": a,
         "off": off, "idx": idx}
    st = R.store(K, V, cent, 1, a)
    cfgs = [(8, 64, 128), (16, 64, 128), (0, 64, 128), (4, 32, 7), (2, 4096, 128), (8, 64, 1),
            (16, 0, 128), (3, 1000, 128)]
    g["cfgs"] = np.array(cfgs, np.uint64)
    for use_der in (1, 0):
        rt = R.centroid_router(cent, bool(use_der))
        for q0 in (0, 4):
            for ci, (probes, recent, bs) in enumerate(cfgs):
                o, ks, mv, em = st.sparse_attention(rt, qr[q0:q0 + 4], qd[q0:q0 + 4], probes, bs,
                                                    recent=recent)
                key = f"sp_d{use_der}_q{q0}_c{ci}"
                g[key + "_out"] = o
                g[key + "_stats"] = np.array([ks, mv, int(em)], np.uint64)
                g[key + "_sel"] = rt.select(qr[q0:q0 + 4], qd[q0:q0 + 4], probes) if probes else \
                    np.zeros(0, np.uint32)
        for l in (1, 4, 8, 16):
            g[f"sel_d{use_der}_l{l}"] = R.centroid_select(cent, qr[:4], qd[:4], l, bool(use_der))
    g["full"] = R.full_attention(qr[:4], K, V)
    g["cov"] = np.array([st.coverage(qr[:4], [3, 7, 11], 64), st.coverage(qr[:4], [], 64),
                         st.coverage(qr[:4], list(range(16)), 64)])
    pos = np.arange(1, 2048, dtype=np.uint64)
    g["derope"] = R.rope_remove_block(K[1:65], pos[:64], spec.rope_base)
    a2, off2, idx2 = R.build_context_store(K, V, spec.rope_base, cent, 1)
    g["store_assign"], g["store_off"], g["store_idx"] = a2, off2, idx2
    # Q-model router with perturbed BN running stats
    m = R.qmodel_init(32, 64, 16, 3)
    rs = np.random.RandomState(0)
    m["bn_run_mean"] = rs.randn(1, 64) * 0.1
    m["bn_run_var"] = 1 + rs.rand(1, 64)
    m["b1"] = rs.randn(1, 64) * 0.05
    m["b2"] = rs.randn(1, 16) * 0.05
    for k, v in m.items():
        g["qm_" + k] = v
    for l in (1, 3, 8, 16):
        g[f"qmsel_l{l}"] = R.qmodel_select(m, qd[:4], l)
    g["qm_probs"] = R.qmodel_forward(m, qd[:4])
    return g


def main():
    R = oracle.ref()
    g = small_case(R)
    np.savez_compressed(os.path.join(OUT, "saap_small.npz"), **g)
    print("wrote", os.path.join(OUT, "saap_small.npz"), len(g), "arrays")


if __name__ == "__main__":
    main()
