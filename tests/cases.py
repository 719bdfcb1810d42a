"""Seeded inputs for the parity tests.  Uses the reference's own generator
(synthdata.cpp via oracle/_ref) when it is built, else a clustered numpy
generator; every tensor is bf16-rounded (the parity contract)."""
import numpy as np

import oracle
from oracle import HeadSpec, bf16_round


def unit_rows(x):
    x = np.asarray(x, np.float64)
    return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)


def make_case(d=128, n=8192, C=256, n_q=8, seed=1, drift=0.0, use_ref=True, sink=1):
    rs = np.random.RandomState(seed)
    if use_ref and oracle.ref_available() and n >= 600:
        R = oracle.ref()
        spec = HeadSpec(dim=d, seed=seed, drift_rate=drift,
                        lowfreq_pairs=4 if d == 32 else 8,
                        longrange_threshold=min(1024, n // 4),
                        window_guard=min(2112, n // 3),
                        local_range=16 if d == 32 else 64)
        p = R.generate_prompt(spec, n, n_q, 0)
        K, V, Kd = bf16_round(p["keys_roped"]), bf16_round(p["values"]), bf16_round(p["keys_deroped"])
        qr, qd = bf16_round(p["q_roped"]), bf16_round(p["q_deroped"])
        sub = Kd[sink:][rs.choice(n - sink, min(n - sink, max(2 * C, 2048)), replace=False)]
        cent = R.kmeans_train(sub, C, 3, seed)
    else:
        centers = unit_rows(rs.randn(max(C // 2, 1), d))
        lab = rs.randint(0, centers.shape[0], n)
        Kd = bf16_round(centers[lab] * 4 + rs.randn(n, d))
        K = Kd.copy()
        V = bf16_round(rs.randn(n, d))
        tq = rs.randint(0, centers.shape[0], n_q)
        qd = bf16_round(centers[tq] * 6 + rs.randn(n_q, d))
        qr = qd.copy()
        cent = unit_rows(Kd[rs.choice(n, C, replace=False)] + 0.01 * rs.randn(C, d))
    return dict(K=K, V=V, Kd=Kd, qr=qr, qd=qd, cent=np.ascontiguousarray(cent, np.float32))


def port_index(port, case, C, sink=1):
    a = port.assign_keys(case["Kd"][sink:], case["cent"])
    off, idx = port.build_ivf(a, C)
    return a, off, idx
