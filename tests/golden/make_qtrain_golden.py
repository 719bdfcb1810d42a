"""Golden Q-model training fixture from the *reference itself* (oracle/_ref):
qmodel_init -> attention_target_rows -> 4 x train_step_on_target
(qmodel.cpp:227-433).  python tests/golden/make_qtrain_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "qtrain_small.npz")


def main():
    R = oracle.ref()
    r = np.random.default_rng(11)
    d, h, C, n, K, N = 16, 48, 12, 24, 4, 300
    init = R.qmodel_init(d, h, C, 5)
    keys = r.normal(0, 1, (N, d)).astype(np.float32)
    assign = r.integers(0, C, N).astype(np.uint32)
    q_roped = r.normal(0, 1, (K * n, d)).astype(np.float32)
    tgt = R.attention_target(q_roped, keys, assign, C)
    qd = r.normal(0, 1, (K, n, d)).astype(np.float32)
    qd[0, 3, :5] = 0.0  # zero inputs exercise the mm zero skip
    params, losses = R.qtrain_steps(init, 1e-3, qd, tgt.reshape(K, n, C))
    rec = {f"init_{k}": v for k, v in init.items()}
    rec.update({f"out_{k}": v for k, v in params.items()})
    np.savez_compressed(OUT, keys=keys, assign=assign, q_roped=q_roped, target=tgt, qd=qd,
                        losses=losses, lr=np.array(1e-3), **rec)
    print("wrote", OUT, os.path.getsize(OUT), "losses", losses)


if __name__ == "__main__":
    main()
