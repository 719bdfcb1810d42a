"""Device Q-model training step timing at QTrainOptions' shape
(experiments.hpp:46-53: hidden 1024, batch 64; d=128, C=1024) against the
reference's train_step_on_target on the host (oracle/_ref, one thread, the
reference as written).  Wall time per step through the public API (host
batch + target in, loss out).  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (reference timing only)
import paper_2502_08246_b200 as sb  # noqa: E402


def main(d=128, h=1024, C=1024, n=64, steps=200, ref_steps=3):
    ctx = sb.default_context()
    R = oracle.ref()
    init = R.qmodel_init(d, h, C, 7)
    r = np.random.default_rng(0)
    qd = r.normal(0, 1, (steps, n, d)).astype(np.float32)
    t = r.random((steps, n, C))
    t /= t.sum(axis=2, keepdims=True)
    tr = sb.QModelTrainer(init, sb.TrainerState(lr=1e-3), ctx)
    for k in range(5):
        tr.train_step_on_target(qd[k], t[k])
    t0 = time.perf_counter()
    for k in range(steps):
        tr.train_step_on_target(qd[k], t[k])
    gpu_ms = (time.perf_counter() - t0) / steps * 1e3
    t0 = time.perf_counter()
    R.qtrain_steps(init, 1e-3, qd[:ref_steps], t[:ref_steps])
    cpu_ms = (time.perf_counter() - t0) / ref_steps * 1e3
    print(json.dumps({"shape": {"d": d, "hidden": h, "C": C, "batch": n},
                      "device_ms_per_step": round(gpu_ms, 3),
                      "reference_cpu_ms_per_step": round(cpu_ms, 1), "cpu_threads": 1,
                      "speedup": round(cpu_ms / gpu_ms, 1),
                      "qtrain_1200_steps_s": round(gpu_ms * 1.2, 2)}))


if __name__ == "__main__":
    main()
