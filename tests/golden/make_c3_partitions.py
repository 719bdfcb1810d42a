"""Reference-trained partitions for the C3 benchmark inputs.

train_head_partition(spec, 131072, 1024, 10, 1) (experiments.cpp:284-295)
for the 8 KV heads of layer 0: HeadSpec defaults with dim=128, drift_rate=0,
seed = 1 + 8*layer + kv_head.  Run by the compiled reference (oracle/_ref),
one process per head (~5 min each, single-threaded k-means).  bench.py's
reference arm routes with these centroids; its GPU arm re-trains them with
the device k-means and checks the result is bit-identical.

    python tests/golden/make_c3_partitions.py [--drift 0.0] [--out FILE]
"""
import argparse
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

N_KEYS, C, ITERS, SINK, KV_HEADS = 131072, 1024, 10, 1, 8


def train(args):
    h, drift = args
    import oracle
    spec = oracle.HeadSpec(dim=128, seed=1 + h, drift_rate=drift)
    return oracle.ref().train_head_partition(spec, N_KEYS, C, ITERS, SINK)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--drift", type=float, default=0.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c3_partitions_drift0.npz"))
    a = ap.parse_args()
    with ProcessPoolExecutor(KV_HEADS) as ex:
        cents = list(ex.map(train, [(h, a.drift) for h in range(KV_HEADS)]))
    np.savez_compressed(a.out, centroids=np.stack(cents).astype(np.float32),
                        seeds=np.arange(1, KV_HEADS + 1, dtype=np.uint64),
                        meta=np.array([N_KEYS, C, ITERS, SINK], np.uint64),
                        drift=np.array([a.drift]))
    print("wrote", a.out, np.stack(cents).shape)


if __name__ == "__main__":
    main()
