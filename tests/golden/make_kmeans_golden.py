"""Generate tests/golden/kmeans_small.npz from the *reference itself*
(oracle/_ref: the unmodified kmeans_train, partition.cpp:52-179).

Run in the dev container (where /root/reference exists):
    python tests/golden/make_kmeans_golden.py
Cases follow partition_test.cpp's k-means tests (one point per cluster,
antipodal clusters, random blocks, a zero key) plus duplicate-heavy inputs
that force empty-cluster repairs and head-dim clustered keys.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "kmeans_small.npz")


def cases():
    r = np.random.default_rng(2502)
    out = []
    k = np.zeros((4, 4), np.float32)
    k[0, 0], k[1, 1], k[2, 2], k[3, 3] = 2.0, 3.0, 1.5, 2.5
    out.append(("pinned", k, 4, 10, 11))
    a = r.normal(0, 0.05, 64)
    b = np.pi + r.normal(0, 0.05, 64)
    k = np.concatenate([np.stack([np.cos(a), np.sin(a)], 1),
                        np.stack([np.cos(b), np.sin(b)], 1)]).astype(np.float32)
    out.append(("antipodal", k, 2, 10, 12))
    for run in range(3):
        out.append((f"random{run}", r.normal(0, 1, (256, 8)).astype(np.float32), 16, 10, 13 + run))
    k = r.normal(0, 1, (32, 4)).astype(np.float32)
    k[5] = 0.0
    k[9] = -0.0
    out.append(("zero_key", k, 4, 5, 15))
    # 8 distinct directions, each repeated: seeds collide -> empty clusters
    base = r.normal(0, 1, (8, 16)).astype(np.float32)
    k = base[r.integers(0, 8, 96)]
    out.append(("duplicates", k, 12, 4, 21))
    k = np.repeat(r.normal(0, 1, (3, 8)).astype(np.float32), [1, 1, 30], axis=0)
    out.append(("repair_then_stuck", k, 6, 3, 22))
    k = r.normal(0, 1, (10, 4)).astype(np.float32)
    k[[1, 3, 4, 6, 8]] = 0.0
    k[7] = -0.0
    out.append(("zero_seeds", k, 5, 3, 26))
    k = np.array([[1, 0], [-1, 0], [0, 1], [0, -1], [2, 0], [-2, 0]], np.float32)
    out.append(("cancel", k, 1, 2, 27))
    cen = r.normal(0, 1, (24, 128))
    k = (cen[r.integers(0, 24, 1024)] * 3 + r.normal(0, 1, (1024, 128))).astype(np.float32)
    out.append(("clustered_d128", k, 32, 5, 23))
    k = r.normal(0, 1, (700, 64)).astype(np.float32)
    out.append(("random_d64", k, 40, 3, 24))
    k = r.normal(0, 1, (300, 3)).astype(np.float32)
    out.append(("odd_dim3", k, 7, 6, 25))
    return out


def main():
    R = oracle.ref()
    rec = {}
    names = []
    for name, keys, C, iters, seed in cases():
        cent, obj, zk, rep, nxt = R.kmeans_train_stats(keys, C, iters, seed)
        rec[f"{name}_keys"] = keys
        rec[f"{name}_cfg"] = np.array([C, iters, seed], np.uint64)
        rec[f"{name}_cent"] = cent
        rec[f"{name}_obj"] = obj
        rec[f"{name}_stats"] = np.array([zk, rep, nxt], np.uint64)
        rec[f"{name}_seeds"] = R.kmeans_seed_rows(seed, keys.shape[0], C)
        names.append(name)
        print(f"{name}: n={keys.shape[0]} d={keys.shape[1]} C={C} iters={iters} "
              f"zero={zk} repairs={rep} obj={obj[-1]:.6f}")
    rec["names"] = np.array(names)
    np.savez_compressed(OUT, **rec)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
