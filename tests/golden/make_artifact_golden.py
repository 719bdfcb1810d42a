"""Write SAAPTNS1 artifacts with the *reference itself* (oracle/_ref:
tensor_write / u64_write / partition_save (= tensor_write of the centroids) /
ivf_save / qmodel_save) into tests/golden/artifacts/, and record what the
reference reads back in tests/golden/artifacts_expect.npz.

    python tests/golden/make_artifact_golden.py
"""
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

G = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(G, "artifacts")


def main():
    R = oracle.ref()
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    r = np.random.default_rng(7)
    keys = r.normal(0, 1, (200, 16)).astype(np.float32)
    cent = R.kmeans_train(keys, 8, 4, 20)
    a = R.assign_keys(keys, cent)
    off, idx = R.build_ivf(a, 8)
    assert R.tensor_write(cent, os.path.join(OUT, "partition.tensor")) is None
    assert R.u64_write(off, os.path.join(OUT, "off.tensor")) is None
    assert R.u64_write(idx, os.path.join(OUT, "idx.tensor")) is None
    assert R.tensor_write(keys[:5], os.path.join(OUT, "block.tensor")) is None
    assert R.tensor_write(np.zeros((0, 4), np.float32), os.path.join(OUT, "empty.tensor")) is None
    assert R.u64_write(np.zeros(0, np.uint64), os.path.join(OUT, "empty_u64.tensor")) is None
    assert R.qmodel_save_init(os.path.join(OUT, "qmodel"), 16, 32, 8, 9) is None
    qm, e = R.qmodel_load(os.path.join(OUT, "qmodel"))
    assert e is None
    blk, _ = R.tensor_read(os.path.join(OUT, "block.tensor"))
    np.savez_compressed(os.path.join(G, "artifacts_expect.npz"), cent=cent, off=off, idx=idx,
                        block=blk, keys=keys, **{f"qm_{k}": v for k, v in qm.items()})
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
