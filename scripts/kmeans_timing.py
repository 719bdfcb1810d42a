"""Device k-means timing at the partition-training scales SURVEY §8(f) names
(C4/C5): one call of saap_kmeans_train (host keys in, centroids out, so the
H2D of the keys is included).  Prints one JSON line per case."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_08246_b200 as sb  # noqa: E402

CASES = [(131071, 128, 1024, 10), (1048575, 128, 4096, 3), (1048575, 128, 16384, 1)]


def main():
    ctx = sb.default_context()
    r = np.random.default_rng(0)
    sel = os.environ.get("KM_CASES")
    cases = [CASES[int(i)] for i in sel.split(",")] if sel else CASES
    for n, d, C, iters in cases:
        cen = r.normal(0, 1, (256, d)).astype(np.float32)
        keys = (cen[r.integers(0, 256, n)] * 2 + r.normal(0, 1, (n, d))).astype(np.float32)
        sb.kmeans_train(keys[:4096], 64, 1, sb.Rng(1), ctx=ctx)  # warm the module
        st = sb.KMeansStats()
        t0 = time.perf_counter()
        sb.kmeans_train(keys, C, iters, sb.Rng(1), st, ctx=ctx)
        dt = time.perf_counter() - t0
        fma = n * C * d * (iters + 1)
        print(json.dumps({"n": n, "d": d, "C": C, "iters": iters, "s": round(dt, 3),
                          "s_per_iter": round(dt / iters, 4),
                          "assign_fp64_tflops": round(2 * fma / dt / 1e12, 2),
                          "repairs": st.empty_cluster_repairs,
                          "objective": st.objective_per_iter[-1]}), flush=True)


if __name__ == "__main__":
    main()
