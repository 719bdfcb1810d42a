"""Summarise trace_step tile/CTA npy files (profiling aid)."""
import sys
import numpy as np
import json

def main(prefix, r=2):
    t = np.load(prefix + "_tiles.npy"); c = np.load(prefix + "_cta.npy")
    m = json.load(open(prefix + ".json"))["median"]
    print({k: m[k] for k in ("decode", "combine", "decode_cta_end_us", "decode_cta_first_tile_us", "decode_cta_start_us")})
    for rr in range(len(t)):
        T = t[rr]; land = T[:, :, 1].ravel(); land = land[~np.isnan(land)]
        h, _ = np.histogram(land, bins=np.arange(0, 60, 4))
        print(rr, "TB/s per 4us:", np.round(h * 65536 / 4e-6 / 1e12, 1))
    st, ft, en, nt = c[r]
    print("tiles/cta", np.percentile(nt, [0, 50, 100]), "end", np.round(np.percentile(en, [0, 10, 50, 90, 100]), 1))
    T = t[r]
    for b in list(np.argsort(en)[-3:]) + list(np.argsort(en)[:2]):
        n = int(nt[b]); ce = [i for i in range(min(n, 48)) if int(T[b, i, 8]) & 32]
        print(b, "start %.1f end %.1f n %d" % (st[b], en[b], n), "chunk ends", ce, "issues",
              np.round(T[b, max(0, n - 8):n, 0], 1), "done", np.round(T[b, max(0, n - 8):n, 2], 1))

if __name__ == "__main__":
    main(sys.argv[1])
