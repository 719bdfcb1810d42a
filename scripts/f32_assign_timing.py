"""Host f32 build: tcgen05 split-key assignment vs the fp64 kernel (timing aid)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2502_08246_b200 as sb
from tests.cases import unit_rows

ctx = sb.Context(0)
rs = np.random.RandomState(3)
G, n, C = 8, 131072, 1024
cent = unit_rows(rs.randn(C, 128))
K = (rs.randn(G * n, 128) * 2).astype(np.float32)
V = rs.randn(G * n, 128).astype(np.float32)
part = sb.Partition(cent, ctx)
res = {}
for tc in (1, 0):
    ctx.set_option("assign_f32_tc", tc)
    L = sb.Layer([n] * G, 128, C, 1, 2047, ctx)
    ts = []
    for rep in range(3):
        ctx.enable_timing(True)
        L.build([part] * G, K, V, K)
        ctx.synchronize()
        ts.append(L.build_timing())
        ctx.enable_timing(False)
    used, refined = L.assign_info()
    a = L.read_index(0)[0]
    res[tc] = {"assign_ms": round(min(t[0] for t in ts), 3), "pack_ms": round(min(t[1] for t in ts), 3),
               "tensor_cores": used, "refined_keys": refined, "keys": G * (n - 1)}
    res[tc]["_a"] = a
same = bool(np.array_equal(res[0]["_a"], res[1]["_a"]))
for r in res.values():
    r.pop("_a")
print(json.dumps({"tcgen05_split": res[1], "fp64": res[0], "assignments_equal": same}))
