"""tcgen05 decode vs mma.sync decode on one C3 layer (sparse + dense), then
timings.  Profiling / bring-up aid."""
import argparse, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx-len", type=int, default=131072)
    args = ap.parse_args()
    import torch
    import paper_2502_08246_b200 as sb
    a = argparse.Namespace(ctx_len=args.ctx_len, batch=8, kv_heads=8, q_heads=32, dim=128, buckets=1024,
                           probes=32, recent=2047, sink=1, kmeans_iters=10)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    ctx = sb.Context(0)
    ctx.set_stream(stream.cuda_stream)
    lay = bench.build_c3_layer(sb, torch, ctx, a, 0, 0.0, 8, 0, dev, stream, len(os.sched_getaffinity(0)))
    cfg = sb.SparseAttnConfig(a.probes, 128, sb.DenseWindow(1, a.recent))
    res = {}
    for tc in (0, 1):
        ctx.set_option("decode_tc", tc)
        out = torch.zeros(64, 4, 128, device=dev)
        stats = torch.zeros(64, 3, dtype=torch.int64, device=dev)
        lay.L.sparse_attention_dev(lay.routers, lay.qr_t, lay.qd_t, 4, cfg, out, stats)
        ctx.synchronize()
        outd = torch.zeros(64, 4, 128, device=dev)
        lay.kv.dense_attention_dev(lay.qr_t, 4, outd)
        ctx.synchronize()
        res[tc] = (out.clone(), outd.clone(), stats.clone())
        print("tc", tc, "ok", float(out.abs().sum()), float(outd.abs().sum()), flush=True)
    def rel(x, y):
        return float(((x - y).abs() / y.abs().clamp_min(1e-3)).max())
    print("sparse max rel diff", rel(res[1][0], res[0][0]), "dense", rel(res[1][1], res[0][1]),
          "stats equal", bool(torch.equal(res[0][2], res[1][2])), flush=True)
    bad = ((res[1][0] - res[0][0]).abs() > 1e-3 * res[0][0].abs().clamp_min(1e-3)).nonzero()
    print("bad entries", bad.shape[0], bad[:8].tolist(), flush=True)
    # repeated steps agree
    ctx.set_option("decode_tc", 1)
    out = torch.zeros(64, 4, 128, device=dev)
    stats = torch.zeros(64, 3, dtype=torch.int64, device=dev)
    for i in range(20):
        lay.L.sparse_attention_dev(lay.routers, lay.qr_t, lay.qd_t, 4, cfg, out, stats)
    ctx.synchronize()
    print("after 20 steps rel", rel(out, res[0][0]), flush=True)


if __name__ == "__main__":
    main()
