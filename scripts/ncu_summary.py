#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (committed evidence).

    python scripts/ncu_summary.py REPORT.ncu-rep [--out profiles/NAME.md] [--json profiles/NAME.json]
    python scripts/ncu_summary.py --launches LAUNCHES.csv --out profiles/NAME_launches.md

Per kernel: duration, DRAM bytes (read+write = "traffic"), DRAM throughput,
SM/tensor-pipe utilisation, occupancy, registers, top stall reasons.
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
              "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
              "s": 1.0}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, zip(r, units))) for r in rows[2:]]


def num(v, u=""):
    try:
        x = float(v.replace(",", ""))
    except Exception:
        return None
    return x * UNIT_SCALE.get(u, 1)


def summarise(rep):
    res = []
    for r in raw_rows(rep):
        k = {"kernel": r.get("Kernel Name", ("?", ""))[0]}
        for m, name in METRICS.items():
            if m in r:
                k[name] = num(*r[m])
        stalls = {}
        for m, (v, u) in r.items():
            if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued"):
                x = num(v)
                if x:
                    stalls[m.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
        tot = sum(stalls.values()) or 1
        k["top_stalls"] = {s: round(v / tot, 3) for s, v in
                           sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        if k.get("dram_read") is not None and k.get("dram_write") is not None:
            k["traffic_bytes"] = k["dram_read"] + k["dram_write"]
        if k.get("duration") and k.get("traffic_bytes"):
            k["dram_gbs"] = k["traffic_bytes"] / k["duration"] / 1e9
        res.append(k)
    return res


def launches(path):
    agg = defaultdict(list)
    lines = [l for l in open(path) if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"]].append(num(r["Metric Value"], r.get("Metric Unit", "")))
    total = sum(sum(v) for v in agg.values())
    rows = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        rows.append({"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v) * 1e6,
                     "share": sum(v) / total if total else 0})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--out")
    ap.add_argument("--json")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    lines = [f"# {a.title or (a.report or a.launches)}", ""]
    data = None
    if a.report:
        data = summarise(a.report)
        lines.append("| kernel | µs | DRAM bytes | DRAM GB/s | DRAM % | SM % | tensor % | occ % | regs | top stalls |")
        lines.append("|---|---|---|---|---|---|---|---|---|---|")
        for k in data:
            st = ", ".join(f"{s} {v:.0%}" for s, v in k["top_stalls"].items())
            lines.append(
                f"| {k['kernel'][:60]} | {k.get('duration', 0) * 1e6:.1f} | "
                f"{k.get('traffic_bytes', 0) / 1e6:.1f} MB | {k.get('dram_gbs', 0):.0f} | "
                f"{k.get('dram_pct') or 0:.1f} | {k.get('sm_pct') or 0:.1f} | "
                f"{k.get('tensor_pipe_pct') or 0:.1f} | {k.get('occupancy_pct') or 0:.1f} | "
                f"{k.get('registers') or 0:.0f} | {st} |")
    if a.launches:
        data = launches(a.launches)
        lines.append("| kernel | launches | mean µs | share of GPU time |")
        lines.append("|---|---|---|---|")
        for r in data:
            lines.append(f"| {r['kernel'][:70]} | {r['launches']} | {r['mean_us']:.1f} | {r['share']:.1%} |")
    text = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(text)
    print(text)
    if a.json:
        json.dump(data, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
