"""Summarise gpurun_out/ ncu artefacts into profiles/<round>/ (tracked).

    python tools/summarize_profiles.py r01
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(io.StringIO("".join(lines)))
    hdr = next(rd)
    iK, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iU = hdr.index("Metric Unit")
    for r in rd:
        if r[iM] != "gpu__time_duration.sum":
            continue
        v = float(r[iV].replace(",", ""))
        unit = r[iU]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        rows.append((r[iK].split("(")[0].replace("void ", ""), ns))
    agg = defaultdict(lambda: [0, 0.0])
    for k, ns in rows:
        agg[k][0] += 1
        agg[k][1] += ns
    tot = sum(v[1] for v in agg.values())
    summary = sorted(({"kernel": k, "launches": c, "total_ms": t / 1e6, "share": t / tot}
                      for k, (c, t) in agg.items()), key=lambda x: -x["total_ms"])
    return {"command": "python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-predict",
            "note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); "
                    "compare SHARES, not absolute times",
            "total_launches": len(rows), "kernels": summary}


def raw_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = r[0], r[1], r[2]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_bytes.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in want or (h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")):
            try:
                fv = float(v.replace(",", ""))
                if h.startswith("smsp__average_warps_issue_stalled") and fv < 0.2:
                    continue
                out[h] = [fv, u]
            except ValueError:
                out[h] = [v, u]
    return out


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        json.dump(launches(tag), open(os.path.join(dst, "launch_list_summary.json"), "w"), indent=1)
    for name in ["h8_full", "knn_full"]:
        rep = os.path.join(OUT, name + ".ncu-rep")
        if os.path.exists(rep):
            json.dump(raw_metrics(rep), open(os.path.join(dst, name + "_ncu_summary.json"), "w"), indent=1)
    print("wrote", os.listdir(dst))


if __name__ == "__main__":
    main()
