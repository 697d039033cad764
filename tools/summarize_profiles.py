"""Summarise one profiling pass (tools/gpu_r2_prof.sh outputs in gpurun_out/) into profiles/<round>/:
    python tools/summarize_profiles.py TAG ROUND_DIR
-> <ROUND_DIR>/h8_full_ncu_summary.json, knn_full_ncu_summary.json (selected metrics of the
   `ncu --set full` raw page) and launch_list_summary.json (per-kernel share of the launch list)."""
import csv, io, json, os, sys
from collections import defaultdict

tag, out = sys.argv[1], sys.argv[2]
src = "gpurun_out"
KEEP = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sector_hit_rate.pct",
        "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "Kernel Name")


def raw_summary(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units, vals = rows[i], rows[i + 1], rows[i + 2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEEP or (h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")):
            try:
                d[h] = [float(v.replace(",", "")), u]
            except ValueError:
                d[h] = [v, u]
    d["source"] = f"ncu --set full --clock-control none, {os.path.basename(path)} (tools/gpu_r2_prof.sh, TAG={tag})"
    return d


os.makedirs(out, exist_ok=True)
for name, fn in (("h8", "h8_full_ncu_summary.json"), ("knn", "knn_full_ncu_summary.json")):
    p = os.path.join(src, f"{tag}_{name}_raw.csv")
    if os.path.exists(p):
        json.dump(raw_summary(p), open(os.path.join(out, fn), "w"), indent=1)
        print("wrote", fn)

p = os.path.join(src, f"{tag}_launches.csv")
if os.path.exists(p):
    lines = [l for l in open(p) if l.startswith('"')]
    rows = [r for r in csv.DictReader(io.StringIO("".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
    # the bench steps only (3 warm-up + 3 timed = prepare from k_scale through
    # loglik's k_final, 6 times), not the loglik-only / graph / gradient /
    # prediction measurements that follow them in the same process
    names = [r["Kernel Name"] for r in rows]
    finals = [i for i, nm in enumerate(names) if "k_final" in nm]
    if len(finals) >= 6:
        rows = rows[: finals[5] + 1]
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(r["Metric Unit"], 1.0)
        k = r["Kernel Name"].split("(")[0]
        tot[k] += v * scale
        cnt[k] += 1
    s = sum(tot.values())
    ks = sorted(tot, key=lambda k: -tot[k])
    json.dump({"command": "python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-predict",
               "note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); "
                       "the 6 bench steps (3 warm-up + 3 timed, prepare + loglik) only; compare SHARES, not absolute times",
               "tag": tag, "total_launches": sum(cnt.values()),
               "kernels": [{"kernel": k, "launches": cnt[k], "total_ms": tot[k], "share": tot[k] / s} for k in ks]},
              open(os.path.join(out, "launch_list_summary.json"), "w"), indent=1)
    print("wrote launch_list_summary.json", [(k, round(tot[k] / s, 3)) for k in ks[:4]])
