"""Summarise an ncu report: key metrics, stall reasons, top SASS lines, opcode mix."""
import csv, subprocess, sys, io
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum"]
for h, u, v in zip(hdr, units, vals):
    if h in want or (h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")):
        try:
            if h.startswith("smsp__average_warps_issue_stalled") and float(v) < 0.3: continue
        except ValueError: pass
        print(f"{h[:80]:80s} {v} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(x[iW]) for x in data if x[iW].isdigit())
c, ce = Counter(), Counter()
for x in data:
    if not x[iW].isdigit(): continue
    t = x[iS].strip().split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += int(x[iW]); ce[op.split(".")[0]] += int(x[iE])
print("stall samples by opcode:", [(k, round(100 * v / tot, 1)) for k, v in c.most_common(12)])
print("executed by opcode:", ce.most_common(14))
top = sorted(range(len(data)), key=lambda i: -(int(data[i][iW]) if data[i][iW].isdigit() else 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for i in sorted(top):
    print(i, round(100 * int(data[i][iW]) / tot, 1), data[i][iE], data[i][iS].strip()[:90])
