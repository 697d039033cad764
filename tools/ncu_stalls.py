"""Per-function warp-stall breakdown of an ncu report (source page, CUDA lines).
    python tools/ncu_stalls.py gpurun_out/x.ncu-rep [source-file]
Each CUDA source line's samples are attributed to the enclosing function /
task-type region of the source file."""
import csv, io, re, subprocess, sys
from collections import Counter, defaultdict
rep = sys.argv[1]
srcf = sys.argv[2] if len(sys.argv) > 2 else "paper_2504_12004_b200/csrc/h8_kernel.cuh"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = [r for r in rows if r and r[0] == "Line No"][0]
iS = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
src = open(srcf).read().split("\n")
marks = []  # (line, name) of function starts / labelled regions
for i, l in enumerate(src):
    m = re.match(r"(?:template <[^>]*>\s*)?__(?:device|global)__.*?(\w+)\(", l)
    if m:
        marks.append((i + 1, m.group(1)))
    m2 = re.search(r"// region: (\w+)", l)
    if m2:
        marks.append((i + 1, m2.group(1)))
marks.sort()
def region(ln):
    r = "?"
    for a, n in marks:
        if a <= ln: r = n
    return r
tot = 0.0
agg = defaultdict(Counter)
lines = Counter()
cur = ""
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if not r or not r[0].isdigit() or len(r) <= iS: continue
    try: s = float(r[iS] or 0)
    except ValueError: continue
    ln = int(r[0])
    if not cur.endswith(srcf.split("/")[-1]):
        reg = "hdr:" + cur.split("/")[-1]
        tot += s
        agg[reg]["samples"] += s
        for i, h in stall_cols:
            try: agg[reg][h] += float(r[i] or 0)
            except ValueError: pass
        continue
    reg = region(ln)
    tot += s
    agg[reg]["samples"] += s
    lines[(ln, src[ln - 1].strip()[:70])] += s
    for i, h in stall_cols:
        try: agg[reg][h] += float(r[i] or 0)
        except ValueError: pass
print(f"total samples {tot:.0f}")
for reg, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
    top = sorted(((v, h[6:]) for h, v in c.items() if h != "samples"), reverse=True)[:4]
    print(f"{c['samples']/tot*100:5.1f}%  {reg:18s} " + "  ".join(f"{h}={v/tot*100:.1f}" for v, h in top))
print("\ntop lines")
for (ln, t), s in lines.most_common(25):
    print(f"{s/tot*100:5.1f}% {ln:5d} {t}")
