"""Warp-stall samples of an ncu report attributed to INLINED CALL SITES.
    python tools/ncu_callsites.py gpurun_out/x.ncu-rep path/to/kernel.cubin kernel_symbol
Joins the ncu SASS page (per-instruction samples, absolute addresses) with
nvdisasm -gi line info (offset -> innermost line + 'inlined at' chain)."""
import csv, io, re, subprocess, sys
from collections import Counter, defaultdict
rep, cubin, sym = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
iA, iS = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
addrs = []
for r in data:
    try:
        addrs.append((int(r[iA], 16), float(r[iS] or 0), {h: float(r[i] or 0) for i, h in stalls}))
    except ValueError:
        pass
base = min(a for a, _, _ in addrs)
dis = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(dis) if l.startswith(".text." + sym + ":")][0]
info = {}
cur = ("?", 0, ())
for l in dis[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    m = re.search(r'File "([^"]+)", line (\d+)(.*)', l)
    if m:
        chain = tuple((f.split("/")[-1], int(n)) for f, n in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3)))
        cur = (m.group(1).split("/")[-1], int(m.group(2)), chain)
        continue
    mm = re.match(r"\s+/\*([0-9a-f]+)\*/", l)
    if mm:
        info[int(mm.group(1), 16)] = cur
tot = sum(s for _, s, _ in addrs)
site = Counter(); site_st = defaultdict(Counter)
for a, s, st in addrs:
    f, ln, chain = info.get(a - base, ("?", 0, ()))
    # attribute to the outermost frame inside the kernel file (the call site in k_h8)
    key = chain[-1] if chain else (f, ln)
    site[key] += s
    for h, v in st.items():
        site_st[key][h] += v
src = {}
for f, ln in site:
    pass
print(f"total samples {tot:.0f}")
for (f, ln), s in site.most_common(30):
    top = sorted(((v, h[6:]) for h, v in site_st[(f, ln)].items()), reverse=True)[:3]
    print(f"{s/tot*100:5.1f}%  {f}:{ln}  " + " ".join(f"{h}={v/tot*100:.1f}" for v, h in top))
