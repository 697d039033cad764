"""H8 per-task timeline (tool; needs a -DSBV_TRACE=1 build of libsbv):

    SBV_LIB=paper_2504_12004_b200/variants/libsbv_trace.so python tools/h8_trace.py [cfg] [n]

Runs one prepare + one loglik, dumps the k_h8 trace (one record per task per
warp: clock64 at grab, after the dependency waits, at the end) and prints a
summary: where the warps' time goes (dependency waits, task bodies by type,
staging, end-of-block barrier), per-panel chain timing and block spans.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(cfg, n):
    import torch
    import sbv_inputs as si
    import paper_2504_12004_b200 as sbv
    c = dict(si.CONFIGS[cfg])
    if n:
        c["n"] = n
    X = torch.from_numpy(si.make_X(c["n"], c["d"], seed=1)).cuda()
    y = torch.from_numpy(si.make_y(si.make_X(c["n"], c["d"], seed=1), seed=2, kind="iid")).cuda()
    theta = si.default_theta(c["d"], nu=c["nu"], tau2=1e-4)
    h = sbv.Handle(seed=3, profile=True)
    h.prepare(X, c["bs"], c["m"], si.default_scale(c["d"]))
    h.loglik(y, theta)  # warm
    out = os.path.abspath("gpurun_out/h8_trace.bin")
    os.environ["SBV_TRACE_OUT"] = out
    h.loglik(y, theta)
    del os.environ["SBV_TRACE_OUT"]
    return out, h.stage_times(False)["H8_block_llh"], h.stats()


def analyse(path):
    r = np.fromfile(path, dtype=np.uint64).reshape(-1, 6).astype(np.int64)
    t0, t1, t2, item, code, cw = r.T
    cta, warp = cw >> 8, cw & 0xFF
    typ = (code >> 24) & 0xFF
    j = (code >> 12) & 0xFFF
    ch = code & 0xFFF
    names = {0: "A", 1: "F", 2: "C0", 3: "BC", 4: "BCF"}
    res = {"records": int(len(r))}
    task = typ < 0xF0
    # per-CTA span: first record to last record
    spans = {}
    tot_warp_time = 0
    for c in np.unique(cta):
        m = cta == c
        spans[int(c)] = (int(t0[m].min()), int(t2[m].max()))
    nwarps = int(warp.max()) + 1
    tot_warp_time = sum((b - a) * nwarps for a, b in spans.values())
    wait = (t1 - t0)[task].sum()
    res["warp_time_cycles"] = int(tot_warp_time)
    res["frac_dependency_wait"] = float(wait / tot_warp_time)
    for tcode, nm in names.items():
        mm = task & (typ == tcode)
        if mm.any():
            res[f"frac_body_{nm}"] = float((t2 - t1)[mm].sum() / tot_warp_time)
            res[f"mean_body_{nm}_cycles"] = float((t2 - t1)[mm].mean())
            res[f"count_{nm}"] = int(mm.sum())
    # staging: block-start record (0xFE) -> first task grab of that block in the CTA
    st = typ == 0xFE
    en = typ == 0xFF
    accounted = wait + (t2 - t1)[task].sum()
    res["frac_other (staging, barriers, tail)"] = float(1 - accounted / tot_warp_time)
    # block spans and per-panel F chain
    bspan, fgap, nlist = [], [], []
    key = item * 100000 + cta
    starts = {(int(i), int(c)): int(t) for i, c, t in zip(item[st], cta[st], t0[st])}
    ends = {(int(i), int(c)): int(t) for i, c, t in zip(item[en], cta[en], t0[en])}
    Ns = {(int(i), int(c)): int(cd & 0xFFFFFF) for i, c, cd in zip(item[en], cta[en], code[en])}
    for k_, s in starts.items():
        if k_ in ends:
            bspan.append(ends[k_] - s)
            nlist.append(Ns[k_])
    res["block_span_cycles_mean"] = float(np.mean(bspan)) if bspan else None
    res["block_N_mean"] = float(np.mean(nlist)) if nlist else None
    # F-chain: end of F(j) -> end of F(j+1) within a block
    fm = task & ((typ == 1) | (typ == 4))  # F(j) or BCF(j-1) = BC(j-1,1) + F(j)
    jf = np.where(typ == 4, j + 1, j)
    order = np.lexsort((jf[fm], item[fm]))
    fi, fj, fe, fs, fr = item[fm][order], jf[fm][order], t2[fm][order], t0[fm][order], t1[fm][order]
    gaps = []
    for a_ in range(1, len(fi)):
        if fi[a_] == fi[a_ - 1] and fj[a_] == fj[a_ - 1] + 1:
            gaps.append(fe[a_] - fe[a_ - 1])
    res["F_to_F_cycles_mean"] = float(np.mean(gaps)) if gaps else None
    res["F_wait_cycles_mean"] = float((fr - fs).mean()) if len(fs) else None
    # concurrency: average number of warps in a task body (not waiting), sampled
    res["nwarps_per_cta"] = nwarps
    # per-type body time by panel j (first 12 panels)
    byj = {}
    for tcode, nm in names.items():
        mm = task & (typ == tcode)
        if not mm.any():
            continue
        byj[nm] = [float((t2 - t1)[mm & (j == jj)].mean()) if (mm & (j == jj)).any() else None
                   for jj in range(0, 12)]
    res["body_cycles_by_panel"] = byj
    # dependency-wait by type
    for tcode, nm in names.items():
        mm = task & (typ == tcode)
        if mm.any():
            res[f"frac_wait_{nm}"] = float((t1 - t0)[mm].sum() / tot_warp_time)
    return res


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    path, h8_ms, stats = run(cfg, n)
    res = analyse(path)
    res["h8_ms"] = h8_ms
    res["flops"] = stats["flops"]
    print(json.dumps(res, indent=1))
