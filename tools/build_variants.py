"""Build experimental libsbv variants (CPU side):
    python tools/build_variants.py name1="-DFOO" name2="-DBAR=2" ...
-> paper_2504_12004_b200/variants/libsbv_<name>.so ; probe on the GPU with
    SBV_LIB=<path> python tools/probe_perf.py cfg2 2
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
out = os.path.join(ROOT, "paper_2504_12004_b200", "variants")
os.makedirs(out, exist_ok=True)
for spec in sys.argv[1:]:
    name, _, flags = spec.partition("=")
    os.environ["SBV_NVCC_EXTRA"] = flags
    os.environ["SBV_LIB_OUT"] = os.path.join(out, f"libsbv_{name}.so")
    import importlib
    import paper_2504_12004_b200.build as b
    importlib.reload(b)
    b.build(force=True)
    print("built", name, flags)
