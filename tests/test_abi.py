"""CPU checks of the C boundary: libsbv.so builds/loads, exports every symbol
include/sbv.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sbv.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void)\s+(sbv_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def libsbv():
    from paper_2504_12004_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ["sbv_prepare", "sbv_loglik", "sbv_block_terms", "sbv_num_blocks", "sbv_get_blocks",
              "sbv_get_neighbors", "sbv_comm_init", "sbv_last_error", "sbv_destroy"]:
        assert s in syms


def test_library_exports_every_declared_symbol(libsbv):
    for s in declared_symbols():
        assert hasattr(libsbv, s), s


def test_binding_lists_every_export():
    from paper_2504_12004_b200 import sbv
    assert sorted(sbv.EXPORTS) == [s for s in declared_symbols() if s in sbv.EXPORTS]
    assert set(declared_symbols()) == set(sbv.EXPORTS)


def test_abi_version(libsbv):
    assert libsbv.sbv_abi_version() == 2


def test_library_is_sm100a_and_uses_dmma(libsbv):
    import subprocess
    from paper_2504_12004_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core path of the fused per-block kernel


def test_no_oracle_in_product_path():
    pkg = os.path.join(ROOT, "paper_2504_12004_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "sbv_oracle" not in txt and "liboracle" not in txt, f


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is None and
                    __import__("torch").cuda.is_available(), reason="GPU present")
def test_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_12004_b200 import SBVError, prepare
    with pytest.raises(SBVError):
        prepare([[0.0, 1.0]], 1, 0, [1.0, 1.0])
