"""The product K_nu (paper_2504_12004_b200/csrc/bessel_k.cuh, Temme series +
Steed continued fraction, used by k_h8 for general smoothness)
compiled for the host and checked against scipy.special.kv (CPU, no GPU)."""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest
from scipy import special

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bk():
    out = os.path.join(tempfile.mkdtemp(), "bk.so")
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", os.path.join(ROOT, "tools", "dbg", "besselk_host.cpp"),
                    "-o", out], check=True)
    L = ctypes.CDLL(out)
    L.sbv_test_besselk.restype = ctypes.c_double
    L.sbv_test_besselk.argtypes = [ctypes.c_double, ctypes.c_double]
    return L.sbv_test_besselk


@pytest.mark.parametrize("nu", [0.0, 0.1, 0.25, 0.5, 0.75, 1.0, 1.3, 1.5, 2.0, 2.5, 3.7, 6.4, 10.2, 19.9])
def test_besselk_matches_scipy(bk, nu):
    # scipy's own error reaches ~7e-14 near x = 2; the oracle's integral agrees with
    # the product code to ~1e-15 there (tests/test_oracle_pins.py pins it to scipy)
    for x in np.concatenate([np.geomspace(1e-8, 700, 400), [0.999, 1.0, 1.5, 1.999999, 2.0, 2.000001]]):
        ref = special.kv(nu, x)
        if ref > 1e-300:
            assert abs(bk(nu, x) - ref) <= 2e-13 * ref, (nu, x)


def test_besselk_half_integer_closed_forms(bk):
    """K_{1/2}(x) = sqrt(pi/(2x)) e^-x, K_{3/2} = K_{1/2} (1 + 1/x)."""
    for x in [1e-3, 0.5, 1.7, 2.3, 9.0, 60.0]:
        k12 = np.sqrt(np.pi / (2 * x)) * np.exp(-x)
        assert abs(bk(0.5, x) - k12) <= 1e-14 * k12
        assert abs(bk(1.5, x) - k12 * (1 + 1 / x)) <= 1e-14 * k12 * (1 + 1 / x)
