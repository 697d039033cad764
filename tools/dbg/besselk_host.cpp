// host build of the product K_nu (paper_2504_12004_b200/csrc/bessel_k.cuh) for tests/test_besselk.py
#include "../../paper_2504_12004_b200/csrc/bessel_k.cuh"
extern "C" double sbv_test_besselk(double nu, double x) { return sbv::besselk(nu, x); }
