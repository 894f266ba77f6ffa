"""Accuracy of the rasterizer's fp64 exp (csrc/common.cuh exp_neg) via its
host twin (tests/native/exp_twin.c: same IEEE operation sequence, fma() ==
DFMA), against long-double expl over the domain the kernel uses."""

import ctypes
import os
import subprocess

import pytest

from tests.conftest import ROOT


@pytest.fixture(scope="module")
def twin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("exp") / "exp_twin.so")
    src = os.path.join(ROOT, "tests", "native", "exp_twin.c")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", out, src, "-lm"],
                   check=True)
    lib = ctypes.CDLL(out)
    lib.exp_twin_max_ulp.restype = ctypes.c_double
    lib.exp_twin_max_ulp.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64)]
    lib.exp_twin.restype = ctypes.c_double
    lib.exp_twin.argtypes = [ctypes.c_double]
    return lib


def test_faithful_over_the_alpha_domain(twin):
    # power in [log(1/255) - margin, 0] after the prefilter; test a wider range
    nd = ctypes.c_int64()
    worst = twin.exp_twin_max_ulp(-7.0, 1e-12, 2_000_000, ctypes.byref(nd))
    assert worst < 1.0, worst
    assert nd.value < 0.1 * 2_000_000  # mostly bit-identical to glibc exp


def test_special_points(twin):
    import math
    assert twin.exp_twin(0.0) == 1.0
    for x in (-1e-300, -1e-17, -0.5, -1.0, -5.5451774444795623):
        assert abs(twin.exp_twin(x) - math.exp(x)) <= 2.3e-16 * math.exp(x)
