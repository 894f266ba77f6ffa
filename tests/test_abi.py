"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/potr_b200.h declares.  No compute calls here."""

import ctypes
import os
import re

import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "potr_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(potr_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_14821_b200 import _native
    return _native.load()


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("potr_forward_stats", "potr_score_views", "potr_render", "potr_compact",
                 "potr_forward_stats_host", "potr_compact_host", "potr_bin"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2601_14821_b200 import _native
    for name in declared_functions():
        assert hasattr(lib, name), f"{name} missing from libpotr_b200.so"
        assert name in _native._SIGNATURES, f"{name} has no ctypes signature"
    assert lib.potr_abi_version() == 1


def test_library_targets_sm100a():
    from paper_2601_14821_b200 import _native
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.library_path()],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    assert lib.potr_create(0, ctypes.byref(h)) != 0
    from paper_2601_14821_b200 import rasterizer
    from paper_2601_14821_b200.fixture import make_fixture
    splats, cams = make_fixture(10, 1, 0, 16)
    with pytest.raises(RuntimeError, match="CUDA"):
        rasterizer.render_image(splats, cams[0])


def test_null_context_is_an_argument_error(lib):
    assert lib.potr_forward_stats(None, None, 0, None, None, None, None, None, None) == -1
    assert lib.potr_synchronize(None) == -1
