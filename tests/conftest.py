import functools
import hashlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger-scale parity runs")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def fingerprint(splats, cams):
    """Same digest as oracle/gen_golden.py."""
    h = hashlib.sha256()
    for a in (splats.positions, splats.sh, splats.opacities, splats.scales, splats.rotations):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    for c in cams:
        h.update(np.asarray(c.eye, dtype=np.float64).tobytes())
        h.update(np.asarray(c.rotation, dtype=np.float64).tobytes())
        h.update(np.array([c.fx, c.fy, c.cx, c.cy, c.width, c.height], dtype=np.float64).tobytes())
    return h.hexdigest()


def perturbed(splats):
    out = splats.copy()
    out.opacities = out.opacities * 0.97
    return out


def small_scene():
    from paper_2601_14821_b200.fixture import make_fixture
    return make_fixture(num_splats=1500, num_cameras=6, seed=3, resolution=48)


def sh_scene():
    from paper_2601_14821_b200.fixture import make_fixture, shell_splats
    from paper_2601_14821_b200.scene import Splats
    splats, cams = make_fixture(num_splats=600, num_cameras=6, seed=5, resolution=48)
    extra = shell_splats(3, seed=9)
    extra.positions = extra.positions + np.array([0.0, 40.0, 0.0])
    splats = Splats(*(np.concatenate([getattr(splats, f), getattr(extra, f)]) for f in
                      ("positions", "sh", "opacities", "scales", "rotations")))
    return splats, cams


@functools.lru_cache(maxsize=1)
def c3_scene():
    """The C3-shaped synthetic scene (3M splats, 200 views at 1237x822),
    generated once per session; callers must not modify it."""
    from paper_2601_14821_b200.fixture import config_scene
    return config_scene("C3")


def oracle_scene(seed):
    from paper_2601_14821_b200.fixture import random_scene
    rng = np.random.default_rng(seed + 1000)
    ns = int(rng.integers(20, 51))
    nc = int(rng.integers(2, 5))
    return random_scene(seed, num_splats=ns, num_cameras=nc)


def score_close(got, ref, rel=1e-4, floor=0.0):
    """SURVEY.md 8(a) score check: |gpu - ref| <= rel*|ref| + floor."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    return bool(np.all(np.abs(got - ref) <= rel * np.abs(ref) + floor))


def have_reference():
    return os.path.isdir(os.path.join(REFERENCE_SRC, "potr"))


@pytest.fixture(scope="session")
def reference():
    """The reference package (development container only)."""
    if not have_reference():
        pytest.skip("reference package not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import potr  # noqa: F401
    return potr


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def sh_degenerate_scene():
    """Rank-deficient SH systems (compaction.py:138-145; pkg/tests/
    test_compaction.py:203-210): 400 splats near the origin, four cameras of
    which two share an eye, sparse importances, so most splats see one or two
    distinct directions.  At lambda = 0 their normal equations are singular:
    with weights ~1e-2 the 1e-10 jitter rescues them (status 1), with weights
    ~1e5 it is lost in the rounding of G and the solve fails (RidgeError,
    status 2: the splat keeps its original coefficients)."""
    from paper_2601_14821_b200.fixture import look_at
    from paper_2601_14821_b200.scene import Camera, Splats
    rng = np.random.default_rng(0)
    n = 400
    pos = rng.uniform(-0.2, 0.2, (n, 3))
    sh = 0.3 * rng.standard_normal((n, 3, 16))
    sh[:, :, 0] += 1.0
    splats = Splats(pos, sh, np.full(n, 0.9), np.full((n, 3), 0.05),
                    np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)))
    eyes = np.array([[3.0, 0.1, 0.2], [3.0, 0.1, 0.2], [0.2, 3.0, 0.1], [0.1, 0.2, 3.0]])
    cams = [Camera(eye=e, rotation=look_at(e), fx=40.0, fy=40.0, cx=16.0, cy=16.0, width=32,
                   height=32) for e in eyes]
    ci = rng.uniform(0.0, 0.02, (4, n)) * (rng.uniform(size=(4, n)) < 0.5)
    return splats, cams, ci


# (camera_importance scale, lambda_y, parallel_threshold) of the degenerate cases
SH_DEGENERATE_CASES = [(1.0, 0.0, 1.0), (1.0, 0.0, 0.9999), (1e7, 0.0, 1.0), (1e7, 0.0, 0.9999),
                       (1.0, 1e-12, 0.9999)]
