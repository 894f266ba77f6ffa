"""ctypes front end of the CPU oracle (oracle/potr_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py as the parity checker.  The
product package (paper_2601_14821_b200) never imports it.

Each function mirrors one reference function (file:line in
/root/reference/pkg/src/potr) and takes any object exposing the reference's
Splats / Camera attributes.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpotr_oracle.so")
_lib = None


class OCam(ctypes.Structure):
    _fields_ = [("eye", ctypes.c_double * 3), ("rot", ctypes.c_double * 9),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


def build():
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _splat_arrays(splats):
    n = int(splats.positions.shape[0])
    return (n, _f64(splats.positions, (n, 3)), _f64(splats.sh, (n, 3, 16)),
            _f64(splats.opacities, (n,)), _f64(splats.scales, (n, 3)),
            _f64(splats.rotations, (n, 4)))


def _cam(c):
    o = OCam()
    o.eye[:] = [float(v) for v in np.asarray(c.eye, dtype=np.float64).reshape(3)]
    o.rot[:] = [float(v) for v in np.asarray(c.rotation, dtype=np.float64).reshape(9)]
    o.fx, o.fy, o.cx, o.cy = float(c.fx), float(c.fy), float(c.cx), float(c.cy)
    o.width, o.height = int(c.width), int(c.height)
    return o


def _cams(cams):
    arr = (OCam * max(1, len(cams)))()
    for i, c in enumerate(cams):
        arr[i] = _cam(c)
    return arr


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed ({rc})")


def project(splats, cam):
    """project_splats (rasterizer.py:56-97) + splat_colors (:100-110) for all
    splats.  Returns a dict of arrays."""
    n, pos, sh, op, sc, rot = _splat_arrays(splats)
    out = {"mean2d": np.empty((n, 2)), "cov2d": np.empty((n, 3)), "view_depth": np.empty(n),
           "radius": np.empty(n), "valid": np.empty(n, dtype=np.uint8),
           "colors": np.empty((n, 3))}
    c = _cam(cam)
    _check(lib().oracle_project(ctypes.c_int64(n), _p(pos), _p(sh), _p(op), _p(sc), _p(rot),
                                ctypes.byref(c), _p(out["mean2d"]), _p(out["cov2d"]),
                                _p(out["view_depth"]), _p(out["radius"]), _p(out["valid"]),
                                _p(out["colors"])), "project")
    out["valid"] = out["valid"].astype(bool)
    return out


def depth_order(splats, cam):
    """ids = nonzero(valid); ids[argsort(depth, stable)] (rasterizer.py:248-250)."""
    n, pos, sh, op, sc, rot = _splat_arrays(splats)
    order = np.empty(max(n, 1), dtype=np.int64)
    nv = ctypes.c_int64(0)
    c = _cam(cam)
    _check(lib().oracle_depth_order(ctypes.c_int64(n), _p(pos), _p(sc), _p(rot), ctypes.byref(c),
                                    _p(order), ctypes.byref(nv)), "depth_order")
    return order[:nv.value].copy()


def render(splats, cam, records=False):
    """render_image (rasterizer.py:270) / render_with_records (:246-267).
    Returns (image, trans) or (image, trans, records dict)."""
    n, pos, sh, op, sc, rot = _splat_arrays(splats)
    h, w = int(cam.height), int(cam.width)
    image = np.empty((h, w, 3))
    trans = np.empty((h, w))
    nrec = ctypes.c_int64(0)
    c = _cam(cam)
    L = lib()
    args = [ctypes.c_int64(n), _p(pos), _p(sh), _p(op), _p(sc), _p(rot), ctypes.byref(c),
            _p(image), _p(trans), ctypes.byref(nrec)]
    _check(L.oracle_render(*args, None, None, None, None, None, ctypes.c_int64(0)), "render")
    if not records:
        return image, trans
    m = nrec.value
    rec = {"splat_ids": np.empty(m, dtype=np.int32), "pixels": np.empty(m, dtype=np.int32),
           "alphas": np.empty(m), "trans_at": np.empty(m), "partials": np.empty((m, 3))}
    _check(L.oracle_render(*args, _p(rec["splat_ids"]), _p(rec["pixels"]), _p(rec["alphas"]),
                           _p(rec["trans_at"]), _p(rec["partials"]), ctypes.c_int64(m)),
           "render")
    rec["splat_ids"] = rec["splat_ids"].astype(np.int64)
    rec["pixels"] = rec["pixels"].astype(np.int64)
    return image, trans, rec


def forward_stats(splats, cams, targets=None, threads=1):
    """forward_stats (rasterizer.py:311-352).  Returns
    (importance, camera_importance, delta_mse or None, mse or None)."""
    n, pos, sh, op, sc, rot = _splat_arrays(splats)
    S = len(cams)
    imp = np.empty(n)
    cam_imp = np.empty((S, n))
    dm = np.empty(n) if targets is not None else None
    mse = ctypes.c_double(0.0)
    tptr = None
    keep = None
    if targets is not None:
        keep = [_f64(t, (int(cams[s].height), int(cams[s].width), 3)) for s, t in enumerate(targets)]
        tptr = (ctypes.c_void_p * S)(*[t.ctypes.data for t in keep])
    _check(lib().oracle_forward_stats(ctypes.c_int64(n), _p(pos), _p(sh), _p(op), _p(sc), _p(rot),
                                      ctypes.c_int(S), _cams(cams), tptr, ctypes.c_int(threads),
                                      _p(imp), _p(cam_imp), _p(dm), ctypes.byref(mse)),
           "forward_stats")
    return imp, cam_imp, dm, (mse.value if targets is not None else None)


def tile_lists(splats, cam, tile_w=8, tile_h=4):
    """Per-tile splat lists in (tile, depth, id) order, restated from the
    reference's clipped bbox (rasterizer.py:135-151) and stable depth order
    (:248-250).  Returns (offsets (ntiles+1,), splat ids)."""
    n, pos, sh, op, sc, rot = _splat_arrays(splats)
    tw = (int(cam.width) + tile_w - 1) // tile_w
    th = (int(cam.height) + tile_h - 1) // tile_h
    offsets = np.empty(tw * th + 1, dtype=np.int64)
    total = ctypes.c_int64(0)
    c = _cam(cam)
    L = lib()
    _check(L.oracle_tile_lists(ctypes.c_int64(n), _p(pos), _p(sc), _p(rot), ctypes.byref(c),
                               ctypes.c_int(tile_w), ctypes.c_int(tile_h), _p(offsets), None, ctypes.c_int64(0),
                               ctypes.byref(total)), "tile_lists")
    ids = np.empty(max(total.value, 1), dtype=np.int32)
    _check(L.oracle_tile_lists(ctypes.c_int64(n), _p(pos), _p(sc), _p(rot), ctypes.byref(c),
                               ctypes.c_int(tile_w), ctypes.c_int(tile_h), _p(offsets), _p(ids), ctypes.c_int64(total.value),
                               ctypes.byref(total)), "tile_lists")
    return offsets, ids[:total.value].copy()


def compact(splats, cams, camera_importance, lambda_y, parallel_threshold, zero_threshold,
            threads=1):
    """compact_scene (compaction.py:195-243).  Returns (rgb (N,3,16),
    ycocg (N,3,16), status int8 (N,): 0 ok, 1 jitter, 2 failed, 3 DC fallback)."""
    n, pos, sh, op, sc, rot = _splat_arrays(splats)
    S = len(cams)
    ci = _f64(camera_importance, (S, n))
    rgb = np.empty((n, 3, 16))
    yc = np.empty((n, 3, 16))
    status = np.empty(n, dtype=np.int8)
    _check(lib().oracle_compact(ctypes.c_int64(n), _p(pos), _p(sh), ctypes.c_int(S), _cams(cams),
                                _p(ci), ctypes.c_double(lambda_y),
                                ctypes.c_double(parallel_threshold),
                                ctypes.c_double(zero_threshold), ctypes.c_int(threads), _p(rgb),
                                _p(yc), _p(status)), "compact")
    return rgb, yc, status


def num_threads():
    return int(lib().oracle_num_threads())
