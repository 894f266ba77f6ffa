"""ctypes binding of libpotr_b200.so (include/potr_b200.h).

There is no CPU fallback: if the library is missing, or no CUDA device is
present, every entry point raises.  The build is in-tree
(paper_2601_14821_b200/_lib/libpotr_b200.so, see build.py).
"""

import ctypes
import os
import threading

import numpy as np

from . import build as _build

POTR_OK = 0
POTR_E_ARG = -1
POTR_E_CUDA = -2
POTR_E_NOMEM = -3
POTR_E_CAPACITY = -4
NEQ_STRIDE = 185
OPT_VIEW_BATCH = 1
OPT_RAW_DEPTH_KEYS = 2
OPT_TILE_CULL = 3
OPT_SPATIAL_RECORDS = 4
OPT_LOOKAHEAD = 5
STAGES = ["preprocess", "depth_sort", "scan", "duplicate", "tile_sort", "raster", "reduce",
          "sh_accumulate", "sh_solve"]

c_double_p = ctypes.POINTER(ctypes.c_double)


class PotrCamera(ctypes.Structure):
    """potr_camera (scene.py:64-77 Camera)."""
    _fields_ = [("eye", ctypes.c_double * 3), ("rot", ctypes.c_double * 9),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class PotrSplats(ctypes.Structure):
    """potr_splats (scene.py:42-61 Splats), device pointers."""
    _fields_ = [("n", ctypes.c_int64), ("positions", ctypes.c_void_p), ("sh", ctypes.c_void_p),
                ("opacities", ctypes.c_void_p), ("scales", ctypes.c_void_p),
                ("rotations", ctypes.c_void_p)]


class PotrError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


_lib = None
_lock = threading.Lock()

# Every exported symbol of include/potr_b200.h, with its ctypes signature.
_SIGNATURES = {
    "potr_abi_version": (ctypes.c_int, []),
    "potr_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "potr_destroy": (None, [ctypes.c_void_p]),
    "potr_set_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "potr_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "potr_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "potr_kernel_launches": (ctypes.c_int64, [ctypes.c_void_p]),
    "potr_forward_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats), ctypes.c_int,
                                          ctypes.POINTER(PotrCamera), ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "potr_score_views": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats), ctypes.c_int,
                                        ctypes.POINTER(PotrCamera), ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]),
    "potr_score_views_rows": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                             ctypes.c_int, ctypes.POINTER(PotrCamera),
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p]),
    "potr_score_views_self": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                             ctypes.c_int, ctypes.POINTER(PotrCamera),
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p]),
    "potr_finalize_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "potr_copy_to_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int64]),
    "potr_upload_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_int64]),
    "potr_upload_wait": (ctypes.c_int, [ctypes.c_void_p]),
    "potr_removal_order": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_void_p]),
    "potr_sort_pairs_u64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "potr_render": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                   ctypes.POINTER(PotrCamera), ctypes.c_void_p, ctypes.c_void_p]),
    "potr_render_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats), ctypes.c_int,
                                         ctypes.POINTER(PotrCamera), ctypes.c_void_p,
                                         ctypes.c_void_p]),
    "potr_render_records": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                           ctypes.POINTER(PotrCamera), ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "potr_project": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                    ctypes.POINTER(PotrCamera), ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p]),
    "potr_bin": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                ctypes.POINTER(PotrCamera), ctypes.c_void_p,
                                ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "potr_compact": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats), ctypes.c_int,
                                    ctypes.POINTER(PotrCamera), ctypes.c_void_p, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p]),
    "potr_sh_accumulate": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                          ctypes.c_int, ctypes.POINTER(PotrCamera),
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "potr_sh_normal_equations": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats),
                                                ctypes.c_int, ctypes.POINTER(PotrCamera),
                                                ctypes.c_void_p, ctypes.c_void_p]),
    "potr_sh_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PotrSplats), ctypes.c_void_p,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "potr_octree_decode": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "potr_attribute_decode": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p]),
    "potr_set_option": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "potr_profile_enable": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "potr_profile_read": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "potr_counters_enable": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "potr_counters_read": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "potr_octree": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p]),
    "potr_attribute_streams": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
                                              ctypes.c_int64, ctypes.c_void_p]),
    "potr_image_compare": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "potr_forward_stats_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_int,
                                               ctypes.POINTER(PotrCamera), ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p]),
    "potr_compact_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(PotrCamera),
                                         ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]),
}


def library_path():
    # POTR_B200_LIB: load an alternative in-tree build (A/B experiments)
    return os.environ.get("POTR_B200_LIB", _build.LIB)


def load(build_if_missing=True):
    """Load (building in-tree first if needed) and return the ctypes CDLL."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if path == _build.LIB and build_if_missing and (not os.path.exists(path) or
                                                        _build.needs_build()):
            _build.build()
        if not os.path.exists(path):
            raise ImportError(f"libpotr_b200.so not found at {path}; run "
                              "`python -m paper_2601_14821_b200.build`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.potr_abi_version() != 1:
            raise ImportError("libpotr_b200.so ABI version mismatch")
        _lib = lib
        return lib


def exported_symbols():
    return sorted(_SIGNATURES)


def camera_struct(cam):
    c = PotrCamera()
    c.eye[:] = [float(v) for v in np.asarray(cam.eye, dtype=np.float64).reshape(3)]
    c.rot[:] = [float(v) for v in np.asarray(cam.rotation, dtype=np.float64).reshape(9)]
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def camera_array(cams):
    arr = (PotrCamera * max(1, len(cams)))()
    for i, cam in enumerate(cams):
        arr[i] = camera_struct(cam)
    return arr


class Context:
    """One potr_ctx bound to a CUDA device, ordered on torch's current stream."""

    def __init__(self, device_index):
        self.lib = load()
        self.device_index = int(device_index)
        h = ctypes.c_void_p()
        rc = self.lib.potr_create(self.device_index, ctypes.byref(h))
        if rc != POTR_OK:
            raise PotrError(f"potr_create(device={device_index}) failed ({rc}): "
                            "no usable CUDA device")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and self.lib is not None:
            try:
                self.lib.potr_destroy(h)
            except Exception:
                pass
            self.handle = None

    def set_stream(self, stream_handle):
        self.check(self.lib.potr_set_stream(self.handle, ctypes.c_void_p(stream_handle)),
                   "potr_set_stream")

    def check(self, rc, what):
        if rc == POTR_OK:
            return
        msg = self.lib.potr_last_error(self.handle)
        msg = msg.decode() if msg else ""
        if rc == POTR_E_ARG:
            raise ValueError(f"{what}: {msg}")
        if rc == POTR_E_NOMEM:
            raise MemoryError(f"{what}: {msg}")
        raise PotrError(f"{what} failed ({rc}): {msg}")

    def call(self, name, *args):
        self.check(getattr(self.lib, name)(self.handle, *args), name)

    def launches(self):
        return int(self.lib.potr_kernel_launches(self.handle))

    def profile(self, enable=True):
        """Start (reset) or stop live per-stage CUDA-event timing."""
        self.call("potr_profile_enable", int(bool(enable)))

    def profile_read(self):
        """{stage: (total ms, launches)} since profile() (synchronizes)."""
        ms = (ctypes.c_double * len(STAGES))()
        cnt = (ctypes.c_int64 * len(STAGES))()
        self.call("potr_profile_read", ctypes.cast(ms, ctypes.c_void_p),
                  ctypes.cast(cnt, ctypes.c_void_p))
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(STAGES)}

    def counters(self, enable=True):
        self.call("potr_counters_enable", int(bool(enable)))

    def counters_read(self):
        """(E bbox evaluations, live evaluations, contributions M, pairs K)."""
        out = (ctypes.c_uint64 * 4)()
        self.call("potr_counters_read", ctypes.cast(out, ctypes.c_void_p))
        return tuple(int(v) for v in out)
