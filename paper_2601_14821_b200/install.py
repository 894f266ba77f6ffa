"""Rebind the reference package (potr) to the B200 implementations.

The reference binds names at import time, so patching
potr.rasterizer alone would miss potr.pruning's `compute_delta_mse`,
potr.pipeline's `compute_importance` / `render_targets` / `compact_scene`,
and so on.  install() rebinds every import site listed below and returns an
uninstall callable.
"""

import importlib

from . import codec as _codec
from . import compaction as _comp
from . import metrics as _met
from . import rasterizer as _rast

PATCH_SET = {
    "potr.rasterizer": {
        "forward_stats": _rast.forward_stats,
        "compute_delta_mse": _rast.compute_delta_mse,
        "compute_importance": _rast.compute_importance,
        "render_targets": _rast.render_targets,
        "render_image": _rast.render_image,
        "render_with_records": _rast.render_with_records,
        "project_splats": _rast.project_splats,
        "splat_colors": _rast.splat_colors,
    },
    "potr.pruning": {"compute_delta_mse": _rast.compute_delta_mse},
    "potr.pipeline": {
        "compute_importance": _rast.compute_importance,
        "render_targets": _rast.render_targets,
        "compact_scene": _comp.compact_scene,
        "encode_container": _codec.encode_container,
        "decode_container": "decode_container",
    },
    "potr.bitstream": {
        "encode_container": _codec.encode_container,
        "decode_container": "decode_container",
    },
    "potr.cli": {
        "compute_importance": _rast.compute_importance,
        "render_targets": _rast.render_targets,
    },
    "potr.compaction": {
        "render_image": _rast.render_image,
        "compact_scene": _comp.compact_scene,
    },
    "potr.metrics": {
        "render_image": _rast.render_image,
        "ssim": _met.ssim,
        "compare_renders": _met.compare_renders,
        "compute_metrics": _met.compute_metrics,
    },
}


def _decode_container_raising_reference_errors():
    """codec.decode_container, re-raising the reference's own exception
    classes (bitstream.py:53-62, quantize.py:22) so callers that catch
    potr.bitstream.IntegrityError and friends keep working."""
    ref_bs = importlib.import_module("potr.bitstream")
    ref_q = importlib.import_module("potr.quantize")

    def decode_container(data):
        try:
            return _codec.decode_container(data)
        except _codec.OctreeError as e:
            raise ref_q.OctreeError(str(e)) from None
        except _codec.ContainerError as e:
            raise getattr(ref_bs, type(e).__name__)(str(e)) from None

    decode_container.__doc__ = _codec.decode_container.__doc__
    return decode_container


_FACTORIES = {"decode_container": _decode_container_raising_reference_errors}


def install(modules=None):
    """Patch the reference modules in place; returns uninstall()."""
    saved = []
    made = {}
    for modname, names in PATCH_SET.items():
        if modules is not None and modname not in modules:
            continue
        try:
            mod = importlib.import_module(modname)
        except ImportError:
            continue
        for name, fn in names.items():
            if hasattr(mod, name):
                if isinstance(fn, str):
                    if fn not in made:
                        made[fn] = _FACTORIES[fn]()
                    fn = made[fn]
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, fn)

    def uninstall():
        for mod, name, old in reversed(saved):
            setattr(mod, name, old)

    return uninstall
