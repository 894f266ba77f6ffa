"""Tile-binning evidence (kernel (b)): the GPU's global depth order and its
per-tile splat lists, for parity against the reference-derived lists.

depth_order == ids[np.argsort(view_depth[ids], kind="stable")] of
rasterizer.py:248-250; tile lists are the 8x4-pixel tiles each splat's clipped
bbox (rasterizer.py:135-151) touches, in (tile, depth, id) order.
"""

import ctypes

import numpy as np
import torch

from . import _native
from . import device as D

TILE_W, TILE_H = 8, 4  # csrc/common.cuh kTileW x kTileH


def tile_lists(splats, camera):
    """Returns (depth order of valid splats, tile offsets (ntiles+1,),
    concatenated per-tile splat ids) from the GPU binning."""
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n = ds.n
    cam = _native.camera_struct(camera)
    tw = (int(camera.width) + TILE_W - 1) // TILE_W
    th = (int(camera.height) + TILE_H - 1) // TILE_H
    order = D.empty(max(n, 1), dev, torch.int64)
    offsets = D.empty(tw * th + 1, dev, torch.int64)
    nv = ctypes.c_int64(0)
    K = ctypes.c_int64(0)
    ctx.call("potr_bin", ctypes.byref(ds.struct()), ctypes.byref(cam), D.ptr(order),
             ctypes.byref(nv), D.ptr(offsets), None, ctypes.c_int64(0), ctypes.byref(K))
    lists = D.empty(max(K.value, 1), dev, torch.int32)
    ctx.call("potr_bin", ctypes.byref(ds.struct()), ctypes.byref(cam), D.ptr(order),
             ctypes.byref(nv), D.ptr(offsets), D.ptr(lists), ctypes.c_int64(max(K.value, 1)),
             ctypes.byref(K))
    return (order[:nv.value].cpu().numpy(), offsets.cpu().numpy(),
            lists[:K.value].cpu().numpy().astype(np.int64))


def depth_order(splats, camera):
    return tile_lists(splats, camera)[0]
