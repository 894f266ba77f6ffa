"""Codec back end with its data-parallel parts on the device (SURVEY.md 8f
row 4; reference: potr/quantize.py, potr/bitstream.py, potr/varint.py).

encode_container keeps the reference's signature and output bytes: the
camera-adaptive octree is built and serialised by potr_octree
(csrc/codec.cu), the 55 quantised attribute streams by
potr_attribute_streams, and only the header packing and the zstd frame
(libzstd, for byte identity) run on the host.  The reference builds the
octree by Python recursion (96 s for 300k splats on one core); here it is a
few sorts and scans.

Host-side pieces kept in numpy because their rounding is numpy's: the root
cube (_root_cube, quantize.py:79-89), log(scales) and the RGB -> YCoCg
coefficient transform (compaction.py:80-82).
"""

import ctypes
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from . import device as D
from . import _zstd

DEFAULT_MAX_DEPTH = 24
MAGIC = b"POTR"
VERSION = 1
NUM_STREAMS = 56
_HEADER_FMT = "<4sBI11fBB" + f"{NUM_STREAMS}I"
HEADER_SIZE = struct.calcsize(_HEADER_FMT)


@dataclass
class QuantParams:
    """quantize.py:26-36."""
    sf_sh: float
    sf_opacity: float
    sf_rotation: float
    sf_scale: float

    def __post_init__(self):
        for name in ("sf_sh", "sf_opacity", "sf_rotation", "sf_scale"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")


def root_cube(positions):
    """_root_cube (quantize.py:79-89): the AABB centre rounded to float32 and
    the max |p - centre| rounded outward to float32."""
    positions = np.asarray(positions, dtype=np.float64)
    lo = positions.min(axis=0)
    hi = positions.max(axis=0)
    center = np.float64(np.asarray((lo + hi) * 0.5, dtype=np.float32))
    half_needed = float(np.abs(positions - center).max()) if len(positions) else 0.0
    half = np.float32(half_needed)
    if np.float64(half) < half_needed:
        half = np.nextafter(half, np.float32(np.inf), dtype=np.float32)
    return center, float(np.float64(half))


def octree_stream(positions, camera_eyes, beta, gamma, max_depth=DEFAULT_MAX_DEPTH,
                  root_cube_=None):
    """serialize_octree(build_octree(...)) (quantize.py:98-170) on the device.
    Returns (stream bytes, DFS order (int64, original indices), centre (3,),
    half)."""
    positions = np.asarray(positions, dtype=np.float64)
    if positions.ndim != 2 or positions.shape[0] < 1:
        raise ValueError("need at least one position")
    if gamma <= 0 or beta < 0:
        raise ValueError("gamma must be > 0 and beta >= 0")
    if root_cube_ is None:
        center, half = root_cube(positions)
    else:
        center = np.float64(np.asarray(root_cube_[0], dtype=np.float32))
        half = float(np.float64(np.float32(root_cube_[1])))
    n = positions.shape[0]
    dev = D.current_device()
    pos = D.to_device(positions, dev, (n, 3))
    eyes = np.ascontiguousarray(np.asarray(camera_eyes, dtype=np.float64).reshape(-1, 3))
    cap = n * (max_depth + 6)
    out = torch.empty(max(cap, 1), dtype=torch.uint8, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    ln = ctypes.c_int64(0)
    c = (ctypes.c_double * 3)(*[float(x) for x in center])
    D.context().call("potr_octree", ctypes.c_int64(n), D.ptr(pos), int(eyes.shape[0]),
                     eyes.ctypes.data_as(ctypes.c_void_p) if len(eyes) else None,
                     ctypes.c_double(beta), ctypes.c_double(gamma), c, ctypes.c_double(half),
                     int(max_depth), D.ptr(out), ctypes.c_int64(cap), ctypes.byref(ln),
                     D.ptr(order))
    return (D.to_host(out[:ln.value]).tobytes(), D.to_host(order), np.asarray(center), half)


def _attribute_streams_device(splats, params, order_dev, sh_ycocg):
    from .compaction import coeffs_rgb_to_ycocg
    n = len(splats.positions)
    dev = D.current_device()
    yc = coeffs_rgb_to_ycocg(splats.sh) if sh_ycocg is None else sh_ycocg
    yc_d = D.to_device(yc, dev, (n, 3, 16))
    op_d = D.to_device(splats.opacities, dev, (n,))
    ls_d = D.to_device(np.log(np.asarray(splats.scales, dtype=np.float64)), dev, (n, 3))
    rot_d = D.to_device(splats.rotations, dev, (n, 4))
    cap = 550 * n
    out = torch.empty(max(cap, 1), dtype=torch.uint8, device=dev)
    lens = (ctypes.c_int64 * 55)()
    D.context().call("potr_attribute_streams", ctypes.c_int64(n), D.ptr(order_dev), D.ptr(yc_d),
                     D.ptr(op_d), D.ptr(ls_d), D.ptr(rot_d), ctypes.c_double(params.sf_sh),
                     ctypes.c_double(params.sf_opacity), ctypes.c_double(params.sf_rotation),
                     ctypes.c_double(params.sf_scale), D.ptr(out), ctypes.c_int64(cap), lens)
    total = int(sum(lens))
    return D.to_host(out[:total]), list(lens)


def _split(blob, lens):
    streams, pos = [], 0
    for L in lens:
        streams.append(blob[pos:pos + L].tobytes())
        pos += L
    return streams


def encode_attribute_streams(splats, params: QuantParams, sh_ycocg=None):
    """bitstream.py:116-155 for splats already in octree DFS order: the 55
    non-octree streams."""
    n = len(splats.positions)
    if n == 0:
        return [b""] * (NUM_STREAMS - 1)
    order = torch.arange(n, dtype=torch.int64, device=D.current_device())
    return _split(*_attribute_streams_device(splats, params, order, sh_ycocg))


def pack_header(splat_count, q, params, beta, gamma, root_center, root_half, max_depth,
                zstd_level, stream_lengths):
    """ContainerHeader.pack (bitstream.py:77-85)."""
    return struct.pack(_HEADER_FMT, MAGIC, VERSION, splat_count, q, params.sf_sh,
                       params.sf_opacity, params.sf_rotation, params.sf_scale, beta, gamma,
                       float(root_center[0]), float(root_center[1]), float(root_center[2]),
                       root_half, max_depth, zstd_level, *stream_lengths)


def encode_container(splats, params: QuantParams, q, beta, gamma, zstd_level=19,
                     max_depth=DEFAULT_MAX_DEPTH, root_cube=None, sh_ycocg=None, camera_eyes=()):
    """bitstream.py:232-259: octree the positions, quantise and serialise every
    attribute in DFS order, compress.  Returns (container bytes, DFS order)."""
    n = len(splats.positions)
    if n == 0:
        streams = [b""] * NUM_STREAMS
        header = pack_header(0, q, params, beta, gamma, np.zeros(3), 0.0, max_depth,
                             zstd_level, [0] * NUM_STREAMS)
        return header + _zstd.compress(b"", zstd_level), np.empty(0, dtype=np.int64)
    octree, order, center, half = octree_stream(splats.positions, camera_eyes, beta, gamma,
                                                max_depth=max_depth, root_cube_=root_cube)
    order_dev = torch.from_numpy(np.ascontiguousarray(order)).to(D.current_device())
    # the attribute streams come back as one blob in stream order: the
    # payload is the octree stream followed by it
    blob, lens = _attribute_streams_device(splats, params, order_dev, sh_ycocg)
    header = pack_header(n, q, params, beta, gamma, center, half, max_depth, zstd_level,
                         [len(octree)] + lens)
    payload = np.concatenate([np.frombuffer(octree, dtype=np.uint8), blob])
    return header + _zstd.compress(payload, zstd_level), order


# ---------------------------------------------------------------------------
# Decode side (bitstream.py:53-112, :169-247, :278-292; quantize.py:173-226)

STREAM_OCTREE = 0
STREAM_DC = (1, 2, 3)
STREAM_AC0 = 4
STREAM_OPACITY = 49
STREAM_SCALE = (50, 51, 52)
STREAM_ROTATION = (53, 54, 55)
# bitstream.py:37-50
PROPERTY_STREAMS = {
    "position": [STREAM_OCTREE],
    "scale": list(STREAM_SCALE),
    "opacity": [STREAM_OPACITY],
    "rotation": list(STREAM_ROTATION),
    "dc_sh": list(STREAM_DC),
    "ac_sh": list(range(STREAM_AC0, STREAM_AC0 + 45)),
}
UNCOMPRESSED_BYTES_PER_SPLAT = {
    "position": 12, "scale": 12, "opacity": 4, "rotation": 16, "dc_sh": 12, "ac_sh": 180,
}
_CLAMP_WARN = "quaternions outside the unit ball, clamped"


class ContainerError(ValueError):
    pass


class UnsupportedFormatError(ContainerError):
    pass


class IntegrityError(ContainerError):
    pass


class OctreeError(ValueError):
    pass


@dataclass
class ContainerHeader:
    """bitstream.py:66-106 (fields and unpack)."""
    splat_count: int
    q: float
    params: QuantParams
    beta: float
    gamma: float
    root_center: np.ndarray
    root_half: float
    max_depth: int = DEFAULT_MAX_DEPTH
    zstd_level: int = 19
    stream_lengths: list = None

    def pack(self) -> bytes:
        return pack_header(self.splat_count, self.q, self.params, self.beta, self.gamma,
                           self.root_center, self.root_half, self.max_depth, self.zstd_level,
                           self.stream_lengths or [0] * NUM_STREAMS)

    @classmethod
    def unpack(cls, data: bytes):
        if len(data) < HEADER_SIZE:
            raise IntegrityError("file shorter than the container header")
        fields = struct.unpack_from(_HEADER_FMT, data)
        if fields[0] != MAGIC:
            raise UnsupportedFormatError("bad magic, not a POTR container")
        if fields[1] != VERSION:
            raise UnsupportedFormatError(f"unsupported container version {fields[1]}")
        (_, _, count, q, sf_sh, sf_op, sf_rot, sf_sc, beta, gamma,
         cx, cy, cz, half, max_depth, level) = fields[:16]
        return cls(splat_count=count, q=q, params=QuantParams(sf_sh, sf_op, sf_rot, sf_sc),
                   beta=beta, gamma=gamma, root_center=np.array([cx, cy, cz], dtype=np.float64),
                   root_half=float(half), max_depth=max_depth, zstd_level=level,
                   stream_lengths=list(fields[16:]))


def write_container(header, streams, zstd_level=None) -> bytes:
    """bitstream.py:226-232: the header (its stream lengths and, if given, its
    level updated) followed by one zstd frame over the streams."""
    if zstd_level is not None:
        header.zstd_level = zstd_level
    header.stream_lengths = [len(s) for s in streams]
    return header.pack() + _zstd.compress(b"".join(streams), header.zstd_level)


def size_report(data: bytes):
    """bitstream.py:300-315: per-property compressed bytes, by ablating each
    property's streams and re-compressing at the container's level.  The six
    re-compressions are independent: they run on host threads (libzstd
    releases the GIL through ctypes); each is the same one-shot compress, so
    the report is the reference's."""
    from concurrent.futures import ThreadPoolExecutor
    header, streams = read_container(data)
    payload_size = len(data) - HEADER_SIZE

    def ablated_size(indices):
        keep = b"".join(s for i, s in enumerate(streams) if i not in indices)
        return len(_zstd.compress(keep, header.zstd_level))

    props = list(PROPERTY_STREAMS.items())
    with ThreadPoolExecutor(max_workers=len(props)) as pool:
        sizes = list(pool.map(lambda kv: ablated_size(kv[1]), props))
    return {
        "payload_bytes": payload_size,
        "header_bytes": HEADER_SIZE,
        "splat_count": header.splat_count,
        "property_bytes": {k: payload_size - a for (k, _), a in zip(props, sizes)},
    }


def _read_payload(data):
    header = ContainerHeader.unpack(data)
    expected = sum(header.stream_lengths)
    try:
        payload = _zstd.decompress(bytes(data[HEADER_SIZE:]), expected)
    except _zstd.ZstdError as e:
        raise IntegrityError(str(e)) from e
    return header, payload


def read_container(data: bytes):
    """bitstream.py:235-247: the header and the 56 streams (host zstd)."""
    header, payload = _read_payload(data)
    streams = []
    pos = 0
    for length in header.stream_lengths:
        streams.append(payload[pos:pos + length])
        pos += length
    return header, streams


@dataclass
class DecodedOctree:
    """quantize.py:173-177 without the Python node tree (positions and depths
    are what decode_container consumes)."""
    positions: np.ndarray
    depths: np.ndarray
    tree: object = None


def _octree_call(data, center, half, max_depth, capacity):
    ctx = D.context()
    buf = data if isinstance(data, np.ndarray) else np.frombuffer(bytes(data), dtype=np.uint8)
    c = np.ascontiguousarray(center, dtype=np.float64)
    pos = np.empty((max(capacity, 1), 3), dtype=np.float64)
    dep = np.empty(max(capacity, 1), dtype=np.int32)
    cnt = ctypes.c_int64(0)
    try:
        ctx.call("potr_octree_decode", buf.ctypes.data_as(ctypes.c_void_p) if buf.size else None,
                 ctypes.c_int64(buf.size), c.ctypes.data_as(ctypes.c_void_p), ctypes.c_double(half),
                 int(max_depth), ctypes.c_int64(capacity), pos.ctypes.data_as(ctypes.c_void_p),
                 dep.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt))
    except (ValueError, _native.PotrError) as e:
        if "octree: " not in str(e):
            raise
        raise OctreeError(str(e).split("octree: ", 1)[1]) from None
    return pos, dep, int(cnt.value)


def deserialize_octree(data: bytes, center, half, max_depth=DEFAULT_MAX_DEPTH, expected=None):
    """quantize.py:180-226: leaf centres (repeated per count) and depths in
    DFS order (libpotr_b200 potr_octree_decode: a preorder stream's node
    boundaries are only known by parsing it, so this walk runs on the host).
    expected: the splat count to size the output for (a container header's);
    a stream holding more is walked a second time."""
    center = np.float64(np.asarray(center, dtype=np.float32))
    half = float(np.float64(np.float32(half)))
    cap = 0 if expected is None else max(int(expected), 0)
    pos, dep, count = _octree_call(data, center, half, max_depth, cap)
    if count > cap:
        pos, dep, count = _octree_call(data, center, half, max_depth, count)
    return DecodedOctree(positions=pos[:count], depths=dep[:count].astype(np.int64))


def decode_attribute_streams(streams, header: ContainerHeader, positions):
    """bitstream.py:169-220 on the GPU (potr_attribute_decode): the scene in
    DFS order with RGB coefficients; streams is the full 56-stream list."""
    attr = streams[1:]
    lengths = np.array([len(s) for s in attr], dtype=np.int64)
    blob = np.frombuffer(b"".join(bytes(s) for s in attr), dtype=np.uint8)
    return _decode_attributes(blob, lengths, header, positions)


def _decode_attributes(blob, lengths, header, positions):
    """The 55 attribute streams, back to back in `blob` (uint8), lengths[i]
    bytes each."""
    import warnings
    from .scene import Splats
    n = header.splat_count
    p = header.params
    dev = D.current_device()
    sh = torch.empty((n, 3, 16), dtype=torch.float64, device=dev)
    opac = torch.empty(n, dtype=torch.float64, device=dev)
    scales = torch.empty((n, 3), dtype=torch.float64, device=dev)
    rot = torch.empty((n, 4), dtype=torch.float64, device=dev)
    clamped = ctypes.c_int64(0)
    try:
        D.context().call("potr_attribute_decode", ctypes.c_int64(n),
                         blob.ctypes.data_as(ctypes.c_void_p) if blob.size else
                         ctypes.c_void_p(lengths.ctypes.data),
                         lengths.ctypes.data_as(ctypes.c_void_p), ctypes.c_double(p.sf_sh),
                         ctypes.c_double(p.sf_opacity), ctypes.c_double(p.sf_rotation),
                         ctypes.c_double(p.sf_scale), D.ptr(sh), D.ptr(opac), D.ptr(scales),
                         D.ptr(rot), ctypes.byref(clamped))
    except (ValueError, _native.PotrError) as e:
        msg = str(e)
        if "integrity: " in msg:
            raise IntegrityError(msg.split("integrity: ", 1)[1]) from None
        if "varint: " in msg:
            raise ValueError(msg.split("varint: ", 1)[1]) from None
        raise
    if clamped.value:
        warnings.warn(f"{int(clamped.value)} {_CLAMP_WARN}", RuntimeWarning)
    return Splats(positions=np.asarray(positions, dtype=np.float64).reshape(n, 3),
                  sh=D.to_host(sh), opacities=D.to_host(opac), scales=D.to_host(scales),
                  rotations=D.to_host(rot))


def decode_container(data: bytes):
    """bitstream.py:278-292: (splats in DFS order, header)."""
    from .scene import Splats
    header, payload = _read_payload(data)  # one buffer: streams are views into it
    if header.splat_count == 0:
        empty = Splats(np.empty((0, 3)), np.empty((0, 3, 16)), np.empty(0),
                       np.empty((0, 3)), np.empty((0, 4)))
        return empty, header
    L0 = header.stream_lengths[STREAM_OCTREE]
    buf = np.frombuffer(payload, dtype=np.uint8)
    # the header's count sizes the walk's output, bounded by the payload (a
    # valid container spends at least one byte per splat in each attribute
    # stream), so a corrupted count cannot demand a huge allocation
    decoded = deserialize_octree(buf[:L0], header.root_center, header.root_half,
                                 header.max_depth, min(header.splat_count, len(payload)))
    if decoded.positions.shape[0] != header.splat_count:
        raise IntegrityError(
            f"octree stream decodes {decoded.positions.shape[0]} splats, "
            f"header says {header.splat_count}")
    lengths = np.array(header.stream_lengths[1:], dtype=np.int64)
    splats = _decode_attributes(buf[L0:], lengths, header, decoded.positions)
    return splats, header
