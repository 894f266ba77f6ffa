"""Device residency: HBM copies of splats and targets, one potr context per GPU.

PyTorch is the plumbing here -- device allocations, pinned staging and the
current CUDA stream -- and every tensor is handed to the C ABI as a raw
pointer.  There is no CPU path: without a CUDA device these raise.
"""

import ctypes
import warnings

import numpy as np
import torch

from . import _native

_contexts = {}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2601_14821_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")


def current_device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def context(device=None):
    """The potr context of `device` (default: current), bound to torch's
    current stream on that device."""
    dev = current_device() if device is None else torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    ctx = _contexts.get(idx)
    if ctx is None:
        ctx = _native.Context(idx)
        _contexts[idx] = ctx
    ctx.set_stream(torch.cuda.current_stream(idx).cuda_stream)
    return ctx


def ptr(t):
    """Raw device pointer of a tensor (None for an absent tensor)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def to_device(arr, device, shape=None):
    """float64 C-contiguous device copy of a host array (or tensor)."""
    if isinstance(arr, torch.Tensor):
        t = arr.to(device=device, dtype=torch.float64)
        return t.contiguous() if shape is None else t.reshape(shape).contiguous()
    a = np.ascontiguousarray(arr, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    if a.size == 0:
        return torch.empty(a.shape, dtype=torch.float64, device=device)
    with warnings.catch_warnings():
        # read-only inputs (the reference freezes its targets) are only read here
        warnings.simplefilter("ignore", UserWarning)
        src = torch.from_numpy(a)
        if a.nbytes >= _STAGED_MIN and not src.is_pinned():
            # pageable (the reference's own arrays): the library's staged
            # upload, host threads filling a pinned ring under the DMA
            dst = torch.empty(a.shape, dtype=torch.float64, device=device)
            context(device).call("potr_copy_to_device", ptr(dst), ctypes.c_void_p(a.ctypes.data),
                                 ctypes.c_int64(a.nbytes))
            return dst
        return src.to(device, non_blocking=False)


_STAGED_MIN = 8 << 20          # pageable sources from this size use potr_copy_to_device
_ASYNC_GEOMETRY_MIN = 32 << 20  # geometry arrays from this size are queued (potr_upload_async)


_PINNED_MAX = 256 << 20        # results up to this size land in pinned memory directly
_STAGE_BYTES = 64 << 20        # larger ones stream through one pinned staging buffer
_stage = None


def to_host(t):
    """Device tensor -> fresh numpy array, through pinned memory.

    A pageable destination makes the driver stage the copy at ~2 GB/s (22 ms
    for forward_stats' 48 MB at C3, 2.4 s for 200 targets); pinned memory
    takes the DMA at PCIe speed.  Results up to 256 MB are returned as views
    of a pinned tensor (torch's caching host allocator recycles it once the
    array is dropped); larger ones are copied through a 64 MB pinned buffer."""
    global _stage
    t = t.detach().contiguous()
    nbytes = t.numel() * t.element_size()
    if not t.is_cuda or nbytes == 0:
        return t.cpu().numpy()
    if nbytes <= _PINNED_MAX:
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t)
        return out.numpy()
    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    if _stage is None:
        _stage = torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True)
    src = t.reshape(-1).view(torch.uint8)
    dst = out.reshape(-1).view(np.uint8)
    stage_np = _stage.numpy()
    for off in range(0, nbytes, _STAGE_BYTES):
        m = min(_STAGE_BYTES, nbytes - off)
        _stage[:m].copy_(src[off:off + m])
        dst[off:off + m] = stage_np[:m]
    return out


def empty(shape, device, dtype=torch.float64):
    """Device buffer; never zero-sized (the C ABI wants a real pointer)."""
    t = torch.empty(shape, dtype=dtype, device=device)
    if t.numel() == 0:
        return torch.empty(max(1, t.numel()), dtype=dtype, device=device)[:0].reshape(shape)
    return t


class DeviceSplats:
    """Splat attributes resident in HBM, float64 in the reference layouts."""

    def __init__(self, positions, sh, opacities, scales, rotations):
        self.positions = positions
        self.sh = sh
        self.opacities = opacities
        self.scales = scales
        self.rotations = rotations
        self.n = int(positions.shape[0])
        self.device = positions.device
        # keep 1-element backing storage for n == 0 so pointers stay valid
        self._keep = [torch.empty(64, dtype=torch.float64, device=self.device)]

    @classmethod
    def from_host(cls, splats, device=None, async_sh=False):
        """Upload host splats.  async_sh: the five arrays are queued on the
        library's upload worker (potr_upload_async), the SH rows (81% of the
        bytes) last -- the next scoring call waits only for the geometry and
        bins its first view batches while the rows arrive; every other library
        call waits for all of them first.  The host arrays are kept referenced
        until the copies are complete."""
        if isinstance(splats, DeviceSplats):
            return splats
        dev = current_device() if device is None else torch.device(device)
        n = int(np.asarray(splats.positions).shape[0]) if not isinstance(
            splats.positions, torch.Tensor) else int(splats.positions.shape[0])
        fields = (("positions", (n, 3)), ("opacities", (n,)), ("scales", (n, 3)),
                  ("rotations", (n, 4)), ("sh", (n, 3, 16)))
        host = {f: getattr(splats, f) for f, _ in fields}
        if async_sh and not any(isinstance(a, torch.Tensor) for a in host.values()):
            arrs = {f: np.ascontiguousarray(host[f], dtype=np.float64).reshape(shape)
                    for f, shape in fields}
            if arrs["sh"].nbytes >= _STAGED_MIN:
                ctx = context(dev)
                out = {}
                for f, shape in fields:
                    a = arrs[f]
                    if f != "sh" and a.nbytes < _ASYNC_GEOMETRY_MIN:
                        # small geometry arrays: faster on this thread (a queued
                        # copy costs ~0.5 ms of worker overhead each)
                        out[f] = to_device(a, dev, shape)
                        continue
                    out[f] = torch.empty(shape, dtype=torch.float64, device=dev)
                    ctx.call("potr_upload_async", ptr(out[f]), ctypes.c_void_p(a.ctypes.data),
                             ctypes.c_int64(a.nbytes))
                ds = cls(out["positions"], out["sh"], out["opacities"], out["scales"],
                         out["rotations"])
                ds._pending_host = arrs
                return ds
        ds = cls(*(to_device(host[f], dev, shape) for f, shape in
                   (("positions", (n, 3)), ("sh", (n, 3, 16)), ("opacities", (n,)),
                    ("scales", (n, 3)), ("rotations", (n, 4)))))
        ds._pending_host = None
        return ds

    def wait_upload(self):
        """Complete a pending async SH upload (potr_upload_wait)."""
        if getattr(self, "_pending_host", None) is not None:
            context(self.device).call("potr_upload_wait")
            self._pending_host = None

    def _p(self, t):
        return t.data_ptr() if t.numel() > 0 else self._keep[0].data_ptr()

    def struct(self):
        s = _native.PotrSplats()
        s.n = self.n
        s.positions = self._p(self.positions)
        s.sh = self._p(self.sh)
        s.opacities = self._p(self.opacities)
        s.scales = self._p(self.scales)
        s.rotations = self._p(self.rotations)
        return s

    def __len__(self):
        return self.n


def _frozen(t):
    """A read-only ndarray none of whose ndarray bases is writable (a
    read-only view of a writable array can still change under it)."""
    if not isinstance(t, np.ndarray) or t.flags.writeable:
        return False
    b = t.base
    while isinstance(b, np.ndarray):
        if b.flags.writeable:
            return False
        b = b.base
    return True


def _fingerprint(t):
    """256 strided samples of the array's bytes: a cheap check, on every cache
    hit, that a frozen array was not unfrozen, modified and frozen again."""
    flat = t.reshape(-1)
    step = max(1, flat.size // 256)
    return hash(flat[::step][:256].tobytes())


class TargetCache:
    """Device copies of the fixed reference renders.

    The targets are fixed for a whole encode (the reference makes
    them read-only, rasterizer.py:375-376 / scene.py:86-93), and run_pruning
    passes the same arrays on every one of its 48 iterations.  A frozen array
    (read-only, and no writable ndarray base under it) that is the same object
    as last time, with the same sampled fingerprint, is therefore served from
    HBM; anything else is re-uploaded on every call.
    """

    def __init__(self):
        self._entries = {}

    def get(self, targets, cameras, device):
        out = []
        keep = {}
        for s, t in enumerate(targets):
            shape = (int(cameras[s].height), int(cameras[s].width), 3)
            frozen = _frozen(t)
            fp = _fingerprint(t) if frozen else None
            hit = self._entries.get(id(t))
            if (frozen and hit is not None and hit[0] is t and hit[2] == fp
                    and hit[1].device == device and tuple(hit[1].shape) == shape):
                dt = hit[1]
            else:
                dt = to_device(t, device, shape)
            if frozen:
                keep[id(t)] = (t, dt, fp)
            out.append(dt)
        self._entries = keep
        return out

    def clear(self):
        self._entries = {}


targets_cache = TargetCache()


class LazyHostArray:
    """A device-resident result that becomes a numpy array on first use.

    forward_stats returns camera_importance (S, N) -- 4.8 GB at 3M splats and
    200 views -- that the pruning controller never reads; the SH recompute
    reads it straight from HBM.  Any numpy use (np.asarray, indexing,
    attribute access) copies it to the host once.
    """

    def __init__(self, tensor):
        self._tensor = tensor
        self._host = None

    @property
    def device_tensor(self):
        return self._tensor

    def numpy(self):
        if self._host is None:
            self._host = to_host(self._tensor)
        return self._host

    def __array__(self, dtype=None, copy=None):
        a = self.numpy()
        if dtype is not None and a.dtype != dtype:
            return a.astype(dtype)
        return a.copy() if copy else a

    @property
    def shape(self):
        return tuple(self._tensor.shape)

    @property
    def dtype(self):
        return np.dtype(np.float64)

    @property
    def ndim(self):
        return self._tensor.dim()

    def __len__(self):
        return int(self._tensor.shape[0])

    def __getitem__(self, item):
        return self.numpy()[item]

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self.numpy(), name)

    def __repr__(self):
        return f"LazyHostArray(shape={self.shape}, device={self._tensor.device})"

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        conv = tuple(np.asarray(x) if isinstance(x, LazyHostArray) else x for x in inputs)
        return getattr(ufunc, method)(*conv, **kwargs)


def as_device_matrix(a, shape, device):
    """Device float64 view of a (possibly lazy) host matrix."""
    if isinstance(a, LazyHostArray) and a.device_tensor.device == device:
        return a.device_tensor.reshape(shape)
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float64).reshape(shape).contiguous()
    return to_device(np.asarray(a), device, shape)
