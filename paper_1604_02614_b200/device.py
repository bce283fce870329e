"""Device plumbing: torch is used only to own fp64 device buffers and streams."""

import numpy as np
import torch

from . import _native as N

F64 = torch.float64


_CUDA_OK = False
_DEVICES = {}


def require_cuda():
    global _CUDA_OK
    if _CUDA_OK:
        return
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1604_02614_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    _CUDA_OK = True


def device():
    # hot on small grids: one cached torch.device per device index, no availability probe
    require_cuda()
    i = torch._C._cuda_getDevice()
    d = _DEVICES.get(i)
    if d is None:
        d = _DEVICES[i] = torch.device("cuda", i)
    return d


def is_host(x):
    return not isinstance(x, torch.Tensor)


def to_device(x):
    """fp64 contiguous CUDA tensor view/copy of x (numpy, list or tensor)."""
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            x = x.to(device())
        if x.dtype != F64:
            x = x.to(F64)
        return x.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=float))
    t = torch.from_numpy(arr)
    return t.to(device(), non_blocking=False)


def to_host(t):
    return t.detach().to("cpu").numpy()


def empty(n):
    return torch.empty(int(n), dtype=F64, device=device())


def zeros(n):
    return torch.zeros(int(n), dtype=F64, device=device())


def ptr(t):
    return None if t is None else t.data_ptr()


def stream_handle():
    # the raw cudaStream_t of torch's current stream (no Stream object per call)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


class Scratch:
    """Small device scalars + pinned host mirror for one sync point."""

    def __init__(self, n):
        self.dev = torch.zeros(int(n), dtype=F64, device=device())
        self.host = torch.zeros(int(n), dtype=F64, pin_memory=True)

    def read(self, k=None):
        k = self.dev.numel() if k is None else k
        self.host[:k].copy_(self.dev[:k], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.host[:k].numpy()


class Ctx:
    """Owner of one libemhd context (one grid / physics / slab placement)."""

    def __init__(self, geometry, physics, max_vectors):
        require_cuda()
        L = N.lib()
        self.lib = L
        h = N.c_vp()
        self.geometry = geometry
        self.physics = physics
        N.check(L.emhd_ctx_create(ctypes_byref(h), ctypes_byref(geometry), ctypes_byref(physics),
                                  int(max_vectors)), "ctx_create")
        self.h = h
        self.max_vectors = int(max_vectors)
        self._stream = None
        # RHS evaluations the device counted for speculative Arnoldi iterations that were
        # discarded (the reference never performs them); subtracted from StepStats.rhs_evals
        self.rhs_discount = 0
        # stencil launches whose status is checked later (a step's RHS / remainder Jv): each is
        # tagged with its own epoch DEFER_BASE + k, so the first one that failed is known and
        # its admissibility report names the reference's cell (mhd.py:111-131)
        self.deferred = []

    def sync_stream(self):
        s = stream_handle()
        if s != self._stream:
            self.lib.emhd_set_stream(self.h, s)
            self._stream = s
        return self.h

    def status(self):
        st = N.Status()
        N.check(self.lib.emhd_status_read(self.sync_stream(), ctypes_byref(st)), "status_read")
        return st

    def stencil_path(self, **kw):
        """Current stencil launch selection as a dict; keyword arguments (kernel, rows_per_cta,
        strip, bulk, min_rows, tile_rows) change it for every later launch on this context."""
        sp = N.StencilPath()
        N.check(self.lib.emhd_get_stencil_path(self.h, ctypes_byref(sp)), "get_stencil_path")
        if kw:
            for k, v in kw.items():
                setattr(sp, k, int(v))
            N.check(self.lib.emhd_set_stencil_path(self.h, ctypes_byref(sp)), "set_stencil_path")
        return {k: getattr(sp, k) for k, _ in N.StencilPath._fields_}

    def fused_orth(self, on):
        """Small grids: run an Arnoldi iteration's orthogonalisation as one launch (default on;
        off: the separate multi-dot / update launches, bit-identical)."""
        N.check(self.lib.emhd_set_fused_orth(self.h, int(bool(on))), "set_fused_orth")

    def last_stencil(self):
        """What the last stencil launch on this context ran (kernel 1 marching / 2 tile, ...)."""
        sp = N.StencilPath()
        N.check(self.lib.emhd_last_stencil(self.h, ctypes_byref(sp)), "last_stencil")
        return {k: getattr(sp, k) for k, _ in N.StencilPath._fields_}

    DEFER_BASE = -(2 ** 31)

    def defer(self, report_args, keep=()):
        """Tag the next stencil launch as deferred (status read later); keep its inputs alive."""
        k = len(self.deferred)
        self.deferred.append((report_args, keep))
        N.check(self.lib.emhd_set_epoch(self.sync_stream(), self.DEFER_BASE + k), "set_epoch")

    def undefer(self):
        N.check(self.lib.emhd_set_epoch(self.sync_stream(), -1), "set_epoch")

    def deferred_report(self, st):
        """Report arguments of the deferred launch that flagged first, or None."""
        k = st.fail_iter - self.DEFER_BASE
        if 0 <= k < len(self.deferred):
            return self.deferred[k][0]
        return None

    def reset_status(self):
        N.check(self.lib.emhd_status_reset(self.sync_stream()), "status_reset")

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and self.h.value:
                self.lib.emhd_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


def ctypes_byref(x):
    import ctypes
    return ctypes.byref(x)
