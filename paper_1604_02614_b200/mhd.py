"""GPU drop-in for the reference RHS interface (pkg/src/expmhd/mhd.py).

Same public names and semantics as the reference: ``Grid2D`` (mhd.py:31-64),
``MhdParams`` (:67-81), ``BoundaryPolicy`` (:84-96), ``AdmissibilityError``
(:27-28), ``energy_from`` (:134-141), ``state_to_vector`` /
``vector_to_state`` (:99-103) and ``make_rhs`` (:280-285).  ``make_rhs``
returns a :class:`GpuRhs`: calling it evaluates the fused sm_100a stencil
(csrc/stencil.cu) on a device vector (torch CUDA fp64) and returns a fresh
device vector; NumPy input is copied to the device and the result copied
back, so reference-style code runs unchanged.
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as D
from .slab import Comm, halo_shape, make_layout

NVARS = 8
RHO, MX, MY, MZ, BX, BY, BZ, EN = range(NVARS)


class AdmissibilityError(ValueError):
    """State with non-positive density or pressure (reference mhd.py:27-28)."""


@dataclass(frozen=True)
class Grid2D:
    """Uniform cell-centred grid on [x_lo, x_hi] x [y_lo, y_hi]."""

    nx: int
    ny: int
    x_lo: float
    x_hi: float
    y_lo: float
    y_hi: float

    def __post_init__(self):
        if self.nx < 4 or self.ny < 4:
            raise ValueError("grid needs at least 4 cells per direction")
        if self.x_hi <= self.x_lo or self.y_hi <= self.y_lo:
            raise ValueError("domain bounds must be increasing")

    @property
    def hx(self):
        return (self.x_hi - self.x_lo) / self.nx

    @property
    def hy(self):
        return (self.y_hi - self.y_lo) / self.ny

    def cell_centers(self):
        x = self.x_lo + (np.arange(self.nx) + 0.5) * self.hx
        y = self.y_lo + (np.arange(self.ny) + 0.5) * self.hy
        return x, y

    @property
    def n_dof(self):
        return NVARS * self.nx * self.ny


@dataclass(frozen=True)
class MhdParams:
    mu: float = 0.0
    eta: float = 0.0
    kappa: float = 0.0
    gamma: float = 5.0 / 3.0
    b_half: bool = True

    def __post_init__(self):
        if min(self.mu, self.eta, self.kappa) < 0:
            raise ValueError("dissipation parameters must be non-negative")
        if self.gamma <= 1.0:
            raise ValueError("gamma must exceed 1")


@dataclass(frozen=True)
class BoundaryPolicy:
    x: str = "periodic"
    y: str = "reflect"

    _VALID = ("periodic", "reflect", "zero-gradient")

    def __post_init__(self):
        for pol in (self.x, self.y):
            if pol not in self._VALID:
                raise ValueError(f"unknown boundary policy {pol!r}")


def state_to_vector(U):
    if isinstance(U, torch.Tensor):
        return U.contiguous().reshape(-1)
    return np.ascontiguousarray(U).reshape(-1)


def vector_to_state(y, grid):
    return y.reshape(NVARS, grid.nx, grid.ny)


def energy_from(rho, v, B, p, params):
    """Total energy density from primitives (host-side IC helper, mhd.py:134-141)."""
    v = np.asarray(v)
    B = np.asarray(B)
    kin = 0.5 * rho * (v[0] ** 2 + v[1] ** 2 + v[2] ** 2)
    mag = B[0] ** 2 + B[1] ** 2 + B[2] ** 2
    mag = 0.5 * mag if params.b_half else mag
    return p / (params.gamma - 1.0) + kin + mag


def agree_status(st, comm):
    """Combine the status words of all slab ranks (OR of flags, min of indices).

    Every rank must take the same exception path, or the next collective hangs.
    """
    if comm is None or not comm.layout.distributed:
        return st
    err = st.flags & (N.ST_RHO | N.ST_PRESSURE | N.ST_NONFINITE | N.ST_DENSE)
    t = torch.tensor([float(err & N.ST_RHO), float(err & N.ST_PRESSURE), float(err & N.ST_NONFINITE),
                      float(err & N.ST_DENSE)], dtype=D.F64, device=D.device())
    comm.allreduce_max(t)
    mn = torch.tensor([float(st.first_nonfinite if st.first_nonfinite < 2 ** 62 else 2 ** 62),
                       float(st.fail_iter)], dtype=D.F64, device=D.device())
    comm.allreduce_min(mn)
    out = N.Status()
    bits = t.cpu().numpy()
    out.flags = (st.flags & ~(N.ST_RHO | N.ST_PRESSURE | N.ST_NONFINITE | N.ST_DENSE)) | \
        sum(int(b) for b in bits)
    mnv = mn.cpu().numpy()
    out.rhs_evals = st.rhs_evals
    out.rhs_evals_mark = st.rhs_evals_mark
    out.first_nonfinite = int(mnv[0])
    out.breakdown = st.breakdown
    out.fail_iter = int(mnv[1])
    out.local_flags = st.flags
    return out


def raise_status(ctx, st, report_args=None, comm=None):
    """Map the device status word to the reference's exception types.

    Priority follows the reference: density (mhd.py:123-125), then pressure
    (:128-130), then a non-finite perturbed RHS (fdjac.py:45-48).  With a slab
    communicator the decision is taken on the combined status of all ranks.
    """
    st = agree_status(st, comm)
    flags = st.flags
    local = getattr(st, "local_flags", flags)
    if not flags & (N.ST_RHO | N.ST_PRESSURE | N.ST_NONFINITE | N.ST_DENSE):
        return
    ctx.reset_status()
    if not flags & (N.ST_RHO | N.ST_PRESSURE | N.ST_NONFINITE):
        raise FloatingPointError("overflow in augmented-matrix exponential")
    if flags & (N.ST_RHO | N.ST_PRESSURE):
        msg = None
        if report_args is not None and local & (N.ST_RHO | N.ST_PRESSURE):
            rep = N.Report()
            mode, a, ah, v, vh, sc = report_args
            N.check(ctx.lib.emhd_admissibility_report(ctx.sync_stream(), mode, a, ah, v, vh, sc,
                                                      D.ctypes_byref(rep)), "admissibility_report")
            if rep.which == 1:
                msg = f"non-positive density at cell {(rep.i, rep.j)}: {rep.value}"
            elif rep.which == 2:
                msg = f"non-positive pressure at cell {(rep.i, rep.j)}: {rep.value}"
        if msg is None:
            kind = "density" if flags & N.ST_RHO else "pressure"
            msg = f"non-positive {kind} in the ghost-padded state"
        raise AdmissibilityError(msg)
    raise FloatingPointError(
        f"non-finite rhs value at component {st.first_nonfinite} during Jacobian apply")


class GpuRhs:
    """Device RHS closure: the fused stencil behind ``make_rhs`` (mhd.py:280-285).

    ``rhs(y)`` with y a CUDA fp64 vector of the local slab returns F(y) on the
    device; with a NumPy vector it returns NumPy.  ``slab``/``comm`` select the
    rank's x-slab (default: the whole grid on the current GPU).
    """

    def __init__(self, params, grid, bc, check=True, layout=None, comm=None, max_vectors=136):
        D.require_cuda()
        self.params, self.grid, self.bc, self.check = params, grid, bc, bool(check)
        self.layout = layout or make_layout(grid.nx, grid.ny, bc.x)
        self.comm = comm or Comm(self.layout)
        L = self.layout
        geo = N.Geometry(L.nx_local, grid.ny, grid.nx, L.x_offset, grid.hx, grid.hy,
                         N.BC[L.bc_lo], N.BC[L.bc_hi], N.BC[bc.y])
        phys = N.Physics(params.mu, params.eta, params.kappa, params.gamma,
                         int(bool(params.b_half)), int(self.check))
        self.ctx = D.Ctx(geo, phys, max_vectors)
        self.n = L.n_local
        self._send = None
        if L.distributed:
            self._send = torch.empty(halo_shape(grid.ny), dtype=D.F64, device=D.device())
        # slab collectives inside the library (slab.NativeComm): the stencil entry points then
        # exchange the halo of the vector they perturb themselves, overlapped with the interior
        self.native = bool(getattr(self.comm, "native", False)) and L.distributed
        if self.native:
            self.comm.attach(self.ctx)

    @property
    def defer_halo(self):
        """True when hot-path callers should pass no halo and let the library exchange it
        (overlapped with the stencil's interior rows)."""
        return self.native

    # -- halos -------------------------------------------------------------
    def halo(self, x, out=None):
        """Exchanged x-halo of a local vector (None when the rank has no neighbours)."""
        if not self.layout.distributed:
            return None
        h = self.ctx.sync_stream()
        if out is None:
            out = torch.zeros(halo_shape(self.grid.ny), dtype=D.F64, device=D.device())
        if self.native:
            N.check(self.ctx.lib.emhd_halo_exchange(h, D.ptr(x), D.ptr(out)), "halo_exchange")
            return out
        N.check(self.ctx.lib.emhd_pack_edges(h, D.ptr(x), D.ptr(self._send)), "pack_edges")
        self.comm.exchange(self._send, out)
        return out

    # -- launches ------------------------------------------------------------
    def launch(self, y, out, y_halo=None):
        N.check(self.ctx.lib.emhd_rhs(self.ctx.sync_stream(), D.ptr(y), D.ptr(y_halo), D.ptr(out)),
                "rhs")
        return out

    def check_status(self, report_args=None):
        raise_status(self.ctx, self.ctx.status(), report_args, self.comm)

    def __call__(self, y):
        host = D.is_host(y)
        yd = D.to_device(y).reshape(-1)
        if yd.numel() != self.n:
            raise ValueError(f"state has {yd.numel()} entries, expected {self.n}")
        yh = None if self.defer_halo else self.halo(yd)
        out = torch.empty_like(yd)
        self.launch(yd, out, yh)
        if self.check:
            self.check_status((0, D.ptr(yd), D.ptr(yh), None, None, None))
        return D.to_host(out) if host else out


def make_rhs(params, grid, bc, check=True, layout=None, comm=None):
    """Flat-vector right-hand-side closure for the time integrators (mhd.py:280-285)."""
    return GpuRhs(params, grid, bc, check=check, layout=layout, comm=comm)


def local_rows(y_global, grid, layout):
    """The slab of a global state vector owned by `layout` (host or device)."""
    U = y_global.reshape(NVARS, grid.nx, grid.ny)
    sl = U[:, layout.x_offset:layout.x_offset + layout.nx_local, :]
    if isinstance(sl, torch.Tensor):
        return sl.contiguous().reshape(-1)
    return np.ascontiguousarray(sl).reshape(-1)


_DIAG = {}


def _diag_ctx(grid, bc, layout=None, comm=None):
    key = (grid, bc, layout)
    if key not in _DIAG:
        _DIAG[key] = GpuRhs(MhdParams(), grid, bc, check=False, layout=layout, comm=comm)
    return _DIAG[key]


def div_B(U, grid, bc, layout=None, comm=None):
    """Centred divergence of the in-plane field and its max |.| (mhd.py:288-296), on the GPU."""
    host = D.is_host(U)
    f = _diag_ctx(grid, bc, layout, comm)
    u = D.to_device(U).reshape(-1)
    nxl = f.layout.nx_local
    d = torch.empty(nxl * grid.ny, dtype=D.F64, device=D.device())
    mx = D.zeros(1)
    N.check(f.ctx.lib.emhd_div_b(f.ctx.sync_stream(), D.ptr(u), D.ptr(f.halo(u)), D.ptr(d), D.ptr(mx)),
            "div_b")
    f.comm.allreduce_max(mx)
    d = d.view(nxl, grid.ny)
    peak = float(mx.item())
    return (D.to_host(d) if host else d), peak


def current_J(U, grid, bc, layout=None, comm=None):
    """Centred current J = curl B, shape (3, nx, ny) (mhd.py:299-309), on the GPU."""
    host = D.is_host(U)
    f = _diag_ctx(grid, bc, layout, comm)
    u = D.to_device(U).reshape(-1)
    nxl = f.layout.nx_local
    J = torch.empty(3 * nxl * grid.ny, dtype=D.F64, device=D.device())
    N.check(f.ctx.lib.emhd_current_j(f.ctx.sync_stream(), D.ptr(u), D.ptr(f.halo(u)), D.ptr(J)),
            "current_j")
    J = J.view(3, nxl, grid.ny)
    return D.to_host(J) if host else J
