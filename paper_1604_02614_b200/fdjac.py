"""GPU drop-in for the forward-difference Jacobian (reference fdjac.py:19-49).

``FdJacobianOperator(rhs, a, f_a=None)`` keeps the reference signature and
semantics (sigma = sqrt(eps)/||v||_inf, sigma = 1 below sqrt(eps), cached
F(a), zero direction -> zeros without an RHS call, non-finite F(a + sigma v)
-> FloatingPointError naming the first bad component).

When ``rhs`` is the fused MHD stencil (:class:`~.mhd.GpuRhs`) the whole
apply is ONE sm_100a kernel (a + sigma v formed on load, (F - F(a))/sigma in
the epilogue); inside the Arnoldi loop the normalisation v_j = w / h_{j,j-1}
is fused in as well (krylov.py).  Any other callable on device vectors gets
the generic path: ||v||_inf, a + sigma v and (F - F(a))/sigma on the device
through the exact-order vector kernels, the user's rhs in between.
"""

import math

import numpy as np
import torch

from . import _native as N
from . import device as D
from .mhd import GpuRhs, raise_status

EPS_MACHINE = np.finfo(float).eps
SQRT_EPS = math.sqrt(EPS_MACHINE)


class LinearOperator:
    """Matrix-free operator v -> A v of fixed dimension (krylov.py:39-52)."""

    def __init__(self, n, matvec):
        self.n = int(n)
        self._matvec = matvec

    def __call__(self, v):
        return self._matvec(v)

    @classmethod
    def from_matrix(cls, M):
        Md = D.to_device(M)
        if Md.dim() != 2:
            raise ValueError("from_matrix needs a 2-D matrix")

        def mv(v):
            host = D.is_host(v)
            out = torch.mv(Md, D.to_device(v).reshape(-1))
            return D.to_host(out) if host else out
        op = cls(Md.shape[0], mv)
        op.matrix = Md
        return op


def host_rhs(f):
    """Adapt a NumPy right-hand side ``y -> F(y)`` to device vectors.

    For small user-defined (non-MHD) systems such as the reference's test problems; the
    user's function itself runs wherever the user wrote it to run.
    """
    def g(y):
        if isinstance(y, torch.Tensor):
            return D.to_device(np.asarray(f(D.to_host(y)), dtype=float))
        return f(y)
    g.__wrapped__ = f
    return g


def unwrap_gpu_rhs(rhs):
    """The fused stencil behind rhs (directly or through a counting wrapper)."""
    seen = 0
    while rhs is not None and seen < 4:
        if isinstance(rhs, GpuRhs):
            return rhs
        rhs = getattr(rhs, "rhs", None)
        seen += 1
    return None


def _lincomb(ctx, terms, out, post=None, post_div=False, max_out=None, len_max=0):
    xs, cs, hs = [], [], []
    for t in terms:
        if isinstance(t, tuple):
            c, x = t
            xs.append(D.ptr(x)); cs.append(c); hs.append(1)
        else:
            xs.append(D.ptr(t)); cs.append(1.0); hs.append(0)
    has_post = 0 if post is None else (2 if post_div else 1)
    N.check(ctx.lib.emhd_lincomb(ctx.sync_stream(), len(xs), N.ptr_array(xs), N.dbl_array(cs),
                                 N.int_array(hs), 0.0 if post is None else float(post), has_post,
                                 D.ptr(out), out.numel(), int(len_max), D.ptr(max_out)), "lincomb")
    return out


class FdJacobianOperator(LinearOperator):
    """Forward-difference approximation of the Jacobian of ``rhs`` at ``a``."""

    def __init__(self, rhs, a, f_a=None, ctx=None):
        self.rhs = rhs
        self.gpu = unwrap_gpu_rhs(rhs)
        self.a = D.to_device(a).reshape(-1)
        if f_a is None:
            fa = rhs(self.a)
            self.f_a = D.to_device(fa).reshape(-1)
        else:
            self.f_a = D.to_device(f_a).reshape(-1)
        self.a_halo = self.gpu.halo(self.a) if self.gpu is not None else None
        self.ctx = self.gpu.ctx if self.gpu is not None else (ctx or _generic_ctx())
        self._scr = D.Scratch(4)
        # no bound method stored on self (the reference passes self._apply as the matvec):
        # that would be a reference cycle, and the operator's a / F(a) (2 W of HBM per step)
        # would then live until the garbage collector happens to run
        super().__init__(self.a.numel(), None)

    def __call__(self, v):
        return self._apply(v)

    # raw device apply (no status check); vnorm_dev: device scalar ||v||_inf or None
    def apply_device(self, v, out=None, vnorm_dev=None, v_halo=None):
        v = v.reshape(-1)
        if out is None:
            out = torch.empty_like(self.a)
        if vnorm_dev is None:
            vnorm_dev = self._scr.dev[0:2]
            self.vnorm_into(v, vnorm_dev)
        if self.gpu is not None:
            if v_halo is None and not self.gpu.defer_halo:
                v_halo = self.gpu.halo(v)
            N.check(self.ctx.lib.emhd_jv(self.ctx.sync_stream(), D.ptr(self.a), D.ptr(self.a_halo),
                                         D.ptr(self.f_a), D.ptr(v), D.ptr(v_halo), D.ptr(vnorm_dev),
                                         D.ptr(out)), "jv")
            return out
        return self._generic_apply(v, out, vnorm_dev)

    def vnorm_into(self, v, dev2):
        N.check(self.ctx.lib.emhd_norms(self.ctx.sync_stream(), D.ptr(v), 0, v.numel(), D.ptr(dev2)),
                "norms")
        if self.gpu is not None and self.gpu.layout.distributed:
            self.gpu.comm.allreduce_max(dev2[1:2])
        # emhd_norms writes {sumsq, max}; the stencil reads scal[0] -> shift max into slot 0
        dev2[0:1].copy_(dev2[1:2])
        return dev2

    def _generic_apply(self, v, out, vnorm_dev):
        vnorm = float(vnorm_dev[0].item())
        if vnorm == 0.0:
            out.zero_()
            return out
        sigma = SQRT_EPS / vnorm if vnorm > SQRT_EPS else 1.0
        pert = torch.empty_like(self.a)
        _lincomb(self.ctx, [self.a, (sigma, v)], pert)
        fp = D.to_device(self.rhs(pert)).reshape(-1)
        bad = torch.nonzero(~torch.isfinite(fp))
        if bad.numel():
            raise FloatingPointError(
                f"non-finite rhs value at component {int(bad[0, 0])} during Jacobian apply")
        _lincomb(self.ctx, [fp, (-1.0, self.f_a)], out, post=sigma, post_div=True)
        return out

    def _apply(self, v):
        host = D.is_host(v)
        vd = D.to_device(v).reshape(-1)
        if self.gpu is None:
            out = self.apply_device(vd)
            return D.to_host(out) if host else out
        vh = None if self.gpu.defer_halo else self.gpu.halo(vd)
        scal = self._scr.dev[0:2]
        self.vnorm_into(vd, scal)
        out = self.apply_device(vd, vnorm_dev=scal, v_halo=vh)
        raise_status(self.ctx, self.ctx.status(), comm=self.gpu.comm, report_args=
                     (1, D.ptr(self.a), D.ptr(self.a_halo), D.ptr(vd), D.ptr(vh), D.ptr(scal)))
        return D.to_host(out) if host else out


_GENERIC = None


def _generic_ctx():
    """A tiny context used only for its vector kernels (generic operators)."""
    global _GENERIC
    if _GENERIC is None:
        geo = N.Geometry(4, 4, 4, 0, 1.0, 1.0, 0, 0, 0)
        phys = N.Physics(0.0, 0.0, 0.0, 5.0 / 3.0, 1, 0)
        _GENERIC = D.Ctx(geo, phys, 136)
    return _GENERIC
