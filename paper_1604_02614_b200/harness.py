"""GPU backend of the reference harness's numerical pieces (pkg/src/expmhd/harness.py).

* ``integrate_rk4``  — classical explicit RK4 with the last step clipped (harness.py:182-199),
  the cross-check integrator of ``reference_solution``; every stage runs on the device:
  the fused RHS stencil plus exact-order stage combinations (``emhd_lincomb`` /
  ``emhd_lincomb_onto``), so trajectories are bit-identical to the reference's.
* ``rk4_stable_dt`` — the conservative explicit step (harness.py:166-179) from a device
  max-reduction of the fast signal speed (``emhd_max_signal_speed``; bitwise).
* ``error_norm``   — max over components of the grid-weighted l2 difference
  (harness.py:153-163) from per-field device sums (``emhd_field_sqdiff``).
* ``integrate``    — the harness's method switch (``_integrate``, harness.py:202-216) on the
  GPU integrators, for a reference ``ExperimentConfig`` (duck-typed).

All accept slab layouts (``layout``/``comm``) like the rest of the package.
"""

import time as _time

import torch

from . import _native as N
from . import device as D
from .epirk import StepController, StepStats, integrate_adaptive, integrate_fixed
from .fdjac import _generic_ctx, _lincomb, host_rhs, unwrap_gpu_rhs
from .mhd import AdmissibilityError, BoundaryPolicy, _diag_ctx, agree_status, make_rhs, raise_status


def _state_ctx(grid, layout=None, comm=None, params=None):
    if params is None:
        return _diag_ctx(grid, BoundaryPolicy("periodic", "periodic"), layout, comm)
    key = ("speed", params)
    f = _diag_ctx(grid, BoundaryPolicy("periodic", "periodic"), layout, comm)
    cache = f.__dict__.setdefault("_speed_ctx", {})
    if key not in cache:
        from .mhd import GpuRhs
        cache[key] = GpuRhs(params, grid, BoundaryPolicy("periodic", "periodic"), check=True,
                            layout=f.layout, comm=f.comm, max_vectors=1)
    return cache[key]


def error_norm(U, U_ref, grid, layout=None, comm=None):
    """max_f sqrt(sum_cells (U_f - R_f)^2 * hx * hy) over the whole (slab-decomposed) grid."""
    f = _state_ctx(grid, layout, comm)
    nxl = f.layout.nx_local
    shape_u, shape_r = tuple(U.shape), tuple(U_ref.shape)
    if shape_u != shape_r or shape_u[1:] != (nxl, grid.ny):
        raise ValueError(f"state shapes {shape_u} / {shape_r} do not "
                         f"match grid ({grid.nx}, {grid.ny})")
    u = D.to_device(U).reshape(-1)
    r = D.to_device(U_ref).reshape(-1)
    sums = D.zeros(8)
    N.check(f.ctx.lib.emhd_field_sqdiff(f.ctx.sync_stream(), D.ptr(u), D.ptr(r), D.ptr(sums)),
            "field_sqdiff")
    f.comm.allreduce_sum(sums)
    area = grid.hx * grid.hy
    return float(torch.sqrt(sums * area).max().item())


def rk4_stable_dt(U, grid, params, layout=None, comm=None):
    """Conservative explicit RK4 step size (harness.py:166-179), bitwise the reference's."""
    f = _state_ctx(grid, layout, comm, params)
    u = D.to_device(U).reshape(-1)
    cmax = D.zeros(1)
    f.ctx.reset_status()
    N.check(f.ctx.lib.emhd_max_signal_speed(f.ctx.sync_stream(), D.ptr(u), D.ptr(cmax)),
            "max_signal_speed")
    f.comm.allreduce_max(cmax)
    st = f.ctx.status()
    if st.flags & (N.ST_RHO | N.ST_PRESSURE):
        f.ctx.reset_status()
        kind = "density" if st.flags & N.ST_RHO else "pressure"
        raise AdmissibilityError(f"non-positive {kind} in the state")
    h = min(grid.hx, grid.hy)
    dt_wave = 0.3 * h / float(cmax.item())
    diff = max(params.mu, params.eta,
               params.gamma * params.mu * params.kappa / (params.gamma - 1.0), 1e-30)
    return min(dt_wave, 0.2 * h * h / diff)


class _Rk4Stages:
    """Device buffers and launches of one RK4 step (k1..k4, the stage input, the next y).

    ``rhs`` is the fused stencil (GpuRhs) or, for a user callable (the reference accepts
    any rhs), ``call`` evaluates it on the device vector; the stage algebra is on the device
    either way."""

    def __init__(self, rhs, n, call=None, ctx=None):
        self.rhs = rhs
        self.call = call
        self.ctx = ctx if ctx is not None else rhs.ctx
        mk = lambda: torch.empty(n, dtype=D.F64, device=D.device())   # noqa: E731
        self.k = [mk() for _ in range(4)]
        self.stage = mk()
        self.ynew = mk()
        self.halo = None
        if call is None and rhs.layout.distributed:
            from .slab import halo_shape
            self.halo = torch.zeros(halo_shape(rhs.grid.ny), dtype=D.F64, device=D.device())

    def f(self, x, out):
        if self.call is not None:
            out.copy_(D.to_device(self.call(x)).reshape(-1))
            return
        xh = self.rhs.halo(x, self.halo) if self.halo is not None else None
        self.rhs.launch(x, out, xh)

    def step(self, y, dt):
        k1, k2, k3, k4 = self.k
        c = 0.5 * dt                                       # 0.5 * step * k (left to right)
        self.f(y, k1)
        _lincomb(self.ctx, [y, (c, k1)], self.stage)        # y + (0.5*step)*k1
        self.f(self.stage, k2)
        _lincomb(self.ctx, [y, (c, k2)], self.stage)
        self.f(self.stage, k3)
        _lincomb(self.ctx, [y, (dt, k3)], self.stage)       # y + step*k3
        self.f(self.stage, k4)
        # y + (step / 6) * (((k1 + 2 k2) + 2 k3) + k4)   (harness.py:194)
        xs = N.ptr_array([D.ptr(k1), D.ptr(k2), D.ptr(k3), D.ptr(k4)])
        N.check(self.ctx.lib.emhd_lincomb_onto(self.ctx.sync_stream(), D.ptr(y), 4, xs,
                                               N.dbl_array([1.0, 2.0, 2.0, 1.0]),
                                               N.int_array([0, 1, 1, 0]), dt / 6.0, 1,
                                               D.ptr(self.ynew), self.ynew.numel()), "lincomb_onto")
        return self.ynew

    def replay_checked(self, y, dt):
        """Error path: the step's stages again, one checked RHS call at a time, so the raised
        exception (type and offending cell) is the reference's."""
        c = 0.5 * dt
        k1 = self.rhs(y)
        k2 = self.rhs(_lincomb(self.ctx, [y, (c, k1)], self.stage).clone())
        k3 = self.rhs(_lincomb(self.ctx, [y, (c, k2)], self.stage).clone())
        self.rhs(_lincomb(self.ctx, [y, (dt, k3)], self.stage).clone())


def integrate_rk4(rhs, y0, t0, t_end, h):
    """Classical explicit RK4 with the last step clipped (harness.py:182-199).

    ``rhs`` is a ``make_rhs`` closure (the fused stencil) or any other callable, as in the
    reference; ``y0`` a host or device vector (a host input returns a host result).  The
    stage algebra runs on the device in the reference's operation order.  With admissibility
    checks on, the status word is read once per step (one
    device sync); a flagged step is replayed stage by stage from the state before it (still
    resident: the three step buffers rotate) to raise the reference's exception.
    """
    g = unwrap_gpu_rhs(rhs)
    host = D.is_host(y0)
    y = D.to_device(y0).reshape(-1).clone()
    stats = StepStats()
    start = _time.perf_counter()
    if g is None:
        # any other callable (the reference takes one): evaluated as given, on device vectors
        # for torch-aware callables or through the host for NumPy ones
        S = _Rk4Stages(None, y.numel(), call=host_rhs(rhs), ctx=_generic_ctx())
        return _rk4_loop(S, None, y, t0, t_end, h, stats, start, host)
    S = _Rk4Stages(g, y.numel())
    return _rk4_loop(S, g, y, t0, t_end, h, stats, start, host)


def _rk4_loop(S, g, y, t0, t_end, h, stats, start, host):
    prev = torch.empty_like(y)
    t = t0
    check = g is not None and g.check
    while t < t_end - 1e-14 * max(1.0, abs(t_end)):
        step = min(h, t_end - t)
        ynew = S.step(y, step)
        y, prev, S.ynew = ynew, y, prev          # prev: the state this step started from
        if check:
            st = agree_status(g.ctx.status(), g.comm)
            if st.flags & (N.ST_RHO | N.ST_PRESSURE):
                g.ctx.reset_status()
                S.replay_checked(prev, step)
                raise_status(g.ctx, st, None, g.comm)
        t += step
        stats.steps_accepted += 1
        stats.rhs_evals += 4
    torch.cuda.current_stream().synchronize()
    stats.wall_time = _time.perf_counter() - start
    return (D.to_host(y) if host else y), stats


def integrate(cfg, control, y0, t0, t_end, grid, layout=None, comm=None):
    """The harness's per-method integrator switch (harness.py:202-216) on the GPU."""
    rhs = make_rhs(cfg.params(), grid, cfg.bc(), layout=layout, comm=comm)
    if cfg.method == "epirk5p1":
        return integrate_adaptive(rhs, y0, t0, t_end, StepController(tol=control),
                                  recoverable=(AdmissibilityError,))
    if cfg.method in ("epirk4-fixed", "epirk5p1-fixed"):
        return integrate_fixed(cfg.method.split("-")[0], rhs, y0, t0, t_end, control,
                               tol_krylov=cfg.krylov_tol)
    return integrate_rk4(rhs, y0, t0, t_end, control)


__all__ = ["error_norm", "rk4_stable_dt", "integrate_rk4", "integrate"]
