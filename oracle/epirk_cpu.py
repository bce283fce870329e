"""Oracle: EpiRK steps and drivers around the Krylov path.  TEST INFRASTRUCTURE ONLY.

Restates reference ``pkg/src/expmhd/epirk.py``:

* coefficients      EPIRK5P1_DECIMALS          epirk.py:23-38
* ``Controller``    StepController             epirk.py:134-166
* ``remainder``     remainder                  epirk.py:179-181
* ``step5p1``       epirk5p1_step              epirk.py:184-228
* ``step4``         epirk4_step                epirk.py:231-268
* ``run_fixed``     integrate_fixed            epirk.py:323-347
* ``run_adaptive``  integrate_adaptive         epirk.py:350-411

Counters mirror ``StepStats`` (epirk.py:104-131).
"""

import math
from dataclasses import dataclass

import numpy as np

from .jvp import FdJv
from .krylov_cpu import CapReached, multi_scale, phi_combination

C5 = {k: float(v) for k, v in {
    "a11": "0.35129592695058193092", "a21": "0.84405472011657126298",
    "a22": "1.6905891609568963624", "b1": "1.0", "b2": "1.2727127317356892397",
    "b3": "2.2714599265422622275", "g11": "0.35129592695058193092",
    "g21": "0.84405472011657126298", "g22": "0.5", "g31": "1.0",
    "g32": "0.71111095364366870359", "g33": "0.62378111953371494809"}.items()}


class StiffnessStop(RuntimeError):
    def __init__(self, message, t, h, last_error):
        super().__init__(message)
        self.t, self.h, self.last_error = t, h, last_error


@dataclass
class Tally:
    steps_accepted: int = 0
    steps_rejected: int = 0
    projections: int = 0
    rhs_evals: int = 0
    operator_applies: int = 0
    substeps: int = 0
    max_basis_size: int = 0

    def add_krylov(self, k):
        self.projections += k.projections
        self.operator_applies += k.operator_applies
        self.substeps += k.substeps
        self.max_basis_size = max(self.max_basis_size, k.max_basis_size)

    def add(self, o):
        for f in ("steps_accepted", "steps_rejected", "projections", "rhs_evals",
                  "operator_applies", "substeps"):
            setattr(self, f, getattr(self, f) + getattr(o, f))
        self.max_basis_size = max(self.max_basis_size, o.max_basis_size)


@dataclass
class Controller:
    tol: float
    safety: float = 0.9
    order: int = 4
    h_min: float = 1e-12
    h_max: float = math.inf
    clamp: tuple = (0.2, 5.0)
    h_init: float = None

    def error_norm(self, err_vec, y):
        w = self.tol + self.tol * np.abs(y)
        return float(np.sqrt(np.mean((err_vec / w) ** 2)))

    def next_h(self, h, err):
        if err == 0.0:
            fac = self.clamp[1]
        else:
            fac = min(max(self.safety * err ** (-1.0 / (self.order + 1)),
                          self.clamp[0]), self.clamp[1])
        return min(max(h * fac, self.h_min), self.h_max)


class _Counted:
    def __init__(self, f):
        self.f, self.calls = f, 0

    def __call__(self, y):
        self.calls += 1
        return self.f(y)


def remainder(rhs, y_n, f_n, jop, y):
    return rhs(y) - f_n - jop(y - y_n)


def _setup(rhs, y_n, f_n):
    cf = _Counted(rhs)
    y_n = np.asarray(y_n, dtype=float)
    f_n = cf(y_n) if f_n is None else np.asarray(f_n, dtype=float)
    return cf, y_n, f_n, FdJv(cf, y_n, f_n)


def step5p1(rhs, y_n, h, tol, knobs=None, f_n=None):
    if h <= 0:
        raise ValueError("step size must be positive")
    cf, y_n, f_n, J = _setup(rhs, y_n, f_n)
    T = Tally()
    (u11, u21, u31), k = multi_scale(J, h, h * f_n, [C5["g11"], C5["g21"], C5["g31"]],
                                     tol, knobs)
    T.add_krylov(k)
    y1 = y_n + C5["a11"] * u11
    r1 = remainder(cf, y_n, f_n, J, y1)
    (w22, w32), k = multi_scale(J, h, h * r1, [C5["g22"], C5["g32"]], tol, knobs)
    T.add_krylov(k)
    y2 = y_n + C5["a21"] * u21 + C5["a22"] * w22
    r2 = remainder(cf, y_n, f_n, J, y2)
    n = y_n.size
    w33, k = phi_combination(J, h, C5["g33"],
                             [np.zeros(n), np.zeros(n), h * (r2 - 2.0 * r1)], tol, knobs)
    T.add_krylov(k)
    corr = C5["b3"] * w33
    y_next = y_n + C5["b1"] * u31 + C5["b2"] * w32 + corr
    T.rhs_evals = cf.calls
    T.steps_accepted = 1
    return y_next, corr, T


def step4(rhs, y_n, h, tol, knobs=None, f_n=None):
    if h <= 0:
        raise ValueError("step size must be positive")
    cf, y_n, f_n, J = _setup(rhs, y_n, f_n)
    T = Tally()
    (u_h, u_23, u_1), k = multi_scale(J, h, h * f_n, [0.5, 2.0 / 3.0, 1.0], tol, knobs)
    T.add_krylov(k)
    r1 = remainder(cf, y_n, f_n, J, y_n + 0.5 * u_h)
    r2 = remainder(cf, y_n, f_n, J, y_n + (2.0 / 3.0) * u_23)
    n = y_n.size
    v3 = h * (32.0 * r1 - 13.5 * r2)
    v4 = h * (-144.0 * r1 + 81.0 * r2)
    w, k = phi_combination(J, h, 1.0, [np.zeros(n), np.zeros(n), v3, v4], tol, knobs)
    T.add_krylov(k)
    T.rhs_evals = cf.calls
    T.steps_accepted = 1
    return y_n + u_1 + w, T


def run_fixed(method, rhs, y0, t0, t_end, h, tol=1e-12, knobs=None, max_steps=None):
    if t_end <= t0:
        raise ValueError("t_end must exceed t0")
    if h <= 0:
        raise ValueError("step size must be positive")
    y, t, tot = np.asarray(y0, dtype=float).copy(), t0, Tally()
    while t < t_end - 1e-14 * max(1.0, abs(t_end)):
        if max_steps is not None and tot.steps_accepted >= max_steps:
            break
        dt = min(h, t_end - t)
        if method == "epirk4":
            y, s = step4(rhs, y, dt, tol, knobs)
        elif method == "epirk5p1":
            y, _, s = step5p1(rhs, y, dt, tol, knobs)
        else:
            raise ValueError(f"unknown method {method!r}")
        tot.add(s)
        t += dt
    return y, tot


def run_adaptive(rhs, y0, t0, t_end, ctl, knobs=None, recoverable=(), max_steps=None):
    if t_end <= t0:
        raise ValueError("t_end must exceed t0")
    y, t = np.asarray(y0, dtype=float).copy(), t0
    h = ctl.h_init if ctl.h_init is not None else (t_end - t0) / 100.0
    h = min(h, ctl.h_max)
    tot = Tally()
    while t < t_end - 1e-14 * max(1.0, abs(t_end)):
        if max_steps is not None and tot.steps_accepted >= max_steps:
            break
        h = min(h, t_end - t)
        try:
            y_new, err_vec, s = step5p1(rhs, y, h, ctl.tol, knobs)
        except CapReached:
            tot.steps_rejected += 1
            h = h / 2.0
            if h < ctl.h_min:
                raise StiffnessStop(f"step size {h:.3e} below h_min at t = {t:.6g} "
                                    f"(Krylov non-convergence)", t, h, math.nan)
            continue
        except recoverable:
            tot.steps_rejected += 1
            if h <= ctl.h_min:
                raise StiffnessStop("trial step rejected by the right-hand side at the "
                                    f"minimum size {h:.3e}, t = {t:.6g}", t, h, math.inf)
            h = max(ctl.h_min, 0.2 * h)
            continue
        err = ctl.error_norm(err_vec, y_new)
        if not math.isfinite(err):
            err = math.inf
        if err <= 1.0:
            tot.add(s)
            y = y_new
            t += h
        else:
            tot.steps_rejected += 1
            tot.projections += s.projections
            tot.rhs_evals += s.rhs_evals
            tot.operator_applies += s.operator_applies
            if h <= ctl.h_min:
                raise StiffnessStop(f"step rejected at the minimum size {h:.3e}, "
                                    f"t = {t:.6g} (error norm {err:.3e})", t, h, err)
        h = ctl.next_h(h, err)
    return y, tot
