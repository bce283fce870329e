"""Oracle: forward-difference Jacobian action.  TEST INFRASTRUCTURE ONLY.

Restates reference ``pkg/src/expmhd/fdjac.py:15-49``:
sigma = sqrt(eps) / ||v||_inf (sigma = 1 when ||v||_inf <= sqrt(eps)),
Jv = (F(a + sigma v) - F(a)) / sigma, F(a) cached, v = 0 -> zeros without an
RHS call, a non-finite perturbed RHS raises FloatingPointError naming the
first bad component.
"""

import math

import numpy as np

SQRT_EPS = math.sqrt(np.finfo(float).eps)     # == 2**-26 exactly


class FdJv:
    """Callable v -> J(a) v with the reference's scaling rule."""

    def __init__(self, rhs, a, f_a=None):
        self.rhs = rhs
        self.a = np.asarray(a, dtype=float)
        self.f_a = rhs(self.a) if f_a is None else np.asarray(f_a, dtype=float)
        self.n = self.a.size
        self.rhs_calls = 0

    @staticmethod
    def sigma_for(vnorm):
        return SQRT_EPS / vnorm if vnorm > SQRT_EPS else 1.0

    def __call__(self, v):
        v = np.asarray(v, dtype=float)
        vmax = float(np.max(np.abs(v))) if v.size else 0.0
        if vmax == 0.0:
            return np.zeros_like(self.a)
        s = self.sigma_for(vmax)
        self.rhs_calls += 1
        fp = self.rhs(self.a + s * v)
        finite = np.isfinite(fp)
        if not finite.all():
            first = int(np.flatnonzero(~finite)[0])
            raise FloatingPointError(
                f"non-finite rhs value at component {first} during Jacobian apply")
        return (fp - self.f_a) / s
