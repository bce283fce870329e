"""Oracle: Arnoldi / phi-function Krylov layer.  TEST INFRASTRUCTURE ONLY.

Restates reference ``pkg/src/expmhd/krylov.py`` and ``phifuncs.py``:

* ``Arnoldi``            _ArnoldiProcess            krylov.py:127-188
  (modified Gram–Schmidt + one full re-orthogonalisation pass, breakdown when
  h_{j+1,j} <= 1e-12 * max(||A v_j||, 1))
* ``arnoldi``            arnoldi                    krylov.py:191-206
* ``resid``              residual_estimate          krylov.py:209-231
* ``phi_block``          phi_dense                  phifuncs.py:65-107
* ``multi_scale``        multi_scale_eval           krylov.py:327-383
* ``phi_combination``    phi_comb (+ apply_aug)     krylov.py:241-324

Counters follow ``KrylovStats`` (krylov.py:55-68) field for field.
"""

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg

BREAKDOWN_RTOL = 1e-12


@dataclass
class Knobs:
    """Same fields and defaults as the reference ``KrylovConfig`` (krylov.py:71-82)."""
    m_init: int = 10
    m_max: int = 100
    soft_cap: int = 25
    grow_threshold: int = 10
    substep_growth: float = 4.0 / 3.0
    min_substep: float = 1.0 / 1024.0
    max_substep: float = 1.0
    reorthogonalize: bool = True


@dataclass
class Counters:
    operator_applies: int = 0
    substeps: int = 0
    max_basis_size: int = 0
    projections: int = 0


class CapReached(RuntimeError):
    """Twin of ``KrylovConvergenceError`` (krylov.py:31-36)."""

    def __init__(self, message, residual):
        super().__init__(message)
        self.residual = residual


class Arnoldi:
    """Growable Arnoldi factorisation, one basis vector per ``grow()``."""

    def __init__(self, op, seed, cap):
        self.op = op
        self.n = len(seed)
        self.cap = min(cap, self.n)
        self.beta = float(np.linalg.norm(seed))
        if self.beta == 0.0:
            raise ValueError("Arnoldi seed vector must be nonzero")
        self.V = np.empty((self.n, self.cap + 1))
        self.V[:, 0] = seed / self.beta
        self.H = np.zeros((self.cap + 1, self.cap))
        self.m = 0
        self.broke = False
        self.applies = 0

    def grow(self):
        if self.broke or self.m >= self.cap:
            return False
        j = self.m
        w = self.op(self.V[:, j])
        self.applies += 1
        w_norm0 = np.linalg.norm(w)
        for _sweep in range(2):                      # MGS, then one re-pass
            for i in range(j + 1):
                c = np.dot(w, self.V[:, i])
                self.H[i, j] += c
                w = w - c * self.V[:, i]
        h = np.linalg.norm(w)
        self.m = j + 1
        if h <= BREAKDOWN_RTOL * max(w_norm0, 1.0):
            self.broke = True
            return False
        self.H[j + 1, j] = h
        self.V[:, j + 1] = w / h
        return True

    @property
    def Hm(self):
        return self.H[:self.m, :self.m]

    @property
    def h_next(self):
        return 0.0 if self.broke else self.H[self.m, self.m - 1]

    def snapshot(self):
        """(V, H) as the reference ``ArnoldiBasis`` would hold them."""
        m = self.m
        if self.broke:
            return self.V[:, :m].copy(), self.H[:m, :m].copy()
        return self.V[:, :m + 1].copy(), self.H[:m + 1, :m].copy()


def arnoldi(op, v, m):
    v = np.asarray(v, dtype=float)
    if np.linalg.norm(v) == 0.0:
        raise ValueError("Arnoldi seed vector must be nonzero")
    if m > op.n:
        raise ValueError(f"basis size {m} exceeds operator dimension {op.n}")
    proc = Arnoldi(op, v, m)
    while proc.m < m and proc.grow():
        pass
    return proc


def resid(h_next, y):
    """|h_{m+1,m}| |y_m| / ||y|| (krylov.py:209-231)."""
    y = np.asarray(y, dtype=float)
    nrm = np.linalg.norm(y)
    return 0.0 if nrm == 0.0 else abs(h_next) * abs(y[-1]) / nrm


def phi_block(k_max, H):
    """[phi_0(H), ..., phi_kmax(H)] from one block-augmented expm (phifuncs.py:65-107)."""
    H = np.asarray(H, dtype=float)
    if not np.all(np.isfinite(H)):
        raise FloatingPointError("H contains non-finite entries")
    n = H.shape[0]
    if k_max == 0:
        return [scipy.linalg.expm(H)]
    big = np.zeros(((k_max + 1) * n,) * 2)
    big[:n, :n] = H
    for j in range(k_max):
        big[j * n:(j + 1) * n, (j + 1) * n:(j + 2) * n] = np.eye(n)
    E = scipy.linalg.expm(big)
    if not np.all(np.isfinite(E)):
        raise FloatingPointError("overflow in augmented-matrix exponential")
    return [E[:n, j * n:(j + 1) * n] for j in range(k_max + 1)]


def _phi_times_e1(Hm, order, scale, beta):
    return phi_block(order, scale * Hm)[order][:, 0] * beta


def multi_scale(op, h, v, scales, tol, knobs=None, order=1):
    """phi_order(c h J) v for all c in scales from one basis (krylov.py:327-375)."""
    knobs = knobs or Knobs()
    scales = list(scales)
    if not scales or any(not (0.0 < c <= 1.0) for c in scales):
        raise ValueError("scales must lie in (0, 1]")
    cnt = Counters(projections=1)
    v = np.asarray(v, dtype=float)
    n = op.n
    if np.all(v == 0.0):
        return [np.zeros(n) for _ in scales], cnt
    c_big = max(scales)
    proc = Arnoldi(op, v, min(knobs.m_max, n))
    while proc.m < min(knobs.m_init, n) and proc.grow():
        pass
    while True:
        y = _phi_times_e1(proc.Hm, order, c_big * h, proc.beta)
        res = resid(proc.h_next, y) * c_big * h
        if res <= tol or proc.broke or proc.m >= proc.n:
            break
        before = proc.m
        proc.grow()
        if proc.m == before:
            cnt.operator_applies += proc.applies
            raise CapReached(
                f"Krylov basis cap {knobs.m_max} reached in multi-scale "
                f"evaluation (residual {res:.3e} > {tol:.3e})", residual=res)
    cnt.operator_applies += proc.applies
    cnt.max_basis_size = proc.m
    cnt.substeps = 1
    Vm = proc.V[:, :proc.m]
    return [Vm @ _phi_times_e1(proc.Hm, order, c * h, proc.beta) for c in scales], cnt


def phi_combination(op, h, c, vectors, tol, knobs=None):
    """sum_k phi_k(c h J) v_k via the augmented exponential (krylov.py:241-324)."""
    knobs = knobs or Knobs()
    cnt = Counters(projections=1)
    n = op.n
    p = len(vectors)
    vs = [np.asarray(x, dtype=float) for x in vectors]
    if all(np.all(x == 0.0) for x in vs):
        return np.zeros(n), cnt
    ch = c * h
    Bmat = np.column_stack(vs[::-1])

    def aug(x):
        u, q = x[:n], x[n:]
        shifted = np.zeros(p)
        shifted[:p - 1] = q[1:]
        return np.concatenate([ch * op(u) + Bmat @ q, shifted])

    naug = n + p
    u = np.zeros(n)
    t, delta = 0.0, 1.0
    while t < 1.0:
        delta = min(delta, knobs.max_substep, 1.0 - t)
        q0 = np.array([t ** (p - 1 - i) / math.factorial(p - 1 - i) for i in range(p)])
        proc = Arnoldi(aug, np.concatenate([u, q0]), min(knobs.m_max, naug))
        while proc.m < min(knobs.m_init, naug) and proc.grow():
            pass
        while True:
            e1 = np.zeros(proc.m)
            e1[0] = proc.beta
            y = scipy.linalg.expm(delta * proc.Hm) @ e1
            res = resid(proc.h_next, y) * delta
            tol_sub = tol * max(delta, 1e-2)
            if res <= tol_sub or proc.broke or proc.m >= proc.n:
                break
            if proc.m >= knobs.soft_cap and delta > knobs.min_substep:
                delta = delta / 2.0
                continue
            before = proc.m
            proc.grow()
            if proc.m == before:
                if delta > knobs.min_substep:
                    delta = delta / 2.0
                    continue
                cnt.operator_applies += proc.applies
                raise CapReached(
                    f"Krylov basis cap {knobs.m_max} reached at substep "
                    f"{delta:.3e} (residual {res:.3e} > {tol_sub:.3e})", residual=res)
        cnt.operator_applies += proc.applies
        u = (proc.V[:, :proc.m] @ y)[:n]
        t = t + delta
        cnt.substeps += 1
        cnt.max_basis_size = max(cnt.max_basis_size, proc.m)
        if proc.m <= knobs.grow_threshold:
            delta = delta * knobs.substep_growth
    return u, cnt
