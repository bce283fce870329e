"""Seeded initial states of the BASELINE configurations (host-side input setup).

``reconnection_ic`` / ``kh_ic`` / ``default_bc`` and the spec dataclasses
restate reference problems.py:17-122 (checked bit-for-bit against the
reference in tests/test_problems.py).  ``kh_shear_ic`` (BASELINE config 1)
and ``fourier_state`` (config 2) are the generators SURVEY.md §8(d) fixes,
which the reference cannot express.  These build NumPy arrays once; they are
not on the timed path.
"""

from dataclasses import dataclass

import numpy as np

from .mhd import (BX, BY, BZ, EN, MX, MY, MZ, NVARS, RHO, BoundaryPolicy, Grid2D, MhdParams,
                  energy_from)


@dataclass(frozen=True)
class ReconnectionSpec:
    x_r: float = 12.8
    y_r: float = 6.4
    psi0: float = 0.1

    @property
    def k_x(self):
        return np.pi / self.x_r

    @property
    def k_y(self):
        return np.pi / (2.0 * self.y_r)

    def grid(self, nx, ny):
        return Grid2D(nx, ny, -self.x_r, self.x_r, -self.y_r, self.y_r)


@dataclass(frozen=True)
class KhSpec:
    eps_x: float = 0.1
    eps_y: float = 0.1
    v0: float = 0.5
    omega_x: float = 2.0
    omega_y: float = 2.0
    p: float = 0.25
    B_x: float = 0.1
    B_z: float = 10.0
    shear_width: float = 0.1
    L_x: float = 1.0
    L_y: float = 1.0

    def grid(self, nx, ny):
        return Grid2D(nx, ny, -self.L_x / 2, self.L_x / 2, -self.L_y / 2, self.L_y / 2)


def _mesh(grid):
    x, y = grid.cell_centers()
    return np.meshgrid(x, y, indexing="ij")


def reconnection_ic(grid, spec=None, params=None):
    """Harris-type sheet with a single-mode flux perturbation (problems.py:66-87)."""
    spec = spec or ReconnectionSpec()
    params = params or MhdParams()
    X, Y = _mesh(grid)
    th = np.tanh(2.0 * Y)
    rho = 1.2 - th ** 2
    p = 0.5 * rho
    bx = th - spec.psi0 * spec.k_y * np.cos(spec.k_x * X) * np.sin(spec.k_y * Y)
    by = spec.psi0 * spec.k_x * np.sin(spec.k_x * X) * np.cos(spec.k_y * Y)
    zero = 0.0 * X
    U = np.zeros((NVARS, grid.nx, grid.ny))
    U[RHO], U[BX], U[BY] = rho, bx, by
    U[EN] = energy_from(rho, (zero, zero, zero), (bx, by, zero), p, params)
    return U


def kh_ic(grid, spec=None, params=None):
    """Perturbed shear layer in an oblique field (problems.py:90-115)."""
    spec = spec or KhSpec()
    params = params or MhdParams()
    X, Y = _mesh(grid)
    pert = spec.eps_x * np.cos(2.0 * np.pi * spec.omega_x * X / spec.L_x) \
        + spec.eps_y * np.sin(np.pi * (2.0 * spec.omega_y - 1.0) * Y / spec.L_y)
    vx = spec.v0 * np.tanh(Y / spec.shear_width) + pert
    rho = np.ones_like(X)
    bx = np.full_like(X, spec.B_x)
    bz = np.full_like(X, spec.B_z)
    U = np.zeros((NVARS, grid.nx, grid.ny))
    U[RHO] = rho
    U[MX] = rho * vx
    U[BX] = bx
    U[BZ] = bz
    U[EN] = energy_from(rho, (vx, 0.0 * X, 0.0 * X), (bx, 0.0 * X, bz), spec.p, params)
    return U


def default_bc(problem):
    if problem in ("reconnection", "kh"):
        return BoundaryPolicy(x="periodic", y="reflect")
    raise ValueError(f"unknown problem {problem!r}")


def kh_shear_ic(grid, params, seed=1604):
    """BASELINE config 1: vx = 0.5 tanh(y/0.05), Bx = 0.1, rho = p = 1, seeded vy noise.

    vy = 1e-3 U(-1, 1) exp(-y^2 / 0.01) per cell from default_rng(seed).
    """
    X, Y = _mesh(grid)
    rng = np.random.default_rng(seed)
    vx = 0.5 * np.tanh(Y / 0.05)
    vy = 1e-3 * rng.uniform(-1.0, 1.0, X.shape) * np.exp(-Y ** 2 / 0.01)
    rho = np.ones_like(X)
    zero = 0.0 * X
    bx = np.full_like(X, 0.1)
    U = np.zeros((NVARS, grid.nx, grid.ny))
    U[RHO] = rho
    U[MX] = rho * vx
    U[MY] = rho * vy
    U[BX] = bx
    U[EN] = energy_from(rho, (vx, vy, zero), (bx, zero, zero), np.ones_like(X), params)
    return U


def kh_shear_grid(n=256):
    return Grid2D(n, n, 0.0, 1.0, -1.0, 1.0)


def fourier_state(grid, params, seed=1604, modes=16, amplitude=0.1):
    """BASELINE config 2: smooth random 8-field state (SURVEY §8d generator).

    Primitives (rho, vx, vy, vz, Bx, By, Bz, p) with bases (1,0,0,0,1,0,0,1), each
    base + amplitude * (sum of `modes` random-phase Fourier modes) / modes.
    Returns (U, rng) so the caller can draw the Krylov start vector next.
    """
    rng = np.random.default_rng(seed)
    X, Y = _mesh(grid)
    bases = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 1.0)
    prim = []
    for base in bases:
        acc = np.zeros_like(X)
        for _ in range(modes):
            k, l = rng.integers(-4, 5, size=2)
            while k == 0 and l == 0:
                k, l = rng.integers(-4, 5, size=2)
            acc = acc + np.cos(2 * np.pi * (k * X + l * Y) + rng.uniform(0, 2 * np.pi))
        prim.append(base + amplitude * acc / float(modes))
    rho, vx, vy, vz, bx, by, bz, p = prim
    U = np.zeros((NVARS, grid.nx, grid.ny))
    U[RHO] = rho
    U[MX], U[MY], U[MZ] = rho * vx, rho * vy, rho * vz
    U[BX], U[BY], U[BZ] = bx, by, bz
    U[EN] = energy_from(rho, (vx, vy, vz), (bx, by, bz), p, params)
    return U, rng


def fourier_grid(n=1024):
    return Grid2D(n, n, 0.0, 1.0, 0.0, 1.0)


def unit_start_vector(rng, n):
    v = rng.standard_normal(n)
    return v / np.linalg.norm(v)
