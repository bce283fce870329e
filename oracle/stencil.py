"""Oracle: 2.5D resistive-MHD right-hand side, restated cell-primitive first.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Restates reference ``pkg/src/expmhd/mhd.py``:

* ghost fill            ``apply_ghosts``      mhd.py:144-171
* pressure + admissibility ``pressure``       mhd.py:106-131
* ideal-MHD fluxes      ``hyperbolic_flux``   mhd.py:174-197
* centred differences   ``_ddx`` / ``_ddy``   mhd.py:200-206
* diffusive fluxes      ``diffusive_flux``    mhd.py:209-266
* divergence / closure  ``rhs`` / ``make_rhs`` mhd.py:269-285

The arithmetic is written in exactly the reference's evaluation order
(NumPy evaluates ``a + b + c`` as ``(a + b) + c`` and never contracts into
FMA), so the result is bit-identical to the reference.  The structure is
different: ghosts come from an index map per axis, primitives are computed
once on the padded field and shared by both flux families.

Grid / params / bc arguments are duck-typed: anything with ``nx, ny, hx, hy``;
``mu, eta, kappa, gamma, b_half``; and ``x, y`` policy strings.
"""

import numpy as np

NF = 8
I_RHO, I_MX, I_MY, I_MZ, I_BX, I_BY, I_BZ, I_EN = range(NF)
FLIP_X = (I_MX, I_BX)     # odd under a mirror in x (mhd.py:23)
FLIP_Y = (I_MY, I_BY)     # odd under a mirror in y (mhd.py:24)


class InadmissibleState(ValueError):
    """Oracle-side twin of the reference ``AdmissibilityError`` (mhd.py:27)."""


def axis_map(n, width, policy):
    """(source index, mirrored?) for every padded position -width..n+width-1.

    periodic -> np.pad 'wrap', zero-gradient -> 'edge', reflect -> 'symmetric'
    (the edge cell is repeated: ghosts [U1, U0 | U0 .. Un-1 | Un-1, Un-2]).
    """
    k = np.arange(-width, n + width)
    if policy == "periodic":
        return k % n, np.zeros(k.shape, bool)
    if policy == "zero-gradient":
        return np.clip(k, 0, n - 1), np.zeros(k.shape, bool)
    if policy == "reflect":
        src = np.where(k < 0, -k - 1, np.where(k >= n, 2 * n - 1 - k, k))
        return src, (k < 0) | (k >= n)
    raise ValueError(f"unknown boundary policy {policy!r}")


def pad_state(U, bc, width=2):
    """Ghost-padded copy of U (8, nx, ny) -> (8, nx+2w, ny+2w)."""
    _, nx, ny = U.shape
    sx, mx = axis_map(nx, width, bc.x)
    sy, my = axis_map(ny, width, bc.y)
    P = U[:, sx, :][:, :, sy]
    for c in FLIP_X:
        P[c, mx, :] *= -1.0
    for c in FLIP_Y:
        P[c, :, my] *= -1.0
    return P


def _first_min_cell(a):
    flat = int(np.argmin(a))
    return tuple(int(t) for t in np.unravel_index(flat, a.shape))


class Primitives:
    """Per-cell primitives of a (padded) conserved field, computed once."""

    def __init__(self, P, params, check=True):
        rho = P[I_RHO]
        if check and np.any(rho <= 0.0):
            c = _first_min_cell(rho)
            raise InadmissibleState(f"non-positive density at cell {c}: {rho[c]}")
        m2 = P[I_MX] ** 2 + P[I_MY] ** 2 + P[I_MZ] ** 2
        b2 = P[I_BX] ** 2 + P[I_BY] ** 2 + P[I_BZ] ** 2
        kinetic = 0.5 * m2 / rho
        magnetic = 0.5 * b2 if params.b_half else b2
        p = (params.gamma - 1.0) * (P[I_EN] - kinetic - magnetic)
        if check and np.any(p <= 0.0):
            c = _first_min_cell(p)
            raise InadmissibleState(f"non-positive pressure at cell {c}: {p[c]}")
        self.U = P
        self.rho = rho
        self.vel = P[I_MX:I_MZ + 1] / rho
        self.mag = P[I_BX:I_BZ + 1]
        self.p = p
        # total pressure always carries |B|^2/2, independent of b_half (mhd.py:180)
        self.ptot = p + 0.5 * b2
        self.temp = p / rho


def pressure_field(U, params, check=True):
    """Reference ``pressure`` (mhd.py:116-131) on an unpadded field."""
    return Primitives(U, params, check).p


def ideal_flux(pr):
    """Ideal-MHD (x, y) flux pair on every cell of ``pr`` (mhd.py:174-197)."""
    U, rho, v, B, ptot = pr.U, pr.rho, pr.vel, pr.mag, pr.ptot
    bv = B[0] * v[0] + B[1] * v[1] + B[2] * v[2]
    out = []
    for a in (0, 1):                     # flux direction x, y
        F = np.empty_like(U)
        F[I_RHO] = U[I_MX + a]
        for d in range(3):
            F[I_MX + d] = rho * v[d] * v[a] - B[d] * B[a]
            F[I_BX + d] = v[a] * B[d] - B[a] * v[d]
        F[I_MX + a] += ptot
        F[I_EN] = (U[I_EN] + ptot) * v[a] - B[a] * bv
        out.append(F)
    return out[0], out[1]


def dx_c(f, hx):
    """Centred x-difference, shrinking both axes by one (mhd.py:200-202)."""
    return (f[..., 2:, 1:-1] - f[..., :-2, 1:-1]) / (2.0 * hx)


def dy_c(f, hy):
    """Centred y-difference, shrinking both axes by one (mhd.py:205-206)."""
    return (f[..., 1:-1, 2:] - f[..., 1:-1, :-2]) / (2.0 * hy)


def viscous_resistive_flux(pr, params, hx, hy):
    """Diffusive (x, y) flux on the once-shrunk field (mhd.py:209-266)."""
    mu, eta, kap, g = params.mu, params.eta, params.kappa, params.gamma
    gv_x, gv_y = dx_c(pr.vel, hx), dy_c(pr.vel, hy)
    gb_x, gb_y = dx_c(pr.mag, hx), dy_c(pr.mag, hy)
    gt_x, gt_y = dx_c(pr.temp, hx), dy_c(pr.temp, hy)
    vc = pr.vel[:, 1:-1, 1:-1]
    bc = pr.mag[:, 1:-1, 1:-1]

    div_v = gv_x[0] + gv_y[1]
    s_xx = 2.0 * gv_x[0] - (2.0 / 3.0) * div_v
    s_yy = 2.0 * gv_y[1] - (2.0 / 3.0) * div_v
    s_xy = gv_y[0] + gv_x[1]
    s_zx, s_zy = gv_x[2], gv_y[2]
    curl_z = gb_x[1] - gb_y[0]

    Fx = np.zeros((NF,) + div_v.shape)
    Fy = np.zeros((NF,) + div_v.shape)
    Fx[I_MX], Fx[I_MY], Fx[I_MZ] = mu * s_xx, mu * s_xy, mu * s_zx
    Fy[I_MX], Fy[I_MY], Fy[I_MZ] = mu * s_xy, mu * s_yy, mu * s_zy
    Fx[I_BY] = eta * curl_z
    Fy[I_BX] = -Fx[I_BY]
    Fx[I_BZ] = eta * gb_x[2]
    Fy[I_BZ] = eta * gb_y[2]

    k_heat = g * mu * kap / (g - 1.0)
    Fx[I_EN] = mu * (s_xx * vc[0] + s_xy * vc[1] + s_zx * vc[2]) \
        + k_heat * gt_x \
        + eta * (bc[1] * curl_z + bc[2] * gb_x[2])
    Fy[I_EN] = mu * (s_xy * vc[0] + s_yy * vc[1] + s_zy * vc[2]) \
        + k_heat * gt_y \
        + eta * (bc[0] * (gb_y[0] - gb_x[1]) + bc[2] * gb_y[2])
    return Fx, Fy


def mhd_rhs(U, params, grid, bc, check=True):
    """dU/dt for U of shape (8, nx, ny) (reference ``rhs``, mhd.py:269-277)."""
    pr = Primitives(pad_state(np.asarray(U, dtype=float), bc, 2), params, check)
    hx, hy = grid.hx, grid.hy
    Hx, Hy = ideal_flux(pr)
    Dx, Dy = viscous_resistive_flux(pr, params, hx, hy)
    Gx = Hx[:, 1:-1, 1:-1] - Dx
    Gy = Hy[:, 1:-1, 1:-1] - Dy
    return -dx_c(Gx, hx) - dy_c(Gy, hy)


def rhs_closure(params, grid, bc, check=True):
    """Flat-vector closure (reference ``make_rhs``, mhd.py:280-285)."""
    shape = (NF, grid.nx, grid.ny)

    def f(y):
        U = np.asarray(y, dtype=float).reshape(shape)
        return np.ascontiguousarray(mhd_rhs(U, params, grid, bc, check)).reshape(-1)
    return f


def divergence_B(U, grid, bc):
    """Centred div B field and its max |.| (reference ``div_B``, mhd.py:288-296)."""
    P = pad_state(np.asarray(U, dtype=float), bc, 1)
    d = (P[I_BX, 2:, 1:-1] - P[I_BX, :-2, 1:-1]) / (2.0 * grid.hx) \
        + (P[I_BY, 1:-1, 2:] - P[I_BY, 1:-1, :-2]) / (2.0 * grid.hy)
    return d, float(np.max(np.abs(d)))


def mhd_rhs_slab(U_local, halo_lo, halo_hi, params, grid, bc, check=True):
    """RHS of an x-slab whose x-ghost rows are given explicitly (None: boundary policy).

    Oracle for the slab decomposition: the padded field is [halo_lo | U_local |
    halo_hi] along x, then y-padded exactly as ``pad_state`` would, so for
    consistent halos the result equals the matching rows of ``mhd_rhs``.
    """
    U_local = np.asarray(U_local, dtype=float)
    _, nxl, ny = U_local.shape
    sx, mx = axis_map(nxl, 2, bc.x)
    Px = U_local[:, sx, :].copy()
    for c in FLIP_X:
        Px[c, mx, :] *= -1.0
    if halo_lo is not None:
        Px[:, :2, :] = halo_lo
    if halo_hi is not None:
        Px[:, -2:, :] = halo_hi
    sy, my = axis_map(ny, 2, bc.y)
    P = Px[:, :, sy]
    for c in FLIP_Y:
        P[c, :, my] *= -1.0
    pr = Primitives(P, params, check)
    hx, hy = grid.hx, grid.hy
    Hx, Hy = ideal_flux(pr)
    Dx, Dy = viscous_resistive_flux(pr, params, hx, hy)
    Gx = Hx[:, 1:-1, 1:-1] - Dx
    Gy = Hy[:, 1:-1, 1:-1] - Dy
    return -dx_c(Gx, hx) - dy_c(Gy, hy)
