"""CPU restatement of the reference's output side (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module; the
product path (paper_1604_02614_b200) never does.

Restates, in NumPy:
* the .mhd25 binary snapshot and its CSV twin (reference pkg/src/expmhd/snapshot.py:1-99):
  96-byte little-endian header, then the state transposed to cell-major (nx, ny, 8);
* explicit classical RK4 with the last step clipped (harness.py:182-199);
* the conservative RK4 step size (harness.py:166-179);
* the harness error norm (harness.py:153-163).
Pinned by tests/test_oracle_golden.py against files and runs of the reference itself
(tests/golden/snapshot_recon16x12.*, rk4_recon32x16.npz).
"""

import struct

import numpy as np

from . import stencil

MAGIC = b"MHD25\x00"
VERSION = 1
# magic, version, nx, ny, 4 bounds, time, gamma mu eta kappa, 8 reserved bytes (snapshot.py:33)
HEADER = struct.Struct("<6sHII4dd4d8x")


def snapshot_bytes(U, grid, time, params):
    """File image of write_snapshot (snapshot.py:43-57)."""
    head = HEADER.pack(MAGIC, VERSION, grid.nx, grid.ny, grid.x_lo, grid.x_hi, grid.y_lo,
                       grid.y_hi, float(time), params.gamma, params.mu, params.eta, params.kappa)
    cells = np.transpose(np.asarray(U, dtype=float), (1, 2, 0)).astype("<f8")
    return head + np.ascontiguousarray(cells).tobytes()


def snapshot_csv(U, grid, time, params):
    """Text of write_snapshot_csv (snapshot.py:83-99): repr() of Python floats."""
    x, y = grid.cell_centers()
    lines = [f"# MHD25 csv time={time!r} nx={grid.nx} ny={grid.ny}",
             f"# domain=[{grid.x_lo!r},{grid.x_hi!r}]x[{grid.y_lo!r},{grid.y_hi!r}]",
             f"# gamma={params.gamma!r} mu={params.mu!r} eta={params.eta!r} kappa={params.kappa!r}",
             "x,y,rho,mx,my,mz,Bx,By,Bz,e"]
    for i in range(grid.nx):
        for j in range(grid.ny):
            row = [float(x[i]), float(y[j])] + [float(U[k, i, j]) for k in range(8)]
            lines.append(",".join(repr(v) for v in row))
    return "\n".join(lines) + "\n"


def rk4_stable_dt(U, grid, params):
    """harness.py:166-179, term by term in the reference's order."""
    rho = U[0]
    v2 = (U[1] ** 2 + U[2] ** 2 + U[3] ** 2) / rho ** 2
    b2 = U[4] ** 2 + U[5] ** 2 + U[6] ** 2
    p = stencil.pressure_field(U, params)
    c_fast = np.sqrt((params.gamma * p + b2) / rho) + np.sqrt(v2)
    h = min(grid.hx, grid.hy)
    dt_wave = 0.3 * h / float(np.max(c_fast))
    diff = max(params.mu, params.eta,
               params.gamma * params.mu * params.kappa / (params.gamma - 1.0), 1e-30)
    return min(dt_wave, 0.2 * h * h / diff)


def rk4(f, y0, t0, t_end, h):
    """Classical RK4, last step clipped (harness.py:182-199); returns (y, steps, rhs_evals)."""
    y = np.array(y0, dtype=float)
    t = t0
    steps = 0
    while t < t_end - 1e-14 * max(1.0, abs(t_end)):
        dt = min(h, t_end - t)
        k1 = f(y)
        k2 = f(y + 0.5 * dt * k1)
        k3 = f(y + 0.5 * dt * k2)
        k4 = f(y + dt * k3)
        y = y + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        t += dt
        steps += 1
    return y, steps, 4 * steps


def error_norm(U, U_ref, grid):
    """max_f sqrt(sum (U_f - R_f)^2 * hx * hy) (harness.py:153-163)."""
    d = np.asarray(U) - np.asarray(U_ref)
    return float(np.max(np.sqrt(np.sum(d * d, axis=(1, 2)) * (grid.hx * grid.hy))))
