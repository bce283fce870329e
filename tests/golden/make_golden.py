"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

It imports ``expmhd`` from /root/reference/pkg/src and writes small .npz /
.json fixtures next to this file.  Nothing in the GPU tests reads
/root/reference; they read these committed fixtures.  Inputs are seeded
synthetic states (the reference ships no data), generated here with the
reference's own problem builders where it has them.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import expmhd as R  # noqa: E402
from expmhd import mhd as Rm  # noqa: E402


def rand_state(rng, nx, ny, emin=40.0):
    U = np.zeros((8, nx, ny))
    U[0] = 1.0 + 0.3 * rng.random((nx, ny))
    U[1:4] = 0.3 * rng.standard_normal((3, nx, ny))
    U[4:7] = rng.standard_normal((3, nx, ny))
    U[7] = emin + rng.random((nx, ny))
    return U


def params_tuple(P):
    return np.array([P.mu, P.eta, P.kappa, P.gamma, float(P.b_half)])


def grid_tuple(g):
    return np.array([g.nx, g.ny, g.x_lo, g.x_hi, g.y_lo, g.y_hi], dtype=float)


BCS = {"periodic": 0, "reflect": 1, "zero-gradient": 2}


def rhs_cases():
    rng = np.random.default_rng(20160408)
    cases = {}
    specs = [
        (16, 12, "periodic", "reflect", True, (1e-2, 3e-3, 2e-2)),
        (12, 16, "reflect", "zero-gradient", False, (1e-2, 3e-3, 2e-2)),
        (8, 8, "zero-gradient", "periodic", True, (0.0, 0.0, 0.0)),
        (40, 70, "periodic", "periodic", True, (1e-3, 1e-3, 1e-3)),
        (33, 130, "periodic", "reflect", True, (2e-2, 1e-2, 3e-2)),
        (130, 37, "reflect", "reflect", False, (1e-4, 5e-4, 1e-3)),
    ]
    for k, (nx, ny, bx, by, bh, (mu, eta, kap)) in enumerate(specs):
        g = R.Grid2D(nx, ny, -1.0, 2.0, -0.7, 0.9)
        bc = R.BoundaryPolicy(bx, by)
        P = R.MhdParams(mu=mu, eta=eta, kappa=kap, b_half=bh)
        U = rand_state(rng, nx, ny)
        F = Rm.rhs(U, P, g, bc)
        cases[f"c{k}_U"] = U
        cases[f"c{k}_F"] = F
        cases[f"c{k}_grid"] = grid_tuple(g)
        cases[f"c{k}_params"] = params_tuple(P)
        cases[f"c{k}_bc"] = np.array([BCS[bx], BCS[by]])
        # Jv on the same state
        f = R.make_rhs(P, g, bc)
        a = U.reshape(-1)
        v = rng.standard_normal(a.size)
        op = R.FdJacobianOperator(f, a)
        cases[f"c{k}_v"] = v
        cases[f"c{k}_Jv"] = op(v)
        small = v * (0.25 * R.fdjac.SQRT_EPS / np.max(np.abs(v)))   # unscaled branch (sigma = 1)
        cases[f"c{k}_vsmall"] = small
        cases[f"c{k}_Jvsmall"] = op(small)
        d, peak = Rm.div_B(U, g, bc)                     # diagnostics (mhd.py:288-309)
        cases[f"c{k}_divB"] = d
        cases[f"c{k}_divBmax"] = np.array([peak])
        cases[f"c{k}_J"] = Rm.current_J(U, g, bc)
    cases["ncases"] = np.array([len(specs)])
    np.savez_compressed(os.path.join(OUT, "rhs_jv_cases.npz"), **cases)


def config0():
    spec = R.ReconnectionSpec()
    g = spec.grid(64, 64)
    P = R.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    bc = R.default_bc("reconnection")
    U0 = R.reconnection_ic(g, params=P)
    f = R.make_rhs(P, g, bc)
    y0 = U0.reshape(-1)
    F0 = f(y0)
    y, st = R.integrate_fixed("epirk4", f, y0, 0.0, 2.0, 0.1, tol_krylov=1e-10)
    y1, st1 = R.epirk4_step(f, y0, 0.1, 1e-10)
    np.savez_compressed(os.path.join(OUT, "config0_recon64.npz"), U0=U0, F0=F0, y20=y, y1=y1)
    keys = ["steps_accepted", "steps_rejected", "projections", "rhs_evals", "operator_applies",
            "substeps", "max_basis_size"]
    with open(os.path.join(OUT, "config0_stats.json"), "w") as fh:
        json.dump({"run20": {k: getattr(st, k) for k in keys},
                   "step1": {k: getattr(st1, k) for k in keys}}, fh, indent=1)


def krylov_dense():
    rng = np.random.default_rng(11)
    out = {}
    n = 12
    A = rng.standard_normal((n, n))
    A = 3.0 * (A - (np.abs(A).sum() / n) * np.eye(n)) / np.linalg.norm(A)
    v = rng.standard_normal(n)
    b = R.arnoldi(R.LinearOperator.from_matrix(A), v, 8)
    out.update(A=A, v=v, V=b.V, H=b.H, beta=np.array([b.beta]))
    # phi_dense of a few matrices
    for k, scale in enumerate((0.05, 0.7, 3.0, 40.0)):
        M = scale * rng.standard_normal((6, 6))
        out[f"phiM{k}"] = M
        out[f"phi{k}"] = np.stack(R.phi_dense(4, M))
    # multi-scale and phi_comb on the dense operator
    op = R.LinearOperator.from_matrix(A)
    outs, st = R.multi_scale_eval(op, 0.9, v, [0.5, 2.0 / 3.0, 1.0], 1e-11)
    out["ms_out"] = np.stack(outs)
    out["ms_stats"] = np.array([st.operator_applies, st.substeps, st.max_basis_size, st.projections])
    vecs = [rng.standard_normal(n) for _ in range(3)]
    out["pc_vecs"] = np.stack(vecs)
    w, st = R.phi_comb(R.PhiCombRequest(operator=op, h=1.3, c=0.8, vectors=vecs, tol=1e-10))
    out["pc_w"] = w
    out["pc_stats"] = np.array([st.operator_applies, st.substeps, st.max_basis_size, st.projections])
    w2, st2 = R.phi_comb(R.PhiCombRequest(operator=op, h=1.0, c=1.0, vectors=vecs, tol=1e-8),
                         R.KrylovConfig(m_max=n + 3, max_substep=0.25))
    out["pc_w_sub"] = w2
    out["pc_stats_sub"] = np.array([st2.operator_applies, st2.substeps, st2.max_basis_size,
                                    st2.projections])
    np.savez_compressed(os.path.join(OUT, "krylov_dense.npz"), **out)


def krylov_mhd():
    """Arnoldi / multi-scale / phi_comb with the FD Jacobian of the MHD RHS (32 x 16)."""
    spec = R.ReconnectionSpec()
    g = spec.grid(32, 16)
    P = R.MhdParams(mu=1e-2, eta=1e-3, kappa=1e-2)
    bc = R.default_bc("reconnection")
    U = R.reconnection_ic(g, params=P)
    f = R.make_rhs(P, g, bc)
    a = U.reshape(-1)
    fa = f(a)
    op = R.FdJacobianOperator(f, a, fa)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(a.size)
    b = R.arnoldi(op, v, 12)
    outs, st = R.multi_scale_eval(op, 0.5, 0.5 * fa, [0.5, 2.0 / 3.0, 1.0], 1e-10)
    vec3 = rng.standard_normal(a.size) * 1e-3
    w, st2 = R.phi_comb(R.PhiCombRequest(operator=op, h=0.5, c=1.0,
                                         vectors=[np.zeros(a.size), np.zeros(a.size), vec3, 0.5 * vec3],
                                         tol=1e-10))
    np.savez_compressed(os.path.join(OUT, "krylov_mhd.npz"), a=a, fa=fa, v=v, H=b.H,
                        beta=np.array([b.beta]), V=b.V, ms_out=np.stack(outs),
                        ms_stats=np.array([st.operator_applies, st.substeps, st.max_basis_size]),
                        vec3=vec3, pc_w=w,
                        pc_stats=np.array([st2.operator_applies, st2.substeps, st2.max_basis_size]),
                        grid=grid_tuple(g), params=params_tuple(P))


def epirk_small():
    """EpiRK5P1 adaptive on a downscaled config 1 (KH shear, 32 x 32) for a few steps."""
    sys.path.insert(0, os.path.join(OUT, "..", ".."))
    from paper_1604_02614_b200.problems import kh_shear_grid, kh_shear_ic  # host-only builder
    g0 = kh_shear_grid(32)
    g = R.Grid2D(g0.nx, g0.ny, g0.x_lo, g0.x_hi, g0.y_lo, g0.y_hi)
    P = R.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-4)
    bc = R.BoundaryPolicy("periodic", "reflect")
    U0 = kh_shear_ic(g0, P)
    f = R.make_rhs(P, g, bc)
    ctl = R.StepController(tol=1e-6)
    y, st = R.integrate_adaptive(f, U0.reshape(-1), 0.0, 0.05, ctl)
    keys = ["steps_accepted", "steps_rejected", "projections", "rhs_evals", "operator_applies",
            "substeps", "max_basis_size"]
    np.savez_compressed(os.path.join(OUT, "epirk5p1_kh32.npz"), U0=U0, y=y)
    with open(os.path.join(OUT, "epirk5p1_kh32.json"), "w") as fh:
        json.dump({k: getattr(st, k) for k in keys}, fh, indent=1)


def config1_256(t_end=0.03):
    """BASELINE config 1 at its full size (KH shear 256 x 256, EpiRK5P1 tol 1e-6) for the first
    few adaptive steps (t <= 0.03: ~1 min of the reference on one core).  The 4 MB state is not
    committed: the fixture holds every 64th entry of the result, its norm and the counters; the
    initial condition is rebuilt by the same host builder the test uses."""
    sys.path.insert(0, os.path.join(OUT, "..", ".."))
    from paper_1604_02614_b200.problems import kh_shear_grid, kh_shear_ic
    g0 = kh_shear_grid(256)
    g = R.Grid2D(g0.nx, g0.ny, g0.x_lo, g0.x_hi, g0.y_lo, g0.y_hi)
    P = R.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-4)
    bc = R.BoundaryPolicy("periodic", "reflect")
    U0 = kh_shear_ic(g0, P)
    f = R.make_rhs(P, g, bc)
    y, st = R.integrate_adaptive(f, U0.reshape(-1), 0.0, t_end, R.StepController(tol=1e-6))
    keys = ["steps_accepted", "steps_rejected", "projections", "rhs_evals", "operator_applies",
            "substeps", "max_basis_size"]
    np.savez_compressed(os.path.join(OUT, "config1_kh256_short.npz"), y_sub=y[::64],
                        y_norm=np.array([np.linalg.norm(y)]), u0_norm=np.array([np.linalg.norm(U0)]),
                        t_end=np.array([t_end]))
    with open(os.path.join(OUT, "config1_kh256_short.json"), "w") as fh:
        json.dump({k: getattr(st, k) for k in keys}, fh, indent=1)


def errors():
    out = {}
    g = R.Grid2D(6, 5, 0.0, 1.0, 0.0, 1.0)
    P = R.MhdParams()
    rng = np.random.default_rng(3)
    U = rand_state(rng, 6, 5)
    U[0, 4, 1] = -0.5
    try:
        Rm.rhs(U, P, g, R.BoundaryPolicy("periodic", "reflect"))
    except R.AdmissibilityError as e:
        out["density"] = {"U": U.tolist(), "msg": str(e)}
    U = rand_state(rng, 6, 5)
    U[7, 2, 3] = 0.01
    try:
        Rm.rhs(U, P, g, R.BoundaryPolicy("reflect", "zero-gradient"))
    except R.AdmissibilityError as e:
        out["pressure"] = {"U": U.tolist(), "msg": str(e)}
    with open(os.path.join(OUT, "errors.json"), "w") as fh:
        json.dump(out, fh)


def harness_fixtures():
    """Output side: .mhd25 / CSV snapshots written by the reference's
    own writer, and a short explicit-RK4 run with the reference's stable step."""
    from expmhd import harness as Rh
    from expmhd import snapshot as Rs
    from expmhd.problems import ReconnectionSpec, reconnection_ic
    P = R.MhdParams(mu=1e-3, eta=2e-3, kappa=3e-3)
    g = ReconnectionSpec().grid(16, 12)
    U = reconnection_ic(g, params=P)
    U = U + 1e-3 * np.random.default_rng(11).standard_normal(U.shape)
    Rs.write_snapshot(os.path.join(OUT, "snapshot_recon16x12.mhd25"), U, g, 0.75, P)
    Rs.write_snapshot_csv(os.path.join(OUT, "snapshot_recon16x12.csv"), U, g, 0.75, P)
    np.save(os.path.join(OUT, "snapshot_recon16x12_U.npy"), U)

    g = ReconnectionSpec().grid(32, 16)
    P = R.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    U0 = reconnection_ic(g, params=P)
    dt = Rh._rk4_stable_dt(U0, g, P)
    f = Rm.make_rhs(P, g, R.default_bc("reconnection"))
    y, st = Rh.integrate_rk4(f, Rm.state_to_vector(U0), 0.0, 7.3 * dt, dt)
    err = Rh.error_norm(Rm.vector_to_state(y, g), U0, g)
    np.savez_compressed(os.path.join(OUT, "rk4_recon32x16.npz"), U0=U0, y=y,
                        scal=np.array([dt, 7.3 * dt, err]),
                        counts=np.array([st.steps_accepted, st.rhs_evals]))


if __name__ == "__main__":
    if sys.argv[1:] == ["harness"]:
        harness_fixtures()
    elif sys.argv[1:] == ["config1"]:
        config1_256()
    else:
        rhs_cases()
        config0()
        krylov_dense()
        krylov_mhd()
        epirk_small()
        config1_256()
        errors()
        harness_fixtures()
    print("fixtures written to", OUT)
