"""Pin the CPU oracle (oracle/) against the reference's golden fixtures (CPU only)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, Obj, case_objects, golden
from oracle import epirk_cpu, jvp, krylov_cpu, stencil


def test_rhs_bitwise_all_cases():
    z = golden("rhs_jv_cases.npz")
    for k in range(int(z["ncases"][0])):
        g, P, bc = case_objects(z, k)
        F = stencil.mhd_rhs(z[f"c{k}_U"], P, g, bc)
        assert np.array_equal(F, z[f"c{k}_F"]), f"case {k}"


def test_jv_bitwise_all_cases():
    z = golden("rhs_jv_cases.npz")
    for k in range(int(z["ncases"][0])):
        g, P, bc = case_objects(z, k)
        f = stencil.rhs_closure(P, g, bc)
        op = jvp.FdJv(f, z[f"c{k}_U"].reshape(-1))
        assert np.array_equal(op(z[f"c{k}_v"]), z[f"c{k}_Jv"]), f"case {k}"
        assert np.array_equal(op(z[f"c{k}_vsmall"]), z[f"c{k}_Jvsmall"]), f"case {k} small"


def test_jv_zero_direction_no_rhs_call():
    calls = []

    def f(y):
        calls.append(1)
        return y * 2.0
    op = jvp.FdJv(f, np.ones(4))
    assert np.all(op(np.zeros(4)) == 0.0)
    assert len(calls) == 1


def test_admissibility_messages_match_reference():
    with open(os.path.join(GOLDEN, "errors.json")) as fh:
        errs = json.load(fh)
    from paper_1604_02614_b200.mhd import BoundaryPolicy, Grid2D, MhdParams
    g = Grid2D(6, 5, 0.0, 1.0, 0.0, 1.0)
    for key, bc in (("density", BoundaryPolicy("periodic", "reflect")),
                    ("pressure", BoundaryPolicy("reflect", "zero-gradient"))):
        U = np.array(errs[key]["U"])
        with pytest.raises(stencil.InadmissibleState) as info:
            stencil.mhd_rhs(U, MhdParams(), g, bc)
        assert str(info.value) == errs[key]["msg"]


def test_config0_one_step_and_counters():
    z = golden("config0_recon64.npz")
    with open(os.path.join(GOLDEN, "config0_stats.json")) as fh:
        st = json.load(fh)["step1"]
    from paper_1604_02614_b200.problems import ReconnectionSpec, default_bc
    from paper_1604_02614_b200.mhd import MhdParams
    g = ReconnectionSpec().grid(64, 64)
    P = MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    f = stencil.rhs_closure(P, g, default_bc("reconnection"))
    y1, T = epirk_cpu.step4(f, z["U0"].reshape(-1), 0.1, 1e-10)
    rel = np.linalg.norm(y1 - z["y1"]) / np.linalg.norm(z["y1"])
    assert rel <= 1e-10
    for k, v in st.items():
        assert getattr(T, k) == v, k


def test_arnoldi_dense_matches_reference():
    z = golden("krylov_dense.npz")
    A = z["A"]

    class Op:
        n = A.shape[0]

        def __call__(self, v):
            return A @ v
    proc = krylov_cpu.arnoldi(Op(), z["v"], 8)
    V, H = proc.snapshot()
    assert np.max(np.abs(H - z["H"])) <= 1e-12
    assert np.max(np.abs(V - z["V"])) <= 1e-12


def test_phi_block_matches_reference():
    z = golden("krylov_dense.npz")
    for k in range(4):
        got = np.stack(krylov_cpu.phi_block(4, z[f"phiM{k}"]))
        want = z[f"phi{k}"]
        assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))


def test_multiscale_and_phicomb_dense():
    z = golden("krylov_dense.npz")
    A = z["A"]

    class Op:
        n = A.shape[0]

        def __call__(self, v):
            return A @ v
    outs, c = krylov_cpu.multi_scale(Op(), 0.9, z["v"], [0.5, 2.0 / 3.0, 1.0], 1e-11)
    assert np.max(np.abs(np.stack(outs) - z["ms_out"])) <= 1e-12
    assert [c.operator_applies, c.substeps, c.max_basis_size, c.projections] == list(z["ms_stats"])
    vecs = list(z["pc_vecs"])
    w, c = krylov_cpu.phi_combination(Op(), 1.3, 0.8, vecs, 1e-10)
    assert np.max(np.abs(w - z["pc_w"])) <= 1e-12
    assert [c.operator_applies, c.substeps, c.max_basis_size, c.projections] == list(z["pc_stats"])
    w, c = krylov_cpu.phi_combination(Op(), 1.0, 1.0, vecs, 1e-8,
                                      krylov_cpu.Knobs(m_max=15, max_substep=0.25))
    assert np.max(np.abs(w - z["pc_w_sub"])) <= 1e-12
    assert [c.operator_applies, c.substeps, c.max_basis_size, c.projections] == list(z["pc_stats_sub"])


def test_krylov_mhd_fd_operator():
    z = golden("krylov_mhd.npz")
    gt, pt = z["grid"], z["params"]
    g = Obj(nx=int(gt[0]), ny=int(gt[1]), hx=(gt[3] - gt[2]) / gt[0], hy=(gt[5] - gt[4]) / gt[1])
    P = Obj(mu=pt[0], eta=pt[1], kappa=pt[2], gamma=pt[3], b_half=bool(pt[4]))
    bc = Obj(x="periodic", y="reflect")
    f = stencil.rhs_closure(P, g, bc)
    assert np.array_equal(f(z["a"]), z["fa"])
    op = jvp.FdJv(f, z["a"], z["fa"])
    proc = krylov_cpu.arnoldi(op, z["v"], 12)
    V, H = proc.snapshot()
    assert np.linalg.norm(H - z["H"]) <= 1e-8 * np.linalg.norm(z["H"])
    outs, c = krylov_cpu.multi_scale(op, 0.5, 0.5 * z["fa"], [0.5, 2.0 / 3.0, 1.0], 1e-10)
    assert [c.operator_applies, c.substeps, c.max_basis_size] == list(z["ms_stats"])
    rel = np.linalg.norm(np.stack(outs) - z["ms_out"]) / np.linalg.norm(z["ms_out"])
    assert rel <= 1e-9


def test_epirk5p1_adaptive_kh32():
    z = golden("epirk5p1_kh32.npz")
    with open(os.path.join(GOLDEN, "epirk5p1_kh32.json")) as fh:
        st = json.load(fh)
    from paper_1604_02614_b200.problems import kh_shear_grid
    from paper_1604_02614_b200.mhd import BoundaryPolicy, MhdParams
    g = kh_shear_grid(32)
    f = stencil.rhs_closure(MhdParams(mu=1e-4, eta=1e-4, kappa=1e-4), g,
                            BoundaryPolicy("periodic", "reflect"))
    y, T = epirk_cpu.run_adaptive(f, z["U0"].reshape(-1), 0.0, 0.05, epirk_cpu.Controller(tol=1e-6))
    assert np.linalg.norm(y - z["y"]) <= 1e-10 * np.linalg.norm(z["y"])
    for k, v in st.items():
        assert getattr(T, k) == v, k


def test_config1_full_size_first_steps():
    """The oracle on BASELINE config 1 at its own size (KH shear 256^2, EpiRK5P1 tol 1e-6) for
    the first four adaptive steps, against the unmodified reference's run (~45 s on one core)."""
    z = golden("config1_kh256_short.npz")
    with open(os.path.join(GOLDEN, "config1_kh256_short.json")) as fh:
        st = json.load(fh)
    from paper_1604_02614_b200.problems import kh_shear_grid, kh_shear_ic
    from paper_1604_02614_b200.mhd import BoundaryPolicy, MhdParams
    g = kh_shear_grid(256)
    prm = MhdParams(mu=1e-4, eta=1e-4, kappa=1e-4)
    f = stencil.rhs_closure(prm, g, BoundaryPolicy("periodic", "reflect"))
    U0 = kh_shear_ic(g, prm)
    y, T = epirk_cpu.run_adaptive(f, U0.reshape(-1), 0.0, float(z["t_end"][0]), epirk_cpu.Controller(tol=1e-6))
    assert np.linalg.norm(y[::64] - z["y_sub"]) <= 1e-10 * np.linalg.norm(z["y_sub"])
    assert abs(np.linalg.norm(y) - float(z["y_norm"][0])) <= 1e-11 * float(z["y_norm"][0])
    for k, v in st.items():
        assert getattr(T, k) == v, k


@pytest.mark.slow
def test_config0_full_trajectory():
    z = golden("config0_recon64.npz")
    with open(os.path.join(GOLDEN, "config0_stats.json")) as fh:
        st = json.load(fh)["run20"]
    from paper_1604_02614_b200.problems import ReconnectionSpec, default_bc
    from paper_1604_02614_b200.mhd import MhdParams
    g = ReconnectionSpec().grid(64, 64)
    f = stencil.rhs_closure(MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3), g, default_bc("reconnection"))
    y, T = epirk_cpu.run_fixed("epirk4", f, z["U0"].reshape(-1), 0.0, 2.0, 0.1, tol=1e-10)
    assert np.linalg.norm(y - z["y20"]) <= 1e-9 * np.linalg.norm(z["y20"])
    for k, v in st.items():
        assert getattr(T, k) == v, k


def test_divergence_oracle_bitwise():
    z = golden("rhs_jv_cases.npz")
    for k in range(int(z["ncases"][0])):
        g, P, bc = case_objects(z, k)
        d, peak = stencil.divergence_B(z[f"c{k}_U"], g, bc)
        assert np.array_equal(d, z[f"c{k}_divB"]) and peak == z[f"c{k}_divBmax"][0]


def test_harness_oracle_matches_reference_outputs():
    """oracle/harness_cpu.py against the reference's own snapshot files and RK4 run."""
    from oracle import harness_cpu as H
    from paper_1604_02614_b200.mhd import MhdParams
    from paper_1604_02614_b200.problems import ReconnectionSpec, default_bc
    U = np.load(os.path.join(GOLDEN, "snapshot_recon16x12_U.npy"))
    g = ReconnectionSpec().grid(16, 12)
    P = MhdParams(mu=1e-3, eta=2e-3, kappa=3e-3)
    with open(os.path.join(GOLDEN, "snapshot_recon16x12.mhd25"), "rb") as fh:
        assert H.snapshot_bytes(U, g, 0.75, P) == fh.read()
    with open(os.path.join(GOLDEN, "snapshot_recon16x12.csv")) as fh:
        assert H.snapshot_csv(U, g, 0.75, P) == fh.read()
    z = golden("rk4_recon32x16.npz")
    g = ReconnectionSpec().grid(32, 16)
    P = MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    dt = H.rk4_stable_dt(z["U0"], g, P)
    assert dt == z["scal"][0]
    f = stencil.rhs_closure(P, g, default_bc("reconnection"))
    y, steps, evals = H.rk4(f, z["U0"].reshape(-1), 0.0, z["scal"][1], dt)
    assert np.array_equal(y, z["y"]) and [steps, evals] == list(z["counts"])
    assert H.error_norm(y.reshape(8, 32, 16), z["U0"], g) == z["scal"][2]


def test_snapshot_header_parsing_host_logic():
    """The product's header parser (host logic, no GPU) on the reference file and broken ones."""
    from paper_1604_02614_b200.snapshot import HEADER_SIZE, SnapshotFormatError, _parse_header
    with open(os.path.join(GOLDEN, "snapshot_recon16x12.mhd25"), "rb") as fh:
        raw = fh.read()
    grid, t, P = _parse_header("f", raw[:HEADER_SIZE])
    assert (grid.nx, grid.ny, t, P.mu, P.eta, P.kappa) == (16, 12, 0.75, 1e-3, 2e-3, 3e-3)
    assert (grid.x_lo, grid.x_hi, grid.y_lo, grid.y_hi) == (-12.8, 12.8, -6.4, 6.4)
    for blob, msg in ((raw[:95], "truncated header"), (b"MHD26\x00" + raw[6:96], "bad magic"),
                      (raw[:6] + b"\x07\x00" + raw[8:96], "unsupported version 7")):
        with pytest.raises(SnapshotFormatError, match=msg):
            _parse_header("f", blob)
