"""Output side on the GPU: .mhd25 snapshots of device states are
byte-identical to the reference writer's; explicit RK4, its stable step and the harness error
norm reproduce the reference's own run (tests/golden/rk4_recon32x16.npz) bit for bit."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden
from oracle import harness_cpu, stencil

pytestmark = pytest.mark.gpu

SNAP = f"{GOLDEN}/snapshot_recon16x12"


def _snap_case():
    import paper_1604_02614_b200 as P
    U = np.load(SNAP + "_U.npy")
    return P, U, P.ReconnectionSpec().grid(16, 12), P.MhdParams(mu=1e-3, eta=2e-3, kappa=3e-3)


def test_snapshot_bytes_match_reference(tmp_path):
    P, U, g, prm = _snap_case()
    path = tmp_path / "s.mhd25"
    P.write_snapshot(str(path), torch.from_numpy(U).cuda(), g, 0.75, prm)
    assert path.read_bytes() == open(SNAP + ".mhd25", "rb").read()
    # host input takes the same device path
    P.write_snapshot(str(path), U, g, 0.75, prm)
    assert path.read_bytes() == open(SNAP + ".mhd25", "rb").read()


def test_snapshot_read_roundtrip():
    P, U, g, prm = _snap_case()
    R, g2, t, p2 = P.read_snapshot(SNAP + ".mhd25")
    assert R.is_cuda and tuple(R.shape) == (8, 16, 12)
    assert np.array_equal(R.cpu().numpy(), U)
    assert (g2, t) == (g, 0.75)
    assert (p2.mu, p2.eta, p2.kappa, p2.gamma) == (prm.mu, prm.eta, prm.kappa, prm.gamma)


def test_snapshot_csv_matches_reference(tmp_path):
    P, U, g, prm = _snap_case()
    path = tmp_path / "s.csv"
    P.write_snapshot_csv(str(path), torch.from_numpy(U).cuda(), g, 0.75, prm)
    assert path.read_text() == open(SNAP + ".csv").read()


def test_snapshot_format_errors(tmp_path):
    P, U, g, prm = _snap_case()
    raw = open(SNAP + ".mhd25", "rb").read()
    cases = {"trunc": raw[:50], "magic": b"XHD25\x00" + raw[6:], "version": raw[:6] + b"\x02\x00" + raw[8:],
             "size": raw[:-8]}
    msgs = {"trunc": "truncated header", "magic": "bad magic", "version": "unsupported version 2",
            "size": "expected 1536 values, found 1535"}
    for k, blob in cases.items():
        p = tmp_path / f"{k}.mhd25"
        p.write_bytes(blob)
        with pytest.raises(P.SnapshotFormatError, match=msgs[k]):
            P.read_snapshot(str(p))
    with pytest.raises(ValueError, match=r"state shape \(8, 16, 11\) does not match grid \(8, 16, 12\)"):
        P.write_snapshot(str(tmp_path / "x.mhd25"), U[:, :, :11], g, 0.0, prm)


def test_rk4_matches_reference_bitwise():
    import paper_1604_02614_b200 as P
    z = golden("rk4_recon32x16.npz")
    g = P.ReconnectionSpec().grid(32, 16)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    U0 = torch.from_numpy(z["U0"]).cuda()
    dt = P.rk4_stable_dt(U0, g, prm)
    assert dt == z["scal"][0]
    f = P.make_rhs(prm, g, P.default_bc("reconnection"))
    y, st = P.integrate_rk4(f, U0.reshape(-1), 0.0, z["scal"][1], dt)
    assert y.is_cuda and np.array_equal(y.cpu().numpy(), z["y"])
    assert [st.steps_accepted, st.rhs_evals] == list(z["counts"])
    # host in, host out
    yh, _ = P.integrate_rk4(f, z["U0"].reshape(-1), 0.0, z["scal"][1], dt)
    assert isinstance(yh, np.ndarray) and np.array_equal(yh, z["y"])
    err = P.error_norm(y.view(8, 32, 16), U0, g)
    assert abs(err - z["scal"][2]) <= 1e-13 * z["scal"][2]


def test_rk4_inadmissible_raises_reference_error():
    import paper_1604_02614_b200 as P
    g = P.ReconnectionSpec().grid(32, 16)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    U = P.reconnection_ic(g, params=prm)
    U[7, 5, 3] = 1e-6                                   # pressure < 0 at one cell
    bc = P.default_bc("reconnection")
    with pytest.raises(stencil.InadmissibleState) as want:
        harness_cpu.rk4(stencil.rhs_closure(prm, g, bc), U.reshape(-1), 0.0, 0.01, 0.005)
    f = P.make_rhs(prm, g, bc)
    with pytest.raises(P.AdmissibilityError) as got:
        P.integrate_rk4(f, U.reshape(-1), 0.0, 0.01, 0.005)
    assert str(got.value) == str(want.value)
    with pytest.raises(P.AdmissibilityError):
        P.rk4_stable_dt(U, g, prm)


def test_error_norm_reference_properties():
    """harness.py:153-163 behaviour: zero on identical states, closed form for one cell,
    invariance under a permutation of the components, grid mismatch rejected."""
    import math
    import paper_1604_02614_b200 as P
    g = P.Grid2D(8, 8, 0.0, 1.0, 0.0, 1.0)
    U = np.random.default_rng(0).standard_normal((8, 8, 8))
    assert P.error_norm(U, U, g) == 0.0
    g = P.Grid2D(10, 5, 0.0, 2.0, 0.0, 1.0)
    U = np.zeros((8, 10, 5))
    V = U.copy()
    V[3, 4, 2] += 0.37
    assert abs(P.error_norm(U, V, g) - 0.37 * math.sqrt(g.hx * g.hy)) <= 1e-14 * 0.37
    g = P.Grid2D(6, 6, 0.0, 1.0, 0.0, 1.0)
    rng = np.random.default_rng(1)
    U, V = rng.standard_normal((8, 6, 6)), rng.standard_normal((8, 6, 6))
    perm = rng.permutation(8)
    a, b = P.error_norm(U, V, g), P.error_norm(U[perm], V[perm], g)
    assert abs(a - b) <= 1e-14 * a
    g = P.Grid2D(8, 8, 0.0, 1.0, 0.0, 1.0)
    with pytest.raises(ValueError, match="grid"):
        P.error_norm(np.zeros((8, 8, 8)), np.zeros((8, 8, 4)), g)


def test_rk4_generic_rhs_is_fourth_order():
    """Any callable rhs, as the reference accepts (harness.py:182-199): y' = -2y."""
    import math
    import paper_1604_02614_b200 as P
    errs = []
    for h in (0.1, 0.05, 0.025):
        y, st = P.integrate_rk4(lambda y: -2.0 * y, np.array([1.0]), 0.0, 1.0, h)
        errs.append(abs(y[0] - math.exp(-2.0)))
        assert st.rhs_evals == 4 * st.steps_accepted
    assert abs(math.log2(errs[0] / errs[1]) - 4.0) <= 0.3
    # same arithmetic as the oracle restatement, step for step
    yo, steps, _ = harness_cpu.rk4(lambda y: -2.0 * y, np.array([1.0]), 0.0, 1.0, 0.3)
    y, st = P.integrate_rk4(lambda y: -2.0 * y, np.array([1.0]), 0.0, 1.0, 0.3)
    assert np.array_equal(y, yo) and st.steps_accepted == steps


def test_snapshot_layout_details(tmp_path):
    """Header fields at their byte offsets; the data block starts with cell (0, 0)'s 8 values."""
    P, U, g, prm = _snap_case()
    path = tmp_path / "s.mhd25"
    P.write_snapshot(str(path), torch.from_numpy(U).cuda(), g, 0.0, prm)
    raw = path.read_bytes()
    assert raw[:6] == b"MHD25\x00" and len(raw) == 96 + 16 * 12 * 64
    assert int.from_bytes(raw[8:12], "little") == 16 and int.from_bytes(raw[12:16], "little") == 12
    assert np.frombuffer(raw[16:48], dtype="<f8").tolist() == [g.x_lo, g.x_hi, g.y_lo, g.y_hi]
    assert np.array_equal(np.frombuffer(raw[96:96 + 64], dtype="<f8"), U[:, 0, 0])
