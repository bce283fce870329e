"""Small grids: the one-launch orthogonalisation of an Arnoldi iteration (orth_small_kernel:
multi-dot, update, selective re-orthogonalisation decision and, when needed, the second
Gram-Schmidt pass separated by grid barriers) against the four separate launches.

Reference semantics: _ArnoldiProcess.extend, krylov.py:144-168.  Tile ownership, per-CTA
partials and summation order of the fused kernel are those of the separate kernels, so the
factorisation must be BIT-IDENTICAL: H, V, the second-pass flags, and through them every
trajectory counter.  The oracle bar (H within 1e-8) is checked on top.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1604_02614_b200 as P
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _factorise(P, f, y0, m, fused):
    f.ctx.fused_orth(fused)
    yd = dev(y0)
    op = P.FdJacobianOperator(f, yd)
    b = P.arnoldi(op, f(yd), m)
    f.ctx.fused_orth(True)
    sp = b.second_pass.cpu().numpy() if b.second_pass is not None else np.ones(b.m)
    return b.H.cpu().numpy(), b.V.cpu().numpy(), sp, b.m, b.breakdown


@pytest.mark.parametrize("eta", [0.5, 2.0 ** -0.5, 0.0])
def test_fused_orthogonalisation_bitwise_config0(P, eta, monkeypatch):
    """Config 0's state (64^2) takes both selective re-orthogonalisation branches and
    mispredicted re-projections; eta = 0 runs both passes in every iteration."""
    from paper_1604_02614_b200 import krylov
    monkeypatch.setattr(krylov, "REORTH_ETA", eta)
    g = P.ReconnectionSpec().grid(64, 64)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    f = P.make_rhs(prm, g, P.default_bc("reconnection"))
    y0 = P.reconnection_ic(g, params=prm).reshape(-1)
    a = _factorise(P, f, y0, 40, True)
    b = _factorise(P, f, y0, 40, False)
    assert a[3] == b[3] == 40 and not a[4] and not b[4]
    assert np.array_equal(a[0], b[0]), "H differs between the fused and the separate launches"
    assert np.array_equal(a[1], b[1]), "V differs"
    if eta > 0.0:
        assert np.array_equal(a[2], b[2])
        assert 0 < a[2].sum() < len(a[2]), "both branches should occur on this state"
    V = a[1]
    assert np.abs(V.T @ V - np.eye(V.shape[1])).max() <= 1e-12


@pytest.mark.parametrize("shape", [(40, 50), (33, 130), (96, 96), (128, 128)])
def test_fused_orthogonalisation_bitwise_ragged_sizes(P, shape):
    """Vector lengths that are not multiples of the 512 / 1024-element tiles, up to the largest
    grid the fused kernel takes (128^2: 256 update CTAs on 148 SMs, two per SM), against the
    separate launches and the oracle's MGS2."""
    from oracle import jvp, krylov_cpu, stencil
    nx, ny = shape
    g = P.Grid2D(nx, ny, -0.3, 1.1, 0.2, 0.9)
    prm = P.MhdParams(mu=2e-2, eta=1e-2, kappa=3e-2)
    bc = P.BoundaryPolicy("periodic", "reflect")
    rng = np.random.default_rng(nx * 1000 + ny)
    U = np.zeros((8, nx, ny))
    U[0] = 1.0 + 0.3 * rng.random((nx, ny))
    U[1:4] = 0.3 * rng.standard_normal((3, nx, ny))
    U[4:7] = rng.standard_normal((3, nx, ny))
    U[7] = 40.0 + rng.random((nx, ny))
    y0 = U.reshape(-1)
    f = P.make_rhs(prm, g, bc)
    a = _factorise(P, f, y0, 12, True)
    b = _factorise(P, f, y0, 12, False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    if nx * ny <= 40 * 130:
        fo = stencil.rhs_closure(prm, g, bc)
        ref = krylov_cpu.arnoldi(jvp.FdJv(fo, y0), fo(y0), 12)
        _, Href = ref.snapshot()
        assert np.linalg.norm(a[0] - Href) <= 1e-8 * np.linalg.norm(Href)


def test_fused_orthogonalisation_projections_and_step(P):
    """multi_scale_eval / phi_comb (augmented tail: vector length n + p) and a whole EpiRK4 step
    of config 0: identical outputs and counters with the fused launch on and off."""
    from conftest import golden
    zk = golden("krylov_mhd.npz")
    gt, pt = zk["grid"], zk["params"]
    g = P.Grid2D(int(gt[0]), int(gt[1]), gt[2], gt[3], gt[4], gt[5])
    prm = P.MhdParams(mu=pt[0], eta=pt[1], kappa=pt[2], gamma=pt[3], b_half=bool(pt[4]))
    f = P.make_rhs(prm, g, P.BoundaryPolicy("periodic", "reflect"))
    n = zk["a"].size
    res = []
    for fused in (True, False):
        f.ctx.fused_orth(fused)
        op = P.FdJacobianOperator(f, zk["a"], zk["fa"])
        outs, st = P.multi_scale_eval(op, 0.5, 0.5 * zk["fa"], [0.5, 2.0 / 3.0, 1.0], 1e-10)
        assert [st.operator_applies, st.substeps, st.max_basis_size] == list(zk["ms_stats"])
        w, st2 = P.phi_comb(P.PhiCombRequest(operator=op, h=0.5, c=1.0,
                                             vectors=[np.zeros(n), np.zeros(n), zk["vec3"], 0.5 * zk["vec3"]],
                                             tol=1e-10))
        assert [st2.operator_applies, st2.substeps, st2.max_basis_size] == list(zk["pc_stats"])
        res.append((outs, w))
    f.ctx.fused_orth(True)
    for x, y in zip(res[0][0], res[1][0]):
        assert np.array_equal(x, y)
    assert np.array_equal(res[0][1], res[1][1])
    z0 = golden("config0_recon64.npz")
    g0 = P.ReconnectionSpec().grid(64, 64)
    prm0 = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    f0 = P.make_rhs(prm0, g0, P.default_bc("reconnection"))
    ys = []
    for fused in (True, False):
        f0.ctx.fused_orth(fused)
        y1, S = P.epirk4_step(f0, z0["U0"].reshape(-1), 0.1, 1e-10)
        ys.append((y1, (S.operator_applies, S.rhs_evals, S.max_basis_size)))
    f0.ctx.fused_orth(True)
    assert ys[0][1] == ys[1][1]
    assert np.array_equal(ys[0][0], ys[1][0])
    assert np.linalg.norm(ys[0][0] - z0["y1"]) <= 1e-8 * np.linalg.norm(z0["y1"])
