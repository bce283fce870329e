"""Property-based GPU parity (hypothesis): random grid shapes, boundary policies and
physics against the CPU oracle — bit-identical RHS and Jv for every shape (tile edges,
partial strips, tiny grids), phi_dense to round-off for random matrices."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

BCS = ["periodic", "reflect", "zero-gradient"]


def _state(rng, nx, ny):
    U = np.zeros((8, nx, ny))
    U[0] = 1.0 + 0.3 * rng.random((nx, ny))
    U[1:4] = 0.3 * rng.standard_normal((3, nx, ny))
    U[4:7] = rng.standard_normal((3, nx, ny))
    U[7] = 40.0 + rng.random((nx, ny))
    return U


@settings(max_examples=30, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(nx=st.integers(4, 70), ny=st.integers(4, 300), bx=st.sampled_from(BCS),
       by=st.sampled_from(BCS), b_half=st.booleans(),
       mu=st.sampled_from([0.0, 1e-4, 2e-2]), eta=st.sampled_from([0.0, 1e-3, 5e-2]),
       kappa=st.sampled_from([0.0, 1e-3, 3e-2]), seed=st.integers(0, 2 ** 31 - 1))
def test_rhs_and_jv_bitwise_random_shapes(nx, ny, bx, by, b_half, mu, eta, kappa, seed):
    import paper_1604_02614_b200 as P
    from oracle import jvp, stencil
    rng = np.random.default_rng(seed)
    g = P.Grid2D(nx, ny, -0.3, 1.7, -1.1, 0.4)
    prm = P.MhdParams(mu=mu, eta=eta, kappa=kappa, b_half=b_half)
    bc = P.BoundaryPolicy(bx, by)
    U = _state(rng, nx, ny)
    y = U.reshape(-1)
    f = P.make_rhs(prm, g, bc)
    fo = stencil.rhs_closure(prm, g, bc)
    assert np.array_equal(f(y), fo(y))
    v = rng.standard_normal(y.size)
    assert np.array_equal(P.FdJacobianOperator(f, y)(v), jvp.FdJv(fo, y)(v))


@settings(max_examples=25, deadline=None)
@given(n=st.integers(1, 14), scale=st.floats(0.01, 40.0), k=st.integers(0, 4),
       seed=st.integers(0, 2 ** 31 - 1))
def test_phi_dense_random_matrices(n, scale, k, seed):
    import paper_1604_02614_b200 as P
    from oracle import krylov_cpu
    M = scale * np.random.default_rng(seed).standard_normal((n, n)) / np.sqrt(n)
    got = P.phi_dense(k, M)
    want = krylov_cpu.phi_block(k, M)
    for a, b in zip(got, want):
        assert np.max(np.abs(a - b)) <= 1e-11 * max(1.0, np.max(np.abs(b)))


@settings(max_examples=12, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])
@given(nx=st.integers(8, 40), ny=st.integers(8, 90), bx=st.sampled_from(BCS), by=st.sampled_from(BCS),
       m=st.integers(3, 24), seed=st.integers(0, 2 ** 31 - 1))
def test_selective_reorth_fd_arnoldi_random(nx, ny, bx, by, m, seed):
    """Fused FD Arnoldi on random states: the selective second pass (eta = 0.5) and the
    reference's always-two-pass order give the oracle's H (1e-8, FD round-off amplification)
    and an orthonormal basis."""
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import krylov
    from oracle import jvp, krylov_cpu, stencil
    rng = np.random.default_rng(seed)
    g = P.Grid2D(nx, ny, 0.0, 1.0, 0.0, 2.0)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    bc = P.BoundaryPolicy(bx, by)
    U = _state(rng, nx, ny)
    y = U.reshape(-1)
    v = rng.standard_normal(y.size)
    ref = krylov_cpu.arnoldi(jvp.FdJv(stencil.rhs_closure(prm, g, bc), y), v, m)
    _, Href = ref.snapshot()
    f = P.make_rhs(prm, g, bc)
    old = krylov.REORTH_ETA
    try:
        for eta in (0.0, 0.5):
            krylov.REORTH_ETA = eta
            b = P.arnoldi(P.FdJacobianOperator(f, y), v, m)
            assert b.m == ref.m and b.breakdown == ref.broke
            k = min(b.H.shape[0], Href.shape[0])
            assert np.linalg.norm(b.H[:k] - Href[:k]) <= 1e-8 * np.linalg.norm(Href), eta
            assert np.max(np.abs(b.V.T @ b.V - np.eye(b.V.shape[1]))) <= 1e-12, eta
    finally:
        krylov.REORTH_ETA = old
