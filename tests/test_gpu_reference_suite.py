"""The reference's own unit tests of the hot path (pkg/tests/test_krylov.py, test_phifuncs.py,
test_epirk.py, test_jacobian.py), re-pointed at the GPU mirror.  Same operators, tolerances
and assertions; NumPy test problems are adapted with ``host_rhs``."""

import math

import numpy as np
import pytest
import scipy.linalg

pytestmark = pytest.mark.gpu

rng = np.random.default_rng(11)


@pytest.fixture(scope="module")
def P():
    import paper_1604_02614_b200 as P
    return P


def stable_matrix(n, scale=1.0):
    A = rng.standard_normal((n, n))
    return scale * (A - (np.abs(A).sum() / n) * np.eye(n)) / np.linalg.norm(A)


def phi_series(k, M, terms=80):
    n = M.shape[0]
    acc = np.zeros((n, n))
    term = np.eye(n) / math.factorial(k)
    for j in range(terms):
        acc = acc + term
        term = (M @ term) / (j + k + 1)
    return acc


def dense_comb(A, h, c, vectors):
    return sum(phi_series(k, c * h * A) @ v for k, v in enumerate(vectors, start=1))


# --------------------------------------------------------------- krylov (test_krylov.py)

def test_arnoldi_symmetric_gives_tridiagonal(P):
    A = rng.standard_normal((9, 9))
    A = A + A.T
    b = P.arnoldi(P.LinearOperator.from_matrix(A), rng.standard_normal(9), 6)
    H = b.H[:b.m, :b.m]
    for i in range(b.m):
        for j in range(b.m):
            if abs(i - j) > 1:
                assert abs(H[i, j]) <= 1e-10


def test_arnoldi_factorization_residual_and_orthonormality(P):
    n = 8
    A = rng.standard_normal((n, n))
    b = P.arnoldi(P.LinearOperator.from_matrix(A), rng.standard_normal(n), n)
    V, H = b.V, b.H
    Vm = V[:, :b.m]
    assert np.max(np.abs(Vm.T @ Vm - np.eye(b.m))) <= 1e-10
    if b.breakdown:
        assert np.max(np.abs(A @ Vm - Vm @ H)) <= 1e-10
    else:
        assert np.max(np.abs(A @ Vm - V @ H)) <= 1e-10


def test_phi_comb_diagonal_oracle(P):
    lam = np.array([-3.0, -1.0, -0.1, 0.2])
    op = P.LinearOperator.from_matrix(np.diag(lam))
    v = np.array([1.0, -2.0, 0.5, 3.0])
    w, _ = P.phi_comb(P.PhiCombRequest(operator=op, h=0.7, c=0.5, vectors=[v], tol=1e-12))
    want = np.array([P.phi_scalar(1, 0.5 * 0.7 * z) for z in lam]) * v
    assert np.max(np.abs(w - want)) <= 1e-11


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_phi_comb_exact_on_full_space(P, p):
    n = 12
    A = stable_matrix(n, scale=4.0)
    vectors = [rng.standard_normal(n) for _ in range(p)]
    req = P.PhiCombRequest(operator=P.LinearOperator.from_matrix(A), h=0.9, c=0.8,
                           vectors=vectors, tol=1e-12)
    w, _ = P.phi_comb(req, P.KrylovConfig(m_init=n + p, m_max=n + p))
    want = dense_comb(A, 0.9, 0.8, vectors)
    assert np.linalg.norm(w - want) <= 1e-10 * max(1.0, np.linalg.norm(want))


def test_phi_comb_substep_consistency(P):
    n = 12
    A = stable_matrix(n, scale=6.0)
    vectors = [rng.standard_normal(n) for _ in range(3)]
    tol = 1e-8
    req = P.PhiCombRequest(operator=P.LinearOperator.from_matrix(A), h=1.0, c=1.0,
                           vectors=vectors, tol=tol)
    w_single, _ = P.phi_comb(req, P.KrylovConfig(m_max=n + 3))
    w_forced, s_forced = P.phi_comb(req, P.KrylovConfig(m_max=n + 3, max_substep=0.25))
    assert s_forced.substeps >= 4
    scale = max(1.0, np.linalg.norm(w_single))
    assert np.linalg.norm(w_forced - w_single) <= 10.0 * tol * scale
    assert np.linalg.norm(w_forced - dense_comb(A, 1.0, 1.0, vectors)) <= 10.0 * tol * scale


def test_phi_comb_meets_tolerance_on_large_operator(P):
    n = 400
    A = 200.0 * (np.diag(-2.0 * np.ones(n)) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1))
    v = rng.standard_normal(n)
    for tol in (1e-4, 1e-8):
        w, stats = P.phi_comb(P.PhiCombRequest(operator=P.LinearOperator.from_matrix(A), h=1.0,
                                               c=1.0, vectors=[v], tol=tol))
        want = np.linalg.solve(A, scipy.linalg.expm(A) @ v - v)
        assert stats.max_basis_size < n
        assert np.linalg.norm(w - want) <= 100.0 * tol * np.linalg.norm(want)


def test_phi_comb_raises_when_cap_and_min_substep_hit(P):
    n = 60
    A = 1e4 * stable_matrix(n, scale=1.0)
    req = P.PhiCombRequest(operator=P.LinearOperator.from_matrix(A), h=1.0, c=1.0,
                           vectors=[rng.standard_normal(n)], tol=1e-14)
    with pytest.raises(P.KrylovConvergenceError) as info:
        P.phi_comb(req, P.KrylovConfig(m_max=5, soft_cap=5, min_substep=0.5))
    assert info.value.residual > 0.0


def test_request_validation(P):
    op = P.LinearOperator.from_matrix(np.eye(3))
    v = np.zeros(3)
    for bad in (dict(c=1.5, vectors=[v]), dict(c=1.0, vectors=[v] * 6),
                dict(c=1.0, vectors=[np.zeros(4)])):
        with pytest.raises(ValueError):
            P.PhiCombRequest(operator=op, h=0.1, tol=1e-8, **bad)
    with pytest.raises(ValueError):
        P.PhiCombRequest(operator=op, h=0.1, c=1.0, vectors=[v], tol=0.0)


def test_multi_scale_diagonal_oracle(P):
    lam = np.array([-2.0, -0.5, 0.1, 0.4, -1.1])
    v = rng.standard_normal(5)
    scales = [0.5, 2.0 / 3.0, 1.0]
    outs, stats = P.multi_scale_eval(P.LinearOperator.from_matrix(np.diag(lam)), 0.9, v, scales, 1e-12)
    assert stats.projections == 1
    for c, out in zip(scales, outs):
        want = np.array([P.phi_scalar(1, c * 0.9 * z) for z in lam]) * v
        assert np.max(np.abs(out - want)) <= 1e-10


def test_multi_scale_higher_order(P):
    n = 10
    A = stable_matrix(n, scale=2.0)
    v = rng.standard_normal(n)
    c = 0.62378111953371494809
    outs, _ = P.multi_scale_eval(P.LinearOperator.from_matrix(A), 1.0, v, [c], 1e-12, order=3)
    want = scipy.linalg.expm(np.block([[c * A, np.eye(n), np.zeros((n, 2 * n))],
                                       [np.zeros((n, 2 * n)), np.eye(n), np.zeros((n, n))],
                                       [np.zeros((n, 3 * n)), np.eye(n)],
                                       [np.zeros((n, 4 * n))]]))[:n, 3 * n:] @ v
    assert np.linalg.norm(outs[0] - want) <= 1e-10


def test_multi_scale_rejects_bad_scales(P):
    op = P.LinearOperator.from_matrix(np.eye(3))
    with pytest.raises(ValueError):
        P.multi_scale_eval(op, 1.0, np.ones(3), [], 1e-8)
    with pytest.raises(ValueError):
        P.multi_scale_eval(op, 1.0, np.ones(3), [0.5, 1.2], 1e-8)


def test_residual_zero_after_breakdown(P):
    b = P.arnoldi(P.LinearOperator.from_matrix(np.eye(4)), np.ones(4), 3)
    assert P.residual_estimate(b, 1.0, 1.0, np.array([1.0])) == 0.0


# ------------------------------------------------------------ phi (test_phifuncs.py)

@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_phi_dense_matches_series(P, k):
    M = rng.standard_normal((7, 7)) * 0.8
    got = P.phi_dense(4, M)[k]
    assert np.max(np.abs(got - phi_series(k, M, terms=60))) <= 1e-12


def test_phi_dense_rejects_nonfinite(P):
    M = np.eye(3)
    M[1, 1] = np.nan
    with pytest.raises(FloatingPointError):
        P.phi_dense(2, M)


# ----------------------------------------------------------- epirk (test_epirk.py)

def brusselator(y):
    a, b = 1.0, 3.0
    return np.array([a + y[0] ** 2 * y[1] - (b + 1.0) * y[0], b * y[0] - y[0] ** 2 * y[1]])


def test_zero_rhs_steps_are_identity(P):
    rhs = P.host_rhs(lambda y: np.zeros_like(y))
    y0 = np.array([1.0, -2.0, 3.0])
    y1, corr, _ = P.epirk5p1_step(rhs, y0, 0.5, 1e-12)
    assert np.all(y1 == y0) and np.all(corr == 0.0)
    y1, _ = P.epirk4_step(rhs, y0, 0.5, 1e-12)
    assert np.all(y1 == y0)


@pytest.mark.parametrize("step", ["epirk4", "epirk5p1"])
def test_linear_problem_exactness_with_exact_jacobian(P, step):
    n = 8
    M = rng.standard_normal((n, n))
    M = M / np.linalg.norm(M)
    y0 = rng.standard_normal(n)
    h = 0.7
    rhs = P.host_rhs(lambda y: M @ y)
    jop = P.LinearOperator.from_matrix(M)
    want = scipy.linalg.expm(h * M) @ y0
    if step == "epirk4":
        y1, _ = P.epirk4_step(rhs, y0, h, 1e-12, jop=jop)
    else:
        y1, _, _ = P.epirk5p1_step(rhs, y0, h, 1e-12, jop=jop)
    assert np.linalg.norm(y1 - want) <= 1e-10 * np.linalg.norm(want)


def test_projection_counts(P):
    rhs = P.host_rhs(brusselator)
    _, st = P.epirk4_step(rhs, np.array([1.0, 3.0]), 0.05, 1e-10)
    assert st.projections == 2
    _, _, st = P.epirk5p1_step(rhs, np.array([1.0, 3.0]), 0.05, 1e-10)
    assert st.projections == 3


def test_riccati_scalar_accuracy(P):
    rhs = P.host_rhs(lambda y: y ** 2)
    errs = []
    for h in (0.1, 0.05, 0.025, 0.0125):
        y, _ = P.integrate_fixed("epirk5p1", rhs, np.array([1.0]), 0.0, 0.5, h, tol_krylov=1e-13)
        errs.append(abs(y[0] - 2.0))
    slopes = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert np.mean(slopes) >= 4.5


def test_integrate_fixed_clips_last_step(P):
    y, stats = P.integrate_fixed("epirk4", P.host_rhs(lambda y: -y), np.array([1.0]), 0.0, 1.0, 0.3)
    assert stats.steps_accepted == 4
    assert y[0] == pytest.approx(math.exp(-1.0), rel=1e-6)


def test_adaptive_counts_rejections(P):
    ctl = P.StepController(tol=1e-8, h_init=0.4)
    y, stats = P.integrate_adaptive(P.host_rhs(lambda y: np.array([y[0] ** 2])), np.array([1.0]),
                                    0.0, 0.5, ctl)
    assert y[0] == pytest.approx(2.0, abs=1e-6)
    assert stats.steps_rejected >= 1 and stats.steps_accepted >= 1


def test_adaptive_raises_stiffness_failure(P):
    ctl = P.StepController(tol=1e-6, h_min=1e-3)
    with pytest.raises(P.StiffnessFailure) as info:
        P.integrate_adaptive(P.host_rhs(lambda y: np.array([y[0] ** 2])), np.array([1.0]), 0.0, 2.0, ctl)
    assert info.value.t < 2.0
    assert info.value.h <= 1e-3 * (1.0 + 1e-9)


def test_adaptive_recoverable_rhs_guard(P):
    class Guard(ValueError):
        pass

    def make(trips):
        budget = {"n": trips}

        def f(y):
            if budget["n"] > 0:
                budget["n"] -= 1
                raise Guard("state out of bounds")
            return -y
        return P.host_rhs(f)

    with pytest.raises(Guard):
        P.integrate_adaptive(make(2), np.array([1.0]), 0.0, 1.0, P.StepController(tol=1e-6))
    y, stats = P.integrate_adaptive(make(2), np.array([1.0]), 0.0, 1.0, P.StepController(tol=1e-6),
                                    recoverable=(Guard,))
    assert stats.steps_rejected >= 2
    assert abs(y[0] - np.exp(-1.0)) < 1e-4


def test_generic_tableau_matches_specialized_steppers(P):
    y0 = np.array([1.5, 3.0, 0.5])
    rhs = P.host_rhs(lambda y: np.array([-y[0] + y[1] * y[2], y[0] - y[1] ** 2, y[0] * y[1] - 2.0 * y[2]]))
    y5, _, _ = P.epirk5p1_step(rhs, y0, 0.1, 1e-13)
    yt, _ = P.epirk_tableau_step(P.EPIRK5P1, rhs, y0, 0.1, 1e-13)
    assert np.linalg.norm(y5 - yt) <= 1e-12 * np.linalg.norm(y5)
    y4, _ = P.epirk4_step(rhs, y0, 0.1, 1e-13)
    yt, _ = P.epirk_tableau_step(P.EPIRK4, rhs, y0, 0.1, 1e-13)
    assert np.linalg.norm(y4 - yt) <= 1e-10 * np.linalg.norm(y4)


# ------------------------------------------------------ jacobian (test_jacobian.py)

def test_linear_map_recovered_to_fd_accuracy(P):
    r = np.random.default_rng(3)
    M = r.standard_normal((6, 6))
    op = P.FdJacobianOperator(P.host_rhs(lambda y: M @ y), r.standard_normal(6))
    for _ in range(5):
        v = r.standard_normal(6)
        assert np.linalg.norm(op(v) - M @ v) <= 100.0 * P.SQRT_EPS * np.linalg.norm(M) * np.linalg.norm(v)


def test_small_direction_used_unscaled(P):
    seen = []

    def f(y):
        seen.append(np.array(y, copy=True))
        return y * 2.0
    op = P.FdJacobianOperator(P.host_rhs(f), np.array([1.0, 1.0]))
    v = np.array([0.5 * P.SQRT_EPS, 0.0])
    op(v)
    assert np.allclose(seen[-1], np.array([1.0, 1.0]) + v)


def test_nonfinite_rhs_identifies_component(P):
    def f(y):
        out = np.array(y, copy=True)
        if y[1] != 0.5:
            out[1] = np.inf
        return out
    op = P.FdJacobianOperator(P.host_rhs(f), np.array([0.0, 0.5, 0.0]))
    with pytest.raises(FloatingPointError, match="component 1"):
        op(np.array([0.0, 1.0, 0.0]))
