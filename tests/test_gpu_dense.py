"""The small dense exponential (phifuncs.py:65-107 via scipy.linalg.expm; krylov.py:209-238) on
one CTA and on an 8-CTA thread-block cluster: same algorithm and decisions, so the cluster's
exponential equals the one-CTA result (bitwise when the exact 1-norms, summed in a different
order, select the same degree and scaling) and scipy's to round-off."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1604_02614_b200  # noqa: F401
    from paper_1604_02614_b200.fdjac import _generic_ctx
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return _generic_ctx()


def expm_dev(ctx, H, cluster_min):
    from paper_1604_02614_b200 import _native as N
    prev = ctx.lib.emhd_set_dense_cluster(cluster_min)
    try:
        n = H.shape[0]
        A = torch.from_numpy(np.ascontiguousarray(H)).cuda()
        E = torch.empty_like(A)
        work = torch.zeros(n + 8, dtype=torch.float64, device="cuda")
        N.check(ctx.lib.emhd_expm(ctx.sync_stream(), A.data_ptr(), n, E.data_ptr(), work.data_ptr()), "expm")
        return E.cpu().numpy()
    finally:
        ctx.lib.emhd_set_dense_cluster(prev)


@pytest.mark.parametrize("n", [40, 64, 100, 110, 141])
def test_cluster_exponential_matches_one_cta_and_scipy(ctx, n):
    import scipy.linalg
    rng = np.random.default_rng(n)
    for scale in (0.3, 20.0, 200.0):
        H = np.triu(rng.standard_normal((n, n)), -1) * scale / np.sqrt(n)     # Hessenberg-like
        one = expm_dev(ctx, H, 0)
        clu = expm_dev(ctx, H, 1)
        ref = scipy.linalg.expm(H)
        den = max(1.0, np.max(np.abs(ref)))
        assert np.max(np.abs(one - ref)) <= 1e-12 * den * max(1.0, scale / 10), (n, scale)
        assert np.max(np.abs(clu - ref)) <= 1e-12 * den * max(1.0, scale / 10), (n, scale)
        assert np.max(np.abs(clu - one)) <= 1e-14 * den * max(1.0, scale / 10), (n, scale)


def test_cluster_residual_batch_matches_one_cta(ctx):
    """Speculative residual checks (emhd_phi_small_batch, order 1) of one factorisation at
    m = 40 .. 47 on clusters and on single CTAs: identical Y and residuals."""
    from paper_1604_02614_b200 import _native as N
    rng = np.random.default_rng(7)
    m_cap = 60
    H = np.triu(rng.standard_normal((m_cap + 1, m_cap)), -1) * 3.0 / np.sqrt(m_cap)
    Hd = torch.from_numpy(H).cuda()
    brk = torch.zeros(m_cap + 1, dtype=torch.float64, device="cuda")
    beta = torch.ones(1, dtype=torch.float64, device="cuda")
    ms = list(range(40, 48))
    out = []
    for cmin in (0, 1):
        prev = ctx.lib.emhd_set_dense_cluster(cmin)
        try:
            Y = torch.zeros((len(ms), m_cap + 1), dtype=torch.float64, device="cuda")
            res = torch.zeros(len(ms), dtype=torch.float64, device="cuda")
            N.check(ctx.lib.emhd_phi_small_batch(ctx.sync_stream(), Hd.data_ptr(), m_cap, N.int_array(ms), 1,
                                                 len(ms), N.dbl_array([0.7] * len(ms)), brk.data_ptr(),
                                                 beta.data_ptr(), Y.data_ptr(), m_cap + 1, res.data_ptr()),
                    "phi_small_batch")
            out.append((Y.cpu().numpy(), res.cpu().numpy()))
        finally:
            ctx.lib.emhd_set_dense_cluster(prev)
    assert np.max(np.abs(out[0][0] - out[1][0])) <= 1e-14 * np.max(np.abs(out[0][0]))
    assert np.allclose(out[0][1], out[1][1], rtol=1e-12, atol=0.0)


@pytest.mark.parametrize("n", [24, 31, 57, 96, 110, 128])
def test_blocked_solve_matches_unblocked_and_scipy(ctx, n):
    """The Pade solve by blocked Gauss-Jordan (eight pivot columns per step, rows not moved)
    against the unblocked solve and scipy, on Hessenberg-like and on full matrices whose
    denominators need row exchanges (large off-diagonal entries), one CTA and cluster."""
    import scipy.linalg
    rng = np.random.default_rng(1000 + n)
    mats = [np.triu(rng.standard_normal((n, n)), -1) * 20.0 / np.sqrt(n),
            rng.standard_normal((n, n)) * 6.0 / np.sqrt(n) + 4.0 * np.eye(n)[::-1],
            rng.standard_normal((n, n)) * 60.0 / np.sqrt(n)]
    for k, H in enumerate(mats):
        ref = scipy.linalg.expm(H)
        den = max(1.0, np.max(np.abs(ref)))
        for cmin in (0, 1):
            res = {}
            for on in (1, 0):
                prev = ctx.lib.emhd_set_dense_gj_blocked(on)
                try:
                    res[on] = expm_dev(ctx, H, cmin)
                finally:
                    ctx.lib.emhd_set_dense_gj_blocked(prev)
            assert np.max(np.abs(res[1] - ref)) <= 2e-11 * den, (n, k, cmin)
            assert np.max(np.abs(res[1] - res[0])) <= 1e-12 * den, (n, k, cmin)
