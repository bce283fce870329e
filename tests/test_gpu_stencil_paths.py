"""Every stencil kernel variant against the CPU oracle, bit for bit.

The launcher picks the row-marching strip kernel (``stencil_kernel``) for grids of 1024^2 and
up — the bench, BASELINE configs 2-4 — and the 2D-tile kernel on small grids.  Here the path
is forced per context (``emhd_set_stencil_path``) so that the marching kernel's own load
pipeline runs on grids the oracle finishes in milliseconds: bulk-copied interior strips and
per-thread cp.async edge strips, ragged strips and ragged row chunks, every mode
(RHS, Jv, normalised Jv of the Arnoldi loop, the augmented phi_comb epilogue in both) and all
nine boundary pairs.  Each case asserts which kernel actually ran (``emhd_last_stencil``).

Reference semantics (cited on the oracle side): mhd.py:269-277 (rhs), fdjac.py:38-49 (Jv),
krylov.py:167 + :149 (v_j = w / h, then J v_j), krylov.py:268-273 (augmented apply).
The augmented top row is compared bitwise with ch*Jv + b_1 q_1 + b_2 q_2 + ... summed left
to right (what the device evaluates), and to 1e-15 relative with the reference's
``ch * op(u) + B @ q`` (a BLAS dgemv whose summation order NumPy does not fix).
"""

import itertools

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

BCS = ["periodic", "reflect", "zero-gradient"]


@pytest.fixture(scope="module")
def P():
    import paper_1604_02614_b200 as P
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rand_state(rng, nx, ny):
    U = np.zeros((8, nx, ny))
    U[0] = 1.0 + 0.3 * rng.random((nx, ny))
    U[1:4] = 0.3 * rng.standard_normal((3, nx, ny))
    U[4:7] = rng.standard_normal((3, nx, ny))
    U[7] = 40.0 + rng.random((nx, ny))
    return U


def lib_ptr(t):
    return None if t is None else t.data_ptr()


class Case:
    """One grid / physics / BC with its oracle closures and device operator."""

    def __init__(self, P, g, prm, bc, U, seed=0):
        from oracle import jvp, stencil
        self.P, self.g, self.prm, self.bc = P, g, prm, bc
        self.U = U
        self.a = U.reshape(-1)
        self.fo = stencil.rhs_closure(prm, g, bc)
        self.jo = jvp.FdJv(self.fo, self.a)
        self.f = P.make_rhs(prm, g, bc)
        self.ctx = self.f.ctx
        self.a_d = dev(self.a)
        self.fa_d = dev(self.jo.f_a)
        self.rng = np.random.default_rng(seed)

    def force(self, **kw):
        self.ctx.stencil_path(**kw)

    def ran(self):
        return self.ctx.last_stencil()

    # device entry points, straight through the C ABI
    def rhs(self):
        out = torch.empty_like(self.a_d)
        self.f.launch(self.a_d, out)
        return out.cpu().numpy()

    def jv(self, v):
        vd = dev(v)
        vn = torch.tensor([np.max(np.abs(v)), 0.0], dtype=torch.float64).cuda()
        out = torch.empty_like(self.a_d)
        L = self.ctx.lib
        from paper_1604_02614_b200 import _native as N
        N.check(L.emhd_jv(self.ctx.sync_stream(), lib_ptr(self.a_d), None, lib_ptr(self.fa_d),
                          lib_ptr(vd), None, lib_ptr(vn), lib_ptr(out)), "jv")
        return out.cpu().numpy()

    def jv_normalized(self, w, h, p=0, ch=1.0, bcols=(), bidx=(), brk=0.0):
        """v_j = w / h and out = J v_j (+ augmented epilogue when p > 0)."""
        from paper_1604_02614_b200 import _native as N
        n = self.a.size
        wd = dev(w)
        scal = dev(np.array([h, np.max(np.abs(w[:n])), brk, 0.0]))
        out = torch.zeros(n + p, dtype=torch.float64, device="cuda")
        vout = torch.zeros(n + p, dtype=torch.float64, device="cuda")
        bd = [dev(b) for b in bcols]
        L = self.ctx.lib
        N.check(L.emhd_jv_normalized(self.ctx.sync_stream(), lib_ptr(self.a_d), None, lib_ptr(self.fa_d),
                                     lib_ptr(wd), None, lib_ptr(scal), lib_ptr(vout), p, ch, len(bd),
                                     N.ptr_array([lib_ptr(b) for b in bd]), N.int_array(list(bidx)),
                                     lib_ptr(out)), "jv_normalized")
        return out.cpu().numpy(), vout.cpu().numpy()

    def jv_aug(self, u, q, ch, bcols, bidx):
        from paper_1604_02614_b200 import _native as N
        n = self.a.size
        p = len(q)
        ud = dev(u)
        vn = torch.tensor([np.max(np.abs(u)), 0.0], dtype=torch.float64).cuda()
        qd = dev(np.asarray(q, dtype=float))
        out = torch.zeros(n + p, dtype=torch.float64, device="cuda")
        bd = [dev(b) for b in bcols]
        L = self.ctx.lib
        N.check(L.emhd_jv_aug(self.ctx.sync_stream(), lib_ptr(self.a_d), None, lib_ptr(self.fa_d),
                              lib_ptr(ud), None, lib_ptr(vn), lib_ptr(qd), p, ch, len(bd),
                              N.ptr_array([lib_ptr(b) for b in bd]), N.int_array(list(bidx)),
                              lib_ptr(out)), "jv_aug")
        return out.cpu().numpy()

    # oracle side
    def aug_ref(self, u, q, ch, bcols, bidx):
        """(device-order top, reference top, tail) of the augmented apply (krylov.py:268-273)."""
        Ju = self.jo(u)
        top = ch * Ju
        for b, k in zip(bcols, bidx):
            top = top + b * q[k]
        p = len(q)
        B = np.zeros((u.size, p))
        for b, k in zip(bcols, bidx):
            B[:, k] = b
        ref = ch * Ju + B @ q
        tail = np.zeros(p)
        tail[:p - 1] = q[1:]
        return top, ref, tail


def check_all_modes(case, label, expect_kernel):
    """RHS, Jv, normalised Jv, both augmented modes, zero direction and queued-after-breakdown,
    each against the oracle, with the forced kernel asserted."""
    n = case.a.size
    rng = case.rng
    # (a) RHS
    assert np.array_equal(case.rhs(), case.fo(case.a)), f"rhs {label}"
    assert case.ran()["kernel"] == expect_kernel, (label, case.ran())
    # (b) Jv with a generic and an unscaled (||v|| < sqrt(eps): sigma = 1) direction
    v = rng.standard_normal(n)
    assert np.array_equal(case.jv(v), case.jo(v)), f"jv {label}"
    vs = 1e-9 * rng.standard_normal(n)
    assert np.array_equal(case.jv(vs), case.jo(vs)), f"jv unscaled {label}"
    # (c) Arnoldi operator step: v_j = w / h (written) and J v_j
    w = rng.standard_normal(n)
    h = float(np.linalg.norm(w))
    out, vout = case.jv_normalized(w, h)
    vj = w / h
    assert np.array_equal(vout, vj), f"v_j {label}"
    assert np.array_equal(out, case.jo(vj)), f"jv_normalized {label}"
    assert case.ran()["kernel"] == expect_kernel
    # (d) augmented epilogue (phi_comb, p = 3, two non-zero B columns) in both modes
    p = 3
    bcols = [rng.standard_normal(n), rng.standard_normal(n)]
    bidx = [0, 2]
    ch = 0.37
    u = rng.standard_normal(n)
    q = rng.standard_normal(p)
    got = case.jv_aug(u, q, ch, bcols, bidx)
    top, ref, tail = case.aug_ref(u, q, ch, bcols, bidx)
    assert np.array_equal(got[:n], top), f"jv_aug top {label}"
    assert np.linalg.norm(got[:n] - ref) <= 1e-15 * np.linalg.norm(ref) + 1e-300
    assert np.array_equal(got[n:], tail)
    wa = np.concatenate([rng.standard_normal(n), rng.standard_normal(p)])
    ha = 1.7
    out, vout = case.jv_normalized(wa, ha, p, ch, bcols, bidx)
    va = wa / ha
    assert np.array_equal(vout, va), f"augmented v_j {label}"
    top, _, tail = case.aug_ref(va[:n], va[n:], ch, bcols, bidx)
    assert np.array_equal(out[:n], top), f"jv_normalized aug top {label}"
    assert np.array_equal(out[n:], tail)
    # (e) zero direction with a non-zero tail: no stencil, top = ch*0 + B q
    got = case.jv_aug(np.zeros(n), q, ch, bcols, bidx)
    ztop = ch * np.zeros(n)
    for b, k in zip(bcols, bidx):
        ztop = ztop + b * q[k]
    assert np.array_equal(got[:n], ztop), f"zero-direction aug {label}"
    # (f) launch queued after a breakdown (scal[2] != 0): zero output, no RHS count
    before = case.ctx.status().rhs_evals
    out, _ = case.jv_normalized(w, h, brk=1.0)
    assert not out.any() and case.ctx.status().rhs_evals == before, f"post-breakdown {label}"


# strip width, rows per CTA, ny: edge strips (cp.async), interior strips (bulk copies), a ragged
# last strip, ragged and single-row chunks; odd ny disables bulk copies everywhere
MARCHING = [
    dict(strip=32, rows_per_cta=3, ny=100, bulk=True),     # edge | bulk | bulk | ragged edge
    dict(strip=32, rows_per_cta=1, ny=66, bulk=True),      # one interior strip, 1 row per CTA
    dict(strip=64, rows_per_cta=4, ny=130, bulk=True),     # exactly one interior strip
    dict(strip=64, rows_per_cta=7, ny=99, bulk=False),     # odd ny: per-thread cp.async only
    dict(strip=128, rows_per_cta=10, ny=300, bulk=True),   # one chunk per strip
    dict(strip=128, rows_per_cta=2, ny=64, bulk=False),    # strip wider than the grid
]


@pytest.mark.parametrize("spacing", ["pow2", "general"])
@pytest.mark.parametrize("mi", range(len(MARCHING)))
def test_marching_kernel_all_modes_all_bcs(P, mi, spacing):
    m = MARCHING[mi]
    nx, ny = 10, m["ny"]
    if spacing == "pow2":
        g = P.Grid2D(nx if nx & (nx - 1) == 0 else 16, ny, 0.0, 1.0, 0.0, 2.0 ** -3 * ny / 8)
        nx = g.nx
    else:
        g = P.Grid2D(nx, ny, -0.3, 1.1, 0.2, 0.9)
    rng = np.random.default_rng(100 + mi)
    U = rand_state(rng, nx, ny)
    prm = P.MhdParams(mu=2e-2, eta=1e-2, kappa=3e-2, b_half=bool(mi % 2))
    for k, (bx, by) in enumerate(itertools.product(BCS, BCS)):
        case = Case(P, g, prm, P.BoundaryPolicy(bx, by), U, seed=mi)
        # the normalised-Jv stencil with one and with two input rows staged ahead
        case.force(kernel=1, strip=m["strip"], rows_per_cta=m["rows_per_cta"], bulk=int(m["bulk"]),
                   raw_rows=1 + (k + mi) % 2)
        check_all_modes(case, (m, spacing, bx, by), expect_kernel=1)
        r = case.ran()
        assert r["strip"] == m["strip"] and r["rows_per_cta"] == m["rows_per_cta"]
        want_bulk = m["bulk"] and ny % 2 == 0 and ny >= 2 * m["strip"] + 2
        assert r["bulk"] == int(want_bulk), (m, r)


def test_tile_kernel_all_modes_all_bcs(P):
    g = P.Grid2D(11, 37, -0.3, 1.1, 0.2, 0.9)
    U = rand_state(np.random.default_rng(7), 11, 37)
    prm = P.MhdParams(mu=2e-2, eta=1e-2, kappa=3e-2)
    for bx, by in itertools.product(BCS, BCS):
        case = Case(P, g, prm, P.BoundaryPolicy(bx, by), U, seed=3)
        case.force(kernel=2)
        check_all_modes(case, ("tile", bx, by), expect_kernel=2)


def test_auto_path_selection(P):
    """AUTO: 2D tiles below tile_rows marching rows per CTA, the marching kernel above."""
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    bc = P.BoundaryPolicy("periodic", "periodic")
    f = P.make_rhs(prm, P.Grid2D(64, 64, 0, 1, 0, 1), bc)
    f(np.ones(8 * 64 * 64) * np.repeat([1, 0, 0, 0, 0, 0, 0, 2.0], 64 * 64))
    assert f.ctx.last_stencil()["kernel"] == 2
    f.ctx.stencil_path(tile_rows=0)
    f(np.ones(8 * 64 * 64) * np.repeat([1, 0, 0, 0, 0, 0, 0, 2.0], 64 * 64))
    assert f.ctx.last_stencil()["kernel"] == 1
    with pytest.raises(Exception):
        f.ctx.stencil_path(strip=48)


# ---------------------------------------------------------------- headline sizes vs the oracle

def test_config2_jv_and_normalised_jv_bitwise_1024(P):
    """The bench's own operator (config 2, 1024^2, marching kernel with bulk copies): Jv and
    the fused normalise + Jv of the Arnoldi loop, bitwise against the oracle."""
    from paper_1604_02614_b200.problems import fourier_grid, fourier_state, unit_start_vector
    g = fourier_grid(1024)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    bc = P.BoundaryPolicy("periodic", "periodic")
    U, rng = fourier_state(g, prm, seed=1604)
    v = unit_start_vector(rng, U.size)
    case = Case(P, g, prm, bc, U)
    assert np.array_equal(case.jv(v), case.jo(v))
    r = case.ran()
    assert r["kernel"] == 1 and r["bulk"] == 1, r
    # the default launch shape of the Jv variants: 64-column strips (4 CTAs/SM), one wave
    assert r["strip"] == 64, r
    w = case.jo(v)
    h = float(np.linalg.norm(w))
    out, vout = case.jv_normalized(w, h)
    assert case.ran()["strip"] == 64
    assert np.array_equal(vout, w / h)
    assert np.array_equal(out, case.jo(w / h))
    # the RHS keeps 128-column strips with one staged row
    assert np.array_equal(case.rhs(), case.fo(case.a))
    assert case.ran()["strip"] == 128, case.ran()
    # through the public operator as well
    op = P.FdJacobianOperator(case.f, case.a_d)
    assert np.array_equal(op(v), case.jo(v))


def test_config2_fd_arnoldi_three_iterations_vs_oracle_1024(P):
    """3 FD-Arnoldi iterations on the config-2 operator (the bench step's first iterations, the
    marching normalise + Jv kernel) against the oracle's MGS2 factorisation: H to 1e-8."""
    from oracle import krylov_cpu
    from paper_1604_02614_b200.problems import fourier_grid, fourier_state, unit_start_vector
    g = fourier_grid(1024)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    bc = P.BoundaryPolicy("periodic", "periodic")
    U, rng = fourier_state(g, prm, seed=1604)
    v = unit_start_vector(rng, U.size)
    case = Case(P, g, prm, bc, U)
    ref = krylov_cpu.arnoldi(case.jo, v, 3)
    Vr, Hr = ref.snapshot()
    for eta in (None, 0.0):
        from paper_1604_02614_b200 import krylov
        old = krylov.REORTH_ETA
        if eta is not None:
            krylov.REORTH_ETA = eta
        try:
            op = P.FdJacobianOperator(case.f, case.a_d, case.fa_d)
            b = P.arnoldi(op, dev(v), 3)
        finally:
            krylov.REORTH_ETA = old
        assert case.ran()["kernel"] == 1
        H = b.H.cpu().numpy()
        assert np.linalg.norm(H - Hr) <= 1e-8 * np.linalg.norm(Hr), (eta, np.linalg.norm(H - Hr))
        V = b.V.cpu().numpy()
        assert np.max(np.abs(V[:, 0] - Vr[:, 0])) <= 1e-15
        assert np.linalg.norm(V - Vr) <= 1e-8 * np.linalg.norm(Vr)


def test_harris_2048_jv_bitwise(P):
    """Config 3's grid (Harris sheet at 2048^2, non-power-of-two spacing: corrected-reciprocal
    divisions; periodic x, reflecting walls in y) — one Jv bitwise against the oracle."""
    g = P.ReconnectionSpec().grid(2048, 2048)
    prm = P.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-3)
    U = P.reconnection_ic(g, params=prm)
    case = Case(P, g, prm, P.default_bc("reconnection"), U)
    v = np.random.default_rng(2048).standard_normal(U.size)
    ref = case.jo(v)
    assert np.array_equal(case.jv(v), ref)
    assert case.ran()["kernel"] == 1 and case.ran()["strip"] == 64
    # the Arnoldi-loop launch on the same grid: v_j = w / h written and J v_j
    h = float(np.linalg.norm(ref))
    out, vout = case.jv_normalized(ref, h)
    assert np.array_equal(vout, ref / h)
    assert np.array_equal(out, case.jo(ref / h))


@pytest.mark.slow
def test_harris_4096_jv_bitwise(P):
    """Config 4's grid (4096^2, 1 GiB vectors) — one Jv bitwise against the oracle."""
    g = P.ReconnectionSpec().grid(4096, 4096)
    prm = P.MhdParams(mu=1e-4, eta=1e-5, kappa=1e-3)
    U = P.reconnection_ic(g, params=prm)
    case = Case(P, g, prm, P.default_bc("reconnection"), U)
    v = np.random.default_rng(4096).standard_normal(U.size)
    got = case.jv(v)
    assert case.ran()["kernel"] == 1
    assert np.array_equal(got, case.jo(v))


@pytest.mark.parametrize("kernel,strip", [(1, 32), (1, 64), (2, 0)])
def test_nonfinite_component_named_by_every_kernel(P, kernel, strip):
    """The first non-finite Jv component (fdjac.py:47-48) is named identically by the marching
    kernel (either strip width) and the 2D-tile kernel: several fields and cells go non-finite,
    the reference reports the smallest flat index."""
    from oracle import jvp, stencil
    g = P.Grid2D(12, 70, 0.0, 1.0, 0.0, 1.0)
    prm = P.MhdParams()
    bc = P.BoundaryPolicy("periodic", "periodic")
    U = np.zeros((8, 12, 70))
    U[0] = 1.0
    U[7] = 2.0
    U[1, 5, 40] = 1e200          # momentum^2 overflows in the perturbed state
    U[7, 5, 40] = 1e308
    U[2, 9, 3] = 1e200
    U[7, 9, 3] = 1e308
    v = np.zeros(U.size)
    v[5] = 1.0
    fa = np.zeros(U.size)
    ref = jvp.FdJv(stencil.rhs_closure(prm, g, bc, check=False), U.reshape(-1), fa)
    with pytest.raises(FloatingPointError) as want:
        ref(v)
    f = P.make_rhs(prm, g, bc, check=False)
    if kernel == 1:
        f.ctx.stencil_path(kernel=1, strip=strip, rows_per_cta=5)
    else:
        f.ctx.stencil_path(kernel=2)
    op = P.FdJacobianOperator(f, U.reshape(-1), fa)
    with pytest.raises(FloatingPointError) as got:
        op(v)
    assert f.ctx.last_stencil()["kernel"] == kernel
    assert str(got.value) == str(want.value)
