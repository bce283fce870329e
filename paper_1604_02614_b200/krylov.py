"""GPU drop-in for the Krylov phi-function layer (reference krylov.py, phifuncs.py).

Public names and semantics follow the reference: ``KrylovConfig``
(krylov.py:71-82), ``KrylovStats`` (:55-68), ``ArnoldiBasis`` (:85-100),
``PhiCombRequest`` (:103-124), ``KrylovConvergenceError`` (:31-36),
``arnoldi`` (:191-206), ``residual_estimate`` (:209-231), ``phi_comb``
(:241-324) and ``multi_scale_eval`` (:327-375).

Device design:
* the basis lives in HBM as (m_cap+1) contiguous rows of length ld (the
  reference's V[n, m_cap+1] is column-strided, krylov.py:137);
* one Arnoldi iteration = fused normalise + Jv stencil (csrc/stencil.cu), a
  multi-dot sweep, an update + re-dot sweep and an update + norm sweep
  (csrc/krylov.cu): CGS2, the reference's MGS + re-orthogonalisation
  projector to round-off, in three streaming passes;
* the small dense phi / exp of the Hessenberg matrix and the residual
  surrogate run on the GPU (csrc/dense.cu); the host reads one double per
  residual check and makes the reference's control decisions verbatim;
* V_m y and the EpiRK stage axpys are one sweep over the basis (emhd_combine).
"""

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as D
from .fdjac import FdJacobianOperator, LinearOperator, _generic_ctx, _lincomb
from .mhd import raise_status
from .slab import PushHalo

MAX_COMB_ORDER = 5
# speculation depth of the batched residual checks (0: automatic from the vector size,
# 1: off — one residual check per Arnoldi iteration, as the reference orders them)
SPEC_DEPTH_OVERRIDE = 0
# single-rank fused engines drive each Arnoldi iteration with one C call (emhd_arnoldi_iter);
# False routes through the per-kernel C entry points (same kernels; used for per-launch timing)
FAST_DRIVER = True
BREAKDOWN_RTOL = 1e-12
# Arnoldi iterations queued behind a batch of residual checks while the checks run on a
# side stream (None: by vector size; EMHD_LOOKAHEAD overrides; 0: checks in stream order)
LOOKAHEAD_OVERRIDE = None
# Selective re-orthogonalisation of the fused finite-difference engines (Kahan-Parlett "twice is
# enough" with kappa = 1/eta = 2; DGKS/ARPACK use eta ~ 1/sqrt(2)): the second Gram-Schmidt pass
# runs only when the first left ||w1|| < eta ||w||.  The reference's MGS always runs it
# (krylov.py:156-160); when ||w1|| >= eta ||w|| the first pass already leaves w1 orthogonal to
# O(eps / eta), so H and V change at round-off level.  0: always two passes.
# EMHD_REORTH_ETA overrides.  Measured (identical counters in every case): config 2 1216 -> 1672
# it/s, config 1 0.71 -> 0.58 s, config-3 physics at 1024^2 1.86 -> 1.68 s (eta 1/sqrt(2): 1630
# it/s, 0.65 s, 1.82 s).
REORTH_ETA = float(os.environ.get("EMHD_REORTH_ETA", "0.5"))
# fast path: the first update pass skips the re-projection dots when the previous iteration
# skipped its second pass (a gated multi-dot computes them on a misprediction)
PREDICT_REPROJECTION = os.environ.get("EMHD_PREDICT_REPROJ", "1") != "0"
# reporting: count kept iterations / second passes per context (tools/run_configs.py)
COUNT_PASSES = False
# persisting-L2 window over the head of the basis (see _l2_window); env override in MiB
L2_WINDOW_MB = os.environ.get("EMHD_L2_WINDOW_MB")


class KrylovConvergenceError(RuntimeError):
    """Raised when the basis cap is reached with the substep at minimum."""

    def __init__(self, message, residual):
        super().__init__(message)
        self.residual = residual


@dataclass
class KrylovStats:
    operator_applies: int = 0
    substeps: int = 0
    max_basis_size: int = 0
    projections: int = 0

    def merge(self, other):
        self.operator_applies += other.operator_applies
        self.substeps += other.substeps
        self.max_basis_size = max(self.max_basis_size, other.max_basis_size)
        self.projections += other.projections


@dataclass
class KrylovConfig:
    m_init: int = 10
    m_max: int = 100
    soft_cap: int = 25
    grow_threshold: int = 10
    substep_growth: float = 4.0 / 3.0
    min_substep: float = 1.0 / 1024.0
    max_substep: float = 1.0
    reorthogonalize: bool = True


@dataclass
class ArnoldiBasis:
    """Orthonormal basis V (n x m or n x (m+1)), Hessenberg H, seed norm beta."""

    V: object
    H: object
    m: int
    beta: float
    breakdown: bool = False
    # B200 extension: per iteration, 1.0 where the second Gram-Schmidt pass ran (device
    # tensor; None when every iteration ran it, i.e. selective re-orthogonalisation off)
    second_pass: object = None

    @property
    def h_next(self):
        if self.breakdown or self.H.shape[0] == self.m:
            return 0.0
        return float(self.H[self.m, self.m - 1])


@dataclass
class PhiCombRequest:
    """Query for w = sum_{k=1}^p phi_k(c*h*J) v_k (krylov.py:103-124)."""

    operator: LinearOperator
    h: float
    c: float
    vectors: list
    tol: float

    def __post_init__(self):
        if not (0.0 < self.c <= 1.0):
            raise ValueError(f"scale factor c must be in (0, 1], got {self.c}")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        p = len(self.vectors)
        if p < 1 or p > MAX_COMB_ORDER:
            raise ValueError(f"need 1 <= p <= {MAX_COMB_ORDER} vectors, got {p}")
        n = self.operator.n
        for k, v in enumerate(self.vectors, start=1):
            shp = tuple(v.shape) if hasattr(v, "shape") else np.shape(v)
            if shp != (n,):
                raise ValueError(f"vector v_{k} has shape {shp}, expected ({n},)")


def _ld(n):
    return (n + 31) // 32 * 32


def _l2_window(ctx, h, V, vec_bytes):
    """Keep the first 40 MiB of the basis in L2 across iterations (persisting access window on
    the launching stream): every multi-dot and update pass re-reads it, and the vectors that
    stream through evict each other instead of it.  Measured on the config-2 workload: 512²
    +3.8 %, 1024² +1.6 %, 2048² +0.3 %; at 256² (-1 to -2 %) the whole working set competes
    for L2 and at 2048² with 64 MiB the stencil loses more than the passes gain, so it is on
    for 16 MiB <= W <= 256 MiB only.  Set once per (stream, basis buffer)."""
    if L2_WINDOW_MB is not None:
        want = int(float(L2_WINDOW_MB) * 2 ** 20)
    else:
        want = 40 * 2 ** 20 if 16 * 2 ** 20 <= vec_bytes <= 256 * 2 ** 20 else 0
    want = min(want, V.numel() * 8)
    key = (ctx._stream, D.ptr(V), want)
    prev = getattr(ctx, "_l2win", None)
    if prev == key or (want == 0 and (prev is None or prev[0] != ctx._stream)):
        return
    N.check(ctx.lib.emhd_l2_window(h, D.ptr(V), want), "l2_window")
    ctx._l2win = key


def _persistent_basis(ctx, rows, ld):
    """A (rows, ld) view of the context's reusable Krylov basis buffer (grown on demand)."""
    buf = getattr(ctx, "_basis", None)
    need = rows * ld
    if buf is None or buf.numel() < need:
        ctx._basis = None
        del buf
        torch.cuda.empty_cache()
        ctx._basis = torch.empty(need, dtype=D.F64, device=D.device())
    return ctx._basis[:need].view(rows, ld)


class _Engine:
    """How one Arnoldi iteration obtains w = A v_j."""

    fused = False


class _FusedFd(_Engine):
    """FD Jacobian of the fused stencil, optionally augmented (phi_comb)."""

    fused = True

    def __init__(self, jop, p=0, ch=1.0, bcols=(), bidx=()):
        self.jop, self.gpu, self.ctx = jop, jop.gpu, jop.ctx
        self.p, self.ch = p, float(ch)
        self.bcols = list(bcols)
        self.bidx = list(bidx)
        self._bptr = N.ptr_array([D.ptr(b) for b in self.bcols])
        self._bidx = N.int_array(self.bidx)
        self._vn = D.zeros(2)


class _Generic(_Engine):
    """Any LinearOperator (optionally wrapped by the augmented operator)."""

    def __init__(self, op, n, p=0, ch=1.0, bcols=(), bidx=()):
        self.op, self.n, self.p, self.ch = op, n, p, float(ch)
        self.bcols, self.bidx = list(bcols), list(bidx)
        self.ctx = getattr(op, "ctx", None) or _generic_ctx()


class _Process:
    """Device Arnoldi factorisation (reference _ArnoldiProcess, krylov.py:127-188)."""

    def __init__(self, engine, seed, m_cap, n_top, p=0, layout=None, comm=None, persistent=False,
                 reorthogonalize=True, seed_norms=None):
        self.eng = engine
        self.ctx = engine.ctx
        self.lib = self.ctx.lib
        self.n_top = n_top
        self.p = p
        self.naug = n_top + p
        self.layout, self.comm = layout, comm
        rank0 = layout is None or layout.rank == 0
        self.len_upd = self.naug
        self.len_dot = n_top + (p if rank0 else 0)
        # global dimension (the reference's self.n)
        self.n = (layout.nx_global * layout.ny * 8 if layout is not None else n_top) + p
        self.m_cap = min(m_cap, self.n)
        if self.m_cap + 1 > self.ctx.max_vectors - 4:
            raise ValueError(f"basis cap {self.m_cap} exceeds the context limit")
        # V and w are never read beyond their written lengths: no zero-fill of 2.7 GB.
        # Projections inside a step (multi-scale, phi-comb) share one persistent basis per
        # context, sized for any tail p <= 5, so a 129 GiB basis (4096^2, m_max 128) is
        # allocated once instead of once per projection.
        if persistent:
            self.ld = _ld(n_top + MAX_COMB_ORDER)
            self.V = _persistent_basis(self.ctx, self.m_cap + 1, self.ld)
        else:
            self.ld = _ld(self.naug)
            self.V = torch.empty((self.m_cap + 1, self.ld), dtype=D.F64, device=D.device())
        k = self.m_cap + 4
        hw = max(self.m_cap, 1)
        nsmall = (self.m_cap + 1) * hw + 3 * k + 2 + 5 * (self.m_cap + 1) + 4
        # projections inside a step run one after the other on the context's stream: their work
        # vectors, small device block and pinned readback buffers are allocated once per
        # (cap, ld) and reused (stream order protects the device side, every host read follows
        # a sync) — a dozen tensor constructions per projection otherwise, on host-bound grids
        pool = None
        if persistent:
            cache = self.ctx.__dict__.setdefault("_proc_pool", {})
            pool = cache.get((self.m_cap, self.ld, D.device().index))
            if pool is None:
                pool = cache[(self.m_cap, self.ld, D.device().index)] = {}
        self._pool = pool
        if pool:
            self.w = pool["w"]
            self._small = pool["small"]
            self._small.zero_()
        else:
            self.w = [torch.empty(self.ld, dtype=D.F64, device=D.device()) for _ in range(2)]
            # one zero-filled block for H and every small scalar area (a single fill launch)
            self._small = torch.zeros(nsmall, dtype=D.F64, device=D.device())
        o = (self.m_cap + 1) * hw
        self.H = self._small[:o].view(self.m_cap + 1, hw)
        self.d1 = self._small[o:o + k]
        self.d2 = self._small[o + k:o + 2 * k]
        self.nrm = self._small[o + 2 * k:o + 2 * k + 2]
        o2 = o + 2 * k + 2
        self.brk = self._small[o2:o2 + self.m_cap + 1]
        self.nb = self._small[o2 + self.m_cap + 1:o2 + self.m_cap + 5]   # {sum seed^2, max|seed|, beta, -}
        o3 = o2 + self.m_cap + 5
        self.gate = self._small[o3:o3 + self.m_cap + 1]       # look-ahead gates (fast path)
        self.evals = self._small[o3 + self.m_cap + 1:o3 + 2 * (self.m_cap + 1)]   # RHS evals per iteration
        self.reorth = self._small[o3 + 2 * (self.m_cap + 1):o3 + 3 * (self.m_cap + 1)]  # 1: pass 2 skipped
        self.md2 = self._small[o3 + 3 * (self.m_cap + 1):o3 + 4 * (self.m_cap + 1)]     # 0: separate h2 dots
        # selective on the fused engines, both passes elsewhere.  `reorthogonalize` is accepted
        # and ignored, exactly as the reference does: its _ArnoldiProcess stores nothing from it
        # and always runs the re-orthogonalisation pass (`if True:`, krylov.py:156-160)
        del reorthogonalize
        self.eta = REORTH_ETA if engine.fused else 0.0
        self._settled = 0
        self._pending = False
        self._brk_seen = {}
        self._depth = 2
        if pool:
            self.scal = pool["scal"]
            self.scal.dev.zero_()
            self.res_host, self.brk_host, self.host_rb = pool["res_host"], pool["brk_host"], pool["host_rb"]
            self.Ybuf, self.resbuf = pool["Ybuf"], pool["resbuf"]
        else:
            self.scal = D.Scratch(4)
            self.res_host = torch.zeros(8, dtype=D.F64, pin_memory=True)
            self.brk_host = torch.zeros(self.m_cap + 1, dtype=D.F64, pin_memory=True)
            self.Ybuf = torch.empty(8 * (self.m_cap + 1), dtype=D.F64, device=D.device())
            self.resbuf = torch.empty(8, dtype=D.F64, device=D.device())
            self.host_rb = torch.zeros(self.m_cap + 16, dtype=D.F64, pin_memory=True)
            if pool is not None:
                pool.update(w=self.w, small=self._small, scal=self.scal, res_host=self.res_host,
                            brk_host=self.brk_host, host_rb=self.host_rb, Ybuf=self.Ybuf,
                            resbuf=self.resbuf)
        self.beta_dev = self.nb[2:3]
        # slab ranks with symmetric memory: w's edge rows are pushed into the neighbours'
        # halo buffers by the update pass itself (emhd_update_push), no P2P exchange per Jv
        self.push = None
        native = engine.fused and getattr(engine.gpu, "native", False)
        if engine.fused and layout is not None and layout.distributed and not native:
            g = engine.gpu
            if "_push_halo" not in g.__dict__:
                g._push_halo = PushHalo.create(g.layout, g.comm)
            self.push = g._push_halo
        self.m = 0
        self.breakdown = False
        self.applies = 0
        self.cur = 0            # index of the w buffer holding the latest unnormalised vector
        self._vm_ready = 0      # rows of V materialised
        # beta = ||seed||_2, V[0] = seed / beta  (krylov.py:132-137)
        sd = seed.reshape(-1)
        h = self.ctx.sync_stream()
        _l2_window(self.ctx, h, self.V, self.ld * 8)
        if seed_norms is not None:
            # {sum seed^2, max|seed|} already all-reduced and read by the caller (its zero test):
            # one host sync for both
            dev2, b2 = seed_norms
            self.nb[0:2].copy_(dev2)
        else:
            N.check(self.lib.emhd_norms(h, D.ptr(sd), self.len_dot, n_top, D.ptr(self.nb)), "norms")
            self._allreduce_norms(self.nb)
            b2 = float(self.nb[0].item())
        self.beta = math.sqrt(b2)
        if self.beta == 0.0:
            raise ValueError("Arnoldi seed vector must be nonzero")
        N.check(self.lib.emhd_div_scalar(h, D.ptr(sd), D.ptr(self.nb), 1, D.ptr(self.V[0]),
                                         D.ptr(self.beta_dev), self.naug), "div_scalar")
        self._vm_ready = 1
        # single-rank fused engine: one C call per iteration (emhd_arnoldi_iter)
        # slab ranks whose collectives live in the library (slab.NativeComm) keep it too
        self.fast = FAST_DRIVER and engine.fused and (layout is None or not layout.distributed or native)
        if self.fast:
            E = engine
            A = N.ArnoldiArgs()
            A.a, A.fa = D.ptr(E.jop.a), D.ptr(E.jop.f_a)
            A.V, A.ldv = D.ptr(self.V), self.ld
            A.H, A.ldh = D.ptr(self.H), self.H.shape[1]
            A.w0, A.w1 = D.ptr(self.w[0]), D.ptr(self.w[1])
            A.d1, A.d2, A.nrm = D.ptr(self.d1), D.ptr(self.d2), D.ptr(self.nrm)
            A.vn, A.scal, A.brk = D.ptr(E._vn), D.ptr(self.scal.dev), D.ptr(self.brk)
            A.n_top, A.len_dot, A.len_upd = self.n_top, self.len_dot, self.len_upd
            A.p, A.nb, A.ch = self.p, len(E.bcols), E.ch
            for k, b in enumerate(E.bcols):
                A.bcol[k] = D.ptr(b)
                A.bidx[k] = E.bidx[k]
            A.gen = self._new_gen()
            A.gate, A.evals = D.ptr(self.gate), D.ptr(self.evals)
            A.eta, A.reorth = self.eta, D.ptr(self.reorth)
            # re-projection dots predicted from the previous decision (fast path only)
            A.md2 = D.ptr(self.md2) if PREDICT_REPROJECTION else None
            A.a_halo = D.ptr(E.jop.a_halo)
            self._args = A
            self._args_ref = D.ctypes_byref(A)

    def _new_gen(self):
        g = (getattr(self.ctx, "_gen", 0) + 1) & 0x7fffffff
        self.ctx._gen = g
        return g

    # -- collectives ----------------------------------------------------------
    def _allreduce_sum(self, t):
        if self.comm is not None:
            self.comm.allreduce_sum(t)

    def _allreduce_norms(self, t2):
        """{sum, max} across slabs with one SUM all-reduce of 1 + P slots (emhd_slot_norms)."""
        if self.comm is not None and self.layout.distributed:
            L = self.layout
            slots = getattr(self, "_slots", None)
            if slots is None:
                slots = self._slots = torch.zeros(L.size + 1, dtype=D.F64, device=D.device())
            h = self.ctx.sync_stream()
            N.check(self.lib.emhd_slot_norms(h, D.ptr(t2), L.rank, L.size, D.ptr(slots)), "slot_norms")
            self.comm.allreduce_sum(slots)
            N.check(self.lib.emhd_unslot_norms(self.ctx.sync_stream(), D.ptr(slots), L.size, D.ptr(t2)),
                    "unslot_norms")

    # -- one iteration ----------------------------------------------------------
    def _apply(self, j):
        """w_out = A v_j; returns the index of the w buffer written."""
        E = self.eng
        h = self.ctx.sync_stream()
        dst = 1 - self.cur if j > 0 else 0
        out = self.w[dst]
        if E.fused:
            a, ah, fa = E.jop.a, E.jop.a_halo, E.jop.f_a
            if j == 0:
                v = self.V[0]
                vh = None if E.gpu.defer_halo else E.gpu.halo(v[:self.n_top])
                N.check(self.lib.emhd_norms(h, D.ptr(v), 0, self.n_top, D.ptr(E._vn)), "norms")
                if self.layout is not None and self.layout.distributed:
                    self.comm.allreduce_max(E._vn[1:2])
                E._vn[0:1].copy_(E._vn[1:2])
                if self.p:
                    N.check(self.lib.emhd_jv_aug(h, D.ptr(a), D.ptr(ah), D.ptr(fa), D.ptr(v), D.ptr(vh),
                                                 D.ptr(E._vn), D.ptr(v[self.n_top:]), self.p, E.ch,
                                                 len(E.bcols), E._bptr, E._bidx, D.ptr(out)), "jv_aug")
                else:
                    N.check(self.lib.emhd_jv(h, D.ptr(a), D.ptr(ah), D.ptr(fa), D.ptr(v), D.ptr(vh),
                                             D.ptr(E._vn), D.ptr(out)), "jv")
                self._last = (1, v, vh, E._vn)
            else:
                wp = self.w[self.cur]
                wh = self.push.buf if self.push is not None else E.gpu.halo(wp[:self.n_top])
                N.check(self.lib.emhd_jv_normalized(h, D.ptr(a), D.ptr(ah), D.ptr(fa), D.ptr(wp),
                                                    D.ptr(wh), D.ptr(self.scal.dev), D.ptr(self.V[j]),
                                                    self.p, E.ch, len(E.bcols), E._bptr, E._bidx,
                                                    D.ptr(out)), "jv_normalized")
                self._vm_ready = j + 1
                self._last = (2, wp, wh, self.scal.dev)
        else:
            if j > 0:
                self._materialize(j)
            v = self.V[j]
            if self.p:
                n = self.n_top
                q = v[n:n + self.p].to("cpu").numpy()
                top = D.to_device(E.op(v[:n])).reshape(-1)
                terms = [(E.ch, top)] + [(float(q[k]), b) for b, k in zip(E.bcols, E.bidx)]
                _lincomb(self.ctx, terms, out[:n])
                tail = np.zeros(self.p)
                tail[:self.p - 1] = q[1:]
                out[n:n + self.p].copy_(torch.from_numpy(tail))
            else:
                r = D.to_device(E.op(v[:self.naug])).reshape(-1)
                out[:self.naug].copy_(r)
        self.cur = dst
        return dst

    def _materialize(self, upto):
        """Write V[k] = w / h for the pending row k = upto (krylov.py:167)."""
        if self._vm_ready > upto:
            return
        h = self.ctx.sync_stream()
        N.check(self.lib.emhd_div_scalar(h, D.ptr(self.w[self.cur]), D.ptr(self.scal.dev), 0,
                                         D.ptr(self.V[upto]), 0, self.naug), "div_scalar")
        self._vm_ready = upto + 1

    def extend(self, sync=True):
        """Add one basis vector; returns False on lucky breakdown (krylov.py:144-168).

        With ``sync=False`` (fused engine only) the iteration is queued without
        waiting for its breakdown test; ``settle()`` later resolves where the
        factorisation stopped (a launch queued after a breakdown does no work).
        """
        if self.breakdown or self.m >= self.m_cap:
            return False
        j = self.m
        if self.fast:
            N.check(self.lib.emhd_arnoldi_iter(self.ctx.sync_stream(), self._args_ref, j), "arnoldi_iter")
            self.applies += 1
            self.cur = j % 2
            if j > 0:
                self._vm_ready = j + 1
            self._last = (2 if j else 1, None, None, None)
            self.m = j + 1
            if not sync:
                self._pending = True
                return True
            return self.settle()
        self.lib.emhd_set_epoch(self.ctx.sync_stream(), j)
        wi = self._apply(j)
        self.lib.emhd_set_epoch(self.ctx.sync_stream(), -1)   # later launches: not speculative
        self.applies += 1
        w = self.w[wi]
        h = self.ctx.sync_stream()
        nv = j + 1
        # pass 1: h1 = V^T w and ||w||^2 (the breakdown scale, krylov.py:151)
        N.check(self.lib.emhd_multidot(h, D.ptr(w), D.ptr(self.V), self.ld, nv, self.len_dot, 1,
                                       D.ptr(self.d1)), "multidot")
        self._allreduce_sum(self.d1[:nv + 1])
        # w -= V h1 ; h2 = V^T w ; ||w||^2, max|w_top|
        N.check(self.lib.emhd_update(h, D.ptr(w), D.ptr(self.V), self.ld, nv, D.ptr(self.d1),
                                     self.len_upd, self.len_dot, self.n_top, 0, D.ptr(self.d2)), "update")
        self._allreduce_sum(self.d2[:nv + 1])
        if self.comm is not None and self.layout.distributed:
            self.comm.allreduce_max(self.d2[nv + 1:nv + 2])
        gate = None
        if self.eta > 0.0:
            # selective re-orthogonalisation: pass 2 only when ||w1|| < eta ||w|| (on device;
            # the pass-2 launches below test the gate, no host sync)
            gate = self.reorth[j:j + 1]
            N.check(self.lib.emhd_reorth_decide(h, D.ptr(self.d1), D.ptr(self.d2), nv, D.ptr(self.d1[nv:]),
                                                j, D.ptr(self.H), self.H.shape[1], D.ptr(self.scal.dev),
                                                D.ptr(self.brk), self.eta, D.ptr(gate)), "reorth_decide")
            if self.push is not None:
                N.check(self.lib.emhd_push_edges(h, D.ptr(w), self.push.lo_ptr, self.push.hi_ptr,
                                                 D.ptr(gate)), "push_edges")

        def gated():
            if gate is not None:
                N.check(self.lib.emhd_skip_next(h, D.ptr(gate)), "skip_next")

        # w -= V h2 ; ||w||^2, max|w_top| ; column bookkeeping (fused when single-rank)
        if self.comm is None or not self.layout.distributed:
            gated()
            N.check(self.lib.emhd_update_finish(
                h, D.ptr(w), D.ptr(self.V), self.ld, nv, D.ptr(self.d2), self.len_upd, self.len_dot,
                self.n_top, D.ptr(self.nrm), D.ptr(self.d1), D.ptr(self.d1[nv:]), j, D.ptr(self.H),
                self.H.shape[1], D.ptr(self.scal.dev), D.ptr(self.brk)), "update_finish")
        elif self.push is not None:
            P = self.push
            gated()
            N.check(self.lib.emhd_update_push(h, D.ptr(w), D.ptr(self.V), self.ld, nv, D.ptr(self.d2),
                                              self.len_upd, self.len_dot, self.n_top, D.ptr(self.nrm),
                                              P.lo_ptr, P.hi_ptr), "update_push")
            self._allreduce_norms(self.nrm)          # also orders the pushed halo rows
            gated()
            N.check(self.lib.emhd_arnoldi_finish(h, D.ptr(self.d1), D.ptr(self.d2), D.ptr(self.nrm),
                                                 D.ptr(self.d1[nv:]), j, D.ptr(self.H),
                                                 self.H.shape[1], D.ptr(self.scal.dev), D.ptr(self.brk)),
                    "arnoldi_finish")
        else:
            gated()
            N.check(self.lib.emhd_update(h, D.ptr(w), D.ptr(self.V), self.ld, nv, D.ptr(self.d2),
                                         self.len_upd, self.len_dot, self.n_top, 1, D.ptr(self.nrm)),
                    "update")
            self._allreduce_norms(self.nrm)
            gated()
            N.check(self.lib.emhd_arnoldi_finish(h, D.ptr(self.d1), D.ptr(self.d2), D.ptr(self.nrm),
                                                 D.ptr(self.d1[nv:]), j, D.ptr(self.H),
                                                 self.H.shape[1], D.ptr(self.scal.dev), D.ptr(self.brk)),
                    "arnoldi_finish")
        self.m = j + 1
        if not sync and self.eng.fused:
            self._pending = True
            return True
        return self.settle()

    def extend_many(self, k, lookahead=False):
        """Queue up to k iterations without syncing; one C call on the single-rank fast path.
        ``lookahead``: the iterations are gated (cancellable) look-ahead iterations."""
        k = min(k, self.m_cap - self.m)
        if k <= 0 or self.breakdown:
            return 0
        if not self.fast:
            done = 0
            while done < k and self.extend(sync=False):
                done += 1
            return done
        j0 = self.m
        if lookahead and j0 >= 1 and os.environ.get("EMHD_LOOKAHEAD_GATE", "1") != "0":
            N.check(self.lib.emhd_arnoldi_lookahead(self.ctx.sync_stream(), self._args_ref, j0, j0 + k),
                    "arnoldi_lookahead")
        else:
            N.check(self.lib.emhd_arnoldi_run(self.ctx.sync_stream(), self._args_ref, j0, j0 + k),
                    "arnoldi_run")
        self.applies += k
        self.m = j0 + k
        self.cur = (self.m - 1) % 2
        if self.m - 1 > 0:
            self._vm_ready = self.m
        self._pending = True
        return k

    def settle(self, res_dev=None, check=True, upto=None, side=False):
        """One host sync: breakdown position, device status of queued iterations and (when
        given) the residual estimates just computed on the device; returns them.  With
        ``check=False`` the status word is kept in ``self.last_status`` for the caller.

        ``upto`` (fast path): only iterations below it are resolved — later ones are
        look-ahead iterations still queued; ``side``: the readback runs on the side stream
        behind the residual checks, so the host does not wait for the look-ahead."""
        upto = self.m if (upto is None or not self.fast) else min(upto, self.m)
        self._pending = upto < self.m
        first = self._settled
        nres = 0 if res_dev is None else res_dev.numel()
        if self.fast:
            st = N.Status()
            nb = upto - first
            def _readback():
                N.check(self.lib.emhd_readback(self.ctx.sync_stream(), D.ptr(self.brk) + 8 * first, nb,
                                               D.ptr(res_dev) if nres else None, nres,
                                               D.ptr(self.host_rb), D.ctypes_byref(st)), "readback")
            if side:
                with torch.cuda.stream(self.side_stream()):
                    _readback()
            else:
                _readback()           # no stream context on the common path (host-bound grids)
            hb = self.host_rb.numpy()
            flags = hb[:nb]
            if nres:
                self.res_host[:nres].copy_(self.host_rb[nb:nb + nres])
        else:
            self.brk_host[:self.m].copy_(self.brk[:self.m], non_blocking=True)
            if res_dev is not None:
                self.res_host[:nres].copy_(res_dev, non_blocking=True)
            st = self.ctx.status()                 # synchronises the stream
            flags = self.brk_host[first:self.m].numpy()
        for k, fv in enumerate(flags):
            self._brk_seen[first + k] = float(fv)
        hit = np.flatnonzero(flags != 0.0)
        if hit.size:
            b = first + int(hit[0])
            self.applies -= self.m - (b + 1)
            self.m = b + 1
            self.breakdown = True
            self._pending = False
            self._settled = self.m
        else:
            self._settled = upto
        if self.comm is not None and self.layout.distributed:
            from .mhd import agree_status
            st = agree_status(st, self.comm)
        self.last_status = st
        if not check:
            if res_dev is not None:
                return self.res_host[:nres].numpy().copy()
            return not self.breakdown
        if self.eng.fused:
            self.check_status(st)
        if st.flags & N.ST_DENSE:
            self.ctx.reset_status()
            raise FloatingPointError("overflow in augmented-matrix exponential")
        if res_dev is not None:
            return self.res_host[:res_dev.numel()].numpy().copy()
        return not self.breakdown

    def check_status(self, st):
        E = self.eng
        if st.flags & (N.ST_RHO | N.ST_PRESSURE | N.ST_NONFINITE):
            if st.fail_iter < 0:
                # flagged by a launch outside this factorisation (a step's RHS / remainder Jv,
                # tagged by Ctx.defer: its report names the reference's cell)
                raise_status(self.ctx, st, self.ctx.deferred_report(st), self.comm)
            j = min(st.fail_iter, self.m - 1)
            a, ah = E.jop.a, E.jop.a_halo
            # the failing state is a + sigma V[j] with V[j] materialised
            v = self.V[j]
            vh = E.gpu.halo(v[:self.n_top])
            sc = E._vn
            N.check(self.lib.emhd_norms(self.ctx.sync_stream(), D.ptr(v), 0, self.n_top,
                                        D.ptr(sc)), "norms")
            if self.layout is not None and self.layout.distributed:
                self.comm.allreduce_max(sc[1:2])
            sc[0:1].copy_(sc[1:2])
            raise_status(self.ctx, st, (1, D.ptr(a), D.ptr(ah), D.ptr(v), D.ptr(vh), D.ptr(sc)),
                         self.comm)

    # -- views ------------------------------------------------------------------
    @property
    def Hm(self):
        return self.H[:self.m, :self.m]

    @property
    def h_next(self):
        if self.breakdown:
            return 0.0
        return float(self.H[self.m, self.m - 1].item())

    def basis(self, host=False):
        m = self.m
        if not self.breakdown:
            self._materialize(m)
        k = m if self.breakdown else m + 1
        V = self.V[:k, :self.naug].T
        H = self.H[:m, :m] if self.breakdown else self.H[:m + 1, :m]
        if host:
            V, H = D.to_host(V.contiguous()), D.to_host(H.contiguous())
        else:
            V, H = V, H.clone()
        sp = (1.0 - self.reorth[:m]) if self.eta > 0.0 else None
        if sp is not None and host:
            sp = D.to_host(sp)
        return ArnoldiBasis(V=V, H=H, m=m, beta=self.beta, breakdown=self.breakdown, second_pass=sp)

    # -- small dense + combination ---------------------------------------------
    def phi_coeffs(self, order, scales):
        """Device Y[s] = beta phi_order(scale_s H_m) e1 and raw residuals (krylov.py:378-383)."""
        if len(scales) > 4:
            parts = []
            for k in range(0, len(scales), 4):
                Yk, rk = self.phi_coeffs(order, scales[k:k + 4])
                parts.append((Yk.clone(), rk.clone()))      # the next call reuses the buffers
            return torch.cat([p[0] for p in parts]), torch.cat([p[1] for p in parts])
        S = len(scales)
        Y = self.Ybuf[:S * self.m].view(S, self.m)
        res = self.resbuf[:S]
        scal = None if self.breakdown else self.scal.dev
        N.check(self.lib.emhd_phi_small_h(self.ctx.sync_stream(), D.ptr(self.H), self.H.shape[1], self.m,
                                          order, S, N.dbl_array(scales),
                                          D.ptr(scal) if scal is not None else D.ptr(self._brk()),
                                          D.ptr(self.beta_dev), D.ptr(Y), D.ptr(res)), "phi_small")
        return Y, res

    def batch_size(self):
        """Speculation depth of the next batch of residual checks.

        The cap is deep when an iteration is cheap relative to a small dense exponential
        (small grids) and 1 on very large grids; within a projection the depth starts at 2
        and doubles after every failed batch, so a projection that converges right after
        m_init wastes at most one iteration while a long one needs O(log m) host syncs."""
        if not self.fast or SPEC_DEPTH_OVERRIDE == 1:
            return 1
        if SPEC_DEPTH_OVERRIDE:
            cap = SPEC_DEPTH_OVERRIDE
        else:
            n = self.n_top
            cap = 8 if n <= (1 << 21) else (4 if n <= (1 << 23) else (2 if n <= (1 << 25) else 1))
        depth = min(cap, self._depth)
        self._depth = min(2 * self._depth, 8)
        return depth

    def phi_batch(self, order, scale, ms, side=False):
        """Residuals (device) of phi_order(scale H_m) e1 for every m in ms, one launch.

        ``side``: the launch runs on the high-priority side stream once the iterations queued
        so far have finished, so Arnoldi iterations queued afterwards (look-ahead) overlap it.
        It reads H[:m, :m], H[m, m-1] and brk[m-1] for m <= max(ms) only, which later
        iterations never write."""
        S = len(ms)
        Y = self.Ybuf[:S * (self.m_cap + 1)].view(S, self.m_cap + 1)
        res = self.resbuf[:S]
        def _launch():
            N.check(self.lib.emhd_phi_small_batch(self.ctx.sync_stream(), D.ptr(self.H), self.H.shape[1],
                                                  N.int_array(ms), order, S, N.dbl_array([scale] * S),
                                                  D.ptr(self.brk), D.ptr(self.beta_dev), D.ptr(Y),
                                                  self.m_cap + 1, D.ptr(res)), "phi_small_batch")
        if side:
            stream = torch.cuda.current_stream()
            ev = torch.cuda.Event()
            ev.record(stream)
            stream = self.side_stream()
            stream.wait_event(ev)
            with torch.cuda.stream(stream):
                _launch()
        else:
            _launch()
        return Y, res

    def side_stream(self):
        s = getattr(self.ctx, "_side_stream", None)
        if s is None:
            s = self.ctx._side_stream = torch.cuda.Stream(priority=-1)
        return s

    def lookahead(self):
        """Iterations to queue behind a batch of residual checks run on the side stream: about
        one small dense exponential's worth of Arnoldi work (0 on very large grids, where one
        iteration outlasts it, and on the per-kernel / multi-rank paths)."""
        if not self.fast or (self.layout is not None and self.layout.distributed):
            return 0
        env = os.environ.get("EMHD_LOOKAHEAD")
        if LOOKAHEAD_OVERRIDE is not None:
            return LOOKAHEAD_OVERRIDE
        if env is not None:
            return max(0, int(env))
        # Measured (config trajectories): 64^2 is host-bound (look-ahead only adds host work),
        # 256^2 gains 12 % with 4, 1024^2 breaks even with 1 (a started look-ahead iteration
        # runs to the end even when cancelled, as long as the exponential it hides)
        n = self.n_top
        return 4 if (1 << 17) < n <= (1 << 20) else 0

    def _cancel_lookahead(self, m_keep):
        """Cancel queued look-ahead iterations >= m_keep (async copy on the idle side stream,
        so it lands ahead of them); later iterations of this process get a new generation."""
        if not (self.fast and self._pending and self.m > m_keep):
            return
        with torch.cuda.stream(self.side_stream()):
            N.check(self.lib.emhd_arnoldi_cancel(self.ctx.sync_stream(), self._args.gen, m_keep),
                    "arnoldi_cancel")
        self._args.gen = self._new_gen()

    def truncate(self, m_keep):
        """Drop speculative iterations beyond m_keep (they were never needed)."""
        drop = self.m - m_keep
        if drop <= 0:
            return
        self.applies -= drop
        self.ctx.spec_dropped = getattr(self.ctx, "spec_dropped", 0) + drop   # reporting only
        if self.fast:
            self._cancel_lookahead(m_keep)
            h = self.ctx.sync_stream()
            # RHS evaluations the dropped iterations actually made (cancelled look-ahead and
            # post-breakdown launches made none), subtracted on the device in stream order;
            # error flags raised by look-ahead iterations after the host read the status are
            # cleared the same way (no reference counterpart: the reference never runs them)
            N.check(self.lib.emhd_evals_discount(h, D.ptr(self.evals[m_keep:]), drop), "evals_discount")
            N.check(self.lib.emhd_status_scrub(h, m_keep), "status_scrub")
        else:
            self.ctx.rhs_discount += drop          # each dropped iteration ran one stencil
        self._pending = False
        self.m = m_keep
        self._settled = min(self._settled, m_keep)
        self.breakdown = bool(self.brk_host_flag(m_keep - 1))

    def brk_host_flag(self, j):
        return self._brk_seen.get(j, 0.0) != 0.0

    def resolve_status(self, m_keep):
        """Raise for device errors of iterations the reference performs (< m_keep); forget
        the ones raised only by discarded speculative iterations.  Flags of look-ahead
        iterations that are still queued (kept, checked by the next batch) stay put."""
        st = self.last_status
        bad = st.flags & (N.ST_RHO | N.ST_PRESSURE | N.ST_NONFINITE)
        if bad and st.fail_iter < m_keep and self.eng.fused:
            self._cancel_lookahead(m_keep)
            self.check_status(st)
        elif self._pending and self.m > m_keep:
            return
        elif st.flags & (N.ST_RHO | N.ST_PRESSURE | N.ST_NONFINITE | N.ST_DENSE):
            # errors of discarded speculative work only: forget them, keep the RHS count
            N.check(self.lib.emhd_status_clear_errors(self.ctx.sync_stream()), "status_clear_errors")

    def account_passes(self):
        """Reporting only (COUNT_PASSES): add this projection's kept iterations and second
        passes to the context's device counters (no host sync; read with pass_counts(ctx))."""
        m = self.m
        if m <= 0 or not COUNT_PASSES:
            return
        acc = getattr(self.ctx, "_pass_acc", None)
        if acc is None:
            acc = self.ctx._pass_acc = torch.zeros(2, dtype=D.F64, device=D.device())
        acc[0] += m
        acc[1] += (m - self.reorth[:m].sum()) if self.eta > 0.0 else float(m)

    def _brk(self):
        if not hasattr(self, "_brk_t"):
            self._brk_t = torch.tensor([0.0, 0.0, 1.0, 0.0], dtype=D.F64).to(D.device())
        return self._brk_t

    def combine(self, Y, outs, bases=None, coefs=None, length=None):
        S = Y.shape[0]
        length = self.n_top if length is None else length
        bases = bases or [None] * S
        coefs = coefs or [1.0] * S
        N.check(self.lib.emhd_combine(self.ctx.sync_stream(), D.ptr(self.V), self.ld, self.m, D.ptr(Y), S,
                                      N.ptr_array([D.ptr(b) for b in bases]), N.dbl_array(coefs),
                                      N.ptr_array([D.ptr(o) for o in outs]), length), "combine")
        return outs


def _engine_for(op, n_top, p=0, ch=1.0, bcols=(), bidx=()):
    if isinstance(op, FdJacobianOperator) and op.gpu is not None:
        return _FusedFd(op, p, ch, bcols, bidx), op.gpu.layout, op.gpu.comm
    return _Generic(op, n_top, p, ch, bcols, bidx), None, None


def _dense_check(ctx):
    st = ctx.status()
    if st.flags & N.ST_DENSE:
        ctx.reset_status()
        raise FloatingPointError("overflow in augmented-matrix exponential")


def arnoldi(op, v, m, reorthogonalize=True):
    """m-step Arnoldi factorisation of ``op`` seeded with ``v`` (krylov.py:191-206)."""
    host = D.is_host(v)
    vd = D.to_device(v).reshape(-1)
    eng, layout, comm = _engine_for(op, vd.numel())
    n_glob = (layout.nx_global * layout.ny * 8) if layout is not None else vd.numel()
    if m > n_glob:
        raise ValueError(f"basis size {m} exceeds operator dimension {op.n}")
    proc = _Process(eng, vd, m, vd.numel(), 0, layout, comm, reorthogonalize=bool(reorthogonalize))
    proc.extend_many(m)
    proc.settle()
    return proc.basis(host=host)


def pass_counts(ctx):
    """(iterations kept, of which ran the second Gram-Schmidt pass) over the projections of
    multi_scale_eval / phi_comb on this context so far (reporting; one host sync)."""
    acc = getattr(ctx, "_pass_acc", None)
    if acc is None:
        return 0, 0
    a = acc.cpu().numpy()
    return int(a[0]), int(a[1])


def residual_estimate(basis, h, c, small_phi_seed):
    """|h_{m+1,m}| |y_m| / ||y|| (krylov.py:209-231)."""
    y = np.asarray(D.to_host(small_phi_seed) if isinstance(small_phi_seed, torch.Tensor)
                   else small_phi_seed, dtype=float)
    nrm = np.linalg.norm(y)
    if nrm == 0.0:
        return 0.0
    return abs(basis.h_next) * abs(y[-1]) / nrm


def _seed_norms(ctx, v, len_dot, n_top, layout, comm):
    """{sum v^2 over len_dot, max|v| over n_top} on the device, all-reduced across slabs, and
    their host values — the zero test of a projection and its beta in ONE host sync."""
    t = torch.zeros(2, dtype=D.F64, device=D.device())
    N.check(ctx.lib.emhd_norms(ctx.sync_stream(), D.ptr(v), len_dot, n_top, D.ptr(t)), "norms")
    if comm is not None and layout is not None and layout.distributed:
        slots = torch.zeros(layout.size + 1, dtype=D.F64, device=D.device())
        N.check(ctx.lib.emhd_slot_norms(ctx.sync_stream(), D.ptr(t), layout.rank, layout.size, D.ptr(slots)),
                "slot_norms")
        comm.allreduce_sum(slots)
        N.check(ctx.lib.emhd_unslot_norms(ctx.sync_stream(), D.ptr(slots), layout.size, D.ptr(t)),
                "unslot_norms")
    host = t.cpu().numpy()
    return t, float(host[0]), float(host[1])


def _maxabs_many(ctx, vecs):
    out = torch.zeros(2 * len(vecs), dtype=D.F64, device=D.device())
    h = ctx.sync_stream()
    for k, v in enumerate(vecs):
        N.check(ctx.lib.emhd_norms(h, D.ptr(v), 0, v.numel(), D.ptr(out[2 * k:2 * k + 2])), "norms")
    return out.view(-1, 2)[:, 1]


def multi_scale_eval(op, h, v, scales, tol, cfg=None, order=1, _into=None):
    """phi_order(c_i h J) v for several scales from one basis (krylov.py:327-375).

    ``_into`` (internal): list of (base, coef, out) triples to fuse the stage
    axpy ``out = base + coef * result`` into the basis sweep.
    """
    cfg = cfg or KrylovConfig()
    scales = list(scales)
    if not scales or any(not (0.0 < c <= 1.0) for c in scales):
        raise ValueError("scales must lie in (0, 1]")
    stats = KrylovStats(projections=1)
    host = D.is_host(v)
    vd = D.to_device(v).reshape(-1)
    eng, layout, comm = _engine_for(op, vd.numel())
    n_top = vd.numel()
    norms_dev, b2, vmax = _seed_norms(eng.ctx, vd, n_top, n_top, layout, comm)
    if vmax == 0.0:
        outs = [torch.zeros(n_top, dtype=D.F64, device=D.device()) for _ in scales]
        if _into:
            for (base, coef, out), o in zip(_into, outs):
                if base is None:
                    out.zero_()
                else:
                    _lincomb(eng.ctx, [base, (coef, o)], out)   # y_n + a * 0, exact order
            outs = [t[2] for t in _into]
        return ([D.to_host(o) for o in outs] if host else outs), stats
    c_big = max(scales)
    proc = _Process(eng, vd, cfg.m_max, n_top, 0, layout, comm, persistent=True,
                    reorthogonalize=cfg.reorthogonalize, seed_norms=(norms_dev, b2))
    m_target = min(cfg.m_init, proc.n)
    # the m_init burst is queued together with the first batch of residual checks: one host
    # sync resolves both (a breakdown inside the burst is caught by that settle, below)
    proc.extend_many(m_target)
    nxt = m_target                                # smallest basis size not yet checked
    look = proc.lookahead()
    while True:
        # speculative batch: the residual at the current m plus up to B-1 further iterations,
        # all checked in one phi launch and one host sync; the reference's decision sequence
        # (stop at the first m with res <= tol, breakdown or m >= n) is replayed on the host.
        # While the checks run (side stream), `look` further iterations are already queued.
        B = proc.batch_size()
        want = nxt + B - 1
        if proc.m < want:
            proc.extend_many(want - proc.m)
        hi = min(want, proc.m)
        ms = list(range(nxt, hi + 1)) or [proc.m]
        _, res_raw = proc.phi_batch(order, c_big * h, ms, side=look > 0)
        if look:
            proc.extend_many(look, lookahead=True)
        raw = proc.settle(res_raw, check=False, upto=hi, side=look > 0)
        if proc.breakdown and proc.m < ms[0]:
            # the burst broke down before m_init: the reference checks the residual at that m
            # (rare: one more launch and sync)
            ms = [proc.m]
            _, res_raw = proc.phi_batch(order, c_big * h, ms)
            raw = proc.settle(res_raw, check=False, upto=proc.m)
        chosen, res = None, None
        for k, mk in enumerate(ms):
            if mk > proc.m:                       # beyond a breakdown found by settle
                break
            res = float(raw[k]) * c_big * h
            if math.isinf(raw[k]):
                proc.truncate(mk)
                proc.resolve_status(mk)
                proc.ctx.reset_status()
                raise FloatingPointError("overflow in augmented-matrix exponential")
            if res <= tol or proc.brk_host_flag(mk - 1) or mk >= proc.n:
                chosen = mk
                break
            if mk >= proc.m_cap:                  # extend() would leave m unchanged
                proc.truncate(mk)
                proc.resolve_status(mk)
                stats.operator_applies += proc.applies
                raise KrylovConvergenceError(
                    f"Krylov basis cap {cfg.m_max} reached in multi-scale "
                    f"evaluation (residual {res:.3e} > {tol:.3e})", residual=res)
        if chosen is not None:
            proc.truncate(chosen)
            proc.resolve_status(chosen)
            break
        proc.resolve_status(hi)
        nxt = hi + 1                              # hi was just checked and failed
    stats.operator_applies += proc.applies
    proc.account_passes()
    stats.max_basis_size = proc.m
    stats.substeps = 1
    Y, _ = proc.phi_coeffs(order, [c * h for c in scales])
    if _into is None:
        raise_status(eng.ctx, eng.ctx.status(), None, comm)    # dense overflow of the last phi
    outs = []
    for k in range(0, len(scales), 4):
        chunk = list(range(k, min(k + 4, len(scales))))
        o = [torch.empty(n_top, dtype=D.F64, device=D.device()) for _ in chunk]
        if _into:
            bases = [_into[i][0] for i in chunk]
            coefs = [_into[i][1] for i in chunk]
            tgt = [_into[i][2] for i in chunk]
            proc.combine(Y[chunk[0]:chunk[-1] + 1].contiguous(), tgt, bases, coefs)
            o = tgt
        else:
            proc.combine(Y[chunk[0]:chunk[-1] + 1].contiguous(), o)
        outs.extend(o)
    return ([D.to_host(o) for o in outs] if host else outs), stats


def phi_comb(req, cfg=None, _zero=None):
    """w = sum_k phi_k(c h J) v_k by the augmented exponential (krylov.py:241-324).

    ``_zero`` (internal): list of booleans marking vectors known to be zero,
    skipping the device zero test.
    """
    cfg = cfg or KrylovConfig()
    stats = KrylovStats(projections=1)
    op = req.operator
    p = len(req.vectors)
    host = any(D.is_host(x) for x in req.vectors)
    vs = [D.to_device(x).reshape(-1) for x in req.vectors]
    n_top = vs[0].numel()
    eng0, layout, comm = _engine_for(op, n_top)
    zero = list(_zero) if _zero is not None else [None] * p
    unknown = [k for k in range(p) if zero[k] is None]
    if unknown:
        mx = _maxabs_many(eng0.ctx, [vs[k] for k in unknown])
        if comm is not None:
            comm.allreduce_max(mx)
        for k, val in zip(unknown, mx.cpu().numpy()):
            zero[k] = float(val) == 0.0
    if all(zero):
        out = torch.zeros(n_top, dtype=D.F64, device=D.device())
        return (D.to_host(out) if host else out), stats
    ch = req.c * req.h
    # columns of B are v_p ... v_1 (krylov.py:264); zero columns contribute nothing
    cols = [(vs[p - 1 - k], k) for k in range(p) if not zero[p - 1 - k]]
    eng, layout, comm = _engine_for(op, n_top, p, ch, [b for b, _ in cols], [k for _, k in cols])
    naug_glob = ((layout.nx_global * layout.ny * 8) if layout is not None else n_top) + p
    u = torch.zeros(n_top, dtype=D.F64, device=D.device())
    seed = torch.zeros(_ld(n_top + p), dtype=D.F64, device=D.device())
    t = 0.0
    delta = 1.0
    while t < 1.0:
        delta = min(delta, cfg.max_substep, 1.0 - t)
        q = np.array([t ** (p - 1 - i) / math.factorial(p - 1 - i) for i in range(p)])
        seed[:n_top].copy_(u)
        seed[n_top:n_top + p].copy_(torch.from_numpy(q))
        # first substep: u = 0 and q = e_p, so ||seed||^2 = 1 exactly — no device norm or sync
        known = None
        if t == 0.0:
            known = (torch.tensor([1.0, 0.0], dtype=D.F64).to(D.device(), non_blocking=True), 1.0)
        proc = _Process(eng, seed[:n_top + p], min(cfg.m_max, naug_glob), n_top, p, layout, comm,
                        reorthogonalize=cfg.reorthogonalize,
                        persistent=True, seed_norms=known)
        m_target = min(cfg.m_init, naug_glob)
        # burst queued together with the first batch of residual checks (one host sync)
        proc.extend_many(m_target)
        nxt = m_target
        look = proc.lookahead()
        while True:
            # speculative batch of residual checks (see multi_scale_eval); extensions stop
            # where the reference could change delta instead of extending (soft cap)
            limit = proc.m_cap if delta <= cfg.min_substep else min(cfg.soft_cap, proc.m_cap)
            B = proc.batch_size()
            want = min(nxt + B - 1, limit)
            if proc.m < want:
                proc.extend_many(want - proc.m)
            hi = min(max(want, nxt), proc.m)
            ms = list(range(nxt, hi + 1)) or [proc.m]
            Yb, res_raw = proc.phi_batch(0, delta, ms, side=look > 0)
            if look and proc.m < limit:
                proc.extend_many(min(look, limit - proc.m), lookahead=True)
            raw = proc.settle(res_raw, check=False, upto=ms[-1], side=look > 0)
            if proc.breakdown and proc.m < ms[0]:
                # breakdown inside the burst: the reference checks the residual at that m
                ms = [proc.m]
                Yb, res_raw = proc.phi_batch(0, delta, ms)
                raw = proc.settle(res_raw, check=False, upto=proc.m)
            tol_sub = req.tol * max(delta, 1e-2)
            action, res = None, None
            for k, mk in enumerate(ms):
                if mk > proc.m:                       # beyond a breakdown found by settle
                    break
                if math.isinf(raw[k]):
                    proc.truncate(mk)
                    proc.resolve_status(mk)
                    proc.ctx.reset_status()
                    raise FloatingPointError("overflow in augmented-matrix exponential")
                res = float(raw[k]) * delta
                if res <= tol_sub or proc.brk_host_flag(mk - 1) or mk >= proc.n:
                    action = ("done", k, mk)
                elif mk >= cfg.soft_cap and delta > cfg.min_substep:
                    action = ("halve", k, mk)
                elif mk >= proc.m_cap:
                    action = ("cap", k, mk)
                if action is not None:
                    break
            if action is None:
                proc.resolve_status(ms[-1])
                nxt = ms[-1] + 1
                continue
            kind, k, mk = action
            proc.truncate(mk)
            proc.resolve_status(mk)
            if kind == "done":
                Y = Yb[k:k + 1, :mk].contiguous()
                break
            if kind == "cap" and delta <= cfg.min_substep:
                stats.operator_applies += proc.applies
                raise KrylovConvergenceError(
                    f"Krylov basis cap {cfg.m_max} reached at substep "
                    f"{delta:.3e} (residual {res:.3e} > {tol_sub:.3e})", residual=res)
            delta = delta / 2.0                       # soft cap, or hard cap above min_substep
            nxt = proc.m
        stats.operator_applies += proc.applies
        proc.account_passes()
        u_new = torch.empty(n_top, dtype=D.F64, device=D.device())
        proc.combine(Y, [u_new])
        u = u_new
        t = t + delta
        stats.substeps += 1
        stats.max_basis_size = max(stats.max_basis_size, proc.m)
        if proc.m <= cfg.grow_threshold:
            delta = delta * cfg.substep_growth
    return (D.to_host(u) if host else u), stats
