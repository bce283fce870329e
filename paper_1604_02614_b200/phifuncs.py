"""phi functions (reference phifuncs.py).

``phi_dense`` evaluates phi_0..phi_kmax of a small dense matrix with ONE
exponential of the block upper-bidiagonal augmented matrix, on the GPU
(emhd_expm, csrc/dense.cu — the Al-Mohy & Higham 2009 scaling-and-squaring
algorithm that the reference reaches through scipy.linalg.expm,
phifuncs.py:65-107).  ``phi_scalar`` is the reference's scalar formula
(phifuncs.py:32-62); it is host arithmetic on one number, not vector work.
"""

import math

import numpy as np
import torch

from . import _native as N
from . import device as D
from .fdjac import _generic_ctx

MAX_ORDER = 4
SMALL_ARG_THRESHOLD = 0.5
SERIES_TERMS = 20


def _check_order(k):
    if not isinstance(k, (int, np.integer)) or k < 0 or k > MAX_ORDER:
        raise ValueError(f"phi order must be an integer in [0, {MAX_ORDER}], got {k!r}")


def phi_scalar(k, z):
    _check_order(k)
    z = complex(z) if np.iscomplexobj(z) or isinstance(z, complex) else float(z)
    if k == 0:
        return np.exp(z)
    if abs(z) < SMALL_ARG_THRESHOLD:
        acc = 0.0
        zp = 1.0
        for j in range(SERIES_TERMS):
            acc += zp / math.factorial(j + k)
            zp = zp * z
        return acc
    val = np.exp(z)
    for j in range(k):
        val = (val - 1.0 / math.factorial(j)) / z
    return val


def expm(A):
    """exp(A) of a small dense matrix on the GPU (host in -> host out)."""
    host = D.is_host(A)
    Ad = D.to_device(A)
    if Ad.dim() != 2 or Ad.shape[0] != Ad.shape[1]:
        raise ValueError(f"A must be square, got shape {tuple(Ad.shape)}")
    n = Ad.shape[0]
    E = torch.empty_like(Ad)
    work = D.zeros(n + 8)
    ctx = _generic_ctx()
    N.check(ctx.lib.emhd_expm(ctx.sync_stream(), D.ptr(Ad), n, D.ptr(E), D.ptr(work)), "expm")
    st = ctx.status()
    if st.flags & N.ST_DENSE:
        ctx.reset_status()
        raise FloatingPointError("overflow in augmented-matrix exponential")
    return D.to_host(E) if host else E


def phi_dense(k_max, H):
    """[phi_0(H), ..., phi_kmax(H)] via one augmented exponential (phifuncs.py:65-107)."""
    _check_order(k_max)
    host = D.is_host(H)
    Hh = np.asarray(D.to_host(H) if not host else H, dtype=float)
    if Hh.ndim != 2 or Hh.shape[0] != Hh.shape[1]:
        raise ValueError(f"H must be square, got shape {Hh.shape}")
    if not np.all(np.isfinite(Hh)):
        raise FloatingPointError("H contains non-finite entries")
    n = Hh.shape[0]
    dim = (k_max + 1) * n
    A = np.zeros((dim, dim))
    A[:n, :n] = Hh
    for j in range(k_max):
        blk = (j + 1) * n
        A[j * n:blk, blk:blk + n] = np.eye(n)
    E = expm(D.to_device(A))
    out = [E[:n, j * n:(j + 1) * n].contiguous() for j in range(k_max + 1)]
    return [D.to_host(x) for x in out] if host else out
