"""Host-side logic on CPU: input generators, slab placement, multi-rank halo exchange.

The multi-rank tests run world_size 2 and 3 with the gloo backend on CPU: they
drive the same Comm / SlabLayout code the GPU path uses, with the oracle's
slab RHS standing in for the kernel, and require bit-identical rows.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden
from oracle import stencil
from paper_1604_02614_b200.mhd import BoundaryPolicy, Grid2D, MhdParams
from paper_1604_02614_b200.problems import (ReconnectionSpec, fourier_grid, fourier_state,
                                            reconnection_ic)
from paper_1604_02614_b200.slab import Comm, make_layout, pack_edges_torch, split_rows


def test_reconnection_ic_matches_reference_bitwise():
    z = golden("config0_recon64.npz")
    g = ReconnectionSpec().grid(64, 64)
    U = reconnection_ic(g, params=MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3))
    assert np.array_equal(U, z["U0"])


def test_fourier_state_is_seeded_and_admissible():
    g = fourier_grid(32)
    U1, rng1 = fourier_state(g, MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3))
    U2, _ = fourier_state(g, MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3))
    assert np.array_equal(U1, U2)
    assert U1[0].min() > 0.5
    p = stencil.pressure_field(U1, MhdParams())
    assert p.min() > 0.5


def test_split_rows_balanced():
    for nx in (16, 17, 1024, 4096):
        for P in (1, 2, 3, 4, 8):
            c, o = split_rows(nx, P)
            assert sum(c) == nx and max(c) - min(c) <= 1
            assert o[0] == 0 and all(o[k] + c[k] == o[k + 1] for k in range(P - 1))


def test_layout_neighbours():
    L = make_layout(64, 32, "periodic", 0, 4)
    assert (L.lo_neighbor, L.hi_neighbor, L.bc_lo, L.bc_hi) == (3, 1, "external", "external")
    L = make_layout(64, 32, "reflect", 0, 4)
    assert (L.lo_neighbor, L.hi_neighbor, L.bc_lo, L.bc_hi) == (-1, 1, "reflect", "external")
    L = make_layout(64, 32, "reflect", 3, 4)
    assert (L.lo_neighbor, L.hi_neighbor, L.bc_lo, L.bc_hi) == (2, -1, "external", "reflect")
    L = make_layout(64, 32, "periodic", 0, 1)
    assert not L.distributed and L.bc_lo == "periodic"
    with pytest.raises(ValueError):
        make_layout(4, 8, "periodic", 0, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _slab_worker(rank, size, port, bcx, nx, ny):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        g = Grid2D(nx, ny, -1.0, 2.0, -0.7, 0.9)
        bc = BoundaryPolicy(bcx, "reflect")
        P = MhdParams(mu=1e-2, eta=3e-3, kappa=2e-2)
        rng = np.random.default_rng(7)
        U = np.zeros((8, nx, ny))
        U[0] = 1 + 0.3 * rng.random((nx, ny))
        U[1:4] = 0.3 * rng.standard_normal((3, nx, ny))
        U[4:7] = rng.standard_normal((3, nx, ny))
        U[7] = 40 + rng.random((nx, ny))
        F_global = stencil.mhd_rhs(U, P, g, bc)
        L = make_layout(nx, ny, bcx, rank, size)
        Ul = np.ascontiguousarray(U[:, L.x_offset:L.x_offset + L.nx_local, :])
        send = pack_edges_torch(torch.from_numpy(Ul).reshape(-1), L.nx_local, ny)
        recv = torch.full_like(send, float("nan"))
        Comm(L).exchange(send, recv)
        lo = recv[0].numpy() if L.bc_lo == "external" else None
        hi = recv[1].numpy() if L.bc_hi == "external" else None
        Fl = stencil.mhd_rhs_slab(Ul, lo, hi, P, g, bc)
        want = F_global[:, L.x_offset:L.x_offset + L.nx_local, :]
        assert np.array_equal(Fl, want), f"rank {rank}: slab RHS differs"
        # the Arnoldi reductions: partial dots + all-reduce == global dot (to round-off)
        w = np.sin(np.arange(U.size) * 0.37).reshape(U.shape)
        part = torch.tensor([float(np.sum(w[:, L.x_offset:L.x_offset + L.nx_local, :] * Ul)),
                             float(np.max(np.abs(Ul)))], dtype=torch.float64)
        c = Comm(L)
        c.allreduce_sum(part[0:1])
        c.allreduce_max(part[1:2])
        assert abs(part[0].item() - float(np.sum(w * U))) <= 1e-12 * abs(float(np.sum(w * U)))
        assert part[1].item() == float(np.max(np.abs(U)))
        # one-collective norms (emhd_slot_norms layout): {sum, max of rank r at 1 + r}
        slots = torch.zeros(size + 1, dtype=torch.float64)
        slots[0] = float(np.sum(Ul * Ul))
        slots[1 + rank] = float(np.max(np.abs(Ul)))
        c.allreduce_sum(slots)
        assert abs(slots[0].item() - float(np.sum(U * U))) <= 1e-12 * float(np.sum(U * U))
        assert slots[1:].max().item() == float(np.max(np.abs(U)))
        # peer-memory halo push needs NCCL + symmetric memory: gloo keeps the exchange
        from paper_1604_02614_b200.slab import PushHalo
        assert PushHalo.create(L, c) is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size,bcx", [(2, "periodic"), (2, "reflect"), (3, "periodic"),
                                      (3, "zero-gradient")])
def test_gloo_slab_halo_exchange_matches_single_domain(size, bcx):
    mp.spawn(_slab_worker, args=(size, _free_port(), bcx, 13, 9), nprocs=size, join=True)
