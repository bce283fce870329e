"""Slab ranks with their collectives inside the library (slab.NativeComm, emhd_comm_init_*).

The slab path then keeps the one-C-call-per-iteration Arnoldi driver: the dot / norm
all-reduces of krylov.py:151,153,158,161 are issued from C between the kernels, and the x-halo
of the vector a stencil perturbs is exchanged on a second stream while the stencil's interior
rows [2, nx-2) run (the edge rows follow).

* ring of one (this GPU is its own lo and hi neighbour, periodic x): every slab code path —
  EXTERNAL boundaries, NCCL send/recv + all-reduce (1-rank communicator), the interior / edge
  split — against the single-domain result and the oracle, for both transports;
* 2 and 3 processes sharing one GPU through the host transport (gloo): the multi-rank control
  flow of the C driver against the reference fixtures (no kernel waits on another rank);
* 2 processes on 2 GPUs over NCCL when the box has them (skipped on one GPU).
"""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT, case_objects, golden

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def P():
    import paper_1604_02614_b200 as P
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("transport", ["nccl", "host"])
def test_ring_of_one_matches_single_domain(P, transport):
    from oracle import jvp, stencil
    from paper_1604_02614_b200 import krylov
    from paper_1604_02614_b200.slab import Comm, NativeComm, make_ring_layout
    z = golden("rhs_jv_cases.npz")
    for k in range(int(z["ncases"][0])):
        g, prm, bc = case_objects(z, k)
        if bc.x != "periodic" or g.nx < 4:
            continue
        ring = make_ring_layout(g.nx, g.ny)
        f = P.make_rhs(prm, g, bc, layout=ring, comm=NativeComm(ring, transport=transport))
        assert f.native and f.layout.distributed
        U = z[f"c{k}_U"].reshape(-1)
        for kernel in (1, 2):             # marching strips (interior / edge split) and 2D tiles
            f.ctx.stencil_path(kernel=kernel)
            assert np.array_equal(f(U), z[f"c{k}_F"].reshape(-1)), (k, kernel, "rhs")
            op = P.FdJacobianOperator(f, U)
            assert np.array_equal(op(z[f"c{k}_v"]), z[f"c{k}_Jv"]), (k, kernel, "jv")
            if kernel == 1 and transport == "nccl" and g.nx > 4:
                assert f.ctx.last_stencil()["rows_per_cta"] == 2     # the edge-row launch ran last
        f.ctx.stencil_path(kernel=0)

    # Arnoldi through the C slab driver == the single-domain C driver bit for bit (same kernels,
    # same predicted re-projection, 1-rank reductions), the Python per-kernel slab path and the
    # reference fixture to the FD bar
    zk = golden("krylov_mhd.npz")
    gt, pt = zk["grid"], zk["params"]
    g = P.Grid2D(int(gt[0]), int(gt[1]), gt[2], gt[3], gt[4], gt[5])
    prm = P.MhdParams(mu=pt[0], eta=pt[1], kappa=pt[2], gamma=pt[3], b_half=bool(pt[4]))
    bc = P.BoundaryPolicy("periodic", "reflect")
    ring = make_ring_layout(g.nx, g.ny)
    fn = P.make_rhs(prm, g, bc, layout=ring, comm=NativeComm(ring, transport=transport))
    fp = P.make_rhs(prm, g, bc, layout=ring, comm=Comm(ring))
    fs = P.make_rhs(prm, g, bc)
    out = []
    for f in (fn, fs, fp):
        op = P.FdJacobianOperator(f, zk["a"], zk["fa"])
        b = P.arnoldi(op, zk["v"], 12)
        out.append(b)
        assert b.m == 12 and not b.breakdown
        assert np.linalg.norm(b.H - zk["H"]) <= 1e-8 * np.linalg.norm(zk["H"])
    assert np.array_equal(out[0].H, out[1].H) and np.array_equal(out[0].V, out[1].V)
    # the fast (C-driver) path was taken on the native ring
    proc_fast = krylov._Process(krylov._FusedFd(P.FdJacobianOperator(fn, zk["a"], zk["fa"])),
                                dev(zk["v"]), 4, zk["a"].size, 0, ring, fn.comm)
    assert proc_fast.fast

    # multi-scale / phi-comb counters and one config-0 EpiRK4 step on the ring
    op = P.FdJacobianOperator(fn, zk["a"], zk["fa"])
    outs, st = P.multi_scale_eval(op, 0.5, 0.5 * zk["fa"], [0.5, 2.0 / 3.0, 1.0], 1e-10)
    assert [st.operator_applies, st.substeps, st.max_basis_size] == list(zk["ms_stats"])
    n = zk["a"].size
    w, st = P.phi_comb(P.PhiCombRequest(operator=op, h=0.5, c=1.0,
                                        vectors=[np.zeros(n), np.zeros(n), zk["vec3"], 0.5 * zk["vec3"]],
                                        tol=1e-10))
    assert [st.operator_applies, st.substeps, st.max_basis_size] == list(zk["pc_stats"])
    assert np.linalg.norm(w - zk["pc_w"]) <= 1e-8 * np.linalg.norm(zk["pc_w"])
    z0 = golden("config0_recon64.npz")
    with open(os.path.join(GOLDEN, "config0_stats.json")) as fh:
        s1 = json.load(fh)["step1"]
    g = P.ReconnectionSpec().grid(64, 64)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    ring = make_ring_layout(64, 64)
    f = P.make_rhs(prm, g, P.default_bc("reconnection"), layout=ring,
                   comm=NativeComm(ring, transport=transport))
    y1, S = P.epirk4_step(f, z0["U0"].reshape(-1), 0.1, 1e-10)
    assert np.linalg.norm(y1 - z0["y1"]) <= 1e-8 * np.linalg.norm(z0["y1"])
    for key, v in s1.items():
        assert getattr(S, key) == v, key


def _worker(rank, size, port, transport, ndev):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev_i = rank % ndev
    torch.cuda.set_device(dev_i)
    if transport == "host":
        dist.init_process_group("gloo", rank=rank, world_size=size)
    else:
        dist.init_process_group("nccl", rank=rank, world_size=size, device_id=torch.device("cuda", dev_i))
    try:
        import paper_1604_02614_b200 as P
        from paper_1604_02614_b200.mhd import local_rows
        from paper_1604_02614_b200.slab import NativeComm, make_layout
        from conftest import case_objects, golden

        z = golden("rhs_jv_cases.npz")
        for k in (0, 3, 4):
            g, prm, bc = case_objects(z, k)
            L = make_layout(g.nx, g.ny, bc.x, rank, size)
            f = P.make_rhs(prm, g, bc, layout=L, comm=NativeComm(L, transport=transport))
            a = local_rows(z[f"c{k}_U"].reshape(-1), g, L)
            assert np.array_equal(f(a), local_rows(z[f"c{k}_F"].reshape(-1), g, L)), (k, "rhs")
            op = P.FdJacobianOperator(f, a)
            assert np.array_equal(op(local_rows(z[f"c{k}_v"], g, L)), local_rows(z[f"c{k}_Jv"], g, L)), (k, "jv")

        zk = golden("krylov_mhd.npz")
        gt, pt = zk["grid"], zk["params"]
        g = P.Grid2D(int(gt[0]), int(gt[1]), gt[2], gt[3], gt[4], gt[5])
        prm = P.MhdParams(mu=pt[0], eta=pt[1], kappa=pt[2], gamma=pt[3], b_half=bool(pt[4]))
        bc = P.BoundaryPolicy("periodic", "reflect")
        L = make_layout(g.nx, g.ny, bc.x, rank, size)
        f = P.make_rhs(prm, g, bc, layout=L, comm=NativeComm(L, transport=transport))
        op = P.FdJacobianOperator(f, local_rows(zk["a"], g, L), local_rows(zk["fa"], g, L))
        b = P.arnoldi(op, local_rows(zk["v"], g, L), 12)
        assert b.m == 12
        assert np.linalg.norm(b.H - zk["H"]) <= 1e-8 * np.linalg.norm(zk["H"])
        outs, st = P.multi_scale_eval(op, 0.5, local_rows(0.5 * zk["fa"], g, L),
                                      [0.5, 2.0 / 3.0, 1.0], 1e-10)
        assert [st.operator_applies, st.substeps, st.max_basis_size] == list(zk["ms_stats"])
        w, st = P.phi_comb(P.PhiCombRequest(
            operator=op, h=0.5, c=1.0,
            vectors=[np.zeros(L.n_local), np.zeros(L.n_local), local_rows(zk["vec3"], g, L),
                     local_rows(0.5 * zk["vec3"], g, L)], tol=1e-10))
        assert [st.operator_applies, st.substeps, st.max_basis_size] == list(zk["pc_stats"])
        assert np.linalg.norm(w - local_rows(zk["pc_w"], g, L)) <= 1e-8 * np.linalg.norm(zk["pc_w"])

        z0 = golden("config0_recon64.npz")
        with open(os.path.join(GOLDEN, "config0_stats.json")) as fh:
            s1 = json.load(fh)["step1"]
        g = P.ReconnectionSpec().grid(64, 64)
        prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
        bc = P.default_bc("reconnection")
        L = make_layout(g.nx, g.ny, bc.x, rank, size)
        f = P.make_rhs(prm, g, bc, layout=L, comm=NativeComm(L, transport=transport))
        y1, S = P.epirk4_step(f, local_rows(z0["U0"].reshape(-1), g, L), 0.1, 1e-10)
        assert np.linalg.norm(y1 - local_rows(z0["y1"], g, L)) <= 1e-8 * np.linalg.norm(z0["y1"]) / np.sqrt(size)
        for key, v in s1.items():
            assert getattr(S, key) == v, key
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3])
def test_host_transport_ranks_on_one_gpu_match_reference(size):
    mp.spawn(_worker, args=(size, _port(), "host", 1), nprocs=size, join=True)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (one NCCL rank per GPU)")
def test_nccl_ranks_on_two_gpus_match_reference():
    mp.spawn(_worker, args=(2, _port(), "nccl", torch.cuda.device_count()), nprocs=2, join=True)


def test_ring_of_one_predicted_reprojection_both_branches(P):
    """Config 0's state drives both selective re-orthogonalisation branches (and mispredicted
    re-projections): the slab C driver on a ring of one equals the single-domain C driver bit
    for bit over 40 iterations (decision taken by a separate kernel from the all-reduced sums,
    gated multi-dot into scratch + all-reduce + gated copy on a misprediction)."""
    from paper_1604_02614_b200.slab import NativeComm, make_ring_layout
    g = P.ReconnectionSpec().grid(64, 64)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    bc = P.default_bc("reconnection")
    y0 = P.reconnection_ic(g, params=prm).reshape(-1)
    ring = make_ring_layout(64, 64)
    res = []
    for f in (P.make_rhs(prm, g, bc), P.make_rhs(prm, g, bc, layout=ring, comm=NativeComm(ring))):
        yd = dev(y0)
        op = P.FdJacobianOperator(f, yd)
        b = P.arnoldi(op, f(yd), 40)
        res.append((b.H.cpu().numpy(), b.V.cpu().numpy(), b.second_pass.cpu().numpy()))
    sp = res[0][2]
    assert 0 < sp.sum() < len(sp)
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])
