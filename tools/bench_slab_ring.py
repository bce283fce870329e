#!/usr/bin/env python
"""Cost of the slab path on one GPU: BASELINE config 2's step (arnoldi(FdJacobianOperator, v, 40))
on the whole grid vs. on a ring of one slab rank (this GPU is its own lo / hi neighbour, x
periodic) whose collectives run inside the library (slab.NativeComm, NCCL 1-rank
communicators): every iteration then issues the all-reduces from C and exchanges the halo on a
second stream while the stencil's interior rows run.  Same arithmetic, device-timed.

    python tools/bench_slab_ring.py [n ...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_steps(fn, steps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200.problems import fourier_grid, fourier_state, unit_start_vector
    from paper_1604_02614_b200.slab import Comm, NativeComm, make_ring_layout
    sizes = [int(x) for x in sys.argv[1:]] or [256, 1024]
    for n in sizes:
        g = fourier_grid(n)
        prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
        bc = P.BoundaryPolicy("periodic", "periodic")
        U, rng = fourier_state(g, prm, seed=1604)
        a = torch.from_numpy(U.reshape(-1)).cuda()
        v = torch.from_numpy(unit_start_vector(rng, U.size)).cuda()
        steps = 10 if n <= 1024 else 3
        row = {"grid": n, "m": 40}
        ref = None
        for name, mk in (("single_domain", lambda: P.make_rhs(prm, g, bc)),
                         ("ring_native_nccl", lambda: P.make_rhs(prm, g, bc, layout=make_ring_layout(n, n),
                                                                 comm=NativeComm(make_ring_layout(n, n)))),
                         ("ring_python_per_kernel", lambda: P.make_rhs(prm, g, bc, layout=make_ring_layout(n, n),
                                                                       comm=Comm(make_ring_layout(n, n))))):
            f = mk()
            op = P.FdJacobianOperator(f, a)
            box = {}

            def step():
                box["b"] = P.arnoldi(op, v, 40)
            ms = time_steps(step, steps)
            H = box["b"].H.cpu().numpy()
            if ref is None:
                ref = H
            row[name] = {"ms_per_step": ms, "iterations_per_s": 40 / (ms / 1e3),
                         "H_rel_diff_vs_single": float(np.linalg.norm(H - ref) / np.linalg.norm(ref))}
            del op, f, box
            torch.cuda.empty_cache()
        row["native_overhead"] = row["ring_native_nccl"]["ms_per_step"] / row["single_domain"]["ms_per_step"] - 1
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
