#!/usr/bin/env python
"""Per-rank proxy for strong scaling: one GPU runs the Arnoldi of a P-way x-slab (nx/P x ny
grid, periodic) through the fast C driver and through the per-kernel Python path that slab
ranks use, to show where host overhead caps the multi-rank iteration rate.

    python tools/probe_slab_host.py [n] [P...]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import krylov as K
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    parts = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    m = 40
    out = []
    from paper_1604_02614_b200.problems import fourier_grid, fourier_state, unit_start_vector
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    gfull = fourier_grid(n)
    Ufull, rng = fourier_state(gfull, prm)             # bench.py's config-2 state at n x n
    vfull = unit_start_vector(rng, Ufull.size).reshape(Ufull.shape)
    for p in parts:
        # rank 0's slab of a P-way x-decomposition (periodic wrap in place of the halo: same work)
        g = P.Grid2D(n // p, n, 0.0, 1.0 / p, 0.0, 1.0)
        U = np.ascontiguousarray(Ufull[:, :n // p, :])
        f = P.make_rhs(prm, g, P.BoundaryPolicy("periodic", "periodic"))
        a = torch.from_numpy(U.reshape(-1)).cuda()
        v = torch.from_numpy(np.ascontiguousarray(vfull[:, :n // p, :]).reshape(-1)).cuda()
        op = P.FdJacobianOperator(f, a)
        row = {"P": p, "rank_grid": [n // p, n]}
        for fast in (True, False):
            K.FAST_DRIVER = fast
            for _ in range(2):
                P.arnoldi(op, v, m)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            reps = 5
            for _ in range(reps):
                P.arnoldi(op, v, m)
            e1.record()
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) / reps / m * 1e6
            dev = e0.elapsed_time(e1) * 1e3 / reps / m
            row["fast" if fast else "per_kernel_python"] = {"us_per_iteration": dev, "wall_us": wall}
        K.FAST_DRIVER = True
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
