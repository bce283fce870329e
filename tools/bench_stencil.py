#!/usr/bin/env python
"""Micro-benchmark of the fused stencil (RHS and Jv) over grid sizes; CUDA-event timed."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200.problems import fourier_grid, fourier_state
    sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["64", "256", "1024", "2048"])]
    res = []
    for n in sizes:
        g = fourier_grid(n)
        prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
        U, rng = fourier_state(g, prm)
        a = torch.from_numpy(U.reshape(-1)).cuda()
        v = torch.from_numpy(rng.standard_normal(U.size)).cuda()
        f = P.make_rhs(prm, g, P.BoundaryPolicy("periodic", "periodic"))
        op = P.FdJacobianOperator(f, a)
        vn = torch.zeros(2, dtype=torch.float64, device="cuda")
        op.vnorm_into(v, vn)
        out = torch.empty_like(a)
        reps = max(10, int(2e9 / (a.numel() * 8 * 4)))
        for kind in ("rhs", "jv"):
            for _ in range(3):
                f.launch(a, out) if kind == "rhs" else op.apply_device(v, out, vn)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                f.launch(a, out) if kind == "rhs" else op.apply_device(v, out, vn)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            byts = (2 if kind == "rhs" else 4) * a.numel() * 8
            res.append({"n": n, "kind": kind, "us": us, "GBps": byts / us / 1e3,
                        "Gcell_per_s": n * n / us / 1e3})
    print(json.dumps({"ty": os.environ.get("EMHD_STENCIL_TY"), "min_rows": os.environ.get("EMHD_MIN_ROWS"),
                      "results": res}))


if __name__ == "__main__":
    main()
