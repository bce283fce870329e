#!/usr/bin/env python
"""Micro-benchmark of the on-device small dense exponential (emhd_expm) vs scipy on the host."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import scipy.linalg
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import _native as N
    from paper_1604_02614_b200 import device as D
    from paper_1604_02614_b200.fdjac import _generic_ctx
    rng = np.random.default_rng(0)
    out = []
    for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "10,20,40,80,110,160,256".split(","))]:
        for scale in (0.5, 20.0):
            H = np.triu(rng.standard_normal((n, n)), -1) * scale / np.sqrt(n)   # Hessenberg-like
            A = D.to_device(H)
            E = torch.empty_like(A)
            work = D.zeros(n + 8)
            ctx = _generic_ctx()
            for _ in range(2):
                N.check(ctx.lib.emhd_expm(ctx.sync_stream(), D.ptr(A), n, D.ptr(E), D.ptr(work)))
            reps = 5
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                N.check(ctx.lib.emhd_expm(ctx.sync_stream(), D.ptr(A), n, D.ptr(E), D.ptr(work)))
            torch.cuda.synchronize()
            gpu_us = (time.perf_counter() - t0) / reps * 1e6
            t0 = time.perf_counter()
            for _ in range(reps):
                Eh = scipy.linalg.expm(H)
            cpu_us = (time.perf_counter() - t0) / reps * 1e6
            err = float(np.max(np.abs(E.cpu().numpy() - Eh)) / max(1.0, np.max(np.abs(Eh))))
            out.append({"n": n, "norm": float(np.linalg.norm(H, 1)), "gpu_us": gpu_us, "scipy_us": cpu_us,
                        "rel_err": err})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
