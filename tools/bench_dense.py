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


def phi_residual_bench():
    """emhd_phi_small_h (order 1, one scale): the residual check of a multi-scale projection."""
    import scipy.linalg
    from paper_1604_02614_b200 import _native as N
    from paper_1604_02614_b200 import device as D
    from paper_1604_02614_b200.fdjac import _generic_ctx
    rng = np.random.default_rng(1)
    out = []
    for m in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "10,20,30,40,60,84,100".split(","))]:
        for scale in (1.0, 30.0):
            H = np.triu(rng.standard_normal((m + 1, m)), -1) * scale / np.sqrt(m)
            Hd = D.to_device(H)
            scal = D.to_device(np.array([abs(H[m, m - 1]), 1.0, 0.0, 0.0]))
            beta = D.to_device(np.array([1.0]))
            Y = D.zeros(m)
            res = D.zeros(1)
            ctx = _generic_ctx()
            h = ctx.sync_stream()
            sc = N.dbl_array([1.0])
            call = lambda: N.check(ctx.lib.emhd_phi_small_h(h, D.ptr(Hd), m, m, 1, 1, sc, D.ptr(scal),   # noqa
                                                            D.ptr(beta), D.ptr(Y), D.ptr(res)))
            for _ in range(3):
                call()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / reps * 1e3
            Ab = np.zeros((m + 1, m + 1))
            Ab[:m, :m] = H[:m, :m]
            Ab[0, m] = 1.0
            want = scipy.linalg.expm(Ab)[:m, m]
            err = float(np.max(np.abs(Y.cpu().numpy() - want)) / max(1e-300, np.max(np.abs(want))))
            out.append({"m": m, "norm": float(np.linalg.norm(H[:m, :m], 1)), "gpu_us": us, "rel_err": err})
    print(json.dumps({"phi_small_residual": out}))


if __name__ == "__main__":
    if sys.argv[1:2] == ["phi"]:
        phi_residual_bench()
    else:
        main()
