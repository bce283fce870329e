#!/usr/bin/env python
"""Micro-benchmark of the Arnoldi-loop stencil (fused normalise + Jv, MODE_JVN) per kernel
variant: python tools/bench_jvn.py 1024,2048 [raw_rows,...] [strip,...] [mode]   (raw rows staged ahead:
1 or 2; strip width 0 = default, 32 / 64 / 96 / 128; mode jvn (default) / jv / rhs: the plain Jv
(4W) and RHS (2W) launches of the same marching kernel)
CUDA-event timed, back-to-back launches on inputs larger than L2 only from 2048^2 up; at 1024^2
the a / w / F(a) / out set (320 MB) already exceeds the 126 MB L2."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import _native as N
    from paper_1604_02614_b200.problems import fourier_grid, fourier_state
    sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1024"])]
    variants = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2"])]
    strips = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0"])]
    mode = sys.argv[4] if len(sys.argv) > 4 else "jvn"
    nw = {"jvn": 5, "jvna": 7, "jv": 4, "rhs": 2}[mode]   # jvna: augmented epilogue, p = 3, two B columns
    res = []
    for n in sizes:
        g = fourier_grid(n)
        prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
        U, rng = fourier_state(g, prm)
        a = torch.from_numpy(U.reshape(-1)).cuda()
        w = torch.from_numpy(rng.standard_normal(U.size)).cuda()
        f = P.make_rhs(prm, g, P.BoundaryPolicy("periodic", "periodic"))
        fa = torch.empty_like(a)
        f.launch(a, fa)
        scal = torch.tensor([float(w.norm()), float(w.abs().max()), 0.0, 0.0], dtype=torch.float64).cuda()
        npad = 8 if mode == "jvna" else 0
        out = torch.empty(a.numel() + npad, dtype=a.dtype, device=a.device)
        vout = torch.empty(a.numel() + npad, dtype=a.dtype, device=a.device)
        if mode == "jvna":
            w = torch.cat([w, torch.from_numpy(rng.standard_normal(npad)).cuda()])
            bcols = [torch.from_numpy(rng.standard_normal(U.size)).cuda() for _ in range(2)]
        L = f.ctx.lib
        ref = None
        for rr, strip in [(r, st) for r in variants for st in strips]:
            f.ctx.stencil_path(kernel=1, raw_rows=rr, strip=strip)

            vn = scal[1:2] / scal[0:1]

            def go():
                if mode == "rhs":
                    f.launch(a, out)
                    return
                if mode == "jv":
                    N.check(L.emhd_jv(f.ctx.sync_stream(), a.data_ptr(), None, fa.data_ptr(), w.data_ptr(),
                                      None, vn.data_ptr(), out.data_ptr()), "jv")
                    return
                if mode == "jvna":
                    N.check(L.emhd_jv_normalized(f.ctx.sync_stream(), a.data_ptr(), None, fa.data_ptr(),
                                                 w.data_ptr(), None, scal.data_ptr(), vout.data_ptr(), 3, 0.37, 2,
                                                 N.ptr_array([b.data_ptr() for b in bcols]), N.int_array([0, 2]),
                                                 out.data_ptr()), "jvna")
                    return
                N.check(L.emhd_jv_normalized(f.ctx.sync_stream(), a.data_ptr(), None, fa.data_ptr(),
                                             w.data_ptr(), None, scal.data_ptr(), vout.data_ptr(), 0, 1.0, 0,
                                             N.ptr_array([]), N.int_array([]), out.data_ptr()), "jvn")
            for _ in range(5):
                go()
            torch.cuda.synchronize()
            same = None
            if ref is None:
                ref = (out.clone(), vout.clone())
            else:
                same = bool(torch.equal(out, ref[0]) and torch.equal(vout, ref[1]))
            reps = max(20, int(4e9 / (U.size * 8 * 5)))
            best = 1e30
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    go()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
            byts = nw * U.size * 8
            res.append({"mode": mode, "n": n, "raw_rows": rr, "us": round(best, 2), "GBps": round(byts / best / 1e3, 1),
                        "ran": f.ctx.last_stencil(), "same_as_first": same})
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
