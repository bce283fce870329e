#!/usr/bin/env python
"""Micro-benchmark of the Arnoldi streaming kernels (multidot, update modes 0/1) vs nvec."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1604_02614_b200 import _native as N
    from paper_1604_02614_b200 import device as D
    from paper_1604_02614_b200.fdjac import _generic_ctx
    n = int(os.environ.get("NELEM", 8 * 1024 * 1024))
    ld = (n + 31) // 32 * 32
    nv_list = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "4,8,16,24,32,40".split(","))]
    V = torch.randn(max(nv_list) + 1, ld, dtype=torch.float64, device="cuda")
    w = torch.randn(ld, dtype=torch.float64, device="cuda")
    h = torch.randn(256, dtype=torch.float64, device="cuda") * 1e-3
    out = torch.zeros(256, dtype=torch.float64, device="cuda")
    ctx = _generic_ctx()
    L = ctx.lib
    hs = ctx.sync_stream()
    res = []
    for nv in nv_list:
        for kind in ("multidot", "update0", "update1"):
            def run():
                if kind == "multidot":
                    L.emhd_multidot(hs, D.ptr(w), D.ptr(V), ld, nv, n, 1, D.ptr(out))
                else:
                    L.emhd_update(hs, D.ptr(w), D.ptr(V), ld, nv, D.ptr(h), n, n, n,
                                  0 if kind == "update0" else 1, D.ptr(out))
            for _ in range(3):
                run()
            reps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            byts = 8.0 * n * ((nv + 1) if kind == "multidot" else (nv + 2))
            res.append({"nvec": nv, "kernel": kind, "us": round(us, 1), "GBps": round(byts / us / 1e3, 1)})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
