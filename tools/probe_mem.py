#!/usr/bin/env python
"""Device-memory probe of the EpiRK4 driver: live bytes after each run and after gc.collect().

    python tools/probe_mem.py [n]          # config-4 physics on an n x n grid, default 1024

Reports torch.cuda.memory_allocated() (live tensors) and the peak of each run; memory that a
gc.collect() frees was held by reference cycles (garbage the driver should not leave behind).
"""
import gc
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1604_02614_b200 as P
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    gc.disable()
    g = P.ReconnectionSpec().grid(n, n)
    prm = P.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-3)
    bc = P.default_bc("reconnection")
    y0 = torch.from_numpy(P.reconnection_ic(g, params=prm).reshape(-1)).cuda()
    f = P.make_rhs(prm, g, bc)
    cfg = P.KrylovConfig(m_max=128)
    W = y0.numel() * 8
    rows = []
    for k in range(3):
        torch.cuda.reset_peak_memory_stats()
        y, st = P.integrate_fixed("epirk4", f, y0, 0.0, 0.24, 0.12, tol_krylov=1e-10, cfg=cfg)
        torch.cuda.synchronize()
        del y
        a0 = torch.cuda.memory_allocated()
        peak = torch.cuda.max_memory_allocated()
        freed = gc.collect()
        a1 = torch.cuda.memory_allocated()
        rows.append({"run": k, "live_W": a0 / W, "after_gc_W": a1 / W, "peak_W": peak / W,
                     "gc_objects": freed, "basis_W": getattr(f.ctx, "_basis", torch.empty(0)).numel() * 8 / W})
    # what the cycles are made of: one more run, garbage saved instead of freed
    y, st = P.integrate_fixed("epirk4", f, y0, 0.0, 0.24, 0.12, tol_krylov=1e-10, cfg=cfg)
    del y
    gc.set_debug(gc.DEBUG_SAVEALL)
    gc.collect()
    from collections import Counter
    kinds = Counter(type(o).__qualname__ for o in gc.garbage)
    big = []
    for o in gc.garbage:
        if isinstance(o, torch.Tensor) and o.is_cuda and o.numel() * 8 >= W // 2:
            holders = [type(r).__qualname__ for r in gc.get_referrers(o) if r is not gc.garbage][:4]
            big.append({"numel": o.numel(), "holders": holders})
    cyc = []
    for o in gc.garbage:
        if type(o).__qualname__ in ("_Process", "_FusedFd", "_Generic", "FdJacobianOperator", "frame", "function", "cell"):
            cyc.append(type(o).__qualname__ + (":" + o.f_code.co_name if hasattr(o, "f_code") else "") +
                       (":" + o.__qualname__ if type(o).__name__ == "function" else ""))
    print(json.dumps({"n": n, "W_bytes": W, "runs": rows, "garbage_kinds": kinds.most_common(25),
                      "big_tensors": big[:20], "named": cyc[:60]}))


if __name__ == "__main__":
    main()
