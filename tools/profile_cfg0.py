#!/usr/bin/env python
"""cProfile of the host side of config 0 (64^2 reconnection, EpiRK4 x 20): where the interpreter
time between the sync points goes.  python tools/profile_cfg0.py [n_top]"""
import cProfile
import io
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1604_02614_b200 as P
    top = int(sys.argv[1]) if len(sys.argv) > 1 else 45
    g = P.ReconnectionSpec().grid(64, 64)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    f = P.make_rhs(prm, g, P.default_bc("reconnection"))
    y0 = torch.from_numpy(P.reconnection_ic(g, params=prm).reshape(-1)).cuda()
    run = lambda: P.integrate_fixed("epirk4", f, y0, 0.0, 2.0, 0.1, tol_krylov=1e-10)   # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        run()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print("wall ms (5 runs):", [round(t * 1e3, 2) for t in ts])
    pr = cProfile.Profile()
    pr.enable()
    run()
    torch.cuda.synchronize()
    pr.disable()
    for key in ("tottime", "cumtime"):
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats(key).print_stats(top)
        print(s.getvalue())


if __name__ == "__main__":
    main()
