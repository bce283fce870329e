#!/usr/bin/env python
"""Where a small-grid trajectory's wall time goes on the host: time blocked in the sync points
(Arnoldi settle / readback, seed-norm and zero-test readbacks, status reads) against the rest
(Python + launches).  python tools/probe_host_waits.py   (config 0: 64^2, EpiRK4 x 20)"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import device as D
    from paper_1604_02614_b200 import krylov as K
    acc = {}

    def wrap(obj, name, key):
        fn = getattr(obj, name)

        def w(*a, **k):
            t0 = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                d = acc.setdefault(key, [0, 0.0])
                d[0] += 1
                d[1] += time.perf_counter() - t0
        setattr(obj, name, w)

    wrap(K._Process, "settle", "settle (readback + sync)")
    wrap(K, "_seed_norms", "seed norms readback")
    wrap(K, "_maxabs_many", "zero-test launch")
    wrap(D.Ctx, "status", "status read")
    wrap(K._Process, "__init__", "_Process.__init__")
    wrap(K._Process, "extend_many", "extend_many (launches)")
    wrap(K._Process, "phi_batch", "phi_batch launch")
    wrap(K._Process, "truncate", "truncate")
    wrap(K._Process, "combine", "combine")
    wrap(torch.Tensor, "cpu", "tensor.cpu()")
    g = P.ReconnectionSpec().grid(64, 64)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    f = P.make_rhs(prm, g, P.default_bc("reconnection"))
    y0 = torch.from_numpy(P.reconnection_ic(g, params=prm).reshape(-1)).cuda()
    run = lambda: P.integrate_fixed("epirk4", f, y0, 0.0, 2.0, 0.1, tol_krylov=1e-10)   # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    acc.clear()
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    T = time.perf_counter() - t0
    print(json.dumps({"wall_ms": T * 1e3,
                      "blocked_or_spent_ms": {k: [n, round(t * 1e3, 3)] for k, (n, t) in acc.items()}}, indent=1))


if __name__ == "__main__":
    main()
