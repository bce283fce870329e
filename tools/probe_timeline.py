#!/usr/bin/env python
"""GPU busy time vs wall time of a trajectory (torch.profiler / CUPTI): how much of a run is
host-induced idle.  python tools/probe_timeline.py [config] (0 = 64^2 EpiRK4 x 20, 1 = KH 256^2)"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200.problems import kh_shear_grid, kh_shear_ic
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    if cfg == 0:
        g = P.ReconnectionSpec().grid(64, 64)
        prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
        f = P.make_rhs(prm, g, P.default_bc("reconnection"))
        y0 = torch.from_numpy(P.reconnection_ic(g, params=prm).reshape(-1)).cuda()
        run = lambda: P.integrate_fixed("epirk4", f, y0, 0.0, 2.0, 0.1, tol_krylov=1e-10)   # noqa: E731
    else:
        g = kh_shear_grid(256)
        prm = P.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-4)
        f = P.make_rhs(prm, g, P.BoundaryPolicy("periodic", "reflect"))
        y0 = torch.from_numpy(kh_shear_ic(g, prm).reshape(-1)).cuda()
        run = lambda: P.integrate_adaptive(f, y0, 0.0, 2.0, P.StepController(tol=1e-6))     # noqa: E731
    run()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        run()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    spans = sorted((e.time_range.start, e.time_range.end) for e in ev if e.time_range.end > e.time_range.start)
    busy = 0.0
    cur_s, cur_e = None, None
    for s, e in spans:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    wall = spans[-1][1] - spans[0][0] if spans else 0.0
    kern = {}
    for e in ev:
        k = e.name.split("(")[0][:50]
        a = kern.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    top = sorted(kern.items(), key=lambda kv: -kv[1][1])[:12]
    print(json.dumps({"config": cfg, "gpu_busy_ms": busy / 1e3, "gpu_span_ms": wall / 1e3,
                      "kernels": len(ev), "top": [[k, n, t / 1e3] for k, (n, t) in top]}, indent=1))


if __name__ == "__main__":
    main()
