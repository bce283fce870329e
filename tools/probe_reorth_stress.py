"""Probe for the selective re-orthogonalisation stress test: per-column H differences of
eta = 0.5 / 1/sqrt(2) against always-two-pass, and of two-pass against itself on a seed
perturbed by one ulp (the FD operator's own chaotic floor)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import krylov
    from oracle import jvp, stencil
    from test_gpu_parity import _invariant_pair_seed
    n = 32
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 120
    amp = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-5
    g = P.Grid2D(n, n, 0.0, 1.0, 0.0, 1.0)
    prm = P.MhdParams(mu=1e-2, eta=1e-2, kappa=1e-2)
    bc = P.BoundaryPolicy("periodic", "periodic")
    U = np.zeros((8, n, n)); U[0] = 1.0; U[4] = 1.0; U[7] = 2.0
    x = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(x, x, indexing="ij")
    u = _invariant_pair_seed(jvp.FdJv(stencil.rhs_closure(prm, g, bc), U.reshape(-1)), n, X, Y, 1, 1)
    rng = np.random.default_rng(5)
    v = u.copy()
    for (k, l) in ((2, 1), (0, 3)):
        v += (amp * rng.standard_normal((8, 1, 1)) * np.cos(2 * np.pi * (k * X + l * Y) + rng.uniform(0, 6))).reshape(-1)
    op = P.FdJacobianOperator(P.make_rhs(prm, g, bc), U.reshape(-1))
    runs = {}
    for name, eta, seed in (("two", 0.0, v), ("two_ulp", 0.0, np.nextafter(v, 2 * v)),
                            ("e05", 0.5, v), ("e07", 1 / np.sqrt(2), v)):
        krylov.REORTH_ETA = eta
        b = P.arnoldi(op, torch.from_numpy(seed).cuda(), m)
        V = b.V.clone()
        G = (V.T @ V).cpu().numpy()
        runs[name] = dict(H=b.H.cpu().numpy(), m=b.m, orth=float(np.max(np.abs(G - np.eye(G.shape[0])))),
                          sp=None if b.second_pass is None else b.second_pass.cpu().numpy())
    H2 = runs["two"]["H"]
    colnorm = np.linalg.norm(H2, axis=0)
    out = {}
    for name in ("two_ulp", "e05", "e07"):
        H = runs[name]["H"]
        d = np.linalg.norm(H - H2, axis=0) / colnorm
        first = [int(np.argmax(d > t)) if np.any(d > t) else None for t in (1e-10, 1e-8, 1e-6, 1e-3)]
        cum = [float(np.linalg.norm(H[:, :k + 1] - H2[:, :k + 1]) / np.linalg.norm(H2[:, :k + 1])) for k in range(H.shape[1])]
        out[name] = {"m": runs[name]["m"], "orth": runs[name]["orth"],
                     "first_col_over_1e-10_1e-8_1e-6_1e-3": first,
                     "cum_rel_at_20_40_60_80_100_119": [cum[k] for k in (20, 40, 60, 80, 100, min(119, len(cum) - 1))],
                     "second_passes": None if runs[name]["sp"] is None else int(runs[name]["sp"].sum())}
    rat = [H2[j + 1, j] / np.linalg.norm(H2[:j + 2, j]) for j in range(H2.shape[1])]
    out["two_ratio_min_first10"] = [float(r) for r in rat[:10]]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
