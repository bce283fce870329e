import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libemhd.so")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


class Obj:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def case_objects(z, k):
    """(grid, params, bc) duck-typed objects for rhs_jv_cases case k."""
    gt = z[f"c{k}_grid"]
    pt = z[f"c{k}_params"]
    bt = z[f"c{k}_bc"]
    names = ["periodic", "reflect", "zero-gradient"]
    from paper_1604_02614_b200.mhd import BoundaryPolicy, Grid2D, MhdParams
    g = Grid2D(int(gt[0]), int(gt[1]), gt[2], gt[3], gt[4], gt[5])
    P = MhdParams(mu=pt[0], eta=pt[1], kappa=pt[2], gamma=pt[3], b_half=bool(pt[4]))
    bc = BoundaryPolicy(names[int(bt[0])], names[int(bt[1])])
    return g, P, bc
