#!/usr/bin/env python
"""Measurement of the output-side rows on one GPU.

    python tools/bench_output.py [n1,n2,...]        # default 1024,4096

Per grid (Harris-sheet state of BASELINE configs 3/4, eta = mu = 1e-4, kappa = 1e-3):
div_B, current_J, error_norm, rk4_stable_dt, one explicit RK4 step through integrate_rk4,
and a .mhd25 snapshot write + read of the device state.  Device work is timed with CUDA
events after warm-up; algorithmic bytes per call (C = nx * ny cells, W = 64 C bytes):

  div_B          read Bx, By, write divB              3 * 8C
  current_J      read Bx, By, Bz, write 3 planes      6 * 8C
  error_norm     read U, U_ref                        2W
  rk4_stable_dt  read U                               1W
  RK4 step       4 RHS (2W) + 3 stage inputs (3W) + final combination (6W) = 23W

Snapshots are file-system bound: wall-clock GB/s of the whole write / read (GPU transpose +
PCIe + file), reported beside the device-only pack/unpack kernels.
"""
import json
import os
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dev_time(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import device as D
    from paper_1604_02614_b200.mhd import _diag_ctx
    sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,4096").split(",")]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except Exception:
        peak = 6650.0
    out = []
    for n in sizes:
        g = P.ReconnectionSpec().grid(n, n)
        prm = P.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-3)
        bc = P.default_bc("reconnection")
        U = torch.from_numpy(P.reconnection_ic(g, params=prm)).cuda()
        U2 = U * (1.0 + 1e-9)
        C = n * n
        W = 64 * C
        reps = max(5, int(4e9 / W))
        rows = []

        def rec(name, us, nbytes):
            rows.append({"op": name, "us": us, "GBps": nbytes / us / 1e3,
                         "frac_of_hbm": nbytes / us / 1e3 / peak})

        # public API calls (each returns a host scalar: one sync per call) ...
        rec("div_B (API)", dev_time(lambda: P.div_B(U, g, bc), reps), 3 * 8 * C)
        rec("current_J (API)", dev_time(lambda: P.current_J(U, g, bc), reps), 6 * 8 * C)
        rec("error_norm (API)", dev_time(lambda: P.error_norm(U, U2, g), reps), 2 * W)
        rec("rk4_stable_dt (API)", dev_time(lambda: P.rk4_stable_dt(U, g, prm), reps), W)
        # ... and their kernels alone through the C ABI
        from paper_1604_02614_b200.harness import _state_ctx
        u = U.reshape(-1)
        dq = _diag_ctx(g, bc)
        hq = dq.halo(u)
        dbuf, mx = torch.empty(C, dtype=torch.float64, device="cuda"), D.zeros(1)
        Jbuf = torch.empty(3 * C, dtype=torch.float64, device="cuda")
        sums = D.zeros(8)
        sp = _state_ctx(g, None, None, prm)
        Lq, hdl = dq.ctx.lib, dq.ctx.sync_stream
        rec("div_b kernel", dev_time(lambda: Lq.emhd_div_b(hdl(), D.ptr(u), D.ptr(hq), D.ptr(dbuf), D.ptr(mx)), reps), 3 * 8 * C)
        rec("current_j kernel", dev_time(lambda: Lq.emhd_current_j(hdl(), D.ptr(u), D.ptr(hq), D.ptr(Jbuf)), reps), 6 * 8 * C)
        e_ctx = _state_ctx(g)
        rec("field_sqdiff kernel", dev_time(lambda: e_ctx.ctx.lib.emhd_field_sqdiff(e_ctx.ctx.sync_stream(), D.ptr(u), D.ptr(U2), D.ptr(sums)), reps), 2 * W)
        rec("max_signal_speed kernel", dev_time(lambda: sp.ctx.lib.emhd_max_signal_speed(sp.ctx.sync_stream(), D.ptr(u), D.ptr(mx)), reps), W)
        f = P.make_rhs(prm, g, bc)
        y = U.reshape(-1)
        h = P.rk4_stable_dt(U, g, prm)
        k = 4
        us = dev_time(lambda: P.integrate_rk4(f, y, 0.0, k * h, h), max(2, reps // 8)) / k
        rec("rk4_step", us, 23 * W)
        # device-only transposes of the snapshot path
        dc = _diag_ctx(g, P.BoundaryPolicy("periodic", "periodic"))
        cells = torch.empty_like(y)
        lib, s = dc.ctx.lib, dc.ctx.sync_stream
        rec("cells_pack", dev_time(lambda: lib.emhd_cells_pack(s(), D.ptr(y), C, D.ptr(cells)), reps), 2 * W)
        back = torch.empty_like(y)
        rec("cells_unpack", dev_time(lambda: lib.emhd_cells_unpack(s(), D.ptr(cells), C, D.ptr(back)), reps), 2 * W)
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "s.mhd25")
            P.write_snapshot(path, U, g, 0.0, prm)
            t0 = time.perf_counter()
            P.write_snapshot(path, U, g, 0.0, prm)
            tw = time.perf_counter() - t0
            P.read_snapshot(path)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            R, _, _, _ = P.read_snapshot(path)
            torch.cuda.synchronize()
            tr = time.perf_counter() - t0
            assert torch.equal(R, U), "snapshot round trip differs"
        rows.append({"op": "write_snapshot (wall, file)", "us": tw * 1e6, "GBps": W / tw / 1e9})
        rows.append({"op": "read_snapshot (wall, file)", "us": tr * 1e6, "GBps": W / tr / 1e9})
        out.append({"n": n, "W_bytes": W, "results": rows})
    print(json.dumps({"peak_GBps": peak, "state": "reconnection_ic, mu=eta=1e-4, kappa=1e-3",
                      "grids": out}))


if __name__ == "__main__":
    main()
