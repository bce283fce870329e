#!/usr/bin/env python
"""Benchmark of the B200 EpiRK/Krylov hot path on BASELINE config 2.

Workload (BASELINE.json configs[2]): seeded smooth random 8-field
state (16 random-phase Fourier modes per primitive) on a 1024 x 1024 grid,
fp64, mu = eta = kappa = 1e-3, periodic x and y; a seeded unit start vector.
One step = ``arnoldi(FdJacobianOperator(make_rhs(...), a), v, 40)``: 40
Jv+Arnoldi iterations (each one fused normalise+Jv stencil, a multi-dot and
two update sweeps — the reference's _ArnoldiProcess.extend, krylov.py:144-168).
The config's 100 standalone Jv products are timed beside it and reported as
grid-point updates/s.  Vectors are 64 MiB and the basis 2.7 GB, far larger
than L2, so no L2 flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the grid is slab-decomposed in x across ranks (NCCL
halo exchange + all-reduces, strong scaling); timings are the max over ranks.
``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port in oracle/, the reference itself being pure Python that cannot
travel to the GPU box) on this host's cores, rank 0 only.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Jv+Arnoldi iterations/s (fp64)"
UNIT = "iterations/s"
FALLBACK_HBM = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=1024, help="grid is n x n")
    p.add_argument("--m", type=int, default=40, help="Krylov dimension")
    p.add_argument("--jv", type=int, default=100, help="standalone Jv products per step")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--quick", action="store_true", help="timed region only (for ncu)")
    p.add_argument("--no-trajectory", action="store_true", help="skip the config-1 trajectory")
    p.add_argument("--no-two-pass", action="store_true", help="skip the always-two-pass record")
    p.add_argument("--comm", default="native", choices=["native", "python"],
                   help="slab collectives: inside libemhd (C driver) or torch.distributed")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the config-3 trajectory and the config-4 4096^2 Arnoldi line")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def _reorth_eta():
    try:
        from paper_1604_02614_b200 import krylov
        return krylov.REORTH_ETA
    except Exception:
        return float("nan")


def config_dict(args, world):
    return {
        "workload": f"config2: {args.n}x{args.n} seeded Fourier state, "
                    f"arnoldi(FdJacobianOperator(make_rhs), v, {args.m}) per step "
                    f"+ {args.jv} standalone Jv products",
        "grid": [args.n, args.n], "krylov_dim": args.m, "jv_products": args.jv,
        "fields": 8, "mu": 1e-3, "eta": 1e-3, "kappa": 1e-3, "bc": "periodic/periodic",
        "decomposition": f"x-slabs x{world}", "parallelism": f"slab{world}",
        "slab_collectives": ("libemhd NCCL (C driver, halo exchange overlapped with interior rows)"
                             if getattr(args, "comm", "native") == "native" else "torch.distributed")
                            if world > 1 else None,
        "l2": "inputs larger than L2 (64 MiB vectors, 2.7 GB basis); no flush needed",
        "orthogonalisation": "classical Gram-Schmidt, second pass when ||w1|| < eta ||w|| "
                             "(selective re-orthogonalisation, eta = %.4g; 0 = always two passes; "
                             "the reference runs MGS + a full second pass)" % _reorth_eta(),
        "seed": 1604,
    }


def make_inputs(args):
    from paper_1604_02614_b200.mhd import MhdParams
    from paper_1604_02614_b200.problems import fourier_grid, fourier_state, unit_start_vector
    g = fourier_grid(args.n)
    prm = MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    U, rng = fourier_state(g, prm, seed=1604)
    v = unit_start_vector(rng, U.size)
    return g, prm, U, v


# ------------------------------------------------------------------ clocks
class Clocks:
    """SM clock and throttle-reason sampling during the timed region (B200_PROFILING.md clocks
    line): NVML every 10 ms from a thread (nvidia-smi -lms 200 as a fallback)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []          # (sm_mhz, max_mhz, set(reasons))
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def loop():
                while not self._stop.is_set():
                    try:
                        sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, mx, {k for k, b in bits.items() if r & b}))
                    except Exception:
                        pass
                    self._stop.wait(0.01)
            self._nvml = nv
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self.t.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for s_, m_, r_ in self.samples:
            sm.append(s_)
            mx = m_
            reasons |= r_
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(self.NAMES, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else "nvidia-smi"}


# ------------------------------------------------------ kernel instrumentation
# emhd_profile_read kinds (include/emhd.h EMHD_K_*), reported under the C-ABI entry names
KIND_NAMES = {0: "emhd_jv", 1: "emhd_jv_normalized", 2: "emhd_multidot", 3: "emhd_update",
              4: "emhd_multidot (second pass)", 5: "emhd_update_finish", 6: "emhd_norms",
              7: "emhd_div_scalar", 8: "gate"}


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200 import _native as N
    from paper_1604_02614_b200.mhd import local_rows
    from paper_1604_02614_b200.slab import Comm, NativeComm, make_layout

    g, prm, U, v = make_inputs(args)
    bc = P.BoundaryPolicy("periodic", "periodic")
    layout = make_layout(g.nx, g.ny, bc.x, rank, world)
    # slab ranks: collectives inside the library (C driver, stream-ordered NCCL all-reduces,
    # halo exchange overlapped with the interior rows); --comm python: torch.distributed calls
    comm = NativeComm(layout) if (world > 1 and args.comm == "native") else Comm(layout)
    f = P.make_rhs(prm, g, bc, layout=layout, comm=comm)
    a_host = local_rows(U.reshape(-1), g, layout)
    v_host = local_rows(v, g, layout)
    a_pin = torch.from_numpy(a_host).pin_memory()
    v_pin = torch.from_numpy(v_host).pin_memory()
    a = a_pin.cuda()
    vd = v_pin.cuda()
    op = P.FdJacobianOperator(f, a)
    n_local = a.numel()
    cells_global = g.nx * g.ny

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        return P.arnoldi(op, vd, args.m)

    def maxall(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        b = step()
    assert b.m == args.m and not b.breakdown, "unexpected breakdown in the bench workload"

    # ---- headline: K steps, device-timed, max over ranks
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with Clocks(local) as clk:
        e0.record()
        for _ in range(args.steps):
            b = step()
        e1.record()
        barrier()
    t_ms = maxall(e0.elapsed_time(e1))
    iters = args.m * args.steps
    value = iters / (t_ms / 1e3)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_dict(args, world), "clocks": clk.summary()}
    if args.quick:
        if rank == 0:
            print(json.dumps(out), flush=True)
        return

    # ---- 100 standalone Jv products (grid-point updates/s)
    vn = torch.zeros(2, dtype=torch.float64, device="cuda")
    op.vnorm_into(vd, vn)
    jout = torch.empty_like(a)
    vh = f.halo(vd)
    for _ in range(3):
        op.apply_device(vd, jout, vn, vh)
    barrier()
    j0, j1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    j0.record()
    for _ in range(args.jv):
        op.apply_device(vd, jout, vn, vh)
    j1.record()
    barrier()
    jv_ms = maxall(j0.elapsed_time(j1))
    jv_per_s = args.jv / (jv_ms / 1e3)
    hbm, hbm_src = peaks()
    jv_gbs = 4.0 * 8.0 * n_local * world / (jv_ms / 1e3 / args.jv) / 1e9
    out["jv"] = {"products": args.jv, "jv_per_s": jv_per_s,
                 "grid_point_updates_per_s": jv_per_s * cells_global,
                 "us_per_jv": jv_ms * 1e3 / args.jv, "alg_GBps_per_gpu": jv_gbs / world,
                 "frac_of_hbm": jv_gbs / world / hbm}

    # ---- the Arnoldi loop's stencil (fused normalise + Jv, 5W) launched back to back: the same
    # kernel as the `emhd_jv_normalized` entry of `kernels` below, without the loop's power-capped
    # clocks and without the per-launch event bracketing of the profile run (single rank only)
    if world == 1:
        from paper_1604_02614_b200 import _native as N
        L = f.ctx.lib
        wv = jout.clone()
        sc = torch.tensor([float(wv.norm()), float(wv.abs().max()), 0.0, 0.0], dtype=torch.float64,
                          device="cuda")
        vout = torch.empty_like(a)
        nout = torch.empty_like(a)

        def jvn():
            N.check(L.emhd_jv_normalized(f.ctx.sync_stream(), a.data_ptr(), None, op.f_a.data_ptr(),
                                         wv.data_ptr(), None, sc.data_ptr(), vout.data_ptr(), 0, 1.0, 0,
                                         N.ptr_array([]), N.int_array([]), nout.data_ptr()), "jv_normalized")
        for _ in range(3):
            jvn()
        torch.cuda.synchronize()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0.record()
        for _ in range(args.jv):
            jvn()
        n1.record()
        torch.cuda.synchronize()
        jvn_us = n0.elapsed_time(n1) * 1e3 / args.jv
        jvn_gbs = 5.0 * 8.0 * n_local / (jvn_us * 1e-6) / 1e9
        out["jv_normalized_back_to_back"] = {"launches": args.jv, "us": jvn_us, "alg_GBps": jvn_gbs,
                                             "frac_of_hbm": jvn_gbs / hbm, "ran": f.ctx.last_stencil()}
        del wv, vout, nout

    # ---- the same K steps with the second Gram-Schmidt pass in every iteration (the
    # reference's order of work: selective re-orthogonalisation off, EMHD_REORTH_ETA=0)
    if not args.no_two_pass:
        from paper_1604_02614_b200 import krylov as K
        saved = K.REORTH_ETA
        K.REORTH_ETA = 0.0
        try:
            for _ in range(2):
                step()
            barrier()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(args.steps):
                b2 = step()
            t1.record()
            barrier()
        finally:
            K.REORTH_ETA = saved
        assert b2.second_pass is None
        tp_ms = maxall(t0.elapsed_time(t1))
        W2 = 8.0 * n_local
        canon2 = sum((3 * j + 11) * W2 for j in range(args.m))
        hbm2, _ = peaks()
        out["two_pass"] = {
            "value": iters / (tp_ms / 1e3), "unit": UNIT, "ms_per_step": tp_ms / args.steps,
            "steps": args.steps,
            "iteration_roofline": {"alg_GB_per_step_per_gpu": canon2 / 1e9,
                                   "achieved_GBps_per_gpu": canon2 / (tp_ms / args.steps / 1e3) / 1e9,
                                   "frac": canon2 / (tp_ms / args.steps / 1e3) / 1e9 / hbm2,
                                   "rule": "(3j+11)W per iteration (SURVEY 8d, both passes)"},
            "orthogonalisation": "classical Gram-Schmidt twice in every iteration (CGS2)"}

    # ---- profiled pass (same K steps, same fast path): the library brackets every launch of
    # the Arnoldi iterations with CUDA events on the launching stream (emhd_profile); a launch
    # that a device gate turned into a no-op (skipped second pass, cancelled look-ahead)
    # counts zero algorithmic bytes
    import ctypes
    lib = N.lib()
    hctx = op.ctx.h
    N.check(lib.emhd_profile(hctx, 1), "profile")
    barrier()
    passes = []
    records = []
    cap = 64 * args.m + 64
    kinds = (ctypes.c_int * cap)()
    pms = (ctypes.c_double * cap)()
    pby = (ctypes.c_double * cap)()
    for _ in range(args.steps):
        bb = step()
        nrec = lib.emhd_profile_read(hctx, cap, kinds, pms, pby)
        if nrec < 0:
            raise RuntimeError("emhd_profile_read failed")
        records += [(KIND_NAMES.get(kinds[i], str(kinds[i])), pms[i], pby[i]) for i in range(nrec)]
        passes.append(None if bb.second_pass is None else bb.second_pass.cpu().numpy())
    barrier()
    N.check(lib.emhd_profile(hctx, 0), "profile")
    table = {}
    for name, ms_, by_ in records:
        a_ = table.setdefault(name, {"launches": 0, "ms": 0.0, "bytes": 0.0})
        a_["launches"] += 1
        a_["ms"] += ms_
        a_["bytes"] += by_
    launches_per_step = sum(1 for r in records if r[0] != "gate") / args.steps
    kern = []
    for name, a_ in sorted(table.items(), key=lambda kv: -kv[1]["ms"]):
        avg_us = a_["ms"] * 1e3 / a_["launches"]
        gbs = a_["bytes"] / (a_["ms"] / 1e3) / 1e9 if a_["ms"] > 0 else 0.0
        kern.append({"kernel": name, "launches": a_["launches"], "avg_us": avg_us,
                     "share_of_step": a_["ms"] / args.steps / (t_ms / args.steps),
                     "alg_GBps": gbs, "frac": gbs / hbm})
    top = kern[0]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(top["kernel"])
    out["roofline"] = {"bound": "hbm", "achieved": top["alg_GBps"], "peak": hbm, "unit": "GB/s",
                       "frac": top["alg_GBps"] / hbm, "traffic": traffic,
                       "kernel": top["kernel"], "peak_source": hbm_src,
                       "traffic_of": "ncu --set full capture of ONE launch of this kernel (profiles/*_ncu_full.json "
                                     "via profiles/summarize.py): compare it with that launch's own algorithmic "
                                     "bytes, (nvec+2)*L*8 with nvec = round(traffic / (L*8)) - 2; `achieved` "
                                     "averages the launches j = 0..m-1 of the timed steps",
                       "alg_bytes_rule": "multidot (nvec+1)*L*8, update (nvec+2)*L*8, "
                                         "jv_normalized 5W, jv 4W, rhs 2W (SURVEY 8d)"}
    out["kernels"] = kern
    out["gpu_launches"] = int(round(launches_per_step * args.steps))
    # whole-iteration roofline.  SURVEY 8d's canonical (3j + 11) W per iteration assumes both
    # Gram-Schmidt passes; with selective re-orthogonalisation an iteration whose second pass
    # is skipped needs (2j + 8) W (fused Jv + pass-1 dots (j + 5) W, update + re-projection
    # (j + 3) W), one that runs it (3j + 11) W.
    W = 8.0 * n_local
    sp = passes[-1] if passes and passes[-1] is not None else [1.0] * args.m
    alg_iter = sum(((3 * j + 11) if sp[j] else (2 * j + 8)) * W for j in range(args.m))
    canon = sum((3 * j + 11) * W for j in range(args.m))
    out["iteration_roofline"] = {"alg_GB_per_step_per_gpu": alg_iter / 1e9,
                                 "achieved_GBps_per_gpu": alg_iter / (t_ms / args.steps / 1e3) / 1e9,
                                 "frac": alg_iter / (t_ms / args.steps / 1e3) / 1e9 / hbm,
                                 "second_pass_iterations": int(sum(1 for x in sp if x)),
                                 "two_pass_canonical_GB_per_step": canon / 1e9,
                                 "rule": "(3j+11)W with the second Gram-Schmidt pass, (2j+8)W without "
                                         "(selective re-orthogonalisation, eta = %g)" % _reorth_eta()}

    # ---- end to end through the public API with host buffers
    if not args.no_e2e:
        hb = torch.empty((args.m + 1) * args.m, dtype=torch.float64).pin_memory()

        def e2e_step():
            a_d = a_pin.to("cuda", non_blocking=True)
            v_d = v_pin.to("cuda", non_blocking=True)
            jop = P.FdJacobianOperator(f, a_d)
            bb = P.arnoldi(jop, v_d, args.m)
            hb.copy_(bb.H.reshape(-1), non_blocking=True)
            return bb
        for _ in range(2):
            e2e_step()
        barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record()
        for _ in range(args.steps):
            e2e_step()
        q1.record()
        barrier()
        e2e_ms = maxall(q0.elapsed_time(q1))
        out["e2e"] = {"value": iters / (e2e_ms / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": int(2 * 8 * n_local),
                      "d2h_bytes_per_step": int(8 * (args.m + 1) * args.m),
                      "ms_per_step": e2e_ms / args.steps,
                      "path": "numpy-pinned host a, v -> FdJacobianOperator(make_rhs) -> arnoldi -> H"}

    # ---- secondary: BASELINE configs 0 (reconnection 64^2, EpiRK4 x 20) and 1 (KH shear 256^2,
    # EpiRK5P1 tol 1e-6 to t=2) trajectories
    if rank == 0 and world == 1 and not args.no_trajectory:
        out["trajectory_config0"] = trajectory_config0()
        out["trajectory_config1"] = trajectory_config1()

    # ---- secondary: BASELINE configs 4 (4096^2 Arnoldi, m = 40) and 3 (2048^2 EpiRK5P1, 50 steps)
    if rank == 0 and world == 1 and not args.no_secondary:
        out["config4_arnoldi"] = config4_arnoldi(args)
        out["trajectory_config3"] = trajectory_config3()

    # ---- CPU baseline (rank 0, N = 1): the oracle port, bounded j-sampled extends
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, g, prm, U, v, b)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def trajectory_config0(repeat=3):
    """BASELINE config 0 (reconnection 64^2, EpiRK4 dt = 0.1 x 20 steps, Krylov tol 1e-10)
    through integrate_fixed: the latency-bound, host-sync-bound configuration (best of 3)."""
    import torch
    import paper_1604_02614_b200 as P
    g = P.ReconnectionSpec().grid(64, 64)
    prm = P.MhdParams(mu=1e-3, eta=1e-3, kappa=1e-3)
    f = P.make_rhs(prm, g, P.default_bc("reconnection"))
    y0 = torch.from_numpy(P.reconnection_ic(g, params=prm).reshape(-1)).cuda()
    P.integrate_fixed("epirk4", f, y0, 0.0, 0.2, 0.1, tol_krylov=1e-10)      # warm-up
    best, st = None, None
    for _ in range(repeat):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y, st = P.integrate_fixed("epirk4", f, y0, 0.0, 2.0, 0.1, tol_krylov=1e-10)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        best = sec if best is None else min(best, sec)
    keys = ["steps_accepted", "projections", "rhs_evals", "operator_applies", "max_basis_size"]
    return {"workload": "config0: reconnection 64x64, EpiRK4 dt 0.1 x 20, Krylov tol 1e-10",
            "seconds": best, "iterations_per_s": st.operator_applies / best,
            "stats": {k: getattr(st, k) for k in keys}}


def trajectory_config1():
    """Whole EpiRK5P1 run of BASELINE config 1 through the public API (device-timed wall)."""
    import torch
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200.problems import kh_shear_grid, kh_shear_ic
    g = kh_shear_grid(256)
    prm = P.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-4)
    f = P.make_rhs(prm, g, P.BoundaryPolicy("periodic", "reflect"))
    y0 = torch.from_numpy(kh_shear_ic(g, prm).reshape(-1)).cuda()
    P.integrate_adaptive(f, y0, 0.0, 0.05, P.StepController(tol=1e-6))      # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y, st = P.integrate_adaptive(f, y0, 0.0, 2.0, P.StepController(tol=1e-6))
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    keys = ["steps_accepted", "steps_rejected", "projections", "rhs_evals", "operator_applies",
            "substeps", "max_basis_size"]
    return {"workload": "config1: KH shear 256x256, mu=eta=kappa=1e-4, EpiRK5P1 tol 1e-6, t 0->2",
            "seconds": sec, "iterations_per_s": st.operator_applies / sec,
            "cell_steps_per_s": g.nx * g.ny * st.steps_accepted / sec,
            "stats": {k: getattr(st, k) for k in keys}}


def config4_arnoldi(args, n=4096, steps=3):
    """BASELINE config 4's grid (Harris sheet 4096^2, eta = mu = 1e-4, kappa = 1e-3): the
    config-2 step (arnoldi(FdJacobianOperator(make_rhs), v, 40)) on 1 GiB vectors, device-timed,
    with its whole-iteration roofline (a 41 GiB basis: one B200)."""
    import torch
    import paper_1604_02614_b200 as P
    from paper_1604_02614_b200.problems import unit_start_vector
    g = P.ReconnectionSpec().grid(n, n)
    prm = P.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-3)
    f = P.make_rhs(prm, g, P.default_bc("reconnection"))
    a = torch.from_numpy(P.reconnection_ic(g, params=prm).reshape(-1)).cuda()
    v = torch.from_numpy(unit_start_vector(np.random.default_rng(1604), a.numel())).cuda()
    op = P.FdJacobianOperator(f, a)
    b = P.arnoldi(op, v, args.m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        b = P.arnoldi(op, v, args.m)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    W = 8.0 * a.numel()
    sp = b.second_pass.cpu().numpy() if b.second_pass is not None else [1.0] * args.m
    alg = sum(((3 * j + 11) if sp[j] else (2 * j + 8)) * W for j in range(args.m))
    hbm, _ = peaks()
    res = {"workload": f"config4 grid: Harris {n}x{n}, mu=eta=1e-4, kappa=1e-3, periodic/reflect; "
                       f"arnoldi(FdJacobianOperator(make_rhs), v, {args.m}) per step",
           "steps": steps, "ms_per_step": ms, "iterations_per_s": args.m / (ms / 1e3),
           "iteration_roofline": {"alg_GB_per_step": alg / 1e9, "frac": alg / (ms / 1e3) / 1e9 / hbm,
                                  "second_pass_iterations": int(sum(1 for x in sp if x)),
                                  "rule": "(3j+11)W with the second Gram-Schmidt pass, (2j+8)W without"},
           "breakdown": bool(b.breakdown), "m": int(b.m)}
    del b, op, a, v, f
    torch.cuda.empty_cache()
    return res


def trajectory_config3(n=2048, steps=50):
    """BASELINE config 3: Harris sheet 2048^2, mu = eta = 1e-4, kappa = 1e-3, EpiRK5P1 with
    rtol = atol = 1e-6 for 50 accepted steps (max_steps driver extension; h0 = 0.05)."""
    import torch
    import paper_1604_02614_b200 as P
    g = P.ReconnectionSpec().grid(n, n)
    prm = P.MhdParams(mu=1e-4, eta=1e-4, kappa=1e-3)
    f = P.make_rhs(prm, g, P.default_bc("reconnection"))
    y0 = torch.from_numpy(P.reconnection_ic(g, params=prm).reshape(-1)).cuda()
    ctl = P.StepController(tol=1e-6, h_init=0.05)
    P.integrate_adaptive(f, y0, 0.0, 1e3, ctl, max_steps=2,
                         recoverable=(P.AdmissibilityError,))          # warm-up (allocations)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y, st = P.integrate_adaptive(f, y0, 0.0, 1e3, P.StepController(tol=1e-6, h_init=0.05),
                                 max_steps=steps, recoverable=(P.AdmissibilityError,))
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    keys = ["steps_accepted", "steps_rejected", "projections", "rhs_evals", "operator_applies",
            "substeps", "max_basis_size"]
    res = {"workload": f"config3: Harris {n}x{n}, mu=eta=1e-4, kappa=1e-3, EpiRK5P1 tol 1e-6, "
                       f"{steps} accepted steps (h0 0.05)",
           "seconds": sec, "iterations_per_s": st.operator_applies / sec,
           "cell_steps_per_s": g.nx * g.ny * st.steps_accepted / sec,
           "stats": {k: getattr(st, k) for k in keys}}
    del y, y0, f
    torch.cuda.empty_cache()
    return res


def sample_js(m, k):
    """k iterations stratified over j in [0, m): the midpoint of each of k equal bins."""
    return [min(m - 1, int((i + 0.5) * m / k)) for i in range(k)]


def timed_extends(proc, js, clock=time.perf_counter):
    """Time the reference algorithm's extend at each j of js on a factorisation that already
    holds at least max(js) + 1 basis vectors: before each sample the process is rewound to
    m = j (column j of H cleared; extend recomputes it and overwrites V[:, j + 1])."""
    ts = []
    for j in js:
        proc.m = j
        proc.broke = False
        proc.H[:, j] = 0.0
        t0 = clock()
        proc.grow()
        ts.append(clock() - t0)
    return ts


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        return int(info[0]["num_threads"]) if info else 1
    except Exception:
        return 1


def cpu_baseline(args, g, prm, U, v, basis, samples=5):
    """The oracle's Arnoldi extend (the reference's MGS + full second pass, krylov.py:144-168, on
    the reference's column-strided n x (m+1) basis) timed at `samples` iterations stratified
    over j in [0, m).  The factorisation it extends is the device's (copied into the oracle's
    layout) so the sample needs no 160 s CPU build; the cost of extend does not depend on
    the values."""
    from oracle import jvp, krylov_cpu, stencil
    bc = type("BC", (), {"x": "periodic", "y": "periodic"})()
    f = stencil.rhs_closure(prm, g, bc)
    a = U.reshape(-1)
    op = jvp.FdJv(f, a)
    proc = krylov_cpu.Arnoldi(op, v, args.m)
    Vd = basis.V.T.contiguous().cpu().numpy()          # (m + 1, n) rows of the device basis
    proc.V[:, :] = Vd.T
    del Vd
    proc.H[:, :] = basis.H.cpu().numpy()
    proc.m = args.m
    js = sample_js(args.m, samples)
    ts = timed_extends(proc, js)
    per = sum(ts) / len(ts)
    threads = blas_threads()
    return {"value": 1.0 / per, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle (numpy restatement of the reference's _ArnoldiProcess.extend: MGS + "
                      f"full re-orthogonalisation pass, FdJacobianOperator, mhd.rhs) on the full "
                      f"{args.n}^2 config-2 state with the reference's n x {args.m + 1} "
                      f"column-strided basis; {samples} iterations timed at j = {js} "
                      f"(stratified over [0, {args.m})) on the device's m = {args.m} "
                      f"factorisation copied to the host; value = 1 / mean seconds per "
                      f"iteration; OpenBLAS threads {threads} (dots), NumPy elementwise 1 thread",
            "j_sampled": js, "measured_iter_s": ts}


# ----------------------------------------------------------- reference arm
def run_reference(args):
    """The reference algorithm's CPU implementation (the oracle port; the reference is pure
    Python and cannot travel to the GPU box) on config 2's workload: the m = 40 factorisation
    (cap 40, V n x 41 column-strided, as the reference's arnoldi(op, v, 40) allocates) is built
    once in warm-up; every step then re-runs extend at one j of a stratified sample of
    [0, 40) on that factorisation (rewound to m = j), so the timed work is the printed config's
    iteration mix, not its cheapest iterations."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import jvp, krylov_cpu, stencil
    g, prm, U, v = make_inputs(args)
    bc = type("BC", (), {"x": "periodic", "y": "periodic"})()
    f = stencil.rhs_closure(prm, g, bc)
    a = U.reshape(-1)
    op = jvp.FdJv(f, a)
    tb = time.perf_counter()
    proc = krylov_cpu.Arnoldi(op, v, args.m)
    build = []
    while proc.m < args.m:
        t0 = time.perf_counter()
        if not proc.grow():
            break
        build.append(time.perf_counter() - t0)
    build_s = time.perf_counter() - tb
    assert proc.m == args.m, "unexpected breakdown in the reference build"
    timed_extends(proc, sample_js(args.m, max(args.warmup, 1)))        # warm-up samples
    js = sample_js(args.m, args.steps)
    ts = timed_extends(proc, js)
    T = sum(ts)
    value = len(ts) / T
    threads = blas_threads()
    cfg = config_dict(args, world)
    cfg["orthogonalisation"] = ("modified Gram-Schmidt + one full re-orthogonalisation pass "
                                "(the reference's _ArnoldiProcess.extend, krylov.py:144-168)")
    cfg["basis_layout"] = f"numpy n x {args.m + 1} C-order (column-strided basis vectors, krylov.py:137)"
    cfg["m_sampled"] = args.m
    cfg["j_sampled"] = js
    sample = (f"oracle port (numpy restatement of the reference's arnoldi/_ArnoldiProcess.extend + "
              f"FdJacobianOperator + mhd.rhs; the reference is pure Python) on the full "
              f"{args.n}^2 config-2 state: the m={args.m} factorisation built once in warm-up "
              f"({build_s:.1f} s, also the full-run reference time), then one extend per step at "
              f"j = {js}; OpenBLAS threads {threads} (dots), NumPy elementwise 1 thread")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": T / len(ts) * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": cfg, "impl": "reference",
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                            "sample": sample},
           "full_build": {"seconds": build_s, "iterations_per_s": len(build) / build_s,
                          "per_iteration_s": build},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
