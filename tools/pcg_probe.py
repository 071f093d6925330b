"""Per-iteration cost of the device PCG (graph WHILE loop) vs its parts.

    python tools/pcg_probe.py [--workload cfg2]

Times solves capped at k iterations (slope = per-iteration cost, intercept =
per-solve setup), a warm SpMV and the LDL^T apply on the bench workload.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def timed(fn, reps=20):
    import torch

    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    args = ap.parse_args()
    import torch
    from paper_2306_05893_b200 import _lib, krylov

    W = bench.build_workload(args.workload)
    a, b, _ = W["integ"].assemble_system(W["state"])
    x = torch.empty(a.ncols, dtype=torch.float64, device="cuda")
    out = {}
    for kind, name, ld in ((_lib.PRECOND_JACOBI, "jacobi", None), (_lib.PRECOND_IDENTITY, "cg", None),
                           (_lib.PRECOND_LDLT, "ldlt", W["factors"].device())):
        pts = []
        for k in (1, 2, 4, 8, 16):
            us = timed(lambda: krylov.solve_device(a, b, x, kind, ld, 1e-30, k, sync=False))
            pts.append((k, us))
        ks = np.array([p[0] for p in pts], dtype=float)
        us = np.array([p[1] for p in pts])
        slope, icpt = np.polyfit(ks, us, 1)
        krylov.solve_device(a, b, x, kind, ld, 1e-30, 16, sync=True)
        ph = np.zeros(6, dtype=np.int64)
        _lib.load().tsb_pcg_phase_times(krylov._handle(a.nrows).h, ph.ctypes.data, _lib.stream_ptr())
        names = ["spmv", "barrier_alpha", "update", "barrier_beta", "precond", "loop"]
        out[name] = {"us_per_iteration": float(slope), "us_per_solve_setup": float(icpt),
                     "phase_us_per_iteration": {k: round(float(v) / 16e3, 2) for k, v in zip(names, ph)},
                     "points": [[int(k), round(float(u), 1)] for k, u in pts]}
    xv = torch.randn(a.ncols, dtype=torch.float64, device="cuda")
    out["spmv_warm_us"] = timed(lambda: krylov.spmv(a, xv))
    dev = W["factors"].device()
    r = torch.randn(a.ncols, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    out["ldlt_apply_warm_us"] = timed(lambda: dev.run("apply", r, z))
    out["assemble_us"] = timed(lambda: W["integ"]._assemble_device(
        W["integ"]._flat_dev(W["state"].positions), W["integ"]._flat_dev(W["state"].velocities),
        W["integ"]._flat_dev(W["state"].f_ext)))
    out["step_jacobi_us"] = timed(lambda: W["integ"].compute_step(W["state"], W["solvers"]["jacobi"]), 10)
    out["step_ldlt_us"] = timed(lambda: W["integ"].compute_step(W["state"], W["solvers"]["ldlt"]), 10)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
