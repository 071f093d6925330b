"""Isolated SpMV timing (tsb_spmv, CUDA events, L2 flushed) on the bench
workload's matrix, plus a bit-exactness check against the reference order.

    TSB_SPMV_VARIANT=k python tools/spmv_bench.py [--workload cfg3]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    args = ap.parse_args()
    import torch
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import krylov
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState
    from oracle import tetsim_oracle as O

    w = bench.WORKLOADS[args.workload]
    mesh = P.generate_beam(*w["dims"], 0.1)
    mesh = mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))
    integ = BackwardEulerIntegrator(mesh, P.make_model(w["law"], mesh, P.MaterialParams(1e5, 0.3, 1000.0)),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    st = SimState.rest(mesh, device=True)
    cfg = krylov.SolverConfig(1e-9, 8000)
    integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    W = {"integ": integ, "state": st}
    r = bench.time_spmv(W, 30, bench.L2Flush())
    a, _, _ = integ.assemble_system(st)
    x = np.random.default_rng(0).standard_normal(a.ncols)
    exact = bool(np.array_equal(krylov.spmv(a, x), O.spmv(a.row_ptr, a.col_ind, a.values, x)))
    print(json.dumps({"workload": args.workload, "variant": os.environ.get("TSB_SPMV_VARIANT", "0"),
                      "spmv_us": r["ms"] * 1e3, "gbs": r["gbs"], "bit_exact": exact}))


if __name__ == "__main__":
    main()
