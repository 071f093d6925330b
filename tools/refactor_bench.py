"""Device LDL^T refactorisation timing (csrc/refactor.cu) on a bench workload.

    python tools/refactor_bench.py [--workload cfg2] [--host]

Builds the scenario matrix of step 3, plans the refactorisation once, then
times tsb_refactor_run with CUDA events (median of 5 after 2 warm-ups) and
reports the dense fp64 rate; --host also times the host multifrontal
factorisation + pack of the same matrix and checks the device image
against it.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--host", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import _ldlt_pack as K, krylov, ndprecond as ND, refactor as R
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState

    w = bench.WORKLOADS[args.workload]
    mesh = P.generate_beam(*w["dims"], 0.1)
    mesh = mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))
    integ = BackwardEulerIntegrator(mesh, P.make_model(w["law"], mesh, P.MaterialParams(1e5, 0.3, 1000.0)),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    cfg = krylov.SolverConfig(1e-9, 8000)
    st = SimState.rest(mesh, device=True)
    for _ in range(3):
        res = integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    a = res.matrix
    t0 = time.perf_counter()
    plan = ND.expand_plan(ND.nested_dissection(P.vertex_adjacency(mesh), bench.LEAF))
    t_nd = time.perf_counter() - t0
    t0 = time.perf_counter()
    rf = R.DeviceRefactor(a, plan)
    t_plan = time.perf_counter() - t0
    out = {"workload": args.workload, "n": a.nrows, "fronts": len(rf.rplan.fronts),
           "heights": int(rf.rplan.heights.max()) + 1, "ops": len(rf.rplan.prog),
           "workspace_gb": rf.workspace_bytes / 1e9, "gflop": rf.rplan.flops / 1e9,
           "t_nd_s": t_nd, "t_plan_s": t_plan}
    img = rf.images[0]
    ts = []
    for i in range(2 + args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rf.enqueue(a, img)
        e1.record()
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    assert rf.failed_block() < 0
    ms = float(np.median(ts))
    out.update(refactor_ms=ms, tflops=rf.rplan.flops / ms / 1e9, samples_ms=ts)
    # PCG with the fresh factor on the matrix it was computed from
    f = R.make_factors(rf, img, 3)
    a2, b2, _ = integ.assemble_system(st)
    x, rep = krylov.pcg(a, b2, f, cfg)
    out.update(pcg_iterations_fresh=int(rep.iterations))
    if args.host:
        t0 = time.perf_counter()
        hf = ND.ldlt_factor(a, plan)
        t1 = time.perf_counter()
        H = K.pack(hf)
        t2 = time.perf_counter()
        g = img.t["g"].cpu().numpy()
        rel = float(np.abs(g - H["g"]).max() / np.abs(H["g"]).max())
        out.update(host_factor_s=t1 - t0, host_pack_s=t2 - t1, rel_vs_host_pack=rel)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
