"""Contact stage timing on a dropped beam (device path).

    python tools/contact_bench.py [--dims 10 10 100] [--steps 6]

A free beam falls on the plane z = -0.001 (bottom face contacts after a few
steps).  Per contact step: the whole pipeline step (free motion + contact
resolution + correction) with (a) the factor path (W = Y^T D^-1 Y from m
lower sweeps, one upper sweep) and (b) the reference's column path
(apply_inverse = factors.apply per column, m full applies), both with LDL^T
factors of the previous step's matrix computed on the device.
"""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[10, 10, 100])
    ap.add_argument("--steps", type=int, default=6)
    args = ap.parse_args()
    import torch
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import contact as CT, krylov, ndprecond as ND
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState

    mesh = P.generate_beam(*args.dims, 0.1)
    params = P.MaterialParams(1e5, 0.3, 1000.0)
    plan = ND.expand_plan(ND.nested_dissection(P.vertex_adjacency(mesh), 64))
    cfg = krylov.SolverConfig(1e-9, 8000)
    solve = lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg)  # noqa: E731
    out = {"dims": args.dims, "n": mesh.ndof}
    for mode in ("factors", "columns"):
        integ = BackwardEulerIntegrator(mesh, P.make_model("corotational", mesh, params), IntegratorConfig(dt=0.01))
        pipe = CT.PlaneContactPipeline(integ, -0.001)
        st = SimState.rest(mesh, device=True)
        rf = None
        f = None
        rows = []
        for k in range(40):
            ai = None if f is None else (f if mode == "factors" else (lambda rhs, f=f: f.apply(rhs)))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            info = pipe.step(st, solve, ai)
            e1.record()
            e1.synchronize()
            wall = (time.perf_counter() - t0) * 1e3
            if info.ncontacts and f is not None:
                rows.append({"step": k, "contacts": info.ncontacts, "ms": e0.elapsed_time(e1), "wall_ms": wall,
                             "residual": info.complementarity_residual, "maxpen": info.max_penetration})
                if len(rows) >= args.steps:
                    break
            if rf is None:
                from paper_2306_05893_b200.refactor import DeviceRefactor
                rf = DeviceRefactor(info.result.matrix, plan, buffers=2)
            f = rf.factor(info.result.matrix, source_step=k)
        out[mode] = rows
    print(json.dumps(out))


if __name__ == "__main__":
    main()
