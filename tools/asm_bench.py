"""Assembly timing (fused device assembly of one step), CUDA events, L2 flushed.

    python tools/asm_bench.py [--workload cfg3] [--law corotational]
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--law", default=None)
    args = ap.parse_args()
    import torch
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import krylov
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState

    w = bench.WORKLOADS[args.workload]
    mesh = P.generate_beam(*w["dims"], 0.1)
    mesh = mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))
    law = args.law or w["law"]
    integ = BackwardEulerIntegrator(mesh, P.make_model(law, mesh, P.MaterialParams(1e5, 0.3, 1000.0)),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    st = SimState.rest(mesh, device=True)
    cfg = krylov.SolverConfig(1e-9, 8000)
    for _ in range(3):
        integ.step(st, lambda a, b: krylov.pcg(a, b, krylov.jacobi_precond(a), cfg))
    flush = bench.L2Flush()
    x, v, fe = (integ._flat_dev(a) for a in (st.positions, st.velocities, st.f_ext))
    for _ in range(3):
        integ._assemble_device(x, v, fe)
    ts = []
    for _ in range(20):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        integ._assemble_device(x, v, fe)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    nnz = len(integ.assembler.pattern["col_ind"])
    m, N = mesh.element_count, mesh.node_count
    byts = 8 * nnz + m * (16 + 104 + 64) + N * 144
    print(json.dumps({"workload": args.workload, "law": law, "assembly_ms": ms, "algorithmic_MB": byts / 1e6,
                      "gbs": byts / (ms * 1e-3) / 1e9}))


if __name__ == "__main__":
    main()
