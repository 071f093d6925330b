"""Dump the bench workload's step matrix, a random x and the reference
y = A x (oracle order) as raw binaries for tools/spmv_variants.cu.

    python tools/spmv_dump.py [--workload cfg3] [--out /tmp/spmv]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--out", default="/tmp/spmv")
    args = ap.parse_args()
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200.integrator import BackwardEulerIntegrator, IntegratorConfig, SimState
    from paper_2306_05893_b200 import krylov

    w = bench.WORKLOADS[args.workload]
    mesh = P.generate_beam(*w["dims"], 0.1)
    mesh = mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))
    integ = BackwardEulerIntegrator(mesh, P.make_model(w["law"], mesh, P.MaterialParams(1e5, 0.3, 1000.0)),
                                    IntegratorConfig(dt=0.01, gravity=(0.0, -9.81, 0.0)))
    st = SimState.rest(mesh, device=True)
    a, _, _ = integ.assemble_system(st)
    x = np.random.default_rng(0).standard_normal(a.ncols)
    y = krylov.spmv(a, x)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    np.asarray(a.row_ptr, dtype=np.int32).tofile(out / "rp.bin")
    np.asarray(a.col_ind, dtype=np.int32).tofile(out / "ci.bin")
    np.asarray(a.values, dtype=np.float64).tofile(out / "val.bin")
    x.tofile(out / "x.bin")
    np.asarray(y, dtype=np.float64).tofile(out / "y.bin")
    print(f"dumped n={a.nrows} nnz={a.nnz} to {out}")


if __name__ == "__main__":
    main()
