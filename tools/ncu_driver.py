"""Minimal driver for ncu captures of the step's kernels on one workload:
builds the bench workload once, then runs --reps of each: the fused
assembly (elem_kernel + gather_kernel), the isolated SpMV, the LDL^T apply
(lower_sweep + upper_sweep) and one Jacobi and one LDL^T PCG solve
(pcg_persistent).  Not a timing tool -- numbers printed under ncu are not
bench values.

    ncu ... python tools/ncu_driver.py [--workload cfg3] [--reps 2]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2306_05893_b200 import _lib, krylov

    W = bench.build_workload(args.workload)
    integ, st = W["integ"], W["state"]
    x, v, fe = (integ._flat_dev(a) for a in (st.positions, st.velocities, st.f_ext))
    a, b, _ = integ.assemble_system(st)
    f = W["factors"]
    dev = f.device()
    r = torch.randn(f.plan.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    y = torch.empty_like(r)
    d_rp, d_ci = a.device_pattern()
    lib = _lib.load()
    for _ in range(args.reps):
        integ._assemble_device(x, v, fe)
        lib.tsb_spmv(a.nrows, _lib.ptr(d_rp), _lib.ptr(d_ci), _lib.ptr(a.device_values()), _lib.ptr(r),
                     _lib.ptr(y), _lib.stream_ptr())
        dev.run("apply", r, z)
        W["solvers"]["jacobi"](a, b)[1].iterations
        W["solvers"]["ldlt"](a, b)[1].iterations
    torch.cuda.synchronize()
    print("ncu driver done")


if __name__ == "__main__":
    main()
