"""LDL^T apply cost in sequence: standalone applies back to back and after an
L2 flush, and PCG solves capped at k iterations (flushed before each), to see
whether the per-apply cost depends on what ran just before.

    python tools/apply_seq.py [--workload cfg3]
"""
import argparse
import json
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
    from paper_2306_05893_b200 import _lib, krylov

    W = bench.build_workload(args.workload)
    f = W["factors"]
    dev = f.device()
    r = torch.randn(f.plan.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    flush = bench.L2Flush()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    out = {}
    for mode in ("back_to_back", "flushed"):
        ts = []
        for i in range(16):
            if mode == "flushed":
                flush()
            a, b = ev(), ev()
            a.record()
            dev.run("apply", r, z)
            b.record()
            b.synchronize()
            ts.append(round(a.elapsed_time(b) * 1e3, 1))
        out[mode] = ts
    # a long burst: 16 applies in one timed region
    a, b = ev(), ev()
    flush()
    a.record()
    for _ in range(16):
        dev.run("apply", r, z)
    b.record()
    b.synchronize()
    out["burst16_us_each"] = a.elapsed_time(b) * 1e3 / 16
    A, B, _ = W["integ"].assemble_system(W["state"])
    x = torch.empty(A.ncols, dtype=torch.float64, device="cuda")
    h = krylov._handle(A.nrows)
    lib = _lib.load()
    pts = []
    for k in (1, 2, 3, 4, 6, 8, 12, 16, 24):
        ts, pre = [], []
        for _ in range(5):
            flush()
            a, b = ev(), ev()
            a.record()
            krylov.solve_device(A, B, x, _lib.PRECOND_LDLT, dev, 1e-30, k, sync=False)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
            ph = np.zeros(6, dtype=np.int64)
            lib.tsb_pcg_phase_times(h.h, ph.ctypes.data, _lib.stream_ptr())
            pre.append(ph[4] / 1e3)
        pts.append({"k": k, "solve_us": round(float(np.median(ts)), 1),
                    "loop_precond_us_per_it": round(float(np.median(pre)) / max(k - 1, 1), 1)})
    out["pcg"] = pts
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
