"""Pattern build time: host topology_pattern vs the device build (csrc/pattern.cu).

    python tools/pattern_bench.py [--workload cfg3]
"""

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
    ap.add_argument("--workload", default="cfg3")
    args = ap.parse_args()
    import torch
    import paper_2306_05893_b200 as P
    from paper_2306_05893_b200 import _plan

    w = bench.WORKLOADS[args.workload]
    mesh = P.generate_beam(*w["dims"], 0.1)
    mesh = mesh.with_fixed_nodes(np.flatnonzero(mesh.nodes[:, 2] == 0.0))
    t0 = time.perf_counter()
    h = _plan.topology_pattern(mesh)
    t_host = time.perf_counter() - t0
    _plan.device_topology_pattern(mesh)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        d = _plan.device_topology_pattern(mesh, keep_device=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    same = all(np.array_equal(np.asarray(h[k]), np.asarray(d[k])) for k in
               ("row_ptr", "col_ind", "fixed_diag_slots", "blk", "blk_list", "node_ptr", "node_list"))
    print(json.dumps({"workload": args.workload, "nnz": int(len(h["col_ind"])), "host_s": t_host,
                      "device_s_incl_download": float(np.median(ts)), "identical": same}))


if __name__ == "__main__":
    main()
