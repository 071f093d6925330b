"""Run the sweep building-block micro-benchmarks (tools/ubench.cu) on cuda:0.

    python tools/ubench.py [--build-only]
"""

from __future__ import annotations

import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
SO = ROOT / "tools" / "libubench.so"


def build():
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-I", str(ROOT / "include"),
           "-I", str(ROOT / "paper_2306_05893_b200" / "csrc"), str(ROOT / "tools" / "ubench.cu"),
           "-o", str(SO), "-lcudart_static"]
    subprocess.run(cmd, check=True)


def main():
    build()
    if "--build-only" in sys.argv:
        return
    import torch

    sys.path.insert(0, str(ROOT))
    from paper_2306_05893_b200._ldlt_pack import packed_inverse

    lib = C.CDLL(str(SO))
    vp = C.c_void_p
    res = {}
    # panel triangle solve, w = 128 (8 tiles) and 64
    for w in (128, 64, 32):
        rng = np.random.default_rng(0)
        L = np.tril(rng.standard_normal((w, w)) * 0.01, -1) + np.eye(w)
        blob = list(packed_inverse(L))
        blob = torch.from_numpy(np.concatenate(blob)).cuda()
        cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
        out = torch.zeros(128, dtype=torch.float64, device="cuda")
        lib.ub_forward(vp(blob.data_ptr()), C.c_int64(blob.numel()), w, 50, vp(cyc.data_ptr()), vp(out.data_ptr()))
        c = cyc.cpu().numpy()
        res[f"panel_w{w}_cycles"] = {"forward": int(c[0]), "backward": int(c[1])}
    # streaming: TMA bulk vs plain loads, 1 CTA and 148/296 CTAs, 32/96 KB per copy
    buf = torch.zeros(2 * 1024 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # 2 GB, > L2
    ns = torch.zeros(512, dtype=torch.int64, device="cuda")
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    for kb in (32, 96):
        byts = kb * 1024
        stride = byts // 8
        for grid in (1, 148, 296):
            iters = max(1, min(200, (buf.numel() // stride) // grid))
            lib.ub_tma(vp(buf.data_ptr()), C.c_int64(stride), C.c_uint32(byts), iters, grid, vp(ns.data_ptr()))
            t = ns[:grid].cpu().numpy().max() / 1e9
            res[f"tma_{kb}KB_grid{grid}"] = {"GBps_total": byts * iters * grid / t / 1e9,
                                             "us_per_copy": t / iters * 1e6}
            lib.ub_ldg(vp(buf.data_ptr()), C.c_int64(stride), C.c_uint32(byts), iters, grid, vp(ns.data_ptr()),
                       vp(sink.data_ptr()))
            t = ns[:grid].cpu().numpy().max() / 1e9
            res[f"ldg_{kb}KB_grid{grid}"] = {"GBps_total": byts * iters * grid / t / 1e9,
                                             "us_per_copy": t / iters * 1e6}
    bar = torch.zeros(64, dtype=torch.int32, device="cuda")
    for grid in (148, 296, 592):
        lib.ub_barrier(vp(bar.data_ptr()), 1000, grid, vp(ns.data_ptr()))
        res[f"grid_barrier_us_grid{grid}"] = float(ns[0].item()) / 1000 / 1e3
    print(json.dumps(res, indent=1))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "ubench.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
