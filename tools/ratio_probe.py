"""Lower-input mode threshold probe: apply / lower-sweep time per GATHER_RATIO.

    python tools/ratio_probe.py cfg2|cfg3
"""
import json, os, statistics, sys
sys.path.insert(0, "/root/repo")
import bench
import torch
from paper_2306_05893_b200 import _ldlt_pack as K
from paper_2306_05893_b200._ldlt_pack import DevicePanels
wl = sys.argv[1]
W = bench.build_workload(wl)
f = W["factors"]
flush = bench.L2Flush()
r = torch.randn(f.plan.n, dtype=torch.float64, device="cuda")
out = {}
for ratio in (0.0, 0.1, 0.3, 1.0, 3.0, 1e9):
    K.GATHER_RATIO = ratio
    dev = DevicePanels(f)
    z = torch.empty_like(r)
    for _ in range(3):
        dev.run("apply", r, z)
    ts = {"apply": [], "lower": []}
    for mode in ("apply", "lower"):
        for _ in range(15):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); dev.run(mode, r, z); b.record(); b.synchronize()
            ts[mode].append(a.elapsed_time(b))
    out[ratio] = {k: round(statistics.median(v), 4) for k, v in ts.items()}
    del dev
print(wl, json.dumps(out))
