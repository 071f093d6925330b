"""Steady state of AsyncPreconditioner(device=True) on cfg2 (bench.time_async_device).
    TSB_PCG_CTAS_PER_SM=2 python tools/async_probe.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402

W = bench.build_workload("cfg2")
print(json.dumps(bench.time_async_device(W, 40, bench.L2Flush())))
