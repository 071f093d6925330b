"""Packing constants probe: apply time per (HOP, SCHED_WORKERS) of the list
schedule, or per FIN_CONTRIB (finaliser granularity) with --fin.

    python tools/sched_probe.py cfg2|cfg3 [--fin]
"""
import itertools
import json
import statistics
import sys

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402


def main():
    import torch
    from paper_2306_05893_b200 import _ldlt_pack as K
    from paper_2306_05893_b200._ldlt_pack import DevicePanels

    W = bench.build_workload(sys.argv[1])
    f = W["factors"]
    flush = bench.L2Flush()
    r = torch.randn(f.plan.n, dtype=torch.float64, device="cuda")
    out = {}
    fin = "--fin" in sys.argv
    grid = [(None, None, c) for c in (1024, 2048, 4096, 16384)] if fin else \
        [(h, w, None) for h, w in itertools.product((0.5, 1.5, 4.0), (296, 444, 888))]
    for hop, workers, fc in grid:
        if fin:
            K.FIN_CONTRIB = fc
        else:
            K.HOP, K.SCHED_WORKERS = hop, workers
        dev = DevicePanels(f)
        z = torch.empty_like(r)
        for _ in range(3):
            dev.run("apply", r, z)
        ts = []
        for _ in range(15):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dev.run("apply", r, z)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        out[f"fin{fc}" if fin else f"{hop}/{workers}"] = round(statistics.median(ts), 4)
        del dev
    print(sys.argv[1], json.dumps(out))


if __name__ == "__main__":
    main()
