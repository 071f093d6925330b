"""Apply time of the LDL^T sweeps vs the item granularity (segments per chunk
item, TMA groups per small-tile item): packs the bench workload's factors
once per setting and times dev.run("apply") with CUDA events, L2 flushed.

    python tools/item_tune.py [--workload cfg3] [--segs 1,2,4,8] [--groups 1,2,4] [--ratios 0,1]

--ratios sweeps the lower input-mode threshold (K.GATHER_RATIO); the lower
and upper sweeps are timed separately too.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2306_05893_b200 import _ldlt_pack as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--segs", default="1,2,4,8")
    ap.add_argument("--groups", default="1,2,4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ratios", default="")
    ap.add_argument("--segs-lower", default="", help="lower-sweep segments per chunk (default: --segs)")
    ap.add_argument("--whole", default="", help="segments per whole-tiles item (default: --segs)")
    ap.add_argument("--few", default="", help="K.GATHER_FEW values")
    ap.add_argument("--cbcap", type=int, default=None, help="K.CB_CAP (contribution staging; 0 = sum from L2)")
    args = ap.parse_args()
    import torch

    W = bench.build_workload(args.workload)
    f = W["factors"]
    flush = bench.L2Flush()
    r = torch.randn(f.plan.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    out = []

    def timed(dev, mode):
        for _ in range(3):
            dev.run(mode, r, z)
        ts = []
        for _ in range(args.reps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.run(mode, r, z)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    if args.cbcap is not None:
        K.CB_CAP = args.cbcap
    ratios = [float(v) for v in args.ratios.split(",")] if args.ratios else [None]
    lowers = [int(v) for v in args.segs_lower.split(",")] if args.segs_lower else [None]
    wholes = [int(v) for v in args.whole.split(",")] if args.whole else [None]
    fews = [int(v) for v in args.few.split(",")] if args.few else [K.GATHER_FEW]
    for ratio, sl, wh, fw in [(r_, l_, w_, f_) for r_ in ratios for l_ in lowers for w_ in wholes for f_ in fews]:
        K.SEGS_LOWER, K.WHOLE_SEGS, K.GATHER_FEW = sl, wh, fw
        K.GATHER_RATIO = ratio
        for sg in map(int, args.segs.split(",")):
            for gr in map(int, args.groups.split(",")):
                K.SEGS_PER_ITEM, K.GROUPS_PER_ITEM = sg, min(gr, K.MAX_GROUPS)  # overrides of item_granularity (csrc kGroupsPerItem)
                dev = K.DevicePanels(f)
                row = {"segs": sg, "segs_lower": sl, "whole": wh, "few": fw, "groups": gr, "ratio": ratio, "apply_ms": timed(dev, "apply"),
                       "lower_ms": timed(dev, "lower"), "upper_ms": timed(dev, "upper"), "items": dev.n_items}
                print(json.dumps(row), flush=True)
                out.append(row)
                del dev
    print(json.dumps({"workload": args.workload, "best": min(out, key=lambda x: x["apply_ms"])}))


if __name__ == "__main__":
    main()
