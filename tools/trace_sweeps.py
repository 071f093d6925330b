"""Per-item timeline of the persistent LDL^T sweep kernels (globaltimer trace).

    python tools/trace_sweeps.py [--workload cfg2] [--out gpurun_out/trace_cfg2.json]

Prints, per sweep: wall time, items by type with mean wait (take -> ready)
and execute (ready -> end) times, and the fraction of CTA-time spent waiting
on dependencies -- the evidence for where the level-scheduled latency goes.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2306_05893_b200._ldlt_pack import DevicePanels  # noqa: E402


def summarize(tr, kinds, names):
    t0 = tr[:, 0].min()
    take, ready, end = tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 2] - t0
    out = {"wall_us": float(end.max() / 1e3), "items": int(len(tr))}
    per = {}
    for ty in np.unique(kinds):
        m = kinds == ty
        per[names[int(ty)]] = {
            "count": int(m.sum()),
            "wait_us_mean": float(((ready - take)[m]).mean() / 1e3),
            "exec_us_mean": float(((end - ready)[m]).mean() / 1e3),
            "stage_us_mean": float(((tr[:, 4] - tr[:, 1])[m]).mean() / 1e3),
            "compute_us_mean": float(((tr[:, 5] - tr[:, 4])[m]).mean() / 1e3),
            "publish_us_mean": float(((tr[:, 2] - tr[:, 5])[m]).mean() / 1e3),
        }
    out["by_kind"] = per
    busy = float((end - ready).sum())
    wait = float((ready - take).sum())
    out["wait_fraction_of_item_time"] = wait / max(busy + wait, 1.0)
    out["sms_used"] = int(len(np.unique(tr[:, 3])))
    bins = np.linspace(0, end.max(), 11)
    conc = []
    for a, b in zip(bins[:-1], bins[1:]):
        ov = np.clip(np.minimum(end, b) - np.maximum(ready, a), 0, None).sum() / max(b - a, 1)
        conc.append(round(float(ov), 1))
    out["mean_executing_items_per_decile"] = conc
    return out


def lower_chain(tr, items, H):
    """Critical chain of the lower sweep: from the last item back through the
    child item that completed each block's input."""
    t0 = tr[:, 0].min()
    end = (tr[:, 2] - t0) / 1e3
    ready = (tr[:, 1] - t0) / 1e3
    blk = items[:, 0]
    by_block = {}
    for i, b in enumerate(blk):
        by_block.setdefault(int(b), []).append(i)
    cur = int(np.argmax(end))
    chain = []
    while True:
        chain.append(cur)
        kids = H["children"][int(blk[cur])]
        if not kids:
            break
        cand = [i for c in kids for i in by_block[c]]
        cur = max(cand, key=lambda i: end[i])
    chain.reverse()
    return [{"block": int(blk[i]), "m": int(H["blocks"][blk[i]]["m"]), "ready": round(float(ready[i]), 2),
             "end": round(float(end[i]), 2)} for i in chain]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    W = bench.build_workload(args.workload)
    f = W["factors"]
    dev = DevicePanels(f, trace=True)
    r = torch.randn(f.plan.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    flush = bench.L2Flush()
    res = []
    for _ in range(args.reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.run("apply", r, z)
        e1.record()
        e1.synchronize()
        res.append(e0.elapsed_time(e1))
    H = dev.host
    plain = DevicePanels(f)  # same kernels without the trace instrumentation
    res_plain = []
    for _ in range(args.reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plain.run("apply", r, z)
        e1.record()
        e1.synchronize()
        res_plain.append(e0.elapsed_time(e1))
    report = {
        "workload": args.workload, "apply_ms_median": float(np.median(res)),
        "apply_ms_untraced": float(np.median(res_plain)), "blocks": H["nb"],
        "n": H["n"], "grid_note": "persistent grid = SMs x resident CTAs",
        "lower": summarize(dev.trace_l.cpu().numpy(), (H["blocks"]["target_l"][H["items_l"][:, 0]] > 0).astype(int),
                           {0: "leaf", 1: "inner"}),
        "upper": summarize(dev.trace_u.cpu().numpy(), (H["blocks"]["na"][H["items_u"][:, 0]] > 0).astype(int),
                           {0: "root", 1: "inner"}),
        "lower_chain": lower_chain(dev.trace_l.cpu().numpy(), H["items_l"], H),
    }
    txt = json.dumps(report, indent=1)
    print(txt)
    if args.out:
        Path(args.out).write_text(txt)
        keep = {k: H[k] for k in ("items_l", "items_u", "parent")}
        keep.update(np_l=H["tiles_l"]["np"], np_u=H["tiles_u"]["np"], m=H["blocks"]["m"], na=H["blocks"]["na"],
                    mode=H["blocks"]["mode"])
        np.savez_compressed(Path(args.out).with_suffix(".npz"), trace_l=dev.trace_l.cpu().numpy(),
                            trace_u=dev.trace_u.cpu().numpy(), **keep)


if __name__ == "__main__":
    main()
