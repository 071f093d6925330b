"""Summarise a saved sweep trace (tools/trace_sweeps.py --out X.json -> X.npz):
per item kind the mean take->ready / ready->staged / staged->computed /
computed->end times (us) and the items in flight per 50 us bin.

    python tools/trace_stats.py gpurun_out/r2_trace_cfg3.npz
"""
import sys

import numpy as np


def main(path):
    z = np.load(path)
    for nm in ("trace_l", "trace_u"):
        tr = z[nm].astype(np.int64)
        it = z["items_l" if nm == "trace_l" else "items_u"]
        t0 = tr[:, 0].min()
        take, ready, end, st, cp = [(tr[:, k] - t0) / 1e3 for k in (0, 1, 2, 4, 5)]
        seg = it[:, 3]
        print(nm, "items", len(tr), "wall %.1f us" % end.max())
        WHOLE = 1 << 20  # csrc kWhole: whole-tiles items
        for name, mask in (("chunk", (seg > 0) & (seg != WHOLE)), ("whole", seg == WHOLE), ("small", seg == 0),
                           ("fin", seg < 0)):
            if mask.sum() == 0:
                continue
            if name == "fin":
                print("  fin %d take->ready %.2f total %.2f" % (mask.sum(), np.mean((ready - take)[mask]),
                                                              np.mean((end - take)[mask])))
                continue
            print("  %s %d take->ready %.2f ready->staged %.2f staged->computed %.2f computed->end %.2f total %.2f" % (
                name, mask.sum(), np.mean((ready - take)[mask]), np.mean((st - ready)[mask]),
                np.mean((cp - st)[mask]), np.mean((end - cp)[mask]), np.mean((end - take)[mask])))
        bins = np.arange(0, end.max() + 50, 50)
        print("  in flight per 50 us:", [int(((take < b + 50) & (end > b)).sum()) for b in bins[:-1]])
        busy = np.zeros(len(bins) - 1)
        for a, b_ in zip(ready, end):
            pass
        print("  executing (ready..end) per 50 us:",
              [round(float(np.clip(np.minimum(end, b + 50) - np.maximum(ready, b), 0, None).sum() / 50), 1)
               for b in bins[:-1]])


if __name__ == "__main__":
    main(sys.argv[1])
