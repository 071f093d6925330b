"""Summarise a tools/trace_sweeps.py output: per-sweep stats + critical chains.

    python tools/trace_report.py gpurun_out/trace_cfg2.json
"""
import json
import sys

import numpy as np

path = sys.argv[1]
d = json.load(open(path))
for k in ("apply_ms_median", "apply_ms_untraced", "blocks"):
    print(k, d[k])
for sw in ("lower", "upper"):
    x = d[sw]
    print(sw, x["wall_us"], x["items"], "waitfrac", round(x["wait_fraction_of_item_time"], 2),
          x["mean_executing_items_per_decile"])
    for k, v in x["by_kind"].items():
        print("   ", k, {a: round(b, 2) for a, b in v.items()})
z = np.load(path.replace(".json", ".npz"), allow_pickle=True)
par = z["parent"]
for sw, up in (("l", False), ("u", True)):
    tr = z["trace_" + sw].astype(float)
    it = z["items_" + sw]
    T = (tr - tr[:, 0].min()) / 1e3
    end = T[:, 2]
    byb = {}
    for i, b in enumerate(it[:, 0]):
        byb.setdefault(int(b), []).append(i)
    kids = {}
    for b, p in enumerate(par):
        kids.setdefault(int(p), []).append(b)
    cur = int(np.argmax(end))
    chain = []
    while True:
        chain.append(cur)
        b = int(it[cur, 0])
        nxt = [int(par[b])] if up else kids.get(b, [])
        nxt = [q for q in nxt if q >= 0]
        if not nxt:
            break
        cur = max((i for q in nxt for i in byb[q]), key=lambda i: end[i])
    print(f"{sw} chain ({len(chain)} hops):")
    for i in reversed(chain):
        print("   blk %4d rows %4d-%4d take %7.2f ready %7.2f staged %7.2f computed %7.2f end %7.2f" % (
            it[i, 0], it[i, 1], it[i, 2], T[i, 0], T[i, 1], T[i, 4], T[i, 5], T[i, 2]))
