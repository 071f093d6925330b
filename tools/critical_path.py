"""Critical path of a traced lower sweep (tools/trace_sweeps.py --out X.json -> X.npz).

Walks back from the last DIAG: each DIAG waits on its latest-finishing
contribution chunk, each chunk on its panel's DIAG.  Prints the chain with the
per-hop split: execution, pickup delay (item taken after its dependency was
already done) and handoff (dependency done -> item ready)."""
import sys

import numpy as np

z = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace_cfg2.npz")
tr, it = z["trace_l"], z["items_l"]
t0 = tr[:, 0].min()
take, ready, end = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
deps = z["deps"]
P = int(z["p_w"].shape[0])
diag_item = {int(it[i, 1]): i for i in range(len(it)) if it[i, 0] == 0}
chunks_to = {p: [] for p in range(P)}
for i in range(len(it)):
    if it[i, 0] == 1:
        for t in deps[it[i, 4]: it[i, 4] + it[i, 5]]:
            chunks_to[int(t)].append(i)
cur = max(diag_item.values(), key=lambda i: end[i])
chain = []
while True:
    chain.append(cur)
    if it[cur, 0] == 0:
        src = chunks_to[int(it[cur, 1])]
        if not src:
            break
        cur = max(src, key=lambda i: end[i])
    else:
        cur = diag_item[int(it[cur, 1])]
chain.reverse()
tot = {"exec": 0.0, "wait_after_take": 0.0, "pickup_late": 0.0}
prev_end = 0.0
for i in chain:
    late = max(0.0, take[i] - prev_end)       # dependency done before this item was even taken
    wait = ready[i] - max(take[i], prev_end)  # spin after take (incl. handoff latency)
    tot["exec"] += end[i] - ready[i]
    tot["wait_after_take"] += max(wait, 0.0)
    tot["pickup_late"] += late
    prev_end = end[i]
print(f"chain: {len(chain)} items ({sum(it[i,0]==0 for i in chain)} DIAG), ends at {end[chain[-1]]:.1f} us of {end.max():.1f}")
print({k: round(v, 1) for k, v in tot.items()})
for i in chain[-12:]:
    print(f"  {['DIAG','OFF'][it[i,0]]:5s} p={it[i,1]:4d} w={z['p_w'][it[i,1]]:3d} rows={it[i,3]-it[i,2]:4d} take={take[i]:7.1f} ready={ready[i]:7.1f} end={end[i]:7.1f}")
