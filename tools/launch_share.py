"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_share.py launches.csv [--after KERNEL_SUBSTRING]

--after keeps the launches from the last occurrence of KERNEL_SUBSTRING on
(e.g. the last refactorisation of a repeated run)."""

import collections
import csv
import sys

UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def main():
    path = sys.argv[1]
    after = sys.argv[sys.argv.index("--after") + 1] if "--after" in sys.argv else None
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if after:
        idx = [i for i, d in enumerate(data) if after in d["Kernel Name"]]
        data = data[idx[-1]:] if idx else data
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {n[:60]:60s} {c:6d} {t:11.1f} us {100 * t / tot:5.1f}%  ({t / c:.1f} us/launch)")


if __name__ == "__main__":
    main()
