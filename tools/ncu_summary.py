"""Summarise ncu captures (tools/profile.sh output) into profiles/.

    python tools/ncu_summary.py gpurun_out/ncu_r1_cfg2 profiles/r1_ncu_cfg2 [--bytes kernel=B ...]

Writes <out>.md (one table: duration, DRAM traffic, GB/s, occupancy, top
stall reasons per kernel + the per-kernel share of the launch list) and
<out>.json (the raw numbers).  `--bytes` gives the algorithmic bytes per
launch of a kernel so the table also shows algorithmic GB/s.
"""

from __future__ import annotations

import collections
import csv
import json
import re
import subprocess
import sys
from pathlib import Path

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dyn_B": "launch__shared_mem_per_block_dynamic",
}
UNIT = {"Mbyte": 1.0, "Kbyte": 1e-3, "Gbyte": 1e3, "byte": 1e-6, "us": 1.0, "ms": 1e3, "ns": 1e-3}


def raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def num(m, key):
    if key not in m:
        return None
    u, v = m[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * UNIT.get(u, 1.0)


def stalls(m, top=4):
    st = {}
    for h, (u, v) in m.items():
        g = re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_(\w+?)", h)
        if g and not h.endswith("_not_issued"):
            try:
                st[g.group(1)] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    return [(k, round(100 * v / tot, 1)) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:top]]


def launch_shares(path: Path):
    rows = list(csv.reader(path.read_text().splitlines()))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
            agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "total_us": round(sum(v), 1), "avg_us": round(sum(v) / len(v), 2),
                "share_pct": round(100 * sum(v) / tot, 1)} for k, v in agg.items()}


def main():
    src, out = Path(sys.argv[1]), Path(sys.argv[2])
    algo = {}
    for a in sys.argv[3:]:
        if "=" in a:
            k, v = a.split("=", 1)
            algo[k] = float(v)
    res = {"kernels": {}, "launch_list": None}
    if (src / "launches.csv").exists():
        res["launch_list"] = launch_shares(src / "launches.csv")
    for rep in sorted(src.glob("full_*.ncu-rep")):
        m = raw(rep)
        k = rep.stem[len("full_"):]
        d = {name: num(m, key) for name, key in KEYS.items()}
        d["stalls_top"] = stalls(m)
        if d["duration_us"] and d["dram_read_MB"] is not None:
            d["traffic_MB"] = round(d["dram_read_MB"] + d["dram_write_MB"], 3)
            d["dram_GBs"] = round(d["traffic_MB"] / d["duration_us"] * 1e3, 1)
            if k in algo:
                d["algorithmic_MB"] = algo[k] / 1e6
                d["algorithmic_GBs"] = round(algo[k] / 1e6 / d["duration_us"] * 1e3, 1)
        res["kernels"][k] = d
    out.with_suffix(".json").write_text(json.dumps(res, indent=1))
    lines = [f"# ncu summary: {src.name}", "",
             "Captured with tools/profile.sh (`ncu --set full --clock-control none`, one launch per kernel,",
             "cold cache, serialised).  GB/s = (dram read + write) / duration.", "",
             "| kernel | grid x block | regs | us | DRAM MB (r+w) | DRAM GB/s | algo MB | algo GB/s | DRAM % | SM % | warps active % | top stalls (% of samples) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, d in res["kernels"].items():
        def f(x, p=1):
            return "-" if x is None else f"{x:.{p}f}"
        lines.append(f"| {k} | {f(d['grid'],0)} x {f(d['block'],0)} | {f(d['regs'],0)} | {f(d['duration_us'])} | "
                     f"{f(d.get('traffic_MB'),2)} | {f(d.get('dram_GBs'))} | {f(d.get('algorithmic_MB'),2)} | "
                     f"{f(d.get('algorithmic_GBs'))} | {f(d['dram_pct'])} | {f(d['sm_pct'])} | "
                     f"{f(d['warps_active_pct'])} | {', '.join(f'{a} {b}' for a, b in d['stalls_top'])} |")
    if res["launch_list"]:
        lines += ["", "## Launch list (gpu__time_duration per launch, whole short bench run)", "",
                  "| kernel | launches | total us | avg us | share % |", "|---|---|---|---|---|"]
        for k, d in sorted(res["launch_list"].items(), key=lambda kv: -kv[1]["total_us"]):
            lines.append(f"| {k} | {d['launches']} | {d['total_us']} | {d['avg_us']} | {d['share_pct']} |")
    out.with_suffix(".md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
