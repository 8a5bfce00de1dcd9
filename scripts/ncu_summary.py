#!/usr/bin/env python
"""Summarise an ncu launch list of bench.py into per-kernel-kind numbers.

Input: the CSV written by
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -c 400 --csv --log-file <csv> python bench.py --steps 3 ...
Takes the last complete iteration (launches between two k_tick markers) and
aggregates per kernel kind (td_avg, td, cur, obs, pred, spmv, tick): launch
count, summed device time (cold-cache, serialised: compare SHARES) and DRAM
bytes.  Writes/updates profiles/ncu_traffic.json (read by bench.py for the
roofline "traffic" field) and prints a markdown table.

  python scripts/ncu_summary.py gpurun_out/launches_dram.csv --workload goofspiel5 --variant pcfr+
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import re
from collections import OrderedDict

LK = {0: "td_avg", 1: "td", 2: "cur", 3: "obs", 4: "pred"}


def kind_of(name: str, predictive: bool) -> str:
    m = re.search(r"k_level(?:_gp?)?<(\d+)", name)
    if m:
        k = LK[int(m.group(1))]
        if k == "obs" and not predictive:
            return "obs_rm"
        return k
    for key in ("k_spmv", "k_tick", "k_avg0", "k_small", "k_persistent"):
        if key in name:
            return {"k_spmv": "spmv", "k_tick": "tick", "k_avg0": "td_avg",
                    "k_small": "persistent", "k_persistent": "persistent"}[key]
    return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--workload", default="goofspiel5")
    ap.add_argument("--variant", default="pcfr+")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "ncu_traffic.json"))
    args = ap.parse_args()
    lines = open(args.csv).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    launches: "OrderedDict[str, dict]" = OrderedDict()
    for r in rows[1:]:
        lid = r[col["ID"]]
        d = launches.setdefault(lid, {"name": r[col["Kernel Name"]], "grid": r[col["Grid Size"]]})
        val = float(r[col["Metric Value"]].replace(",", ""))
        unit = r[col["Metric Unit"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
                 "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1)
        d[r[col["Metric Name"]]] = val * scale
    seq = list(launches.values())
    ticks = [i for i, d in enumerate(seq) if "k_tick" in d["name"]]
    # the longest tick-to-tick window holding only iteration kernels (creates,
    # reads and checks run other kernels between iterations; with overlapped
    # alt iterations the last window is the epilogue, a partial iteration)
    best = None
    for a, b in zip(ticks, ticks[1:]):
        win = seq[a + 1:b + 1]
        if all("k_level" in d["name"] or "k_tick" in d["name"] or "k_spmv" in d["name"]
               or "k_avg0" in d["name"] for d in win) and (best is None or len(win) >= len(best)):
            best = win
    if best is not None:
        seq = best
    pred = args.variant in ("pcfr", "pcfr+")
    agg: dict = {}
    for d in seq:
        k = kind_of(d["name"], pred)
        a = agg.setdefault(k, {"launches": 0, "seconds": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["seconds"] += d.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(a["seconds"] for a in agg.values()) or 1.0
    print(f"| kind | launches | ncu time (us) | share | DRAM bytes/launch | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    out = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["seconds"]):
        per = a["dram_bytes"] / a["launches"]
        gbs = a["dram_bytes"] / a["seconds"] / 1e9 if a["seconds"] else 0.0
        print(f"| {k} | {a['launches']} | {a['seconds'] * 1e6:.1f} | {a['seconds'] / total:.2f} | "
              f"{per:.3e} | {gbs:.0f} |")
        out[k] = per
    # the longest launch of each kind (bench.py's roofline names the longest
    # launch of the step): its own DRAM bytes, key "<kind>@top"
    for k in list(out):
        ds = [d for d in seq if kind_of(d["name"], pred) == k]
        top = max(ds, key=lambda d: d.get("gpu__time_duration.sum", 0.0))
        out[k + "@top"] = top.get("dram__bytes_read.sum", 0.0) + top.get("dram__bytes_write.sum", 0.0)
        print(f"longest {k}: {top['name'][:60]} grid {top['grid']} {top.get('gpu__time_duration.sum', 0) * 1e6:.1f} us "
              f"{out[k + '@top'] / 1e6:.2f} MB DRAM")
    db = {}
    if os.path.exists(args.out):
        with open(args.out) as fh:
            db = json.load(fh)
    db[args.workload] = out
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(db, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
