#!/usr/bin/env python
"""profiles/traffic.json from the per-config ncu CSVs of profiles/tools/capture.sh.

    python profiles/tools/traffic.py profiles/r02_v3

Each traffic_<cfg>.csv holds dram__bytes_read.sum / dram__bytes_write.sum / gpu__time_duration.sum
of two launches of the dominant kernel (tg_mma_kernel, or the gather walk); the entry written
is the mean read + write bytes per launch.  bench.py reports it as roofline.traffic.
"""
from __future__ import annotations

import csv
import glob
import json
import os
import sys


def per_launch(path: str) -> tuple[float, float]:
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ii, mi, ui, vi = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    by_id: dict[str, dict[str, float]] = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        if r[mi].startswith("dram__bytes"):
            v *= scale[r[ui]]
        by_id.setdefault(r[ii], {})[r[mi]] = v
    tot = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in by_id.values()]
    us = [d["gpu__time_duration.sum"] for d in by_id.values()]
    return sum(tot) / len(tot), sum(us) / len(us)


def main() -> None:
    d = sys.argv[1]
    out = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel "
                    "(ncu --clock-control none, mean of two launches), written by profiles/tools/traffic.py",
           "_source": d}
    for p in sorted(glob.glob(os.path.join(d, "traffic_*.csv"))):
        name = os.path.basename(p)[len("traffic_"):-len(".csv")]
        key = name[:-len("_gather")] + ":gather" if name.endswith("_gather") else name + ":mma"
        b, t = per_launch(p)
        out[key] = int(round(b))
        print(f"{key:24s} {b / 1e6:10.2f} MB per launch   ({t:.1f} under ncu, unit as exported)")
    out["cfg3:mma"] = out.get("cfg3_s1_2:mma")
    root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    with open(os.path.join(root, "profiles", "traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
