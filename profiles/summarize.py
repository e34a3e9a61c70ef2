"""Summaries of the ncu captures kept under profiles/ (run here, on the files gpurun brought back).

  python profiles/summarize.py launches <launches.csv> [title]   per-kernel launch count / mean / share
  python profiles/summarize.py raw <raw.csv>                      key metrics of a --set full capture
"""

from __future__ import annotations

import csv
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__t_sector_hit_rate.pct",
]


def launches(path: str, title: str = "") -> None:
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        per.setdefault(r[ki], []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in per.values())
    if title:
        print(title)
    for k, v in per.items():
        print(f"{k[:70]:70s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:9.2f} us  share={sum(v) / total:6.1%}")


def raw(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("----")
        print(f"  Kernel Name  {name[:100]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:80s} {units[i]:>8s} {r[i]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    else:
        raw(sys.argv[2])
