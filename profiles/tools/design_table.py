#!/usr/bin/env python
"""Markdown tables of DESIGN.md section 5 from a capture directory's bench lines and timelines.

    python profiles/tools/design_table.py profiles/r02_v3            # print
    python profiles/tools/design_table.py profiles/r02_v3 --write    # and replace them in DESIGN.md
"""
from __future__ import annotations

import json
import os
import sys


def line(d: str, name: str):
    p = os.path.join(d, name)
    if not os.path.exists(p):
        return None
    txt = open(p).read().strip().splitlines()
    return json.loads(txt[-1]) if txt else None


def timelines(d: str) -> str:
    """The milestone table of the four step timelines (profiles/tools/gtrace.py output)."""
    def col(name):
        out = {}
        for l in open(os.path.join(d, name)).read().splitlines()[1:]:
            pr = l.split()
            if "last" not in pr:
                continue
            j = len(pr) - 1 - pr[::-1].index("last")
            out[" ".join(pr[1:j - 2])] = (pr[j - 1], pr[j + 1])
        return out

    cols = [col(f) for f in ("timeline_cfg4.txt", "timeline_cfg4_outliers_8x100.txt", "timeline_cfg2.txt",
                             "timeline_cfg2_outliers_8x100.txt")]
    names = [("split CTA start", "X split: CTA start"), ("split row done", "X split: row done"),
             ("GEMM CTA start", "GEMM CTA resident (programmatic launch)"),
             ("dep wait returned", "`griddepcontrol.wait` returns"), ("first MMA commit", "first MMA stage committed"),
             ("outlier terms: start", "epilogue: outlier lookups start (first unit)"),
             ("outlier terms: done", "epilogue: outlier lookups done"), ("last MMA issued", "last MMA issued"),
             ("accumulator ready", "accumulator ready"), ("epilogue done", "epilogue done"), ("CTA exit", "CTA exit")]
    rows = ["| milestone (first – last CTA) | cfg4 | cfg4, 8 channels at 100× | cfg2 | cfg2, 8 channels at 100× |",
            "|---|---|---|---|---|"]
    for k, label in names:
        rows.append(f"| {label} | " + " | ".join(f"{c[k][0]} – {c[k][1]}" for c in cols) + " |")
    return "\n".join(rows)


def write_design(d: str, tables: str) -> None:
    """Replace the bench tables and the timeline table of DESIGN.md section 5."""
    root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    path = os.path.join(root, "DESIGN.md")
    s = open(path).read()
    a, b = s.index("| config | step | split / GEMM |"), s.index("(`cfg1` is launch-bound;")
    s = s[:a] + tables + "\n\n" + s[b:]
    a, b = s.index("| milestone (first – last CTA) |"), s.index("cfg4 spends ")
    s = s[:a] + timelines(d) + "\n\n" + s[b:]
    open(path, "w").write(s)


def main() -> None:
    d = sys.argv[1]
    if "--write" in sys.argv:
        import contextlib
        import io

        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            sys.argv.remove("--write")
            main()
        parts = buf.getvalue().strip().split("\n\n")
        write_design(d, parts[0] + "\n\n" + parts[1])
        print(buf.getvalue())
        return
    rows = [("cfg1 64×512×512", "bench_cfg1.json"), ("cfg2 256×4096×4096 +PReLU", "bench_cfg2.json"),
            ("cfg3 512×8192² s=1/16", "bench_cfg3_s1_16.json"), ("cfg3 s=1/8", "bench_cfg3_s1_8.json"),
            ("cfg3 s=1/4", "bench_cfg3_s1_4.json"), ("cfg3 s=1/2", "bench_cfg3_s1_2.json"),
            ("cfg4 16×4096×11008 +PReLU", "bench_cfg4.json"), ("**cfg5 8192×8192×16384 (default)**", "bench_default.json")]
    print("| config | step | split / GEMM | effective | × north-star roofline (GEMM kernel) | int8 tensor frac (burst / sustained peak) | DRAM per launch vs TCSC bytes | e2e (public API, host buffers) | CPU reference (16 cores) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for label, f in rows:
        j = line(d, f)
        if not j:
            continue
        r, e, t = j["roofline"], j.get("e2e") or {}, j["roofline"].get("tensor") or {}
        us = 1e3
        step = j["ms_per_step"] * us
        stepf = f"{step:.1f} µs" if step < 1000 else f"{step / 1000:.2f} ms"
        pr, ru = j["breakdown_ms"]["prepare"] * us, j["breakdown_ms"]["run"] * us
        prf = f"{pr:.1f} / {ru:.1f} µs" if ru < 1000 else f"{pr / 1000:.2f} / {ru / 1000:.2f} ms"
        tr = r.get("traffic")
        trf = f"{tr / 1e6:.1f} / {r['algorithmic_bytes_per_launch'] / 1e6:.0f} MB" if tr else "—"
        clk = j["clocks"]
        note = f" ({', '.join(clk['reasons'])}, {clk['sm_mhz']:.0f} MHz)" if clk["reasons"] else ""
        cpu = (j.get("cpu_baseline") or {}).get("value")
        ems = e.get("ms_per_step")
        print(f"| {label} | {stepf}{note} | {prf} | {j['value'] / 1e3:.1f} TOP/s | {r['frac']:.2f} ({r['bound']}) | "
              f"{t.get('frac', 0):.2f} / {t.get('frac_of_sustained', 0):.2f} | {trf} | "
              f"{e.get('value', 0) / 1e3:.2f} TOP/s ({ems:.3f} ms) | {cpu:.1f} GOP/s |")
    print()
    print("| heavy-tailed X (8 channels at 100×) | step | split / GEMM | plain X step | ratio | rows: exact walk / shed / listed entries | normwise, scaled error |")
    print("|---|---|---|---|---|---|---|")
    for label, f, g in [("cfg4", "bench_cfg4_outliers_8x100.json", "bench_cfg4.json"),
                        ("cfg2", "bench_cfg2_outliers_8x100.json", "bench_cfg2.json"),
                        ("cfg5", "bench_cfg5_outliers_8x100.json", "bench_default.json")]:
        j, k = line(d, f), line(d, g)
        if not j or not k:
            continue
        x = j["run"]["x_rows"]
        sc = 1e3 if j["ms_per_step"] < 1 else 1
        un = "µs" if sc == 1e3 else "ms"
        print(f"| {label} | {j['ms_per_step'] * sc:.2f} {un} | {j['breakdown_ms']['prepare'] * sc:.2f} / {j['breakdown_ms']['run'] * sc:.2f} {un} | "
              f"{k['ms_per_step'] * sc:.2f} {un} | {j['ms_per_step'] / k['ms_per_step']:.2f} | {x['exact_rows']} / {x['outlier_rows']} / {x['outlier_entries']} | "
              f"{j['parity']['normwise_vs_fp64']:.1e}, {j['parity']['scaled_vs_fp64']:.1e} |")
    ref = line(d, "bench_ref_default.json")
    if ref:
        print()
        print(f"reference arm: {ref['value']:.1f} GOP/s, {ref['ms_per_step']:.0f} ms per step, kind {ref['cpu_baseline']['kind']}, "
              f"{ref['cpu_baseline']['cores']} cores; {ref['cpu_baseline']['sample']}")
    g = line(d, "bench_cfg2_gather.json")
    if g:
        print(f"gather cfg2: {g['ms_per_step']:.3f} ms, {g['value'] / 1e3:.2f} TOP/s, frac {g['roofline']['frac']:.3f}; e2e {g['e2e']['ms_per_step']:.3f} ms")


if __name__ == "__main__":
    main()
