#!/usr/bin/env python
"""Summarise ncu evidence for profiles/.

  python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
      --report gpurun_out/prof.ncu-rep --tag r01b --config C1 --reads 1000000

Writes profiles/<tag>_launches_<config>.csv (the launch list, copied),
profiles/<tag>_ncu_<config>.md (per-kernel share of the step from the launch
list; key metrics, stall breakdown and top source lines of the full capture)
and updates profiles/ncu_traffic.json[<config>] with the captured kernel's
DRAM bytes per launch, which bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (registers), blocks"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit %"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "L1 global load requests"),
]


def _num(s: str) -> float:
    return float(s.replace(",", ""))


def launches(path: str) -> list[tuple[str, float]]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(r[ki], _num(r[vi])) for r in rows[1:] if r[h.index("Metric Name")] == "gpu__time_duration.sum"]


def raw(report: str) -> tuple[list[dict], dict]:
    """One dict per captured kernel launch, and the units."""
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    return [dict(zip(h, d)) for d in rows[2:]], dict(zip(h, u))


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return _num(v) * scale.get(unit, 1)


def source_lines(report: str, top: int = 25) -> list[tuple[str, int, float, float, str]]:
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, rows = None, []
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur = os.path.basename(r[1])
            continue
        if r[0] in ("Function Name", "Line No") or len(r) < 8 or r[2] != "-":
            continue
        try:
            rows.append((cur, int(r[0]), _num(r[4]), _num(r[7]), r[1].strip()[:80]))
        except ValueError:
            pass
    ts = sum(x[2] for x in rows) or 1
    ti = sum(x[3] for x in rows) or 1
    rows.sort(key=lambda x: -x[2])
    return [(f, ln, 100 * s / ts, 100 * i / ti, src) for f, ln, s, i, src in rows[:top]]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", required=True)
    ap.add_argument("--report", required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="C1")
    ap.add_argument("--reads", type=int, default=1_000_000)
    ap.add_argument("--alg-bytes-per-read", type=float, default=None)
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(args.launches, os.path.join(PROF, f"{args.tag}_launches_{args.config}.csv"))

    lst = launches(args.launches)
    agg = collections.OrderedDict()
    for name, ns in lst:
        short = name.split("(")[0].replace("void ", "")[:70]
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += ns
    ds, u = raw(args.report)
    lines = [f"# ncu evidence {args.tag} ({args.config}, {args.reads} reads per launch)", "",
             "## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold, serialised)", "",
             "| kernel | launches | total us | mean us |", "|---|---|---|---|"]
    for k, (c, t) in agg.items():
        lines.append(f"| `{k}` | {c} | {t / 1e3:.1f} | {t / 1e3 / c:.1f} |")
    hot = [t for n, t in lst if any(k in n for k in ("seed_kernel", "solo_kernel", "resolve_kernel", "align_kernel",
                                                       "prune_kernel"))]
    if hot:
        steps = max(c for c, _ in agg.values())
        lines += ["", f"Hot-path kernels (seed, solo, resolve, warp, prune, global-table; all launches in the list): "
                      f"{sum(hot) / 1e6:.3f} ms total, {sum(hot) / 1e6 / steps:.3f} ms per step."]
    dram = 0.0
    for d in ds:
        lines += ["", f"## Full capture: `{d.get('Kernel Name', '?')[:80]}`", "", "| metric | value |", "|---|---|"]
        for key, label in METRICS:
            if key in d:
                lines.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
        if "dram__bytes_read.sum" in d:
            b = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + to_bytes(
                d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
            dram += b
            lines.append(f"| DRAM bytes per read | {b / args.reads:.0f} B |")
        st = {}
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k:
                try:
                    st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = _num(v)
                except ValueError:
                    pass
        tot = sum(st.values()) or 1
        lines += ["", "Warp-state samples: " + ", ".join(
            f"{k} {100 * v / tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8])]
    if args.alg_bytes_per_read:
        lines += ["", f"Algorithmic bytes per read (DESIGN.md §5): {args.alg_bytes_per_read:.0f} B; DRAM bytes per "
                      f"read of the captured kernels together: {dram / args.reads:.0f} B."]
    lines += ["", "## Top source lines by stall samples", "", "| file:line | samples | inst | source |",
              "|---|---|---|---|"]
    for f, ln, s, i, src in source_lines(args.report):
        lines.append(f"| {f}:{ln} | {s:.1f}% | {i:.1f}% | `{src.replace('|', '/')}` |")
    with open(os.path.join(PROF, f"{args.tag}_ncu_{args.config}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tp = os.path.join(PROF, "ncu_traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    if dram:
        tj[args.config] = {"dram_bytes_per_launch": dram, "reads_per_launch": args.reads, "tag": args.tag,
                           "kernels": [d.get("Kernel Name", "")[:80] for d in ds],
                           "source": "ncu --set full --clock-control none, one launch of each kernel, summed"}
        json.dump(tj, open(tp, "w"), indent=1)
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
