#!/usr/bin/env python
"""Per-source-line instructions and stall samples of one kernel in an ncu
report:  python scripts/ncu_lines.py REPORT KERNEL_SUBSTRING [TOP]"""
import csv
import os
import subprocess
import sys


def main():
    rep, want = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, cur_fn, rows = None, None, []
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = os.path.basename(r[1])
            continue
        if r[0] == "Function Name":
            cur_fn = r[1]
            continue
        if r[0] == "Line No" or len(r) < 8 or r[2] != "-" or want not in (cur_fn or ""):
            continue
        try:
            rows.append((cur_file, int(r[0]), float(r[4].replace(",", "")), float(r[7].replace(",", "")),
                         r[1].strip()[:90]))
        except ValueError:
            pass
    ts = sum(x[2] for x in rows) or 1
    ti = sum(x[3] for x in rows) or 1
    print(f"total samples {ts:.0f}, warp instructions {ti:.3e}")
    for f, ln, s, i, src in sorted(rows, key=lambda x: -x[3])[:top]:
        print(f"{f}:{ln:5d}  inst {100 * i / ti:5.1f}%  stall {100 * s / ts:5.1f}%  {src}")


if __name__ == "__main__":
    main()
