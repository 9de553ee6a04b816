#!/bin/bash
# Per-kernel time / instructions of one bench step (C1), for the two-kernel path.
cd "$(dirname "$0")/.."
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"seed_kernel|align_kernel" -c ${1:-3} --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null \
  | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>14 and r[0].isdigit()]
for r in rows: print(r[0], r[4][:45], r[12], r[14])
"
