#!/bin/bash
# C2 e2e and device time vs the solo kernel's grid cap (SA_SOLO_GRID)
O=gpurun_out; mkdir -p $O; : > $O/sologrid.log
for g in 888 1776 4000000; do
  echo "SA_SOLO_GRID=$g" >> $O/sologrid.log
  SA_SOLO_GRID=$g timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 2>&1 | grep chunk >> $O/sologrid.log
  SA_SOLO_GRID=$g SA_DEBUG_NOCOPY=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 2>&1 | grep chunk >> $O/sologrid.log
done
