#!/bin/bash
O=gpurun_out; mkdir -p $O; : > $O/c4ramp.log
for r in 1024 4096 16384; do
P="timeout 600 python scripts/e2e_probe.py --config C4 --reads 50000 --calls 4"
SA_RAMP0=$r $P --pageable 2>&1 | grep chunk | sed "s/^/ramp=$r /" >> $O/c4ramp.log
SA_RAMP0=$r $P 2>&1 | grep chunk | sed "s/^/ramp=$r pinned /" >> $O/c4ramp.log
done
for r in 1024 16384; do
SA_RAMP0=$r timeout 600 python scripts/e2e_probe.py --config C3 --reads 500000 --calls 4 2>&1 | grep chunk | sed "s/^/C3 ramp=$r pinned /" >> $O/c4ramp.log
done
