#!/bin/bash
# C2 e2e from pageable caller buffers: staging copy threads vs host packing
O=gpurun_out; mkdir -p $O; : > $O/pageable.log
P="timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 5"
$P --pageable 2>&1 | grep chunk | sed 's/^/default /' >> $O/pageable.log
SA_STAGE_THREADS=16 $P --pageable 2>&1 | grep chunk | sed 's/^/stage16 /' >> $O/pageable.log
SA_PACK_THREADS=8 $P --pageable 2>&1 | grep chunk | sed 's/^/pack8 /' >> $O/pageable.log
SA_PACK_THREADS=16 $P --pageable 2>&1 | grep chunk | sed 's/^/pack16 /' >> $O/pageable.log
SA_PACK_THREADS=16 $P 2>&1 | grep chunk | sed 's/^/pack16-pinned /' >> $O/pageable.log
