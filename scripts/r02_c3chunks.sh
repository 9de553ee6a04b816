#!/bin/bash
# C3 e2e vs chunk size
O=gpurun_out; mkdir -p $O; : > $O/c3chunks.log
for c in 262144 393216 524288; do
  SA_CHUNK_READS=$c timeout 600 python scripts/e2e_probe.py --config C3 --reads 500000 --calls 4 2>&1 | grep chunk >> $O/c3chunks.log
  SA_CHUNK_READS=$c SA_DEBUG_NOCOPY=1 timeout 600 python scripts/e2e_probe.py --config C3 --reads 500000 --calls 4 2>&1 | grep chunk | sed 's/^/nocopy /' >> $O/c3chunks.log
done
