#!/bin/bash
# C2 e2e vs smaller chunk sizes (run under gpurun)
O=gpurun_out; mkdir -p $O; : > $O/chunks_small.log
for c in 196608 262144 327680 425984; do
SA_CHUNK_READS=$c timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 8 2>&1 | grep chunk >> $O/chunks_small.log
done
