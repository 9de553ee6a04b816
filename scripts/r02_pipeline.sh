#!/bin/bash
# C2 e2e pipeline diagnostics (run under gpurun)
O=gpurun_out; mkdir -p $O
SA_PIPE_SINGLE=1 timeout 600 python scripts/ktime.py C2 > $O/ktime_c2.log 2>&1
timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --copy-floor > $O/e2e_c2.log 2>&1
for c in 425984 1048576 2097152; do
SA_DEBUG_NOCOPY=1 SA_CHUNK_READS=$c timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 >> $O/e2e_c2_nocopy.log 2>&1
done
