#!/bin/bash
# C2 e2e vs chunk size / first ramp size (run under gpurun)
O=gpurun_out; mkdir -p $O; : > $O/chunks.log
for c in 425984 655360 1048576 1572864; do for r in 16384 65536; do
SA_CHUNK_READS=$c SA_RAMP0=$r timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 2>&1 | grep chunk | sed "s/^/ramp=$r /" >> $O/chunks.log
done; done
