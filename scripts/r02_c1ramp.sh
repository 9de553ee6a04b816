#!/bin/bash
# C1 e2e vs chunk size and first ramp size
O=gpurun_out; mkdir -p $O; : > $O/c1ramp.log
for c in 32768 49152 65536; do for r in 4096 8192 16384; do
  SA_CHUNK_READS=$c SA_RAMP0=$r timeout 300 python scripts/e2e_probe.py --config C1 --reads 1000000 --calls 8 2>&1 | grep chunk | sed "s/^/ramp=$r /" >> $O/c1ramp.log
done; done
timeout 300 python scripts/e2e_probe.py --config C1 --reads 1000000 --calls 8 --copy-floor 2>&1 | grep "H2D\|chunk" >> $O/c1ramp.log
