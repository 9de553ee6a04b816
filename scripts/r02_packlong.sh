#!/bin/bash
# long reads from pinned buffers: ASCII vs host-packed vs end-of-batch overflow pass
O=gpurun_out; mkdir -p $O; : > $O/packlong.log
P="timeout 600 python scripts/e2e_probe.py --config C3 --reads 500000 --calls 4"
$P 2>&1 | grep chunk | sed "s/^/C3 ascii /" >> $O/packlong.log
SA_CHUNK_OVERFLOW=0 $P 2>&1 | grep chunk | sed "s/^/C3 ascii-endpass /" >> $O/packlong.log
SA_PACK_THREADS=16 $P 2>&1 | grep chunk | sed "s/^/C3 pack16 /" >> $O/packlong.log
SA_PACK_THREADS=8 $P 2>&1 | grep chunk | sed "s/^/C3 pack8 /" >> $O/packlong.log
