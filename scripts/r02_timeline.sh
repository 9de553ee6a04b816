#!/bin/bash
# C2 batch-pipeline timeline (SA_DEBUG_TIMELINE): chunk, kernel tag, event time
O=gpurun_out; mkdir -p $O
SA_DEBUG_TIMELINE=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 1 > $O/timeline_c2.log 2>&1
SA_DEBUG_TIMELINE=1 SA_CHUNK_READS=1048576 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 1 > $O/timeline_c2_1m.log 2>&1
