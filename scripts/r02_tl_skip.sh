#!/bin/bash
O=gpurun_out; mkdir -p $O
SA_DEBUG_TIMELINE=1 SA_DEBUG_NOCOPY=1 SA_DEBUG_SKIP_LISTED=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 1 > $O/timeline_skip.log 2>&1
SA_DEBUG_TIMELINE=1 SA_DEBUG_NOCOPY=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 1 > $O/timeline_nocopy.log 2>&1
