#!/bin/bash
# timing experiment: how much of the C2 pipeline and of one device launch the listed-read kernels cost
O=gpurun_out; mkdir -p $O; : > $O/skiplisted.log
P="timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 5"
$P 2>&1 | grep chunk | sed 's/^/full /' >> $O/skiplisted.log
SA_DEBUG_SKIP_LISTED=1 $P 2>&1 | grep chunk | sed 's/^/skip /' >> $O/skiplisted.log
SA_DEBUG_NOCOPY=1 $P 2>&1 | grep chunk | sed 's/^/full-nocopy /' >> $O/skiplisted.log
SA_DEBUG_NOCOPY=1 SA_DEBUG_SKIP_LISTED=1 $P 2>&1 | grep chunk | sed 's/^/skip-nocopy /' >> $O/skiplisted.log
SA_DEBUG_SKIP_LISTED=1 timeout 600 python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('device skip', d['roofline']['kernel_ms'])" >> $O/skiplisted.log 2>&1
