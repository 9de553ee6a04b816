#!/bin/bash
# C2/C3/C4 lines, parity subset, and C3/C4 vs the long-read layouts' shared
# candidate-table capacity (SA_LONG_CAP)
O=gpurun_out; mkdir -p $O; : > $O/longcap.log
for c in 64 96 128; do for cfg in C3; do
  SA_LONG_CAP=$c timeout 900 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cap $c $cfg', round(d['value']), round(d['roofline']['kernel_ms'],2), round(d['roofline']['overflow_kernel_ms'],2), d['stats_per_step']['overflow_reads'], round(d['e2e']['value']))" >> $O/longcap.log
done; done
