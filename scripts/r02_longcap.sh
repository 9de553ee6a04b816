#!/bin/bash
# C2/C3/C4 lines, parity subset, and C3/C4 vs the long-read layouts' shared
# candidate-table capacity (SA_LONG_CAP)
O=gpurun_out; mkdir -p $O; : > $O/longcap.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline > $O/b_c2.json 2>/dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -q -x -m gpu > $O/t_par3.log 2>&1; echo rc=$? >> $O/t_par3.log
for c in 64 128 256; do for cfg in C3 C4; do
  SA_LONG_CAP=$c timeout 900 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cap $c $cfg', round(d['value']), round(d['roofline']['kernel_ms'],2), round(d['roofline']['overflow_kernel_ms'],2), d['stats_per_step']['overflow_reads'], round(d['e2e']['value']))" >> $O/longcap.log
done; done
