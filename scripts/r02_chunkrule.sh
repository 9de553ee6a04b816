#!/bin/bash
# chunk-size rule scaled by read length: parity + e2e at C1/C2/C3
O=gpurun_out; mkdir -p $O; : > $O/chunkrule.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c3" > $O/t_c3.log 2>&1; echo rc=$? >> $O/t_c3.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $O/t_par5.log 2>&1; echo rc=$? >> $O/t_par5.log
for c in C1 C2 C3; do
  n=1000000; [ $c = C2 ] && n=10000000; [ $c = C3 ] && n=500000
  timeout 600 python scripts/e2e_probe.py --config $c --reads $n --calls 5 2>&1 | grep chunk | sed "s/^/$c /" >> $O/chunkrule.log
done
