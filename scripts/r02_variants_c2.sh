#!/bin/bash
# C2 / C1 device+e2e per library variant (lib/variants/*.so beside the default)
O=gpurun_out; mkdir -p $O
bash scripts/variants.sh --steps 10 > $O/variants_c2.log 2>&1
bash scripts/variants.sh --steps 20 --config C1 > $O/variants_c1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $O/t_par2.log 2>&1; echo rc=$? >> $O/t_par2.log
