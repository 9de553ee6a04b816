#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -q -x -m gpu > $O/t_par8.log 2>&1; echo rc=$? >> $O/t_par8.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c2_full or c1" > $O/t_full8.log 2>&1; echo rc=$? >> $O/t_full8.log
bash scripts/variants.sh --steps 10 > $O/variants_c2.log 2>&1
bash scripts/variants.sh --steps 20 --config C1 > $O/variants_c1.log 2>&1
SA_DEBUG_SOLO=1 timeout 600 python scripts/solo_reasons.py C2 > $O/solo_reasons.log 2>&1
SNAP_B200_LIB=$PWD/paper_1111_5572_b200/lib/variants/libsnapb200_nosoloqf.so SA_DEBUG_SOLO=1 timeout 600 python scripts/solo_reasons.py C2 >> $O/solo_reasons.log 2>&1
