#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline > $O/b_c4g.json 2> $O/b_c4g.err
SA_NO_GPLANES=1 timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline > $O/b_c4ng.json 2> $O/b_c4ng.err
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c4" > $O/t_c4g.log 2>&1; echo rc=$? >> $O/t_c4g.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -q -x -m gpu > $O/t_par.log 2>&1; echo rc=$? >> $O/t_par.log
SA_SOLO_DYN=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 > $O/e2e_solodyn.log 2>&1
SA_SOLO_DYN=1 SA_DEBUG_NOCOPY=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 >> $O/e2e_solodyn.log 2>&1
