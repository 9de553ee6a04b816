#!/bin/bash
# Re-entry check on one B200: GPU suite, smoke, C2 bench line, then the C2
# launch list and --set full captures of every hot kernel (r02_ncu_c2.sh).
TAG=${1:-r02y}
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/gputest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
bash scripts/r02_ncu_c2.sh $TAG
