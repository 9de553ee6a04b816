#!/bin/bash
# Quick state check on one B200: GPU tests, smoke, bench C2 and C4.
TAG=${1:-r02q}
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/host_$TAG.txt
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1
echo "pytest rc=$?" >> $O/gputest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1
timeout 900 python bench.py --steps 10 > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline > $O/bench_${TAG}_C4.json 2> $O/bench_${TAG}_C4.err
timeout 900 python bench.py --config C3 --steps 3 --no-cpu-baseline > $O/bench_${TAG}_C3.json 2> $O/bench_${TAG}_C3.err
