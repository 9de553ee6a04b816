#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun from the repo root).
#   $1 = tag; $2 = "tests" to run pytest -m gpu first
TAG=${1:-r02a}
O=gpurun_out
mkdir -p $O
nproc > $O/host_$TAG.txt; free -g >> $O/host_$TAG.txt; nvidia-smi -L >> $O/host_$TAG.txt
if [ "$2" = "tests" ]; then
  timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1
  echo "pytest rc=$?" >> $O/gputest_$TAG.log
fi
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
timeout 900 python bench.py --config C1 > $O/bench_${TAG}_C1.json 2> $O/bench_${TAG}_C1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_l_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:seed_kernel|solo_kernel|align_kernel' -c 4 \
    -o $O/prof_c2_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f_$TAG.log 2>&1
