#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun from the repo root):
#   r02_evidence.sh TAG [tests]
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nproc > $O/host_$TAG.txt; free -g >> $O/host_$TAG.txt; nvidia-smi -L >> $O/host_$TAG.txt
if [ "$2" = "tests" ]; then
  timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1
  echo "pytest rc=$?" >> $O/gputest_$TAG.log
  python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1
fi
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
for c in C1 C0 C3 C4; do
  timeout 900 python bench.py --config $c --steps 5 > $O/bench_${TAG}_$c.json 2> $O/bench_${TAG}_$c.err
done
timeout 900 python bench.py --box --box-devices 0,0 --steps 5 > $O/bench_${TAG}_box00.json 2> $O/bench_${TAG}_box00.err
K='regex:seed_kernel|solo_kernel|resolve_kernel|align_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 10 --csv --log-file $O/launches_${TAG}_C2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_l_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 10 --csv --log-file $O/launches_${TAG}_C1.csv \
    python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_l1_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k "$K" -c 5 \
    -o $O/prof_${TAG}_C2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k "$K" -c 5 \
    -o $O/prof_${TAG}_C1 -f python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f1_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:align_kernel' -c 1 \
    -o $O/prof_${TAG}_C4 -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f4_$TAG.log 2>&1
