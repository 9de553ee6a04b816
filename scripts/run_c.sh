# tests (parity subset), C2 bench, ncu full capture of the C2 device step's kernels
TAG=${1:-c}
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py tests/test_boundary.py -x -q -m gpu > $O/gputest_$TAG.log 2>&1
echo "rc=$?" >> $O/gputest_$TAG.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:seed_kernel|solo_kernel|resolve_kernel|prune_kernel|align_kernel' -c 6 \
    -o $O/prof_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_$TAG.log 2>&1
