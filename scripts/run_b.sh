set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_b.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py tests/test_boundary.py -x -q -m gpu > gpurun_out/gputest_b.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_b.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
SA_NO_PRUNE_BATCH=1 timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_b_nopb.json 2> gpurun_out/bench_b_nopb.err
timeout 600 python bench.py --config C1 --steps 10 --no-cpu-baseline > gpurun_out/bench_b_C1.json 2> gpurun_out/bench_b_C1.err
