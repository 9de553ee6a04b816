O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -x -q -m gpu > $O/gputest_p.log 2>&1
echo "rc=$?" >> $O/gputest_p.log
bash scripts/run_variants.sh p "C2 C3 C4 C0 C1" default
