O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -x -q -m gpu > $O/gputest_n.log 2>&1
echo "rc=$?" >> $O/gputest_n.log
bash scripts/run_variants.sh n C2 default
SA_PRUNE_SPLIT=0 bash scripts/run_variants.sh n C2 default
bash scripts/run_variants.sh n C3 default r01 d682caf 68e918c 3d4b19d
