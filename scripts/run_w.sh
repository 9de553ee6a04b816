O=gpurun_out
for v in "X=1" "SA_PRUNE_SPLIT=0" "SA_EAGER_PROBES=0" "SA_PRUNE_SPLIT=0 SA_EAGER_PROBES=0" "SA_CHUNK_OVERFLOW=0"; do
  echo "== $v" >> $O/e2e_w.log
  env $v SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | grep -v "seed 0.000" | tail -2 >> $O/e2e_w.log
done
