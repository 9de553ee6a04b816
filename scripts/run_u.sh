O=gpurun_out
for c in 262144 524288 1048576 2097152; do
  echo "== chunk $c" >> $O/e2e_u.log
  SA_CHUNK_READS=$c SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | grep -v "seed 0.000" | tail -2 >> $O/e2e_u.log
done
