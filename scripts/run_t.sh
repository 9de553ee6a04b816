O=gpurun_out
for v in default stages8 stages10; do
  if [ "$v" = default ]; then L=""; else L="SNAP_B200_LIB=paper_1111_5572_b200/lib/variants/libsnapb200_$v.so"; fi
  echo "== $v" >> $O/e2e_t.log
  env $L SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | tail -2 >> $O/e2e_t.log
  echo "== $v chunk_overflow=0" >> $O/e2e_t.log
  env $L SA_CHUNK_OVERFLOW=0 SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | tail -2 >> $O/e2e_t.log
done
