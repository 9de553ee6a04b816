O=gpurun_out
for c in 425984 1048576; do
SA_DEBUG_PIPE=1 SA_CHUNK_READS=$c timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 > $O/pipe_span_$c.log 2>&1
done
