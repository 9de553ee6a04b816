O=gpurun_out
echo "== nocopy (results garbage beyond stage 6: timing only)" >> $O/e2e_v.log
SA_DEBUG_NOCOPY=1 SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | grep -v "seed 0.000" | tail -2 >> $O/e2e_v.log
echo "== normal" >> $O/e2e_v.log
SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | grep -v "seed 0.000" | tail -2 >> $O/e2e_v.log
