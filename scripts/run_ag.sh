O=gpurun_out
for g in 888 1776 3552 100000; do
  echo "== solo grid cap $g" >> $O/e2e_ag.log
  SA_SOLO_GRID=$g SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | grep -v "seed 0.000" | tail -2 >> $O/e2e_ag.log
  SA_SOLO_GRID=$g SA_PIPE_SINGLE=1 SA_DEBUG_NOCOPY=1 SA_DEBUG_PIPE=1 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 3 2>&1 | grep "seed" | tail -1 >> $O/e2e_ag.log
done
