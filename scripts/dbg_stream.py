import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1111_5572_b200 import api, synth
cfg = synth.CONFIGS["C1"].scaled(genome_len=2_000_000, n_reads=int(sys.argv[1]) if len(sys.argv) > 1 else 100_000)
g = synth.make_genome(cfg)
packed, nmask = synth.pack_genome(g)
bases, offs, _, _ = synth.make_reads(cfg, g)
genome = api.PackedGenome(packed, nmask, g.size)
idx = api.SeedIndex.build(genome, 20)
al = api.Aligner(idx, genome, cfg.params)
for it in range(3):
    try:
        r = al.align_arrays(bases, offs)
        print("ok", it, r["kind"][:5], al.last_timing(), flush=True)
    except Exception as e:
        print("ERR", it, type(e).__name__, e, flush=True)
