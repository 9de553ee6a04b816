"""Diagnostics: why the solo kernel hands reads to the warp kernel
(SA_DEBUG_SOLO=1 prints the counts), on one device-resident launch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SA_DEBUG_SOLO"] = "1"
import torch  # noqa: E402

from paper_1111_5572_b200 import api, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_reads
g = synth.make_genome(cfg)
packed, nmask = synth.pack_genome(g)
bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=n)
genome = api.PackedGenome(packed, nmask, g.size)
al = api.Aligner(api.SeedIndex.build(genome, cfg.params.seed_size), genome, cfg.params)
dev = torch.device("cuda", 0)
db = torch.from_numpy(bases).to(dev)
do = torch.from_numpy(offs.view(np.int64)).to(dev)
dr = torch.empty(n * 24, dtype=torch.uint8, device=dev)
ds = torch.zeros(20, dtype=torch.int64, device=dev)
s = torch.cuda.current_stream(dev).cuda_stream
al.align_device(db.data_ptr(), do.data_ptr(), n, cfg.read_len, dr.data_ptr(), ds.data_ptr(), s)
al.sync(s)
print(dict(zip(api.STAT_FIELDS, ds.cpu().tolist())))
