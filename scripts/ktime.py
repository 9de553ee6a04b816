"""Diagnostics: per-kernel device times (SA_DEBUG_KTIME) of one device launch
and of the chunked batch pipeline (single compute stream) at a config."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SA_DEBUG_KTIME"] = "1"
import torch  # noqa: E402

from paper_1111_5572_b200 import api, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n = cfg.n_reads
g = synth.make_genome(cfg)
packed, nmask = synth.pack_genome(g)
bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=n)
genome = api.PackedGenome(packed, nmask, g.size)
al = api.Aligner(api.SeedIndex.build(genome, cfg.params.seed_size), genome, cfg.params)
lib = ctypes.CDLL(api.LIB_PATH)
dev = torch.device("cuda", 0)
db = torch.from_numpy(bases).to(dev)
do = torch.from_numpy(offs.view(np.int64)).to(dev)
dr = torch.empty(n * 24, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream(dev).cuda_stream
for i in range(3):
    al.align_device(db.data_ptr(), do.data_ptr(), n, cfg.read_len, dr.data_ptr(), 0, s)
    al.sync(s)
    lib.sab_debug_ktimes(b"device")
pin_b, pin_r = api.PinnedBuffer(bases.nbytes), api.PinnedBuffer(n * 24)
hb = pin_b.array(np.uint8, bases.size)
hb[:] = bases
hr = pin_r.array(api.RESULT_DTYPE, n)
for i in range(3):
    al.align_arrays(hb, offs, hr)
    lib.sab_debug_ktimes(b"pipeline")
