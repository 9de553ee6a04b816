"""H2D bandwidth alone vs with the align kernel running (device path) concurrently."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
x = torch.empty(108_000_000, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
s = torch.cuda.Stream()
def h2d(chunks):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        n = x.numel() // chunks
        for i in range(chunks):
            y[i*n:(i+1)*n].copy_(x[i*n:(i+1)*n], non_blocking=True)
        e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1)
for c in (1, 8, 64):
    h2d(c); print("H2D alone chunks", c, "ms %.3f" % h2d(c))
# concurrent: a busy kernel on the default stream
from paper_1111_5572_b200 import api, synth
import numpy as np
cfg = synth.CONFIGS["C1"]
g = synth.make_genome(cfg); packed, nmask = synth.pack_genome(g)
bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=1_000_000)
genome = api.PackedGenome(packed, nmask, g.size)
al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
db = torch.from_numpy(bases).cuda(); do = torch.from_numpy(offs.view(np.int64)).cuda()
dr = torch.empty(len(offs) * 24, dtype=torch.uint8, device="cuda"); ds = torch.zeros(20, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for c in (1, 8):
    al.align_device(db.data_ptr(), do.data_ptr(), 1_000_000, 100, dr.data_ptr(), ds.data_ptr(), st.cuda_stream)
    t = h2d(c)
    torch.cuda.synchronize()
    print("H2D with align kernel running, chunks", c, "ms %.3f" % t)
