"""Do host<->device copies slow the kernels down?  Device-resident
seed + align over 1 M C1 reads, timed with CUDA events, alone and while
another stream streams H2D (and D2H) copies in a loop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1111_5572_b200 import api, synth

cfg = synth.CONFIGS["C1"]
g = synth.make_genome(cfg)
packed, nmask = synth.pack_genome(g)
bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=1_000_000)
genome = api.PackedGenome(packed, nmask, g.size)
al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
db = torch.from_numpy(bases).cuda()
do = torch.from_numpy(offs.view(np.int64)).cuda()
dr = torch.empty(len(offs) * 24, dtype=torch.uint8, device="cuda")
ds = torch.zeros(20, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
x = torch.empty(216_000_000, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
rh = torch.empty(48_000_000, dtype=torch.uint8).pin_memory()
r = torch.empty(48_000_000, dtype=torch.uint8, device="cuda")
cs = torch.cuda.Stream()
cs2 = torch.cuda.Stream()


def kern(n=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        al.align_device(db.data_ptr(), do.data_ptr(), 1_000_000, 100, dr.data_ptr(), ds.data_ptr(), st.cuda_stream)
    e1.record(st)
    return e0, e1, n


def done(t):
    e0, e1, n = t
    e1.synchronize()
    return e0.elapsed_time(e1) / n


for _ in range(3):
    done(kern())
print("kernels alone          %.3f ms / 1M reads" % done(kern()))
for mode in ("h2d", "h2d+d2h"):
    torch.cuda.synchronize()
    with torch.cuda.stream(cs):
        for i in range(20):
            y.copy_(x, non_blocking=True)
    if mode == "h2d+d2h":
        with torch.cuda.stream(cs2):
            for i in range(60):
                rh.copy_(r, non_blocking=True)
    t = kern(5)
    print(f"kernels during {mode:8s} %.3f ms / 1M reads" % done(t))
    torch.cuda.synchronize()

# the same 1 M reads as device-resident calls of one chunk each
for cr in (16_384, 65_536, 110_000, 250_000, 1_000_000):
    def chunked():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for r0 in range(0, 1_000_000, cr):
            n = min(cr, 1_000_000 - r0)
            al.align_device(db.data_ptr(), do.data_ptr() + 8 * r0, n, 100, dr.data_ptr() + 24 * r0, ds.data_ptr(),
                            st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1)
    chunked()
    print(f"chunks of {cr:8d} reads: %.3f ms / 1M reads" % min(chunked() for _ in range(3)))
