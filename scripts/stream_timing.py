"""Streamed vs chunked batch path: e2e event time and kernel time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1111_5572_b200 import api, synth
cfg = synth.CONFIGS["C1"]
g = synth.make_genome(cfg)
packed, nmask = synth.pack_genome(g)
bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=1_000_000)
genome = api.PackedGenome(packed, nmask, g.size)
al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
pb, po, pr = api.PinnedBuffer(bases.nbytes), api.PinnedBuffer(offs.nbytes), api.PinnedBuffer(len(offs) * 24)
hb, ho, hr = pb.array(np.uint8, bases.size), po.array(np.uint64, offs.size), pr.array(api.RESULT_DTYPE, offs.size - 1)
hb[:] = bases; ho[:] = offs
for mode in ("stream", "chunked", "stream"):
    if mode == "stream": os.environ["SA_STREAM"] = "1"
    else: os.environ.pop("SA_STREAM", None)
    for _ in range(3): al.align_arrays(hb, ho, hr)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); al.align_arrays(hb, ho, hr); ts.append(time.perf_counter() - t0)
        e, k = al.last_timing()
    print(mode, "wall ms %.3f" % (1000 * np.median(ts)), "event e2e ms %.3f kernel ms %.3f launches %d" % (e, k, al.last_launches()), flush=True)
