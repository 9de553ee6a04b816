"""LV work rates per config: dp_cells (LV cells touched: wavefront slide
steps, or 64 per bit-parallel word step) per second of the step's kernels, on
one device-resident launch.  python scripts/lv_rates.py C2 C3 C4"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1111_5572_b200 import api, synth  # noqa: E402

for name in sys.argv[1:] or ["C2", "C3", "C4"]:
    cfg = synth.CONFIGS[name]
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, cfg.params.seed_size), genome, cfg.params)
    n = offs.size - 1
    dev = torch.device("cuda", 0)
    db = torch.from_numpy(bases).to(dev)
    do = torch.from_numpy(offs.view(np.int64)).to(dev)
    dr = torch.empty(n * 24, dtype=torch.uint8, device=dev)
    ds = torch.zeros(20, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    for _ in range(2):
        al.align_device(db.data_ptr(), do.data_ptr(), n, cfg.read_len, dr.data_ptr(), 0, s)
    al.sync(s)
    ds.zero_()
    al.align_device(db.data_ptr(), do.data_ptr(), n, cfg.read_len, dr.data_ptr(), ds.data_ptr(), s)
    al.sync(s)
    f, sl = al.last_kernel_times()
    st = dict(zip(api.STAT_FIELDS, ds.cpu().tolist()))
    ms = f + sl
    print(f"{name}: {n} reads, kernels {ms:.2f} ms, distance_calls {st['distance_calls']}, dp_cells {st['dp_cells']}, "
          f"{st['dp_cells'] / ms / 1e6:.2f} G cells/s, {st['distance_calls'] / ms / 1e3:.1f} M LV calls/s", flush=True)
    del al, db, do, dr
