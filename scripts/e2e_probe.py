"""e2e probe (default C1, --config C2 ...): sa_align_batch wall time per call from pinned buffers,
beside the plain H2D of the same bytes (the copy floor).  Run with
SA_DEBUG_PIPE=1 for the pipeline's span lines, SA_CHUNK_READS=n to force
the chunk size.

  python scripts/e2e_probe.py [--reads N] [--calls K]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reads", type=int, default=1_000_000)
    ap.add_argument("--calls", type=int, default=8)
    ap.add_argument("--copy-floor", action="store_true")
    ap.add_argument("--config", default="C1")
    ap.add_argument("--pageable", action="store_true", help="time the call from ordinary (pageable) numpy buffers")
    args = ap.parse_args()
    import torch

    from paper_1111_5572_b200 import api, synth

    cfg = synth.CONFIGS[args.config]
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=args.reads)
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, cfg.params.seed_size), genome, cfg.params)
    pin_b, pin_o, pin_r = api.PinnedBuffer(bases.nbytes), api.PinnedBuffer(offs.nbytes), api.PinnedBuffer(args.reads * 24)
    hb, ho = pin_b.array(np.uint8, bases.size), pin_o.array(np.uint64, offs.size)
    hr = pin_r.array(api.RESULT_DTYPE, args.reads)
    hb[:] = bases
    ho[:] = offs
    if args.pageable:
        hb, ho, hr = bases, offs, np.zeros(args.reads, api.RESULT_DTYPE)
    for _ in range(3):
        al.align_arrays(hb, ho, hr)
    ms = []
    for _ in range(args.calls):
        t0 = time.perf_counter()
        al.align_arrays(hb, ho, hr)
        ms.append(1000 * (time.perf_counter() - t0))
    ms.sort()
    print(f"{'pageable ' if args.pageable else ''}chunk={os.environ.get('SA_CHUNK_READS', 'auto')} e2e ms min {ms[0]:.3f} median {ms[len(ms)//2]:.3f} "
          f"-> {args.reads / ms[len(ms)//2] / 1e3:.1f} M reads/s; event span {al.last_timing()[0]:.3f} ms", flush=True)
    if args.copy_floor:
        x = torch.from_numpy(hb)  # pinned
        y = torch.empty(x.numel(), dtype=torch.uint8, device="cuda")
        for chunk in (48_000 * 100, 4_800_000 * 2, x.numel()):
            best = 1e9
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for o in range(0, x.numel(), chunk):
                    y[o:o + chunk].copy_(x[o:o + chunk], non_blocking=True)
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(f"H2D {x.numel() / 1e6:.0f} MB in {chunk / 1e6:.1f} MB copies: {best:.3f} ms = "
                  f"{x.numel() / best / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
