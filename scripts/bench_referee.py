#!/usr/bin/env python
"""GPU referee at C1 scale, ours vs the reference's CPU
oracle_align (REF src/eval.cpp:270-306), plus criterion-1-style agreement of
the aligner with the referee (REF tests/acceptance/acceptance_main.cpp:194-289).

Synthetic C1 inputs (100 Mbp genome, seed 2; C1 reads).  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (test infrastructure: the reference arm)
from paper_1111_5572_b200 import api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--reads", type=int, default=100_000)
    ap.add_argument("--ref-reads", type=int, default=2_000)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=args.reads)
    genome = api.PackedGenome(packed, nmask, g.size)
    line = {"workload": f"{cfg.name}: {g.size} bp genome, {args.reads} reads of {cfg.read_len} bp"}
    t0 = time.perf_counter()
    rf = api.Referee(genome)
    line["ours_context_s"] = time.perf_counter() - t0
    rf.align_arrays(cfg.params, bases[:int(offs[1000])], offs[:1001])  # warm-up
    t0 = time.perf_counter()
    got = rf.align_arrays(cfg.params, bases, offs)
    dt = time.perf_counter() - t0
    line["ours_reads_per_s"] = args.reads / dt
    line["ours_seconds"] = dt

    t0 = time.perf_counter()
    ref = O.RefReferee(packed, nmask, g.size)
    line["reference_context_s"] = time.perf_counter() - t0
    n = args.ref_reads
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    want = ref.align(cfg.params, bases[:int(offs[n])], offs[:n + 1], threads=cores)
    dt = time.perf_counter() - t0
    line["reference_reads_per_s"] = n / dt
    line["reference_threads"] = cores
    line["reference_sample_reads"] = n
    line["parity_mismatches_on_sample"] = len(O.compare_results(got[:n], want))

    # criterion-1 style: the aligner against the referee on every read
    al = api.Aligner(api.SeedIndex.build(genome, cfg.params.seed_size), genome, cfg.params)
    res = al.align_arrays(bases, offs)
    same_kind = (res["kind"] == got["kind"])
    single = (res["kind"] == 0) & (got["kind"] == 0)
    same_pos = single & (res["position"] == got["position"]) & (res["direction"] == got["direction"])
    line["aligner_vs_referee"] = {"kind_agreement": float(same_kind.mean()),
                                  "single_single_same_locus": float(same_pos.sum() / max(1, single.sum())),
                                  "referee_single": int((got["kind"] == 0).sum()),
                                  "aligner_single": int((res["kind"] == 0).sum())}
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(line, f, indent=1)


if __name__ == "__main__":
    main()
