#!/usr/bin/env python
"""File-level timings at C1 scale, ours vs the reference:

  index:  FASTA -> SNAPIDX1  (sa_run_index, GPU CSR)   vs reference run_index
  align:  index + FASTQ -> SAM (sa_run_align, GPU)     vs reference run_align
          (same threads, stable order; SAM files compared byte for byte)

Synthetic inputs: the C1 genome (100 Mbp, seed 2) as a 4-contig FASTA, and
C1 reads written as FASTQ with truth-encoded names ("chrN_pos1_F|R_serial",
REF src/simulator.cpp:44-48).  Prints one JSON line; --out also writes it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (test infrastructure: the reference arm)
from paper_1111_5572_b200 import api, synth  # noqa: E402


def write_fasta(path, g: np.ndarray, n_contigs: int):
    cuts = np.linspace(0, g.size, n_contigs + 1).astype(int)
    with open(path, "wb") as f:
        for i in range(n_contigs):
            f.write(f">chr{i + 1}\n".encode())
            seg = g[cuts[i]:cuts[i + 1]]
            for j in range(0, seg.size, 80):
                f.write(seg[j:j + 80].tobytes() + b"\n")
    return [(f"chr{i + 1}", int(cuts[i])) for i in range(n_contigs)]


def write_fastq(path, bases, offs, tpos, tdir, contigs):
    starts = np.array([c[1] for c in contigs])
    with open(path, "wb") as f:
        buf = []
        for i in range(offs.size - 1):
            p = int(tpos[i])
            ci = int(np.searchsorted(starts, p, side="right") - 1)
            name = f"{contigs[ci][0]}_{p - contigs[ci][1] + 1}_{'R' if tdir[i] else 'F'}_{i}"
            s = bases[int(offs[i]):int(offs[i + 1])].tobytes()
            buf.append(b"@" + name.encode() + b"\n" + s + b"\n+\n" + b"I" * len(s) + b"\n")
            if len(buf) >= 100_000:
                f.write(b"".join(buf))
                buf = []
        f.write(b"".join(buf))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reads", type=int, default=1_000_000)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--ref-reads", type=int, default=400_000, help="reads for the reference run_align")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = synth.CONFIGS["C1"]
    tmp = tempfile.mkdtemp(prefix="snapfiles_")
    g = synth.make_genome(cfg)
    fa = os.path.join(tmp, "c1.fa")
    contigs = write_fasta(fa, g, 4)
    bases, offs, tpos, tdir = synth.make_reads(cfg, g, n_reads=args.reads)
    fq = os.path.join(tmp, "c1.fq")
    write_fastq(fq, bases, offs, tpos, tdir, contigs)
    fq_ref = os.path.join(tmp, "c1_ref.fq")
    write_fastq(fq_ref, bases[:int(offs[args.ref_reads])], offs[:args.ref_reads + 1], tpos, tdir, contigs)
    line = {"workload": f"C1 genome as 4-contig FASTA ({g.size} bp); {args.reads} x {cfg.read_len} bp FASTQ "
                        f"({os.path.getsize(fq) / 1e6:.0f} MB)", "threads": args.threads}

    idx = os.path.join(tmp, "ours.idx")
    t0 = time.perf_counter()
    api.run_index(fa, idx, 20)
    line["index_ours_s"] = time.perf_counter() - t0
    ref_idx = os.path.join(tmp, "ref.idx")
    t0 = time.perf_counter()
    assert O.ref_run_index(fa, ref_idx, 20) == 0
    line["index_reference_s"] = time.perf_counter() - t0
    line["index_files_identical"] = open(idx, "rb").read() == open(ref_idx, "rb").read()
    gidx = os.path.join(tmp, "ours.gpuidx")
    api.run_index(fa, gidx, 20, fmt=api.SA_INDEX_SNAPGPU1)
    line["index_bytes"] = {"snapidx1": os.path.getsize(idx), "snapgpu1": os.path.getsize(gidx)}

    p = cfg.params
    for name, path in (("snapidx1", idx), ("snapgpu1", gidx)):
        sam = os.path.join(tmp, f"ours_{name}.sam")
        t0 = time.perf_counter()
        rep = api.run_align(path, fq, sam, p, threads=args.threads, stable_order=True,
                            verify_index=(name == "snapidx1"))
        dt = time.perf_counter() - t0
        line[f"align_ours_{name}"] = {"seconds": dt, "reads_per_s_align_phase": args.reads / rep.elapsed_seconds,
                                      "single": rep.single, "correct": rep.correct, "wrong": rep.wrong,
                                      "report_elapsed_s": rep.elapsed_seconds}
    # reference on a prefix of the same FASTQ (its own run_align, all threads)
    sam_ref = os.path.join(tmp, "ref.sam")
    t0 = time.perf_counter()
    txt = O.ref_run_align(ref_idx, fq_ref, sam_ref, p, threads=args.threads, stable=True)
    dt = time.perf_counter() - t0
    el = float(dict(ln.split("=", 1) for ln in txt.strip().splitlines())["elapsed_sec"])
    line["align_reference"] = {"seconds": dt, "reads": args.ref_reads, "report_elapsed_s": el,
                               "reads_per_s_align_phase": args.ref_reads / el,
                               "note": "seconds = process wall incl. index load; report_elapsed_s = workers only"}
    sam_ours_prefix = os.path.join(tmp, "ours_prefix.sam")
    api.run_align(idx, fq_ref, sam_ours_prefix, p, threads=args.threads, stable_order=True)
    line["sam_identical_on_reference_sample"] = open(sam_ref, "rb").read() == open(sam_ours_prefix, "rb").read()
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(line, f, indent=1)
    subprocess.run(["rm", "-rf", tmp])


if __name__ == "__main__":
    main()
