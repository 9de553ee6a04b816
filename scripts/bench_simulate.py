"""run_simulate throughput: this library's sa_run_simulate vs the reference's
run_simulate (oracle/_ref), same FASTA, profile and count; the two FASTQ
files are compared byte for byte.  Prints one JSON line.

  python scripts/bench_simulate.py [--genome-bp N] [--reads N] [--read-len L]
"""
import argparse
import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1111_5572_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--genome-bp", type=int, default=20_000_000)
    ap.add_argument("--reads", type=int, default=1_000_000)
    ap.add_argument("--read-len", type=int, default=100)
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    tmp = tempfile.mkdtemp(prefix="simbench")
    fa = os.path.join(tmp, "g.fa")
    seq = np.frombuffer(b"ACGT", np.uint8)[np.random.default_rng(5).integers(0, 4, args.genome_bp)]
    with open(fa, "wb") as f:
        f.write(b">chr1\n")
        for i in range(0, seq.size, 80):
            f.write(seq[i:i + 80].tobytes() + b"\n")
    # the C1-style profile the reference simulator can express
    prof = dict(read_length=args.read_len, snp_rate=0.0009, indel_mutation_rate=0.0001, seq_error_rate=0.015,
                indel_error_fraction=0.07, rng_seed=1001)
    ref_fq, our_fq = os.path.join(tmp, "ref.fq"), os.path.join(tmp, "our.fq")
    t0 = time.perf_counter()
    O.ref_run_simulate(fa, ref_fq, args.reads, **prof)
    t_ref = time.perf_counter() - t0
    t0 = time.perf_counter()
    api.run_simulate(fa, our_fq, args.reads, api.SimProfile(**prof), threads=args.threads)
    t_our = time.perf_counter() - t0

    def digest(p):
        h = hashlib.sha256()
        with open(p, "rb") as f:
            for blk in iter(lambda: f.read(1 << 24), b""):
                h.update(blk)
        return h.hexdigest()

    same = digest(ref_fq) == digest(our_fq)
    print(json.dumps({"what": "run_simulate FASTA -> FASTQ (REF src/driver.cpp:158-168)",
                      "genome_bp": args.genome_bp, "reads": args.reads, "read_len": args.read_len,
                      "profile": prof, "reference_s": round(t_ref, 3), "ours_s": round(t_our, 3),
                      "reference_reads_per_s": round(args.reads / t_ref), "ours_reads_per_s": round(args.reads / t_our),
                      "speedup": round(t_ref / t_our, 2), "byte_identical": same,
                      "host_threads": args.threads or os.cpu_count(), "fastq_bytes": os.path.getsize(our_fq)}))
    for p in (fa, ref_fq, our_fq):
        os.remove(p)


if __name__ == "__main__":
    main()
