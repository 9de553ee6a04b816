"""FASTQ -> SAM end to end: sa_run_align against the
reference's own run_align (REF src/driver.cpp:47-156) on the same index file
and FASTQ, both produced by the reference (run_index, run_simulate).

Bar: with stable order the SAM files are byte-identical; the metrics report
matches line for line except wall-clock fields and dp_cells (implementation-
specific); every error keeps the reference's class and
message.  Reads come from the reference's ReadSimulator, so names carry the
truth and the correct/wrong counts are compared too.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1111_5572_b200 import api, synth

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

VOLATILE = ("elapsed_sec", "reads_per_sec", "dp_cells")


def _fasta(tmp_path, contigs):
    p = tmp_path / "ref.fa"
    with open(p, "w") as f:
        for name, seq in contigs:
            f.write(f">{name} synthetic\n")
            for i in range(0, len(seq), 70):
                f.write(seq[i:i + 70] + "\n")
    return str(p)


@pytest.fixture(scope="module")
def corpus(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("ra")
    cfg = synth.CONFIGS["C1"].scaled(genome_len=2_000_000)
    g = synth.make_genome(cfg).tobytes().decode()
    g = g[:700_000] + "N" * 300 + g[700_300:]
    fa = _fasta(tmp, [("chr1", g[:1_200_000]), ("chr_2_x", g[1_200_000:1_900_000]), ("chrM", g[1_900_000:])])
    idx = str(tmp / "ref.idx")
    assert O.ref_run_index(fa, idx, 20) == 0
    fq = str(tmp / "reads.fq")
    O.ref_run_simulate(fa, fq, 30_000, read_length=100, seq_error_rate=0.02, indel_error_fraction=0.1,
                       rng_seed=7)
    params = api.AlignerParams(seed_size=20, seeds_to_try=10, max_distance=10, confidence_threshold=2,
                               max_hits=300, bucket_size=32)
    return dict(tmp=tmp, fa=fa, idx=idx, fq=fq, params=params)


def _report_lines(text):
    return {k: v for k, v in (ln.split("=", 1) for ln in text.strip().splitlines()) if k not in VOLATILE}


def _run_both(c, name, threads=4, chunk_min=1 << 20, stable=True, fq=None, params=None):
    fq = fq or c["fq"]
    params = params or c["params"]
    ref_sam = str(c["tmp"] / f"{name}.ref.sam")
    our_sam = str(c["tmp"] / f"{name}.our.sam")
    our_rep = str(c["tmp"] / f"{name}.our.txt")
    ref_text = O.ref_run_align(c["idx"], fq, ref_sam, params, threads=threads, chunk_min=chunk_min, stable=stable,
                               command_line="seedaln align test")
    rep = api.run_align(c["idx"], fq, our_sam, params, threads=threads, chunk_min_bytes=chunk_min,
                        stable_order=stable, report_path=our_rep, command_line="seedaln align test")
    return ref_sam, our_sam, ref_text, rep, our_rep


def test_sam_byte_identical_and_report(corpus):
    ref_sam, our_sam, ref_text, rep, our_rep = _run_both(corpus, "a")
    assert open(our_sam, "rb").read() == open(ref_sam, "rb").read()
    assert _report_lines(rep.to_text()) == _report_lines(ref_text)
    assert open(our_rep).read() == rep.to_text()
    assert rep.total == 30_000 and rep.correct > 0.95 * rep.total


@pytest.mark.parametrize("threads,chunk_min", [(1, 4 << 20), (3, 4096), (16, 1000)])
def test_thread_and_chunk_invariance(corpus, threads, chunk_min):
    # REF tests/test_driver.cpp:160-193: output independent of threads/chunking
    ref_sam, our_sam, ref_text, rep, _ = _run_both(corpus, f"t{threads}", threads=threads, chunk_min=chunk_min)
    assert open(our_sam, "rb").read() == open(ref_sam, "rb").read()
    assert _report_lines(rep.to_text()) == _report_lines(ref_text)


def test_unstable_order_same_records(corpus):
    ref_sam, our_sam, _, _, _ = _run_both(corpus, "u", threads=8, chunk_min=4096, stable=False)
    a = open(ref_sam).read().splitlines()
    b = open(our_sam).read().splitlines()
    assert a[:5] == b[:5]  # header
    assert sorted(a) == sorted(b)


def test_crlf_lowercase_iupac_and_short_reads(corpus):
    # hand-made FASTQ: CRLF endings, lowercase / IUPAC bases, a read shorter
    # than s, an empty read, '+name' separators, no trailing newline
    g = api.PackedGenome.from_fasta(corpus["fa"])
    seq = g.substring(5000, 300)
    recs = [("r1", seq[:100].lower(), "I" * 100), ("r2", seq[50:150].replace("A", "R", 3), "#" * 100),
            ("short", seq[:12], "I" * 12), ("empty", "", ""), ("chr1_5001_F_9", seq[:100], "5" * 100)]
    text = "".join(f"@{n} extra\r\n{s}\r\n+{n}\r\n{q}\r\n" for n, s, q in recs).rstrip("\r\n")
    fq = str(corpus["tmp"] / "odd.fq")
    open(fq, "w", newline="").write(text)
    ref_sam, our_sam, ref_text, rep, _ = _run_both(corpus, "odd", threads=2, fq=fq)
    assert open(our_sam, "rb").read() == open(ref_sam, "rb").read()
    assert _report_lines(rep.to_text()) == _report_lines(ref_text)


@pytest.mark.parametrize("text", [
    "not a fastq\n",                                  # does not start with a FASTQ record
    "@r1\nACGT\n+\nIIII\nr2\nACGT\n+\nIIII\n",        # record without '@'
    "@r1\nACGT\n+\nIIII\n@\nACGT\n+\nIIII\n",         # empty name
    "@r1\nACGT\n+\nIIII\n@r2\nACGT\n",                # truncated
    "@r1\nACGT\n+\nIIII\n@r2\nACGT\nx\nIIII\n",       # missing '+'
    "@r1\nACGT\n+\nIIII\n@r2\nACGT\n+\nIII\n",        # length mismatch
    "@r1\nACGT\n+\nIIII\n@r2\nAC-T\n+\nIIII\n",       # illegal base
])
def test_fastq_errors_match_reference(corpus, text):
    fq = str(corpus["tmp"] / "bad.fq")
    open(fq, "w").write(text)
    with pytest.raises(O.RefError) as re_:
        O.ref_run_align(corpus["idx"], fq, str(corpus["tmp"] / "x.sam"), corpus["params"], threads=1)
    with pytest.raises(api.ParseError) as oe:
        api.run_align(corpus["idx"], fq, str(corpus["tmp"] / "y.sam"), corpus["params"], threads=1)
    assert re_.value.code == api.SA_EPARSE and str(oe.value) == re_.value.msg


def test_seed_size_mismatch_and_missing_files(corpus):
    p = api.AlignerParams(**{**corpus["params"].__dict__, "seed_size": 16})
    with pytest.raises(O.RefError) as re_:
        O.ref_run_align(corpus["idx"], corpus["fq"], str(corpus["tmp"] / "x.sam"), p)
    with pytest.raises(api.FormatError) as oe:
        api.run_align(corpus["idx"], corpus["fq"], str(corpus["tmp"] / "y.sam"), p)
    assert str(oe.value) == re_.value.msg
    with pytest.raises(api.IoError, match="cannot open"):
        api.run_align(str(corpus["tmp"] / "none.idx"), corpus["fq"], str(corpus["tmp"] / "y.sam"))
    with pytest.raises(api.IoError, match="cannot stat"):
        api.run_align(corpus["idx"], str(corpus["tmp"] / "none.fq"), str(corpus["tmp"] / "y.sam"),
                      corpus["params"])
    bad = api.AlignerParams(**{**corpus["params"].__dict__, "seeds_to_try": 0})
    with pytest.raises(ValueError):
        api.run_align(corpus["idx"], corpus["fq"], str(corpus["tmp"] / "y.sam"), bad)


def test_run_index_then_align(corpus):
    # our GPU run_index output drives both aligners identically
    idx = str(corpus["tmp"] / "ours.idx")
    api.run_index(corpus["fa"], idx, 20)
    assert open(idx, "rb").read() == open(corpus["idx"], "rb").read()
    gidx = str(corpus["tmp"] / "ours.gpuidx")
    api.run_index(corpus["fa"], gidx, 20, fmt=api.SA_INDEX_SNAPGPU1)
    a = str(corpus["tmp"] / "g1.sam")
    b = str(corpus["tmp"] / "g2.sam")
    api.run_align(idx, corpus["fq"], a, corpus["params"], threads=4, stable_order=True)
    api.run_align(gidx, corpus["fq"], b, corpus["params"], threads=4, stable_order=True)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert os.path.getsize(gidx) < os.path.getsize(idx) / 10
