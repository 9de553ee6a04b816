"""Read simulator parity: sa_simulator_* / sa_run_simulate against the
reference's own ReadSimulator and run_simulate (REF src/simulator.cpp:90-206,
src/driver.cpp:158-168), compiled from /root/reference into oracle/_ref.

Host code only (the simulator is one sequential mt19937_64 stream), so these
run without a GPU.  Parity bar: the FASTQ files are byte-identical, which
covers every read's bases, name (truth) and order.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1111_5572_b200 import api

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference library (oracle/_ref) not built")


def _fasta(tmp, contigs, name="g.fa"):
    p = tmp / name
    with open(p, "w") as f:
        for nm, seq in contigs:
            f.write(f">{nm} description\n")
            for i in range(0, len(seq), 61):
                f.write(seq[i:i + 61] + "\n")
    return str(p)


def _seq(n, seed):
    return np.frombuffer(b"ACGT", np.uint8)[np.random.default_rng(seed).integers(0, 4, n)].tobytes().decode()


@pytest.fixture(scope="module")
def genomes(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("sim")
    a = _seq(400_000, 11)
    # N runs inside contigs, a contig shorter than most read lengths, an empty
    # contig, and a last contig whose windows are truncated by the genome end
    multi = [("chr1", a[:150_000] + "N" * 500 + a[150_000:200_000]),
             ("short", a[200_000:200_040]),
             ("empty", ""),
             ("chr_2_x", a[200_040:260_000] + "NNNNNNNNNN" + a[260_000:300_000]),
             ("tail", a[300_000:300_600])]
    return dict(tmp=tmp, plain=_fasta(tmp, [("chr1", a)], "plain.fa"), multi=_fasta(tmp, multi, "multi.fa"),
                nheavy=_fasta(tmp, [("n", ("N" * 97 + "ACG") * 300)], "nheavy.fa"),
                allN=_fasta(tmp, [("n", "N" * 5000)], "alln.fa"))


PROFILES = [
    dict(),  # SimProfile{} defaults
    dict(read_length=100, snp_rate=0.0, indel_mutation_rate=0.0, seq_error_rate=0.01, indel_error_fraction=0.0,
         rng_seed=1001),  # the C0 profile
    dict(read_length=150, snp_rate=0.05, indel_mutation_rate=0.03, seq_error_rate=0.04, indel_error_fraction=0.3,
         rng_seed=7),
    dict(read_length=36, snp_rate=0.3, indel_mutation_rate=0.3, seq_error_rate=0.5, indel_error_fraction=0.5,
         rng_seed=123456789),
    dict(read_length=1, seq_error_rate=1.0, indel_error_fraction=1.0, rng_seed=3),
    dict(read_length=1000, snp_rate=0.01, indel_mutation_rate=0.005, seq_error_rate=0.05,
         indel_error_fraction=0.4, rng_seed=2 ** 63 + 5),
    dict(read_length=120, snp_rate=1.0, indel_mutation_rate=0.0, seq_error_rate=0.0, rng_seed=9),
    dict(read_length=80, snp_rate=0.0, indel_mutation_rate=1.0, seq_error_rate=0.0, rng_seed=10),
]


def _both(g, fa, count, prof, name, threads=0):
    ref = str(g["tmp"] / f"{name}.ref.fq")
    our = str(g["tmp"] / f"{name}.our.fq")
    O.ref_run_simulate(fa, ref, count, **prof)
    api.run_simulate(fa, our, count, api.SimProfile(**prof), threads=threads)
    return open(ref, "rb").read(), open(our, "rb").read()


@pytest.mark.parametrize("k", range(len(PROFILES)))
@pytest.mark.parametrize("which", ["plain", "multi"])
def test_run_simulate_byte_identical(genomes, which, k):
    prof = PROFILES[k]
    if which == "multi" and prof.get("read_length", 100) > 600:
        prof = dict(prof, read_length=590)  # still fits chr1 / chr_2_x / tail
    n = 300 if prof.get("read_length", 100) >= 590 else 3000
    ref, our = _both(genomes, genomes[which], n, prof, f"{which}{k}")
    assert our.count(b"\n") == 4 * n
    assert our == ref


def test_n_heavy_genome_redraws(genomes):
    # 97 of every 100 bases are N: most loci are redrawn (REF simulator.cpp:131-133, 183-185)
    ref, our = _both(genomes, genomes["nheavy"], 200, dict(read_length=3, seq_error_rate=0.2, rng_seed=4), "nh")
    assert our == ref


def test_thread_count_invariance(genomes):
    prof = dict(read_length=100, seq_error_rate=0.03, indel_error_fraction=0.2, rng_seed=77)
    outs = []
    for t in (1, 3, 16):
        p = str(genomes["tmp"] / f"t{t}.fq")
        api.run_simulate(genomes["multi"], p, 5000, api.SimProfile(**prof), threads=t)
        outs.append(open(p, "rb").read())
    assert outs[0] == outs[1] == outs[2]


def test_simulator_stream_matches_file(genomes):
    """ReadSimulator::next in batches of any size is the same stream the file holds."""
    prof = dict(read_length=50, snp_rate=0.01, seq_error_rate=0.05, indel_error_fraction=0.2, rng_seed=21)
    ref = str(genomes["tmp"] / "stream.ref.fq")
    O.ref_run_simulate(genomes["multi"], ref, 1000, **prof)
    lines = open(ref).read().splitlines()
    sim = api.ReadSimulator(api.PackedGenome.from_fasta(genomes["multi"]), api.SimProfile(**prof))
    got = []
    for n in (1, 7, 92, 400, 500):
        bases, truth = sim.next_batch(n)
        for i in range(n):
            tr = sim.truth_of(truth[i])
            got.append((api.encode_truth(tr), bases[i].tobytes().decode()))
    assert len(got) == 1000
    for i, (name, b) in enumerate(got):
        assert lines[4 * i] == "@" + name
        assert lines[4 * i + 1] == b
        assert lines[4 * i + 3] == "I" * 50
    # truths: serials in order, positions inside the named contig
    contigs = {c[0]: c for c in api.PackedGenome.from_fasta(genomes["multi"]).contigs()}
    for i, (name, _) in enumerate(got):
        c, pos1, d, ser = name.rsplit("_", 3)
        assert int(ser) == i and d in "FR" and 1 <= int(pos1) <= contigs[c][2] - 50 + 1


def test_errors_match_reference(genomes, tmp_path):
    fa = genomes["plain"]
    out = str(tmp_path / "x.fq")
    cases = [
        (fa, out, 0, dict(), ValueError),
        (fa, out, 5, dict(read_length=0), ValueError),
        (fa, out, 5, dict(snp_rate=-0.1), ValueError),
        (fa, out, 5, dict(indel_mutation_rate=1.5), ValueError),
        (fa, out, 5, dict(seq_error_rate=float("nan")), ValueError),
        (fa, out, 5, dict(indel_error_fraction=2.0), ValueError),
        (fa, out, 5, dict(read_length=400_001), ValueError),  # no contig long enough
        (str(tmp_path / "missing.fa"), out, 5, dict(), api.IoError),
        (fa, str(tmp_path / "no" / "dir.fq"), 5, dict(), api.IoError),
        (genomes["allN"], out, 5, dict(read_length=10), RuntimeError),  # failed to place a read
    ]
    for fasta, o, n, prof, exc in cases:
        with pytest.raises(O.RefError) as rerr:
            O.ref_run_simulate(fasta, o, n, **prof)
        with pytest.raises(exc) as ours:
            api.run_simulate(fasta, o, n, api.SimProfile(**prof))
        assert str(ours.value) == rerr.value.msg, (prof, str(ours.value), rerr.value.msg)


def test_simulator_create_errors(genomes):
    g = api.PackedGenome.from_fasta(genomes["multi"])
    with pytest.raises(ValueError, match="no contig is long enough"):
        api.ReadSimulator(g, api.SimProfile(read_length=10**6))
    with pytest.raises(ValueError, match="snp rate must be in"):
        api.ReadSimulator(g, api.SimProfile(snp_rate=3))
    gn = api.PackedGenome.from_fasta(genomes["allN"])
    sim = api.ReadSimulator(gn, api.SimProfile(read_length=10))
    with pytest.raises(RuntimeError, match="failed to place a read"):
        sim.next_batch(2)
