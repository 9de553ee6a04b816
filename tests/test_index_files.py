"""Genome and index files: PackedGenome::from_fasta, SNAPIDX1 save/load
(REF src/genome.cpp:48-94,158-179; src/seed_index.cpp:145-228;
src/driver.cpp:37-45), checked against the reference library itself
(oracle/_ref).

CPU tests: FASTA parsing (words, contigs, checksum, every error message) and
the index loader's format checks, which all run before any GPU work.
GPU tests: SNAPIDX1 files written from the GPU-built CSR are byte-identical to
the reference's run_index output; reference-written files load and align
exactly like the reference; tampered tables are caught by verification.
"""
import os
import struct

import numpy as np
import pytest

from oracle import oracle as O
from paper_1111_5572_b200 import api, synth

need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

ACGT = "ACGT"


def _random_fasta(rng, n_contigs=4, max_len=3000, n_frac=0.01, wrap=60, crlf=False, lower=False,
                  iupac=False, empty_contig=False) -> str:
    out = []
    for c in range(n_contigs):
        L = int(rng.integers(1, max_len))
        seq = rng.choice(list(ACGT), L)
        if n_frac:
            seq[rng.random(L) < n_frac] = "N"
        if iupac:
            seq[rng.random(L) < 0.01] = rng.choice(list("RYSWKMBDHVU"))
        s = "".join(seq)
        if lower:
            s = "".join(ch.lower() if rng.random() < 0.3 else ch for ch in s)
        nl = "\r\n" if crlf else "\n"
        out.append(f">ctg_{c} some description{nl}")
        for i in range(0, len(s), wrap):
            out.append(s[i:i + wrap] + nl)
        if rng.random() < 0.3:
            out.append(nl)  # blank lines are skipped
        if empty_contig and c == 1:
            out.append(f">empty{nl}")
    return "".join(out)


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


# ------------------------------------------------------------------ FASTA (CPU)

@need_ref
@pytest.mark.parametrize("kw", [dict(), dict(crlf=True), dict(lower=True, iupac=True), dict(empty_contig=True),
                                dict(n_contigs=1, wrap=1000, n_frac=0.2), dict(n_contigs=30, max_len=70)])
def test_fasta_matches_reference(tmp_path, kw):
    rng = np.random.default_rng(len(str(kw)))
    path = _write(tmp_path, "g.fa", _random_fasta(rng, **kw))
    g = api.PackedGenome.from_fasta(path)
    packed, nmask, n, contigs, ck = O.ref_genome_from_fasta(path)
    assert g.size() == n
    assert np.array_equal(g.packed, packed) and np.array_equal(g.nmask, nmask)
    assert g.contigs() == contigs
    assert g.checksum() == ck


@need_ref
@pytest.mark.parametrize("text", [
    "",                                 # empty FASTA input
    "\n\n",
    "ACGT\n>c\nACGT\n",                 # sequence before any header
    ">\nACGT\n",                        # empty name
    "> x\nACGT\n",                      # name is the first token: empty
    ">c\nACGT\nAC-GT\n",                # illegal character
    ">c\nACGT\nACXGT\n",
])
def test_fasta_errors_match_reference(tmp_path, text):
    path = _write(tmp_path, "bad.fa", text)
    code, msg = O.ref_genome_from_fasta(path)
    with pytest.raises(api.ParseError) as ei:
        api.PackedGenome.from_fasta(path)
    assert code == api.SA_EPARSE and str(ei.value) == msg


def test_fasta_missing_file(tmp_path):
    with pytest.raises(api.IoError, match="cannot open"):
        api.PackedGenome.from_fasta(str(tmp_path / "nope.fa"))


# ------------------------------------------------------------------ loader format checks (CPU)

def _ref_index_file(tmp_path, seed=12, s=20):
    rng = np.random.default_rng(seed)
    fa = _write(tmp_path, "g.fa", _random_fasta(rng, n_contigs=3, max_len=5000))
    idx = str(tmp_path / "g.idx")
    assert O.ref_run_index(fa, idx, s) == 0
    return fa, idx


def _load_errors(path):
    """(reference code, message) and ours for loading `path`."""
    try:
        O.RefLoadedIndex(path)
        ref = (0, "")
    except O.RefError as e:
        ref = (e.code, e.msg)
    try:
        api.SeedIndex.load(path)
        ours = (0, "")
    except (api.FormatError, api.IoError, ValueError, RuntimeError) as e:
        ours = ({api.FormatError: 3, api.IoError: 5, ValueError: 1}.get(type(e), 2), str(e))
    return ref, ours


def _mutate(data: bytes, at: int, new: bytes) -> bytes:
    return data[:at] + new + data[at + len(new):]


@need_ref
@pytest.mark.parametrize("case", ["magic", "version", "seed0", "seed33", "truncated_header", "truncated_words",
                                  "end_marker", "checksum", "tables", "array_size", "contig_count", "empty"])
def test_loader_format_errors_match_reference(tmp_path, case):
    _, idx = _ref_index_file(tmp_path)
    data = open(idx, "rb").read()
    if case == "magic":
        data = _mutate(data, 0, b"SNAPIDX2")
    elif case == "version":
        data = _mutate(data, 8, struct.pack("<I", 2))
    elif case == "seed0":
        data = _mutate(data, 12, struct.pack("<I", 0))
    elif case == "seed33":
        data = _mutate(data, 12, struct.pack("<I", 33))
    elif case == "truncated_header":
        data = data[:20]
    elif case == "truncated_words":
        data = data[:len(data) // 2]
    elif case == "end_marker":
        data = data[:-8] + b"SNAPEND2"
    elif case == "checksum":
        data = _mutate(data, 16, struct.pack("<Q", 12345))
    elif case == "tables":  # offsets' last entry no longer equals the position count
        arr = _array_starts(data)  # packed, nmask, keys, offsets, positions
        n_off = struct.unpack("<Q", data[arr[3]:arr[3] + 8])[0]
        n_pos = struct.unpack("<Q", data[arr[4]:arr[4] + 8])[0]
        data = _mutate(data, arr[3] + 8 + 8 * (n_off - 1), struct.pack("<Q", n_pos + 1))
    elif case == "array_size":  # packed-word count beyond the sane limit
        at = _packed_count_at(data)
        data = _mutate(data, at, struct.pack("<Q", 1 << 41))
    elif case == "contig_count":
        data = _mutate(data, 24, struct.pack("<Q", 1 << 41))
    elif case == "empty":
        data = b""
    bad = str(tmp_path / "bad.idx")
    open(bad, "wb").write(data)
    ref, ours = _load_errors(bad)
    assert ref[0] != 0
    assert ours == ref, (ours, ref)


def _array_starts(data: bytes) -> list[int]:
    """Byte offsets of the five word arrays' counts: packed, nmask, keys,
    offsets, positions (REF include/seedaln/seed_index.hpp:74-85)."""
    at = _packed_count_at(data)
    out = []
    for _ in range(5):
        out.append(at)
        n = struct.unpack("<Q", data[at:at + 8])[0]
        at += 8 + 8 * n
    return out


def _packed_count_at(data: bytes) -> int:
    at = 24
    n_contigs = struct.unpack("<Q", data[at:at + 8])[0]
    at += 8
    for _ in range(n_contigs):
        ln = struct.unpack("<I", data[at:at + 4])[0]
        at += 4 + ln + 16
    return at + 8  # after genome_length


def test_loader_missing_file(tmp_path):
    with pytest.raises(api.IoError, match="cannot open"):
        api.SeedIndex.load(str(tmp_path / "nope.idx"))


# ------------------------------------------------------------------ GPU: write / load / verify

@need_ref
@pytest.mark.gpu
@pytest.mark.parametrize("s", [4, 11, 20, 31, 32])
def test_snapidx1_bytes_identical_to_reference(tmp_path, s):
    rng = np.random.default_rng(s)
    fa = _write(tmp_path, "g.fa", _random_fasta(rng, n_contigs=5, max_len=20000, n_frac=0.02, lower=True,
                                                iupac=True, empty_contig=True))
    ref_idx = str(tmp_path / "ref.idx")
    assert O.ref_run_index(fa, ref_idx, s) == 0
    g = api.PackedGenome.from_fasta(fa)
    ours = str(tmp_path / "ours.idx")
    api.save_index_file(s, g, ours)
    assert open(ours, "rb").read() == open(ref_idx, "rb").read()


@need_ref
@pytest.mark.gpu
def test_snapidx1_repeats_and_palindromes(tmp_path):
    # repeat-dense genome: long position lists, palindromic keys, N runs
    g0 = synth.make_repeat_genome(9, 300_000, 30, min_len=100, max_len=800, min_copies=5, max_copies=60,
                                  min_div=0.0, max_div=0.03)
    g0[1000:1100] = ord("N")
    seq = g0.tobytes().decode()
    fa = _write(tmp_path, "r.fa", ">a\n" + seq[:150_000] + "\n>b\n" + seq[150_000:] + "\n")
    for s in (8, 20):
        ref_idx = str(tmp_path / f"ref{s}.idx")
        assert O.ref_run_index(fa, ref_idx, s) == 0
        ours = str(tmp_path / f"ours{s}.idx")
        api.save_index_file(s, api.PackedGenome.from_fasta(fa), ours)
        assert open(ours, "rb").read() == open(ref_idx, "rb").read()


@need_ref
@pytest.mark.gpu
def test_load_reference_file_aligns_like_reference(tmp_path):
    cfg = synth.CONFIGS["C1"].scaled(genome_len=3_000_000, n_reads=20_000)
    gen = synth.make_genome(cfg)
    fa = _write(tmp_path, "g.fa", ">chrA\n" + gen[:1_000_000].tobytes().decode() + "\n>chrB\n"
                + gen[1_000_000:].tobytes().decode() + "\n")
    ref_idx = str(tmp_path / "ref.idx")
    assert O.ref_run_index(fa, ref_idx, 20) == 0
    idx, g = api.SeedIndex.load(ref_idx)
    assert [c[0] for c in g.contigs()] == ["chrA", "chrB"]
    bases, offs, _, _ = synth.make_reads(cfg, gen)
    got = api.Aligner(idx, g, cfg.params).align_arrays(bases, offs)
    want, _ = O.RefLoadedIndex(ref_idx).align_arrays(cfg.params, bases, offs, threads=8)
    assert O.compare_results(got, want) == []


@need_ref
@pytest.mark.gpu
def test_verify_catches_tampered_tables(tmp_path):
    _, idx = _ref_index_file(tmp_path, s=12)
    data = bytearray(open(idx, "rb").read())
    # swap two position values at the end of the positions array: the file
    # stays structurally valid and its genome checksum still matches
    end = len(data) - 8
    a, b = data[end - 16:end - 8], data[end - 8:end]
    data[end - 16:end - 8], data[end - 8:end] = b, a
    bad = str(tmp_path / "tampered.idx")
    open(bad, "wb").write(bytes(data))
    O.RefLoadedIndex(bad)  # the reference accepts it
    with pytest.raises(api.FormatError, match="do not match"):
        api.SeedIndex.load(bad)
    api.SeedIndex.load(bad, verify=False)  # opt-out: rebuilt from the genome


@pytest.mark.gpu
def test_snapgpu1_roundtrip(tmp_path):
    cfg = synth.CONFIGS["C0"]
    gen = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(gen)
    g = api.PackedGenome(packed, nmask, gen.size, [("x", 0, 400_000), ("y", 400_000, gen.size - 400_000)])
    path = str(tmp_path / "g.gpuidx")
    api.save_index_file(20, g, path, fmt=api.SA_INDEX_SNAPGPU1)
    assert os.path.getsize(path) < 400_000  # genome only: ~0.27 B/base
    idx, g2 = api.SeedIndex.load(path)
    assert g2.contigs() == g.contigs() and g2.checksum() == g.checksum()
    bases, offs, _, _ = synth.make_reads(cfg, gen)
    a = api.Aligner(idx, g2, cfg.params).align_arrays(bases, offs)
    b = api.Aligner(api.SeedIndex.build(g, 20), g, cfg.params).align_arrays(bases, offs)
    assert O.compare_results(a, b) == []


@pytest.mark.gpu
def test_index_csr_matches_oracle():
    rng = np.random.default_rng(4)
    seq = rng.choice(np.frombuffer(b"ACGT", np.uint8), 50_000)
    seq[rng.random(seq.size) < 0.01] = ord("N")
    packed, nmask = O.pack_genome(seq.tobytes())
    g = api.PackedGenome(packed, nmask, seq.size)
    for s in (3, 16, 20):
        keys, offs, pos = api.index_csr(g, s)
        oi = O.OracleIndex(packed, nmask, seq.size, s)
        assert keys.size == oi.ix.n_keys and pos.size == oi.ix.n_positions
        ok = np.ctypeslib.as_array(C_u64p(oi.ix.keys), (oi.ix.n_keys,))
        oo = np.ctypeslib.as_array(C_u64p(oi.ix.offsets), (oi.ix.n_keys + 1,))
        op = np.ctypeslib.as_array(C_u32p(oi.ix.positions), (oi.ix.n_positions,))
        assert np.array_equal(keys, ok) and np.array_equal(offs, oo) and np.array_equal(pos, op.astype(np.uint64))


def C_u64p(addr):
    import ctypes
    return ctypes.cast(addr, ctypes.POINTER(ctypes.c_uint64))


def C_u32p(addr):
    import ctypes
    return ctypes.cast(addr, ctypes.POINTER(ctypes.c_uint32))
