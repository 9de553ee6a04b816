"""Parity of the CUDA path (through the C-ABI) against the oracle.

Bar: bit-exact -- every AlignmentResult field (kind, has_position, position,
direction, distance, gap) and every AlignStats counter the reference defines
except dp_cells (implementation-specific), for every read.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1111_5572_b200 import api, synth

pytestmark = pytest.mark.gpu

ACGT = np.frombuffer(b"ACGT", np.uint8)


def _case(name, genome_len, n_reads, n_runs=0, read_n_frac=0.0, seed=7):
    cfg = synth.CONFIGS[name].scaled(genome_len=genome_len, n_reads=n_reads)
    g = synth.make_genome(cfg)
    rng = np.random.default_rng(seed)
    for p in rng.integers(0, genome_len - 50, n_runs):
        g[p:p + int(rng.integers(1, 40))] = ord("N")
    packed, nmask = synth.pack_genome(g)
    bases, offs, tp, td = synth.make_reads(cfg, g)
    if read_n_frac:
        for i in rng.integers(0, n_reads, int(n_reads * read_n_frac)):
            bases[int(offs[i]) + int(rng.integers(0, cfg.read_len))] = ord("N")
    return cfg, g, packed, nmask, bases, offs


def _gpu_vs_oracle(cfg, g, packed, nmask, bases, offs, params=None):
    params = params or cfg.params
    genome = api.PackedGenome(packed, nmask, g.size)
    idx = api.SeedIndex.build(genome, params.seed_size)
    al = api.Aligner(idx, genome, params)
    got = al.align_arrays(bases, offs)
    want, wst = O.OracleIndex(packed, nmask, g.size, params.seed_size).align_arrays(params, bases, offs, threads=8)
    bad = O.compare_results(got, want)
    assert not bad, f"{len(bad)} reads differ; first {bad[:5]}: gpu {got[bad[:3]]} oracle {want[bad[:3]]}"
    gst = al.stats().values
    for f in O.STAT_FIELDS[:16] + ("hits_consumed", "window_bases", "read_bases"):
        if f == "dp_cells":
            continue
        assert gst[f] == wst[f], f"stat {f}: gpu {gst[f]} oracle {wst[f]}"
    return got, gst


# ----------------------------------------------------------------- LV

def test_lv_known_answers():
    # REF tests/test_edit_distance.cpp:37-68
    cases = [("ACGT", "ACGTAA", 2, 0), ("ACGT", "AGGTAA", 2, 1), ("ACGTACGT", "ACGACGTCCC", 2, 1),
             ("AAAA", "TTTTTT", 2, None), ("AC", "ACGTGT", 3, 0), ("ACGT", "AC", 3, 2), ("ACGT", "", 4, 4),
             ("AN", "AN", 2, 1), ("ANNA", "AGGA", 4, 2), ("ACGT", "ACGN", 2, 1)]
    got = api.bounded_distance_batch([(r, w, d) for r, w, d, _ in cases])
    assert got == [e for *_, e in cases]
    with pytest.raises(ValueError):
        api.bounded_distance("A", "A", -1)


def _random_triples(rng, n, max_len=100, max_edits=11, max_dl=16):
    out = []
    for _ in range(n):
        L = int(rng.integers(1, max_len + 1))
        read = ACGT[rng.integers(0, 4, L)].tobytes().decode()
        win = list(read)
        for _ in range(int(rng.integers(0, max_edits))):
            if not win:
                break
            i = int(rng.integers(0, len(win)))
            op = int(rng.integers(0, 3))
            if op == 0:
                win[i] = "ACGT"[int(rng.integers(0, 4))]
            elif op == 1:
                win.insert(i, "ACGT"[int(rng.integers(0, 4))])
            else:
                del win[i]
        win += list(ACGT[rng.integers(0, 4, 8)].tobytes().decode())
        if rng.integers(0, 16) == 0:
            win[int(rng.integers(0, len(win)))] = "N"
        if rng.integers(0, 16) == 0:
            read = read[:-1] + "N"
        dl = int(rng.integers(0, max_dl))
        out.append((read, "".join(win)[:L + dl], dl))
    return out


def test_lv_random_vs_oracle():
    # acceptance criterion 2 style (REF tests/acceptance/acceptance_main.cpp:293-333)
    rng = np.random.default_rng(0xC2C2)
    triples = _random_triples(rng, 20000)
    got = api.bounded_distance_batch(triples)
    want = [O.or_bounded_distance(r, w, d) for r, w, d in triples]
    assert got == want
    full = [O.or_full_dp(r, w) for r, w, d in triples[:3000]]
    for (r, w, d), gv, f in zip(triples, got, full):
        assert gv == (f if f <= d else None)


def test_lv_wide_limits_vs_oracle():
    rng = np.random.default_rng(11)
    triples = []
    for _ in range(300):
        L = int(rng.integers(200, 3000))
        t = _random_triples(rng, 1, max_len=1, max_edits=1, max_dl=1)  # noqa: F841
        read = ACGT[rng.integers(0, 4, L)].tobytes().decode()
        win = list(read)
        for _ in range(int(rng.integers(0, L // 8))):
            i = int(rng.integers(0, len(win)))
            op = int(rng.integers(0, 3))
            if op == 0:
                win[i] = "ACGT"[int(rng.integers(0, 4))]
            elif op == 1:
                win.insert(i, "ACGT"[int(rng.integers(0, 4))])
            else:
                del win[i]
        dl = int(rng.integers(16, 400))
        win = "".join(win) + ACGT[rng.integers(0, 4, dl)].tobytes().decode()
        triples.append((read, win[:L + dl], dl))
    got = api.bounded_distance_batch(triples)
    want = [O.or_bounded_distance(r, w, d) for r, w, d in triples]
    assert got == want


def test_lv_long_limits_vs_oracle():
    """Long reads at long-read limits (256-960: the systolic lv_sys serves
    them, C4's 607 among them): close and diverged windows, windows cut short
    (genome end), N bases on both sides."""
    rng = np.random.default_rng(607)
    triples = []
    for t in range(48):
        L = int(rng.integers(1500, 10001))
        read = list(ACGT[rng.integers(0, 4, L)].tobytes().decode())
        for _ in range(int(rng.integers(0, 4))):
            read[int(rng.integers(0, L))] = "N"
        read = "".join(read)
        win = list(read)
        rate = [0.01, 0.05, 0.08, 0.12, 0.3][t % 5]
        for _ in range(int(L * rate)):
            i = int(rng.integers(0, len(win)))
            op = int(rng.integers(0, 3))
            if op == 0:
                win[i] = "ACGTN"[int(rng.integers(0, 5))]
            elif op == 1:
                win.insert(i, "ACGT"[int(rng.integers(0, 4))])
            else:
                del win[i]
        dl = int(rng.integers(256, 961))
        win = "".join(win) + ACGT[rng.integers(0, 4, dl)].tobytes().decode()
        cut = L + dl if t % 3 else int(rng.integers(max(1, L - dl), L + dl))
        triples.append((read, win[:cut], dl))
    got = api.bounded_distance_batch(triples)
    want = [O.or_bounded_distance(r, w, d) for r, w, d in triples]
    assert got == want
    assert any(v is None for v in want) and any(v is not None for v in want)


def test_lv_long_limits_edges_vs_oracle():
    """Edges of the long-read LVs (lv_sys from 256; lv_bitpar_warp above 960):
    reads ending exactly on / one past a 64-row block, windows shorter than
    m - d_limit (nothing reachable), empty windows, all-N and N-rich reads,
    limits at 256, 607, 960, 961 and 1023, limits above the read length."""
    rng = np.random.default_rng(960)
    triples = []
    for m in (255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 4096, 4097):
        read = ACGT[rng.integers(0, 4, m)].tobytes().decode()
        for dl in (256, 607, 960, 961, 1023):
            win = list(read)
            for _ in range(int(rng.integers(0, max(1, m // 10)))):
                i = int(rng.integers(0, len(win)))
                op = int(rng.integers(0, 3))
                if op == 0:
                    win[i] = "ACGT"[int(rng.integers(0, 4))]
                elif op == 1:
                    win.insert(i, "ACGT"[int(rng.integers(0, 4))])
                else:
                    del win[i]
            win = "".join(win) + ACGT[rng.integers(0, 4, dl)].tobytes().decode()
            triples.append((read, win[:m + dl], dl))
            triples.append((read, win[:max(0, m - dl - 1)], dl))  # row m out of reach
            triples.append((read, "", dl))
    n_read = "N" * 700
    triples += [(n_read, ACGT[rng.integers(0, 4, 1000)].tobytes().decode(), 700),
                (n_read, n_read, 700), (n_read, n_read, 699)]
    nr = list(ACGT[rng.integers(0, 4, 3000)].tobytes().decode())
    for i in rng.integers(0, 3000, 200):
        nr[int(i)] = "N"
    nr = "".join(nr)
    triples += [(nr, nr + "ACGT" * 100, 300), (nr, nr.replace("N", "A") + "ACGT" * 100, 250)]
    got = api.bounded_distance_batch(triples)
    want = [O.or_bounded_distance(r, w, d) for r, w, d in triples]
    assert got == want


# ----------------------------------------------------------------- lookup

@pytest.mark.parametrize("s", [3, 4, 7, 8, 20, 31, 32])
def test_lookup_vs_oracle(s):
    rng = np.random.default_rng(s)
    for trial in range(6):
        L = int(rng.integers(max(s, 50), 20000))
        seq = ACGT[rng.integers(0, 4, L)]
        if trial % 3 == 0:
            seq[rng.random(L) < 0.03] = ord("N")
        seq = seq.tobytes()
        packed, nmask = O.pack_genome(seq)
        gi = api.SeedIndex.build(api.PackedGenome(packed, nmask, L), s)
        oi = O.OracleIndex(packed, nmask, L, s)
        probes = []
        for p in range(200):
            if p % 2 == 0 and L > s:
                at = int(rng.integers(0, L - s + 1))
                probes.append(seq[at:at + s].decode())
            else:
                probes.append(ACGT[rng.integers(0, 4, s)].tobytes().decode())
        res = gi.lookup_batch(probes, cap=L)
        for q, r in zip(probes, res):
            f, rc = oi.lookup(q)
            assert (r.forward, r.rc) == (f, rc), q
        assert gi.total_positions() == oi.ix.n_positions


def test_lookup_palindrome_and_rc():
    # REF tests/test_seed_index.cpp:67-95
    g = api.PackedGenome.from_sequence("ACGTACGTAC")
    idx = api.SeedIndex.build(g, 4)
    assert idx.total_positions() == 7
    r = idx.lookup("ACGT")
    assert r.forward == [0, 4] and r.rc == [0, 4] and r.count() == 4
    assert idx.lookup("CGTA").forward == [1, 5]
    g2 = api.PackedGenome.from_sequence("AACCGG")
    r2 = api.SeedIndex.build(g2, 4).lookup("GGTT")
    assert r2.forward == [] and r2.rc == [0] and r2.count() == 1
    g3 = api.PackedGenome.from_sequence("ACNTA")
    i3 = api.SeedIndex.build(g3, 3)
    assert i3.total_positions() == 0 and i3.lookup("ACN").count() == 0


# ----------------------------------------------------------------- aligner

@pytest.mark.parametrize("name,glen,nreads,runs,nfrac", [
    ("C0", 1_000_000, 10_000, 0, 0.0),
    ("C1", 5_000_000, 30_000, 20, 0.02),
    ("C2", 8_000_000, 30_000, 20, 0.02),
    ("C3", 8_000_000, 2_000, 10, 0.01),
    ("C4", 3_000_000, 60, 5, 0.0),
])
def test_align_parity(name, glen, nreads, runs, nfrac):
    cfg, g, packed, nmask, bases, offs = _case(name, glen, nreads, runs, nfrac)
    got, st = _gpu_vs_oracle(cfg, g, packed, nmask, bases, offs)
    assert st["reads"] == nreads


def test_align_heavily_edited_reads():
    """Reads carrying 0-16 edits each (substitutions, 1-3 base insertions and
    deletions, N) at d_max 12: every LV length from an exact match to a
    wavefront that fails at the limit -- the solo kernel's serial iterations,
    the warp's lane-per-diagonal finish of the longer ones (lv_warp_resume)
    and the warp kernel's own LV (test_gpu_solo.py forces each)."""
    cfg, g, packed, nmask, bases, offs = _case("C1", 3_000_000, 20_000)
    rng = np.random.default_rng(11)
    reads = []
    for i in range(20_000):
        L = int(rng.integers(90, 130))
        st = int(rng.integers(0, g.size - L - 8))
        r = bytearray(g[st:st + L].tobytes())
        for _ in range(int(rng.integers(0, 17))):
            q = int(rng.integers(0, len(r)))
            kind = int(rng.integers(0, 10))
            if kind < 6:
                r[q] = ACGT[int(rng.integers(0, 4))]
            elif kind < 8:
                del r[q:q + int(rng.integers(1, 4))]
            elif kind < 9:
                r[q:q] = bytes(ACGT[int(v)] for v in rng.integers(0, 4, int(rng.integers(1, 4))))
            else:
                r[q] = ord("N")
        if i % 2:
            r = bytearray(bytes(r).translate(bytes.maketrans(b"ACGT", b"TGCA"))[::-1])
        reads.append(bytes(r))
    buf, offs2 = api.reads_to_buffer(reads)
    _gpu_vs_oracle(cfg, g, packed, nmask, np.frombuffer(buf, np.uint8).copy(), offs2)


def test_align_force_max_dlimit_parity():
    cfg, g, packed, nmask, bases, offs = _case("C2", 4_000_000, 10_000, 10, 0.01)
    p = synth.CONFIGS["C2"].params
    forced = api.AlignerParams(**{**p.__dict__, "force_max_dlimit": True})
    _gpu_vs_oracle(cfg, g, packed, nmask, bases, offs, params=forced)


def test_align_ragged_and_short_reads():
    cfg, g, packed, nmask, bases, offs = _case("C1", 2_000_000, 3000)
    rng = np.random.default_rng(3)
    reads = []
    for i in range(3000):
        L = int(rng.integers(0, 260))
        st = int(rng.integers(0, g.size - L - 1))
        r = bytearray(g[st:st + L].tobytes())
        for _ in range(int(rng.integers(0, 4))):
            if L:
                r[int(rng.integers(0, L))] = ACGT[int(rng.integers(0, 4))]
        reads.append(bytes(r))
    buf, offs2 = api.reads_to_buffer(reads)
    b = np.frombuffer(buf, np.uint8).copy()
    _gpu_vs_oracle(cfg, g, packed, nmask, b, offs2)


def test_invalid_character_raises():
    cfg, g, packed, nmask, bases, offs = _case("C0", 200_000, 10)
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
    b = bases.copy()
    b[5] = ord("x")
    with pytest.raises(ValueError):
        al.align_arrays(b, offs)
    # a read shorter than s is never inspected (REF aligner.cpp:231-235)
    assert al.align_batch(["ACGx"])[0].kind == api.ResultKind.NotFound


@pytest.mark.parametrize("read_len", [100, 1500])
def test_every_byte_outside_acgtn_raises(read_len):
    """Every byte value other than A/C/G/T/N, at positions spread over the read
    (word offsets 0-3, every 32-base block, the last base), fails the batch
    (REF genome.cpp:182-200); reads of A/C/G/T/N only never do. 100 bp reads
    are decoded by the seed kernel, 1.5 kbp reads by the long-read kernel."""
    cfg, g, packed, nmask, bases, offs = _case("C0", 200_000, 10)
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
    rng = np.random.default_rng(7)
    base = bytearray(rng.choice(np.frombuffer(b"ACGTN", np.uint8), size=read_len).tobytes())
    ok = al.align_batch([bytes(base).decode()] * 3)
    assert len(ok) == 3
    for v in range(256):
        if v in b"ACGTN":
            continue
        r = bytearray(base)
        r[(v * 37) % read_len] = v
        buf, offs2 = api.reads_to_buffer([bytes(base), bytes(r), bytes(base)])
        with pytest.raises(ValueError):
            al.align_arrays(np.frombuffer(buf, np.uint8).copy(), offs2)


# ----------------------------------------------------------------- golden fixtures (reference outputs)

import json  # noqa: E402
import os  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_lv_golden_gpu():
    d = np.load(os.path.join(GOLD, "lv_golden.npz"))
    rb, ro, wb, wo = d["reads"].tobytes(), d["read_off"], d["wins"].tobytes(), d["win_off"]
    triples = [(rb[ro[i]:ro[i + 1]].decode(), wb[wo[i]:wo[i + 1]].decode(), int(d["d_limits"][i]))
               for i in range(d["d_limits"].size)]
    got = api.bounded_distance_batch(triples)
    assert [-1 if v is None else v for v in got] == d["expected"].tolist()


def test_lookup_golden_gpu():
    with open(os.path.join(GOLD, "lookup_golden.json")) as f:
        data = json.load(f)
    for s, dd in data.items():
        g = api.PackedGenome.from_sequence(dd["genome"])
        idx = api.SeedIndex.build(g, int(s))
        assert idx.total_positions() == dd["total"]
        assert idx.distinct_seeds() == dd["distinct"]
        res = idx.lookup_batch(dd["queries"], cap=len(dd["genome"]))
        for q, r, f, rc in zip(dd["queries"], res, dd["fwd"], dd["rc"]):
            assert (r.forward, r.rc) == (f, rc), (s, q)


@pytest.mark.parametrize("case", ["C1", "C2", "C2_force", "C3", "C4", "REP"])
def test_align_golden_gpu(case):
    d = np.load(os.path.join(GOLD, "align_golden.npz"))
    g = d[f"{case}__genome"]
    pa = [int(v) for v in d[f"{case}__params"]]
    p = api.AlignerParams(seed_size=pa[0], seeds_to_try=pa[1], max_distance=pa[2], confidence_threshold=pa[3],
                          max_hits=pa[4], bucket_size=pa[5], force_max_dlimit=bool(pa[6]))
    packed, nmask = synth.pack_genome(g)
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, p.seed_size), genome, p)
    got = al.align_arrays(d[f"{case}__bases"], d[f"{case}__offsets"])
    want = d[f"{case}__results"].view(api.RESULT_DTYPE)
    assert O.compare_results(got, want) == []
    st = al.stats().values
    exp = d[f"{case}__stats"].tolist()
    for i, f in enumerate(api.REFERENCE_STAT_FIELDS):
        if f != "dp_cells":
            assert st[f] == exp[i], f


@pytest.mark.parametrize("parts", [3, 17])
def test_partitioned_index_build_identical(parts, monkeypatch):
    """The key-hash-partitioned build (used automatically for 3.1 Gbp genomes)
    yields the same index as the one-pass build: same lookups, same alignments."""
    cfg, g, packed, nmask, bases, offs = _case("C2", 4_000_000, 8_000, 10, 0.01)
    genome = api.PackedGenome(packed, nmask, g.size)
    one = api.SeedIndex.build(genome, 20)
    monkeypatch.setenv("SA_INDEX_PARTS", str(parts))
    many = api.SeedIndex.build(genome, 20)
    monkeypatch.delenv("SA_INDEX_PARTS")
    assert (one.distinct_seeds(), one.total_positions()) == (many.distinct_seeds(), many.total_positions())
    rng = np.random.default_rng(parts)
    probes = [g[p:p + 20].tobytes().decode() for p in rng.integers(0, g.size - 20, 3000)]
    a, b = one.lookup_batch(probes, cap=4096), many.lookup_batch(probes, cap=4096)
    assert [(r.forward, r.rc) for r in a] == [(r.forward, r.rc) for r in b]
    ra = api.Aligner(one, genome, cfg.params).align_arrays(bases, offs)
    rb = api.Aligner(many, genome, cfg.params).align_arrays(bases, offs)
    assert not O.compare_results(ra, rb)


@pytest.mark.parametrize("mode", ["deferred", "kernel"])
def test_overflow_paths_parity(mode, monkeypatch):
    """Reads with more candidates than the 64-entry shared table: collected
    batch-wide and redone by one global-table pass at the end of the batch
    (default), or by a global-table kernel after every chunk
    (SA_OVERFLOW_KERNEL) -- same results, same stats."""
    if mode == "kernel":
        monkeypatch.setenv("SA_OVERFLOW_KERNEL", "1")
    g = synth.make_repeat_genome(5, 2_000_000, 60, min_len=200, max_len=1500, min_copies=20, max_copies=150,
                                 min_div=0.0, max_div=0.04)
    packed, nmask = synth.pack_genome(g)
    cfg = synth.CONFIGS["C3"].scaled(genome_len=g.size, n_reads=4000)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    _, st = _gpu_vs_oracle(cfg, g, packed, nmask, bases, offs)
    assert st["overflow_reads"] > 0


def _streamed_case():
    cfg = synth.CONFIGS["C1"].scaled(genome_len=5_000_000, n_reads=100_000)
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    # interleave a few long reads (beyond the streamed layout: deferred to the
    # end-of-batch pass) and short reads (< s) into later chunks
    rng = np.random.default_rng(12)
    reads = [bases[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(offs.size - 1)]
    for i in rng.integers(20_000, 100_000, 60):
        st = int(rng.integers(0, g.size - 400))
        reads[int(i)] = g[st:st + int(rng.integers(129, 400))].tobytes()
    for i in rng.integers(20_000, 100_000, 30):
        reads[int(i)] = reads[int(i)][:int(rng.integers(0, 20))]
    buf, offs2 = api.reads_to_buffer(reads)
    return cfg, g, packed, nmask, np.frombuffer(buf, np.uint8).copy(), offs2


def test_streamed_batch_matches_chunked_and_oracle(monkeypatch):
    """sa_align_batch's single-launch streamed path (SA_STREAM=1: chunk flags
    written by stream memory ops, per-chunk copy-out gated on done counts)
    against the chunked pipeline (the default) and the oracle: pageable and pinned
    result buffers, deferred long reads, short reads."""
    monkeypatch.setenv("SA_STREAM", "1")
    cfg, g, packed, nmask, bases, offs = _streamed_case()
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
    a = al.align_arrays(bases, offs)
    st_a = dict(al.stats().values)
    pin = api.PinnedBuffer(offs.size * 24)
    hr = pin.array(api.RESULT_DTYPE, offs.size - 1)
    al.align_arrays(bases, offs, hr)
    assert O.compare_results(hr.copy(), a) == []
    monkeypatch.delenv("SA_STREAM")
    al2 = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
    b = al2.align_arrays(bases, offs)
    assert O.compare_results(a, b) == []
    for f in api.REFERENCE_STAT_FIELDS:
        assert st_a[f] == al2.stats().values[f], f
    want, _ = O.OracleIndex(packed, nmask, g.size, 20).align_arrays(cfg.params, bases, offs, threads=8)
    assert O.compare_results(a, want) == []


def test_streamed_batch_errors(monkeypatch):
    monkeypatch.setenv("SA_STREAM", "1")
    cfg, g, packed, nmask, bases, offs = _streamed_case()
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
    bad = bases.copy()
    bad[int(offs[90_000]) + 5] = ord("X")  # a late chunk: the error still surfaces
    with pytest.raises(ValueError, match="read 90000"):
        al.align_arrays(bad, offs)
    o2 = offs.copy()
    o2[70_001] = o2[70_000] - 1  # offsets not ascending inside a late chunk
    with pytest.raises(ValueError, match="ascending"):
        al.align_arrays(bases, o2)
    # the context stays usable after both errors
    again = al.align_arrays(bases, offs)
    want, _ = O.OracleIndex(packed, nmask, g.size, 20).align_arrays(cfg.params, bases, offs, threads=8)
    assert O.compare_results(again, want) == []


@pytest.mark.parametrize("pack", ["0", "3"])
def test_batch_pipeline_fixed_length_ramp_and_packing(pack, monkeypatch):
    """The seeded chunk pipeline on 400 k equal-length reads (offsets never
    copied in; chunk sizes ramp up and back down) and on ragged reads with
    deferred long ones, with ASCII input and with host-packed bit planes
    (SA_PACK_THREADS); bad characters still fail the right read."""
    monkeypatch.setenv("SA_PACK_THREADS", pack)
    cfg, g, packed, nmask, bases, offs = _case("C1", 5_000_000, 400_000, 10, 0.01)
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
    oi = O.OracleIndex(packed, nmask, g.size, 20)
    got = al.align_arrays(bases, offs)
    want, wst = oi.align_arrays(cfg.params, bases, offs, threads=8)
    assert O.compare_results(got, want) == []
    for f in api.REFERENCE_STAT_FIELDS:
        if f != "dp_cells":
            assert al.stats().values[f] == wst[f], f
    bad = bases.copy()
    bad[int(offs[399_990]) + 7] = ord("x")  # in the last (ramp-down) chunk
    with pytest.raises(ValueError, match="read 399990"):
        al.align_arrays(bad, offs)
    cfg2, g2, packed2, nmask2, b2, o2 = _streamed_case()
    genome2 = api.PackedGenome(packed2, nmask2, g2.size)
    al2 = api.Aligner(api.SeedIndex.build(genome2, 20), genome2, cfg2.params)
    want2, _ = O.OracleIndex(packed2, nmask2, g2.size, 20).align_arrays(cfg2.params, b2, o2, threads=8)
    assert O.compare_results(al2.align_arrays(b2, o2), want2) == []


@pytest.mark.parametrize("bs,c,dmax,n,hmax", [
    (32, 2, -1, 10, 300),   # automatic d_max (ceil(12 L / 100))
    (16, 1, 6, 25, 300),
    (8, 3, 8, 3, 50),
    (4, 2, 10, 10, 2),      # tiny h_max: most repeat seeds are popular
    (1, 2, 5, 10, 300),
    (7, 2, 8, 10, 300),     # not a power of two: the warp kernel only
    (64, 2, 10, 10, 300),   # wider than the solo kernel's 32-bit anchor mask
])
def test_align_param_sweep(bs, c, dmax, n, hmax):
    """AlignerParams away from the configs' values (bucket size, confidence,
    d_max, seeds, h_max) on a repeat-rich genome, in a batch large enough for
    the solo kernel: bit-exact with the oracle, counters included."""
    g = synth.make_repeat_genome(9, 3_000_000, 40, min_len=150, max_len=800, min_copies=2, max_copies=12,
                                 min_div=0.0, max_div=0.06)
    packed, nmask = synth.pack_genome(g)
    cfg = synth.CONFIGS["C1"].scaled(genome_len=g.size, n_reads=14_000)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    p = api.AlignerParams(seed_size=20, seeds_to_try=n, max_distance=dmax, confidence_threshold=c, max_hits=hmax,
                          bucket_size=bs)
    _gpu_vs_oracle(cfg, g, packed, nmask, bases, offs, params=p)


def test_pageable_and_pinned_buffers_agree():
    """sa_align_batch with the caller's buffers pageable (the library stages
    them through its own pinned buffers, input and results), pinned, or
    mixed: identical results, equal to the oracle, over many chunks."""
    cfg, g, packed, nmask, bases, offs = _case("C1", 3_000_000, 300_000, 5, 0.005)
    genome = api.PackedGenome(packed, nmask, g.size)
    al = api.Aligner(api.SeedIndex.build(genome, 20), genome, cfg.params)
    pageable = al.align_arrays(bases, offs)
    pin_b, pin_r = api.PinnedBuffer(bases.nbytes), api.PinnedBuffer(pageable.nbytes)
    hb = pin_b.array(np.uint8, bases.size)
    hb[:] = bases
    hr = pin_r.array(api.RESULT_DTYPE, pageable.size)
    al.align_arrays(hb, offs, hr)
    assert O.compare_results(hr.copy(), pageable) == []
    mixed = al.align_arrays(hb, offs)                 # pinned in, pageable out
    assert O.compare_results(mixed, pageable) == []
    hr[:] = np.zeros(1, api.RESULT_DTYPE)
    al.align_arrays(bases, offs, hr)                  # pageable in, pinned out
    assert O.compare_results(hr.copy(), pageable) == []
    want, _ = O.OracleIndex(packed, nmask, g.size, 20).align_arrays(cfg.params, bases, offs, threads=8)
    assert O.compare_results(pageable, want) == []
