"""GPU referee: sa_referee_align / sa_referee_scan
against the reference's own oracle_align / oracle_scan (REF src/eval.cpp:
122-306, oracle/_ref).  Bar: identical results for every read and identical
hit lists (positions, distances, strands, order)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1111_5572_b200 import api, synth

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


def _genome(name, glen, repeats=False, n_runs=0, seed=5):
    if repeats:
        g = synth.make_repeat_genome(seed, glen, max(1, glen // 20000), min_len=150, max_len=1200, min_copies=4,
                                     max_copies=40, min_div=0.0, max_div=0.05)
    else:
        g = synth.make_genome(synth.CONFIGS[name].scaled(genome_len=glen))
    rng = np.random.default_rng(seed)
    for p in rng.integers(0, glen - 60, n_runs):
        g[p:p + int(rng.integers(1, 50))] = ord("N")
    packed, nmask = synth.pack_genome(g)
    return g, packed, nmask


def _both(g, packed, nmask, params, bases, offs):
    ours = api.Referee(api.PackedGenome(packed, nmask, g.size))
    ref = O.RefReferee(packed, nmask, g.size)
    a = ours.align_arrays(params, bases, offs)
    b = ref.align(params, bases, offs, threads=16)
    return a, b, ours, ref


@pytest.mark.parametrize("name,glen,nreads,rep,runs,nfrac", [
    ("C0", 1_000_000, 3000, False, 0, 0.0),
    ("C1", 400_000, 3000, False, 10, 0.01),
    ("C2", 300_000, 2000, True, 5, 0.01),
])
def test_referee_align_matches_reference(name, glen, nreads, rep, runs, nfrac):
    g, packed, nmask = _genome(name, glen, rep, runs)
    cfg = synth.CONFIGS[name].scaled(genome_len=glen, n_reads=nreads)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    rng = np.random.default_rng(3)
    for i in rng.integers(0, nreads, int(nreads * nfrac)):
        bases[int(offs[i]) + int(rng.integers(0, cfg.read_len))] = ord("N")
    a, b, _, _ = _both(g, packed, nmask, cfg.params, bases, offs)
    bad = O.compare_results(a, b)
    assert bad == [], f"{len(bad)} differ; first {bad[:3]}: ours {a[bad[:2]]} ref {b[bad[:2]]}"


def test_referee_wide_limits_and_edge_reads():
    # C3-like limits (d_max 80) on a small genome; N-heavy reads force the
    # small-q tables or the every-position scan; short reads are NotFound
    g, packed, nmask = _genome("C1", 60_000, n_runs=3)
    cfg = synth.CONFIGS["C3"].scaled(genome_len=g.size, n_reads=40)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    reads = [bases[int(offs[i]):int(offs[i + 1])].tobytes() for i in range(40)]
    gs = g.tobytes()
    reads += [gs[100:160], gs[2000:2019], b"N" * 30 + gs[5000:5070], gs[7000:7100].replace(b"A", b"N"), b"", b"ACG"]
    buf, offs2 = api.reads_to_buffer(reads)
    bb = np.frombuffer(buf, np.uint8)
    for params in (cfg.params, api.AlignerParams(seed_size=20, seeds_to_try=10, max_distance=-1,
                                                 confidence_threshold=2, max_hits=300, bucket_size=16)):
        a, b, _, _ = _both(g, packed, nmask, params, bb, offs2)
        assert O.compare_results(a, b) == []


@pytest.mark.parametrize("d_limit,bucket", [(0, 32), (3, 32), (11, 32), (11, 7), (40, 64)])
def test_referee_scan_hits_match_reference(d_limit, bucket):
    g, packed, nmask = _genome("C2", 200_000, repeats=True, n_runs=4, seed=8)
    # d_limit 40 leaves 2-base pieces: no q-gram table applies and every
    # genome position is verified (REF eval.cpp:188-190) -- a few reads only,
    # the reference's scan is single-threaded here
    cfg = synth.CONFIGS["C1"].scaled(genome_len=g.size, n_reads=200 if d_limit < 20 else 3)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    ours = api.Referee(api.PackedGenome(packed, nmask, g.size))
    ref = O.RefReferee(packed, nmask, g.size)
    ho, hits = ours.scan_arrays(d_limit, bucket, bases, offs)
    total = 0
    for i in range(offs.size - 1):
        want = ref.scan(bases[int(offs[i]):int(offs[i + 1])].tobytes(), d_limit, bucket)
        got = [(int(h["position"]), int(h["distance"]), int(h["direction"])) for h in hits[int(ho[i]):int(ho[i + 1])]]
        assert got == want, i
        total += len(want)
    assert total > 0


def test_referee_rejects_bad_characters():
    g, packed, nmask = _genome("C0", 50_000)
    ours = api.Referee(api.PackedGenome(packed, nmask, g.size))
    buf, offs = api.reads_to_buffer([g[:100].tobytes().decode().lower()])
    with pytest.raises(ValueError, match="non-base"):
        ours.align_arrays(synth.CONFIGS["C0"].params, np.frombuffer(buf, np.uint8), offs)
