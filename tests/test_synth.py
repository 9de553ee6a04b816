"""Synthetic inputs are deterministic and have the configured shape (CPU)."""
import numpy as np

from paper_1111_5572_b200 import synth


def test_random_genome_deterministic_and_uniform():
    cfg = synth.CONFIGS["C0"]
    a = synth.make_genome(cfg)
    b = synth.make_genome(cfg)
    assert a.size == 1_000_000 and (a == b).all()
    counts = np.bincount(a, minlength=256)[[65, 67, 71, 84]]
    assert counts.sum() == a.size and counts.min() > 0.24 * a.size


def test_reads_shape_and_truth():
    cfg = synth.CONFIGS["C0"].scaled(n_reads=500)
    g = synth.make_genome(cfg)
    bases, offs, pos, dirs = synth.make_reads(cfg, g)
    assert bases.size == 500 * 100 and offs[-1] == bases.size
    comp = bytes.maketrans(b"ACGT", b"TGCA")
    mism = []
    for i in range(500):
        r = bases[offs[i]:offs[i + 1]].tobytes()
        if dirs[i]:
            r = r.translate(comp)[::-1]
        t = g[pos[i]:pos[i] + 100].tobytes()
        mism.append(sum(x != y for x, y in zip(r, t)))
    assert 0.5 < np.mean(mism) < 1.6  # 1% substitutions, no indels in C0
    assert 0.4 < dirs.mean() < 0.6
    b2, _, p2, _ = synth.make_reads(cfg, g)
    assert (b2 == bases).all() and (p2 == pos).all()


def test_repeat_genome_has_repeats():
    g = synth.make_repeat_genome(5, 200_000, 10, min_div=0.0, max_div=0.0)
    seeds = {}
    for p in range(0, g.size - 20, 7):
        k = g[p:p + 20].tobytes()
        seeds[k] = seeds.get(k, 0) + 1
    assert max(seeds.values()) >= 4
