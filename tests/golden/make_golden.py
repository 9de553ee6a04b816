"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs here (where /root/reference exists) against oracle/_ref/libseedaln_ref.so,
the unmodified reference library compiled by `make -C oracle ref`.  Outputs
are committed so the C restatement stays pinned on machines without
/root/reference (the GPU box).  Inputs are seeded synthetic data.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1111_5572_b200 import synth  # noqa: E402

ACGT = np.frombuffer(b"ACGT", np.uint8)


def _cat(strs):
    b = b"".join(s.encode() for s in strs)
    off = np.zeros(len(strs) + 1, np.uint64)
    off[1:] = np.cumsum([len(s) for s in strs])
    return np.frombuffer(b, np.uint8), off


def lv(rng):
    reads, wins, dls = [], [], []
    for t in range(4000):
        L = int(rng.integers(0 if t < 20 else 1, 101))
        read = ACGT[rng.integers(0, 4, L)].tobytes().decode()
        w = list(read)
        for _ in range(int(rng.integers(0, 11))):
            if not w:
                break
            i = int(rng.integers(0, len(w)))
            op = int(rng.integers(0, 3))
            if op == 0:
                w[i] = "ACGT"[int(rng.integers(0, 4))]
            elif op == 1:
                w.insert(i, "ACGT"[int(rng.integers(0, 4))])
            else:
                del w[i]
        w += list(ACGT[rng.integers(0, 4, 8)].tobytes().decode())
        if rng.integers(0, 16) == 0 and w:
            w[int(rng.integers(0, len(w)))] = "N"
        if rng.integers(0, 16) == 0 and read:
            read = read[:-1] + "N"
        dl = int(rng.integers(0, 24))
        wins.append("".join(w)[:L + dl])
        reads.append(read)
        dls.append(dl)
    exp = [O.ref_bounded_distance(r, w, d) for r, w, d in zip(reads, wins, dls)]
    full = [O.rlib().ref_full_dp_distance(r.encode(), len(r), w.encode(), len(w)) for r, w in zip(reads, wins)]
    rb, ro = _cat(reads)
    wb, wo = _cat(wins)
    np.savez_compressed(os.path.join(HERE, "lv_golden.npz"), reads=rb, read_off=ro, wins=wb, win_off=wo,
                        d_limits=np.array(dls, np.int32),
                        expected=np.array([-1 if e is None else e for e in exp], np.int32),
                        full_dp=np.array(full, np.int32))


def offsets(rng):
    cases = [(100, 20, 9), (25, 20, 4), (19, 20, 3), (40, 20, 25), (100, 20, 8), (100, 20, 10),
             (125, 20, 12), (1000, 20, 40), (10000, 22, 200)]
    for _ in range(400):
        cases.append((int(rng.integers(1, 400)), int(rng.integers(1, 33)), int(rng.integers(1, 60))))
    out = [{"len": L, "s": s, "n": n, "offsets": O.ref_seed_offsets(L, s, n)} for L, s, n in cases]
    with open(os.path.join(HERE, "seed_offsets_golden.json"), "w") as f:
        json.dump(out, f)


def lookup(rng):
    data = {}
    for s, L, npct in [(4, 3000, 0), (8, 5000, 3), (20, 20000, 1), (31, 4000, 0), (32, 4000, 2)]:
        seq = ACGT[rng.integers(0, 4, L)]
        seq[rng.random(L) < npct / 100] = ord("N")
        seq = seq.tobytes()
        packed, nmask = O.pack_genome(seq)
        ri = O.RefIndex(packed, nmask, L, s)
        qs = []
        for p in range(300):
            if p % 2 == 0:
                at = int(rng.integers(0, L - s + 1))
                qs.append(seq[at:at + s].decode())
            else:
                qs.append(ACGT[rng.integers(0, 4, s)].tobytes().decode())
        fw, rc = [], []
        for q in qs:
            f, r = ri.lookup(q)
            fw.append(f)
            rc.append(r)
        d, t = ri.info()
        data[str(s)] = {"genome": seq.decode(), "queries": qs, "fwd": fw, "rc": rc, "distinct": d, "total": t}
    with open(os.path.join(HERE, "lookup_golden.json"), "w") as f:
        json.dump(data, f)


def align(rng):
    cases = {}
    for name, glen, nreads, force in [("C1", 200_000, 2000, False), ("C2", 250_000, 2000, False),
                                      ("C2", 250_000, 1000, True), ("C3", 200_000, 200, False),
                                      ("C4", 120_000, 12, False)]:
        cfg = synth.CONFIGS[name].scaled(genome_len=glen, n_reads=nreads)
        g = synth.make_genome(cfg)
        for p in rng.integers(0, glen - 50, 5):
            g[p:p + int(rng.integers(1, 30))] = ord("N")
        packed, nmask = synth.pack_genome(g)
        bases, offs, _, _ = synth.make_reads(cfg, g)
        for i in rng.integers(0, nreads, nreads // 40):
            bases[int(offs[i]) + int(rng.integers(0, cfg.read_len))] = ord("N")
        p = cfg.params
        if force:
            p = synth.AlignerParams(**{**p.__dict__, "force_max_dlimit": True})
        ri = O.RefIndex(packed, nmask, g.size, p.seed_size)
        res, st = ri.align_arrays(p, bases, offs, threads=8)
        key = f"{name}{'_force' if force else ''}"
        cases[key] = dict(genome=g, bases=bases, offsets=offs, results=res.view(np.uint8),
                          stats=np.array([st[f] for f in O.STAT_FIELDS[:16]], np.uint64),
                          params=np.array([p.seed_size, p.seeds_to_try, p.max_distance, p.confidence_threshold,
                                           p.max_hits, p.bucket_size, int(p.force_max_dlimit)], np.int32))
    # repeat-dense corpus: diverged and exact families, popular seeds (h_max 40)
    g = synth.make_repeat_genome(77, 150_000, 25, min_len=150, max_len=900, min_copies=4, max_copies=120,
                                 min_div=0.0, max_div=0.06, repeat_fraction=0.6)
    g[5000:5600] = ord("A")
    packed, nmask = synth.pack_genome(g)
    cfg = synth.CONFIGS["C1"].scaled(genome_len=g.size, n_reads=2000)
    cfg = synth.Config(**{**cfg.__dict__, "sub_rate": 0.03, "indel_rate": 0.004})
    bases, offs, _, _ = synth.make_reads(cfg, g)
    p = synth.AlignerParams(seed_size=20, seeds_to_try=10, max_distance=10, confidence_threshold=2,
                            max_hits=40, bucket_size=32)
    ri = O.RefIndex(packed, nmask, g.size, 20)
    res, st = ri.align_arrays(p, bases, offs, threads=8)
    cases["REP"] = dict(genome=g, bases=bases, offsets=offs, results=res.view(np.uint8),
                        stats=np.array([st[f] for f in O.STAT_FIELDS[:16]], np.uint64),
                        params=np.array([20, 10, 10, 2, 40, 32, 0], np.int32))
    flat = {f"{k}__{f}": v for k, d in cases.items() for f, v in d.items()}
    np.savez_compressed(os.path.join(HERE, "align_golden.npz"), **flat)


if __name__ == "__main__":
    if not O.ref_available():
        O.build(with_ref=True)
    rng = np.random.default_rng(20261019)
    lv(rng)
    offsets(rng)
    lookup(rng)
    align(rng)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
