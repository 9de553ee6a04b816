"""CPU evidence for the long-read LV's q-gram pre-test (csrc/lv.cuh
qgram_reject): replays the reference's seed loop (REF src/aligner.cpp:223-316)
in Python on C3 reads against the oracle index, records every
bounded_distance call (read orientation, window, d_limit, result), and
counts how many of the failing calls each filter variant would have rejected
(asserting it never rejects a call whose distance is <= d_limit).

  python scripts/qgram_filter_model.py [n_reads]
"""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1111_5572_b200 import synth
from oracle import oracle as O
cfg = synth.CONFIGS['C3']; p = cfg.params
g = synth.make_genome(cfg); packed, nmask = synth.pack_genome(g)
NR = int(sys.argv[1]) if len(sys.argv) > 1 else 200
bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=NR)
oi = O.OracleIndex(packed, nmask, g.size, p.seed_size, for_reads=(p.seeds_to_try, bases, offs), threads=8)
G = g  # uint8 ascii? check
gs = bytes(G[:100]) ; print('genome sample', gs[:20])
COMP = bytes.maketrans(b'ACGTN', b'TGCAN')
def rc(s): return s.translate(COMP)[::-1]
calls = []  # (read_idx, d_limit, result, read, window)
for r in range(NR):
    read = bytes(bases[offs[r]:offs[r+1]]); L = len(read); rcr = rc(read)
    s = p.seed_size; d_max = p.max_distance if p.max_distance >= 0 else (12*L+99)//100; c = p.confidence_threshold
    offsets = O.or_seed_offsets(L, s, p.seeds_to_try); tier0 = L // s
    cands = {}; order = []
    dbest = dsec = 1 << 30; bpos = 0; bdir = 0; tested = 0
    def observe(d, pos, dr):
        global dbest, dsec, bpos, bdir
    for i, off in enumerate(offsets):
        seed = read[off:off+s].decode()
        if 'N' in seed: continue
        fw, rv = oi.lookup(seed)
        if len(fw) + len(rv) > p.max_hits: continue
        if i < tier0: tested += 1
        for pp in fw:
            a = max(0, pp - off); key = (a // p.bucket_size, 0)
            if key not in cands: cands[key] = [0, 0, False]; order.append(key)
            cands[key][0] += 1; cands[key][1] |= 1 << (a - key[0]*p.bucket_size)
        for pp in rv:
            a = max(0, pp - (L - s - off)); key = (a // p.bucket_size, 1)
            if key not in cands: cands[key] = [0, 0, False]; order.append(key)
            cands[key][0] += 1; cands[key][1] |= 1 << (a - key[0]*p.bucket_size)
        # score best
        best = None
        for k in order:
            cc = cands[k]
            if cc[2]: continue
            amin = k[0]*p.bucket_size + ((cc[1] & -cc[1]).bit_length() - 1)
            key2 = (-cc[0], amin, k[1])
            if best is None or key2 < best[0]: best = (key2, k)
        if best is None: continue
        k = best[1]; cc = cands[k]; cc[2] = True
        if dbest > d_max: dl = d_max + c - 1
        elif dsec >= dbest + c: dl = dbest + c - 1
        else: dl = dbest - 1
        if dl < 0: continue
        ori = read if k[1] == 0 else rcr
        bd = 1 << 30; ba = 0
        m = cc[1]
        while m:
            a = k[0]*p.bucket_size + ((m & -m).bit_length() - 1); m &= m - 1
            if a >= g.size: continue
            win = bytes(G[a:a + L + dl])
            v = O.or_bounded_distance(ori.decode(), win.decode(), dl)
            calls.append((r, dl, v, ori, win))
            if v is not None and v < bd: bd, ba = v, a
        if bd < (1 << 30):
            # tracker observe (REF aligner.cpp:87-109)
            if dbest < (1 << 30) and k[1] == bdir and abs(ba - bpos) <= p.bucket_size:
                if bd < dbest: dbest, bpos = bd, ba
            elif bd < dbest: dsec, dbest, bpos, bdir = dbest, bd, ba, k[1]
            elif bd < dsec: dsec = bd
        if dbest < c and dsec < dbest + c: break
        if tested >= dbest + c: break  # (pruning loop omitted: C3 never gets here)
print('reads', NR, 'calls', len(calls), 'fail', sum(v is None for _,_,v,_,_ in calls))
def qgrams(s, q):
    return [s[i:i+q] for i in range(len(s) - q + 1)]
for q in (5, 6, 7, 8):
    rej = okfail = kept_ok = 0
    for r, dl, v, ori, win in calls:
        m = len(ori)
        # banded: read q-gram at i occurs in win[i-dl .. i+dl+q)
        cnt = 0
        wq = {}
        for j, x in enumerate(qgrams(win, q)): wq.setdefault(x, []).append(j)
        for i, x in enumerate(qgrams(ori, q)):
            if b'N' in x: continue
            js = wq.get(x)
            if js and any(abs(j - i) <= dl for j in js): cnt += 1
        thr = (m - q + 1) - dl * q
        if cnt < thr:
            rej += 1
            assert v is None, (cnt, thr, v)
        elif v is None: okfail += 1
        else: kept_ok += 1
    print('q', q, 'rejected', rej, 'passed-but-failed', okfail, 'passed-ok', kept_ok)
print('--- unbanded (set of window q-grams)')
for q in (6, 7, 8, 9, 10):
    rej = okfail = 0
    for r, dl, v, ori, win in calls:
        m = len(ori)
        ws = set(qgrams(win, q))
        cnt = sum(1 for x in qgrams(ori, q) if b'N' not in x and x in ws)
        thr = (m - q + 1) - dl * q
        if cnt < thr:
            rej += 1
            assert v is None
        elif v is None: okfail += 1
    print('q', q, 'rejected', rej, 'passed-but-failed', okfail)
print('--- segment-banded (window q-grams in 64-position segments, bands rounded out)')
for q in (6, 7, 8):
  for S in (64, 128, 256):
    rej = 0
    for r, dl, v, ori, win in calls:
        m = len(ori)
        segs = {}
        for j, x in enumerate(qgrams(win, q)): segs.setdefault(j // S, set()).add(x)
        cnt = 0
        for i, x in enumerate(qgrams(ori, q)):
            if b'N' in x: continue
            lo, hi = max(0, i - dl) // S, (i + dl) // S
            if any(x in segs.get(sg, ()) for sg in range(lo, hi + 1)): cnt += 1
        thr = (m - q + 1) - dl * q
        if cnt < thr:
            rej += 1
            assert v is None
    print('q', q, 'S', S, 'rejected', rej)
print('--- piece-wise banded (pieces of P read q-gram starts; window slice [a-dl, b-1+dl])')
def piece_count(ori, win, dl, q, P):
    m, w = len(ori), len(win)
    total = 0
    nq = m - q + 1
    for a in range(0, nq, P):
        b = min(nq, a + P)
        lo, hi = max(0, a - dl), min(w - q, b - 1 + dl)
        ws = set(win[j:j+q] for j in range(lo, hi + 1) if b'N' not in win[j:j+q])
        total += sum(1 for i in range(a, b) if b'N' not in ori[i:i+q] and ori[i:i+q] in ws)
    return total
for q in (6, 7):
  for P in (128, 256, 512):
    rej = 0
    for r, dl, v, ori, win in calls:
        cnt = piece_count(ori, win, dl, q, P)
        if cnt < (len(ori) - q + 1) - dl * q:
            rej += 1
            assert v is None
    print('q', q, 'P', P, 'rejected', rej)
