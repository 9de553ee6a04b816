"""CPU model of the systolic long-read LV (csrc/lv.cuh lv_sys), step for
step, lane for lane, checked against the oracle's bounded_distance (REF
src/edit_distance.cpp:19-75).  This pins the algorithm -- the row-block
layout ending at row m, the virtual rows, the band bounds ("+1 per row"
under the block above, hin = +1 past it), K columns per step with a
one-step skew (the kernel runs K = 2; 1 and 4 are checked too: measured
1 / 2 / generic 3-4 columns per step, C4 87 / 77 / 78-79 ms), and the early stop -- on small sizes the CPU runs in seconds; the kernel itself is
checked on the GPU by tests/test_gpu_parity.py::test_lv_long_limits_vs_oracle
and the lowered-threshold LV suite (tests/test_gpu_solo.py)."""
import random

import pytest

from oracle import oracle as O

M64 = (1 << 64) - 1


def _popc(x: int) -> int:
    return bin(x & M64).count("1")


def lv_sys_model(read: str, win: str, dl: int, K: int = 2) -> int | None:
    """lv_sys as the warp runs it: 32 lanes, lane l owns blocks l, l + 32, ...;
    block b runs columns K (p - 1) + 1 .. K p at step p + b (the kernel: K = 2)."""
    m, w = len(read), len(win)
    B = (m + 63) >> 6
    jend = min(w, m + dl)
    inf, never = 0x3FFFFFFF, 1 << 30
    best = [m if m <= dl else inf] * 32
    if jend >= 1 and B > 0:
        L = [dict(b=lane - 32, tsw=1 if lane < B else never, ts=never, te=-1, js=0, je=0, ae=-never,
                  Pv=0, Mv=0, q={}, sc=0, fresh=False, pub=0, act=False, gp=0) for lane in range(32)]
        for t in range(1, (jend + K - 1) // K + B):
            pubs = [s["pub"] for s in L]  # the shuffle reads last step's values
            for lane, s in enumerate(L):
                rcv = pubs[(lane + 31) % 32]
                if t == s["tsw"]:  # next block of this lane
                    b = s["b"] = s["b"] + 32
                    r0 = m - 64 * (B - b) + 1
                    js, je = max(1, r0 - dl), min(jend, r0 + 63 + dl)
                    s["js"], s["je"] = js, je
                    s["ts"], s["te"] = (js + K - 1) // K + b, (je + K - 1) // K + b
                    s["tsw"] = s["te"] + 1 if b + 32 < B else never
                    s["ae"] = min(jend, r0 - 1 + dl) if b > 0 else -never
                    s["q"] = {c: sum(1 << k for k in range(64) if 0 <= r0 - 1 + k < m and read[r0 - 1 + k] == c)
                              for c in "ACGT"}
                    if js == 1:  # exact column 0
                        t1 = 1 - r0
                        s["Pv"] = M64 if t1 <= 0 else (0 if t1 >= 64 else (M64 << t1) & M64)
                        s["Mv"], s["sc"], s["fresh"] = ~s["Pv"] & M64, abs(r0 + 63), False
                    else:  # upper bound below the block above
                        s["Pv"], s["Mv"], s["fresh"] = M64, 0, True
                    s["gp"] = js - 1
                b = s["b"]
                s["act"] = act = s["ts"] <= t <= s["te"]
                if not act:
                    continue
                j0 = K * (t - b - 1) + 1
                sce = rcv >> (2 * K)
                ha = [((rcv >> (2 * (K - 1 - c))) & 3) - 1 for c in range(K)]  # the block above's houts
                hout = [0] * K
                for c in range(K):
                    j = j0 + c
                    if j < s["js"] or j > s["je"]:
                        continue
                    hin = ha[c] if j <= s["ae"] else 1
                    if s["fresh"]:  # the block above's D at column j, + 64 ("+1 per row")
                        above = sce - sum(ha[c2] for c2 in range(c + 1, K) if j0 + c2 <= s["ae"])
                        s["sc"], s["fresh"] = above - hin + 64, False
                    g = win[s["gp"]]
                    s["gp"] += 1
                    eq0 = 0 if g == "N" else s["q"][g]
                    hneg = 1 if hin < 0 else 0
                    Pv, Mv = s["Pv"], s["Mv"]
                    Xv = eq0 | Mv
                    eq = eq0 | hneg
                    Xh = ((((eq & Pv) + Pv) & M64) ^ Pv) | eq
                    Ph = (Mv | ~(Xh | Pv)) & M64
                    Mh = Pv & Xh
                    hout[c] = (Ph >> 63) - (Mh >> 63)
                    Ph = ((Ph << 1) & M64) | (1 if hin > 0 else 0)
                    Mh = ((Mh << 1) & M64) | hneg
                    s["Pv"], s["Mv"] = (Mh | ~(Xv | Ph)) & M64, Ph & Xv
                    s["sc"] += hout[c]
                    if b == B - 1:
                        best[lane] = min(best[lane], s["sc"])  # D[m][j]
                pub = s["sc"]
                for c in range(K):
                    pub = (pub << 2) | (hout[c] + 1)
                s["pub"] = pub
            if t % 64 == 0:  # early stop (K-column skew between neighbours: + K)
                thr = min(dl + K, min(best) + K - 1)
                if all(not s["act"] or s["sc"] - _popc(s["Pv"]) > thr for s in L):
                    break
    v = min(best)
    return v if v <= dl else None


def _mutate(rng: random.Random, s: str, rate: float) -> str:
    out = []
    for ch in s:
        r = rng.random()
        if r < rate / 3:
            out.append(rng.choice("ACGTN"))
        elif r < 2 * rate / 3:
            pass
        elif r < rate:
            out += [ch, rng.choice("ACGT")]
        else:
            out.append(ch)
    return "".join(out)


@pytest.mark.parametrize("K", [1, 2, 4])
def test_lv_sys_model_vs_oracle(K):
    rng = random.Random(960 + K)
    n = 0
    for _ in range(160):
        m = rng.choice([1, 2, 5, 30, 63, 64, 65, 127, 128, 129, 200, 257])
        dl = rng.choice([16, 17, 20, 33, 40, 64, 70])
        read = "".join(rng.choice("ACGTN" if rng.random() < 0.1 else "ACGT") for _ in range(m))
        win = _mutate(rng, read, rng.choice([0.0, 0.02, 0.1, 0.3, 0.6])) + \
            "".join(rng.choice("ACGT") for _ in range(dl + 5))
        win = win[:rng.choice([len(win), min(len(win), m + dl), max(0, m - rng.randint(0, 20))] +
                           [max(0, m + dl - k) for k in (1, 2, 3)])]
        assert lv_sys_model(read, win, dl, K) == O.or_bounded_distance(read, win, dl), (m, dl, len(win))
        n += 1
    assert n == 160
