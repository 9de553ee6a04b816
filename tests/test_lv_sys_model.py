"""CPU model of the systolic long-read LV (csrc/lv.cuh lv_sys), step for
step, lane for lane, checked against the oracle's bounded_distance (REF
src/edit_distance.cpp:19-75).  This pins the algorithm -- the row-block
layout ending at row m, the virtual rows, the band bounds ("+1 per row"
under the block above, hin = +1 past it), the one-step skew and the early
stop -- on small sizes the CPU runs in seconds; the kernel itself is
checked on the GPU by tests/test_gpu_parity.py::test_lv_long_limits_vs_oracle
and the lowered-threshold LV suite (tests/test_gpu_solo.py)."""
import random

from oracle import oracle as O

M64 = (1 << 64) - 1


def _popc(x: int) -> int:
    return bin(x & M64).count("1")


def lv_sys_model(read: str, win: str, dl: int) -> int | None:
    """lv_sys as the warp runs it: 32 lanes, lane l owns blocks l, l + 32, ..."""
    m, w = len(read), len(win)
    B = (m + 63) >> 6
    jend = min(w, m + dl)
    inf = 0x3FFFFFFF
    best = [m if m <= dl else inf] * 32
    if jend >= 1 and B > 0:
        L = [dict(b=lane - 32, r0=0, js=1, je=0, ae=0, Pv=0, Mv=0, q={}, sc=0, fresh=False, pub=0, act=False)
             for lane in range(32)]
        for t in range(1, jend + B):
            pubs = [s["pub"] for s in L]  # the shuffle reads last step's values
            for lane, s in enumerate(L):
                rcv = pubs[(lane + 31) % 32]
                if t - s["b"] > s["je"] and s["b"] + 32 < B:  # next block of this lane
                    b = s["b"] = s["b"] + 32
                    r0 = s["r0"] = m - 64 * (B - b) + 1
                    s["js"], s["je"], s["ae"] = max(1, r0 - dl), min(jend, r0 + 63 + dl), min(jend, r0 - 1 + dl)
                    s["q"] = {c: sum(1 << k for k in range(64) if 0 <= r0 - 1 + k < m and read[r0 - 1 + k] == c)
                              for c in "ACGT"}
                    if s["js"] == 1:  # exact column 0
                        t1 = 1 - r0
                        s["Pv"] = M64 if t1 <= 0 else (0 if t1 >= 64 else (M64 << t1) & M64)
                        s["Mv"], s["sc"], s["fresh"] = ~s["Pv"] & M64, abs(r0 + 63), False
                    else:  # upper bound below the block above
                        s["Pv"], s["Mv"], s["fresh"] = M64, 0, True
                b = s["b"]
                j = t - b
                s["act"] = act = b >= 0 and s["js"] <= j <= s["je"]
                if not act:
                    continue
                g = win[j - 1]
                eq0 = 0 if g == "N" else s["q"][g]
                hin, scin = 1, 0
                if b > 0 and j <= s["ae"]:
                    hin, scin = (rcv & 3) - 1, rcv >> 2
                hneg = 1 if hin < 0 else 0
                Pv, Mv = s["Pv"], s["Mv"]
                Xv = eq0 | Mv
                eq = eq0 | hneg
                Xh = ((((eq & Pv) + Pv) & M64) ^ Pv) | eq
                Ph = (Mv | ~(Xh | Pv)) & M64
                Mh = Pv & Xh
                hout = (Ph >> 63) - (Mh >> 63)
                Ph = ((Ph << 1) & M64) | (1 if hin > 0 else 0)
                Mh = ((Mh << 1) & M64) | hneg
                s["Pv"], s["Mv"] = (Mh | ~(Xv | Ph)) & M64, Ph & Xv
                if s["fresh"]:
                    s["sc"], s["fresh"] = scin + _popc(s["Pv"]) - _popc(s["Mv"]), False
                else:
                    s["sc"] += hout
                s["pub"] = (s["sc"] << 2) | (hout + 1)
                if b == B - 1:
                    best[lane] = min(best[lane], s["sc"])  # D[m][j]
            if t % 64 == 0:  # early stop
                thr = min(dl + 1, min(best))
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


def test_lv_sys_model_vs_oracle():
    rng = random.Random(960)
    n = 0
    for _ in range(160):
        m = rng.choice([1, 5, 30, 63, 64, 65, 127, 128, 129, 200, 257])
        dl = rng.choice([16, 20, 33, 40, 64, 70])
        read = "".join(rng.choice("ACGTN" if rng.random() < 0.1 else "ACGT") for _ in range(m))
        win = _mutate(rng, read, rng.choice([0.0, 0.02, 0.1, 0.3, 0.6])) + \
            "".join(rng.choice("ACGT") for _ in range(dl + 5))
        win = win[:rng.choice([len(win), min(len(win), m + dl), max(0, m - rng.randint(0, 20))])]
        assert lv_sys_model(read, win, dl) == O.or_bounded_distance(read, win, dl), (m, dl, len(win))
        n += 1
    assert n == 160
