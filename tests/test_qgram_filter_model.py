"""CPU model of the long-read LV's exact q-gram pre-test (csrc/lv.cuh
qgram_reject): whenever it rejects a (read, window, d_limit), the oracle's
bounded_distance (REF src/edit_distance.cpp:19-75) must be "more than
d_limit".  Random pairs across the close / diverged / unrelated range, with
N bases and cut windows, at limits where the bound can bite."""
import random

from oracle import oracle as O

Q, PIECE = 6, 128  # kQfQ, kQfPiece


def qgram_reject_model(read: str, win: str, dl: int) -> bool:
    m, w = len(read), len(win)
    nq = m - Q + 1
    thr = nq - dl * Q
    if thr <= 0:
        return False
    total = 0
    for a0 in range(0, nq, PIECE):
        b0 = min(nq, a0 + PIECE)
        lo, hi = max(0, a0 - dl), min(w - Q, b0 - 1 + dl)
        band = {win[j:j + Q] for j in range(lo, hi + 1) if "N" not in win[j:j + Q]}
        total += sum(1 for i in range(a0, b0) if "N" not in read[i:i + Q] and read[i:i + Q] in band)
        if total >= thr:
            return False
        if total + (nq - b0) < thr:
            return True
    return total < thr


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


def test_qgram_filter_never_rejects_a_close_window():
    rng = random.Random(83)
    rejected = kept_close = 0
    for _ in range(400):
        m = rng.choice([40, 100, 250, 600, 1000])
        dl = rng.choice([2, 5, 10, 20, 40, 83])
        read = "".join(rng.choice("ACGTN" if rng.random() < 0.02 else "ACGT") for _ in range(m))
        win = _mutate(rng, read, rng.choice([0.0, 0.01, 0.03, 0.06, 0.1, 0.2, 0.4])) + \
            "".join(rng.choice("ACGT") for _ in range(dl + 5))
        win = win[:rng.choice([len(win), min(len(win), m + dl), max(0, m - rng.randint(0, 30))])]
        want = O.or_bounded_distance(read, win, dl)
        if qgram_reject_model(read, win, dl):
            rejected += 1
            assert want is None, (m, dl, len(win), want)
        elif want is not None:
            kept_close += 1
    assert rejected > 50 and kept_close > 50  # the test exercises both sides
