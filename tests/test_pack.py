"""Host read packer (csrc/pack.cpp) on CPU: the batch path ships reads to the
GPU as three bit planes {lo, hi, n} instead of ASCII.  Every ISA variant must
equal a numpy restatement of the encoding, including ragged tails and bytes
outside {A,C,G,T,N} (marked lo = n = 1 so the seed kernel still fails the
read, REF src/genome.cpp:182-200)."""
import ctypes as C
import time

import numpy as np
import pytest

from paper_1111_5572_b200 import api


def _planes_np(b: np.ndarray, wpp: int) -> np.ndarray:
    n = b.size
    c = b.view(np.uint8)
    bad = ~np.isin(c, np.frombuffer(b"ACGTN", np.uint8))
    lo = (c == ord("C")) | (c == ord("T")) | bad
    hi = (c == ord("G")) | (c == ord("T"))
    nn = (c == ord("N")) | bad
    out = np.zeros((3, wpp), np.uint32)
    words = (n + 31) // 32
    for p, bits in enumerate((lo, hi, nn)):
        pad = np.zeros(words * 32, bool)
        pad[:n] = bits
        out[p, :words] = np.packbits(pad.reshape(-1, 32)[:, ::-1], axis=1).view(">u4").ravel()
    return out


def _pack(b: np.ndarray, isa: int):
    lib = api._load()
    f = lib.sab_debug_pack
    f.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_int]
    n = b.size
    wpp = (n + 31) // 32 + 2
    out = np.full((3, wpp), 0xDEADBEEF, np.uint32)
    rc = f(b.ctypes.data, n, out.ctypes.data, wpp, isa)
    return rc, out, wpp


@pytest.mark.parametrize("isa", [1, 2, 3])
@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 63, 64, 65, 1000, 4099])
def test_pack_matches_numpy(isa, n):
    rng = np.random.default_rng(n * 7 + isa)
    b = rng.choice(np.frombuffer(b"ACGTACGTACGTN", np.uint8), n).astype(np.uint8)
    if n > 10:  # a few bad characters: lowercase, IUPAC, punctuation, NUL
        for ch in b"acRY.\x00":
            b[rng.integers(0, n)] = ch
    rc, got, wpp = _pack(b, isa)
    if rc == api.SA_ERUNTIME:
        pytest.skip("ISA not supported on this CPU")
    assert rc == 0
    np.testing.assert_array_equal(got, _planes_np(b, wpp))


def test_pack_throughput_report():
    """Not a gate: prints the single-thread packing rate of the best ISA."""
    b = np.random.default_rng(0).choice(np.frombuffer(b"ACGT", np.uint8), 64 << 20).astype(np.uint8)
    for isa in (3, 2, 1):
        rc, _, _ = _pack(b[:64], isa)
        if rc == 0:
            break
    t0 = time.perf_counter()
    rc, _, _ = _pack(b, isa)
    dt = time.perf_counter() - t0
    assert rc == 0
    print(f"pack isa={isa}: {b.size / dt / 1e9:.1f} GB/s single thread")
