"""TEST INFRASTRUCTURE ONLY -- ctypes access to the parity oracles.

  OracleIndex / or_*   plain-C restatement (oracle/snap_oracle.c), built by
                       `make -C oracle` into oracle/build/liboracle.so
  RefIndex / ref_*     the reference library itself, compiled in place from
                       /root/reference by `make -C oracle ref` into
                       oracle/_ref/libseedaln_ref.so (travels prebuilt)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libseedaln_ref.so")
REF_DIR = "/root/reference/proj"

RESULT_DTYPE = np.dtype(
    [("position", "<u8"), ("distance", "<i4"), ("gap", "<i4"), ("kind", "u1"),
     ("has_position", "u1"), ("direction", "u1"), ("reserved", "u1", (5,))]
)
STAT_FIELDS = (
    "reads", "reads_too_short", "seed_lookups", "seeds_skipped_n", "seeds_skipped_popular",
    "reads_all_seeds_popular", "distance_calls", "distance_calls_after_first",
    "early_out_after_first", "dp_cells", "multi_early_exits", "pruning_exits",
    "first_scored_was_best", "single_hits", "multiple_hits", "not_found",
    "hits_consumed", "window_bases", "read_bases", "overflow_reads",
)


class Params(C.Structure):
    _fields_ = [("seed_size", C.c_int32), ("seeds_to_try", C.c_int32),
                ("max_distance", C.c_int32), ("confidence_threshold", C.c_int32),
                ("max_hits", C.c_int32), ("bucket_size", C.c_int32),
                ("force_max_dlimit", C.c_int32)]

    @classmethod
    def of(cls, p) -> "Params":
        return cls(p.seed_size, p.seeds_to_try, p.max_distance, p.confidence_threshold, p.max_hits,
                   p.bucket_size, 1 if p.force_max_dlimit else 0)


class Stats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in STAT_FIELDS]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f in STAT_FIELDS}


def build(with_ref: bool | None = None) -> None:
    """make -C oracle (and `ref` when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if with_ref is None:
        with_ref = os.path.isdir(REF_DIR)
    if with_ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REF_DIR}"], check=True)
        # the C++ drop-in test program (needs the product library built first)
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1111_5572_b200", "lib", "libsnapb200.so")):
            subprocess.run(["make", "-s", "-C", HERE, "dropin", f"REF={REF_DIR}"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


_o = None
_r = None
P64 = C.POINTER(C.c_uint64)


def _u64p(a):
    return a.ctypes.data_as(P64)


class _OrIndex(C.Structure):
    _fields_ = [("seed_size", C.c_int), ("n_keys", C.c_uint64), ("n_positions", C.c_uint64),
                ("keys", C.c_void_p), ("offsets", C.c_void_p), ("positions", C.c_void_p),
                ("n_queries", C.c_uint64), ("queries", C.c_void_p), ("misses", C.c_uint64)]


class _OrGenome(C.Structure):
    _fields_ = [("len", C.c_uint64), ("packed", C.c_void_p), ("nmask", C.c_void_p)]


def olib():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            build(with_ref=False)
        lib = C.CDLL(ORACLE_SO)
        lib.or_seed_offsets.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int)]
        lib.or_pack_seed.argtypes = [C.c_char_p, C.c_int, P64]
        lib.or_packed_rc.argtypes = [C.c_uint64, C.c_int]
        lib.or_packed_rc.restype = C.c_uint64
        lib.or_index_build.argtypes = [C.POINTER(_OrGenome), C.c_int, C.POINTER(_OrIndex)]
        lib.or_index_build_for_reads.argtypes = [C.POINTER(_OrGenome), C.c_int, C.c_int, C.c_void_p, P64,
                                                 C.c_uint64, C.c_int, C.POINTER(_OrIndex)]
        lib.or_index_free.argtypes = [C.POINTER(_OrIndex)]
        lib.or_lookup.argtypes = [C.POINTER(_OrIndex), C.c_char_p, C.POINTER(C.c_void_p), P64,
                                  C.POINTER(C.c_void_p), P64]
        lib.or_bounded_distance.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, C.c_int, P64]
        lib.or_full_dp_distance.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64]
        lib.or_align_batch.argtypes = [C.POINTER(_OrIndex), C.POINTER(_OrGenome), C.POINTER(Params),
                                       C.c_void_p, P64, C.c_uint64, C.c_void_p, C.POINTER(Stats), C.c_int]
        lib.or_pack_genome.argtypes = [C.c_char_p, C.c_uint64, P64, P64]
        _o = lib
    return _o


def rlib():
    global _r
    if _r is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref needs /root/reference)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_create.argtypes = [P64, C.c_uint64, P64, C.c_uint64, C.c_uint64, C.c_int]
        lib.ref_create.restype = C.c_void_p
        lib.ref_create_from_csr.argtypes = [P64, C.c_uint64, P64, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p,
                                            C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64]
        lib.ref_create_from_csr.restype = C.c_void_p
        lib.ref_destroy.argtypes = [C.c_void_p]
        lib.ref_index_info.argtypes = [C.c_void_p, P64, P64]
        lib.ref_genome_checksum.argtypes = [C.c_void_p]
        lib.ref_genome_checksum.restype = C.c_uint64
        lib.ref_lookup.argtypes = [C.c_void_p, C.c_char_p, C.c_int, P64, P64, P64, P64, C.c_uint64]
        lib.ref_bounded_distance.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.c_int, P64]
        lib.ref_full_dp_distance.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64]
        lib.ref_seed_offsets.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int)]
        lib.ref_pack_seed.argtypes = [C.c_char_p, C.c_int, P64]
        lib.ref_packed_rc.argtypes = [C.c_uint64, C.c_int]
        lib.ref_packed_rc.restype = C.c_uint64
        lib.ref_tracker_replay.argtypes = [C.c_int, C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int64)]
        lib.ref_align_batch.argtypes = [C.c_void_p, C.POINTER(Params), C.c_void_p, P64, C.c_uint64,
                                        C.c_void_p, C.POINTER(Stats), C.c_int]
        lib.ref_genome_from_fasta.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.ref_genome_free.argtypes = [C.c_void_p]
        lib.ref_genome_info.argtypes = [C.c_void_p, P64, P64, P64]
        lib.ref_genome_words.argtypes = [C.c_void_p, C.POINTER(P64), P64, C.POINTER(P64), P64]
        lib.ref_genome_contig.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_char_p), P64, P64]
        lib.ref_run_index.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        lib.ref_load_index.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.ref_referee_create.argtypes = [P64, C.c_uint64, P64, C.c_uint64, C.c_uint64]
        lib.ref_referee_create.restype = C.c_void_p
        lib.ref_referee_destroy.argtypes = [C.c_void_p]
        lib.ref_oracle_align.argtypes = [C.c_void_p, C.POINTER(Params), C.c_void_p, P64, C.c_uint64, C.c_void_p,
                                         C.c_int]
        lib.ref_oracle_scan.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_int, C.c_int, P64,
                                        C.POINTER(C.c_int32), C.POINTER(C.c_uint8), C.c_uint64]
        lib.ref_oracle_scan.restype = C.c_int64
        lib.ref_run_simulate.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_uint64, C.c_double,
                                         C.c_double, C.c_double, C.c_double, C.c_uint64]
        _r = lib
    return _r


# ----------------------------------------------------------------- pure helpers

def or_seed_offsets(length: int, s: int, n: int) -> list[int]:
    buf = (C.c_int * max(n, 1))()
    k = olib().or_seed_offsets(length, s, n, buf)
    return list(buf[:k])


def ref_seed_offsets(length: int, s: int, n: int) -> list[int]:
    buf = (C.c_int * max(n, 1))()
    k = rlib().ref_seed_offsets(length, s, n, buf)
    return list(buf[:k])


def or_bounded_distance(read: str, win: str, d_limit: int) -> int | None | str:
    cells = C.c_uint64()
    v = olib().or_bounded_distance(read.encode(), len(read), win.encode(), len(win), d_limit, C.byref(cells))
    return "throws" if v == -2 else (None if v < 0 else v)


def ref_bounded_distance(read: str, win: str, d_limit: int) -> int | None | str:
    cells = C.c_uint64()
    v = rlib().ref_bounded_distance(read.encode(), len(read), win.encode(), len(win), d_limit, C.byref(cells))
    return "throws" if v == -2 else (None if v < 0 else v)


def or_full_dp(read: str, win: str) -> int:
    return olib().or_full_dp_distance(read.encode(), len(read), win.encode(), len(win))


def or_packed_rc(key: int, s: int) -> int:
    return olib().or_packed_rc(key, s)


def or_pack_seed(seed: str) -> int | None:
    k = C.c_uint64()
    return k.value if olib().or_pack_seed(seed.encode(), len(seed), C.byref(k)) else None


def pack_genome(seq: bytes) -> tuple[np.ndarray, np.ndarray]:
    n = len(seq)
    packed = np.zeros(max(1, (n + 31) // 32), np.uint64)
    nmask = np.zeros(max(1, (n + 63) // 64), np.uint64)
    if olib().or_pack_genome(seq, n, _u64p(packed), _u64p(nmask)) != 0:
        raise ValueError("illegal character")
    return packed[:(n + 31) // 32], nmask[:(n + 63) // 64]


# ----------------------------------------------------------------- indexes

class OracleIndex:
    """C restatement: CSR index + Aligner::align.

    With `for_reads=(n_seeds, bases, offsets)` the index is restricted to the
    keys those reads can probe (or_index_build_for_reads): the oracle for
    3.1 Gbp genomes, where the full CSR would not fit this container.  Any
    probe of another key is counted in `misses()`; align_arrays asserts 0.
    """

    def __init__(self, packed: np.ndarray, nmask: np.ndarray, length: int, s: int, for_reads=None,
                 threads: int = 8):
        self.packed = np.ascontiguousarray(packed, np.uint64)
        self.nmask = np.ascontiguousarray(nmask, np.uint64)
        self.g = _OrGenome(length, self.packed.ctypes.data, self.nmask.ctypes.data)
        self.ix = _OrIndex()
        if for_reads is None:
            rc = olib().or_index_build(C.byref(self.g), s, C.byref(self.ix))
        else:
            n_seeds, bases, offsets = for_reads
            offsets = np.ascontiguousarray(offsets, np.uint64)
            b = np.ascontiguousarray(bases, np.uint8)
            rc = olib().or_index_build_for_reads(C.byref(self.g), s, n_seeds, b.ctypes.data, _u64p(offsets),
                                                 offsets.size - 1, threads, C.byref(self.ix))
        if rc:
            raise ValueError(f"oracle index build failed ({rc})")

    def misses(self) -> int:
        return int(self.ix.misses)

    def __del__(self):
        if _o is not None and getattr(self, "ix", None) is not None:
            _o.or_index_free(C.byref(self.ix))
            self.ix = None

    def lookup(self, seed: str) -> tuple[list[int], list[int]]:
        f, r = C.c_void_p(), C.c_void_p()
        nf, nr = C.c_uint64(), C.c_uint64()
        olib().or_lookup(C.byref(self.ix), seed.encode(), C.byref(f), C.byref(nf), C.byref(r), C.byref(nr))
        fw = list(C.cast(f, C.POINTER(C.c_uint32))[:nf.value]) if nf.value else []
        rv = list(C.cast(r, C.POINTER(C.c_uint32))[:nr.value]) if nr.value else []
        return fw, rv

    def align_arrays(self, params, bases, offsets, threads: int = 1):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        res = np.zeros(n, RESULT_DTYPE)
        st = Stats()
        p = Params.of(params)
        b = np.ascontiguousarray(np.frombuffer(bases, np.uint8) if isinstance(bases, (bytes, bytearray)) else bases,
                                 np.uint8)
        rc = olib().or_align_batch(C.byref(self.ix), C.byref(self.g), C.byref(p), b.ctypes.data,
                                   _u64p(offsets), n, res.ctypes.data, C.byref(st), threads)
        if rc:
            raise ValueError(f"or_align_batch failed ({rc})")
        if self.ix.queries and self.ix.misses:
            raise AssertionError(f"restricted oracle index probed {self.ix.misses} keys it was not built for")
        return res, st.as_dict()


class RefIndex:
    """The reference library (oracle/_ref): SeedIndex::build + Aligner::align."""

    def __init__(self, packed: np.ndarray, nmask: np.ndarray, length: int, s: int):
        lib = rlib()
        self.packed = np.ascontiguousarray(packed, np.uint64)
        self.nmask = np.ascontiguousarray(nmask, np.uint64)
        self.h = lib.ref_create(_u64p(self.packed), self.packed.size, _u64p(self.nmask), self.nmask.size,
                                length, s)
        if not self.h:
            raise ValueError(lib.ref_last_error().decode())
        self.s = s

    @classmethod
    def from_restricted(cls, oi: "OracleIndex") -> "RefIndex":
        """The reference's own SeedIndex + Aligner over the key-restricted CSR
        of an OracleIndex built with for_reads=: loaded through the
        reference's load_index_file (ref_create_from_csr), so the reference's
        unmodified lookup and Aligner::align run at 3.1 Gbp, where its
        single-threaded full build does not fit a bounded run.  Exact for the
        reads the restricted index was built for."""
        self = cls.__new__(cls)
        lib = rlib()
        self.packed, self.nmask = oi.packed, oi.nmask
        self.h = lib.ref_create_from_csr(_u64p(self.packed), self.packed.size, _u64p(self.nmask), self.nmask.size,
                                         oi.g.len, oi.ix.seed_size, oi.ix.keys, oi.ix.n_keys, oi.ix.offsets,
                                         oi.ix.positions, oi.ix.n_positions)
        if not self.h:
            raise ValueError(lib.ref_last_error().decode())
        self.s = oi.ix.seed_size
        return self

    def __del__(self):
        if _r is not None and getattr(self, "h", None):
            _r.ref_destroy(self.h)
            self.h = None

    def info(self) -> tuple[int, int]:
        d, t = C.c_uint64(), C.c_uint64()
        rlib().ref_index_info(self.h, C.byref(d), C.byref(t))
        return d.value, t.value

    def lookup(self, seed: str, cap: int = 1 << 16) -> tuple[list[int], list[int]]:
        f = np.zeros(cap, np.uint64)
        r = np.zeros(cap, np.uint64)
        nf, nr = C.c_uint64(), C.c_uint64()
        rc = rlib().ref_lookup(self.h, seed.encode(), len(seed), _u64p(f), C.byref(nf), _u64p(r),
                               C.byref(nr), cap)
        if rc:
            raise ValueError(rlib().ref_last_error().decode())
        return [int(x) for x in f[:nf.value]], [int(x) for x in r[:nr.value]]

    def align_arrays(self, params, bases, offsets, threads: int = 1):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        res = np.zeros(n, RESULT_DTYPE)
        st = Stats()
        p = Params.of(params)
        b = np.ascontiguousarray(np.frombuffer(bases, np.uint8) if isinstance(bases, (bytes, bytearray)) else bases,
                                 np.uint8)
        rc = rlib().ref_align_batch(self.h, C.byref(p), b.ctypes.data, _u64p(offsets), n,
                                    res.ctypes.data, C.byref(st), threads)
        if rc:
            raise ValueError(rlib().ref_last_error().decode())
        return res, st.as_dict()


# ----------------------------------------------------------------- reference files

def ref_genome_from_fasta(path: str):
    """PackedGenome::from_fasta of the reference -> (packed, nmask, length,
    contigs [(name, start, length)], checksum), or (code, message) on error."""
    lib = rlib()
    h = C.c_void_p()
    rc = lib.ref_genome_from_fasta(os.fsencode(path), C.byref(h))
    if rc:
        return rc, lib.ref_last_error().decode()
    try:
        n, nc, ck = C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib.ref_genome_info(h, C.byref(n), C.byref(nc), C.byref(ck))
        pp, pn = P64(), P64()
        a, b = C.c_uint64(), C.c_uint64()
        lib.ref_genome_words(h, C.byref(pp), C.byref(a), C.byref(pn), C.byref(b))
        packed = np.ctypeslib.as_array(pp, (a.value,)).copy() if a.value else np.zeros(0, np.uint64)
        nmask = np.ctypeslib.as_array(pn, (b.value,)).copy() if b.value else np.zeros(0, np.uint64)
        contigs = []
        for i in range(nc.value):
            nm, st, ln = C.c_char_p(), C.c_uint64(), C.c_uint64()
            lib.ref_genome_contig(h, i, C.byref(nm), C.byref(st), C.byref(ln))
            contigs.append((nm.value.decode(), st.value, ln.value))
        return packed, nmask, n.value, contigs, ck.value
    finally:
        lib.ref_genome_free(h)


def ref_run_index(fasta: str, index_path: str, seed_size: int):
    """run_index (REF src/driver.cpp:37-45): 0, or (code, message)."""
    lib = rlib()
    rc = lib.ref_run_index(os.fsencode(fasta), os.fsencode(index_path), seed_size)
    return 0 if rc == 0 else (rc, lib.ref_last_error().decode())


def ref_run_simulate(fasta: str, out: str, count: int, read_length: int = 100, snp_rate: float = 0.0009,
                     indel_mutation_rate: float = 0.0001, seq_error_rate: float = 0.02,
                     indel_error_fraction: float = 0.0, rng_seed: int = 1):
    """run_simulate (REF src/driver.cpp:158-168): FASTQ with truth-encoded names."""
    lib = rlib()
    rc = lib.ref_run_simulate(os.fsencode(fasta), os.fsencode(out), count, read_length, snp_rate,
                              indel_mutation_rate, seq_error_rate, indel_error_fraction, rng_seed)
    if rc:
        raise RefError(rc, lib.ref_last_error().decode())


REF_CLI = os.path.join(HERE, "_ref", "seedaln_ref_cli")


def ref_run_align(index_path: str, fastq: str, out: str, params, threads: int = 1, chunk_min: int = 4 << 20,
                  stable: bool = True, tolerance: int = 50, report_path: str | None = None,
                  command_line: str = "seedaln align") -> str:
    """run_align (REF src/driver.cpp:47-156) of the reference, run out of
    process (oracle/ref_cli.cpp explains why); returns EvalReport::to_text()."""
    p = params
    args = [REF_CLI, "align", index_path, fastq, out, str(p.seed_size), str(p.seeds_to_try), str(p.max_distance),
            str(p.confidence_threshold), str(p.max_hits), str(p.bucket_size), "1" if p.force_max_dlimit else "0",
            str(threads), str(chunk_min), "1" if stable else "0", str(tolerance), report_path or "-", command_line]
    r = subprocess.run(args, capture_output=True, text=True)
    if r.returncode != 0:
        line = (r.stdout.strip().splitlines() or ["ERROR 2 " + r.stderr.strip()])[-1]
        _, code, msg = line.split(" ", 2)
        raise RefError(int(code), msg)
    return r.stdout


class RefLoadedIndex(RefIndex):
    """load_index_file (REF src/seed_index.cpp:173-228) of the reference."""

    def __init__(self, path: str):  # noqa: D401 -- no RefIndex.__init__ (no build)
        lib = rlib()
        h = C.c_void_p()
        rc = lib.ref_load_index(os.fsencode(path), C.byref(h))
        if rc:
            self.h = None
            raise RefError(rc, lib.ref_last_error().decode())
        self.h = h.value


class RefReferee:
    """OracleContext + oracle_align / oracle_scan of the reference (REF src/eval.cpp:122-306)."""

    def __init__(self, packed, nmask, length):
        lib = rlib()
        self.packed = np.ascontiguousarray(packed, np.uint64)
        self.nmask = np.ascontiguousarray(nmask, np.uint64)
        self.h = lib.ref_referee_create(_u64p(self.packed), self.packed.size, _u64p(self.nmask), self.nmask.size,
                                        length)
        if not self.h:
            raise RuntimeError(lib.ref_last_error().decode())

    def __del__(self):
        if _r is not None and getattr(self, "h", None):
            _r.ref_referee_destroy(self.h)
            self.h = None

    def align(self, params, bases, offsets, threads=8):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        res = np.zeros(n, RESULT_DTYPE)
        b = np.ascontiguousarray(bases, np.uint8)
        p = Params.of(params)
        if rlib().ref_oracle_align(self.h, C.byref(p), b.ctypes.data, _u64p(offsets), n, res.ctypes.data, threads):
            raise RefError(1, rlib().ref_last_error().decode())
        return res

    def scan(self, read: bytes, d_limit: int, bucket: int, cap: int = 1 << 16):
        pos = np.zeros(cap, np.uint64)
        dist = np.zeros(cap, np.int32)
        dr = np.zeros(cap, np.uint8)
        n = rlib().ref_oracle_scan(self.h, read, len(read), d_limit, bucket, _u64p(pos),
                                   dist.ctypes.data_as(C.POINTER(C.c_int32)), dr.ctypes.data_as(C.POINTER(C.c_uint8)),
                                   cap)
        if n < 0:
            raise RefError(1, rlib().ref_last_error().decode())
        n = min(n, cap)
        return [(int(pos[i]), int(dist[i]), int(dr[i])) for i in range(n)]


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code, self.msg = code, msg


def ref_tracker_replay(merge_radius: int, ops: list[tuple[int, int, int]]) -> list[tuple[int, int, int, int]]:
    flat = (C.c_int64 * (3 * len(ops)))(*[v for op in ops for v in op])
    out = (C.c_int64 * (4 * len(ops)))()
    rlib().ref_tracker_replay(merge_radius, flat, len(ops), out)
    return [tuple(out[4 * i:4 * i + 4]) for i in range(len(ops))]


def compare_results(a: np.ndarray, b: np.ndarray) -> list[int]:
    """Indices of reads whose AlignmentResult differs in any field
    (kind, has_position, position, direction, distance, gap)."""
    diff = np.zeros(a.size, bool)
    for f in ("kind", "has_position", "position", "direction", "distance", "gap"):
        diff |= a[f] != b[f]
    return np.nonzero(diff)[0].tolist()
