"""Python mirror of the reference's hot-path API over the C-ABI (ctypes).

Same names, argument meaning and error behaviour as the reference library
(REF = /root/reference/proj):

  AlignerParams / validate / effective_max_distance   REF include/seedaln/aligner.hpp:19-30
  ResultKind, Direction, AlignmentResult, AlignStats  REF aligner.hpp:32-66, seed_index.hpp:14
  PackedGenome (packed words + N mask)                REF include/seedaln/genome.hpp:36-85
  SeedIndex.build / lookup -> LookupResult            REF include/seedaln/seed_index.hpp:24-71
  Aligner(index, genome, params).align(read)          REF aligner.hpp:116-158
  align_read, seed_offsets, bounded_distance          REF aligner.hpp:160-163, :72, edit_distance.hpp:122

C++ exceptions map to Python ones: std::invalid_argument -> ValueError,
FormatError -> FormatError, runtime failures -> RuntimeError.

Every computation runs in libsnapb200.so on a CUDA device.  There is no CPU
fallback: if the library or a GPU is missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SNAP_B200_LIB") or os.path.join(_HERE, "lib", "libsnapb200.so")
SYNTH_PATH = os.path.join(_HERE, "lib", "libsnap_synth.so")

SA_OK, SA_EINVAL, SA_ERUNTIME, SA_EFORMAT, SA_EPARSE, SA_EIO = 0, 1, 2, 3, 4, 5
SA_INDEX_SNAPIDX1, SA_INDEX_SNAPGPU1 = 0, 1

RESULT_DTYPE = np.dtype(
    [("position", "<u8"), ("distance", "<i4"), ("gap", "<i4"), ("kind", "u1"),
     ("has_position", "u1"), ("direction", "u1"), ("reserved", "u1", (5,))]
)
assert RESULT_DTYPE.itemsize == 24

STAT_FIELDS = (
    "reads", "reads_too_short", "seed_lookups", "seeds_skipped_n", "seeds_skipped_popular",
    "reads_all_seeds_popular", "distance_calls", "distance_calls_after_first",
    "early_out_after_first", "dp_cells", "multi_early_exits", "pruning_exits",
    "first_scored_was_best", "single_hits", "multiple_hits", "not_found",
    # extensions
    "hits_consumed", "window_bases", "read_bases", "overflow_reads",
)
REFERENCE_STAT_FIELDS = STAT_FIELDS[:16]


class FormatError(RuntimeError):
    """Bad binary artifact or mismatched index (REF include/seedaln/errors.hpp:22-25)."""


class ParseError(RuntimeError):
    """Malformed FASTA/FASTQ text (REF include/seedaln/errors.hpp:10-19)."""


class IoError(RuntimeError):
    """File cannot be opened or written (REF include/seedaln/errors.hpp:27-30)."""


class ResultKind(enum.IntEnum):  # REF aligner.hpp:32
    SingleHit = 0
    MultipleHits = 1
    NotFound = 2


class Direction(enum.IntEnum):  # REF seed_index.hpp:14
    Forward = 0
    ReverseComplement = 1


class _Params(C.Structure):
    _fields_ = [("seed_size", C.c_int32), ("seeds_to_try", C.c_int32),
                ("max_distance", C.c_int32), ("confidence_threshold", C.c_int32),
                ("max_hits", C.c_int32), ("bucket_size", C.c_int32),
                ("force_max_dlimit", C.c_int32)]


class _Stats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in STAT_FIELDS]


class _AlignOptions(C.Structure):  # sa_align_options
    _fields_ = [("index_path", C.c_char_p), ("fastq_path", C.c_char_p), ("output_path", C.c_char_p),
                ("params", _Params), ("threads", C.c_uint32), ("chunk_min_bytes", C.c_uint64),
                ("stable_order", C.c_int32), ("tolerance", C.c_uint64), ("report_path", C.c_char_p),
                ("command_line", C.c_char_p), ("devices", C.POINTER(C.c_int32)), ("n_devices", C.c_int32),
                ("verify_index", C.c_int32)]


class _SimProfile(C.Structure):  # sa_sim_profile = SimProfile (REF simulator.hpp:17-26)
    _fields_ = [("read_length", C.c_uint64), ("snp_rate", C.c_double), ("indel_mutation_rate", C.c_double),
                ("seq_error_rate", C.c_double), ("indel_error_fraction", C.c_double), ("rng_seed", C.c_uint64)]


TRUTH_DTYPE = np.dtype([("contig", "<u8"), ("position", "<u8"), ("serial", "<u8"), ("direction", "u1"),
                        ("pad", "u1", (7,))])
assert TRUTH_DTYPE.itemsize == 32


class _EvalReport(C.Structure):  # sa_eval_report
    _fields_ = [(f, C.c_uint64) for f in ("total", "single", "multiple", "notfound", "correct", "wrong",
                                           "no_truth")] + [("elapsed_seconds", C.c_double), ("stats", _Stats)]


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -m paper_1111_5572_b200.build` "
            "(the aligner has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "sa_default_params": (None, [P(_Params)]),
        "sa_validate_params": (C.c_int, [P(_Params)]),
        "sa_seed_offsets": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32)]),
        "sa_create": (C.c_int, [P(C.c_uint64), C.c_uint64, P(C.c_uint64), C.c_uint64, C.c_uint64,
                                C.c_int32, P(C.c_int32), C.c_int32, P(C.c_void_p)]),
        "sa_destroy": (None, [C.c_void_p]),
        "sa_last_error": (C.c_char_p, [C.c_void_p]),
        "sa_align_batch": (C.c_int, [C.c_void_p, P(_Params), C.c_void_p, P(C.c_uint64), C.c_uint64,
                                     C.c_void_p, P(_Stats)]),
        "sa_align_device": (C.c_int, [C.c_void_p, P(_Params), C.c_void_p, C.c_void_p, C.c_uint64,
                                      C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
        "sa_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
        "sa_lookup_batch": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, P(C.c_uint32),
                                      P(C.c_uint64), P(C.c_uint32), P(C.c_uint64), P(C.c_uint32),
                                      C.c_uint32]),
        "sa_index_info": (C.c_int, [C.c_void_p, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]),
        "sa_bounded_distance_batch": (C.c_int, [C.c_char_p, P(C.c_uint64), C.c_char_p,
                                                P(C.c_uint64), P(C.c_int32), C.c_uint64,
                                                P(C.c_int32), C.c_int32]),
        "sa_host_alloc": (C.c_int, [P(C.c_void_p), C.c_uint64]),
        "sa_host_free": (None, [C.c_void_p]),
        "sa_last_timing": (C.c_int, [C.c_void_p, P(C.c_float), P(C.c_float)]),
        "sa_last_launches": (C.c_int, [C.c_void_p, P(C.c_uint64)]),
        "sa_last_kernel_times": (C.c_int, [C.c_void_p, P(C.c_float), P(C.c_float)]),
        "sa_genome_from_fasta": (C.c_int, [C.c_char_p, P(C.c_void_p)]),
        "sa_genome_from_words": (C.c_int, [P(C.c_uint64), C.c_uint64, P(C.c_uint64), C.c_uint64, C.c_uint64,
                                           P(C.c_char_p), P(C.c_uint64), P(C.c_uint64), C.c_uint64,
                                           P(C.c_void_p)]),
        "sa_genome_free": (None, [C.c_void_p]),
        "sa_genome_info": (C.c_int, [C.c_void_p, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]),
        "sa_genome_words": (C.c_int, [C.c_void_p, P(P(C.c_uint64)), P(C.c_uint64), P(P(C.c_uint64)),
                                      P(C.c_uint64)]),
        "sa_genome_contig": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_char_p), P(C.c_uint64), P(C.c_uint64)]),
        "sa_create_from_genome": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_int32), C.c_int32, P(C.c_void_p)]),
        "sa_index_write": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_char_p]),
        "sa_index_load": (C.c_int, [C.c_char_p, P(C.c_int32), C.c_int32, C.c_int32, P(C.c_void_p),
                                    P(C.c_void_p)]),
        "sa_index_csr": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, P(C.c_uint64), P(C.c_uint64),
                                   P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]),
        "sa_index_seed_size": (C.c_int, [C.c_void_p, P(C.c_int32)]),
        "sa_referee_create": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_void_p)]),
        "sa_referee_destroy": (None, [C.c_void_p]),
        "sa_referee_align": (C.c_int, [C.c_void_p, P(_Params), C.c_void_p, P(C.c_uint64), C.c_uint64, C.c_void_p]),
        "sa_referee_scan": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, P(C.c_uint64), C.c_uint64,
                                      P(C.c_uint64), C.c_void_p, C.c_uint64]),
        "sa_default_align_options": (None, [P(_AlignOptions)]),
        "sa_run_index": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int32, C.c_int32, C.c_int32]),
        "sa_run_align": (C.c_int, [P(_AlignOptions), P(_EvalReport)]),
        "sa_report_text": (C.c_int, [P(_EvalReport), C.c_char_p, C.c_uint64, P(C.c_uint64)]),
        "sa_default_sim_profile": (None, [P(_SimProfile)]),
        "sa_simulator_create": (C.c_int, [C.c_void_p, P(_SimProfile), P(C.c_void_p)]),
        "sa_simulator_destroy": (None, [C.c_void_p]),
        "sa_simulator_next": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
        "sa_run_simulate": (C.c_int, [C.c_char_p, C.c_char_p, C.c_uint64, P(_SimProfile), C.c_uint32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    """Names of the C-ABI entry points declared in include/snap_b200.h."""
    hdr = os.path.join(os.path.dirname(_HERE), "include", "snap_b200.h")
    import re
    txt = open(hdr).read()
    return sorted(set(re.findall(r"\b(sa_[a-z_]+)\s*\(", txt)))


def _raise(code: int, ctx=None):
    lib = _load()
    msg = lib.sa_last_error(ctx).decode(errors="replace")
    if code == SA_EINVAL:
        raise ValueError(msg)
    if code == SA_EFORMAT:
        raise FormatError(msg)
    if code == SA_EPARSE:
        raise ParseError(msg)
    if code == SA_EIO:
        raise IoError(msg)
    raise RuntimeError(msg)


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# ----------------------------------------------------------------------- params

@dataclass
class AlignerParams:
    """REF include/seedaln/aligner.hpp:19-30 (same defaults)."""
    seed_size: int = 20
    seeds_to_try: int = 25
    max_distance: int = -1
    confidence_threshold: int = 2
    max_hits: int = 300
    bucket_size: int = 32
    force_max_dlimit: bool = False

    def _c(self) -> _Params:
        return _Params(self.seed_size, self.seeds_to_try, self.max_distance,
                       self.confidence_threshold, self.max_hits, self.bucket_size,
                       1 if self.force_max_dlimit else 0)

    def validate(self) -> None:  # REF src/aligner.cpp:11-24
        lib = _load()
        p = self._c()
        rc = lib.sa_validate_params(C.byref(p))
        if rc:
            _raise(rc)

    def effective_max_distance(self, read_length: int) -> int:  # REF aligner.cpp:26-29
        if self.max_distance >= 0:
            return self.max_distance
        return (12 * read_length + 99) // 100


@dataclass
class AlignmentResult:  # REF aligner.hpp:36-44
    kind: ResultKind = ResultKind.NotFound
    has_position: bool = False
    position: int = 0
    direction: Direction = Direction.Forward
    distance: int = -1
    gap: int = 0


@dataclass
class AlignStats:  # REF aligner.hpp:47-66 (+ extensions)
    values: dict = field(default_factory=lambda: {f: 0 for f in STAT_FIELDS})

    def __getattr__(self, name):
        if name in STAT_FIELDS:
            return self.values[name]
        raise AttributeError(name)

    def merge(self, other: "AlignStats") -> None:
        for f in STAT_FIELDS:
            self.values[f] += other.values[f]

    @classmethod
    def _from_c(cls, s: _Stats) -> "AlignStats":
        return cls({f: int(getattr(s, f)) for f in STAT_FIELDS})


def results_to_objects(arr: np.ndarray) -> list[AlignmentResult]:
    return [AlignmentResult(ResultKind(int(r["kind"])), bool(r["has_position"]), int(r["position"]),
                            Direction(int(r["direction"])), int(r["distance"]), int(r["gap"]))
            for r in arr]


# ----------------------------------------------------------------------- genome

_CODE = np.full(256, 255, dtype=np.uint8)
for _c, _v in zip(b"ACGTacgt", [0, 1, 2, 3, 0, 1, 2, 3]):
    _CODE[_c] = _v
for _c in b"UNRYSWKMBDHVunryswkmbdhv":
    _CODE[_c] = 4


def pack_sequence(seq: bytes | np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """ASCII -> (packed_words, n_mask_words) in PackedGenome layout
    (REF src/genome.cpp:39-46).  Raises ValueError on illegal characters."""
    a = np.frombuffer(seq, dtype=np.uint8) if isinstance(seq, (bytes, bytearray)) else np.asarray(seq, np.uint8)
    n = a.size
    codes = _CODE[a]
    if n and codes.max() == 255:
        bad = int(np.argmax(codes == 255))
        raise ValueError(f"illegal base {chr(a[bad])!r}")
    isn = codes == 4
    c2 = np.where(isn, 0, codes).astype(np.uint64)
    pad32 = (-n) % 32
    c2 = np.concatenate([c2, np.zeros(pad32, np.uint64)]).reshape(-1, 32)
    packed = np.bitwise_or.reduce(c2 << (2 * np.arange(32, dtype=np.uint64)), axis=1).astype(np.uint64)
    pad64 = (-n) % 64
    nb = np.concatenate([isn.astype(np.uint64), np.zeros(pad64, np.uint64)]).reshape(-1, 64)
    nmask = np.bitwise_or.reduce(nb << np.arange(64, dtype=np.uint64), axis=1).astype(np.uint64)
    return packed, nmask


class PackedGenome:
    """2-bit packed genome + N mask + contig table (REF include/seedaln/genome.hpp:36-100).
    Without an explicit contig table the genome is one contig "chr1"."""

    def __init__(self, packed: np.ndarray, nmask: np.ndarray, length: int,
                 contigs: Sequence[tuple[str, int, int]] | None = None):
        self.packed = np.ascontiguousarray(packed, dtype=np.uint64)
        self.nmask = np.ascontiguousarray(nmask, dtype=np.uint64)
        self.length = int(length)
        if self.packed.size != (self.length + 31) // 32 or self.nmask.size != (self.length + 63) // 64:
            raise FormatError("packed/n-mask sizes do not match the genome length")
        self._contigs = [tuple(c) for c in contigs] if contigs is not None else [("chr1", 0, self.length)]

    @classmethod
    def from_sequence(cls, seq: bytes | str) -> "PackedGenome":
        if isinstance(seq, str):
            seq = seq.encode()
        packed, nmask = pack_sequence(seq)
        return cls(packed, nmask, len(seq))

    @classmethod
    def from_contigs(cls, named_seqs: Sequence[tuple[str, str]]) -> "PackedGenome":
        # REF src/genome.cpp:96-112: contigs tile the genome in order
        # (alignment windows ignore contig boundaries, REF genome.cpp:114-123)
        contigs, start = [], 0
        for name, sq in named_seqs:
            contigs.append((name, start, len(sq)))
            start += len(sq)
        g = cls.from_sequence("".join(sq for _, sq in named_seqs))
        g._contigs = contigs
        return g

    @classmethod
    def from_fasta(cls, path: str) -> "PackedGenome":  # REF src/genome.cpp:48-94
        lib = _load()
        h = C.c_void_p()
        rc = lib.sa_genome_from_fasta(os.fsencode(path), C.byref(h))
        if rc:
            _raise(rc)
        try:
            return cls._from_handle(h.value)
        finally:
            lib.sa_genome_free(h)

    @classmethod
    def _from_handle(cls, h) -> "PackedGenome":
        lib = _load()
        n, nc = C.c_uint64(), C.c_uint64()
        lib.sa_genome_info(h, C.byref(n), C.byref(nc), None)
        pp, pn = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)()
        np_, nn = C.c_uint64(), C.c_uint64()
        lib.sa_genome_words(h, C.byref(pp), C.byref(np_), C.byref(pn), C.byref(nn))
        packed = np.ctypeslib.as_array(pp, (np_.value,)).copy() if np_.value else np.zeros(0, np.uint64)
        nmask = np.ctypeslib.as_array(pn, (nn.value,)).copy() if nn.value else np.zeros(0, np.uint64)
        contigs = []
        for i in range(nc.value):
            nm, st, ln = C.c_char_p(), C.c_uint64(), C.c_uint64()
            lib.sa_genome_contig(h, i, C.byref(nm), C.byref(st), C.byref(ln))
            contigs.append((nm.value.decode(), st.value, ln.value))
        return cls(packed, nmask, n.value, contigs)

    def _handle(self):
        """A native sa_genome for this genome (caller frees with sa_genome_free)."""
        lib = _load()
        names = (C.c_char_p * max(1, len(self._contigs)))(*[c[0].encode() for c in self._contigs])
        starts = np.array([c[1] for c in self._contigs], np.uint64)
        lens = np.array([c[2] for c in self._contigs], np.uint64)
        h = C.c_void_p()
        rc = lib.sa_genome_from_words(_u64p(self.packed), self.packed.size, _u64p(self.nmask), self.nmask.size,
                                      self.length, names, _u64p(starts), _u64p(lens), len(self._contigs),
                                      C.byref(h))
        if rc:
            _raise(rc)
        return h

    def contigs(self) -> list[tuple[str, int, int]]:  # REF genome.hpp:91 (name, start, length)
        return list(self._contigs)

    def checksum(self) -> int:  # REF src/genome.cpp:158-179
        lib = _load()
        h = self._handle()
        try:
            v = C.c_uint64()
            lib.sa_genome_info(h, None, None, C.byref(v))
            return v.value
        finally:
            lib.sa_genome_free(h)

    def size(self) -> int:
        return self.length

    def at(self, pos: int) -> int:  # REF genome.hpp:50-54; 4 = N
        if (int(self.nmask[pos >> 6]) >> (pos & 63)) & 1:
            return 4
        return (int(self.packed[pos >> 5]) >> ((pos & 31) * 2)) & 3

    def substring(self, pos: int, length: int) -> str:  # REF genome.cpp:114-123
        if pos >= self.length:
            raise IndexError(f"genome position {pos} past end {self.length}")
        n = min(length, self.length - pos)
        return "".join("ACGTN"[self.at(pos + i)] for i in range(n))

    def to_contig_coordinate(self, pos: int) -> tuple[str, int]:  # REF genome.cpp:121-131
        if pos >= self.length:
            raise IndexError(f"genome position {pos} past end {self.length}")
        starts = [c[1] for c in self._contigs]
        import bisect
        i = bisect.bisect_right(starts, pos) - 1
        return self._contigs[i][0], pos - self._contigs[i][1]


def save_index_file(seed_size: int, g: PackedGenome, path: str, fmt: int = SA_INDEX_SNAPIDX1,
                    device: int = 0) -> None:
    """run_index / save_index_file (REF src/driver.cpp:37-45, src/seed_index.cpp:145-170):
    CSR tables built on the GPU; SNAPIDX1 byte-identical to the reference's."""
    lib = _load()
    h = g._handle()
    try:
        rc = lib.sa_index_write(h, seed_size, fmt, device, os.fsencode(path))
        if rc:
            _raise(rc)
    finally:
        lib.sa_genome_free(h)


def index_csr(g: PackedGenome, seed_size: int, device: int = 0) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """The reference SeedIndex's keys_/offsets_/positions_ (REF seed_index.hpp:69-71), GPU-built."""
    lib = _load()
    h = g._handle()
    try:
        nk, npos = C.c_uint64(0), C.c_uint64(0)
        rc = lib.sa_index_csr(h, seed_size, device, C.byref(nk), C.byref(npos), None, None, None)
        if rc:
            _raise(rc)
        keys = np.zeros(nk.value, np.uint64)
        offs = np.zeros(nk.value + 1, np.uint64)
        pos = np.zeros(npos.value, np.uint64)
        rc = lib.sa_index_csr(h, seed_size, device, C.byref(nk), C.byref(npos), _u64p(keys), _u64p(offs),
                              _u64p(pos))
        if rc:
            _raise(rc)
        return keys, offs, pos
    finally:
        lib.sa_genome_free(h)


# ----------------------------------------------------------------------- index

@dataclass
class LookupResult:  # REF seed_index.hpp:27-32
    forward: list
    rc: list

    def count(self) -> int:
        return len(self.forward) + len(self.rc)


class SeedIndex:
    """GPU seed index (replaces REF SeedIndex, src/seed_index.cpp:80-143).
    Holds one replica per device in ``devices``."""

    def __init__(self, ctx: int, seed_size: int, genome: PackedGenome):
        self._ctx = ctx
        self._seed_size = seed_size
        self._genome = genome

    @classmethod
    def build(cls, g: PackedGenome, seed_size: int, devices: Iterable[int] | None = None) -> "SeedIndex":
        lib = _load()
        devs = list(devices) if devices is not None else [0]
        darr = (C.c_int32 * len(devs))(*devs)
        out = C.c_void_p()
        rc = lib.sa_create(_u64p(g.packed), g.packed.size, _u64p(g.nmask), g.nmask.size, g.length,
                           seed_size, darr, len(devs), C.byref(out))
        if rc:
            _raise(rc)
        return cls(out.value, seed_size, g)

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx and _lib is not None:
            _lib.sa_destroy(ctx)
            self._ctx = None

    @classmethod
    def load(cls, path: str, devices: Iterable[int] | None = None, verify: bool = True
             ) -> tuple["SeedIndex", PackedGenome]:
        """load_index_file (REF src/seed_index.cpp:173-228) -> (index, genome)."""
        lib = _load()
        devs = list(devices) if devices is not None else [0]
        darr = (C.c_int32 * len(devs))(*devs)
        gh, ctx = C.c_void_p(), C.c_void_p()
        rc = lib.sa_index_load(os.fsencode(path), darr, len(devs), 1 if verify else 0, C.byref(gh), C.byref(ctx))
        if rc:
            _raise(rc)
        try:
            g = PackedGenome._from_handle(gh.value)
        finally:
            lib.sa_genome_free(gh)
        s = C.c_int32()
        lib.sa_index_seed_size(ctx.value, C.byref(s))
        return cls(ctx.value, s.value, g), g

    def seed_size(self) -> int:
        return self._seed_size

    def _info(self):
        d, t, b = C.c_uint64(), C.c_uint64(), C.c_uint64()
        rc = _load().sa_index_info(self._ctx, C.byref(d), C.byref(t), C.byref(b))
        if rc:
            _raise(rc, self._ctx)
        return d.value, t.value, b.value

    def distinct_seeds(self) -> int:
        return self._info()[0]

    def total_positions(self) -> int:
        return self._info()[1]

    def device_bytes(self) -> int:
        return self._info()[2]

    def lookup_counts(self, seeds: Sequence[str] | bytes) -> np.ndarray:
        buf = seeds if isinstance(seeds, (bytes, bytearray)) else "".join(seeds).encode()
        n = len(buf) // self._seed_size
        counts = np.zeros(n, np.uint32)
        rc = _load().sa_lookup_batch(self._ctx, bytes(buf), n, counts.ctypes.data_as(C.POINTER(C.c_uint32)),
                                     None, None, None, None, 0)
        if rc:
            _raise(rc, self._ctx)
        return counts

    def lookup_batch(self, seeds: Sequence[str], cap: int = 4096) -> list[LookupResult]:
        for sd in seeds:  # REF seed_index.cpp:129-130
            if len(sd) != self._seed_size:
                raise ValueError("seed length does not match index seed size")
        n = len(seeds)
        if n == 0:
            return []
        buf = "".join(seeds).encode()
        counts = np.zeros(n, np.uint32)
        nf = np.zeros(n, np.uint32)
        nr = np.zeros(n, np.uint32)
        fo = np.zeros(n * cap, np.uint64)
        ro = np.zeros(n * cap, np.uint64)
        P32 = C.POINTER(C.c_uint32)
        rc = _load().sa_lookup_batch(self._ctx, buf, n, counts.ctypes.data_as(P32), _u64p(fo),
                                     nf.ctypes.data_as(P32), _u64p(ro), nr.ctypes.data_as(P32), cap)
        if rc:
            _raise(rc, self._ctx)
        out = []
        for i in range(n):
            if nf[i] > cap or nr[i] > cap:
                raise ValueError("lookup list longer than cap")
            out.append(LookupResult([int(v) for v in fo[i * cap:i * cap + nf[i]]],
                                    [int(v) for v in ro[i * cap:i * cap + nr[i]]]))
        return out

    def lookup(self, seed: str) -> LookupResult:  # REF seed_index.cpp:128-143
        return self.lookup_batch([seed])[0]


# ----------------------------------------------------------------------- aligner

def reads_to_buffer(reads: Sequence[str | bytes]) -> tuple[bytes, np.ndarray]:
    bs = [r.encode() if isinstance(r, str) else bytes(r) for r in reads]
    offs = np.zeros(len(bs) + 1, np.uint64)
    if bs:
        offs[1:] = np.cumsum([len(b) for b in bs])
    return b"".join(bs), offs


class Aligner:
    """REF include/seedaln/aligner.hpp:116-158.  ``align`` is a batch of one
    (for tests); ``align_batch`` / ``align_arrays`` are the production calls."""

    def __init__(self, idx: SeedIndex, g: PackedGenome, params: AlignerParams):
        params.validate()  # REF aligner.cpp:119
        if idx.seed_size() != params.seed_size:  # REF aligner.cpp:120-121
            raise ValueError("index seed size does not match params")
        self._idx = idx
        self._g = g
        self._params = params
        self._stats = AlignStats()

    def params(self) -> AlignerParams:
        return self._params

    def stats(self) -> AlignStats:
        return self._stats

    def align_arrays(self, bases, offsets: np.ndarray, results: np.ndarray | None = None) -> np.ndarray:
        """bases: bytes / uint8 array (may be pinned); offsets: uint64[n+1]."""
        lib = _load()
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        if results is None:
            results = np.zeros(n, RESULT_DTYPE)
        st = _Stats()
        p = self._params._c()
        if isinstance(bases, (bytes, bytearray)):
            bptr = C.cast(C.c_char_p(bytes(bases)), C.c_void_p)
            keep = bases
        else:
            arr = np.ascontiguousarray(bases, dtype=np.uint8)
            bptr = C.c_void_p(arr.ctypes.data)
            keep = arr
        rc = lib.sa_align_batch(self._idx._ctx, C.byref(p), bptr, _u64p(offsets), n,
                                C.c_void_p(results.ctypes.data), C.byref(st))
        del keep
        if rc:
            _raise(rc, self._idx._ctx)
        self._stats.merge(AlignStats._from_c(st))
        return results

    def align_batch(self, reads: Sequence[str | bytes]) -> list[AlignmentResult]:
        buf, offs = reads_to_buffer(reads)
        return results_to_objects(self.align_arrays(buf, offs))

    def align(self, read) -> AlignmentResult:  # REF aligner.cpp:223
        bases = read.bases if hasattr(read, "bases") else read
        return self.align_batch([bases])[0]

    def last_timing(self) -> tuple[float, float]:
        e, k = C.c_float(), C.c_float()
        _load().sa_last_timing(self._idx._ctx, C.byref(e), C.byref(k))
        return e.value, k.value

    def last_launches(self) -> int:
        v = C.c_uint64()
        _load().sa_last_launches(self._idx._ctx, C.byref(v))
        return v.value

    def last_kernel_times(self) -> tuple[float, float]:
        """(fused kernel ms, overflow kernel ms) of the last call (CUDA events)."""
        f, s = C.c_float(), C.c_float()
        rc = _load().sa_last_kernel_times(self._idx._ctx, C.byref(f), C.byref(s))
        if rc:
            _raise(rc, self._idx._ctx)
        return f.value, s.value

    def align_device(self, d_bases: int, d_offsets: int, n_reads: int, max_read_length: int,
                     d_results: int, d_stats: int = 0, stream: int = 0) -> None:
        """Device-resident batch (raw CUDA pointers, e.g. torch data_ptr()); async on stream."""
        p = self._params._c()
        rc = _load().sa_align_device(self._idx._ctx, C.byref(p), C.c_void_p(d_bases), C.c_void_p(d_offsets),
                                     n_reads, max_read_length, C.c_void_p(d_results),
                                     C.c_void_p(d_stats) if d_stats else None,
                                     C.c_void_p(stream) if stream else None)
        if rc:
            _raise(rc, self._idx._ctx)

    def sync(self, stream: int = 0) -> None:
        rc = _load().sa_sync(self._idx._ctx, C.c_void_p(stream) if stream else None)
        if rc:
            _raise(rc, self._idx._ctx)


def align_read(read, idx: SeedIndex, g: PackedGenome, params: AlignerParams,
               stats: AlignStats | None = None) -> AlignmentResult:  # REF aligner.cpp:366-373
    a = Aligner(idx, g, params)
    r = a.align(read)
    if stats is not None:
        stats.merge(a.stats())
    return r


def seed_offsets(read_length: int, s: int, n: int) -> list[int]:  # REF aligner.cpp:50-79
    lib = _load()
    buf = (C.c_int32 * max(n, 1))()
    cnt = C.c_int32()
    rc = lib.sa_seed_offsets(read_length, s, n, buf, C.byref(cnt))
    if rc:
        _raise(rc)
    return list(buf[:cnt.value])


def classify_confidence(d_best: int, d_second: int, d_max: int, c: int) -> ResultKind:
    # REF aligner.cpp:81-85 (scalar helper; the kernel applies the same rule)
    if d_best <= d_max and d_second >= d_best + c:
        return ResultKind.SingleHit
    if d_best <= d_max:
        return ResultKind.MultipleHits
    return ResultKind.NotFound


def bounded_distance_batch(pairs: Sequence[tuple[str, str, int]], device: int = 0) -> list[int | None]:
    """bounded_distance (REF src/edit_distance.cpp:19-75) for many
    (read, window, d_limit) triples on the GPU; None = exceeds the limit."""
    lib = _load()
    if not pairs:
        return []
    rb, ro = reads_to_buffer([p[0] for p in pairs])
    wb, wo = reads_to_buffer([p[1] for p in pairs])
    dl = np.array([p[2] for p in pairs], np.int32)
    out = np.zeros(len(pairs), np.int32)
    P32 = C.POINTER(C.c_int32)
    rc = lib.sa_bounded_distance_batch(rb, _u64p(ro), wb, _u64p(wo), dl.ctypes.data_as(P32),
                                       len(pairs), out.ctypes.data_as(P32), device)
    if rc:
        _raise(rc)
    return [None if v < 0 else int(v) for v in out]


def bounded_distance(read: str, window: str, d_limit: int) -> int | None:
    return bounded_distance_batch([(read, window, d_limit)])[0]


class PinnedBuffer:
    """Page-locked host buffer from sa_host_alloc, viewable as a numpy array."""

    def __init__(self, nbytes: int):
        lib = _load()
        p = C.c_void_p()
        rc = lib.sa_host_alloc(C.byref(p), nbytes)
        if rc:
            _raise(rc)
        self.ptr = p.value
        self.nbytes = nbytes

    def array(self, dtype, count: int | None = None) -> np.ndarray:
        dt = np.dtype(dtype)
        count = self.nbytes // dt.itemsize if count is None else count
        buf = (C.c_char * (count * dt.itemsize)).from_address(self.ptr)
        return np.frombuffer(buf, dtype=dt, count=count)

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.sa_host_free(self.ptr)
            self.ptr = None


# ----------------------------------------------------------------------- driver

@dataclass
class EvalReport:  # REF include/seedaln/eval.hpp:24-46
    total: int = 0
    single: int = 0
    multiple: int = 0
    notfound: int = 0
    correct: int = 0
    wrong: int = 0
    no_truth: int = 0
    elapsed_seconds: float = 0.0
    stats: AlignStats = field(default_factory=AlignStats)
    _c: object = None

    def to_text(self) -> str:  # REF src/eval.cpp:75-120
        lib = _load()
        n = C.c_uint64()
        lib.sa_report_text(C.byref(self._c), None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        lib.sa_report_text(C.byref(self._c), buf, n.value + 1, C.byref(n))
        return buf.value.decode()


def run_index(fasta_path: str, index_path: str, seed_size: int = 20, fmt: int = SA_INDEX_SNAPIDX1,
              device: int = 0) -> None:
    """run_index (REF src/driver.cpp:37-45) with the CSR built on the GPU."""
    rc = _load().sa_run_index(os.fsencode(fasta_path), os.fsencode(index_path), seed_size, fmt, device)
    if rc:
        _raise(rc)


def run_align(index_path: str, fastq_path: str, output_path: str, params: AlignerParams | None = None,
              threads: int = 1, chunk_min_bytes: int = 4 << 20, stable_order: bool = False, tolerance: int = 50,
              report_path: str | None = None, command_line: str = "seedaln align",
              devices: Iterable[int] | None = None, verify_index: bool = True) -> EvalReport:
    """run_align (REF src/driver.cpp:47-156): FASTQ -> SAM through the GPU."""
    lib = _load()
    o = _AlignOptions()
    lib.sa_default_align_options(C.byref(o))
    keep = [os.fsencode(index_path), os.fsencode(fastq_path), os.fsencode(output_path),
            os.fsencode(report_path) if report_path else None, command_line.encode()]
    o.index_path, o.fastq_path, o.output_path, o.report_path, o.command_line = keep
    o.params = (params or AlignerParams())._c()
    o.threads = threads
    o.chunk_min_bytes = chunk_min_bytes
    o.stable_order = 1 if stable_order else 0
    o.tolerance = tolerance
    devs = list(devices) if devices is not None else [0]
    darr = (C.c_int32 * len(devs))(*devs)
    o.devices = darr
    o.n_devices = len(devs)
    o.verify_index = 1 if verify_index else 0
    rep = _EvalReport()
    rc = lib.sa_run_align(C.byref(o), C.byref(rep))
    del keep
    if rc:
        _raise(rc)
    return EvalReport(rep.total, rep.single, rep.multiple, rep.notfound, rep.correct, rep.wrong, rep.no_truth,
                      rep.elapsed_seconds, AlignStats._from_c(rep.stats), rep)


# ----------------------------------------------------------------------- referee

REFEREE_HIT_DTYPE = np.dtype([("position", "<u8"), ("distance", "<i4"), ("direction", "u1"), ("reserved", "u1", (3,))])


class Referee:
    """OracleContext / oracle_align / oracle_scan on the GPU (REF include/seedaln/eval.hpp:49-117)."""

    def __init__(self, g: PackedGenome, device: int = 0):
        lib = _load()
        h = g._handle()
        try:
            out = C.c_void_p()
            rc = lib.sa_referee_create(h, device, C.byref(out))
            if rc:
                _raise(rc)
            self._r = out.value
        finally:
            lib.sa_genome_free(h)

    def __del__(self):
        r = getattr(self, "_r", None)
        if r and _lib is not None:
            _lib.sa_referee_destroy(r)
            self._r = None

    def align_arrays(self, params: AlignerParams, bases, offsets: np.ndarray) -> np.ndarray:
        """oracle_align per read (REF src/eval.cpp:270-306)."""
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        res = np.zeros(n, RESULT_DTYPE)
        b = np.ascontiguousarray(np.frombuffer(bases, np.uint8) if isinstance(bases, (bytes, bytearray)) else bases,
                                 np.uint8)
        p = params._c()
        rc = _load().sa_referee_align(self._r, C.byref(p), C.c_void_p(b.ctypes.data), _u64p(offsets), n,
                                      C.c_void_p(res.ctypes.data))
        if rc:
            _raise(rc)
        return res

    def scan_arrays(self, d_limit: int, bucket_size: int, bases, offsets: np.ndarray):
        """oracle_scan per read (REF src/eval.cpp:244-268): (hit_offsets, hits)."""
        lib = _load()
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        b = np.ascontiguousarray(np.frombuffer(bases, np.uint8) if isinstance(bases, (bytes, bytearray)) else bases,
                                 np.uint8)
        ho = np.zeros(n + 1, np.uint64)
        rc = lib.sa_referee_scan(self._r, d_limit, bucket_size, C.c_void_p(b.ctypes.data), _u64p(offsets), n,
                                 _u64p(ho), None, 0)
        if rc:
            _raise(rc)
        hits = np.zeros(int(ho[-1]), REFEREE_HIT_DTYPE)
        rc = lib.sa_referee_scan(self._r, d_limit, bucket_size, C.c_void_p(b.ctypes.data), _u64p(offsets), n,
                                 _u64p(ho), C.c_void_p(hits.ctypes.data), hits.size)
        if rc:
            _raise(rc)
        return ho, hits


# ----------------------------------------------------------------------- simulator

@dataclass
class SimProfile:  # REF include/seedaln/simulator.hpp:17-26 (same defaults)
    read_length: int = 100
    snp_rate: float = 0.0009
    indel_mutation_rate: float = 0.0001
    seq_error_rate: float = 0.02
    indel_error_fraction: float = 0.0
    rng_seed: int = 1

    def _c(self) -> _SimProfile:
        return _SimProfile(self.read_length, self.snp_rate, self.indel_mutation_rate, self.seq_error_rate,
                           self.indel_error_fraction, self.rng_seed)


@dataclass
class Truth:  # REF simulator.hpp:30-36
    contig: str
    position: int
    direction: Direction
    serial: int


def encode_truth(t: Truth) -> str:  # REF src/simulator.cpp:43-48
    return f"{t.contig}_{t.position + 1}_{'F' if t.direction == Direction.Forward else 'R'}_{t.serial}"


class ReadSimulator:
    """ReadSimulator(genome, profile) (REF src/simulator.cpp:90-192) in
    libsnapb200.so: the reference's mt19937_64 draw stream, so next() yields
    the reference's reads in the same order."""

    def __init__(self, g: PackedGenome, profile: SimProfile | None = None):
        lib = _load()
        self._g = g
        self.profile = profile or SimProfile()
        self._gh = g._handle()
        h = C.c_void_p()
        rc = lib.sa_simulator_create(self._gh, C.byref(self.profile._c()), C.byref(h))
        if rc:
            lib.sa_genome_free(self._gh)
            self._gh = None
            _raise(rc)
        self._h = h
        self._names = [c[0] for c in g.contigs()]

    def __del__(self):
        lib = _lib
        if lib is not None:
            if getattr(self, "_h", None):
                lib.sa_simulator_destroy(self._h)
                self._h = None
            if getattr(self, "_gh", None):
                lib.sa_genome_free(self._gh)
                self._gh = None

    def next_batch(self, count: int) -> tuple[np.ndarray, np.ndarray]:
        """`count` reads: (bases uint8[count, read_length], truth TRUTH_DTYPE[count])."""
        L = self.profile.read_length
        bases = np.empty((count, L), dtype=np.uint8)
        truth = np.zeros(count, dtype=TRUTH_DTYPE)
        rc = _load().sa_simulator_next(self._h, count, bases.ctypes.data, truth.ctypes.data)
        if rc:
            _raise(rc)
        return bases, truth

    def truth_of(self, t) -> Truth:
        return Truth(self._names[int(t["contig"])], int(t["position"]), Direction(int(t["direction"])),
                     int(t["serial"]))

    def next(self) -> tuple[str, str, Truth]:  # REF simulator.cpp:117: (name, bases, truth)
        b, t = self.next_batch(1)
        tr = self.truth_of(t[0])
        return encode_truth(tr), b[0].tobytes().decode(), tr


def run_simulate(fasta_path: str, output_path: str, count: int, profile: SimProfile | None = None,
                 threads: int = 0) -> None:
    """run_simulate (REF src/driver.cpp:158-168): FASTA -> FASTQ, the reference's bytes."""
    p = (profile or SimProfile())._c()
    rc = _load().sa_run_simulate(os.fsencode(fasta_path), os.fsencode(output_path), count, C.byref(p), threads)
    if rc:
        _raise(rc)
