"""The drop-in boundary without a GPU: the C-ABI library loads, exports every
entry point include/snap_b200.h declares, and its host-side logic (parameter
validation, seed schedule, error codes) matches the reference.  No compute
calls are made here."""
import ctypes as C
import json
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1111_5572_b200 import api
from tests.conftest import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _declared():
    txt = open(os.path.join(ROOT, "include", "snap_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sa_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = api._load()
    decl = _declared()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", api.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sa_[a-z_]+)", out))
    assert set(decl) <= exported
    assert exported <= set(decl), f"undeclared exports {exported - set(decl)}"


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", api.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_params_match_reference():
    # REF include/seedaln/aligner.hpp:20-26
    p = api._Params()
    api._load().sa_default_params(C.byref(p))
    assert (p.seed_size, p.seeds_to_try, p.max_distance, p.confidence_threshold, p.max_hits,
            p.bucket_size, p.force_max_dlimit) == (20, 25, -1, 2, 300, 32, 0)
    d = api.AlignerParams()
    assert (d.seed_size, d.seeds_to_try, d.max_distance, d.confidence_threshold, d.max_hits,
            d.bucket_size) == (20, 25, -1, 2, 300, 32)


def test_params_validation():
    # REF src/aligner.cpp:11-24, tests/test_aligner.cpp:111-123
    p = api.AlignerParams()
    p.validate()
    assert p.effective_max_distance(100) == 12
    assert p.effective_max_distance(1000) == 120
    p.max_distance = 5
    assert p.effective_max_distance(100) == 5
    for field, bad in [("bucket_size", 65), ("bucket_size", 0), ("seed_size", 0), ("seed_size", 33),
                       ("seeds_to_try", 0), ("max_distance", -2), ("confidence_threshold", 0),
                       ("max_hits", 0)]:
        q = api.AlignerParams(**{field: bad})
        with pytest.raises(ValueError):
            q.validate()


def test_seed_offsets_host_matches_golden():
    with open(os.path.join(GOLD, "seed_offsets_golden.json")) as f:
        for c in json.load(f):
            assert api.seed_offsets(c["len"], c["s"], c["n"]) == c["offsets"], c


def test_classify_confidence():
    # REF tests/test_aligner.cpp:72-78
    K = api.ResultKind
    inf = 0x7FFFFFFF // 4
    assert api.classify_confidence(1, 5, 8, 2) == K.SingleHit
    assert api.classify_confidence(1, 2, 8, 2) == K.MultipleHits
    assert api.classify_confidence(9, inf, 8, 2) == K.NotFound
    assert api.classify_confidence(0, inf, 8, 2) == K.SingleHit
    assert api.classify_confidence(8, 9, 8, 2) == K.MultipleHits


def test_create_argument_errors():
    lib = api._load()
    packed = np.zeros(1, np.uint64)
    out = C.c_void_p()
    P = C.POINTER(C.c_uint64)
    pp = packed.ctypes.data_as(P)
    # seed size out of range -> invalid_argument (REF seed_index.cpp:81-82)
    assert lib.sa_create(pp, 1, pp, 1, 10, 0, None, 0, C.byref(out)) == api.SA_EINVAL
    assert lib.sa_create(pp, 1, pp, 1, 10, 33, None, 0, C.byref(out)) == api.SA_EINVAL
    # genome shorter than the seed (REF :83-84)
    assert lib.sa_create(pp, 1, pp, 1, 4, 5, None, 0, C.byref(out)) == api.SA_EINVAL
    # word counts inconsistent with the length -> FormatError
    assert lib.sa_create(pp, 1, pp, 1, 100, 4, None, 0, C.byref(out)) == api.SA_EFORMAT
    assert b"seed" in lib.sa_last_error(None) or b"match" in lib.sa_last_error(None)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    g = api.PackedGenome.from_sequence("ACGT" * 100)
    with pytest.raises(RuntimeError, match="CUDA"):
        api.SeedIndex.build(g, 8)


def test_pack_sequence_matches_oracle_layout():
    from oracle import oracle as O

    rng = np.random.default_rng(4)
    for L in (1, 31, 32, 33, 63, 64, 65, 1000):
        seq = bytes(rng.choice(list(b"ACGTNacgtn"), L).tolist())
        a = api.pack_sequence(seq)
        b = O.pack_genome(seq)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    with pytest.raises(ValueError):
        api.pack_sequence(b"ACGX")


def test_product_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_1111_5572_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|liboracle|seedaln_ref|snap_oracle", txt, re.M), f


def test_cpp_adapter_compiles_and_links(tmp_path):
    """include/snap_b200.hpp (the C++ drop-in shape) compiles against the C ABI
    and links against libsnapb200.so (no GPU call is made)."""
    src = tmp_path / "use.cpp"
    src.write_text(
        '#include "snap_b200.hpp"\n'
        "int main(int argc, char**) {\n"
        "  if (argc > 5) { snap_b200::SeedIndex idx({0}, {0}, 20, 20);\n"
        "    snap_b200::Aligner al(idx, snap_b200::default_params());\n"
        "    auto r = al.align(\"ACGT\"); return r.kind; }\n"
        "  if (argc > 6) { auto g = snap_b200::Genome::from_fasta(\"x.fa\");\n"
        "    snap_b200::save_index_file(g, 20, \"x.idx\");\n"
        "    auto [idx, g2] = snap_b200::load_index_file(\"x.idx\");\n"
        "    sa_align_options o; sa_default_align_options(&o); snap_b200::run_align(o);\n"
        "    snap_b200::Referee rf(g2); return static_cast<int>(idx.seed_size()); }\n"
        "  if (argc > 7) { auto g = snap_b200::Genome::from_fasta(\"x.fa\"); sa_sim_profile sp;\n"
        "    sa_default_sim_profile(&sp); snap_b200::ReadSimulator sim(g, sp); std::string b;\n"
        "    std::vector<sa_sim_truth> t; sim.next(10, b, t); snap_b200::run_simulate(\"x.fa\", \"x.fq\", 10, sp);\n"
        "    return static_cast<int>(t[0].serial); }\n"
        "  return 0; }\n")
    exe = tmp_path / "use"
    r = subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                        api.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(api.LIB_PATH)}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0


@pytest.mark.gpu
def test_cpp_dropin_runs_against_the_reference():
    """The C++ drop-in executed (tests/cpp/dropin_main.cpp, built by
    oracle.build() where the reference headers are): the reference's
    Aligner and snap_b200::Aligner in one process over the same
    run_align-style pageable reads (REF src/driver.cpp:99-132), every
    AlignmentResult field and counter equal over three parameter sets, and
    the same exception types for bad params, a seed-size mismatch and a bad
    character."""
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([exe, "200000"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "DROPIN OK 600000 0" in r.stdout
