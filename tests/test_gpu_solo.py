"""The thread-per-read solo kernel (align.cu solo_kernel) against the oracle.

The solo kernel finishes the reads whose seeds have few hits (at most 6 each,
8 candidates in all) and hands every other read to the warp kernel, so by
default each batch is split between the two kernels.  These runs force each side: SA_SOLO_MIN_READS=1
puts every launch (small batches, ragged and short reads, N seeds, the
repeat corpora whose reads bail part-way, force_max_dlimit, the golden
corpora) through the solo kernel first; SA_NO_SOLO=1 runs the warp kernel
alone.  Both must match the oracle read for read and counter for counter.
The switches are read once per process, so each run is a subprocess.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SELECT = "align_parity or ragged or heavily_edited or force_max or align_golden or overflow_paths or fixed_length or param_sweep"


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"SA_SOLO_MIN_READS": "1"}, {"SA_NO_SOLO": "1"}], ids=["solo-everywhere", "warp-only"])
def test_parity_with_solo_forced(env):
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-x", "-q",
                        "-m", "gpu", "-k", SELECT, "-p", "no:cacheprovider"],
                       cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.gpu
def test_bitparallel_lv_vs_oracle():
    """lv_bitpar (the solo kernel's banded bit-parallel LV) through the
    standalone LV entry point (SA_LV_BITPAR=1: lane 0 of each warp runs it for
    limits <= 15): the reference's known answers, the golden LV triples and
    random pairs with edits and N against the oracle."""
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-x", "-q",
                        "-m", "gpu", "-k", "lv_known or lv_random or lv_wide or lv_golden", "-p", "no:cacheprovider"],
                       cwd=ROOT, env={**os.environ, "SA_LV_BITPAR": "1"}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.gpu
def test_referee_wavefront_verify_still_matches():
    """The referee's verify stage uses lv_bitpar for limits <= 15; the
    wavefront LV it replaced (SA_REF_WAVEFRONT=1) must still give the
    reference's hit lists and results."""
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_referee.py"), "-x", "-q",
                        "-m", "gpu", "-p", "no:cacheprovider"],
                       cwd=ROOT, env={**os.environ, "SA_REF_WAVEFRONT": "1", "SA_REF_BUCKET_SERIAL": "1", "SA_REF_MERGE_SERIAL": "1"}, capture_output=True, text=True,
                       timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.gpu
def test_parity_multichunk_and_grid_stride():
    """Every launch split into many small chunks (SA_CHUNK_READS=1024, so the
    overflow pass of SA_OVERFLOW_KERNEL runs per chunk with chunk-relative
    read ids) and every kernel run with a single block (SA_SOLO_GRID=1,
    SA_SEED_GRID=1: grid-stride loops take many iterations and the
    lane-distributed counters accumulate across them), the solo kernel on for
    every launch."""
    env = {"SA_CHUNK_READS": "1024", "SA_SOLO_GRID": "1", "SA_SEED_GRID": "1", "SA_SOLO_MIN_READS": "1"}
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-x", "-q",
                        "-m", "gpu", "-k", "align_parity or overflow_paths or param_sweep", "-p", "no:cacheprovider"],
                       cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["sys", "bitpar"])
def test_warp_bitparallel_lv_vs_oracle(variant):
    """The long-read LVs through the standalone LV entry with their threshold
    lowered to 16 (SA_LV_WARP_BITPAR_MIN): lv_sys (systolic: lane per row
    block, blocks skewed in time, the default) and lv_bitpar_warp (band
    spread over the warp, carries scanned across lanes; SA_LV_LONG=bitpar).
    The reference's known answers, the golden LV triples, random pairs and
    wide limits (16-400 on reads of 200-3000 bases) against the oracle."""
    env = {**os.environ, "SA_LV_WARP_BITPAR_MIN": "16"}
    if variant == "bitpar":
        env["SA_LV_LONG"] = "bitpar"
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-x", "-q",
                        "-m", "gpu", "-k", "lv_known or lv_random or lv_wide or lv_golden", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
