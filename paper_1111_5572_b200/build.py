"""In-tree build of the native libraries (no JIT cache, so the .so files
travel to the GPU box with the repo snapshot).

  lib/libsnapb200.so     CUDA sm_100a kernels + C-ABI (include/snap_b200.h)
  lib/libsnap_synth.so   synthetic genome/read generator (host only)

Run ``python -m paper_1111_5572_b200.build`` or call ``build()``.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib")
OBJ = os.path.join(HERE, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_SOURCES = ["index.cu", "align.cu", "capi.cu", "csr.cu", "genome_io.cpp", "run_align.cpp", "referee.cu", "pack.cpp", "simulate.cpp"]
HEADERS = ["common.cuh", "align_kernels.cuh", "device_index.h", "host_common.h", "lv.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-diag-suppress", "550",
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build(verbose: bool = False) -> dict[str, str]:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "snap_b200.h")]
    objs = []
    jobs = []
    for src in CUDA_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        if _stale(o, [s] + hdrs):
            jobs.append([NVCC, *NVCC_FLAGS, "-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for _ in ex.map(_run, jobs):
            pass
    so = os.path.join(LIB, "libsnapb200.so")
    if jobs or _stale(so, objs):
        _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
              "-o", so, *objs])
    synth_src = os.path.join(CSRC, "synth.cpp")
    synth_so = os.path.join(LIB, "libsnap_synth.so")
    if _stale(synth_so, [synth_src]):
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-o", synth_so, synth_src, "-lpthread"])
    if verbose:
        print(f"built {so}\nbuilt {synth_so}")
    return {"cuda": so, "synth": synth_so}


def build_variant(name: str, defines: list[str]) -> str:
    """Experimental build with extra -D flags into lib/variants/ (select at
    run time with SNAP_B200_LIB=<path>); the default library is untouched."""
    vdir = os.path.join(LIB, "variants")
    vobj = os.path.join(OBJ, name)
    os.makedirs(vdir, exist_ok=True)
    os.makedirs(vobj, exist_ok=True)
    objs, jobs = [], []
    for src in CUDA_SOURCES:
        o = os.path.join(vobj, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        jobs.append([NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", o])
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        for _ in ex.map(_run, jobs):
            pass
    so = os.path.join(vdir, f"libsnapb200_{name}.so")
    _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-o", so, *objs])
    return so


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
