"""In-tree build of libmscg.so (sm_100a) — no JIT cache, so the .so travels
with the gpurun snapshot.

    python -m paper_1104_3349_b200.build [--force] [-v]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libmscg.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
# Host setup code must reproduce the reference's arithmetic bit-for-bit:
# no FMA contraction.
CXXFLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
            "-Wno-unused-parameter", "-I", os.path.join(CUDA, "include")] + INC
NVFLAGS = ARCH + ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
                  "-Xptxas", "-v"] + INC

# The device Oseen assembly must round exactly like the host generator.
PER_FILE = {"device/oseen.cu": ["--fmad=false"]}

SOURCES = [
    "host/oseen.cpp", "host/partition.cpp", "host/schur.cpp", "host/mmio.cpp", "capi.cpp",
    "device/runtime.cu", "device/spmv.cu", "device/factor.cu", "device/trisolve.cu",
    "device/precond.cu", "device/correct.cu", "device/gmres.cu", "device/schur.cu", "device/oseen.cu",
    "device/dissect.cu", "device/partition.cu",
]
HEADERS = ["host/csr.hpp", "host/setup.hpp", "device/common.cuh", "device/internal.hpp"]


def _newest_header() -> float:
    hs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "mscg.h")]
    return max(os.path.getmtime(h) for h in hs)


def _obj(src: str) -> str:
    return os.path.join(OBJ, src.replace("/", "_") + ".o")


def _compile(src: str, force: bool, verbose: bool) -> tuple[str, str]:
    path = os.path.join(CSRC, src)
    out = _obj(src)
    if (not force and os.path.exists(out)
            and os.path.getmtime(out) >= max(os.path.getmtime(path), _newest_header())):
        return out, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + PER_FILE.get(src, []) + ["-c", path, "-o", out]
    else:
        cmd = [os.environ.get("CXX", "g++")] + CXXFLAGS + ["-c", path, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out, (r.stdout + r.stderr) if verbose else ""


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            sys.stderr.write(log)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(map(os.path.getmtime, objs)):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        shutil.move(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
