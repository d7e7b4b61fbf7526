"""Build librepops.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2502_19405_b200.build [--force] [--verbose]

Flags that matter for bits:
  -fmad=false        no contraction of a separate multiply and add into FFMA
  -ftz=false         gradual underflow (IEEE subnormals)
  -prec-div=true     IEEE correctly rounded division (__fdiv_rn also explicit)
  -prec-sqrt=true    IEEE correctly rounded sqrt
  never --use_fast_math
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librepops.so")
OBJ = os.path.join(HERE, "build_obj")
SOURCES = ["abi.cu", "gemm.cu", "gemm_tn.cu", "rowops.cu", "elementwise.cu", "sha256.cu", "p2p.cu", "attention.cu"]
HEADERS = ["common.cuh", "gemm.cuh", "rowops.cuh", "elementwise.cuh", "sha256.cuh", "p2p.cuh", "attention.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NUMERIC = ["-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-O3"]


def _deps_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(os.path.dirname(HERE), "include", "repops.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def _includes(path: str, seen: set) -> set:
    """the file and every quoted #include it reaches (transitively)"""
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as f:
        for line in f:
            m = re.match(r'\s*#include\s+"([^"]+)"', line)
            if m:
                _includes(os.path.normpath(os.path.join(os.path.dirname(path), m.group(1))), seen)
    return seen


def _src_deps_mtime(src: str) -> float:
    """newest of the object's source, the headers it includes and this script"""
    files = _includes(os.path.join(CSRC, src), set()) | {os.path.abspath(__file__)}
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, verbose: bool, force: bool = True) -> str:
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    if not force and not os.environ.get("RO_NVCC_DEFS") and os.path.exists(obj) \
            and os.path.getmtime(obj) >= _src_deps_mtime(src):
        return obj  # up to date
    extra = os.environ.get("RO_NVCC_DEFS", "").split()  # tuning variants only (tools/sha_tune.sh)
    cmd = [NVCC, *ARCH, *NUMERIC, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd[1:1] = ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, force), SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
