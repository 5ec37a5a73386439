"""Build libakv.so in-tree for sm_100a (explicit nvcc; no JIT cache).

    python -m paper_2409_16546_b200.build [--force] [--verbose]

Each .cu compiles to an object in parallel, then one nvcc link produces
paper_2409_16546_b200/libakv.so (cudart linked statically).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "akv")
LIB = os.path.join(PKG, "libakv.so")
SOURCES = ["akv_append.cu", "akv_qk.cu", "akv_select.cu", "akv_pv.cu", "akv_api.cu", "akv_analysis.cu"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))] + [
        os.path.join(INCLUDE, "akv.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def _compile(src: str):
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    cmd = [nvcc(), ARCH, *FLAGS, f"-I{INCLUDE}", f"-I{CSRC}", "-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return obj, cmd, res


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    log_lines = []
    failed = False
    for obj, cmd, res in results:
        log_lines.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        failed |= res.returncode != 0
    if not failed:
        tmp = LIB + ".tmp"
        cmd = [nvcc(), ARCH, "-shared", "-o", tmp] + [r[0] for r in results]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log_lines.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        failed = res.returncode != 0
    log = os.path.join(BUILD, "build.log")
    with open(log, "w") as f:
        f.write("\n".join(log_lines))
    if failed:
        sys.stderr.write("\n".join(log_lines)[-20000:])
        raise RuntimeError(f"nvcc failed; see {log}")
    if verbose:
        sys.stderr.write("\n".join(log_lines))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
