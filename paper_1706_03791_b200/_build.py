"""Build libebz200.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

Every translation unit is compiled with ``-fmad=false`` (the arithmetic
contract forbids FMA contraction) and ``-lineinfo``
(so ncu source pages map to the code), then linked into one shared library
that the ctypes loader in ``_native.py`` opens.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libebz200.so")
ROOT = os.path.dirname(PKG)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
         f"-I{os.path.join(ROOT, 'include')}"]
# A/B experiments (tools/ab_build.sh): extra nvcc flags, built into
# build_<tag>/ and ab/<tag>.so instead of the product library
_AB_TAG = os.environ.get("EBZ_AB_TAG")
if _AB_TAG:
    FLAGS = FLAGS + os.environ.get("EBZ_NVCC_EXTRA", "").split()
    BUILD = BUILD + "_" + _AB_TAG
    LIB = os.path.join(ROOT, "ab", _AB_TAG + ".so")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "ebz200.h"))
    objs = []
    jobs = []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as pool:
        list(pool.map(run, jobs))
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or jobs or _stale(LIB, objs):
        run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt",
             "-lpthread", "-ldl"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
