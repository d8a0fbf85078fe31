"""Build the sm_100a shared library in-tree (no JIT cache).

    python -m paper_2503_08040_b200.build        # or __graft_entry__.build()

Produces paper_2503_08040_b200/lib/libfbq_b200.so from csrc/*.cu and
csrc/host/*.cpp with nvcc -gencode arch=compute_100a,code=sm_100a.  Objects
are rebuilt only when a source or header is newer (parallel nvcc jobs).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build_obj")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libfbq_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -ftz=false / IEEE division: the bit-exact rounding in fbq_round.cuh (the
# parity-denormal RTN fix, subnormal scales and products) needs
# fp32 denormals preserved; nvcc defines no macro for -ftz, so the flags are
# pinned here and checked below (never add --use_fast_math).
CU_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ftz=false",
                   "-prec-div=true", "-prec-sqrt=true",
                   "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]
assert not any(f in CU_FLAGS for f in ("--use_fast_math", "-use_fast_math", "-ftz=true")), \
    "fbq kernels require IEEE denormals (no FTZ / fast math)"
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off",
             "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include"]


def _sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    return cu, cpp


def _headers():
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "host", "*.h*"))
    hs += glob.glob(os.path.join(ROOT, "include", "*.h"))
    return hs


def _stale(obj: str, src: str, newest_header: float) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return t < os.path.getmtime(src) or t < newest_header


def build(verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    cu, cpp = _sources()
    newest_h = max([os.path.getmtime(h) for h in _headers()] + [0.0])
    jobs = []
    objs = []
    for src in cu:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, src, newest_h):
            jobs.append([NVCC, *CU_FLAGS, "-c", src, "-o", obj])
    for src in cpp:
        obj = os.path.join(OBJ, "host_" + os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, src, newest_h):
            jobs.append(["g++", *CXX_FLAGS, "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print("[fbq build]", os.path.basename(cmd[-3]), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print("[fbq build] linked", LIB, flush=True)
    return LIB


if __name__ == "__main__":
    build(verbose="-q" not in sys.argv)
