"""Build the sm_100a CUDA library in-tree: paper_1805_05225_b200/lib/libseqloom_cuda.so.

    python -m paper_1805_05225_b200.build [--verbose-ptxas] [--force]

Each csrc/*.cu is compiled with nvcc for sm_100a only (no PTX fallback, no
other arch) and linked into one shared library exporting the C ABI declared in
include/seqloom_cuda.h.  Incremental: an object is rebuilt when its source or
any header in csrc/ or include/ is newer.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
# SL_EXPERIMENTS=1: a separate build with the measurement hooks (-DSL_EXPERIMENTS:
# per-step trace stamps, the experimental kernels) into build_obj_exp/ and lib_exp/;
# load it with SL_LIB_PATH=paper_1805_05225_b200/lib_exp/libseqloom_cuda.so
EXPERIMENTS = os.environ.get("SL_EXPERIMENTS", "") not in ("", "0")
OBJ = os.path.join(PKG, "build_obj_exp" if EXPERIMENTS else "build_obj")
LIB_DIR = os.path.join(PKG, "lib_exp" if EXPERIMENTS else "lib")
LIB = os.path.join(LIB_DIR, "libseqloom_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
                  "-diag-suppress", "177,550", "--diag-error", "20013,20014,20015"] + \
    (["-DSL_EXPERIMENTS"] if EXPERIMENTS else [])


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
            glob.glob(os.path.join(ROOT, "include", "*.h")) +
            glob.glob(os.path.join(ROOT, "include", "**", "*.hpp"), recursive=True))


def _stale(src: str, obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *deps])


def _compile(src: str, obj: str, ptxas_v: bool) -> str:
    if src.endswith(".cu"):
        cmd = [NVCC, *NVFLAGS, *(["-Xptxas", "-v"] if ptxas_v else []), "-c", src, "-o", obj]
    else:  # host C++ on top of the C ABI
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-I" + os.path.join(ROOT, "include"),
               "-I/usr/local/cuda/include", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(force: bool = False, ptxas_v: bool = False, quiet: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(HOST, "*.cpp")))
    deps = _headers()
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(s, o, deps):
            jobs.append((s, o))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for (s, _), log in zip(jobs, ex.map(lambda j: _compile(j[0], j[1], ptxas_v), jobs)):
            if log and (ptxas_v or not quiet):
                print(f"== {os.path.basename(s)}\n{log}", file=sys.stderr)
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda", "-Xlinker", "-Bsymbolic"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose-ptxas", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, ptxas_v=a.verbose_ptxas, quiet=False))
