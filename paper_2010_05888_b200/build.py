"""Build libgar.so (sm_100a) in-tree: nvcc -gencode arch=compute_100a,code=sm_100a.

Objects go to ``_build/``; units are compiled in parallel and only rebuilt
when their source or any header is newer.  This file imports nothing from the
package, so it can run on a clean checkout before libgar.so exists:

    python paper_2010_05888_b200/build.py        (or python -m paper_2010_05888_b200.build)

Concurrent builders (one per torchrun rank) serialise on ``_build/.lock``; the
later ones find everything up to date.
"""
from __future__ import annotations

import concurrent.futures as cf
import fcntl
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libgar.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", CSRC, "-I", os.path.join(ROOT, "include")]


def _headers():
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hs.append(os.path.join(ROOT, "include", "gar.h"))
    return hs


def _regen_networks():
    gen = os.path.join(CSRC, "gen_networks.py")
    out = os.path.join(CSRC, "networks.cuh")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(gen):
        subprocess.check_call([sys.executable, gen, out])


def _compile(src, obj, log):
    cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stderr[-4000:]}")
    os.replace(obj + ".tmp", obj)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with open(os.path.join(OBJ, ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            return _build_locked(verbose, jobs)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build_locked(verbose: bool, jobs: int | None) -> str:
    _regen_networks()
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    todo, objs = [], []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_mtime):
            todo.append((s, o, o[:-2] + ".log"))
    stale = [o for o in glob.glob(os.path.join(OBJ, "*.o")) if o not in objs]
    for o in stale:                       # a removed source: drop its object and log, and relink below
        os.remove(o)
        if os.path.exists(o[:-2] + ".log"):
            os.remove(o[:-2] + ".log")
    if todo:
        jobs = jobs or max(1, os.cpu_count() or 1)
        if verbose:
            print(f"[libgar] compiling {len(todo)} units with {jobs} jobs", flush=True)
        with cf.ThreadPoolExecutor(jobs) as ex:
            for o in ex.map(lambda t: _compile(*t), todo):
                if verbose:
                    print(f"[libgar]   {os.path.basename(o)}", flush=True)
    if todo or stale or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcuda"])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
