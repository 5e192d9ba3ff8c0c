"""Build libffsat.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

Each translation unit compiles in parallel to an object file, then nvcc links the shared library."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SRC = [os.path.join(CSRC, f) for f in ("ffsat.cu", "eval.cu", "eval_f32.cu", "eval_f64.cu", "sym_f32.cu", "sym_f64.cu",
                                       "host.cpp")]
OBJDIR = os.path.join(HERE, "build")
OUT = os.path.join(HERE, "libffsat.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]


def deps():
    return SRC + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        [os.path.join(os.path.dirname(HERE), "include", "ffsat.h"), __file__]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in deps())


def _obj(src):
    return os.path.join(OBJDIR, os.path.basename(src) + ".o")


def build(force: bool = False, verbose: bool = False, extra=()) -> str:
    if not (force or needs_build()):
        return OUT
    os.makedirs(OBJDIR, exist_ok=True)
    cmds = [[NVCC, *FLAGS, *extra, "-c", "-o", _obj(s), s] for s in SRC]

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        return subprocess.run(cmd, capture_output=True, text=True)
    with ThreadPoolExecutor(len(cmds)) as ex:
        results = list(ex.map(run, cmds))
    for r in results:
        if r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        if r.returncode:
            raise RuntimeError("nvcc failed: " + " ".join(r.args))
    link = [NVCC, *ARCH, "-shared", "-o", OUT, *[_obj(s) for s in SRC]]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.check_call(link)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, extra=["-Xptxas", "-v"] if "--ptxas-v" in sys.argv else [])
