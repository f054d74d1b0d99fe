"""Build libapnn.so (sm_100a) in-tree with nvcc.

Every .cu under csrc/ is compiled with
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
and linked into paper_2106_12169_b200/libapnn.so (static cudart, no torch
dependency: the library is a plain C ABI).  Objects go to build/ next to it.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
SO = os.path.join(HERE, "libapnn.so")
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "--split-compile=0",  # parallel device optimisation (gemm_tc.cu 4.3 -> 1.5 min)
         "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "apnn.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), so_path: str = None, build_dir: str = None) -> str:
    """Compile every csrc/*.cu; `extra`/`so_path`/`build_dir` build experiment variants side by side."""
    global BUILD, SO
    if so_path or build_dir:
        BUILD, SO = build_dir or BUILD + "_exp", so_path or SO
    os.makedirs(BUILD, exist_ok=True)
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "apnn.h")]
    jobs = []
    objs = []
    for src in _sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append([NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(SO, objs):
        tmp = SO + f".tmp{os.getpid()}"
        run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
        os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    # python build.py [--force] [--variant NAME -DFOO=1 ...]  (variant -> libapnn_NAME.so)
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        name = args[i + 1]
        defs = [a for a in args[i + 2:] if a.startswith("-D")]
        print(build(force=True, verbose=False, extra=defs, so_path=os.path.join(HERE, f"libapnn_{name}.so"),
                    build_dir=os.path.join(HERE, f"build_{name}")))
    else:
        print(build(force="--force" in args, verbose=True))
