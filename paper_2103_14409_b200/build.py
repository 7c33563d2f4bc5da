"""Build liblscat.so (all CUDA sources, sm_100a) in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, one object per source (parallel),
linked against the NCCL that ships with torch (the same libnccl.so.2 torch loads).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "liblscat.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return os.path.join(d, "include"), os.path.join(d, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def flags():
    inc, _ = nccl_dirs()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                   "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
                   "-I", inc]


def _compile(src, extra):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "lscat.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj, None
    cmd = [NVCC] + flags() + extra + os.environ.get("LSCAT_NVCC_EXTRA", "").split() + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"{' '.join(cmd)}\n{r.stdout}\n{r.stderr}"
    return obj, None


# per-file extra flags: the reducer/generator need IEEE-exact double arithmetic (explicit _rn
# intrinsics are used too; --fmad=false is a second guard)
EXTRA = {"reduce.cu": ["--fmad=false"], "gen.cu": ["--fmad=false"], "stats.cu": ["--fmad=false"]}


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(jobs or os.cpu_count() or 4) as ex:
        res = list(ex.map(lambda s: _compile(s, EXTRA.get(os.path.basename(s), [])), srcs))
    errs = [e for _, e in res if e]
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n\n".join(errs))
    objs = [o for o, _ in res]
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _, libdir = nccl_dirs()
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
