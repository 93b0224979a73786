"""Build libbf200.so (the C-ABI library) for sm_100a with nvcc.

Compiles csrc/*.cu and the generated instantiation shards csrc/gen/*.cu in
parallel (one nvcc per translation unit) and links them into
paper_2512_15595_b200/libbf200.so (in-tree, so it travels with the repo to the
GPU box).  Incremental: a translation unit is rebuilt only if a source or
header is newer than its object.

-lineinfo: the hand-written translation units always carry it.  The generated
specializations (~1,200 kernels) carry it only in the profiling build
(`python -m paper_2512_15595_b200.build --lineinfo` ->
libbf200_lineinfo.so, selected with BF200_LIB=... for ncu --import-source
captures): with -lineinfo ptxas embeds the PTX text of every kernel twice,
which made the default library 4x larger (126 MB) for no run-time effect.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build", "obj")
LIB = os.path.join(PKG, "libbf200.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
LIB_LINEINFO = os.path.join(PKG, "libbf200_lineinfo.so")
FLAGS = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", INCLUDE, "-I", CSRC]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(INCLUDE, "bf.h")]


def sources():
    gen = os.path.join(CSRC, "gen_instances.py")
    shards = sorted(glob.glob(os.path.join(CSRC, "gen", "inst_*.cu")))
    if not shards or any(os.path.getmtime(gen) > os.path.getmtime(s) for s in shards):
        subprocess.check_call([sys.executable, gen], cwd=CSRC)
        shards = sorted(glob.glob(os.path.join(CSRC, "gen", "inst_*.cu")))
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + shards


def _compile(src, hdr_mtime, verbose, lineinfo_all=False):
    gen = os.sep + "gen" + os.sep in src
    lineinfo = lineinfo_all or not gen
    sub = OBJ + ("_li" if lineinfo_all and gen else "")
    os.makedirs(sub, exist_ok=True)
    obj = os.path.join(sub, os.path.relpath(src, CSRC).replace(os.sep, "_") + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj, False
    cmd = [NVCC, *ARCH, *FLAGS, *(["-lineinfo"] if lineinfo else []), "-c", src, "-o", obj + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj, True


def build(verbose: bool = False, jobs: int | None = None, lineinfo: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()
    hdr = max(os.path.getmtime(h) for h in _headers())
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    with ThreadPoolExecutor(jobs) as ex:
        res = list(ex.map(lambda s: _compile(s, hdr, verbose, lineinfo), srcs))
    objs = [o for o, _ in res]
    lib = LIB_LINEINFO if lineinfo else LIB
    if any(c for _, c in res) or not os.path.exists(lib) or \
            any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs):
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, lineinfo="--lineinfo" in sys.argv))
