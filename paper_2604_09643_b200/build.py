"""Build libpa.so in-tree with nvcc for sm_100a (no JIT cache, so the .so travels with the repo).

The library is split into translation units (host API + small kernels, and one unit per operator-kernel
family) compiled in parallel, then linked into one shared object."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SRC = [os.path.join(CSRC, f) for f in ("pa_api.cu", "k_dep.cu", "k_tay.cu", "k_svd.cu", "k_direct_gauss.cu",
                                       "k_direct_exp.cu", "k_direct_pow.cu", "k_generic.cu")]
HDRS = [os.path.join(CSRC, f) for f in ("pa_kernels.cuh", "pa_plan.h", "k_direct_impl.cuh")] + \
    [os.path.join(ROOT, "include", "pa.h")]
DEPS = SRC + HDRS
LIB = os.path.join(HERE, "libpa.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", *ARCH, "-lineinfo", "-ftz=true", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]


def source_hash() -> str:
    """sha256 (16 hex) of every source libpa is built from: stamps ncu captures (profiles/) so bench.py can
    refuse counters measured on another build."""
    import hashlib

    h = hashlib.sha256()
    for p in sorted(DEPS):
        with open(p, "rb") as fh:
            h.update(os.path.basename(p).encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, defs=(), lib: str = LIB, objdir: str = OBJ) -> str:
    """Compile every translation unit (in parallel) and link libpa.so; `defs` are extra -D flags (variants)."""
    if not (force or stale(lib)):
        return lib
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *defs, *inc, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, flush=True)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(len(SRC), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SRC))
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
