"""Build the in-tree C-ABI library librqmc.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librqmc.so")
SOURCES = [os.path.join(CSRC, f) for f in
           ("rqmc_plan.cpp", "rqmc_gen.cu", "rqmc_gemm.cu", "rqmc_fine.cu", "rqmc_tree.cu", "rqmc_fft.cu")]
HEADERS = [os.path.join(CSRC, "rqmc_internal.h"), os.path.join(CSRC, "rqmc_device.cuh"),
           os.path.join(CSRC, "rqmc_exp2_table.h"), os.path.join(ROOT, "include", "rqmc.h")]
DEPS = SOURCES + HEADERS
OBJDIR = os.path.join(PKG, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def needs_build(lib: str = LIB, defines=()) -> bool:
    """lib missing, older than a source / header, or (variants) built with other -D flags."""
    if not os.path.exists(lib):
        return True
    if lib != LIB:
        stamp = lib + ".defs"
        if not os.path.exists(stamp) or open(stamp).read() != " ".join(defines):
            return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _compile(src: str, verbose: bool, objdir: str = OBJDIR, defines=()) -> str:
    """One translation unit -> object (the units compile in parallel; the .cu files are heavy)."""
    obj = os.path.join(objdir, os.path.basename(src) + ".o")
    if os.path.exists(obj) and all(os.path.getmtime(obj) > os.path.getmtime(d) for d in [src, *HEADERS]):
        return obj
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c",
           "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"),
           *[f"-D{d}" for d in defines], "-o", obj + ".tmp", src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build librqmc.so; `variant` + `defines` build an A/B experiment library librqmc_<variant>.so
    (loaded only when RQMC_LIB points at it)."""
    lib = LIB if not variant else os.path.join(PKG, f"librqmc_{variant}.so")
    objdir = OBJDIR if not variant else os.path.join(OBJDIR, variant)
    if not force and not needs_build(lib, defines):
        return lib
    os.makedirs(objdir, exist_ok=True)
    if force:
        for f in os.listdir(objdir):
            if f.endswith(".o"):
                os.remove(os.path.join(objdir, f))
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, objdir, defines), SOURCES))
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", lib + ".tmp", *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking librqmc.so")
    os.replace(lib + ".tmp", lib)
    if variant:
        with open(lib + ".defs", "w") as fh:
            fh.write(" ".join(defines))
    return lib


if __name__ == "__main__":
    # python _build.py [--force] [-v] [--variant NAME -DMACRO[=V] ...]
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else ""
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv, verbose="-v" in argv, variant=var, defines=defs))
