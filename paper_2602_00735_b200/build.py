"""Build libhelm.so in-tree: nvcc for sm_100a only (no other architectures, no JIT cache)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libhelm.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nccl_dirs():
    """(include, lib) of the NCCL that torch's wheel set ships (nvidia-nccl), or None."""
    try:
        import nvidia.nccl as m
        base = list(m.__path__)[0]
    except Exception:
        base = None
    for b in [base, "/usr"]:
        if b and os.path.exists(os.path.join(b, "include", "nccl.h")):
            lib = os.path.join(b, "lib")
            if os.path.exists(os.path.join(lib, "libnccl.so")) or os.path.exists(os.path.join(lib, "libnccl.so.2")):
                return os.path.join(b, "include"), lib
    return None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """One object per .cu, compiled in parallel (whole-file device code: no relocatable device linking), then one
    shared link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    base = [nvcc, *flags, *os.environ.get("HELM_NVCC_EXTRA", "").split(), "-I", INCLUDE, "-I", CSRC]
    nd = nccl_dirs()
    if nd:
        inc, lib = nd
        libname = "nccl" if os.path.exists(os.path.join(lib, "libnccl.so")) else ":libnccl.so.2"
        base += ["-DHELM_HAVE_NCCL", "-I", inc]
        link = ["-L", lib, "-l" + libname, "-Xlinker", "-rpath=" + lib]
    else:
        link = []
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]

    def compile_one(so):
        src, obj = so
        return subprocess.run(base + ["-c", src, "-o", obj], capture_output=True, text=True), src

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, zip(srcs, objs)))
    lcmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, *link, "-o", LIB + ".tmp"]
    log = os.path.join(PKG, "build.log")
    with open(log, "w") as f:
        for r, src in results:
            f.write(" ".join(base + ["-c", src]) + "\n" + r.stdout + r.stderr)
    bad = [(r, src) for r, src in results if r.returncode != 0]
    if bad:
        sys.stderr.write("".join(r.stderr[-6000:] for r, _ in bad))
        raise RuntimeError(f"nvcc failed on {[os.path.basename(s) for _, s in bad]} (see {log})")
    res = subprocess.run(lcmd, capture_output=True, text=True)
    with open(log, "a") as f:
        f.write(" ".join(lcmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError(f"nvcc link failed (see {log})")
    if verbose:
        sys.stderr.write("".join(r.stderr for r, _ in results))
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
