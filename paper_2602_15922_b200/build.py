"""Build libdz.so in-tree with nvcc for sm_100a only.

    python -m paper_2602_15922_b200.build [--force] [--verbose]

Sources: csrc/*.cu (kernels), csrc/dz.cpp (C ABI).  cudart is linked
statically; NCCL is the torch-bundled libnccl.so.2 (rpath to its directory).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdz.so")
TRACE_LIB = os.path.join(HERE, "libdz_trace.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    for base in [sysconfig.get_paths()["purelib"], *sys.path]:
        inc = os.path.join(base, "nvidia", "nccl", "include")
        lib = os.path.join(base, "nvidia", "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("nccl.h / libnccl.so.2 not found (expected the torch-bundled nvidia-nccl wheel)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + [os.path.join(CSRC, "dz.cpp")]


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "dz.h")]


def source_sha() -> str:
    """Identity of a build: sha256 (16 hex) over every source the library compiles from and this build
    script (its flags).  The linked libdz.so is not byte-reproducible (the device-link step embeds
    nvcc's temporary file names), the objects and their SASS are."""
    import hashlib
    h = hashlib.sha256()
    for p in sorted(deps()) + [os.path.abspath(__file__)]:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """trace=True builds the diagnostics variant libdz_trace.so (-DDZ_TRACE: K2 cycle trace and
    per-CTA timeline, see dz_debug_trace); tools load it through DZ_LIB_PATH."""
    out = TRACE_LIB if trace else LIB
    extra = os.environ.get("DZ_BUILD_EXTRA", "").split()  # experiments: extra nvcc flags ...
    if extra:
        out = os.environ["DZ_BUILD_OUT"]                      # ... built into a separate library
    if not force and not trace and not extra and up_to_date():
        return LIB
    inc, lib = nccl_dirs()
    objdir = os.path.join(HERE, "build_x" if extra else ("build_trace" if trace else "build"))
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden", *ARCH,
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc] + (["-DDZ_TRACE"] if trace else []) + extra
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *common, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "cu"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = out + f".tmp{os.getpid()}"
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath,{lib}", "-lrt", "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.check_call(link)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, trace="--trace" in sys.argv))
