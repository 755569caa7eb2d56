"""Builds libndgi.so in-tree with nvcc for sm_100a (B200).

    python paper_2604_12625_b200/build.py [--verbose]

Every .cu under csrc/ is compiled with
`-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo` into one shared
library exporting the C ABI of include/ndgi.h.  The CUDA runtime is linked
statically so the library does not depend on torch's cudart.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libndgi.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ndgi.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(verbose: bool = False, force: bool = False, out: str | None = None, defines=()) -> str:
    lib = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    # experiment variants keep their objects outside the repo (gpurun snapshot size)
    objdir = os.path.join(HERE, "build") if out is None else os.path.join("/tmp", "ndgi_" + os.path.basename(lib).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    extra = (["-Xptxas", "-v"] if verbose else []) + [f"-D{d}" for d in defines]

    hdr_t = max(os.path.getmtime(d) for d in _deps() if not d.endswith(".cu"))
    stamp = os.path.join(objdir, "flags.txt")
    flags_key = " ".join(FLAGS + extra)
    same_flags = os.path.exists(stamp) and open(stamp).read() == flags_key

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        # incremental: an object newer than its source and every header, built
        # with the same flags, is reused
        if (same_flags and os.path.exists(obj) and
                os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t)):
            return obj
        cmd = [NVCC, *FLAGS, *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    with open(stamp, "w") as f:
        f.write(flags_key)
    # objects of deleted sources must not be linked
    for o in glob.glob(os.path.join(objdir, "*.o")):
        if o not in objs:
            os.remove(o)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-Xcompiler", "-fPIC", *objs, "-o", lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


CHECKED_LIB = os.path.join(HERE, "libndgi_checked.so")


def build_checked(force: bool = False) -> str:
    """The self-checking test build (NDGI_CHECKED: bounds checks that trap;
    NDGI_JITTER: random per-warp delays at every synchronisation point) used
    by tests/test_gpu_selfcheck.py in place of compute-sanitizer."""
    if not force and os.path.exists(CHECKED_LIB) and os.path.getmtime(CHECKED_LIB) >= max(
            os.path.getmtime(d) for d in _deps()):
        return CHECKED_LIB
    return build(out=CHECKED_LIB, defines=["NDGI_CHECKED=1", "NDGI_JITTER=1"])


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True))
