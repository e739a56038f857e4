"""Build libwino.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2201_10369_b200.build [--force] [--verbose]

Device code: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
(-fmad=false: nothing is contracted behind the explicit __fmaf_rn / fma.rn.f32x2 chains,
DESIGN.md §2.3).  Host code: -O2 -ffp-contract=off (recipe R64 is bit-exact only without
contraction).

Provenance: the library is stamped with the SHA-256 of every source, header and compiler
flag (libwino.so.stamp).  needs_build() compares CONTENTS, not mtimes, so a library copied
to another machine is reused only when it was built from exactly these sources, and any
edit forces a rebuild (objects are rebuilt per translation unit by the same rule).
Concurrent builders (one per torchrun rank) serialise on an fcntl lock and link through a
per-process temporary file.
"""
from __future__ import annotations

import concurrent.futures as cf
import contextlib
import fcntl
import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libwino.so")
STAMP = LIB + ".stamp"
LOCK = os.path.join(HERE, ".build.lock")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
          "-Xcompiler", "-fPIC,-O2,-ffp-contract=off,-fno-fast-math", "--expt-relaxed-constexpr"]
LINK = ["-shared", "-lcudart"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(HERE, "..", "include", "wino.h")])


def _digest(paths, extra=()) -> str:
    h = hashlib.sha256()
    for p in paths:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    for e in extra:
        h.update(str(e).encode())
    return h.hexdigest()


def _lib_digest() -> str:
    return _digest(_sources() + _headers(), [NVCC, ARCH, COMMON, LINK])


def _obj(src: str) -> str:
    return os.path.join(BUILD, os.path.basename(src) + ".o")


def _obj_digest(src: str) -> str:
    return _digest([src] + _headers(), [NVCC, ARCH, COMMON])


def _read(path: str) -> str:
    try:
        with open(path) as f:
            return f.read().strip()
    except OSError:
        return ""


def needs_build() -> bool:
    return not os.path.exists(LIB) or _read(STAMP) != _lib_digest()


def _compile(src: str, verbose: bool) -> str:
    obj = _obj(src)
    tmp = f"{obj}.{os.getpid()}.tmp"
    cmd = [NVCC, *ARCH, *COMMON, "-c", src, "-o", tmp]
    if verbose and src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, obj)
    with open(obj + ".stamp", "w") as f:
        f.write(_obj_digest(src))
    return obj


@contextlib.contextmanager
def _locked():
    with open(LOCK, "w") as f:
        fcntl.flock(f, fcntl.LOCK_EX)
        try:
            yield
        finally:
            fcntl.flock(f, fcntl.LOCK_UN)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    with _locked():
        if not force and not needs_build():   # another process finished it meanwhile
            return LIB
        os.makedirs(BUILD, exist_ok=True)
        srcs = _sources()
        todo = [s for s in srcs if force or _read(_obj(s) + ".stamp") != _obj_digest(s) or not os.path.exists(_obj(s))]
        # longest translation units first (they bound the parallel build time)
        todo.sort(key=lambda s: -os.path.getsize(s))
        with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            list(ex.map(lambda s: _compile(s, verbose), todo))
        objs = [_obj(s) for s in srcs]
        tmp = f"{LIB}.{os.getpid()}.tmp"
        r = subprocess.run([NVCC, *ARCH, "-o", tmp, *objs, *LINK], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
        with open(STAMP, "w") as f:
            f.write(_lib_digest())
    return LIB


def build_info() -> dict:
    """Which library is loaded and whether it matches the sources (reported by smoke())."""
    return {"lib": LIB, "stamp": _read(STAMP), "sources_digest": _lib_digest(), "up_to_date": not needs_build()}


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
