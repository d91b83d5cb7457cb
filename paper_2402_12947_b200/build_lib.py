"""Build the in-tree sm_100a shared library (no GPU needed: nvcc cross-compiles).

    python -m paper_2402_12947_b200.build_lib [--force]

Produces ``paper_2402_12947_b200/lib/libsimplexmg_b200.so`` (C-ABI declared in
``include/simplexmg_b200.h``) with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo``; ptxas register/spill report goes to ``lib/ptxas.log``.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libsimplexmg_b200.so")
HEADER = os.path.join(ROOT, "include", "simplexmg_b200.h")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
COMPILE_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-Xptxas", "-v",
]
LINK_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-shared",
    "-Xlinker", "-rpath=/usr/local/cuda/lib64",
]
EXTRA = os.environ.get("SMG_NVCC_EXTRA", "").split()


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER, __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def _compile(src: str, objdir: str, force: bool):
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER, __file__]
    if (not force and os.path.exists(obj)
            and all(os.path.getmtime(p) <= os.path.getmtime(obj) for p in deps)):
        return obj, None, ""
    cmd = [NVCC] + COMPILE_FLAGS + EXTRA + ["-c", "-o", obj, src]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return obj, res.returncode, " ".join(cmd) + "\n" + res.stdout + res.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc per source file, in parallel (objects cached under lib/obj by
    mtime), then one link."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, objdir, force), srcs))
    log_path = os.path.join(LIBDIR, "ptxas.log")
    old_log = {}
    if os.path.exists(log_path):
        # keep the register/spill report of sources that were not recompiled
        for blk in open(log_path).read().split("\n#### ")[1:]:
            old_log[blk.split("\n", 1)[0]] = blk.split("\n", 1)[1] if "\n" in blk else ""
    with open(log_path, "w") as f:
        for src, (obj, rc, out) in zip(srcs, results):
            name = os.path.basename(src)
            f.write("\n#### " + name + "\n" + (out if rc is not None else old_log.get(name, "")))
    for src, (obj, rc, out) in zip(srcs, results):
        if rc not in (None, 0):
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)} with exit code {rc}")
    tmp = LIB + ".tmp"
    cmd = [NVCC] + LINK_FLAGS + ["-o", tmp] + [r[0] for r in results]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"link failed with exit code {res.returncode}")
    os.replace(tmp, LIB)
    if verbose:
        print(open(log_path).read())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
