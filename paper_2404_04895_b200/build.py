"""Build libtaco.so in-tree for sm_100a (``python -m paper_2404_04895_b200.build``).

Plain nvcc, no torch extension machinery: the C ABI (include/taco.h) has no
torch types, and the shared object travels to the GPU box with the repo.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("TACO_BUILD_OUT") or os.path.join(HERE, "lib", "libtaco.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    # A/B experiments only (scripts/ab_variant.sh): extra -D flags
    *os.environ.get("TACO_NVCC_EXTRA", "").split(),
]
OBJ_DIR = os.path.join(os.path.dirname(HERE), "build",
                       "taco_obj" if not os.environ.get("TACO_BUILD_OUT") else
                       "taco_obj_" + os.path.basename(os.environ["TACO_BUILD_OUT"]).replace(".so", ""))


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    newest = max(os.path.getmtime(p) for p in deps)
    return newest > os.path.getmtime(OUT)


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu into lib/libtaco.so (skipped when up to date)."""
    if not force and not _stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    os.makedirs(OBJ_DIR, exist_ok=True)
    # one nvcc per translation unit, in parallel, then a shared link
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, "-I", INCLUDE, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
        objs.append(obj)
    for cmd, proc in procs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, cmd)
    tmp = OUT + ".tmp"
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    subprocess.run(link, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
