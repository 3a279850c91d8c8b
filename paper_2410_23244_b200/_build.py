"""In-tree build of the sm_100a library (`lib/libbart_b200.so`).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the build
container; the .so travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libbart_b200.so")
SOURCES = ["propose.cu", "sweep.cu", "forest.cu", "binning.cu", "capi.cu"]
HEADERS = ["common.cuh", "internal.h", "propose.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the decision arithmetic must round exactly like numpy/numba: no FMA contraction
    "-fmad=false",
    "--shared", "-Xcompiler", "-fPIC", "-cudart", "static",
]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "bart_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Compile the library; `out`/`defines` build instrumented or experiment variants elsewhere."""
    lib = out or LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", lib + ".tmp",
           *[os.path.join(CSRC, f) for f in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose:
        print(res.stderr, file=sys.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


TIMELINE_LIB = os.path.join(PKG, "lib", "libbart_b200_timeline.so")


def build_timeline(defines: tuple = ()) -> str:
    """The instrumented variant tools/timeline.py loads (per-phase clock stamps)."""
    if defines:
        tag = "_".join(d.replace("=", "") for d in defines)
        return build(out=TIMELINE_LIB.replace(".so", f"_{tag}.so"), defines=("BART_TIMELINE=1", *defines))
    return build(out=TIMELINE_LIB, defines=("BART_TIMELINE=1",))


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
