"""Build liblw_b200.so in-tree for sm_100a (called by __graft_entry__.build()).

nvcc flags that matter for correctness:
  -fmad=false            no mul+add contraction: device FP64 matches the CPU oracle and the
                         reference bit for bit (explicit __fma_rn is kept where glibc fuses)
  -Xcompiler -ffp-contract=off   same for host code (alias tables)
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(BUILD, "liblw_b200.so")
SOURCES = ["lw_capi.cu", "lw_bvh_build.cu", "lw_render.cu", "lw_sah_build.cu"]
# every header of the library (any change rebuilds all translation units)
HEADERS = sorted(f for f in os.listdir(HERE) if f.endswith((".cuh", ".h"))) + [os.path.join("..", "..", "include", "lw_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-warn-spills",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + HEADERS + ["build.py"]
    return any(os.path.getmtime(os.path.join(HERE, d)) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile liblw_b200.so (or an experiment variant with extra -D defines into `out`)."""
    lib = out or LIB
    if not force and not defines and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    objs = []
    env = dict(os.environ)
    env.pop("CC", None)
    env.pop("CXX", None)
    for src in SOURCES:
        tag = "_".join(d.replace("=", "") for d in defines)
        obj = os.path.join(BUILD, os.path.splitext(src)[0] + f"{tag}.o")
        cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(HERE, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.run(cmd, check=True, env=env)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
                    "-cudart", "static"], check=True, env=env)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None))
