"""Compile the CUDA library in-tree (libghostmg_b200.so next to this file).

nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false: sm_100a only, and
no multiply-add contraction (the kernels restate the reference's rounding
order; the only FMAs are explicit __fma_rn calls).
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libghostmg_b200.so")
SOURCES = ["context.cu", "gs_sweep.cu", "gs_small.cu", "gs_stream.cu", "gs_diag.cu", "gs_chain.cu", "coarse_dense.cu", "setup_ops.cu", "ghost_ops.cu", "grid_ops.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-cudart", "static",
]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "ghostmg_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(verbose=False, force=False, csrc=CSRC, lib=LIB, defines=()):
    """Compile `csrc` into `lib` (an alternate source tree / output path is
    for A/B experiments with tools/build_alt.sh)."""
    if not force and lib == LIB and not needs_build():
        return LIB
    objs = []
    build_dir = os.path.join(os.path.dirname(lib), "..", "build", "csrc") if lib == LIB else os.path.join(
        os.path.dirname(lib), "obj")
    os.makedirs(build_dir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(csrc, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose and out:
            sys.stderr.write(out.decode())
    tmp = lib + ".tmp"
    cmd = [NVCC, *FLAGS, "-shared", *objs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(LIB)
