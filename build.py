"""Build the sm_100a CUDA library in-tree (nvcc, no cmake):
paper_2411_16786_b200/_dice_b200.so. Usage: python build.py [--force]"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2411_16786_b200")
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_dice_b200.so")
SOURCES = ["dice_gemm.cu", "dice_ops.cu", "dice_ep.cu"]
HEADERS = ["dice_gemm.h", "dice_ptx.cuh", os.path.join("..", "..", "include", "dice_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = OUT) -> str:
    """defines / out: an experiment build (-D switches) written elsewhere
    (loaded by the probes through DICE_LIB_PATH); the product build has none."""
    if out == OUT and not defines and not force and not _stale():
        return OUT
    objs = []
    for src in SOURCES:
        obj = os.path.join(os.path.dirname(out), src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = out + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, out)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    # python build.py [--force] [-v] [--variant NAME -DSWITCH ...]
    args = sys.argv[1:]
    if "--variant" in args:
        name = args[args.index("--variant") + 1]
        d = os.path.join(ROOT, "build", "variants", name)
        os.makedirs(d, exist_ok=True)
        print(build(defines=[a[2:] for a in args if a.startswith("-D")],
                    out=os.path.join(d, "_dice_b200.so")))
    else:
        print(build(force="--force" in args, verbose="-v" in args))
