"""Build libnslct.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_1707_03688_b200.build            # incremental (skips if up to date)
    python -m paper_1707_03688_b200.build --force
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnslct.so")
SOURCES = [os.path.join(CSRC, f) for f in ("nslct.cu", "bluestein.cu", "planner.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("kernels.cuh", "planner.h", "bluestein.h")] + \
    [os.path.join(ROOT, "include", "nslct.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("NSLCT_NVCC_EXTRA", "").split()
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v"]


def nccl_include():
    """Directory of nccl.h (types only: the library dlopens libnccl.so.2 at run time).
    The NCCL wheel PyTorch ships with, else the system header."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for loc in (spec.submodule_search_locations or []) if spec else []:
            d = os.path.join(loc, "include")
            if os.path.exists(os.path.join(d, "nccl.h")):
                return d
    except Exception:
        pass
    return "/usr/include"


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force=False, verbose=False):
    """Compile every source to an object in parallel (one nvcc per translation unit),
    then link the shared library."""
    if not force and up_to_date():
        return LIB
    objs, procs, logs = [], [], []
    for src in SOURCES:
        obj = os.path.join(HERE, "build_" + os.path.basename(src) + ".o")
        cmd = [NVCC] + FLAGS + EXTRA + ["-I", os.path.join(ROOT, "include"), "-I", nccl_include(), "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    ok = True
    for cmd, pr in procs:
        out, err = pr.communicate()
        logs.append(" ".join(cmd) + "\n" + out + err)
        if pr.returncode != 0:
            ok = False
            sys.stderr.write(err[-4000:])
    if ok:
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp"] + objs + ["-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            ok = False
            sys.stderr.write(res.stderr[-4000:])
    with open(os.path.join(HERE, "build.log"), "w") as f:
        f.write("\n".join(logs))
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    if not ok:
        raise RuntimeError("nvcc failed (see %s)" % os.path.join(HERE, "build.log"))
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
