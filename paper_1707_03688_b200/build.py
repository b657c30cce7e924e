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
SOURCES = [os.path.join(CSRC, f) for f in ("nslct.cu", "planner.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("kernels.cuh", "planner.h")] + \
    [os.path.join(ROOT, "include", "nslct.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("NSLCT_NVCC_EXTRA", "").split()
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-O3", "-shared", "-Xptxas", "-v", "--threads", "0"]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    cmd = [NVCC] + FLAGS + EXTRA + ["-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp"] + SOURCES
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError("nvcc failed (see %s)" % log)
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
