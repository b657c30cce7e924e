"""One 16384^2 complex64 transform through the library (for ncu captures of the large-N
passes).  Usage: python tools/c5_once.py [n] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1707_03688_b200 import nslct  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mr, _ = synth.config_streams(5)
M = synth.random_symplectic(mr)
g = torch.Generator(device="cuda")
g.manual_seed(5)
x = torch.randn((1, n, n), dtype=torch.complex64, device="cuda", generator=g)
with nslct.Plan(n, M, 1) as p:
    for _ in range(reps):
        y = p.exec(x)
    torch.cuda.synchronize()
print("ok", n, float(y.abs().mean()))
