"""Per-pass times of ONE batched n x n complex64 transform measured the way
tools/slab_pass_timing.py measures the slab passes: each pass launched alone
(nslct_exec_pass) between two events with a device synchronize after it, so the two
numbers compare like with like (a pass timed alone starts on an idle GPU with a cold L2;
inside nslct_exec the passes run back to back).  Usage: python tools/batched_pass_timing.py [n] [reps]"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1707_03688_b200 import nslct  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mr, _ = synth.config_streams(5)
M = synth.random_symplectic(mr)
g = torch.Generator(device="cuda")
g.manual_seed(5)
x = torch.randn((1, n, n), dtype=torch.complex64, device="cuda", generator=g)
bufs = [torch.empty_like(x), torch.empty_like(x)]
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
with nslct.Plan(n, M, 1, profile=True) as p:
    npass = p.info()["n_passes"]
    tot = [0.0] * npass
    for rep in range(reps + 1):
        cur = x
        for k in range(npass):
            dst = bufs[k % 2]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nslct.lib().nslct_exec_pass(p._h, k, ctypes.c_void_p(cur.data_ptr()), ctypes.c_void_p(dst.data_ptr()), stream)
            e1.record()
            torch.cuda.synchronize()
            if rep > 0:
                tot[k] += e0.elapsed_time(e1) / reps
            cur = dst
    out = torch.empty_like(x)
    for _ in range(3):
        p.exec(x, out)
    torch.cuda.synchronize()
    p.pass_ms()
    for _ in range(reps):
        p.exec(x, out)
    torch.cuda.synchronize()
    inside = p.pass_ms()
print(json.dumps({"n": n, "pass_ms_alone": [round(t, 4) for t in tot], "pass_ms_inside_exec": [round(t, 4) for t in inside]}))
