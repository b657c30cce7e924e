"""A/B of the large-N kernels (the default vs the generic one-CTA-per-line kernels) on one GPU:
per-pass CUDA-event times of one n x n complex64 transform, and the C5 slab passes of one
rank.  Usage: python tools/large_n_ab.py [n] [batch]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1707_03688_b200 import nslct  # noqa: E402


def run(n, batch, kernels, reps=10):
    mr, _ = synth.config_streams(5)
    M = synth.random_symplectic(mr)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn((batch, n, n), dtype=torch.complex64, device="cuda", generator=g)
    out = torch.empty_like(x)
    with nslct.Plan(n, M, batch, profile=True, kernels=kernels) as p:
        for _ in range(3):
            p.exec(x, out)
        torch.cuda.synchronize()
        p.pass_ms()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            p.exec(x, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        pms = p.pass_ms()
    return {"n": n, "batch": batch, "kernels": kernels, "ms": round(ms, 4),
            "transforms_per_s": round(batch / (ms * 1e-3), 2), "pass_ms": [round(t, 4) for t in pms],
            "hbm_frac_per_pass": [round(batch * 2 * n * n * 8 / (t * 1e-3) / 6532.2e9, 3) for t in pms]}, out


n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ref = None
for k in ("auto", "generic"):
    r, out = run(n, batch, k)
    if ref is None:
        ref = out.clone()
    else:
        r["rel_diff_vs_auto"] = float(torch.linalg.vector_norm((out - ref).to(torch.complex128)) /
                                      torch.linalg.vector_norm(ref.to(torch.complex128)))
    print(json.dumps(r), flush=True)
