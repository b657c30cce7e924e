"""Per-rank pass times of the row-slab mode, measured on ONE GPU by running every rank's
passes one after another (the all-to-all replaced by device block copies, as in
tests/slab_emulation.py).  Prints one JSON line: per-pass ms summed over ranks (= one GPU doing
all ranks' HBM work) and divided by P (the per-GPU HBM time of a P-GPU run, without the
exchange).  Usage: python tools/slab_pass_timing.py [n] [P] [reps] [exchange_chunks]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1707_03688_b200 import nslct  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    chunks = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    L = n // P
    mr, _ = synth.config_streams(5)
    M = synth.random_symplectic(mr)
    plans = [nslct.SlabPlan(n, M, P, r, exchange_chunks=chunks) for r in range(P)]
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = [torch.randn((L, n), dtype=torch.complex64, device="cuda", generator=g) for _ in range(P)]
    out = [torch.empty_like(t) for t in x]
    npass = plans[0].n_passes
    tot = [0.0] * npass
    for rep in range(reps + 1):
        cur = x
        for k in range(npass):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for r in range(P):
                plans[r].exec_pass(k, cur[r], out[r])
            e1.record()
            torch.cuda.synchronize()
            if rep > 0:
                tot[k] += e0.elapsed_time(e1) / reps
            cur = out   # layout-only stand-in for the exchange: the timing is what matters
            out = [torch.empty_like(t) for t in x]
    hbm = 2.0 * n * n * 8
    res = {"n": n, "P": P, "exchange_chunks": chunks, "pair_kernels": True,
           "pass_ms_all_ranks": [round(t, 3) for t in tot],
           "per_gpu_ms": round(sum(tot) / P, 3),
           "hbm_TBps_per_pass": [round(hbm / (t * 1e-3) / 1e12, 2) for t in tot]}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
