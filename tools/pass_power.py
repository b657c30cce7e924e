"""Power and SM clock of each pass kind of the C4 step run alone (nslct_exec_pass on the
batched plan, the same launch many times back to back) and of the whole step, sampled with
nvidia-smi every 100 ms.  Usage: python tools/pass_power.py [seconds per case]"""
import ctypes
import json
import os
import subprocess
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1707_03688_b200 import nslct  # noqa: E402

SECS = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
n, batch = 4096, 32
mr, _ = synth.config_streams(4)
M = synth.random_symplectic(mr)
g = torch.Generator(device="cuda")
g.manual_seed(4)
x = torch.randn((batch, n, n), dtype=torch.complex64, device="cuda", generator=g)
bufs = [torch.empty_like(x), torch.empty_like(x)]
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def sample(fn, reps_hint):
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=f, stderr=subprocess.DEVNULL)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    n_done = 0
    e0.record()
    while time.time() - t0 < SECS:
        for _ in range(reps_hint):
            fn()
        n_done += reps_hint
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_done
    p.terminate()
    p.wait()
    f.seek(0)
    rows = [r.split(",") for r in f.read().strip().splitlines()]
    os.unlink(f.name)
    # the second half of the samples: the power controller has settled
    rows = rows[len(rows) // 2:]
    clk = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    return {"ms": round(ms, 4), "sm_mhz_median": clk[len(clk) // 2], "power_w_median": pw[len(pw) // 2],
            "power_w_max": pw[-1], "samples": len(rows)}


with nslct.Plan(n, M, batch) as p:
    npass = p.info()["n_passes"]
    # intermediate buffers of each pass as nslct_exec chains them
    cur = x
    srcs = []
    for k in range(npass):
        dst = bufs[k % 2]
        nslct.lib().nslct_exec_pass(p._h, k, ctypes.c_void_p(cur.data_ptr()), ctypes.c_void_p(dst.data_ptr()), stream)
        srcs.append((cur, dst))
        cur = dst
    torch.cuda.synchronize()
    out = torch.empty_like(x)
    res = {"step": sample(lambda: p.exec(x, out), 10)}
    for k in range(npass):
        s, d = srcs[k]
        res["K%d" % (k + 1)] = sample(lambda: nslct.lib().nslct_exec_pass(
            p._h, k, ctypes.c_void_p(s.data_ptr()), ctypes.c_void_p(d.data_ptr()), stream), 40)
    # a plain device copy of the same bytes for comparison
    res["copy"] = sample(lambda: bufs[0].copy_(x), 40)
for k, v in res.items():
    v["joule_per_launch"] = round(v["power_w_median"] * v["ms"] * 1e-3, 3)
    print(k, json.dumps(v), flush=True)
