"""On-chip (F2) vs line-pass schedule over N, dtype and batch (L2-resident and HBM-sized).

Times each schedule with CUDA events around nslct_exec after an L2 flush (512 MiB memset),
median of 7, and prints one JSON line per case (used to pick NSLCT_SCHEDULE_AUTO's rule).
"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1707_03688_b200 import nslct  # noqa: E402

flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device="cuda")
mr, _ = synth.config_streams(2)
M = synth.random_symplectic(mr)


def timeit(p, x, out, reps=7):
    ts = []
    for _ in range(2):
        p.exec(x, out)
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p.exec(x, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


cases = []
for dtype, ns in (("c64", (32, 64, 128, 256)), ("c128", (32, 64, 128))):
    S = 8 if dtype == "c64" else 16
    for n in ns:
        for total_mb in (1, 16, 1024):
            batch = max(1, (total_mb * 2 ** 20) // (n * n * S))
            cases.append((dtype, n, batch))
cases.append(("c128", 32, 1))   # C1
for dtype, n, batch in cases:
    S = 8 if dtype == "c64" else 16
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    x = torch.randn((batch, n, n), dtype=tdt, device="cuda")
    out = torch.empty_like(x)
    r = {"dtype": dtype, "n": n, "batch": batch, "MB": batch * n * n * S / 2 ** 20}
    for sch in ("auto", "line_passes"):
        with nslct.Plan(n, M, batch, dtype=dtype, schedule=sch) as p:
            ms = timeit(p, x, out)
            r[sch + "_ms"] = ms
            r[sch + "_per_s"] = batch / (ms * 1e-3)
            r[sch + "_onchip"] = p.info()["on_chip"]
    r["speedup_onchip"] = r["line_passes_ms"] / r["auto_ms"]
    print(json.dumps(r), flush=True)
    del x, out
