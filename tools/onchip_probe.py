"""Run one on-chip plan (n, dtype) on cuda:0 and compare with the line-pass schedule."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1707_03688_b200 import nslct  # noqa: E402

n, dtype = int(sys.argv[1]), sys.argv[2]
mr, ir = synth.config_streams(2)
M = synth.random_symplectic(mr)
x = torch.from_numpy(synth.iid_cn(ir, (3, n, n)).astype(np.complex64 if dtype == "c64" else np.complex128)).cuda()
with nslct.Plan(n, M, 3, dtype=dtype) as p, nslct.Plan(n, M, 3, dtype=dtype, schedule="line_passes") as q:
    print("on_chip", p.info()["on_chip"])
    a = p.exec(x)
    b = q.exec(x)
    torch.cuda.synchronize()
    print("rel diff", float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)))
