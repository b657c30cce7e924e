"""Debug: N = 16384 auto (pair2) vs generic kernels, repeated execs, profile on/off."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth
from paper_1707_03688_b200 import nslct
n = 16384
mr, _ = synth.config_streams(5)
M = synth.random_symplectic(mr)
g = torch.Generator(device="cuda"); g.manual_seed(5)
x = torch.randn((1, n, n), dtype=torch.complex64, device="cuda", generator=g)
def rd(a, b):
    return float(torch.linalg.vector_norm((a - b).to(torch.complex128)) / torch.linalg.vector_norm(b.to(torch.complex128)))
with nslct.Plan(n, M, 1, kernels="generic") as p:
    ref = p.exec(x)
torch.cuda.synchronize()
for prof in (False, True):
    with nslct.Plan(n, M, 1, profile=prof) as p:
        out = torch.empty_like(x)
        res = []
        for i in range(5):
            p.exec(x, out)
            torch.cuda.synchronize()
            res.append(rd(out, ref))
        o2 = p.exec(x)
        torch.cuda.synchronize()
        res.append(rd(o2, ref))
        print(json.dumps({"profile": prof, "rel_diffs": res, "info_kind": p.info()["kind"]}), flush=True)
