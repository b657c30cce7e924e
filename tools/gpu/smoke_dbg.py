import sys; sys.path.insert(0, '.')
import numpy as np, torch, synth
from oracle import metrics, operators, planner
from paper_1707_03688_b200 import nslct
mr, ir = synth.config_streams(1)
M = synth.random_symplectic(mr)
for n in (64, 256, 1024, 4096):
    x = synth.iid_cn(ir, (2, n, n)).astype(np.complex64)
    pl = planner.plan(M)
    with nslct.Plan(n, M, 2, h_fixed=pl["h"]) as p:
        G = p.exec(torch.from_numpy(x).cuda()).cpu().numpy()
        info = p.info()
    errs = []
    for i in range(2 if n <= 1024 else 1):
        ref, _ = operators.nsdlct(x[i].astype(np.complex128), M, pl=pl)
        errs.append(metrics.rel_l2(G[i], ref))
    print(n, info["on_chip"], ["%.6e" % e for e in errs], flush=True)
