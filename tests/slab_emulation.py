"""Single-GPU emulation of the row-slab (multi-GPU) mode, for the parity tests only.

nranks slab plans (nslct_plan_slab) run one after another on ONE GPU, each pass through
nslct_exec_pass / nslct_exec_pass_peer, and the exchange between passes is done here by
block copies on the device (or, for the peer-store form, by the passes' own stores into
the other "ranks'" receive buffers).  No kernel waits on another.  The product path for
real multi-GPU runs is nslct.Plan(..., comm=...), where the library itself runs the passes
and the exchanges (include/nslct.h nslct_exec)."""
import torch

from paper_1707_03688_b200 import nslct


def emulate_slabs(n, M, x_full, nranks, dtype="c64", **kw):
    """x_full: CUDA tensor [n, n].  The all-to-all moves block s of rank r's pass output
    ([n][L] = nranks row-blocks of L x L) to block r of rank s's next input.  Returns the
    assembled [n, n] output."""
    L = n // nranks
    plans = [nslct.SlabPlan(n, M, nranks, r, dtype=dtype, **kw) for r in range(nranks)]
    cur = [x_full[r * L:(r + 1) * L].contiguous() for r in range(nranks)]
    outs = [torch.empty_like(c) for c in cur]
    np_ = plans[0].n_passes
    for k in range(np_):
        last = (k == np_ - 1)
        for r in range(nranks):
            plans[r].exec_pass(k, cur[r], outs[r])
        if last:
            break
        nxt = [torch.empty_like(c) for c in cur]
        for r in range(nranks):
            src = outs[r].view(nranks, L * L)
            for s_ in range(nranks):
                nxt[s_].view(nranks, L * L)[r].copy_(src[s_])
        cur = nxt
        outs = [torch.empty_like(c) for c in cur]
    for p in plans:
        p.close()
    return torch.cat(outs, dim=0)


def emulate_slabs_peer(n, M, x_full, nranks, dtype="c64", **kw):
    """The fused peer-store exchange: each transposing pass stores its row-blocks straight
    into the other "ranks'" receive buffers (all on this GPU), double-buffered across
    passes.  Returns the assembled [n, n] output."""
    L = n // nranks
    plans = [nslct.SlabPlan(n, M, nranks, r, dtype=dtype, **kw) for r in range(nranks)]
    cur = [x_full[r * L:(r + 1) * L].contiguous() for r in range(nranks)]
    recv = [[torch.empty_like(cur[0]) for _ in range(nranks)] for _ in range(2)]
    np_ = plans[0].n_passes
    for k in range(np_ - 1):
        ptrs = [t.data_ptr() for t in recv[k % 2]]
        for r in range(nranks):
            plans[r].exec_pass_peer(k, cur[r], ptrs)
        cur = recv[k % 2]
    outs = [torch.empty_like(c) for c in cur]
    for r in range(nranks):
        plans[r].exec_pass(np_ - 1, cur[r], outs[r])
    for p in plans:
        p.close()
    return torch.cat(outs, dim=0)
