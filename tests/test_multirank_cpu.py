"""World-size-2 gloo test (CPU) of the multi-rank host logic of bench.py: the timing is
the MAX over ranks and the work is the SUM over ranks (weak scaling, no collective on the
data path).  Rendezvous on 127.0.0.1."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, r, lr = bench.dist_env()
        t = bench.max_over_ranks(1.5 + rank, w)           # rank-dependent step time
        units = bench.sum_over_ranks(32, w)                # per-rank batch of 32 images
        q.put((rank, w, r, t, units))
    finally:
        dist.destroy_process_group()


def test_bench_rank_aggregation_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for rank, w, r, t, units in res:
        assert w == 2 and r == rank
        assert t == 2.5            # max over ranks of (1.5, 2.5)
        assert units == 64.0       # weak scaling: 2 x 32 images per step


def test_bench_single_rank_defaults(monkeypatch):
    import bench
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    assert bench.dist_env() == (1, 0, 0)
    assert bench.max_over_ranks(3.0, 1) == 3.0
    assert bench.sum_over_ranks(32, 1) == 32.0


def _slab_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1707_03688_b200.nslct import torch_all_to_all
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, L = 8, 8 // world
        # a pass output on rank r: [n][L] with element (e, l_local) = code of
        # (global element e, global line r*L + l_local)
        e = torch.arange(n).view(n, 1)
        l = torch.arange(L).view(1, L) + rank * L
        send = (1000 * e + l).to(torch.complex64)
        recv = torch.empty_like(send)
        torch_all_to_all()(send, recv)
        q.put((rank, recv.real.to(torch.int64).tolist()))
    finally:
        dist.destroy_process_group()


def test_slab_all_to_all_layout_gloo():
    """The slab protocol (include/nslct.h, nslct_plan_slab): after the all-to-all, rank s
    holds block r of every rank r at offset r*L*L, i.e. its next-pass line q_local (global
    s*L + q_local) with element m at (m / L)*L*L + q_local*L + m % L."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, L = 8, 4
    for _ in range(world):
        s, recv = q.get(timeout=10)
        flat = [v for row in recv for v in row]
        for ql in range(L):
            for m in range(n):
                # the value at that position is the pass output (element = s*L+ql, line = m)
                assert flat[(m // L) * L * L + ql * L + m % L] == 1000 * (s * L + ql) + m


class _FakeSlab:
    """Host-side stand-in for nslct.SlabPlan (no GPU): pass k maps this rank's [L][n] lines
    x to y = x * (k + 2) + rank code, then "stores" y transposed ([n][L], row-block s for
    rank s) -- into the all-to-all send buffer (exec_pass) or straight into every rank's
    receive buffer at block offset rank*L*L (exec_pass_peer, given the shared tensors)."""

    def __init__(self, n, nranks, rank, n_passes=3):
        self.n, self.nranks, self.rank, self.n_passes = n, nranks, rank, n_passes
        self.L = n // nranks

    def _pass(self, k, x):
        # the chunked input layout the next pass reads is "transposed back" here
        return (x * (k + 2) + (self.rank + 1) * 1000).T.contiguous()   # [n][L]

    def exec_pass(self, k, x, out, stream=None):
        y = self._pass(k, x.view(self.L, self.n) if k == 0 else self._unchunk(x))
        if k == self.n_passes - 1:
            out.copy_(y.T)
        else:
            out.view(-1).copy_(y.reshape(-1))
        return out

    def exec_pass_peer(self, k, x, peers, stream=None):
        y = self._pass(k, x.view(self.L, self.n) if k == 0 else self._unchunk(x))
        L = self.L
        for s in range(self.nranks):
            peers[s].view(-1)[self.rank * L * L:(self.rank + 1) * L * L].copy_(y[s * L:(s + 1) * L].reshape(-1))

    def _unchunk(self, x):
        # received layout: block r at offset r*L*L holds [L (my lines)][L (r's elements)]
        L = self.L
        blocks = x.view(-1).view(self.nranks, L, L)
        return torch.cat([blocks[r] for r in range(self.nranks)], dim=1)   # [L][n]


import torch  # noqa: E402


def _peer_worker(rank, world, port, shared, q):
    import torch.distributed as dist

    from paper_1707_03688_b200 import nslct
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 8
        fake = _FakeSlab(n, world, rank)
        L = fake.L
        x = (torch.arange(L * n, dtype=torch.float32).view(L, n) + 100 * rank).to(torch.complex64)
        # reference: the all-to-all path (the loop of SlabPlan.run, whose CUDA-tensor
        # checks a host test cannot pass)
        exchange = nslct.torch_all_to_all()
        send, rcv, cur = torch.empty_like(x), torch.empty_like(x), x
        for k in range(fake.n_passes - 1):
            fake.exec_pass(k, cur, send)
            exchange(send, rcv)
            cur = rcv.clone()
        ref = fake.exec_pass(fake.n_passes - 1, cur, torch.empty_like(x))
        recv = [shared[0][rank], shared[1][rank]]
        peers = [[shared[b][s] for s in range(world)] for b in range(2)]
        got = nslct.SlabPlan.run_peer(fake, x, recv, peers, dist.barrier)
        q.put((rank, bool(torch.equal(got, ref))))
    finally:
        dist.destroy_process_group()


def test_slab_fused_exchange_protocol_gloo():
    """SlabPlan.run_peer's protocol (double-buffered receive buffers, one cross-rank
    barrier per transposing pass) with world size 2 over gloo and shared host tensors as
    the "peer memory": identical to the all-to-all path (SlabPlan.run) for the same passes."""
    world, n = 2, 8
    L = n // world
    shared = torch.zeros((2, world, L, n), dtype=torch.complex64).share_memory_()
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, shared, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(world))
    assert res == {0: True, 1: True}
