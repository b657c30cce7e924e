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
        dist.all_to_all_single(recv.view(-1), send.view(-1))
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


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` (no torchrun environment) starts 2 ranks itself
    (torch.distributed.run, 127.0.0.1) and reports n_gpus = 2 with the global batch of 32
    sharded 16 per rank (BASELINE configs[3]); --dry-run swaps the GPU step for a CPU
    stand-in and NCCL for gloo, keeping the spawn / max-over-ranks / sum-over-ranks path."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks_reporting"] == 2
    assert d["config"]["global_batch"] == 32 and d["config"]["per_gpu_batch"] == 16
    assert d["scaling"] == "strong" and d["value"] > 0
    # the C5 slab sub-record runs in child processes of the ranks (their own rendezvous, a
    # timeout; a failure there cannot cost the main line): here the dry-run child, 2 ranks
    c5 = d["sub"]["C5_slab"]
    assert "error" not in c5, c5
    assert c5["n_gpus"] == 2
