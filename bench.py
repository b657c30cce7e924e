"""Benchmark of the B200 NsDLCT (BASELINE.json metric: 2D NsLCT transforms/s and achieved
HBM GB/s as a fraction of the roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (default, config C4 of BASELINE.json): 4096 x 4096 complex64 HA-NsDLCT, batch 32
images PER GPU (weak scaling: images are independent, no collective on the data path),
random symplectic ABCD G(rng) of SURVEY.md §8(d), i.i.d. CN(0,1) input.  One step = one
nslct_exec of the batch (all 5 fused passes).  Inputs are 4 GiB per GPU, far larger than
the 126 MB L2, so no L2 flush is needed between steps.

Timing: W untimed warm-up steps, then K steps bracketed by barrier + synchronize, CUDA
events on the exec stream, max over ranks.  The dominant kernel's average launch time
comes from the library's own per-pass CUDA events (nslct_pass_ms) recorded on the same
stream inside the timed region.

--impl reference: the fp64 CPU oracle (oracle/, the only "reference" this paper has) on
the host cores, each step one 4096^2 image of the same workload; rank 0 only.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (n, per-GPU batch, dtype, description)
    1: (32, 1, "c128", "C1: 32x32 complex128, 1 transform/GPU, random symplectic ABCD, iid CN(0,1)"),
    2: (256, 64, "c64", "C2: 256x256 complex64, batch 64/GPU, random symplectic ABCD, iid CN(0,1)"),
    3: (1024, 16, "c64", "C3: 1024x1024 complex64, batch 16/GPU, random symplectic ABCD, iid CN(0,1)"),
    4: (4096, 32, "c64", "C4: 4096x4096 complex64, batch 32/GPU, random symplectic ABCD, iid CN(0,1)"),
    5: (16384, 1, "c64", "C5: 16384x16384 complex64, 1 transform/GPU, random symplectic ABCD, iid CN(0,1)"),
}
METRIC = "2D NsLCT transforms/s (HBM roofline fraction reported in 'roofline')"
UNIT = "transforms/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x, world, device=None):
    """Max of a float over all ranks (torch.distributed all_reduce MAX)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world, device=None):
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = max(smax, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def traffic_from_profiles(cfg_id):
    """ncu --set full DRAM bytes per launch of the dominant kernel, if a capture summary
    for this workload is committed under profiles/ (see profiles/README.md)."""
    p = os.path.join(ROOT, "profiles", "traffic_c%d.json" % cfg_id)
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["dram_bytes_per_launch"]), d.get("kernel")
    except Exception:
        return None, None


def cpu_oracle_sample(x_img, M):
    """Time the fp64 oracle (as it stands) on one image of the workload."""
    import numpy as np
    from oracle import operators
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    g = np.asarray(x_img, np.complex128)
    t0 = time.perf_counter()
    operators.nsdlct(g, M)
    dt = time.perf_counter() - t0
    return dt, cores


def cpu_fft_sample(x_img, M):
    """Time the plain CPU FFT-based decomposition (baselines/cpu_fft.py, fp64, scipy.fft on
    every host core) on one image of the workload; the plan comes from the oracle planner."""
    import numpy as np
    from baselines import cpu_fft
    from oracle import planner
    cores = os.cpu_count()
    pl = planner.plan(M)
    g = np.asarray(x_img, np.complex128)
    n = g.shape[-1]
    t0 = time.perf_counter()
    cpu_fft.transform(g, pl["chain"], math.sqrt(2.0 * math.pi / n), workers=cores)
    return time.perf_counter() - t0, cores


def cpu_direct_sample(x_img, M, k=128):
    """Time the direct method (Eq. Intro32, oracle/direct.py, O(N^2) per output pixel) on k
    sampled output pixels of one image; returns the extrapolated seconds per transform
    (x N^2 / k) and the BLAS thread count."""
    import numpy as np
    from oracle import direct
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    g = np.asarray(x_img, np.complex128)
    n = g.shape[-1]
    dx = math.sqrt(2.0 * math.pi / n)
    rs = np.random.default_rng(0)
    idx = rs.integers(0, n, (k, 2))
    pts = (idx - n // 2) * dx
    t0 = time.perf_counter()
    direct.direct(g, M, dx, out_points=pts)
    dt = time.perf_counter() - t0
    return dt * n * n / k, cores


def run_reference(args):
    """Reference arm: the fp64 oracle, as it stands, on the host cores (rank 0 only).

    A full oracle transform of one 4096^2 image takes seconds, so one "step" is ONE
    operator of the oracle's HA chain (a CC = F^-1 CM F, or a CM; Eq. HA28) applied to the
    running image, in order: 4 consecutive steps are one complete transform.  This keeps
    any --steps K --warmup W run within minutes while timing exactly the oracle's code."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import synth
    from oracle import operators, planner
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    n, batch, dtype, desc = CONFIGS[args.config]
    mr, ir = synth.config_streams(args.config)
    M = synth.random_symplectic(mr)
    x = synth.iid_cn(ir, (n, n)).astype(np.complex64).astype(np.complex128)
    dx = math.sqrt(2.0 * math.pi / n)
    plan = planner.plan(M)
    chain = plan["chain"]
    g = x
    times = []
    for i in range(args.warmup + args.steps):
        op = chain[i % len(chain)]
        t0 = time.perf_counter()
        g = operators.apply_chain(g, [op], dx)
        dt = time.perf_counter() - t0
        if (i + 1) % len(chain) == 0:
            g = x
        if i >= args.warmup:
            times.append(dt)
    total = sum(times)
    val = (len(times) / len(chain)) / total        # complete transforms per second
    ms_step = total / len(times) * 1e3
    sample = ("one operator of the %d-operator HA chain (CC or CM) of one %dx%d image per step; "
              "%d steps = one transform" % (len(chain), n, n, len(chain)))
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
           "config": {"workload": desc, "n": n, "per_gpu_batch": batch, "step": sample,
                      "oracle": "fp64 O_plan, dense-DFT products (numpy/OpenBLAS)"},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def run_ours(args):
    import numpy as np
    import torch

    import synth
    from paper_1707_03688_b200 import nslct

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    n, batch, dtype, desc = CONFIGS[args.config]
    if args.batch:   # exploration only: the config's workload at another per-GPU batch
        desc = desc.replace("batch %d/GPU" % batch, "batch %d/GPU" % args.batch)
        batch = args.batch
    mr, _ = synth.config_streams(args.config)
    M = synth.random_symplectic(mr)                 # same matrix on every rank
    if args.variant == "LC":   # the first G(rng) draw whose LC plan has a y-axis H (3 passes)
        while nslct.nslct_plan_describe(n, M, variant="LC")["lc_axis"] != "y":
            M = synth.random_symplectic(mr)
    if args.config == 5 and world > 1:
        return run_slab(args, n, M, dtype, desc, world, rank, local, dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(synth.SEED_BASE + 1000 * args.config + rank)
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    x = torch.randn((batch, n, n), dtype=tdt, device=dev, generator=gen)   # CN(0,1)
    out = torch.empty_like(x)
    plan = nslct.Plan(n, M, batch, dtype=dtype, profile=True, device=local, schedule=args.schedule,
                      variant=args.variant)
    info = plan.info()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # inputs + outputs smaller than 2x the 126 MB L2 (C2): flush L2 before every timed step
    # (a 512 MiB memset outside the per-step events); larger workloads stream through HBM.
    S = 8 if dtype == "c64" else 16
    flush = None
    if 2 * batch * n * n * S < 256 * 2 ** 20:
        flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        plan.exec(x, out, stream)
    torch.cuda.synchronize()
    plan.pass_ms()                                  # reset the per-pass averages
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            plan.exec(x, out, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_local = e0.elapsed_time(e1) / args.steps
    else:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            plan.exec(x, out, stream)
            b.record(stream)
        torch.cuda.synchronize()
        ms_local = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    barrier()
    clk = clocks.stop()
    pass_ms = plan.pass_ms()
    ms = max_over_ranks(ms_local, world, dev)
    total_units = sum_over_ranks(batch, world, dev)
    value = total_units / (ms * 1e-3)

    # dominant kernel roofline: algorithmic bytes per launch = batch * 2 * N^2 * S
    ki = max(range(len(pass_ms)), key=lambda k: pass_ms[k])
    bytes_launch = batch * 2.0 * n * n * S
    peak, peak_src = peaks()
    achieved = bytes_launch / (pass_ms[ki] * 1e-3) / 1e9
    traffic, tr_kernel = traffic_from_profiles(args.config)
    step_alg_bytes = info["n_launches"] * bytes_launch
    if info["on_chip"]:
        names = ["on-chip: all %d passes, image in shared memory" % info["n_passes"]]
    elif info["n_passes"] == 5:
        names = ["K1 CM+FFT_y (transposed store)", "K2 FFT_x CM IFFT_x", "K3 IFFT_y CM FFT_y",
                 "K4 FFT_x CM IFFT_x", "K5 IFFT_y CM"]
    elif info["n_passes"] == 3:
        names = ["P1 (y lines)", "P2 FFT_x CM IFFT_x", "P3 (y lines)"]
    else:
        names = ["B0 gather"]

    # end-to-end through the public C API with host buffers (H2D + exec + D2H per step)
    e2e = None
    if not args.no_e2e:
        hin = torch.empty((batch, n, n), dtype=tdt).pin_memory()
        hin.copy_(x.cpu())
        hout = torch.empty_like(hin).pin_memory()
        plan.exec_host(hin, hout, stream)        # exec_host records no per-pass events
        nst = max(1, min(args.steps, args.e2e_steps))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(nst):
            plan.exec_host(hin, hout, stream)      # synchronises the stream each call
        t_e2e = (time.perf_counter() - t0) / nst
        barrier()
        t_e2e = max_over_ranks(t_e2e, world, dev)
        # the PCIe ceiling of this e2e number: plain pinned copies of the same bytes, each
        # direction alone (exec_host overlaps H2D, passes and D2H chunk by chunk)
        dbuf = torch.empty((batch, n, n), dtype=tdt, device=dev)
        t_dir = []
        for direction in ("h2d", "d2h"):
            ts = []
            for _ in range(2):
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                if direction == "h2d":
                    dbuf.copy_(hin, non_blocking=True)
                else:
                    hout.copy_(dbuf, non_blocking=True)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t1)
            t_dir.append(min(ts))
        # both directions at once on two streams (what the pipelined call needs)
        dbuf2 = torch.empty_like(dbuf)
        s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            with torch.cuda.stream(s1):
                dbuf.copy_(hin, non_blocking=True)
            with torch.cuda.stream(s2):
                hout.copy_(dbuf2, non_blocking=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t1)
        t_bidir = min(ts)
        del dbuf, dbuf2
        e2e = {"value": total_units / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(hin.numel() * S),
               "d2h_bytes_per_step": int(hout.numel() * S), "steps": nst,
               "h2d_gbs": hin.numel() * S / t_dir[0] / 1e9, "d2h_gbs": hout.numel() * S / t_dir[1] / 1e9,
               "bidir_gbs": (hin.numel() + hout.numel()) * S / t_bidir / 1e9,
               "pcie_bound_value": total_units / max(max(t_dir), t_bidir),
               "how": "nslct_exec_host: pinned host in -> device, %d launches, device -> pinned host out, "
                      "pipelined in ~64 MiB image chunks over two copy streams; wall clock per call "
                      "(each call returns with the result on the host)" % info["n_launches"]}

    cpu = None
    cpu_fft_line = None
    cpu_direct_line = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        img0 = x[0].cpu().numpy()
        dt, cores = cpu_oracle_sample(img0, M)
        cpu = {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": "1 of the %d %dx%d images of one step (image 0), fp64 dense-DFT O_plan" % (batch, n, n)}
        dtf, coresf = cpu_fft_sample(img0, M)
        cpu_fft_line = {"value": 1.0 / dtf, "unit": UNIT, "cores": coresf, "kind": "cpu_fft_decomposition",
                        "sample": "image 0 of the step, fp64, scipy.fft (workers=%d): baselines/cpu_fft.py" % coresf}
        dtd, coresd = cpu_direct_sample(img0, M)
        cpu_direct_line = {"value": 1.0 / dtd, "unit": UNIT, "cores": coresd, "kind": "oracle_direct_eq_intro32",
                           "sample": "128 sampled output pixels of image 0 (O(N^2) each), extrapolated x N^2/128"}

    plan.close()
    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": desc + ("" if args.variant == "HA" else ", LC-NsDLCT variant"), "n": n,
                       "variant": info["variant"], "per_gpu_batch": batch, "global_batch": int(total_units),
                       "plan_kind": info["kind"], "parallelism": "dp%d (independent images, no collective)" % world,
                       "l2": ("L2 flushed before every step (512 MiB memset outside the step events)" if flush is not None
                              else "each pass reads and writes %.2f GiB/GPU (>= 2x the 126 MB L2); no flush"
                              % (2 * batch * n * n * S / 2 ** 30)),
                       "schedule": "on-chip (1 launch)" if info["on_chip"] else "%d line passes" % info["n_passes"], "hbm_alg_bytes_per_step": step_alg_bytes},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": names[ki],
                         "alg_bytes_per_launch": bytes_launch, "launch_ms": pass_ms[ki],
                         "peak_source": peak_src, "traffic_kernel": tr_kernel,
                         "step_frac_of_peak": step_alg_bytes / (ms * 1e-3) / 1e9 / peak,
                         "step_frac_of_8TBs": step_alg_bytes / (ms * 1e-3) / 1e9 / 8000.0,
                         "pass_ms": pass_ms},
            "cpu_baseline": cpu,
            "cpu_fft_baseline": cpu_fft_line,
            "cpu_direct_baseline": cpu_direct_line,
            "e2e": e2e,
            "gpu_launches": info["n_launches"] * args.steps,
            "clocks": clk,
        }
        print(json.dumps(res))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_slab(args, n, M, dtype, desc, world, rank, local, dev):
    """C5: ONE n x n transform as row slabs over `world` GPUs, NCCL all-to-all between the
    5 passes (nslct_plan_slab / nslct_exec_pass).  Strong scaling."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_1707_03688_b200 import nslct
    L = n // world
    gen = torch.Generator(device=dev)
    gen.manual_seed(synth.SEED_BASE + 5000 + rank)
    x = torch.randn((L, n), dtype=torch.complex64, device=dev, generator=gen)
    out = torch.empty_like(x)
    plan = nslct.SlabPlan(n, M, world, rank, device=local)
    stream = torch.cuda.current_stream(dev)
    if args.exchange == "peer":
        # the all-to-all fused into the transposing passes' stores (nslct_exec_pass_peer)
        # into torch symmetric-memory receive buffers over NVLink
        recv, ptrs, sbar = nslct.symm_mem_exchange(L, n)

        def step():
            plan.run_peer(x, recv, ptrs, sbar, out, stream)
    else:
        exchange = nslct.torch_all_to_all()

        def step():
            plan.run(x, exchange, out, stream)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    passes = plan.n_passes
    plan.close()
    hbm_bytes_gpu = passes * 2.0 * n * L * 8
    a2a_bytes_gpu = (passes - 1) * (world - 1) / world * n * L * 8     # per GPU per direction
    nvlink_gbs = 900.0
    if rank == 0:
        res = {
            "metric": METRIC, "value": 1.0 / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": desc + ", row slabs of %d x %d per GPU" % (L, n), "n": n, "global_batch": 1,
                       "parallelism": "row-slab x%d, %s" % (world, "all-to-all fused into the pass stores "
                                                            "(NVLink peer memory)" if args.exchange == "peer"
                                                            else "NCCL all-to-all between passes")},
            "roofline": {"bound": "nvlink", "achieved": a2a_bytes_gpu / (ms * 1e-3) / 1e9, "peak": nvlink_gbs,
                         "unit": "GB/s", "frac": a2a_bytes_gpu / (ms * 1e-3) / 1e9 / nvlink_gbs, "traffic": None,
                         "hbm_alg_bytes_per_gpu": hbm_bytes_gpu, "alltoall_bytes_per_gpu_per_dir": a2a_bytes_gpu,
                         "nvlink_bound_ms": a2a_bytes_gpu / nvlink_gbs / 1e6},
            "cpu_baseline": None, "e2e": None, "gpu_launches": passes * args.steps, "clocks": clk,
        }
        print(json.dumps(res))
    dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", choices=("nccl", "peer"), default="nccl",
                    help="config 5 under torchrun: NCCL all-to-all between passes, or the exchange "
                         "fused into the transposing passes' stores to peer memory")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--schedule", default="auto", choices=["auto", "line_passes", "on_chip"],
                    help="on-chip kernel where available (auto) or one launch per pass")
    ap.add_argument("--variant", default="HA", choices=["HA", "LC"], help="planner variant")
    ap.add_argument("--batch", type=int, default=0,
                    help="override the config's per-GPU batch (exploration; the default run uses the config's)")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
