"""Benchmark of the B200 NsDLCT (BASELINE.json metric: 2D NsLCT transforms/s and achieved
HBM GB/s as a fraction of the roofline, at 1/2/4/8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]

--gpus N > 1 without a torchrun environment re-launches this script under
torch.distributed.run (one process per GPU, NCCL, rendezvous on 127.0.0.1) and checks that
the world size is N.

Headline workload (default, BASELINE.json configs[3] = C4): 4096 x 4096 complex64
HA-NsDLCT, GLOBAL batch 32 sharded 32/N images per GPU (strong scaling: images are
independent, no collective on the data path), random symplectic ABCD G(rng) of SURVEY.md
§8(d), i.i.d. CN(0,1) input.  One step = one nslct_exec of the rank's images (all 5
fused passes).  Each pass reads and writes >= 1 GiB per GPU (far more than the 126 MB
L2), so no L2 flush is needed; the small configs flush L2 before every step.

Sub-records in the same JSON line (N = 1): C1 latency, C2 (L2-flushed, % of B_min and of
B_alg), the C3 special-case sweep (DFT / gyrator / separable / B = 0, with the B = 0
gather's roofline) and C5 on one GPU; at N > 1 the C5 row-slab transform over all N GPUs
through the library's comm plans (NCCL chunked exchange and fused peer stores) against a
measured bare all-to-all of the same blocks.

Timing: W untimed warm-up steps, then K steps bracketed by barrier + synchronize, CUDA
events on the exec stream, max over ranks.  The dominant kernel's launch time comes from
the library's own per-pass CUDA events (nslct_pass_ms) recorded on the same stream inside
the timed region.

--impl reference: the fp64 CPU oracle (oracle/, the only "reference" this paper has) on
the host cores, each step one operator of the oracle chain on one image of the workload;
rank 0 only.
--dry-run: the multi-process plumbing (spawn, gloo process group, max/sum over ranks, the
JSON line) with a CPU stand-in step -- no GPU; used by tests/test_multirank_cpu.py.
"""
import argparse
import json
import math
import os
import platform
import socket
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (n, GLOBAL batch, dtype, description) -- BASELINE.json configs[id - 1]
    1: (32, 1, "c128", "C1: 32x32 complex128, single transform, random symplectic ABCD, iid CN(0,1)"),
    2: (256, 64, "c64", "C2: 256x256 complex64, batch 64, random symplectic ABCD, Gaussian-windowed chirps + 5% noise"),
    3: (1024, 16, "c64", "C3: 1024x1024 complex64, batch 16 per sub-case, special-case sweep "
                         "(DFT, gyrator, separable, B=0), unit-amplitude random-phase images"),
    4: (4096, 32, "c64", "C4: 4096x4096 complex64, global batch 32 sharded 32/N per GPU, random symplectic ABCD, "
                         "iid CN(0,1)"),
    5: (16384, 1, "c64", "C5: 16384x16384 complex64 single transform, random symplectic ABCD, iid CN(0,1)"),
}
METRIC = "2D NsLCT transforms/s (HBM roofline fraction reported in 'roofline')"
UNIT = "transforms/s"
NVLINK_GBS = 900.0   # nominal per direction per GPU (NVLink 5), context only


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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn(argv, n):
    """Re-run this script as n ranks under torch.distributed.run (stdout passes through)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % n,
           "--master-addr=127.0.0.1", "--master-port=%d" % _free_port(), os.path.abspath(__file__)] + list(argv)
    return subprocess.run(cmd).returncode


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
        return self

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
        sm, smax, reasons, pw = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = max(smax, float(r[2]))
                try:
                    pw.append(float(r[3]))
                except Exception:
                    pass
                for nm, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        sm.sort()
        pw.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": pw[len(pw) // 2] if pw else None,
                "power_w_max": pw[-1] if pw else None}


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


# ------------------------------------------------------------------------ CPU baselines
def host_facts():
    """CPU model, core count, BLAS threads and affinity of this process."""
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity_cpus": aff, "blas": blas}


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def _timed(fn, reps=1):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2]


def cpu_baselines(full=False):
    """BASELINE.md §3 on the host cores.  Default: a bounded set (C1 in full, C2 all 64
    images of the FFT baseline and 4 oracle images, one C3 image per sub-case, 2 C4 oracle
    images, C4 O_direct on 4096 sampled pixels, c64 + c128 FFT decomposition on C4 image
    0).  full=True adds the rest of §3 (C2 O_direct in full, all 4 images per C3 sub-case,
    the C3 DFT O_direct in full, the C5 transform for every baseline).  Returns the list of
    records and the headline cpu_baseline (the oracle on C4)."""
    import numpy as np

    import synth
    from baselines import cpu_fft
    from oracle import direct, operators, planner
    recs = []
    cores = blas_threads()

    def add(cfg, kind, dtype, sec_per_transform, sample, extrapolated=False):
        recs.append({"config": cfg, "kind": kind, "dtype": dtype, "value": 1.0 / sec_per_transform,
                     "unit": UNIT, "sec_per_transform": sec_per_transform, "cores": cores,
                     "sample": sample, "extrapolated": extrapolated})

    def imgs(cfg, k):
        n = CONFIGS[cfg][0]
        mr, ir = synth.config_streams(cfg)
        if cfg == 2:
            x = synth.chirp_gauss_field(ir, n, k)
        elif cfg == 3:
            x = synth.random_phase_field(ir, (k, n, n))
        else:
            x = synth.iid_cn(ir, (k, n, n))
        M = synth.random_symplectic(mr) if cfg != 3 else synth.c3_sweep_matrices(mr)
        cast = np.complex128 if CONFIGS[cfg][2] == "c128" else np.complex64
        return M, x.astype(cast).astype(np.complex128)

    def oracle_rec(cfg, M, x, label):
        pl = planner.plan(M)
        t = _timed(lambda: [operators.nsdlct(g, M, pl=pl) for g in x]) / len(x)
        add(cfg, "oracle O_plan (fp64 dense-DFT zgemm)", "c128", t, label)
        return t

    def fft_rec(cfg, M, x, label):
        n = x.shape[-1]
        pl = planner.plan(M)
        for dt, name in ((np.complex64, "c64"), (np.complex128, "c128")):
            if pl["kind"] == "B0":
                continue
            t = _timed(lambda: [cpu_fft.transform(g, pl["chain"], math.sqrt(2 * math.pi / n),
                                                  workers=os.cpu_count(), dtype=dt) for g in x],
                       reps=3 if x.size * 8 < 2 ** 28 else 1) / len(x)
            add(cfg, "cpu_fft_decomposition (scipy.fft workers=%d)" % os.cpu_count(), name, t, label)

    def direct_rec(cfg, M, g, k, label):
        n = g.shape[-1]
        dx = math.sqrt(2.0 * math.pi / n)
        if k is None or k >= n * n:
            t = _timed(lambda: direct.direct(g, M, dx))
            add(cfg, "oracle O_direct (Eq. Intro32)", "c128", t, label + ", all %d outputs" % (n * n))
        else:
            rs = np.random.default_rng(0)
            pts = (rs.integers(0, n, (k, 2)) - n // 2) * dx
            t = _timed(lambda: direct.direct(g, M, dx, out_points=pts)) * n * n / k
            add(cfg, "oracle O_direct (Eq. Intro32)", "c128", t, label + ", %d sampled outputs x N^2/%d" % (k, k),
                extrapolated=True)

    M, x = imgs(1, 1)
    oracle_rec(1, M, x, "C1 in full")
    direct_rec(1, M, x[0], None, "C1")
    M, x = imgs(2, 64)
    oracle_rec(2, M, x if full else x[:4], "C2: %d of 64 images" % (64 if full else 4))
    fft_rec(2, M, x, "C2: all 64 images")
    direct_rec(2, M, x[0], None if full else 4096, "C2 image 0")
    subs, x3 = imgs(3, 4 if full else 1)
    for name in ("dft", "gyrator", "separable", "b0"):
        oracle_rec(3, subs[name], x3, "C3 %s: %d image(s)" % (name, len(x3)))
        fft_rec(3, subs[name], x3[:1], "C3 %s: image 0" % name)
    direct_rec(3, subs["dft"], x3[0], None if full else 4096, "C3 dft image 0")
    M, x = imgs(4, 2)
    t4 = oracle_rec(4, M, x, "C4: 2 of 32 images")
    fft_rec(4, M, x[:1], "C4 image 0")
    direct_rec(4, M, x[0], 4096, "C4 image 0")
    if full:
        M, x = imgs(5, 1)
        oracle_rec(5, M, x, "C5 single transform")
        fft_rec(5, M, x, "C5 single transform")
        direct_rec(5, M, x[0], 4096, "C5")
    head = {"value": 1.0 / t4, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "2 of the 32 C4 4096x4096 images (images 0, 1 of the config-4 stream), fp64 dense-DFT "
                      "O_plan on all host cores (median of 1)"}
    return recs, head


# ------------------------------------------------------------------------ reference arm
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
    cores = blas_threads()
    n, batch, dtype, desc = CONFIGS[args.config]
    mr, ir = synth.config_streams(args.config)
    M = synth.random_symplectic(mr) if args.config != 3 else synth.c3_sweep_matrices(mr)["gyrator"]
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
           "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic",
           "config": {"workload": desc, "n": n, "global_batch": batch, "step": sample,
                      "oracle": "fp64 O_plan, dense-DFT products (numpy/OpenBLAS)"},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "host": host_facts()}
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------ GPU measurement
def time_exec(plan, x, out, stream, steps, warmup, flush=None, barrier=None):
    """Average ms per nslct_exec over `steps` timed calls (CUDA events on `stream`; with
    `flush`, L2 is overwritten before every step outside the per-step events)."""
    import torch
    for _ in range(warmup):
        plan.exec(x, out, stream)
    torch.cuda.synchronize()
    if plan.profile:
        plan.pass_ms()   # reset the per-pass averages
    if barrier:
        barrier()
    torch.cuda.synchronize()
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            plan.exec(x, out, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    else:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            plan.exec(x, out, stream)
            b.record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    if barrier:
        barrier()
    return ms


def pass_names(info):
    if info["on_chip"]:
        return ["on-chip: all %d passes, image in shared memory" % info["n_passes"]]
    if info["kind"] == "B0":
        return ["B0 chirp x bilinear gather"]
    if info["n_passes"] == 5:
        return ["K1 CM+FFT_y (transposed store)", "K2 FFT_x CM IFFT_x", "K3 IFFT_y CM FFT_y",
                "K4 FFT_x CM IFFT_x", "K5 IFFT_y CM"]
    return ["P1 (y lines)", "P2 FFT_x CM IFFT_x", "P3 (y lines)"]


def line_flops(n, mode_ffts):
    """Algorithmic real flops of one line of a pass: mode_ffts line FFTs of 5 N log2 N
    (radix-2 convention) + one chirp complex multiply (6 flops) per element."""
    return mode_ffts * 5.0 * n * math.log2(n) + 6.0 * n


def ffts_of_pass(info, k):
    if info["kind"] == "B0" or info["on_chip"]:
        return 0
    if info["n_passes"] == 5:
        return (1, 2, 2, 2, 1)[k]
    return (3, 2, 1)[k] if info["kind"] == "I" else (1, 2, 3)[k]


def measure_batched(nslct, torch, dev, stream, n, batch, dtype, M, x=None, steps=20, warmup=5, flush_l2=None,
                    barrier=None, seed=0, **plan_kw):
    """One batched plan timed through nslct_exec; returns a dict with ms, pass_ms, info."""
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    if x is None:
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        x = torch.randn((batch, n, n), dtype=tdt, device=dev, generator=gen)   # CN(0,1)
    out = torch.empty_like(x)
    S = 8 if dtype == "c64" else 16
    flush = None
    if flush_l2 is None:
        flush_l2 = 2 * batch * n * n * S < 256 * 2 ** 20
    if flush_l2:
        flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    plan = nslct.Plan(n, M, batch, dtype=dtype, profile=True, device=dev.index, **plan_kw)
    info = plan.info()
    ms = time_exec(plan, x, out, stream, steps, warmup, flush, barrier)
    pms = plan.pass_ms()
    plan.close()
    return {"ms": ms, "pass_ms": pms, "info": info, "flushed": flush is not None, "x": x, "S": S}


def roofline_of(r, n, batch, peak, peak_src, fp32_peak=None):
    """Dominant kernel: achieved = algorithmic bytes per launch (batch * 2 N^2 S) / its
    average launch time; plus the whole step against B_alg (and B_min for small N)."""
    info, pms, S = r["info"], r["pass_ms"], r["S"]
    names = pass_names(info)
    ki = max(range(len(pms)), key=lambda k: pms[k])
    bytes_launch = batch * 2.0 * n * n * S
    achieved = bytes_launch / (pms[ki] * 1e-3) / 1e9
    step_alg = info["n_launches"] * bytes_launch if not info["on_chip"] else info["n_passes"] * bytes_launch
    b_min = bytes_launch
    ro = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
          "kernel": names[ki], "alg_bytes_per_launch": bytes_launch, "launch_ms": pms[ki],
          "peak_source": peak_src, "pass_ms": pms,
          "step_alg_bytes": step_alg,
          "step_frac_of_peak": step_alg / (r["ms"] * 1e-3) / 1e9 / peak,
          "step_frac_of_8TBs": step_alg / (r["ms"] * 1e-3) / 1e9 / 8000.0,
          "step_frac_of_peak_bmin": b_min / (r["ms"] * 1e-3) / 1e9 / peak}
    nf = ffts_of_pass(info, ki)
    if fp32_peak and nf and S == 8:
        fl = batch * n * line_flops(n, nf)
        ach = fl / (pms[ki] * 1e-3) / 1e12
        ro["alu"] = {"bound": "fp32", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak,
                     "flops_per_launch": fl,
                     "count": "%d line FFT(s) x 5 N log2 N + 6 N (chirp) real flops per line, radix-2 convention; "
                              "peak = nslct_fp32_peak (measured FFMA rate)" % nf}
    return ro


def run_ours(args):
    import numpy as np
    import torch

    import synth
    from paper_1707_03688_b200 import nslct

    world, rank, local = dist_env()
    assert world == args.gpus, "world size %d != --gpus %d" % (world, args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    n, gbatch, dtype, desc = CONFIGS[args.config]
    if args.batch:   # exploration only: another global batch of the config's workload
        desc = desc.replace("batch %d" % gbatch, "batch %d" % args.batch)
        gbatch = args.batch
    peak, peak_src = peaks()
    fp32_peak = nslct.fp32_peak_tflops(local)
    stream = torch.cuda.current_stream(dev)
    mr, ir = synth.config_streams(args.config)
    sub = {}

    clocks = ClockSampler(local).start()
    if args.config == 5 and world > 1:
        M = synth.random_symplectic(mr)
        main = run_slab(args, nslct, torch, dev, stream, n, M, world, rank, barrier)
        value, ms, units = main["value"], main["ms"], 1
        ro, e2e, info = main["roofline"], None, None
        launches = main["launches"]
        cfg = {"workload": desc + ", row slabs of %d x %d per GPU" % (n // world, n), "n": n, "global_batch": 1,
               "parallelism": "row-slab x%d: comm plan, %s" % (world, main["exchange"]),
               "ms_by_exchange": main["ms_by_exchange"], "exchange_errors": main.get("errors")}
        scaling = "strong"
    else:
        if gbatch % world:
            raise SystemExit("global batch %d not divisible by %d GPUs" % (gbatch, world))
        batch = gbatch // world
        if args.config == 3:   # the special-case sweep: all four sub-cases, batch each
            subs = synth.c3_sweep_matrices(mr)
            tot_ms, recs = 0.0, {}
            for name in ("dft", "gyrator", "separable", "b0"):
                r = measure_batched(nslct, torch, dev, stream, n, batch, dtype, subs[name], steps=args.steps,
                                    warmup=args.warmup, barrier=barrier, seed=synth.SEED_BASE + 3000 + rank,
                                    schedule=args.schedule)
                tot_ms += r["ms"]
                recs[name] = {"ms": r["ms"], "transforms_per_s": batch / (r["ms"] * 1e-3), "plan_kind": r["info"]["kind"],
                              "roofline": roofline_of(r, n, batch, peak, peak_src, fp32_peak)}
                last = r
            ms_local = tot_ms
            units_local = 4 * batch
            info = last["info"]
            ro = recs["gyrator"]["roofline"]
            ro = dict(ro, sweep=recs)
            sub["C3_sweep"] = recs
        else:
            M = synth.random_symplectic(mr)              # same matrix on every rank
            if args.variant == "LC":   # the first G(rng) draw whose LC plan has a y-axis H (3 passes)
                while nslct.nslct_plan_describe(n, M, variant="LC")["lc_axis"] != "y":
                    M = synth.random_symplectic(mr)
            r = measure_batched(nslct, torch, dev, stream, n, batch, dtype, M, steps=args.steps, warmup=args.warmup,
                                barrier=barrier, seed=synth.SEED_BASE + 1000 * args.config + rank,
                                schedule=args.schedule, variant=args.variant)
            ms_local, units_local, info = r["ms"], batch, r["info"]
            ro = roofline_of(r, n, batch, peak, peak_src, fp32_peak)
            main_x = r["x"]
        ms = max_over_ranks(ms_local, world, dev)
        units = sum_over_ranks(units_local, world, dev)
        value = units / (ms * 1e-3)
        traffic, tr_kernel = traffic_from_profiles(args.config)
        ro["traffic"] = traffic
        ro["traffic_kernel"] = tr_kernel
        launches = info["n_launches"] * args.steps * (4 if args.config == 3 else 1)
        cfg = {"workload": desc + ("" if args.variant == "HA" else ", LC-NsDLCT variant"), "n": n,
               "global_batch": int(units), "per_gpu_batch": batch,
               "plan_kind": info["kind"], "variant": info["variant"],
               "parallelism": "dp%d (global batch sharded %d per GPU, no collective on the data path)" % (world, batch),
               "l2": ("L2 flushed before every step (512 MiB memset outside the step events)"
                      if 2 * batch * n * n * (8 if dtype == "c64" else 16) < 256 * 2 ** 20
                      else "each pass reads and writes %.2f GiB/GPU (>= 2x the 126 MB L2); no flush"
                      % (2 * batch * n * n * 8 / 2 ** 30)),
               "schedule": "on-chip (1 launch)" if info["on_chip"] else "%d line passes" % info["n_passes"]}
        scaling = "strong"
        # end-to-end through the public C API with host buffers (H2D + passes + D2H per step)
        e2e = None
        if not args.no_e2e and args.config != 3:
            e2e = measure_e2e(nslct, torch, dev, stream, n, batch, dtype, M, main_x, args, world, barrier, units)
    clk = clocks.stop()

    # sub-records (one GPU): the other configs of BASELINE.json through the same library
    if not args.no_sub and world == 1 and args.config == 4:
        sub.update(sub_records(nslct, torch, dev, stream, peak, peak_src, fp32_peak, args))
    if not args.no_sub and world > 1 and args.config == 4:
        # C5 as row slabs over the same GPUs, in CHILD processes (one per rank, their own
        # rendezvous): the comm plans have only ever run on one GPU, and a fault or a hang
        # there must not cost the C4 line
        port = int(max_over_ranks(_free_port() if rank == 0 else 0, world, dev))
        sub["C5_slab"] = slab_child(args, world, rank, local, port)

    cpu, cpu_recs = None, None
    if rank == 0 and not args.no_cpu_baseline:
        cpu_recs, cpu = cpu_baselines(full=args.cpu_full)
    barrier()
    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": dtype, "data": "synthetic", "config": cfg,
            "roofline": ro, "cpu_baseline": cpu, "cpu_baselines": cpu_recs, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk, "sub": sub, "host": host_facts(),
            "fp32_peak_tflops": fp32_peak,
        }
        print(json.dumps(res), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def measure_e2e(nslct, torch, dev, stream, n, batch, dtype, M, x, args, world, barrier, units):
    """The same metric through nslct_exec_host: pinned host in -> device -> passes -> pinned
    host out inside the timed region, every step (wall clock per call, max over ranks)."""
    S = 8 if dtype == "c64" else 16
    plan = nslct.Plan(n, M, batch, dtype=dtype, device=dev.index)
    hin = torch.empty(tuple(x.shape), dtype=x.dtype).pin_memory()
    hin.copy_(x.cpu())
    hout = torch.empty_like(hin).pin_memory()
    plan.exec_host(hin, hout, stream)
    nst = max(1, min(args.steps, args.e2e_steps))
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(nst):
        plan.exec_host(hin, hout, stream)      # returns with the result on the host
    t_e2e = (time.perf_counter() - t0) / nst
    barrier()
    plan.close()
    t_e2e = max_over_ranks(t_e2e, world, dev)
    dbuf = torch.empty(tuple(x.shape), dtype=x.dtype, device=dev)
    t_dir = []
    for direction in ("h2d", "d2h"):
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            if direction == "h2d":
                dbuf.copy_(hin, non_blocking=True)
            else:
                hout.copy_(dbuf, non_blocking=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t1)
        t_dir.append(min(ts))
    # both directions at once (what the pipelined call needs: PCIe is full duplex, but the
    # host memory system and the copy engines are shared)
    dbuf2 = torch.empty_like(dbuf)
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ts = []
    for _ in range(4):   # the first repetition warms the two streams' copy engines up
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        with torch.cuda.stream(s_in):
            dbuf.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s_out):
            hout.copy_(dbuf2, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t1)
    t_bidir = min(ts)
    del dbuf, dbuf2
    return {"value": units / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(hin.numel() * S),
            "d2h_bytes_per_step": int(hout.numel() * S), "steps": nst,
            "h2d_gbs": hin.numel() * S / t_dir[0] / 1e9, "d2h_gbs": hout.numel() * S / t_dir[1] / 1e9,
            "pcie_bound_value": units / max(t_dir),
            "pcie_bidir_gbs": 2 * hin.numel() * S / t_bidir / 1e9,
            "pcie_bidir_bound_value": units / t_bidir,
            "frac_of_bidir_bound": t_bidir / t_e2e,
            "how": "nslct_exec_host per rank: pinned host in -> device, passes, device -> pinned host out, "
                   "pipelined in ~64 MiB image chunks over two copy streams; wall clock per call, max over ranks"}


def sub_records(nslct, torch, dev, stream, peak, peak_src, fp32_peak, args):
    """C1, C2, C3 sweep and C5 (one GPU) through the same library, each with its roofline."""
    import numpy as np

    import synth
    out = {}
    steps = max(10, args.steps)
    clocks = ClockSampler(dev.index).start()
    # C1: latency of one 32x32 complex128 transform (on-chip kernel, launch-bound)
    mr, ir = synth.config_streams(1)
    r = measure_batched(nslct, torch, dev, stream, 32, 1, "c128", synth.random_symplectic(mr), steps=200,
                        warmup=20, flush_l2=False)
    out["C1"] = {"transforms_per_s": 1.0 / (r["ms"] * 1e-3), "us_per_transform": r["ms"] * 1e3,
                 "note": "latency-bound (one launch, 16 KiB image); no L2 flush"}
    # C2: 256^2 c64 batch 64 (32 MiB: L2-resident) -- L2 flushed before every step
    mr, ir = synth.config_streams(2)
    M2 = synth.random_symplectic(mr)
    x2 = torch.from_numpy(synth.chirp_gauss_field(ir, 256, 64).astype(np.complex64)).to(dev)
    r = measure_batched(nslct, torch, dev, stream, 256, 64, "c64", M2, x=x2, steps=steps, warmup=5, flush_l2=True)
    ro = roofline_of(r, 256, 64, peak, peak_src, fp32_peak)
    out["C2"] = {"transforms_per_s": 64 / (r["ms"] * 1e-3), "ms": r["ms"], "roofline": ro,
                 "frac_of_peak_vs_B_min": ro["step_frac_of_peak_bmin"],
                 "note": "L2 flushed before each step; B_min = one HBM round trip per image (SURVEY §8(d))"}
    # C3: the special-case sweep, batch 16 each; B = 0 gather roofline 2 N^2 S per transform
    mr, ir = synth.config_streams(3)
    subs = synth.c3_sweep_matrices(mr)
    x3 = torch.from_numpy(synth.random_phase_field(ir, (16, 1024, 1024)).astype(np.complex64)).to(dev)
    tot, recs = 0.0, {}
    for name in ("dft", "gyrator", "separable", "b0"):
        r = measure_batched(nslct, torch, dev, stream, 1024, 16, "c64", subs[name], x=x3, steps=steps, warmup=5,
                            flush_l2=True)
        tot += r["ms"]
        recs[name] = {"ms": r["ms"], "transforms_per_s": 16 / (r["ms"] * 1e-3), "plan_kind": r["info"]["kind"],
                      "roofline": roofline_of(r, 1024, 16, peak, peak_src, fp32_peak)}
    out["C3"] = {"transforms_per_s": 64 / (tot * 1e-3), "sweep": recs,
                 "note": "4 sub-cases x 16 images (128 MiB each, L2 flushed before each step)"}
    # C5 on one GPU: one 16384^2 transform (cluster-pair kernels)
    mr, ir = synth.config_streams(5)
    r = measure_batched(nslct, torch, dev, stream, 16384, 1, "c64", synth.random_symplectic(mr),
                        steps=max(10, args.steps // 2), warmup=3, seed=5)
    out["C5_1gpu"] = {"transforms_per_s": 1.0 / (r["ms"] * 1e-3), "ms": r["ms"],
                      "roofline": roofline_of(r, 16384, 1, peak, peak_src, fp32_peak)}
    out["clocks"] = clocks.stop()
    # C4 sustained: the headline step repeated for ~3 s with its own clock / power samples.
    # Every pass (and a plain copy of the same bytes) runs at the board's power limit when
    # sustained, so the 20-step `value` is a burst figure; this is the
    # steady state.
    mr, ir = synth.config_streams(4)
    ck = ClockSampler(dev.index).start()
    r = measure_batched(nslct, torch, dev, stream, 4096, 32, "c64", synth.random_symplectic(mr),
                        steps=300, warmup=5, seed=synth.SEED_BASE + 4000)
    out["C4_sustained"] = {"transforms_per_s": 32 / (r["ms"] * 1e-3), "ms": r["ms"], "steps": 300,
                           "pass_ms": r["pass_ms"], "clocks": ck.stop()}
    return out


def slab_child(args, world, rank, local, port, timeout=300, extra=()):
    """`bench.py --config 5 --gpus world` as a child of every rank (rank 0's child prints the
    line, returned here as the sub-record); killed after `timeout` seconds.  Never raises."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
               LOCAL_RANK=str(local), WORLD_SIZE=str(world))
    for k in [k for k in env if k.startswith("TORCHELASTIC_")]:
        env.pop(k)   # the child ranks rendezvous among themselves (no agent store)
    cmd = [sys.executable, os.path.abspath(__file__), "--config", "5", "--gpus", str(world),
           "--steps", str(max(5, args.steps // 2)), "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-sub"]
    cmd += list(extra)
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": "timeout after %d s (child killed)" % timeout}
    except Exception as e:   # noqa: BLE001
        return {"error": repr(e)}
    if rank != 0:
        return None
    for line in reversed(r.stdout.strip().splitlines()):
        try:
            d = json.loads(line)
            return {"value": d["value"], "ms": d["ms_per_step"], "n_gpus": d["n_gpus"], "steps": d["steps"],
                    "config": d.get("config"), "roofline": d.get("roofline"), "launches": d.get("gpu_launches")}
        except Exception:   # noqa: BLE001
            continue
    return {"error": "child rc=%d: %s" % (r.returncode, (r.stderr or r.stdout)[-400:])}


def run_slab(args, nslct, torch, dev, stream, n, M, world, rank, barrier, steps=None):
    """C5: ONE n x n transform as row slabs over `world` GPUs through the library's comm
    plans (nslct_exec runs every pass and exchange): NCCL chunked send/recv and the fused
    peer-store exchange, against a measured bare NCCL all-to-all of the same blocks."""
    import torch.distributed as dist
    import synth
    steps = steps or args.steps
    L = n // world
    gen = torch.Generator(device=dev)
    gen.manual_seed(synth.SEED_BASE + 5000 + rank)
    x = torch.randn((L, n), dtype=torch.complex64, device=dev, generator=gen)
    out = torch.empty_like(x)
    comm = nslct.Communicator()
    res, errors, np_ = {}, {}, 5
    for exch in ("nccl", "peer"):
        # a plan-time failure (e.g. no CUDA IPC between the GPUs) is the same on every rank:
        # record it and go on with the other exchange; the flag is agreed over the ranks
        plan, err = None, None
        try:
            plan = nslct.Plan(n, M, 1, comm=comm, exchange=exch, device=dev.index)
        except Exception as e:   # noqa: BLE001
            err = repr(e)
        if max_over_ranks(1.0 if err else 0.0, world, dev) > 0:
            errors[exch] = err or "failed on another rank"
            if plan is not None:
                plan.close()
            continue
        np_ = plan.info()["n_passes"]
        ms_l = time_exec(plan, x, out, stream, steps, 3, None, barrier)
        plan.close()
        res[exch] = max_over_ranks(ms_l, world, dev)
    if not res:
        raise SystemExit("slab mode: no exchange available: %r" % errors)
    # the bare exchange: (n_passes - 1) all-to-alls of the same [L][n] slabs
    send, recv = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        dist.all_to_all_single(recv.view(-1), send.view(-1))
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        for _ in range(np_ - 1):
            dist.all_to_all_single(recv.view(-1), send.view(-1))
    e1.record(stream)
    torch.cuda.synchronize()
    a2a_ms = max_over_ranks(e0.elapsed_time(e1) / steps, world, dev)
    comm.close()
    best = min(res, key=lambda k: res[k])
    ms = res[best]
    a2a_bytes = (np_ - 1) * (world - 1) / world * n * L * 8.0    # per GPU per direction
    hbm_bytes = np_ * 2.0 * n * L * 8
    return {"value": 1.0 / (ms * 1e-3), "ms": ms, "exchange": best, "ms_by_exchange": res, "errors": errors or None,
            "launches": np_ * steps,
            "roofline": {"bound": "nvlink (all-to-all)", "achieved": a2a_bytes / (ms * 1e-3) / 1e9,
                         "peak": a2a_bytes / (a2a_ms * 1e-3) / 1e9, "unit": "GB/s", "frac": a2a_ms / ms,
                         "traffic": None, "peak_source": "measured: bare NCCL all_to_all_single of the same "
                                                         "[L][n] slabs, (n_passes - 1) per transform",
                         "alltoall_ms_measured": a2a_ms, "alltoall_bytes_per_gpu_per_dir": a2a_bytes,
                         "nvlink_nominal_bound_ms": a2a_bytes / NVLINK_GBS / 1e6,
                         "hbm_alg_bytes_per_gpu": hbm_bytes}}


# ------------------------------------------------------------------------ dry run (CPU)
def run_dry(args):
    """The multi-process plumbing without a GPU: gloo process group, a CPU stand-in step
    (the CPU FFT baseline on a small image per local image), max/sum over ranks, the JSON
    line of rank 0.  Checks what the GPU run relies on: world size = --gpus, strong-scaled
    shard sizes, MAX time, SUM units."""
    import numpy as np
    import torch.distributed as dist

    import synth
    from baselines import cpu_fft
    from oracle import planner
    world, rank, _ = dist_env()
    assert world == args.gpus, "world size %d != --gpus %d" % (world, args.gpus)
    if world > 1:
        dist.init_process_group("gloo")
    gbatch = CONFIGS[args.config][1] if not args.batch else args.batch
    batch = gbatch // world
    mr, ir = synth.config_streams(args.config)
    M = synth.random_symplectic(mr)
    pl = planner.plan(M)
    g = synth.iid_cn(ir, (64, 64))
    for _ in range(args.warmup):
        cpu_fft.transform(g, pl["chain"], 0.3, workers=1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(batch):
            cpu_fft.transform(g, pl["chain"], 0.3, workers=1)
    ms = max_over_ranks((time.perf_counter() - t0) / args.steps * 1e3, world)
    units = sum_over_ranks(batch, world)
    ranks = sum_over_ranks(1, world)
    sub = {}
    if world > 1 and args.config == 4 and not args.no_sub:   # the child-process plumbing of run_ours
        port = int(max_over_ranks(_free_port() if rank == 0 else 0, world))
        sub["C5_slab"] = slab_child(args, world, rank, int(os.environ.get("LOCAL_RANK", "0")), port,
                                    timeout=120, extra=("--dry-run",))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": units / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "sub": sub,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "strong", "dry_run": True, "ranks_reporting": int(ranks),
                          "config": {"global_batch": int(units), "per_gpu_batch": batch}}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-full", action="store_true", help="every CPU baseline of BASELINE.md §3 (adds minutes)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub-records (other configs)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--schedule", default="auto", choices=["auto", "line_passes", "on_chip"],
                    help="on-chip kernel where available (auto) or one launch per pass")
    ap.add_argument("--variant", default="HA", choices=["HA", "LC"], help="planner variant")
    ap.add_argument("--batch", type=int, default=0,
                    help="override the config's global batch (exploration; the default run uses the config's)")
    ap.add_argument("--dry-run", action="store_true", help="CPU-only plumbing check (gloo), no GPU")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(argv, args.gpus)
    if args.dry_run:
        return run_dry(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
