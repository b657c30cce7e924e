"""Thin ctypes binding of libnslct.so (include/nslct.h).

Argument marshalling only: every step of the transform runs in the library's CUDA
kernels.  There is no CPU fallback: if libnslct.so is missing or fails to load, every
entry point raises.  PyTorch is used only for device memory and streams.
"""
import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# NSLCT_LIB: an alternative in-tree build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("NSLCT_LIB") or os.path.join(_HERE, "libnslct.so")

C64, C128 = 0, 1
VARIANTS = {"HA": 0, "LC": 1, "FIXED_H": 2, "DING": 3}
DISPATCH = {"reversible": 0, "formI": 1}
STATUS = {0: "OK", 1: "E_ARG", 2: "E_NOT_SYMPLECTIC", 3: "E_NO_DECOMP", 4: "E_UNSUPPORTED_N",
          5: "E_CUDA", 6: "E_NCCL", 7: "E_OOM"}
KINDS = {0: "B0", 1: "I", 2: "II", 3: "DING"}

# every symbol include/nslct.h declares
EXPORTS = ("nslct_opts_default", "nslct_plan", "nslct_plan_ex", "nslct_exec", "nslct_exec_host",
           "nslct_plan_info", "nslct_plan_describe", "nslct_pass_ms", "nslct_destroy",
           "nslct_last_error", "nslct_abi_version", "nslct_plan_slab", "nslct_exec_pass",
           "nslct_exec_pass_peer")


class NslctError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status
        self.name = STATUS.get(status, str(status))


class nslct_opts(ctypes.Structure):
    _fields_ = [("dx", ctypes.c_double), ("variant", ctypes.c_int), ("dispatch", ctypes.c_int),
                ("h_fixed", ctypes.c_double * 3), ("device", ctypes.c_int), ("profile", ctypes.c_int),
                ("schedule", ctypes.c_int), ("n_in", ctypes.c_int), ("reserved", ctypes.c_int * 4)]


class nslct_plan_desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("variant", ctypes.c_int), ("lc_axis", ctypes.c_int),
                ("n_passes", ctypes.c_int),
                ("H", ctypes.c_double * 3), ("Bp", ctypes.c_double * 3), ("P2", ctypes.c_double * 3),
                ("P4", ctypes.c_double * 3), ("Q", (ctypes.c_double * 3) * 5),
                ("dx", ctypes.c_double), ("objective", ctypes.c_double),
                ("sym_residual", ctypes.c_double), ("recomposition_residual", ctypes.c_double),
                ("dispatch_key", ctypes.c_double), ("n_launches", ctypes.c_int), ("on_chip", ctypes.c_int),
                ("fft_len", ctypes.c_int), ("n_in", ctypes.c_int)]


_LIB = None


def lib():
    """Load libnslct.so (fails loudly when it is missing: there is no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libnslct.so not built (run python -m paper_1707_03688_b200.build)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        L.nslct_opts_default.argtypes = [ctypes.POINTER(nslct_opts)]
        L.nslct_opts_default.restype = None
        L.nslct_plan.argtypes = [ctypes.POINTER(vp), i64, dp, i64, ctypes.c_int]
        L.nslct_plan_ex.argtypes = [ctypes.POINTER(vp), i64, dp, i64, ctypes.c_int, ctypes.POINTER(nslct_opts)]
        L.nslct_exec.argtypes = [vp, vp, vp, vp]
        L.nslct_plan_slab.argtypes = [ctypes.POINTER(vp), i64, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(nslct_opts)]
        L.nslct_exec_pass.argtypes = [vp, ctypes.c_int, vp, vp, vp]
        L.nslct_exec_pass_peer.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(vp), ctypes.c_int, vp]
        L.nslct_exec_host.argtypes = [vp, vp, vp, vp]
        L.nslct_plan_info.argtypes = [vp, ctypes.POINTER(nslct_plan_desc)]
        L.nslct_plan_describe.argtypes = [i64, dp, ctypes.POINTER(nslct_opts), ctypes.POINTER(nslct_plan_desc)]
        L.nslct_pass_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.nslct_destroy.argtypes = [vp]
        L.nslct_last_error.restype = ctypes.c_char_p
        L.nslct_abi_version.restype = ctypes.c_int
        for f in ("nslct_plan", "nslct_plan_ex", "nslct_exec", "nslct_exec_host", "nslct_plan_info",
                  "nslct_plan_describe", "nslct_pass_ms", "nslct_destroy", "nslct_plan_slab",
                  "nslct_exec_pass", "nslct_exec_pass_peer"):
            getattr(L, f).restype = ctypes.c_int
        _LIB = L
    return _LIB


def _check(st):
    if st != 0:
        raise NslctError(st, lib().nslct_last_error().decode(errors="replace"))


def _abcd(M):
    a = np.ascontiguousarray(np.asarray(M, dtype=np.float64).reshape(16))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


SCHEDULES = {"auto": 0, "line_passes": 1, "on_chip": 2}


def make_opts(dx=None, variant="HA", dispatch="reversible", h_fixed=None, device=None, profile=False,
              schedule="auto", n_in=None):
    o = nslct_opts()
    lib().nslct_opts_default(ctypes.byref(o))
    o.dx = float(dx) if dx else 0.0
    o.variant = VARIANTS[variant]
    o.dispatch = DISPATCH[dispatch]
    if h_fixed is not None:
        o.variant = VARIANTS["FIXED_H"]
        for i in range(3):
            o.h_fixed[i] = float(h_fixed[i])
    o.device = -1 if device is None else int(device)
    o.profile = 1 if profile else 0
    o.schedule = SCHEDULES[schedule]
    o.n_in = 0 if n_in is None else int(n_in)
    return o


def _desc_dict(d):
    s = lambda a: np.array([[a[0], a[2]], [a[2], a[1]]])
    return dict(kind=KINDS[d.kind], variant={0: "HA", 1: "LC", 2: "FIXED_H", 3: "DING"}[d.variant],
                lc_axis={0: None, 1: "x", 2: "y"}[d.lc_axis], n_passes=d.n_passes,
                h=np.array(list(d.H)), H=s(d.H), Bp=s(d.Bp), P2=s(d.P2), P4=s(d.P4),
                Q=[s(d.Q[i]) for i in range(5)], dx=d.dx, objective=d.objective,
                sym_residual=d.sym_residual, recomposition_residual=d.recomposition_residual,
                dispatch_key=d.dispatch_key, n_launches=d.n_launches, on_chip=bool(d.on_chip),
                fft_len=d.fft_len, n_in=d.n_in)


def nslct_plan_describe(n, M, **kw):
    """Host-only planning (no GPU needed): returns the plan description dict."""
    a, ap = _abcd(M)
    o = make_opts(**kw)
    d = nslct_plan_desc()
    _check(lib().nslct_plan_describe(int(n), ap, ctypes.byref(o), ctypes.byref(d)))
    return _desc_dict(d)


class Plan:
    """RAII wrapper of nslct_plan_t.  exec() takes torch CUDA tensors (complex64/128).
    n_in (< n): fused zero-padding -- inputs are [batch, n_in, n_in], outputs [batch, n, n]."""

    def __init__(self, n, M, batch, dtype="c64", dx=None, variant="HA", dispatch="reversible",
                 h_fixed=None, device=None, profile=False, schedule="auto", n_in=None):
        self.n, self.batch = int(n), int(batch)
        self.n_in = self.n if n_in is None else int(n_in)
        self.dtype = dtype
        a, ap = _abcd(M)
        o = make_opts(dx, variant, dispatch, h_fixed, device, profile, schedule, n_in)
        h = ctypes.c_void_p()
        _check(lib().nslct_plan_ex(ctypes.byref(h), self.n, ap, self.batch,
                                   C64 if dtype == "c64" else C128, ctypes.byref(o)))
        self._h = h
        self.profile = profile

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().nslct_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def info(self):
        d = nslct_plan_desc()
        _check(lib().nslct_plan_info(self._h, ctypes.byref(d)))
        return _desc_dict(d)

    def exec_ptr(self, in_ptr, out_ptr, stream_ptr=0):
        _check(lib().nslct_exec(self._h, ctypes.c_void_p(in_ptr), ctypes.c_void_p(out_ptr),
                                ctypes.c_void_p(stream_ptr)))

    def exec(self, x, out=None, stream=None):
        """x: torch CUDA tensor [batch, n_in, n_in] of complex64 (c64) / complex128 (c128)."""
        import torch
        want = torch.complex64 if self.dtype == "c64" else torch.complex128
        ni = self.n_in
        if not (x.is_cuda and x.dtype == want and x.is_contiguous()
                and tuple(x.shape[-2:]) == (ni, ni) and x.numel() == self.batch * ni * ni):
            raise ValueError("exec expects a contiguous CUDA %s tensor of %d x %d x %d"
                             % (want, self.batch, ni, ni))
        if out is None:
            out = torch.empty((self.batch, self.n, self.n), dtype=want, device=x.device)
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        self.exec_ptr(x.data_ptr(), out.data_ptr(), s.cuda_stream)
        return out

    def exec_host(self, host_in, host_out, stream=None):
        """host_in/host_out: CPU torch tensors or numpy arrays (pinned for full speed)."""
        def ptr(t):
            return t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data
        sp = 0
        if stream is not None:
            sp = stream.cuda_stream
        _check(lib().nslct_exec_host(self._h, ctypes.c_void_p(ptr(host_in)),
                                     ctypes.c_void_p(ptr(host_out)), ctypes.c_void_p(sp)))
        return host_out

    def pass_ms(self):
        buf = (ctypes.c_float * 8)()
        nw = ctypes.c_int(0)
        _check(lib().nslct_pass_ms(self._h, buf, 8, ctypes.byref(nw)))
        return [buf[i] for i in range(nw.value)]


class SlabPlan(Plan):
    """One n x n transform sharded as row slabs over nranks (nslct_plan_slab).

    run(x_slab, exchange) executes the passes of this rank's slab of L = n/nranks rows;
    exchange(send, recv) must perform the all-to-all of nranks blocks of L*L elements
    between passes (torch_all_to_all() for NCCL/gloo process groups)."""

    def __init__(self, n, M, nranks, rank, dtype="c64", dx=None, variant="HA", dispatch="reversible",
                 h_fixed=None, device=None):
        self.n, self.batch, self.dtype = int(n), 1, dtype
        self.nranks, self.rank = int(nranks), int(rank)
        self.L = self.n // self.nranks
        a, ap = _abcd(M)
        o = make_opts(dx, variant, dispatch, h_fixed, device, False)
        h = ctypes.c_void_p()
        _check(lib().nslct_plan_slab(ctypes.byref(h), self.n, ap, self.nranks, self.rank,
                                     C64 if dtype == "c64" else C128, ctypes.byref(o)))
        self._h = h
        self.profile = False
        self.n_passes = self.info()["n_passes"]

    def exec_pass(self, k, x, out, stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        _check(lib().nslct_exec_pass(self._h, int(k), ctypes.c_void_p(x.data_ptr()),
                                     ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
        return out

    def exec_pass_peer(self, k, x, peer_ptrs, stream=None):
        """Transposing pass k with the exchange fused into its store: row-block s goes to
        peer_ptrs[s] (device pointers, one per rank) at block offset rank*L*L."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        arr = (ctypes.c_void_p * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
        _check(lib().nslct_exec_pass_peer(self._h, int(k), ctypes.c_void_p(x.data_ptr()), arr,
                                          len(peer_ptrs), ctypes.c_void_p(s.cuda_stream)))

    def run_peer(self, x_slab, recv, peer_ptrs, barrier, out=None, stream=None):
        """The slab transform with every all-to-all fused into the producing pass's store
        (nslct_exec_pass_peer).  recv: this rank's two receive buffers [L, n] (double
        buffering across passes); peer_ptrs[b][s]: rank s's receive buffer b; barrier():
        a stream-ordered cross-rank barrier run after each transposing pass."""
        import torch
        out = torch.empty_like(x_slab) if out is None else out
        cur = x_slab
        for k in range(self.n_passes - 1):
            self.exec_pass_peer(k, cur, peer_ptrs[k % 2], stream)
            barrier()
            cur = recv[k % 2]
        self.exec_pass(self.n_passes - 1, cur, out, stream)
        return out

    def run(self, x_slab, exchange, out=None, stream=None):
        """x_slab: contiguous CUDA tensor [L, n] (this rank's rows).  Returns [L, n]."""
        import torch
        want = torch.complex64 if self.dtype == "c64" else torch.complex128
        if not (x_slab.is_cuda and x_slab.dtype == want and x_slab.is_contiguous()
                and tuple(x_slab.shape) == (self.L, self.n)):
            raise ValueError("run expects a contiguous CUDA %s tensor of %d x %d" % (want, self.L, self.n))
        send = torch.empty_like(x_slab)    # pass outputs: nranks row-blocks of [L][L]
        recv = torch.empty_like(x_slab)    # all-to-all results: the next pass's input
        out = torch.empty_like(x_slab) if out is None else out
        cur = x_slab
        for k in range(self.n_passes):
            if k == self.n_passes - 1:
                self.exec_pass(k, cur, out, stream)
            else:
                self.exec_pass(k, cur, send, stream)
                exchange(send, recv)   # stream-ordered after pass k; recv was last read by pass k
                cur = recv
        return out


def torch_all_to_all(group=None):
    """exchange(send, recv) for SlabPlan.run over a torch.distributed process group
    (NCCL on GPUs): nranks equal blocks of L*L elements."""
    import torch.distributed as dist

    def exchange(send, recv):
        dist.all_to_all_single(recv.view(-1), send.view(-1), group=group)
    return exchange


def symm_mem_exchange(L, n, dtype="c64", group=None):
    """Receive buffers for SlabPlan.run_peer in torch symmetric memory (CUDA peer memory
    over NVLink on a multi-GPU node): returns (recv, peer_ptrs, barrier).  Multi-GPU only;
    not exercised by this round's single-GPU tests (the kernel path is, through
    emulate_slabs_peer)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    want = torch.complex64 if dtype == "c64" else torch.complex128
    grp = group if group is not None else dist.group.WORLD
    recv, handles = [], []
    for _ in range(2):
        b = symm.empty(L, n, dtype=want, device=torch.device("cuda", torch.cuda.current_device()))
        handles.append(symm.rendezvous(b, grp))
        recv.append(b)
    peer_ptrs = [list(h.buffer_ptrs) for h in handles]
    return recv, peer_ptrs, (lambda: handles[0].barrier())


def emulate_slabs_peer(n, M, x_full, nranks, dtype="c64", **kw):
    """Single-GPU emulation of the fused peer-store exchange: nranks slab plans run one
    after another, each transposing pass storing its row-blocks straight into the other
    "ranks'" receive buffers (all on this GPU; no kernel waits on another).  Returns the
    assembled [n, n] output."""
    import torch
    L = n // nranks
    plans = [SlabPlan(n, M, nranks, r, dtype=dtype, **kw) for r in range(nranks)]
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


def emulate_slabs(n, M, x_full, nranks, dtype="c64", **kw):
    """Single-GPU emulation of the row-slab mode: nranks slab plans run one after another,
    the all-to-all done by block copies on the device (no kernel waits on another).
    x_full: CUDA tensor [n, n].  Returns the assembled [n, n] output."""
    import torch
    L = n // nranks
    plans = [SlabPlan(n, M, nranks, r, dtype=dtype, **kw) for r in range(nranks)]
    cur = [x_full[r * L:(r + 1) * L].contiguous() for r in range(nranks)]
    outs = [torch.empty_like(c) for c in cur]
    np_ = plans[0].n_passes
    for k in range(np_):
        last = (k == np_ - 1)
        for r in range(nranks):
            plans[r].exec_pass(k, cur[r], outs[r])
        if last:
            break
        # all-to-all: block s of rank r's output -> block r of rank s's input
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


def default_dx(n):
    return math.sqrt(2.0 * math.pi / n)


def inverse_matrix(M):
    """M^-1 = (D^T, -B^T; -C^T, A^T) (Eq. CCCMCCCM20): the inverse transform's matrix."""
    M = np.asarray(M, dtype=np.float64).reshape(4, 4)
    A, B, C, D = M[:2, :2], M[:2, 2:], M[2:, :2], M[2:, 2:]
    return np.block([[D.T, -B.T], [-C.T, A.T]])


def nsdlct(x, M, variant="HA", dispatch="reversible", dx=None, n=None, h_fixed=None, stream=None):
    """One-shot NsDLCT of x ([n_in, n_in] or [batch, n_in, n_in], complex64/complex128) for
    the 4x4 ABCD matrix M: plan, execute, free.  CUDA tensors run on their device; numpy
    arrays or CPU tensors go through nslct_exec_host (host in, host out).  n (>= n_in)
    zero-pads the input to n x n inside the first pass.  Returns the
    same kind of array, [.., n, n].  For repeated calls build a Plan once instead."""
    import torch
    is_np = isinstance(x, np.ndarray)
    t = torch.from_numpy(np.ascontiguousarray(x)) if is_np else x
    if t.dtype not in (torch.complex64, torch.complex128):
        raise ValueError("nsdlct expects complex64 or complex128 input")
    dtype = "c64" if t.dtype == torch.complex64 else "c128"
    squeeze = t.dim() == 2
    if squeeze:
        t = t.unsqueeze(0)
    b, n_in = t.shape[0], t.shape[-1]
    n_out = n_in if n is None else int(n)
    kw = dict(dtype=dtype, dx=dx, variant=variant, dispatch=dispatch, h_fixed=h_fixed,
              n_in=(n_in if n_out != n_in else None))
    if t.is_cuda:
        with torch.cuda.device(t.device):
            with Plan(n_out, M, b, device=t.device.index, **kw) as p:
                out = p.exec(t.contiguous(), stream=stream)
                (stream or torch.cuda.current_stream(t.device)).synchronize()   # before the plan is freed
    else:
        with Plan(n_out, M, b, **kw) as p:
            out = torch.empty((b, n_out, n_out), dtype=t.dtype)
            p.exec_host(t.contiguous(), out, stream)
    if squeeze:
        out = out[0]
    return out.numpy() if is_np else out


def nsdlct_inverse(G, M, **kw):
    """The inverse NsDLCT: nsdlct on M^-1 (with the reversible dispatch the pair is exact
    to rounding)."""
    return nsdlct(G, inverse_matrix(M), **kw)
