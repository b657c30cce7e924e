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
           "nslct_exec_pass_peer", "nslct_inverse_matrix", "nslct_comm_unique_id", "nslct_comm_init",
           "nslct_comm_info", "nslct_comm_destroy", "nslct_fp32_peak")
ABI_VERSION = 4
KERNELS = {"auto": 0, "generic": 1}
EXCHANGES = {"nccl": 0, "peer": 1}


class NslctError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status
        self.name = STATUS.get(status, str(status))


class nslct_opts(ctypes.Structure):
    _fields_ = [("dx", ctypes.c_double), ("variant", ctypes.c_int), ("dispatch", ctypes.c_int),
                ("h_fixed", ctypes.c_double * 3), ("device", ctypes.c_int), ("profile", ctypes.c_int),
                ("schedule", ctypes.c_int), ("n_in", ctypes.c_int), ("kernels", ctypes.c_int),
                ("host_chunk_kb", ctypes.c_int), ("comm", ctypes.c_void_p), ("exchange_chunks", ctypes.c_int),
                ("exchange", ctypes.c_int), ("reserved", ctypes.c_int * 4)]


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
        L.nslct_inverse_matrix.argtypes = [dp, dp]
        L.nslct_comm_unique_id.argtypes = [ctypes.c_char_p]
        L.nslct_comm_init.argtypes = [ctypes.POINTER(vp), ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
        L.nslct_comm_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.nslct_comm_destroy.argtypes = [vp]
        L.nslct_fp32_peak.argtypes = [ctypes.c_int, dp]
        L.nslct_last_error.restype = ctypes.c_char_p
        L.nslct_abi_version.restype = ctypes.c_int
        for f in ("nslct_plan", "nslct_plan_ex", "nslct_exec", "nslct_exec_host", "nslct_plan_info",
                  "nslct_plan_describe", "nslct_pass_ms", "nslct_destroy", "nslct_plan_slab",
                  "nslct_exec_pass", "nslct_exec_pass_peer", "nslct_inverse_matrix", "nslct_comm_unique_id",
                  "nslct_comm_init", "nslct_comm_info", "nslct_comm_destroy", "nslct_fp32_peak"):
            getattr(L, f).restype = ctypes.c_int
        if L.nslct_abi_version() != ABI_VERSION:
            raise ImportError("libnslct.so ABI %d, binding expects %d: rebuild (python -m paper_1707_03688_b200.build)"
                              % (L.nslct_abi_version(), ABI_VERSION))
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
              schedule="auto", n_in=None, kernels="auto", host_chunk_kb=0, comm=None, exchange_chunks=0,
              exchange="nccl"):
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
    o.kernels = KERNELS[kernels]
    o.host_chunk_kb = int(host_chunk_kb)
    o.comm = None if comm is None else comm.handle
    o.exchange_chunks = int(exchange_chunks)
    o.exchange = EXCHANGES[exchange]
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


def _want_dtype(dtype):
    import torch
    return torch.complex64 if dtype == "c64" else torch.complex128


class Plan:
    """RAII wrapper of nslct_plan_t.  exec() takes torch CUDA tensors (complex64/128).
    n_in (< n): fused zero-padding -- inputs are [batch, n_in, n_in], outputs [batch, n, n].
    comm (a Communicator): ONE n x n transform row-slab sharded over the communicator's
    ranks -- batch must be 1 and exec() takes this rank's slab [n/nranks, n]; the library
    runs every pass and every exchange itself (exchange="nccl": chunked NCCL all-to-all
    overlapping the passes; "peer": stores straight into the peers' buffers over NVLink).
    Creating a comm plan is collective over the communicator."""

    def __init__(self, n, M, batch, dtype="c64", dx=None, variant="HA", dispatch="reversible",
                 h_fixed=None, device=None, profile=False, schedule="auto", n_in=None, kernels="auto",
                 host_chunk_kb=0, comm=None, exchange_chunks=0, exchange="nccl"):
        self.n, self.batch = int(n), int(batch)
        self.n_in = self.n if n_in is None else int(n_in)
        self.dtype = dtype
        self.comm = comm
        if device is None:
            try:
                import torch
                device = torch.cuda.current_device() if torch.cuda.is_available() else None
            except ImportError:
                device = None
        self.device = device
        a, ap = _abcd(M)
        o = make_opts(dx, variant, dispatch, h_fixed, device, profile, schedule, n_in, kernels, host_chunk_kb,
                      comm, exchange_chunks, exchange)
        h = ctypes.c_void_p()
        _check(lib().nslct_plan_ex(ctypes.byref(h), self.n, ap, self.batch,
                                   C64 if dtype == "c64" else C128, ctypes.byref(o)))
        self._h = h
        self.profile = profile
        if comm is not None:
            self.rows = self.n // comm.nranks
            self.in_shape = self.out_shape = (self.rows, self.n)
        else:
            self.in_shape = (self.batch, self.n_in, self.n_in)
            self.out_shape = (self.batch, self.n, self.n)

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

    def _check_dev(self, t, name, shape):
        want = _want_dtype(self.dtype)
        if not (t.is_cuda and t.dtype == want and t.is_contiguous() and tuple(t.shape) == tuple(shape)):
            raise ValueError("%s must be a contiguous CUDA %s tensor of shape %s (got %s %s %s)"
                             % (name, want, tuple(shape), t.device, t.dtype, tuple(t.shape)))
        if self.device is not None and t.device.index != self.device:
            raise ValueError("%s is on %s, the plan on cuda:%d" % (name, t.device, self.device))

    def exec(self, x, out=None, stream=None):
        """x: torch CUDA tensor of the plan's input shape ([batch, n_in, n_in], or the
        slab [n/nranks, n] of a comm plan), complex64 (c64) / complex128 (c128).  out:
        optional tensor of the output shape (may be x unless the plan zero-pads)."""
        import torch
        if x.dim() == 2 and self.comm is None and self.batch == 1:
            x = x.unsqueeze(0)
        self._check_dev(x, "x", self.in_shape)
        if out is None:
            out = torch.empty(self.out_shape, dtype=x.dtype, device=x.device)
        else:
            self._check_dev(out, "out", self.out_shape)
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        self.exec_ptr(x.data_ptr(), out.data_ptr(), s.cuda_stream)
        return out

    def exec_host(self, host_in, host_out, stream=None):
        """host_in/host_out: CPU torch tensors or numpy arrays (pinned for full speed) of the
        plan's input/output shapes and dtype, C-contiguous."""
        want = np.complex64 if self.dtype == "c64" else np.complex128

        def ptr(t, name, shape):
            if hasattr(t, "data_ptr"):
                import torch
                ok = (not t.is_cuda and t.dtype == _want_dtype(self.dtype) and t.is_contiguous()
                      and tuple(t.shape) == tuple(shape))
                p = t.data_ptr()
            else:
                ok = (isinstance(t, np.ndarray) and t.dtype == want and t.flags.c_contiguous
                      and tuple(t.shape) == tuple(shape))
                p = t.ctypes.data if ok else 0
            if not ok:
                raise ValueError("%s must be a C-contiguous host %s array of shape %s" % (name, want.__name__, tuple(shape)))
            return p
        if self.comm is not None:
            raise ValueError("exec_host: not for comm (slab) plans")
        pi = ptr(host_in, "host_in", self.in_shape)
        po = ptr(host_out, "host_out", self.out_shape)
        sp = 0
        if stream is not None:
            sp = stream.cuda_stream
        _check(lib().nslct_exec_host(self._h, ctypes.c_void_p(pi), ctypes.c_void_p(po), ctypes.c_void_p(sp)))
        return host_out

    def pass_ms(self):
        buf = (ctypes.c_float * 8)()
        nw = ctypes.c_int(0)
        _check(lib().nslct_pass_ms(self._h, buf, 8, ctypes.byref(nw)))
        return [buf[i] for i in range(nw.value)]


class Communicator:
    """nslct_comm_t: the library's own NCCL communicator (one process per GPU).
    Communicator(group): over a torch.distributed process group -- rank 0's NCCL unique id
    is broadcast through the group, then every rank initialises on its current CUDA device.
    Communicator.local(): a one-rank communicator (no process group needed)."""

    def __init__(self, group=None, _uid=None, _rank=None, _nranks=None):
        if _uid is None:
            import torch.distributed as dist
            uid = ctypes.create_string_buffer(128)
            if dist.get_rank(group) == 0:
                _check(lib().nslct_comm_unique_id(uid))
            obj = [bytes(uid.raw)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
            _uid, _rank, _nranks = obj[0], dist.get_rank(group), dist.get_world_size(group)
        h = ctypes.c_void_p()
        _check(lib().nslct_comm_init(ctypes.byref(h), _uid, int(_rank), int(_nranks)))
        self.handle = h
        r, nr = ctypes.c_int(), ctypes.c_int()
        _check(lib().nslct_comm_info(h, ctypes.byref(r), ctypes.byref(nr)))
        self.rank, self.nranks = r.value, nr.value

    @classmethod
    def local(cls):
        uid = ctypes.create_string_buffer(128)
        _check(lib().nslct_comm_unique_id(uid))
        return cls(_uid=bytes(uid.raw), _rank=0, _nranks=1)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().nslct_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class SlabPlan(Plan):
    """One pass at a time of a row-slab transform (nslct_plan_slab / nslct_exec_pass /
    nslct_exec_pass_peer): the entry points a caller uses to run the slab passes with its
    own exchange -- e.g. the single-GPU multi-rank emulation in the tests.  The product
    path for multi-GPU is Plan(..., comm=Communicator(...)), which runs every pass and
    exchange inside the library."""

    def __init__(self, n, M, nranks, rank, dtype="c64", dx=None, variant="HA", dispatch="reversible",
                 h_fixed=None, device=None, kernels="auto", exchange_chunks=0):
        self.n, self.batch, self.dtype = int(n), 1, dtype
        self.nranks, self.rank = int(nranks), int(rank)
        self.L = self.n // self.nranks
        self.comm = None
        self.device = device
        a, ap = _abcd(M)
        o = make_opts(dx, variant, dispatch, h_fixed, device, False, kernels=kernels, exchange_chunks=exchange_chunks)
        h = ctypes.c_void_p()
        _check(lib().nslct_plan_slab(ctypes.byref(h), self.n, ap, self.nranks, self.rank,
                                     C64 if dtype == "c64" else C128, ctypes.byref(o)))
        self._h = h
        self.profile = False
        self.in_shape = self.out_shape = (self.L, self.n)
        self.n_passes = self.info()["n_passes"]

    def exec_pass(self, k, x, out, stream=None):
        import torch
        self._check_dev(x, "x", self.in_shape)
        self._check_dev(out, "out", self.out_shape)
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        _check(lib().nslct_exec_pass(self._h, int(k), ctypes.c_void_p(x.data_ptr()),
                                     ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
        return out

    def exec_pass_peer(self, k, x, peer_ptrs, stream=None):
        """Transposing pass k with the exchange fused into its store: row-block s goes to
        peer_ptrs[s] (device pointers, one per rank) at block offset rank*L*L."""
        import torch
        self._check_dev(x, "x", self.in_shape)
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        arr = (ctypes.c_void_p * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
        _check(lib().nslct_exec_pass_peer(self._h, int(k), ctypes.c_void_p(x.data_ptr()), arr,
                                          len(peer_ptrs), ctypes.c_void_p(s.cuda_stream)))


def fp32_peak_tflops(device=0):
    """Measured FP32 FMA throughput of the device (nslct_fp32_peak), TFLOP/s."""
    t = ctypes.c_double(0.0)
    _check(lib().nslct_fp32_peak(int(device), ctypes.byref(t)))
    return t.value


def default_dx(n):
    return math.sqrt(2.0 * math.pi / n)


def inverse_matrix(M):
    """M^-1 = (D^T, -B^T; -C^T, A^T) (Eq. CCCMCCCM20), computed by the
    library (nslct_inverse_matrix): the inverse transform's matrix."""
    a, ap = _abcd(M)
    out = np.empty(16, np.float64)
    _check(lib().nslct_inverse_matrix(ap, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return out.reshape(4, 4)


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
