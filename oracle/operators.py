"""Discrete operators and the full NsDLCT O_plan (oracle; test infrastructure only).

Index convention (reading R1): centered indices
m, p in [-floor(N/2), ceil(N/2) - 1], stored at array index m + floor(N/2).
Grid (reading R2): input and output spacing dx (Delta_u = Delta_x);
the frequency grid of the DFT has spacing dw = 2 pi / (N dx).

Every DFT here is a dense matrix product with W[p, m] = exp(-2 pi j ((p m) mod N) / N)
built from exact integer products -- the definition of Eq. BasicDFT16, no FFT.
"""
import math

import numpy as np

from . import planner as _planner


def centered(n):
    """Centered sample indices of reading R1."""
    return np.arange(n, dtype=np.int64) - n // 2


def dft_kernel(n):
    """W[p, m] = exp(-j 2 pi p m / N) on centered p, m (Eq. BasicDFT16),
    the product p*m reduced mod N exactly in integers before the exponential."""
    k = centered(n)
    pm = np.mod(np.outer(k, k), n)
    return np.exp(-2j * math.pi * pm.astype(np.float64) / n)


_W_CACHE = {}


def _W(n):
    if n not in _W_CACHE:
        if len(_W_CACHE) > 4:
            _W_CACHE.clear()
        _W_CACHE[n] = dft_kernel(n)
    return _W_CACHE[n]


def dft2(g, dx):
    """Discrete 2D FT F_{x,y} of Eq. BasicDFT16:
    G[p,q] = (dx dy / (j 2 pi)) sum_m sum_n exp(-j 2 pi (pm + qn)/N) g[m,n].
    Output lives on the frequency grid dw = 2 pi / (N dx)."""
    g = np.asarray(g, np.complex128)
    W = _W(g.shape[-1])
    c = dx * dx / (2j * math.pi)
    return c * (W @ g @ W.T)


def idft2_exact(G, dx):
    """Exact inverse of dft2 (reading R3; the printed Eq. BasicDFT20, PAPER.md:184,
    carries the constant of Eq. BasicDFT16 and would give F^{-1}F = -I):
    g[m,n] = (j 2 pi / (dx dy)) (1/N^2) sum_p sum_q exp(+j 2 pi (pm + qn)/N) G[p,q]."""
    G = np.asarray(G, np.complex128)
    n = G.shape[-1]
    Wc = np.conj(_W(n))
    c = (2j * math.pi) / (dx * dx) / (n * n)
    return c * (Wc @ G @ Wc.T)


def idft2_printed(G, dx):
    """Eq. BasicDFT20 exactly as printed: constant dx dy/(j 2 pi), kernel
    exp(+j 2 pi (pm+qn)/N).  Used only to pin reading R3 (printed = -exact inverse)."""
    G = np.asarray(G, np.complex128)
    Wc = np.conj(_W(G.shape[-1]))
    return dx * dx / (2j * math.pi) * (Wc @ G @ Wc.T)


def chirp(n, Q, d):
    """exp(j/2 (q11 p^2 d^2 + 2 q12 p q d^2 + q22 q^2 d^2)) on the centered grid of
    spacing d (the kernel of Eq. BasicCM12)."""
    k = centered(n).astype(np.float64) * d
    P, Qg = np.meshgrid(k, k, indexing="ij")
    q11, q22 = Q[0, 0], Q[1, 1]
    q12 = 0.5 * (Q[0, 1] + Q[1, 0])
    return np.exp(0.5j * (q11 * P * P + 2.0 * q12 * P * Qg + q22 * Qg * Qg))


def cm(g, Q, d):
    """2D discrete CM O_CM^Q (Eq. BasicCM12) on spacing d."""
    g = np.asarray(g, np.complex128)
    return chirp(g.shape[-1], Q, d) * g


def cc(g, B, dx):
    """2D discrete CC O_CC^B = F^{-1} O_CM^{-B} F (Eq. BasicCC20);
    the middle CM is sampled on the frequency grid dw = 2 pi/(N dx) (reading R2)."""
    n = np.asarray(g).shape[-1]
    dw = 2.0 * math.pi / (n * dx)
    return idft2_exact(cm(dft2(g, dx), -np.asarray(B), dw), dx)


def cc1d(g, h, axis, dx):
    """1D discrete CC along x (axis 'x', rows index m) or y: F_x^{-1} CM F_x with
    chirp exp(-j/2 h p^2 dw^2) (Eq. LC12).  The 1D DFT pair is the
    x- or y-factor of Eq. BasicDFT16 and its exact inverse; their constants cancel."""
    g = np.asarray(g, np.complex128)
    n = g.shape[-1]
    W = _W(n)
    dw = 2.0 * math.pi / (n * dx)
    k = centered(n).astype(np.float64) * dw
    ch = np.exp(-0.5j * h * k * k)
    if axis == "x":
        return (np.conj(W) @ (ch[:, None] * (W @ g))) / n
    return ((g @ W.T) * ch[None, :]) @ np.conj(W).T / n


def affine_bilinear(g, Dm):
    """2D discrete affine transform with bilinear interpolation, Eq. BasicAffine12/16
    (PAPER.md:361-371), input and output on the same grid (Delta_u = Delta_x), so
    p1 = d11 p + d21 q,  q1 = d12 p + d22 q,  p2 = floor(p1), k = p1 - p2, etc.
    Taps outside the N x N grid read 0 (reading R10).  Without the sqrt(det D) factor."""
    g = np.asarray(g, np.complex128)
    n = g.shape[-1]
    off = n // 2
    k = centered(n).astype(np.float64)
    P, Qg = np.meshgrid(k, k, indexing="ij")
    p1 = Dm[0, 0] * P + Dm[1, 0] * Qg
    q1 = Dm[0, 1] * P + Dm[1, 1] * Qg
    p2 = np.floor(p1)
    q2 = np.floor(q1)
    kk = p1 - p2
    ll = q1 - q2
    p2i = p2.astype(np.int64) + off
    q2i = q2.astype(np.int64) + off

    def tap(i, j):
        ok = (i >= 0) & (i < n) & (j >= 0) & (j < n)
        out = np.zeros(P.shape, np.complex128)
        out[ok] = g[i[ok], j[ok]]
        return out

    return ((1 - kk) * (1 - ll) * tap(p2i, q2i) + (1 - kk) * ll * tap(p2i, q2i + 1)
            + kk * (1 - ll) * tap(p2i + 1, q2i) + kk * ll * tap(p2i + 1, q2i + 1))


def b0_transform(g, C, Dm, dx):
    """B = 0 case, Eq. Intro20:
    G(z') = sqrt(det D) exp(j/2 z'^T C D^T z') g(D^T z'), with g(D^T z') from the
    bilinear affine transform of Eq. BasicAffine12; principal sqrt (reading R10)."""
    sq = np.sqrt(complex(np.linalg.det(Dm)))
    S = C @ Dm.T
    S = 0.5 * (S + S.T)
    return sq * cm(affine_bilinear(g, Dm), S, dx)


def apply_chain(g, chain, dx, n1d=None):
    """Apply a plan's operator list (application order) to g."""
    out = np.asarray(g, np.complex128)
    for op in chain:
        if op[0] == "CM":
            out = cm(out, op[1], dx)
        elif op[0] == "CC":
            out = cc(out, op[1], dx)
        elif op[0] == "CC1":
            out = cc1d(out, op[1], op[2], dx)
        elif op[0] == "B0":
            out = b0_transform(out, op[1], op[2], dx)
        else:
            raise ValueError(op[0])
    return out


def lc_chain(pl):
    """LC-NsDLCT (Eq. LC12; form II Eq. CCCMCCCM44): the CC(H) with
    H = (h,0;0,0) or (0,0;0,h) becomes a 1D CC along x or y."""
    out = list(pl["chain"])
    if pl.get("axis") is None:
        return out                       # LC not applicable: HA fallback
    i = 0 if pl["kind"] == "I" else 3    # CC(H) is applied first in form I, last in form II
    Hm = out[i][1]
    h = Hm[0, 0] if pl["axis"] == "x" else Hm[1, 1]
    out[i] = ("CC1", h, pl["axis"])
    return out


def zero_pad(g, n_out):
    """Zero-padding of the input to (N + dN) x (N + dN):
    every sample keeps its centered coordinate (reading R1: array index m + floor(N/2)),
    so sample m lands at index m + floor(N'/2); everything else is 0.  The padded field
    is on the same spacing dx as the original."""
    g = np.asarray(g, np.complex128)
    n = g.shape[-1]
    if n_out < n:
        raise ValueError("n_out must be >= N")
    off = n_out // 2 - n // 2
    out = np.zeros(g.shape[:-2] + (n_out, n_out), np.complex128)
    out[..., off:off + n, off:off + n] = g
    return out


def nsdlct(g, M, dx=None, variant="HA", policy="reversible", h_override=None, pl=None):
    """O_plan: the paper's NsDLCT of g for ABCD matrix M.

    HA: Eq. HA28 in form I, Eq. CCCMCCCM40 in
    form II, dispatched by Eq. Reversible08 (+ reading R7).  LC: Eq. LC12 / CCCMCCCM44.
    B = 0: Eq. Intro20 with bilinear resampling.  g may be (N,N) or (batch,N,N).
    Returns (G, plan)."""
    g = np.asarray(g, np.complex128)
    n = g.shape[-1]
    if dx is None:
        dx = math.sqrt(2.0 * math.pi / n)
    if pl is None:
        pl = _planner.plan(M, variant=variant, policy=policy, h_override=h_override)
    chain = lc_chain(pl) if variant == "LC" else pl["chain"]
    if g.ndim == 2:
        return apply_chain(g, chain, dx), pl
    return np.stack([apply_chain(x, chain, dx) for x in g]), pl
