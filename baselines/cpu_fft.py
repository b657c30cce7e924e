"""A plain CPU FFT-based decomposition of the NsDLCT chain: the baseline BASELINE.json's
north_star asks bench.py to time next to the fp64 oracle ("a plain CPU FFT-based
decomposition on the box's host cores").

It evaluates the same operator list as the oracle (CM / CC stages of Eq. HA28 or
CCCMCCCM40, PAPER.md:773-787 / 1010-1019) with FFTs instead of dense DFT matrices:
  CM_Q g   = exp(j/2 z^T Q z) g on the centred grid of spacing dx       (Eq. BasicCM12)
  CC_B g   = F^-1 CM_{-B}(dw) F g, dw = 2 pi / (N dx)                   (Eq. BasicCC20)
with the centred DFT F = fftshift . fft2 . ifftshift (N even); the constants of
Eq. BasicDFT16 and of its exact inverse cancel inside a CC.  fp64, scipy.fft with
`workers` threads.  It is a reported baseline only: the plan (the chain) is an input,
and tests/test_cpu_fft_baseline.py checks it against the oracle on small N.
"""
import math

import numpy as np
import scipy.fft as sfft


def _chirp(n, Q, d):
    k = (np.arange(n, dtype=np.float64) - n // 2) * d
    q11, q22, q12 = Q[0][0], Q[1][1], 0.5 * (Q[0][1] + Q[1][0])
    # exp(j/2 (q11 p^2 + 2 q12 p q + q22 q^2)) as an outer structure: rows p, columns q
    return np.exp(0.5j * (q11 * k[:, None] ** 2 + 2.0 * q12 * k[:, None] * k[None, :] + q22 * k[None, :] ** 2))


def _F(g, workers):
    return sfft.fftshift(sfft.fft2(sfft.ifftshift(g), workers=workers))


def _Finv(G, workers):
    return sfft.fftshift(sfft.ifft2(sfft.ifftshift(G), workers=workers))


def transform(g, chain, dx, workers=-1, dtype=np.complex128):
    """g: (N, N) complex; chain: [("CM", Q) | ("CC", B), ...] in application order.
    dtype: complex128 (fp64 FFTs) or complex64 (fp32 FFTs; chirps computed in fp64 and
    rounded)."""
    out = np.asarray(g, dtype)
    n = out.shape[-1]
    dw = 2.0 * math.pi / (n * dx)
    for kind, Q in chain:
        Q = np.asarray(Q, np.float64)
        if kind == "CM":
            out = _chirp(n, Q, dx).astype(dtype) * out
        elif kind == "CC":
            out = _Finv(_chirp(n, -Q, dw).astype(dtype) * _F(out, workers), workers)
        else:
            raise ValueError("the FFT baseline covers the HA chain only (%s)" % kind)
    return out
