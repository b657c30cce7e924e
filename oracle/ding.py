"""Ding's 2D NsDLCT (§3.2, Eq. Ding04-16) -- oracle only.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The decomposition (Eq. Ding04)
    (A, B; C, D) = (I, 0; D B^-1, I) (B, 0; 0, B^-T) (0, I; -I, 0) (I, 0; B^-1 A, I)
gives (Eq. Ding12)
    O_Ding = O_CM^{D B^-1}  O_Affine^{B^-T}  F_{x,y}  O_CM^{B^-1 A},
with the discrete CM of Eq. BasicCM12, the DFT of Eq. BasicDFT16 and the bilinear affine
transform of Eq. BasicAffine12/16.  Readings (R14):
  * "two-times upsampling is performed in F": the input of F is
    zero-padded to N' = 2N (oracle.operators.zero_pad), so F's output lies on the
    frequency grid dw = 2 pi / (N' dx) with N' x N' samples;
  * the affine transform maps that grid to the N x N output grid du = dx:
    p1 = (d11 p du + d21 q du) / dw (Eq. BasicAffine16 with input spacing dw);
    taps outside the N' x N' grid read 0 and sqrt(det D) takes the principal branch
    (reading R10, as for the B = 0 case);
  * both CMs are on the space grid dx (input: N x N before padding; output: N x N).
"""
import math

import numpy as np

from . import operators as op
from .symplectic import blocks


def affine_bilinear_grid(g, Dm, d_in, d_out, n_out):
    """Eq. BasicAffine12/16 between grids: g on the centered
    N_in x N_in grid of spacing d_in, output on the centered n_out x n_out grid of
    spacing d_out; p1 = (d11 p d_out + d21 q d_out)/d_in, q1 = (d12 p d_out + d22 q
    d_out)/d_in, p2 = floor(p1), k = p1 - p2, ...  Taps outside the input grid read 0.
    Without the sqrt(det D) factor."""
    g = np.asarray(g, np.complex128)
    n_in = g.shape[-1]
    k_out = op.centered(n_out).astype(np.float64)
    P, Qg = np.meshgrid(k_out, k_out, indexing="ij")
    r = d_out / d_in
    p1 = (Dm[0, 0] * P + Dm[1, 0] * Qg) * r
    q1 = (Dm[0, 1] * P + Dm[1, 1] * Qg) * r
    p2 = np.floor(p1)
    q2 = np.floor(q1)
    kk = p1 - p2
    ll = q1 - q2
    off = n_in // 2
    p2i = p2.astype(np.int64) + off
    q2i = q2.astype(np.int64) + off

    def tap(i, j):
        ok = (i >= 0) & (i < n_in) & (j >= 0) & (j < n_in)
        out = np.zeros(P.shape, np.complex128)
        out[ok] = g[i[ok], j[ok]]
        return out

    return ((1 - kk) * (1 - ll) * tap(p2i, q2i) + (1 - kk) * ll * tap(p2i, q2i + 1)
            + kk * (1 - ll) * tap(p2i + 1, q2i) + kk * ll * tap(p2i + 1, q2i + 1))


def ding(g, M, dx=None, up=2):
    """O_Ding of Eq. Ding12 applied to the N x N field g (det B != 0), `up`-times
    upsampled F.  Returns the N x N output on spacing dx."""
    g = np.asarray(g, np.complex128)
    n = g.shape[-1]
    if dx is None:
        dx = math.sqrt(2.0 * math.pi / n)
    A, B, C, D = blocks(M)
    Bi = np.linalg.inv(B)
    h = op.cm(g, Bi @ A, dx)                        # O_CM^{B^-1 A}
    n2 = up * n
    Fh = op.dft2(op.zero_pad(h, n2), dx)            # F_{x,y} on dw = 2 pi/(n2 dx)
    dw = 2.0 * math.pi / (n2 * dx)
    Dm = Bi.T                                       # O_Affine^{B^-T}
    G = np.sqrt(complex(np.linalg.det(Dm))) * affine_bilinear_grid(Fh, Dm, dw, dx, n)
    return op.cm(G, D @ Bi, dx)                     # O_CM^{D B^-1}
