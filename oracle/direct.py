"""Direct method O_direct (oracle; test infrastructure only, see oracle/__init__.py).

Eq. Intro32:
  G[p,q] = dx dy / (2 pi sqrt(-det B)) sum_m sum_n
           exp[j/2 (r'^T D B^{-1} r' - 2 r^T B^{-1} r' + r^T B^{-1} A r)] g[m,n],
  r = (m dx, n dy), r' = (p du, q dv).
sqrt(-det B) takes the principal branch; the metaplectic sign of the fast operator can
differ by -1 (reading R4), so cross-operator comparisons are made modulo a global sign.

Evaluated as  G_k = pre * chi_out(r'_k) * sum_m E_A[k,m] sum_n h[m,n] E_B[k,n]
with h = chi_in * g, E_A[k,m] = exp(-j a_k x_m), E_B[k,n] = exp(-j b_k y_n),
(a_k, b_k) = B^{-1} r'_k -- an O(K N^2) BLAS-batched evaluation of the same sum.
"""
import math

import numpy as np

from .symplectic import blocks


def direct(g, M, dx_in, dx_out=None, n_out=None, out_points=None, chunk=2048):
    """O_direct(g) on output grid (n_out, dx_out) or at explicit output points.

    g: (N, N) samples g[m, n] on the centered grid of spacing dx_in.
    out_points: optional (K, 2) array of output coordinates r' (overrides the grid).
    Returns (n_out, n_out) or (K,) complex128."""
    g = np.asarray(g, np.complex128)
    n = g.shape[-1]
    A, B, C, D = blocks(M)
    Bi = np.linalg.inv(B)
    BiA = Bi @ A
    DBi = D @ Bi
    x = (np.arange(n) - n // 2) * dx_in
    X, Y = np.meshgrid(x, x, indexing="ij")
    h = g * np.exp(0.5j * (BiA[0, 0] * X * X + (BiA[0, 1] + BiA[1, 0]) * X * Y + BiA[1, 1] * Y * Y))
    if out_points is None:
        n_out = n if n_out is None else n_out
        dx_out = dx_in if dx_out is None else dx_out
        u = (np.arange(n_out) - n_out // 2) * dx_out
        U, V = np.meshgrid(u, u, indexing="ij")
        pts = np.stack([U.ravel(), V.ravel()], axis=1)
        shape = (n_out, n_out)
    else:
        pts = np.asarray(out_points, float)
        shape = (pts.shape[0],)
    pre = dx_in * dx_in / (2.0 * math.pi * np.sqrt(complex(-np.linalg.det(B))))
    out = np.empty(pts.shape[0], np.complex128)
    for s in range(0, pts.shape[0], chunk):
        P = pts[s:s + chunk]
        ab = P @ Bi.T                      # rows (a_k, b_k) = B^{-1} r'_k
        EA = np.exp(-1j * np.outer(ab[:, 0], x))
        EB = np.exp(-1j * np.outer(ab[:, 1], x))
        inner = np.sum((EA @ h) * EB, axis=1)
        chi_out = np.exp(0.5j * (DBi[0, 0] * P[:, 0] ** 2 + (DBi[0, 1] + DBi[1, 0]) * P[:, 0] * P[:, 1]
                                 + DBi[1, 1] * P[:, 1] ** 2))
        out[s:s + chunk] = pre * chi_out * inner
    return out.reshape(shape)


def direct_1d(g, a, b, d, dx_in, dx_out=None, n_out=None):
    """1D direct LCT sum (the 1D analogue of Eq. Intro32):
    G[p] = dx / sqrt(j 2 pi b) sum_m exp[j/2 (d/b u^2 - 2 x u / b + a/b x^2)] g[m],
    principal square root.  Used to pin the 2D constant on separable matrices (P6)."""
    g = np.asarray(g, np.complex128)
    n = g.shape[-1]
    n_out = n if n_out is None else n_out
    dx_out = dx_in if dx_out is None else dx_out
    x = (np.arange(n) - n // 2) * dx_in
    u = (np.arange(n_out) - n_out // 2) * dx_out
    K = np.exp(0.5j * ((d / b) * u[:, None] ** 2 - 2.0 * np.outer(u, x) / b + (a / b) * x[None, :] ** 2))
    return dx_in / np.sqrt(complex(2j * math.pi * b)) * (K @ g)
