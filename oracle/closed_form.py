"""Closed forms used to pin the oracle (test infrastructure only).

* Hermite-Gaussian inputs, Eq. Acc12/Acc16, evaluated with the
  orthonormal Hermite-function recurrence (SPEC.md DESIGN DECISIONS of module grid):
  psi_0 = pi^{-1/4} e^{-x^2/2}, psi_1 = sqrt(2) x psi_0,
  psi_{k+1} = sqrt(2/(k+1)) x psi_k - sqrt(k/(k+1)) psi_{k-1}.
* Gaussian-beam law of the continuous NsLCT (obtained from Eq. Intro08 by a Gaussian
  integral): for g(z) = exp(j/2 z^T K z) with Im K > 0,
      G(z') = +- det(A + B K)^{-1/2} exp(j/2 z'^T (C + D K)(A + B K)^{-1} z').
  The +- is the metaplectic sign (reading R4); it is NOT fixed here.
"""
import math

import numpy as np

from .symplectic import blocks


def hermite_function(k, x):
    """HG_k(x) of Eq. Acc12."""
    x = np.asarray(x, float)
    p0 = math.pi ** -0.25 * np.exp(-0.5 * x * x)
    if k == 0:
        return p0
    p1 = math.sqrt(2.0) * x * p0
    for j in range(1, k):
        p0, p1 = p1, math.sqrt(2.0 / (j + 1)) * x * p1 - math.sqrt(j / (j + 1.0)) * p0
    return p1


def hg2d(orders, n, dx):
    """sum over (k,l) of HG_{k,l}(x,y) = HG_k(x) HG_l(y) (Eq. Acc16/Acc20) on the
    centered N x N grid of spacing dx (x along the first array axis)."""
    x = (np.arange(n) - n // 2) * dx
    out = np.zeros((n, n), np.complex128)
    for k, l in orders:
        out += np.outer(hermite_function(k, x), hermite_function(l, x))
    return out


def gaussian(K, n, dx):
    """g(z) = exp(j/2 z^T K z) sampled on the centered grid."""
    x = (np.arange(n) - n // 2) * dx
    X, Y = np.meshgrid(x, x, indexing="ij")
    return np.exp(0.5j * (K[0, 0] * X * X + (K[0, 1] + K[1, 0]) * X * Y + K[1, 1] * Y * Y))


def gaussian_lct(M, K, n, dx):
    """Closed-form NsLCT of gaussian(K) sampled on the centered output grid (up to the
    metaplectic sign): det(A+BK)^{-1/2} exp(j/2 z'^T (C+DK)(A+BK)^{-1} z')."""
    A, B, C, D = blocks(M)
    K = np.asarray(K, complex)
    T = A + B @ K
    Kout = (C + D @ K) @ np.linalg.inv(T)
    amp = 1.0 / np.sqrt(np.linalg.det(T))
    return amp * gaussian(Kout, n, dx)
