"""Error metrics (test infrastructure only).

NMSE of Eq. Acc04, Eq. Add16 and Eq. Rev08
 all have the form sum|a - b|^2 / sum|b|^2.
"""
import math

import numpy as np


def nmse(a, ref):
    a = np.asarray(a); ref = np.asarray(ref)
    return float(np.sum(np.abs(a - ref) ** 2) / np.sum(np.abs(ref) ** 2))


def rel_l2(a, ref):
    return math.sqrt(nmse(a, ref))


def align_sign(a, ref):
    """a multiplied by s = sign Re<a, ref> (reading R4: comparisons across operators are
    made modulo the metaplectic +-1)."""
    s = 1.0 if np.real(np.vdot(a, ref)) >= 0 else -1.0
    return s * np.asarray(a)


def nmse_pm(a, ref):
    return nmse(align_sign(a, ref), ref)


def psnr(rec, ref):
    """PSNR in dB with peak = max|ref|."""
    mse = float(np.mean(np.abs(np.asarray(rec) - np.asarray(ref)) ** 2))
    peak = float(np.max(np.abs(ref)))
    return 10.0 * math.log10(peak * peak / mse) if mse > 0 else math.inf
