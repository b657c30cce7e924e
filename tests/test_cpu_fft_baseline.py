"""The CPU FFT-based baseline bench.py reports (baselines/cpu_fft.py) computes the same
operator as the oracle: checked on small N, both dispatch forms."""
import math

import numpy as np
import pytest

import synth
from baselines import cpu_fft
from oracle import metrics as me
from oracle import operators as op
from oracle import planner as opl


@pytest.mark.parametrize("n", [32, 64])
@pytest.mark.parametrize("policy", ["reversible", "formI"])
def test_fft_baseline_matches_oracle(n, policy):
    rng = np.random.default_rng(7 + n)
    for _ in range(3):
        M = synth.random_symplectic(rng)
        g = synth.iid_cn(rng, (n, n))
        ref, pl = op.nsdlct(g, M, policy=policy)
        got = cpu_fft.transform(g, pl["chain"], math.sqrt(2 * math.pi / n), workers=1)
        assert me.rel_l2(got, ref) < 1e-12


def test_fft_baseline_complex64():
    """The complex64 variant (reported next to the c64 GPU numbers) is the same operator at
    fp32 rounding."""
    rng = np.random.default_rng(3)
    M = synth.random_symplectic(rng)
    g = synth.iid_cn(rng, (64, 64))
    ref, pl = op.nsdlct(g, M)
    got = cpu_fft.transform(g, pl["chain"], math.sqrt(2 * math.pi / 64), workers=1, dtype=np.complex64)
    assert got.dtype == np.complex64 and me.rel_l2(got, ref) < 1e-5
