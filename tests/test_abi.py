"""CPU tests of the C-ABI library: it loads, exports every symbol include/nslct.h declares,
and its host planner (nslct_plan_describe, no CUDA call) agrees with the oracle planner.
No compute calls (no GPU here)."""
import math
import os
import re

import numpy as np
import pytest

import synth
from oracle import planner as opl
from oracle import symplectic as sy
from paper_1707_03688_b200 import nslct

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "nslct.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nslct_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = nslct.lib()
    declared = header_functions()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(nslct.EXPORTS) == declared
    assert L.nslct_abi_version() == nslct.ABI_VERSION == 4


def test_describe_errors():
    with pytest.raises(nslct.NslctError) as e:
        nslct.nslct_plan_describe(32, np.eye(4) * 1.1)
    assert e.value.name == "E_NOT_SYMPLECTIC"
    Z = np.zeros((2, 2))
    R = np.array([[0.0, 1.0], [-1.0, 0.0]])
    with pytest.raises(nslct.NslctError) as e:
        nslct.nslct_plan_describe(32, np.block([[Z, R], [-R, Z]]))
    assert e.value.name == "E_NO_DECOMP"
    M = np.eye(4)
    M[0, 1] = np.nan
    with pytest.raises(nslct.NslctError) as e:
        nslct.nslct_plan_describe(32, M)
    assert e.value.name == "E_ARG"


def test_b0_and_special_plans():
    assert nslct.nslct_plan_describe(32, np.eye(4))["kind"] == "B0"
    d = nslct.nslct_plan_describe(32, synth.dft_matrix4())
    assert d["kind"] == "I" and np.abs(d["h"]).max() == 0.0 and d["objective"] == 64.0
    d = nslct.nslct_plan_describe(32, synth.idft_matrix4())
    assert d["kind"] == "II"
    assert nslct.nslct_plan_describe(32, synth.idft_matrix4(), dispatch="formI")["kind"] == "I"
    assert abs(nslct.nslct_plan_describe(64, np.eye(4))["dx"] - math.sqrt(2 * math.pi / 64)) < 1e-15


def _oracle_Q(p):
    """The five executed chirps implied by the oracle plan (application order)."""
    Z = np.zeros((2, 2))
    if p["kind"] == "I":
        return [Z, -p["H"], p["P2"], -p["Bp"], p["P4"]]
    ch = p["chain"]   # CM(Q_right), CC(B1'), CM(Q_left), CC(H1)
    return [ch[0][1], -ch[1][1], ch[2][1], -ch[3][1], Z]


@pytest.mark.parametrize("variant", ["HA", "LC"])
def test_planner_parity_with_oracle(variant):
    """The C++ planner (mirror formulas for form II) and the oracle planner (literal
    Eq. CCCMCCCM08-16) agree on kind, objective (1e-9 rel) and executed chirps."""
    r, _ = synth.config_streams(50)
    mats = [synth.random_symplectic(r) for _ in range(12)]
    mats += [synth.gyrator_matrix4(a) for a in (0.7, 2.5)]
    mats += [sy.polar_project(np.array(x, float)) for x in (
        [[0, 1.1217, -0.7754, -0.3765], [-1.0934, -1.8826, 1.1005, 1.3878],
         [0.1697, -1.4013, -0.5352, 1.2447], [-0.2014, -0.5209, -0.5916, 0.3141]],)]
    for M in mats:
        d = nslct.nslct_plan_describe(64, M, variant=variant)
        p = opl.plan(M, variant=variant)
        assert d["kind"] == p["kind"]
        assert abs(d["objective"] - p["J"]) <= 1e-9 * p["J"]
        assert d["recomposition_residual"] <= 1e-9
        assert d["lc_axis"] == p["axis"]
        # both searches follow reading R5 and end on the same optimum (to the Nelder-Mead
        # tolerance): H and every executed chirp agree, unconditionally
        assert np.abs(d["h"] - p["h"]).max() < 1e-7, (d["h"], p["h"])
        for qc, qo in zip(d["Q"], _oracle_Q(p)):
            assert np.abs(qc - qo).max() <= 1e-6 * max(1.0, np.abs(qo).max())


def test_fixed_h_reproduces_oracle_chain():
    """With the oracle's H passed in (VARIANT_FIXED_H) the C++ chirps equal the oracle's
    to rounding -- this is how GPU parity pins the discrete operator."""
    r, _ = synth.config_streams(51)
    for _ in range(6):
        M = synth.random_symplectic(r)
        p = opl.plan(M)
        d = nslct.nslct_plan_describe(64, M, h_fixed=p["h"])
        for qc, qo in zip(d["Q"], _oracle_Q(p)):
            assert np.abs(qc - qo).max() <= 1e-12 * max(1.0, np.abs(qo).max())


def test_planner_is_fast():
    import time
    r, _ = synth.config_streams(52)
    M = synth.random_symplectic(r)
    t = time.time()
    for _ in range(5):
        nslct.nslct_plan_describe(4096, M)
    assert (time.time() - t) / 5 < 0.05


def test_inverse_matrix_matches_oracle():
    """nslct.inverse_matrix (the user-facing M^-1 of Eq. CCCMCCCM20) equals the oracle's
    symplectic inverse and inverts M."""
    from oracle import symplectic as sy
    r, _ = synth.config_streams(21)
    for _ in range(3):
        M = synth.random_symplectic(r)
        Mi = nslct.inverse_matrix(M)
        assert np.allclose(Mi, sy.inverse(M), atol=1e-14)
        assert np.allclose(Mi @ M, np.eye(4), atol=1e-12)


def test_ding_plan_describe():
    """Ding plans on the host (no GPU): kind DING, 3 passes, Q0 = B^-1 A and Q4 = D B^-1
    of Eq. Ding12; B = 0 takes the Eq. Intro20 path; a singular B != 0
    has no Ding decomposition."""
    r, _ = synth.config_streams(23)
    M = synth.random_symplectic(r)
    d = nslct.nslct_plan_describe(64, M, variant="DING")
    assert d["kind"] == "DING" and d["n_passes"] == 3 and d["variant"] == "DING"
    A, B, C, D = M[:2, :2], M[:2, 2:], M[2:, :2], M[2:, 2:]
    Bi = np.linalg.inv(B)
    assert np.allclose(d["Q"][0], 0.5 * (Bi @ A + (Bi @ A).T), atol=1e-12)
    assert np.allclose(d["Q"][4], 0.5 * (D @ Bi + (D @ Bi).T), atol=1e-12)
    assert d["recomposition_residual"] < 1e-9
    assert nslct.nslct_plan_describe(64, np.eye(4), variant="DING")["kind"] == "B0"
    # B = [[1, 0], [0, 0]] (rank 1): a valid matrix (free space along x, identity in y)
    Ms = np.eye(4)
    Ms[0, 2] = 1.0
    with pytest.raises(nslct.NslctError) as e:
        nslct.nslct_plan_describe(64, Ms, variant="DING")
    assert e.value.name == "E_NO_DECOMP"
