"""fp64 CPU oracle for the 2D NsDLCT of arxiv 1707.03688.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything
under `oracle/`.  The product path (`paper_1707_03688_b200`, `libnslct.so`)
never imports, calls or links it, and the oracle shares no code, tables or
constants with the CUDA path: it is written from PAPER.md directly.

Modules
  symplectic  -- ABCD algebra: validity (Eq. Intro12), inverse (Eq. CCCMCCCM20),
                 composition, symplectic polar projection (reading R6).
  planner     -- decomposition planning: CM-CC-CM-CC (Eq. Bnonsym08), HA objective
                 (Eq. HA16/HA24), LC rule (Eq. LC08/LC10), CC-CM-CC-CM (Eq.
                 CCCMCCCM08-16), reversible dispatch (Eq. Reversible08 + reading R7).
  operators   -- the discrete operators: CM (Eq. BasicCM12), DFT/IDFT (Eq.
                 BasicDFT16, exact inverse per reading R3), CC (Eq. BasicCC20),
                 bilinear affine (Eq. BasicAffine12/16), B=0 case (Eq. Intro20),
                 and O_plan = the full HA/LC NsDLCT (Eq. HA28 / LC12 / CCCMCCCM40/44).
  direct      -- the direct method O_direct (Eq. Intro32), O(N^4).
  closed_form -- Hermite-Gaussian inputs (Eq. Acc12/16) and the Gaussian-beam
                 closed form of the continuous NsLCT (derived from Eq. Intro08).
  metrics     -- NMSE (Eq. Acc04 / Add16 / Rev08), relative L2, PSNR.
  ding        -- Ding's NsDLCT (Eq. Ding12), the paper's comparison system (row F4).

Parity status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py except where its docstring says "parity unpinned"
(see DESIGN.md "Oracle pins").
"""
from . import symplectic, planner, operators, direct, closed_form, metrics, ding  # noqa: F401
