"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the NsDLCT method itself (no chirps, no
DFTs, no planning): only random-number draws and the construction of valid
ABCD matrices / input fields from them, following the recipe of SURVEY.md
§8(d) and DESIGN.md "Input recipe".  Both `oracle/` and the product package
may import it; it imports neither.
"""
from .generators import *  # noqa: F401,F403
