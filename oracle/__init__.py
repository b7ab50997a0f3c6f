"""fp64 CPU oracle for the randomized Tucker/HOSVD hot path.

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline and ``--impl reference`` legs).  The product package
``paper_2001_07124_b200`` never imports, links or executes anything here, and the
oracle shares no code with the CUDA path (only ``gen.synth`` inputs are shared).

Every function cites the PAPER.md passage it follows.  Pins: tests/test_oracle_pins.py.
Parity unpinned (no closed form; only the oracle defines them): the exact E,
factors and cores of cfg2-cfg5.
"""
from .rtucker import *  # noqa: F401,F403
from .tensor import fold, fro, multi_ttm, reconstruct, ttm, unfold  # noqa: F401
