"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This package holds NO arithmetic of the simulation method (no gate
application, no readout): it only writes circuits in the IR text format and
draws seeded initial states.  Both the CPU oracle (``oracle/``) and the CUDA
path (``paper_2106_13995_b200``) consume what it produces; neither imports
the other.

* ``circuits``  -- supremacy-style grids,
  reversible shift-and-add multipliers,
  QFT, random circuits over the full gate set, inverse ("mirror") circuits,
  and the IR text writer.
* ``states``    -- seeded random normalised complex states and basis inputs.
"""

from .circuits import (  # noqa: F401
    Circuit,
    GateSpec,
    supremacy,
    multiplier,
    qft,
    random_circuit,
    inverse,
    concat,
    basis_prep,
    to_text,
    gate_count,
    remove_random_qubit,
    width_sweep,
    family_at_width,
    supremacy_grid,
    random_unitary,
)
from .states import random_state, round_to_c64  # noqa: F401
