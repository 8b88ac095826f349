"""Seeded initial states (inputs only).

Recipe: numpy PCG64(seed), re and im drawn from standard_normal,
normalised in fp64 (SURVEY 8(c) comparison procedure step 1).  For complex64 runs the
state is rounded to complex64 first and the rounded values are what both sides get.
"""

from __future__ import annotations

import numpy as np


def random_state(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    d = 1 << n
    psi = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    psi /= np.sqrt(np.sum(np.abs(psi) ** 2))
    return psi.astype(np.complex128)


def round_to_c64(psi: np.ndarray) -> np.ndarray:
    """Round to complex64 and return the up-cast complex128 copy both sides consume."""
    return psi.astype(np.complex64).astype(np.complex128)
