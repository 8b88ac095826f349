"""Comparison helpers (SURVEY 8(c) comparison procedure; EquivalenceReport S:335-339 extended)."""

import numpy as np

U_C64 = 2.0 ** -24
U_C128 = 2.0 ** -53


def report(got: np.ndarray, ref: np.ndarray) -> dict:
    d = np.abs(got.astype(np.complex128) - ref)
    worst = int(np.argmax(d))  # lowest index among equal maxima (R19)
    l2 = float(np.sqrt(np.sum(d * d)))
    fid = float(abs(np.vdot(got.astype(np.complex128), ref)) ** 2)
    return {"max_abs": float(d[worst]), "worst_index": worst, "l2": l2, "fidelity": fid}


def assert_close(got, ref, dtype: str, ngates: int, tol_c64=1e-4, tol_c128=1e-10):
    """Tolerances: north_star max|d| <= 1e-10 (c128) / 1e-4 (c64), plus the scale-free
    ||d||_2 <= 8 G u bound of reading R9 (u = unit roundoff of the state dtype)."""
    r = report(got, ref)
    u = U_C64 if dtype == "c64" else U_C128
    tol = tol_c64 if dtype == "c64" else tol_c128
    assert r["max_abs"] <= tol, r
    assert r["l2"] <= 8 * max(ngates, 1) * u + (4 * u if dtype == "c64" else 0), r
    return r
