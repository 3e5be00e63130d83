"""Parity helpers shared by the GPU tests (no estimator arithmetic: error measures only).

Two bars, both against the complex128 oracle on the same seeded inputs:
- north_star's per-instance relative Frobenius error <= 1e-4;
- a row-level bar on top of it: for every (instance t, antenna m, user k, window w) the kept output segment
  h[t, m, k, o_w:o_{w+1}] must be within 1e-3 relative error of the oracle's.  A per-instance norm dilutes a
  localised fault (one wrong edge-window row of config 3 at 1e-3 reads ~3e-5 per instance); the row bar does not.
"""
from __future__ import annotations

import numpy as np

import oracle

TOL = 1e-4
ROW_TOL = 1e-3


def row_rel_err_max(h: np.ndarray, ref: np.ndarray, N: int, b: int, s: int) -> float:
    """max over (t, m, k, window) of ||h_seg - ref_seg|| / ||ref_seg|| (segments with a zero reference skipped)."""
    h = np.asarray(h).astype(np.complex128)
    ref = np.asarray(ref)
    worst = 0.0
    for (_a, o, o1) in oracle.window_table(N, b, s):
        d = np.linalg.norm(h[..., o:o1] - ref[..., o:o1], axis=-1)
        n = np.linalg.norm(ref[..., o:o1], axis=-1)
        ok = n > 0
        if ok.any():
            worst = max(worst, float((d[ok] / n[ok]).max()))
        if (~ok).any() and d[~ok].max() > 0:      # zero reference segment: the estimate must be zero too
            worst = float("inf")
    return worst


def assert_parity(h: np.ndarray, ref: np.ndarray, N: int, b: int, s: int, tol: float = TOL,
                  row_tol: float = ROW_TOL):
    """Both bars; returns (per-instance errors, worst row error)."""
    err = oracle.rel_fro_error_per_instance(h, ref)
    assert np.all(err <= tol), f"per-instance rel Frobenius error {err.max():.3e} > {tol}"
    row = row_rel_err_max(h, ref, N, b, s)
    assert row <= row_tol, f"worst row (t, m, k, window) rel error {row:.3e} > {row_tol}"
    assert np.isfinite(h).all()
    return err, row
