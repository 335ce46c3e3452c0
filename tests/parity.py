"""Parity comparators between the B200 path and the CPU oracle.

Criteria (BASELINE.json north_star):
  * per-lambda epoch counts identical;
  * per-checkpoint active-set sizes identical, final active sets and supports
    identical;
  * coefficients: max|d beta| <= 1e-8 * max(1, max|beta|)  (fp64);
  * duality gaps: |d G| <= 1e-8 |G| + 64 u ||y||^2  (u = 2^-53; the gap is
    cancellation-limited at G ~ eps).
"""

from __future__ import annotations

import numpy as np

U = 2.0 ** -53


def gap_close(g_gpu: float, g_ref: float, y_norm_sq: float, rel: float = 1e-8) -> bool:
    return abs(g_gpu - g_ref) <= rel * abs(g_ref) + 64 * U * y_norm_sq


def beta_close(b_gpu, b_ref, rel: float = 1e-8) -> bool:
    scale = max(1.0, float(np.max(np.abs(b_ref))) if b_ref.size else 1.0)
    return float(np.max(np.abs(b_gpu - b_ref))) <= rel * scale if b_ref.size else True


def compare_states(a, b, y_norm_sq: float, rel: float = 1e-8, where: str = ""):
    """a: GPU SolverState, b: oracle SolverState."""
    assert a.passes_done == b.passes_done, f"{where}: epochs {a.passes_done} vs {b.passes_done}"
    assert a.converged == b.converged, f"{where}: converged {a.converged} vs {b.converged}"
    assert len(a.screen_trace) == len(b.screen_trace), f"{where}: checkpoints differ"
    for k, (ra, rb) in enumerate(zip(a.screen_trace, b.screen_trace)):
        assert ra[0] == rb[0], f"{where}: trace passes row {k}: {ra} vs {rb}"
        assert ra[1] == rb[1], f"{where}: trace |A| row {k}: {ra} vs {rb}"
        assert gap_close(ra[2], rb[2], y_norm_sq, rel), f"{where}: trace gap row {k}: {ra} vs {rb}"
    assert np.array_equal(a.active, b.active), f"{where}: final active sets differ"
    assert np.array_equal(np.flatnonzero(a.beta), np.flatnonzero(b.beta)), f"{where}: supports differ"
    assert beta_close(a.beta, b.beta, rel), \
        f"{where}: beta max diff {np.max(np.abs(a.beta - b.beta))}"
    assert gap_close(a.cert.gap, b.cert.gap, y_norm_sq, rel), \
        f"{where}: gap {a.cert.gap} vs {b.cert.gap}"


def compare_paths(ra, rb, y_norm_sq: float, rel: float = 1e-8):
    assert len(ra.states) == len(rb.states)
    for t, (a, b) in enumerate(zip(ra.states, rb.states)):
        compare_states(a, b, y_norm_sq, rel, where=f"lambda[{t}]")
    assert np.array_equal(ra.converged, rb.converged)
