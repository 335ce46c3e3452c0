"""Parity comparators between the B200 path and the CPU oracle.

Criteria (BASELINE.json north_star):
  * per-lambda epoch counts identical;
  * per-checkpoint active-set sizes identical (and the sets themselves, element
    by element, when both runs tracked them), final active sets and supports
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
    if getattr(a, "active_history", None) and getattr(b, "active_history", None):
        # per-checkpoint active sets, element by element (track_active runs)
        assert len(a.active_history) == len(b.active_history), f"{where}: checkpoint count"
        for k, (ha, hb) in enumerate(zip(a.active_history, b.active_history)):
            assert np.array_equal(np.asarray(ha), np.asarray(hb)), f"{where}: active set at checkpoint {k}"
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


def path_report(ra, rb, y_norm_sq: float, rel: float = 1e-8) -> dict:
    """Non-raising summary of ``compare_paths`` over the common prefix of two
    paths (bench.py's parity block)."""
    k = min(len(ra.states), len(rb.states))
    out = {"lambdas_compared": k, "epochs_equal": True, "checkpoints_equal": True,
           "active_sets_equal": True, "supports_equal": True, "max_beta_rel": 0.0,
           "gaps_within_tol": True, "first_mismatch": None}
    for t in range(k):
        a, b = ra.states[t], rb.states[t]
        try:
            compare_states(a, b, y_norm_sq, rel, where=f"lambda[{t}]")
        except AssertionError as e:
            if out["first_mismatch"] is None:
                out["first_mismatch"] = str(e)[:300]
        out["epochs_equal"] &= a.passes_done == b.passes_done
        ta = [(r[0], r[1]) for r in a.screen_trace]
        tb = [(r[0], r[1]) for r in b.screen_trace]
        out["checkpoints_equal"] &= ta == tb
        ha_, hb_ = getattr(a, "active_history", []), getattr(b, "active_history", [])
        hist = (len(ha_) == len(hb_)
                and all(np.array_equal(np.asarray(x), np.asarray(z))
                        for x, z in zip(ha_, hb_)))
        out["active_sets_equal"] &= bool(hist and np.array_equal(a.active, b.active))
        out["supports_equal"] &= bool(np.array_equal(np.flatnonzero(a.beta), np.flatnonzero(b.beta)))
        scale = max(1.0, float(np.max(np.abs(b.beta))) if b.beta.size else 1.0)
        d = float(np.max(np.abs(a.beta - b.beta))) / scale if b.beta.size else 0.0
        out["max_beta_rel"] = max(out["max_beta_rel"], d)
        out["gaps_within_tol"] &= bool(gap_close(a.cert.gap, b.cert.gap, y_norm_sq, rel)
                                       and all(gap_close(x[2], z[2], y_norm_sq, rel)
                                               for x, z in zip(a.screen_trace, b.screen_trace)))
    out["ok"] = out["first_mismatch"] is None and k > 0
    return out
