"""Seeded synthetic inputs for BASELINE.json configs 0-4.

No public dataset is involved: every config is synthetic, and the paper's
datasets (Leukemia, 20newsgroup, RCV1) are not available, so cfg0 only
borrows Leukemia's shape.  The GPU run and the CPU oracle consume the very
same host arrays produced here.

Conventions (discrepancies D5/D6):
  * seeds: ``np.random.default_rng(cfg_index)``; cfg2 blocks use
    ``default_rng([2, block])``; cfg4 problem b uses ``default_rng([4, b])``;
  * AR(1) design along the feature index: x_0 = z_0,
    x_j = rho x_{j-1} + sqrt(1 - rho^2) z_j, then columns centred and
    scaled to unit l2 norm;
  * SNR is the amplitude ratio ||X beta*|| / ||noise|| of the reference's
    own generator (datasets.py:146-151);
  * the gap tolerance is absolute: epsilon = tol * ||y||^2.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class LassoPathCase:
    name: str
    X: object                 # F-ordered ndarray (n, p) or scipy CSC matrix
    y: np.ndarray
    n_lambdas: int
    delta: float              # grid goes from lambda_max to lambda_max / 10**delta
    tol: float                # relative gap tolerance; epsilon = tol * ||y||^2
    beta_star: np.ndarray
    meta: dict

    @property
    def epsilon(self) -> float:
        return float(self.tol * np.dot(self.y, self.y))


def ar1_design(rng, n: int, p: int, corr: float, dtype=np.float64) -> np.ndarray:
    """Gaussian rows with AR(1) correlation along features, centred, unit
    norm columns; returned F-ordered (column j contiguous)."""
    z = rng.standard_normal((p, n))           # row j of z = feature j
    s = np.sqrt(1.0 - corr * corr)
    for j in range(1, p):
        z[j] *= s
        z[j] += corr * z[j - 1]
    z -= z.mean(axis=1, keepdims=True)
    z /= np.sqrt(np.einsum("ij,ij->i", z, z))[:, None]
    return np.asfortranarray(z.T.astype(dtype, copy=False))


def _response(rng, X, beta_star, snr):
    signal = np.asarray(X @ beta_star).ravel()
    noise = rng.standard_normal(signal.size)
    noise *= np.linalg.norm(signal) / (snr * np.linalg.norm(noise))
    return signal + noise


def _support(rng, p, k, values):
    beta = np.zeros(p)
    idx = rng.choice(p, size=k, replace=False)
    if values == "pm1":
        beta[idx] = rng.choice([-1.0, 1.0], size=k)
    else:
        beta[idx] = rng.standard_normal(k)
    return beta


def make_dense_case(name, seed, n, p, corr, k, values, snr, T, delta, tol):
    rng = np.random.default_rng(seed)
    X = ar1_design(rng, n, p, corr)
    beta = _support(rng, p, k, values)
    y = _response(rng, X, beta, snr)
    return LassoPathCase(name, X, y, T, delta, tol, beta,
                         dict(n=n, p=p, ar=corr, k=k, values=values, snr=snr,
                              storage="dense-f64"))


def cfg0(p=7129):
    """configs[0]: 72 x 7129 AR(1) rho=0.5, 20 +-1, SNR 3, 100 lambdas to /1e3."""
    return make_dense_case("cfg0", 0, 72, p, 0.5, 20, "pm1", 3.0, 100, 3.0, 1e-8)


def cfg1(p=100_000, n=1000):
    """configs[1]: 1000 x 100000 AR(1) rho=0.3, 100 N(0,1), SNR 3, 100 lambdas to /1e2."""
    return make_dense_case("cfg1", 1, n, p, 0.3, 100, "normal", 3.0, 100, 2.0, 1e-8)


def cfg2(p=1_000_000, n=10_000, k=500, block=10_000):
    """configs[2]: n x p i.i.d. N(0,1) float32 entries, generated per
    10000-column block with ``default_rng([2, block])``, columns scaled to
    unit norm with float64 norms and stored as float32; 500 +-1
    coefficients; SNR 3 (unstated in BASELINE.json: recorded in ``meta``);
    50 lambdas to lambda_max / 20; tolerance 1e-5.  The full size is a
    40 GB design: tests use a column prefix (``p``), which is the same
    generator's first blocks."""
    X = np.empty((n, p), dtype=np.float32, order="F")
    for b0 in range(0, p, block):
        b1 = min(p, b0 + block)
        Z = np.random.default_rng([2, b0 // block]).standard_normal((b1 - b0, n), dtype=np.float32)
        Zd = Z.astype(np.float64)
        Zd /= np.sqrt(np.einsum("ij,ij->i", Zd, Zd))[:, None]
        X[:, b0:b1] = Zd.T.astype(np.float32)
    rng = np.random.default_rng(2)
    beta = _support(rng, p, min(k, p), "pm1")
    y = _response(rng, X, beta, 3.0)
    return LassoPathCase("cfg2", X, y, 50, float(np.log10(20.0)), 1e-5, beta,
                         dict(n=n, p=p, k=min(k, p), values="pm1", snr=3.0, snr_note="unstated in BASELINE; 3 used",
                              storage="dense-f32"))


def cfg2_block(b: int, n: int = 10_000, block: int = 10_000, width: int | None = None) -> np.ndarray:
    """Columns [b*block, b*block + width) of the cfg2 design: i.i.d. N(0,1)
    float32 draws of ``default_rng([2, b])``, unit norm (float64 norms),
    stored float32, F-ordered (n, width) -- exactly ``cfg2``'s block b."""
    width = block if width is None else width
    Z = np.random.default_rng([2, b]).standard_normal((width, n), dtype=np.float32)
    Zd = Z.astype(np.float64)
    Zd /= np.sqrt(np.einsum("ij,ij->i", Zd, Zd))[:, None]
    return np.asfortranarray(Zd.T.astype(np.float32))


def cfg2_streamed(p=1_000_000, n=10_000, k=500, block=10_000, col_range=None, on_block=None):
    """configs[2] without ever holding the 40 GB design on the host: the
    blocks of ``cfg2`` are generated one at a time; the response is
    y = sum_blocks X_b beta*_b + noise with the block signals accumulated in
    float64 in block order (``cfg2`` itself multiplies the whole matrix at
    once, so the two responses agree to round-off, not bit for bit: this is
    its own seeded instance family, used for the full-size and the
    column-sharded runs).  Returns (X_shard, y, beta*, meta): ``X_shard`` holds
    the columns ``col_range`` (default: none, pass ``on_block(b0, Xb)`` to
    consume the blocks instead, e.g. to upload them)."""
    rng = np.random.default_rng(2)
    beta = _support(rng, p, min(k, p), "pm1")
    lo, hi = (0, 0) if col_range is None else col_range
    Xs = np.empty((n, hi - lo), dtype=np.float32, order="F") if hi > lo else None
    signal = np.zeros(n)
    for b0 in range(0, p, block):
        b1 = min(p, b0 + block)
        Xb = cfg2_block(b0 // block, n, block, b1 - b0)
        nzb = np.flatnonzero(beta[b0:b1])
        if nzb.size:
            signal += Xb[:, nzb].astype(np.float64) @ beta[b0:b1][nzb]
        if hi > lo and b1 > lo and b0 < hi:
            a, z = max(b0, lo), min(b1, hi)
            Xs[:, a - lo:z - lo] = Xb[:, a - b0:z - b0]
        if on_block is not None:
            on_block(b0, Xb)
    noise = rng.standard_normal(n)
    noise *= np.linalg.norm(signal) / (3.0 * np.linalg.norm(noise))
    y = signal + noise
    meta = dict(n=n, p=p, k=min(k, p), values="pm1", snr=3.0, block=block,
                response="block-accumulated signal (cfg2_streamed)", storage="dense-f32")
    return Xs, y, beta, meta


def cfg3(p=1_000_000, n=20_000, nnz_per_col=20):
    """configs[3]: CSC n x p, exactly ``nnz_per_col`` rows per column drawn
    uniformly without replacement, lognormal(0,1) values, unit column norms,
    200 +-1 coefficients, SNR 5, 100 lambdas to /1e2."""
    rng = np.random.default_rng(3)
    # per-column uniform sample of distinct rows: draw, then redraw the
    # (rare) columns that contain a repeated row
    rows = rng.integers(0, n, size=(p, nnz_per_col), dtype=np.int64)
    while True:
        srt = np.sort(rows, axis=1)
        bad = np.flatnonzero(np.any(srt[:, 1:] == srt[:, :-1], axis=1))
        if bad.size == 0:
            break
        rows[bad] = rng.integers(0, n, size=(bad.size, nnz_per_col), dtype=np.int64)
    rows = rows.astype(np.int32)
    rows.sort(axis=1)
    vals = rng.lognormal(0.0, 1.0, size=(p, nnz_per_col))
    vals /= np.sqrt(np.einsum("ij,ij->i", vals, vals))[:, None]
    indptr = np.arange(0, (p + 1) * nnz_per_col, nnz_per_col, dtype=np.int64)
    X = sp.csc_matrix((vals.ravel(), rows.ravel(), indptr), shape=(n, p))
    beta = _support(rng, p, 200, "pm1")
    y = _response(rng, X, beta, 5.0)
    return LassoPathCase("cfg3", X, y, 100, 2.0, 1e-8, beta,
                         dict(n=n, p=p, nnz_per_col=nnz_per_col, k=200, values="pm1",
                              snr=5.0, storage="csc-f64"))


def cfg4_shared(n0=1000, p=50_000):
    """Shared design of configs[4]: 1000 x 50000 AR(1) rho=0.5, centred,
    unit-norm columns; y0 from 50 +-1 coefficients at SNR 3."""
    rng = np.random.default_rng(4)
    X0 = ar1_design(rng, n0, p, 0.5)
    beta = _support(rng, p, 50, "pm1")
    y0 = _response(rng, X0, beta, 3.0)
    return X0, y0, beta


def cfg4_rows(b: int, n0: int = 1000, n: int = 500) -> np.ndarray:
    """Bootstrap rows of problem b (with replacement)."""
    return np.random.default_rng([4, b]).integers(0, n0, n)


def by_name(name: str, **kw) -> LassoPathCase:
    return {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3}[name](**kw)
