"""Kernel-level parity of the sm_100a kernels against the CPU oracle
(oracle/kernels.c == reference numba kernels, _kernels.py:14-92).

Exact-order twins must match bit for bit; production kernels (FMA,
CTA-parallel reductions, certified-zero skipping) within fp64 round-off.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gapsafe_oracle as O

gs = pytest.importorskip("paper_1505_03410_b200")
pytestmark = pytest.mark.gpu


def _dense(seed, n, p, dtype=np.float64):
    rng = np.random.default_rng(seed)
    X = np.asfortranarray(rng.standard_normal((n, p)).astype(dtype))
    return X, rng


def _csc(seed, n, p, density):
    rng = np.random.default_rng(seed)
    X = sp.random(n, p, density=density, random_state=np.random.RandomState(seed), format="csc",
                  data_rvs=lambda k: np.random.RandomState(seed + 1).lognormal(size=k))
    X.sort_indices()
    return X, rng


@pytest.mark.parametrize("n,p", [(1, 1), (7, 13), (72, 300), (1000, 257), (4096, 40)])
def test_tdot_exact_order_bitwise(n, p):
    X, rng = _dense(n * 31 + p, n, p)
    v = rng.standard_normal(n)
    cols = rng.permutation(p)[: max(1, p // 2)].astype(np.int64)
    ref = np.empty(cols.size)
    O.tdot_dense(X, v, cols, 0.0, ref)
    D = gs.DesignMatrix(X)
    out = D.transpose_dot(v, cols, exact_order=True)
    assert np.array_equal(out, ref)


def test_tdot_exact_order_bitwise_f32_storage():
    X32, rng = _dense(5, 333, 91, np.float32)
    v = rng.standard_normal(333)
    cols = np.arange(91, dtype=np.int64)
    ref = np.empty(91)
    O.tdot_dense(np.asfortranarray(X32.astype(np.float64)), v, cols, 0.0, ref)
    out = gs.DesignMatrix(X32).transpose_dot(v, cols, exact_order=True)
    assert np.array_equal(out, ref)


def test_tdot_exact_order_bitwise_csc():
    X, rng = _csc(3, 500, 400, 0.05)
    v = rng.standard_normal(500)
    cols = np.arange(400, dtype=np.int64)[::3].copy()
    ref = np.empty(cols.size)
    O.tdot_csc(X.data, X.indices, X.indptr, 500, v, cols, 0.0, ref)
    out = gs.DesignMatrix(X).transpose_dot(v, cols, exact_order=True)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("n,p", [(72, 500), (1000, 300), (1, 5), (33, 7)])
def test_tdot_fast_close(n, p):
    X, rng = _dense(n + 7 * p, n, p)
    v = rng.standard_normal(n)
    D = gs.DesignMatrix(X)
    full = D.transpose_dot(v)
    ref = X.T @ v
    bound = 4 * (n + 2) * 2.0 ** -53 * (np.abs(X).T @ np.abs(v))
    assert np.all(np.abs(full - ref) <= bound + 1e-300)
    cols = np.arange(p, dtype=np.int64)[::2].copy()
    np.testing.assert_array_equal(D.transpose_dot(v, cols), full[cols])


@pytest.mark.parametrize("n,p,lam_frac", [(72, 400, 0.3), (1000, 200, 0.1), (20, 50, 0.05),
                                          (500, 123, 0.5)])
def test_cd_pass_exact_order_bitwise(n, p, lam_frac):
    X, rng = _dense(11 * n + p, n, p)
    y = rng.standard_normal(n)
    nsq = np.einsum("ij,ij->j", X, X)
    lam = lam_frac * np.max(np.abs(X.T @ y))
    active = np.sort(rng.choice(p, size=p * 3 // 4, replace=False)).astype(np.int64)
    b_ref, r_ref = np.zeros(p), y.copy()
    b_gpu, r_gpu = np.zeros(p), y.copy()
    D = gs.DesignMatrix(X)
    lib = D._lib
    from paper_1505_03410_b200 import _lib
    for _ in range(6):
        O.cd_pass_dense(X, b_ref, r_ref, active, lam, nsq, 0.0)
        _lib.check(lib.gs_cd_pass(D.handle, _lib.f64p(b_gpu), _lib.f64p(r_gpu), _lib.i64p(active),
                                  active.size, lam, _lib.f64p(nsq), 0.0, 1))
        assert np.array_equal(b_gpu, b_ref)
        assert np.array_equal(r_gpu, r_ref)


def test_cd_pass_exact_order_bitwise_csc():
    X, rng = _csc(9, 400, 300, 0.04)
    y = rng.standard_normal(400)
    nsq = np.asarray(X.multiply(X).sum(axis=0)).ravel()
    keep = np.flatnonzero(nsq > 0).astype(np.int64)
    lam = 0.2 * np.max(np.abs(X.T @ y))
    b_ref, r_ref = np.zeros(300), y.copy()
    b_gpu, r_gpu = np.zeros(300), y.copy()
    D = gs.DesignMatrix(X)
    from paper_1505_03410_b200 import _lib
    for _ in range(5):
        O.cd_pass_csc(X.data, X.indices, X.indptr, 400, b_ref, r_ref, keep, lam, nsq, 0.0)
        _lib.check(D._lib.gs_cd_pass(D.handle, _lib.f64p(b_gpu), _lib.f64p(r_gpu), _lib.i64p(keep),
                                     keep.size, lam, _lib.f64p(nsq), 0.0, 1))
    assert np.array_equal(b_gpu, b_ref)
    assert np.array_equal(r_gpu, r_ref)


@pytest.mark.parametrize("n,p,lam_frac", [(72, 700, 0.1), (1000, 400, 0.05), (300, 300, 0.02),
                                          (1024, 60, 0.1), (130, 90, 0.3)])
def test_cd_pass_production_close(n, p, lam_frac):
    """Production epoch (certified skipping, CTA reductions) tracks the
    sequential reference to round-off; supports agree."""
    X, rng = _dense(3 * n + p, n, p)
    X /= np.linalg.norm(X, axis=0)
    X = np.asfortranarray(X)
    y = rng.standard_normal(n)
    nsq = np.einsum("ij,ij->j", X, X)
    lam = lam_frac * np.max(np.abs(X.T @ y))
    active = np.arange(p, dtype=np.int64)
    b_ref, r_ref = np.zeros(p), y.copy()
    D = gs.DesignMatrix(X)
    st = gs.SolverState(beta=np.zeros(p), residual=y.copy(), active=active, theta=None, cert=None,
                        passes_done=0, converged=False)
    prob = gs.LassoProblem(D, y, lam)
    for _ in range(8):
        O.cd_pass_dense(X, b_ref, r_ref, active, lam, nsq, 0.0)
        gs.cd_pass(st, prob)
    assert np.array_equal(np.flatnonzero(st.beta), np.flatnonzero(b_ref))
    np.testing.assert_allclose(st.beta, b_ref, rtol=0, atol=1e-11 * max(1, np.abs(b_ref).max()))
    np.testing.assert_allclose(st.residual, r_ref, rtol=0, atol=1e-11 * np.abs(y).max())


def test_cd_pass_production_csc_close():
    X, rng = _csc(21, 2000, 3000, 0.01)
    X = sp.csc_matrix(X @ sp.diags(1.0 / np.maximum(np.sqrt(np.asarray(X.multiply(X).sum(0)).ravel()), 1e-300)))
    y = rng.standard_normal(2000)
    D = gs.DesignMatrix(X)
    nsq = np.asarray(X.multiply(X).sum(axis=0)).ravel()
    active = np.flatnonzero(nsq > 0).astype(np.int64)
    lam = 0.05 * np.max(np.abs(X.T @ y))
    b_ref, r_ref = np.zeros(3000), y.copy()
    st = gs.SolverState(beta=np.zeros(3000), residual=y.copy(), active=active, theta=None, cert=None,
                        passes_done=0, converged=False)
    prob = gs.LassoProblem(D, y, lam)
    for _ in range(5):
        O.cd_pass_csc(X.data, X.indices, X.indptr, 2000, b_ref, r_ref, active, lam, nsq, 0.0)
        gs.cd_pass(st, prob)
    assert np.array_equal(np.flatnonzero(st.beta), np.flatnonzero(b_ref))
    np.testing.assert_allclose(st.beta, b_ref, rtol=0, atol=1e-11)


def test_matvec_axpy_maxcorr():
    X, rng = _dense(17, 64, 90)
    D = gs.DesignMatrix(X)
    beta = np.zeros(90)
    beta[[3, 17, 40]] = [1.5, -2.0, 0.25]
    np.testing.assert_allclose(D.matvec(beta), X @ beta, rtol=1e-14, atol=1e-14)
    v = rng.standard_normal(64)
    w = v.copy()
    D.axpy_col(17, 0.7, w)
    ref = v.copy()
    ref[:] += 0.7 * X[:, 17]
    assert np.array_equal(w, ref)                     # elementwise, separate roundings
    val, j = D.max_abs_correlation(v)
    c = np.abs(X.T @ v)
    assert j == int(np.argmax(c)) and val == pytest.approx(c.max(), rel=1e-13)
    with pytest.raises(IndexError):
        D.col_dot(90, v)
    with pytest.raises(ValueError):
        D.max_abs_correlation(v, restrict=np.array([], dtype=np.int64))


def test_max_abs_correlation_tie_smallest_index():
    D = gs.DesignMatrix(np.eye(3))
    assert D.max_abs_correlation(np.ones(3))[1] == 0


@pytest.mark.parametrize("sparse", [False, True])
def test_screen_matches_oracle(sparse):
    rng = np.random.default_rng(8)
    n, p = 60, 2000
    if sparse:
        Xh = sp.random(n, p, density=0.1, random_state=np.random.RandomState(8), format="csc")
    else:
        Xh = np.asfortranarray(rng.standard_normal((n, p)))
    D, Dor = gs.DesignMatrix(Xh), O.DesignMatrix(Xh)
    c = rng.standard_normal(n) * 0.05
    for r in (0.0, 0.01, 0.1):
        a = gs.screen(gs.Sphere(center=c, radius=r), D)
        b = O.screen(O.Sphere(center=c, radius=r), Dor)
        # identical masks except features within 1e-10 of the threshold
        near = np.abs(b.mu - (1 - gs.SCREEN_SAFETY)) <= 1e-10
        diff = np.setxor1d(a.active_set, b.active_set)
        assert np.all(near[diff])
        np.testing.assert_allclose(a.mu, b.mu, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("n", [40, 72, 200, 384, 640, 1000, 1500])
def test_cd_pipeline_stress(n):
    """Many epochs of the warp-specialized CD (all warp-group sizes and ring
    depths, several active-set sizes incl. multi-tile) against the sequential
    reference; a protocol hang would trip the device watchdog and raise."""
    rng = np.random.default_rng(n)
    p = 9000 if n <= 72 else 2500
    X = np.asfortranarray(rng.standard_normal((n, p)))
    X /= np.linalg.norm(X, axis=0)
    X = np.asfortranarray(X)
    y = X[:, :12] @ rng.standard_normal(12) + 0.1 * rng.standard_normal(n)
    nsq = np.einsum("ij,ij->j", X, X)
    D = gs.DesignMatrix(X)
    for lam_frac in (0.5, 0.1, 0.02):
        lam = lam_frac * np.max(np.abs(X.T @ y))
        active = np.arange(p, dtype=np.int64)
        b_ref, r_ref = np.zeros(p), y.copy()
        st = gs.SolverState(beta=np.zeros(p), residual=y.copy(), active=active, theta=None, cert=None,
                            passes_done=0, converged=False)
        prob = gs.LassoProblem(D, y, lam)
        for _ in range(4):
            O.cd_pass_dense(X, b_ref, r_ref, active, lam, nsq, 0.0)
            gs.cd_pass(st, prob)
        assert np.array_equal(np.flatnonzero(st.beta), np.flatnonzero(b_ref))
        np.testing.assert_allclose(st.beta, b_ref, rtol=0, atol=1e-10 * max(1, np.abs(b_ref).max()))


def _fused_screen_case(kind):
    rng = np.random.default_rng(21)
    if kind == "dense_f64_wide":          # 4096 x 8 B = 32 KB columns: whole-CTA column reduction
        n, p = 4096, 900
        Xh = np.asfortranarray(rng.standard_normal((n, p)) / np.sqrt(n))
    elif kind == "dense_f32_wide":        # cfg2's column shape: 10000 x 4 B = 40 KB
        n, p = 10_000, 700
        Xh = np.asfortranarray((rng.standard_normal((n, p)) / np.sqrt(n)).astype(np.float32))
    elif kind == "dense_f32_odd_wide":    # wide with a ragged last vector per thread
        n, p = 5003, 450
        Xh = np.asfortranarray((rng.standard_normal((n, p)) / np.sqrt(n)).astype(np.float32))
    elif kind == "dense_f64_staged":      # cfg1's column shape (TMA-staged warp-per-column form)
        n, p = 1000, 3000
        Xh = np.asfortranarray(rng.standard_normal((n, p)) / np.sqrt(n))
    elif kind == "csc_short":             # cfg3's column shape: 20 nonzeros per column
        n, p = 20_000, 6000
        idx = np.concatenate([np.sort(rng.choice(n, 20, replace=False)) for _ in range(p)])
        Xh = sp.csc_matrix((rng.lognormal(size=20 * p) / np.sqrt(20.0), idx, np.arange(0, 20 * p + 1, 20)),
                           shape=(n, p))
    elif kind == "csc_short_ragged":      # 0 .. 40 nonzeros per column, some empty, some past the unrolled trips
        n, p = 3000, 5000
        lens = rng.integers(0, 41, p)
        lens[::97] = 0
        idx = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens] + [np.empty(0, np.int64)])
        ptr = np.concatenate([[0], np.cumsum(lens)])
        Xh = sp.csc_matrix((rng.lognormal(size=int(ptr[-1])) / 4.0, idx.astype(np.int32), ptr), shape=(n, p))
    else:                                 # long CSC columns: warp-per-column form
        n, p = 2000, 1200
        Xh = sp.random(n, p, density=0.05, random_state=np.random.RandomState(3), format="csc")
        Xh.sort_indices()
    return Xh, rng


@pytest.mark.parametrize("kind", ["dense_f64_wide", "dense_f32_wide", "dense_f32_odd_wide", "dense_f64_staged",
                                  "csc_short", "csc_short_ragged", "csc_long"])
def test_fused_screen_pass_matches_oracle(kind):
    """The persistent kernel's fused full-p screening pass (group_gemv G_MU in
    each of its GEMV forms) keeps exactly the oracle's survivors, except
    features within 1e-10 of the 1 - 1e-9 threshold (regions.py:129-139)."""
    Xh, rng = _fused_screen_case(kind)
    X64 = Xh.astype(np.float64) if not sp.issparse(Xh) else Xh
    D = gs.DesignMatrix(Xh)
    Dor = O.DesignMatrix(np.asfortranarray(X64) if not sp.issparse(Xh) else X64)
    n = Xh.shape[0]
    y = rng.standard_normal(n)
    lmax, _ = Dor.max_abs_correlation(y)
    c = y / lmax
    for r in (0.0, 0.02, 0.2):
        b = O.screen(O.Sphere(center=c, radius=r), Dor)
        a = gs.PathTimer.screen_pass_active(D, c, r)
        near = np.abs(b.mu - (1 - gs.SCREEN_SAFETY)) <= 1e-10
        diff = np.setxor1d(a, b.active_set)
        assert np.all(near[diff]), (kind, r, diff[:5])
        assert a.size > 0 or b.active_set.size == 0


def test_design_constructors_blockwise_and_device():
    """Block-wise upload (designs larger than a host array), the device-buffer
    constructor (columns received over NCCL) and the device column gather give
    the same design as the host-array constructor."""
    torch = pytest.importorskip("torch")
    for dtype in (np.float64, np.float32):
        X, rng = _dense(31, 130, 700, dtype)
        v = rng.standard_normal(130)
        D = gs.DesignMatrix(X)
        blocks = ((j0, X[:, j0:j0 + 256]) for j0 in range(0, 700, 256))
        Db = gs.DesignMatrix.from_blocks(130, 700, dtype, blocks)
        assert np.array_equal(Db.col_norms_sq, D.col_norms_sq)
        assert np.array_equal(Db.transpose_dot(v), D.transpose_dot(v))
        assert Db.max_abs_correlation(v) == D.max_abs_correlation(v)
        idx = np.array([699, 0, 17, 17, 345], dtype=np.int64)
        assert np.array_equal(D.columns_to_host(idx), X[:, idx])
        # device buffer -> design: the gathered columns as a (k, n) CUDA tensor
        tdt = torch.float32 if dtype == np.float32 else torch.float64
        buf = torch.empty((idx.size, 130), dtype=tdt, device="cuda")
        D.gather_columns_to_device(idx, buf.data_ptr(), 130)
        torch.cuda.synchronize()
        Dd = gs.DesignMatrix.from_device(buf.data_ptr(), 130, idx.size, 130, dtype)
        ref = gs.DesignMatrix(np.asfortranarray(X[:, idx]))
        assert np.array_equal(Dd.col_norms_sq, ref.col_norms_sq)
        assert np.array_equal(Dd.transpose_dot(v), ref.transpose_dot(v))
        with pytest.raises(ValueError):
            Dd.toarray()
    with pytest.raises(IndexError):
        D.columns_to_host(np.array([700], dtype=np.int64))
