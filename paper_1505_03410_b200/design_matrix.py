"""Device-resident design matrix (drop-in for gapsafe.design_matrix.DesignMatrix,
/root/reference/pkg/src/gapsafe/design_matrix.py:22-187).

Storage is uploaded once to HBM: dense input as column-major fp64 (or fp32
storage with fp64 arithmetic, for float32 inputs), sparse input as canonical
CSC (sorted, deduplicated; design_matrix.py:37-43) plus a CSR copy for the
row-parallel residual resync.  Column norms are computed on the device.  Every
method runs a CUDA kernel through the C ABI; host arrays are only the
caller's inputs and outputs.

Elastic-Net tail (design_matrix.py:54-65,100-158): with
``tail_weight > 0`` the reference keeps the rows ``sqrt(tail_weight) I_p``
implicit.  Here they are stored: the device copy is the CSC of
``[X; sqrt(w) I_p]`` (one extra entry per column, row ``n_base + j``, last in
its column since indices are sorted), so every device kernel -- the products,
the persistent solve, the sparse CD waves -- runs unchanged on the augmented
problem.  The tail entry is the last term of each column's sequential sum,
which is the reference's order (``s += tail_scale * v[n_base + j]`` after the
base dot, _kernels.py tdot_*/cd_pass_*).  Column norms are the reference's
``base_sq + tail_weight`` (:56), passed to the device, not recomputed.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _lib


class DesignMatrix:
    """n x p feature matrix with cached per-column Euclidean norms."""

    def __init__(self, storage, tail_weight: float = 0.0):
        if tail_weight < 0:
            raise ValueError("tail_weight must be non-negative")
        lib = _lib.load()
        handle = ctypes.c_void_p()
        if sp.issparse(storage):
            mat = sp.csc_matrix(storage).astype(np.float64)
            mat.sum_duplicates()
            mat.sort_indices()
            self._mat = mat
            self.is_sparse = True
            self.n_base, self.n_cols = mat.shape
            if self.n_base < 1 or self.n_cols < 1:
                raise ValueError("matrix must have at least one row and column")
            self._indptr64 = np.ascontiguousarray(mat.indptr, dtype=np.int64)
            data = np.ascontiguousarray(mat.data, dtype=np.float64)
            indices = np.ascontiguousarray(mat.indices, dtype=np.int32)
            _lib.check(lib.gs_matrix_csc(_lib.f64p(data), _lib.i32p(indices), _lib.i64p(self._indptr64),
                                         self.n_base, self.n_cols, None, ctypes.byref(handle)))
            self.dtype = np.float64
        else:
            arr = np.asarray(storage)
            if arr.dtype != np.float32:
                arr = np.asarray(arr, dtype=np.float64)
            arr = np.asfortranarray(arr)
            if arr.ndim != 2:
                raise ValueError("storage must be 2-dimensional")
            self._mat = arr
            self.is_sparse = False
            self.n_base, self.n_cols = arr.shape
            if self.n_base < 1 or self.n_cols < 1:
                raise ValueError("matrix must have at least one row and column")
            self.dtype = arr.dtype.type
            dt = _lib.GS_DTYPE_F32 if arr.dtype == np.float32 else _lib.GS_DTYPE_F64
            _lib.check(lib.gs_matrix_dense(arr.ctypes.data_as(ctypes.c_void_p), dt, self.n_base,
                                           self.n_cols, self.n_base, None, ctypes.byref(handle)))
        self._h = handle
        self._lib = lib
        self.tail_weight = float(tail_weight)
        self.tail_scale = float(np.sqrt(tail_weight))
        nsq = np.empty(self.n_cols, dtype=np.float64)
        _lib.check(lib.gs_matrix_norms_sq(self._h, _lib.f64p(nsq)))
        if self.tail_weight > 0.0:
            nsq = nsq + self.tail_weight                          # design_matrix.py:56
            self._h = self._upload_augmented(nsq)
            lib.gs_matrix_free(handle)
            self.dtype = np.float64
        self._col_norms_sq = nsq
        self._col_norms = np.sqrt(nsq)

    def _upload_augmented(self, nsq: np.ndarray) -> ctypes.c_void_p:
        """Device CSC of [X; tail_scale I_p] with the reference's norms."""
        base = self._mat if self.is_sparse else sp.csc_matrix(np.asarray(self._mat, dtype=np.float64))
        tail = sp.identity(self.n_cols, dtype=np.float64, format="csc") * self.tail_scale
        aug = sp.vstack([base, tail], format="csc")
        aug.sort_indices()
        self._aug_indptr64 = np.ascontiguousarray(aug.indptr, dtype=np.int64)
        data = np.ascontiguousarray(aug.data, dtype=np.float64)
        indices = np.ascontiguousarray(aug.indices, dtype=np.int32)
        handle = ctypes.c_void_p()
        _lib.check(self._lib.gs_matrix_csc(_lib.f64p(data), _lib.i32p(indices), _lib.i64p(self._aug_indptr64),
                                           self.n_base + self.n_cols, self.n_cols, _lib.f64p(nsq),
                                           ctypes.byref(handle)))
        return handle

    @classmethod
    def from_device(cls, dev_ptr: int, n: int, p: int, ld: int, dtype) -> "DesignMatrix":
        """Dense design from a device buffer (column j at ``dev_ptr + j*ld``
        elements): device-to-device copy, no host storage.  The column-sharded
        path builds the survivors' sub-design from columns received over NCCL
        this way; the caller synchronises the producer of
        the buffer first."""
        lib = _lib.load()
        self = cls.__new__(cls)
        handle = ctypes.c_void_p()
        dt = _lib.GS_DTYPE_F32 if np.dtype(dtype) == np.float32 else _lib.GS_DTYPE_F64
        _lib.check(lib.gs_matrix_dense_dev(ctypes.c_void_p(int(dev_ptr)), dt, int(n), int(p), int(ld),
                                           ctypes.byref(handle)))
        self._h, self._lib, self._mat = handle, lib, None
        self.is_sparse = False
        self.n_base, self.n_cols = int(n), int(p)
        self.dtype = np.dtype(dtype).type
        self.tail_weight = 0.0
        self.tail_scale = 0.0
        nsq = np.empty(self.n_cols, dtype=np.float64)
        _lib.check(lib.gs_matrix_norms_sq(self._h, _lib.f64p(nsq)))
        self._col_norms_sq = nsq
        self._col_norms = np.sqrt(nsq)
        return self

    @classmethod
    def from_blocks(cls, n: int, p: int, dtype, blocks) -> "DesignMatrix":
        """Dense design uploaded block by block: ``blocks`` yields
        ``(j0, Xb)`` with ``Xb`` an (n, k) array of the columns j0 .. j0+k.
        The host never holds more than one block (configs[2] is a 40 GB
        design); no host copy is kept."""
        lib = _lib.load()
        self = cls.__new__(cls)
        handle = ctypes.c_void_p()
        npdt = np.dtype(dtype)
        dt = _lib.GS_DTYPE_F32 if npdt == np.float32 else _lib.GS_DTYPE_F64
        _lib.check(lib.gs_matrix_dense_alloc(dt, int(n), int(p), ctypes.byref(handle)))
        self._h, self._lib, self._mat = handle, lib, None
        for j0, Xb in blocks:
            Xb = np.asfortranarray(Xb, dtype=npdt)
            if Xb.shape[0] != n:
                raise ValueError("block has the wrong number of rows")
            _lib.check(lib.gs_matrix_dense_set_columns(handle, int(j0), int(Xb.shape[1]),
                                                       Xb.ctypes.data_as(ctypes.c_void_p), int(n)))
        _lib.check(lib.gs_matrix_dense_finalize(handle))
        self.is_sparse = False
        self.n_base, self.n_cols = int(n), int(p)
        self.dtype = npdt.type
        self.tail_weight = 0.0
        self.tail_scale = 0.0
        nsq = np.empty(self.n_cols, dtype=np.float64)
        _lib.check(lib.gs_matrix_norms_sq(self._h, _lib.f64p(nsq)))
        self._col_norms_sq = nsq
        self._col_norms = np.sqrt(nsq)
        return self

    def columns_to_host(self, idx: np.ndarray) -> np.ndarray:
        """(n, k) host copy of the columns ``idx`` of a dense design (gathered on
        the device, one D2H copy): the column-subsampled parity checks of
        designs that have no host copy."""
        import torch
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        tdt = torch.float32 if self.dtype == np.float32 else torch.float64
        buf = torch.empty((max(1, idx.size), self.n_base), dtype=tdt, device="cuda")
        if idx.size:
            self.gather_columns_to_device(idx, buf.data_ptr(), self.n_base)
        return np.asfortranarray(buf[: idx.size].cpu().numpy().T)

    def gather_columns_to_device(self, idx: np.ndarray, dst_ptr: int, ld_dst: int) -> None:
        """Columns ``idx`` into the device buffer at ``dst_ptr`` (``ld_dst``
        elements per column): the send buffer of the X_A gather."""
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        _lib.check(self._lib.gs_matrix_gather_columns_dev(self._h, _lib.i64p(idx), idx.size,
                                                          ctypes.c_void_p(int(dst_ptr)), int(ld_dst)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.gs_matrix_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def device_bytes(self) -> int:
        return int(self._lib.gs_matrix_device_bytes(self._h))

    # ------------------------------------------------------------------
    @property
    def n_rows(self) -> int:
        """Logical rows, the tail included (design_matrix.py:60-65)."""
        if self.tail_weight > 0:
            return self.n_base + self.n_cols
        return self.n_base

    @property
    def col_norms(self) -> np.ndarray:
        return self._col_norms

    @property
    def col_norms_sq(self) -> np.ndarray:
        return self._col_norms_sq

    @property
    def zero_norm_cols(self) -> np.ndarray:
        return np.flatnonzero(self._col_norms == 0.0)

    def with_tail(self, tail_weight: float) -> "DesignMatrix":
        return DesignMatrix(self._mat, tail_weight=tail_weight)

    def normalized(self) -> "DesignMatrix":
        """Copy with unit-norm columns (zero columns left untouched)."""
        if self.tail_weight > 0:
            raise ValueError("cannot normalize an augmented matrix")
        norms = self._col_norms.copy()
        norms[norms == 0.0] = 1.0
        if self.is_sparse:
            return DesignMatrix(self._mat @ sp.diags(1.0 / norms))
        return DesignMatrix(self._mat / norms)

    # ------------------------------------------------------------------
    def _check_col(self, j: int) -> None:
        if not 0 <= j < self.n_cols:
            raise IndexError(f"column index {j} out of range [0, {self.n_cols})")

    def _vec(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.shape != (self.n_rows,):
            raise ValueError("vector length does not match n_rows")
        return v

    def col_dot(self, j: int, v: np.ndarray) -> float:
        """x_j^T v (design_matrix.py:100-113)."""
        self._check_col(j)
        return float(self.transpose_dot(v, cols=np.array([j], dtype=np.int64))[0])

    def axpy_col(self, j: int, a: float, v: np.ndarray) -> None:
        """In place v += a x_j (design_matrix.py:115-128)."""
        self._check_col(j)
        if v.shape != (self.n_rows,):
            raise ValueError("vector length does not match n_rows")
        if a == 0.0:
            return
        buf = np.ascontiguousarray(v, dtype=np.float64)
        _lib.check(self._lib.gs_axpy_col(self._h, int(j), float(a), _lib.f64p(buf)))
        if buf is not v:
            v[...] = buf

    def matvec(self, beta: np.ndarray) -> np.ndarray:
        """X @ beta (design_matrix.py:130-137)."""
        beta = np.ascontiguousarray(beta, dtype=np.float64)
        if beta.shape != (self.n_cols,):
            raise ValueError("beta has wrong length")
        out = np.empty(self.n_rows, dtype=np.float64)
        _lib.check(self._lib.gs_matvec(self._h, _lib.f64p(beta), _lib.f64p(out)))
        return out

    def transpose_dot(self, v: np.ndarray, cols: np.ndarray | None = None,
                      exact_order: bool = False) -> np.ndarray:
        """X^T v, optionally restricted to ``cols`` (design_matrix.py:139-158).

        ``exact_order`` selects the reference kernels' sequential non-FMA
        summation (bit-exact with _kernels.tdot_*)."""
        v = self._vec(v)
        if cols is None:
            out = np.empty(self.n_cols, dtype=np.float64)
            _lib.check(self._lib.gs_tdot(self._h, _lib.f64p(v), None, 0, 0.0, _lib.f64p(out),
                                         int(exact_order)))
            return out
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(cols.size, dtype=np.float64)
        if cols.size:
            _lib.check(self._lib.gs_tdot(self._h, _lib.f64p(v), _lib.i64p(cols), cols.size, 0.0,
                                         _lib.f64p(out), int(exact_order)))
        return out

    def max_abs_correlation(self, v: np.ndarray,
                            restrict: np.ndarray | None = None) -> tuple[float, int]:
        """(max_j |x_j^T v|, argmax j), ties to the smallest index (:160-174)."""
        v = self._vec(v)
        val = ctypes.c_double()
        arg = ctypes.c_int64()
        if restrict is not None:
            restrict = np.ascontiguousarray(restrict, dtype=np.int64)
            if restrict.size == 0:
                raise ValueError("empty restriction set")
            _lib.check(self._lib.gs_max_abs_correlation(self._h, _lib.f64p(v), _lib.i64p(restrict),
                                                        restrict.size, ctypes.byref(val),
                                                        ctypes.byref(arg)))
        else:
            _lib.check(self._lib.gs_max_abs_correlation(self._h, _lib.f64p(v), None, 0,
                                                        ctypes.byref(val), ctypes.byref(arg)))
        return float(val.value), int(arg.value)

    # ------------------------------------------------------------------
    def toarray(self) -> np.ndarray:
        if self._mat is None:
            raise ValueError("this design was built from device memory and keeps no host copy")
        base = self._mat.toarray() if self.is_sparse else np.array(self._mat, dtype=np.float64)
        if self.tail_scale > 0.0:                               # design_matrix.py:177-183
            return np.asfortranarray(np.vstack([base, self.tail_scale * np.eye(self.n_cols)]))
        return np.asfortranarray(base)

    def raw(self):
        """Host storage handle (the uploaded copy lives on the device)."""
        return self._mat
