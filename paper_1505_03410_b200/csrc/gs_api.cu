// Host side of libgapsafe_b200: device-resident DesignMatrix, the primitive
// entry points and the solve / sequential-screen state machine
// (solver.py:149-246, path.py:82-91), all behind the C ABI of
// include/gapsafe_b200.h.
#include "../../include/gapsafe_b200.h"
#include "gs_kernels.cuh"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace gs;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(GS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CKL()                                                                          \
    do {                                                                               \
        cudaError_t e_ = cudaGetLastError();                                           \
        if (e_ != cudaSuccess)                                                         \
            return fail(GS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

#define TRY(x)                  \
    do {                        \
        int r_ = (x);           \
        if (r_ != GS_OK) return r_; \
    } while (0)

static int g_device = -1;

static int ensure_device() {
    if (g_device >= 0) return GS_OK;
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt <= 0)
        return fail(GS_ERR_NODEVICE, "gapsafe_b200 requires a CUDA device (sm_100a); none found"
                    " -- there is no CPU fallback");
    CK(cudaSetDevice(0));
    g_device = 0;
    return GS_OK;
}

template <typename T>
static int dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    CK(cudaMalloc((void**)p, count * sizeof(T)));
    return GS_OK;
}

static inline unsigned grid_for(int64_t n, int block, int64_t cap = 148 * 16) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ---------------------------------------------------------------------------
// matrix
// ---------------------------------------------------------------------------
struct gs_matrix {
    int sparse = 0, dtype = GS_DTYPE_F64;
    int64_t n = 0, p = 0, ld = 0, nnz = 0;
    void* X = nullptr;                       // dense
    double* data = nullptr;                  // CSC
    int32_t* indices = nullptr;
    int64_t* indptr = nullptr;
    double* csr_data = nullptr;              // CSR copy (resync row products)
    int32_t* csr_cols = nullptr;
    int64_t* csr_rowptr = nullptr;
    double* norms_sq = nullptr;
    double* norms = nullptr;
    int64_t bytes = 0;
    cudaStream_t st = nullptr;
};

static void matrix_release(gs_matrix* M) {
    if (!M) return;
    cudaFree(M->X); cudaFree(M->data); cudaFree(M->indices); cudaFree(M->indptr);
    cudaFree(M->csr_data); cudaFree(M->csr_cols); cudaFree(M->csr_rowptr);
    cudaFree(M->norms_sq); cudaFree(M->norms);
    if (M->st) cudaStreamDestroy(M->st);
    delete M;
}

static int matrix_norms(gs_matrix* M, const double* norms_sq_host) {
    TRY(dalloc(&M->norms_sq, M->p));
    TRY(dalloc(&M->norms, M->p));
    if (norms_sq_host) {
        CK(cudaMemcpyAsync(M->norms_sq, norms_sq_host, M->p * sizeof(double), cudaMemcpyHostToDevice, M->st));
    } else if (M->sparse) {
        k_col_norms_sq_csc<<<grid_for(M->p * 32, 256), 256, 0, M->st>>>(M->data, M->indptr, M->p, M->norms_sq);
    } else if (M->dtype == GS_DTYPE_F64) {
        k_col_norms_sq_dense<double><<<grid_for(M->p * 32, 256), 256, 0, M->st>>>((const double*)M->X, M->ld, (int)M->n, M->p, M->norms_sq);
    } else {
        k_col_norms_sq_dense<float><<<grid_for(M->p * 32, 256), 256, 0, M->st>>>((const float*)M->X, M->ld, (int)M->n, M->p, M->norms_sq);
    }
    CKL();
    k_sqrt_vec<<<grid_for(M->p, 256), 256, 0, M->st>>>(M->norms_sq, 0.0, M->p, M->norms_sq, M->norms);
    CKL();
    CK(cudaStreamSynchronize(M->st));
    M->bytes += 2 * M->p * 8;
    return GS_OK;
}

extern "C" int gs_init(int device) {
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt <= 0)
        return fail(GS_ERR_NODEVICE, "gapsafe_b200 requires a CUDA device (sm_100a); none found"
                    " -- there is no CPU fallback");
    if (device < 0 || device >= cnt) return fail(GS_ERR_VALUE, "device index out of range");
    CK(cudaSetDevice(device));
    g_device = device;
    return GS_OK;
}

extern "C" int gs_device_count(int* count) {
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess) cnt = 0;
    *count = cnt;
    return GS_OK;
}

extern "C" const char* gs_last_error(void) { return g_err.c_str(); }
extern "C" const char* gs_version(void) { return "gapsafe_b200 0.1.0 (sm_100a)"; }

extern "C" int gs_matrix_dense(const void* X, int dtype, int64_t n, int64_t p, int64_t ld_host,
                               const double* norms_sq, gs_matrix** out) {
    TRY(ensure_device());
    if (n < 1 || p < 1) return fail(GS_ERR_VALUE, "matrix must have at least one row and column");
    if (n > (1 << 30)) return fail(GS_ERR_VALUE, "too many rows");
    if (dtype != GS_DTYPE_F64 && dtype != GS_DTYPE_F32) return fail(GS_ERR_VALUE, "dtype must be f64 or f32");
    gs_matrix* M = new gs_matrix();
    M->dtype = dtype; M->n = n; M->p = p;
    const size_t es = dtype == GS_DTYPE_F64 ? 8 : 4;
    const int64_t align = dtype == GS_DTYPE_F64 ? 2 : 4;      // 16-B aligned columns
    M->ld = (n + align - 1) / align * align;
    int rc;
    if ((rc = [&]() -> int {
            CK(cudaStreamCreateWithFlags(&M->st, cudaStreamNonBlocking));
            CK(cudaMalloc(&M->X, (size_t)M->ld * p * es));
            M->bytes += (int64_t)M->ld * p * es;
            if (M->ld != n) CK(cudaMemsetAsync(M->X, 0, (size_t)M->ld * p * es, M->st));
            CK(cudaMemcpy2DAsync(M->X, M->ld * es, X, ld_host * es, n * es, p, cudaMemcpyHostToDevice, M->st));
            return matrix_norms(M, norms_sq);
        }()) != GS_OK) {
        matrix_release(M);
        return rc;
    }
    *out = M;
    return GS_OK;
}

extern "C" int gs_matrix_csc(const double* data, const int32_t* indices, const int64_t* indptr, int64_t n,
                             int64_t p, const double* norms_sq, gs_matrix** out) {
    TRY(ensure_device());
    if (n < 1 || p < 1) return fail(GS_ERR_VALUE, "matrix must have at least one row and column");
    gs_matrix* M = new gs_matrix();
    M->sparse = 1; M->n = n; M->p = p;
    const int64_t nnz = indptr[p];
    M->nnz = nnz;
    int rc;
    if ((rc = [&]() -> int {
            CK(cudaStreamCreateWithFlags(&M->st, cudaStreamNonBlocking));
            TRY(dalloc(&M->data, nnz)); TRY(dalloc(&M->indices, nnz)); TRY(dalloc(&M->indptr, p + 1));
            CK(cudaMemcpyAsync(M->data, data, nnz * 8, cudaMemcpyHostToDevice, M->st));
            CK(cudaMemcpyAsync(M->indices, indices, nnz * 4, cudaMemcpyHostToDevice, M->st));
            CK(cudaMemcpyAsync(M->indptr, indptr, (p + 1) * 8, cudaMemcpyHostToDevice, M->st));
            // CSR copy for the row-parallel resync (built once on the host).
            std::vector<int64_t> rowptr(n + 1, 0);
            for (int64_t q = 0; q < nnz; ++q) rowptr[indices[q] + 1]++;
            for (int64_t r = 0; r < n; ++r) rowptr[r + 1] += rowptr[r];
            std::vector<int64_t> fill(rowptr.begin(), rowptr.end() - 1);
            std::vector<double> cd(nnz);
            std::vector<int32_t> cc(nnz);
            for (int64_t j = 0; j < p; ++j)
                for (int64_t q = indptr[j]; q < indptr[j + 1]; ++q) {
                    const int64_t dst = fill[indices[q]]++;
                    cd[dst] = data[q];
                    cc[dst] = (int32_t)j;
                }
            TRY(dalloc(&M->csr_data, nnz)); TRY(dalloc(&M->csr_cols, nnz)); TRY(dalloc(&M->csr_rowptr, n + 1));
            CK(cudaMemcpyAsync(M->csr_data, cd.data(), nnz * 8, cudaMemcpyHostToDevice, M->st));
            CK(cudaMemcpyAsync(M->csr_cols, cc.data(), nnz * 4, cudaMemcpyHostToDevice, M->st));
            CK(cudaMemcpyAsync(M->csr_rowptr, rowptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice, M->st));
            CK(cudaStreamSynchronize(M->st));
            M->bytes += nnz * 24 + (p + 1) * 8 + (n + 1) * 8;
            return matrix_norms(M, norms_sq);
        }()) != GS_OK) {
        matrix_release(M);
        return rc;
    }
    *out = M;
    return GS_OK;
}

extern "C" int gs_matrix_norms_sq(const gs_matrix* M, double* out) {
    CK(cudaMemcpy(out, M->norms_sq, M->p * 8, cudaMemcpyDeviceToHost));
    return GS_OK;
}

extern "C" int64_t gs_matrix_device_bytes(const gs_matrix* M) { return M ? M->bytes : 0; }
extern "C" void gs_matrix_free(gs_matrix* M) { matrix_release(M); }

// ---------------------------------------------------------------------------
// launch helpers shared by primitives and the solver
// ---------------------------------------------------------------------------
struct Scratch {   // reusable device buffers sized for one (n, p)
    double* blk_val = nullptr;
    int64_t* blk_idx = nullptr;
    int32_t* cnt = nullptr;
    int64_t* off = nullptr;
    int64_t nblk = 0;
    int alloc(int64_t p) {
        nblk = std::max<int64_t>(p / 8 + 2, (p + kCompactChunk - 1) / kCompactChunk + 2);
        TRY(dalloc(&blk_val, nblk)); TRY(dalloc(&blk_idx, nblk));
        TRY(dalloc(&cnt, nblk)); TRY(dalloc(&off, nblk));
        return GS_OK;
    }
    void release() { cudaFree(blk_val); cudaFree(blk_idx); cudaFree(cnt); cudaFree(off); }
};

static int gemv_cpb(int64_t m) {
    int64_t c = (m + 148 * 4 - 1) / (148 * 4);
    return (int)std::max<int64_t>(8, std::min<int64_t>(512, c));
}

// Launch the screening / restricted GEMV over m columns (cols == nullptr: 0..m-1).
static int launch_gemv(const gs_matrix* M, cudaStream_t st, GemvArgs a, int64_t* nblocks_out) {
    if (a.m <= 0) { if (nblocks_out) *nblocks_out = 0; return GS_OK; }
    a.ld = M->ld;
    a.n = (int)M->n;
    a.cpb = gemv_cpb(a.m);
    const int64_t nb = (a.m + a.cpb - 1) / a.cpb;
    if (nblocks_out) *nblocks_out = nb;
    if (M->sparse) {
        k_gemv_t_csc<<<(unsigned)nb, 256, 0, st>>>(M->data, M->indices, M->indptr, a);
    } else {
        const bool vsm = (M->n + 2) * 8 <= 48 * 1024;
        const size_t sm = vsm ? (size_t)(M->n + 2) * 8 : 0;
        if (M->dtype == GS_DTYPE_F64) {
            if (vsm) k_gemv_t_dense<double, true><<<(unsigned)nb, 256, sm, st>>>((const double*)M->X, a);
            else k_gemv_t_dense<double, false><<<(unsigned)nb, 256, 0, st>>>((const double*)M->X, a);
        } else {
            if (vsm) k_gemv_t_dense<float, true><<<(unsigned)nb, 256, sm, st>>>((const float*)M->X, a);
            else k_gemv_t_dense<float, false><<<(unsigned)nb, 256, 0, st>>>((const float*)M->X, a);
        }
    }
    CKL();
    return GS_OK;
}

static int launch_compact(cudaStream_t st, Scratch& s, const uint8_t* flags, int64_t m, const int32_t* cols,
                          int32_t* out, int64_t* count_dev) {
    const int64_t nb = (m + kCompactChunk - 1) / kCompactChunk;
    if (m <= 0) {
        CK(cudaMemsetAsync(count_dev, 0, sizeof(int64_t), st));
        return GS_OK;
    }
    k_compact_count<<<(unsigned)nb, 256, 0, st>>>(flags, m, s.cnt);
    k_scan_counts<<<1, 1024, 0, st>>>(s.cnt, nb, s.off, count_dev);
    k_compact_scatter<<<(unsigned)nb, 256, 0, st>>>(flags, m, cols, s.off, out);
    CKL();
    return GS_OK;
}

// ---------------------------------------------------------------------------
// primitives
// ---------------------------------------------------------------------------
struct TmpBuf {
    std::vector<void*> ptrs;
    template <typename T> int get(T** p, size_t count) {
        TRY(dalloc(p, count));
        ptrs.push_back(*p);
        return GS_OK;
    }
    ~TmpBuf() { for (void* q : ptrs) cudaFree(q); }
};

static int upload_cols(cudaStream_t st, TmpBuf& tb, const gs_matrix* M, const int64_t* cols, int64_t k,
                       int32_t** out) {
    std::vector<int32_t> c32(std::max<int64_t>(k, 1));
    for (int64_t i = 0; i < k; ++i) {
        if (cols[i] < 0 || cols[i] >= M->p)
            return fail(GS_ERR_INDEX, "column index " + std::to_string(cols[i]) + " out of range [0, " +
                                           std::to_string(M->p) + ")");
        c32[i] = (int32_t)cols[i];
    }
    TRY(tb.get(out, k));
    CK(cudaMemcpyAsync(*out, c32.data(), k * 4, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return GS_OK;
}

extern "C" int gs_tdot(const gs_matrix* M, const double* v, const int64_t* cols, int64_t k, double tail_scale,
                       double* out, int exact_order) {
    TRY(ensure_device());
    cudaStream_t st = M->st;
    TmpBuf tb;
    const int64_t n = M->n;
    const int64_t vlen = n + (tail_scale > 0.0 ? M->p : 0);
    double* dv; double* dout; int32_t* dcols = nullptr;
    TRY(tb.get(&dv, vlen + 2));
    CK(cudaMemcpyAsync(dv, v, vlen * 8, cudaMemcpyHostToDevice, st));
    const int64_t m = cols ? k : M->p;
    if (m == 0) return GS_OK;
    TRY(tb.get(&dout, m));
    if (cols) TRY(upload_cols(st, tb, M, cols, k, &dcols));
    if (exact_order || tail_scale > 0.0) {
        if (!dcols) {
            std::vector<int64_t> all(m);
            for (int64_t i = 0; i < m; ++i) all[i] = i;
            TRY(upload_cols(st, tb, M, all.data(), m, &dcols));
        }
        if (M->sparse)
            k_tdot_exact_csc<<<grid_for(m, 128), 128, 0, st>>>(M->data, M->indices, M->indptr, (int)n, dv, dcols, m, tail_scale, dout);
        else if (M->dtype == GS_DTYPE_F64)
            k_tdot_exact_dense<double><<<grid_for(m, 128), 128, 0, st>>>((const double*)M->X, M->ld, (int)n, dv, dcols, m, tail_scale, dout);
        else
            k_tdot_exact_dense<float><<<grid_for(m, 128), 128, 0, st>>>((const float*)M->X, M->ld, (int)n, dv, dcols, m, tail_scale, dout);
        CKL();
    } else {
        GemvArgs a{};
        a.v = dv; a.cols = dcols; a.m = m; a.mode = GEMV_RAW; a.out_c = dout;
        TRY(launch_gemv(M, st, a, nullptr));
    }
    CK(cudaMemcpyAsync(out, dout, m * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GS_OK;
}

static int matvec_dev(const gs_matrix* M, cudaStream_t st, TmpBuf& tb, const double* dbeta, const double* dy,
                      double* dout) {
    // support = nonzero coordinates of beta over all p
    const int64_t p = M->p, n = M->n;
    if (M->sparse) {
        k_resync_csr<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(M->csr_data, M->csr_cols, M->csr_rowptr, (int)n, dbeta, dy, dout);
        CKL();
        return GS_OK;
    }
    uint8_t* flags; int32_t* S; int64_t* cnt; double* partial;
    Scratch s;
    TRY(s.alloc(p));
    TRY(tb.get(&flags, p)); TRY(tb.get(&S, p)); TRY(tb.get(&cnt, 1));
    k_flags_beta_nz<<<grid_for(p, 256), 256, 0, st>>>(nullptr, p, dbeta, flags);
    int rc = launch_compact(st, s, flags, p, nullptr, S, cnt);
    if (rc == GS_OK) {
        const int nch = (int)std::min<int64_t>(256, std::max<int64_t>(1, (p + 31) / 32));
        rc = tb.get(&partial, (size_t)nch * n);
        if (rc == GS_OK) {
            dim3 g((unsigned)((n + 255) / 256), (unsigned)nch);
            if (M->dtype == GS_DTYPE_F64)
                k_resync_partial_dense<double><<<g, 256, 0, st>>>((const double*)M->X, M->ld, (int)n, S, cnt, dbeta, nch, partial);
            else
                k_resync_partial_dense<float><<<g, 256, 0, st>>>((const float*)M->X, M->ld, (int)n, S, cnt, dbeta, nch, partial);
            k_resync_final<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dy, partial, nch, (int)n, dout);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail(GS_ERR_CUDA, cudaGetErrorString(e));
        }
    }
    CK(cudaStreamSynchronize(st));
    s.release();
    return rc;
}

extern "C" int gs_matvec(const gs_matrix* M, const double* beta, double* out) {
    TRY(ensure_device());
    cudaStream_t st = M->st;
    TmpBuf tb;
    double *db, *dout;
    TRY(tb.get(&db, M->p)); TRY(tb.get(&dout, M->n));
    CK(cudaMemcpyAsync(db, beta, M->p * 8, cudaMemcpyHostToDevice, st));
    TRY(matvec_dev(M, st, tb, db, nullptr, dout));
    CK(cudaMemcpy(out, dout, M->n * 8, cudaMemcpyDeviceToHost));
    return GS_OK;
}

extern "C" int gs_max_abs_correlation(const gs_matrix* M, const double* v, const int64_t* rcols, int64_t k,
                                      double* val, int64_t* arg) {
    TRY(ensure_device());
    if (rcols && k == 0) return fail(GS_ERR_VALUE, "empty restriction set");
    cudaStream_t st = M->st;
    TmpBuf tb;
    Scratch s;
    TRY(s.alloc(M->p));
    double* dv; int32_t* dcols = nullptr; double* dval; int64_t* didx;
    TRY(tb.get(&dv, M->n + 2)); TRY(tb.get(&dval, 1)); TRY(tb.get(&didx, 1));
    CK(cudaMemcpyAsync(dv, v, M->n * 8, cudaMemcpyHostToDevice, st));
    if (rcols) TRY(upload_cols(st, tb, M, rcols, k, &dcols));
    GemvArgs a{};
    a.v = dv; a.cols = dcols; a.m = rcols ? k : M->p; a.mode = GEMV_MAX;
    a.blk_val = s.blk_val; a.blk_idx = s.blk_idx;
    int64_t nb = 0;
    TRY(launch_gemv(M, st, a, &nb));
    k_max_finalize<<<1, 1024, 0, st>>>(s.blk_val, s.blk_idx, nb, dval, didx);
    CKL();
    int64_t pos = 0;
    CK(cudaMemcpyAsync(val, dval, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&pos, didx, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    s.release();
    *arg = rcols ? rcols[pos] : pos;
    return GS_OK;
}

extern "C" int gs_axpy_col(const gs_matrix* M, int64_t j, double a, double* v) {
    TRY(ensure_device());
    if (j < 0 || j >= M->p)
        return fail(GS_ERR_INDEX, "column index " + std::to_string(j) + " out of range [0, " + std::to_string(M->p) + ")");
    if (a == 0.0) return GS_OK;
    cudaStream_t st = M->st;
    TmpBuf tb;
    double *dv, *db; int32_t* dl; int64_t* dc;
    TRY(tb.get(&dv, M->n)); TRY(tb.get(&db, M->p)); TRY(tb.get(&dl, 1)); TRY(tb.get(&dc, 1));
    CK(cudaMemcpyAsync(dv, v, M->n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(db, 0, M->p * 8, st));
    CK(cudaMemcpyAsync(db + j, &a, 8, cudaMemcpyHostToDevice, st));
    const int32_t j32 = (int32_t)j;
    const int64_t one = 1;
    CK(cudaMemcpyAsync(dl, &j32, 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dc, &one, 8, cudaMemcpyHostToDevice, st));
    if (M->sparse)
        k_drop_axpy_csc<<<1, 256, 0, st>>>(M->data, M->indices, M->indptr, dl, dc, db, dv);
    else if (M->dtype == GS_DTYPE_F64)
        k_drop_axpy_dense<double><<<grid_for(M->n, 256, 1 << 30), 256, 0, st>>>((const double*)M->X, M->ld, (int)M->n, dl, dc, db, dv);
    else
        k_drop_axpy_dense<float><<<grid_for(M->n, 256, 1 << 30), 256, 0, st>>>((const float*)M->X, M->ld, (int)M->n, dl, dc, db, dv);
    CKL();
    CK(cudaMemcpyAsync(v, dv, M->n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GS_OK;
}

extern "C" int gs_vec_stats(const double* a, const double* b, int64_t n, double* dot, double* asum) {
    TRY(ensure_device());
    TmpBuf tb;
    double *da, *db = nullptr, *dout;
    TRY(tb.get(&da, n)); TRY(tb.get(&dout, 2));
    CK(cudaMemcpy(da, a, n * 8, cudaMemcpyHostToDevice));
    if (b) { TRY(tb.get(&db, n)); CK(cudaMemcpy(db, b, n * 8, cudaMemcpyHostToDevice)); }
    k_vec_stats<<<1, 1024>>>(da, db, n, dout);
    CKL();
    double h[2];
    CK(cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost));
    if (dot) *dot = h[0];
    if (asum) *asum = h[1];
    return GS_OK;
}

// CD epoch launch: (block, rows-per-thread) from n.
template <typename T>
static int launch_cd_dense(const gs_matrix* M, cudaStream_t st, const CdArgs& a) {
    const int64_t n = M->n;
    const T* X = (const T*)M->X;
    if (n <= 128) k_cd_epoch_dense<T, 1><<<1, 128, 0, st>>>(X, a);
    else if (n <= 256) k_cd_epoch_dense<T, 1><<<1, 256, 0, st>>>(X, a);
    else if (n <= 512) k_cd_epoch_dense<T, 2><<<1, 256, 0, st>>>(X, a);
    else if (n <= 1024) k_cd_epoch_dense<T, 4><<<1, 256, 0, st>>>(X, a);
    else if (n <= 2048) k_cd_epoch_dense<T, 8><<<1, 256, 0, st>>>(X, a);
    else if (n <= 4096) k_cd_epoch_dense<T, 8><<<1, 512, 0, st>>>(X, a);
    else return fail(GS_ERR_VALUE, "dense CD kernel supports n <= 4096 in this build");
    CKL();
    return GS_OK;
}

static int launch_cd(const gs_matrix* M, cudaStream_t st, const CdArgs& a) {
    if (M->sparse) {
        const size_t sm = (size_t)M->n * 8;
        if (sm > 200 * 1024) return fail(GS_ERR_VALUE, "sparse CD kernel supports n <= 25600 in this build");
        if (sm > 48 * 1024) CK(cudaFuncSetAttribute(k_cd_epoch_csc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_cd_epoch_csc<<<1, 1024, sm, st>>>(M->data, M->indices, M->indptr, a);
        CKL();
        return GS_OK;
    }
    return M->dtype == GS_DTYPE_F64 ? launch_cd_dense<double>(M, st, a) : launch_cd_dense<float>(M, st, a);
}

// ---------------------------------------------------------------------------
// solver
// ---------------------------------------------------------------------------
struct gs_solver {
    const gs_matrix* M = nullptr;
    cudaStream_t st = nullptr;
    int64_t n = 0, p = 0;
    double *y = nullptr, *beta = nullptr, *rho = nullptr, *theta = nullptr, *c = nullptr, *t = nullptr;
    int32_t *A = nullptr, *A2 = nullptr, *S = nullptr, *Dl = nullptr;
    uint8_t *flags = nullptr, *flags2 = nullptr, *mark = nullptr;
    double* partial = nullptr;
    int nch_max = 0;
    Scratch s;
    DevScalars* sc = nullptr;     // device
    DevScalars* hs = nullptr;     // pinned host mirror
    TraceRow* trace = nullptr;
    int64_t trace_cap = 0;
    double lmax = 0.0, y_norm_sq = 0.0;
    int64_t jstar = 0;
    int64_t m = 0;                // current active count (host mirror)
    bool has_prev = false;
    double prev_margin = 1.0;
    int prev_interp = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

static void solver_release(gs_solver* S) {
    if (!S) return;
    cudaFree(S->y); cudaFree(S->beta); cudaFree(S->rho); cudaFree(S->theta); cudaFree(S->c); cudaFree(S->t);
    cudaFree(S->A); cudaFree(S->A2); cudaFree(S->S); cudaFree(S->Dl);
    cudaFree(S->flags); cudaFree(S->flags2); cudaFree(S->mark); cudaFree(S->partial);
    cudaFree(S->sc); cudaFreeHost(S->hs); cudaFree(S->trace);
    S->s.release();
    if (S->ev0) cudaEventDestroy(S->ev0);
    if (S->ev1) cudaEventDestroy(S->ev1);
    if (S->st) cudaStreamDestroy(S->st);
    delete S;
}

static int sc_upload(gs_solver* S) {
    CK(cudaMemcpyAsync(S->sc, S->hs, sizeof(DevScalars), cudaMemcpyHostToDevice, S->st));
    return GS_OK;
}
static int sc_download(gs_solver* S) {
    CK(cudaMemcpyAsync(S->hs, S->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, S->st));
    CK(cudaStreamSynchronize(S->st));
    return GS_OK;
}

extern "C" int gs_solver_create(const gs_matrix* M, const double* y, gs_solver** out) {
    TRY(ensure_device());
    gs_solver* S = new gs_solver();
    S->M = M; S->n = M->n; S->p = M->p;
    int rc = [&]() -> int {
        const int64_t n = S->n, p = S->p;
        CK(cudaStreamCreateWithFlags(&S->st, cudaStreamNonBlocking));
        CK(cudaEventCreate(&S->ev0)); CK(cudaEventCreate(&S->ev1));
        TRY(dalloc(&S->y, n + 2)); TRY(dalloc(&S->rho, n + 2)); TRY(dalloc(&S->theta, n + 2));
        TRY(dalloc(&S->beta, p)); TRY(dalloc(&S->c, p)); TRY(dalloc(&S->t, p));
        TRY(dalloc(&S->A, p)); TRY(dalloc(&S->A2, p)); TRY(dalloc(&S->S, p)); TRY(dalloc(&S->Dl, p));
        TRY(dalloc(&S->flags, p)); TRY(dalloc(&S->flags2, p)); TRY(dalloc(&S->mark, p));
        S->nch_max = (int)std::min<int64_t>(256, std::max<int64_t>(1, (p + 31) / 32));
        if (!M->sparse) TRY(dalloc(&S->partial, (size_t)S->nch_max * n));
        TRY(S->s.alloc(p));
        TRY(dalloc(&S->sc, 1));
        CK(cudaMallocHost((void**)&S->hs, sizeof(DevScalars)));
        memset(S->hs, 0, sizeof(DevScalars));
        CK(cudaMemsetAsync(S->mark, 0, p, S->st));
        CK(cudaMemsetAsync(S->beta, 0, p * 8, S->st));
        CK(cudaMemsetAsync(S->y, 0, (n + 2) * 8, S->st));
        CK(cudaMemcpyAsync(S->y, y, n * 8, cudaMemcpyHostToDevice, S->st));
        TRY(sc_upload(S));
        // lambda_max = |X^T y|_inf, j_star (problem.py:50), ||y||^2 (problem.py:54)
        GemvArgs a{};
        a.v = S->y; a.m = p; a.mode = GEMV_MAX; a.blk_val = S->s.blk_val; a.blk_idx = S->s.blk_idx;
        int64_t nb = 0;
        TRY(launch_gemv(M, S->st, a, &nb));
        k_max_finalize<<<1, 1024, 0, S->st>>>(S->s.blk_val, S->s.blk_idx, nb, &S->sc->corr, &S->sc->corr_arg);
        double* tmp;
        TRY(dalloc(&tmp, 2));
        k_vec_stats<<<1, 1024, 0, S->st>>>(S->y, S->y, n, tmp);
        CKL();
        double h[2];
        CK(cudaMemcpyAsync(h, tmp, 16, cudaMemcpyDeviceToHost, S->st));
        TRY(sc_download(S));
        cudaFree(tmp);
        S->lmax = S->hs->corr;
        S->jstar = S->hs->corr_arg;
        S->y_norm_sq = h[0];
        S->hs->y_norm_sq = h[0];
        return GS_OK;
    }();
    if (rc != GS_OK) { solver_release(S); return rc; }
    *out = S;
    return GS_OK;
}

extern "C" int gs_solver_lambda_max(gs_solver* S, double* lambda_max, int64_t* j_star, double* y_norm_sq) {
    if (lambda_max) *lambda_max = S->lmax;
    if (j_star) *j_star = S->jstar;
    if (y_norm_sq) *y_norm_sq = S->y_norm_sq;
    return GS_OK;
}

extern "C" int gs_solver_set_beta(gs_solver* S, const double* beta) {
    if (beta) CK(cudaMemcpyAsync(S->beta, beta, S->p * 8, cudaMemcpyHostToDevice, S->st));
    else CK(cudaMemsetAsync(S->beta, 0, S->p * 8, S->st));
    CK(cudaStreamSynchronize(S->st));
    return GS_OK;
}

extern "C" void gs_solver_free(gs_solver* S) { solver_release(S); }

static int status_error(int32_t st, const DevScalars* h, bool seq) {
    char buf[256];
    if (st == ST_INFEASIBLE) {
        snprintf(buf, sizeof buf, "dual point infeasible: margin=%.17g", seq ? h->margin : h->margin);
        return fail(GS_ERR_INFEASIBLE, buf);
    }
    if (st == ST_NEG_GAP) {
        snprintf(buf, sizeof buf, "negative duality gap beyond tolerance: %.17g", h->gap_pre);
        return fail(GS_ERR_NUMERICAL, buf);
    }
    return GS_OK;
}

// rho = y - X beta over the current support (beta is zero off A)
static int resync(gs_solver* S) {
    const gs_matrix* M = S->M;
    cudaStream_t st = S->st;
    const int n = (int)S->n;
    if (M->sparse) {
        k_resync_csr<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(M->csr_data, M->csr_cols, M->csr_rowptr, n, S->beta, S->y, S->rho);
        CKL();
        return GS_OK;
    }
    const int64_t m = S->m;
    k_flags_beta_nz<<<grid_for(std::max<int64_t>(m, 1), 256), 256, 0, st>>>(S->A, m, S->beta, S->flags);
    CKL();
    TRY(launch_compact(st, S->s, S->flags, m, S->A, S->S, &S->sc->n_supp));
    const int nch = (int)std::min<int64_t>(S->nch_max, std::max<int64_t>(1, (m + 31) / 32));
    dim3 g((unsigned)((n + 255) / 256), (unsigned)nch);
    if (M->dtype == GS_DTYPE_F64)
        k_resync_partial_dense<double><<<g, 256, 0, st>>>((const double*)M->X, M->ld, n, S->S, &S->sc->n_supp, S->beta, nch, S->partial);
    else
        k_resync_partial_dense<float><<<g, 256, 0, st>>>((const float*)M->X, M->ld, n, S->S, &S->sc->n_supp, S->beta, nch, S->partial);
    k_resync_final<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(S->y, S->partial, nch, n, S->rho);
    CKL();
    return GS_OK;
}

// restricted (A) or unrestricted (all p) |X^T rho|_inf into sc->corr; dots into c.
static int dual_corr(gs_solver* S, bool restricted) {
    GemvArgs a{};
    a.v = S->rho; a.cols = restricted ? S->A : nullptr; a.m = restricted ? S->m : S->p;
    a.mode = GEMV_MAX; a.out_c = restricted ? S->c : nullptr;
    a.blk_val = S->s.blk_val; a.blk_idx = S->s.blk_idx;
    int64_t nb = 0;
    TRY(launch_gemv(S->M, S->st, a, &nb));
    k_max_finalize<<<1, 1024, 0, S->st>>>(S->s.blk_val, S->s.blk_idx, nb, &S->sc->corr, &S->sc->corr_arg);
    CKL();
    return GS_OK;
}

static int cd_epoch(gs_solver* S, bool certify) {
    const gs_matrix* M = S->M;
    if (S->m == 0) return GS_OK;
    if (certify) {
        GemvArgs a{};
        a.v = S->rho; a.cols = S->A; a.m = S->m; a.mode = GEMV_CERT; a.out_c = S->c; a.out_t = S->t;
        a.blk_val = S->s.blk_val; a.blk_idx = S->s.blk_idx; a.norms = M->norms; a.beta = S->beta;
        a.lam = S->hs->lam; a.rho_norm_dev = &S->sc->rho_norm_ub; a.gam = gamma_n(M->sparse ? 64 : M->n);
        if (M->sparse) {
            // CSC columns are short; bound with the true max column length
            a.gam = gamma_n(std::min<int64_t>(M->n, M->nnz));
        }
        TRY(launch_gemv(M, S->st, a, nullptr));
    }
    CdArgs c{};
    c.ld = M->ld; c.n = (int)M->n; c.A = S->A; c.m = S->m; c.tcert = certify ? S->t : nullptr;
    c.beta = S->beta; c.rho = S->rho; c.nsq = M->norms_sq; c.norms = M->norms; c.lam = S->hs->lam; c.sc = S->sc;
    return launch_cd(M, S->st, c);
}

static int copy_active_host(gs_solver* S, int64_t* out) {
    std::vector<int32_t> tmp(std::max<int64_t>(S->m, 1));
    if (S->m) CK(cudaMemcpyAsync(tmp.data(), S->A, S->m * 4, cudaMemcpyDeviceToHost, S->st));
    CK(cudaStreamSynchronize(S->st));
    for (int64_t i = 0; i < S->m; ++i) out[i] = tmp[i];
    return GS_OK;
}

static int fire_hook(gs_solver* S, const gs_solve_config* cfg) {
    if (!cfg->on_checkpoint) return GS_OK;
    std::vector<int64_t> act(std::max<int64_t>(S->m, 1));
    TRY(copy_active_host(S, act.data()));
    cfg->on_checkpoint(act.data(), S->m, cfg->user);
    return GS_OK;
}

// screen all p with a sphere whose radius lives in sc->radius (seq screen)
// or is given (lambda_max shortcut, radius 0); result into S->A, count sc->m.
static int screen_all(gs_solver* S, const double* center, const double* radius_dev, double radius_host) {
    GemvArgs a{};
    a.v = center; a.m = S->p; a.mode = GEMV_MU; a.scale = 1.0; a.radius_dev = radius_dev;
    a.radius_host = radius_host; a.thresh = 1.0 - 1e-9; a.norms = S->M->norms; a.flags = S->flags;
    TRY(launch_gemv(S->M, S->st, a, nullptr));
    TRY(launch_compact(S->st, S->s, S->flags, S->p, nullptr, S->A, &S->sc->m));
    return GS_OK;
}

extern "C" int gs_solver_seq_screen(gs_solver* S, double lam, int64_t* n_active) {
    if (!S->has_prev) return fail(GS_ERR_VALUE, "sequential screen needs a previous solve");
    S->hs->lam = lam;
    TRY(sc_upload(S));
    k_seq_gap<<<1, 1024, 0, S->st>>>(S->rho, S->y, S->theta, (int)S->n, S->beta, S->A, S->m, S->prev_margin, S->sc);
    CKL();
    TRY(screen_all(S, S->theta, &S->sc->radius, 0.0));
    TRY(sc_download(S));
    if (S->hs->status != ST_OK) {
        S->hs->margin = S->prev_margin;
        return status_error(S->hs->status, S->hs, true);
    }
    S->m = S->hs->m;
    *n_active = S->m;
    return GS_OK;
}

static int solve_outputs(gs_solver* S, gs_solve_result* R, int64_t n_trace) {
    cudaStream_t st = S->st;
    if (R->beta) CK(cudaMemcpyAsync(R->beta, S->beta, S->p * 8, cudaMemcpyDeviceToHost, st));
    if (R->residual) CK(cudaMemcpyAsync(R->residual, S->rho, S->n * 8, cudaMemcpyDeviceToHost, st));
    if (R->theta) CK(cudaMemcpyAsync(R->theta, S->theta, S->n * 8, cudaMemcpyDeviceToHost, st));
    if (R->active) TRY(copy_active_host(S, R->active));
    std::vector<TraceRow> tr(std::max<int64_t>(n_trace, 1));
    if (n_trace > 0 && S->trace)
        CK(cudaMemcpyAsync(tr.data(), S->trace, n_trace * sizeof(TraceRow), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t nt = std::min<int64_t>(n_trace, R->trace_cap);
    for (int64_t i = 0; i < nt; ++i) {
        if (R->trace_passes) R->trace_passes[i] = tr[i].passes;
        if (R->trace_active) R->trace_active[i] = tr[i].n_active;
        if (R->trace_gap) R->trace_gap[i] = tr[i].gap;
        if (R->trace_radius) R->trace_radius[i] = tr[i].radius;
    }
    R->n_trace = n_trace;
    R->n_active = S->m;
    return GS_OK;
}

static int ensure_trace(gs_solver* S, int64_t rows) {
    if (rows <= S->trace_cap) return GS_OK;
    cudaFree(S->trace);
    S->trace = nullptr;
    TRY(dalloc(&S->trace, rows));
    S->trace_cap = rows;
    return GS_OK;
}

extern "C" int gs_solver_solve(gs_solver* S, double lam, const gs_solve_config* cfg, const int64_t* active0,
                               int64_t n0, int active0_mode, gs_solve_result* R) {
    if (!(lam > 0)) return fail(GS_ERR_VALUE, "lambda must be positive");
    if (cfg->epsilon <= 0) return fail(GS_ERR_VALUE, "epsilon must be positive");
    if (cfg->screen_every < 1) return fail(GS_ERR_VALUE, "screen_every must be at least 1");
    if (cfg->max_passes < 1) return fail(GS_ERR_VALUE, "max_passes must be at least 1");
    const gs_matrix* M = S->M;
    cudaStream_t st = S->st;
    const int64_t p = S->p;
    const bool gap_rule = cfg->rule == GS_RULE_GAP_SPHERE;
    const bool certify = cfg->certify != 0;
    const int64_t f = cfg->screen_every;
    TRY(ensure_trace(S, cfg->max_passes / f + 4));
    DevScalars* h = S->hs;
    h->lam = lam; h->eps = cfg->epsilon; h->y_norm_sq = S->y_norm_sq;
    h->visits = h->uncertified = h->nonzero = 0;
    h->status = ST_OK;
    TRY(sc_upload(S));
    CK(cudaEventRecord(S->ev0, st));
    memset(&R->n_active, 0, sizeof(gs_solve_result) - offsetof(gs_solve_result, n_active));

    // ---- lambda >= lambda_max: _solve_at_lambda_max (solver.py:129-146, 160-161)
    if (lam >= S->lmax * (1 - 1e-14)) {
        CK(cudaMemsetAsync(S->beta, 0, p * 8, st));
        CK(cudaMemcpyAsync(S->rho, S->y, S->n * 8, cudaMemcpyDeviceToDevice, st));
        k_scale_vec<<<grid_for(S->n, 256), 256, 0, st>>>(S->y, lam, S->n, S->theta, 1);
        CKL();
        if (gap_rule) {
            TRY(screen_all(S, S->theta, nullptr, 0.0));
        } else {
            k_flags_norm_pos<<<grid_for(p, 256), 256, 0, st>>>(nullptr, p, M->norms, S->flags);
            CKL();
            TRY(launch_compact(st, S->s, S->flags, p, nullptr, S->A, &S->sc->m));
        }
        TRY(sc_download(S));
        S->m = h->m;
        TraceRow row{0, S->m, 0.0, 0.0};
        CK(cudaMemcpyAsync(S->trace, &row, sizeof row, cudaMemcpyHostToDevice, st));
        TRY(fire_hook(S, cfg));
        R->converged = 1; R->margin = 0.0; R->interpolating = 0; R->lambda_max_shortcut = 1;
        R->primal = 0.5 * S->y_norm_sq; R->dual = 0.5 * S->y_norm_sq; R->gap = 0.0;
        R->passes_done = 0; R->checkpoints = 0;
        TRY(solve_outputs(S, R, 1));
        S->has_prev = true; S->prev_margin = 0.0; S->prev_interp = 0;
        CK(cudaEventRecord(S->ev1, st));
        CK(cudaEventSynchronize(S->ev1));
        float ms = 0; cudaEventElapsedTime(&ms, S->ev0, S->ev1);
        R->device_ms = ms;
        return GS_OK;
    }

    // ---- active set init (solver.py:171-178): active0 filtered to nonzero norms
    if (active0_mode == 1) {
        TmpBuf tb;
        int32_t* d0 = nullptr;
        if (n0 > 0) {
            TRY(upload_cols(st, tb, M, active0, n0, &d0));
            CK(cudaMemcpyAsync(S->A2, d0, n0 * 4, cudaMemcpyDeviceToDevice, st));
        }
        k_flags_norm_pos<<<grid_for(std::max<int64_t>(n0, 1), 256), 256, 0, st>>>(S->A2, n0, M->norms, S->flags);
        CKL();
        TRY(launch_compact(st, S->s, S->flags, n0, S->A2, S->A, &S->sc->m));
        CK(cudaStreamSynchronize(st));
    } else if (active0_mode == 2) {
        const int64_t m0 = S->m;
        k_flags_norm_pos<<<grid_for(std::max<int64_t>(m0, 1), 256), 256, 0, st>>>(S->A, m0, M->norms, S->flags);
        CKL();
        TRY(launch_compact(st, S->s, S->flags, m0, S->A, S->A2, &S->sc->m));
        std::swap(S->A, S->A2);
    } else {
        k_flags_norm_pos<<<grid_for(p, 256), 256, 0, st>>>(nullptr, p, M->norms, S->flags);
        CKL();
        TRY(launch_compact(st, S->s, S->flags, p, nullptr, S->A, &S->sc->m));
    }
    CK(cudaMemcpyAsync(&S->hs->m, &S->sc->m, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    S->m = h->m;
    if (S->m > 0) {
        k_set_mark<<<grid_for(S->m, 256), 256, 0, st>>>(S->A, S->m, S->mark);
        CKL();
    }
    k_zero_unmarked<<<grid_for(p, 256), 256, 0, st>>>(S->beta, S->mark, p);
    CKL();

    int64_t passes = 0, ntrace = 0, nckpt = 0;
    bool converged = false;
    const double thresh = 1.0 - 1e-9;
    for (int64_t k = 1; k <= cfg->max_passes; ++k) {
        if (f == 1 || k % f == 1) {
            ++nckpt;
            TRY(resync(S));
            if (S->m == 0) {
                // everything screened: unrestricted dual point (solver.py:190-203)
                TRY(dual_corr(S, false));
                k_ckpt_dual<<<1, 1024, 0, st>>>(S->rho, S->y, (int)S->n, S->beta, S->A, 0, S->theta, S->sc, 0);
                CKL();
                k_ckpt_post<<<1, 1024, 0, st>>>(S->rho, (int)S->n, S->beta, S->A, S->sc, S->trace, ntrace, passes);
                CKL();
                TRY(sc_download(S));
                if (h->status != ST_OK) return status_error(h->status, h, false);
                ++ntrace;
                TRY(fire_hook(S, cfg));
                converged = h->gap_post <= cfg->epsilon;
                break;
            }
            TRY(dual_corr(S, true));
            k_ckpt_dual<<<1, 1024, 0, st>>>(S->rho, S->y, (int)S->n, S->beta, S->A, S->m, S->theta, S->sc, gap_rule ? 1 : 0);
            CKL();
            if (gap_rule) {
                k_ckpt_keep<<<grid_for(S->m, 256), 256, 0, st>>>(S->c, S->A, S->m, M->norms, S->beta, S->sc, thresh, S->flags, S->flags2);
                CKL();
                TRY(launch_compact(st, S->s, S->flags2, S->m, S->A, S->Dl, &S->sc->n_drop));
                if (M->sparse)
                    k_drop_axpy_csc<<<1, 256, 0, st>>>(M->data, M->indices, M->indptr, S->Dl, &S->sc->n_drop, S->beta, S->rho);
                else if (M->dtype == GS_DTYPE_F64)
                    k_drop_axpy_dense<double><<<(unsigned)((S->n + 255) / 256), 256, 0, st>>>((const double*)M->X, M->ld, (int)S->n, S->Dl, &S->sc->n_drop, S->beta, S->rho);
                else
                    k_drop_axpy_dense<float><<<(unsigned)((S->n + 255) / 256), 256, 0, st>>>((const float*)M->X, M->ld, (int)S->n, S->Dl, &S->sc->n_drop, S->beta, S->rho);
                k_zero_listed<<<grid_for(S->m, 256), 256, 0, st>>>(S->beta, S->Dl, &S->sc->n_drop);
                CKL();
                TRY(launch_compact(st, S->s, S->flags, S->m, S->A, S->A2, &S->sc->m));
                std::swap(S->A, S->A2);
            }
            k_ckpt_post<<<1, 1024, 0, st>>>(S->rho, (int)S->n, S->beta, S->A, S->sc, S->trace, ntrace, passes);
            CKL();
            TRY(sc_download(S));
            if (h->status != ST_OK) return status_error(h->status, h, false);
            S->m = h->m;
            ++ntrace;
            TRY(fire_hook(S, cfg));
            if (h->gap_post <= cfg->epsilon) { converged = true; break; }
            if (S->m == 0) break;
        } else if (k % 100 == 0) {
            TRY(resync(S));
            k_rho_norm_ub<<<1, 1024, 0, st>>>(S->rho, (int)S->n, S->sc);
            CKL();
        }
        TRY(cd_epoch(S, certify));
        ++passes;
    }
    double primal, dual, gap;
    if (!converged) {
        // budget exhausted or early break: certify the final iterate (solver.py:237-245)
        TRY(resync(S));
        TRY(dual_corr(S, S->m > 0));
        k_ckpt_dual<<<1, 1024, 0, st>>>(S->rho, S->y, (int)S->n, S->beta, S->A, S->m, S->theta, S->sc, 0);
        CKL();
        TRY(sc_download(S));
        if (h->status != ST_OK) return status_error(h->status, h, false);
        primal = h->primal; dual = h->dual; gap = h->gap_pre;
        converged = gap <= cfg->epsilon;
    } else {
        primal = h->primal_post; dual = h->dual; gap = h->gap_post;
    }
    R->converged = converged; R->margin = h->margin; R->interpolating = h->interp;
    R->primal = primal; R->dual = dual; R->gap = gap;
    R->passes_done = passes; R->checkpoints = nckpt;
    R->cd_visits = h->visits; R->cd_uncertified = h->uncertified; R->cd_nonzero = h->nonzero;
    TRY(solve_outputs(S, R, ntrace));
    S->has_prev = true; S->prev_margin = h->margin; S->prev_interp = h->interp;
    CK(cudaEventRecord(S->ev1, st));
    CK(cudaEventSynchronize(S->ev1));
    float ms = 0; cudaEventElapsedTime(&ms, S->ev0, S->ev1);
    R->device_ms = ms;
    return GS_OK;
}

// ---------------------------------------------------------------------------
// kernel twin: one CD epoch over a host active list
// ---------------------------------------------------------------------------
extern "C" int gs_cd_pass(const gs_matrix* M, double* beta, double* rho, const int64_t* active, int64_t k,
                          double lam, const double* norms_sq, double tail_scale, int exact_order) {
    TRY(ensure_device());
    cudaStream_t st = M->st;
    TmpBuf tb;
    const int64_t n = M->n, p = M->p;
    const int64_t nrho = n + (tail_scale > 0.0 ? p : 0);
    double *db, *dr, *dns, *dnorm;
    int32_t* dA = nullptr;
    TRY(tb.get(&db, p)); TRY(tb.get(&dr, nrho + 2));
    CK(cudaMemcpyAsync(db, beta, p * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dr, rho, nrho * 8, cudaMemcpyHostToDevice, st));
    if (k > 0) TRY(upload_cols(st, tb, M, active, k, &dA));
    if (norms_sq) {
        TRY(tb.get(&dns, p)); TRY(tb.get(&dnorm, p));
        CK(cudaMemcpyAsync(dns, norms_sq, p * 8, cudaMemcpyHostToDevice, st));
        k_sqrt_vec<<<grid_for(p, 256), 256, 0, st>>>(dns, 0.0, p, dns, dnorm);
        CKL();
    } else {
        dns = M->norms_sq; dnorm = M->norms;
    }
    if (k > 0) {
        if (exact_order || tail_scale > 0.0) {
            if (M->sparse)
                k_cd_pass_exact_csc<<<1, 256, 0, st>>>(M->data, M->indices, M->indptr, (int)n, db, dr, dA, k, lam, dns, tail_scale);
            else if (M->dtype == GS_DTYPE_F64)
                k_cd_pass_exact_dense<double><<<1, 256, 0, st>>>((const double*)M->X, M->ld, (int)n, db, dr, dA, k, lam, dns, tail_scale);
            else
                k_cd_pass_exact_dense<float><<<1, 256, 0, st>>>((const float*)M->X, M->ld, (int)n, db, dr, dA, k, lam, dns, tail_scale);
            CKL();
        } else {
            // production path: certification anchor at the incoming rho
            DevScalars* sc; double *c, *t;
            TRY(tb.get(&sc, 1)); TRY(tb.get(&c, k)); TRY(tb.get(&t, k));
            CK(cudaMemsetAsync(sc, 0, sizeof(DevScalars), st));
            k_rho_norm_ub<<<1, 1024, 0, st>>>(dr, (int)n, sc);
            Scratch s;
            TRY(s.alloc(k));
            GemvArgs a{};
            a.v = dr; a.cols = dA; a.m = k; a.mode = GEMV_CERT; a.out_c = c; a.out_t = t;
            a.blk_val = s.blk_val; a.blk_idx = s.blk_idx; a.norms = dnorm; a.beta = db; a.lam = lam;
            a.rho_norm_dev = &sc->rho_norm_ub; a.gam = gamma_n(n);
            int rc = launch_gemv(M, st, a, nullptr);
            if (rc == GS_OK) {
                CdArgs cda{};
                cda.ld = M->ld; cda.n = (int)n; cda.A = dA; cda.m = k; cda.tcert = t; cda.beta = db; cda.rho = dr;
                cda.nsq = dns; cda.norms = dnorm; cda.lam = lam; cda.sc = sc;
                rc = launch_cd(M, st, cda);
            }
            CK(cudaStreamSynchronize(st));
            s.release();
            if (rc != GS_OK) return rc;
        }
    }
    CK(cudaMemcpyAsync(beta, db, p * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rho, dr, nrho * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GS_OK;
}

// ---------------------------------------------------------------------------
// sphere screening over host inputs
// ---------------------------------------------------------------------------
extern "C" int gs_screen_sphere(const gs_matrix* M, const double* center, double radius, const int64_t* cols,
                                int64_t k, double tol, double* mu, int64_t* active_out, int64_t* n_active) {
    TRY(ensure_device());
    cudaStream_t st = M->st;
    TmpBuf tb;
    const int64_t m = cols ? k : M->p;
    double *dv, *dmu;
    int32_t *dcols = nullptr, *dout;
    uint8_t* flags;
    int64_t* dcount;
    TRY(tb.get(&dv, M->n + 2)); TRY(tb.get(&dmu, m)); TRY(tb.get(&dout, m)); TRY(tb.get(&flags, m));
    TRY(tb.get(&dcount, 1));
    CK(cudaMemcpyAsync(dv, center, M->n * 8, cudaMemcpyHostToDevice, st));
    if (cols && k > 0) TRY(upload_cols(st, tb, M, cols, k, &dcols));
    if (m == 0) { *n_active = 0; return GS_OK; }
    Scratch s;
    TRY(s.alloc(m));
    GemvArgs a{};
    a.v = dv; a.cols = dcols; a.m = m; a.mode = GEMV_MU; a.scale = 1.0; a.radius_host = radius;
    a.thresh = 1.0 - tol; a.norms = M->norms; a.out_mu = dmu; a.flags = flags;
    int rc = launch_gemv(M, st, a, nullptr);
    if (rc == GS_OK) rc = launch_compact(st, s, flags, m, dcols, dout, dcount);
    int64_t cnt = 0;
    if (rc == GS_OK) {
        CK(cudaMemcpyAsync(&cnt, dcount, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<int32_t> tmp(std::max<int64_t>(cnt, 1));
        if (cnt) CK(cudaMemcpyAsync(tmp.data(), dout, cnt * 4, cudaMemcpyDeviceToHost, st));
        if (mu) CK(cudaMemcpyAsync(mu, dmu, m * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t i = 0; i < cnt; ++i) active_out[i] = tmp[i];
        *n_active = cnt;
    }
    s.release();
    return rc;
}
