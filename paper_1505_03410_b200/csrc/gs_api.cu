// Host side of libgapsafe_b200: device-resident DesignMatrix, the primitive
// entry points and the solve / sequential-screen state machine
// (solver.py:149-246, path.py:82-91), all behind the C ABI of
// include/gapsafe_b200.h.
#include "../../include/gapsafe_b200.h"
#include "gs_solve.cuh"
#include "gs_launch.h"

#include <cmath>
#include <cstdlib>
#include <cstddef>

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
static int64_t g_launches = 0;   // kernels launched by this library (bench evidence)
#define COUNT_LAUNCH(k) (g_launches += (k))

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
    int64_t max_col_nnz = 0;                 // CSC: longest column
    void* X = nullptr;                       // dense
    double* data = nullptr;                  // CSC
    int32_t* indices = nullptr;
    int64_t* indptr = nullptr;
    double* csr_data = nullptr;              // CSR copy (resync row products)
    int32_t* csr_cols = nullptr;
    int64_t* csr_rowptr = nullptr;
    double* norms_sq = nullptr;
    double* norms = nullptr;
    double* inv_nsq = nullptr;                // RN(1/norms_sq)
    int64_t bytes = 0;
    cudaStream_t st = nullptr;
};

static void matrix_release(gs_matrix* M) {
    if (!M) return;
    cudaFree(M->X); cudaFree(M->data); cudaFree(M->indices); cudaFree(M->indptr);
    cudaFree(M->csr_data); cudaFree(M->csr_cols); cudaFree(M->csr_rowptr);
    cudaFree(M->norms_sq); cudaFree(M->norms); cudaFree(M->inv_nsq);
    if (M->st) cudaStreamDestroy(M->st);
    delete M;
}

static int matrix_norms(gs_matrix* M, const double* norms_sq_host) {
    TRY(dalloc(&M->norms_sq, M->p));
    TRY(dalloc(&M->norms, M->p));
    TRY(dalloc(&M->inv_nsq, M->p));
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
    k_sqrt_vec<<<grid_for(M->p, 256), 256, 0, M->st>>>(M->norms_sq, 0.0, M->p, M->norms_sq, M->norms, M->inv_nsq);
    CKL();
    CK(cudaStreamSynchronize(M->st));
    M->bytes += 3 * M->p * 8;
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
extern "C" int64_t gs_launch_count(void) { return g_launches; }

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
    for (int64_t j = 0; j < p; ++j) M->max_col_nnz = std::max<int64_t>(M->max_col_nnz, indptr[j + 1] - indptr[j]);
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

// dense design from a DEVICE buffer (column-major, ld_dev rows per column):
// device-to-device copy into owned storage, norms on the device.  Used by the
// column-sharded path: the survivors' columns arrive over NCCL in device
// memory and never touch the host (sharded.py).
extern "C" int gs_matrix_dense_dev(const void* X_dev, int dtype, int64_t n, int64_t p, int64_t ld_dev,
                                   gs_matrix** out) {
    TRY(ensure_device());
    if (n < 1 || p < 1) return fail(GS_ERR_VALUE, "matrix must have at least one row and column");
    if (n > (1 << 30)) return fail(GS_ERR_VALUE, "too many rows");
    if (dtype != GS_DTYPE_F64 && dtype != GS_DTYPE_F32) return fail(GS_ERR_VALUE, "dtype must be f64 or f32");
    if (ld_dev < n) return fail(GS_ERR_VALUE, "ld_dev must be at least n");
    gs_matrix* M = new gs_matrix();
    M->dtype = dtype; M->n = n; M->p = p;
    const size_t es = dtype == GS_DTYPE_F64 ? 8 : 4;
    const int64_t align = dtype == GS_DTYPE_F64 ? 2 : 4;
    M->ld = (n + align - 1) / align * align;
    int rc;
    if ((rc = [&]() -> int {
            CK(cudaStreamCreateWithFlags(&M->st, cudaStreamNonBlocking));
            CK(cudaMalloc(&M->X, (size_t)M->ld * p * es));
            M->bytes += (int64_t)M->ld * p * es;
            if (M->ld != n) CK(cudaMemsetAsync(M->X, 0, (size_t)M->ld * p * es, M->st));
            // the source was produced on another stream (torch / NCCL): the caller
            // synchronises it before this call; the copy itself is stream-ordered here
            CK(cudaMemcpy2DAsync(M->X, M->ld * es, X_dev, ld_dev * es, n * es, p, cudaMemcpyDeviceToDevice, M->st));
            return matrix_norms(M, nullptr);
        }()) != GS_OK) {
        matrix_release(M);
        return rc;
    }
    *out = M;
    return GS_OK;
}

// Dense design built block by block (designs larger than a comfortable host
// array: configs[2] is 40 GB): allocate zeroed device storage, upload column
// blocks from (reusable) host buffers, then compute the norms.
extern "C" int gs_matrix_dense_alloc(int dtype, int64_t n, int64_t p, gs_matrix** out) {
    TRY(ensure_device());
    if (n < 1 || p < 1) return fail(GS_ERR_VALUE, "matrix must have at least one row and column");
    if (n > (1 << 30)) return fail(GS_ERR_VALUE, "too many rows");
    if (dtype != GS_DTYPE_F64 && dtype != GS_DTYPE_F32) return fail(GS_ERR_VALUE, "dtype must be f64 or f32");
    gs_matrix* M = new gs_matrix();
    M->dtype = dtype; M->n = n; M->p = p;
    const size_t es = dtype == GS_DTYPE_F64 ? 8 : 4;
    const int64_t align = dtype == GS_DTYPE_F64 ? 2 : 4;
    M->ld = (n + align - 1) / align * align;
    int rc;
    if ((rc = [&]() -> int {
            CK(cudaStreamCreateWithFlags(&M->st, cudaStreamNonBlocking));
            CK(cudaMalloc(&M->X, (size_t)M->ld * p * es));
            M->bytes += (int64_t)M->ld * p * es;
            CK(cudaMemsetAsync(M->X, 0, (size_t)M->ld * p * es, M->st));
            CK(cudaStreamSynchronize(M->st));
            return GS_OK;
        }()) != GS_OK) {
        matrix_release(M);
        return rc;
    }
    *out = M;
    return GS_OK;
}

extern "C" int gs_matrix_dense_set_columns(gs_matrix* M, int64_t j0, int64_t k, const void* X, int64_t ld_host) {
    if (M->sparse || M->norms) return fail(GS_ERR_VALUE, "set_columns needs a dense design that is not finalized yet");
    if (j0 < 0 || k < 0 || j0 + k > M->p) return fail(GS_ERR_INDEX, "column block out of range");
    if (ld_host < M->n) return fail(GS_ERR_VALUE, "ld_host must be at least n");
    if (k == 0) return GS_OK;
    const size_t es = M->dtype == GS_DTYPE_F64 ? 8 : 4;
    CK(cudaMemcpy2DAsync((char*)M->X + (size_t)j0 * M->ld * es, M->ld * es, X, ld_host * es, M->n * es, k,
                         cudaMemcpyHostToDevice, M->st));
    CK(cudaStreamSynchronize(M->st));      // the host buffer may be reused on return
    return GS_OK;
}

extern "C" int gs_matrix_dense_finalize(gs_matrix* M) {
    if (M->sparse || M->norms) return fail(GS_ERR_VALUE, "finalize needs a dense design that is not finalized yet");
    return matrix_norms(M, nullptr);
}

template <typename T>
static __global__ void k_gather_cols(const T* __restrict__ X, int64_t ld, int n, const int64_t* __restrict__ idx,
                                     int64_t k, T* __restrict__ dst, int64_t ld_dst) {
    // one block per gathered column (grid-stride), threads over rows; rows n..ld_dst-1 zeroed
    for (int64_t c = blockIdx.x; c < k; c += gridDim.x) {
        const T* src = X + idx[c] * ld;
        T* d = dst + c * ld_dst;
        for (int64_t r = threadIdx.x; r < ld_dst; r += blockDim.x) d[r] = r < n ? src[r] : (T)0;
    }
}

// columns idx[0..k) of a dense design into a DEVICE buffer (column-major,
// ld_dst rows per column): the send buffer of the X_A gather
extern "C" int gs_matrix_gather_columns_dev(const gs_matrix* M, const int64_t* idx, int64_t k, void* dst_dev,
                                            int64_t ld_dst) {
    TRY(ensure_device());
    if (M->sparse) return fail(GS_ERR_VALUE, "column gather needs a dense design");
    if (ld_dst < M->n) return fail(GS_ERR_VALUE, "ld_dst must be at least n");
    if (k == 0) return GS_OK;
    for (int64_t c = 0; c < k; ++c)
        if (idx[c] < 0 || idx[c] >= M->p) return fail(GS_ERR_INDEX, "column index out of range");
    int64_t* didx = nullptr;
    TRY(dalloc(&didx, k));
    struct Free { void* q; ~Free() { cudaFree(q); } } guard{didx};
    CK(cudaMemcpyAsync(didx, idx, k * 8, cudaMemcpyHostToDevice, M->st));
    const unsigned grid = (unsigned)std::min<int64_t>(k, 148 * 8);
    if (M->dtype == GS_DTYPE_F64)
        k_gather_cols<double><<<grid, 256, 0, M->st>>>((const double*)M->X, M->ld, (int)M->n, didx, k, (double*)dst_dev, ld_dst);
    else
        k_gather_cols<float><<<grid, 256, 0, M->st>>>((const float*)M->X, M->ld, (int)M->n, didx, k, (float*)dst_dev, ld_dst);
    CKL();
    CK(cudaStreamSynchronize(M->st));     // the buffer is handed to another stream (NCCL) next
    return GS_OK;
}

extern "C" int gs_matrix_norms_sq(const gs_matrix* M, double* out) {
    CK(cudaMemcpyAsync(out, M->norms_sq, M->p * 8, cudaMemcpyDeviceToHost, M->st));
    CK(cudaStreamSynchronize(M->st));
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
    COUNT_LAUNCH(1);
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
    COUNT_LAUNCH(3);
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
        CK(cudaStreamSynchronize(st));   // callers copy dout on another stream
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
    CK(cudaMemcpyAsync(out, dout, M->n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
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

// ---------------------------------------------------------------------------
// persistent solve: launch configuration
// ---------------------------------------------------------------------------
constexpr int kSolveThreads = 256;

struct CdShape { int R, W; };

static CdShape cd_shape(int64_t n) {
    // rows per lane R (template) and CD warp-group size W: W*32*R >= n
    // W compute warps (one more warp is the producer, 8 warps per CTA)
    if (n <= 32) return {1, 1};
    if (n <= 64) return {2, 1};
    if (n <= 512) return {4, (int)((n + 127) / 128)};
    if (n <= 1792) return {8, (int)((n + 255) / 256)};
    if (n <= 10752) return {48, (int)((n + 1535) / 1536)};     // cfg2 (n = 10000): rho rows in registers, columns streamed
    return {0, 0};
}

// CD consumer per shape (measured on B200, profiles/r01/cd_modes.md): Gram
// windows win only for a single-warp chain (cfg0: 10.8 s vs 12.9 s); with a
// cross-warp reduction per coordinate (cfg1, cfg4) the direct chain is faster.
static int cd_gram_default(int64_t n) { return (cd_shape(n).R <= 4 && cd_shape(n).W == 1) ? 1 : 0; }

// blocked-chain consumer (gs_cd_blk.cuh): rows per thread R and compute warps
// NW <= 7 (the warp after them is the producer: threshold scan + TMA issue)
static CdShape cd_shape_blk(int64_t n) {
    if (n <= 32) return {1, 1};
    if (n <= 64) return {2, 1};
    if (n <= 128) return {4, 1};
    if (n <= 256) return {4, 2};
    if (n <= 512) return {4, 4};
    if (n <= 896) return {4, 7};
    if (n <= 1120) return {5, 7};     // cfg1 (n = 1000): 5 rows per thread, 7 compute warps
    return {0, 0};
}

// dense CD plan: consumer mode (0 direct, 1 Gram windows, 2 blocked chain;
// GS_CD_GRAM overrides), template R and warps.  The blocked chain is the
// default wherever it applies (n <= 1120).
struct CdPlan { int mode, R, W; };
static CdPlan cd_plan(int64_t n) {
    const char* eg = getenv("GS_CD_GRAM");
    int mode = eg ? atoi(eg) : (cd_shape_blk(n).R ? 2 : cd_gram_default(n));
    if (mode == 2 && cd_shape_blk(n).R == 0) mode = 0;
    const CdShape s = mode == 2 ? cd_shape_blk(n) : cd_shape(n);
    return {mode, s.R, s.W};
}
static int blk_mfac() {
    const char* e = getenv("GS_BLK_MFAC");
    return e ? atoi(e) : 32;
}

static int launch_solve(const gs_matrix* M, cudaStream_t st, const SolveDev* dprobs, int G, int nprob, size_t smem,
                        int R) {
    const bool f64 = M->sparse || M->dtype == GS_DTYPE_F64;
    COUNT_LAUNCH(1);
    CK(f64 ? gs_launch_solve_f64(R, st, dprobs, G, nprob, smem) : gs_launch_solve_f32(R, st, dprobs, G, nprob, smem));
    return GS_OK;
}

static int launch_cdpass(const gs_matrix* M, cudaStream_t st, const SolveDev* dprobs, size_t smem, int R) {
    const bool f64 = M->sparse || M->dtype == GS_DTYPE_F64;
    COUNT_LAUNCH(1);
    CK(f64 ? gs_launch_cdpass_f64(R, st, dprobs, smem) : gs_launch_cdpass_f32(R, st, dprobs, smem));
    return GS_OK;
}

static int vs_cap_for(const gs_matrix* M) { return M->sparse ? 24576 : 6144; }

static size_t cd_bytes_for(const gs_matrix* M) {
    if (M->sparse) return 0;
    const int es = M->dtype == GS_DTYPE_F64 ? 8 : 4;
    const size_t b = std::max(cd_smem_bytes_rt(M->ld, es), cd_shape_blk(M->n).R ? blk_smem_bytes(M->ld, es) : (size_t)0);
    return (b + 15) / 16 * 16;
}

// GEMV modes per shape (gs_solve.cuh): whole-CTA column reduction for dense
// columns of 16 KB and more; 8 lanes per column for short CSC columns
static bool gemv_wide_for(const gs_matrix* M) {
    if (M->sparse) return false;
    const char* e = getenv("GS_GEMV_WIDE");
    if (e) return atoi(e) != 0 && M->n <= 256 * kWideRows;
    const int64_t colb = M->ld * (M->dtype == GS_DTYPE_F64 ? 8 : 4);
    return colb >= 16 * 1024 && M->n <= 256 * kWideRows;
}
static bool csc_short_for(const gs_matrix* M) {
    if (!M->sparse) return false;
    const char* e = getenv("GS_CSC_SHORT");
    if (e) return atoi(e) != 0;
    return M->p > 0 && M->nnz <= 24 * M->p;
}

static size_t solve_smem(const gs_matrix* M) {
    const int64_t n = M->n;
    const size_t vs = (n <= vs_cap_for(M) && !gemv_wide_for(M)) ? (size_t)(n + 2) * 8 : 0;
    if (M->sparse) return std::max(vs, cd_csc_smem_bytes(n));
    size_t b = cd_bytes_for(M) + vs;     // dense: CD tile + column ring stay resident beside the GEMV staging
    if (gemv_wide_for(M)) {
        // the column ring of the wide GEMV takes all of it: as many whole columns as fit (up to 8)
        const size_t colb = (size_t)M->ld * (M->dtype == GS_DTYPE_F64 ? 8 : 4);
        const size_t cap = 216 * 1024;          // leaves room for the kernels' static shared memory
        const size_t want = std::min<size_t>((cap - kWidePartBytes) / colb, kWideSlots) * colb + kWidePartBytes;
        b = std::max(b, want);
    }
    return b;
}

// shared-memory / GEMV plan fields of a SolveDev
static void set_plan(const gs_matrix* M, SolveDev& d) {
    d.vs_cap = gemv_wide_for(M) ? 0 : vs_cap_for(M);
    d.cd_bytes = (int)cd_bytes_for(M);
    d.gemv_wide = gemv_wide_for(M) ? 1 : 0;
    d.csc_short = csc_short_for(M) ? 1 : 0;
    d.smem_total = (int)solve_smem(M);
    const char* efl = getenv("GS_CSC_FLAT");
    d.csc_flat = efl ? atoi(efl) : 1;
    const char* el2 = getenv("GS_L2_HINT");
    d.l2_hint = el2 ? atoi(el2) : 1;
    const char* els = getenv("GS_LDS_EXPLICIT");
    d.lds_explicit = els ? atoi(els) : 1;
    const char* ech = getenv("GS_CD_CHUNK");
    d.cd_chunk_pos = M->sparse ? (ech ? atoi(ech) : 16384) : 0;   // cfg3 sweep: 2048 -> 219 s, 16384 -> 201 s
}

static int check_shape(const gs_matrix* M) {
    if (M->sparse) {
        if (solve_smem(M) > 225 * 1024) return fail(GS_ERR_VALUE, "sparse solver supports n <= 22400 in this build");
        return GS_OK;
    }
    if (cd_shape(M->n).R == 0) return fail(GS_ERR_VALUE, "dense solver supports n <= 10752 in this build");
    return GS_OK;
}

// ---------------------------------------------------------------------------
// solver
// ---------------------------------------------------------------------------
struct gs_solver {
    const gs_matrix* M = nullptr;
    cudaStream_t st = nullptr;
    int64_t n = 0, p = 0;
    double *y = nullptr, *beta = nullptr, *rho = nullptr, *theta = nullptr, *c = nullptr;
    ColInfo* cinfo = nullptr;
    float *t = nullptr, *t2 = nullptr;
    int32_t *A = nullptr, *A2 = nullptr, *S = nullptr, *Dl = nullptr;
    uint8_t *flags = nullptr, *mark = nullptr;
    double* partial = nullptr;
    int nch_max = 0;
    Scratch s;
    DevScalars* sc = nullptr;     // device
    DevScalars* hs = nullptr;     // pinned host mirror
    SolveCtl* ctl = nullptr;
    SolveCtl* hctl = nullptr;
    GroupBar* bar = nullptr;
    double* cta_val = nullptr;
    int64_t* cta_idx = nullptr;
    int64_t* cta_cnt = nullptr;
    SolveDev* dprob = nullptr;
    TraceRow* trace = nullptr;
    int64_t trace_cap = 0;
    int G = 1;
    double lmax = 0.0, y_norm_sq = 0.0;
    int64_t jstar = 0;
    int* rowmark = nullptr;       // [n] row map of the parallel CSC waves
    double* q = nullptr;          // X^T y (static / dynamic / ST3 / dome centres)
    double* gstar = nullptr;      // X^T x_jstar (ST3), built on first use
    bool gstar_ready = false;
    int64_t m = 0;                // active count after the last solve
    bool has_prev = false, seq_pending = false;
    double seq_lam = 0.0;
    double prev_margin = 1.0;
    int prev_interp = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t tev0 = nullptr, tev1 = nullptr;   // gs_solver_timer (bench)
};

static void solver_release(gs_solver* S) {
    if (!S) return;
    cudaFree(S->y); cudaFree(S->beta); cudaFree(S->rho); cudaFree(S->theta); cudaFree(S->c); cudaFree(S->cinfo);
    cudaFree(S->t); cudaFree(S->t2);
    cudaFree(S->A); cudaFree(S->A2); cudaFree(S->S); cudaFree(S->Dl);
    cudaFree(S->flags); cudaFree(S->mark); cudaFree(S->partial);
    cudaFree(S->sc); cudaFreeHost(S->hs); cudaFree(S->ctl); cudaFreeHost(S->hctl); cudaFree(S->bar);
    cudaFree(S->cta_val); cudaFree(S->cta_idx); cudaFree(S->cta_cnt); cudaFree(S->dprob); cudaFree(S->trace);
    cudaFree(S->q); cudaFree(S->gstar); cudaFree(S->rowmark);
    S->s.release();
    if (S->ev0) cudaEventDestroy(S->ev0);
    if (S->ev1) cudaEventDestroy(S->ev1);
    if (S->tev0) cudaEventDestroy(S->tev0);
    if (S->tev1) cudaEventDestroy(S->tev1);
    if (S->st) cudaStreamDestroy(S->st);
    delete S;
}

static int sc_upload(gs_solver* S) {
    CK(cudaMemcpyAsync(S->sc, S->hs, sizeof(DevScalars), cudaMemcpyHostToDevice, S->st));
    return GS_OK;
}
static int sc_download(gs_solver* S) {
    CK(cudaMemcpyAsync(S->hs, S->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, S->st));
    CK(cudaMemcpyAsync(S->hctl, S->ctl, sizeof(SolveCtl), cudaMemcpyDeviceToHost, S->st));
    CK(cudaStreamSynchronize(S->st));
    return GS_OK;
}

// CTAs cooperating on one problem: enough to stream the design at HBM rate,
// few enough that the group barrier stays cheap for small problems.
static int choose_group(const gs_matrix* M) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* env = getenv("GS_GROUP_CTAS");
    if (env && atoi(env) > 0) return std::min(atoi(env), sms);
    const double bytes = M->sparse ? (double)M->nnz * 12.0 : (double)M->ld * M->p * (M->dtype == GS_DTYPE_F64 ? 8 : 4);
    // one CTA per 512 KiB of design: even a 4 MB design (cfg0) runs its restricted GEMVs and
    // compactions faster on 8 CTAs than the group barrier costs (5.87 s -> 4.68 s measured)
    const int g = (int)std::ceil(bytes / (512.0 * 1024.0));
    return std::max(1, std::min(sms, g));
}

extern "C" int gs_solver_create(const gs_matrix* M, const double* y, gs_solver** out) {
    TRY(ensure_device());
    TRY(check_shape(M));
    gs_solver* S = new gs_solver();
    S->M = M; S->n = M->n; S->p = M->p;
    int rc = [&]() -> int {
        const int64_t n = S->n, p = S->p;
        S->G = choose_group(M);
        CK(cudaStreamCreateWithFlags(&S->st, cudaStreamNonBlocking));
        CK(cudaEventCreate(&S->ev0)); CK(cudaEventCreate(&S->ev1));
        CK(cudaEventCreate(&S->tev0)); CK(cudaEventCreate(&S->tev1));
        TRY(dalloc(&S->y, n + 2)); TRY(dalloc(&S->rho, n + 2)); TRY(dalloc(&S->theta, n + 2));
        TRY(dalloc(&S->beta, p)); TRY(dalloc(&S->c, p)); TRY(dalloc(&S->cinfo, p)); TRY(dalloc(&S->t, p)); TRY(dalloc(&S->t2, p));
        TRY(dalloc(&S->A, p)); TRY(dalloc(&S->A2, p)); TRY(dalloc(&S->S, p)); TRY(dalloc(&S->Dl, p));
        TRY(dalloc(&S->flags, p)); TRY(dalloc(&S->mark, p));
        S->nch_max = (int)std::min<int64_t>(256, std::max<int64_t>(1, (p + 15) / 16));
        if (!M->sparse) TRY(dalloc(&S->partial, (size_t)S->nch_max * n));
        TRY(S->s.alloc(p));
        TRY(dalloc(&S->sc, 1)); TRY(dalloc(&S->ctl, 1)); TRY(dalloc(&S->bar, 1));
        TRY(dalloc(&S->cta_val, S->G)); TRY(dalloc(&S->cta_idx, S->G)); TRY(dalloc(&S->cta_cnt, 2 * S->G));
        TRY(dalloc(&S->dprob, 1));
        CK(cudaMallocHost((void**)&S->hs, sizeof(DevScalars)));
        CK(cudaMallocHost((void**)&S->hctl, sizeof(SolveCtl)));
        memset(S->hs, 0, sizeof(DevScalars));
        memset(S->hctl, 0, sizeof(SolveCtl));
        CK(cudaMemsetAsync(S->bar, 0, sizeof(GroupBar), S->st));
        CK(cudaMemsetAsync(S->mark, 0, p, S->st));
        CK(cudaMemsetAsync(S->beta, 0, p * 8, S->st));
        CK(cudaMemsetAsync(S->y, 0, (n + 2) * 8, S->st));
        CK(cudaMemsetAsync(S->rho, 0, (n + 2) * 8, S->st));
        CK(cudaMemsetAsync(S->theta, 0, (n + 2) * 8, S->st));
        CK(cudaMemcpyAsync(S->y, y, n * 8, cudaMemcpyHostToDevice, S->st));
        TRY(sc_upload(S));
        // lambda_max = |X^T y|_inf, j_star (problem.py:50), ||y||^2 (problem.py:54)
        TRY(dalloc(&S->q, p));
        if (M->sparse) {
            TRY(dalloc(&S->rowmark, n + 1));
            CK(cudaMemsetAsync(S->rowmark, 0x7f, (n + 1) * sizeof(int), S->st));
        }
        GemvArgs a{};
        a.v = S->y; a.m = p; a.mode = GEMV_MAX; a.blk_val = S->s.blk_val; a.blk_idx = S->s.blk_idx;
        a.out_c = S->q;                    // X^T y kept for the static/dynamic/ST3/dome centres
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

extern "C" int gs_solver_set_lambda_max(gs_solver* S, double lambda_max) {
    if (!S) return fail(GS_ERR_VALUE, "null solver");
    if (!(lambda_max > 0)) return fail(GS_ERR_VALUE, "lambda_max must be positive");
    S->lmax = lambda_max;
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

static int status_error(int32_t st, double margin, double gap) {
    char buf[256];
    if (st == ST_INFEASIBLE) {
        snprintf(buf, sizeof buf, "dual point infeasible: margin=%.17g", margin);
        return fail(GS_ERR_INFEASIBLE, buf);
    }
    if (st == ST_NEG_GAP) {
        snprintf(buf, sizeof buf, "negative duality gap / inner radius beyond tolerance: %.17g", gap);
        return fail(GS_ERR_NUMERICAL, buf);
    }
    if (st == ST_VALUE) return fail(GS_ERR_VALUE, "theta must be dual feasible");
    return GS_OK;
}

static int copy_active_host(gs_solver* S, int64_t m, int64_t* out) {
    std::vector<int32_t> tmp(std::max<int64_t>(m, 1));
    if (m) CK(cudaMemcpyAsync(tmp.data(), S->A, m * 4, cudaMemcpyDeviceToHost, S->st));
    CK(cudaStreamSynchronize(S->st));
    for (int64_t i = 0; i < m; ++i) out[i] = tmp[i];
    return GS_OK;
}

// Sequential screen of path.py:82-91: runs fused at the start of the next
// solve (init_mode 2) from the device-resident previous (beta, theta, rho).
extern "C" int gs_solver_seq_screen(gs_solver* S, double lam, int64_t* n_active) {
    if (!S->has_prev) return fail(GS_ERR_VALUE, "sequential screen needs a previous solve");
    S->seq_pending = true;
    S->seq_lam = lam;
    if (n_active) *n_active = -1;
    return GS_OK;
}

static int solve_outputs(gs_solver* S, gs_solve_result* R, int64_t n_trace, int64_t m) {
    cudaStream_t st = S->st;
    if (R->beta) CK(cudaMemcpyAsync(R->beta, S->beta, S->p * 8, cudaMemcpyDeviceToHost, st));
    if (R->residual) CK(cudaMemcpyAsync(R->residual, S->rho, S->n * 8, cudaMemcpyDeviceToHost, st));
    if (R->theta) CK(cudaMemcpyAsync(R->theta, S->theta, S->n * 8, cudaMemcpyDeviceToHost, st));
    if (R->active) TRY(copy_active_host(S, m, R->active));
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
    R->n_active = m;
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

static void fill_dev(gs_solver* S, SolveDev& d) {
    const gs_matrix* M = S->M;
    memset(&d, 0, sizeof d);
    d.X = M->X; d.ld = M->ld; d.n = (int)M->n; d.dtype = M->dtype; d.p = M->p; d.sparse = M->sparse;
    d.data = M->data; d.indices = M->indices; d.indptr = M->indptr;
    d.csr_data = M->csr_data; d.csr_cols = M->csr_cols; d.csr_rowptr = M->csr_rowptr;
    d.norms = M->norms; d.nsq = M->norms_sq; d.inv_nsq = M->inv_nsq;
    d.y = S->y; d.cinfo = S->cinfo; d.beta = S->beta; d.rho = S->rho; d.theta = S->theta; d.c = S->c; d.t = S->t; d.t2 = S->t2;
    d.A = S->A; d.A2 = S->A2; d.S = S->S; d.Dl = S->Dl; d.mark = S->mark;
    d.partial = S->partial; d.nch_max = S->nch_max;
    d.sc = S->sc; d.ctl = S->ctl; d.trace = S->trace; d.trace_cap = S->trace_cap; d.bar = S->bar;
    d.cta_val = S->cta_val; d.cta_idx = S->cta_idx; d.cta_cnt = S->cta_cnt;
    const CdPlan cs = cd_plan(M->n);
    d.cd_warps = M->sparse ? 1 : cs.W;
    d.blk_mfac = blk_mfac();
    set_plan(M, d);
    const char* env = getenv("GS_REFRESH_EXCESS");
    d.refresh_excess = env ? atoi(env) : 32;
    d.cd_gram = cs.mode;
    const char* ep = getenv("GS_CD_PROF");
    d.cd_prof = ep ? atoi(ep) : 0;
    d.q = S->q; d.gstar = S->gstar; d.lmax_path = S->lmax; d.jstar = S->jstar;
    d.rowmark = S->rowmark;
    // CSC waves: fully parallel when rows are plentiful relative to column
    // length (conflicts between a wave's members are rare); otherwise the
    // conflict-free admission (profiles/r01/cd_modes.md)
    const char* ec = getenv("GS_CSC_PAR");
    d.csc_par = ec ? atoi(ec) : (M->sparse && M->n >= 256 * std::max<int64_t>(M->max_col_nnz, 1) ? 1 : 0);
}

// column j of the design as a dense f64 n-vector (regions.py:187: X.matvec(e_j))
static __global__ void k_densify_col(const void* X, int dtype, int64_t ld, const double* data, const int32_t* indices,
                                     const int64_t* indptr, int sparse, int64_t j, int n, double* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (sparse) {          // out was zeroed by the caller
        if (blockIdx.x == 0)
            for (int64_t q = indptr[j] + threadIdx.x; q < indptr[j + 1]; q += blockDim.x) out[indices[q]] = data[q];
    } else if (r < n) {
        out[r] = dtype == GS_DTYPE_F64 ? ((const double*)X)[j * ld + r] : (double)((const float*)X)[j * ld + r];
    }
}

// gstar = X^T x_jstar for the ST3 centre (regions.py:186-196), once per solver
static int ensure_gstar(gs_solver* S) {
    if (S->gstar_ready) return GS_OK;
    const gs_matrix* M = S->M;
    cudaStream_t st = S->st;
    if (!S->gstar) TRY(dalloc(&S->gstar, S->p));
    double* col;
    TRY(dalloc(&col, S->n + 2));
    CK(cudaMemsetAsync(col, 0, (S->n + 2) * 8, st));
    const int blocks = M->sparse ? 1 : (int)((S->n + 255) / 256);
    if (M->sparse && S->n > 0) {
        // one block: zero then scatter (single-block kernel keeps the order)
        k_densify_col<<<1, 1024, 0, st>>>(nullptr, 0, 0, M->data, M->indices, M->indptr, 1, S->jstar, 0, col);
    } else {
        k_densify_col<<<blocks, 256, 0, st>>>(M->X, M->dtype, M->ld, nullptr, nullptr, nullptr, 0, S->jstar,
                                              (int)S->n, col);
    }
    CKL();
    GemvArgs a{};
    a.v = col; a.m = S->p; a.mode = GEMV_RAW; a.out_c = S->gstar;
    TRY(launch_gemv(M, st, a, nullptr));
    CK(cudaStreamSynchronize(st));
    cudaFree(col);
    S->gstar_ready = true;
    return GS_OK;
}

extern "C" int gs_solver_solve(gs_solver* S, double lam, const gs_solve_config* cfg, const int64_t* active0,
                               int64_t n0, int active0_mode, gs_solve_result* R) {
    if (!(lam > 0)) return fail(GS_ERR_VALUE, "lambda must be positive");
    if (cfg->epsilon <= 0) return fail(GS_ERR_VALUE, "epsilon must be positive");
    if (cfg->screen_every < 1) return fail(GS_ERR_VALUE, "screen_every must be at least 1");
    if (cfg->max_passes < 1) return fail(GS_ERR_VALUE, "max_passes must be at least 1");
    if (cfg->rule < GS_RULE_NONE || cfg->rule > GS_RULE_GAP_DOME) return fail(GS_ERR_VALUE, "unknown rule");
    if (active0_mode == 2 && !(S->seq_pending && S->seq_lam == lam))
        return fail(GS_ERR_VALUE, "active0_mode 2 needs gs_solver_seq_screen at the same lambda");
    if (active0_mode == 2 && cfg->rule != GS_RULE_GAP_SPHERE && cfg->rule != GS_RULE_GAP_DOME)
        return fail(GS_ERR_VALUE, "the sequential screen is defined for the gap sphere and gap dome rules");
    S->seq_pending = false;
    const gs_matrix* M = S->M;
    cudaStream_t st = S->st;
    if (cfg->rule == GS_RULE_ST3) TRY(ensure_gstar(S));
    const int64_t p = S->p;
    const bool screening = cfg->rule != GS_RULE_NONE;
    const int64_t f = cfg->screen_every;
    TRY(ensure_trace(S, cfg->max_passes / f + 4));
    DevScalars* h = S->hs;
    h->lam = lam; h->eps = cfg->epsilon; h->y_norm_sq = S->y_norm_sq;
    h->visits = h->uncertified = h->nonzero = 0;
    h->status = ST_OK;
    h->m = S->m;
    CK(cudaEventRecord(S->ev0, st));
    memset(&R->n_active, 0, sizeof(gs_solve_result) - offsetof(gs_solve_result, n_active));

    // ---- lambda >= lambda_max: _solve_at_lambda_max (solver.py:129-146, 160-161)
    if (lam >= S->lmax * (1 - 1e-14)) {
        TRY(sc_upload(S));
        CK(cudaMemsetAsync(S->beta, 0, p * 8, st));
        CK(cudaMemcpyAsync(S->rho, S->y, S->n * 8, cudaMemcpyDeviceToDevice, st));
        k_scale_vec<<<grid_for(S->n, 256), 256, 0, st>>>(S->y, lam, S->n, S->theta, 1);
        CKL();
        if (screening) {
            GemvArgs a{};
            a.v = S->theta; a.m = p; a.mode = GEMV_MU; a.scale = 1.0; a.radius_host = 0.0;
            a.thresh = 1.0 - 1e-9; a.norms = M->norms; a.flags = S->flags;
            TRY(launch_gemv(M, st, a, nullptr));
        } else {
            k_flags_norm_pos<<<grid_for(p, 256), 256, 0, st>>>(nullptr, p, M->norms, S->flags);
            CKL();
        }
        TRY(launch_compact(st, S->s, S->flags, p, nullptr, S->A, &S->sc->m));
        TRY(sc_download(S));
        S->m = h->m;
        TraceRow row{0, S->m, 0.0, 0.0};
        CK(cudaMemcpyAsync(S->trace, &row, sizeof row, cudaMemcpyHostToDevice, st));
        if (cfg->on_checkpoint) {
            std::vector<int64_t> act(std::max<int64_t>(S->m, 1));
            TRY(copy_active_host(S, S->m, act.data()));
            cfg->on_checkpoint(act.data(), S->m, cfg->user);
        }
        R->converged = 1; R->margin = 0.0; R->interpolating = 0; R->lambda_max_shortcut = 1;
        R->primal = 0.5 * S->y_norm_sq; R->dual = 0.5 * S->y_norm_sq; R->gap = 0.0;
        R->passes_done = 0; R->checkpoints = 0;
        TRY(solve_outputs(S, R, 1, S->m));
        S->has_prev = true; S->prev_margin = 0.0; S->prev_interp = 0;
        CK(cudaEventRecord(S->ev1, st));
        CK(cudaEventSynchronize(S->ev1));
        float ms = 0; cudaEventElapsedTime(&ms, S->ev0, S->ev1);
        R->device_ms = ms;
        return GS_OK;
    }

    // ---- the persistent solve
    if (active0_mode == 1) {
        // the device marks the listed columns (the active set is their
        // ascending, duplicate-free compaction), so a list is deduplicated
        // here: at most p entries reach S->A2 (p slots)
        std::vector<char> seen((size_t)p, 0);
        std::vector<int32_t> c32;
        c32.reserve((size_t)std::min<int64_t>(std::max<int64_t>(n0, 1), p));
        for (int64_t i = 0; i < n0; ++i) {
            if (active0[i] < 0 || active0[i] >= p) return fail(GS_ERR_INDEX, "active0 index out of range");
            if (!seen[(size_t)active0[i]]) { seen[(size_t)active0[i]] = 1; c32.push_back((int32_t)active0[i]); }
        }
        const int64_t nu = (int64_t)c32.size();
        if (nu) {
            CK(cudaMemcpyAsync(S->A2, c32.data(), nu * 4, cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));   // c32 is a host temporary
        }
        h->cnt = nu;
    }
    TRY(sc_upload(S));
    memset(S->hctl, 0, sizeof(SolveCtl));
    CK(cudaMemcpyAsync(S->ctl, S->hctl, sizeof(SolveCtl), cudaMemcpyHostToDevice, st));
    SolveDev d;
    fill_dev(S, d);
    d.lam = lam; d.eps = cfg->epsilon; d.max_passes = cfg->max_passes; d.f = f;
    d.rule = cfg->rule; d.certify = cfg->certify; d.stop_at_ckpt = cfg->on_checkpoint ? 1 : 0;
    d.init_mode = active0_mode == 2 ? 2 : (active0_mode == 1 ? 1 : 0);
    d.prev_margin = S->prev_margin;
    CK(cudaMemcpyAsync(S->dprob, &d, sizeof d, cudaMemcpyHostToDevice, st));
    const size_t smem = solve_smem(M);
    const int Rr = M->sparse ? 1 : cd_plan(M->n).R;
    int64_t hook_fired = 0, launches = 0;
    while (true) {
        TRY(launch_solve(M, st, S->dprob, S->G, 1, smem, Rr));
        ++launches;
        TRY(sc_download(S));
        const SolveCtl* c = S->hctl;
        if (h->status != ST_OK) {
            S->has_prev = false;
            return status_error(h->status, h->margin, h->gap_pre);
        }
        if (cfg->on_checkpoint && c->nckpt > hook_fired) {
            std::vector<int64_t> act(std::max<int64_t>(h->m, 1));
            TRY(copy_active_host(S, h->m, act.data()));
            cfg->on_checkpoint(act.data(), h->m, cfg->user);
            hook_fired = c->nckpt;
        }
        if (c->done) break;
    }
    const SolveCtl* c = S->hctl;
    S->m = h->m;
    R->converged = c->converged;
    R->margin = h->margin; R->interpolating = h->interp;
    if (c->final_done) { R->primal = h->primal; R->dual = h->dual; R->gap = h->gap_pre; }
    else { R->primal = h->primal_post; R->dual = h->dual; R->gap = h->gap_post; }
    R->passes_done = c->passes; R->checkpoints = c->nckpt;
    R->cd_visits = h->visits; R->cd_uncertified = h->uncertified; R->cd_nonzero = h->nonzero;
    R->screen_ms = c->t_screen * 1e-6; R->ckpt_ms = c->t_ckpt * 1e-6;
    R->refresh_ms = c->t_refresh * 1e-6; R->cd_ms = c->t_cd * 1e-6;
    R->n_screen = c->n_screen; R->n_refresh = c->n_refresh; R->launches = launches;
    R->cd_candidates = c->n_cand; R->cd_skipped = c->n_skip; R->cd_requeues = c->n_requeue;
    TRY(solve_outputs(S, R, c->ntrace, S->m));
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
    double *db, *dr, *dns, *dnorm, *dinv;
    ColInfo* dci;
    int32_t* dA = nullptr;
    TRY(tb.get(&db, p)); TRY(tb.get(&dr, nrho + 2)); TRY(tb.get(&dci, p));
    CK(cudaMemcpyAsync(db, beta, p * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dr, rho, nrho * 8, cudaMemcpyHostToDevice, st));
    if (k > 0) TRY(upload_cols(st, tb, M, active, k, &dA));
    if (norms_sq) {
        TRY(tb.get(&dns, p)); TRY(tb.get(&dnorm, p)); TRY(tb.get(&dinv, p));
        CK(cudaMemcpyAsync(dns, norms_sq, p * 8, cudaMemcpyHostToDevice, st));
        k_sqrt_vec<<<grid_for(p, 256), 256, 0, st>>>(dns, 0.0, p, dns, dnorm, dinv);
        CKL();
    } else {
        dns = M->norms_sq; dnorm = M->norms; dinv = M->inv_nsq;
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
            TRY(check_shape(M));
            DevScalars* sc; SolveCtl* ctl; double* c; float* t; SolveDev* dp; double* cval; int64_t* cidx;
            TRY(tb.get(&sc, 1)); TRY(tb.get(&ctl, 1)); TRY(tb.get(&c, k)); TRY(tb.get(&t, k)); TRY(tb.get(&dp, 1));
            TRY(tb.get(&cval, 1)); TRY(tb.get(&cidx, 1));
            DevScalars hs{};
            hs.m = k;
            CK(cudaMemcpyAsync(sc, &hs, sizeof hs, cudaMemcpyHostToDevice, st));
            CK(cudaMemsetAsync(ctl, 0, sizeof(SolveCtl), st));
            SolveDev d;
            memset(&d, 0, sizeof d);
            d.X = M->X; d.ld = M->ld; d.n = (int)n; d.dtype = M->dtype; d.p = p; d.sparse = M->sparse;
            d.data = M->data; d.indices = M->indices; d.indptr = M->indptr;
            d.norms = dnorm; d.nsq = dns; d.inv_nsq = dinv; d.cinfo = dci; d.beta = db; d.rho = dr; d.c = c; d.t = t; d.A = dA;
            d.sc = sc; d.ctl = ctl; d.lam = lam; d.certify = 1; d.cta_val = cval; d.cta_idx = cidx;
            const CdPlan cp = cd_plan(n);
            d.cd_gram = cp.mode;
            d.blk_mfac = blk_mfac();
            d.cd_warps = M->sparse ? 1 : cp.W;
            set_plan(M, d);
            CK(cudaMemcpyAsync(dp, &d, sizeof d, cudaMemcpyHostToDevice, st));
            TRY(launch_cdpass(M, st, dp, solve_smem(M), M->sparse ? 1 : cp.R));
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

// ---------------------------------------------------------------------------
// measurement support
// ---------------------------------------------------------------------------
extern "C" int gs_solver_timer(gs_solver* S, int op, double* ms) {
    if (op == 0) {
        CK(cudaStreamSynchronize(S->st));
        CK(cudaEventRecord(S->tev0, S->st));
        return GS_OK;
    }
    CK(cudaEventRecord(S->tev1, S->st));
    CK(cudaEventSynchronize(S->tev1));
    float f = 0.0f;
    CK(cudaEventElapsedTime(&f, S->tev0, S->tev1));
    if (ms) *ms = f;
    return GS_OK;
}

extern "C" int gs_screen_timed(const gs_matrix* M, const double* center, double radius, int reps, double* ms,
                               int64_t* n_active, int32_t* active_out) {
    TRY(ensure_device());
    if (reps < 1) reps = 1;
    cudaStream_t st = M->st;
    TmpBuf tb;
    double* dv; uint8_t* mark; int32_t* out; int64_t* cnt; SolveDev* dp;
    TRY(tb.get(&dv, M->n + 2)); TRY(tb.get(&mark, M->p)); TRY(tb.get(&out, M->p)); TRY(tb.get(&cnt, 1));
    TRY(tb.get(&dp, 1));
    CK(cudaMemcpyAsync(dv, center, M->n * 8, cudaMemcpyHostToDevice, st));
    SolveDev d;
    memset(&d, 0, sizeof d);
    d.X = M->X; d.ld = M->ld; d.n = (int)M->n; d.dtype = M->dtype; d.p = M->p; d.sparse = M->sparse;
    d.data = M->data; d.indices = M->indices; d.indptr = M->indptr; d.norms = M->norms; d.nsq = M->norms_sq;
    d.inv_nsq = M->inv_nsq;
    d.theta = dv; d.mark = mark;
    set_plan(M, d);
    CK(cudaMemcpyAsync(dp, &d, sizeof d, cudaMemcpyHostToDevice, st));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = solve_smem(M);
    Scratch s;
    TRY(s.alloc(M->p));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    int rc = GS_OK;
    const bool f64 = M->sparse || M->dtype == GS_DTYPE_F64;
    auto gemv = [&]() -> int {
        COUNT_LAUNCH(1);
        CK(f64 ? gs_launch_screen_full_f64(st, dp, radius, sms, smem) : gs_launch_screen_full_f32(st, dp, radius, sms, smem));
        return GS_OK;
    };
    // warm-up pass (GEMV + compaction), then `reps` GEMV launches timed with
    // events on this stream (the design, > L2, is streamed from HBM each time)
    rc = gemv();
    if (rc == GS_OK) rc = launch_compact(st, s, mark, M->p, nullptr, out, cnt);
    if (rc == GS_OK) {
        CK(cudaEventRecord(e0, st));
        for (int r = 0; r < reps && rc == GS_OK; ++r) rc = gemv();
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float f = 0.0f;
        cudaEventElapsedTime(&f, e0, e1);
        *ms = f / reps;
        CK(cudaMemcpyAsync(n_active, cnt, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (active_out && *n_active > 0) {
            // survivors of the warm-up pass (the timed launches recompute the same marks)
            CK(cudaMemcpyAsync(active_out, out, (size_t)*n_active * 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    s.release();
    return rc;
}

extern "C" int gs_host_alloc(int64_t bytes, void** out) {
    TRY(ensure_device());
    CK(cudaMallocHost(out, (size_t)std::max<int64_t>(bytes, 1)));
    return GS_OK;
}

extern "C" void gs_host_free(void* ptr) { cudaFreeHost(ptr); }

// ---------------------------------------------------------------------------
// batched independent problems (cfg4): one CTA per problem, whole path on device
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ X0, int64_t ld0, const int32_t* __restrict__ rows, int n,
                              int64_t ld, int64_t p, int64_t B, T* __restrict__ Xb) {
    // block (j-chunk, b); threads over rows
    const int64_t b = blockIdx.y;
    const int32_t* rw = rows + b * n;
    T* dst = Xb + b * ld * p;
    for (int64_t j = blockIdx.x; j < p; j += gridDim.x) {
        const T* col = X0 + j * ld0;
        for (int r = threadIdx.x; r < ld; r += blockDim.x) dst[j * ld + r] = r < n ? col[rw[r]] : (T)0;
    }
}

__global__ void k_gather_y(const double* __restrict__ y0, const int32_t* __restrict__ rows, int n, int64_t B,
                           double* __restrict__ yb, int64_t ldy) {
    const int64_t b = blockIdx.x;
    for (int r = threadIdx.x; r < ldy; r += blockDim.x) yb[b * ldy + r] = r < n ? y0[rows[b * n + r]] : 0.0;
}

struct gs_batch {
    int64_t B = 0, n = 0, p = 0, ld = 0, ldy = 0;
    int dtype = GS_DTYPE_F64;
    gs_matrix shape;                  // shape descriptor (no storage) for launch configuration
    void* X = nullptr;                // B designs, column-major, ld rows each
    double *y = nullptr, *norms_sq = nullptr, *norms = nullptr, *inv = nullptr;
    double *beta = nullptr, *rho = nullptr, *theta = nullptr, *c = nullptr;
    ColInfo* cinfo = nullptr;
    float *t = nullptr, *t2 = nullptr;
    int32_t *A = nullptr, *A2 = nullptr, *S = nullptr, *Dl = nullptr;
    uint8_t* mark = nullptr;
    double* partial = nullptr;
    int nch_max = 1;
    DevScalars* sc = nullptr;
    SolveCtl* ctl = nullptr;
    TraceRow* trace = nullptr;
    int64_t trace_cap = 0;
    double* cta_val = nullptr;
    int64_t* cta_idx = nullptr;
    int64_t* cta_cnt = nullptr;
    SolveDev* dprobs = nullptr;
    BatchOut* douts = nullptr;
    std::vector<double> lmax;
    std::vector<double> ynsq;
    cudaStream_t st = nullptr;
};

static void batch_release(gs_batch* Bt) {
    if (!Bt) return;
    void* ptrs[] = {Bt->X, Bt->y, Bt->norms_sq, Bt->norms, Bt->inv, Bt->beta, Bt->rho, Bt->theta, Bt->c,
                    Bt->cinfo, Bt->t, Bt->t2, Bt->A, Bt->A2, Bt->S, Bt->Dl, Bt->mark, Bt->partial, Bt->sc,
                    Bt->ctl, Bt->trace, Bt->cta_val, Bt->cta_idx, Bt->cta_cnt, Bt->dprobs, Bt->douts};
    for (void* q : ptrs) cudaFree(q);
    if (Bt->st) cudaStreamDestroy(Bt->st);
    delete Bt;
}

extern "C" int gs_batch_create(const gs_matrix* X0, const double* y0, const int32_t* rows, int64_t B, int64_t n,
                               gs_batch** out) {
    TRY(ensure_device());
    if (X0->sparse) return fail(GS_ERR_VALUE, "batched problems need a dense design");
    if (B < 1 || n < 1) return fail(GS_ERR_VALUE, "batch needs B >= 1 problems of n >= 1 rows");
    for (int64_t i = 0; i < B * n; ++i)
        if (rows[i] < 0 || rows[i] >= X0->n) return fail(GS_ERR_INDEX, "row index out of range");
    gs_batch* Bt = new gs_batch();
    int rc = [&]() -> int {
        Bt->B = B; Bt->n = n; Bt->p = X0->p; Bt->dtype = X0->dtype;
        const int64_t align = X0->dtype == GS_DTYPE_F64 ? 2 : 4;
        Bt->ld = (n + align - 1) / align * align;
        Bt->ldy = n + 2;
        Bt->shape.n = n; Bt->shape.p = X0->p; Bt->shape.ld = Bt->ld; Bt->shape.dtype = X0->dtype;
        if (cd_shape(n).R == 0 || cd_shape(n).R > 8) return fail(GS_ERR_VALUE, "batched solver supports n <= 1792");
        const int64_t p = Bt->p, ld = Bt->ld;
        const size_t es = X0->dtype == GS_DTYPE_F64 ? 8 : 4;
        CK(cudaStreamCreateWithFlags(&Bt->st, cudaStreamNonBlocking));
        cudaStream_t st = Bt->st;
        CK(cudaMalloc(&Bt->X, (size_t)B * ld * p * es));
        TRY(dalloc(&Bt->y, B * Bt->ldy)); TRY(dalloc(&Bt->norms_sq, B * p)); TRY(dalloc(&Bt->norms, B * p));
        TRY(dalloc(&Bt->inv, B * p)); TRY(dalloc(&Bt->beta, B * p)); TRY(dalloc(&Bt->rho, B * Bt->ldy));
        TRY(dalloc(&Bt->theta, B * Bt->ldy)); TRY(dalloc(&Bt->c, B * p)); TRY(dalloc(&Bt->cinfo, B * p));
        TRY(dalloc(&Bt->t, B * p)); TRY(dalloc(&Bt->t2, B * p)); TRY(dalloc(&Bt->A, B * p));
        TRY(dalloc(&Bt->A2, B * p)); TRY(dalloc(&Bt->S, B * p)); TRY(dalloc(&Bt->Dl, B * p));
        TRY(dalloc(&Bt->mark, B * p));
        Bt->nch_max = (int)std::min<int64_t>(32, std::max<int64_t>(1, (p + 15) / 16));
        TRY(dalloc(&Bt->partial, B * Bt->nch_max * n));
        TRY(dalloc(&Bt->sc, B)); TRY(dalloc(&Bt->ctl, B));
        TRY(dalloc(&Bt->cta_val, B)); TRY(dalloc(&Bt->cta_idx, B)); TRY(dalloc(&Bt->cta_cnt, 2 * B));
        TRY(dalloc(&Bt->dprobs, B)); TRY(dalloc(&Bt->douts, B));
        CK(cudaMemsetAsync(Bt->mark, 0, B * p, st));
        CK(cudaMemsetAsync(Bt->beta, 0, B * p * 8, st));
        CK(cudaMemsetAsync(Bt->rho, 0, B * Bt->ldy * 8, st));
        CK(cudaMemsetAsync(Bt->theta, 0, B * Bt->ldy * 8, st));
        CK(cudaMemsetAsync(Bt->sc, 0, B * sizeof(DevScalars), st));
        int32_t* drows;
        TRY(dalloc(&drows, B * n));
        CK(cudaMemcpyAsync(drows, rows, B * n * 4, cudaMemcpyHostToDevice, st));
        double* dy0;
        TRY(dalloc(&dy0, X0->n));
        CK(cudaMemcpyAsync(dy0, y0, X0->n * 8, cudaMemcpyHostToDevice, st));
        dim3 gg((unsigned)std::min<int64_t>(p, 4096), (unsigned)B);
        if (X0->dtype == GS_DTYPE_F64)
            k_gather_rows<double><<<gg, 256, 0, st>>>((const double*)X0->X, X0->ld, drows, (int)n, ld, p, B, (double*)Bt->X);
        else
            k_gather_rows<float><<<gg, 256, 0, st>>>((const float*)X0->X, X0->ld, drows, (int)n, ld, p, B, (float*)Bt->X);
        k_gather_y<<<(unsigned)B, 256, 0, st>>>(dy0, drows, (int)n, B, Bt->y, Bt->ldy);
        CKL();
        // column norms of all B * p columns at once
        if (X0->dtype == GS_DTYPE_F64)
            k_col_norms_sq_dense<double><<<grid_for(B * p * 32, 256), 256, 0, st>>>((const double*)Bt->X, ld, (int)n, B * p, Bt->norms_sq);
        else
            k_col_norms_sq_dense<float><<<grid_for(B * p * 32, 256), 256, 0, st>>>((const float*)Bt->X, ld, (int)n, B * p, Bt->norms_sq);
        k_sqrt_vec<<<grid_for(B * p, 256), 256, 0, st>>>(Bt->norms_sq, 0.0, B * p, Bt->norms_sq, Bt->norms, Bt->inv);
        CKL();
        // lambda_max and ||y||^2 per problem
        Scratch sc;
        TRY(sc.alloc(p));
        double *dval, *dvs;
        int64_t* didx;
        TRY(dalloc(&dval, B)); TRY(dalloc(&didx, B)); TRY(dalloc(&dvs, 2 * B));
        for (int64_t b = 0; b < B; ++b) {
            gs_matrix Mb = Bt->shape;
            Mb.X = (char*)Bt->X + (size_t)b * ld * p * es;
            GemvArgs a{};
            a.v = Bt->y + b * Bt->ldy; a.m = p; a.mode = GEMV_MAX; a.blk_val = sc.blk_val; a.blk_idx = sc.blk_idx;
            int64_t nb = 0;
            TRY(launch_gemv(&Mb, st, a, &nb));
            k_max_finalize<<<1, 1024, 0, st>>>(sc.blk_val, sc.blk_idx, nb, dval + b, didx + b);
            k_vec_stats<<<1, 1024, 0, st>>>(Bt->y + b * Bt->ldy, Bt->y + b * Bt->ldy, n, dvs + 2 * b);
        }
        CKL();
        Bt->lmax.resize(B);
        std::vector<double> vs(2 * B);
        CK(cudaMemcpyAsync(Bt->lmax.data(), dval, B * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(vs.data(), dvs, 2 * B * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        Bt->ynsq.resize(B);
        for (int64_t b = 0; b < B; ++b) Bt->ynsq[b] = vs[2 * b];
        sc.release();
        cudaFree(dval); cudaFree(didx); cudaFree(dvs); cudaFree(drows); cudaFree(dy0);
        return GS_OK;
    }();
    if (rc != GS_OK) { batch_release(Bt); return rc; }
    *out = Bt;
    return GS_OK;
}

extern "C" int gs_batch_lambda_max(gs_batch* Bt, double* lmax) {
    for (int64_t b = 0; b < Bt->B; ++b) lmax[b] = Bt->lmax[b];
    return GS_OK;
}

extern "C" void gs_batch_free(gs_batch* Bt) { batch_release(Bt); }

extern "C" int gs_batch_run_paths(gs_batch* Bt, const double* grids, int64_t T, const gs_solve_config* cfg,
                                  const double* eps, double* betas, int64_t* passes, double* gaps,
                                  int32_t* converged, int64_t* n_active, double* device_ms) {
    // eps: per-problem gap tolerances [B] (solver.py:37,226 takes epsilon per
    // solve); NULL runs every problem at cfg->epsilon
    if (!eps && cfg->epsilon <= 0) return fail(GS_ERR_VALUE, "epsilon must be positive");
    if (eps)
        for (int64_t b = 0; b < Bt->B; ++b)
            if (!(eps[b] > 0)) return fail(GS_ERR_VALUE, "epsilon must be positive");
    if (cfg->screen_every < 1 || cfg->max_passes < 1) return fail(GS_ERR_VALUE, "bad solver configuration");
    if (cfg->on_checkpoint) return fail(GS_ERR_VALUE, "checkpoint hooks are not available in batched mode");
    if (cfg->rule != GS_RULE_NONE && cfg->rule != GS_RULE_GAP_SPHERE)
        return fail(GS_ERR_VALUE, "batched problems run the none / gap_sphere rules");
    const int64_t B = Bt->B, p = Bt->p, n = Bt->n, ld = Bt->ld;
    cudaStream_t st = Bt->st;
    const size_t es = Bt->dtype == GS_DTYPE_F64 ? 8 : 4;
    const int64_t cap = cfg->max_passes / cfg->screen_every + 4;
    if (cap * B > Bt->trace_cap) {
        cudaFree(Bt->trace);
        TRY(dalloc(&Bt->trace, cap * B));
        Bt->trace_cap = cap * B;
    }
    double *dgrid, *dbetas = nullptr, *dgaps;
    int64_t *dpasses, *dnact;
    int32_t* dconv;
    TmpBuf tb;
    TRY(tb.get(&dgrid, B * T)); TRY(tb.get(&dgaps, B * T)); TRY(tb.get(&dpasses, B * T));
    TRY(tb.get(&dnact, B * T)); TRY(tb.get(&dconv, B * T));
    if (betas) TRY(tb.get(&dbetas, B * T * p));
    CK(cudaMemcpyAsync(dgrid, grids, B * T * 8, cudaMemcpyHostToDevice, st));
    std::vector<SolveDev> probs(B);
    std::vector<BatchOut> outs(B);
    std::vector<DevScalars> hsc(B);
    const CdPlan cs = cd_plan(n);
    for (int64_t b = 0; b < B; ++b) {
        SolveDev& d = probs[b];
        memset(&d, 0, sizeof d);
        d.X = (char*)Bt->X + (size_t)b * ld * p * es; d.ld = ld; d.n = (int)n; d.dtype = Bt->dtype; d.p = p;
        d.norms = Bt->norms + b * p; d.nsq = Bt->norms_sq + b * p; d.inv_nsq = Bt->inv + b * p;
        d.y = Bt->y + b * Bt->ldy; d.beta = Bt->beta + b * p; d.rho = Bt->rho + b * Bt->ldy;
        d.theta = Bt->theta + b * Bt->ldy; d.cinfo = Bt->cinfo + b * p; d.c = Bt->c + b * p;
        d.t = Bt->t + b * p; d.t2 = Bt->t2 + b * p; d.A = Bt->A + b * p; d.A2 = Bt->A2 + b * p;
        d.S = Bt->S + b * p; d.Dl = Bt->Dl + b * p; d.mark = Bt->mark + b * p;
        d.partial = Bt->partial + b * Bt->nch_max * n; d.nch_max = Bt->nch_max;
        d.sc = Bt->sc + b; d.ctl = Bt->ctl + b; d.trace = Bt->trace + b * cap; d.trace_cap = cap;
        d.cta_val = Bt->cta_val + b; d.cta_idx = Bt->cta_idx + b; d.cta_cnt = Bt->cta_cnt + 2 * b;
        d.eps = eps ? eps[b] : cfg->epsilon; d.max_passes = cfg->max_passes; d.f = cfg->screen_every; d.rule = cfg->rule;
        d.certify = cfg->certify; d.cd_warps = cs.W;
        set_plan(&Bt->shape, d);
        const char* env = getenv("GS_REFRESH_EXCESS");
        d.refresh_excess = env ? atoi(env) : 32;
        d.cd_gram = cs.mode;
        d.blk_mfac = blk_mfac();
        BatchOut& o = outs[b];
        o.grid = dgrid + b * T; o.lmax = Bt->lmax[b]; o.betas = dbetas ? dbetas + b * T * p : nullptr;
        o.passes = dpasses + b * T; o.gaps = dgaps + b * T; o.converged = dconv + b * T; o.n_active = dnact + b * T;
        o.T = (int)T;
        memset(&hsc[b], 0, sizeof(DevScalars));
        hsc[b].eps = d.eps; hsc[b].y_norm_sq = Bt->ynsq[b];
    }
    CK(cudaMemcpyAsync(Bt->dprobs, probs.data(), B * sizeof(SolveDev), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(Bt->douts, outs.data(), B * sizeof(BatchOut), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(Bt->sc, hsc.data(), B * sizeof(DevScalars), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(Bt->beta, 0, B * p * 8, st));
    const size_t smem = solve_smem(&Bt->shape);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    COUNT_LAUNCH(1);
    const bool f64 = Bt->dtype == GS_DTYPE_F64;
    CK(f64 ? gs_launch_batch_f64(cs.R, st, Bt->dprobs, Bt->douts, (int)B, smem)
        : gs_launch_batch_f32(cs.R, st, Bt->dprobs, Bt->douts, (int)B, smem));
    CKL();
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (passes) CK(cudaMemcpyAsync(passes, dpasses, B * T * 8, cudaMemcpyDeviceToHost, st));
    if (gaps) CK(cudaMemcpyAsync(gaps, dgaps, B * T * 8, cudaMemcpyDeviceToHost, st));
    if (converged) CK(cudaMemcpyAsync(converged, dconv, B * T * 4, cudaMemcpyDeviceToHost, st));
    if (n_active) CK(cudaMemcpyAsync(n_active, dnact, B * T * 8, cudaMemcpyDeviceToHost, st));
    if (betas) CK(cudaMemcpyAsync(betas, dbetas, B * T * p * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (converged)
        for (int64_t i = 0; i < B * T; ++i)
            if (converged[i] < 0) return fail(GS_ERR_NUMERICAL, "a batched problem hit an infeasible / negative-gap status");
    return GS_OK;
}
