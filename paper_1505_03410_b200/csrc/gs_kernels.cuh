// sm_100a kernels of the Gap Safe Lasso hot path.
//
//   k_gemv_t_*      screening / restricted X^T v pass (A2, A4, A5b, A6) with
//                   fused epilogues: |.|-argmax, sphere test mu >= 1 - tol,
//                   per-column certification thresholds for the CD kernel.
//   k_compact_*     stable (ascending) stream compaction of surviving indices.
//   k_resync_*      residual rho = y - X beta over the support only (A5a).
//   k_ckpt_*        checkpoint scalar algebra: Eq. 10 dual point, P, D, G,
//                   radius, drop axpys, post-drop certificate, trace (A5b-d).
//   k_cd_epoch_*    one cyclic CD epoch over the active set, one CTA per
//                   problem, with exact certified-zero skipping (A7).
//   k_*_exact       kernel-level twins of _kernels.py in the reference's own
//                   summation order (sequential, non-FMA) for bit-exact tests.
#pragma once
#include "gs_device.cuh"

namespace gs {

// ---------------------------------------------------------------------------
// device-resident scalar block of one solve (read back once per checkpoint)
// ---------------------------------------------------------------------------
struct DevScalars {
    // problem
    double lam, eps, y_norm_sq;
    // dual point (problem.py:98-123)
    double rho_sq, y_rho, corr, alpha, margin;
    int64_t corr_arg;
    int32_t interp, status;
    // certificates (problem.py:57-86, regions.py:213-218)
    double l1, primal, dual, gap_pre, radius, primal_post, gap_post, radius_post;
    // certification anchor
    double rho_norm_ub;
    // screening-rule region (regions.py:159-273): |theta - y/lam|^2, radius,
    // ST3 centre coefficient, dome outer radius R, ball radius R/2, cut ratio;
    // trace radius for the rules whose trace reports the region radius
    double dsq, rule_r, rule_coef, rule_R, rule_rd, rule_a, rule_trace_r;
    int32_t rule_trace_fixed, rule_pad;
    // counts
    int64_t m;            // active-set size
    int64_t cnt;          // generic compaction output count
    int64_t n_supp;       // support size (resync)
    int64_t n_drop;       // dropped columns with beta != 0
    // CD statistics
    unsigned long long visits, uncertified, nonzero;
};

struct TraceRow { int64_t passes, n_active; double gap, radius; };

enum Status : int32_t {
    ST_OK = 0,
    ST_INFEASIBLE = 1,     // InfeasibleDualError   (problem.py:74-76)
    ST_NEG_GAP = 2,        // NumericalInconsistencyError (regions.py:215-217, 266-268)
    ST_VALUE = 3,          // ValueError: dome/dynamic/ST3 centre infeasible (regions.py:170, 183, 258)
};

enum RuleId : int32_t { R_NONE = 0, R_GAP_SPHERE = 1, R_STATIC = 2, R_DYNAMIC = 3, R_ST3 = 4, R_GAP_DOME = 5 };

// Dome support test (regions.py:82-97) for the gap dome of regions.py:250-273:
// qy = x^T y / lam, th = x^T theta, centre (y/lam + theta)/2, unit normal
// (y/lam - theta)/R, ball radius r = R/2, clamped cut ratio a.
__device__ __forceinline__ double dome_mu(double qy, double th, double R, double r, double a, double nrm) {
    if (R == 0.0) return fabs(th);                       // Sphere(theta, 0)
    const double ct = 0.5 * qy + 0.5 * th;
    const double nt = (qy - th) / R;
    const double cross = r * sqrt(fmax(nrm * nrm - nt * nt, 0.0) * (1.0 - a * a));
    const double sp = (nt < -a * nrm) ? ct + r * nrm : ct - r * a * nt + cross;
    const double sn = (-nt < -a * nrm) ? -ct + r * nrm : -ct + r * a * nt + cross;
    return fmax(sp, sn);
}

// ---------------------------------------------------------------------------
// column dot products (warp per column), fixed order, FMA
// ---------------------------------------------------------------------------
template <typename T> struct ColDot;

template <> struct ColDot<double> {
    // ld must be even: column start is 16-B aligned, rows read as double2.
    static __device__ __forceinline__ double run(const double* __restrict__ x,
                                                 const double* __restrict__ v, int n, int lane) {
        const double2* x2 = reinterpret_cast<const double2*>(x);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const int n2 = n >> 1;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
        for (int q = lane; q < n2; q += kWarp) {
            const double2 xv = __ldg(x2 + q);
            const double2 vv = v2[q];
            a0 = fma(xv.x, vv.x, a0);
            a1 = fma(xv.y, vv.y, a1);
        }
        if ((n & 1) && lane == 0) a0 = fma(__ldg(x + n - 1), v[n - 1], a0);
        return warp_sum(a0 + a1);
    }
};

template <> struct ColDot<float> {
    // ld must be a multiple of 4: rows read as float4.
    static __device__ __forceinline__ double run(const float* __restrict__ x,
                                                 const double* __restrict__ v, int n, int lane) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const int n4 = n >> 2;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int q = lane; q < n4; q += kWarp) {
            const float4 xv = __ldg(x4 + q);
            const double2 va = v2[2 * q], vb = v2[2 * q + 1];
            a0 = fma((double)xv.x, va.x, a0);
            a1 = fma((double)xv.y, va.y, a1);
            a0 = fma((double)xv.z, vb.x, a0);
            a1 = fma((double)xv.w, vb.y, a1);
        }
        for (int r = (n4 << 2) + lane; r < n; r += kWarp) a0 = fma((double)__ldg(x + r), v[r], a0);
        return warp_sum(a0 + a1);
    }
};


// two columns per warp in flight (doubles the bytes in flight per warp);
// per-column summation order identical to ColDot<T>::run.
template <typename T> struct ColDot2;

template <> struct ColDot2<double> {
    static __device__ __forceinline__ void run(const double* __restrict__ x0, const double* __restrict__ x1,
                                               const double* __restrict__ v, int n, int lane, double& c0,
                                               double& c1) {
        const double2* p0 = reinterpret_cast<const double2*>(x0);
        const double2* p1 = reinterpret_cast<const double2*>(x1);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const int n2 = n >> 1;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll 8
        for (int q = lane; q < n2; q += kWarp) {
            const double2 xa = __ldg(p0 + q);
            const double2 xb = __ldg(p1 + q);
            const double2 vv = v2[q];
            a0 = fma(xa.x, vv.x, a0);
            a1 = fma(xa.y, vv.y, a1);
            b0 = fma(xb.x, vv.x, b0);
            b1 = fma(xb.y, vv.y, b1);
        }
        if ((n & 1) && lane == 0) {
            a0 = fma(__ldg(x0 + n - 1), v[n - 1], a0);
            b0 = fma(__ldg(x1 + n - 1), v[n - 1], b0);
        }
        double s0 = a0 + a1, s1 = b0 + b1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        c0 = s0;
        c1 = s1;
    }
};

template <> struct ColDot2<float> {
    static __device__ __forceinline__ void run(const float* __restrict__ x0, const float* __restrict__ x1,
                                               const double* __restrict__ v, int n, int lane, double& c0,
                                               double& c1) {
        const float4* p0 = reinterpret_cast<const float4*>(x0);
        const float4* p1 = reinterpret_cast<const float4*>(x1);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const int n4 = n >> 2;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll 4
        for (int q = lane; q < n4; q += kWarp) {
            const float4 xa = __ldg(p0 + q);
            const float4 xb = __ldg(p1 + q);
            const double2 va = v2[2 * q], vb = v2[2 * q + 1];
            a0 = fma((double)xa.x, va.x, a0);
            a1 = fma((double)xa.y, va.y, a1);
            a0 = fma((double)xa.z, vb.x, a0);
            a1 = fma((double)xa.w, vb.y, a1);
            b0 = fma((double)xb.x, va.x, b0);
            b1 = fma((double)xb.y, va.y, b1);
            b0 = fma((double)xb.z, vb.x, b0);
            b1 = fma((double)xb.w, vb.y, b1);
        }
        for (int r = (n4 << 2) + lane; r < n; r += kWarp) {
            a0 = fma((double)__ldg(x0 + r), v[r], a0);
            b0 = fma((double)__ldg(x1 + r), v[r], b0);
        }
        double s0 = a0 + a1, s1 = b0 + b1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        c0 = s0;
        c1 = s1;
    }
};

// one column out of shared memory; per-lane partition, accumulation order and
// butterfly identical to ColDot2 (bit-identical results)
template <typename T> struct ColDotS;

template <> struct ColDotS<double> {
    static __device__ __forceinline__ double run(const double* x, const double* v, int n, int lane) {
        const double2* p = reinterpret_cast<const double2*>(x);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const int n2 = n >> 1;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int q = lane; q < n2; q += kWarp) {
            const double2 xa = p[q];
            const double2 vv = v2[q];
            a0 = fma(xa.x, vv.x, a0);
            a1 = fma(xa.y, vv.y, a1);
        }
        if ((n & 1) && lane == 0) a0 = fma(x[n - 1], v[n - 1], a0);
        double s = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        return s;
    }
};

template <> struct ColDotS<float> {
    static __device__ __forceinline__ double run(const float* x, const double* v, int n, int lane) {
        const float4* p = reinterpret_cast<const float4*>(x);
        const double2* v2 = reinterpret_cast<const double2*>(v);
        const int n4 = n >> 2;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int q = lane; q < n4; q += kWarp) {
            const float4 xa = p[q];
            const double2 va = v2[2 * q], vb = v2[2 * q + 1];
            a0 = fma((double)xa.x, va.x, a0);
            a1 = fma((double)xa.y, va.y, a1);
            a0 = fma((double)xa.z, vb.x, a0);
            a1 = fma((double)xa.w, vb.y, a1);
        }
        for (int r = (n4 << 2) + lane; r < n; r += kWarp) a0 = fma((double)x[r], v[r], a0);
        double s = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        return s;
    }
};

// ---------------------------------------------------------------------------
// screening / restricted GEMV with fused epilogues
// ---------------------------------------------------------------------------
enum GemvMode : int {
    GEMV_RAW = 0,    // out_c[i] = x_{j}^T v
    GEMV_MAX = 1,    // + per-block max |c| (smallest index on ties)
    GEMV_MU = 2,     // sphere test: mu = |c| * scale + r * ||x_j||; flags = mu >= thresh
    GEMV_CERT = 3,   // out_c, per-column certification threshold out_t, + block max
};

struct GemvArgs {
    int64_t ld;
    int n;
    const double* v;           // [n]
    const int32_t* cols;       // nullable -> identity (i -> column i)
    int64_t m;                 // number of columns processed
    int cpb;                   // columns per block
    int mode;
    double* out_c;             // [m] nullable
    double* blk_val;           // [grid] (MAX, CERT)
    int64_t* blk_idx;          // [grid]
    // MU
    double scale;
    const double* radius_dev;  // nullable -> radius_host
    double radius_host;
    double thresh;             // 1 - tol
    const double* norms;       // [p] column norms
    double* out_mu;            // [m] nullable
    uint8_t* flags;            // [m]
    // CERT
    double* out_t;             // [m]
    const double* beta;        // [p]
    double lam;
    const double* rho_norm_dev;
    double gam;                // gamma_n
};

// Certification threshold: with
// c = fl(x^T rho0) and Delta >= ||rho - rho0||, the CD kernel's own dot
// g = fl(x^T rho) obeys |g| <= |c| + 2 gam ||x|| ||rho0|| + (1+gam)^2 ||x|| Delta,
// so Delta < t guarantees |g| <= lam, hence z = fl(g/nsq) in [-u, u], hence a
// zero update (for beta_j == 0).  All operations round toward the safe side.
__device__ __forceinline__ double cert_threshold(double c, double norm, double lam,
                                                 double rho0, double gam) {
    const double k = 1.0 + 4.0 * gam + 1e-13;
    // certified against lam (1 - 1e-15): |g| stays a few ulps inside lam, so the blocked
    // chain's z = fl(g * RN(1/nsq)) (no division) is still within [-u, u] for u = RN(lam/nsq)
    const double lam_s = __dmul_rd(lam, 1.0 - 1e-15);
    const double num = __dsub_rd(__dsub_rd(lam_s, fabs(c)), __dmul_ru(__dmul_ru(2.0 * k, gam), __dmul_ru(norm, rho0)));
    const double den = __dmul_ru(norm, __dmul_ru(k, k));
    if (!(num > 0.0)) return -1.0;
    return __ddiv_rd(num, den);
}

template <typename T, bool VSMEM>
static __global__ void __launch_bounds__(256) k_gemv_t_dense(const T* __restrict__ X, GemvArgs a) {
    extern __shared__ double smem_v[];
    __shared__ double s_val[8];
    __shared__ int64_t s_idx[8];
    __shared__ int s_cnt[8];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * a.cpb;
    const int64_t i1 = min(a.m, i0 + (int64_t)a.cpb);
    if (VSMEM) {
        for (int r = tid; r < a.n; r += blockDim.x) smem_v[r] = a.v[r];
        if (tid == 0 && (a.n & 1)) smem_v[a.n] = 0.0;
        __syncthreads();
    }
    const double* v = VSMEM ? smem_v : a.v;
    const double radius = (a.mode == GEMV_MU) ? (a.radius_dev ? *a.radius_dev : a.radius_host) : 0.0;
    const double rho0 = (a.mode == GEMV_CERT) ? *a.rho_norm_dev : 0.0;
    double bmax = -1.0;
    int64_t barg = INT64_MAX;
    int cnt = 0;
    for (int64_t i = i0 + w; i < i1; i += nw) {
        const int64_t j = a.cols ? (int64_t)a.cols[i] : i;
        const double c = ColDot<T>::run(X + j * a.ld, v, a.n, lane);
        if (lane == 0) {
            if (a.out_c) a.out_c[i] = c;
            if (a.mode == GEMV_MAX || a.mode == GEMV_CERT) argmax_merge(bmax, barg, fabs(c), i);
            if (a.mode == GEMV_MU) {
                const double mu = fabs(c) * a.scale + radius * a.norms[j];
                if (a.out_mu) a.out_mu[i] = mu;
                const bool keep = mu >= a.thresh;
                a.flags[i] = keep;
                cnt += keep;
            } else if (a.mode == GEMV_CERT) {
                a.out_t[i] = (a.beta[j] != 0.0) ? -1.0 : cert_threshold(c, a.norms[j], a.lam, rho0, a.gam);
            }
        }
    }
    if (a.mode == GEMV_MAX || a.mode == GEMV_CERT) {
        if (lane == 0) { s_val[w] = bmax; s_idx[w] = barg; }
        __syncthreads();
        if (tid == 0) {
            for (int k = 1; k < nw; ++k) argmax_merge(bmax, barg, s_val[k], s_idx[k]);
            a.blk_val[blockIdx.x] = bmax;
            a.blk_idx[blockIdx.x] = barg;
        }
    }
    (void)s_cnt;
}

// CSC: warp per column, entries in storage order (sorted rows).
static __global__ void __launch_bounds__(256) k_gemv_t_csc(const double* __restrict__ data,
                                                    const int32_t* __restrict__ indices,
                                                    const int64_t* __restrict__ indptr, GemvArgs a) {
    __shared__ double s_val[8];
    __shared__ int64_t s_idx[8];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * a.cpb;
    const int64_t i1 = min(a.m, i0 + (int64_t)a.cpb);
    const double radius = (a.mode == GEMV_MU) ? (a.radius_dev ? *a.radius_dev : a.radius_host) : 0.0;
    const double rho0 = (a.mode == GEMV_CERT) ? *a.rho_norm_dev : 0.0;
    double bmax = -1.0;
    int64_t barg = INT64_MAX;
    for (int64_t i = i0 + w; i < i1; i += nw) {
        const int64_t j = a.cols ? (int64_t)a.cols[i] : i;
        const int64_t lo = __ldg(indptr + j), hi = __ldg(indptr + j + 1);
        double acc = 0.0;
        for (int64_t q = lo + lane; q < hi; q += kWarp)
            acc = fma(__ldg(data + q), __ldg(a.v + __ldg(indices + q)), acc);
        const double c = warp_sum(acc);
        if (lane == 0) {
            if (a.out_c) a.out_c[i] = c;
            if (a.mode == GEMV_MAX || a.mode == GEMV_CERT) argmax_merge(bmax, barg, fabs(c), i);
            if (a.mode == GEMV_MU) {
                const double mu = fabs(c) * a.scale + radius * a.norms[j];
                if (a.out_mu) a.out_mu[i] = mu;
                a.flags[i] = mu >= a.thresh;
            } else if (a.mode == GEMV_CERT) {
                a.out_t[i] = (a.beta[j] != 0.0) ? -1.0 : cert_threshold(c, a.norms[j], a.lam, rho0, a.gam);
            }
        }
    }
    if (a.mode == GEMV_MAX || a.mode == GEMV_CERT) {
        if (lane == 0) { s_val[w] = bmax; s_idx[w] = barg; }
        __syncthreads();
        if (tid == 0) {
            for (int k = 1; k < nw; ++k) argmax_merge(bmax, barg, s_val[k], s_idx[k]);
            a.blk_val[blockIdx.x] = bmax;
            a.blk_idx[blockIdx.x] = barg;
        }
    }
}

// second stage of the block max: one block; writes (max, position) to out.
static __global__ void k_max_finalize(const double* __restrict__ bv, const int64_t* __restrict__ bi,
                               int64_t nb, double* out_val, int64_t* out_idx) {
    __shared__ double s_val[32];
    __shared__ int64_t s_idx[32];
    double v = -1.0;
    int64_t i = INT64_MAX;
    for (int64_t k = threadIdx.x; k < nb; k += blockDim.x) argmax_merge(v, i, bv[k], bi[k]);
    warp_argmax(v, i);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if (lane == 0) { s_val[w] = v; s_idx[w] = i; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < nw; ++k) argmax_merge(v, i, s_val[k], s_idx[k]);
        *out_val = v < 0.0 ? 0.0 : v;
        *out_idx = i == INT64_MAX ? 0 : i;
    }
}

// ---------------------------------------------------------------------------
// stable stream compaction (ascending), chunk = 4 elements/thread x 256 threads
// ---------------------------------------------------------------------------
constexpr int kCompactChunk = 1024;

__device__ __forceinline__ int block_excl_scan(int v, int* sh, int& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < nw ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) sh[lane] = s;
    }
    __syncthreads();
    total = sh[nw - 1];
    const int excl = (w ? sh[w - 1] : 0) + x - v;
    __syncthreads();
    return excl;
}

static __global__ void __launch_bounds__(256) k_compact_count(const uint8_t* __restrict__ flags, int64_t m,
                                                       int32_t* __restrict__ cnt) {
    __shared__ int sh[32];
    const int64_t base = (int64_t)blockIdx.x * kCompactChunk + threadIdx.x * 4;
    int c = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) c += (base + k < m) ? (int)flags[base + k] : 0;
    int total;
    block_excl_scan(c, sh, total);
    if (threadIdx.x == 0) cnt[blockIdx.x] = total;
}

// exclusive scan of block counts (one block), writes offsets and total.
static __global__ void k_scan_counts(const int32_t* __restrict__ cnt, int64_t nb, int64_t* __restrict__ off,
                              int64_t* total_out) {
    __shared__ int64_t sh[1024];
    const int t = threadIdx.x, T = blockDim.x;
    const int64_t per = (nb + T - 1) / T;
    const int64_t lo = t * per, hi = min(nb, lo + per);
    int64_t s = 0;
    for (int64_t k = lo; k < hi; ++k) s += cnt[k];
    sh[t] = s;
    __syncthreads();
    if (t == 0) {
        int64_t acc = 0;
        for (int k = 0; k < T; ++k) { int64_t v = sh[k]; sh[k] = acc; acc += v; }
        *total_out = acc;
    }
    __syncthreads();
    int64_t acc = sh[t];
    for (int64_t k = lo; k < hi; ++k) { off[k] = acc; acc += cnt[k]; }
}

// out[off + rank] = cols ? cols[i] : i, for flagged i in ascending order.
static __global__ void __launch_bounds__(256) k_compact_scatter(const uint8_t* __restrict__ flags, int64_t m,
                                                         const int32_t* __restrict__ cols,
                                                         const int64_t* __restrict__ off,
                                                         int32_t* __restrict__ out) {
    __shared__ int sh[32];
    const int64_t base = (int64_t)blockIdx.x * kCompactChunk + threadIdx.x * 4;
    int f[4], c = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) { f[k] = (base + k < m) ? (int)flags[base + k] : 0; c += f[k]; }
    int total;
    int pos = block_excl_scan(c, sh, total);
    const int64_t o = off[blockIdx.x];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (f[k]) { const int64_t i = base + k; out[o + pos++] = cols ? cols[i] : (int32_t)i; }
}

// ---------------------------------------------------------------------------
// small element-wise kernels
// ---------------------------------------------------------------------------
static __global__ void k_flags_norm_pos(const int32_t* __restrict__ cols, int64_t m, const double* __restrict__ norms,
                                 uint8_t* __restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = cols ? cols[i] : i;
        flags[i] = norms[j] > 0.0;
    }
}

static __global__ void k_flags_beta_nz(const int32_t* __restrict__ cols, int64_t m, const double* __restrict__ beta,
                                uint8_t* __restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = cols ? cols[i] : i;
        flags[i] = beta[j] != 0.0;
    }
}

static __global__ void k_set_mark(const int32_t* __restrict__ cols, int64_t m, uint8_t* __restrict__ mark) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        mark[cols[i]] = 1;
}

// beta_j = 0 where mark_j == 0 (solver.py:176-178), then clears mark.
static __global__ void k_zero_unmarked(double* __restrict__ beta, uint8_t* __restrict__ mark, int64_t p) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        if (!mark[j]) beta[j] = 0.0;
        mark[j] = 0;
    }
}

static __global__ void k_scale_vec(const double* __restrict__ x, double s, int64_t n, double* __restrict__ out,
                            int divide) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = divide ? x[i] / s : x[i] * s;
}

// ---------------------------------------------------------------------------
// residual resync over the support only (design_matrix.py:130-137 semantics)
// ---------------------------------------------------------------------------
// partial[c*n + r] = sum_{k in chunk c} X[r, S[k]] * beta[S[k]]  (ascending k, FMA)
template <typename T>
static __global__ void __launch_bounds__(256) k_resync_partial_dense(const T* __restrict__ X, int64_t ld, int n,
                                                              const int32_t* __restrict__ S,
                                                              const int64_t* __restrict__ s_count,
                                                              const double* __restrict__ beta, int nchunks,
                                                              double* __restrict__ partial) {
    const int64_t s = *s_count;
    const int c = blockIdx.y;
    const int64_t per = (s + nchunks - 1) / nchunks;
    const int64_t k0 = (int64_t)c * per, k1 = min(s, k0 + per);
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double acc = 0.0;
    for (int64_t k = k0; k < k1; ++k) {
        const int64_t j = S[k];
        acc = fma(to_d(__ldg(X + j * ld + r)), beta[j], acc);
    }
    partial[(int64_t)c * n + r] = acc;
}

// out[r] = (y ? y[r] - sum : sum) over chunks in ascending order.
static __global__ void k_resync_final(const double* __restrict__ y, const double* __restrict__ partial, int nchunks,
                               int n, double* __restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += partial[(int64_t)c * n + r];
    out[r] = y ? y[r] - s : s;
}

// CSR row products: out[r] = (y ? y[r] - sum : sum), sum over the row in column order.
static __global__ void k_resync_csr(const double* __restrict__ data, const int32_t* __restrict__ cols,
                             const int64_t* __restrict__ rowptr, int n, const double* __restrict__ beta,
                             const double* __restrict__ y, double* __restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double s = 0.0;
    for (int64_t q = rowptr[r]; q < rowptr[r + 1]; ++q) s = fma(data[q], beta[cols[q]], s);
    out[r] = y ? y[r] - s : s;
}

// rho += beta_j x_j for dropped j in ascending order (numpy: v += a * x,
// separate roundings), thread per row.
template <typename T>
static __global__ void k_drop_axpy_dense(const T* __restrict__ X, int64_t ld, int n, const int32_t* __restrict__ D,
                                  const int64_t* __restrict__ d_count, const double* __restrict__ beta,
                                  double* __restrict__ rho) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nd = *d_count;
    if (r >= n || nd == 0) return;
    double q = rho[r];
    for (int64_t k = 0; k < nd; ++k) {
        const int64_t j = D[k];
        q = __dadd_rn(q, __dmul_rn(beta[j], to_d(X[j * ld + r])));
    }
    rho[r] = q;
}

// CSC variant: one block, columns in ascending order, a barrier between
// columns (rows inside one column are distinct).
static __global__ void k_drop_axpy_csc(const double* __restrict__ data, const int32_t* __restrict__ indices,
                                const int64_t* __restrict__ indptr, const int32_t* __restrict__ D,
                                const int64_t* __restrict__ d_count, const double* __restrict__ beta,
                                double* __restrict__ rho) {
    const int64_t nd = *d_count;
    for (int64_t k = 0; k < nd; ++k) {
        const int64_t j = D[k];
        const double bj = beta[j];
        for (int64_t q = indptr[j] + threadIdx.x; q < indptr[j + 1]; q += blockDim.x)
            rho[indices[q]] = __dadd_rn(rho[indices[q]], __dmul_rn(bj, data[q]));
        __syncthreads();
    }
}

// generic dot / abs-sum over device vectors (problem.py scalar algebra for
// the drop-in helper functions).  out[0] = sum a*b, out[1] = sum |a|.
static __global__ void __launch_bounds__(1024) k_vec_stats(const double* __restrict__ a, const double* __restrict__ b,
                                                    int64_t n, double* out) {
    __shared__ double red[32];
    double s = 0.0, t = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double x = a[i];
        if (b) s = fma(x, b[i], s);
        t += fabs(x);
    }
    s = block_sum(s, red);
    t = block_sum(t, red);
    if (threadIdx.x == 0) { out[0] = s; out[1] = t; }
}

// ---------------------------------------------------------------------------
// exact-order kernel twins (reference summation order, for bit-exact tests)
// ---------------------------------------------------------------------------
template <typename T>
static __global__ void k_tdot_exact_dense(const T* __restrict__ X, int64_t ld, int n, const double* __restrict__ v,
                                   const int32_t* __restrict__ cols, int64_t k, double tail_scale,
                                   double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = cols[i];
        const T* x = X + j * ld;
        double s = 0.0;
        for (int r = 0; r < n; ++r) s = __dadd_rn(s, __dmul_rn(to_d(x[r]), v[r]));
        if (tail_scale > 0.0) s = __dadd_rn(s, __dmul_rn(tail_scale, v[n + j]));
        out[i] = s;
    }
}

static __global__ void k_tdot_exact_csc(const double* __restrict__ data, const int32_t* __restrict__ indices,
                                 const int64_t* __restrict__ indptr, int n, const double* __restrict__ v,
                                 const int32_t* __restrict__ cols, int64_t k, double tail_scale,
                                 double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = cols[i];
        double s = 0.0;
        for (int64_t q = indptr[j]; q < indptr[j + 1]; ++q) s = __dadd_rn(s, __dmul_rn(data[q], v[indices[q]]));
        if (tail_scale > 0.0) s = __dadd_rn(s, __dmul_rn(tail_scale, v[n + j]));
        out[i] = s;
    }
}

// one block: thread 0 forms the sequential non-FMA dot, all threads apply the
// axpy with separate roundings (_kernels.py:39-92 arithmetic, bit for bit).
template <typename T>
static __global__ void k_cd_pass_exact_dense(const T* __restrict__ X, int64_t ld, int n, double* __restrict__ beta,
                                      double* __restrict__ rho, const int32_t* __restrict__ A, int64_t k,
                                      double lam, const double* __restrict__ nsq, double tail_scale) {
    __shared__ double s_d;
    for (int64_t i = 0; i < k; ++i) {
        const int64_t j = A[i];
        const T* x = X + j * ld;
        if (threadIdx.x == 0) {
            double g = 0.0;
            for (int r = 0; r < n; ++r) g = __dadd_rn(g, __dmul_rn(to_d(x[r]), rho[r]));
            if (tail_scale > 0.0) g = __dadd_rn(g, __dmul_rn(tail_scale, rho[n + j]));
            const double z = __dadd_rn(beta[j], __ddiv_rn(g, nsq[j]));
            const double u = __ddiv_rn(lam, nsq[j]);
            const double nb = z > u ? __dsub_rn(z, u) : (z < -u ? __dadd_rn(z, u) : 0.0);
            const double d = __dsub_rn(nb, beta[j]);
            if (d != 0.0) beta[j] = nb;
            s_d = d;
        }
        __syncthreads();
        const double d = s_d;
        if (d != 0.0) {
            for (int r = threadIdx.x; r < n; r += blockDim.x) rho[r] = __dsub_rn(rho[r], __dmul_rn(d, to_d(x[r])));
            if (tail_scale > 0.0 && threadIdx.x == 0) rho[n + j] = __dsub_rn(rho[n + j], __dmul_rn(d, tail_scale));
        }
        __syncthreads();
    }
}

static __global__ void k_cd_pass_exact_csc(const double* __restrict__ data, const int32_t* __restrict__ indices,
                                    const int64_t* __restrict__ indptr, int n, double* __restrict__ beta,
                                    double* __restrict__ rho, const int32_t* __restrict__ A, int64_t k, double lam,
                                    const double* __restrict__ nsq, double tail_scale) {
    __shared__ double s_d;
    for (int64_t i = 0; i < k; ++i) {
        const int64_t j = A[i];
        const int64_t lo = indptr[j], hi = indptr[j + 1];
        if (threadIdx.x == 0) {
            double g = 0.0;
            for (int64_t q = lo; q < hi; ++q) g = __dadd_rn(g, __dmul_rn(data[q], rho[indices[q]]));
            if (tail_scale > 0.0) g = __dadd_rn(g, __dmul_rn(tail_scale, rho[n + j]));
            const double z = __dadd_rn(beta[j], __ddiv_rn(g, nsq[j]));
            const double u = __ddiv_rn(lam, nsq[j]);
            const double nb = z > u ? __dsub_rn(z, u) : (z < -u ? __dadd_rn(z, u) : 0.0);
            const double d = __dsub_rn(nb, beta[j]);
            if (d != 0.0) beta[j] = nb;
            s_d = d;
        }
        __syncthreads();
        const double d = s_d;
        if (d != 0.0) {
            for (int64_t q = lo + threadIdx.x; q < hi; q += blockDim.x)
                rho[indices[q]] = __dsub_rn(rho[indices[q]], __dmul_rn(d, data[q]));
            if (tail_scale > 0.0 && threadIdx.x == 0) rho[n + j] = __dsub_rn(rho[n + j], __dmul_rn(d, tail_scale));
        }
        __syncthreads();
    }
}

// column norms: warp per column, FMA, ascending rows per lane then butterfly.
template <typename T>
static __global__ void __launch_bounds__(256) k_col_norms_sq_dense(const T* __restrict__ X, int64_t ld, int n, int64_t p,
                                                            double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = wg; j < p; j += nwg) {
        const T* x = X + j * ld;
        double a = 0.0;
        for (int r = lane; r < n; r += kWarp) { const double q = to_d(__ldg(x + r)); a = fma(q, q, a); }
        a = warp_sum(a);
        if (lane == 0) out[j] = a;
    }
}

static __global__ void __launch_bounds__(256) k_col_norms_sq_csc(const double* __restrict__ data,
                                                          const int64_t* __restrict__ indptr, int64_t p,
                                                          double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = wg; j < p; j += nwg) {
        double a = 0.0;
        for (int64_t q = indptr[j] + lane; q < indptr[j + 1]; q += kWarp) { const double v = data[q]; a = fma(v, v, a); }
        a = warp_sum(a);
        if (lane == 0) out[j] = a;
    }
}

static __global__ void k_sqrt_vec(const double* __restrict__ a, double add, int64_t p, double* __restrict__ out_sq,
                           double* __restrict__ out, double* __restrict__ out_inv) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        const double s = a[j] + add;
        out_sq[j] = s;
        out[j] = sqrt(s);
        if (out_inv) out_inv[j] = s > 0.0 ? 1.0 / s : 0.0;
    }
}

}  // namespace gs
