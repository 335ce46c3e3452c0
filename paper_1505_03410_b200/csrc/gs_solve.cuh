// Persistent per-problem solve kernel: Algorithm 1 of the paper
// (solver.py:149-246) as ONE cooperative launch per lambda.
//
// A "group" of G co-resident CTAs owns one problem.  Phases that stream the
// design (residual resync, restricted X^T rho, sequential full-p screen,
// certification refresh) are split over all G CTAs; the scalar algebra and
// the serial CD epoch run on CTA 0 while the rest wait at the group barrier.
// There is no host round trip between checkpoints: the host launches once
// per lambda (or once per checkpoint when a checkpoint hook needs the active
// set on the host).
//
// Certified-zero skipping (exact): every active position i carries a
// threshold t_i (gs_kernels.cuh: cert_threshold) computed from an anchor
// residual rho0; Delta >= ||rho - rho0|| is accumulated rigorously (round-up)
// over CD updates and checkpoint drop-axpys.  A position with beta == 0 and
// Delta < t_i provably yields a zero update and is skipped without reading
// its column.  The anchor is refreshed (one GEMV over X_A by the whole group)
// only when skipping degrades, and after every residual resync.
#pragma once
#include "gs_kernels.cuh"

#include <cstdio>

namespace gs {

static __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
static __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

struct alignas(16) ColInfo {        // per column, rebuilt per lambda (u), beta kept current
    double ns, inv, nr, u, beta, pad;
};

struct GroupBar {
    unsigned count;
    unsigned gen;
};

// loop / control state of one solve, persistent across (hook-mode) launches
struct SolveCtl {
    int64_t k, passes, ntrace, nckpt;
    int32_t started, resume, pending, done, converged, status, need_refresh, final_done;
    double cd_delta, anchor_norm, cd_gstep;
    int64_t n_requeue, n_cand, n_skip;
    int64_t epoch_unc, epoch_nz;
    int64_t n_refresh;
    // device-side phase timers (%globaltimer, ns), CTA 0 thread 0
    unsigned long long t_screen, t_ckpt, t_refresh, t_cd;
    int64_t n_screen;
    // Gram-window consumer phase cycles (warp 0, clock64), GS_CD_PROF=1
    unsigned long long c_form, c_wait, c_red, c_chain, c_upd, n_win, n_mem;
    unsigned long long c_w1[6];   // blocked chain: phase cycles of a second compute warp ([5]: producer idle)
    unsigned long long c_pr[2];   // blocked chain: producer scan / descriptor + TMA issue cycles
};

static __device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

enum Pending : int32_t { PEND_NONE = 0, PEND_CONTINUE = 1, PEND_CONVERGED = 2, PEND_BREAK = 3 };

struct SolveDev {
    // design
    const void* X;
    int64_t ld;
    int n;
    int dtype;
    int64_t p;
    int sparse;
    const double* data;
    const int32_t* indices;
    const int64_t* indptr;
    const double* csr_data;
    const int32_t* csr_cols;
    const int64_t* csr_rowptr;
    const double* norms;
    const double* nsq;
    const double* inv_nsq;   // RN(1/nsq), 0 for empty columns
    // state
    const double* y;
    double* beta;
    double* rho;
    double* theta;
    struct ColInfo* cinfo;   // per column (nsq, 1/nsq, ||x||, lam/nsq, beta), rebuilt per lambda
    double* c;
    float* t;
    float* t2;
    int32_t* A;
    int32_t* A2;
    int32_t* S;
    int32_t* Dl;
    uint8_t* mark;
    double* partial;
    int nch_max;
    DevScalars* sc;
    SolveCtl* ctl;
    TraceRow* trace;
    int64_t trace_cap;
    GroupBar* bar;
    double* cta_val;     // [G]
    int64_t* cta_idx;    // [G]
    int64_t* cta_cnt;    // [2 G]
    // parameters
    double lam, eps;
    int64_t max_passes, f;
    int rule;            // GS_RULE_*
    int certify;
    int stop_at_ckpt;    // hook mode: return to the host after every checkpoint
    int init_mode;       // 0 all nonzero-norm columns, 1 host list in A2 (count in sc->cnt), 2 sequential screen
    double prev_margin;
    int refresh_excess;
    int cd_warps;        // CD warp-group size
    int cd_bytes;        // dense CD shared-memory region (tile + ring), GEMV staging after it
    int vs_cap;          // max n staged in shared memory for the GEMV
    int cd_gram;         // dense CD: Gram-window consumer (1) or one reduction per coordinate (0)
    // screening rules other than the gap sphere: q = X^T y, gstar = X^T x_jstar (ST3)
    const double* q;
    const double* gstar;
    double lmax_path;
    int64_t jstar;
    int cd_prof;         // print Gram-window phase cycles at the end of each solve (debug)
    int csc_par;         // CSC CD: fully parallel waves (cd_epoch_csc_par)
    int* rowmark;        // [n] row map of cd_epoch_csc_par (kRowFree between waves)
    int blk_mfac;        // blocked-chain CD: window drift bound Dp = D + blk_mfac * gstep
    int gemv_wide;       // dense GEMV: whole CTA per column (columns >= 16 KB), v in registers
    int csc_short;       // CSC GEMV: 8 lanes per column (short columns), 32 columns per warp round
    int smem_total;      // dynamic shared memory of the launch (bytes)
    int cd_chunk_pos;    // sparse CD: positions per re-anchored chunk of an epoch (0: whole epoch)
    int csc_flat;        // CSC full-p pass: flat coalesced loads + products in shared memory
    int l2_hint;         // TMA copies carry L2 eviction-priority hints (GEMV evict_first, CD columns evict_last)
    int lds_explicit;    // staged GEMV reads shared memory through ld.shared on 32-bit addresses
};

struct Group {
    int G, c;
    GroupBar* bar;
};

static __device__ __forceinline__ void group_sync(const Group& g) {
    __syncthreads();
    if (g.G > 1) {
        if (threadIdx.x == 0) {
            volatile unsigned* genp = &g.bar->gen;
            const unsigned my = *genp;
            __threadfence();
            const unsigned arrived = atomicAdd(&g.bar->count, 1u);
            if (arrived == (unsigned)g.G - 1u) {
                atomicExch(&g.bar->count, 0u);
                __threadfence();
                atomicAdd(&g.bar->gen, 1u);
            } else {
                // exponential backoff: CTAs idle through a CD epoch must not
                // flood L2 with polls while CTA 0 runs the latency-bound chain
                const unsigned long long t0 = gtimer();
                unsigned ns = 32;
                while (*genp == my) {
                    __nanosleep(ns);
                    ns = ns < 1024 ? ns * 2 : ns;
                    if (gtimer() - t0 > 60000000000ull) __trap();   // never hang the GPU
                }
            }
            __threadfence();   // acquire: also invalidates this SM's L1
        }
        __syncthreads();
    }
}

static __device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// bounded spin: a protocol error traps (launch failure) instead of hanging the
// GPU; the message names the wait and the queue state
static __device__ __noinline__ void spin_fail(int where, int a, int b, int c, int d) {
    printf("gapsafe_b200 watchdog: wait %d expired (block %d thread %d: %d %d %d %d)\n", where, (int)blockIdx.x,
           (int)threadIdx.x, a, b, c, d);
    __trap();
}
static __device__ __forceinline__ void spin_guard(unsigned long long t0, int where = 0, int a = 0, int b = 0, int c = 0,
                                           int d = 0) {
    if (gtimer() - t0 > 20000000000ull) spin_fail(where, a, b, c, d);
}

static __device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

static __device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_expect_tx_s(unsigned b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mbar_arrive_s(unsigned b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
static __device__ __forceinline__ bool mbar_test_s(unsigned b, unsigned parity) {
    unsigned ok;
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(b), "r"(parity) : "memory");
    return ok != 0;
}
static __device__ __forceinline__ void tma_bulk_g2s_s(unsigned dst, const void* src, unsigned bytes, unsigned b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(b) : "memory");
}
// The same with an L2 eviction-priority hint.  The group GEMVs stream the
// whole active design (70-120 MB on cfg1) through L2 at every checkpoint and
// refresh; without a hint they evict the few thousand columns the CD chain
// re-reads every epoch, and the chain's TMA fetches then pay DRAM latency.
// GEMV traffic is marked evict_first, the CD columns evict_last.
static __device__ __forceinline__ unsigned long long l2_policy_evict_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
static __device__ __forceinline__ unsigned long long l2_policy_evict_last() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
static __device__ __forceinline__ void tma_bulk_g2s_hint(unsigned dst, const void* src, unsigned bytes, unsigned b,
                                                         unsigned long long pol, int use_hint = 1) {
    if (!use_hint) { tma_bulk_g2s_s(dst, src, bytes, b); return; }
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(b), "l"(pol) : "memory");
}
static __device__ __forceinline__ int ld_vol(const int* p) { return *(const volatile int*)p; }
// CTA-scope acquire load / release store on shared memory (the load is a
// plain LDS on sm_100a; the store is MEMBAR.ALL.CTA + STS)
static __device__ __forceinline__ int ld_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
static __device__ __forceinline__ void st_rel(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// the same on precomputed 32-bit shared addresses: no generic->shared
// conversion (S2UR SR_CgaCtaId) inside the serial loops
static __device__ __forceinline__ int ld_acq_s(unsigned a) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
static __device__ __forceinline__ void st_rel_s(unsigned a, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
static __device__ __forceinline__ void st_vol_f64_s(unsigned a, double v) {
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
static __device__ __forceinline__ double ld_vol_f64_s(unsigned a) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}

// ---------------------------------------------------------------------------
// group-wide stable compaction over positions [0, m): each CTA owns one
// contiguous range, counts, then scatters at its prefix offset.  Two
// independent predicates are compacted in the same two phases.
// ---------------------------------------------------------------------------
template <class PredA, class EmitA, class PredB, class EmitB>
static __device__ void group_compact2(const Group& g, const SolveDev& P, int64_t m, PredA pa, EmitA ea, PredB pb,
                               EmitB eb, int64_t* total_a, int64_t* total_b, int* sh) {
    const int64_t per = (m + g.G - 1) / g.G;
    const int64_t lo = min(m, (int64_t)g.c * per), hi = min(m, lo + per);
    int ca = 0, cb = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) { ca += pa(i) ? 1 : 0; cb += pb(i) ? 1 : 0; }
    int tot;
    block_excl_scan(ca, sh, tot);
    const int64_t cta_a = tot;
    block_excl_scan(cb, sh, tot);
    const int64_t cta_b = tot;
    if (threadIdx.x == 0) { P.cta_cnt[2 * g.c] = cta_a; P.cta_cnt[2 * g.c + 1] = cta_b; }
    group_sync(g);
    int64_t oa = 0, ob = 0, ta = 0, tb = 0;
    for (int k = 0; k < g.G; ++k) {
        const int64_t va = P.cta_cnt[2 * k], vb = P.cta_cnt[2 * k + 1];
        if (k < g.c) { oa += va; ob += vb; }
        ta += va; tb += vb;
    }
    // stable scatter, blockDim positions per round
    for (int64_t base = lo; base < hi; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int fa = (i < hi && pa(i)) ? 1 : 0;
        const int fb = (i < hi && pb(i)) ? 1 : 0;
        int na, nb;
        const int ra = block_excl_scan(fa, sh, na);
        const int rb = block_excl_scan(fb, sh, nb);
        if (fa) ea(i, oa + ra);
        if (fb) eb(i, ob + rb);
        oa += na;
        ob += nb;
    }
    if (g.c == 0 && threadIdx.x == 0) {
        if (total_a) *total_a = ta;
        if (total_b) *total_b = tb;
    }
}

// ---------------------------------------------------------------------------
// group GEMV over positions (cols == nullptr: identity), warp per column,
// columns interleaved over all warps of the group.  v staged in shared memory
// when it fits.  Emits per-CTA (max |c|, position) into P.cta_val/cta_idx.
// ---------------------------------------------------------------------------
enum GMode : int { G_DUAL = 0, G_CERT = 1, G_MU = 2 };

constexpr int kGStages = 4;     // TMA stages of the staged dense GEMV

// explicit shared-space loads on 32-bit addresses: a pointer that reaches a
// helper through function arguments is generic to the compiler, and generic
// loads of shared memory take the long-scoreboard path (LD.E, resolved at run
// time) instead of LDS
static __device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
static __device__ __forceinline__ double2 lds_f64x2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
static __device__ __forceinline__ float4 lds_f32x4(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
static __device__ __forceinline__ float lds_f32x1(unsigned a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
static __device__ __forceinline__ uint4 lds_u32x4(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// one column out of shared memory against a centre vector in shared memory,
// both by 32-bit shared addresses; per-lane partition, accumulation order and
// butterfly identical to ColDotS / ColDot2 (bit-identical results)
template <typename T> struct ColDotSS;
template <> struct ColDotSS<double> {
    static __device__ __forceinline__ double run(unsigned x_s, unsigned v_s, int n, int lane) {
        const int n2 = n >> 1;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int q = lane; q < n2; q += kWarp) {
            const double2 xa = lds_f64x2(x_s + 16u * (unsigned)q);
            const double2 vv = lds_f64x2(v_s + 16u * (unsigned)q);
            a0 = fma(xa.x, vv.x, a0);
            a1 = fma(xa.y, vv.y, a1);
        }
        if ((n & 1) && lane == 0) a0 = fma(lds_f64(x_s + 8u * (unsigned)(n - 1)), lds_f64(v_s + 8u * (unsigned)(n - 1)), a0);
        double s = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        return s;
    }
};
template <> struct ColDotSS<float> {
    static __device__ __forceinline__ double run(unsigned x_s, unsigned v_s, int n, int lane) {
        const int n4 = n >> 2;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
        for (int q = lane; q < n4; q += kWarp) {
            const float4 xa = lds_f32x4(x_s + 16u * (unsigned)q);
            const double2 va = lds_f64x2(v_s + 32u * (unsigned)q), vb = lds_f64x2(v_s + 32u * (unsigned)q + 16u);
            a0 = fma((double)xa.x, va.x, a0);
            a1 = fma((double)xa.y, va.y, a1);
            a0 = fma((double)xa.z, vb.x, a0);
            a1 = fma((double)xa.w, vb.y, a1);
        }
        for (int r = (n4 << 2) + lane; r < n; r += kWarp)
            a0 = fma((double)lds_f32x1(x_s + 4u * (unsigned)r), lds_f64(v_s + 8u * (unsigned)r), a0);
        double s = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        return s;
    }
};

// ---------------------------------------------------------------------------
// Wide-column dense GEMV (P.gemv_wide: columns of 16 KB and more, cfg2's
// 40 KB f32 columns).  A whole column no longer fits several times in a
// stage, so the warp-per-column form would leave 7 of 8 warps idle.  Here the
// CTA streams its contiguous share of positions through a ring of whole-column
// slots (cp.async.bulk, one mbarrier per slot) and ALL warps reduce each
// column: thread t owns the 16-byte vectors t, t + 256, ... of every column
// and keeps the matching entries of v in registers (no shared-memory reads of
// v at all); per column one butterfly per warp and a fixed-order sum of the
// warp partials by thread 0, which also runs the epilogue and re-issues the
// slot.  One __syncthreads per column.
// ---------------------------------------------------------------------------
constexpr int kWideRows = 44;      // entries of v per thread: n <= 256 * 44 = 11264
constexpr int kWideSlots = 8;
constexpr int kWidePartBytes = 2 * 32 * 8 * 8;     // warp partials of two epilogue batches (tail of the dynamic region)

template <typename T, class Epi>
static __device__ __noinline__ void group_gemv_wide(const Group& g, const SolveDev& P, const double* __restrict__ v,
                                                       const int32_t* cols, int64_t m, int mode, unsigned char* stg,
                                                       int64_t stg_bytes, Epi epilogue) {
    constexpr int E = 16 / (int)sizeof(T);          // elements per 16-byte vector
    constexpr int KV = kWideRows / E;               // vectors per thread
    constexpr int GV = 8;                           // vectors loaded per group (all issued before the first FMA)
    constexpr int kEB = 32;                         // columns per epilogue batch (one lane each)
    static_assert(kWidePartBytes == 2 * kEB * 8 * 8, "partials region");
    __shared__ unsigned long long s_wbar[kWideSlots];
    // warp partials of two epilogue batches: the last kWidePartBytes of the dynamic region
    double (*s_wpart)[kEB][8] = reinterpret_cast<double (*)[kEB][8]>(stg + stg_bytes - kWidePartBytes);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, W = blockDim.x >> 5;
    const int n = P.n;
    const T* X = (const T*)P.X;
    const int64_t ldx = P.ld;
    const double* __restrict__ p_norms = P.norms;
    const double* p_beta = P.beta;
    const int use_hint = P.l2_hint;
    const int64_t colb = ldx * (int64_t)sizeof(T);
    const int NS = (int)min((int64_t)kWideSlots, (stg_bytes - kWidePartBytes) / colb);
    const int nvec = (int)(ldx / E);
    const int64_t per = (m + g.G - 1) / g.G;
    const int64_t lo = min(m, (int64_t)g.c * per), hi = min(m, lo + per);
    const int nst = (int)(hi - lo);
    const unsigned bar0 = smem_u32(&s_wbar[0]);
    const unsigned stg0 = smem_u32(stg);
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&s_wbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // this thread's entries of v (rows past n are zero: the column padding is zero too)
    double th[KV * E];
#pragma unroll
    for (int k = 0; k < KV; ++k) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int r = (tid + k * 256) * E + e;
            th[k * E + e] = r < n ? v[r] : 0.0;
        }
    }
    __syncthreads();
    const unsigned long long pol_stream = l2_policy_evict_first();
    auto issue = [&](int k) {                       // thread 0: column lo + k into slot k % NS
        const int s = k % NS;
        const int64_t i = lo + k;
        const int64_t j = cols ? (int64_t)cols[i] : i;
        const unsigned b = bar0 + 8u * s;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx_s(b, (unsigned)colb);
        tma_bulk_g2s_hint(stg0 + (unsigned)(s * colb), X + j * ldx, (unsigned)colb, b, pol_stream, use_hint);
    };
    // epilogues run lane-parallel, one batch of kEB columns at a time, by the warp
    // whose turn it is (batch index mod W): coalesced norm loads and mark stores,
    // and no per-column serial tail on one thread
    auto run_epilogues = [&](int kb0, int cnt) {    // columns kb0 .. kb0 + cnt of this CTA's share
        if (lane < cnt) {
            const int k = kb0 + lane;
            const int64_t i = lo + k;
            const int64_t j = cols ? (int64_t)cols[i] : i;
            const double nrm = __ldg(p_norms + j);
            const double bj = (mode == G_CERT) ? p_beta[j] : 0.0;
            const double* pp = &s_wpart[(k / kEB) & 1][k % kEB][0];
            double cval = 0.0;
            for (int q = 0; q < W; ++q) cval += pp[q];
            epilogue(i, j, cval, nrm, bj);
        }
    };
    if (tid == 0)
        for (int k = 0; k < min(nst, NS); ++k) issue(k);
    for (int k = 0; k < nst; ++k) {
        const int s = k % NS;
        {
            const unsigned b = bar0 + 8u * s, par = (unsigned)((k / NS) & 1);
            if (!mbar_test_s(b, par)) {
                const unsigned long long t0 = gtimer();
                while (!mbar_test_s(b, par)) spin_guard(t0, 6, k, nst, (int)g.c, 0);
            }
        }
        const unsigned base_s = stg0 + (unsigned)(s * colb);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int g0 = 0; g0 < KV; g0 += GV) {
            if (g0 * 256 >= nvec) break;            // uniform
            uint4 raw[GV];
#pragma unroll
            for (int u = 0; u < GV; ++u) {
                const int q = tid + (g0 + u) * 256;
                raw[u] = (g0 + u < KV && q < nvec) ? lds_u32x4(base_s + 16u * (unsigned)q) : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < GV; ++u) {
                if (g0 + u < KV) {
                    const int kk = g0 + u;
                    if constexpr (E == 2) {
                        if (u & 1) {
                            a2 = fma(__hiloint2double((int)raw[u].y, (int)raw[u].x), th[kk * 2], a2);
                            a3 = fma(__hiloint2double((int)raw[u].w, (int)raw[u].z), th[kk * 2 + 1], a3);
                        } else {
                            a0 = fma(__hiloint2double((int)raw[u].y, (int)raw[u].x), th[kk * 2], a0);
                            a1 = fma(__hiloint2double((int)raw[u].w, (int)raw[u].z), th[kk * 2 + 1], a1);
                        }
                    } else {
                        a0 = fma((double)__uint_as_float(raw[u].x), th[kk * 4], a0);
                        a1 = fma((double)__uint_as_float(raw[u].y), th[kk * 4 + 1], a1);
                        a2 = fma((double)__uint_as_float(raw[u].z), th[kk * 4 + 2], a2);
                        a3 = fma((double)__uint_as_float(raw[u].w), th[kk * 4 + 3], a3);
                    }
                }
            }
        }
        double sum = (a0 + a1) + (a2 + a3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) s_wpart[(k / kEB) & 1][k % kEB][w] = sum;
        __syncthreads();                             // slot fully read, partials visible
        if (tid == 0 && k + NS < nst) issue(k + NS);
        if ((k % kEB) == kEB - 1 && w == ((k / kEB) % W)) run_epilogues(k - (kEB - 1), kEB);
    }
    // the last, partial batch (its partials were published by the loop's last barrier)
    if (nst % kEB != 0 && w == ((nst / kEB) % W)) run_epilogues(nst - nst % kEB, nst % kEB);
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < NS; ++s) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&s_wbar[s])) : "memory");
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Short-column CSC GEMV (P.csc_short: about 24 nonzeros per column or fewer,
// cfg3's 20).  A warp takes 32 consecutive positions per round: lane l loads
// the column pointers, norm (and beta) of position l; the columns are then
// reduced by 8-lane groups, four columns at a time, with the loads of all
// eight batches issued before the first gather (24 values + 24 row indices in
// flight per lane).  Three shuffle steps per column instead of five, no idle
// lanes, and the per-column epilogues run lane-parallel.
// ---------------------------------------------------------------------------
// streamed once: read-only loads that do not allocate in L1 (with ~210 KB of the
// SM's 256 KB in use as shared memory, the few L1 lines left would be evicted
// between the trips that touch them and re-fetched from L2)
static __device__ __forceinline__ double ldg_stream_f64(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
static __device__ __forceinline__ int32_t ldg_stream_s32(const int32_t* p) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

template <class Epi>
static __device__ __noinline__ void group_gemv_csc_short(const Group& g, const SolveDev& P, const double* vv,
                                                            const bool staged, const int32_t* cols, int64_t m, int mode,
                                                            Epi epilogue) {
    // P lives in global memory: keep its pointers in registers (the loads below would
    // otherwise re-read them from the descriptor before every access)
    const double* __restrict__ p_data = P.data;
    const int32_t* __restrict__ p_indices = P.indices;
    const int64_t* __restrict__ p_indptr = P.indptr;
    const double* __restrict__ p_norms = P.norms;
    const double* p_beta = P.beta;
    const unsigned vs_s = staged ? smem_u32(vv) : 0u;
    auto vget = [&](int32_t r) -> double { return staged ? lds_f64(vs_s + 8u * (unsigned)r) : __ldg(vv + r); };
    constexpr int T3 = 3;                            // unrolled trips of 8 nonzeros
    constexpr int CPR = 16;                          // positions per warp round (two rounds in flight per warp)
    constexpr int NB = CPR / 4;                      // batches of four columns
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int sub = lane >> 3, sl = lane & 7;
    const int64_t GW = (int64_t)g.G * W;
    const int64_t nround = (m + CPR - 1) / CPR;
    // software pipeline over this warp's rounds: the column pointers of round
    // r + 2 and the values / row indices of round r + 1 are in flight while
    // round r is reduced (two register buffers, the loop unrolled by two)
    struct Meta { int64_t j, plo, phi; double nrm, bj; bool valid; };
    auto load_meta = [&](int64_t rd) {
        Meta mt;
        const int64_t i = rd * CPR + lane;
        mt.valid = rd < nround && lane < CPR && i < m;
        mt.j = mt.valid ? (cols ? (int64_t)cols[i] : i) : 0;
        mt.plo = 0; mt.phi = 0; mt.nrm = 0.0; mt.bj = 0.0;
        if (mt.valid) {
            mt.plo = __ldg(p_indptr + mt.j);
            mt.phi = __ldg(p_indptr + mt.j + 1);
            mt.nrm = __ldg(p_norms + mt.j);
            if (mode == G_CERT) mt.bj = p_beta[mt.j];
        }
        return mt;
    };
    struct Buf { double dv[NB][T3]; int32_t iv[NB][T3]; int64_t qlo[NB], qhi[NB]; };
    auto load_buf = [&](const Meta& mt, Buf& B) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int src = 4 * b + sub;
            B.qlo[b] = __shfl_sync(FULL, mt.plo, src) + sl;
            B.qhi[b] = __shfl_sync(FULL, mt.phi, src);
#pragma unroll
            for (int t = 0; t < T3; ++t) {
                const int64_t q = B.qlo[b] + 8 * t;
                const bool ok = q < B.qhi[b];
                B.dv[b][t] = ok ? ldg_stream_f64(p_data + q) : 0.0;
                B.iv[b][t] = ok ? ldg_stream_s32(p_indices + q) : 0;
            }
        }
    };
    auto reduce_buf = [&](int64_t rd, const Meta& mt, const Buf& B) {
        double cval = 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            double a = 0.0;
#pragma unroll
            for (int t = 0; t < T3; ++t) a = fma(B.dv[b][t], vget(B.iv[b][t]), a);
            for (int64_t q = B.qlo[b] + 8 * T3; q < B.qhi[b]; q += 8) a = fma(__ldg(p_data + q), vget(__ldg(p_indices + q)), a);
            a += __shfl_xor_sync(FULL, a, 4);
            a += __shfl_xor_sync(FULL, a, 2);
            a += __shfl_xor_sync(FULL, a, 1);
            // column 4 b + sub sits in the lanes of group `sub`; lane l wants column l
            const double got = __shfl_sync(FULL, a, (lane & 3) * 8);
            if ((lane >> 2) == b) cval = got;
        }
        if (mt.valid) epilogue(rd * CPR + lane, mt.j, cval, mt.nrm, mt.bj);
    };
    const int64_t r0 = (int64_t)g.c * W + w;
    if (r0 >= nround) return;
    Buf A, B;
    Meta m0 = load_meta(r0), m1 = load_meta(r0 + GW);
    load_buf(m0, A);
    for (int64_t rd = r0; rd < nround; rd += 2 * GW) {
        // even round: values in A; fetch the odd round into B
        Meta m2 = load_meta(rd + 2 * GW);
        if (rd + GW < nround) load_buf(m1, B);
        reduce_buf(rd, m0, A);
        if (rd + GW >= nround) break;
        // odd round: values in B; fetch the next even round into A
        Meta m3 = load_meta(rd + 3 * GW);
        if (rd + 2 * GW < nround) load_buf(m2, A);
        reduce_buf(rd + GW, m1, B);
        m0 = m2;
        m1 = m3;
    }
}

// ---------------------------------------------------------------------------
// Short-column CSC GEMV over CONSECUTIVE columns (the full-p screening pass):
// flat, fully coalesced loads.  The 8-lane form above asks the memory system
// for 64-byte (values) and 32-byte (row indices) pieces, four separate ones
// per load instruction; with ~18 MB of such requests in flight it still
// delivers only ~1.4 TB/s.  Here a warp round (32 consecutive columns) reads
// its CONTIGUOUS nonzero range [indptr[c0], indptr[c0+32]) exactly like a
// copy -- lane l takes entries l, l+32, ... (256-byte and 128-byte requests,
// every line touched once) -- multiplies each value by its centre entry
// (gather from the staged centre) and parks the products in a per-warp
// shared-memory buffer; the columns are then summed out of that buffer by
// 8-lane groups (conflict-free contiguous reads, three shuffle steps).  The
// next round's loads are in flight while the current one is reduced.
// Rounds with more nonzeros than the buffer holds fall back to direct loads.
// ---------------------------------------------------------------------------
template <class Epi>
static __device__ __noinline__ void group_gemv_csc_flat(const Group& g, const SolveDev& P, const double* vv,
                                                           int64_t m, int mode, double* sbuf_all, int capw, Epi epilogue) {
    constexpr int CPR = 16;                          // columns per warp round (two rounds in flight per warp:
                                                     // 32 would need ~170 live registers for the two buffers)
    constexpr int TU = 10;                           // unrolled trips of 32 entries (320 per round)
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int sub = lane >> 3, sl = lane & 7;
    const int64_t GW = (int64_t)g.G * W;
    const int64_t nround = (m + CPR - 1) / CPR;
    const double* __restrict__ p_data = P.data;
    const int32_t* __restrict__ p_indices = P.indices;
    const int64_t* __restrict__ p_indptr = P.indptr;
    const double* __restrict__ p_norms = P.norms;
    const double* p_beta = P.beta;
    const unsigned vs_s = smem_u32(vv);
    const unsigned sb_s = smem_u32(sbuf_all + (size_t)w * capw);
    struct Meta { int64_t plo, phi; double nrm, bj; bool valid; };
    auto load_meta = [&](int64_t rd) {
        Meta mt;
        const int64_t j = rd * CPR + lane;
        mt.valid = rd < nround && lane < CPR && j < m;
        mt.plo = 0; mt.phi = 0; mt.nrm = 0.0; mt.bj = 0.0;
        if (mt.valid) {
            mt.plo = __ldg(p_indptr + j);
            mt.phi = __ldg(p_indptr + j + 1);
            mt.nrm = __ldg(p_norms + j);
            if (mode == G_CERT) mt.bj = p_beta[j];
        }
        return mt;
    };
    struct Buf { double dv[TU]; int32_t iv[TU]; int64_t qa; int total; };
    auto load_buf = [&](const Meta& mt, Buf& B) {
        // the round's nonzero range: first column's start .. last valid column's end
        const unsigned vmask = __ballot_sync(FULL, mt.valid);
        const int lastl = 31 - __clz((int)vmask);
        B.qa = __shfl_sync(FULL, mt.plo, 0);
        B.total = (int)(__shfl_sync(FULL, mt.phi, lastl < 0 ? 0 : lastl) - B.qa);
        if (vmask == 0u) B.total = 0;
        const int lim = B.total <= capw ? B.total : 0;      // oversized rounds load nothing here
        const double* dbase = p_data + B.qa + lane;         // one 64-bit address per round, immediates per trip
        const int32_t* ibase = p_indices + B.qa + lane;
        const int lim_l = lim - lane;
#pragma unroll
        for (int t = 0; t < TU; ++t) {
            const bool ok = 32 * t < lim_l;
            B.dv[t] = ok ? ldg_stream_f64(dbase + 32 * t) : 0.0;
            B.iv[t] = ok ? ldg_stream_s32(ibase + 32 * t) : 0;
        }
    };
    auto reduce_buf = [&](int64_t rd, const Meta& mt, const Buf& B) {
        double cval = 0.0;
        if (B.total <= capw) {
            // products into the warp's buffer (entry e at slot e)
#pragma unroll
            for (int t = 0; t < TU; ++t) {
                const int e = 32 * t + lane;
                if (e < B.total) {
                    const double pr = B.dv[t] * lds_f64(vs_s + 8u * (unsigned)B.iv[t]);
                    asm volatile("st.shared.f64 [%0], %1;" ::"r"(sb_s + 8u * (unsigned)e), "d"(pr) : "memory");
                }
            }
            for (int e = 32 * TU + lane; e < B.total; e += 32) {
                const double pr = __ldg(p_data + B.qa + e) * lds_f64(vs_s + 8u * (unsigned)__ldg(p_indices + B.qa + e));
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(sb_s + 8u * (unsigned)e), "d"(pr) : "memory");
            }
            __syncwarp();
#pragma unroll
            for (int b = 0; b < CPR / 4; ++b) {
                const int src = 4 * b + sub;
                const int64_t clo = __shfl_sync(FULL, mt.plo, src), chi = __shfl_sync(FULL, mt.phi, src);
                const int off = (int)(clo - B.qa), len = (int)(chi - clo);
                double a = 0.0;
                const unsigned cb_s = sb_s + 8u * (unsigned)(off + sl);
                if (sl < len) a = lds_f64(cb_s);
                if (sl + 8 < len) a += lds_f64(cb_s + 64u);
                if (sl + 16 < len) a += lds_f64(cb_s + 128u);
                for (int u = sl + 24; u < len; u += 8) a += lds_f64(sb_s + 8u * (unsigned)(off + u));
                a += __shfl_xor_sync(FULL, a, 4);
                a += __shfl_xor_sync(FULL, a, 2);
                a += __shfl_xor_sync(FULL, a, 1);
                const double got = __shfl_sync(FULL, a, (lane & 3) * 8);
                if ((lane >> 2) == b) cval = got;
            }
            __syncwarp();                            // the buffer is rewritten by the next round
        } else {
            // a round too large for the buffer: direct 8-lane sums from global memory
#pragma unroll
            for (int b = 0; b < CPR / 4; ++b) {
                const int src = 4 * b + sub;
                const int64_t clo = __shfl_sync(FULL, mt.plo, src), chi = __shfl_sync(FULL, mt.phi, src);
                double a = 0.0;
                for (int64_t q = clo + sl; q < chi; q += 8) a = fma(__ldg(p_data + q), lds_f64(vs_s + 8u * (unsigned)__ldg(p_indices + q)), a);
                a += __shfl_xor_sync(FULL, a, 4);
                a += __shfl_xor_sync(FULL, a, 2);
                a += __shfl_xor_sync(FULL, a, 1);
                const double got = __shfl_sync(FULL, a, (lane & 3) * 8);
                if ((lane >> 2) == b) cval = got;
            }
        }
        if (mt.valid) epilogue(rd * CPR + lane, rd * CPR + lane, cval, mt.nrm, mt.bj);
    };
    const int64_t r0 = (int64_t)g.c * W + w;
    if (r0 >= nround) return;
    Buf A, B;
    Meta m0 = load_meta(r0), m1 = load_meta(r0 + GW);
    load_buf(m0, A);
    for (int64_t rd = r0; rd < nround; rd += 2 * GW) {
        Meta m2 = load_meta(rd + 2 * GW);
        if (rd + GW < nround) load_buf(m1, B);
        reduce_buf(rd, m0, A);
        if (rd + GW >= nround) break;
        Meta m3 = load_meta(rd + 3 * GW);
        if (rd + 2 * GW < nround) load_buf(m2, A);
        reduce_buf(rd + GW, m1, B);
        m0 = m2;
        m1 = m3;
    }
}

// __noinline__: solve_body calls this from seven places; inlined, the kernel grew to
// ~170 k instructions and the register pressure at the call sites pushed spills into
// the CD chain's window loop (local-memory loads on the serial path).
template <typename T>
static __device__ __forceinline__ void group_gemv_impl(const Group& g, const SolveDev& P, const double* v, const int32_t* cols, int64_t m,
                           int mode, double* out_c, float* out_t, double rho0, double gam, double radius,
                           double* vs, unsigned char* stg = nullptr, int64_t stg_bytes = 0,
                           int* tile_valid = nullptr) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int n = P.n;
    const bool wide = !P.sparse && P.gemv_wide && stg != nullptr &&
                      (int64_t)P.smem_total >= 2 * P.ld * (int64_t)sizeof(T) + kWidePartBytes;
    const bool stage = n <= P.vs_cap && !wide;
    if (stage) {
        if (n >= 2048 && (n & 1) == 0 && (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
            // long centre vector (cfg3: 160 KB): one TMA bulk copy per 32 KB instead of 8-byte loads
            __shared__ unsigned long long s_vbar;
            const unsigned vb = smem_u32(&s_vbar);
            __syncthreads();                     // earlier readers of vs are done before the async-proxy writes
            if (threadIdx.x == 0) {
                mbar_init(&s_vbar, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx_s(vb, (unsigned)(n * 8));
                for (int off = 0; off < n; off += 4096) {
                    const int cnt = min(4096, n - off);
                    tma_bulk_g2s_s(smem_u32(vs + off), v + off, (unsigned)(cnt * 8), vb);
                }
                vs[n] = 0.0; vs[n + 1] = 0.0;
            }
            __syncthreads();
            if (!mbar_test_s(vb, 0)) {
                const unsigned long long t0 = gtimer();
                while (!mbar_test_s(vb, 0)) spin_guard(t0, 7, n, 0, 0, 0);
            }
            __syncthreads();
            if (threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(vb) : "memory");
        } else {
            for (int r = threadIdx.x; r < n + 2; r += blockDim.x) vs[r] = r < n ? v[r] : 0.0;
        }
        __syncthreads();
    }
    const double* vv = stage ? vs : v;
    const unsigned vs_s = stage ? smem_u32(vs) : 0u;
    double bmax = -1.0;
    int64_t barg = INT64_MAX;
    const int64_t GW = (int64_t)g.G * W;
    // P lives in global memory and every store below could alias it as far as the compiler
    // knows, so each use would re-load the field (a dependent global load per column):
    // the fields the epilogue needs are read once, here
    const bool e_dome = P.rule == R_GAP_DOME && P.q != nullptr;
    const double* __restrict__ e_q = P.q;
    const double e_lam = P.lam;
    const double e_R = e_dome ? P.sc->rule_R : 0.0, e_rd = e_dome ? P.sc->rule_rd : 0.0, e_a = e_dome ? P.sc->rule_a : 0.0;
    uint8_t* const e_mark = P.mark;
    // per-column epilogue (lane 0); nrm/bj were loaded before the dot
    auto epilogue = [&](int64_t i, int64_t j, double cval, double nrm, double bj) {
        if (mode == G_MU) {
            const double mu = e_dome ? dome_mu(__ldg(e_q + j) / e_lam, cval, e_R, e_rd, e_a, nrm)
                                     : fabs(cval) + radius * nrm;
            e_mark[j] = (mu >= 1.0 - 1e-9) && nrm > 0.0;
        } else {
            if (out_c) out_c[i] = cval;
            argmax_merge(bmax, barg, fabs(cval), i);
            if (mode == G_CERT) {
                const double tt = (bj != 0.0) ? -1.0 : cert_threshold(cval, nrm, e_lam, rho0, gam);
                out_t[i] = __double2float_rd(tt);
            }
        }
    };
    if (P.sparse && P.csc_short && stage && !cols && P.csc_flat &&
        (int64_t)P.smem_total - (int64_t)(n + 2) * 8 >= (int64_t)W * 8 * 320) {
        // consecutive columns (the full-p pass): flat coalesced loads, products parked in the
        // shared memory left free beside the staged centre
        const int64_t room = ((int64_t)P.smem_total - (int64_t)(n + 2) * 8) / ((int64_t)W * 8);
        const int capw = (int)min((int64_t)512, room) & ~31;
        group_gemv_csc_flat(g, P, vv, m, mode, vs + n + 2, capw, epilogue);
    } else if (P.sparse && P.csc_short) {
        group_gemv_csc_short(g, P, vv, stage, cols, m, mode, epilogue);
    } else if (wide) {
        // vs is not staged in this mode: the ring takes the whole dynamic shared memory
        group_gemv_wide<T>(g, P, v, cols, m, mode, stg, (int64_t)P.smem_total, epilogue);
        if (tile_valid && threadIdx.x == 0) *tile_valid = 0;   // the CD threshold tile was overwritten
        __syncthreads();
    } else if (P.sparse) {
        for (int64_t i = (int64_t)g.c * W + w; i < m; i += GW) {
            const int64_t j = cols ? (int64_t)cols[i] : i;
            const double nrm = __ldg(P.norms + j);
            const double bj = (mode == G_CERT) ? P.beta[j] : 0.0;
            const int64_t lo = __ldg(P.indptr + j), hi = __ldg(P.indptr + j + 1);
            double acc = 0.0;
            for (int64_t q = lo + lane; q < hi; q += kWarp) acc = fma(__ldg(P.data + q), vv[__ldg(P.indices + q)], acc);
            const double cval = warp_sum(acc);
            if (lane == 0) epilogue(i, j, cval, nrm, bj);
        }
    } else if (stg_bytes >= (int64_t)kGStages * P.ld * (int64_t)sizeof(T)) {
        // TMA-staged: this CTA streams its contiguous share of positions
        // through kGStages shared-memory stages (cp.async.bulk, mbarrier
        // tx-count); its warps reduce the columns out of shared memory.  Per
        // column the lane partition and butterfly are those of ColDot2, so the
        // values are bit-identical to the direct path below.
        __shared__ unsigned long long s_gbar[kGStages];
        const T* X = (const T*)P.X;
        const int64_t ldx = P.ld;
        const double* __restrict__ p_norms = P.norms;
        const double* p_beta = P.beta;
        const int use_hint = P.l2_hint, use_lds = P.lds_explicit;
        const int64_t colb = ldx * (int64_t)sizeof(T);
        const int64_t sb = stg_bytes / kGStages / 16 * 16;
        const int C = (int)min((int64_t)(32 * W), sb / colb);      // columns per stage
        const int64_t per = (m + g.G - 1) / g.G;
        const int64_t lo = min(m, (int64_t)g.c * per), hi = min(m, lo + per);
        const int nst = (int)((hi - lo + C - 1) / C);
        const unsigned bar0 = smem_u32(&s_gbar[0]);
        const unsigned stg0 = smem_u32(stg);
        if (threadIdx.x == 0) {
            for (int s = 0; s < kGStages; ++s) mbar_init(&s_gbar[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        const unsigned long long pol_stream = l2_policy_evict_first();
        auto issue = [&](int k) {           // warp 0: stage k into slot k % kGStages
            const int s = k % kGStages;
            const int64_t i0 = lo + (int64_t)k * C, i1 = min(hi, i0 + C);
            const unsigned b = bar0 + 8u * s, dst = stg0 + (unsigned)(s * sb);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (lane == 0) mbar_expect_tx_s(b, (unsigned)((i1 - i0) * colb));
            __syncwarp();
            if (!cols) {
                if (lane == 0) tma_bulk_g2s_hint(dst, X + i0 * ldx, (unsigned)((i1 - i0) * colb), b, pol_stream, use_hint);
            } else {
                // one column per lane: the gathered indices load in parallel
                for (int64_t i = i0 + lane; i < i1; i += 32)
                    tma_bulk_g2s_hint(dst + (unsigned)((i - i0) * colb), X + (int64_t)cols[i] * ldx, (unsigned)colb, b,
                                      pol_stream, use_hint);
            }
        };
        if (w == 0)
            for (int k = 0; k < min(nst, kGStages); ++k) issue(k);
        // per-column epilogue inputs, one stage ahead in registers: lane l of
        // warp w holds column w + l*W of the stage
        const int per_w = (C + W - 1) / W;
        auto fetch = [&](int k, int64_t& jj, double& nr, double& bb) {
            const int64_t i = lo + (int64_t)k * C + w + (int64_t)lane * W;
            jj = 0; nr = 0.0; bb = 0.0;
            if (k < nst && lane < per_w && i < min(hi, lo + (int64_t)(k + 1) * C)) {
                jj = cols ? (int64_t)cols[i] : i;
                nr = __ldg(p_norms + jj);
                if (mode == G_CERT) bb = p_beta[jj];
            }
        };
        int64_t jn; double nn, bn;
        fetch(0, jn, nn, bn);
        for (int k = 0; k < nst; ++k) {
            const int64_t jc = jn; const double nc = nn, bc = bn;
            fetch(k + 1, jn, nn, bn);
            const int s = k % kGStages;
            {
                const unsigned b = bar0 + 8u * s, par = (unsigned)((k / kGStages) & 1);
                if (!mbar_test_s(b, par)) {
                    const unsigned long long t0 = gtimer();
                    while (!mbar_test_s(b, par)) spin_guard(t0, 5, k, nst, (int)g.c, 0);
                }
            }
            const int64_t i0 = lo + (int64_t)k * C;
            const int cn = (int)min((int64_t)C, hi - i0);
            const T* base = reinterpret_cast<const T*>(stg + (size_t)s * sb);
            for (int l = 0; w + l * W < cn; ++l) {
                const int cc = w + l * W;
                const double cval = (stage && use_lds) ? ColDotSS<T>::run(stg0 + (unsigned)(s * sb) + (unsigned)(cc * colb), vs_s, n, lane)
                                          : ColDotS<T>::run(base + (int64_t)cc * ldx, vv, n, lane);
                const int64_t j = __shfl_sync(0xffffffffu, jc, l);
                const double nrm = __shfl_sync(0xffffffffu, nc, l);
                const double bj = __shfl_sync(0xffffffffu, bc, l);
                if (lane == 0) epilogue(i0 + cc, j, cval, nrm, bj);
            }
            __syncthreads();                  // slot s fully read
            if (w == 0 && k + kGStages < nst) issue(k + kGStages);
        }
        if (threadIdx.x == 0)
            for (int s = 0; s < kGStages; ++s) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&s_gbar[s])) : "memory");
        if (tile_valid && threadIdx.x == 0) *tile_valid = 0;   // the CD threshold tile was overwritten
        __syncthreads();
    } else {
        const T* X = (const T*)P.X;
        // each warp takes two columns (i, i + GW) per round
        for (int64_t i = (int64_t)g.c * W + w; i < m; i += 2 * GW) {
            const int64_t i1 = i + GW;
            const bool two = i1 < m;
            const int64_t j0 = cols ? (int64_t)cols[i] : i;
            const int64_t j1 = two ? (cols ? (int64_t)cols[i1] : i1) : j0;
            const double nrm0 = __ldg(P.norms + j0), nrm1 = __ldg(P.norms + j1);
            const double bj0 = (mode == G_CERT) ? P.beta[j0] : 0.0;
            const double bj1 = (mode == G_CERT) ? P.beta[j1] : 0.0;
            double c0, c1;
            ColDot2<T>::run(X + j0 * P.ld, X + j1 * P.ld, vv, n, lane, c0, c1);
            if (lane == 0) {
                epilogue(i, j0, c0, nrm0, bj0);
                if (two) epilogue(i1, j1, c1, nrm1, bj1);
            }
        }
    }
    if (mode != G_MU) {
        __shared__ double s_v[32];
        __shared__ int64_t s_i[32];
        warp_argmax(bmax, barg);
        if (lane == 0) { s_v[w] = bmax; s_i[w] = barg; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < W; ++k) argmax_merge(bmax, barg, s_v[k], s_i[k]);
            P.cta_val[g.c] = bmax;
            P.cta_idx[g.c] = barg;
        }
    }
}

template <typename T>
static __device__ __noinline__ void group_gemv(const Group& g, const SolveDev& P, const double* v, const int32_t* cols, int64_t m,
                           int mode, double* out_c, float* out_t, double rho0, double gam, double radius,
                           double* vs, unsigned char* stg = nullptr, int64_t stg_bytes = 0,
                           int* tile_valid = nullptr) {
    group_gemv_impl<T>(g, P, v, cols, m, mode, out_c, out_t, rho0, gam, radius, vs, stg, stg_bytes, tile_valid);
}

// max over the per-CTA partials (every caller thread gets the same answer)
static __device__ __forceinline__ void group_max_result(const Group& g, const SolveDev& P, double& v, int64_t& i) {
    v = -1.0;
    i = INT64_MAX;
    for (int k = 0; k < g.G; ++k) argmax_merge(v, i, P.cta_val[k], P.cta_idx[k]);
    if (v < 0.0) { v = 0.0; i = 0; }
}

// ---------------------------------------------------------------------------
// residual resync rho = y - X beta over the support (design_matrix.py:130-137)
// ---------------------------------------------------------------------------
template <typename T>
static __device__ void group_resync(const Group& g, const SolveDev& P, int64_t m, int* sh) {
    const int n = P.n;
    // support list S = {A_i : beta_{A_i} != 0}, ascending (l1 norms, dense products)
    const int32_t* A = P.A;
    group_compact2(g, P, m,
                   [&](int64_t i) { return P.beta[A[i]] != 0.0; },
                   [&](int64_t i, int64_t o) { P.S[o] = A[i]; },
                   [&](int64_t) { return false; }, [&](int64_t, int64_t) {},
                   &P.sc->n_supp, nullptr, sh);
    group_sync(g);
    if (P.sparse) {
        for (int64_t r = (int64_t)g.c * blockDim.x + threadIdx.x; r < n; r += (int64_t)g.G * blockDim.x) {
            double s = 0.0;
            for (int64_t q = __ldg(P.csr_rowptr + r); q < __ldg(P.csr_rowptr + r + 1); ++q)
                s = fma(__ldg(P.csr_data + q), P.beta[__ldg(P.csr_cols + q)], s);
            P.rho[r] = __ldg(P.y + r) - s;
        }
        group_sync(g);
        return;
    }
    const int64_t s = P.sc->n_supp;
    const int B = blockDim.x;
    const int nrb = (n + B - 1) / B;
    const int nch = (int)imin64(P.nch_max, imax64(1, (s + 15) / 16));
    const int64_t per = (s + nch - 1) / nch;
    const T* X = (const T*)P.X;
    if (s > 0) {
        for (int task = g.c; task < nrb * nch; task += g.G) {
            const int rb = task % nrb, ch = task / nrb;
            const int r = rb * B + threadIdx.x;
            if (r < n) {
                const int64_t k0 = (int64_t)ch * per, k1 = min(s, k0 + per);
                double acc = 0.0;
                for (int64_t k = k0; k < k1; ++k) {
                    const int64_t j = P.S[k];
                    acc = fma(to_d(__ldg(X + j * P.ld + r)), P.beta[j], acc);
                }
                P.partial[(int64_t)ch * n + r] = acc;
            }
        }
    }
    group_sync(g);
    for (int64_t r = (int64_t)g.c * B + threadIdx.x; r < n; r += (int64_t)g.G * B) {
        double sum = 0.0;
        if (s > 0)
            for (int ch = 0; ch < nch; ++ch) sum += P.partial[(int64_t)ch * n + r];
        P.rho[r] = __ldg(P.y + r) - sum;
    }
    group_sync(g);
}

// ---------------------------------------------------------------------------
// checkpoint scalar algebra on CTA 0 (problem.py:98-123, 57-86; regions.py:213-218)
// l1 over the support list (beta is zero elsewhere).
// ---------------------------------------------------------------------------
static __device__ void cta_dual(const SolveDev& P, double corr, int want_radius, bool l1_over_support, int64_t m,
                         double* red) {
    DevScalars* sc = P.sc;
    const double lam = P.lam;
    const int n = P.n;
    double a = 0.0, b = 0.0, aru = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const double q = P.rho[r];
        a = fma(q, q, a);
        b = fma(__ldg(P.y + r), q, b);
        aru = __dadd_ru(aru, __dmul_ru(q, q));
    }
    const double rho_sq = block_sum(a, red);
    const double y_rho = block_sum(b, red);
    const double rho_sq_ru = block_sum_ru(aru, red);
    double alpha = 0.0, margin = 1.0;
    int interp = 0;
    if (rho_sq == 0.0) {
        interp = 1;
    } else {
        const double raw = y_rho / (lam * rho_sq);
        if (corr > 0.0) {
            const double bound = 1.0 / corr;
            alpha = fmin(fmax(raw, -bound), bound);
        } else {
            alpha = raw;
        }
        margin = 1.0 - fabs(alpha) * corr;
    }
    double dd = 0.0, l1 = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const double th = interp ? 0.0 : alpha * P.rho[r];
        P.theta[r] = th;
        const double diff = th - __ldg(P.y + r) / lam;
        dd = fma(diff, diff, dd);
    }
    if (l1_over_support) {
        const int64_t s = sc->n_supp;
        for (int64_t i = threadIdx.x; i < s; i += blockDim.x) l1 += fabs(P.beta[P.S[i]]);
    } else {
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) l1 += fabs(P.beta[P.A[i]]);
    }
    const double dsq = block_sum(dd, red);
    const double l1s = block_sum(l1, red);
    if (threadIdx.x == 0) {
        const double dual = 0.5 * sc->y_norm_sq - 0.5 * (lam * lam) * dsq;
        const double primal = 0.5 * rho_sq + lam * l1s;
        const double gap = primal - dual;
        sc->rho_sq = rho_sq; sc->y_rho = y_rho; sc->alpha = alpha; sc->margin = margin; sc->interp = interp;
        sc->corr = corr; sc->l1 = l1s; sc->primal = primal; sc->dual = dual; sc->gap_pre = gap; sc->dsq = dsq;
        int st = ST_OK;
        if (margin < -1e-9) st = ST_INFEASIBLE;
        else if (want_radius && gap < -1e-10) st = ST_NEG_GAP;
        sc->status = st;
        sc->radius = sqrt(2.0 * fmax(gap, 0.0)) / lam;
        sc->rho_norm_ub = __dsqrt_ru(rho_sq_ru);
    }
    __syncthreads();
}

// mu_C(x_j) of the checkpoint region (regions.py:75-97) from the restricted dot
// c = x_j^T rho (theta = alpha rho) and q_j = x_j^T y (solver.py:104-119)
static __device__ __forceinline__ double rule_mu(const SolveDev& P, const DevScalars* sc, double c, int32_t j,
                                                 double nrm) {
    switch (P.rule) {
        case R_STATIC:
        case R_DYNAMIC: return fabs(__ldg(P.q + j) / P.lam) + sc->rule_r * nrm;
        case R_ST3: return fabs(__ldg(P.q + j) / P.lam - sc->rule_coef * __ldg(P.gstar + j)) + sc->rule_r * nrm;
        case R_GAP_DOME: return dome_mu(__ldg(P.q + j) / P.lam, sc->alpha * c, sc->rule_R, sc->rule_rd, sc->rule_a, nrm);
        default: return fabs(sc->alpha * c) + sc->radius * nrm;
    }
}

// region scalars of the checkpoint (thread 0 of CTA 0, after cta_dual):
// regions.py:162-165 (static), 168-174 (dynamic), 177-197 (ST3), 235-273 (dome)
static __device__ void rule_scalars(const SolveDev& P, DevScalars* sc) {
    const double lam = P.lam;
    sc->rule_trace_fixed = 0;
    if (sc->status != ST_OK) return;
    switch (P.rule) {
        case R_STATIC: {
            const double r = fabs(1.0 / lam - 1.0 / P.lmax_path) * sqrt(sc->y_norm_sq);
            sc->rule_r = r; sc->rule_trace_r = r; sc->rule_trace_fixed = 1;
            break;
        }
        case R_DYNAMIC: {
            const double r = sqrt(sc->dsq);
            sc->rule_r = r; sc->rule_trace_r = r; sc->rule_trace_fixed = 1;
            break;
        }
        case R_ST3: {
            const double big_r = sqrt(sc->dsq);
            const double nrm = __ldg(P.norms + P.jstar);
            const double qs = __ldg(P.q + P.jstar);
            const double sgn = qs > 0.0 ? 1.0 : (qs < 0.0 ? -1.0 : 1.0);
            const double dist = (P.lmax_path / lam - 1.0) / nrm;
            double rad = big_r * big_r - dist * dist;
            if (rad < 0.0) rad = 0.0;
            sc->rule_coef = (dist / nrm) * sgn;
            sc->rule_r = sqrt(rad); sc->rule_trace_r = sc->rule_r; sc->rule_trace_fixed = 1;
            break;
        }
        case R_GAP_DOME: {
            const double big_r = sqrt(sc->dsq);
            sc->rule_R = big_r;
            if (big_r > 0.0) {
                const double val = sc->y_norm_sq - sc->rho_sq - 2.0 * lam * sc->l1;
                double r_in = sqrt(fmax(val, 0.0)) / lam;
                if (r_in > big_r * (1 + 1e-9) + 1e-12) { sc->status = ST_NEG_GAP; return; }
                r_in = fmin(r_in, big_r);
                const double ratio = 2.0 * (r_in / big_r) * (r_in / big_r) - 1.0;
                sc->rule_rd = 0.5 * big_r;
                sc->rule_a = fmin(fmax(ratio, -1.0), 1.0);
            }
            break;
        }
        default: break;
    }
}

// post-drop certificate (solver.py:217-221): zero the dropped beta, add the
// drop-axpy drift to Delta, recompute P with the same theta, trace row.
static __device__ void cta_post(const SolveDev& P, double* red) {
    DevScalars* sc = P.sc;
    SolveCtl* ctl = P.ctl;
    const double lam = P.lam;
    const int n = P.n;
    // drift of the drop axpys (before zeroing beta)
    const int64_t nd = sc->n_drop;
    double dr = 0.0;
    for (int64_t k = threadIdx.x; k < nd; k += blockDim.x) {
        const int32_t j = P.Dl[k];
        dr = __dadd_ru(dr, __dmul_ru(fabs(P.beta[j]), __ldg(P.norms + j)));
    }
    const double drift = block_sum_ru(dr, red);
    for (int64_t k = threadIdx.x; k < nd; k += blockDim.x) P.beta[P.Dl[k]] = 0.0;
    __syncthreads();
    double a = 0.0, aru = 0.0, l1 = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const double q = P.rho[r];
        a = fma(q, q, a);
        aru = __dadd_ru(aru, __dmul_ru(q, q));
    }
    const int64_t s = sc->n_supp;
    for (int64_t i = threadIdx.x; i < s; i += blockDim.x) l1 += fabs(P.beta[P.S[i]]);
    const double rho_sq = block_sum(a, red);
    const double rho_sq_ru = block_sum_ru(aru, red);
    const double l1s = block_sum(l1, red);
    if (threadIdx.x == 0) {
        const double primal = 0.5 * rho_sq + lam * l1s;
        const double gap = primal - sc->dual;
        sc->primal_post = primal;
        sc->gap_post = gap;
        sc->radius_post = sqrt(2.0 * fmax(gap, 0.0)) / lam;
        const double anchor = sc->rho_norm_ub;          // pre-drop rho: the anchor of t
        ctl->anchor_norm = anchor;
        // rigorous drift bound of the drop axpys: sum|b_j||x_j| (1+k) + u (||rho0|| + drift)
        ctl->cd_delta = __dadd_ru(__dmul_ru(drift, 1.0 + 1e-12),
                                  __dmul_ru(2.3e-16 * (double)imax64(nd, 1), __dadd_ru(anchor, drift)));
        if (nd == 0) ctl->cd_delta = 0.0;
        sc->rho_norm_ub = __dsqrt_ru(rho_sq_ru);
        // solver.py:122-126: region radius for static/dynamic/ST3, gap radius otherwise
        const double tr = sc->rule_trace_fixed ? sc->rule_trace_r : sc->radius_post;
        if (ctl->ntrace < P.trace_cap) P.trace[ctl->ntrace] = TraceRow{ctl->passes, sc->m, gap, tr};
        ctl->ntrace++;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// CD epoch, dense, run by the first W warps of CTA 0
// ---------------------------------------------------------------------------
constexpr int kTTile = 8192;   // certification thresholds staged per tile (float), columns <= 16 KB
// threshold-tile length: halved for long columns so the TMA column ring keeps 4 slots
__host__ __device__ inline int cd_tile(int64_t ld, int es) { return ld * es > 16384 ? kTTile / 2 : kTTile; }

static __device__ __forceinline__ int64_t scan_tile(const float* ts, int64_t tb, int64_t tend, int64_t from, double D,
                                             int lane) {
    for (int64_t base = from; base < tend; base += 32) {
        const int64_t q = base + lane;
        const bool unc = q < tend && !(D < (double)ts[q - tb]);
        const unsigned b = __ballot_sync(0xffffffffu, unc);
        if (b) return base + __ffs(b) - 1;
    }
    return tend;
}

static __device__ __forceinline__ double delta_step(double D, double step, double rho0) {
    // ||rho_new - rho|| <= |d| ||x|| (1+u) + u ||rho_new||, ||rho_new|| <= rho0 + D + |d| ||x||
    return __dadd_ru(D, __dadd_ru(__dmul_ru(step, 1.0 + 1e-12), __dmul_ru(2.3e-16, __dadd_ru(__dadd_ru(rho0, D), step))));
}

// Serial CD chain, warp-specialized.
//
//   producer warp (warp W): one ballot over 32 staged thresholds yields every
//     candidate in the window -- positions uncertified under a pessimistic
//     drift bound Dp = Delta_published + margin.  Each lane then issues its own
//     candidate into its own ring slot: two TMA bulk copies (cp.async.bulk,
//     mbarrier complete_tx) for the column x_j (ld*sizeof(T) bytes) and its
//     packed ColInfo (nsq, 1/nsq, ||x||, u = lam/nsq, beta), then the slot
//     header (position, threshold, Dp, generation).  Entries are published
//     through the slot mbarriers (consumers test the entry's phase).
//   compute warps (0..W-1): one poll per entry; skip candidates certified
//     under the current Delta, otherwise run the chain
//     dot -> butterfly [-> cross-warp sum] ->
//     RN(g/nsq) (RN(1/nsq) + Markstein) -> soft threshold -> axpy, then publish
//     Delta.  If Delta outgrew an entry's Dp, positions between candidates may
//     no longer be certified: restart after the last processed position with a
//     new generation; stale entries are drained.
// Candidates are consumed strictly in ascending position order, so the
// arithmetic is exactly the sequential CD over the uncertified positions.
constexpr int kRingMax = 64;

struct alignas(16) SlotHdr {
    ColInfo ci;                      // TMA destination (48 B)
    double tcert;                    // certification threshold of the candidate
    double dp;                       // pessimistic Delta it was selected under
    int32_t pos;                     // candidate position; == m: end of epoch
    int32_t j;
    int32_t gen;
    int32_t flags;                   // kNoData: header-only entry (no column bytes)
};
constexpr int32_t kNoData = 1;

struct alignas(16) CdCtl {
    unsigned long long bar[kRingMax];     // mbarriers (TMA completion), one per slot
    int consumed[8];                      // per compute warp: entries fully read
    double dpub;                          // Delta published by compute warp 0
    int req_gen, req_pos;                 // restart request (compute -> producer)
    int finished, pad0, pad1, pad2;       // compute warps consumed the current-generation end entry
    double req_hint;                      // Gram windows: the restarted generation selects under >= this drift
};

// Gram-window consumer state (shared memory, see cd_consume_gram)
constexpr int kGM = 7;                                // members per window
constexpr int kGDots = kGM + kGM * (kGM - 1) / 2;     // h_b and Gram G(b,b'), b' < b: 28 <= 32 lanes
constexpr int kGEv = 512;                             // window span in positions = P-event capacity
struct alignas(16) GMem {
    double tc, dp, bj, ns, iv, uq, nr, pad;
    int32_t j, pos, pad0, pad1;
};
struct alignas(16) GWin {
    double part[8][32];          // per-warp reduced dots
    double vals[32];             // window dots: h_b at [b], G(b,b') at [kGM + b(b-1)/2 + b']
    GMem mem[kGM];
    double ev_t[kGEv], ev_dp[kGEv];
    int32_t ev_pos[kGEv], ev_gap[kGEv];
    unsigned gmin_t[kGM + 1], gmin_dp[kGM + 1];   // per gap: min t, min dp (float bits, dp rounded down)
    double dres[kGM], nbv[kGM];  // committed updates d_b (0: none) and new coefficients
    double D, gstep, term_dp;
    int ncommit, gen, wstart, done;
};

// first position in [from, lim) with !(D < t) (uncertified under D)
static __device__ __forceinline__ int scan_under(const float* ts, int tb, int lim, int from, double D, int lane) {
    for (int base = from; base < lim; base += 32) {
        const int q = base + lane;
        const bool unc = q < lim && !(D < (double)ts[q - tb]);
        const unsigned b = __ballot_sync(0xffffffffu, unc);
        if (b) return base + __ffs(b) - 1;
    }
    return lim;
}

// Gram-window consumer (P.cd_gram): the compute warps take the ring entries in
// windows of up to kGM "members" (candidates uncertified at the window start
// with a growth allowance: t <= Dq = D_s + Mg, Mg = 2 kGM gstep), load the
// members' rows into registers, and reduce ALL dots of the window at once --
// h_b = x_b^T rho and G(b,b') = x_b^T x_b' (b' < b) -- in one transposed
// butterfly (28 values, lane l ends with dot l).  Warp 0 then runs the
// coordinate chain in registers, every lane redundantly:
//     g_b = h_b - sum_{b'<b} d_b' G(b,b')   (accumulated as the d's appear)
//     z = beta + RN(g/nsq); soft threshold; d_b
// and the members' axpys rho -= d_b x_b are applied afterwards in member order
// with the reference's separate roundings (_kernels.py:60-64), so the stored
// rho is exactly the one sequential CD would store with these d's.
//
// The other candidates in the window span ("P events": certified at the
// window start) are re-checked at their turn against the running drift D: a
// P position that lost its certificate truncates the window there (members
// before it commit; the producer restarts at it), and an entry whose producer
// bound dp no longer covers D (positions between candidates may be
// uncertified) discards the window (nothing committed; restart at the window
// start under a larger drift hint).  Window boundaries are a function of the
// data (thresholds, D), never of timing, so results are bit-identical run to
// run (pkg/tests/test_path.py:124-131).
//
// Safety of skipping with the Gram form of g: relative to x_b^T rho_stored
// it adds the dot errors of h and G (<= gam ||x_b|| (||rho0|| + 2 Delta)),
// the missed axpy roundings x_b^T e_b' (<= ||x_b|| * the rounding part of
// each step, hence the doubled allowance in delta_step_g) and the final
// summation (<= 8u (|h| + sum |d G|)); gamma_n carries +40u for the latter,
// so cert_threshold's bound still implies a zero update.
static __device__ __forceinline__ double delta_step_g(double D, double step, double rho0) {
    return __dadd_ru(D, __dadd_ru(__dmul_ru(step, 1.0 + 1e-12), __dmul_ru(4.6e-16, __dadd_ru(__dadd_ru(rho0, D), step))));
}

template <typename T, int R>
static __device__ __forceinline__ void cd_consume_gram(const SolveDev& P, const int m, const int W,
                                                       const unsigned char* ring, const unsigned sbytes, const int kmask,
                                                       const unsigned bar_s, const int kshift, const unsigned cons_s, const unsigned fin_s,
                                                       const unsigned reqg_s, const unsigned reqp_s, const unsigned dpub_s,
                                                       CdCtl* cc, GWin* gw, float* ts, const bool use_t, const double rho0,
                                                       double (&rr)[R], double& D, double& gstep, int& n_unc, int& n_nz,
                                                       int& n_req, int& n_cand, int& n_skip, const int ct) {
    const int tid = ct, lane = tid & 31, w = tid >> 5, BT = W * 32;
    const unsigned FULL = 0xffffffffu;
    const int n = P.n;
    const unsigned mycons_s = cons_s + 4u * w;
    const unsigned lower = (1u << lane) - 1u;
    int k = 0, gen = 0, wstart = 0;
    double xw[kGM][R];
#pragma unroll
    for (int b = 0; b < kGM; ++b)
#pragma unroll
        for (int q = 0; q < R; ++q) xw[b][q] = 0.0;
    for (;;) {
        const double Mg = use_t ? __dmul_ru((double)kGM, gstep) : 0.0;
        const double Dq = use_t ? __dadd_ru(D, Mg) : 0.0;
        const int span_end = wstart + kGEv;
        int nmem = 0, nev = 0, term = 0, lastpos = -1, termpos = 0, ncand = 0;
        double term_dp = 0.0;
        // member b's header fields live in lane b of warp 0
        double m_tc = 0.0, m_dp = 0.0, m_bj = 0.0, m_ns = 0.0, m_iv = 0.0, m_uq = 0.0, m_nr = 0.0;
        int m_j = 0, m_pos = 0;
        const long long c0 = clock64();
        long long cw = 0;
        // ---------------- formation (every compute warp, identically) ----------------
        unsigned long long t0 = 0;
        while (term == 0) {
            const int idx = k + lane;
            const int s = idx & kmask;
            // entry idx is ready when its slot's phase (idx / K) & 1 completed; only
            // the next K entries can be tested (one use ahead at most)
            const bool rdy = lane <= kmask && mbar_test_s(bar_s + 8u * s, (unsigned)((idx >> kshift) & 1));
            const unsigned rb = __ballot_sync(FULL, rdy);
            const int nr = (rb == FULL) ? 32 : __ffs(~rb) - 1;
            if (nr == 0) {
                const long long cs = clock64();
                if (t0 == 0) t0 = gtimer();
                spin_guard(t0, 6, k, gen, wstart, nmem);
                cw += clock64() - cs;
                continue;
            }
            t0 = 0;
            const SlotHdr* h = reinterpret_cast<const SlotHdr*>(ring + (size_t)s * sbytes);
            int hg = -1, pos = 0, fl = 0;
            double tc = 0.0, dp = 0.0;
            if (lane < nr) { hg = h->gen; pos = h->pos; fl = h->flags; tc = h->tcert; dp = h->dp; }
            const bool live = lane < nr && hg == gen;
            const bool isend = live && pos >= m;
            const bool beyond = live && !isend && pos >= span_end;
            const bool inwin = live && !isend && !beyond;
            const bool isq = inwin && (!use_t || !(Dq < tc));
            const bool anom = live && use_t && ((dp < Dq) || (isq && (fl & kNoData)));
            const unsigned qb = __ballot_sync(FULL, isq);
            const unsigned tb = __ballot_sync(FULL, isend || beyond || anom);
            const int tpos = tb ? __ffs(tb) - 1 : 32;
            const int need = kGM - nmem;
            const int lastq = (__popc(qb) >= need) ? (int)__fns(qb, 0, need) : 32;   // need-th member
            int cut, tkind = 0;
            if (lastq < tpos) {
                cut = lastq + 1;
                tkind = 1;
            } else if (tpos < nr) {
                cut = tpos;
                tkind = __shfl_sync(FULL, anom ? 4 : (isend ? 2 : 3), tpos);
                termpos = __shfl_sync(FULL, pos, tpos);
                term_dp = __shfl_sync(FULL, dp, tpos);
            } else {
                cut = nr;
            }
            const unsigned below = cut >= 32 ? FULL : ((1u << cut) - 1u);
            if (tkind != 4) {
                const unsigned mb = qb & below;
                const unsigned iw = __ballot_sync(FULL, inwin) & below;
                const unsigned pb = iw & ~mb;
                const int cnt = __popc(mb);
                if (w == 0) {
                    if ((pb >> lane) & 1u) {                // P events (position-ordered)
                        const int e = nev + __popc(pb & lower);
                        gw->ev_t[e] = tc;
                        gw->ev_dp[e] = dp;
                        gw->ev_pos[e] = pos;
                        gw->ev_gap[e] = nmem + __popc(mb & lower);
                    }
                    if (cnt) {
                        // members of this batch -> lanes nmem .. nmem+cnt-1
                        double cbj = 0.0, cns = 0.0, civ = 0.0, cuq = 0.0, cnr = 0.0;
                        int cj = 0;
                        if ((mb >> lane) & 1u) {
                            cbj = h->ci.beta; cns = h->ci.ns; civ = h->ci.inv; cuq = h->ci.u; cnr = h->ci.nr; cj = h->j;
                        }
                        const int bi = lane - nmem;
                        const bool take = bi >= 0 && bi < cnt;
                        const int src = take ? (int)__fns(mb, 0, bi + 1) : lane;
                        const double x_tc = __shfl_sync(FULL, tc, src), x_dp = __shfl_sync(FULL, dp, src);
                        const double x_bj = __shfl_sync(FULL, cbj, src), x_ns = __shfl_sync(FULL, cns, src);
                        const double x_iv = __shfl_sync(FULL, civ, src), x_uq = __shfl_sync(FULL, cuq, src);
                        const double x_nr = __shfl_sync(FULL, cnr, src);
                        const int x_j = __shfl_sync(FULL, cj, src), x_pos = __shfl_sync(FULL, pos, src);
                        if (take) {
                            m_tc = x_tc; m_dp = x_dp; m_bj = x_bj; m_ns = x_ns; m_iv = x_iv; m_uq = x_uq; m_nr = x_nr;
                            m_j = x_j; m_pos = x_pos;
                        }
                    }
                }
                // members' rows, one predicated pass (warp-uniform conditions)
#pragma unroll
                for (int b = 0; b < kGM; ++b) {
                    if (b >= nmem && b < nmem + cnt) {
                        const int ml = (int)__fns(mb, 0, b - nmem + 1);
                        const SlotHdr* hm = reinterpret_cast<const SlotHdr*>(ring + (size_t)((k + ml) & kmask) * sbytes);
                        const T* xs = reinterpret_cast<const T*>(hm + 1) + tid;
#pragma unroll
                        for (int q = 0; q < R; ++q) xw[b][q] = (tid + q * BT < n) ? to_d(xs[q * BT]) : 0.0;
                    }
                }
                nev += __popc(pb);
                nmem += cnt;
                ncand += __popc(iw);
                if (iw) lastpos = __shfl_sync(FULL, pos, 31 - __clz(iw));
            }
            k += cut;
            term = tkind;
            __syncwarp();
            if (lane == 0) st_rel_s(mycons_s, k);          // entries before k fully read
        }
        if (term == 4) {
            // the producer's bound does not cover this window: restart at the
            // window start under a larger drift hint (nothing was consumed yet)
            ++gen;
            if (w == 0) ++n_req;
            if (tid == 0) {
                cc->req_hint = __dadd_ru(Dq, __dmul_ru(2.0, Mg));
                st_rel_s(reqp_s, wstart);
                st_rel_s(reqg_s, gen);
            }
            continue;
        }
        // ---------------- all dots of the window, then one transposed butterfly ----------------
        const long long c1 = clock64();
        if (nmem > 0) {
            double v[32];
#pragma unroll
            for (int b = 0; b < kGM; ++b) {
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int q = 0; q < R; q += 2) {
                    a0 = fma(xw[b][q], rr[q], a0);
                    if (q + 1 < R) a1 = fma(xw[b][q + 1], rr[q + 1], a1);
                }
                v[b] = a0 + a1;
#pragma unroll
                for (int b2 = 0; b2 < b; ++b2) {
                    double g0 = 0.0, g1 = 0.0;
#pragma unroll
                    for (int q = 0; q < R; q += 2) {
                        g0 = fma(xw[b][q], xw[b2][q], g0);
                        if (q + 1 < R) g1 = fma(xw[b][q + 1], xw[b2][q + 1], g1);
                    }
                    v[kGM + b * (b - 1) / 2 + b2] = g0 + g1;
                }
            }
#pragma unroll
            for (int i = kGDots; i < 32; ++i) v[i] = 0.0;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < o; ++i) {
                    const double send = up ? v[i] : v[i + o];
                    const double keep = up ? v[i + o] : v[i];
                    v[i] = keep + __shfl_xor_sync(FULL, send, o);
                }
            }
            gw->part[w][lane] = v[0];
        }
        named_bar(1, BT);
        const long long c2 = clock64();
        if (w == 0) {
            // ---------------- the coordinate chain (warp 0; lanes redundant, branch-free) ----------------
            double val = 0.0;
            if (nmem > 0)
                for (int q = 0; q < W; ++q) val += gw->part[q][lane];
            double acc[kGM];
#pragma unroll
            for (int b = 0; b < kGM; ++b) acc[b] = __shfl_sync(FULL, val, b);
            double Dl = D, gsl = gstep;
            double my_d = 0.0, my_nb = 0.0, my_D = D, my_gs = gstep;   // lane b: member b's update / drift before it
            unsigned procm = 0, nzm = 0;
#pragma unroll
            for (int b = 0; b < kGM; ++b) {
                const double tc = __shfl_sync(FULL, m_tc, b), bj = __shfl_sync(FULL, m_bj, b);
                const double ns = __shfl_sync(FULL, m_ns, b), iv = __shfl_sync(FULL, m_iv, b);
                const double uq = __shfl_sync(FULL, m_uq, b), nr = __shfl_sync(FULL, m_nr, b);
                if (lane == b) { my_D = Dl; my_gs = gsl; }
                const bool run = b < nmem && (!use_t || !(Dl < tc));     // certified members: zero update
                const double g = acc[b];
                const double q0 = g * iv;
                const double rq = fma(-q0, ns, g);
                const double qq = fma(rq, iv, q0);            // RN(g / nsq)
                const double z = bj + qq;
                const double nb = z > uq ? z - uq : (z < -uq ? z + uq : 0.0);
                const double d = run ? nb - bj : 0.0;
                procm |= run ? (1u << b) : 0u;
                if (d != 0.0) {
                    nzm |= 1u << b;
#pragma unroll
                    for (int b2 = b + 1; b2 < kGM; ++b2)
                        acc[b2] = fma(-d, __shfl_sync(FULL, val, kGM + b2 * (b2 - 1) / 2 + b), acc[b2]);
                    if (use_t) {
                        const double step = __dmul_ru(fabs(d), nr);
                        Dl = delta_step_g(Dl, step, rho0);
                        gsl = 0.875 * gsl + 0.125 * step;
                    }
                }
                if (lane == b) { my_d = d; my_nb = nb; }
            }
            if (lane == nmem) { my_D = Dl; my_gs = gsl; }            // trailing gap
            // ---- violations, resolved by position: discard (a bound no longer covers D)
            // or truncate (a P position lost its certificate) at the first one
            int kd = 0x7fffffff, kt = 0x7fffffff;
            if (use_t) {
                if (lane < nmem && my_D > m_dp) kd = m_pos;
                for (int e0 = 0; e0 < nev; e0 += 32) {
                    const int e = e0 + lane;
                    const int gp = e < nev ? gw->ev_gap[e] : 0;
                    const double De = __shfl_sync(FULL, my_D, gp);
                    if (e < nev) {
                        const int ps = gw->ev_pos[e];
                        if (De > gw->ev_dp[e]) kd = min(kd, ps);
                        else if (!(De < gw->ev_t[e])) kt = min(kt, ps);
                    }
                }
                kd = __reduce_min_sync(FULL, kd);
                kt = __reduce_min_sync(FULL, kt);
                if (term == 2 && Dl > term_dp) kd = min(kd, m);
            }
            int action = 0, ncommit = nmem, rpos = 0;
            double vio = Dl;
            if (kd != 0x7fffffff && kd <= kt) {
                action = 2;
                vio = Dl;
                ncommit = 0;
            } else if (kt != 0x7fffffff) {
                action = 1;
                rpos = kt;
                ncommit = __popc(__ballot_sync(FULL, lane < nmem && m_pos < kt));
                Dl = __shfl_sync(FULL, my_D, ncommit);
                gsl = __shfl_sync(FULL, my_gs, ncommit);
            }
            if (action == 2) { Dl = D; gsl = gstep; }
            // ---- commit
            int done = 0, nws = wstart;
            if (action == 0) {
                if (term == 2) done = 1;
                else nws = lastpos >= 0 ? lastpos + 1 : termpos;
            } else {
                ++gen;
                ++n_req;
                nws = action == 1 ? rpos : wstart;
                if (lane == 0) {
                    const double mg2 = __dmul_ru(2.0 * kGM, gsl);
                    cc->req_hint = action == 2 ? __dadd_ru(vio, mg2) : __dadd_ru(Dl, mg2);
                    st_rel_s(reqp_s, nws);
                    st_rel_s(reqg_s, gen);
                }
            }
            const unsigned cm = (1u << ncommit) - 1u;
            n_unc += __popc(procm & cm);
            n_nz += __popc(nzm & cm);
            n_skip += ncommit - __popc(procm & cm);
            n_cand += ncand;
            if (lane < kGM) gw->dres[lane] = (lane < ncommit) ? my_d : 0.0;
            if (lane < ncommit && ((nzm >> lane) & 1u)) {
                P.beta[m_j] = my_nb;
                P.cinfo[m_j].beta = my_nb;
                if (use_t && m_bj == 0.0) {
                    P.t[m_pos] = -1.0f;                      // now in the support
                    if (m <= cd_tile(P.ld, (int)sizeof(T))) ts[m_pos] = -1.0f;      // resident tile (single tile only)
                }
            }
            if (lane == 0) {
                gw->ncommit = ncommit;
                gw->D = Dl;
                gw->gstep = gsl;
                gw->gen = gen;
                gw->wstart = nws;
                gw->done = done;
                st_vol_f64_s(dpub_s, Dl);
                if (done) st_rel_s(fin_s, 1);
            }
        }
        named_bar(1, BT);
        const long long c3 = clock64();
        const int nc = gw->ncommit;
#pragma unroll
        for (int b = 0; b < kGM; ++b) {
            if (b < nc) {
                const double d = gw->dres[b];
                if (d != 0.0) {
#pragma unroll
                    for (int q = 0; q < R; ++q) rr[q] = __dsub_rn(rr[q], __dmul_rn(d, xw[b][q]));
                }
            }
        }
        D = gw->D;
        gstep = gw->gstep;
        gen = gw->gen;
        wstart = gw->wstart;
        if (P.cd_prof && tid == 0) {
            SolveCtl* c = P.ctl;
            const long long c4 = clock64();
            c->c_form += c1 - c0 - cw; c->c_wait += cw; c->c_red += c2 - c1; c->c_chain += c3 - c2; c->c_upd += c4 - c3;
            c->n_win += 1; c->n_mem += nmem;
        }
        if (gw->done) break;
    }
}

__host__ __device__ inline int cd_ring_slots(int64_t ld, int es) {
    // power of two, at most 64 slots and ~128 KB of ring
    const int64_t bytes = ld * es + 80;
    int k = 64;
    while (k > 4 && (int64_t)k * bytes > 128 * 1024) k >>= 1;
    return k;
}
__host__ __device__ inline size_t cd_slot_bytes(int64_t ld, int es) {
    return sizeof(SlotHdr) + (size_t)ld * es;          // ld * es is a multiple of 16
}
__host__ __device__ inline size_t cd_smem_bytes_rt(int64_t ld, int es) {
    return (size_t)cd_tile(ld, es) * (sizeof(float) + sizeof(int32_t)) + 64 * sizeof(double) + sizeof(CdCtl) + sizeof(GWin) +
           (size_t)cd_ring_slots(ld, es) * cd_slot_bytes(ld, es);
}

template <typename T, int R>
static __device__ __noinline__ void cd_epoch_dense(const SolveDev& P, int64_t m64, int W, unsigned char* smem,
                                            int* tile_valid) {
    SolveCtl* ctl = P.ctl;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int BT = W * 32;
    const int m = (int)m64;
    float* ts = reinterpret_cast<float*>(smem);
    const int TT = cd_tile(P.ld, (int)sizeof(T));
    int32_t* As = reinterpret_cast<int32_t*>(smem + TT * sizeof(float));
    double* part = reinterpret_cast<double*>(smem + TT * (sizeof(float) + sizeof(int32_t)));   // [2][32]
    CdCtl* cc = reinterpret_cast<CdCtl*>(part + 64);
    GWin* gw = reinterpret_cast<GWin*>(cc + 1);
    unsigned char* ring = reinterpret_cast<unsigned char*>(gw + 1);
    const int K = cd_ring_slots(P.ld, (int)sizeof(T));          // power of two
    const int kmask = K - 1, kshift = __ffs(K) - 1;
    const unsigned sbytes = (unsigned)cd_slot_bytes(P.ld, (int)sizeof(T));
    const unsigned xbytes = (unsigned)(P.ld * sizeof(T));
    const bool use_t = P.certify != 0;
    const int n = P.n;
    if (m == 0) {
        if (tid == 0) { ctl->epoch_unc = 0; ctl->epoch_nz = 0; }
        __syncthreads();
        return;
    }
    // ---- setup (all threads)
    if (tid == 0) {
        for (int s = 0; s < K; ++s) mbar_init(&cc->bar[s], 1);
        for (int k = 0; k < 8; ++k) cc->consumed[k] = 0;
        cc->dpub = use_t ? ctl->cd_delta : 0.0;
        cc->req_gen = 0;
        cc->req_pos = 0;
        cc->req_hint = 0.0;
        cc->finished = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const bool keep_tile = (m <= TT) && *tile_valid;
    if (!keep_tile) {
        const int lim = min(m, TT);
        for (int q = tid; q < lim; q += blockDim.x) {
            As[q] = P.A[q];
            ts[q] = use_t ? P.t[q] : -1.0f;
        }
    }
    __syncthreads();
    const unsigned ring_s = smem_u32(ring);
    const unsigned bar_s = smem_u32(&cc->bar[0]);
    // control words as 32-bit shared addresses, computed once
    const unsigned cons_s = smem_u32(&cc->consumed[0]), fin_s = smem_u32(&cc->finished);
    const unsigned reqg_s = smem_u32(&cc->req_gen), reqp_s = smem_u32(&cc->req_pos);
    const unsigned dpub_s = smem_u32(&cc->dpub);

    // warp roles: the W compute warps take the TOP warp ids and the producer
    // the one below them.  The scheduler of each SMSP (warps w, w+4) issues
    // the highest eligible warp id first, so the serial chain (compute warp 0)
    // never loses an issue slot to the spinning producer.
    const int wbase = (int)(blockDim.x >> 5) - W;
    if (w == wbase - 1) {
        // =================== producer warp ===================
        // Entries are published through the slot mbarriers themselves: the
        // header is written before the arrive (release), the column bytes
        // complete the phase (complete_tx), and consumers test the phase of
        // entry e (parity (e / K) & 1) lane-parallel.  Entry e is issued only
        // after entry e - K was consumed by every compute warp, so a phase is
        // never tested more than one use ahead.
        const T* __restrict__ X = (const T*)P.X;
        const ColInfo* __restrict__ cinfo = P.cinfo;
        const double gs0 = ctl->cd_gstep > 0.0 ? ctl->cd_gstep : 1e-2 * P.lam;
        // Gram windows (cd_gram): candidates are selected under dpub + 6 Mg, and
        // carry column bytes only when t <= dpub + 4 Mg (Mg = the consumer's
        // window-growth allowance); the rest are header-only entries whose
        // certification the consumer re-checks at their turn.
        const bool gram = P.cd_gram != 0;
        const double mg0 = __dmul_ru((double)kGM, gs0);
        const double margin_gs = gram ? __dmul_ru(6.0, mg0) : __dmul_ru(2.0 * K, gs0);
        const double margin_dat = __dmul_ru(4.0, mg0);
        const unsigned FULL = 0xffffffffu;
        double hint = 0.0;
        int tb = 0, tend = min(m, TT);
        int qnext = 0, gen = 0;
        int k_issue = 0;
        bool done = false;
        unsigned long long t0 = gtimer();       // reset on progress (watchdog)
        auto load_tile_p = [&](int from) {
            tb = (from / TT) * TT;
            tend = min(m, tb + TT);
            for (int q = tb + lane; q < tend; q += 32) { As[q - tb] = P.A[q]; ts[q - tb] = use_t ? P.t[q] : -1.0f; }
            __syncwarp();
        };
        asm volatile("fence.proxy.async.global;" ::: "memory");   // cinfo/beta stores before TMA reads
        while (true) {
            // control words: lane 0 fin, lane 1 restart generation, lanes 2.. consumed counters
            int cw = 0;
            if (lane == 0) cw = ld_acq_s(fin_s);
            else if (lane == 1) cw = ld_acq_s(reqg_s);
            else if (lane < 2 + W) cw = ld_acq_s(cons_s + 4u * (lane - 2));
            if (__shfl_sync(FULL, cw, 0)) break;
            const int rg = __shfl_sync(FULL, cw, 1);
            const int cmin = __reduce_min_sync(FULL, (lane >= 2 && lane < 2 + W) ? cw : 0x7fffffff);
            if (rg != gen) {
                gen = rg;
                const int rp = __shfl_sync(FULL, lane == 0 ? ld_acq_s(reqp_s) : 0, 0);
                double hv = lane == 0 ? cc->req_hint : 0.0;
                hint = __shfl_sync(FULL, hv, 0);
                if (rp < tb || rp > tend || (rp == tend && tend < m)) load_tile_p(rp);
                qnext = rp;
                done = false;
            }
            int free_slots = K - (k_issue - cmin);
            if (done || free_slots <= 0) {
                __nanosleep(32);
                spin_guard(t0, 1, k_issue, cmin, gen, (int)done);
                continue;
            }
            t0 = gtimer();
            double dpub = lane == 0 ? ld_vol_f64_s(dpub_s) : 0.0;
            dpub = __shfl_sync(FULL, dpub, 0);
            const double dp = use_t ? fmax(__dadd_ru(dpub, margin_gs), hint) : 0.0;
            const double dd = fmax(__dadd_ru(dpub, margin_dat), hint);   // column bytes for t <= dd (gram)
            // scan and issue until the free slots are used or the epoch ends
            int base = qnext;
            while (free_slots > 0) {
                if (base >= tend) {
                    if (tend >= m) {
                        // end of the epoch: an entry without data
                        if (lane == 0) {
                            const int s = k_issue & kmask;
                            SlotHdr* h = reinterpret_cast<SlotHdr*>(ring + (size_t)s * sbytes);
                            h->pos = m;
                            h->gen = gen;
                            h->dp = dp;                        // positions after the last candidate: certified under dp
                            h->flags = kNoData;
                            mbar_arrive_s(bar_s + 8u * s);     // release: the header is visible with the phase
                        }
                        ++k_issue;
                        done = true;
                        break;
                    }
                    load_tile_p(tend);
                    base = tb;
                    continue;
                }
                const int q = base + lane;
                const bool unc = q < tend && (!use_t || !(dp < (double)ts[q - tb]));
                const unsigned mask = __ballot_sync(FULL, unc);
                if (!mask) { base += 32; continue; }
                const int navail = min(__popc(mask), free_slots);
                const int rank = __popc(mask & ((1u << lane) - 1u));
                if (((mask >> lane) & 1u) && rank < navail) {
                    const int p = base + lane;
                    const int s = (k_issue + rank) & kmask;
                    const int32_t j = As[p - tb];
                    const unsigned slot = ring_s + (unsigned)s * sbytes;
                    const unsigned bb = bar_s + 8u * s;
                    const double tcp = (double)ts[p - tb];
                    const bool nodata = gram && use_t && dd < tcp;
                    SlotHdr* h = reinterpret_cast<SlotHdr*>(ring + (size_t)s * sbytes);
                    h->tcert = tcp;
                    h->dp = dp;
                    h->pos = p;
                    h->j = j;
                    h->gen = gen;
                    h->flags = nodata ? kNoData : 0;
                    if (nodata) {
                        mbar_arrive_s(bb);                     // header only: completes the phase at once
                    } else {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        mbar_expect_tx_s(bb, xbytes + (unsigned)sizeof(ColInfo));
                        tma_bulk_g2s_s(slot + (unsigned)sizeof(SlotHdr), X + (int64_t)j * P.ld, xbytes, bb);
                        tma_bulk_g2s_s(slot, cinfo + j, (unsigned)sizeof(ColInfo), bb);
                    }
                }
                const int lastbit = (int)__fns(mask, 0, navail);
                qnext = base + lastbit + 1;
                base = qnext;
                k_issue += navail;
                free_slots -= navail;
            }
            __syncwarp();
        }
        // drain outstanding transactions before the ring memory is reused:
        // the last min(K, k_issue) entries, one per slot
        {
            const int e = k_issue - 1 - lane;
            bool pend = lane < K && e >= 0;
            while (__any_sync(FULL, pend)) {
                if (pend && mbar_test_s(bar_s + 8u * (e & kmask), (unsigned)((e >> kshift) & 1))) pend = false;
                spin_guard(t0, 2, k_issue, 0, 0, 0);
            }
        }
    } else if (w >= wbase) {
        // =================== compute warps ===================
        const int tid = threadIdx.x - 32 * wbase, w = tid >> 5;     // index within the compute group
        double rr[R];
#pragma unroll
        for (int k = 0; k < R; ++k) { const int r = tid + k * BT; rr[k] = r < n ? P.rho[r] : 0.0; }
        double D = use_t ? ctl->cd_delta : 0.0;
        const double rho0 = ctl->anchor_norm;
        double gstep = ctl->cd_gstep > 0.0 ? ctl->cd_gstep : 1e-2 * P.lam;
        double* __restrict__ beta = P.beta;
        ColInfo* cinfo_w = P.cinfo;
        float* tg = P.t;
        int pb = 0, gen = 0, last = -1;
        int n_unc = 0, n_nz = 0, n_req = 0, n_cand = 0, n_skip = 0;
        const int cmask = min(7, (K >> 2) - 1);     // consumed is signalled every cmask+1 entries
        const unsigned mycons_s = cons_s + 4u * w;
        bool gram = false;
        if constexpr (R <= 4) gram = P.cd_gram != 0;     // member rows held in registers: R <= 4 only
        if (gram) {
            if constexpr (R <= 4)
                cd_consume_gram<T, R>(P, m, W, ring, sbytes, kmask, bar_s, kshift, cons_s, fin_s, reqg_s, reqp_s, dpub_s, cc,
                                      gw, ts, use_t, rho0, rr, D, gstep, n_unc, n_nz, n_req, n_cand, n_skip, tid);
        } else {
        bool pf = false;                 // entry k was prefetched under entry k-1's reduction
        int pf_pos = 0, pf_hg = 0, pf_j = 0;
        double pf_tc = 0.0, pf_dp = 0.0, pf_bj = 0.0, pf_ns = 0.0, pf_iv = 0.0, pf_uq = 0.0, pf_nr = 0.0;
        constexpr int RN = R <= 8 ? R : 1;
        double xvn[RN];
#pragma unroll
        for (int q = 0; q < RN; ++q) xvn[q] = 0.0;
        for (int k = 0;; ++k) {
            const int s = k & kmask;
            // entries before k are fully read: consumed is signalled in batches (release store)
            if (k > 0 && (k & cmask) == 0) { __syncwarp(); if (lane == 0) st_rel_s(mycons_s, k); }
            // one poll per entry (unless it was prefetched under the previous
            // entry's reduction): header and bytes are published together
            // through the slot mbarrier
            int pos, hg, j;
            double tc, dp, bj, ns, iv, uq, nr;
            const bool had_pf = pf;
            pf = false;
            if (had_pf) {
                pos = pf_pos; hg = pf_hg; j = pf_j; tc = pf_tc; dp = pf_dp;
                bj = pf_bj; ns = pf_ns; iv = pf_iv; uq = pf_uq; nr = pf_nr;
            } else {
                const unsigned par = (unsigned)((k >> kshift) & 1);
                if (!mbar_test_s(bar_s + 8u * s, par)) {
                    const unsigned long long t0 = gtimer();
                    while (!mbar_test_s(bar_s + 8u * s, par)) spin_guard(t0, 4, k, gen, last, 0);
                }
                const SlotHdr* h0 = reinterpret_cast<const SlotHdr*>(ring + (size_t)s * sbytes);
                pos = h0->pos; hg = h0->gen; j = h0->j; tc = h0->tcert; dp = h0->dp;
                bj = h0->ci.beta; ns = h0->ci.ns; iv = h0->ci.inv; uq = h0->ci.u; nr = h0->ci.nr;
            }
            const SlotHdr* h = reinterpret_cast<const SlotHdr*>(ring + (size_t)s * sbytes);
            bool process = hg == gen && pos < m;
            if (hg == gen && use_t && D > dp) {
                // drift outgrew the queue's bound (for the end entry: the positions
                // after the last candidate): restart after the last processed position
                ++n_req;
                ++gen;
                if (tid == 0) { st_rel_s(reqp_s, last + 1); st_rel_s(reqg_s, gen); }
                continue;
            }
            if (process && use_t && D < tc) {
                ++n_skip;                              // certified: zero update
                process = false;
            }
            if (!process) {
                if (hg == gen && pos >= m) {
                    if (tid == 0) st_rel_s(fin_s, 1);
                    break;
                }
                if (hg == gen) ++n_cand;
                continue;
            }
            ++n_cand;
            const T* xs = reinterpret_cast<const T*>(h + 1) + tid;
            // ---- critical chain
            constexpr int RX = R <= 8 ? R : 1;
            double xv[RX];
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if constexpr (R <= 8) {
#pragma unroll
                for (int q = 0; q < R; ++q) xv[q] = had_pf ? xvn[q] : ((tid + q * BT < n) ? to_d(xs[q * BT]) : 0.0);
#pragma unroll
                for (int q = 0; q < R; q += 2) {
                    a0 = fma(xv[q], rr[q], a0);
                    if (q + 1 < R) a1 = fma(xv[q + 1], rr[q + 1], a1);
                }
            } else {
                // long columns: stream the slot from shared memory (4 independent chains)
#pragma unroll
                for (int q = 0; q < R; q += 4) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double x = (q + u < R && tid + (q + u) * BT < n) ? to_d(xs[(q + u) * BT]) : 0.0;
                        const double r = q + u < R ? rr[q + u] : 0.0;
                        if (u == 0) a0 = fma(x, r, a0);
                        else if (u == 1) a1 = fma(x, r, a1);
                        else if (u == 2) a2 = fma(x, r, a2);
                        else a3 = fma(x, r, a3);
                    }
                }
            }
            // prefetch entry k+1 (header, ColInfo, this thread's rows) under the
            // reduction.  The slot address is selected by the phase test's
            // result: the loads are data-dependent on the (acquire) test, so
            // they cannot observe the slot before its phase completed, and no
            // branch holds the butterfly below behind the test's latency.
            {
                const int s1 = (k + 1) & kmask;
                pf = mbar_test_s(bar_s + 8u * s1, (unsigned)(((k + 1) >> kshift) & 1));
                const int sl = pf ? s1 : s;
                const SlotHdr* h1 = reinterpret_cast<const SlotHdr*>(ring + (size_t)sl * sbytes);
                pf_pos = h1->pos; pf_hg = h1->gen; pf_j = h1->j; pf_tc = h1->tcert; pf_dp = h1->dp;
                pf_bj = h1->ci.beta; pf_ns = h1->ci.ns; pf_iv = h1->ci.inv; pf_uq = h1->ci.u; pf_nr = h1->ci.nr;
                if constexpr (R <= 8) {
                    const T* xs1 = reinterpret_cast<const T*>(h1 + 1) + tid;
#pragma unroll
                    for (int q = 0; q < R; ++q) xvn[q] = (tid + q * BT < n) ? to_d(xs1[q * BT]) : 0.0;
                }
            }
            double acc = warp_sum((a0 + a1) + (a2 + a3));
            double g;
            if (W > 1) {
                if (lane == 0) part[pb * 32 + w] = acc;
                named_bar(1, BT);
                // warps' partials loaded together, summed in a fixed tree (W <= 7)
                double pw[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pw[q] = q < W ? part[pb * 32 + q] : 0.0;
                g = ((pw[0] + pw[1]) + (pw[2] + pw[3])) + ((pw[4] + pw[5]) + (pw[6] + pw[7]));
                pb ^= 1;
            } else {
                g = acc;
            }
            const double q0 = g * iv;
            const double rq = fma(-q0, ns, g);
            const double qq = fma(rq, iv, q0);            // RN(g / nsq)
            const double z = bj + qq;
            const double nb = z > uq ? z - uq : (z < -uq ? z + uq : 0.0);
            const double d = nb - bj;
            ++n_unc;
            last = pos;
            if (d != 0.0) {
                ++n_nz;
                if constexpr (R <= 8) {
#pragma unroll
                    for (int q = 0; q < R; ++q) rr[q] = __dsub_rn(rr[q], __dmul_rn(d, xv[q]));
                } else {
#pragma unroll
                    for (int q = 0; q < R; ++q)
                        rr[q] = __dsub_rn(rr[q], __dmul_rn(d, (tid + q * BT < n) ? to_d(xs[q * BT]) : 0.0));
                }
                if (use_t) {
                    const double step = __dmul_ru(fabs(d), nr);
                    D = delta_step(D, step, rho0);
                    gstep = 0.875 * gstep + 0.125 * step;
                }
                // bookkeeping stores by one lane that never signals consumption:
                // the consumed release (lane 0 of each warp) does not wait on them
                if (w == W - 1 && lane == 1) {
                    beta[j] = nb;
                    cinfo_w[j].beta = nb;
                    if (use_t && bj == 0.0) {
                        tg[pos] = -1.0f;                       // now in the support
                        if (m <= TT) ts[pos] = -1.0f;      // resident tile (single tile only)
                    }
                }
                if (lane == 0) st_vol_f64_s(dpub_s, D);
            }
        }
        }
        if (W > 1) named_bar(1, BT);
        double s2 = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int r = tid + q * BT;
            if (r < n) { P.rho[r] = rr[q]; s2 = __dadd_ru(s2, __dmul_ru(rr[q], rr[q])); }
        }
        s2 = warp_sum_ru(s2);
        if (W > 1) {
            if (lane == 0) part[pb * 32 + w] = s2;
            named_bar(1, BT);
            double tot = 0.0;
            for (int q = 0; q < W; ++q) tot = __dadd_ru(tot, part[pb * 32 + q]);
            s2 = tot;
        }
        if (tid == 0) {
            P.sc->rho_norm_ub = __dsqrt_ru(s2);
            ctl->cd_delta = D;
            ctl->cd_gstep = gstep;
            ctl->epoch_unc = n_unc;
            ctl->epoch_nz = n_nz;
            ctl->n_requeue += n_req;
            ctl->n_cand += n_cand;
            ctl->n_skip += n_skip;
            P.sc->visits += (unsigned long long)m;
            P.sc->uncertified += (unsigned long long)n_unc;
            P.sc->nonzero += (unsigned long long)n_nz;
        }
    }
    __syncthreads();
    if (tid == 0) {
        *tile_valid = (m <= TT) ? 1 : 0;
        for (int s = 0; s < K; ++s) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&cc->bar[s])) : "memory");
    }
    __syncthreads();
}

// CSC CD epoch: conflict-free waves (rho in shared memory).
//
// Coordinates whose columns share no row commute exactly: each reads and
// writes only the rho entries of its own rows.  Warp 0 schedules a wave over
// the positions [a, b): it walks them in order, skips those certified under a
// pessimistic drift bound dp = Delta + margin, and admits uncertified ones
// ("members") while their row sets are pairwise disjoint (a shared-memory row
// bitmap); the wave ends at the first conflicting candidate, a column with more
// than 32 nonzeros (run alone), 32 members or the tile end.  All warps then
// run the members' updates in parallel -- each reads exactly the rho values the
// sequential order would give it, so the arithmetic is the sequential CD's,
// bit for bit.  Afterwards the real drift of every skipped position is known
// (Delta + the members' steps before it); if one of them is no longer
// certified, the members after it are rolled back exactly (disjoint rows: the
// old rho values are restored) and the next wave starts at that position.
constexpr int kSpTile = 4096;    // thresholds + positions staged per tile
constexpr int kSpMW = 32;        // members per wave (one per lane of warp 0)
constexpr int kRowFree = 0x7f7f7f7f;   // row map value between waves (cudaMemset 0x7f)

struct SpMember {
    int32_t pos, j, nnz, pad;
    double ns, nr, bj, d, nb, step;
    int32_t idx[32];
    double val[32];
};

__host__ __device__ inline size_t cd_csc_smem_bytes(int64_t n) {
    const size_t a = (size_t)kSpTile * 8 + (size_t)n * 8 + (size_t)((n + 31) / 32) * 4;
    return (a + 15) / 16 * 16 + (size_t)kSpMW * sizeof(SpMember);
}

static __device__ __noinline__ void cd_epoch_csc(const SolveDev& P, int64_t m64, unsigned char* smem, int64_t lo64 = 0) {
    SolveCtl* ctl = P.ctl;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, NW = blockDim.x >> 5;
    const int n = P.n, m = (int)m64;
    const unsigned FULL = 0xffffffffu;
    float* ts = reinterpret_cast<float*>(smem);
    int32_t* As = reinterpret_cast<int32_t*>(smem + kSpTile * 4);
    double* srho = reinterpret_cast<double*>(smem + kSpTile * 8);
    const int nbw = (n + 31) / 32;
    unsigned* bm = reinterpret_cast<unsigned*>(srho + n);
    SpMember* mem = reinterpret_cast<SpMember*>(smem + ((size_t)kSpTile * 8 + (size_t)n * 8 + (size_t)nbw * 4 + 15) / 16 * 16);
    __shared__ double s_D;
    __shared__ int s_a, s_b, s_nmem, s_solo, s_tb, s_tend;
    const bool use_t = P.certify != 0;
    const double lam = P.lam;
    const double rho0 = ctl->anchor_norm;
    for (int r = tid; r < n; r += blockDim.x) srho[r] = P.rho[r];
    for (int k = tid; k < nbw; k += blockDim.x) bm[k] = 0u;
    if (tid == 0) { s_D = use_t ? ctl->cd_delta : 0.0; s_a = (int)lo64; s_tb = 0; s_tend = 0; }
    double gstep = ctl->cd_gstep > 0.0 ? ctl->cd_gstep : 1e-2 * lam;     // warp 0's copy
    long long n_unc = 0, n_nz = 0, n_roll = 0, n_mem = 0;                 // warp 0 lane 0
    __syncthreads();
    while (s_a < m) {
        const int a = s_a;
        if (a >= s_tend) {                       // stage the next tile of thresholds / positions
            const int tb = a, tend = min(m, a + kSpTile);
            for (int q = tb + tid; q < tend; q += blockDim.x) {
                As[q - tb] = P.A[q];
                ts[q - tb] = use_t ? P.t[q] : -1.0f;
            }
            __syncthreads();
            if (tid == 0) { s_tb = tb; s_tend = tend; }
            __syncthreads();
        }
        const int tb = s_tb, tend = s_tend;
        // ---------------- schedule (warp 0) ----------------
        if (w == 0) {
            const double D = s_D;
            const double dp = use_t ? __dadd_ru(D, __dmul_ru(2.0 * kSpMW, gstep)) : 0.0;
            int nmem = 0, b = -1, solo = 0;
            for (int base = a; b < 0; base += 32) {
                if (base >= tend) { b = tend; break; }
                const int q = base + lane;
                const bool unc = q < tend && (!use_t || !(dp < (double)ts[q - tb]));
                unsigned mask = __ballot_sync(FULL, unc);
                if (!mask) continue;
                // per-candidate column metadata, loaded in parallel by the candidate lanes
                int cj = 0, cnz = 0;
                int64_t clo = 0;
                double cns = 0.0, cnr = 0.0, cbj = 0.0;
                if (unc) {
                    cj = As[q - tb];
                    clo = __ldg(P.indptr + cj);
                    cnz = (int)(__ldg(P.indptr + cj + 1) - clo);
                    cns = __ldg(P.nsq + cj);
                    cnr = __ldg(P.norms + cj);
                    cbj = P.beta[cj];
                }
                while (mask && b < 0) {
                    // up to 8 candidates: their row lists are loaded together
                    int cl[8];
                    unsigned mm = mask;
#pragma unroll
                    for (int c = 0; c < 8; ++c) { cl[c] = mm ? __ffs(mm) - 1 : -1; if (mm) mm &= mm - 1; }
                    int ridx[8];
                    double rval[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        ridx[c] = -1; rval[c] = 0.0;
                        const int src = cl[c] < 0 ? 0 : cl[c];
                        const int64_t lo_c = __shfl_sync(FULL, clo, src);
                        const int nz_c = __shfl_sync(FULL, cnz, src);
                        if (cl[c] >= 0 && nz_c <= 32 && lane < nz_c) {
                            ridx[c] = __ldg(P.indices + lo_c + lane);
                            rval[c] = __ldg(P.data + lo_c + lane);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (cl[c] < 0 || b >= 0) continue;
                        const int lc = cl[c];
                        const int pos = base + lc;
                        const int nz_c = __shfl_sync(FULL, cnz, lc);
                        if (nz_c > 32) {                  // long column: alone in its wave
                            if (nmem > 0) { b = pos; break; }
                            solo = 1;
                        } else {
                            const int r = ridx[c];
                            const bool hit = r >= 0 && ((bm[r >> 5] >> (r & 31)) & 1u);
                            if (__ballot_sync(FULL, hit)) { b = pos; break; }
                            if (r >= 0) atomicOr(&bm[r >> 5], 1u << (r & 31));
                            if (lane < nz_c) { mem[nmem].idx[lane] = r; mem[nmem].val[lane] = rval[c]; }
                        }
                        if (lane == lc) {
                            SpMember& M = mem[nmem];
                            M.pos = pos; M.j = cj; M.nnz = cnz; M.ns = cns; M.nr = cnr; M.bj = cbj;
                        }
                        __syncwarp();
                        mask &= ~(1u << lc);
                        ++nmem;
                        if (solo || nmem == kSpMW) { b = pos + 1; break; }
                    }
                }
            }
            if (lane == 0) { s_b = b; s_nmem = nmem; s_solo = solo; }
        }
        __syncthreads();
        const int nmem = s_nmem;
        // ---------------- members in parallel (all warps) ----------------
        double oldv[kSpMW / 8 > 0 ? (kSpMW + 7) / 8 : 1];
#pragma unroll
        for (int it = 0; it < (kSpMW + 7) / 8; ++it) {
            oldv[it] = 0.0;
            const int k = w + it * NW;
            if (k >= nmem) continue;
            SpMember& M = mem[k];
            const double bj = M.bj, ns = M.ns;
            double g;
            int r = -1;
            double x = 0.0, o = 0.0;
            if (!s_solo) {
                if (lane < M.nnz) { r = M.idx[lane]; x = M.val[lane]; o = srho[r]; }
                g = warp_sum(fma(x, o, 0.0));
            } else {
                const int64_t lo = __ldg(P.indptr + M.j), hi = __ldg(P.indptr + M.j + 1);
                double acc = 0.0;
                for (int64_t q = lo + lane; q < hi; q += 32) acc = fma(__ldg(P.data + q), srho[__ldg(P.indices + q)], acc);
                g = warp_sum(acc);
            }
            const double z = bj + g / ns;
            const double u = lam / ns;
            const double nb = z > u ? z - u : (z < -u ? z + u : 0.0);
            const double d = nb - bj;
            if (d != 0.0) {
                if (!s_solo) {
                    if (r >= 0) srho[r] = __dsub_rn(o, __dmul_rn(d, x));
                } else {
                    __syncwarp();
                    const int64_t lo = __ldg(P.indptr + M.j), hi = __ldg(P.indptr + M.j + 1);
                    for (int64_t q = lo + lane; q < hi; q += 32) {
                        const int32_t rr = __ldg(P.indices + q);
                        srho[rr] = __dsub_rn(srho[rr], __dmul_rn(d, __ldg(P.data + q)));
                    }
                }
            }
            oldv[it] = o;
            if (lane == 0) { M.d = d; M.nb = nb; M.step = d != 0.0 ? __dmul_ru(fabs(d), M.nr) : 0.0; }
        }
        __syncthreads();
        // ---------------- drift bound, certification check, cut-off (warp 0) ----------------
        if (w == 0) {
            int b = s_b;
            double Dn = 0.0;
            if (use_t) {
                const double D = s_D;
                const double st = lane < nmem ? mem[lane].step : 0.0;
                double incl = st;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double t = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl = __dadd_ru(incl, t);
                }
                const double S = __shfl_sync(FULL, incl, 31);
                double excl = __shfl_up_sync(FULL, incl, 1);
                if (lane == 0) excl = 0.0;
                // per update: |d| ||x|| (1+1e-12) plus a rounding term u ||rho_new||,
                // ||rho_new|| <= rho0 + Delta + 2 S (see delta_step)
                const double err = __dmul_ru(2.3e-16, __dadd_ru(__dadd_ru(rho0, D), __dmul_ru(2.0, S)));
                auto Dk = [&](int k, double ex) {     // bound before member k (ex = steps of members < k)
                    return __dadd_ru(__dadd_ru(D, __dmul_ru(ex, 1.0 + 1e-12)), __dmul_ru((double)k, err));
                };
                Dn = Dk(nmem, S);
                const double dp = __dadd_ru(D, __dmul_ru(2.0 * kSpMW, gstep));
                if (Dn > dp) {
                    // find the first skipped position whose certificate fails under its real drift
                    int cut = -1;
                    for (int base = a; base < b && cut < 0; base += 32) {
                        const int s = base + lane;
                        bool bad = false;
                        if (s < b) {
                            int k = 0;                         // members before s
                            bool is_mem = false;
                            for (int q = 0; q < nmem; ++q) {
                                const int pq = mem[q].pos;
                                k += pq < s ? 1 : 0;
                                is_mem |= pq == s;
                            }
                            if (!is_mem) {
                                double ex = 0.0;               // steps of the members before s
                                for (int q = 0; q < k; ++q) ex = __dadd_ru(ex, mem[q].step);
                                bad = !(Dk(k, ex) < (double)ts[s - tb]);
                            }
                        }
                        const unsigned bb = __ballot_sync(FULL, bad);
                        if (bb) cut = base + __ffs(bb) - 1;
                    }
                    if (cut >= 0) {
                        b = cut;
                        int k = 0;
                        double ex = 0.0;
                        for (int q = 0; q < nmem; ++q)
                            if (mem[q].pos < cut) { ++k; ex = __dadd_ru(ex, mem[q].step); }
                        Dn = Dk(k, ex);
                        if (lane == 0) ++n_roll;
                    }
                }
            }
            // kept members: statistics and the step estimate
            if (lane == 0) {
                for (int q = 0; q < nmem; ++q) {
                    if (mem[q].pos >= b) break;
                    ++n_unc;
                    if (mem[q].d != 0.0) { ++n_nz; gstep = 0.875 * gstep + 0.125 * mem[q].step; }
                }
                n_mem += nmem;
                s_b = b;
                if (use_t) s_D = Dn;
            }
            gstep = __shfl_sync(FULL, gstep, 0);
        }
        __syncthreads();
        // ---------------- commit or roll back; release the rows ----------------
        {
            const int b = s_b;
#pragma unroll
            for (int it = 0; it < (kSpMW + 7) / 8; ++it) {
                const int k = w + it * NW;
                if (k >= nmem) continue;
                const SpMember& M = mem[k];
                const bool keep = M.pos < b;
                if (!s_solo && lane < M.nnz) {
                    const int r = M.idx[lane];
                    if (!keep && M.d != 0.0) srho[r] = oldv[it];
                    atomicAnd(&bm[r >> 5], ~(1u << (r & 31)));
                }
                if (keep && M.d != 0.0 && lane == 0) {
                    P.beta[M.j] = M.nb;
                    if (use_t && M.bj == 0.0) { P.t[M.pos] = -1.0f; ts[M.pos - tb] = -1.0f; }
                }
            }
            if (tid == 0) s_a = b;
        }
        __syncthreads();
    }
    if (tid == 0) {
        ctl->cd_delta = s_D;
        ctl->cd_gstep = gstep;
        ctl->epoch_unc = n_unc;
        ctl->epoch_nz = n_nz;
        ctl->n_requeue += n_roll;
        ctl->n_cand += n_mem;
        P.sc->visits += (unsigned long long)(m - (int)lo64);
        P.sc->uncertified += (unsigned long long)n_unc;
        P.sc->nonzero += (unsigned long long)n_nz;
    }
    __syncthreads();
    __shared__ double red[32];
    double s = 0.0;
    for (int r = tid; r < n; r += blockDim.x) { const double q = srho[r]; P.rho[r] = q; s = __dadd_ru(s, __dmul_ru(q, q)); }
    s = block_sum_ru(s, red);
    if (tid == 0) P.sc->rho_norm_ub = __dsqrt_ru(s);
    __syncthreads();
}


// CSC CD epoch, fully parallel waves (GS_CSC_PAR=1; experimental).
//
// Warp 0 admits the next (up to 32) candidates uncertified under dp with one
// ballot per 32 positions (a column with more than 32 nonzeros ends the wave
// before it, or runs alone).  All warps compute every member's g from the
// wave-start rho and its update d without writing rho.  Nonzero members mark
// their rows in a global row map (atomicMin of the member index); every member
// then checks its rows in parallel: a member that touches a row marked by an
// earlier nonzero member read a stale rho value, and the wave ends there.
// Accepted nonzero members have pairwise disjoint rows, so their axpys are
// applied in parallel -- the arithmetic is the sequential CD's, bit for bit.
// The certification cut-off and the statistics are those of cd_epoch_csc.
static __device__ __noinline__ void cd_epoch_csc_par(const SolveDev& P, int64_t m64, unsigned char* smem, int64_t lo64 = 0) {
    SolveCtl* ctl = P.ctl;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, NW = blockDim.x >> 5;
    const int n = P.n, m = (int)m64;
    const unsigned FULL = 0xffffffffu;
    float* ts = reinterpret_cast<float*>(smem);
    int32_t* As = reinterpret_cast<int32_t*>(smem + kSpTile * 4);
    double* srho = reinterpret_cast<double*>(smem + kSpTile * 8);
    const int nbw = (n + 31) / 32;
    SpMember* mem = reinterpret_cast<SpMember*>(smem + ((size_t)kSpTile * 8 + (size_t)n * 8 + (size_t)nbw * 4 + 15) / 16 * 16);
    int* first = P.rowmark;                      // n ints, kRowFree between waves
    __shared__ double s_D;
    __shared__ int s_a, s_b, s_nmem, s_solo, s_tb, s_tend;
    __shared__ int s_flag[kSpMW];
    __shared__ int64_t s_lo[kSpMW];
    const bool use_t = P.certify != 0;
    const double lam = P.lam;
    const double rho0 = ctl->anchor_norm;
    for (int r = tid; r < n; r += blockDim.x) srho[r] = P.rho[r];
    if (tid == 0) { s_D = use_t ? ctl->cd_delta : 0.0; s_a = (int)lo64; s_tb = 0; s_tend = 0; }
    double gstep = ctl->cd_gstep > 0.0 ? ctl->cd_gstep : 1e-2 * lam;
    long long n_unc = 0, n_nz = 0, n_roll = 0, n_mem = 0;
    __syncthreads();
    while (s_a < m) {
        const int a = s_a;
        if (a >= s_tend) {
            const int tb = a, tend = min(m, a + kSpTile);
            for (int q = tb + tid; q < tend; q += blockDim.x) {
                As[q - tb] = P.A[q];
                ts[q - tb] = use_t ? P.t[q] : -1.0f;
            }
            __syncthreads();
            if (tid == 0) { s_tb = tb; s_tend = tend; }
            __syncthreads();
        }
        const int tb = s_tb, tend = s_tend;
        // ---------------- admission (warp 0) ----------------
        // Pass 1 scans the staged thresholds only (shared memory): up to kSpMW uncertified
        // positions, lane k ends up with candidate k.  Pass 2 loads the candidates' column
        // pointers and constants in ONE parallel round (the round-1 version loaded them
        // inside the scan loop, a dependent global round trip per 32 positions).
        if (w == 0) {
            const double D = s_D;
            const double dp = use_t ? __dadd_ru(D, __dmul_ru(2.0 * kSpMW, gstep)) : 0.0;
            int nmem = 0, b = tend, solo = 0;
            for (int base = a; base < tend && nmem < kSpMW; base += 32) {
                const int q = base + lane;
                const bool unc = q < tend && (!use_t || !(dp < (double)ts[q - tb]));
                const unsigned mask = __ballot_sync(FULL, unc);
                const int cntm = __popc(mask), room = kSpMW - nmem, take = min(cntm, room);
                const int rank = __popc(mask & ((1u << lane) - 1u));
                if (unc && rank < take) s_flag[nmem + rank] = q;          // candidate list (positions)
                nmem += take;
                if (take < cntm) {
                    // the wave ends before the first candidate that did not fit
                    const unsigned nxt = __ballot_sync(FULL, unc && rank == take);
                    b = base + __ffs((int)nxt) - 1;
                    break;
                }
                if (nmem == kSpMW) { b = min(base + 32, tend); break; }
            }
            __syncwarp();
            int q = 0, cj = 0, cnz = 0;
            int64_t clo = 0;
            double c_ns = 0.0, c_nr = 0.0, c_bj = 0.0;
            if (lane < nmem) {
                q = s_flag[lane];
                cj = As[q - tb];
                clo = __ldg(P.indptr + cj);
                cnz = (int)(__ldg(P.indptr + cj + 1) - clo);
                c_ns = __ldg(P.nsq + cj); c_nr = __ldg(P.norms + cj); c_bj = P.beta[cj];
            }
            // a column with more than 32 nonzeros ends the wave before it, or runs alone
            const unsigned longm = __ballot_sync(FULL, lane < nmem && cnz > 32);
            if (longm) {
                const int fl = __ffs((int)longm) - 1;
                if (fl == 0) { nmem = 1; solo = 1; b = __shfl_sync(FULL, q, 0) + 1; }
                else { nmem = fl; b = __shfl_sync(FULL, q, fl); }
            }
            if (lane < nmem) {
                SpMember& M = mem[lane];
                M.pos = q; M.j = cj; M.nnz = cnz;
                M.ns = c_ns; M.nr = c_nr; M.bj = c_bj;
                s_lo[lane] = clo;
            }
            if (lane == 0) { s_b = b; s_nmem = nmem; s_solo = solo; }
        }
        __syncthreads();
        const int nmem = s_nmem;
        // ---------------- g and d of every member from the wave-start rho ----------------
        // the (up to four) members of this warp are loaded together: one global round trip
        // for their row indices and values instead of one per member
        constexpr int kIt = (kSpMW + 7) / 8;
        double oldv[kIt];
        if (!s_solo) {
            int rr_[kIt];
            double xx_[kIt];
#pragma unroll
            for (int it = 0; it < kIt; ++it) {
                const int k = w + it * NW;
                rr_[it] = -1; xx_[it] = 0.0;
                if (k < nmem && lane < mem[k].nnz) {
                    const int64_t lo = s_lo[k];
                    rr_[it] = __ldg(P.indices + lo + lane);
                    xx_[it] = __ldg(P.data + lo + lane);
                }
            }
#pragma unroll
            for (int it = 0; it < kIt; ++it) {
                oldv[it] = 0.0;
                const int k = w + it * NW;
                if (k >= nmem) continue;
                SpMember& M = mem[k];
                const int r = rr_[it];
                const double x = xx_[it];
                const double o = r >= 0 ? srho[r] : 0.0;
                M.idx[lane] = r; M.val[lane] = x;
                const double g = warp_sum(fma(x, o, 0.0));
                const double z = M.bj + g / M.ns;
                const double u = lam / M.ns;
                const double nb = z > u ? z - u : (z < -u ? z + u : 0.0);
                const double d = nb - M.bj;
                oldv[it] = o;
                __syncwarp();
                if (lane == 0) { M.d = d; M.nb = nb; M.step = d != 0.0 ? __dmul_ru(fabs(d), M.nr) : 0.0; }
            }
        } else {
#pragma unroll
            for (int it = 0; it < kIt; ++it) oldv[it] = 0.0;
            if (w == 0 && nmem > 0) {
                SpMember& M = mem[0];
                const int64_t lo = s_lo[0], hi = lo + M.nnz;
                double acc = 0.0;
                for (int64_t q = lo + lane; q < hi; q += 32) acc = fma(__ldg(P.data + q), srho[__ldg(P.indices + q)], acc);
                const double g = warp_sum(acc);
                const double z = M.bj + g / M.ns;
                const double u = lam / M.ns;
                const double nb = z > u ? z - u : (z < -u ? z + u : 0.0);
                const double d = nb - M.bj;
                __syncwarp();
                if (lane == 0) { M.d = d; M.nb = nb; M.step = d != 0.0 ? __dmul_ru(fabs(d), M.nr) : 0.0; }
            }
        }
        __syncthreads();
        // ---------------- conflicts with earlier nonzero members (row map) ----------------
        if (!s_solo && nmem > 1) {
#pragma unroll
            for (int it = 0; it < (kSpMW + 7) / 8; ++it) {
                const int k = w + it * NW;
                if (k < nmem && mem[k].d != 0.0 && lane < mem[k].nnz) atomicMin(first + mem[k].idx[lane], k);
            }
            __syncthreads();
            int own[(kSpMW + 7) / 8];
#pragma unroll
            for (int it = 0; it < (kSpMW + 7) / 8; ++it) {        // the four row-map reads in one round trip
                const int k = w + it * NW;
                own[it] = (k < nmem && lane < mem[k].nnz) ? __ldcg(first + mem[k].idx[lane]) : 0x7fffffff;
            }
#pragma unroll
            for (int it = 0; it < (kSpMW + 7) / 8; ++it) {
                const int k = w + it * NW;
                if (k >= nmem) continue;
                const unsigned hb = __ballot_sync(FULL, own[it] < k);
                if (lane == 0) s_flag[k] = hb != 0u;
            }
            __syncthreads();
            if (w == 0) {
                const bool f = lane < nmem && s_flag[lane];
                const unsigned fb = __ballot_sync(FULL, f);
                if (fb) {
                    const int cut = __ffs(fb) - 1;
                    if (lane >= cut && lane < nmem) mem[lane].step = 0.0;
                    __syncwarp();
                    if (lane == 0) s_b = mem[cut].pos;
                }
                __syncwarp();
            }
            __syncthreads();
        }
        // ---------------- drift bound, certification check, cut-off (warp 0) ----------------
        if (w == 0) {
            int b = s_b;
            double Dn = 0.0;
            if (use_t) {
                const double D = s_D;
                const double st = lane < nmem ? mem[lane].step : 0.0;
                double incl = st;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double t = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl = __dadd_ru(incl, t);
                }
                const double S = __shfl_sync(FULL, incl, 31);
                double excl = __shfl_up_sync(FULL, incl, 1);
                if (lane == 0) excl = 0.0;
                // per update: |d| ||x|| (1+1e-12) plus a rounding term u ||rho_new||,
                // ||rho_new|| <= rho0 + Delta + 2 S (see delta_step)
                const double err = __dmul_ru(2.3e-16, __dadd_ru(__dadd_ru(rho0, D), __dmul_ru(2.0, S)));
                auto Dk = [&](int k, double ex) {     // bound before member k (ex = steps of members < k)
                    return __dadd_ru(__dadd_ru(D, __dmul_ru(ex, 1.0 + 1e-12)), __dmul_ru((double)k, err));
                };
                Dn = Dk(nmem, S);
                const double dp = __dadd_ru(D, __dmul_ru(2.0 * kSpMW, gstep));
                if (Dn > dp) {
                    // find the first skipped position whose certificate fails under its real drift
                    int cut = -1;
                    for (int base = a; base < b && cut < 0; base += 32) {
                        const int s = base + lane;
                        bool bad = false;
                        if (s < b) {
                            int k = 0;                         // members before s
                            bool is_mem = false;
                            for (int q = 0; q < nmem; ++q) {
                                const int pq = mem[q].pos;
                                k += pq < s ? 1 : 0;
                                is_mem |= pq == s;
                            }
                            if (!is_mem) {
                                double ex = 0.0;               // steps of the members before s
                                for (int q = 0; q < k; ++q) ex = __dadd_ru(ex, mem[q].step);
                                bad = !(Dk(k, ex) < (double)ts[s - tb]);
                            }
                        }
                        const unsigned bb = __ballot_sync(FULL, bad);
                        if (bb) cut = base + __ffs(bb) - 1;
                    }
                    if (cut >= 0) {
                        b = cut;
                        int k = 0;
                        double ex = 0.0;
                        for (int q = 0; q < nmem; ++q)
                            if (mem[q].pos < cut) { ++k; ex = __dadd_ru(ex, mem[q].step); }
                        Dn = Dk(k, ex);
                        if (lane == 0) ++n_roll;
                    }
                }
            }
            // kept members: statistics and the step estimate
            if (lane == 0) {
                for (int q = 0; q < nmem; ++q) {
                    if (mem[q].pos >= b) break;
                    ++n_unc;
                    if (mem[q].d != 0.0) { ++n_nz; gstep = 0.875 * gstep + 0.125 * mem[q].step; }
                }
                n_mem += nmem;
                s_b = b;
                if (use_t) s_D = Dn;
            }
            gstep = __shfl_sync(FULL, gstep, 0);
        }
        __syncthreads();
        // ---------------- commit: accepted nonzero members (disjoint rows), release the row map ----------------
        {
            const int b = s_b;
#pragma unroll
            for (int it = 0; it < (kSpMW + 7) / 8; ++it) {
                const int k = w + it * NW;
                if (k >= nmem) continue;
                const SpMember& M = mem[k];
                const bool keep = M.pos < b;
                if (!s_solo) {
                    if (lane < M.nnz && M.d != 0.0) {
                        const int r = M.idx[lane];
                        if (keep) srho[r] = __dsub_rn(oldv[it], __dmul_rn(M.d, M.val[lane]));
                        if (nmem > 1) first[r] = kRowFree;
                    }
                } else if (keep && M.d != 0.0) {
                    const int64_t lo = s_lo[k], hi = lo + M.nnz;
                    for (int64_t q = lo + lane; q < hi; q += 32) {
                        const int32_t rr = __ldg(P.indices + q);
                        srho[rr] = __dsub_rn(srho[rr], __dmul_rn(M.d, __ldg(P.data + q)));
                    }
                }
                if (keep && M.d != 0.0 && lane == 0) {
                    P.beta[M.j] = M.nb;
                    if (use_t && M.bj == 0.0) { P.t[M.pos] = -1.0f; ts[M.pos - tb] = -1.0f; }
                }
            }
            if (tid == 0) s_a = b;
        }
        __syncthreads();
    }
    if (tid == 0) {
        ctl->cd_delta = s_D;
        ctl->cd_gstep = gstep;
        ctl->epoch_unc = n_unc;
        ctl->epoch_nz = n_nz;
        ctl->n_requeue += n_roll;
        ctl->n_cand += n_mem;
        P.sc->visits += (unsigned long long)(m - (int)lo64);
        P.sc->uncertified += (unsigned long long)n_unc;
        P.sc->nonzero += (unsigned long long)n_nz;
    }
    __syncthreads();
    __shared__ double red[32];
    double s = 0.0;
    for (int r = tid; r < n; r += blockDim.x) { const double q = srho[r]; P.rho[r] = q; s = __dadd_ru(s, __dmul_ru(q, q)); }
    s = block_sum_ru(s, red);
    if (tid == 0) P.sc->rho_norm_ub = __dsqrt_ru(s);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// the persistent solve kernel
// ---------------------------------------------------------------------------
}  // namespace gs
#include "gs_cd_blk.cuh"
namespace gs {

// dense CD epoch: blocked chain (cd_gram == 2, R <= 5) or the ring consumers
template <typename T, int R>
static __device__ __forceinline__ void cd_epoch_dense_any(const SolveDev& P, int64_t m, unsigned char* smem,
                                                          int* tile_valid) {
    if constexpr (R <= 5) {
        if (P.cd_gram == 2) { cd_epoch_blk<T, R>(P, m, P.cd_warps, smem, tile_valid); return; }
    }
    cd_epoch_dense<T, R>(P, m, P.cd_warps, smem, tile_valid);
}

template <typename T, int R>
static __device__ void solve_body(const SolveDev& P, const Group& g, unsigned char* smem) {
    __shared__ int sh[32];
    __shared__ double red[32];
    // CSC designs always launch the R = 1 instantiation (gs_api.cu: launch_solve): the
    // long-column instantiation compiles the sparse branches out, which leaves the direct
    // CD chain (96 registers of rho) a leaner caller
    constexpr bool kMaySparse = R < 48;
    const bool sparse_ = kMaySparse && P.sparse;
    DevScalars* sc = P.sc;
    SolveCtl* ctl = P.ctl;
    // dense: [CD tile | vs]; sparse: the CD uses [t tile | rho] and vs aliases it
    double* vs = reinterpret_cast<double*>(smem + (sparse_ ? 0 : P.cd_bytes));
    __shared__ int s_tile_valid;
    if (threadIdx.x == 0) s_tile_valid = 0;
    __syncthreads();
    const bool gap_rule = P.rule == R_GAP_SPHERE;
    const bool screening = P.rule != R_NONE;
    const double gam = gamma_n(sparse_ ? (int64_t)P.n : (int64_t)P.n);

    if (ctl->done) return;

    // ---- init: active set, beta zeroed outside it (solver.py:163-178) ----
    if (!ctl->started) {
        if (P.init_mode == 2) {
            // sequential gap-sphere screen (path.py:82-91): gap at the new lambda
            // for the previous (beta, theta, rho), then the fused full-p test.
            if (g.c == 0) {
                const double lam = P.lam;
                double a = 0.0, dd = 0.0, l1 = 0.0;
                for (int r = threadIdx.x; r < P.n; r += blockDim.x) {
                    const double q = P.rho[r];
                    a = fma(q, q, a);
                    const double diff = P.theta[r] - __ldg(P.y + r) / lam;
                    dd = fma(diff, diff, dd);
                }
                const int64_t m0 = sc->m;
                for (int64_t i = threadIdx.x; i < m0; i += blockDim.x) l1 += fabs(P.beta[P.A[i]]);
                const double rho_sq = block_sum(a, red), dsq = block_sum(dd, red), l1s = block_sum(l1, red);
                if (threadIdx.x == 0) {
                    const double primal = 0.5 * rho_sq + lam * l1s;
                    const double dual = 0.5 * sc->y_norm_sq - 0.5 * (lam * lam) * dsq;
                    const double gap = primal - dual;
                    int st = ST_OK;
                    if (P.rule == R_GAP_DOME) {
                        // region_gap_dome(prob_t, beta_prev, theta_prev, rho_prev) (regions.py:250-273)
                        if (P.prev_margin < -1e-9) st = ST_VALUE;
                        const double big_r = sqrt(dsq);
                        sc->rule_R = big_r;
                        if (st == ST_OK && big_r > 0.0) {
                            const double val = sc->y_norm_sq - rho_sq - 2.0 * lam * l1s;
                            double r_in = sqrt(fmax(val, 0.0)) / lam;
                            if (r_in > big_r * (1 + 1e-9) + 1e-12) st = ST_NEG_GAP;
                            r_in = fmin(r_in, big_r);
                            const double ratio = 2.0 * (r_in / big_r) * (r_in / big_r) - 1.0;
                            sc->rule_rd = 0.5 * big_r;
                            sc->rule_a = fmin(fmax(ratio, -1.0), 1.0);
                        }
                    } else {
                        if (P.prev_margin < -1e-9) st = ST_INFEASIBLE;
                        else if (gap < -1e-10) st = ST_NEG_GAP;
                    }
                    sc->status = st;
                    sc->gap_pre = gap;
                    sc->radius = sqrt(2.0 * fmax(gap, 0.0)) / lam;
                }
            }
            group_sync(g);
            if (sc->status != ST_OK) { if (g.c == 0 && threadIdx.x == 0) ctl->done = 1; return; }
            const unsigned long long ts0 = gtimer();
            group_gemv<T>(g, P, P.theta, nullptr, P.p, G_MU, nullptr, nullptr, 0.0, gam, sc->radius, vs, smem, sparse_ ? 0 : P.cd_bytes, &s_tile_valid);
            group_sync(g);
            if (g.c == 0 && threadIdx.x == 0) { ctl->t_screen += gtimer() - ts0; ctl->n_screen++; }
        } else if (P.init_mode == 0) {
            for (int64_t j = (int64_t)g.c * blockDim.x + threadIdx.x; j < P.p; j += (int64_t)g.G * blockDim.x)
                P.mark[j] = __ldg(P.norms + j) > 0.0;
            group_sync(g);
        } else {
            const int64_t n0 = sc->cnt;
            for (int64_t i = (int64_t)g.c * blockDim.x + threadIdx.x; i < n0; i += (int64_t)g.G * blockDim.x) {
                const int32_t j = P.A2[i];
                if (__ldg(P.norms + j) > 0.0) P.mark[j] = 1;
            }
            group_sync(g);
        }
        // A = {j : mark_j}; beta_j = 0 off A; mark cleared
        group_compact2(g, P, P.p,
                       [&](int64_t j) { return P.mark[j] != 0; },
                       [&](int64_t j, int64_t o) { P.A[o] = (int32_t)j; },
                       [&](int64_t) { return false; }, [&](int64_t, int64_t) {},
                       &sc->m, nullptr, sh);
        group_sync(g);
        for (int64_t j = (int64_t)g.c * blockDim.x + threadIdx.x; j < P.p; j += (int64_t)g.G * blockDim.x) {
            if (!P.mark[j]) P.beta[j] = 0.0;
            P.mark[j] = 0;
            const double ns = __ldg(P.nsq + j);
            if (!sparse_) {
                ColInfo ci;
                ci.ns = ns;
                ci.inv = __ldg(P.inv_nsq + j);
                ci.nr = __ldg(P.norms + j);
                ci.u = ns > 0.0 ? P.lam / ns : 0.0;   // u = lam / nsq (_kernels.py:51), per lambda
                ci.beta = P.beta[j];
                ci.pad = 0.0;
                P.cinfo[j] = ci;
            }
        }
        if (g.c == 0 && threadIdx.x == 0) {
            ctl->started = 1;
            ctl->k = 1;
            ctl->passes = 0;
            ctl->ntrace = 0;
            ctl->nckpt = 0;
            ctl->resume = 0;
            ctl->pending = PEND_NONE;
            ctl->converged = 0;
            ctl->need_refresh = 1;
            ctl->cd_delta = 0.0;
        }
        group_sync(g);
    }

    int64_t k = ctl->k;
    int32_t pending = ctl->pending;
    bool broke = false, converged = false;
    if (pending == PEND_CONVERGED) { converged = true; k = P.max_passes + 1; }
    else if (pending == PEND_BREAK) { broke = true; k = P.max_passes + 1; }

    while (k <= P.max_passes) {
        const bool ckpt_pass = (P.f == 1 || k % P.f == 1);
        const bool is_ckpt = ckpt_pass && pending != PEND_CONTINUE;
        pending = PEND_NONE;
        if (is_ckpt) {
            const unsigned long long tc0 = gtimer();
            int64_t m = sc->m;
            group_resync<T>(g, P, m, sh);
            if (m == 0) {
                // everything screened: unrestricted dual point (solver.py:190-203)
                group_gemv<T>(g, P, P.rho, nullptr, P.p, G_DUAL, nullptr, nullptr, 0.0, gam, 0.0, vs, smem, sparse_ ? 0 : P.cd_bytes, &s_tile_valid);
                group_sync(g);
                if (g.c == 0) {
                    double corr; int64_t ci;
                    group_max_result(g, P, corr, ci);
                    cta_dual(P, corr, 0, true, 0, red);
                    if (threadIdx.x == 0) {
                        sc->n_drop = 0;
                        sc->gap_post = sc->gap_pre;
                        sc->primal_post = sc->primal;
                        sc->radius_post = sqrt(2.0 * fmax(sc->gap_pre, 0.0)) / P.lam;
                        if (ctl->ntrace < P.trace_cap) P.trace[ctl->ntrace] = TraceRow{ctl->passes, 0, sc->gap_pre, sc->radius_post};
                        ctl->ntrace++;
                        ctl->nckpt++;
                        ctl->pending = sc->gap_pre <= P.eps ? PEND_CONVERGED : PEND_BREAK;
                        ctl->k = k;
                    }
                }
                group_sync(g);
                if (sc->status != ST_OK) { if (g.c == 0 && threadIdx.x == 0) ctl->done = 1; return; }
            } else {
                // restricted |X_A^T rho|_inf with the dots kept for mu and the anchor
                group_gemv<T>(g, P, P.rho, P.A, m, G_DUAL, P.c, nullptr, 0.0, gam, 0.0, vs, smem, sparse_ ? 0 : P.cd_bytes, &s_tile_valid);
                group_sync(g);
                if (g.c == 0) {
                    double corr; int64_t ci;
                    group_max_result(g, P, corr, ci);
                    cta_dual(P, corr, gap_rule ? 1 : 0, true, m, red);
                    if (threadIdx.x == 0) rule_scalars(P, sc);
                    __syncthreads();
                }
                group_sync(g);
                if (sc->status != ST_OK) { if (g.c == 0 && threadIdx.x == 0) ctl->done = 1; return; }
                const double alpha = sc->alpha, radius = sc->radius, anchor = sc->rho_norm_ub;
                const bool cert = P.certify != 0;
                if (screening) {
                    // keep = mu >= 1 - 1e-9 with mu = |alpha c| + r ||x|| (solver.py:208-216);
                    // kept positions carry their certification thresholds along.
                    const int32_t* A = P.A;
                    group_compact2(g, P, m,
                                   [&](int64_t i) {
                                       const double mu = rule_mu(P, sc, P.c[i], A[i], __ldg(P.norms + A[i]));
                                       return mu >= 1.0 - 1e-9;
                                   },
                                   [&](int64_t i, int64_t o) {
                                       const int32_t j = A[i];
                                       P.A2[o] = j;
                                       if (cert) {
                                           const double tt = (P.beta[j] != 0.0) ? -1.0 : cert_threshold(P.c[i], __ldg(P.norms + j), P.lam, anchor, gam);
                                           P.t2[o] = __double2float_rd(tt);
                                       }
                                   },
                                   [&](int64_t i) {
                                       const double mu = rule_mu(P, sc, P.c[i], A[i], __ldg(P.norms + A[i]));
                                       return !(mu >= 1.0 - 1e-9) && P.beta[A[i]] != 0.0;
                                   },
                                   [&](int64_t i, int64_t o) { P.Dl[o] = A[i]; },
                                   &sc->m, &sc->n_drop, sh);
                    group_sync(g);
                    // drop axpys rho += beta_j x_j, ascending j (numpy order per element)
                    const int64_t nd = sc->n_drop;
                    if (nd > 0) {
                        if (sparse_) {
                            if (g.c == 0) {
                                for (int64_t q0 = 0; q0 < nd; ++q0) {
                                    const int32_t j = P.Dl[q0];
                                    const double bj = P.beta[j];
                                    for (int64_t q = __ldg(P.indptr + j) + threadIdx.x; q < __ldg(P.indptr + j + 1); q += blockDim.x) {
                                        const int32_t r = __ldg(P.indices + q);
                                        P.rho[r] = __dadd_rn(P.rho[r], __dmul_rn(bj, __ldg(P.data + q)));
                                    }
                                    __syncthreads();
                                }
                            }
                        } else {
                            const T* X = (const T*)P.X;
                            for (int64_t r = (int64_t)g.c * blockDim.x + threadIdx.x; r < P.n; r += (int64_t)g.G * blockDim.x) {
                                double q = P.rho[r];
                                for (int64_t q0 = 0; q0 < nd; ++q0) {
                                    const int64_t j = P.Dl[q0];
                                    q = __dadd_rn(q, __dmul_rn(P.beta[j], to_d(__ldg(X + j * P.ld + r))));
                                }
                                P.rho[r] = q;
                            }
                        }
                    }
                    group_sync(g);
                    if (g.c == 0) {
                        cta_post(P, red);
                        if (threadIdx.x == 0) { ctl->need_refresh = cert ? 0 : 1; }
                    }
                } else {
                    // rule none: no drop; thresholds for all positions at this anchor
                    if (cert) {
                        for (int64_t i = (int64_t)g.c * blockDim.x + threadIdx.x; i < m; i += (int64_t)g.G * blockDim.x) {
                            const int32_t j = P.A[i];
                            const double tt = (P.beta[j] != 0.0) ? -1.0 : cert_threshold(P.c[i], __ldg(P.norms + j), P.lam, anchor, gam);
                            P.t[i] = __double2float_rd(tt);
                        }
                    }
                    if (g.c == 0 && threadIdx.x == 0) { sc->m = m; sc->n_drop = 0; }
                    group_sync(g);
                    if (g.c == 0) {
                        cta_post(P, red);
                        if (threadIdx.x == 0) ctl->need_refresh = 0;
                    }
                }
                if (g.c == 0 && threadIdx.x == 0) {
                    ctl->nckpt++;
                    const int64_t mn = sc->m;
                    ctl->pending = sc->gap_post <= P.eps ? PEND_CONVERGED : (mn == 0 ? PEND_BREAK : PEND_CONTINUE);
                    ctl->k = k;
                }
                group_sync(g);
                if (screening) {
                    // swap A/A2 and t/t2 (device pointers are per launch; the host swaps between launches)
                    // handled by copying back: the compaction wrote the new active set into A2/t2
                    const int64_t mn = sc->m;
                    for (int64_t i = (int64_t)g.c * blockDim.x + threadIdx.x; i < mn; i += (int64_t)g.G * blockDim.x) {
                        P.A[i] = P.A2[i];
                        if (cert) P.t[i] = P.t2[i];
                    }
                    group_sync(g);
                }
            }
            if (g.c == 0 && threadIdx.x == 0) { ctl->t_ckpt += gtimer() - tc0; s_tile_valid = 0; }
            pending = ctl->pending;
            if (P.stop_at_ckpt) {
                if (g.c == 0 && threadIdx.x == 0) { ctl->k = k; }
                return;   // host fires the checkpoint hook, then relaunches
            }
            if (pending == PEND_CONVERGED) { converged = true; break; }
            if (pending == PEND_BREAK) { broke = true; break; }
            pending = PEND_NONE;
        } else if (!ckpt_pass && k % 100 == 0) {
            group_resync<T>(g, P, sc->m, sh);
            if (g.c == 0) {
                double a = 0.0;
                for (int r = threadIdx.x; r < P.n; r += blockDim.x) { const double q = P.rho[r]; a = __dadd_ru(a, __dmul_ru(q, q)); }
                const double s = block_sum_ru(a, red);
                if (threadIdx.x == 0) { sc->rho_norm_ub = __dsqrt_ru(s); ctl->need_refresh = 1; }
            }
            group_sync(g);
        }
        // ---- one CD epoch over the active set ----
        const int64_t m = sc->m;
        // Sparse designs: the epoch runs in position chunks, each re-anchored (c_i, t_i
        // from the current rho, Delta = 0) by the whole group just before CTA 0 walks it.
        // The norm-based drift bound is far too pessimistic for 20-nonzero columns once
        // a few hundred updates have accumulated; with the drift restarted per chunk the
        // uncertified visits fall to about the support (exact skips only, so the
        // arithmetic is unchanged).  One pass over X_A per epoch in total.
        const int nch = (sparse_ && P.certify && P.cd_chunk_pos > 0 && m > 0)
                            ? (int)imin64(256, imax64(1, (m + P.cd_chunk_pos - 1) / P.cd_chunk_pos)) : 1;
        if (nch > 1) {
            int64_t unc = 0, nz = 0;
            for (int ch = 0; ch < nch; ++ch) {
                const int64_t c0 = m * ch / nch, c1 = m * (ch + 1) / nch;
                const unsigned long long tr0 = gtimer();
                const double anchor = sc->rho_norm_ub;
                group_gemv<T>(g, P, P.rho, P.A + c0, c1 - c0, G_CERT, P.c + c0, P.t + c0, anchor, gam, 0.0, vs, smem, 0, &s_tile_valid);
                if (g.c == 0 && threadIdx.x == 0) { ctl->anchor_norm = anchor; ctl->cd_delta = 0.0; ctl->n_refresh++; }
                group_sync(g);
                if (g.c == 0) {
                    const unsigned long long td0 = gtimer();
                    if (threadIdx.x == 0) ctl->t_refresh += td0 - tr0;
                    if (P.csc_par && P.rowmark) cd_epoch_csc_par(P, c1, smem, c0); else cd_epoch_csc(P, c1, smem, c0);
                    if (threadIdx.x == 0) ctl->t_cd += gtimer() - td0;
                    unc += ctl->epoch_unc; nz += ctl->epoch_nz;
                }
                group_sync(g);
            }
            if (g.c == 0 && threadIdx.x == 0) {
                ctl->epoch_unc = unc; ctl->epoch_nz = nz;
                ctl->passes++;
                ctl->need_refresh = 0;
            }
            group_sync(g);
            ++k;
            continue;
        }
        if (P.certify && ctl->need_refresh && m > 0) {
            const unsigned long long tr0 = gtimer();
            const double anchor = sc->rho_norm_ub;
            group_gemv<T>(g, P, P.rho, P.A, m, G_CERT, P.c, P.t, anchor, gam, 0.0, vs, smem, sparse_ ? 0 : P.cd_bytes, &s_tile_valid);
            if (g.c == 0 && threadIdx.x == 0) { ctl->anchor_norm = anchor; ctl->cd_delta = 0.0; ctl->n_refresh++; s_tile_valid = 0; }
            group_sync(g);
            if (g.c == 0 && threadIdx.x == 0) ctl->t_refresh += gtimer() - tr0;
        }
        if (g.c == 0) {
            const unsigned long long td0 = gtimer();
            if (sparse_) { if (P.csc_par && P.rowmark) cd_epoch_csc_par(P, m, smem); else cd_epoch_csc(P, m, smem); }
            else cd_epoch_dense_any<T, R>(P, m, smem, &s_tile_valid);
            if (threadIdx.x == 0) {
                ctl->t_cd += gtimer() - td0;
                ctl->passes++;
                ctl->need_refresh = (ctl->epoch_unc - ctl->epoch_nz > P.refresh_excess) ? 1 : 0;
            }
        }
        group_sync(g);
        ++k;
    }
    // ---- budget exhausted or early break: certify the final iterate (solver.py:237-245)
    if (!converged) {
        const int64_t m = sc->m;
        group_resync<T>(g, P, m, sh);
        if (m > 0) group_gemv<T>(g, P, P.rho, P.A, m, G_DUAL, nullptr, nullptr, 0.0, gam, 0.0, vs, smem, sparse_ ? 0 : P.cd_bytes, &s_tile_valid);
        else group_gemv<T>(g, P, P.rho, nullptr, P.p, G_DUAL, nullptr, nullptr, 0.0, gam, 0.0, vs, smem, sparse_ ? 0 : P.cd_bytes, &s_tile_valid);
        group_sync(g);
        if (g.c == 0) {
            double corr; int64_t ci;
            group_max_result(g, P, corr, ci);
            cta_dual(P, corr, 0, true, m, red);
            if (threadIdx.x == 0) {
                ctl->converged = sc->gap_pre <= P.eps;
                ctl->final_done = 1;
            }
        }
    } else if (g.c == 0 && threadIdx.x == 0) {
        ctl->converged = 1;
    }
    if (g.c == 0 && threadIdx.x == 0) { ctl->done = 1; ctl->k = k; }
    if (P.cd_prof && g.c == 0 && threadIdx.x == 0 && ctl->n_win)
    {
        const double nw = (double)ctl->n_win;
        if (P.cd_gram == 2)
            printf("cdprof lam=%.6e windows=%llu members=%llu cyc/win warp0: wait=%.0f dots=%.0f bar=%.0f chain=%.0f commit=%.0f"
                   " | warp1: wait=%.0f dots=%.0f bar=%.0f chain=%.0f commit=%.0f | producer: idle=%.0f scan=%.0f issue=%.0f\n",
                   P.lam, ctl->n_win, ctl->n_mem,
                   ctl->c_wait / nw, ctl->c_red / nw, ctl->c_upd / nw, ctl->c_chain / nw, ctl->c_form / nw,
                   ctl->c_w1[0] / nw, ctl->c_w1[1] / nw, ctl->c_w1[2] / nw, ctl->c_w1[3] / nw, ctl->c_w1[4] / nw,
                   ctl->c_w1[5] / nw, ctl->c_pr[0] / nw, ctl->c_pr[1] / nw);
        else
            printf("cdprof lam=%.6e windows=%llu members=%llu cyc/win: form=%.0f wait=%.0f red=%.0f chain=%.0f upd=%.0f\n", P.lam,
                   ctl->n_win, ctl->n_mem, ctl->c_form / nw, ctl->c_wait / nw, ctl->c_red / nw, ctl->c_chain / nw,
                   ctl->c_upd / nw);
    }
    (void)broke;
}

template <typename T, int R>
__global__ void __launch_bounds__(256, 1) k_solve(const SolveDev* __restrict__ probs, int G) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x / G;
    const SolveDev& P = probs[prob];
    Group g{G, (int)(blockIdx.x % G), P.bar};
    solve_body<T, R>(P, g, smem);
}

// gs_cd_pass production twin: anchor at the incoming rho, one refresh, one
// certified CD epoch (single CTA).
template <typename T, int R>
__global__ void __launch_bounds__(256, 1) k_cd_pass_prod(const SolveDev* __restrict__ probs) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double red[32];
    const SolveDev& P = probs[0];
    Group g{1, 0, nullptr};
    const int64_t m = P.sc->m;
    if (!P.sparse)
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
            const int32_t j = P.A[i];
            const double ns = __ldg(P.nsq + j);
            ColInfo ci;
            ci.ns = ns; ci.inv = __ldg(P.inv_nsq + j); ci.nr = __ldg(P.norms + j);
            ci.u = ns > 0.0 ? P.lam / ns : 0.0; ci.beta = P.beta[j]; ci.pad = 0.0;
            P.cinfo[j] = ci;
        }
    double a = 0.0;
    for (int r = threadIdx.x; r < P.n; r += blockDim.x) { const double q = P.rho[r]; a = __dadd_ru(a, __dmul_ru(q, q)); }
    const double anchor = __dsqrt_ru(block_sum_ru(a, red));
    const double gam = gamma_n(P.n);
    if (P.certify) group_gemv<T>(g, P, P.rho, P.A, m, G_CERT, P.c, P.t, anchor, gam, 0.0,
                                 reinterpret_cast<double*>(smem + (P.sparse ? 0 : P.cd_bytes)), smem,
                                 P.sparse ? 0 : P.cd_bytes, nullptr);
    if (threadIdx.x == 0) { P.ctl->anchor_norm = anchor; P.ctl->cd_delta = 0.0; }
    __syncthreads();
    __shared__ int s_tile_valid;
    if (threadIdx.x == 0) s_tile_valid = 0;
    __syncthreads();
    if (P.sparse) cd_epoch_csc(P, m, smem);
    else cd_epoch_dense_any<T, R>(P, m, smem, &s_tile_valid);
}

// standalone full-p screening pass (the same group_gemv G_MU code the
// persistent kernel runs for the sequential screen); P.theta = center.
template <typename T>
__global__ void __launch_bounds__(256, 1) k_screen_full(const SolveDev* __restrict__ probs, double radius) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SolveDev& P = probs[0];
    Group g{(int)gridDim.x, (int)blockIdx.x, nullptr};
    group_gemv_impl<T>(g, P, P.theta, nullptr, P.p, G_MU, nullptr, nullptr, 0.0, 0.0, radius,
                  reinterpret_cast<double*>(smem + (P.sparse ? 0 : P.cd_bytes)), smem, P.sparse ? 0 : P.cd_bytes,
                  nullptr);
}

// ---------------------------------------------------------------------------
// Batched independent problems (BASELINE cfg4, stability selection): one CTA
// per problem runs its whole warm-started lambda path on the device -- the
// lambda loop, the lambda_max shortcut, the sequential screen and every solve
// -- so problems never wait for each other (no per-lambda global barrier).
// ---------------------------------------------------------------------------
struct BatchOut {
    const double* grid;     // [T] lambdas of this problem
    double lmax;
    double* betas;          // [T * p] or nullptr
    int64_t* passes;        // [T]
    double* gaps;           // [T]
    int32_t* converged;     // [T]
    int64_t* n_active;      // [T]
    int T;
};

template <typename T, int R>
static __device__ void batch_problem(SolveDev* probs, const BatchOut* outs, const int b, unsigned char* smem) {
    __shared__ SolveDev sp;
    __shared__ int sh[32];
    if (threadIdx.x == 0) sp = probs[b];
    __syncthreads();
    const BatchOut& o = outs[b];
    Group g{1, 0, nullptr};
    DevScalars* sc = sp.sc;
    SolveCtl* ctl = sp.ctl;
    const int64_t p = sp.p;
    const int n = sp.n;
    double prev_margin = 1.0;
    int prev_interp = 0;
    const bool gap_rule = sp.rule == 1;
    for (int t = 0; t < o.T; ++t) {
        const double lam = o.grid[t];
        if (lam >= o.lmax * (1 - 1e-14)) {
            // _solve_at_lambda_max (solver.py:129-146): beta = 0, theta = y/lam, rho = y,
            // active = {|x_j^T theta| >= 1 - 1e-9} (rule gap) or nonzero-norm columns
            for (int64_t j = threadIdx.x; j < p; j += blockDim.x) sp.beta[j] = 0.0;
            for (int r = threadIdx.x; r < n; r += blockDim.x) {
                const double y = sp.y[r];
                sp.rho[r] = y;
                sp.theta[r] = y / lam;
            }
            __syncthreads();
            if (gap_rule) {
                group_gemv<T>(g, sp, sp.theta, nullptr, p, G_MU, nullptr, nullptr, 0.0, 0.0, 0.0,
                              reinterpret_cast<double*>(smem + (sp.sparse ? 0 : sp.cd_bytes)), smem,
                              sp.sparse ? 0 : sp.cd_bytes, nullptr);
            } else {
                for (int64_t j = threadIdx.x; j < p; j += blockDim.x) sp.mark[j] = __ldg(sp.norms + j) > 0.0;
            }
            __syncthreads();
            group_compact2(g, sp, p,
                           [&](int64_t j) { return sp.mark[j] != 0; },
                           [&](int64_t j, int64_t q) { sp.A[q] = (int32_t)j; },
                           [&](int64_t) { return false; }, [&](int64_t, int64_t) {},
                           &sc->m, nullptr, sh);
            __syncthreads();
            for (int64_t j = threadIdx.x; j < p; j += blockDim.x) sp.mark[j] = 0;
            if (threadIdx.x == 0) {
                o.passes[t] = 0;
                o.gaps[t] = 0.0;
                o.converged[t] = 1;
                o.n_active[t] = sc->m;
            }
            prev_margin = 0.0;
            prev_interp = 0;
        } else {
            if (threadIdx.x == 0) {
                sp.lam = lam;
                sp.init_mode = (gap_rule && t > 0 && !prev_interp) ? 2 : 0;
                sp.prev_margin = prev_margin;
                sc->lam = lam;
                sc->status = ST_OK;
                SolveCtl z{};
                *ctl = z;
            }
            __syncthreads();
            solve_body<T, R>(sp, g, smem);
            __syncthreads();
            if (threadIdx.x == 0) {
                o.passes[t] = ctl->passes;
                o.gaps[t] = ctl->final_done ? sc->gap_pre : sc->gap_post;
                o.converged[t] = sc->status != ST_OK ? -1 : ctl->converged;
                o.n_active[t] = sc->m;
            }
            prev_margin = sc->margin;
            prev_interp = sc->interp;
            if (sc->status != ST_OK) break;   // error status: stop this problem (host raises)
        }
        if (o.betas) {
            double* dst = o.betas + (int64_t)t * p;
            for (int64_t j = threadIdx.x; j < p; j += blockDim.x) dst[j] = sp.beta[j];
        }
        __syncthreads();
    }
}

// Persistent batched driver: min(B, #SM) CTAs claim problems from a global
// counter, so long and short bootstrap paths pack dynamically instead of in
// static waves of one problem per CTA.  Each problem's arithmetic does not
// depend on which CTA runs it (results are bit-identical to any schedule).
template <typename T, int R>
__global__ void __launch_bounds__(256, 1) k_batch_path(SolveDev* probs, const BatchOut* outs, int B, int* next) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_b;
    for (;;) {
        if (threadIdx.x == 0) s_b = atomicAdd(next, 1);
        __syncthreads();
        const int b = s_b;
        __syncthreads();
        if (b >= B) break;
        batch_problem<T, R>(probs, outs, b, smem);
        __syncthreads();
    }
}

}  // namespace gs
