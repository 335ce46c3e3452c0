// Sequential CSC CD epoch with a producer warp (P.csc_seq; columns of at most
// 32 nonzeros: cfg3's 20).  cd_pass_csc (_kernels.py:67-92) one coordinate at a
// time, in the reference's order, on ONE warp -- with everything that is not
// the arithmetic taken off that warp's path.
//
// Why not waves: after the per-chunk re-anchoring (gs_solve.cuh, chunked
// epochs) nearly every uncertified coordinate is a support member, so a wave of
// "commuting" members is cut by a row conflict after ~16 members, and each wave
// pays ~10 us of admission, row-map round trips and block barriers: 0.4-0.6 us
// per member.  A short column needs only a 20-row gather from rho (shared
// memory), one butterfly, a division and a 20-row scatter: ~350 cycles.
//
// Roles (one CTA):
//   * producer (warp 1): scans the staged thresholds for the next window of up
//     to kSqW uncertified positions under a drift bound Dp, loads the members'
//     column pointers and constants (one parallel round), writes the window
//     descriptor and issues the TMA bulk copies of their values and row
//     indices (16-byte aligned spans that contain the column) into a ring of
//     kSqSlots window slots, one mbarrier per slot;
//   * consumer (warp 0): rho in shared memory; per member: gather, dot
//     (the wave kernel's lane partition and butterfly, so the value is
//     bit-identical to it), z = beta + g / nsq, soft threshold, scatter with
//     the reference's separate roundings, drift update.  A member after which
//     D > Dp ends the window there and posts a restart request (position,
//     drift) under a new generation; windows of the old generation are
//     discarded unread.
// The arithmetic of a processed coordinate does not depend on which other
// positions are members, so -- unlike the blocked dense chain -- the bound may
// follow the published drift at any time without affecting results.
#pragma once

namespace gs {

constexpr int kSqW = 16;          // members per window
constexpr int kSqSlots = 4;       // window slots in flight
constexpr int kSqCap = 40;        // entries per member copy: 32 + alignment slack, multiple of 4
constexpr int kSqTile = 2048;     // thresholds + positions staged per tile
constexpr int kSqMaxNnz = 32;

struct alignas(16) SqDesc {
    double dp;
    int32_t cnt, last, gen, pad;
    int32_t pos[kSqW], j[kSqW], nnz[kSqW], off[kSqW];
    double ns[kSqW], nr[kSqW], bj[kSqW], u[kSqW];
};
struct alignas(16) SqSlot {
    double val[kSqW][kSqCap];
    int32_t idx[kSqW][kSqCap];
};
struct alignas(16) SqCtl {
    unsigned long long bar[kSqSlots];
    SqDesc desc[kSqSlots];
    double d_pub, g_pub, req_d, req_g;
    int cons, req_gen, req_pos, done;
};

__host__ __device__ inline size_t cd_csc_seq_smem_bytes(int64_t n) {
    const size_t a = (size_t)kSqTile * 8 + (size_t)n * 8;
    return (a + 15) / 16 * 16 + sizeof(SqCtl) + (size_t)kSqSlots * sizeof(SqSlot);
}

static __device__ __noinline__ void cd_epoch_csc_seq(const SolveDev& P, int64_t m64, unsigned char* smem, int64_t lo64 = 0) {
    SolveCtl* ctl = P.ctl;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n = P.n, m = (int)m64, lo = (int)lo64;
    const unsigned FULL = 0xffffffffu;
    float* ts = reinterpret_cast<float*>(smem);
    int32_t* As = reinterpret_cast<int32_t*>(smem + kSqTile * 4);
    double* srho = reinterpret_cast<double*>(smem + kSqTile * 8);
    SqCtl* sc_ = reinterpret_cast<SqCtl*>(smem + ((size_t)kSqTile * 8 + (size_t)n * 8 + 15) / 16 * 16);
    SqSlot* slots = reinterpret_cast<SqSlot*>(sc_ + 1);
    const bool use_t = P.certify != 0;
    const double lam = P.lam;
    const double D0 = use_t ? ctl->cd_delta : 0.0;
    const double gstep0 = ctl->cd_gstep > 0.0 ? ctl->cd_gstep : 1e-2 * lam;
    for (int r = tid; r < n; r += blockDim.x) srho[r] = P.rho[r];
    if (tid == 0) {
        for (int s = 0; s < kSqSlots; ++s) mbar_init(&sc_->bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sc_->d_pub = D0; sc_->g_pub = gstep0; sc_->req_d = 0.0; sc_->req_g = 0.0;
        sc_->cons = 0; sc_->req_gen = 0; sc_->req_pos = 0; sc_->done = 0;
    }
    __syncthreads();
    const unsigned bar_s = smem_u32(&sc_->bar[0]);
    const unsigned cons_s = smem_u32(&sc_->cons), reqg_s = smem_u32(&sc_->req_gen), done_s = smem_u32(&sc_->done);
    const double mfac = 2.0 * kSqW;

    if (w == 1) {
        // ================= producer =================
        const double* __restrict__ p_data = P.data;
        const int32_t* __restrict__ p_indices = P.indices;
        const int64_t* __restrict__ p_indptr = P.indptr;
        const double* __restrict__ p_nsq = P.nsq;
        const double* __restrict__ p_norms = P.norms;
        const double* p_beta = P.beta;
        const int32_t* p_A = P.A;
        const float* p_t = P.t;
        int cur = lo, tb = lo, tend = lo;              // first scan step loads a tile
        int gen = 0, q = 0;
        bool emitted_last = false;
        double Dp = use_t ? __dadd_ru(D0, __dmul_ru(mfac, gstep0)) : 0.0;
        for (;;) {
            bool stop = false;
            {
                const unsigned long long t0 = gtimer();
                for (;;) {
                    if (ld_acq_s(done_s)) { stop = true; break; }
                    const int rg = ld_acq_s(reqg_s);
                    if (rg != gen) {
                        gen = rg;
                        cur = *(volatile int*)&sc_->req_pos;
                        if (cur < tb || cur >= tend) { tb = cur; tend = cur; }     // reload at the next scan step
                        Dp = use_t ? __dadd_ru(*(volatile double*)&sc_->req_d, __dmul_ru(mfac, *(volatile double*)&sc_->req_g)) : 0.0;
                        emitted_last = false;
                    }
                    if (!emitted_last && ld_acq_s(cons_s) >= q - (kSqSlots - 1)) break;
                    spin_guard(t0, 21, q, gen, cur, 0);
                }
            }
            if (stop) break;
            if (use_t)
                Dp = fmax(Dp, __dadd_ru(*(volatile double*)&sc_->d_pub, __dmul_ru(mfac, *(volatile double*)&sc_->g_pub)));
            const int slot = q % kSqSlots;
            SqDesc* dsc = &sc_->desc[slot];
            int found = 0;
            while (found < kSqW && cur < m) {
                if (cur >= tend) {
                    tb = cur;
                    tend = min(m, tb + kSqTile);
                    for (int qq = tb + lane; qq < tend; qq += 32) { As[qq - tb] = p_A[qq]; ts[qq - tb] = use_t ? p_t[qq] : -1.0f; }
                    __syncwarp();
                }
                const int qp = cur + lane;
                const bool unc = qp < tend && !(Dp < (double)ts[qp - tb]);
                const unsigned mask = __ballot_sync(FULL, unc);
                const int avail = __popc(mask), take = min(avail, kSqW - found);
                const int rank = __popc(mask & ((1u << lane) - 1u));
                if (unc && rank < take) { dsc->pos[found + rank] = qp; dsc->j[found + rank] = As[qp - tb]; }
                if (take < avail) {
                    const unsigned nxt = __ballot_sync(FULL, unc && rank == take);
                    cur += __ffs((int)nxt) - 1;
                } else {
                    cur = min(cur + 32, tend);
                }
                found += take;
            }
            const int last = (cur >= m) ? 1 : 0;
            __syncwarp();
            // the members' pointers and constants: one parallel round of loads
            int64_t lo4 = 0;
            int cnt4 = 0;
            if (lane < found) {
                const int j = dsc->j[lane];
                const int64_t plo = __ldg(p_indptr + j), phi = __ldg(p_indptr + j + 1);
                const double ns = __ldg(p_nsq + j);
                const int nnz = (int)(phi - plo);
                lo4 = plo & ~(int64_t)3;
                const int off = (int)(plo - lo4);
                cnt4 = nnz > 0 ? ((off + nnz + 3) & ~3) : 0;
                dsc->nnz[lane] = nnz; dsc->off[lane] = off;
                dsc->ns[lane] = ns; dsc->nr[lane] = __ldg(p_norms + j); dsc->bj[lane] = p_beta[j];
                dsc->u[lane] = lam / ns;                       // u = lam / nsq (_kernels.py:79), off the consumer's path
            }
            int bytes = cnt4 * 12;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(FULL, bytes, o);
            if (lane == 0) { dsc->dp = Dp; dsc->cnt = found; dsc->last = last; dsc->gen = gen; }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            const unsigned bb = bar_s + 8u * slot;
            if (lane == 0) {
                if (bytes) mbar_expect_tx_s(bb, (unsigned)bytes);
                else mbar_arrive_s(bb);
            }
            __syncwarp();
            if (lane < found && cnt4) {
                tma_bulk_g2s_s(smem_u32(&slots[slot].val[lane][0]), p_data + lo4, (unsigned)(cnt4 * 8), bb);
                tma_bulk_g2s_s(smem_u32(&slots[slot].idx[lane][0]), p_indices + lo4, (unsigned)(cnt4 * 4), bb);
            }
            if (last) emitted_last = true;
            ++q;
        }
    } else if (w == 0) {
        // ================= consumer =================
        const double rho0 = ctl->anchor_norm;
        double* const p_beta = P.beta;
        float* const p_t = P.t;
        double D = D0, gstep = gstep0;
        long long n_unc = 0, n_nz = 0, n_req = 0;
        int gen = 0, k = 0;
        for (;;) {
            const int s = k % kSqSlots;
            {
                const unsigned b = bar_s + 8u * s, par = (unsigned)((k / kSqSlots) & 1);
                if (!mbar_test_s(b, par)) {
                    const unsigned long long t0 = gtimer();
                    while (!mbar_test_s(b, par)) spin_guard(t0, 22, k, gen, 0, 0);
                }
            }
            const SqDesc* dsc = &sc_->desc[s];
            const int cnt = dsc->cnt, last = dsc->last;
            const double dpw = dsc->dp;
            if (dsc->gen != gen) {
                __syncwarp();
                if (lane == 0) st_rel_s(cons_s, k + 1);
                ++k;
                continue;
            }
            const SqSlot* sl = &slots[s];
            int done_b = cnt;
            bool viol = false;
            for (int b = 0; b < cnt; ++b) {
                const int nnz = dsc->nnz[b], off = dsc->off[b];
                const double ns = dsc->ns[b], bj = dsc->bj[b], u = dsc->u[b];
                double x = 0.0, o = 0.0;
                int r = -1;
                if (lane < nnz) { x = sl->val[b][off + lane]; r = sl->idx[b][off + lane]; o = srho[r]; }
                const double g = warp_sum(fma(x, o, 0.0));
                const double z = bj + g / ns;
                const double nb = z > u ? z - u : (z < -u ? z + u : 0.0);
                const double d = nb - bj;
                ++n_unc;
                if (d != 0.0) {
                    if (r >= 0) srho[r] = __dsub_rn(o, __dmul_rn(d, x));
                    ++n_nz;
                    const double step = __dmul_ru(fabs(d), dsc->nr[b]);
                    if (use_t) D = delta_step(D, step, rho0);
                    gstep = 0.875 * gstep + 0.125 * step;
                    if (lane == 0) {
                        const int j = dsc->j[b], pos = dsc->pos[b];
                        p_beta[j] = nb;
                        if (use_t && bj == 0.0) {
                            p_t[pos] = -1.0f;                         // now in the support
                            if (m - lo <= kSqTile) ts[pos - lo] = -1.0f;   // resident tile (positions lo .. m)
                        }
                    }
                    __syncwarp();                                    // the scatter precedes the next member's gather
                    if (use_t && D > dpw) { done_b = b + 1; viol = true; break; }
                }
            }
            __syncwarp();
            if (lane == 0) {
                *(volatile double*)&sc_->d_pub = D;
                *(volatile double*)&sc_->g_pub = gstep;
            }
            if (viol) {
                n_unc -= 0;
                ++n_req;
                ++gen;
                if (lane == 0) {
                    *(volatile int*)&sc_->req_pos = dsc->pos[done_b - 1] + 1;
                    *(volatile double*)&sc_->req_d = D;
                    *(volatile double*)&sc_->req_g = gstep;
                    st_rel_s(reqg_s, gen);
                }
            }
            __syncwarp();
            if (lane == 0) st_rel_s(cons_s, k + 1);              // the slot (descriptor and data) is free
            if (!viol && last) break;
            ++k;
        }
        if (lane == 0) {
            st_rel_s(done_s, 1);
            ctl->cd_delta = D;
            ctl->cd_gstep = gstep;
            ctl->epoch_unc = n_unc;
            ctl->epoch_nz = n_nz;
            ctl->n_requeue += n_req;
            ctl->n_cand += n_unc;
            P.sc->visits += (unsigned long long)(m - lo);
            P.sc->uncertified += (unsigned long long)n_unc;
            P.sc->nonzero += (unsigned long long)n_nz;
        }
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < kSqSlots; ++s)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&sc_->bar[s])) : "memory");
    __shared__ double red[32];
    double s2 = 0.0;
    for (int r = tid; r < n; r += blockDim.x) { const double q = srho[r]; P.rho[r] = q; s2 = __dadd_ru(s2, __dmul_ru(q, q)); }
    s2 = block_sum_ru(s2, red);
    if (tid == 0) P.sc->rho_norm_ub = __dsqrt_ru(s2);
    __syncthreads();
}

}  // namespace gs
