// Blocked-chain dense CD epoch (P.cd_gram == 2): the serial coordinate chain
// of cd_pass_dense (_kernels.py:39-64) advanced kBW coordinates at a time.
//
// The epoch walks the active positions in ascending order in WINDOWS of up to
// kBW = 7 "members": positions not certified zero under the window's drift
// bound Dp (t_i <= Dp; the support has t = -1).  Positions between members
// carry t > Dp and are skipped (certified zero updates, gs_solve.cuh header).
//
// Per window (every compute warp; rows of rho in registers, R per thread):
//   1. the member columns and ColInfo records arrive in a shared-memory slot
//      by TMA (cp.async.bulk, one mbarrier per slot), issued one window
//      AHEAD by warp 0 (the scan of the next window runs under the same Dp,
//      so it is valid as long as the drift stays <= Dp);
//   2. ALL dots of the window at once -- h_b = x_b^T rho and the Gram entries
//      G(b,c) = x_b^T x_c, c < b (28 values) -- FMA partials per thread, one
//      transposed butterfly per warp (lane l ends with dot l), warps combined
//      through shared memory in fixed order: ONE barrier per window;
//   3. the coordinate chain in registers, every lane of every warp
//      redundantly (no broadcast of the d's is needed afterwards):
//         g_b = h_b - sum_{c<b} d_c G(b,c)   (folded in as the d's appear)
//         z = beta_b + RN(g_b/nsq_b); soft threshold; d_b
//      and the running drift bound D (round-up, doubled rounding allowance:
//      delta_step_g);
//   4. the first member after which D > Dp ends the window there (the gap
//      after it may hold a position that lost its certificate): members up
//      to it commit, warp 0 re-scans from the next position under
//      Dp = D + margin and re-issues the (now stale) next window;
//   5. the committed members' axpys rho -= d_b x_b, in member order with the
//      reference's separate roundings, so the stored rho is exactly the one
//      sequential CD stores with these d's.
// Window boundaries depend only on the data (thresholds, D), never on timing:
// paths are bit-identical run to run (pkg/tests/test_path.py:124-131).
//
// Safety of the Gram form for certified skips is the argument of
// cd_consume_gram (gs_solve.cuh): gamma_n carries +40u for the <= 8-term
// final summation and delta_step_g doubles the rounding allowance.
#pragma once

namespace gs {

constexpr int kBW = 7;                                 // members per window
constexpr int kBDots = kBW + kBW * (kBW - 1) / 2;      // h_b and G(b,c), c < b: 28 <= 32 lanes
constexpr int kBSlots = 2;                             // column slots (window k in slot k & 1)
constexpr int kBInfo = 3;                              // descriptor / ColInfo slots (window k in k % 3)
constexpr int kBTile = 8192;                           // thresholds + positions staged per tile

struct alignas(16) BlkDesc {
    double dp;                   // drift bound the members were selected under
    int32_t cnt, last;           // members; the scan reached the end of the active set
    int32_t pos[kBW];
    int32_t j[kBW];
};

struct alignas(16) BlkCtl {
    unsigned long long bar[kBSlots];
    BlkDesc desc[kBInfo];
    ColInfo info[kBInfo][kBW];   // TMA destination
    double part[2][8][32];       // per-warp partial dots, double-buffered by window parity
};

__host__ __device__ inline size_t blk_col_bytes(int64_t ld, int es) { return (size_t)ld * es; }   // multiple of 16
__host__ __device__ inline size_t blk_smem_bytes(int64_t ld, int es) {
    return (size_t)kBTile * (sizeof(float) + sizeof(int32_t)) + sizeof(BlkCtl) +
           (size_t)kBSlots * kBW * blk_col_bytes(ld, es);
}

// wait until phase `use` (0-based count of issues into this slot) completed;
// phases complete in order, so waiting for each in turn is unambiguous
static __device__ __forceinline__ void blk_wait(unsigned bar, int& waited, int use, int where) {
    for (; waited <= use; ++waited) {
        const unsigned par = (unsigned)(waited & 1);
        if (!mbar_test_s(bar, par)) {
            const unsigned long long t0 = gtimer();
            while (!mbar_test_s(bar, par)) spin_guard(t0, where, waited, use, 0, 0);
        }
    }
}

template <typename T, int R>
static __device__ __noinline__ void cd_epoch_blk(const SolveDev& P, int64_t m64, int NW, unsigned char* smem,
                                                 int* tile_valid) {
    SolveCtl* ctl = P.ctl;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int BT = NW * 32;
    const int m = (int)m64;
    const int n = P.n;
    const unsigned FULL = 0xffffffffu;
    float* ts = reinterpret_cast<float*>(smem);
    int32_t* As = reinterpret_cast<int32_t*>(smem + kBTile * sizeof(float));
    BlkCtl* bc = reinterpret_cast<BlkCtl*>(smem + kBTile * (sizeof(float) + sizeof(int32_t)));
    unsigned char* cols = reinterpret_cast<unsigned char*>(bc + 1);
    const unsigned cbytes = (unsigned)blk_col_bytes(P.ld, (int)sizeof(T));
    const unsigned slot_bytes = cbytes * kBW;
    const bool use_t = P.certify != 0;
    if (m == 0) {
        if (tid == 0) { ctl->epoch_unc = 0; ctl->epoch_nz = 0; }
        __syncthreads();
        return;
    }
    if (tid == 0) {
        for (int s = 0; s < kBSlots; ++s) mbar_init(&bc->bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const bool keep_tile = (m <= kBTile) && *tile_valid;
    if (!keep_tile) {
        const int lim = min(m, kBTile);
        for (int q = tid; q < lim; q += blockDim.x) {
            As[q] = P.A[q];
            ts[q] = use_t ? P.t[q] : -1.0f;
        }
    }
    __syncthreads();
    const unsigned bar_s = smem_u32(&bc->bar[0]);
    const unsigned cols_s = smem_u32(cols);

    if (w < NW) {
        const double rho0 = ctl->anchor_norm;
        double D = use_t ? ctl->cd_delta : 0.0;
        double gstep = ctl->cd_gstep > 0.0 ? ctl->cd_gstep : 1e-2 * P.lam;
        const double mfac = (double)P.blk_mfac;
        double rr[R];
#pragma unroll
        for (int q = 0; q < R; ++q) { const int r = tid + q * BT; rr[q] = r < n ? P.rho[r] : 0.0; }
        int n_unc = 0, n_nz = 0, n_req = 0;
        int uses[kBSlots] = {0, 0}, waited[kBSlots] = {0, 0};

        // ---- producer state (warp 0): scan cursor, bound, threshold tile
        int cur = 0, tb = 0, tend = min(m, kBTile);
        double Dp = use_t ? __dadd_ru(D, __dmul_ru(mfac, gstep)) : 0.0;
        const T* __restrict__ X = (const T*)P.X;
        // scan the next window from `cur` under Dp and issue it into (slot, info slot)
        auto produce = [&](int slot, int islot) {
            int found = 0, mpos = 0, mj = 0;
            while (found < kBW && cur < m) {
                if (cur >= tend) {
                    tb = cur;
                    tend = min(m, tb + kBTile);
                    for (int q = tb + lane; q < tend; q += 32) { As[q - tb] = P.A[q]; ts[q - tb] = use_t ? P.t[q] : -1.0f; }
                    __syncwarp();
                }
                const int q = cur + lane;
                const bool unc = q < tend && !(Dp < (double)ts[q - tb]);
                const unsigned mask = __ballot_sync(FULL, unc);
                const int avail = __popc(mask), take = min(avail, kBW - found);
                const int src = (lane >= found && lane < found + take) ? (int)__fns(mask, 0, lane - found + 1) : lane;
                const int qs = __shfl_sync(FULL, q, src);
                const int js = __shfl_sync(FULL, unc ? As[q - tb] : 0, src);
                if (lane >= found && lane < found + take) { mpos = qs; mj = js; }
                if (take < avail) cur = __shfl_sync(FULL, q, (int)__fns(mask, 0, take)) + 1;
                else cur = min(cur + 32, tend);
                found += take;
            }
            const int last = (cur >= m) ? 1 : 0;
            BlkDesc* dsc = &bc->desc[islot];
            if (lane < found) { dsc->pos[lane] = mpos; dsc->j[lane] = mj; }
            if (lane == 0) { dsc->dp = Dp; dsc->cnt = found; dsc->last = last; }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            const unsigned bb = bar_s + 8u * slot;
            if (lane == 0) {
                if (found) mbar_expect_tx_s(bb, (unsigned)found * (cbytes + (unsigned)sizeof(ColInfo)));
                else mbar_arrive_s(bb);   // empty window: the phase completes at once
            }
            __syncwarp();
            if (lane < found) {
                tma_bulk_g2s_s(cols_s + (unsigned)slot * slot_bytes + (unsigned)lane * cbytes, X + (int64_t)mj * P.ld,
                               cbytes, bb);
                tma_bulk_g2s_s(smem_u32(&bc->info[islot][lane]), P.cinfo + mj, (unsigned)sizeof(ColInfo), bb);
            }
        };

        if (w == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");   // cinfo / beta stores before TMA reads
            produce(0, 0);
        }
        uses[0] = 1;
        int k = 0;
        for (;;) {
            const int s = k & 1, i3 = k % kBInfo;
            blk_wait(bar_s + 8u * s, waited[s], uses[s] - 1, 11);
            const BlkDesc* dsc = &bc->desc[i3];
            const int cnt = dsc->cnt, last = dsc->last;
            const double dpw = dsc->dp;
            // speculative next window (same bound): its column slot was last read
            // before the previous window's barrier, its info slot two windows ago
            if (!last) {
                if (w == 0) {
                    // rolling bound: the window two ahead of the last finished one is
                    // selected under the current drift plus the allowance (never lowered,
                    // so earlier gaps stay covered by their own window's bound)
                    if (use_t) Dp = fmax(Dp, __dadd_ru(D, __dmul_ru(mfac, gstep)));
                    produce(s ^ 1, (k + 1) % kBInfo);
                }
                uses[s ^ 1]++;
            }
            // ---- dots of the window: h_b and G(b,c), c < b
            double xw[kBW][R];
            const T* xs0 = reinterpret_cast<const T*>(cols + (size_t)s * slot_bytes) + tid;
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                const T* xs = reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(xs0) + (size_t)b * cbytes);
#pragma unroll
                for (int q = 0; q < R; ++q) xw[b][q] = (b < cnt && tid + q * BT < n) ? to_d(xs[q * BT]) : 0.0;
            }
            double* part = &bc->part[k & 1][0][0];
            {
                double v[32];
#pragma unroll
                for (int b = 0; b < kBW; ++b) {
                    double a0 = 0.0, a1 = 0.0;
#pragma unroll
                    for (int q = 0; q < R; q += 2) {
                        a0 = fma(xw[b][q], rr[q], a0);
                        if (q + 1 < R) a1 = fma(xw[b][q + 1], rr[q + 1], a1);
                    }
                    v[b] = a0 + a1;
#pragma unroll
                    for (int c = 0; c < b; ++c) {
                        double g0 = 0.0, g1 = 0.0;
#pragma unroll
                        for (int q = 0; q < R; q += 2) {
                            g0 = fma(xw[b][q], xw[c][q], g0);
                            if (q + 1 < R) g1 = fma(xw[b][q + 1], xw[c][q + 1], g1);
                        }
                        v[kBW + b * (b - 1) / 2 + c] = g0 + g1;
                    }
                }
#pragma unroll
                for (int i = kBDots; i < 32; ++i) v[i] = 0.0;
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
                part[w * 32 + lane] = v[0];
            }
            if (NW > 1) named_bar(1, BT);
            else __syncwarp();
            // every warp: the window's dots (lane l: dot l), warps summed in a fixed tree
            double tot;
            {
                double pw[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pw[q] = q < NW ? part[q * 32 + lane] : 0.0;
                tot = ((pw[0] + pw[1]) + (pw[2] + pw[3])) + ((pw[4] + pw[5]) + (pw[6] + pw[7]));
            }
            // ---- the chain (every lane, redundantly)
            double acc[kBW], dv[kBW], nbv[kBW], Dv[kBW];
#pragma unroll
            for (int b = 0; b < kBW; ++b) acc[b] = __shfl_sync(FULL, tot, b);
            const ColInfo* inf = &bc->info[i3][0];
            double Dl = D, gsl = gstep;
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                const double2 nsiv = *reinterpret_cast<const double2*>(&inf[b].ns);     // ns, inv
                const double2 nru = *reinterpret_cast<const double2*>(&inf[b].nr);      // nr, u
                const double bj = inf[b].beta;
                const double g = acc[b];
                const double q0 = g * nsiv.y;
                const double rq = fma(-q0, nsiv.x, g);
                const double qq = fma(rq, nsiv.y, q0);              // RN(g / nsq)
                const double z = bj + qq;
                const double uq = nru.y;
                const double nb = z > uq ? z - uq : (z < -uq ? z + uq : 0.0);
                const double d = (b < cnt) ? nb - bj : 0.0;
#pragma unroll
                for (int c = b + 1; c < kBW; ++c)
                    acc[c] = fma(-d, __shfl_sync(FULL, tot, kBW + c * (c - 1) / 2 + b), acc[c]);
                if (d != 0.0 && use_t) {
                    const double step = __dmul_ru(fabs(d), nru.x);
                    Dl = delta_step_g(Dl, step, rho0);
                    gsl = 0.875 * gsl + 0.125 * step;
                }
                dv[b] = d;
                nbv[b] = nb;
                Dv[b] = Dl;
            }
            // ---- end of the window: the first member after which D > Dp
            int ncommit = cnt;
            bool viol = false;
            if (use_t) {
#pragma unroll
                for (int b = kBW - 1; b >= 0; --b)
                    if (b < cnt && Dv[b] > dpw) { ncommit = b + 1; viol = true; }
            }
            // ---- commit: axpys in member order (separate roundings), bookkeeping
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                const double d = dv[b];
                if (b < ncommit && d != 0.0) {
#pragma unroll
                    for (int q = 0; q < R; ++q) rr[q] = __dsub_rn(rr[q], __dmul_rn(d, xw[b][q]));
                }
            }
            double Dn = D, gn = gstep;
            int nzc = 0;
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                if (b < ncommit) {
                    Dn = Dv[b];
                    if (dv[b] != 0.0) ++nzc;
                }
            }
            // gstep: recompute the EMA over the committed members only
            if (use_t && ncommit < cnt) {
                gn = gstep;
#pragma unroll
                for (int b = 0; b < kBW; ++b)
                    if (b < ncommit && dv[b] != 0.0) gn = 0.875 * gn + 0.125 * __dmul_ru(fabs(dv[b]), inf[b].nr);
            } else {
                gn = gsl;
            }
            if (w == 0 && lane < ncommit && dv[lane] != 0.0) {
                // lane b commits member b (values of its own chain copy)
                double dmine = 0.0, nbmine = 0.0;
#pragma unroll
                for (int b = 0; b < kBW; ++b) if (lane == b) { dmine = dv[b]; nbmine = nbv[b]; }
                const int j = dsc->j[lane], pos = dsc->pos[lane];
                P.beta[j] = nbmine;
                P.cinfo[j].beta = nbmine;
                if (use_t && inf[lane].beta == 0.0) {
                    P.t[pos] = -1.0f;                                  // now in the support
                    if (pos >= tb && pos < tend) ts[pos - tb] = -1.0f;
                }
                (void)dmine;
            }
            n_unc += ncommit;
            n_nz += nzc;
            D = Dn;
            gstep = gn;
            if (viol) {
                // the drift outgrew the bound: restart after the last committed member
                ++n_req;
                const int rpos = dsc->pos[ncommit - 1] + 1;
                if (!last) {
                    // the speculative window is stale: every warp observes its phase
                    // (mbarrier parity waits are only unambiguous one phase behind), and
                    // only then may warp 0 issue the next phase into that slot
                    blk_wait(bar_s + 8u * (s ^ 1), waited[s ^ 1], uses[s ^ 1] - 1, 12);
                    if (NW > 1) named_bar(1, BT);
                }
                if (w == 0) {
                    cur = rpos;
                    if (cur < tb || cur > tend || (cur == tend && tend < m)) {
                        tb = cur; tend = cur;       // forces a reload at the next scan step
                    }
                    Dp = fmax(Dp, __dadd_ru(D, __dmul_ru(mfac, gstep)));
                    produce(s ^ 1, (k + 1) % kBInfo);
                }
                uses[s ^ 1]++;
            } else if (last) {
                break;
            }
            ++k;
        }
        // ---- epilogue: rho back, ||rho|| upper bound for the next anchor
        if (NW > 1) named_bar(1, BT);
        double s2 = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int r = tid + q * BT;
            if (r < n) { P.rho[r] = rr[q]; s2 = __dadd_ru(s2, __dmul_ru(rr[q], rr[q])); }
        }
        s2 = warp_sum_ru(s2);
        double* red = &bc->part[0][0][0];
        if (lane == 0) red[w] = s2;
        if (NW > 1) named_bar(1, BT);
        else __syncwarp();
        if (tid == 0) {
            double tot = 0.0;
            for (int q = 0; q < NW; ++q) tot = __dadd_ru(tot, red[q]);
            P.sc->rho_norm_ub = __dsqrt_ru(tot);
            ctl->cd_delta = D;
            ctl->cd_gstep = gstep;
            ctl->epoch_unc = n_unc;
            ctl->epoch_nz = n_nz;
            ctl->n_requeue += n_req;
            ctl->n_cand += n_unc;
            if (P.cd_prof) { ctl->n_win += (unsigned long long)(k + 1); ctl->n_mem += (unsigned long long)n_unc; }
            P.sc->visits += (unsigned long long)m;
            P.sc->uncertified += (unsigned long long)n_unc;
            P.sc->nonzero += (unsigned long long)n_nz;
        }
    }
    __syncthreads();
    if (tid == 0) {
        *tile_valid = (m <= kBTile) ? 1 : 0;
        for (int s = 0; s < kBSlots; ++s)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bc->bar[s])) : "memory");
    }
    __syncthreads();
}

}  // namespace gs
