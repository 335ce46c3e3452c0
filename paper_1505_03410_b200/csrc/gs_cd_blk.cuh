// Blocked-chain dense CD epoch (P.cd_gram == 2): the serial coordinate chain
// of cd_pass_dense (_kernels.py:39-64) advanced kBW coordinates at a time.
//
// The epoch walks the active positions in ascending order in WINDOWS of up to
// kBW = 7 "members": positions not certified zero under the window's drift
// bound Dp (t_i <= Dp; the support has t = -1).  Positions between members
// carry t > Dp and are skipped (certified zero updates, gs_solve.cuh header).
//
// Roles (warp-specialized, one CTA):
//   * NW <= 7 compute warps (rows of rho in registers, R per thread);
//   * ONE producer warp (warp NW): scans the staged thresholds for the next
//     window, writes the window descriptor and issues the TMA bulk copies
//     (cp.async.bulk, one mbarrier per column slot) of the member columns and
//     their ColInfo records.  It runs up to two windows ahead (two column
//     slots, three descriptor slots), so the scan, the descriptor stores and
//     the TMA issue are off the compute warps' critical path.
//
// Per window, every compute warp:
//   1. waits for the slot's mbarrier phase (window k is the (k/2)-th use of
//      slot k & 1; the producer refills a slot only after every compute warp
//      passed the window's barrier, so a warp is never more than one phase
//      behind and the parity test is unambiguous);
//   2. ALL dots of the window at once -- h_b = x_b^T rho and the Gram entries
//      G(b,c) = x_b^T x_c, c < b (28 values) -- FMA partials per thread, one
//      transposed butterfly per warp (lane l ends with dot l), warps combined
//      through shared memory in fixed order: ONE barrier per window, after
//      which warp 0 releases the column slot to the producer;
//   3. the coordinate chain in registers, every lane of every warp
//      redundantly (no broadcast of the d's is needed afterwards), branch-free:
//         g_b = h_b - sum_{c<b} d_c G(b,c)   (folded in as the d's appear)
//         z = fl(beta_b + g_b RN(1/nsq_b)); soft threshold; d_b
//      then the running drift bound D over the members (round-up adds);
//   4. the first member after which D > Dp ends the window there (the gap
//      after it may hold a position that lost its certificate): members up
//      to it commit, and the compute warps post a restart request (position,
//      drift) under a new generation; windows of the old generation still in
//      the pipe are consumed and discarded;
//   5. the committed members' axpys rho -= d_b x_b, in member order with the
//      reference's separate roundings, so the stored rho is exactly the one
//      sequential CD stores with these d's.
//
// Determinism.  Window membership must not depend on timing (the Gram form's
// roundings depend on the window partition, and paths must be bit-identical
// run to run, pkg/tests/test_path.py:124-131).  The bound of window q is
// therefore a function of the data only: Dp_q = max(Dp_{q-1}, D_{q-3} + mfac *
// gstep_{q-3}), with (D, gstep) as published at the END of window q - 3 (a
// ring of four entries; the producer may start window q only after window
// q - 2 passed its barrier, which orders that publication before the read),
// and a restart sets Dp from the request's own (D, gstep).  How many stale
// windows the producer emitted before it saw a request varies with timing,
// but those are discarded unread and only shift window numbers, not members.
//
// Safety of the Gram form for certified skips is the argument of
// cd_consume_gram (gs_solve.cuh): gamma_n carries +40u for the <= 8-term
// final summation and the drift increments double the rounding allowance.
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
    int32_t gen, pad;            // restart generation the window belongs to
    int32_t pos[kBW + 1];
    int32_t j[kBW + 1];
};

struct alignas(16) BlkCtl {
    unsigned long long bar[kBSlots];
    BlkDesc desc[kBInfo];
    ColInfo info[kBInfo][kBW];   // TMA destination
    double part[2][8][32];       // per-warp partial dots, double-buffered by window parity
    // compute warps -> producer
    double d_ring[4], g_ring[4]; // drift / step scale at the end of window k, slot k & 3
    double req_d, req_g;         // restart request: drift and step scale at the request
    int cons_cols;               // windows whose column slot has been released
    int req_gen, req_pos;        // restart request: generation (release-published last), first position
    int done;                    // epoch finished
};

__host__ __device__ inline size_t blk_col_bytes(int64_t ld, int es) { return (size_t)ld * es; }   // multiple of 16
__host__ __device__ inline size_t blk_smem_bytes(int64_t ld, int es) {
    return (size_t)kBTile * (sizeof(float) + sizeof(int32_t)) + sizeof(BlkCtl) +
           (size_t)kBSlots * kBW * blk_col_bytes(ld, es);
}

// wait until phase `use` (0-based count of issues into this slot) completed
static __device__ __forceinline__ void blk_wait(unsigned bar, int use, int where) {
    const unsigned par = (unsigned)(use & 1);
    if (!mbar_test_s(bar, par)) {
        const unsigned long long t0 = gtimer();
        while (!mbar_test_s(bar, par)) spin_guard(t0, where, use, 0, 0, 0);
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
    const double D0 = use_t ? ctl->cd_delta : 0.0;
    const double gstep0 = ctl->cd_gstep > 0.0 ? ctl->cd_gstep : 1e-2 * P.lam;
    if (tid == 0) {
        for (int s = 0; s < kBSlots; ++s) mbar_init(&bc->bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 4; ++i) { bc->d_ring[i] = D0; bc->g_ring[i] = gstep0; }
        bc->req_d = 0.0; bc->req_g = 0.0;
        bc->cons_cols = 0; bc->req_gen = 0; bc->req_pos = 0; bc->done = 0;
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
    const unsigned cons_s = smem_u32(&bc->cons_cols), reqg_s = smem_u32(&bc->req_gen), done_s = smem_u32(&bc->done);
    const double mfac = (double)P.blk_mfac;

    if (w == NW) {
        // ================= producer warp =================
        const T* __restrict__ X = (const T*)P.X;
        int cur = 0, tb = 0, tend = min(m, kBTile);
        int gen = 0, q = 0;
        bool emitted_last = false;
        double Dp = use_t ? __dadd_ru(D0, __dmul_ru(mfac, gstep0)) : 0.0;
        asm volatile("fence.proxy.async.global;" ::: "memory");   // cinfo / beta stores before TMA reads
        const unsigned long long pol_keep = l2_policy_evict_last();   // the chain's columns stay in L2 across GEMV passes
        // phase cycles (clock64) only in a -DGS_CD_PROFILE build: the counters cost registers,
        // and this function runs at the 255-register limit
#ifdef GS_CD_PROFILE
        const bool pprof = P.cd_prof != 0 && lane == 0;
        long long ppc[3] = {0, 0, 0};
        long long ptprev = pprof ? clock64() : 0;
        auto plap = [&](int i) { if (pprof) { const long long t = clock64(); ppc[i] += t - ptprev; ptprev = t; } };
#else
        auto plap = [](int) {};
#endif
        for (;;) {
            // a free column slot (window q - 2 released), a restart request, or the end
            bool stop = false;
            {
                const unsigned long long t0 = gtimer();
                for (;;) {
                    if (ld_acq_s(done_s)) { stop = true; break; }
                    const int rg = ld_acq_s(reqg_s);
                    if (rg != gen) {
                        gen = rg;
                        cur = *(volatile int*)&bc->req_pos;
                        if (cur < tb || cur > tend || (cur == tend && tend < m)) { tb = cur; tend = cur; }   // reload
                        Dp = use_t ? __dadd_ru(*(volatile double*)&bc->req_d, __dmul_ru(mfac, *(volatile double*)&bc->req_g))
                                   : 0.0;
                        emitted_last = false;
                    }
                    if (!emitted_last && ld_acq_s(cons_s) >= q - 1) break;
                    spin_guard(t0, 13, q, gen, cur, 0);
                }
            }
            if (stop) break;
            plap(0);
            // rolling bound with a fixed lag of three windows (see "Determinism" above)
            if (use_t && q >= 3)
                Dp = fmax(Dp, __dadd_ru(*(volatile double*)&bc->d_ring[(q - 3) & 3],
                                        __dmul_ru(mfac, *(volatile double*)&bc->g_ring[(q - 3) & 3])));
            // ---- scan the next window from `cur` under Dp
            const int slot = q & 1, islot = q % kBInfo;
            BlkDesc* dsc = &bc->desc[islot];
            int found = 0;
            while (found < kBW && cur < m) {
                if (cur >= tend) {
                    tb = cur;
                    tend = min(m, tb + kBTile);
                    for (int qq = tb + lane; qq < tend; qq += 32) { As[qq - tb] = P.A[qq]; ts[qq - tb] = use_t ? P.t[qq] : -1.0f; }
                    __syncwarp();
                }
                const int qp = cur + lane;
                const bool unc = qp < tend && !(Dp < (double)ts[qp - tb]);
                const unsigned mask = __ballot_sync(FULL, unc);
                const int avail = __popc(mask), take = min(avail, kBW - found);
                const int rank = __popc(mask & ((1u << lane) - 1u));
                if (unc && rank < take) { dsc->pos[found + rank] = qp; dsc->j[found + rank] = As[qp - tb]; }
                if (take < avail) {
                    const unsigned nxt = __ballot_sync(FULL, unc && rank == take);
                    cur += __ffs((int)nxt) - 1;                  // the first uncertified position not taken
                } else {
                    cur = min(cur + 32, tend);
                }
                found += take;
            }
            const int last = (cur >= m) ? 1 : 0;
            plap(1);
            if (lane == 0) { dsc->dp = Dp; dsc->cnt = found; dsc->last = last; dsc->gen = gen; }
            __syncwarp();
            const int mj = lane < found ? dsc->j[lane] : 0;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            const unsigned bb = bar_s + 8u * slot;
            if (lane == 0) {
                if (found) mbar_expect_tx_s(bb, (unsigned)found * (cbytes + (unsigned)sizeof(ColInfo)));
                else mbar_arrive_s(bb);   // empty window: the phase completes at once
            }
            __syncwarp();
            if (lane < found) {
                tma_bulk_g2s_hint(cols_s + (unsigned)slot * slot_bytes + (unsigned)lane * cbytes, X + (int64_t)mj * P.ld,
                                  cbytes, bb, pol_keep, P.l2_hint);
                tma_bulk_g2s_s(smem_u32(&bc->info[islot][lane]), P.cinfo + mj, (unsigned)sizeof(ColInfo), bb);
            }
            if (last) emitted_last = true;
            ++q;
            plap(2);
        }
#ifdef GS_CD_PROFILE
        if (pprof) { ctl->c_w1[5] += (unsigned long long)ppc[0]; ctl->c_pr[0] += (unsigned long long)ppc[1]; ctl->c_pr[1] += (unsigned long long)ppc[2]; }
#endif
    } else if (w < NW) {
        // ================= compute warps =================
        const double rho0 = ctl->anchor_norm;
        // P lives in global memory: the pointers the commit needs, read once
        double* const p_beta = P.beta;
        ColInfo* const p_cinfo = P.cinfo;
        float* const p_t = P.t;
        double D = D0;
        double gstep = gstep0;
        double rr[R];
#pragma unroll
        for (int q = 0; q < R; ++q) { const int r = tid + q * BT; rr[q] = r < n ? P.rho[r] : 0.0; }
        int n_unc = 0, n_nz = 0, n_req = 0, gen = 0;
        int k = 0;
        // phase cycles of warp 0 and of a second compute warp, GS_CD_PROF=1
#ifdef GS_CD_PROFILE
        const bool prof = P.cd_prof != 0 && lane == 0 && (w == 0 || w == 1);
        long long pc[5] = {0, 0, 0, 0, 0};
        long long tprev = prof ? clock64() : 0;
        auto lap = [&](int i) { if (prof) { const long long t = clock64(); pc[i] += t - tprev; tprev = t; } };
#else
        auto lap = [](int) {};
#endif
        for (;;) {
            const int s = k & 1, i3 = k % kBInfo;
            blk_wait(bar_s + 8u * s, k >> 1, 11);
            const BlkDesc* dsc = &bc->desc[i3];
            const int cnt = dsc->cnt, last = dsc->last;
            const double dpw = dsc->dp;
            lap(0);
            if (dsc->gen != gen) {
                // a window of an older generation (selected before a restart): discard
                if (NW > 1) named_bar(1, BT);
                if (tid == 0) {
                    *(volatile double*)&bc->d_ring[k & 3] = D;
                    *(volatile double*)&bc->g_ring[k & 3] = gstep;
                    st_rel_s(cons_s, k + 1);
                }
                ++k;
                continue;
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
            lap(1);
            if (NW > 1) named_bar(1, BT);
            else __syncwarp();
            // every compute warp has read the window's columns: the slot may be refilled
            if (tid == 0) st_rel_s(cons_s, k + 1);
            lap(2);
            // every warp: the window's dots (lane l: dot l), warps summed in a fixed tree
            double tot;
            {
                double pw[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pw[q] = q < NW ? part[q * 32 + lane] : 0.0;
                tot = ((pw[0] + pw[1]) + (pw[2] + pw[3])) + ((pw[4] + pw[5]) + (pw[6] + pw[7]));
            }
            // ---- the chain (every lane, redundantly; branch-free)
            double acc[kBW], dv[kBW], nbv[kBW], inc[kBW];
            double Gs[kBW * (kBW - 1) / 2];
#pragma unroll
            for (int b = 0; b < kBW; ++b) acc[b] = __shfl_sync(FULL, tot, b);
#pragma unroll
            for (int i = 0; i < kBW * (kBW - 1) / 2; ++i) Gs[i] = __shfl_sync(FULL, tot, kBW + i);
            const ColInfo* inf = &bc->info[i3][0];
            // the members' constants first (one round of shared-memory loads), then the pure chain
            double c_iv[kBW], c_u[kBW], c_bj[kBW];
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                c_iv[b] = inf[b].inv;
                c_u[b] = inf[b].u;
                c_bj[b] = inf[b].beta;
            }
            // z = fl(beta + g * RN(1/nsq)): one FMA on the serial path instead of the
            // correctly rounded quotient (three dependent operations).  The Gram form of g
            // already differs from the stored-residual dot by a few ulps, so the quotient's
            // last bit is not what parity rests on; the certified skips stay exact because
            // cert_threshold certifies against lam (1 - 1e-15) (gs_kernels.cuh).
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                const double z = fma(acc[b], c_iv[b], c_bj[b]);
                const double uq = c_u[b];
                const double zp = z - uq, zm = z + uq;
                const double nb = z > uq ? zp : (z < -uq ? zm : 0.0);
                const double d = (b < cnt) ? nb - c_bj[b] : 0.0;
#pragma unroll
                for (int c = b + 1; c < kBW; ++c) acc[c] = fma(-d, Gs[c * (c - 1) / 2 + b], acc[c]);
                dv[b] = d;
                nbv[b] = nb;
            }
            // drift increment of a nonzero member: step (1 + 1e-12) + 4.6e-16 (rho0 + D + step), with
            // D <= dpw for every member that commits (round-up arithmetic throughout)
            const double kD = use_t ? __dmul_ru(4.6e-16, __dadd_ru(rho0, dpw)) : 0.0;
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                const double step = __dmul_ru(fabs(dv[b]), inf[b].nr);
                inc[b] = dv[b] != 0.0 ? __dadd_ru(__dmul_ru(step, 1.0 + 1.0001e-12), kD) : 0.0;
            }
            lap(3);
            // ---- drift after each member; the window ends at the first member after which D > Dp
            double Dv[kBW];
            {
                double Dl = D;
#pragma unroll
                for (int b = 0; b < kBW; ++b) { Dl = __dadd_ru(Dl, inc[b]); Dv[b] = Dl; }
            }
            int ncommit = cnt;
            bool viol = false;
            if (use_t) {
#pragma unroll
                for (int b = kBW - 1; b >= 0; --b)
                    if (b < cnt && Dv[b] > dpw) { ncommit = b + 1; viol = true; }
            }
            // ---- commit: axpys in member order (separate roundings), bookkeeping
            double ssum = 0.0, dmine = 0.0, nbmine = 0.0;
            int nzc = 0;
#pragma unroll
            for (int b = 0; b < kBW; ++b) {
                const double d = dv[b];
                if (b < ncommit && d != 0.0) {
#pragma unroll
                    for (int q = 0; q < R; ++q) rr[q] = __dsub_rn(rr[q], __dmul_rn(d, xw[b][q]));
                    ssum += inc[b];
                    ++nzc;
                }
                if (b < ncommit && use_t) D = Dv[b];
                if (lane == b) { dmine = d; nbmine = nbv[b]; }
            }
            if (nzc) gstep = 0.5 * gstep + 0.5 * (ssum / (double)nzc);
            if (w == 0 && lane < ncommit && dmine != 0.0) {
                // lane b commits member b (values of its own chain copy)
                const int j = dsc->j[lane], pos = dsc->pos[lane];
                p_beta[j] = nbmine;
                p_cinfo[j].beta = nbmine;
                if (use_t && inf[lane].beta == 0.0) {
                    p_t[pos] = -1.0f;                                  // now in the support
                    if (m <= kBTile) ts[pos] = -1.0f;                  // resident tile (positions 0 .. m)
                }
            }
            n_unc += ncommit;
            n_nz += nzc;
            if (tid == 0) { *(volatile double*)&bc->d_ring[k & 3] = D; *(volatile double*)&bc->g_ring[k & 3] = gstep; }
            lap(4);
            if (viol) {
                // the drift outgrew the bound: restart after the last committed member
                ++n_req;
                ++gen;
                if (tid == 0) {
                    *(volatile int*)&bc->req_pos = dsc->pos[ncommit - 1] + 1;
                    *(volatile double*)&bc->req_d = D;
                    *(volatile double*)&bc->req_g = gstep;
                    st_rel_s(reqg_s, gen);
                }
            } else if (last) {
                break;
            }
            ++k;
        }
        if (tid == 0) st_rel_s(done_s, 1);
#ifdef GS_CD_PROFILE
        if (prof) {
            if (w == 0) {
                ctl->c_wait += pc[0]; ctl->c_red += pc[1]; ctl->c_upd += pc[2]; ctl->c_chain += pc[3]; ctl->c_form += pc[4];
            } else {
                for (int i = 0; i < 5; ++i) ctl->c_w1[i] += (unsigned long long)pc[i];
            }
        }
#endif
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
        if (w == 0) asm volatile("fence.proxy.async.global;" ::: "memory");   // cinfo stores before the next epoch's TMA reads
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
