// hsgn_multi.cuh -- member-resident multi-step cluster kernel of the SI-IMEX
// hSGN step: the C CTAs of a member (one thread-block cluster, as in
// hsgn_cluster.cuh) load its state once, advance it by K full SI-IMEX steps
// (both stages of P:500-517, the dt rule of P:607-617 with t_end
// clipping) with the state, the stage inputs and every intermediate held in
// shared memory, and store it once.  Per step nothing touches HBM: the tiles
// exchange their edge rows (E2/R2 of stage 2, the filter rows, U^{n+1}), the
// separator data of the exact depth solve and the dt maxima through DSMEM
// (st.async into the receivers' shared memory, completion on their mbarriers).
// Citations: P:n = PAPER.md line n, Ak = DESIGN.md reading k.
//
// Same arithmetic as cl_stage_kernel (phases 1-3, the exact cluster solve),
// with two differences of rounding only: E2 and R2 are formed in
// the H-form (H = K - 3hb/2 is affine in (h, K) at fixed b) and the initial
// dt maxima use the kernel's reciprocal / square root.
#pragma once
#include "hsgn_cluster.cuh"

#ifndef HSGN_MMINB
#define HSGN_MMINB 4                                  // resident CTAs per SM (registers / shared memory)
#endif

namespace hsgn {

// HSGN_EXP_TIMING builds: per-step phase clocks of CTA 0 of member 0 into
// g_clt (row st = stage; tools/res_timing.py)
#if HSGN_EXP_TIMING
#define ML_MARK(st, k) do { if (prof) { const long long t_ = clock64(); g_clt[st][k] += (unsigned long long)(t_ - tml); tml = t_; } } while (0)
#else
#define ML_MARK(st, k) do { } while (0)
#endif

__shared__ double s_dx[C_MAX][4];                     // dt maxima (u, nu), error flag of every CTA
__shared__ __align__(8) unsigned long long s_emb, s_umb, s_dmb;

template <bool BATHY>
__global__ void __launch_bounds__(CNT, HSGN_MMINB) cl_multi_kernel(const Params P, const Bufs B, const int K,
                                                                   const int k0)
{
    double *const sm = hsgn_smem;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int C = P.tiles;
    const int c = blockIdx.x;
    const int m = blockIdx.y;
    const int n = P.n;
    const size_t mo = size_t(m) * n;
    const int s = c * P.T;
    const int Tc = (c == C - 1) ? n - s : P.T;
    const bool cyc = P.bcl == BC_PERIODIC;
    const bool left_phys = !cyc && c == 0, right_phys = !cyc && c == C - 1;
    const bool wall_l = P.bcl == BC_WALL, wall_r = P.bcr == BC_WALL;
    const int cl_ = (c > 0) ? c - 1 : C - 1, cr_ = (c + 1 < C) ? c + 1 : 0;
    const int Tl = (cl_ == C - 1) ? n - (C - 1) * P.T : P.T;        // left neighbour's rows
    const unsigned xmb = (unsigned)__cvta_generic_to_shared(&s_xmb);
    const unsigned fmb = (unsigned)__cvta_generic_to_shared(&s_fmb);
    const unsigned emb = (unsigned)__cvta_generic_to_shared(&s_emb);
    const unsigned umb = (unsigned)__cvta_generic_to_shared(&s_umb);
    const unsigned dmb = (unsigned)__cvta_generic_to_shared(&s_dmb);
    double *const A0 = sm, *const A1 = sm + CARR, *const A2 = sm + 2 * CARR, *const A3 = sm + 3 * CARR;
    double *const A4 = sm + 4 * CARR, *const A5 = sm + 5 * CARR, *const A6 = sm + 6 * CARR;
    double *const A7 = sm + 7 * CARR, *const A8 = sm + 8 * CARR;
    double *const sU[4] = {A0, A1, A2, A3};            // state U (h, q, H, W), later E2
    double *const sQd = A4, *const sHd = A5, *const sBe = A6, *const sDe = A7;
    const double *const sB = BATHY ? A8 : nullptr;
    const int ks = Tc / CMCH - 1;
    const int r0 = tid * CMCH;
    const bool live = r0 < Tc;
    const bool filt = P.filter_sigma > 0.0;
    const bool relax = P.gen_rate > 0.0 || P.sp_rate > 0.0;
    const int nside = (left_phys ? 0 : 1) + (right_phys ? 0 : 1);
    const double lam = P.lam[m], lam3 = lam * (1.0 / 3.0), g = P.g;
    double t = P.t[(k0 & 1) * P.members + m];
    const double t_end = P.ctrl->t_end;

#if HSGN_EXP_TIMING
    const bool prof = m == 0 && c == 0 && tid == 0;
    long long tml = clock64();
#endif
    auto arm = [&](unsigned mb, unsigned bytes) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
    };
    const unsigned XB = unsigned(XPUB * C) * 8u, EB = 160u * nside, FB = 32u * nside, UB = 128u * nside,
                   DB = 24u * unsigned(C);
    if (tid == 0) {
        for (unsigned mb : {xmb, fmb, emb, umb, dmb})
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        arm(xmb, XB); arm(fmb, filt ? FB : 0u); arm(emb, EB); arm(umb, UB); arm(dmb, DB);
    }
    unsigned px = 0u, pf = 0u, pe = 0u, pu = 0u, pd = 0u;   // phase parities

    // ---- load U^n once (H-form), halo rows of the neighbours / mirrors ---------
    {
        auto putU = [&](int r, double h, double q, double H, double W, double b) {
            const int x = swz(r);
            A0[x] = h; A1[x] = q; A2[x] = H; A3[x] = W;
            if (BATHY) A8[x] = b;
        };
        auto ld2 = [&](size_t gc, double (&e)[4][2], double (&bb)[2]) {
#pragma unroll
            for (int f = 0; f < 4; f++) {
                const double2 u = __ldg(reinterpret_cast<const double2 *>(B.Un[f] + gc));
                e[f][0] = u.x; e[f][1] = u.y;
            }
            if (BATHY) {
                const double2 b2 = __ldg(reinterpret_cast<const double2 *>(P.b + (gc - mo)));
                bb[0] = b2.x; bb[1] = b2.y;
                for (int k = 0; k < 2; k++) e[2][k] -= 1.5 * e[0][k] * bb[k];      // H = K - 1.5 h b (A9)
            } else {
                bb[0] = bb[1] = 0.0;
            }
        };
        if (live) {
            double e0[4][2], e1[4][2], b0[2], b1[2];
            ld2(mo + size_t(s + r0), e0, b0);
            ld2(mo + size_t(s + r0 + 2), e1, b1);
            putU(r0, e0[0][0], e0[1][0], e0[2][0], e0[3][0], b0[0]);
            putU(r0 + 1, e0[0][1], e0[1][1], e0[2][1], e0[3][1], b0[1]);
            putU(r0 + 2, e1[0][0], e1[1][0], e1[2][0], e1[3][0], b1[0]);
            putU(r0 + 3, e1[0][1], e1[1][1], e1[2][1], e1[3][1], b1[1]);
        }
        const int hs = (tid == 64 || tid == 65) ? 0 : (tid == 96 || tid == 97) ? 1 : -1;
        if (hs == 0 && !left_phys) {
            const int rr0 = (tid == 64) ? -4 : -2;
            const int gc = (s + rr0 >= 0) ? s + rr0 : n + s + rr0;
            double e[4][2], bb[2];
            ld2(mo + size_t(gc), e, bb);
            putU(rr0, e[0][0], e[1][0], e[2][0], e[3][0], bb[0]);
            putU(rr0 + 1, e[0][1], e[1][1], e[2][1], e[3][1], bb[1]);
        }
        if (hs == 1 && !right_phys) {
            const int rr0 = (tid == 96) ? Tc : Tc + 2;
            const int gc = (s + rr0 < n) ? s + rr0 : s + rr0 - n;
            double e[4][2], bb[2];
            ld2(mo + size_t(gc), e, bb);
            putU(rr0, e[0][0], e[1][0], e[2][0], e[3][0], bb[0]);
            putU(rr0 + 1, e[0][1], e[1][1], e[2][1], e[3][1], bb[1]);
        }
    }
    __syncthreads();
    // mirrored halo rows at physical ends (A10): U and b (b is static)
    auto mirror_halo = [&](double *const *arr, bool withb) {
        if (tid == 0 && left_phys) {
            for (int k = 0; k < 4; k++) {
                const int src = swz(wall_l ? k : 0), dst = swz(-1 - k);
                arr[0][dst] = arr[0][src]; arr[1][dst] = (wall_l ? -1.0 : 1.0) * arr[1][src];
                arr[2][dst] = arr[2][src]; arr[3][dst] = arr[3][src];
                if (BATHY && withb) A8[dst] = A8[src];
            }
        }
        if (tid == ks && right_phys) {
            for (int k = 0; k < 4; k++) {
                const int src = swz(wall_r ? Tc - 1 - k : Tc - 1), dst = swz(Tc + k);
                arr[0][dst] = arr[0][src]; arr[1][dst] = (wall_r ? -1.0 : 1.0) * arr[1][src];
                arr[2][dst] = arr[2][src]; arr[3][dst] = arr[3][src];
                if (BATHY && withb) A8[dst] = A8[src];
            }
        }
    };
    mirror_halo(sU, true);
    __syncthreads();
    cl_arrive_relaxed();
    cl_wait();                                        // every CTA started, mbarriers initialised

    TileAcc acc{0.0, 0.0, 0.0, 0u, 1 << 30, 0};
    // dt maxima of the own rows of U (h, q, H, W in arrays 0..3): max|u|, max(|u| + c) (A7)
    auto local_maxima = [&](double &um, double &nm) {
        um = 0.0; nm = 0.0;
        if (live) {
#pragma unroll
            for (int i = 0; i < CMCH; i++) {
                const int x = swz(r0 + i);
                const double h = A0[x], ih = rcp(h);
                const double u = fabs(A1[x] * ih), sg = A2[x] * ih * ih;
                um = fmax(um, u);
                nm = fmax(nm, u + fsqrt(g * h + lam3 * sg * sg));
            }
        }
        um = warp_max_nonneg(um);
        nm = warp_max_nonneg(nm);
    };
    // cluster-wide maxima and the error flag -> dt of the next step
    auto reduce_dt = [&](double um, double nm, unsigned err, double &dtn) {
        if (lane == 0) { s_red[0][wid] = um; s_red[1][wid] = nm; }
        const unsigned eb = __reduce_or_sync(0xffffffffu, err);
        if (lane == 0) s_redf[wid] = __uint_as_float(eb);
        __syncthreads();
        if (wid == 0) {
            double a = 0.0, b = 0.0;
            unsigned e = 0u;
            for (int q = 0; q < CNT / 32; q++) {
                a = fmax(a, s_red[0][q]); b = fmax(b, s_red[1][q]); e |= __float_as_uint(s_redf[q]);
            }
            if (lane < C) {
                st_remote(&s_dx[c][0], &s_dmb, unsigned(lane), a);
                st_remote(&s_dx[c][1], &s_dmb, unsigned(lane), b);
                st_remote(&s_dx[c][2], &s_dmb, unsigned(lane), double(e));
            }
        }
        mbar_wait(dmb, pd);
        pd ^= 1u;
        // (non-negative doubles: the warp max of the bit patterns, C <= 32 lanes)
        const bool ql = lane < C;
        const double a = warp_max_nonneg(ql ? s_dx[lane][0] : 0.0), b = warp_max_nonneg(ql ? s_dx[lane][1] : 0.0);
        const double e = warp_max_nonneg(ql ? s_dx[lane][2] : 0.0);
        __syncthreads();
        if (tid == 0) arm(dmb, DB);
        double d = dt_rule(P.cfl, P.mcfl, P.dx, P.idx, a, b);
        if (t_end > 0.0) {
            if (!(t < t_end)) d = 0.0;
            else if (t + d >= t_end) d = t_end - t;          // land exactly on t_end
        }
        if (!(d >= 0.0) || !isfinite(d)) { acc.err |= ERR_DT; d = 0.0; }
        if (e != 0.0) d = 0.0;                              // an error anywhere in the member: stop
        dtn = d;
        return b;
    };
    double dtm;
    {
        double um, nm;
        local_maxima(um, nm);
        reduce_dt(um, nm, 0u, dtm);
    }
    int kdone = 0;
    const double kap = P.order == 2 ? 0.25 : 0.0;

#pragma unroll 1
    for (int step = 0; step < K; step++) {
        if (dtm == 0.0) {                              // member at t_end (or stopped): carry
            continue;
        }
        ML_MARK(0, 15);
        // ===== the two IMEX stages; stage 2 inputs E2, R2 =====
#pragma unroll 1
        for (int st = 0; st < 2; st++) {
            const bool st2 = st == 1;
            const StageC S = stage_consts(P, st2 ? P.aI2 : P.aI1, dtm, lam);
            const double tau = S.tau, idx1 = S.idx1, tdx2 = S.tdx2, t2h = S.t2h, lt2 = S.lt2;
            const double lt2h = S.lt2h, ltdx2 = S.ltdx2, ltau = S.ltau;
            // ---- phase 1 (E = arrays 0..3; R: stage 1 = E, stage 2 in the R slots)
            double wd[CMCH], hRv[CMCH];
            {
                RowCtx Cx{};
                Cx.tau = tau; Cx.tdx2 = tdx2; Cx.t2 = S.t2; Cx.lt2 = lt2; Cx.lam = lam; Cx.lam3 = lam3;
                Cx.ltau = ltau; Cx.g = g; Cx.idx = idx1;
                Cx.c23 = (2.0 / 3.0) * lam * lt2;
                // (R = E in stage 1: a runtime choice, one copy of the code for both stages)
                if ((tid == 0 && !left_phys) || (tid == 32 && !right_phys))
                    cl_single_row<BATHY>(Cx, kap, sB, tid == 0 ? -1 : Tc, A0, A1, A2, A3, sQd, sHd, sBe, sDe, !st2);
                if (live) {
                    double wh[3], wq[3], wH[3], wW[3];
#pragma unroll
                    for (int k = 0; k < 3; k++) {
                        const int x = swz(r0 - 2 + k);
                        wh[k] = A0[x]; wq[k] = A1[x]; wH[k] = A2[x]; wW[k] = A3[x];
                    }
                    FState Mm = muscl_minus(wh, wq, wH, wW, kap);
#pragma unroll
                    for (int k = 0; k < 2; k++) { wh[k] = wh[k + 1]; wq[k] = wq[k + 1]; wH[k] = wH[k + 1]; wW[k] = wW[k + 1]; }
                    {
                        const int x = swz(r0 + 1);
                        wh[2] = A0[x]; wq[2] = A1[x]; wH[2] = A2[x]; wW[2] = A3[x];
                    }
                    FState Pn, Mr;
                    muscl_pair(wh, wq, wH, wW, kap, Pn, Mr);
                    Face Fl = rusanov(Mm, Pn);
#pragma unroll
                    for (int i = 0; i < CMCH; i++) {
                        const int r = r0 + i;
                        double ch[3], cq[3], cH[3], cW[3];
#pragma unroll
                        for (int k = 0; k < 3; k++) { ch[k] = wh[k]; cq[k] = wq[k]; cH[k] = wH[k]; cW[k] = wW[k]; }
#pragma unroll
                        for (int k = 0; k < 2; k++) { wh[k] = wh[k + 1]; wq[k] = wq[k + 1]; wH[k] = wH[k + 1]; wW[k] = wW[k + 1]; }
                        {
                            const int x = swz(r + 2);
                            wh[2] = A0[x]; wq[2] = A1[x]; wH[2] = A2[x]; wW[2] = A3[x];
                        }
                        FState Mn;
                        muscl_pair(wh, wq, wH, wW, kap, Pn, Mn);
                        const Face Fr = rusanov(Mr, Pn);
                        Mr = Mn;
                        double beta;
                        cl_row_update<BATHY>(Cx, sB, r, ch, cq, cH, cW, Fl, Fr, sQd, sHd, sBe, sDe, wd[i], beta, hRv[i],
                                             !st2);
                        if (!(beta > 0.0)) acc.err |= ERR_COERC;
                        acc.bhi = max(acc.bhi, __double2hiint(beta));
                        acc.kkey = min(acc.kkey, khi_key(beta));
                        Fl = Fr;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < CMCH; i++) { wd[i] = 0.0; hRv[i] = 0.0; }
                }
            }
            __syncthreads();
            ML_MARK(st, 0);                            // phase 1
            if (tid == 0 && left_phys) {
                const int x = swz(-1), y = swz(0);
                sQd[x] = (wall_l ? -1.0 : 1.0) * sQd[y]; sHd[x] = sHd[y]; sDe[x] = sDe[y]; sBe[x] = -sBe[y];
            }
            if (tid == 32 && right_phys) {
                const int x = swz(Tc), y = swz(Tc - 1);
                sQd[x] = (wall_r ? -1.0 : 1.0) * sQd[y]; sHd[x] = sHd[y]; sDe[x] = sDe[y]; sBe[x] = -sBe[y];
            }
            __syncthreads();
            // ---- phase 2: assembly, partition, PCR (arrays 4..7), exact cluster solve
            double vb[CMCH + 2], vd[CMCH + 2], vH[CMCH + 2], vq[CMCH + 2];
#pragma unroll
            for (int k = 0; k < CMCH + 2; k++) {
                const int x = swz(r0 - 1 + k);
                vb[k] = live ? sBe[x] : 0.0; vd[k] = live ? sDe[x] : 0.0;
                vH[k] = live ? sHd[x] : 0.0; vq[k] = live ? sQd[x] : 0.0;
            }
            double am[CMCH], cm[CMCH], dm[CMCH];
#pragma unroll
            for (int i = 0; i < CMCH; i++) {
                const double rl = t2h * (vb[i] + vb[i + 1]), rr = t2h * (vb[i + 1] + vb[i + 2]);
                const double ml = lt2h * (vd[i] + vd[i + 1]), mr = lt2h * (vd[i + 1] + vd[i + 2]);
                const double rhs = hRv[i] - tdx2 * (vq[i + 2] - vq[i]) + mr * (vH[i + 2] - vH[i + 1])
                                   - ml * (vH[i + 1] - vH[i]);
                const double a = -rl, cc = -rr, dg = 1.0 + rl + rr;
                if (i == 0) {
                    const double inv = rcp(dg);
                    am[0] = a * inv; cm[0] = cc * inv; dm[0] = rhs * inv;
                } else {
                    const double inv = rcp(dg - a * cm[i - 1]);
                    am[i] = -a * am[i - 1] * inv; cm[i] = cc * inv; dm[i] = (rhs - a * dm[i - 1]) * inv;
                }
            }
            const double aE = am[CMCH - 1], cE = cm[CMCH - 1], dE = dm[CMCH - 1];
            {
                double Pn = 0.0, Qn = 0.0, Rn = -1.0;
#pragma unroll
                for (int i = CMCH - 2; i >= 0; i--) {
                    const double Pi = dm[i] - cm[i] * Pn, Qi = am[i] - cm[i] * Qn, Ri = -cm[i] * Rn;
                    dm[i] = Pi; am[i] = Qi; cm[i] = Ri;
                    Pn = Pi; Qn = Qi; Rn = Ri;
                }
            }
            double P1 = __shfl_down_sync(0xffffffffu, dm[0], 1), Q1 = __shfl_down_sync(0xffffffffu, am[0], 1);
            double R1 = __shfl_down_sync(0xffffffffu, cm[0], 1);
            if (lane == 0) { s_cw[wid][0] = dm[0]; s_cw[wid][1] = am[0]; s_cw[wid][2] = cm[0]; }
            __syncthreads();                              // (also: all window loads of arrays 4..7 done)
            if (lane == 31) {
                if (wid + 1 < CNT / 32) { P1 = s_cw[wid + 1][0]; Q1 = s_cw[wid + 1][1]; R1 = s_cw[wid + 1][2]; }
                else { P1 = Q1 = R1 = 0.0; }
            }
            double A_ = aE, C_ = -cE * R1, D_ = dE - cE * P1, V_ = 0.0, W_ = 0.0;
            {
                const double ib = rcp(1.0 - cE * Q1);
                A_ *= ib; C_ *= ib; D_ *= ib;
            }
            if (tid == 0) { V_ = A_; A_ = 0.0; }
            if (tid == ks - 1) { W_ = C_; C_ = 0.0; }
            if (tid >= ks) { A_ = 0.0; C_ = 0.0; D_ = 0.0; V_ = 0.0; W_ = 0.0; }
            double *const pb0 = A4 + PPAD, *const pb1 = A4 + 5 * PSTR + PPAD;
            auto put = [&](double *b, int k, double a, double cc, double d, double v, double w_) {
                b[k] = a; b[PSTR + k] = cc; b[2 * PSTR + k] = d; b[3 * PSTR + k] = v; b[4 * PSTR + k] = w_;
            };
            put(pb0, tid, A_, C_, D_, V_, W_);
            if (tid < 2 * PPAD) {
                const int k = tid < PPAD ? tid - PPAD : CNT + tid - PPAD;
                put(pb0, k, 0.0, 0.0, 0.0, 0.0, 0.0);
                put(pb1, k, 0.0, 0.0, 0.0, 0.0, 0.0);
            }
            {
                const float ea = float(fabs(A_)), ec = float(fabs(C_));
                const float ev = warp_max_nonneg(ea > ec ? ea : ec);
                if (lane == 0) s_redf[wid] = ev;
            }
            __syncthreads();
            int lim = CNT;
            {
                float e0 = 0.0f;
#pragma unroll
                for (int q = 0; q < CNT / 32; q++) e0 = fmaxf(e0, s_redf[q]);
                if (e0 < 0.4f) {
                    const float q = __fdividef(64.0f, -__log2f(e0) - 0.28f);
                    const int qi = int(ceilf(q));
                    lim = qi <= 1 ? 1 : min(CNT, 1 << (32 - __clz(qi - 1)));
                }
            }
            const double *fin = pb0;
            for (int sd = 1, pp = 0; sd < lim; sd <<= 1, pp ^= 1) {
                const double *cur = pp ? pb1 : pb0;
                double *nxt = pp ? pb0 : pb1;
                // a row whose partner tid -/+ sd lies outside 0..CNT-1 has A_ (C_) exactly 0
                // at this level (row 0 starts with A_ = 0, rows >= ks-1 with C_ = 0, and
                // PCR keeps it so), so any finite value may stand in for the partner's:
                // the pads (zeros) for sd <= PPAD, the row's own slot beyond
                int km = tid - sd, kp = tid + sd;
                km = (sd <= PPAD || km >= 0) ? km : tid;
                kp = (sd <= PPAD || kp < CNT) ? kp : tid;
                const double Am = cur[km], Cm = cur[PSTR + km], Dm = cur[2 * PSTR + km], Vm = cur[3 * PSTR + km], Wm = cur[4 * PSTR + km];
                const double Ap = cur[kp], Cp = cur[PSTR + kp], Dp = cur[2 * PSTR + kp], Vp = cur[3 * PSTR + kp], Wp = cur[4 * PSTR + kp];
                const double ib = rcp(1.0 - A_ * Cm - C_ * Ap);
                const double An = -A_ * Am * ib, Cn = -C_ * Cp * ib;
                D_ = (D_ - A_ * Dm - C_ * Dp) * ib;
                V_ = (V_ - A_ * Vm - C_ * Vp) * ib;
                W_ = (W_ - A_ * Wm - C_ * Wp) * ib;
                A_ = An; C_ = Cn;
                put(nxt, tid, A_, C_, D_, V_, W_);
                __syncthreads();
                fin = nxt;
            }
            ML_MARK(st, 1);                            // assembly, partition, PCR
            const double Yl = fin[2 * PSTR + tid - 1], Vl = fin[3 * PSTR + tid - 1], Wl = fin[4 * PSTR + tid - 1];
            const double Yr = fin[2 * PSTR + tid + 1], Vr = fin[3 * PSTR + tid + 1], Wr = fin[4 * PSTR + tid + 1];
            const double Yks = fin[2 * PSTR + ks - 1], Vks = fin[3 * PSTR + ks - 1], Wks = fin[4 * PSTR + ks - 1];
            // publish the separator data to every CTA (DSMEM), wait for all of it
            if (wid == 0 || wid == (ks >> 5)) {
                double v6[6];
                if (wid == 0) {
                    v6[0] = __shfl_sync(0xffffffffu, dm[0], 0); v6[1] = __shfl_sync(0xffffffffu, am[0], 0);
                    v6[2] = __shfl_sync(0xffffffffu, cm[0], 0); v6[3] = __shfl_sync(0xffffffffu, D_, 0);
                    v6[4] = __shfl_sync(0xffffffffu, V_, 0); v6[5] = __shfl_sync(0xffffffffu, W_, 0);
                    for (int i = lane; i < 6 * C; i += 32) {
                        const int rk = i / 6, k = i - rk * 6;
                        st_remote(&s_cx[c][6 + k], &s_xmb, unsigned(rk), cl_pick6(v6, k));
                    }
                }
                if (wid == (ks >> 5)) {
                    const int ls = ks & 31;
                    v6[0] = __shfl_sync(0xffffffffu, aE, ls); v6[1] = __shfl_sync(0xffffffffu, cE, ls);
                    v6[2] = __shfl_sync(0xffffffffu, dE, ls);
                    v6[3] = Yks; v6[4] = Vks; v6[5] = Wks;
                    for (int i = lane; i < 6 * C; i += 32) {
                        const int rk = i / 6, k = i - rk * 6;
                        st_remote(&s_cx[c][k], &s_xmb, unsigned(rk), cl_pick6(v6, k));
                    }
                }
            }
            ML_MARK(st, 2);                            // publish
            mbar_wait(xmb, px);
            px ^= 1u;
            ML_MARK(st, 3);                            // separator wait
            // separator system (lanes = equations, every warp), as in cl_stage_kernel
            double Lm = 0.0, Lc, Lp = 0.0, nx[6];
            {
                double a = 0.0, cc = 0.0, d = 0.0;
                const int j = lane;
                if (j < C) {
                    const int jn = (j + 1 < C) ? j + 1 : (cyc ? 0 : -1);
                    const double aEj = s_cx[j][0], cEj = s_cx[j][1], dEj = s_cx[j][2];
                    const double Yp = s_cx[j][3], Vp = s_cx[j][4], Wp = s_cx[j][5];
                    double P1n = 0, Q1n = 0, R1n = 0, Y0 = 0, V0 = 0, W0 = 0;
                    if (jn >= 0) {
                        P1n = s_cx[jn][6]; Q1n = s_cx[jn][7]; R1n = s_cx[jn][8];
                        Y0 = s_cx[jn][9]; V0 = s_cx[jn][10]; W0 = s_cx[jn][11];
                    }
                    const double cr = cEj * R1n;
                    const double sub = -aEj * Vp, dia = (1.0 - cEj * Q1n) - aEj * Wp + cr * V0, sup = cr * W0;
                    const double rhs = dEj - cEj * P1n - aEj * Yp + cr * Y0;
                    const double id = rcp(dia);
                    a = sub * id; cc = sup * id; d = rhs * id;
                }
                const bool dec = __all_sync(0xffffffffu, fabs(a) <= 5.421010862427522e-20 &&
                                                             fabs(cc) <= 5.421010862427522e-20);
                for (int sd = 1; sd < C && !dec; sd <<= 1) {
                    int jm = j - sd, jp = j + sd;
                    if (cyc) { jm = (jm % C + C) % C; jp = jp % C; }
                    const double am_ = __shfl_sync(0xffffffffu, a, jm & 31), cm2 = __shfl_sync(0xffffffffu, cc, jm & 31);
                    const double dm_ = __shfl_sync(0xffffffffu, d, jm & 31);
                    const double ap_ = __shfl_sync(0xffffffffu, a, jp & 31), cp2 = __shfl_sync(0xffffffffu, cc, jp & 31);
                    const double dp_ = __shfl_sync(0xffffffffu, d, jp & 31);
                    const bool okm = j < C && jm >= 0 && jm < C, okp = j < C && jp >= 0 && jp < C;
                    const double Am = okm ? am_ : 0.0, Cm = okm ? cm2 : 0.0, Dm = okm ? dm_ : 0.0;
                    const double Ap = okp ? ap_ : 0.0, Cp = okp ? cp2 : 0.0, Dp = okp ? dp_ : 0.0;
                    const double ib = rcp(1.0 - a * Cm - cc * Ap);
                    const double na = -a * Am * ib, nc = -cc * Cp * ib;
                    d = (d - a * Dm - cc * Dp) * ib;
                    a = na; cc = nc;
                }
                const double Lj = (cyc && !dec) ? d * rcp(1.0 + a + cc) : d;
                Lm = (c > 0 || cyc) ? __shfl_sync(0xffffffffu, Lj, cl_) : 0.0;
                Lc = __shfl_sync(0xffffffffu, Lj, c);
                Lp = __shfl_sync(0xffffffffu, Lj, cr_);
#pragma unroll
                for (int k = 0; k < 6; k++) nx[k] = s_cx[cr_][6 + k];
            }
            __syncthreads();                          // s_cx read by every warp
            if (tid == 0) arm(xmb, XB);
            ML_MARK(st, 4);                            // separator solve
            double hb[CMCH], hLn, hRn;
            {
                const double Xk = tid < ks ? D_ - V_ * Lm - W_ * Lc : (tid == ks ? Lc : 0.0);
                const double XL = tid == 0 ? Lm : Yl - Vl * Lm - Wl * Lc;
                const double XR = tid + 1 == ks ? Lc : Yr - Vr * Lm - Wr * Lc;
#pragma unroll
                for (int i = 0; i < CMCH; i++) hb[i] = live ? ((i == CMCH - 1) ? Xk : dm[i] - am[i] * XL - cm[i] * Xk) : 1.0;
                hLn = live ? (left_phys && tid == 0 ? hb[0] : XL) : 1.0;
                if (!live) hRn = 1.0;
                else if (tid < ks) hRn = P1 - Q1 * Xk - R1 * XR;
                else if (right_phys) hRn = hb[CMCH - 1];
                else {
                    const double X0n = nx[3] - nx[4] * Lc - nx[5] * Lp;
                    hRn = nx[0] - nx[1] * Lc - nx[2] * X0n;
                }
            }
            acc.rho = fmax(acc.rho, S.t2 * __hiloint2double(acc.bhi + 1, 0));
            // ---- phase 3: back-substitution, own rows; H-form out
            double qbv[CMCH], Hbv[CMCH], Wbv[CMCH];
#pragma unroll
            for (int i = 0; i < CMCH; i++) {
                const int r = r0 + i;
                const double h0 = hb[i];
                const double hl = (i > 0) ? hb[i - 1] : hLn, hr = (i < CMCH - 1) ? hb[i + 1] : hRn;
                double qb = vq[i + 1] - tdx2 * vb[i + 1] * (hr - hl) - ltdx2 * vd[i + 1] * (vH[i + 2] - vH[i]);
                if (BATHY && live) {
                    const double bm = sB[swz(r - 1)], bp = sB[swz(r + 1)];
                    qb -= tau * g * A0[swz(r)] * (bp - bm) * (0.5 * idx1);   // A9
                }
                const double rden = rcp(h0 * h0 + lt2);
                const double HdD = vH[i + 1] * rden;
                qbv[i] = qb;
                Hbv[i] = HdD * (h0 * h0);
                Wbv[i] = wd[i] - ltau * HdD;
                if (live) {
                    if (!(h0 > P.h_min)) acc.err |= ERR_DRY;
                    if (!isfinite(h0 + qb + HdD + Wbv[i])) acc.err |= ERR_NONFINITE;
                }
            }
            __syncthreads();                          // PCR buffers (arrays 4..7) and arrays 0..3 all read
            ML_MARK(st, 5);                            // recovery + phase 3
            if (!st2) {
                // ---- E2, R2 of the own rows -> arrays 0..3 / R slots;
                //      edge rows to the neighbours (DSMEM) or mirrored (A10)
                const double wE = P.wE, wR = P.wR;
                double e[4][CMCH], rr[4][CMCH];
#pragma unroll
                for (int i = 0; i < CMCH; i++) {
                    const int x = swz(r0 + i);                 // U^n of the own rows: still in arrays 0..3
                    const double un[4] = {A0[x], A1[x], A2[x], A3[x]};
                    const double u1[4] = {hb[i], qbv[i], Hbv[i], Wbv[i]};
#pragma unroll
                    for (int f = 0; f < 4; f++) {
                        const double d = u1[f] - un[f];
                        e[f][i] = fma(wE, d, un[f]);
                        rr[f][i] = fma(wR, d, un[f]);
                    }
                }
                if (live) {
#pragma unroll
                    for (int i = 0; i < CMCH; i++) {
                        const int x = swz(r0 + i);
                        A0[x] = e[0][i]; A1[x] = e[1][i]; A2[x] = e[2][i]; A3[x] = e[3][i];
                        sDe[x] = rr[0][i]; sQd[x] = rr[1][i]; sHd[x] = rr[2][i]; sBe[x] = rr[3][i];
                    }
                }
                if (tid == 0 && !left_phys) {         // rows 0..3 -> left neighbour's rows Tl .. Tl+3
                    for (int i = 0; i < CMCH; i++)
                        for (int f = 0; f < 4; f++) st_remote(sU[f] + swz(Tl + i), &s_emb, cl_, e[f][i]);
                    st_remote(sDe + swz(Tl), &s_emb, cl_, rr[0][0]); st_remote(sQd + swz(Tl), &s_emb, cl_, rr[1][0]);
                    st_remote(sHd + swz(Tl), &s_emb, cl_, rr[2][0]); st_remote(sBe + swz(Tl), &s_emb, cl_, rr[3][0]);
                }
                if (tid == ks && !right_phys) {       // rows Tc-4 .. Tc-1 -> right neighbour's rows -4 .. -1
                    for (int i = 0; i < CMCH; i++)
                        for (int f = 0; f < 4; f++) st_remote(sU[f] + swz(i - 4), &s_emb, cr_, e[f][i]);
                    st_remote(sDe + swz(-1), &s_emb, cr_, rr[0][3]); st_remote(sQd + swz(-1), &s_emb, cr_, rr[1][3]);
                    st_remote(sHd + swz(-1), &s_emb, cr_, rr[2][3]); st_remote(sBe + swz(-1), &s_emb, cr_, rr[3][3]);
                }
                __syncthreads();
                mirror_halo(sU, false);
                ML_MARK(0, 6);                         // E2 / R2 formed and sent
                mbar_wait(emb, pe);
                pe ^= 1u;
                __syncthreads();
                if (tid == 0) arm(emb, EB);
                ML_MARK(0, 7);                         // E2 / R2 halo wait
                continue;                             // -> stage 2
            }
            // ---- final stage: A19 filter (rows -2, -1, Tc, Tc+1 via DSMEM), relaxation,
            //      U^{n+1} into arrays 0..3 and to the neighbours' halo rows
            if (filt) {
                double *const sQb = A4, *const sWb = A5;
                if (live) {
#pragma unroll
                    for (int i = 0; i < CMCH; i++) { sQb[swz(r0 + i)] = qbv[i]; sWb[swz(r0 + i)] = Wbv[i]; }
                }
                if (tid == 0) {
                    if (left_phys) {
                        const double pq = wall_l ? -1.0 : 1.0;
                        sQb[swz(-1)] = pq * qbv[0]; sWb[swz(-1)] = Wbv[0];
                        sQb[swz(-2)] = wall_l ? pq * qbv[1] : qbv[0]; sWb[swz(-2)] = wall_l ? Wbv[1] : Wbv[0];
                    } else {
                        st_remote(sQb + swz(Tl), &s_fmb, cl_, qbv[0]); st_remote(sWb + swz(Tl), &s_fmb, cl_, Wbv[0]);
                        st_remote(sQb + swz(Tl + 1), &s_fmb, cl_, qbv[1]); st_remote(sWb + swz(Tl + 1), &s_fmb, cl_, Wbv[1]);
                    }
                }
                if (tid == ks) {
                    if (right_phys) {
                        const double pq = wall_r ? -1.0 : 1.0;
                        sQb[swz(Tc)] = pq * qbv[3]; sWb[swz(Tc)] = Wbv[3];
                        sQb[swz(Tc + 1)] = wall_r ? pq * qbv[2] : qbv[3]; sWb[swz(Tc + 1)] = wall_r ? Wbv[2] : Wbv[3];
                    } else {
                        st_remote(sQb + swz(-2), &s_fmb, cr_, qbv[2]); st_remote(sWb + swz(-2), &s_fmb, cr_, Wbv[2]);
                        st_remote(sQb + swz(-1), &s_fmb, cr_, qbv[3]); st_remote(sWb + swz(-1), &s_fmb, cr_, Wbv[3]);
                    }
                }
                __syncthreads();
                ML_MARK(1, 6);                         // filter rows sent
                mbar_wait(fmb, pf);
                pf ^= 1u;
                ML_MARK(1, 7);                         // filter rows wait
                if (live) {
                    const double sig16 = P.filter_sigma * (1.0 / 16.0);
                    double xq[CMCH + 4], xw[CMCH + 4];
                    xq[0] = sQb[swz(r0 - 2)]; xq[1] = sQb[swz(r0 - 1)];
                    xq[CMCH + 2] = sQb[swz(r0 + CMCH)]; xq[CMCH + 3] = sQb[swz(r0 + CMCH + 1)];
                    xw[0] = sWb[swz(r0 - 2)]; xw[1] = sWb[swz(r0 - 1)];
                    xw[CMCH + 2] = sWb[swz(r0 + CMCH)]; xw[CMCH + 3] = sWb[swz(r0 + CMCH + 1)];
#pragma unroll
                    for (int i = 0; i < CMCH; i++) { xq[i + 2] = qbv[i]; xw[i + 2] = Wbv[i]; }
#pragma unroll
                    for (int i = 0; i < CMCH; i++) {
                        qbv[i] = xq[i + 2] - sig16 * (xq[i] - 4.0 * xq[i + 1] + 6.0 * xq[i + 2] - 4.0 * xq[i + 3] + xq[i + 4]);
                        Wbv[i] = xw[i + 2] - sig16 * (xw[i] - 4.0 * xw[i + 1] + 6.0 * xw[i + 2] - 4.0 * xw[i + 3] + xw[i + 4]);
                        if (!isfinite(qbv[i] + Wbv[i])) acc.err |= ERR_NONFINITE;
                    }
                }
                __syncthreads();
                if (tid == 0) arm(fmb, FB);
            }
            if (relax && live) {
                const double t_new = t + dtm;
#pragma unroll
                for (int i = 0; i < CMCH; i++) {
                    const double bb = BATHY ? sB[swz(r0 + i)] : 0.0;
                    double h0 = hb[i], Ko = Hbv[i] + 1.5 * h0 * bb;
                    relax_cell(P, P.x_min + (double(s + r0 + i) + 0.5) * P.dx, bb, t_new, h0, qbv[i], Ko, Wbv[i]);
                    hb[i] = h0;
                    Hbv[i] = Ko - 1.5 * h0 * bb;
                }
            }
            if (live) {
#pragma unroll
                for (int i = 0; i < CMCH; i++) {
                    const int x = swz(r0 + i);
                    A0[x] = hb[i]; A1[x] = qbv[i]; A2[x] = Hbv[i]; A3[x] = Wbv[i];
                }
            }
            if (tid == 0 && !left_phys) {
                for (int i = 0; i < CMCH; i++) {
                    const double v[4] = {hb[i], qbv[i], Hbv[i], Wbv[i]};
                    for (int f = 0; f < 4; f++) st_remote(sU[f] + swz(Tl + i), &s_umb, cl_, v[f]);
                }
            }
            if (tid == ks && !right_phys) {
                for (int i = 0; i < CMCH; i++) {
                    const double v[4] = {hb[i], qbv[i], Hbv[i], Wbv[i]};
                    for (int f = 0; f < 4; f++) st_remote(sU[f] + swz(i - 4), &s_umb, cr_, v[f]);
                }
            }
            __syncthreads();
            mirror_halo(sU, false);
        }
        // ---- commit the step, dt of the next one from U^{n+1}
        t = (t_end > 0.0 && dtm == t_end - t) ? t_end : t + dtm;
        kdone++;
        ML_MARK(1, 8);                                 // filter, relaxation, U^{n+1} + halos sent
        double um, nm;
        local_maxima(um, nm);
        reduce_dt(um, nm, acc.err, dtm);
        ML_MARK(1, 9);                                 // dt maxima, cluster max, dt
        mbar_wait(umb, pu);
        pu ^= 1u;
        __syncthreads();
        if (tid == 0) arm(umb, UB);
        ML_MARK(1, 10);                                // U halo wait
#if HSGN_EXP_TIMING
        if (prof) g_clt[1][15] += 1ull;
#endif
    }

    // ---- store U (K-form) of the own rows, the member's time and dt maxima
    if (live) {
        const size_t gd = mo + size_t(s + r0);
        double o[4][CMCH];
#pragma unroll
        for (int i = 0; i < CMCH; i++) {
            const int x = swz(r0 + i);
            const double bb = BATHY ? sB[x] : 0.0;
            o[0][i] = A0[x]; o[1][i] = A1[x]; o[2][i] = A2[x] + 1.5 * A0[x] * bb; o[3][i] = A3[x];
        }
#pragma unroll
        for (int f = 0; f < 4; f++) {
            double2 *const op = reinterpret_cast<double2 *>(B.out[f] + gd);
            op[0] = make_double2(o[f][0], o[f][1]);
            op[1] = make_double2(o[f][2], o[f][3]);
        }
    }
    {
        double um, nm;
        local_maxima(um, nm);                     // (warp maxima)
        acc.umax = um;
        acc.numax = nm;
        // error bits, maxima of the final state into slot (k0 + K) % 3, time level
        const unsigned eb = __reduce_or_sync(0xffffffffu, acc.err);
        if (lane == 0 && eb) atomicOr(P.err, eb);
        const int kk = __reduce_min_sync(0xffffffffu, acc.kkey);
        if (lane == 0) {
            const int slot = (k0 + K) % 3;
            atomicMax(P.maxes + (slot * 2 + 0) * P.members + m, (unsigned long long)__double_as_longlong(um));
            atomicMax(P.maxes + (slot * 2 + 1) * P.members + m, (unsigned long long)__double_as_longlong(nm));
            if (kk != 0x7fffffff && P.kmin) atomicMax(P.kmin, ~unsigned(kk));
            const float rf = float(acc.rho);
            if (rf > 0.0f) atomicMax(P.rho_obs, (unsigned long long)__double_as_longlong(double(rf) * (1.0 + 1e-6)));
        }
        if (c == 0 && tid == 0) {
            P.t[((k0 + K) & 1) * P.members + m] = t;
            P.dt[m] = dtm;
        }
    }
    (void)kdone;
    // no remote store may target an exited CTA: the last exchanges were waited for
}

}  // namespace hsgn
