// hsgn_cluster.cuh -- sm_100a cluster stage kernel of the SI-IMEX hSGN step:
// one IMEX stage S(E, R, tau) with the depth system of P:509-512
// solved EXACTLY across the CTAs of a thread-block cluster (no overlap rows,
// no decay check).  Citations: P:n = PAPER.md line n, Ak = DESIGN.md reading k.
//
// Work split.  A member (one periodic or walled 1-D domain of n cells) is
// cut into C contiguous tiles of T rows (the last one n - (C-1) T), one CTA
// each; the C CTAs of a member form one cluster (C <= 16).  Within a CTA every
// thread owns a chunk of CMCH = 4 consecutive rows.
//
// Exact solve (SPIKE inside the cluster).  The depth matrix is tridiagonal
// (cyclic for periodic members).  Each chunk is reduced to its last row (the
// partition method: downward + upward sweeps in registers), giving a
// tridiagonal system in the chunk-end unknowns X_k.  The last chunk end of CTA
// j is its SEPARATOR L_j (row T_j - 1).  Between two separators lie only rows
// of one CTA, so each CTA solves its interior chunk ends X_0 .. X_{ks-1} by PCR
// in shared memory with three right-hand sides:
//     X_k = Y_k - V_k L_{j-1} - W_k L_j
// (V, W: responses to the couplings of its first and last interior rows to the
// two separators).  Every CTA then pushes 12 numbers into the shared memory of
// every CTA of the cluster (DSMEM, st.shared::cluster): the raw reduced row of
// its separator chunk, (Y, V, W) at its last interior slot, and the first-row
// relation and (Y, V, W) of its chunk 0 (what the separator row of the
// previous CTA needs).  After one cluster barrier each CTA forms the C
// separator equations
//     -a V' L_{j-1} + (B - a W' + c R1 V0) L_j + c R1 W0 L_{j+1}
//        = d - c P1 - a Y' + c R1 Y0
// and solves them redundantly by PCR over C lanes of one warp (cyclic for
// periodic members, indices mod C).  X_k and every row then follow exactly.
// The result is the unique solution of the full system (to round-off); PCR
// stops early only once the reduced couplings are below 2^-64 (then the rows
// are decoupled to round-off).
//
// Shared-memory layout.  Phases 1-3 are chunk-parallel (thread t reads rows
// 4t-2 .. 4t+5); a plain row layout would put the 32 threads of a warp on 4
// bank pairs.  Row arrays are therefore stored chunk-major with an XOR swizzle,
//     row r (r in [-4, 4 CNT + 4)):  j = r + 4,  i = j & 3,  c = j >> 2,
//     index = i * CCAP + (c ^ (i << 3)),
// which is conflict-free (2 wavefronts per warp access, the minimum for 8-B
// words) both chunk-parallel (fixed i, consecutive c) and row-parallel
// (consecutive r).  TMA lands the tile in plain row order; one row-parallel
// pass (which also forms E and R of stage 2) rewrites it swizzled
// in place, through registers.
//
// Phases (CNT = 128 threads, rows -4 .. T+3 of the tile in shared memory):
//   load    : TMA bulk copies of U^n (and U1, b) rows -4 .. T+3 (periodic wrap
//             by extra segments; physical ends mirrored in the next pass)
//   pass    : E, R (stage 2), H = K - 1.5 h b, wall parity, swizzle
//   phase 1 : MUSCL + Rusanov faces, predictor, coefficients (rows -1 .. T)
//   phase 2 : assembly, partition sweeps, interior PCR (Y, V, W), DSMEM
//             exchange, separator PCR, recovery -> hbar (rows -1 .. T)
//   phase 3 : back-substitution; final stage: A19 filter with a +-2 row DSMEM
//             halo exchange, dt maxima; staged TMA bulk store
#pragma once
#include "hsgn_kernels.cuh"

#ifndef HSGN_CMINB
#define HSGN_CMINB 4
#endif
#ifndef HSGN_CMINB1            // first-stage kernels: 96 registers fit without spills, 5 CTAs
#define HSGN_CMINB1 5          // per SM (cfg3 stage 1: cluster 468 -> 455 us, SPIKE 699 -> 655
#endif                         // us; the second stage measured slower at 5)

namespace hsgn {

constexpr int CNT = 128;                 // threads per CTA (= chunks)
constexpr int CMCH = 4;                  // rows per chunk
constexpr int CT_MAX = CNT * CMCH;       // 512 rows per CTA
constexpr int CCAP = CNT + 32;           // swizzled capacity in chunks (rows -4 .. T+3; XOR < CCAP)
constexpr int CARR = 4 * CCAP;           // doubles per row array (640)
constexpr int C_MAX = 16;                // CTAs per cluster (16: non-portable size)
constexpr int CNARR = 8;
constexpr size_t CSMEM_BYTES = size_t(CNARR) * CARR * sizeof(double);        // 40 KiB
constexpr size_t CSMEM_BYTES_B = size_t(CNARR + 1) * CARR * sizeof(double);  // + b (45 KiB)
constexpr int XPUB = 12;                 // doubles each CTA publishes to the cluster

__shared__ double s_cx[C_MAX][XPUB];     // separator data of every CTA of the cluster
__shared__ double s_cw[NT / 32][3];      // chunk-relation exchange across warps

__device__ __forceinline__ int swz(int r)
{
    const int j = r + 4, i = j & 3;
    return i * CCAP + ((j >> 2) ^ (i << 3));
}

// Cluster barrier, used once: every CTA arrives (relaxed: no memory ordering,
// only "started, mbarriers initialised" -- fence.mbarrier_init orders those)
// right after its start and waits just before its first remote store.
__device__ __forceinline__ void cl_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory"); }

// shared::cluster address of `p` (a shared variable of this CTA) in CTA `rank`
__device__ __forceinline__ unsigned cl_map(const void *p, unsigned rank)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

// Remote store of one double into CTA `rank`'s shared memory at the address
// of `dst` there, completing 8 transaction bytes on that CTA's mbarrier `mbar`
// (st.async: the receiver waits on its own mbarrier, no cluster barrier).
__device__ __forceinline__ void st_remote(const void *dst, const void *mbar, unsigned rank, double v)
{
    const unsigned a = cl_map(dst, rank), b = cl_map(mbar, rank);
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n"
                 ::"r"(a), "l"((unsigned long long)__double_as_longlong(v)), "r"(b) : "memory");
}

__shared__ __align__(8) unsigned long long s_xmb;   // separator data received from the near CTAs
__shared__ __align__(8) unsigned long long s_xmb2;  // ... from the others (the coupled case only)
__shared__ __align__(8) unsigned long long s_fmb;   // filter halo rows received

// Separator data routing.  Equation j needs the OWN part (values 0..5) of CTA
// j and the LEFT part (values 6..11) of CTA j+1; a CTA c needs equations
// c-1, c, c+1 (and the left part of c+1 for its halo row T), i.e. own parts of
// CTAs c-1 .. c+1 and left parts of c .. c+2.  part = -1: own, 0: left.
__device__ __forceinline__ bool cl_is_near(int s, int r, int C, bool cyc, int part)
{
    // sender s -> receiver r: own near iff s - r in {-1, 0, 1}; left iff s - r in {0, 1, 2}
    // (mod C for periodic members, C a power of two)
    if (cyc) {
        if (C <= 3) return true;
        const int d = (s - r - part) & (C - 1);
        return d <= 2;
    }
    const int d = s - r - part;
    return d >= 0 && d <= 2;
}

// number of distinct near senders of receiver c for a part (see cl_is_near)
__device__ __forceinline__ int cl_near_count(int c, int C, bool cyc, int part)
{
    if (cyc) return C < 3 ? C : 3;
    const int lo = max(c + part, 0), hi = min(c + part + 2, C - 1);
    return hi >= lo ? hi - lo + 1 : 0;
}

__device__ __forceinline__ double cl_pick6(const double (&v)[6], int k)
{
    return k == 0 ? v[0] : k == 1 ? v[1] : k == 2 ? v[2] : k == 3 ? v[3] : k == 4 ? v[4] : v[5];
}

// Predictor (A9) and coefficients at E (A2) of one row r
// of the swizzled tile; same arithmetic as row_update (hsgn_kernels.cuh).
// R = (h, q, H, W) of the row (stage 1: R = E) is read from the row's slot of
// (sDe, sQd, sHd, sBe), which then take delta, q^dag, H^dag, beta.
template <bool BATHY, bool R_IS_E = false>
__device__ __forceinline__ void cl_row_update(const RowCtx &C, const double *sB, int r,
                                              const double (&ch)[3], const double (&cq)[3],
                                              const double (&cH)[3], const double (&cW)[3],
                                              const Face &Fl, const Face &Fr, double *sQd, double *sHd,
                                              double *sBe, double *sDe, double &Wd_out, double &beta_out,
                                              double &hR_out, bool r_is_e = R_IS_E)
{
    const int x = swz(r);
    // R of the row (r_is_e: stage 1, R = E)
    const double hR = r_is_e ? ch[1] : sDe[x], qR = r_is_e ? cq[1] : sQd[x];
    const double HR = r_is_e ? cH[1] : sHd[x], WR = r_is_e ? cW[1] : sBe[x];
    const double hE = ch[1], qE = cq[1], HE = cH[1];
    const double s2 = hE * hE, den = s2 + C.lt2;
    const double Z = rcp(hE * den);
    const double ihE = den * Z, D = hE * Z;
    const double sg = HE * (ihE * ihE);                              // eta/h
    double Dxb = 0.0, hRp = hR, ptil_term = 0.0;
    if (BATHY) {
        const double bm = sB[swz(r - 1)], b0 = sB[x], bp = sB[swz(r + 1)];
        Dxb = (bp - bm) * (0.5 * C.idx);
        const double Gr = C.g * (hE + ch[2]) * 0.5, Gl = C.g * (ch[0] + hE) * 0.5;
        hRp = hR + C.t2 * (Gr * (bp - b0) - Gl * (b0 - bm));          // zeta-form (A9)
        ptil_term = 1.5 * C.tau * C.lam3 * (1.0 - sg) * Dxb;          // p~
    }
    const double Wd = WR - C.tdx2 * (Fr.W - Fl.W) + C.ltau;
    const double Hd = HR - C.tdx2 * (Fr.H - Fl.H) - 1.5 * C.tau * qE * Dxb + C.tau * Wd;
    const double qd = qR - C.tdx2 * (Fr.q - Fl.q) - ptil_term;
    const double t = 2.0 * sg - 1.0;
    const double a2 = fma(C.lam3 * sg, 3.0 * sg - 1.0, C.g * hE);
    const double beta = fma(-C.c23 * t, (D * D) * Hd, a2);
    const double delta = (t * (-1.0 / 3.0)) * (hE * D);
    sQd[x] = qd; sHd[x] = Hd; sBe[x] = beta; sDe[x] = delta;
    hR_out = hRp;
    Wd_out = Wd;
    beta_out = beta;
}

// Phase 1 of one isolated row r (rows -1 and T of the tile): faces r -+ 1/2
// from E rows r-2 .. r+2.
template <bool BATHY, bool R_IS_E = false>
__device__ __forceinline__ void cl_single_row(const RowCtx &C, double kap, const double *sB, int r,
                                              const double *sEh, const double *sEq, const double *sEH,
                                              const double *sEW, double *sQd, double *sHd, double *sBe,
                                              double *sDe, bool r_is_e = R_IS_E)
{
    double xh[5], xq[5], xH[5], xW[5];
#pragma unroll
    for (int k = 0; k < 5; k++) {
        const int x = swz(r - 2 + k);
        xh[k] = sEh[x]; xq[k] = sEq[x]; xH[k] = sEH[x]; xW[k] = sEW[x];
    }
    const double ah[3] = {xh[0], xh[1], xh[2]}, aq[3] = {xq[0], xq[1], xq[2]};
    const double aH[3] = {xH[0], xH[1], xH[2]}, aW[3] = {xW[0], xW[1], xW[2]};
    const double bh[3] = {xh[1], xh[2], xh[3]}, bq[3] = {xq[1], xq[2], xq[3]};
    const double bH[3] = {xH[1], xH[2], xH[3]}, bW[3] = {xW[1], xW[2], xW[3]};
    const double ch[3] = {xh[2], xh[3], xh[4]}, cq[3] = {xq[2], xq[3], xq[4]};
    const double cH[3] = {xH[2], xH[3], xH[4]}, cW[3] = {xW[2], xW[3], xW[4]};
    const FState Mm = muscl_minus(ah, aq, aH, aW, kap);       // M_{r-1}
    FState Pl, Mr;
    muscl_pair(bh, bq, bH, bW, kap, Pl, Mr);                  // Pl_r, M_r
    const FState Pn = muscl_plus(ch, cq, cH, cW, kap);        // Pl_{r+1}
    const Face Fl = rusanov(Mm, Pl), Fr = rusanov(Mr, Pn);
    double Wd, hR, beta;
    cl_row_update<BATHY, R_IS_E>(C, sB, r, bh, bq, bH, bW, Fl, Fr, sQd, sHd, sBe, sDe, Wd, beta, hR, r_is_e);
}

#if HSGN_EXP_TIMING
// per-phase clocks of the cluster kernels, summed over CTAs: [stage][mark]
__device__ unsigned long long g_clt[2][16];
#define CL_MARK(k) do { if (tid == 0) tmk[k] = clock64(); } while (0)
#else
#define CL_MARK(k) do { } while (0)
#endif

// PCR buffers (phase 2, in the dead E arrays 1..3): 2 buffers x 5 columns (A, C, D, V, W) of CNT slots
// with PPAD zero slots on either side, so levels of stride <= PPAD need no
// bounds tests (the pads are identity rows: no coupling, zero right-hand side).
constexpr int PPAD = 16;
constexpr int PSTR = CNT + 2 * PPAD;
static_assert(2 * 5 * PSTR <= 3 * CARR, "PCR buffers fit in arrays 1..3");

// Kernel modes.  CLUSTER: the C tiles of a member are one thread-block cluster,
// the separator data travel by DSMEM.  TIPS / FINISH: tile-level SPIKE for
// members of any size (no cluster; C = tiles per member): TIPS computes each
// tile's reduced system and writes its 12 published values to P.sp_tips;
// sep_solve_kernel solves the separator system of every member exactly into
// P.sp_L; FINISH recomputes the tile (identical arithmetic), takes its L values
// from P.sp_L, and finishes the stage; with the A19 filter the two rows at each
// interior tile end are completed by filter_fix_kernel from P.sp_fb.
enum { CL_MODE_CLUSTER = 0, CL_MODE_TIPS = 1, CL_MODE_FINISH = 2 };

// ---------------------------------------------------------------------------
// The cluster stage kernel.  grid = (C, members), cluster = (C, 1, 1).
// STAGE2: inputs U^n and U1 (E, R formed on load); FINAL: this stage produces
// U^{n+1} (filter, dt maxima, time level).  P.T = tile rows (a multiple of
// 4), P.tiles = C; periodic members (both sides periodic) or physical ends
// on both sides.
// ---------------------------------------------------------------------------
template <bool STAGE2, bool FINAL, bool BATHY, int MODE = CL_MODE_CLUSTER>
__global__ void __launch_bounds__(CNT, STAGE2 ? HSGN_CMINB : HSGN_CMINB1) cl_stage_kernel(const Params P, const Bufs B)
{
    constexpr bool CLU = MODE == CL_MODE_CLUSTER;
    double *const sm = hsgn_smem;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#if HSGN_EXP_TIMING
    long long tmk[12] = {};
#endif
    CL_MARK(0);
    const int C = P.tiles;
    const int c = blockIdx.x;                       // == %cluster_ctarank (cluster spans x)
    const int m = blockIdx.y;
    const int n = P.n;
    const size_t mo = size_t(m) * n;
    const int s = c * P.T;
    const int Tc = (c == C - 1) ? n - s : P.T;
    const bool cyc = P.bcl == BC_PERIODIC;
    // slab sides (BC_HALO, tile-level SPIKE only): the neighbouring slab's rows
    // come from the halo buffers, its separators from the slab interface solve
    const bool left_halo = !CLU && c == 0 && P.bcl == BC_HALO;
    const bool right_halo = !CLU && c == C - 1 && P.bcr == BC_HALO;
    const bool left_phys = !cyc && c == 0 && !left_halo, right_phys = !cyc && c == C - 1 && !right_halo;
    const unsigned xmb = (unsigned)__cvta_generic_to_shared(&s_xmb);
    const unsigned xmb2 = (unsigned)__cvta_generic_to_shared(&s_xmb2);
    const unsigned fmb = (unsigned)__cvta_generic_to_shared(&s_fmb);
    double *const A0 = sm, *const A1 = sm + CARR, *const A2 = sm + 2 * CARR, *const A3 = sm + 3 * CARR;
    double *const A4 = sm + 4 * CARR, *const A5 = sm + 5 * CARR, *const A6 = sm + 6 * CARR;
    double *const A7 = sm + 7 * CARR, *const A8 = sm + 8 * CARR;
    const int ks = Tc / CMCH - 1;                     // separator chunk (last row = Tc - 1)
    const bool filt = FINAL && (P.filter_sigma > 0.0);
    // run control first: its latency overlaps the barrier and the tile load
    const double dtm = P.dt[m];
    const double lam = P.lam[m];
    double tm0 = -1.0, tend0 = -1.0;
    if (FINAL && c == 0 && tid == 0) { tm0 = P.t[P.kpar * P.members + m]; tend0 = P.ctrl->t_end; }

    // ---- load.  Thread t owns rows 4t .. 4t+3 (contiguous: two 16-B loads per
    // field, a warp reads 1 KiB contiguous).  E goes to shared memory
    // (swizzled; neighbours' rows are read in phase 1), R stays in registers
    // (only its own rows are used).  Rows -4..-1 and Tc..Tc+3 (halo) come from
    // the neighbouring tiles (periodic: wrapped) by threads 64, 65 (left) and
    // 96, 97 (right), two rows each, or are mirrored at physical ends (A10);
    // R of rows -1 and Tc goes to s_rh for the threads computing those rows.
    if (CLU && tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xmb) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xmb2) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(fmb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        // separator data: XPUB doubles from each of the C CTAs (incl. this one),
        // the parts the three equations c-1, c, c+1 need on xmb, the rest on xmb2
        const unsigned nb = 48u * unsigned(cl_near_count(c, C, cyc, -1) + cl_near_count(c, C, cyc, 0));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(xmb), "r"(nb) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(xmb2),
                     "r"(unsigned(XPUB * C) * 8u - nb) : "memory");
        // filter halo: rows Tc, Tc+1 (q, W) from the right neighbour, -2, -1 from the left
        const unsigned fbytes = filt ? (left_phys ? 0u : 32u) + (right_phys ? 0u : 32u) : 0u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fmb), "r"(fbytes) : "memory");
    }
    const bool wall_l = P.bcl == BC_WALL, wall_r = P.bcr == BC_WALL;
    const int r0 = tid * CMCH;
    const bool live = r0 < Tc;
    {
        const double wE = P.wE, wR = P.wR;
        // rows [r, r+1] of every field at global cell gc (member offset applied);
        // E and R of the two rows (stage 1: R = E); H = K - 1.5 h b (A9)
        auto load2 = [&](size_t gc, double (&e)[4][2], double (&rr)[4][2], double (&bb)[2]) {
            double2 u[4], v[4];
#pragma unroll
            for (int f = 0; f < 4; f++) u[f] = __ldg(reinterpret_cast<const double2 *>(B.Un[f] + gc));
            if (STAGE2) {
#pragma unroll
                for (int f = 0; f < 4; f++) v[f] = __ldg(reinterpret_cast<const double2 *>(B.U1[f] + gc));
            }
            if (BATHY) {
                const double2 b2 = __ldg(reinterpret_cast<const double2 *>(P.b + (gc - mo)));
                bb[0] = b2.x; bb[1] = b2.y;
            } else {
                bb[0] = bb[1] = 0.0;
            }
#pragma unroll
            for (int f = 0; f < 4; f++) {
                const double x0 = u[f].x, x1 = u[f].y;
                if (STAGE2) {     // (1 - w) U^n + w U1 = U^n + w (U1 - U^n)
                    const double d0 = v[f].x - x0, d1 = v[f].y - x1;
                    e[f][0] = fma(wE, d0, x0); e[f][1] = fma(wE, d1, x1);
                    rr[f][0] = fma(wR, d0, x0); rr[f][1] = fma(wR, d1, x1);
                } else {
                    e[f][0] = x0; e[f][1] = x1;
                    rr[f][0] = x0; rr[f][1] = x1;
                }
            }
            if (BATHY) {
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    e[2][k] -= 1.5 * e[0][k] * bb[k];
                    rr[2][k] -= 1.5 * rr[0][k] * bb[k];
                }
            }
        };
        auto putE = [&](int r, double h, double q, double H, double W, double b) {
            const int x = swz(r);
            A0[x] = h; A1[x] = q; A2[x] = H; A3[x] = W;
            if (BATHY) A8[x] = b;
        };
        auto putR = [&](int r, double h, double q, double H, double W) {   // read back by the row's owner
            const int x = swz(r);
            A7[x] = h; A4[x] = q; A5[x] = H; A6[x] = W;
        };
        if (live) {
            double e0[4][2], e1[4][2], q0[4][2], q1[4][2], b0[2], b1[2];
            load2(mo + size_t(s + r0), e0, q0, b0);
            load2(mo + size_t(s + r0 + 2), e1, q1, b1);
            putR(r0, q0[0][0], q0[1][0], q0[2][0], q0[3][0]);
            putR(r0 + 1, q0[0][1], q0[1][1], q0[2][1], q0[3][1]);
            putR(r0 + 2, q1[0][0], q1[1][0], q1[2][0], q1[3][0]);
            putR(r0 + 3, q1[0][1], q1[1][1], q1[2][1], q1[3][1]);
            putE(r0, e0[0][0], e0[1][0], e0[2][0], e0[3][0], b0[0]);
            putE(r0 + 1, e0[0][1], e0[1][1], e0[2][1], e0[3][1], b0[1]);
            putE(r0 + 2, e1[0][0], e1[1][0], e1[2][0], e1[3][0], b1[0]);
            putE(r0 + 3, e1[0][1], e1[1][1], e1[2][1], e1[3][1], b1[1]);
            // physical ends: mirrored ghosts (A10; q odd at walls, copy for transmissive)
            if (tid == 0 && left_phys) {
                const double pq = wall_l ? -1.0 : 1.0;
                double ef[4][4], bf[4];
#pragma unroll
                for (int f = 0; f < 4; f++) { ef[f][0] = e0[f][0]; ef[f][1] = e0[f][1]; ef[f][2] = e1[f][0]; ef[f][3] = e1[f][1]; }
                bf[0] = b0[0]; bf[1] = b0[1]; bf[2] = b1[0]; bf[3] = b1[1];
#pragma unroll
                for (int k = 0; k < 4; k++) {           // row -1-k <- row k (wall) or row 0
                    const int src = wall_l ? k : 0;
                    putE(-1 - k, ef[0][src], pq * ef[1][src], ef[2][src], ef[3][src], bf[src]);
                }
            }
            if (tid == ks && right_phys) {
                const double pq = wall_r ? -1.0 : 1.0;
                double ef[4][4], bf[4];
#pragma unroll
                for (int f = 0; f < 4; f++) { ef[f][0] = e0[f][0]; ef[f][1] = e0[f][1]; ef[f][2] = e1[f][0]; ef[f][3] = e1[f][1]; }
                bf[0] = b0[0]; bf[1] = b0[1]; bf[2] = b1[0]; bf[3] = b1[1];
#pragma unroll
                for (int k = 0; k < 4; k++) {           // row Tc+k <- row Tc-1-k (wall) or Tc-1
                    const int src = wall_r ? 3 - k : 3;
                    putE(Tc + k, ef[0][src], pq * ef[1][src], ef[2][src], ef[3][src], bf[src]);
                }
            }
        }
        // one row of a neighbouring slab (cell index < 0 or >= n): halo buffers
        // [U^n 0..3][U1 4..7][b 8], H cells per side
        auto load1h = [&](int cell, double (&e)[4], double (&rr)[4], double &bb) {
            const bool lft = cell < 0;
            const int o = lft ? cell + P.H : cell - n;
            const double *const *hp = lft ? P.halo_l : P.halo_r;
            bb = BATHY ? hp[8][o] : 0.0;
#pragma unroll
            for (int f = 0; f < 4; f++) {
                const double x0 = hp[f][o];
                if (STAGE2) {
                    const double d0 = hp[4 + f][o] - x0;
                    e[f] = fma(wE, d0, x0); rr[f] = fma(wR, d0, x0);
                } else {
                    e[f] = x0; rr[f] = x0;
                }
            }
            if (BATHY) { e[2] -= 1.5 * e[0] * bb; rr[2] -= 1.5 * rr[0] * bb; }
        };
        // halo rows of interior or periodic tile ends
        const int hs = (tid == 64 || tid == 65) ? 0 : (tid == 96 || tid == 97) ? 1 : -1;
        if (hs == 0 && left_halo) {
            const int rr0 = (tid == 64) ? -4 : -2;
#pragma unroll
            for (int k = 0; k < 2; k++) {
                double e[4], q[4], bb;
                load1h(rr0 + k, e, q, bb);
                putE(rr0 + k, e[0], e[1], e[2], e[3], bb);
                if (rr0 + k == -1) putR(-1, q[0], q[1], q[2], q[3]);
            }
        } else if (hs == 1 && right_halo) {
            const int rr0 = (tid == 96) ? Tc : Tc + 2;
#pragma unroll
            for (int k = 0; k < 2; k++) {
                double e[4], q[4], bb;
                load1h(s + rr0 + k, e, q, bb);
                putE(rr0 + k, e[0], e[1], e[2], e[3], bb);
                if (rr0 + k == Tc) putR(Tc, q[0], q[1], q[2], q[3]);
            }
        } else if (hs == 0 && !left_phys) {
            const int rr0 = (tid == 64) ? -4 : -2;                    // rows rr0, rr0+1
            const int gc = (s + rr0 >= 0) ? s + rr0 : n + s + rr0;    // (periodic wrap: c == 0)
            double e[4][2], q[4][2], bb[2];
            load2(mo + size_t(gc), e, q, bb);
            putE(rr0, e[0][0], e[1][0], e[2][0], e[3][0], bb[0]);
            putE(rr0 + 1, e[0][1], e[1][1], e[2][1], e[3][1], bb[1]);
            if (tid == 65) putR(-1, q[0][1], q[1][1], q[2][1], q[3][1]);
        }
        if (hs == 1 && !right_phys && !right_halo) {
            const int rr0 = (tid == 96) ? Tc : Tc + 2;
            const int gc = (s + rr0 < n) ? s + rr0 : s + rr0 - n;
            double e[4][2], q[4][2], bb[2];
            load2(mo + size_t(gc), e, q, bb);
            putE(rr0, e[0][0], e[1][0], e[2][0], e[3][0], bb[0]);
            putE(rr0 + 1, e[0][1], e[1][1], e[2][1], e[3][1], bb[1]);
            if (tid == 96) putR(Tc, q[0][0], q[1][0], q[2][0], q[3][0]);
        }
    }
    __syncthreads();                                  // E rows; mbarriers initialised
    if (CLU) cl_arrive_relaxed();                     // cluster phase: every CTA has started
    CL_MARK(1);
    CL_MARK(2);
    CL_MARK(3);

    TileAcc acc{0.0, 0.0, 0.0, 0u, 1 << 30, 0};
    if (dtm == 0.0) {                                 // member at t_end: uniform over the cluster
        if (MODE == CL_MODE_TIPS) return;             // (its separators are not used)
        carry_tile<FINAL, BATHY>(P, B, mo, s, s + Tc, lam, acc);
        __syncwarp();
        if (CLU) cl_wait();
        tile_epilogue<FINAL>(P, c, m, dtm, acc, tm0, tend0);
        return;
    }
    const StageC S = stage_consts(P, STAGE2 ? P.aI2 : P.aI1, dtm, lam);
    const double tau = S.tau, g = S.g, idx1 = S.idx1, tdx2 = S.tdx2, t2h = S.t2h, lt2 = S.lt2;
    const double lt2h = S.lt2h, ltdx2 = S.ltdx2, lam3 = S.lam3, ltau = S.ltau;
    const double *const sEh = A0, *const sEq = A1, *const sEH = A2, *const sEW = A3;
    double *const sQd = A4, *const sHd = A5, *const sBe = A6, *const sDe = A7;
    const double *const sB = BATHY ? A8 : nullptr;

    // ---- phase 1: faces, predictor, coefficients ---------------------------
    double wd[CMCH], hRv[CMCH];
    {
        const double kap = P.order == 2 ? 0.25 : 0.0;
        RowCtx Cx{};
        Cx.tau = tau; Cx.tdx2 = tdx2; Cx.t2 = S.t2; Cx.lt2 = lt2; Cx.lam = lam; Cx.lam3 = lam3;
        Cx.ltau = ltau; Cx.g = g; Cx.idx = idx1;
        Cx.c23 = (2.0 / 3.0) * lam * lt2;
        if (tid == 0 && !left_phys)                   // row -1 (previous CTA's last row)
            cl_single_row<BATHY>(Cx, kap, sB, -1, sEh, sEq, sEH, sEW, sQd, sHd, sBe, sDe);
        if (tid == 32 && !right_phys)                 // row Tc (next CTA's first row)
            cl_single_row<BATHY>(Cx, kap, sB, Tc, sEh, sEq, sEH, sEW, sQd, sHd, sBe, sDe);
        if (live) {
            double wh[3], wq[3], wH[3], wW[3];
#pragma unroll
            for (int k = 0; k < 3; k++) {             // rows r0-2 .. r0
                const int x = swz(r0 - 2 + k);
                wh[k] = sEh[x]; wq[k] = sEq[x]; wH[k] = sEH[x]; wW[k] = sEW[x];
            }
            FState Mm = muscl_minus(wh, wq, wH, wW, kap);          // M_{r0-1}
#pragma unroll
            for (int k = 0; k < 2; k++) { wh[k] = wh[k + 1]; wq[k] = wq[k + 1]; wH[k] = wH[k + 1]; wW[k] = wW[k + 1]; }
            {
                const int x = swz(r0 + 1);
                wh[2] = sEh[x]; wq[2] = sEq[x]; wH[2] = sEH[x]; wW[2] = sEW[x];
            }
            FState Pn, Mr;
            muscl_pair(wh, wq, wH, wW, kap, Pn, Mr);               // Pl_{r0}, M_{r0}
            Face Fl = rusanov(Mm, Pn);                             // face r0 - 1/2
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
                    wh[2] = sEh[x]; wq[2] = sEq[x]; wH[2] = sEH[x]; wW[2] = sEW[x];
                }
                FState Mn;
                muscl_pair(wh, wq, wH, wW, kap, Pn, Mn);           // Pl_{r+1}, M_{r+1}
                const Face Fr = rusanov(Mr, Pn);                   // face r + 1/2
                Mr = Mn;
                double beta;
                cl_row_update<BATHY>(Cx, sB, r, ch, cq, cH, cW, Fl, Fr, sQd, sHd, sBe, sDe, wd[i], beta, hRv[i]);
                if (!(beta > 0.0)) acc.err |= ERR_COERC;           // kappa > 0
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
    // physical ends (A10): derived-field ghosts mirrored, the depth coupling
    // across the end cut (beta_{-1} = -beta_0 makes rho_{-1/2} exactly 0)
    if (tid == 0 && left_phys) {
        const int x = swz(-1), y = swz(0);
        sQd[x] = (wall_l ? -1.0 : 1.0) * sQd[y]; sHd[x] = sHd[y]; sDe[x] = sDe[y]; sBe[x] = -sBe[y];
    }
    if (tid == 32 && right_phys) {
        const int x = swz(Tc), y = swz(Tc - 1);
        sQd[x] = (wall_r ? -1.0 : 1.0) * sQd[y]; sHd[x] = sHd[y]; sDe[x] = sDe[y]; sBe[x] = -sBe[y];
    }
    __syncthreads();
    CL_MARK(4);

    // ---- phase 2: assemble + exact solve (A1, A3) ---------------
    // register windows of the derived fields over rows r0-1 .. r0+4 (arrays
    // 4..7 stay intact: phase 3 reads them again; the PCR buffers go to the
    // dead E arrays 1..3)
    double hb[CMCH], hLn, hRn;
    double am[CMCH], cm[CMCH], dm[CMCH];
    {
    double vb[CMCH + 2], vd[CMCH + 2], vH[CMCH + 2], vq[CMCH + 2];
    if (live) {
#pragma unroll
        for (int k = 0; k < CMCH + 2; k++) {
            const int x = swz(r0 - 1 + k);
            vb[k] = sBe[x]; vd[k] = sDe[x]; vH[k] = sHd[x]; vq[k] = sQd[x];
        }
    } else {
#pragma unroll
        for (int k = 0; k < CMCH + 2; k++) { vb[k] = 0.0; vd[k] = 0.0; vH[k] = 0.0; vq[k] = 0.0; }
    }
#pragma unroll
        for (int i = 0; i < CMCH; i++) {
            const double rl = t2h * (vb[i] + vb[i + 1]);              // rho_{r-1/2}
            const double rr = t2h * (vb[i + 1] + vb[i + 2]);          // rho_{r+1/2}
            const double ml = lt2h * (vd[i] + vd[i + 1]);             // mu (A1)
            const double mr = lt2h * (vd[i + 1] + vd[i + 2]);
            const double rhs = hRv[i] - tdx2 * (vq[i + 2] - vq[i]) + mr * (vH[i + 2] - vH[i + 1])
                               - ml * (vH[i + 1] - vH[i]);
            const double a = -rl, cc = -rr, dg = 1.0 + rl + rr;
            if (i == 0) {
                const double inv = rcp(dg);
                am[0] = a * inv; cm[0] = cc * inv; dm[0] = rhs * inv;
            } else {
                const double inv = rcp(dg - a * cm[i - 1]);
                am[i] = -a * am[i - 1] * inv;
                cm[i] = cc * inv;
                dm[i] = (rhs - a * dm[i - 1]) * inv;
            }
        }
    }
    {
        // chunk-end relation: X_k + aE X_{k-1} + cE x_{next first} = dE;
        // upward: x_i = P_i - Q_i X_{k-1} - R_i X_k (stored in dm, am, cm)
        const double aE = am[CMCH - 1], cE = cm[CMCH - 1], dE = dm[CMCH - 1];
        {
            double Pn = 0.0, Qn = 0.0, Rn = -1.0;
#pragma unroll
            for (int i = CMCH - 2; i >= 0; i--) {
                const double Pi = dm[i] - cm[i] * Pn;
                const double Qi = am[i] - cm[i] * Qn;
                const double Ri = -cm[i] * Rn;
                dm[i] = Pi; am[i] = Qi; cm[i] = Ri;
                Pn = Pi; Qn = Qi; Rn = Ri;
            }
        }
        double P1 = __shfl_down_sync(0xffffffffu, dm[0], 1);
        double Q1 = __shfl_down_sync(0xffffffffu, am[0], 1);
        double R1 = __shfl_down_sync(0xffffffffu, cm[0], 1);
        if (lane == 0) { s_cw[wid][0] = dm[0]; s_cw[wid][1] = am[0]; s_cw[wid][2] = cm[0]; }
        __syncthreads();                              // (also: all window loads of arrays 4..7 done)
        if (lane == 31) {
            if (wid + 1 < CNT / 32) { P1 = s_cw[wid + 1][0]; Q1 = s_cw[wid + 1][1]; R1 = s_cw[wid + 1][2]; }
            else { P1 = 0.0; Q1 = 0.0; R1 = 0.0; }
        }
        // reduced row of chunk end k: A X_{k-1} + X_k + C X_{k+1} = D (normalised)
        double A_ = aE, C_ = -cE * R1, D_ = dE - cE * P1, V_ = 0.0, W_ = 0.0;
        {
            const double ib = rcp(1.0 - cE * Q1);
            A_ *= ib; C_ *= ib; D_ *= ib;
        }
        if (tid == 0) { V_ = A_; A_ = 0.0; }          // coupling to L_{j-1}: right-hand side V
        if (tid == ks - 1) { W_ = C_; C_ = 0.0; }     // coupling to L_j: right-hand side W
        if (tid >= ks) { A_ = 0.0; C_ = 0.0; D_ = 0.0; V_ = 0.0; W_ = 0.0; }   // separator, dead
        double *const pb0 = A1 + PPAD, *const pb1 = A1 + 5 * PSTR + PPAD;       // slot k at [k]
        auto put = [&](double *b, int k, double a, double cc, double d, double v, double w_) {
            b[k] = a; b[PSTR + k] = cc; b[2 * PSTR + k] = d; b[3 * PSTR + k] = v; b[4 * PSTR + k] = w_;
        };
        put(pb0, tid, A_, C_, D_, V_, W_);
        if (tid < 2 * PPAD) {                         // zero pads (identity rows) of both buffers
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
            if (e0 < 0.4f) {     // PCR stop once e^(2^s) <= 2^-64 (see stage_body)
                const float q = __fdividef(64.0f, -__log2f(e0) - 0.28f);
                const int qi = int(ceilf(q));
                lim = qi <= 1 ? 1 : min(CNT, 1 << (32 - __clz(qi - 1)));
            }
        }
        // one PCR level at stride sd, cur -> nxt (pads: no bounds tests for sd <= PPAD)
        auto level = [&](const int sd, const double *cur, double *nxt) {
            int km = tid - sd, kp = tid + sd;
            const bool okm = sd <= PPAD || km >= 0, okp = sd <= PPAD || kp < CNT;
            km = okm ? km : 0; kp = okp ? kp : 0;
            double Am = cur[km], Cm = cur[PSTR + km], Dm = cur[2 * PSTR + km];
            double Vm = cur[3 * PSTR + km], Wm = cur[4 * PSTR + km];
            double Ap = cur[kp], Cp = cur[PSTR + kp], Dp = cur[2 * PSTR + kp];
            double Vp = cur[3 * PSTR + kp], Wp = cur[4 * PSTR + kp];
            if (sd > PPAD) {
                if (!okm) { Am = Cm = Dm = Vm = Wm = 0.0; }
                if (!okp) { Ap = Cp = Dp = Vp = Wp = 0.0; }
            }
            const double ib = rcp(1.0 - A_ * Cm - C_ * Ap);
            const double An = -A_ * Am * ib, Cn = -C_ * Cp * ib;
            D_ = (D_ - A_ * Dm - C_ * Dp) * ib;
            V_ = (V_ - A_ * Vm - C_ * Vp) * ib;
            W_ = (W_ - A_ * Wm - C_ * Wp) * ib;
            A_ = An; C_ = Cn;
            put(nxt, tid, A_, C_, D_, V_, W_);
            __syncthreads();
        };
        static_assert(CNT == 128, "PCR levels below are written out for 128 unknowns");
        const double *fin = pb0;                      // buffer holding the final (Y, V, W)
        if (lim > 1) { level(1, pb0, pb1); fin = pb1; }
        if (lim > 2) { level(2, pb1, pb0); fin = pb0; }
        if (lim > 4) { level(4, pb0, pb1); fin = pb1; }
        if (lim > 8) { level(8, pb1, pb0); fin = pb0; }
        if (lim > 16) { level(16, pb0, pb1); fin = pb1; }
        if (lim > 32) { level(32, pb1, pb0); fin = pb0; }
        if (lim > 64) { level(64, pb0, pb1); fin = pb1; }
        // (Y, V, W) of the neighbouring slots, read before the exchange: after it
        // the neighbours' filter halo rows may land in arrays 2, 3
        const double Yl = fin[2 * PSTR + tid - 1], Vl = fin[3 * PSTR + tid - 1], Wl = fin[4 * PSTR + tid - 1];
        const double Yr = fin[2 * PSTR + tid + 1], Vr = fin[3 * PSTR + tid + 1], Wr = fin[4 * PSTR + tid + 1];
        const double Yks = fin[2 * PSTR + ks - 1], Vks = fin[3 * PSTR + ks - 1], Wks = fin[4 * PSTR + ks - 1];
        CL_MARK(5);
        const int cp_ = (c + 1 < C) ? c + 1 : 0, cm_ = (c > 0) ? c - 1 : C - 1;
        double Lm = 0.0, Lc, Lp = 0.0;
        double nx[6];                                 // the next tile's left part (P1, Q1, R1, Y0, V0, W0)
        if constexpr (MODE == CL_MODE_TIPS) {
            // publish to global memory: the same 12 values as the DSMEM exchange
            double *const tp = P.sp_tips + (size_t(m) * C + c) * XPUB;
            if (tid == 0) { tp[6] = dm[0]; tp[7] = am[0]; tp[8] = cm[0]; tp[9] = D_; tp[10] = V_; tp[11] = W_; }
            if (tid == ks) { tp[0] = aE; tp[1] = cE; tp[2] = dE; tp[3] = Yks; tp[4] = Vks; tp[5] = Wks; }
            return;
        } else if constexpr (MODE == CL_MODE_FINISH) {
            const double *const Lv = P.sp_L + size_t(m) * C;
            Lc = Lv[c];
            if (left_halo) Lm = P.sx_elfr[2 * m];                 // E_{p-1}: left slab's last separator
            else if (c > 0 || cyc) Lm = Lv[cm_];
            if (right_halo) Lp = P.sx_elfr[2 * m + 1];            // F_{p+1}: right slab's first separator
            else if (c + 1 < C || cyc) Lp = Lv[cp_];
            const double *const tn = right_halo ? P.sx_nx + size_t(m) * 6
                                                : P.sp_tips + (size_t(m) * C + cp_) * XPUB + 6;
#pragma unroll
            for (int k = 0; k < 6; k++) nx[k] = tn[k];
        } else {
        // publish (DSMEM, st.async): warp 0 sends the first-row relation of chunk 0
        // and (Y, V, W) of slot 0 (what the previous CTA's separator row needs);
        // the warp of thread ks sends the raw reduced row of the separator chunk
        // and (Y, V, W) of slot ks-1 -- to every CTA of the cluster
        cl_wait();                                    // every CTA of the cluster has started
        if (wid == 0 || wid == (ks >> 5)) {
            double v6[6];
            if (wid == 0) {
                v6[0] = __shfl_sync(0xffffffffu, dm[0], 0); v6[1] = __shfl_sync(0xffffffffu, am[0], 0);
                v6[2] = __shfl_sync(0xffffffffu, cm[0], 0); v6[3] = __shfl_sync(0xffffffffu, D_, 0);
                v6[4] = __shfl_sync(0xffffffffu, V_, 0); v6[5] = __shfl_sync(0xffffffffu, W_, 0);
                for (int i = lane; i < 6 * C; i += 32) {
                    const int rk = i / 6, k = i - rk * 6;
                    const bool nr = cl_is_near(c, rk, C, cyc, 0);       // left part: receivers c-2 .. c
                    st_remote(&s_cx[c][6 + k], nr ? (const void *)&s_xmb : (const void *)&s_xmb2, unsigned(rk),
                              cl_pick6(v6, k));
                }
            }
            if (wid == (ks >> 5)) {
                const int ls = ks & 31;
                v6[0] = __shfl_sync(0xffffffffu, aE, ls); v6[1] = __shfl_sync(0xffffffffu, cE, ls);
                v6[2] = __shfl_sync(0xffffffffu, dE, ls);
                v6[3] = Yks; v6[4] = Vks; v6[5] = Wks;
                for (int i = lane; i < 6 * C; i += 32) {
                    const int rk = i / 6, k = i - rk * 6;
                    const bool nr = cl_is_near(c, rk, C, cyc, -1);      // own part: receivers c-1 .. c+1
                    st_remote(&s_cx[c][k], nr ? (const void *)&s_xmb : (const void *)&s_xmb2, unsigned(rk),
                              cl_pick6(v6, k));
                }
            }
        }
        mbar_wait(xmb, 0u);                           // the data of equations c-1, c, c+1
        CL_MARK(6);
        // separator equation j (lane-independent helper): coefficients of
        // L_{j-1}, L_j, L_{j+1}, normalised by the diagonal
        auto sep_eq = [&](int j, double &a, double &cc, double &d) {
            const int jn = (j + 1 < C) ? j + 1 : (cyc ? 0 : -1);
            const double aEj = s_cx[j][0], cEj = s_cx[j][1], dEj = s_cx[j][2];
            const double Yp = s_cx[j][3], Vp = s_cx[j][4], Wp = s_cx[j][5];
            double P1n = 0, Q1n = 0, R1n = 0, Y0 = 0, V0 = 0, W0 = 0;
            if (jn >= 0) {
                P1n = s_cx[jn][6]; Q1n = s_cx[jn][7]; R1n = s_cx[jn][8];
                Y0 = s_cx[jn][9]; V0 = s_cx[jn][10]; W0 = s_cx[jn][11];
            }
            const double cr = cEj * R1n;
            const double sub = -aEj * Vp;
            const double dia = (1.0 - cEj * Q1n) - aEj * Wp + cr * V0;
            const double sup = cr * W0;
            const double rhs = dEj - cEj * P1n - aEj * Yp + cr * Y0;
            const double id = rcp(dia);
            a = sub * id; cc = sup * id; d = rhs * id;
        };
        {
            // the couplings of neighbouring separators go through the spike tips
            // (~ r^T): usually equations c-1, c, c+1 are decoupled to round-off
            // (the in-CTA PCR's stop test, 2^-64): then L_j = d_j; otherwise all
            // C equations are solved by PCR over the lanes of every warp
            double a = 0.0, cc = 0.0, d = 0.0;
            const int jj = lane == 0 ? cm_ : lane == 1 ? c : cp_;
            const bool has = lane < 3 && (lane == 1 || cyc || (lane == 0 ? c > 0 : c + 1 < C));
            if (has) sep_eq(jj, a, cc, d);
            const bool dec = __all_sync(0xffffffffu, fabs(a) <= 5.421010862427522e-20 &&
                                                         fabs(cc) <= 5.421010862427522e-20);   // 2^-64
            if (dec) {
                Lm = __shfl_sync(0xffffffffu, d, 0);
                Lc = __shfl_sync(0xffffffffu, d, 1);
                Lp = __shfl_sync(0xffffffffu, d, 2);
                if (!(c > 0 || cyc)) Lm = 0.0;
            } else {
                mbar_wait(xmb2, 0u);                  // every CTA's data
                a = cc = d = 0.0;
                const int j = lane;
                if (j < C) sep_eq(j, a, cc, d);
                for (int sd = 1; sd < C; sd <<= 1) {
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
                // cyclic: the last level couples each row to itself (stride C == 0 mod C)
                const double Lj = cyc ? d * rcp(1.0 + a + cc) : d;
                Lm = (c > 0 || cyc) ? __shfl_sync(0xffffffffu, Lj, cm_) : 0.0;
                Lc = __shfl_sync(0xffffffffu, Lj, c);
                Lp = __shfl_sync(0xffffffffu, Lj, cp_);
            }
        }
#pragma unroll
        for (int k = 0; k < 6; k++) nx[k] = s_cx[cp_][6 + k];
        }
        // chunk ends: X_k = Y_k - V_k L_{j-1} - W_k L_j (interior), X_ks = L_j
        const double Xk = tid < ks ? D_ - V_ * Lm - W_ * Lc : (tid == ks ? Lc : 0.0);
        const double XL = tid == 0 ? Lm : Yl - Vl * Lm - Wl * Lc;
        const double XR = tid + 1 == ks ? Lc : Yr - Vr * Lm - Wr * Lc;
        if (live) {
#pragma unroll
            for (int i = 0; i < CMCH; i++) hb[i] = (i == CMCH - 1) ? Xk : dm[i] - am[i] * XL - cm[i] * Xk;
            // hbar of rows r0-1 (= X_{k-1}) and r0+4 (first row of the next chunk,
            // or of the next CTA: from its published relation)
            hLn = left_phys && tid == 0 ? hb[0] : XL;          // Neumann hbar_{-1} := hbar_0
            if (tid < ks) {
                hRn = P1 - Q1 * Xk - R1 * XR;
            } else if (right_phys) {
                hRn = hb[CMCH - 1];                             // Neumann hbar_Tc := hbar_{Tc-1}
            } else {
                const double X0n = nx[3] - nx[4] * Lc - nx[5] * Lp;
                hRn = nx[0] - nx[1] * Lc - nx[2] * X0n;
            }
        } else {
#pragma unroll
            for (int i = 0; i < CMCH; i++) hb[i] = 1.0;
            hLn = hRn = 1.0;
        }
    }
    acc.rho = fmax(acc.rho, S.t2 * __hiloint2double(acc.bhi + 1, 0));
    CL_MARK(7);

    // ---- phase 3: back-substitution, own rows -------------------
    double qbv[CMCH], HdD[CMCH], Wbv[CMCH], bbv[CMCH], ihv[CMCH];
    double vb[CMCH + 2], vd[CMCH + 2], vH[CMCH + 2], vq[CMCH + 2];
#pragma unroll
    for (int k = 0; k < CMCH + 2; k++) {
        const int x = swz(r0 - 1 + k);
        vb[k] = sBe[x]; vd[k] = sDe[x]; vH[k] = sHd[x]; vq[k] = sQd[x];
    }
#pragma unroll
    for (int i = 0; i < CMCH; i++) {
        const int r = r0 + i;
        bbv[i] = 0.0;
        const double h0 = hb[i];
        const double hl = (i > 0) ? hb[i - 1] : hLn;
        const double hr = (i < CMCH - 1) ? hb[i + 1] : hRn;
        double qb = vq[i + 1] - tdx2 * vb[i + 1] * (hr - hl) - ltdx2 * vd[i + 1] * (vH[i + 2] - vH[i]);
        if (BATHY && live) {
            const double bm = sB[swz(r - 1)], bp = sB[swz(r + 1)];
            bbv[i] = sB[swz(r)];
            qb -= tau * g * sEh[swz(r)] * (bp - bm) * (0.5 * idx1);     // A9
        }
        // Hbar = H^dag hbar^2/(hbar^2 + lam tau^2), Wbar; final
        // stage: Z = 1/(hbar (hbar^2 + lam tau^2)) also gives 1/hbar
        const double den = h0 * h0 + lt2;
        double rden;
        if (FINAL) {
            const double Z = rcp(h0 * den);
            rden = h0 * Z;
            ihv[i] = den * Z;
        } else {
            rden = rcp(den);
            ihv[i] = 0.0;
        }
        HdD[i] = vH[i + 1] * rden;
        qbv[i] = qb;
        Wbv[i] = wd[i] - ltau * HdD[i];
        if (live) {
            if (!(h0 > P.h_min)) acc.err |= ERR_DRY;
            if (!isfinite(h0 + qb + HdD[i] + Wbv[i])) acc.err |= ERR_NONFINITE;
        }
    }
    // FINISH mode with the filter: the two rows at an interior tile end need the
    // neighbouring tile's rows -- filter_fix_kernel completes them (and their dt
    // maxima); here they stay unfiltered
    auto fix_row = [&](int i) -> bool {
        return !CLU && filt && ((tid == 0 && i < 2 && !left_phys) || (tid == ks && i >= 2 && !right_phys));
    };
    if (filt) {
        // A19 on q, W: own rows into A2 (q), A3 (W); rows -2, -1, Tc, Tc+1 from
        // the neighbouring CTAs (DSMEM) or mirrored at physical ends (A10)
        double *const sQb = A2, *const sWb = A3;
        if (live) {
#pragma unroll
            for (int i = 0; i < CMCH; i++) { sQb[swz(r0 + i)] = qbv[i]; sWb[swz(r0 + i)] = Wbv[i]; }
        }
        if (tid == 0) {                               // rows 0, 1 -> left neighbour's Tl, Tl+1
            if (left_phys) {
                const double pq = wall_l ? -1.0 : 1.0;
                sQb[swz(-1)] = pq * qbv[0]; sWb[swz(-1)] = Wbv[0];
                sQb[swz(-2)] = wall_l ? pq * qbv[1] : qbv[0]; sWb[swz(-2)] = wall_l ? Wbv[1] : Wbv[0];
            } else if (!CLU) {                        // FINISH: rows 0..3 for filter_fix_kernel
                double *const fb = P.sp_fb + (size_t(m) * C + c) * 16;
#pragma unroll
                for (int i = 0; i < CMCH; i++) { fb[i] = qbv[i]; fb[4 + i] = Wbv[i]; }
            } else {
                const int cl_ = (c > 0) ? c - 1 : C - 1;
                const int Tl = (cl_ == C - 1) ? n - (C - 1) * P.T : P.T;
                st_remote(sQb + swz(Tl), &s_fmb, cl_, qbv[0]);
                st_remote(sWb + swz(Tl), &s_fmb, cl_, Wbv[0]);
                st_remote(sQb + swz(Tl + 1), &s_fmb, cl_, qbv[1]);
                st_remote(sWb + swz(Tl + 1), &s_fmb, cl_, Wbv[1]);
            }
        }
        if (tid == ks) {                              // rows Tc-2, Tc-1 -> right neighbour's -2, -1
            if (right_phys) {
                const double pq = wall_r ? -1.0 : 1.0;
                sQb[swz(Tc)] = pq * qbv[3]; sWb[swz(Tc)] = Wbv[3];
                sQb[swz(Tc + 1)] = wall_r ? pq * qbv[2] : qbv[3]; sWb[swz(Tc + 1)] = wall_r ? Wbv[2] : Wbv[3];
            } else if (!CLU) {                        // FINISH: rows Tc-4..Tc-1
                double *const fb = P.sp_fb + (size_t(m) * C + c) * 16 + 8;
#pragma unroll
                for (int i = 0; i < CMCH; i++) { fb[i] = qbv[i]; fb[4 + i] = Wbv[i]; }
            } else {
                const int cr_ = (c + 1 < C) ? c + 1 : 0;
                st_remote(sQb + swz(-2), &s_fmb, cr_, qbv[2]);
                st_remote(sWb + swz(-2), &s_fmb, cr_, Wbv[2]);
                st_remote(sQb + swz(-1), &s_fmb, cr_, qbv[3]);
                st_remote(sWb + swz(-1), &s_fmb, cr_, Wbv[3]);
            }
        }
        __syncthreads();                              // own rows and mirrored ghosts
        if (CLU) mbar_wait(fmb, 0u);                  // neighbours' rows
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
                if (fix_row(i)) continue;             // FINISH: completed by filter_fix_kernel
                // f_i - (sigma/16)(f_{i-2} - 4 f_{i-1} + 6 f_i - 4 f_{i+1} + f_{i+2})
                qbv[i] = xq[i + 2] - sig16 * (xq[i] - 4.0 * xq[i + 1] + 6.0 * xq[i + 2] - 4.0 * xq[i + 3] + xq[i + 4]);
                Wbv[i] = xw[i + 2] - sig16 * (xw[i] - 4.0 * xw[i + 1] + 6.0 * xw[i + 2] - 4.0 * xw[i + 3] + xw[i + 4]);
                if (!isfinite(qbv[i] + Wbv[i])) acc.err |= ERR_NONFINITE;
            }
        }
    }
    CL_MARK(8);
    // final values, dt maxima, direct 16-B stores of the own rows
    if (live) {
        double oh[CMCH], oK[CMCH];
#pragma unroll
        const bool relax = FINAL && (P.gen_rate > 0.0 || P.sp_rate > 0.0);
        const double t_new = relax ? P.t[P.kpar * P.members + m] + dtm : 0.0;
        for (int i = 0; i < CMCH; i++) {
            double h0 = hb[i];
            const double Hb = HdD[i] * (h0 * h0);
            double Ko = BATHY ? Hb + 1.5 * h0 * bbv[i] : Hb;
            if (relax && !fix_row(i)) {
                // A10 relaxation zones at t^{n+1}, after the filter
                relax_cell(P, P.x_min + (double(s + r0 + i) + 0.5) * P.dx, bbv[i], t_new, h0, qbv[i], Ko, Wbv[i]);
                const double ih = rcp(h0);
                const double u = fabs(qbv[i] * ih), sg = (Ko - 1.5 * h0 * bbv[i]) * ih * ih;
                const double nu = u + fsqrt(g * h0 + lam3 * sg * sg);
                acc.umax = u > acc.umax ? u : acc.umax;
                acc.numax = nu > acc.numax ? nu : acc.numax;
            } else if (FINAL && !fix_row(i)) {
                const double u = fabs(qbv[i] * ihv[i]), sg = HdD[i];
                const double nu = u + fsqrt(g * h0 + lam3 * sg * sg);
                acc.umax = u > acc.umax ? u : acc.umax;
                acc.numax = nu > acc.numax ? nu : acc.numax;
            }
            oh[i] = h0;
            oK[i] = Ko;
        }
        const size_t gd = mo + size_t(s + r0);
        double2 *const o0 = reinterpret_cast<double2 *>(B.out[0] + gd);
        double2 *const o1 = reinterpret_cast<double2 *>(B.out[1] + gd);
        double2 *const o2 = reinterpret_cast<double2 *>(B.out[2] + gd);
        double2 *const o3 = reinterpret_cast<double2 *>(B.out[3] + gd);
        o0[0] = make_double2(oh[0], oh[1]); o0[1] = make_double2(oh[2], oh[3]);
        o1[0] = make_double2(qbv[0], qbv[1]); o1[1] = make_double2(qbv[2], qbv[3]);
        o2[0] = make_double2(oK[0], oK[1]); o2[1] = make_double2(oK[2], oK[3]);
        o3[0] = make_double2(Wbv[0], Wbv[1]); o3[1] = make_double2(Wbv[2], Wbv[3]);
    }
    CL_MARK(9);
    tile_epilogue<FINAL>(P, c, m, dtm, acc, tm0, tend0);
    if (CLU) mbar_wait(xmb2, 0u);                     // no remote store may target an exited CTA
#if HSGN_EXP_TIMING
    CL_MARK(10);
    if (tid == 0) {
        unsigned long long *gg = g_clt[STAGE2 ? 1 : 0];
        for (int k = 1; k <= 10; k++) atomicAdd(gg + k - 1, (unsigned long long)(tmk[k] - tmk[k - 1]));
        atomicAdd(gg + 15, 1ull);
    }
#endif
}

}  // namespace hsgn

namespace hsgn {

// ---------------------------------------------------------------------------
// Tile-level SPIKE, step 2: the separator system of every member (one CTA per
// member), from the tiles' published values (P.sp_tips, CL_MODE_TIPS):
//     -a V' L_{j-1} + (B - a W' + c R1 V0) L_j + c R1 W0 L_{j+1}
//        = d - c P1 - a Y' + c R1 Y0                        (j = 0 .. G-1)
// (the same equations as the cluster kernel's; cyclic for periodic members),
// solved exactly by the same scheme one level up: thread chunks of separators
// eliminated sequentially (partition method, per-row relations in P.sp_S),
// the chunk ends by PCR with two spike columns, the last chunk end (L_{G-1})
// as the block's single separator.  Writes L to P.sp_L.
// ---------------------------------------------------------------------------
// nxr: the right slab's tile-0 relation (P1, Q1, R1, Y0, V0, W0) for the last
// equation of a slab with a BC_HALO right side (else NULL).  Non-cyclic
// members: the outer couplings a_0 L_{-1}, c_{G-1} L_G are dropped (exactly 0 at
// physical ends); slabs carry them as the spike columns of the right-hand
// side: mode 1 -> d = a_0 e_0 (V), mode 2 -> d = c_{G-1} e_{G-1} (W), mode 0 -> Y.
__device__ __forceinline__ void sep_equation(const double *tips, int G, bool cyc, int j, double &a, double &cc,
                                             double &d, const double *nxr = nullptr, int mode = 0)
{
    const double *o = tips + size_t(j) * XPUB;
    const int jn = (j + 1 < G) ? j + 1 : (cyc ? 0 : -1);
    double P1n = 0, Q1n = 0, R1n = 0, Y0 = 0, V0 = 0, W0 = 0;
    const double *l = jn >= 0 ? tips + size_t(jn) * XPUB + 6 : nxr;
    if (l) {
        P1n = l[0]; Q1n = l[1]; R1n = l[2]; Y0 = l[3]; V0 = l[4]; W0 = l[5];
    }
    const double aEj = o[0], cEj = o[1], dEj = o[2], Yp = o[3], Vp = o[4], Wp = o[5];
    const double cr = cEj * R1n;
    const double sub = -aEj * Vp;
    const double dia = (1.0 - cEj * Q1n) - aEj * Wp + cr * V0;
    const double sup = cr * W0;
    const double rhs = dEj - cEj * P1n - aEj * Yp + cr * Y0;
    const double id = rcp(dia);
    a = sub * id; cc = sup * id; d = rhs * id;
    if (mode == 1) d = (j == 0) ? a : 0.0;
    else if (mode == 2) d = (j == G - 1) ? cc : 0.0;
    if (!cyc) {
        if (j == 0) a = 0.0;
        if (j == G - 1) cc = 0.0;
    }
}

// NTS threads: 128, or 1024 for members of more than 1024 tiles (8x shorter
// sequential chunk sweeps); the PCR buffers (2 x 5 x (NTS + 2 PPAD) doubles)
// are dynamic shared memory (sep_smem_bytes).  With 1024 threads the equations'
// (a, c, d) come from sep_coef_kernel (all SMs) and both they and the sweep
// relations are stored chunk-transposed, [field][i][thread] with thread chunk
// i-th separator j = thread * mch + i, so that every sweep access of a warp is
// coalesced (strided per-thread chunks cost 32 L1 wavefronts per load on the
// one SM that runs the block).
constexpr size_t sep_smem_bytes(int nts) { return size_t(2) * 5 * (nts + 2 * PPAD) * sizeof(double); }
__host__ __device__ constexpr size_t sep_scratch(int G)          // doubles per member (P.sp_S)
{
    return G > 1024 ? size_t(6) * ((G + 1023) / 1024) * 1024 : size_t(3) * G;
}

__device__ __forceinline__ const double *sep_nxr(const Params &P, int m)
{
    return P.bcr == BC_HALO ? P.sx_nx + size_t(m) * 6 : nullptr;
}

__global__ void __launch_bounds__(256) sep_coef_kernel(const Params P, const int mode)
{
    const int m = blockIdx.y;
    const int G = P.tiles;
    const int j = blockIdx.x * 256 + threadIdx.x;
    if (j >= G) return;
    const int mch = (G + 1023) / 1024, t = j / mch, i = j - t * mch;
    double a, cc, d;
    sep_equation(P.sp_tips + size_t(m) * G * XPUB, G, P.bcl == BC_PERIODIC, j, a, cc, d, sep_nxr(P, m), mode);
    double *const abc = P.sp_S + size_t(m) * sep_scratch(G) + size_t(3) * mch * 1024;
    abc[(size_t(0) * mch + i) * 1024 + t] = a;
    abc[(size_t(1) * mch + i) * 1024 + t] = cc;
    abc[(size_t(2) * mch + i) * 1024 + t] = d;
}

// mode 0: the separators L (or Y for a slab), 1 / 2: the slab spike columns V / W
// (see sep_equation); out: [members][G] (NULL: P.sp_L)
template <int NTS>
__global__ void __launch_bounds__(NTS) sep_solve_kernel(const Params P, const int mode, double *out)
{
    constexpr int SSTR = NTS + 2 * PPAD;              // PCR array stride
    __shared__ double sw[NTS / 32][3];
    __shared__ float sred[NTS / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int m = blockIdx.x;
    const int G = P.tiles;
    const bool cyc = P.bcl == BC_PERIODIC;
    const double *const tips = P.sp_tips + size_t(m) * G * XPUB;
    double *const Lout = (out ? out : P.sp_L) + size_t(m) * G;
    const double *const nxr = sep_nxr(P, m);
    double *const S = P.sp_S + size_t(m) * sep_scratch(G);
    if (G == 1) {                                     // one tile: its separator couples to itself
        if (tid == 0) {
            double a, cc, d;
            sep_equation(tips, G, cyc, 0, a, cc, d, nxr, mode);
            Lout[0] = cyc ? d * rcp(1.0 + a + cc) : d;
        }
        return;
    }
    const int mch = (G + NTS - 1) / NTS;              // separators per thread chunk
    const int ta = (G + mch - 1) / mch;               // active chunks (>= 2)
    const int ks = ta - 1;                            // the block's separator chunk
    const int j0 = tid * mch, j1 = min(G, j0 + mch);
    const bool live = tid < ta;
    // relation f of separator j (f = 0, 1, 2), and equation j: chunk-transposed for NTS = 1024
    auto Sx = [&](int f, int j) -> double & {
        return NTS == 1024 ? S[(size_t(f) * mch + (j - j0)) * NTS + tid] : S[3 * size_t(j) + f];
    };
    auto eq = [&](int j, double &a, double &cc, double &d) {
        if (NTS == 1024) {
            const double *const abc = S + size_t(3) * mch * NTS;
            const size_t o = size_t(j - j0) * NTS + tid;
            a = abc[o]; cc = abc[size_t(mch) * NTS + o]; d = abc[2 * size_t(mch) * NTS + o];
        } else {
            sep_equation(tips, G, cyc, j, a, cc, d, nxr, mode);
        }
    };
    // forward sweep: x_i + am_i X_{k-1} + cm_i x_{i+1} = dm_i
    double am = 0.0, cm = 0.0, dm = 0.0;
    if (live) {
        for (int j = j0; j < j1; j++) {
            double a, cc, d;
            eq(j, a, cc, d);
            if (j == j0) {
                am = a; cm = cc; dm = d;
            } else {
                const double inv = rcp(1.0 - a * cm);
                am = -a * am * inv;
                cm = cc * inv;
                dm = (d - a * dm) * inv;
            }
            Sx(0, j) = am; Sx(1, j) = cm; Sx(2, j) = dm;
        }
    }
    const double aE = am, cE = cm, dE = dm;
    // upward: x_i = P_i - Q_i X_{k-1} - R_i X_k (X_k = x_{j1-1})
    double P0 = 0.0, Q0 = 0.0, R0 = 0.0;
    if (live) {
        double Pn = 0.0, Qn = 0.0, Rn = -1.0;
        Sx(0, j1 - 1) = 0.0; Sx(1, j1 - 1) = 0.0; Sx(2, j1 - 1) = -1.0;
        for (int j = j1 - 2; j >= j0; j--) {
            const double a_ = Sx(0, j), c_ = Sx(1, j), d_ = Sx(2, j);
            const double Pi = d_ - c_ * Pn, Qi = a_ - c_ * Qn, Ri = -c_ * Rn;
            Sx(0, j) = Pi; Sx(1, j) = Qi; Sx(2, j) = Ri;
            Pn = Pi; Qn = Qi; Rn = Ri;
        }
        P0 = Pn; Q0 = Qn; R0 = Rn;
        if (j1 - j0 == 1) { P0 = 0.0; Q0 = 0.0; R0 = -1.0; }
    }
    // the next chunk's first-row relation (thread ks: chunk 0's, the cyclic wrap)
    double P1 = __shfl_down_sync(0xffffffffu, P0, 1), Q1 = __shfl_down_sync(0xffffffffu, Q0, 1);
    double R1 = __shfl_down_sync(0xffffffffu, R0, 1);
    if (lane == 0) { sw[wid][0] = P0; sw[wid][1] = Q0; sw[wid][2] = R0; }
    __syncthreads();
    if (lane == 31) {
        if (wid + 1 < NTS / 32) { P1 = sw[wid + 1][0]; Q1 = sw[wid + 1][1]; R1 = sw[wid + 1][2]; }
        else { P1 = Q1 = R1 = 0.0; }
    }
    const double P00 = sw[0][0], Q00 = sw[0][1], R00 = sw[0][2];     // chunk 0's first-row relation
    double A_ = aE, C_ = -cE * R1, D_ = dE - cE * P1, V_ = 0.0, W_ = 0.0;
    {
        const double ib = rcp(1.0 - cE * Q1);
        A_ *= ib; C_ *= ib; D_ *= ib;
    }
    if (tid == 0) { V_ = A_; A_ = 0.0; }              // coupling to the separator (cyclic wrap)
    if (tid == ks - 1) { W_ = C_; C_ = 0.0; }         // coupling to the separator
    if (tid >= ks) { A_ = C_ = D_ = V_ = W_ = 0.0; }
    double *const b0 = hsgn_smem + PPAD, *const b1 = hsgn_smem + 5 * SSTR + PPAD;
    auto put = [&](double *b, int k, double a, double cc, double d, double v, double w_) {
        b[k] = a; b[SSTR + k] = cc; b[2 * SSTR + k] = d; b[3 * SSTR + k] = v; b[4 * SSTR + k] = w_;
    };
    put(b0, tid, A_, C_, D_, V_, W_);
    if (tid < 2 * PPAD) {
        const int k = tid < PPAD ? tid - PPAD : NTS + tid - PPAD;
        put(b0, k, 0.0, 0.0, 0.0, 0.0, 0.0);
        put(b1, k, 0.0, 0.0, 0.0, 0.0, 0.0);
    }
    {
        const float ea = float(fabs(A_)), ec = float(fabs(C_));
        const float ev = warp_max_nonneg(ea > ec ? ea : ec);
        if (lane == 0) sred[wid] = ev;
    }
    __syncthreads();
    int lim = NTS;
    {
        float e0 = 0.0f;
        for (int q = 0; q < NTS / 32; q++) e0 = fmaxf(e0, sred[q]);
        if (e0 < 0.4f) {
            const float q = __fdividef(64.0f, -__log2f(e0) - 0.28f);
            const int qi = int(ceilf(q));
            lim = qi <= 1 ? 1 : min(NTS, 1 << (32 - __clz(qi - 1)));
        }
    }
    const double *fin = b0;
    for (int sd = 1, pp = 0; sd < lim; sd <<= 1, pp ^= 1) {
        const double *cur = pp ? b1 : b0;
        double *nxt = pp ? b0 : b1;
        int km = tid - sd, kp = tid + sd;
        const bool okm = km >= -PPAD, okp = kp < NTS + PPAD;
        km = okm ? km : 0; kp = okp ? kp : 0;
        double Am = cur[km], Cm = cur[SSTR + km], Dm = cur[2 * SSTR + km], Vm = cur[3 * SSTR + km], Wm = cur[4 * SSTR + km];
        double Ap = cur[kp], Cp = cur[SSTR + kp], Dp = cur[2 * SSTR + kp], Vp = cur[3 * SSTR + kp], Wp = cur[4 * SSTR + kp];
        if (!okm || tid - sd < 0) { Am = Cm = Dm = Vm = Wm = 0.0; }
        if (!okp || tid + sd >= NTS) { Ap = Cp = Dp = Vp = Wp = 0.0; }
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
    // the block's separator L_s = L_{G-1}: its equation couples to the last
    // interior chunk end (Y', V', W') and, through chunk 0's first row, to chunk
    // end 0 (Y0, V0, W0); cyclic: L_{j-1} = L_{j+1} = L_s (one block)
    __shared__ double sL;
    if (tid == ks) {
        const double Yp = fin[2 * SSTR + ks - 1], Vp = fin[3 * SSTR + ks - 1], Wp = fin[4 * SSTR + ks - 1];
        double Pn = 0, Qn = 0, Rn = 0, Y0 = 0, V0 = 0, W0 = 0;
        if (cyc) {
            Pn = P00; Qn = Q00; Rn = R00;
            Y0 = fin[2 * SSTR]; V0 = fin[3 * SSTR]; W0 = fin[4 * SSTR];
        }
        const double cr = cE * Rn;
        const double sub = -aE * Vp, dia = (1.0 - cE * Qn) - aE * Wp + cr * V0, sup = cr * W0;
        const double rhs = dE - cE * Pn - aE * Yp + cr * Y0;
        sL = cyc ? rhs * rcp(sub + dia + sup) : rhs * rcp(dia);
    }
    __syncthreads();
    const double Ls = sL;
    const double Xk = tid < ks ? D_ - (V_ + W_) * Ls : (tid == ks ? Ls : 0.0);
    double XL = 0.0;
    if (tid == 0) XL = cyc ? Ls : 0.0;
    else if (tid <= ks) XL = (tid - 1 == ks) ? Ls : fin[2 * SSTR + tid - 1] - (fin[3 * SSTR + tid - 1] + fin[4 * SSTR + tid - 1]) * Ls;
    if (live) {
        for (int j = j0; j < j1; j++) {
            const double Pi = Sx(0, j), Qi = Sx(1, j), Ri = Sx(2, j);
            Lout[j] = (j == j1 - 1) ? Xk : Pi - Qi * XL - Ri * Xk;
        }
    }
}

// ---------------------------------------------------------------------------
// Tile-level SPIKE, A19 filter at the interior tile ends (final stage): rows
// T-2, T-1 of tile b-1 and rows 0, 1 of tile b from the unfiltered rows
// T-4 .. T-1 and 0 .. 3 (P.sp_fb), written to the output state; their dt
// maxima join the member's.  Four threads per tile end.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) filter_fix_kernel(const Params P, const Bufs B)
{
    const int m = blockIdx.y;
    const int G = P.tiles;
    const bool cyc = P.bcl == BC_PERIODIC;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int bnd = t >> 2, i = (t & 3) + 2;          // tile end b between tiles b-1 and b; row 2..5
    double um = 0.0, nm = 0.0;
    // slab ends (BC_HALO): end 0 with the left slab's last rows (own rows 4, 5
    // only), end G with the right slab's first rows (own rows 2, 3 only)
    const bool hl = bnd == 0 && P.bcl == BC_HALO, hr = bnd == G && P.bcr == BC_HALO;
    const bool act = (bnd < G && (cyc || bnd > 0 || hl) || hr) && (!hl || i >= 4) && (!hr || i < 4) &&
                     P.dt[m] != 0.0;                  // (dt = 0: the member was carried)
    if (act) {
        const int bl = bnd > 0 ? bnd - 1 : G - 1;
        const int Tl = (bl == G - 1) ? P.n - (G - 1) * P.T : P.T;
        const double *fl = hl ? P.sx_fbl + size_t(m) * 8 : P.sp_fb + (size_t(m) * G + bl) * 16 + 8;  // rows Tl-4 .. Tl-1
        const double *fr = hr ? P.sx_fbr + size_t(m) * 8 : P.sp_fb + (size_t(m) * G + bnd) * 16;     // rows 0 .. 3
        double xq[8], xw[8];
#pragma unroll
        for (int k = 0; k < 4; k++) { xq[k] = fl[k]; xw[k] = fl[4 + k]; xq[4 + k] = fr[k]; xw[4 + k] = fr[4 + k]; }
        const double sig16 = P.filter_sigma * (1.0 / 16.0);
        double qo = 0.0, wo = 0.0;
#pragma unroll
        for (int k = 2; k < 6; k++)
            if (k == i) {
                qo = xq[k] - sig16 * (xq[k - 2] - 4.0 * xq[k - 1] + 6.0 * xq[k] - 4.0 * xq[k + 1] + xq[k + 2]);
                wo = xw[k] - sig16 * (xw[k - 2] - 4.0 * xw[k - 1] + 6.0 * xw[k] - 4.0 * xw[k + 1] + xw[k + 2]);
            }
        const int cell = i < 4 ? bl * P.T + Tl - 4 + i : bnd * P.T + (i - 4);   // (hl: i >= 4; hr: i < 4, bl = G-1)
        const size_t g = size_t(m) * P.n + cell;
        double h = B.out[0][g], K = B.out[2][g];
        const double bb = P.b ? P.b[cell] : 0.0;
        if (P.gen_rate > 0.0 || P.sp_rate > 0.0)           // A10 zones after the filter, at t^{n+1}
            relax_cell(P, P.x_min + (double(cell) + 0.5) * P.dx, bb, P.t[P.kpar * P.members + m] + P.dt[m],
                       h, qo, K, wo);
        B.out[0][g] = h;
        B.out[1][g] = qo;
        B.out[2][g] = K;
        B.out[3][g] = wo;
        if (!isfinite(qo + wo)) atomicOr(P.err, ERR_NONFINITE);
        const double ih = rcp(h);
        const double u = fabs(qo * ih), sg = (K - 1.5 * h * bb) * ih * ih;
        um = u;
        nm = u + fsqrt(P.g * h + P.lam[m] * (1.0 / 3.0) * sg * sg);
    }
    um = warp_max_nonneg(um);
    nm = warp_max_nonneg(nm);
    if ((threadIdx.x & 31) == 0 && nm > 0.0) {
        const int slot_w = (P.kslot + 1) % 3;
        atomicMax(P.maxes + (slot_w * 2 + 0) * P.members + m, (unsigned long long)__double_as_longlong(um));
        atomicMax(P.maxes + (slot_w * 2 + 1) * P.members + m, (unsigned long long)__double_as_longlong(nm));
    }
}


// ---------------------------------------------------------------------------
// SPIKE across slabs.  Slab p's separators satisfy
//     L_j = Y_j - V_j E_{p-1} - W_j F_{p+1}
// (Y, V, W from sep_solve_kernel modes 0, 1, 2 over the slab's G tiles; E_{p-1}
// the left slab's last separator, F_{p+1} the right slab's first), so the end
// separators of all slabs, F_q = L_0^q and E_q = L_{G-1}^q, satisfy the 2P system
//     F_q + V_0^q E_{q-1} + W_0^q F_{q+1} = Y_0^q
//     E_q + V_{G-1}^q E_{q-1} + W_{G-1}^q F_{q+1} = Y_{G-1}^q        (ring in q)
// (V = 0 / W = 0 on physical sides), which every slab solves redundantly from
// the all-gathered (Y, V, W) end values.
// ---------------------------------------------------------------------------
// what 0: tile 0's first-row relation (tips 6..11) -> sx_send[m][0..5] (to the left slab)
// what 1: (Y_0, V_0, W_0, Y_{G-1}, V_{G-1}, W_{G-1}) -> sx_send[m][0..5] (all-gather)
// what 2: tile 0's unfiltered rows 0..3 (q, W) -> sx_send[m][0..7] (to the left),
//         the last tile's rows Tc-4..Tc-1 -> sx_send[M*8 + m*8 ..] (to the right)
__global__ void slab_pack_kernel(const Params P, const int what)
{
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= P.members) return;
    const int G = P.tiles, M = P.members;
    if (what == 0) {
        const double *tp = P.sp_tips + size_t(m) * G * XPUB + 6;
        for (int k = 0; k < 6; k++) P.sx_send[size_t(m) * 6 + k] = tp[k];
    } else if (what == 1) {
        const double *Y = P.sx_yvw + size_t(m) * G, *V = Y + size_t(M) * G, *W = V + size_t(M) * G;
        double *o = P.sx_send + size_t(m) * 6;
        o[0] = Y[0]; o[1] = V[0]; o[2] = W[0]; o[3] = Y[G - 1]; o[4] = V[G - 1]; o[5] = W[G - 1];
    } else {
        const double *f0 = P.sp_fb + size_t(m) * G * 16, *fG = P.sp_fb + (size_t(m) * G + G - 1) * 16 + 8;
        for (int k = 0; k < 8; k++) {
            P.sx_send[size_t(m) * 8 + k] = f0[k];
            P.sx_send[size_t(M) * 8 + size_t(m) * 8 + k] = fG[k];
        }
    }
}

// one block per member, 128 threads: the 2P end-separator system (dense, no
// pivoting: a Schur complement of the M-matrix depth system), then
// L_j = Y_j - V_j E_{p-1} - W_j F_{p+1} into P.sp_L and (E_{p-1}, F_{p+1}) into sx_elfr
__global__ void __launch_bounds__(128) slab_iface_kernel(const Params P)
{
    const int m = blockIdx.x, tid = threadIdx.x;
    const int Ps = P.sx_P, n2 = 2 * Ps, G = P.tiles, M = P.members, p = P.sx_rank;
    double *const A = hsgn_smem;                      // [n2][n2 + 1], augmented
    const int ld = n2 + 1;
    for (int e = tid; e < n2 * ld; e += blockDim.x) A[e] = 0.0;
    __syncthreads();
    if (tid < Ps) {
        const int q = tid;
        const double *v = P.sx_all + (size_t(q) * M + m) * 6;    // Y0, V0, W0, YG, VG, WG of slab q
        const int ql = (q + Ps - 1) % Ps, qr = (q + 1) % Ps;
        double *rF = A + size_t(2 * q) * ld, *rE = A + size_t(2 * q + 1) * ld;
        rF[2 * q] += 1.0; rF[2 * ql + 1] += v[1]; rF[2 * qr] += v[2]; rF[n2] = v[0];
        rE[2 * q + 1] += 1.0; rE[2 * ql + 1] += v[4]; rE[2 * qr] += v[5]; rE[n2] = v[3];
    }
    __syncthreads();
    for (int k = 0; k < n2; k++) {                    // forward elimination
        const double piv = A[size_t(k) * ld + k];
        for (int i = k + 1 + tid; i < n2; i += blockDim.x) {
            const double f = A[size_t(i) * ld + k] / piv;
            if (f != 0.0)
                for (int j = k; j <= n2; j++) A[size_t(i) * ld + j] -= f * A[size_t(k) * ld + j];
        }
        __syncthreads();
    }
    __shared__ double sz[2];
    if (tid == 0) {                                   // back substitution (into column n2)
        for (int i = n2 - 1; i >= 0; i--) {
            double x = A[size_t(i) * ld + n2];
            for (int j = i + 1; j < n2; j++) x -= A[size_t(i) * ld + j] * A[size_t(j) * ld + n2];
            A[size_t(i) * ld + n2] = x / A[size_t(i) * ld + i];
        }
        const int ql = (p + Ps - 1) % Ps, qr = (p + 1) % Ps;
        sz[0] = P.bcl == BC_HALO ? A[size_t(2 * ql + 1) * ld + n2] : 0.0;    // E_{p-1}
        sz[1] = P.bcr == BC_HALO ? A[size_t(2 * qr) * ld + n2] : 0.0;        // F_{p+1}
        P.sx_elfr[2 * m] = sz[0];
        P.sx_elfr[2 * m + 1] = sz[1];
    }
    __syncthreads();
    const double El = sz[0], Fr = sz[1];
    const double *Y = P.sx_yvw + size_t(m) * G, *V = Y + size_t(M) * G, *W = V + size_t(M) * G;
    for (int j = tid; j < G; j += blockDim.x) P.sp_L[size_t(m) * G + j] = Y[j] - V[j] * El - W[j] * Fr;
}

}  // namespace hsgn
