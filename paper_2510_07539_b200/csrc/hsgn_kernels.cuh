// hsgn_kernels.cuh -- sm_100a fp64 kernels of the SI-IMEX hSGN step.
//
// One kernel launch = one IMEX stage S(E, R, tau) over every tile of
// every ensemble member.  Citations: P:n = PAPER.md line n, Ak = DESIGN.md
// reading k.  Nothing here is shared with oracle/ (no code, no constants).
//
// CTA work unit: a TILE of Tk kept cells of one member, extended by an overlap
// of w cells on each side (clipped at physical walls).  The depth system of
// P:509-512 couples the whole domain, but it is a diagonally dominant M-matrix
// whose inverse decays like r^k per cell (r from rho_max),
// so solving the extended tile with Neumann-truncated ends gives the kept rows
// exactly to round-off whenever r^w <= 2^-60; every CTA checks that with its
// own rho_max and latches HSGN_E_OVERLAP otherwise.  Periodic domains wrap.
//
// Phases inside the CTA (NT threads, rows of the extended tile in shared memory):
//   load   : coalesced global -> smem: E (h, q, H, W) on rows -3..L+2, R on
//            rows -1..L (stage 2 forms E and R from U^n and U1)
//   phase 1: per-thread CHUNKS of MCH rows, sliding register window:
//            MUSCL + Rusanov faces, predictor q^dag, H^dag, W^dag
//            (A9), coefficients beta, delta
//   phase 2: per-thread chunk assembly of Delta[h] = h^dag (A1),
//            partition method (downward + upward sweeps in registers), reduced
//            system of NT unknowns by PCR in smem, chunk recovery -> hbar
//   phase 3: back-substitution, optional A19 filter, coalesced
//            stores; final stage: per-member max|u|, max(|u|+c) for the next
//            dt and the step commit by the last CTA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef HSGN_NT
#define HSGN_NT 128
#endif
#ifndef HSGN_MINB
#define HSGN_MINB 4
#endif
#ifndef HSGN_MINB2                      // CTAs per SM of the plain second-stage kernels
#define HSGN_MINB2 5
#endif
#ifndef HSGN_MINB1                      // CTAs per SM of the plain first-stage kernels of a 2-stage
#define HSGN_MINB1 5                    // tableau (42 KB of shared memory each; the others: HSGN_MINB)
#endif
#ifndef HSGN_EXP_TIMING                 // dev builds only: per-CTA phase clocks (tools/*timing.py)
#define HSGN_EXP_TIMING 0
#endif

namespace hsgn {

constexpr int NT = HSGN_NT;           // threads per CTA
#ifndef HSGN_MCH
#define HSGN_MCH 5
#endif
constexpr int MCH = HSGN_MCH;       // rows per thread chunk (odd: conflict-free strided smem)
constexpr int LCAP = NT * MCH;      // 1280 rows per CTA incl. phase-1 halo rows
constexpr int SROWS = LCAP + 16;    // smem row capacity per array (even: 16-B aligned bases;
                                    // rows up to L+MCH+2 past a base shifted by <= 4)
constexpr int NARR = 8;             // smem arrays
// PCR buffers of the stage kernels (arrays 2..3 during phase 2): zero pads of
// PPADR slots around each of the three vectors, two buffers
constexpr int PPADR = NT / 2;                     // largest PCR distance
constexpr int PVS = NT + PPADR;                   // vector stride
constexpr int PBUF = 3 * PVS + PPADR;             // buffer stride (pad, A, pad, C, pad, D, pad)
constexpr size_t SMEM_BYTES = size_t(NARR) * SROWS * sizeof(double);
// one-CTA-per-tile stage kernels with bathymetry: b of the tile's raw rows in a
// ninth array (the per-row global reads of b through the boundary map cost more
// than the rest of the stage, `profiles/r01_ncu_summary.md`); < 48 KiB
constexpr size_t SMEM_BYTES_B = SMEM_BYTES + size_t(SROWS) * sizeof(double);
// Picard kernels (A24): alpha, a^2 of the own rows in two more arrays
constexpr size_t SMEM_BYTES_PIC = SMEM_BYTES + size_t(2 * SROWS) * sizeof(double);
constexpr size_t SMEM_BYTES_PIC_B = SMEM_BYTES_B + size_t(2 * SROWS) * sizeof(double);

enum { BC_PERIODIC = 0, BC_WALL = 1, BC_TRANSMISSIVE = 2, BC_HALO = 3 };
enum { ERR_COERC = 1u, ERR_DRY = 2u, ERR_NONFINITE = 4u, ERR_OVERLAP = 8u, ERR_DT = 16u };

struct Ctrl {            // device-resident run control (read by stage kernels)
    double t_end;        // <= 0: no clipping
    double dt_fixed;     // > 0: fixed step
};

struct Params {
    int n, members, tiles, T, w;
    int bcl, bcr, order;
    double dx, idx, g, h_min;        // idx = 1/dx
    double cfl, mcfl;
    double aI1, aI2, wE, wR;
    double filter_sigma;
    const double *b;                 // [n] or nullptr
    const double *lam;               // [members]
    double *t;                       // [2][members], by step parity
    double *dt;                      // [members]
    unsigned long long *maxes;       // [3 slots][2 kinds][members] (double bits), step % 3
    unsigned int *err;
    long long *steps;
    unsigned int *done;
    unsigned long long *rho_obs;     // max rho over tiles (double bits)
    unsigned int *kmin;              // min kappa = beta seen: max of ~khi_key (see khi_key)
    // tile-level SPIKE (hsgn_cluster.cuh CL_MODE_TIPS / FINISH, sep_solve_kernel,
    // filter_fix_kernel): per member and tile 12 published values, the separator
    // value L, 16 unfiltered boundary values; per member and tile 3 scratch
    double *sp_tips, *sp_L, *sp_fb, *sp_S;
    // SPIKE across slabs (BC_HALO sides), per member:
    // sx_nx[6] the right slab's tile-0 first-row relation, sx_fbl[8] / sx_fbr[8]
    // the neighbouring slabs' unfiltered end rows, sx_elfr[2] the neighbouring
    // slabs' end separators (E_{p-1}, F_{p+1}), sx_yvw[3][G] the local separator
    // solutions Y, V, W; sx_all[P][6] every slab's end values; sx_rank, sx_P
    double *sx_nx, *sx_fbl, *sx_fbr, *sx_elfr, *sx_yvw, *sx_all, *sx_send;
    int sx_rank, sx_P;
    const Ctrl *ctrl;
    int kslot, kpar;                 // host step index k: k mod 3, k mod 2
    // the step's first stage computes the step's dt itself (dt_commit_kernel's
    // rule, no launch of its own: stage_kernel<..., FDT>, small ensembles);
    // commit_prev: it also commits step k - 1
    int fuse_dt, commit_prev;
    // slab decomposition (BC_HALO sides): ghost cells received from the
    // neighbouring slab, H cells each: [0..3] U^n fields, [4..7] U1, [8] b
    const double *halo_l[9];
    const double *halo_r[9];
    int H;
    double inv_tiles;                // 1 / tiles
    double rho_ok;                   // largest rho whose decay r(rho)^w <= 2^-60 (overlap check)
    int picard;                      // A24 Picard passes (stage_kernel<..., PIC = true>)
    // A10 relaxation zones (cfg4), applied to U^{n+1} at t^{n+1} in the final
    // stage; rates <= 0 switch them off.  x_i = x_min + (i + 1/2) dx.
    double x_min, x_max, level, gen_x1, gen_rate, amp, omega, kw, cp, sp_x0, sp_rate;
};

struct Bufs {
    const double *Un[4];
    const double *U1[4];
    double *out[4];
};

#if HSGN_EXP_TIMING
// [stage][load wait, compute + store issue, epilogue + drain, CTAs, in-place + phase 1,
//  phase 2, phase 3 + staging, of phase 2: PCR + recovery]
__device__ unsigned long long g_exp[16];
__shared__ long long s_tph[4];
#define EXP_MARK(k) do { if (threadIdx.x == 0) s_tph[k] = clock64(); } while (0)
#else
#define EXP_MARK(k) do { } while (0)
#endif

// Reciprocal: hardware approximation (MUFU.RCP64H, ~2^-20) refined by one
// cubic step r0 (1 + e + e^2), e = 1 - x r0 (relative error e^3 < 2^-60; 3 DFMA,
// <= 1 ulp from IEEE 1/x, tools/rcp_check.cu) -- replaces the IEEE division
// sequence, whose slow-path branch and longer dependency chain dominated the
// stage's fp64 issue.
__device__ __forceinline__ double rcp(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// Shared memory of the stage kernels: the dynamic row arrays and a few
// per-CTA scratch variables (file scope, so the device helpers can reach them).
extern __shared__ __align__(16) double hsgn_smem[];
__shared__ __align__(8) unsigned long long s_mbar;
__shared__ double s_red[2][NT / 32];
__shared__ float s_redf[NT / 32];
__shared__ int s_redk[NT / 32];
__shared__ double s_xch[NT / 32][3];

__device__ __forceinline__ double *dyn_smem() { return hsgn_smem; }

__device__ __forceinline__ void cp_async8(double *dst_smem, const double *src)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// TMA bulk copy global -> shared (16-B aligned, size a multiple of 16),
// completion signalled on the mbarrier at shared address mbar.
__device__ __forceinline__ void bulk_g2s(double *dst_smem, const double *src, unsigned bytes,
                                         unsigned mbar)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(dst_smem);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(a), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

// TMA bulk copy shared -> global (16-B aligned, size a multiple of 16).
__device__ __forceinline__ void bulk_s2g(double *dst, const double *src_smem, unsigned bytes)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(src_smem);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                 ::"l"(dst), "r"(a), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned mbar, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(mbar), "r"(parity) : "memory");
}

__device__ __forceinline__ int map_cell(int c, int n, int bcl, int bcr, double &par)
{
    par = 1.0;
    if (c < 0) {
        if (bcl == BC_PERIODIC) { c %= n; if (c < 0) c += n; }
        else if (bcl == BC_WALL) { c = -1 - c; par = -1.0; }
        else c = 0;
    } else if (c >= n) {
        if (bcr == BC_PERIODIC) c %= n;
        else if (bcr == BC_WALL) { c = 2 * n - 1 - c; par = -1.0; }
        else c = n - 1;
    }
    return c;
}

__device__ __forceinline__ double bathy_at(const Params &P, int c)
{
    if (c < 0 && P.bcl == BC_HALO) return P.halo_l[8][c + P.H];
    if (c >= P.n && P.bcr == BC_HALO) return P.halo_r[8][c - P.n];
    double par;
    return __ldg(P.b + map_cell(c, P.n, P.bcl, P.bcr, par));
}

// dt rule of P:613-617 (reading A7 for nu_max): dt_bar = CFL dx / nu_max; if
// u_max dt_bar / dx > MCFL use MCFL dx / u_max.  Returns < 0 if undefined.
__device__ __forceinline__ double dt_rule(double cfl, double mcfl, double dx, double idx,
                                          double umax, double numax)
{
    double d;
    if (cfl > 0.0) {
        d = cfl * dx * rcp(numax);
        if (mcfl > 0.0 && umax > 0.0 && umax * d * idx > mcfl) d = mcfl * dx * rcp(umax);
    } else if (mcfl > 0.0 && umax > 0.0) {
        d = mcfl * dx * rcp(umax);
    } else {
        d = -1.0;
    }
    return d;
}

// dt of the step with maxima slot kslot and time parity kpar for member m
// (t_end clipping S:342); negative: invalid (ERR_DT).
__device__ __forceinline__ double member_dt(const Params &P, int kslot, int kpar, int m)
{
    const int members = P.members;
    const double umax = __longlong_as_double((long long)P.maxes[(kslot * 2 + 0) * members + m]);
    const double numax = __longlong_as_double((long long)P.maxes[(kslot * 2 + 1) * members + m]);
    const double t_end = P.ctrl->t_end, dt_fixed = P.ctrl->dt_fixed;
    const double tm = P.t[kpar * members + m];
    double dtm = dt_fixed > 0.0 ? dt_fixed : dt_rule(P.cfl, P.mcfl, P.dx, P.idx, umax, numax);
    if (t_end > 0.0) {
        if (!(tm < t_end)) dtm = 0.0;
        else if (tm + dtm >= t_end) dtm = t_end - tm;   // land exactly on t_end
    }
    return (dtm >= 0.0 && isfinite(dtm)) ? dtm : -1.0;
}

// sqrt(x), x > 0: MUFU.RSQ64H estimate (~1e-6), one Newton step for 1/sqrt
// (~1e-12), one residual correction of x * y, which squares the error again
// (branch-free; correctly rounded on 2^20 log-uniform samples over 1e-8 .. 1e8,
// as with two Newton steps: tools/rcp_check.cu).
__device__ __forceinline__ double fsqrt(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-(0.5 * x) * y, y, 1.5);
    const double s = x * y;
    return fma(fma(-s, s, x), 0.5 * y, s);
}

// MUSCL face states (A5): for the window rows (k-1, k, k+1),
// M_k = v_k + kap (v_{k+1} - v_{k-1}) at face k+1/2 and Pl_k = v_k - kap (...)
// at face k-1/2, kap = 1/4 (order 2) or 0 (order 1: v_k exactly, branch-free);
// u = q/h at the face state.
struct FState { double h, q, H, W, u; };
struct Face { double q, H, W; };

__device__ __forceinline__ FState muscl_minus(const double (&wh)[3], const double (&wq)[3],
                                              const double (&wH)[3], const double (&wW)[3],
                                              double kap)
{
    FState S;
    S.h = wh[1] + kap * (wh[2] - wh[0]); S.q = wq[1] + kap * (wq[2] - wq[0]);
    S.H = wH[1] + kap * (wH[2] - wH[0]); S.W = wW[1] + kap * (wW[2] - wW[0]);
    S.u = S.q * rcp(S.h);
    return S;
}

__device__ __forceinline__ FState muscl_plus(const double (&wh)[3], const double (&wq)[3],
                                             const double (&wH)[3], const double (&wW)[3],
                                             double kap)
{
    FState S;
    S.h = wh[1] - kap * (wh[2] - wh[0]); S.q = wq[1] - kap * (wq[2] - wq[0]);
    S.H = wH[1] - kap * (wH[2] - wH[0]); S.W = wW[1] - kap * (wW[2] - wW[0]);
    S.u = S.q * rcp(S.h);
    return S;
}

// Both face states of the window's centre row with one reciprocal:
// Z = 1/(h- h+), 1/h- = h+ Z, 1/h+ = h- Z (a few ulp from q/h).
__device__ __forceinline__ void muscl_pair(const double (&wh)[3], const double (&wq)[3],
                                           const double (&wH)[3], const double (&wW)[3],
                                           double kap, FState &Pl, FState &M)
{
    const double dh = wh[2] - wh[0], dq = wq[2] - wq[0];
    const double dH = wH[2] - wH[0], dW = wW[2] - wW[0];
    Pl.h = fma(-kap, dh, wh[1]); Pl.q = fma(-kap, dq, wq[1]);
    Pl.H = fma(-kap, dH, wH[1]); Pl.W = fma(-kap, dW, wW[1]);
    M.h = fma(kap, dh, wh[1]); M.q = fma(kap, dq, wq[1]);
    M.H = fma(kap, dH, wH[1]); M.W = fma(kap, dW, wW[1]);
    const double Z = rcp(Pl.h * M.h);
    Pl.u = Pl.q * (M.h * Z);
    M.u = M.q * (Pl.h * Z);
}

// Rusanov flux of R_E at a face (A4): alpha = max(|u-|, |u+|),
// F = 1/2 (F(U-) + F(U+)) - 1/2 alpha (U+ - U-) for F^q = q u, F^H = H u, F^W = W u.
// Returned as 2F (the 1/2 is folded into the tau/(2 dx) of the predictor: exact),
// in the form 2F = v- (u- + alpha) + v+ (u+ - alpha) (two products per field).
__device__ __forceinline__ Face rusanov(const FState &m, const FState &p)
{
    const double am = fabs(m.u), ap = fabs(p.u);
    const double a = am > ap ? am : ap;
    const double cm = m.u + a, cp = p.u - a;
    Face F;
    F.q = fma(m.q, cm, p.q * cp);
    F.H = fma(m.H, cm, p.H * cp);
    F.W = fma(m.W, cm, p.W * cp);
    return F;
}

// Pl state of the row after the window (rows k, k+1 = window[1..2] + (h1, q1, H1, W1)).
__device__ __forceinline__ FState muscl_plus_next(const double (&wh)[3], const double (&wq)[3],
                                                  const double (&wH)[3], const double (&wW)[3],
                                                  double h1, double q1, double H1, double W1,
                                                  double kap)
{
    const double th[3] = {wh[1], wh[2], h1}, tq[3] = {wq[1], wq[2], q1};
    const double tH[3] = {wH[1], wH[2], H1}, tW[3] = {wW[1], wW[2], W1};
    return muscl_plus(th, tq, tH, tW, kap);
}

struct RowCtx { double tau, tdx2, t2, lt2, lam, lam3, ltau, g, idx, c23; };

// Predictor (A9) and coefficients at E (A2) of
// one row r; E rows r-1, r, r+1 in (ch, cq, cH, cW); fluxes at r -+ 1/2.
// Stores q^dag, H^dag, beta, delta at row r unless r < -1 (dead row); returns
// h^R' (R_h plus the hydrostatic term) in hR_out.  Stage 2 reads R_h from the
// delta array (sRh == sDe) before overwriting it with delta.
// WB (reading A25): the delta array takes the face coefficient
// dhat_{r+1/2} = -(2 sigma^ - 1)/(3 h~) b1~ of rows r, r+1 instead (averages of
// sigma = H/h^2, h and 1/beta1 over the two rows).
template <bool BATHY, bool WB = false>
__device__ __forceinline__ void row_update(bool STAGE2, const RowCtx &C, const Params &P, const double *sB,
                                           int r, int start, int n,
                                           const double (&ch)[3], const double (&cq)[3],
                                           const double (&cH)[3], const double (&cW)[3],
                                           const Face &Fl, const Face &Fr, double *sQd,
                                           double *sHd, double *sBe, double *sDe, double &Wd_out,
                                           double &beta_out, double &hR_out)
{
    const bool live = r >= -1;
    const int rr = live ? r : 0;
    const double hE = ch[1], qE = cq[1], HE = cH[1], WE = cW[1];
    // R = E in stage 1; stage 2 combined it on load
    const double hR = STAGE2 ? sDe[rr] : hE, qR = STAGE2 ? sQd[rr] : qE;
    const double HR = STAGE2 ? sHd[rr] : HE, WR = STAGE2 ? sBe[rr] : WE;
    // one reciprocal for 1/h and 1/beta1 = h^2/(h^2 + lam tau^2):
    // Z = 1/(h (h^2 + lam tau^2)), 1/h = (h^2 + lam tau^2) Z, D = h Z
    const double s2 = hE * hE, den = s2 + C.lt2;
    const double Z = rcp(hE * den);
    const double ihE = den * Z, D = hE * Z;
    const double ih2 = ihE * ihE;
    const double sg = HE * ih2;                                      // eta/h
    double Dxb = 0.0, hRp = hR, ptil_term = 0.0;
    if (BATHY) {
        // (sB: b of the tile's raw rows in shared memory, else through the map)
        const double bm = sB ? sB[rr - 1] : bathy_at(P, start + rr - 1);
        const double b0 = sB ? sB[rr] : bathy_at(P, start + rr);
        const double bp = sB ? sB[rr + 1] : bathy_at(P, start + rr + 1);
        Dxb = (bp - bm) * (0.5 * C.idx);
        // hydrostatic term in zeta-form (A9)
        const double Gr = C.g * (hE + ch[2]) * 0.5, Gl = C.g * (ch[0] + hE) * 0.5;
        hRp = hR + C.t2 * (Gr * (bp - b0) - Gl * (b0 - bm));
        ptil_term = 1.5 * C.tau * C.lam3 * (1.0 - sg) * Dxb;        // p~
    }
    // predictor
    // (faces carry 2F: tau/dx (F_r - F_l) = tau/(2 dx) (2F_r - 2F_l))
    const double Wd = WR - C.tdx2 * (Fr.W - Fl.W) + C.ltau;
    const double Hd = HR - C.tdx2 * (Fr.H - Fl.H) - 1.5 * C.tau * qE * Dxb + C.tau * Wd;
    const double qd = qR - C.tdx2 * (Fr.q - Fl.q) - ptil_term;
    // coefficients at E: alpha = -(2 sg - 1)/(3 h), a^2,
    // 1/beta1 = h^2 D, beta2 = 2 lam tau^2 h D^2 with
    // D = 1/(h^2 + lam tau^2); so lam alpha beta2 = -(2/3) lam^2 tau^2 (2 sg - 1) D^2
    // and delta = alpha/beta1 = -(2 sg - 1)/3 h D
    const double t = 2.0 * sg - 1.0;
    const double a2 = fma(C.lam3 * sg, 3.0 * sg - 1.0, C.g * hE);
    const double beta = fma(-C.c23 * t, (D * D) * Hd, a2);
    double delta = (t * (-1.0 / 3.0)) * (hE * D);
    if (WB) {
        const double h1 = ch[2], s21 = h1 * h1, den1 = s21 + C.lt2;
        const double Z1 = rcp(h1 * den1);
        const double ih1 = den1 * Z1;
        const double sg1 = cH[2] * ih1 * ih1;
        const double ib11 = s21 * (h1 * Z1);
        // -(2 (sg + sg1)/2 - 1)/(3 (hE + h1)/2) (ib1 + ib11)/2
        delta = -(sg + sg1 - 1.0) * (s2 * D + ib11) * rcp(3.0 * (hE + h1));
    }
    if (live) { sQd[rr] = qd; sHd[rr] = Hd; sBe[rr] = beta; sDe[rr] = delta; }
    hR_out = hRp;
    Wd_out = Wd;
    beta_out = live ? beta : 2.2250738585072014e-308;   // dead rows: neutral for both checks
}

__device__ __forceinline__ double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Warp maxima of non-negative values on their bit patterns (IEEE order of
// non-negative numbers = unsigned order of their bits): two REDUX per double.
__device__ __forceinline__ double warp_max_nonneg(double v)
{
    const unsigned hi = unsigned(__double2hiint(v)), lo = unsigned(__double2loint(v));
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return __hiloint2double(int(mh), int(ml));
}

__device__ __forceinline__ float warp_max_nonneg(float v)
{
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}

__device__ __forceinline__ double block_max(double v, double *red, double ident = 0.0)
{
    v = warp_max(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = (lane < NT / 32) ? red[lane] : ident;
        v = warp_max(v);
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    v = red[0];
    __syncthreads();
    return v;
}

// ---------------------------------------------------------------------------
// The stage kernel.  STAGE2: inputs are U^n and U1 (E, R formed on load);
// FINAL: this stage produces U^{n+1} (filter, dt maxima, commit).
// ---------------------------------------------------------------------------
// A10 wavemaker / sponge relaxation of one cell (x, b) at time t:
// U -= s (U - U_target), see oracle/README and DESIGN.md A10.
__device__ __forceinline__ void relax_cell(const Params &P, double x, double b, double t, double &h,
                                           double &q, double &K, double &W)
{
    double s = 0.0, th, tq, tK;
    if (P.gen_rate > 0.0 && x <= P.gen_x1) {
        const double r = 1.0 - (x - P.x_min) / (P.gen_x1 - P.x_min);
        s = P.gen_rate * r * r;
        const double eta = P.amp * sin(P.omega * t - P.kw * (x - P.x_min));
        th = P.level + eta - b;
        tq = th * (P.cp * eta / P.level);
        tK = th * (th + 1.5 * b);
    } else if (P.sp_rate > 0.0 && x >= P.sp_x0) {
        const double r = (x - P.sp_x0) / (P.x_max - P.sp_x0);
        s = P.sp_rate * r * r;
        th = P.level - b;
        tq = 0.0;
        tK = th * (th + 1.5 * b);
    }
    if (s > 0.0) {
        h = h - s * (h - th);
        q = q - s * (q - tq);
        K = K - s * (K - tK);
        W = W - s * W;
    }
}

// ---------------------------------------------------------------------------
// Tile geometry of one stage.  Rows r in [0, L) of the extended tile are the
// cells start + r; raw rows -3 .. L+2 sit in shared memory at
// smem[k * SROWS + abase + r] (array k).  The stage delivers rows [klo, khi).
// ---------------------------------------------------------------------------
struct Geom {
    int start, L;                 // first cell, rows
    int wl, wr;                   // overlap rows at either end (truncated ends)
    int klo, khi;                 // rows this stage delivers
    bool left_phys, right_phys;   // tile ends on a physical boundary (Neumann end)
    bool interior;                // raw rows are all cells of [0, n) (no ghosts)
    int abase;
};

// Standalone stage tile of kept cells [s, e) with overlap w.
__device__ __forceinline__ Geom stage_geom(const Params &P, int s, int e, int w)
{
    const bool physL = (P.bcl == BC_WALL || P.bcl == BC_TRANSMISSIVE);
    const bool physR = (P.bcr == BC_WALL || P.bcr == BC_TRANSMISSIVE);
    Geom G;
    G.wl = physL ? min(w, s) : w;
    G.wr = physR ? min(w, P.n - e) : w;
    G.start = s - G.wl;
    G.L = (e - s) + G.wl + G.wr;
    G.klo = G.wl;
    G.khi = G.wl + (e - s);
    G.left_phys = physL && (G.start == 0);
    G.right_phys = physR && (G.start + G.L == P.n);
    G.interior = (G.start - 3 >= 0) && (G.start + G.L + 3 <= P.n);
    G.abase = 3;
    return G;
}

// TMA bulk loads need 16-B aligned destinations: shift the arrays by the parity
// of the first copied cell.  Interior tiles copy one range per field; tiles that
// wrap around a periodic domain of even n copy two (cells a0 .. n-1, then
// 0 .. cnt - seg1 - 1), both 16-B aligned because a0 and n are even.
struct LoadPlan {
    int a0, cnt;      // first copied cell (in [0, n)), count (even)
    int seg1;         // cells in the first range (== cnt unless the tile wraps)
    bool bulk;
};

__device__ __forceinline__ LoadPlan load_plan(const Params &P, size_t mo, Geom &G)
{
    LoadPlan Lp;
    const bool wrap = !G.interior && P.bcl == BC_PERIODIC && P.bcr == BC_PERIODIC && (P.n & 1) == 0;
    const int d = (G.interior || wrap) ? int((mo + size_t(G.start - 3)) & 1) : 0;
    G.abase = 3 + d;
    Lp.a0 = G.start - 3 - d;
    Lp.cnt = (G.L + 6 + d + 1) & ~1;
    Lp.seg1 = Lp.cnt;
    Lp.bulk = G.interior && (Lp.a0 >= 0) && (Lp.a0 + Lp.cnt <= P.n);
    if (wrap && Lp.cnt <= P.n) {
        if (Lp.a0 < 0) Lp.a0 += P.n;
        Lp.seg1 = min(Lp.cnt, P.n - Lp.a0);
        Lp.bulk = true;
    }
    return Lp;
}

// Issue the loads of the raw rows -3 .. L+2 of U^n (arrays 0..3) and, for a
// standalone stage 2, of U1 (arrays 7, 4, 5, 6 = h, q, K, W).  Bulk: thread 0,
// completion on the mbarrier; otherwise per-row cp.async through the BC index
// map or a slab halo (all threads).
// PART: LD_ALL (U^n, and U1 if WITH_U1; arrive + expect_tx), LD_UN (U^n only,
// expect_tx without arrive: a later LD_U1 completes the phase), LD_U1 (U1 only,
// arrive + expect_tx).
enum { LD_ALL = 0, LD_UN = 1, LD_U1 = 2 };

template <bool WITH_U1, int PART = LD_ALL, bool WITH_B = false>
__device__ __forceinline__ void issue_load(const Params &P, const Bufs &B, size_t mo, const Geom &G,
                                           const LoadPlan &Lp, unsigned mb, int tid)
{
    double *const smem = dyn_smem();
    constexpr bool DO_UN = PART != LD_U1;
    constexpr bool DO_U1 = WITH_U1 && PART != LD_UN;
    // b rides the TMA copies when its source is 16-B aligned too (a0 even: b has
    // no member offset), else every thread cp.asyncs it (odd n and odd member)
    const bool b_bulk = WITH_B && Lp.bulk && !(Lp.a0 & 1);
    if (WITH_B && Lp.bulk && !b_bulk) {
        double *const Ab = smem + G.abase + 8 * SROWS;
        for (int r = tid - 3; r < G.L + 3; r += NT) cp_async8(Ab + r, P.b + (G.start + r));
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    if (Lp.bulk) {
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const unsigned bytes = unsigned(Lp.seg1) * 8u;
            const unsigned bytes2 = unsigned(Lp.cnt - Lp.seg1) * 8u;     // wrapped part
            const unsigned tx = unsigned(Lp.cnt) * 8u * ((DO_UN ? 4u : 0u) + (DO_U1 ? 4u : 0u) + (b_bulk ? 1u : 0u));
            if (PART == LD_UN)
                asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(tx) : "memory");
            else
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(tx)
                             : "memory");
            const size_t gsrc = mo + size_t(Lp.a0);
            if (DO_UN) {
#pragma unroll
                for (int f = 0; f < 4; f++) bulk_g2s(smem + f * SROWS, B.Un[f] + gsrc, bytes, mb);
            }
            if (b_bulk) {
                bulk_g2s(smem + 8 * SROWS, P.b + Lp.a0, bytes, mb);
                if (bytes2) bulk_g2s(smem + 8 * SROWS + Lp.seg1, P.b, bytes2, mb);
            }
            if (DO_U1) {
                bulk_g2s(smem + 7 * SROWS, B.U1[0] + gsrc, bytes, mb);
                bulk_g2s(smem + 4 * SROWS, B.U1[1] + gsrc, bytes, mb);
                bulk_g2s(smem + 5 * SROWS, B.U1[2] + gsrc, bytes, mb);
                bulk_g2s(smem + 6 * SROWS, B.U1[3] + gsrc, bytes, mb);
            }
            if (bytes2) {
                const int k2 = Lp.seg1;
                if (DO_UN) {
#pragma unroll
                    for (int f = 0; f < 4; f++) bulk_g2s(smem + f * SROWS + k2, B.Un[f] + mo, bytes2, mb);
                }
                if (DO_U1) {
                    bulk_g2s(smem + 7 * SROWS + k2, B.U1[0] + mo, bytes2, mb);
                    bulk_g2s(smem + 4 * SROWS + k2, B.U1[1] + mo, bytes2, mb);
                    bulk_g2s(smem + 5 * SROWS + k2, B.U1[2] + mo, bytes2, mb);
                    bulk_g2s(smem + 6 * SROWS + k2, B.U1[3] + mo, bytes2, mb);
                }
            }
        }
    } else {
        double *const A = smem + G.abase;
        const int n = P.n;
        for (int r = tid - 3; r < G.L + 3; r += NT) {
            const int c = G.start + r;
            const double *p0, *p1, *p2, *p3, *u0 = nullptr, *u1 = nullptr, *u2 = nullptr, *u3 = nullptr;
            const double *pb = nullptr;
            if (c < 0 && P.bcl == BC_HALO) {
                const int o = c + P.H;
                p0 = P.halo_l[0] + o; p1 = P.halo_l[1] + o; p2 = P.halo_l[2] + o; p3 = P.halo_l[3] + o;
                pb = P.halo_l[8] + o;
                if (DO_U1) { u0 = P.halo_l[4] + o; u1 = P.halo_l[5] + o; u2 = P.halo_l[6] + o; u3 = P.halo_l[7] + o; }
            } else if (c >= n && P.bcr == BC_HALO) {
                const int o = c - n;
                p0 = P.halo_r[0] + o; p1 = P.halo_r[1] + o; p2 = P.halo_r[2] + o; p3 = P.halo_r[3] + o;
                pb = P.halo_r[8] + o;
                if (DO_U1) { u0 = P.halo_r[4] + o; u1 = P.halo_r[5] + o; u2 = P.halo_r[6] + o; u3 = P.halo_r[7] + o; }
            } else {
                double par;
                const int ci = map_cell(c, n, P.bcl, P.bcr, par);
                const size_t gi = mo + size_t(ci);
                pb = P.b + ci;
                p0 = B.Un[0] + gi; p1 = B.Un[1] + gi; p2 = B.Un[2] + gi; p3 = B.Un[3] + gi;
                if (DO_U1) { u0 = B.U1[0] + gi; u1 = B.U1[1] + gi; u2 = B.U1[2] + gi; u3 = B.U1[3] + gi; }
            }
            if (DO_UN) {
                cp_async8(A + r, p0); cp_async8(A + SROWS + r, p1);
                cp_async8(A + 2 * SROWS + r, p2); cp_async8(A + 3 * SROWS + r, p3);
            }
            if (DO_U1) {
                cp_async8(A + 7 * SROWS + r, u0); cp_async8(A + 4 * SROWS + r, u1);
                cp_async8(A + 5 * SROWS + r, u2); cp_async8(A + 6 * SROWS + r, u3);
            }
            if (WITH_B) cp_async8(A + 8 * SROWS + r, pb);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
}

// Wait for the loads issued by issue_load (bulk: mbarrier phase parity).
__device__ __forceinline__ void wait_load(const LoadPlan &Lp, unsigned mb, unsigned &parity)
{
    if (Lp.bulk) {
        mbar_wait(mb, parity);
        parity ^= 1u;
    } else {
        cp_async_wait_all();
    }
}

// Per-stage scalars (P:500-517 with tau = a_ii dt).
struct StageC {
    double tau, g, idx1, tdx, tdx2, t2, t2h, lt2, lt2h, ltdx2, lam, lam3, ltau;
};

__device__ __forceinline__ StageC stage_consts(const Params &P, double aii, double dtm, double lam)
{
    StageC S;
    S.tau = aii * dtm;
    S.g = P.g; S.idx1 = P.idx;
    S.tdx = S.tau * S.idx1;                 // tau / dx
    S.tdx2 = 0.5 * S.tdx;                   // tau / (2 dx)
    S.t2 = S.tdx * S.tdx;                   // tau^2 / dx^2
    S.t2h = 0.5 * S.t2;                     // tau^2 / (2 dx^2)
    S.lt2 = lam * S.tau * S.tau;            // lambda tau^2
    S.lt2h = 0.5 * lam * S.t2;              // lambda tau^2 / (2 dx^2)
    S.ltdx2 = lam * S.tdx2;                 // lambda tau / (2 dx)
    S.lam = lam;
    S.lam3 = lam * (1.0 / 3.0);
    S.ltau = lam * S.tau;
    return S;
}

// Accumulators of one tile.
struct TileAcc {
    double umax, numax, rho;
    unsigned int err;
    int wmin;                     // narrowest truncated overlap (1 << 30: none)
    int bhi;                      // max high word of beta over the rows (rho bound)
    int kkey = 0x7fffffff;        // min beta (= kappa) over the rows, as khi_key of its
                                  // high word (coercivity monitor, to 2^-20 relative)
};

// Order-preserving integer key of the high word of a double (signed order of
// the key = numeric order of the value); the device accumulator keeps ~key
// under atomicMax, so 0 (memset) is "no value yet".
__device__ __forceinline__ int khi_key(double v)
{
    const int hi = __double2hiint(v);
    return hi >= 0 ? hi : (hi ^ 0x7fffffff);
}

// ---------------------------------------------------------------------------
// One IMEX stage S(E, R, tau) on the tile G, data already in
// shared memory: raw U^n (and U1) rows as loaded, output K-form staged at
// arrays 4..7 (h, q, K, W) index r (rows [klo, khi) go out by the bulk store).
// ---------------------------------------------------------------------------
// LAT: the small-ensemble (latency) kernels -- 4 CTAs per SM, values kept in
// registers (one CTA per SM: occupancy does not matter, the per-thread chain does)
template <bool STAGE2, bool FINAL, bool BATHY, bool RELAX, bool PIC = false, bool WB = false, bool LAT = false>
__device__ __forceinline__ void stage_body(const Params &P, const Bufs &B, const Geom &G, int m, int s_cell,
                                           const StageC &S, double dtm, TileAcc &acc)
{
    const bool st2 = STAGE2;
    const bool fin = FINAL;
    double *const smem = dyn_smem();
    const int tid = threadIdx.x;
    const int n = P.n;
    const int start = G.start, L = G.L;
    const bool left_phys = G.left_phys, right_phys = G.right_phys;
    double *const A = smem + G.abase;
    double *sEh = A, *sEq = A + SROWS, *sEH = A + 2 * SROWS, *sEW = A + 3 * SROWS;
    double *sQd = A + 4 * SROWS;   // U1_q -> R_q -> q^dagger
    double *sHd = A + 5 * SROWS;   // U1_K -> R_H -> H^dagger
    double *sBe = A + 6 * SROWS;   // U1_W -> R_W -> beta -> hbar
    double *sDe = A + 7 * SROWS;   // U1_h -> R_h -> delta (R_h read by its own row first)
    // b of the raw rows -3 .. L+2 (one-CTA-per-tile kernels: array 8, loaded with the tile)
    const double *const sBz = BATHY ? A + 8 * SROWS : nullptr;
    auto bz = [&](int r) -> double { return sBz[r]; };
    const double tau = S.tau, g = S.g, idx1 = S.idx1, tdx = S.tdx, tdx2 = S.tdx2, t2 = S.t2;
    const double t2h = S.t2h, lt2 = S.lt2, lt2h = S.lt2h, ltdx2 = S.ltdx2, lam = S.lam;
    const double lam3 = S.lam3, ltau = S.ltau;
    const int members = P.members;

    // ---- in-place pass: E, R, H = K - 1.5 h b (A9), wall parity
    {
        const bool raw = true;                        // inputs not yet in H-form / parity
        // q parity of ghost rows mirrored at a wall (raw rows outside [0, n))
        const bool wall_par = raw && !G.interior && (P.bcl == BC_WALL || P.bcr == BC_WALL);
        if (st2 || (raw && BATHY)) {
            // two rows per thread and iteration with 16-B shared accesses: row r of
            // array k sits at smem[k * SROWS + abase + r], pairs start at even
            // offsets (the spare rows at either end are scratch)
            const double wE = P.wE, wR = P.wR;
            const int pbeg = (G.abase - 3) & ~1;
#pragma unroll 1      // (unrolled, the stage-2 kernel measured 1.5 % slower)
            for (int p = pbeg + 2 * tid; p < G.abase + L + 3; p += 2 * NT) {
                const int r = p - G.abase;
                double2 *v = reinterpret_cast<double2 *>(smem + p);
                double2 eh = v[0], eq = v[SROWS / 2], eK = v[SROWS], eW = v[3 * SROWS / 2];
                // (scratch rows clamped onto rows -3 .. L+2: stay inside slab halos)
                const double b0 = (raw && BATHY) ? bz(max(r, -3)) : 0.0;
                const double b1 = (raw && BATHY) ? bz(min(r + 1, L + 2)) : 0.0;
                if (st2) {
                    const double2 h1 = v[7 * SROWS / 2], q1 = v[2 * SROWS], K1 = v[5 * SROWS / 2],
                                  W1 = v[3 * SROWS];
                    const double q1x = q1.x, q1y = q1.y;
                    // (1 - w) U^n + w U1 = U^n + w (U1 - U^n): one difference, two FMAs
                    const double dhx = h1.x - eh.x, dhy = h1.y - eh.y, dqx = q1x - eq.x, dqy = q1y - eq.y;
                    const double dKx = K1.x - eK.x, dKy = K1.y - eK.y, dWx = W1.x - eW.x, dWy = W1.y - eW.y;
                    double2 rh, rq, rK, rW;
                    rh.x = fma(wR, dhx, eh.x); rh.y = fma(wR, dhy, eh.y);
                    rq.x = fma(wR, dqx, eq.x); rq.y = fma(wR, dqy, eq.y);
                    rK.x = fma(wR, dKx, eK.x); rK.y = fma(wR, dKy, eK.y);
                    rW.x = fma(wR, dWx, eW.x); rW.y = fma(wR, dWy, eW.y);
                    if (raw && BATHY) { rK.x -= 1.5 * rh.x * b0; rK.y -= 1.5 * rh.y * b1; }
                    v[7 * SROWS / 2] = rh; v[2 * SROWS] = rq; v[5 * SROWS / 2] = rK; v[3 * SROWS] = rW;
                    eh.x = fma(wE, dhx, eh.x); eh.y = fma(wE, dhy, eh.y);
                    eq.x = fma(wE, dqx, eq.x); eq.y = fma(wE, dqy, eq.y);
                    eK.x = fma(wE, dKx, eK.x); eK.y = fma(wE, dKy, eK.y);
                    eW.x = fma(wE, dWx, eW.x); eW.y = fma(wE, dWy, eW.y);
                }
                if (raw && BATHY) { eK.x -= 1.5 * eh.x * b0; eK.y -= 1.5 * eh.y * b1; }
                v[0] = eh; v[SROWS / 2] = eq; v[SROWS] = eK;
                if (st2) v[3 * SROWS / 2] = eW;
            }
            __syncthreads();
        }
        // q parity of the ghost rows mirrored at a wall (raw rows -3 .. -1 and L .. L+2
        // at most), after the combination: E and R are linear in (U^n, U1), so
        // negating them equals negating the inputs, bitwise
        if (wall_par) {
            if (tid < 6) {
                const int r = tid < 3 ? tid - 3 : L + (tid - 3);
                double par;
                (void)map_cell(start + r, n, P.bcl, P.bcr, par);
                if (par < 0.0) {
                    sEq[r] = -sEq[r];
                    if (st2) sQd[r] = -sQd[r];               // R_q
                }
            }
            __syncthreads();
        }
    }

    // Every thread owns the rows r0 .. r0+MCH-1 of the tile in all three
    // phases (thread 0 also computes row -1 in phase 1, the owner of row L
    // computes it); values stay in registers between phases, neighbours'
    // rows come from shared memory.  Threads whose rows all lie beyond L+1
    // ("dead" chunks) only take part in the reduced solve, as identity rows.
    const int r0 = tid * MCH;
    const bool live = r0 < L + 2;
    double wd[MCH];                  // W^dagger of own rows (phase 1 -> 3)
    double hRv[MCH];                 // h^R' of own rows (phase 1 -> 2)
    // Row -1 (the tile's left halo row of phase 1) is computed by the last
    // thread when its own chunk is dead (L <= (NT - 1) MCH - 2, every tile but
    // the largest): it runs the ordinary chunk loop over rows -1 .. MCH-2 and
    // stores row -1 only, in parallel with the others; otherwise thread 0 does
    // it before its own chunk.
    const bool m1_last = (NT - 1) * MCH >= L + 2;                // CTA-uniform
    const bool row_m1 = m1_last && tid == NT - 1;
    const int p0 = row_m1 ? -1 : r0;                             // first phase-1 row

    // ---- phase 1: faces, predictor, coefficients --------------------------
    // Branch-free over the MCH own rows (stores predicated on r <= L) so the
    // register window shifts are pure renaming.
    if (live || row_m1) {
        const double kap = P.order == 2 ? 0.25 : 0.0;
        RowCtx C{};
        C.tau = tau; C.tdx2 = tdx2; C.t2 = t2; C.lt2 = lt2; C.lam = lam; C.lam3 = lam3;
        C.ltau = ltau; C.g = g; C.idx = idx1;
        C.c23 = (2.0 / 3.0) * lam * lt2;
        double wh[3], wq[3], wH[3], wW[3];
#pragma unroll
        for (int k = 0; k < 3; k++) {                 // rows p0-2 .. p0
            const int rr = p0 - 2 + k;
            wh[k] = sEh[rr]; wq[k] = sEq[rr]; wH[k] = sEH[rr]; wW[k] = sEW[rr];
        }
        FState Mm = muscl_minus(wh, wq, wH, wW, kap);           // M_{p0-1}
        if (!m1_last && tid == 0) {
            // row -1 (left halo of the tile): faces -3/2 and -1/2
            double xh[3], xq[3], xH[3], xW[3];
#pragma unroll
            for (int k = 0; k < 3; k++) {             // rows -3 .. -1
                xh[k] = sEh[k - 3]; xq[k] = sEq[k - 3]; xH[k] = sEH[k - 3]; xW[k] = sEW[k - 3];
            }
            const FState M2 = muscl_minus(xh, xq, xH, xW, kap);     // M_{-2}
            const FState P1 = muscl_plus(wh, wq, wH, wW, kap);      // Pl_{-1} (rows -2..0)
            const Face Fa = rusanov(M2, P1);                          // face -3/2
            const FState P0 = muscl_plus_next(wh, wq, wH, wW, sEh[1], sEq[1], sEH[1], sEW[1], kap);
            const Face Fb = rusanov(Mm, P0);                          // face -1/2
            double Wd, beta, hRd;
            row_update<BATHY, WB>(st2, C, P, sBz, -1, start, n, wh, wq, wH, wW, Fa, Fb,
                                      sQd, sHd, sBe, sDe, Wd, beta, hRd);
        }
#pragma unroll
        for (int k = 0; k < 2; k++) {
            wh[k] = wh[k + 1]; wq[k] = wq[k + 1]; wH[k] = wH[k + 1]; wW[k] = wW[k + 1];
        }
        wh[2] = sEh[p0 + 1]; wq[2] = sEq[p0 + 1]; wH[2] = sEH[p0 + 1]; wW[2] = sEW[p0 + 1];
        FState Pn, Mr;
        muscl_pair(wh, wq, wH, wW, kap, Pn, Mr);               // Pl_{p0}, M_{p0}
        Face Fl = rusanov(Mm, Pn);                             // face p0-1/2
#pragma unroll
        for (int i = 0; i < MCH; i++) {
            const int r = p0 + i;
            // rows this thread stores: its own rows up to L, or row -1 only
            const bool own = row_m1 ? (i == 0) : (r <= L);
            double ch[3], cq[3], cH[3], cW[3];                 // rows r-1, r, r+1
#pragma unroll
            for (int k = 0; k < 3; k++) { ch[k] = wh[k]; cq[k] = wq[k]; cH[k] = wH[k]; cW[k] = wW[k]; }
#pragma unroll
            for (int k = 0; k < 2; k++) {
                wh[k] = wh[k + 1]; wq[k] = wq[k + 1]; wH[k] = wH[k + 1]; wW[k] = wW[k + 1];
            }
            wh[2] = sEh[r + 2]; wq[2] = sEq[r + 2]; wH[2] = sEH[r + 2]; wW[2] = sEW[r + 2];
            FState Mn;
            muscl_pair(wh, wq, wH, wW, kap, Pn, Mn);           // Pl_{r+1}, M_{r+1}
            const Face Fr = rusanov(Mr, Pn);                   // face r+1/2
            Mr = Mn;
            double beta, hRr;
            row_update<BATHY, WB>(st2, C, P, sBz, own ? r : -1000000, start, n, ch, cq, cH, cW, Fl, Fr,
                                      sQd, sHd, sBe, sDe, wd[i], beta, hRr);
            hRv[i] = own ? hRr : 0.0;                          // rows > L: decoupled, finite
            if (i == 0 && row_m1) beta = 2.2250738585072014e-308;   // row -1: not a tile row
            // coercivity on every row of the tile (overlap rows are real
            // cells, and the kept rows' solve relies on them too); the rho bound
            // of the overlap check from max beta (high words: +1 ulp of 2^-20)
            if (!(beta > 0.0)) acc.err |= ERR_COERC;
            acc.bhi = max(acc.bhi, __double2hiint(beta));
            if (!row_m1 && r < L) acc.kkey = min(acc.kkey, khi_key(beta));
            Fl = Fr;
        }
    } else {
#pragma unroll
        for (int i = 0; i < MCH; i++) { wd[i] = 0.0; hRv[i] = 0.0; }
    }
    __syncthreads();
    EXP_MARK(0);
    // plain second stage (5 CTAs per SM): W^dagger of the own rows parked in
    // array 0 (E_h is dead after phase 1 without bathymetry) until phase 3
    constexpr bool s2x = STAGE2 && FINAL && !BATHY && !RELAX && !PIC && !WB && !LAT;
    if (s2x && live) {
#pragma unroll
        for (int i = 0; i < MCH; i++) sEh[r0 + i] = wd[i];
    }
    // derived-field ghosts at physical boundaries (A10).  The implicit
    // coupling across both tile ends is cut (truncated overlap or Neumann end:
    // r_{-1/2} = r_{L-1/2} = 0): beta_{-1} = -beta_0 and beta_L = -beta_{L-1}
    // make those face coefficients t2 (beta_i + beta_{i+1}) / 2 exactly zero;
    // rows L+1 .. L+MCH+2 (read by the last live chunk, and as the window of
    // every dead chunk) get zero fields and alternating +-beta_{L-1}, so all
    // their couplings vanish too (dead chunks are identity rows).
    auto tile_end_ghosts = [&]() {
        if (tid == 0) {
            if (left_phys) {
                sQd[-1] = (P.bcl == BC_WALL ? -1.0 : 1.0) * sQd[0];
                sHd[-1] = sHd[0]; sDe[-1] = sDe[0];
            }
            sBe[-1] = -sBe[0];
        }
        if (tid == 32) {
            if (right_phys) {
                sQd[L] = (P.bcr == BC_WALL ? -1.0 : 1.0) * sQd[L - 1];
                sHd[L] = sHd[L - 1]; sDe[L] = sDe[L - 1];
            }
            sBe[L] = -sBe[L - 1];
        }
        if (tid >= 64 && tid < 64 + MCH + 2) {
            const int r = L + 1 + (tid - 64);
            sQd[r] = 0.0; sHd[r] = 0.0; sDe[r] = 0.0;
            sBe[r] = ((r - L) & 1) ? sBe[L - 1] : -sBe[L - 1];
        }
    };
    tile_end_ghosts();
    // zero pads around the PCR vectors (arrays 2..3 are free after phase 1):
    // partners outside [0, NT) read exact zeros, no bounds tests in the levels
    {
        double *const pb = smem + 2 * SROWS;
#pragma unroll
        for (int k = tid; k < 8 * PPADR; k += NT) {
            const int b = k / (4 * PPADR), v = (k / PPADR) & 3, o = k % PPADR;
            pb[b * PBUF + v * PVS + o] = 0.0;
        }
    }
    __syncthreads();

    // ---- phase 2: assemble + partition solve (A1, A3) ---------
    // Arrays 1..3 are free after phase 1: hbar in array 1, PCR buffers over
    // arrays 2..3 (later the filter buffers), E_h stays in array 0; arrays
    // 4..7 take the output staging during phase 3.
    double *sHB = sEq;                                           // hbar[r], r in [0, L)
    // two PCR buffers of three vectors (A, C, D) of NT slots, each vector
    // between zero pads of PPADR slots (PVS = NT + PPADR)
    double *pcr0 = smem + 2 * SROWS + PPADR;
    double *pcr1 = pcr0 + PBUF;
    double *sEhc = sEh;                                          // E_h (BATHY)
    // register windows over rows r0-1 .. r0+MCH
    // (dead chunks read the ghost rows L+1 .. L+MCH+2: identity rows)
    double vb[MCH + 2], vd[MCH + 2], vH[MCH + 2], vq[MCH + 2];
    // (the 4-CTA second stages, at the register cap, measured faster with zeroed
    // dead windows: 483 vs 486 us on cfg3; the 5-CTA one reads the ghost rows like
    // the first stage: 444.5 -> 437.9 us)
    if (STAGE2 && !s2x) {
        if (live) {
#pragma unroll
            for (int k = 0; k < MCH + 2; k++) {
                vb[k] = sBe[r0 - 1 + k]; vd[k] = sDe[r0 - 1 + k]; vH[k] = sHd[r0 - 1 + k]; vq[k] = sQd[r0 - 1 + k];
            }
        } else {
#pragma unroll
            for (int k = 0; k < MCH + 2; k++) { vb[k] = 0.0; vd[k] = 0.0; vH[k] = 0.0; vq[k] = 0.0; }
        }
    } else {
        const int wb0 = live ? r0 - 1 : L + 1;
#pragma unroll
        for (int k = 0; k < MCH + 2; k++) {
            vb[k] = sBe[wb0 + k]; vd[k] = sDe[wb0 + k]; vH[k] = sHd[wb0 + k]; vq[k] = sQd[wb0 + k];
        }
    }
    double hb[MCH];
    // PIC: alpha, a^2 at E of the own rows, in two arrays after the tile's (shared
    // memory rather than registers: the Picard kernels were spilling)
    double *const sAl = smem + (BATHY ? 9 : 8) * SROWS;
#pragma unroll 1
    for (int pic = 0; pic <= (PIC ? P.picard : 0); pic++) {
    if (PIC && pic > 0) {
        // A24 Picard pass: beta, delta of the own rows with beta1 = 1 + lam tau^2/hbar^2
        // and beta2 = 2 lam tau^2/(beta1^2 hbar^3) at the latest hbar; alpha, a^2 stay
        // at E (recovered from the first pass: alpha = delta beta1(h^E),
        // a^2 = beta - lam alpha beta2(h^E) H^dag)
        if (live) {
#pragma unroll
            for (int i = 0; i < MCH; i++) {
                const int r = r0 + i;
                if (r >= L) continue;
                double al, a2;
                if (pic == 1) {
                    const double hE = sEh[r], hE2 = hE * hE;
                    const double b1E = 1.0 + lt2 / hE2;
                    const double b2E = 2.0 * lt2 / (b1E * b1E * hE2 * hE);
                    al = vd[i + 1] * b1E;
                    a2 = vb[i + 1] - lam * al * b2E * vH[i + 1];
                    sAl[r] = al;
                    sAl[SROWS + r] = a2;
                } else {
                    al = sAl[r];
                    a2 = sAl[SROWS + r];
                }
                const double hn = hb[i], hn2 = hn * hn;
                const double b1 = 1.0 + lt2 / hn2;
                const double b2 = 2.0 * lt2 / (b1 * b1 * hn2 * hn);
                const double be = a2 + lam * al * b2 * vH[i + 1];
                if (r >= G.klo && r < G.khi && !(be > 0.0)) acc.err |= ERR_COERC;
                acc.bhi = max(acc.bhi, __double2hiint(be));
                acc.kkey = min(acc.kkey, khi_key(be));
                sBe[r] = be;
                sDe[r] = al / b1;
            }
        }
        __syncthreads();
        tile_end_ghosts();
        __syncthreads();
        if (live) {
#pragma unroll
            for (int k = 0; k < MCH + 2; k++) { vb[k] = sBe[r0 - 1 + k]; vd[k] = sDe[r0 - 1 + k]; }
        }
    }
    {
        double am[MCH], cm[MCH], dm[MCH];
#pragma unroll
        for (int i = 0; i < MCH; i++) {
            // (r_{-1/2} = r_{L-1/2} = 0 through the beta ghosts set above)
            const double rl = t2h * (vb[i] + vb[i + 1]);
            const double rr = t2h * (vb[i + 1] + vb[i + 2]);
            // (WB, A25: mu_{r+1/2} = 2 lt2h dhat_{r+1/2}, face values in vd)
            const double ml = WB ? 2.0 * lt2h * vd[i] : lt2h * (vd[i] + vd[i + 1]);
            const double mr = WB ? 2.0 * lt2h * vd[i + 1] : lt2h * (vd[i + 1] + vd[i + 2]);
            const double rhs = hRv[i] - tdx2 * (vq[i + 2] - vq[i]) + mr * (vH[i + 2] - vH[i + 1])
                               - ml * (vH[i + 1] - vH[i]);
            const double a = -rl, c = -rr, dg = 1.0 + rl + rr;
            if (i == 0) {
                const double inv = rcp(dg);
                am[0] = a * inv; cm[0] = c * inv; dm[0] = rhs * inv;
            } else {
                const double inv = rcp(dg - a * cm[i - 1]);
                am[i] = -a * am[i - 1] * inv;
                cm[i] = c * inv;
                dm[i] = (rhs - a * dm[i - 1]) * inv;
            }
        }
        // chunk-end relation (downward) and first-row relation (upward):
        // x_i = P_i - Q_i X_{k-1} - R_i X_k,  X_k = last row of chunk k
        const double aE = am[MCH - 1], cE = cm[MCH - 1], dE = dm[MCH - 1];
        double Pn = 0.0, Qn = 0.0, Rn = -1.0;
#pragma unroll
        for (int i = MCH - 2; i >= 0; i--) {
            const double Pi = dm[i] - cm[i] * Pn;
            const double Qi = am[i] - cm[i] * Qn;
            const double Ri = -cm[i] * Rn;
            dm[i] = Pi; am[i] = Qi; cm[i] = Ri;
            Pn = Pi; Qn = Qi; Rn = Ri;
        }
        // neighbour's (P_0, Q_0, R_0) via shuffles / smem across warps
        const int lane = tid & 31, wid = tid >> 5;
        double P1 = __shfl_down_sync(0xffffffffu, dm[0], 1);
        double Q1 = __shfl_down_sync(0xffffffffu, am[0], 1);
        double R1 = __shfl_down_sync(0xffffffffu, cm[0], 1);
        if (lane == 0) { s_xch[wid][0] = dm[0]; s_xch[wid][1] = am[0]; s_xch[wid][2] = cm[0]; }
        __syncthreads();
        if (lane == 31) {
            if (wid + 1 < NT / 32) { P1 = s_xch[wid + 1][0]; Q1 = s_xch[wid + 1][1]; R1 = s_xch[wid + 1][2]; }
            else { P1 = 0.0; Q1 = 0.0; R1 = 0.0; }
        }
        // reduced row k:  A X_{k-1} + Bd X_k + C X_{k+1} = D, normalised by Bd
        double A_ = aE, C_ = -cE * R1, D_ = dE - cE * P1;
        if (tid == 0) A_ = 0.0;
        {
            const double ib = rcp(1.0 - cE * Q1);
            A_ *= ib; C_ *= ib; D_ *= ib;
        }
        // PCR over NT unknowns, double-buffered, one reciprocal per row and
        // step.  The reduced couplings shrink like e_{s+1} <= e_s^2/(1-2e_s^2)
        // (e = max |A|,|C|), so PCR stops once e^(2^s) <= 2^-64: the rows are
        // then decoupled to below round-off (x_k = D_k).
        EXP_MARK(2);
        pcr0[tid] = A_; pcr0[PVS + tid] = C_; pcr0[2 * PVS + tid] = D_;
        {
            const float ea = float(fabs(A_)), ec = float(fabs(C_));
            const float ev = warp_max_nonneg(ea > ec ? ea : ec);
            if (lane == 0) s_redf[wid] = ev;
        }
        __syncthreads();
        int lim = NT;
        {
            float e0 = 0.0f;
#pragma unroll
            for (int q = 0; q < NT / 32; q++) e0 = fmaxf(e0, s_redf[q]);
            if (e0 < 0.4f) {
                // repeated squaring with a 10 % margin per step, ee_0 = 1.1 e0,
                // ee_{s+1} = 1.1 ee_s^2, stops at the first s with ee_s <= 2^-64:
                // log2 ee_s = 2^s (log2 e0 + 2 log2 1.1) - log2 1.1, so
                // 2^s >= (64 - log2 1.1) / -(log2 e0 + 2 log2 1.1), rounded up to a
                // power of two (margins 64 and 0.28 cover the log2 approximation);
                // e0 = 0 gives q = 0 and no PCR step
                const float q = __fdividef(64.0f, -__log2f(e0) - 0.28f);
                const int qi = int(ceilf(q));
                lim = qi <= 1 ? 1 : min(NT, 1 << (32 - __clz(qi - 1)));
            }
        }
        // one PCR level at distance sd (compile-time), cur -> nxt
        // (partners outside [0, NT) are the zero pads)
        auto level = [&](const int sd, const double *cur, double *nxt) {
            const int km = tid - sd, kp = tid + sd;
            const double Am = cur[km], Cm = cur[PVS + km], Dm = cur[2 * PVS + km];
            const double Ap = cur[kp], Cp = cur[PVS + kp], Dp = cur[2 * PVS + kp];
            const double ib = rcp(1.0 - A_ * Cm - C_ * Ap);
            const double Dn = (D_ - A_ * Dm - C_ * Dp) * ib;
            if (2 * sd < lim) {                  // another level follows (lim: CTA-uniform)
                const double An = -A_ * Am * ib;
                const double Cn = -C_ * Cp * ib;
                A_ = An; C_ = Cn; D_ = Dn;
                nxt[tid] = A_; nxt[PVS + tid] = C_; nxt[2 * PVS + tid] = D_;
                __syncthreads();
            } else {
                D_ = Dn;                         // the last level: x_k = D_, nothing to publish
            }                                    // (the XL exchange below has its own barrier)
        };
        static_assert(NT % 32 == 0 && NT <= 256, "PCR levels below are written out for up to 256 unknowns");
        if (lim > 1) level(1, pcr0, pcr1);
        if (lim > 2) level(2, pcr1, pcr0);
        if (lim > 4) level(4, pcr0, pcr1);
        if (lim > 8) level(8, pcr1, pcr0);
        if (lim > 16) level(16, pcr0, pcr1);
        if (lim > 32) level(32, pcr1, pcr0);
        if (lim > 64) level(64, pcr0, pcr1);
        if (NT > 128 && lim > 128) level(128, pcr1, pcr0);
        const double Xk = D_;
        double XL = __shfl_up_sync(0xffffffffu, Xk, 1);
        if (lane == 31) s_xch[wid][0] = Xk;       // last chunk of this warp
        __syncthreads();
        if (lane == 0) XL = (wid > 0) ? s_xch[wid - 1][0] : 0.0;
#pragma unroll
        for (int i = 0; i < MCH; i++) {
            const int r = r0 + i;
            hb[i] = (i == MCH - 1) ? Xk : dm[i] - am[i] * XL - cm[i] * Xk;
            if (r < L) sHB[r] = hb[i];
        }
    }
    __syncthreads();
    }   // Picard passes

    EXP_MARK(1);
    // rho = max (tau/dx)^2 (beta_i + beta_{i+1})/2 <= t2 max beta
    acc.rho = fmax(acc.rho, t2 * __hiloint2double(acc.bhi + 1, 0));

    // ---- phase 3: back-substitution, own rows ------------------
    const bool filt = fin && (P.filter_sigma > 0.0);
    double *sQb = smem + 2 * SROWS + G.abase;                   // filter (A19)
    double *sWb = sQb + SROWS;
    const int klo = G.klo, khi = G.khi;
    const int flo = filt ? klo - 2 : klo, fhi = filt ? khi + 2 : khi;
    // HdD = H^dag / (hbar^2 + lam tau^2): Hbar = HdD hbar^2 and, in the
    // final stage, sigma = Hbar / hbar^2 = HdD for the dt maxima
    double qbv[MCH], HdD[MCH], Wbv[MCH], bbv[MCH], ihv[MCH];
    // final stage without relaxation: h and K of the kept rows are staged in the
    // first loop (arrays 4..7 are not read in phase 3 then) and the wave speed's
    // root sqv computed there, so only q, W (filtered) and u wait for the filter
    // -- fewer values live across it
    double sqv[MCH];
    // Neumann at physical ends (hbar_{-1} := hbar_0, hbar_L := hbar_{L-1}); at cut
    // tile ends rows 0 and L-1 are overlap rows whose qbar is never used (w >= 3)
    constexpr bool reload = (!STAGE2 && !FINAL && !BATHY && !PIC && !WB && !LAT) || s2x;   // (the 5-CTA kernels)
    constexpr bool early = FINAL && !RELAX;
    if (reload) {
        // the plain kernels: the coefficient windows again from shared memory
        // (arrays 4..7 are intact until the staging), so their registers die after
        // the assembly -- 96 registers without spills, 5 CTAs per SM (cfg3: stage
        // 1 313 -> 287 us, stage 2 481 -> 459 us with W^dagger parked and the
        // early staging)
#pragma unroll
        for (int k = 0; k < MCH + 2; k++) {
            vb[k] = sBe[r0 - 1 + k]; vd[k] = sDe[r0 - 1 + k]; vH[k] = sHd[r0 - 1 + k]; vq[k] = sQd[r0 - 1 + k];
        }
        if (early) __syncthreads();          // (the early staging below overwrites arrays 4, 6)
    }
    const double hLn = r0 > 0 ? ((r0 - 1 < L) ? sHB[r0 - 1] : 0.0) : hb[0];
    double hRn = (r0 + MCH < L) ? sHB[r0 + MCH] : 0.0;
    if (right_phys) {
        if (r0 + MCH == L) hRn = hb[MCH - 1];
#pragma unroll
        for (int i = 1; i < MCH; i++)
            if (r0 + i == L) hb[i] = hb[i - 1];       // (row L itself is not kept)
    }
#pragma unroll
    for (int i = 0; i < MCH; i++) {
        const int r = r0 + i;
        const bool act = (r >= flo) && (r < fhi) && (r < L);   // rows this stage needs
        bbv[i] = 0.0;
        const double h0 = hb[i];
        double hl = (i > 0) ? hb[i - 1] : hLn;
        double hr = (i < MCH - 1) ? hb[i + 1] : hRn;
        double qb;
        if (WB) {
            // A25: qbar = q^dag - tau/(2 dx) (Phi_{r+1/2} + Phi_{r-1/2}) with the face
            // fluxes Phi = beta~ (hbar_R - hbar_L) + lam dhat (H^dag_R - H^dag_L)
            // + g h~ (b_R - b_L) (E-depth h~); zero at physical (and cut) ends
            double Phr = 0.5 * (vb[i + 1] + vb[i + 2]) * (hr - h0) + lam * vd[i + 1] * (vH[i + 2] - vH[i + 1]);
            double Phl = 0.5 * (vb[i] + vb[i + 1]) * (h0 - hl) + lam * vd[i] * (vH[i + 1] - vH[i]);
            if (BATHY && act) {
                const double bm = bz(r - 1), bp = bz(r + 1);
                const double b0 = bz(r);
                const double e0 = sEhc[r];
                bbv[i] = b0;
                Phr += 0.5 * g * (e0 + sEhc[r + 1]) * (bp - b0);
                Phl += 0.5 * g * (sEhc[r - 1] + e0) * (b0 - bm);
            }
            if (r == 0) Phl = 0.0;
            if (r == L - 1) Phr = 0.0;
            qb = vq[i + 1] - tdx2 * (Phr + Phl);
        } else {
            qb = vq[i + 1] - tdx2 * vb[i + 1] * (hr - hl) - ltdx2 * vd[i + 1] * (vH[i + 2] - vH[i]);
        }
        if (BATHY && act && !WB) {
            const double bm = bz(r - 1);
            const double bp = bz(r + 1);
            bbv[i] = bz(r);
            qb -= tau * g * sEhc[r] * (bp - bm) * (0.5 * idx1);     // A9
        }
        // P:514-515 with one reciprocal: Hbar = H^dag hbar^2 / (hbar^2 + lam tau^2),
        // Wbar = W^dag - lam tau H^dag / (hbar^2 + lam tau^2); in the final stage
        // the same reciprocal gives 1/hbar: Z = 1/(hbar (hbar^2 + lam tau^2))
        const double den = h0 * h0 + lt2;
        double rden;
        if (fin && !RELAX) {
            const double Z = rcp(h0 * den);
            rden = h0 * Z;
            ihv[i] = den * Z;
        } else {
            rden = rcp(den);
            ihv[i] = 0.0;
        }
        HdD[i] = vH[i + 1] * rden;
        qbv[i] = qb;
        Wbv[i] = (s2x ? sEh[r] : wd[i]) - ltau * HdD[i];
        if (early) {
            const double Hb = HdD[i] * (h0 * h0);
            const double Ko = BATHY ? Hb + 1.5 * h0 * bbv[i] : Hb;
            sqv[i] = fsqrt(g * h0 + lam3 * HdD[i] * HdD[i]);         // sigma = Hbar / hbar^2 = HdD
            smem[4 * SROWS + r] = h0; smem[6 * SROWS + r] = Ko;     // (staged at row r, unmasked)
        }
        {
            // dry rows among the kept ones; non-finite values among the rows the
            // stage delivers (with the filter: also its +-2 input rows, so the
            // filtered values need no test of their own).  One test for all four:
            // a NaN or inf in any makes the sum non-finite.  Branch-free.
            const bool kept = (r >= klo) && (r < khi);
            const unsigned ed = !(h0 > P.h_min) ? unsigned(ERR_DRY) : 0u;
            const unsigned ef = !isfinite(h0 + qb + HdD[i] + Wbv[i]) ? unsigned(ERR_NONFINITE) : 0u;
            acc.err |= (kept ? ed : 0u) | ((filt ? act : kept) ? ef : 0u);
        }
        if (filt && r < L) { sQb[r] = qb; sWb[r] = Wbv[i]; }
    }
    if (filt || reload) __syncthreads();     // (reads of arrays 4..7 before the staging)
    const double sig16 = P.filter_sigma * (1.0 / 16.0);
    const double t_new = (fin && RELAX) ? P.t[P.kpar * members + m] + dtm : 0.0;
    // filter windows over rows r0-2 .. r0+MCH+1: own rows from registers, two halo
    // rows each side from shared memory (threads whose window meets a physical
    // end mirror per row below)
    const bool fwin = filt && (!(left_phys || right_phys) || (r0 >= 2 && r0 + MCH + 2 <= L));
    double xq[MCH + 4], xw[MCH + 4];
    if (fwin) {
        xq[0] = sQb[r0 - 2]; xq[1] = sQb[r0 - 1]; xq[MCH + 2] = sQb[r0 + MCH]; xq[MCH + 3] = sQb[r0 + MCH + 1];
        xw[0] = sWb[r0 - 2]; xw[1] = sWb[r0 - 1]; xw[MCH + 2] = sWb[r0 + MCH]; xw[MCH + 3] = sWb[r0 + MCH + 1];
#pragma unroll
        for (int i = 0; i < MCH; i++) { xq[i + 2] = qbv[i]; xw[i + 2] = Wbv[i]; }
    }
    // final values into (hb, qbv, HdD := K or H, Wbv)
#pragma unroll
    for (int i = 0; i < MCH; i++) {
        const int r = r0 + i;
        // rows outside [klo, khi) are computed and masked (no per-row branch),
        // except on the relaxation and mirrored-filter paths
        const bool kept = (r >= klo) && (r < khi);
        if (!kept && (RELAX || (filt && !fwin))) continue;
        double qo = qbv[i], wo = Wbv[i];
        if (filt) {
            // A19: f_i - (sigma/16)(f_{i-2} - 4 f_{i-1} + 6 f_i - 4 f_{i+1} + f_{i+2})
            auto f5 = [&](double a0, double a1, double a2, double a3, double a4) {
                return a2 - sig16 * (a0 - 4.0 * a1 + 6.0 * a2 - 4.0 * a3 + a4);
            };
            if (fwin) {
                qo = f5(xq[i], xq[i + 1], xq[i + 2], xq[i + 3], xq[i + 4]);
                wo = f5(xw[i], xw[i + 1], xw[i + 2], xw[i + 3], xw[i + 4]);
            } else {
                double fq[5], fw[5];
#pragma unroll
                for (int k = -2; k <= 2; k++) {
                    int rr = r + k;
                    double pq = 1.0;
                    if (rr < 0) {            // only at a physical left boundary
                        if (P.bcl == BC_WALL) { rr = -1 - rr; pq = -1.0; } else rr = 0;
                    } else if (rr >= L) {    // only at a physical right boundary
                        if (P.bcr == BC_WALL) { rr = 2 * L - 1 - rr; pq = -1.0; } else rr = L - 1;
                    }
                    fq[k + 2] = pq * sQb[rr];
                    fw[k + 2] = sWb[rr];
                }
                qo = f5(fq[0], fq[1], fq[2], fq[3], fq[4]);
                wo = f5(fw[0], fw[1], fw[2], fw[3], fw[4]);
            }
        }
        if (early) {
            const double u = fabs(qo * ihv[i]);
            const double nu = u + sqv[i];
            acc.umax = (kept && u > acc.umax) ? u : acc.umax;
            acc.numax = (kept && nu > acc.numax) ? nu : acc.numax;
            smem[5 * SROWS + r] = qo; smem[7 * SROWS + r] = wo;
            continue;
        }
        double h0 = hb[i];
        const double Hb = HdD[i] * (h0 * h0);
        double Ko = BATHY ? Hb + 1.5 * h0 * bbv[i] : Hb;
        if (fin && RELAX) {
            relax_cell(P, P.x_min + (double(s_cell + (r - klo)) + 0.5) * P.dx, bbv[i], t_new, h0, qo, Ko, wo);
            const double Hf = Ko - 1.5 * h0 * bbv[i];
            const double ih = rcp(h0);
            const double u = fabs(qo * ih), sg = Hf * ih * ih;
            const double nu = u + fsqrt(g * h0 + lam3 * sg * sg);
            acc.umax = u > acc.umax ? u : acc.umax;
            acc.numax = nu > acc.numax ? nu : acc.numax;
        } else if (fin) {
            const double u = fabs(qo * ihv[i]), sg = HdD[i];
            const double nu = u + fsqrt(g * h0 + lam3 * sg * sg);
            acc.umax = (kept && u > acc.umax) ? u : acc.umax;
            acc.numax = (kept && nu > acc.numax) ? nu : acc.numax;
        }
        // staging arrays 4..7 are not read in this phase; every row is staged at
        // its own index r (no mask), store_tile writes rows [klo, khi)
        smem[4 * SROWS + r] = h0; smem[5 * SROWS + r] = qo;
        smem[6 * SROWS + r] = Ko; smem[7 * SROWS + r] = wo;
    }
    // truncated overlap widths for the overlap check
    const int wt = min(left_phys ? 1 << 30 : G.wl, right_phys ? 1 << 30 : G.wr);
    acc.wmin = min(acc.wmin, wt);
}

// Store the staged rows (arrays 4..7, index klo .. klo+Tk-1) to out[] at cells
// [s, s + Tk): bulk (thread 0; read-completion wait deferred) or per element.
__device__ __forceinline__ void store_tile(const Bufs &B, size_t mo, int s, int Tk, int klo)
{
    const int tid = threadIdx.x;
    const size_t gdst = mo + size_t(s);
    const bool bulk_out = ((gdst | size_t(Tk) | size_t(klo)) & 1) == 0;
    double *const smem = dyn_smem() + klo;
    double *const oh = smem + 4 * SROWS, *const oq = smem + 5 * SROWS, *const oK = smem + 6 * SROWS,
                 *const oW = smem + 7 * SROWS;
    if (bulk_out) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            const unsigned bytes = unsigned(Tk) * 8u;
            bulk_s2g(B.out[0] + gdst, oh, bytes);
            bulk_s2g(B.out[1] + gdst, oq, bytes);
            bulk_s2g(B.out[2] + gdst, oK, bytes);
            bulk_s2g(B.out[3] + gdst, oW, bytes);
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    } else {
        __syncthreads();
        for (int k = tid; k < Tk; k += NT) {
            B.out[0][gdst + k] = oh[k]; B.out[1][gdst + k] = oq[k];
            B.out[2][gdst + k] = oK[k]; B.out[3][gdst + k] = oW[k];
        }
    }
}

// Member already at t_end (dt = 0): carry the state of kept cells [s, e) and
// its dt maxima.
template <bool FINAL, bool BATHY>
__device__ __forceinline__ void carry_tile(const Params &P, const Bufs &B, size_t mo, int s, int e,
                                           double lam, TileAcc &acc)
{
    const double lam3 = lam * (1.0 / 3.0);
    for (int i = s + threadIdx.x; i < e; i += NT) {
        const double h = B.Un[0][mo + i], q = B.Un[1][mo + i], K = B.Un[2][mo + i], W = B.Un[3][mo + i];
        B.out[0][mo + i] = h; B.out[1][mo + i] = q; B.out[2][mo + i] = K; B.out[3][mo + i] = W;
        if (FINAL) {
            const double bb = BATHY ? __ldg(P.b + i) : 0.0;
            const double ih = rcp(h);
            const double u = q * ih, sg = (K - 1.5 * h * bb) * ih * ih;
            acc.umax = fmax(acc.umax, fabs(u));
            acc.numax = fmax(acc.numax, fabs(u) + fsqrt(P.g * h + lam3 * sg * sg));
        }
    }
}

// Per-tile epilogue: error bits, overlap check (r^w <= 2^-60 at each truncated
// end), dt maxima of the member (final stage) and its next
// time level (tile 0).
template <bool FINAL>
// tm0, tend0: t^n of the member and t_end, read at the CTA's start by tile 0 of
// a final stage (negative: read here) -- keeps their latency out of the serial tail
__device__ __forceinline__ void tile_epilogue(const Params &P, int j, int m, double dtm, const TileAcc &acc,
                                              double tm0 = -1.0, double tend0 = -1.0)
{
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int members = P.members;
    const unsigned int eb = __reduce_or_sync(0xffffffffu, acc.err);
    if (lane == 0 && eb) { atomicOr(P.err, eb); __threadfence(); }
    double um = 0.0, nm = 0.0;
    if (FINAL) { um = warp_max_nonneg(acc.umax); nm = warp_max_nonneg(acc.numax); }
    float rf = warp_max_nonneg(float(acc.rho));
    int km = __reduce_min_sync(0xffffffffu, acc.kkey);
    // (s_red is only used here; s_redf's last reads in phase 2 precede later barriers)
    if (lane == 0) { s_red[0][wid] = um; s_red[1][wid] = nm; s_redf[wid] = rf; s_redk[wid] = km; }
    __syncthreads();
    if (tid == 0) {
        for (int q = 1; q < NT / 32; q++) {
            um = s_red[0][q] > um ? s_red[0][q] : um; nm = s_red[1][q] > nm ? s_red[1][q] : nm;
            rf = s_redf[q] > rf ? s_redf[q] : rf;
            km = min(km, s_redk[q]);
        }
        if (km != 0x7fffffff && P.kmin) atomicMax(P.kmin, ~unsigned(km));
        if (rf > 0.0f && dtm != 0.0) {
            const double rho = double(rf) * (1.0 + 1e-6);
            if (acc.wmin == P.w) {
                // r(rho)^w <= 2^-60  <=>  rho <= rho_ok = r*/(1 - r*)^2, r* = 2^(-60/w) (host)
                if (rho > P.rho_ok) atomicOr(P.err, ERR_OVERLAP);
            } else if (acc.wmin < (1 << 30)) {
                const double rdec = 2.0 * rho / ((1.0 + 2.0 * rho) + sqrt(1.0 + 4.0 * rho));
                double x = 1.0, b = rdec;          // rdec^wmin by squaring
                for (int k = acc.wmin; k > 0; k >>= 1) { if (k & 1) x *= b; b *= b; }
                if (x > 8.673617379884035e-19) atomicOr(P.err, ERR_OVERLAP);   // 2^-60
            }
            atomicMax(P.rho_obs, (unsigned long long)__double_as_longlong(rho));
        }
        if (FINAL) {
            const int slot_w = (P.kslot + 1) % 3;
            atomicMax(P.maxes + (slot_w * 2 + 0) * members + m, (unsigned long long)__double_as_longlong(um));
            atomicMax(P.maxes + (slot_w * 2 + 1) * members + m, (unsigned long long)__double_as_longlong(nm));
            if (j == 0) {   // t^{n+1} of this member, in the other parity slot
                const double tm = tm0 >= 0.0 ? tm0 : P.t[P.kpar * members + m];
                const double t_end = tend0 >= 0.0 ? tend0 : P.ctrl->t_end;
                P.t[(P.kpar ^ 1) * members + m] = (t_end > 0.0 && dtm == t_end - tm) ? t_end : tm + dtm;
            }
        }
    }
}

__device__ __forceinline__ void init_mbar(unsigned mb)
{
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Standalone stage kernel: one IMEX stage over every (tile, member) CTA.
// STAGE2: inputs U^n and U1 (E, R formed on load); FINAL: this stage produces
// U^{n+1} (filter, relaxation, dt maxima, time level).  The default kernel
// organisation of the overlapped tiles.
// ---------------------------------------------------------------------------
#if HSGN_EXP_TIMING
#define EXP_T(v) long long v = clock64()
#else
#define EXP_T(v)
#endif

// FDT: the small-ensemble kernels (at most two waves of CTAs, Params::fuse_dt):
// the step's first stage computes the step's dt itself, and both stages keep
// the 4-CTA register-resident form (stage_body LAT)
template <bool STAGE2, bool FINAL, bool BATHY, bool RELAX = false, bool PIC = false, bool WB = false,
          bool FDT = false>
__global__ void __launch_bounds__(NT, FDT ? HSGN_MINB
                                     : (!STAGE2 && !FINAL && !BATHY && !PIC && !WB) ? HSGN_MINB1
                                     : (STAGE2 && FINAL && !BATHY && !RELAX && !PIC && !WB) ? HSGN_MINB2 : HSGN_MINB)
    stage_kernel(const Params P, const Bufs B)
{
    EXP_T(t0);
    const int tid = threadIdx.x;
    const int j = blockIdx.x;        // tile
    // member: the second stage walks the members backwards, so its first CTAs read the
    // U1 rows the first stage wrote last (and the next first stage, forwards, the U^{n+1}
    // rows written last) while they are still in L2
    const int m = STAGE2 ? P.members - 1 - int(blockIdx.y) : int(blockIdx.y);
    const size_t mo = size_t(m) * P.n;
    const int s = j * P.T;
    const int e = min(P.n, s + P.T);
    Geom G = stage_geom(P, s, e, P.w);
    const LoadPlan Lp = load_plan(P, mo, G);
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&s_mbar);
    // thread 0 initialises the mbarrier and issues the tile's TMA loads at once;
    // the barrier that publishes the initialised mbarrier to the other threads
    // comes after the issue, off the loads' critical path
    if (Lp.bulk && tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    issue_load<STAGE2, LD_ALL, BATHY>(P, B, mo, G, Lp, mb, tid);
    if (Lp.bulk) __syncthreads();
    // ---- run control: dt of this member was set by dt_commit_kernel, or (the
    // step's first stage with fuse_dt) is computed here by its rule from the
    // previous step's maxima, the loads overlapping the tile's TMA copies; tile
    // 0 stores it and frees the maxima slot of two steps back, tile 0 of
    // member 0 commits the previous step (one launch per step fewer)
    const unsigned int err0 = *((volatile unsigned int *)P.err);
    double dtm;
    if (!STAGE2 && FDT) {
        dtm = member_dt(P, P.kslot, P.kpar, m);
        if (j == 0 && tid == 0 && err0 == 0u) {
            if (m == 0 && P.commit_prev) *P.steps += 1;
            if (dtm < 0.0) {
                atomicOr(P.err, ERR_DT);
            } else {
                const int slot_z = (P.kslot + 2) % 3;
                P.dt[m] = dtm;
                P.maxes[(slot_z * 2 + 0) * P.members + m] = 0ull;
                P.maxes[(slot_z * 2 + 1) * P.members + m] = 0ull;
            }
        }
    } else {
        dtm = P.dt[m];
    }
    const double lam = P.lam[m];
    double tm0 = -1.0, tend0 = -1.0;             // (tile_epilogue: t^{n+1} of tile 0)
    if (FINAL && j == 0 && tid == 0) { tm0 = P.t[P.kpar * P.members + m]; tend0 = P.ctrl->t_end; }
    unsigned parity = 0u;
    wait_load(Lp, mb, parity);
    if (BATHY && Lp.bulk && (Lp.a0 & 1)) cp_async_wait_all();    // b by cp.async (issue_load)
    __syncthreads();
    EXP_T(t1);
    if (err0 || dtm < 0.0) return;

    TileAcc acc{0.0, 0.0, 0.0, 0u, 1 << 30, 0};
    if (dtm == 0.0) {
        carry_tile<FINAL, BATHY>(P, B, mo, s, e, lam, acc);
    } else {
        const StageC S = stage_consts(P, STAGE2 ? P.aI2 : P.aI1, dtm, lam);
        stage_body<STAGE2, FINAL, BATHY, RELAX, PIC, WB, FDT>(P, B, G, m, s, S, dtm, acc);
        store_tile(B, mo, s, e - s, G.klo);
    }
    EXP_T(t2);
    tile_epilogue<FINAL>(P, j, m, dtm, acc, tm0, tend0);
    // shared memory must outlive the bulk stores' reads (no-op if none)
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
#if HSGN_EXP_TIMING
    if (tid == 0) {
        const long long t3 = clock64();
        unsigned long long *g = g_exp + (STAGE2 ? 8 : 0);
        atomicAdd(g + 0, (unsigned long long)(t1 - t0));
        atomicAdd(g + 1, (unsigned long long)(t2 - t1));
        atomicAdd(g + 2, (unsigned long long)(t3 - t2));
        atomicAdd(g + 3, 1ull);
        if (dtm != 0.0) {
            atomicAdd(g + 4, (unsigned long long)(s_tph[0] - t1));
            atomicAdd(g + 5, (unsigned long long)(s_tph[1] - s_tph[0]));
            atomicAdd(g + 6, (unsigned long long)(t2 - s_tph[1]));
            atomicAdd(g + 7, (unsigned long long)(s_tph[1] - s_tph[2]));   // PCR + recovery
        }
    }
#endif
}

// ---------------------------------------------------------------------------
// Explicit hSGN scheme, flat bottom:
//   L_h = -D_x(q),  L_q = -D^_x(q u) - a^2 D_x(h) - lam alpha D_x(h eta),
//   L_H = -D^_x(H u) + W,  L_W = -D^_x(W u) - lam (H/h^2 - 1)
// D_x centred over i+-1, D^_x the Rusanov difference of the MUSCL face
// states (A4, A5: the same faces as the SI predictor), a^2, alpha
// at cell i.  Euler: U + dt L(U); Heun: U1 = U + dt L(U),
// U^{n+1} = (U + U1 + dt L(U1)) / 2; then the optional A19 filter on q, W.
//
// explicit_kernel<HEUN2, FINAL, FILT>: one CTA per tile of XT kept cells of one
// member; the stencil input X (U^n, or U1 for HEUN2) is TMA-loaded into shared
// memory with R = 2 (+2 with the filter) halo rows; the base U^n is read per
// cell from global memory.  Thread t owns rows t, t + XNT, ... (consecutive
// threads on consecutive rows: conflict-free shared accesses, coalesced
// global stores).  With the filter the final q, W of rows -2 .. XT+1 are
// computed (the 4 halo rows redundantly) into shared memory first.
// ---------------------------------------------------------------------------
constexpr int XNT = 256;                 // threads per CTA
#ifndef HSGN_XMINB
#define HSGN_XMINB 3
#endif
constexpr int XMINB = HSGN_XMINB;        // CTAs per SM the registers allow
constexpr int XT = 1024;                 // kept cells per tile
constexpr int XR = 4;                    // halo rows of X (filter: 2 + 2)
constexpr int XROWS = XT + 2 * XR + 8;   // shared rows per X array (+ alignment)
constexpr int XFROWS = XT + 8;           // shared rows of the filter arrays
constexpr size_t XSMEM_BYTES = (size_t(4) * XROWS + 4 * size_t(XFROWS)) * sizeof(double);   // FILT
constexpr size_t XSMEM_BYTES_NF = size_t(4) * XROWS * sizeof(double);                        // no filter

// L(X) at row r of the tile (rows r-2 .. r+2 of the shared arrays).
__device__ __forceinline__ void explicit_rhs(const double *xh, const double *xq, const double *xH,
                                             const double *xW, int r, double kap, double g,
                                             double lam, double idx, double ihdx, double out[4])
{
    double wh[3], wq[3], wH[3], wW[3];
    // face r-1/2: M_{r-1} (rows r-2..r) and Pl_r (rows r-1..r+1)
#pragma unroll
    for (int k = 0; k < 3; k++) { wh[k] = xh[r - 2 + k]; wq[k] = xq[r - 2 + k]; wH[k] = xH[r - 2 + k]; wW[k] = xW[r - 2 + k]; }
    const FState Mm = muscl_minus(wh, wq, wH, wW, kap);
#pragma unroll
    for (int k = 0; k < 3; k++) { wh[k] = xh[r - 1 + k]; wq[k] = xq[r - 1 + k]; wH[k] = xH[r - 1 + k]; wW[k] = xW[r - 1 + k]; }
    FState Pl, M0;
    muscl_pair(wh, wq, wH, wW, kap, Pl, M0);
    const Face Fl = rusanov(Mm, Pl);                       // 2 x flux at r-1/2
    // face r+1/2: M_r and Pl_{r+1} (rows r..r+2)
    const double h2 = xh[r + 2], q2 = xq[r + 2], H2 = xH[r + 2], W2 = xW[r + 2];
    const FState Pr = muscl_plus_next(wh, wq, wH, wW, h2, q2, H2, W2, kap);
    const Face Fr = rusanov(M0, Pr);                       // 2 x flux at r+1/2
    const double h = wh[1], H = wH[1], W = wW[1];
    const double ih = rcp(h);
    const double eta = H * ih, sg = eta * ih;                               // eta, eta/h
    const double alpha = -(2.0 * sg - 1.0) * ih * (1.0 / 3.0);
    const double a2 = g * h + lam * (1.0 / 3.0) * sg * sg - lam * eta * alpha;
    const double Dxq = (wq[2] - wq[0]) * ihdx, Dxh = (wh[2] - wh[0]) * ihdx;
    const double DxH = (wH[2] - wH[0]) * ihdx;
    const double hidx = 0.5 * idx;                          // faces carry 2F
    out[0] = -Dxq;
    out[1] = -(Fr.q - Fl.q) * hidx - a2 * Dxh - lam * alpha * DxH;
    out[2] = -(Fr.H - Fl.H) * hidx + W;
    out[3] = -(Fr.W - Fl.W) * hidx - lam * (sg - 1.0);     // H/h^2 = eta/h
}

template <bool HEUN2, bool FINAL, bool FILT>
__global__ void __launch_bounds__(XNT, XMINB) explicit_kernel(const Params P, const Bufs B)
{
    const int tid = threadIdx.x;
    const int j = blockIdx.x, m = blockIdx.y;
    const int n = P.n;
    const size_t mo = size_t(m) * n;
    const int s = j * P.T;
    const int e = min(n, s + P.T);
    const int Tk = e - s;
    constexpr int R = FILT ? XR : 2;           // halo rows of X needed
    constexpr int RO = FILT ? 2 : 0;           // halo rows of final values
    double *const smem = dyn_smem();
    const double *const *X = HEUN2 ? B.U1 : B.Un;
    // ---- load X rows -R .. Tk+R-1 (TMA for interior tiles, 16-B aligned) -----
    const int a0r = s - R;
    const bool interior = (a0r >= 0) && (s + Tk + R <= n);
    const int d = interior ? int((mo + size_t(a0r)) & 1) : 0;
    const int cnt = (Tk + 2 * R + d + 1) & ~1;
    const bool bulk = interior && (a0r - d >= 0) && (a0r - d + cnt <= n);
    double *const A = smem + d + R;            // row r of array k at A[k * XROWS + r]
    double *xh = A, *xq = A + XROWS, *xH = A + 2 * XROWS, *xW = A + 3 * XROWS;
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&s_mbar);
    if (bulk) {
        init_mbar(mb);
        if (tid == 0) {
            const unsigned bytes = unsigned(cnt) * 8u;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes * 4u)
                         : "memory");
            const size_t gsrc = mo + size_t(a0r - d);
#pragma unroll
            for (int f = 0; f < 4; f++) bulk_g2s(smem + f * XROWS, X[f] + gsrc, bytes, mb);
        }
    } else {
        for (int r = tid - R; r < Tk + R; r += XNT) {
            double par;
            const size_t gi = mo + size_t(map_cell(s + r, n, P.bcl, P.bcr, par));
            cp_async8(xh + r, X[0] + gi); cp_async8(xq + r, X[1] + gi);
            cp_async8(xH + r, X[2] + gi); cp_async8(xW + r, X[3] + gi);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const unsigned int err0 = *((volatile unsigned int *)P.err);
    const double dtm = P.dt[m];
    const double lam = P.lam[m];
    if (bulk) mbar_wait(mb, 0);
    else cp_async_wait_all();
    __syncthreads();
    if (err0) return;
    // wall ghosts: q is odd (A10); the raw copies need the sign
    if (!interior && (P.bcl == BC_WALL || P.bcr == BC_WALL)) {
        for (int r = tid - R; r < Tk + R; r += XNT) {
            double par;
            (void)map_cell(s + r, n, P.bcl, P.bcr, par);
            xq[r] *= par;
        }
        __syncthreads();
    }
    const double kap = P.order == 2 ? 0.25 : 0.0;
    const double g = P.g, idx = P.idx, ihdx = 0.5 * P.idx;
    double umax = 0.0, numax = 0.0;
    unsigned int errbits = 0u;
    double *fq = smem + 4 * XROWS + 2, *fw = fq + XFROWS;   // final q, W rows -2 .. Tk+1 (filter)
    if (dtm == 0.0) {
        // member already at t_end: carry the state (and its dt maxima)
        for (int r = tid; r < Tk; r += XNT) {
            const size_t gi = mo + s + r;
            const double h = B.Un[0][gi], q = B.Un[1][gi], K = B.Un[2][gi], W = B.Un[3][gi];
            B.out[0][gi] = h; B.out[1][gi] = q; B.out[2][gi] = K; B.out[3][gi] = W;
            if (FINAL) {
                const double ih = rcp(h);
                const double u = fabs(q * ih), sg = K * ih * ih;
                const double nu = u + fsqrt(g * h + lam * (1.0 / 3.0) * sg * sg);
                umax = u > umax ? u : umax;
                numax = nu > numax ? nu : numax;
            }
        }
    } else {
    // ---- final values of rows -RO .. Tk+RO-1 ----------------------------------
    double *fh = fw + XFROWS, *fk = fh + XFROWS;            // final h, K of kept rows (filter)
    for (int r = tid - RO; r < Tk + RO; r += XNT) {
        const bool kept = r >= 0 && r < Tk;
        // base U^n first: its global loads overlap the flux arithmetic
        double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
        if (HEUN2) {
            const int c = s + r;
            double par = 1.0;
            const size_t gi = mo + size_t((c >= 0 && c < n) ? c : map_cell(c, n, P.bcl, P.bcr, par));
            b0 = B.Un[0][gi]; b1 = par * B.Un[1][gi]; b2 = B.Un[2][gi]; b3 = B.Un[3][gi];
        }
        double L[4];
        explicit_rhs(xh, xq, xH, xW, r, kap, g, lam, idx, ihdx, L);
        double o[4];
        if (HEUN2) {
            o[0] = 0.5 * b0 + 0.5 * (xh[r] + dtm * L[0]);
            o[1] = 0.5 * b1 + 0.5 * (xq[r] + dtm * L[1]);
            o[2] = 0.5 * b2 + 0.5 * (xH[r] + dtm * L[2]);
            o[3] = 0.5 * b3 + 0.5 * (xW[r] + dtm * L[3]);
        } else {
            o[0] = xh[r] + dtm * L[0];
            o[1] = xq[r] + dtm * L[1];
            o[2] = xH[r] + dtm * L[2];
            o[3] = xW[r] + dtm * L[3];
        }
        if (FILT) { fq[r] = o[1]; fw[r] = o[3]; }
        if (kept) {
            if (!(o[0] > P.h_min)) errbits |= ERR_DRY;
            if (!isfinite(o[0] + o[1] + o[2] + o[3])) errbits |= ERR_NONFINITE;
            if (FILT) {
                fh[r] = o[0]; fk[r] = o[2];
            } else {
                B.out[0][mo + s + r] = o[0]; B.out[1][mo + s + r] = o[1];
                B.out[2][mo + s + r] = o[2]; B.out[3][mo + s + r] = o[3];
            }
            if (FINAL && !FILT) {
                const double ih = rcp(o[0]);
                const double u = fabs(o[1] * ih), sg = o[2] * ih * ih;
                const double nu = u + fsqrt(g * o[0] + lam * (1.0 / 3.0) * sg * sg);
                umax = u > umax ? u : umax;
                numax = nu > numax ? nu : numax;
            }
        }
    }
    if (FILT) {
        __syncthreads();
        const double sig16 = P.filter_sigma * (1.0 / 16.0);
        // stencil rows reach a physical end only in the first / last two cells
        const bool near_phys = (P.bcl != BC_PERIODIC && s < 2) || (P.bcr != BC_PERIODIC && e + 2 > n);
        for (int r = tid; r < Tk; r += XNT) {
            // A19 on q and W; the halo rows are the neighbours' final values
            // (the mirror of the tile itself at a physical end, A10)
            double cq[5], cw[5];
            if (!near_phys) {
#pragma unroll
                for (int k = 0; k < 5; k++) { cq[k] = fq[r + k - 2]; cw[k] = fw[r + k - 2]; }
            } else {
#pragma unroll
            for (int k = 0; k < 5; k++) {
                const int c = s + r + k - 2;
                int rr = r + k - 2;
                double pq = 1.0;
                if (c < 0 && P.bcl != BC_PERIODIC) {
                    if (P.bcl == BC_WALL) { rr = -1 - c - s; pq = -1.0; } else rr = -s;
                } else if (c >= n && P.bcr != BC_PERIODIC) {
                    if (P.bcr == BC_WALL) { rr = 2 * n - 1 - c - s; pq = -1.0; } else rr = n - 1 - s;
                }
                cq[k] = pq * fq[rr];
                cw[k] = fw[rr];
            }
            }
            const double qo = cq[2] - sig16 * (cq[0] - 4.0 * cq[1] + 6.0 * cq[2] - 4.0 * cq[3] + cq[4]);
            const double wo = cw[2] - sig16 * (cw[0] - 4.0 * cw[1] + 6.0 * cw[2] - 4.0 * cw[3] + cw[4]);
            if (!isfinite(qo + wo)) errbits |= ERR_NONFINITE;
            const double h0 = fh[r], K0 = fk[r];
            B.out[0][mo + s + r] = h0; B.out[1][mo + s + r] = qo;
            B.out[2][mo + s + r] = K0; B.out[3][mo + s + r] = wo;
            if (FINAL) {
                const double ih = rcp(h0);
                const double u = fabs(qo * ih), sg = K0 * ih * ih;
                const double nu = u + fsqrt(g * h0 + lam * (1.0 / 3.0) * sg * sg);
                umax = u > umax ? u : umax;
                numax = nu > numax ? nu : numax;
            }
        }
    }
    }   // dtm != 0
    // ---- error bits, dt maxima, next time level --------------------------------
    const int lane = tid & 31, wid = tid >> 5;
    const unsigned int eb = __reduce_or_sync(0xffffffffu, errbits);
    if (lane == 0 && eb) { atomicOr(P.err, eb); __threadfence(); }
    if (FINAL) {
        __shared__ double xred[2][XNT / 32];
        const double um = warp_max_nonneg(umax), nm = warp_max_nonneg(numax);
        if (lane == 0) { xred[0][wid] = um; xred[1][wid] = nm; }
        __syncthreads();
        if (tid == 0) {
            double a = xred[0][0], b = xred[1][0];
            for (int q = 1; q < XNT / 32; q++) {
                a = xred[0][q] > a ? xred[0][q] : a;
                b = xred[1][q] > b ? xred[1][q] : b;
            }
            const int members = P.members;
            const int slot_w = (P.kslot + 1) % 3;
            atomicMax(P.maxes + (slot_w * 2 + 0) * members + m, (unsigned long long)__double_as_longlong(a));
            atomicMax(P.maxes + (slot_w * 2 + 1) * members + m, (unsigned long long)__double_as_longlong(b));
            if (j == 0) {
                const double tm = P.t[P.kpar * members + m];
                const double t_end = P.ctrl->t_end;
                P.t[(P.kpar ^ 1) * members + m] = (t_end > 0.0 && dtm == t_end - tm) ? t_end : tm + dtm;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Classical SGN scheme, flat bottom, on (h, q):
//   L_h = -D^_x(q),  L_q = -D^_x(q u + g h^2/2) + h phi,
//   h phi - (1/(3dx^2)) (c_{i+1/2}(phi_{i+1} - phi_i) - c_{i-1/2}(phi_i - phi_{i-1})) = h*,
// c = h_{i+1/2}^3 (h_{i+1/2} = (h_i + h_{i+1})/2), h* of P:591 with g h^3 (A23);
// Rusanov with alpha = max(|u| + sqrt(g h)) on MUSCL faces (A23).  K, W carried.
//
// sgn_kernel<HEUN2, FINAL>: tiles of ST kept cells with an overlap of w rows
// for the phi system (an M-matrix like the SI depth system: the same
// truncation argument and per-CTA decay check); SNT
// threads own MCH-row chunks (partition method in registers, PCR on the SNT
// chunk ends in shared memory).  The phi decay length is ~h/sqrt(3), so w is
// ~ 40 (h/dx): the tile is 5 x 512 rows.
// ---------------------------------------------------------------------------
constexpr int SNT = 512;
constexpr int SLCAP = SNT * MCH;                 // 2560 rows
constexpr int SROWS_S = SLCAP + 16;
// shared: h, q (stencil input, rows -2-? .. L+?), staged outputs h, q, PCR 2 x 3 x SNT
constexpr size_t SSMEM_BYTES = (size_t(4) * SROWS_S + size_t(6) * SNT) * sizeof(double);
// with bathymetry: b of rows -4 .. L+3 in a fifth array (A26)
constexpr size_t SSMEM_BYTES_B = SSMEM_BYTES + size_t(SROWS_S) * sizeof(double);

template <bool HEUN2, bool FINAL, bool BATHY = false>
__global__ void __launch_bounds__(SNT, 1) sgn_kernel(const Params P, const Bufs B)
{
    __shared__ double xw[SNT / 32][3];
    __shared__ float rw[SNT / 32];
    __shared__ double rd[2][SNT / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int j = blockIdx.x, m = blockIdx.y;
    const int n = P.n;
    const size_t mo = size_t(m) * n;
    Geom G = stage_geom(P, j * P.T, min(n, j * P.T + P.T), P.w);
    const int start = G.start, L = G.L;
    double *const smem = dyn_smem();
    double *sh = smem + 4, *sq = sh + SROWS_S;                  // rows -4 .. L+3 (shift 4)
    double *oh = smem + 2 * SROWS_S, *oq = oh + SROWS_S;        // staged outputs
    double *pcr0 = smem + 4 * SROWS_S, *pcr1 = pcr0 + 3 * SNT;
    double *sb = smem + 4 * SROWS_S + 6 * SNT + 4;               // b rows -4 .. L+3 (BATHY)
    const double *const *X = HEUN2 ? B.U1 : B.Un;
    // ---- load rows -4 .. L+3 of (h, q) of X and, for Heun stage 2, the kept
    // rows of U^n's (h, q) into the output staging (read there by the row's own
    // thread before it writes the result); all by cp.async, q parity of wall
    // ghosts applied after the wait ---------------------------------------------
    for (int r = tid - 4; r < L + 4; r += SNT) {
        const int c = start + r;
        double par = 1.0;
        const size_t gi = mo + size_t((c >= 0 && c < n) ? c : map_cell(c, n, P.bcl, P.bcr, par));
        cp_async8(sh + r, X[0] + gi);
        cp_async8(sq + r, X[1] + gi);
        if (BATHY) cp_async8(sb + r, P.b + (gi - mo));             // (b: even at walls)
    }
    if (HEUN2) {
        const size_t g0 = mo + size_t(start + G.klo);
        for (int k = tid; k < G.khi - G.klo; k += SNT) {
            cp_async8(oh + k, B.Un[0] + g0 + k);
            cp_async8(oq + k, B.Un[1] + g0 + k);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const unsigned int err0 = *((volatile unsigned int *)P.err);
    const double dtm = P.dt[m];
    cp_async_wait_all();
    __syncthreads();
    if (err0) return;
    if ((start - 4 < 0 && P.bcl == BC_WALL) || (start + L + 4 > n && P.bcr == BC_WALL)) {
        for (int r = tid - 4; r < L + 4; r += SNT) {
            double par;
            (void)map_cell(start + r, n, P.bcl, P.bcr, par);
            sq[r] *= par;
        }
        __syncthreads();
    }
    const double g = P.g, dx = P.dx, idx = P.idx;
    const double c3 = 1.0 / (3.0 * dx * dx);
    const double s6 = 1.0 / (6.0 * dx * dx * dx);
    const double kap = P.order == 2 ? 0.25 : 0.0;
    double umax = 0.0, numax = 0.0, rho_loc = 0.0;
    unsigned int errbits = 0u;
    const int r0 = tid * MCH;
    double phi[MCH];
    // ---- phi system on own rows (normalised by h_i), partition solve --------
    {
        // windows: h, u over rows r0-2 .. r0+MCH+1
        double wh[MCH + 4], wu[MCH + 4], wb[MCH + 4];
#pragma unroll
        for (int k = 0; k < MCH + 4; k++) {
            const int rr = min(r0 - 2 + k, L + 3);
            wh[k] = sh[rr];
            wu[k] = sq[rr] * rcp(wh[k]);
            wb[k] = BATHY ? sb[rr] : 0.0;
        }
        double am[MCH], cm[MCH], dm[MCH];
#pragma unroll
        for (int i = 0; i < MCH; i++) {
            const int r = r0 + i;
            const double h0 = wh[i + 2], hp = wh[i + 3], hm = wh[i + 1];
            const double hl = 0.5 * (hm + h0), hr = 0.5 * (h0 + hp);
            const double ih0 = rcp(h0);
            double rl = hl * hl * hl * c3 * ih0, rr = hr * hr * hr * c3 * ih0;
            const double hp3 = hp * hp * hp, hm3 = hm * hm * hm;
            const double up2 = wu[i + 4] - wu[i + 2], um2 = wu[i + 2] - wu[i];
            double rhs, dg;
            double kfac = 1.0;               // (BATHY) decay-check factor for kappa < 0
            if (!BATHY) {
                rhs = -s6 * (g * hp3 * (wh[i + 4] - 2.0 * hp + h0) + 0.5 * hp3 * up2 * up2
                             - g * hm3 * (h0 - 2.0 * hm + wh[i]) - 0.5 * hm3 * um2 * um2) * ih0;
                dg = 1.0 + rl + rr;
            } else {
                // A26: zeta = h + b in the g-term; rho at rows r -+ 1, Q at row r, kappa
                auto z = [&](int k) { return wh[k] + wb[k]; };
                double rhb = -s6 * (g * hp3 * (z(i + 4) - 2.0 * z(i + 3) + z(i + 2)) + 0.5 * hp3 * up2 * up2
                                    - g * hm3 * (z(i + 2) - 2.0 * z(i + 1) + z(i)) - 0.5 * hm3 * um2 * um2);
                const double i2dx = 0.5 * idx, idx2 = idx * idx;
                auto rho = [&](int k) {           // at window row k
                    const double hj = wh[k], uj = wu[k];
                    const double bx = (wb[k + 1] - wb[k - 1]) * i2dx;
                    const double zx = (z(k + 1) - z(k - 1)) * i2dx;
                    const double bxx = (wb[k + 1] - 2.0 * wb[k] + wb[k - 1]) * idx2;
                    return -(hj * hj * bx / 2.0) * g * zx + hj * hj * hj * uj * uj * bxx;
                };
                const double u0 = wu[i + 2];
                const double bx = (wb[i + 3] - wb[i + 1]) * i2dx;
                const double zx = (z(i + 3) - z(i + 1)) * i2dx;
                const double zxx = (z(i + 3) - 2.0 * z(i + 2) + z(i + 1)) * idx2;
                const double bxx = (wb[i + 3] - 2.0 * wb[i + 2] + wb[i + 1]) * idx2;
                const double ux = (wu[i + 3] - wu[i + 1]) * i2dx;
                const double Q = (h0 / 2.0) * g * zxx - (3.0 * g * bx / 4.0) * zx + h0 * ux * ux
                                 + 1.5 * h0 * u0 * u0 * bxx;
                rhb += -(rho(i + 3) - rho(i + 1)) * i2dx - h0 * Q * bx;
                rhs = rhb * ih0;
                const double kap = (hr * hr * (wb[i + 3] - wb[i + 2]) - hl * hl * (wb[i + 2] - wb[i + 1])) * (0.5 * idx2)
                                   + 0.75 * h0 * bx * bx;
                dg = 1.0 + rl + rr + kap * ih0;
                // kappa < 0 weakens the diagonal dominance: scale the coupling in the
                // decay check; a non-positive h + kappa makes the phi operator singular
                if (kap < 0.0) {
                    if (!(h0 + kap > 0.0)) errbits |= ERR_COERC;
                    kfac = 1.0 / (1.0 + kap * ih0);
                }
            }
            // tile ends: truncated (overlap) or physical (phi ghost = p phi_0, A23)
            if (r == 0) {
                if (G.left_phys) dg -= rl * (P.bcl == BC_WALL ? -1.0 : 1.0);
                rl = 0.0;
            }
            if (r == L - 1) {
                if (G.right_phys) dg -= rr * (P.bcr == BC_WALL ? -1.0 : 1.0);
                rr = 0.0;
            }
            if (r >= L) { rl = 0.0; rr = 0.0; dg = 1.0; rhs = 0.0; }
            rho_loc = rr * kfac > rho_loc ? rr * kfac : rho_loc;
            const double a = -rl, c = -rr;
            if (i == 0) {
                const double inv = rcp(dg);
                am[0] = a * inv; cm[0] = c * inv; dm[0] = rhs * inv;
            } else {
                const double inv = rcp(dg - a * cm[i - 1]);
                am[i] = -a * am[i - 1] * inv;
                cm[i] = c * inv;
                dm[i] = (rhs - a * dm[i - 1]) * inv;
            }
        }
        const double aE = am[MCH - 1], cE = cm[MCH - 1], dE = dm[MCH - 1];
        double Pn = 0.0, Qn = 0.0, Rn = -1.0;
#pragma unroll
        for (int i = MCH - 2; i >= 0; i--) {
            const double Pi = dm[i] - cm[i] * Pn;
            const double Qi = am[i] - cm[i] * Qn;
            const double Ri = -cm[i] * Rn;
            dm[i] = Pi; am[i] = Qi; cm[i] = Ri;
            Pn = Pi; Qn = Qi; Rn = Ri;
        }
        double P1 = __shfl_down_sync(0xffffffffu, dm[0], 1);
        double Q1 = __shfl_down_sync(0xffffffffu, am[0], 1);
        double R1 = __shfl_down_sync(0xffffffffu, cm[0], 1);
        if (lane == 0) { xw[wid][0] = dm[0]; xw[wid][1] = am[0]; xw[wid][2] = cm[0]; }
        __syncthreads();
        if (lane == 31) {
            if (wid + 1 < SNT / 32) { P1 = xw[wid + 1][0]; Q1 = xw[wid + 1][1]; R1 = xw[wid + 1][2]; }
            else { P1 = 0.0; Q1 = 0.0; R1 = 0.0; }
        }
        double A_ = aE, C_ = -cE * R1, D_ = dE - cE * P1;
        if (tid == 0) A_ = 0.0;
        {
            const double ib = rcp(1.0 - cE * Q1);
            A_ *= ib; C_ *= ib; D_ *= ib;
        }
        double *cur = pcr0, *nxt = pcr1;
        cur[tid] = A_; cur[SNT + tid] = C_; cur[2 * SNT + tid] = D_;
        {
            const float ea = float(fabs(A_)), ec = float(fabs(C_));
            const float ev = warp_max_nonneg(ea > ec ? ea : ec);
            if (lane == 0) rw[wid] = ev;
        }
        __syncthreads();
        int lim = SNT;
        {
            float e0 = 0.0f;
#pragma unroll
            for (int q = 0; q < SNT / 32; q++) e0 = fmaxf(e0, rw[q]);
            if (e0 < 0.4f) {
                float ee = e0 * 1.1f;
                int sdl = 1;
                while (sdl < SNT && ee > 5.42e-20f) { ee = ee * ee * 1.1f; sdl <<= 1; }
                lim = sdl;
            }
        }
#pragma unroll 1
        for (int sd = 1; sd < lim; sd <<= 1) {
            const int km = tid - sd, kp = tid + sd;
            double Am = 0, Cm = 0, Dm = 0, Ap = 0, Cp = 0, Dp = 0;
            if (km >= 0) { Am = cur[km]; Cm = cur[SNT + km]; Dm = cur[2 * SNT + km]; }
            if (kp < SNT) { Ap = cur[kp]; Cp = cur[SNT + kp]; Dp = cur[2 * SNT + kp]; }
            const double ib = rcp(1.0 - A_ * Cm - C_ * Ap);
            const double An = -A_ * Am * ib;
            const double Cn = -C_ * Cp * ib;
            const double Dn = (D_ - A_ * Dm - C_ * Dp) * ib;
            A_ = An; C_ = Cn; D_ = Dn;
            nxt[tid] = A_; nxt[SNT + tid] = C_; nxt[2 * SNT + tid] = D_;
            __syncthreads();
            double *tmp = cur; cur = nxt; nxt = tmp;
        }
        const double Xk = D_;
        double XL = __shfl_up_sync(0xffffffffu, Xk, 1);
        if (lane == 31) xw[wid][0] = Xk;
        __syncthreads();
        if (lane == 0) XL = (wid > 0) ? xw[wid - 1][0] : 0.0;
#pragma unroll
        for (int i = 0; i < MCH; i++) phi[i] = (i == MCH - 1) ? Xk : dm[i] - am[i] * XL - cm[i] * Xk;
    }
    // ---- shallow-water update of own kept rows ----------------------------------
    {
        double wh[3], wq[3], wH[3], wW[3];     // (H, W unused: zero, keep the MUSCL helpers)
#pragma unroll
        for (int k = 0; k < 3; k++) { wh[k] = sh[r0 - 2 + k]; wq[k] = sq[r0 - 2 + k]; wH[k] = 0.0; wW[k] = 0.0; }
        FState Mm = muscl_minus(wh, wq, wH, wW, kap);
#pragma unroll
        for (int k = 0; k < 2; k++) { wh[k] = wh[k + 1]; wq[k] = wq[k + 1]; }
        wh[2] = sh[min(r0 + 1, L + 3)]; wq[2] = sq[min(r0 + 1, L + 3)];
        FState Pn, Mr;
        muscl_pair(wh, wq, wH, wW, kap, Pn, Mr);
        // Rusanov for the shallow-water fluxes: 2F with alpha = max(|u| + sqrt(g h))
        auto face = [&](const FState &a, const FState &b, double &Fh, double &Fq) {
            const double sa = fabs(a.u) + fsqrt(g * a.h), sb = fabs(b.u) + fsqrt(g * b.h);
            const double al = sa > sb ? sa : sb;
            Fh = (a.q + b.q) - al * (b.h - a.h);
            Fq = fma(a.q, a.u, fma(b.q, b.u, 0.5 * g * (a.h * a.h + b.h * b.h))) - al * (b.q - a.q);
        };
        double Fhl, Fql;
        face(Mm, Pn, Fhl, Fql);
        const double hidx = 0.5 * idx;
#pragma unroll
        for (int i = 0; i < MCH; i++) {
            const int r = r0 + i;
            const double hc = wh[1], qc = wq[1];
#pragma unroll
            for (int k = 0; k < 2; k++) { wh[k] = wh[k + 1]; wq[k] = wq[k + 1]; }
            const int rn = min(r + 2, L + 3);
            wh[2] = sh[rn]; wq[2] = sq[rn];
            FState Mn;
            muscl_pair(wh, wq, wH, wW, kap, Pn, Mn);
            double Fhr, Fqr;
            face(Mr, Pn, Fhr, Fqr);
            Mr = Mn;
            if (r >= G.klo && r < G.khi) {
                const double Lh = -(Fhr - Fhl) * hidx;
                double Lq = -(Fqr - Fql) * hidx + hc * phi[i];
                if (BATHY) Lq -= g * hc * (sb[r + 1] - sb[r - 1]) * hidx;          // A26 hydrostatic source
                double ho, qo;
                if (HEUN2) {
                    ho = 0.5 * oh[r - G.klo] + 0.5 * (hc + dtm * Lh);
                    qo = 0.5 * oq[r - G.klo] + 0.5 * (qc + dtm * Lq);
                } else {
                    ho = hc + dtm * Lh;
                    qo = qc + dtm * Lq;
                }
                if (!(ho > P.h_min)) errbits |= ERR_DRY;
                if (!isfinite(ho + qo)) errbits |= ERR_NONFINITE;
                oh[r - G.klo] = ho; oq[r - G.klo] = qo;
                if (FINAL) {
                    const double u = fabs(qo * rcp(ho));
                    const double nu = u + fsqrt(g * ho);
                    umax = u > umax ? u : umax;
                    numax = nu > numax ? nu : numax;
                }
            }
            Fhl = Fhr; Fql = Fqr;
        }
    }
    __syncthreads();
    {
        const int Tk = G.khi - G.klo;
        const size_t gdst = mo + size_t(G.start + G.klo);
        for (int k = tid; k < Tk; k += SNT) {
            B.out[0][gdst + k] = oh[k]; B.out[1][gdst + k] = oq[k];
            if (FINAL) {                // K, W carried into U^{n+1} (not needed in U1)
                B.out[2][gdst + k] = B.Un[2][gdst + k];
                B.out[3][gdst + k] = B.Un[3][gdst + k];
            }
        }
    }
    // ---- error bits, overlap check, dt maxima, time level ---------------------
    const unsigned int eb = __reduce_or_sync(0xffffffffu, errbits);
    if (lane == 0 && eb) { atomicOr(P.err, eb); __threadfence(); }
    double um = 0.0, nm = 0.0;
    if (FINAL) { um = warp_max_nonneg(umax); nm = warp_max_nonneg(numax); }
    const float rf = warp_max_nonneg(float(rho_loc));
    if (lane == 0) { rd[0][wid] = um; rd[1][wid] = nm; rw[wid] = rf; }
    __syncthreads();
    if (tid == 0) {
        float r = rw[0];
        for (int q = 1; q < SNT / 32; q++) {
            um = rd[0][q] > um ? rd[0][q] : um; nm = rd[1][q] > nm ? rd[1][q] : nm;
            r = rw[q] > r ? rw[q] : r;
        }
        um = rd[0][0] > um ? rd[0][0] : um; nm = rd[1][0] > nm ? rd[1][0] : nm;
        const int wmin = min(G.left_phys ? 1 << 30 : G.wl, G.right_phys ? 1 << 30 : G.wr);
        if (r > 0.0f && dtm != 0.0 && wmin < (1 << 30)) {
            const double rho = double(r) * (1.0 + 1e-6);
            const double rdec = 2.0 * rho / ((1.0 + 2.0 * rho) + sqrt(1.0 + 4.0 * rho));
            double x = 1.0, b = rdec;
            for (int k = wmin; k > 0; k >>= 1) { if (k & 1) x *= b; b *= b; }
            if (x > 8.673617379884035e-19) atomicOr(P.err, ERR_OVERLAP);
            atomicMax(P.rho_obs, (unsigned long long)__double_as_longlong(rho));
        }
        if (FINAL) {
            const int members = P.members;
            const int slot_w = (P.kslot + 1) % 3;
            atomicMax(P.maxes + (slot_w * 2 + 0) * members + m, (unsigned long long)__double_as_longlong(um));
            atomicMax(P.maxes + (slot_w * 2 + 1) * members + m, (unsigned long long)__double_as_longlong(nm));
            if (j == 0) {
                const double tm = P.t[P.kpar * members + m];
                const double t_end = P.ctrl->t_end;
                P.t[(P.kpar ^ 1) * members + m] = (t_end > 0.0 && dtm == t_end - tm) ? t_end : tm + dtm;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Between steps: commit step k-1 (steps += 1 unless an error was latched) and
// set dt of step k for every member from the max|u|, max(|u|+c) of U^k
// (A7), clipped to t_end; free the maxima slot read at
// step k-1 (3-slot rotation, slot = k mod 3 is read, k+1 written).
// Slots and time parity come from the host's step index k (kslot = k mod 3,
// kpar = k mod 2), so no kernel reads a device step counter.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) dt_commit_kernel(const Params P, int commit_prev,
                                                        int compute_dt)
{
    const unsigned int err = *((volatile unsigned int *)P.err);
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid == 0 && commit_prev && err == 0u) *P.steps += 1;
    if (err || !compute_dt) return;
    const int m = tid;
    const int members = P.members;
    if (m >= members) return;
    const int slot_z = (P.kslot + 2) % 3;
    const double dtm = member_dt(P, P.kslot, P.kpar, m);
    if (dtm < 0.0) {
        atomicOr(P.err, ERR_DT);
        return;
    }
    P.dt[m] = dtm;
    P.maxes[(slot_z * 2 + 0) * members + m] = 0ull;
    P.maxes[(slot_z * 2 + 1) * members + m] = 0ull;
}

// ---------------------------------------------------------------------------
// Per-(tile, member) reductions of a state: mass partial sums (deterministic,
// summed on the host), min h, max|u|, max(|u|+c).  Optionally seeds the dt
// maxima slot 0 (after hsgn_set_state).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) reduce_kernel(const double *__restrict__ h,
                                                    const double *__restrict__ q,
                                                    const double *__restrict__ K,
                                                    const double *__restrict__ b,
                                                    const double *__restrict__ lamv, int n, int T,
                                                    double g, double *partials,
                                                    unsigned long long *maxes, int members,
                                                    int sgn)
{
    // sgn: 1 = celerity of the classical SGN scheme, sqrt(g h);
    // 2 = as 1 with partials[2] = max h instead of max |u| (SGN tile geometry)
    __shared__ double red[NT / 32 + 1];
    __shared__ double sred[NT];
    const int j = blockIdx.x, m = blockIdx.y, tid = threadIdx.x;
    const int s = j * T, e = min(n, s + T);
    const size_t mo = size_t(m) * n;
    const double lam = lamv[m];
    double sum = 0.0, mn = 1e300, um = 0.0, nm = 0.0;
    for (int i = s + tid; i < e; i += NT) {
        const double hh = h[mo + i], qq = q[mo + i];
        const double bb = b ? b[i] : 0.0;
        const double H = K[mo + i] - 1.5 * hh * bb;
        const double u = qq / hh, sg = H / hh / hh;
        sum += hh;
        mn = fmin(mn, hh);
        um = fmax(um, sgn == 2 ? hh : fabs(u));
        nm = fmax(nm, fabs(u) + sqrt(g * hh + (sgn ? 0.0 : (lam / 3.0) * sg * sg)));
    }
    // deterministic tree sum
    sred[tid] = sum;
    __syncthreads();
    int p2 = 1;
    while (p2 < NT) p2 <<= 1;                 // any NT (tuning builds use NT = 160, 192)
    for (int o = p2 / 2; o > 0; o >>= 1) {
        if (tid < o && tid + o < NT) sred[tid] += sred[tid + o];
        __syncthreads();
    }
    const double tot = sred[0];
    __syncthreads();
    const double mnn = -block_max(-mn, red, -1e300);
    const double umm = block_max(um, red);
    const double nmm = block_max(nm, red);
    if (tid == 0) {
        const size_t o = (size_t(m) * gridDim.x + j) * 4;
        partials[o + 0] = tot;
        partials[o + 1] = mnn;
        partials[o + 2] = umm;
        partials[o + 3] = nmm;
        if (maxes) {
            atomicMax(maxes + 0 * members + m, (unsigned long long)__double_as_longlong(umm));
            atomicMax(maxes + 1 * members + m, (unsigned long long)__double_as_longlong(nmm));
        }
    }
}

}  // namespace hsgn
