/*
 * hsgn_oracle.c -- plain, slow, fp64 CPU ORACLE of the semi-implicit IMEX step
 * of the hyperbolised Serre-Green-Naghdi (hSGN) system, arXiv 2510.07539.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2510_07539_b200/, libhsgn.so) never links, imports or calls it, and it
 * shares no code, header, constant or helper with the CUDA path.
 *
 * Written as straight loops over fp64 arrays, in the order of the paper's
 * equations, with no blocking, fusion or reordering.  Build with
 *   gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 * so that no FMA contraction happens.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n;
 * "Ak" = reading k of the ambiguity ledger in DESIGN.md (section 3).
 *
 * State per cell (D1 of DESIGN.md): h, q = hu, K, W = hw, where
 * K = h*eta (flat bottom) or K = h*eta~ with eta~ = eta + 3b/2.
 * Internally H := K - 1.5*h*b = h*eta; with b == 0, H == K.
 *
 * Every function here is pinned by a test in tests/test_oracle_*.py against
 * something other than itself (closed forms, the paper's printed numbers,
 * dense LU, Fourier symbols derived from the paper); see DESIGN.md section 4:
 *   SI stage / step / run, dt, filter, relaxation zones: test_oracle_pins.py
 *   explicit hSGN scheme (A22): test_oracle_explicit.py
 *   classical SGN scheme (A23): test_oracle_sgn.py; bathymetric closure (A26):
 *     test_oracle_sgnb.py (against the primitive model of P:175-186)
 *   well-balanced face form (A25): test_oracle_wb.py
 *   Picard passes (A24): test_oracle_picard.py (contraction, rest, mass, time
 *     order) and test_oracle_pins_ops.py (the fixed point equals a dense
 *     Newton solve of the un-frozen depth equation P:268-285 in numpy)
 *   A19 filter and A10 relaxation zones: test_oracle_pins_ops.py (single-mode
 *     symbol, mask, walls; ramp and target against a numpy evaluation)
 * tools/mutation_check.py applies 44 plausible mistakes; every one fails a pin.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- status codes (oracle-local; numerically equal to the product's, by
 * choice, so tests can compare them, but defined independently here) ---- */
#define ORC_OK 0
#define ORC_E_INVALID (-1)
#define ORC_E_DRY (-2)
#define ORC_E_COERCIVITY (-3)
#define ORC_E_SINGULAR (-4)
#define ORC_E_NONFINITE (-5)

/* boundary kinds (A10) */
#define ORC_BC_PERIODIC 0
#define ORC_BC_WALL 1
#define ORC_BC_TRANSMISSIVE 2

/* Problem description, mirrored by a ctypes.Structure in oracle/oracle.py. */
typedef struct {
    int32_t n;          /* number of cells */
    int32_t bc_left;    /* ORC_BC_* */
    int32_t bc_right;   /* ORC_BC_* (periodic requires both periodic) */
    int32_t order;      /* 1: piecewise constant faces, 2: MUSCL */
    double dx;          /* uniform spacing */
    double g;           /* gravity (A14: m/s^2) */
    double lambda;      /* relaxation parameter */
    double h_min;       /* dry-bed floor */
    const double *b;    /* bathymetry at cell centres, length n, or NULL (flat) */
    double filter_sigma;/* A19 filter strength, 0 = off */
    int32_t filter_mask;/* bit1 = q, bit3 = W (bit0 h, bit2 K also accepted) */
    int32_t pad_;
    /* relaxation zones (A10, cfg4), applied after each step at the new time t:
     * U -= s(x) (U - U_target).  x of cell i = x_min + (i + 1/2) dx.
     * Wavemaker zone x <= gen_x1: s = gen_rate (1 - (x - x_min)/(gen_x1 - x_min))^2,
     *   target eta = amp sin(omega t - k (x - x_min)): h = level + eta - b,
     *   u = cp eta / level, h eta_aux = h^2 (+1.5 h b in K), w = 0.
     * Sponge zone x >= sp_x0: s = sp_rate ((x - sp_x0)/(x_max - sp_x0))^2, target
     *   lake at rest h = level - b, q = 0, K = h (h + 1.5 b), W = 0.
     * A rate <= 0 switches a zone off. */
    double x_min, level;
    double gen_x1, gen_rate, amp, omega, k, cp;
    double sp_x0, sp_rate;
    /* Picard re-linearisation of the depth equation (reading A24, SURVEY row
     * f4): after the first solve, `picard` more assemble+solve passes with
     * beta1 = 1 + lam tau^2/h^2 and beta2 = 2 lam tau^2/(beta1^2 h^3) taken at
     * the latest hbar (alpha, a^2 stay at E); 0 = the paper's linearised stage. */
    int32_t picard;
    /* Exactly well-balanced variant (reading A25): face-based
     * delta_{i+1/2} in the depth right-hand side and qbar from face-averaged
     * face fluxes, so that the lake at rest is kept to round-off at lam > 0. */
    int32_t wb;
} orc_problem;

/* Double Butcher tableau. */
typedef struct {
    int32_t stages;     /* 1 (SI Euler, P:213-216 / P:500-517) or 2 */
    int32_t pad_;
    double aE[2][2];    /* explicit, strictly lower triangular */
    double aI[2][2];    /* implicit, lower triangular, a_ii > 0 */
    double b[2];        /* weights (equal for both tableaus) */
} orc_tableau;

/* ------------------------------------------------------------------------ */
/* Pointwise algebra of the hSGN model                                       */
/* ------------------------------------------------------------------------ */

/* c^2 = g h + (lambda/3) (eta/h)^2, eta = H/h. */
double orc_celerity(double g, double lambda, double h, double H)
{
    double eta_over_h = (H / h) / h;
    return sqrt(g * h + (lambda / 3.0) * eta_over_h * eta_over_h);
}

/*
 * Coefficients of the implicit depth equation at one cell,
 * with alpha and a^2 from P:142-143:
 *   alpha = -(1/(3h)) (2 eta/h - 1)
 *   a^2   = c^2 - lambda eta alpha
 *   beta1 = 1 + lambda tau^2 / h^2
 *   beta2 = 2 lambda tau^2 / (beta1^2 h^3)
 *   beta  = a^2 + lambda alpha beta2 (h eta)^dagger   (this is kappa)
 *   delta = alpha / beta1
 * h, H are the stage's explicit input E (A2); Hdag is the predictor (h eta)^dagger.
 * out = {alpha, a2, beta1, beta2, beta, delta}.
 */
void orc_coeffs(double g, double lambda, double tau, double h, double H, double Hdag,
                double out[6])
{
    double eta = H / h;
    double sigma = eta / h;                                   /* eta/h */
    double alpha = -(1.0 / (3.0 * h)) * (2.0 * sigma - 1.0);
    double c2 = g * h + (lambda / 3.0) * sigma * sigma;
    double a2 = c2 - lambda * eta * alpha;
    double beta1 = 1.0 + lambda * tau * tau / (h * h);
    double beta2 = 2.0 * lambda * tau * tau / (beta1 * beta1 * h * h * h);
    double beta = a2 + lambda * alpha * beta2 * Hdag;
    double delta = alpha / beta1;
    out[0] = alpha;
    out[1] = a2;
    out[2] = beta1;
    out[3] = beta2;
    out[4] = beta;
    out[5] = delta;
}

/*
 * Rusanov flux of the convective part R_E at one face (A4):
 *   F^ = 1/2 (F(U-) + F(U+)) - 1/2 alpha (U+ - U-),  alpha = max(|u-|, |u+|)
 * with F^q = q u, F^H = H u (= h u eta), F^W = W u (= h u w), u = q/h.
 * vm, vp = face states (h, q, H, W); out = (F^q, F^H, F^W).
 */
void orc_rusanov_face(const double vm[4], const double vp[4], double out[3])
{
    double um = vm[1] / vm[0], up_ = vp[1] / vp[0];
    double a = fabs(um) > fabs(up_) ? fabs(um) : fabs(up_);
    out[0] = 0.5 * (vm[1] * um + vp[1] * up_) - 0.5 * a * (vp[1] - vm[1]);
    out[1] = 0.5 * (vm[2] * um + vp[2] * up_) - 0.5 * a * (vp[2] - vm[2]);
    out[2] = 0.5 * (vm[3] * um + vp[3] * up_) - 0.5 * a * (vp[3] - vm[3]);
}

/* ------------------------------------------------------------------------ */
/* Tridiagonal solvers (the depth system Delta[h] = h^dagger, A3) */
/* ------------------------------------------------------------------------ */

/* Thomas algorithm: lo[i] x[i-1] + di[i] x[i] + up[i] x[i+1] = rhs[i],
 * lo[0] and up[n-1] ignored.  Returns ORC_E_SINGULAR on a zero pivot. */
int orc_thomas(int n, const double *lo, const double *di, const double *up,
               const double *rhs, double *x)
{
    if (n < 1) return ORC_E_INVALID;
    double *cp = (double *)malloc(sizeof(double) * (size_t)n);
    double *dp = (double *)malloc(sizeof(double) * (size_t)n);
    if (!cp || !dp) { free(cp); free(dp); return ORC_E_INVALID; }
    double piv = di[0];
    if (piv == 0.0) { free(cp); free(dp); return ORC_E_SINGULAR; }
    cp[0] = (n > 1 ? up[0] : 0.0) / piv;
    dp[0] = rhs[0] / piv;
    for (int i = 1; i < n; i++) {
        piv = di[i] - lo[i] * cp[i - 1];
        if (piv == 0.0) { free(cp); free(dp); return ORC_E_SINGULAR; }
        cp[i] = (i < n - 1 ? up[i] : 0.0) / piv;
        dp[i] = (rhs[i] - lo[i] * dp[i - 1]) / piv;
    }
    x[n - 1] = dp[n - 1];
    for (int i = n - 2; i >= 0; i--) x[i] = dp[i] - cp[i] * x[i + 1];
    free(cp);
    free(dp);
    return ORC_OK;
}

/* Cyclic tridiagonal: as orc_thomas plus corner couplings lo[0] (to x[n-1])
 * and up[n-1] (to x[0]); Sherman-Morrison rank-one correction. n >= 3. */
int orc_cyclic_thomas(int n, const double *lo, const double *di, const double *up,
                      const double *rhs, double *x)
{
    if (n < 3) return ORC_E_INVALID;
    double *bb = (double *)malloc(sizeof(double) * (size_t)n);
    double *u = (double *)malloc(sizeof(double) * (size_t)n);
    double *z = (double *)malloc(sizeof(double) * (size_t)n);
    if (!bb || !u || !z) { free(bb); free(u); free(z); return ORC_E_INVALID; }
    double alpha = up[n - 1];  /* A[n-1][0] */
    double beta = lo[0];       /* A[0][n-1] */
    double gam = -di[0];
    if (gam == 0.0) gam = -1.0;
    memcpy(bb, di, sizeof(double) * (size_t)n);
    bb[0] = di[0] - gam;
    bb[n - 1] = di[n - 1] - alpha * beta / gam;
    int st = orc_thomas(n, lo, bb, up, rhs, x);
    if (st == ORC_OK) {
        for (int i = 0; i < n; i++) u[i] = 0.0;
        u[0] = gam;
        u[n - 1] = alpha;
        st = orc_thomas(n, lo, bb, up, u, z);
    }
    if (st == ORC_OK) {
        double vx = x[0] + beta * x[n - 1] / gam;
        double vz = z[0] + beta * z[n - 1] / gam;
        double den = 1.0 + vz;
        if (den == 0.0) st = ORC_E_SINGULAR;
        else {
            double fact = vx / den;
            for (int i = 0; i < n; i++) x[i] = x[i] - fact * z[i];
        }
    }
    free(bb);
    free(u);
    free(z);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Ghost cells (A10)                                                */
/* ------------------------------------------------------------------------ */

/* ext has n + 2G entries, ext[G + i] = f[i].  parity = -1 for fields that are
 * odd under reflection at a wall (q), +1 otherwise.  Periodic wraps; wall
 * mirrors (ghost -k <-> cell k-1) with parity; transmissive copies the nearest
 * interior cell (zero-order extrapolation). */
static void fill_ghosts(const double *f, int n, int G, int bcl, int bcr, double parity,
                        double *ext)
{
    for (int i = 0; i < n; i++) ext[G + i] = f[i];
    for (int k = 1; k <= G; k++) {
        double vl, vr;
        if (bcl == ORC_BC_PERIODIC) vl = f[((-k % n) + n) % n];
        else if (bcl == ORC_BC_WALL) vl = parity * f[k - 1];
        else vl = f[0];
        if (bcr == ORC_BC_PERIODIC) vr = f[(n - 1 + k) % n];
        else if (bcr == ORC_BC_WALL) vr = parity * f[n - k];
        else vr = f[n - 1];
        ext[G - k] = vl;
        ext[G + n - 1 + k] = vr;
    }
}

/* ------------------------------------------------------------------------ */
/* One implicit stage S(E, R, tau)                                           */
/* ------------------------------------------------------------------------ */
/*
 * Computes U_new = R + tau * H~(E, U_new) (P:360 with a_ii dt = tau), i.e. the
 * fully discrete SI stage of P:500-517 with the convective fluxes and the
 * linearisation coefficients taken at the explicit input E and the base values
 * (h, q, h eta, h w on the right-hand sides of P:502-504, 511) taken from R.
 * With E = R = U^n and tau = dt this is literally P:500-517.
 * Bathymetric terms follow reading A9; the half-index coefficients follow A1.
 * On success writes out[0..3] = (h, q, K, W) and *min_beta = min_i beta_i.
 */
/* A25 face coefficient dhat_{f+1/2} = -(2 sigma^ - 1)/(3 h~) b1~ between cells f
 * and f+1 of E (ghost-extended arrays with G ghosts): sigma^ = (sigma_f + sigma_{f+1})/2,
 * h~ = (h_f + h_{f+1})/2, b1~ = (1/beta1_f + 1/beta1_{f+1})/2, beta1 = 1 + lam tau^2/h^2.
 * At the lake at rest (sigma = 1, H = h^2) it makes lam dhat (H^dag_{f+1} - H^dag_f)
 * equal the lam part of -beta_{f+1/2} (h_{f+1} - h_f) exactly. */
static double wb_delta(const double *eh, const double *eH, int f, double lam, double tau, int G)
{
    double h0 = eh[f + G], h1 = eh[f + 1 + G];
    double s0 = (eH[f + G] / h0) / h0, s1 = (eH[f + 1 + G] / h1) / h1;
    double b0 = 1.0 / (1.0 + lam * tau * tau / (h0 * h0));
    double b1 = 1.0 / (1.0 + lam * tau * tau / (h1 * h1));
    double sig = 0.5 * (s0 + s1), ht = 0.5 * (h0 + h1), bt = 0.5 * (b0 + b1);
    return -(2.0 * sig - 1.0) / (3.0 * ht) * bt;
}

static int stage_impl(const orc_problem *P, const double *const E[4],
                      const double *const R[4], double tau, double *const out[4],
                      double *min_beta)
{
    const int n = P->n, G = 3;
    const double dx = P->dx, g = P->g, lam = P->lambda;
    const int bcl = P->bc_left, bcr = P->bc_right;
    const int periodic = (bcl == ORC_BC_PERIODIC);
    const double qpar = -1.0;  /* q is odd under wall reflection (A10) */
    int status = ORC_OK;
    size_t ne = (size_t)(n + 2 * G);
    if (P->wb && P->picard > 0) return ORC_E_INVALID;   /* A25 is defined on the linearised stage */

    double *buf = (double *)calloc(ne * 5 + (size_t)(n + 3) * 3 + (size_t)(n + 2) * 8
                                   + (size_t)n * 10, sizeof(double));
    if (!buf) return ORC_E_INVALID;
    double *eh = buf, *eq = eh + ne, *eH = eq + ne, *eW = eH + ne, *eb = eW + ne;
    double *Fq = eb + ne, *FH = Fq + (n + 3), *FW = FH + (n + 3);
    double *qd = FW + (n + 3), *Hd = qd + (n + 2), *Wd = Hd + (n + 2);
    double *be = Wd + (n + 2), *de = be + (n + 2), *hb = de + (n + 2);
    double *bq = hb + (n + 2), *bH = bq + (n + 2);
    double *lo = bH + (n + 2), *di = lo + n, *up = di + n, *rhs = up + n, *Dxb = rhs + n;
    double *hbar = Dxb + n, *tmp0 = hbar + n, *tmp1 = tmp0 + n, *tmp2 = tmp1 + n;
    double *Hloc = tmp2 + n;
    (void)bq; (void)bH;
    double *alE = (double *)malloc(sizeof(double) * (size_t)n * 2);
    if (!alE) { free(buf); return ORC_E_INVALID; }
    double *a2E = alE + n;

    /* Step 1 (A9): H = K - 1.5 h b on E; ghost-extend E and b. */
    double *bzero = tmp0;
    for (int i = 0; i < n; i++) bzero[i] = P->b ? P->b[i] : 0.0;
    for (int i = 0; i < n; i++) Hloc[i] = E[2][i] - 1.5 * E[0][i] * bzero[i];
    fill_ghosts(E[0], n, G, bcl, bcr, 1.0, eh);
    fill_ghosts(E[1], n, G, bcl, bcr, qpar, eq);
    fill_ghosts(Hloc, n, G, bcl, bcr, 1.0, eH);
    fill_ghosts(E[3], n, G, bcl, bcr, 1.0, eW);
    fill_ghosts(bzero, n, G, bcl, bcr, 1.0, eb);
#define X(a, i) ((a)[(i) + G])

    /* Steps 2-3: MUSCL reconstruction (A5) and Rusanov fluxes
     * (A4) at faces f+1/2 for f = -2..n (array slot f+2). */
    for (int f = -2; f <= n; f++) {
        double vm[4], vp[4];
        const double *ev[4] = {eh, eq, eH, eW};
        for (int k = 0; k < 4; k++) {
            double v0 = X(ev[k], f), v1 = X(ev[k], f + 1);
            if (P->order == 2) {
                /* v'_i dx = (v_{i+1} - v_{i-1}) / 2;  v^-_{i+1/2} = v_i + v'_i dx/2,
                 * v^+_{i+1/2} = v_{i+1} - v'_{i+1} dx/2 */
                double s0 = (X(ev[k], f + 1) - X(ev[k], f - 1)) / 2.0;
                double s1 = (X(ev[k], f + 2) - X(ev[k], f)) / 2.0;
                vm[k] = v0 + s0 / 2.0;
                vp[k] = v1 - s1 / 2.0;
            } else {
                vm[k] = v0;
                vp[k] = v1;
            }
        }
        double F[3];
        orc_rusanov_face(vm, vp, F);
        Fq[f + 2] = F[0];
        FH[f + 2] = F[1];
        FW[f + 2] = F[2];
    }
#define FACE(a, i) ((a)[(i) + 2]) /* flux at face i+1/2 */

    /* Step 4: explicit predictor (A9 bathymetric sources). */
    double mb = INFINITY;
    for (int i = 0; i < n; i++) {
        Dxb[i] = (X(eb, i + 1) - X(eb, i - 1)) / (2.0 * dx);
        double hE = X(eh, i), qE = X(eq, i), HE = X(eH, i);
        double HR = R[2][i] - 1.5 * R[0][i] * bzero[i];
        double ptil = (lam / 3.0) * (1.0 - (HE / hE) / hE);     /* p~ */
        double Wd_ = R[3][i] - (tau / dx) * (FACE(FW, i) - FACE(FW, i - 1)) + lam * tau;
        double Hd_ = HR - (tau / dx) * (FACE(FH, i) - FACE(FH, i - 1))
                     - 1.5 * tau * qE * Dxb[i] + tau * Wd_;
        double qd_ = R[1][i] - (tau / dx) * (FACE(Fq, i) - FACE(Fq, i - 1))
                     - 1.5 * tau * ptil * Dxb[i];
        Wd[i + 1] = Wd_;
        Hd[i + 1] = Hd_;
        qd[i + 1] = qd_;
        /* Step 5: coefficients at E (A2) */
        double c[6];
        orc_coeffs(g, lam, tau, hE, HE, Hd_, c);
        be[i + 1] = c[4];
        de[i + 1] = c[5];
        alE[i] = c[0];
        a2E[i] = c[1];
        if (!(c[4] > 0.0)) status = ORC_E_COERCIVITY;  /* kappa > 0 */
        if (c[4] < mb) mb = c[4];
    }
    if (min_beta) *min_beta = mb;
    if (status != ORC_OK) goto done;

    for (int it = 0; it <= P->picard; it++) {
    if (it > 0) {
        /* A24 Picard pass: beta1, beta2 (hence beta, delta) at the latest hbar,
         * alpha and a^2 at E (the exact elimination has b1 = 1/beta1
         * and d b1/dh at h^{n+1}; the paper freezes them at h^n). */
        for (int i = 0; i < n; i++) {
            double hb = hbar[i];
            double beta1 = 1.0 + lam * tau * tau / (hb * hb);
            double beta2 = 2.0 * lam * tau * tau / (beta1 * beta1 * hb * hb * hb);
            be[i + 1] = a2E[i] + lam * alE[i] * beta2 * Hd[i + 1];
            de[i + 1] = alE[i] / beta1;
            if (!(be[i + 1] > 0.0)) { status = ORC_E_COERCIVITY; goto done; }
        }
    }
    /* Derived-field ghosts (A10): periodic wrap; wall/transmissive mirror-copy,
     * with q^dagger odd at a wall. */
    {
        double ql, qr, Hl, Hr, bl, br, dl, dr;
        if (periodic) {
            ql = qd[n]; qr = qd[1]; Hl = Hd[n]; Hr = Hd[1];
            bl = be[n]; br = be[1]; dl = de[n]; dr = de[1];
        } else {
            ql = (bcl == ORC_BC_WALL ? qpar : 1.0) * qd[1];
            qr = (bcr == ORC_BC_WALL ? qpar : 1.0) * qd[n];
            Hl = Hd[1]; Hr = Hd[n]; bl = be[1]; br = be[n]; dl = de[1]; dr = de[n];
        }
        qd[0] = ql; qd[n + 1] = qr; Hd[0] = Hl; Hd[n + 1] = Hr;
        be[0] = bl; be[n + 1] = br; de[0] = dl; de[n + 1] = dr;
    }

    /* Step 6: assemble Delta[h] = h^dagger (reading A1):
     *   rho_{i+1/2} = (tau^2/dx^2) (beta_i + beta_{i+1})/2
     *   mu_{i+1/2}  = (lambda tau^2 / (2 dx^2)) (delta_i + delta_{i+1})
     * Neumann rows (rho = 0 at the boundary face) for wall/transmissive ends. */
    {
        const double t2 = tau * tau / (dx * dx);
        const double lt2 = lam * tau * tau / (2.0 * dx * dx);
        for (int i = 0; i < n; i++) {
            double rl = t2 * (be[i] + be[i + 1]) / 2.0;      /* rho_{i-1/2} */
            double rr = t2 * (be[i + 1] + be[i + 2]) / 2.0;  /* rho_{i+1/2} */
            double ml = lt2 * (de[i] + de[i + 1]);            /* mu_{i-1/2} */
            double mr = lt2 * (de[i + 1] + de[i + 2]);        /* mu_{i+1/2} */
            if (P->wb) {
                /* A25: mu_{i+1/2} = (lam tau^2/dx^2) dhat_{i+1/2} */
                ml = 2.0 * lt2 * wb_delta(eh, eH, i - 1, lam, tau, G);
                mr = 2.0 * lt2 * wb_delta(eh, eH, i, lam, tau, G);
            }
            if (!periodic && i == 0) rl = 0.0;
            if (!periodic && i == n - 1) rr = 0.0;
            double hd = R[0][i] - (tau / (2.0 * dx)) * (qd[i + 2] - qd[i])
                        + mr * (Hd[i + 2] - Hd[i + 1]) - ml * (Hd[i + 1] - Hd[i]);
            /* A9: hydrostatic bathymetric term in zeta-form,
             * (tau^2/dx^2) [G_{i+1/2}(b_{i+1}-b_i) - G_{i-1/2}(b_i-b_{i-1})],
             * G_{i+1/2} = g (h^E_i + h^E_{i+1})/2 */
            double Gr = g * (X(eh, i) + X(eh, i + 1)) / 2.0;
            double Gl = g * (X(eh, i - 1) + X(eh, i)) / 2.0;
            double dbr = X(eb, i + 1) - X(eb, i), dbl = X(eb, i) - X(eb, i - 1);
            if (!periodic && i == 0) dbl = 0.0;
            if (!periodic && i == n - 1) dbr = 0.0;
            hd = hd + t2 * (Gr * dbr - Gl * dbl);
            lo[i] = -rl;
            up[i] = -rr;
            di[i] = 1.0 + rl + rr;
            rhs[i] = hd;
        }
    }
    /* Step 7: exact solve (A3). */
    status = periodic ? orc_cyclic_thomas(n, lo, di, up, rhs, hbar)
                      : orc_thomas(n, lo, di, up, rhs, hbar);
    if (status != ORC_OK) goto done;
    }   /* Picard passes */

    /* Step 8: back-substitution (A9 hydrostatic term). */
    for (int i = 0; i < n; i++) {
        double hl, hr;
        if (periodic) { hl = hbar[(i - 1 + n) % n]; hr = hbar[(i + 1) % n]; }
        else { hl = (i > 0) ? hbar[i - 1] : hbar[0]; hr = (i < n - 1) ? hbar[i + 1] : hbar[n - 1]; }
        double hn = hbar[i];
        if (!(hn > P->h_min)) { status = ORC_E_DRY; goto done; }
        double qn = qd[i + 1] - (tau / (2.0 * dx)) * be[i + 1] * (hr - hl)
                    - (lam * tau / (2.0 * dx)) * de[i + 1] * (Hd[i + 2] - Hd[i])
                    - tau * g * X(eh, i) * Dxb[i];
        if (P->wb) {
            /* A25: qbar = q^dag - (tau/(2dx)) (Phi_{i+1/2} + Phi_{i-1/2}),
             * Phi_{f} = beta_f (hbar_R - hbar_L) + lam dhat_f (H^dag_R - H^dag_L) + G_f (b_R - b_L) */
            double Phr = 0.5 * (be[i + 1] + be[i + 2]) * (hr - hn)
                         + lam * wb_delta(eh, eH, i, lam, tau, G) * (Hd[i + 2] - Hd[i + 1])
                         + 0.5 * g * (X(eh, i) + X(eh, i + 1)) * (X(eb, i + 1) - X(eb, i));
            double Phl = 0.5 * (be[i] + be[i + 1]) * (hn - hl)
                         + lam * wb_delta(eh, eH, i - 1, lam, tau, G) * (Hd[i + 1] - Hd[i])
                         + 0.5 * g * (X(eh, i - 1) + X(eh, i)) * (X(eb, i) - X(eb, i - 1));
            if (!periodic && i == 0) Phl = 0.0;          /* wall / Neumann face */
            if (!periodic && i == n - 1) Phr = 0.0;
            qn = qd[i + 1] - (tau / (2.0 * dx)) * (Phr + Phl);
        }
        double Hn = Hd[i + 1] / (1.0 + lam * tau * tau / (hn * hn));
        double Wn = Wd[i + 1] - lam * tau * Hn / (hn * hn);
        tmp1[i] = qn;
        tmp2[i] = Hn;
        Hloc[i] = Wn;
    }
    for (int i = 0; i < n; i++) {
        double Kn = tmp2[i] + 1.5 * hbar[i] * bzero[i];
        if (!isfinite(hbar[i]) || !isfinite(tmp1[i]) || !isfinite(Kn) || !isfinite(Hloc[i]))
            status = ORC_E_NONFINITE;
        out[0][i] = hbar[i];
        out[1][i] = tmp1[i];
        out[2][i] = Kn;
        out[3][i] = Hloc[i];
    }
#undef X
#undef FACE
done:
    free(alE);
    free(buf);
    return status;
}

int orc_stage(const orc_problem *P, const double *Eh, const double *Eq, const double *EK,
              const double *EW, const double *Rh, const double *Rq, const double *RK,
              const double *RW, double tau, double *Oh, double *Oq, double *OK, double *OW,
              double *min_beta)
{
    if (!P || P->n < 4 || !(P->dx > 0.0) || (P->order != 1 && P->order != 2)) return ORC_E_INVALID;
    if ((P->bc_left == ORC_BC_PERIODIC) != (P->bc_right == ORC_BC_PERIODIC)) return ORC_E_INVALID;
    const double *E[4] = {Eh, Eq, EK, EW};
    const double *R[4] = {Rh, Rq, RK, RW};
    double *O[4] = {Oh, Oq, OK, OW};
    return stage_impl(P, E, R, tau, O, min_beta);
}

/* ------------------------------------------------------------------------ */
/* A19 stability filter (off unless filter_sigma > 0)                        */
/* f_i <- f_i - (sigma/16)(f_{i-2} - 4 f_{i-1} + 6 f_i - 4 f_{i+1} + f_{i+2}) */
/* ------------------------------------------------------------------------ */
static int apply_filter(const orc_problem *P, double *U[4])
{
    if (!(P->filter_sigma > 0.0)) return ORC_OK;
    const int n = P->n, G = 2;
    double *ext = (double *)malloc(sizeof(double) * (size_t)(n + 2 * G));
    if (!ext) return ORC_E_INVALID;
    for (int k = 0; k < 4; k++) {
        if (!(P->filter_mask & (1 << k))) continue;
        double par = (k == 1) ? -1.0 : 1.0;
        fill_ghosts(U[k], n, G, P->bc_left, P->bc_right, par, ext);
        for (int i = 0; i < n; i++) {
            double d4 = ext[i] - 4.0 * ext[i + 1] + 6.0 * ext[i + 2] - 4.0 * ext[i + 3] + ext[i + 4];
            U[k][i] = ext[i + 2] - (P->filter_sigma / 16.0) * d4;
        }
    }
    free(ext);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Relaxation zones: wavemaker and sponge (A10; cfg4)                        */
/* ------------------------------------------------------------------------ */
static void apply_relaxation(const orc_problem *P, double *U[4], double t)
{
    const double x_max = P->x_min + P->n * P->dx;
    for (int i = 0; i < P->n; i++) {
        double x = P->x_min + (i + 0.5) * P->dx;
        double b = P->b ? P->b[i] : 0.0;
        double s = 0.0, tg[4];
        if (P->gen_rate > 0.0 && x <= P->gen_x1) {
            double r = 1.0 - (x - P->x_min) / (P->gen_x1 - P->x_min);
            s = P->gen_rate * r * r;
            double eta = P->amp * sin(P->omega * t - P->k * (x - P->x_min));
            double h = P->level + eta - b;
            double u = P->cp * eta / P->level;
            tg[0] = h; tg[1] = h * u; tg[2] = h * (h + 1.5 * b); tg[3] = 0.0;
        } else if (P->sp_rate > 0.0 && x >= P->sp_x0) {
            double r = (x - P->sp_x0) / (x_max - P->sp_x0);
            s = P->sp_rate * r * r;
            double h = P->level - b;
            tg[0] = h; tg[1] = 0.0; tg[2] = h * (h + 1.5 * b); tg[3] = 0.0;
        }
        if (s > 0.0)
            for (int k = 0; k < 4; k++) U[k][i] = U[k][i] - s * (U[k][i] - tg[k]);
    }
}

/* ------------------------------------------------------------------------ */
/* Tableau validation and stage weights                          */
/* ------------------------------------------------------------------------ */
/* wE = a^E_21 / a^I_11 and wR = a^I_21 / a^I_11 (efficient form). */
int orc_tableau_weights(const orc_tableau *T, double *wE, double *wR)
{
    if (!T) return ORC_E_INVALID;
    if (T->stages == 1) {
        if (!(T->aI[0][0] > 0.0)) return ORC_E_INVALID;
        *wE = 0.0;
        *wR = 0.0;
        return ORC_OK;
    }
    if (T->stages != 2) return ORC_E_INVALID;
    if (!(T->aI[0][0] > 0.0) || !(T->aI[1][1] > 0.0)) return ORC_E_INVALID;
    if (T->aE[0][0] != 0.0 || T->aE[0][1] != 0.0 || T->aE[1][1] != 0.0 || T->aI[0][1] != 0.0)
        return ORC_E_INVALID;
    /* stiffly accurate: last row of A_I equals b */
    if (T->aI[1][0] != T->b[0] || T->aI[1][1] != T->b[1]) return ORC_E_INVALID;
    *wE = T->aE[1][0] / T->aI[0][0];
    *wR = T->aI[1][0] / T->aI[0][0];
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* One SI-IMEX step                                              */
/* ------------------------------------------------------------------------ */
/* One step starting at time t (t only enters the A10 wavemaker zone). */
int orc_step_t(const orc_problem *P, const orc_tableau *T, double t, double dt, double *h,
               double *q, double *K, double *W, double *min_beta);

int orc_step(const orc_problem *P, const orc_tableau *T, double dt, double *h, double *q,
             double *K, double *W, double *min_beta)
{
    return orc_step_t(P, T, 0.0, dt, h, q, K, W, min_beta);
}

int orc_step_t(const orc_problem *P, const orc_tableau *T, double t, double dt, double *h,
               double *q, double *K, double *W, double *min_beta)
{
    double wE, wR;
    int st = orc_tableau_weights(T, &wE, &wR);
    if (st != ORC_OK) return st;
    const int n = P->n;
    double *buf = (double *)malloc(sizeof(double) * (size_t)n * 16);
    if (!buf) return ORC_E_INVALID;
    double *U1[4], *E2[4], *R2[4], *Un[4];
    for (int k = 0; k < 4; k++) {
        U1[k] = buf + (size_t)n * k;
        E2[k] = buf + (size_t)n * (4 + k);
        R2[k] = buf + (size_t)n * (8 + k);
        Un[k] = buf + (size_t)n * (12 + k);
    }
    double *U[4] = {h, q, K, W};
    for (int k = 0; k < 4; k++) memcpy(Un[k], U[k], sizeof(double) * (size_t)n);
    double mb1 = INFINITY, mb2 = INFINITY;
    if (T->stages == 1) {
        /* U^{n+1} = S(U^n, U^n, a_11 dt): literally P:500-517 (tau = dt when a_11 = 1) */
        st = orc_stage(P, Un[0], Un[1], Un[2], Un[3], Un[0], Un[1], Un[2], Un[3],
                       T->aI[0][0] * dt, U1[0], U1[1], U1[2], U1[3], &mb1);
        if (st == ORC_OK) for (int k = 0; k < 4; k++) memcpy(U[k], U1[k], sizeof(double) * (size_t)n);
    } else {
        /* step 1-2: U_E^(1) = U^n; U_I^(1) = U^n + gamma dt H(U_E^(1), U_I^(1)) */
        st = orc_stage(P, Un[0], Un[1], Un[2], Un[3], Un[0], Un[1], Un[2], Un[3],
                       T->aI[0][0] * dt, U1[0], U1[1], U1[2], U1[3], &mb1);
        if (st == ORC_OK) {
            /* efficient form:
             * U_E^(2) = (1 - c/gamma) U^n + (c/gamma) U_I^(1)
             * base of U_I^(2) = (1 - (1-gamma)/gamma) U^n + ((1-gamma)/gamma) U_I^(1) */
            for (int k = 0; k < 4; k++)
                for (int i = 0; i < n; i++) {
                    E2[k][i] = (1.0 - wE) * Un[k][i] + wE * U1[k][i];
                    R2[k][i] = (1.0 - wR) * Un[k][i] + wR * U1[k][i];
                }
            /* step 4-5: U^{n+1} = U_I^(2), stiffly accurate */
            st = orc_stage(P, E2[0], E2[1], E2[2], E2[3], R2[0], R2[1], R2[2], R2[3],
                           T->aI[1][1] * dt, U[0], U[1], U[2], U[3], &mb2);
        }
    }
    if (st == ORC_OK) st = apply_filter(P, U);
    if (st == ORC_OK) apply_relaxation(P, U, t + dt);
    if (min_beta) *min_beta = mb1 < mb2 ? mb1 : mb2;
    free(buf);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Time-step rule (readings A7, A8)                    */
/* ------------------------------------------------------------------------ */
/* nu_max = max_i (|u_i| + c_i), c from P:127 (A7); u_max = max_i |u_i|.
 * dt_bar = CFL dx / nu_max; if u_max dt_bar / dx > MCFL then dt = MCFL dx / u_max.
 * cfl <= 0 disables the first rule, mcfl <= 0 the second; if u_max = 0 the
 * material rule is inactive. */
int orc_dt(const orc_problem *P, double cfl, double mcfl, const double *h, const double *q,
           const double *K, double *dt, double *nu_max_out, double *u_max_out)
{
    double nu = 0.0, um = 0.0;
    for (int i = 0; i < P->n; i++) {
        if (!(h[i] > P->h_min)) return ORC_E_DRY;
        double b = P->b ? P->b[i] : 0.0;
        double H = K[i] - 1.5 * h[i] * b;
        double u = q[i] / h[i];
        double c = orc_celerity(P->g, P->lambda, h[i], H);
        double s = fabs(u) + c;
        if (s > nu) nu = s;
        if (fabs(u) > um) um = fabs(u);
    }
    if (nu_max_out) *nu_max_out = nu;
    if (u_max_out) *u_max_out = um;
    double d;
    if (cfl > 0.0) {
        d = cfl * P->dx / nu;
        if (mcfl > 0.0 && um > 0.0 && um * d / P->dx > mcfl) d = mcfl * P->dx / um;
    } else if (mcfl > 0.0 && um > 0.0) {
        d = mcfl * P->dx / um;
    } else {
        return ORC_E_INVALID;
    }
    *dt = d;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Run loop: max_steps steps, or until t_end (last step clipped)      */
/* t_end <= t0 means "run exactly max_steps steps".                          */
/* dt_fixed > 0 overrides the rule.                                          */
/* ------------------------------------------------------------------------ */
int orc_run(const orc_problem *P, const orc_tableau *T, double cfl, double mcfl,
            double dt_fixed, double t0, double t_end, int64_t max_steps, double *h, double *q,
            double *K, double *W, double *t_out, int64_t *steps_out, double *min_beta)
{
    double t = t0, mb = INFINITY;
    int64_t s = 0;
    int st = ORC_OK;
    int use_tend = (t_end > t0);
    while (s < max_steps) {
        if (use_tend && !(t < t_end)) break;
        double dt;
        if (dt_fixed > 0.0) dt = dt_fixed;
        else {
            st = orc_dt(P, cfl, mcfl, h, q, K, &dt, NULL, NULL);
            if (st != ORC_OK) break;
        }
        /* last step clipped to land exactly on t_end */
        if (use_tend && t + dt >= t_end) dt = t_end - t;
        double m;
        st = orc_step_t(P, T, t, dt, h, q, K, W, &m);
        if (m < mb) mb = m;
        if (st != ORC_OK) break;
        t = (use_tend && dt == t_end - t) ? t_end : t + dt;
        s++;
    }
    if (t_out) *t_out = t;
    if (steps_out) *steps_out = s;
    if (min_beta) *min_beta = mb;
    return st;
}

/* ------------------------------------------------------------------------ */
/* Explicit hSGN scheme                      */
/* ------------------------------------------------------------------------ */
/*
 * Spatial operator L(U) of the first-order explicit scheme P:444-458, flat
 * bottom (P->b must be NULL):
 *   L_h = -D_x(q)
 *   L_q = -D^_x(q u) - a^2(h, eta) D_x(h) - lambda alpha(h, eta) D_x(h eta)
 *   L_H = -D^_x(h u eta) + h w                      (H = h eta = K, W = h w)
 *   L_W = -D^_x(h u w) - lambda (h eta / h^2 - 1)
 * D_x(F)_i = (F_{i+1/2} - F_{i-1/2})/dx with F_{i+1/2} = (F(U_{i+1}) + F(U_i))/2
 * (P:463), i.e. (F_{i+1} - F_{i-1})/(2 dx); D^_x is the Rusanov difference of
 * P:466 with the MUSCL faces of P:469-478 (order 2) or cell values (order 1),
 * alpha = max(|u-|, |u+|) (A4) -- the same face fluxes as the SI predictor.
 * a^2 and alpha are taken at cell i, time level of U; alpha and
 * a^2 as in orc_coeffs.  Ghosts by A10.
 */
static int explicit_L(const orc_problem *P, const double *const U[4], double *const L[4])
{
    const int n = P->n, G = 2;
    const double dx = P->dx, g = P->g, lam = P->lambda;
    const size_t ne = (size_t)(n + 2 * G);
    if (P->b) return ORC_E_INVALID;   /* flat bottom only */
    double *buf = (double *)calloc(ne * 4 + (size_t)(n + 1) * 3, sizeof(double));
    if (!buf) return ORC_E_INVALID;
    double *eh = buf, *eq = eh + ne, *eH = eq + ne, *eW = eH + ne;
    double *Fq = eW + ne, *FH = Fq + (n + 1), *FW = FH + (n + 1);
    fill_ghosts(U[0], n, G, P->bc_left, P->bc_right, 1.0, eh);
    fill_ghosts(U[1], n, G, P->bc_left, P->bc_right, -1.0, eq);
    fill_ghosts(U[2], n, G, P->bc_left, P->bc_right, 1.0, eH);
    fill_ghosts(U[3], n, G, P->bc_left, P->bc_right, 1.0, eW);
#define XE(a, i) ((a)[(i) + G])
    /* Rusanov fluxes at faces f+1/2, f = -1 .. n-1 (slot f+1) */
    for (int f = -1; f <= n - 1; f++) {
        double vm[4], vp[4];
        const double *ev[4] = {eh, eq, eH, eW};
        for (int k = 0; k < 4; k++) {
            double v0 = XE(ev[k], f), v1 = XE(ev[k], f + 1);
            if (P->order == 2) {
                double s0 = (XE(ev[k], f + 1) - XE(ev[k], f - 1)) / 2.0;
                double s1 = (XE(ev[k], f + 2) - XE(ev[k], f)) / 2.0;
                vm[k] = v0 + s0 / 2.0;
                vp[k] = v1 - s1 / 2.0;
            } else {
                vm[k] = v0;
                vp[k] = v1;
            }
        }
        double F[3];
        orc_rusanov_face(vm, vp, F);
        Fq[f + 1] = F[0];
        FH[f + 1] = F[1];
        FW[f + 1] = F[2];
    }
    int st = ORC_OK;
    for (int i = 0; i < n; i++) {
        double h = XE(eh, i), H = XE(eH, i), W = XE(eW, i);
        if (!(h > P->h_min)) st = ORC_E_DRY;
        double eta = H / h, sigma = eta / h;
        double alpha = -(1.0 / (3.0 * h)) * (2.0 * sigma - 1.0);
        double a2 = g * h + (lam / 3.0) * sigma * sigma - lam * eta * alpha;
        double Dxq = (XE(eq, i + 1) - XE(eq, i - 1)) / (2.0 * dx);
        double Dxh = (XE(eh, i + 1) - XE(eh, i - 1)) / (2.0 * dx);
        double DxH = (XE(eH, i + 1) - XE(eH, i - 1)) / (2.0 * dx);
        L[0][i] = -Dxq;
        L[1][i] = -(Fq[i + 1] - Fq[i]) / dx - a2 * Dxh - lam * alpha * DxH;
        L[2][i] = -(FH[i + 1] - FH[i]) / dx + W;
        L[3][i] = -(FW[i + 1] - FW[i]) / dx - lam * (H / (h * h) - 1.0);
    }
#undef XE
    free(buf);
    return st;
}

/* L(U) as a library call (tests). */
int orc_explicit_rhs(const orc_problem *P, const double *h, const double *q, const double *K,
                     const double *W, double *Lh, double *Lq, double *LK, double *LW)
{
    const double *U[4] = {h, q, K, W};
    double *L[4] = {Lh, Lq, LK, LW};
    return explicit_L(P, U, L);
}

/*
 * One explicit step: stages = 1 forward Euler U + dt L(U);
 * stages = 2 Heun: U1 = U + dt L(U),
 * U^{n+1} = 1/2 U + 1/2 (U1 + dt L(U1)).  Then the optional A19 filter and the
 * A10 relaxation zones at t + dt, as for the SI step.
 */
int orc_explicit_step_t(const orc_problem *P, int stages, double t, double dt, double *h,
                        double *q, double *K, double *W)
{
    if (stages != 1 && stages != 2) return ORC_E_INVALID;
    const int n = P->n;
    double *buf = (double *)malloc(sizeof(double) * (size_t)n * 12);
    if (!buf) return ORC_E_INVALID;
    double *Un[4], *U1[4], *Lb[4];
    for (int k = 0; k < 4; k++) {
        Un[k] = buf + (size_t)n * k;
        U1[k] = buf + (size_t)n * (4 + k);
        Lb[k] = buf + (size_t)n * (8 + k);
    }
    double *U[4] = {h, q, K, W};
    for (int k = 0; k < 4; k++) memcpy(Un[k], U[k], sizeof(double) * (size_t)n);
    int st = explicit_L(P, (const double *const *)Un, Lb);
    if (st == ORC_OK) {
        for (int k = 0; k < 4; k++)
            for (int i = 0; i < n; i++) U1[k][i] = Un[k][i] + dt * Lb[k][i];
        if (stages == 1) {
            for (int k = 0; k < 4; k++) memcpy(U[k], U1[k], sizeof(double) * (size_t)n);
        } else {
            st = explicit_L(P, (const double *const *)U1, Lb);
            if (st == ORC_OK)
                for (int k = 0; k < 4; k++)
                    for (int i = 0; i < n; i++)
                        U[k][i] = 0.5 * Un[k][i] + 0.5 * (U1[k][i] + dt * Lb[k][i]);
        }
    }
    if (st == ORC_OK)
        for (int i = 0; i < n; i++)
            if (!(h[i] > P->h_min)) st = ORC_E_DRY;
    if (st == ORC_OK) st = apply_filter(P, U);
    if (st == ORC_OK) apply_relaxation(P, U, t + dt);
    free(buf);
    return st;
}

/* Explicit run: dt = CFL_EX dx / mu_max (mu = |u| + c, A7) unless
 * dt_fixed > 0; max_steps steps or until t_end (last step clipped). */
int orc_explicit_run(const orc_problem *P, int stages, double cfl, double dt_fixed, double t0,
                     double t_end, int64_t max_steps, double *h, double *q, double *K, double *W,
                     double *t_out, int64_t *steps_out)
{
    double t = t0;
    int64_t s = 0;
    int st = ORC_OK;
    int use_tend = (t_end > t0);
    while (s < max_steps) {
        if (use_tend && !(t < t_end)) break;
        double dt;
        if (dt_fixed > 0.0) dt = dt_fixed;
        else {
            st = orc_dt(P, cfl, 0.0, h, q, K, &dt, NULL, NULL);
            if (st != ORC_OK) break;
        }
        if (use_tend && t + dt >= t_end) dt = t_end - t;
        st = orc_explicit_step_t(P, stages, t, dt, h, q, K, W);
        if (st != ORC_OK) break;
        t = (use_tend && dt == t_end - t) ? t_end : t + dt;
        s++;
    }
    if (t_out) *t_out = t;
    if (steps_out) *steps_out = s;
    return st;
}

/* ------------------------------------------------------------------------ */
/* Classical SGN scheme, with bathymetry      */
/* ------------------------------------------------------------------------ */
/*
 * Explicit scheme for the standard SGN equations in elliptic-hyperbolic form
 * (P:548-556):
 *   h_t + (hu)_x = 0,  (hu)_t + (hu^2 + g h^2/2)_x = h phi,
 *   h_i phi_i - (1/(3 dx^2)) (h^3_{i+1/2}(phi_{i+1} - phi_i) - h^3_{i-1/2}(phi_i - phi_{i-1})) = h*_i,
 *   h*_i = -(1/(6 dx^3)) ( g h^3_{i+1} (h_{i+2} - 2h_{i+1} + h_i) + (h^3_{i+1}/2)(u_{i+2} - u_i)^2
 *                        - g h^3_{i-1} (h_i - 2h_{i-1} + h_{i-2}) - (h^3_{i-1}/2)(u_i - u_{i-2})^2 )
 * Readings (A23): the g-term carries h^3 (P:591 prints g h_{i+1}; the
 * discretisation of -(h^3/3 g h_xx)_x of P:548 needs h^3); h_{i+1/2} =
 * (h_i + h_{i+1})/2; Rusanov fluxes of the shallow-water part on MUSCL faces
 * of (h, q) with the wave speed alpha = max(|u| + sqrt(g h)) of both face
 * states; phi ghosts: periodic wrap, wall phi_{-1} = -phi_0 (phi is an
 * acceleration, odd like q), transmissive phi_{-1} = phi_0.  K and W are not
 * part of this model and are carried unchanged.
 *
 * Bathymetry (eq. SGNb_standard; reading A26): the phi equation
 *   h phi - (h^3/3 phi_x)_x + kappa phi = -(h^3/3 g zeta_xx + 2 h^3/3 u_x^2 + rho)_x - h Q b_x,
 *   kappa = (h^2 b_x/2)_x + 3 h b_x^2/4,  rho = -(h^2 b_x/2) g zeta_x + h^3 u^2 b_xx,
 *   Q = (h/2) g zeta_xx - (3 g b_x/4) zeta_x + h u_x^2 + (3/2) h u^2 b_xx,
 * follows from P:175-186 with phi := Du/Dt + g zeta_x, so the momentum carries
 * the hydrostatic source: (hu)_t + (hu^2 + g h^2/2)_x + g h b_x = h phi (P:566
 * prints it without g h b_x, which would move the lake at rest).  Discretised
 * like the flat scheme: zeta = h + b in the g-term's second differences, rho and
 * the derivatives of zeta, u, b centred at cells i-1, i, i+1, kappa_i =
 * (h^2_{i+1/2}(b_{i+1} - b_i) - h^2_{i-1/2}(b_i - b_{i-1}))/(2 dx^2) + (3/4) h_i (D_x b)_i^2,
 * source -g h_i (D_x b)_i.  b ghosts even.  b = 0 reproduces the flat scheme
 * bit for bit (every added term is a product with a difference of b).
 */
static int sgn_L(const orc_problem *P, const double *h, const double *q, double *Lh, double *Lq)
{
    const int n = P->n, G = 2;
    const double dx = P->dx, g = P->g;
    const size_t ne = (size_t)(n + 2 * G);
    double *buf = (double *)calloc(ne * 4 + (size_t)(n + 1) * 2 + (size_t)n * 4, sizeof(double));
    if (!buf) return ORC_E_INVALID;
    double *eh = buf, *eq = eh + ne, *eu = eq + ne, *eb = eu + ne;
    double *Fh = eb + ne, *Fq = Fh + (n + 1);
    double *lo = Fq + (n + 1), *di = lo + n, *up = di + n, *rhs = up + n;
    double *phi = (double *)calloc((size_t)n, sizeof(double));
    if (!phi) { free(buf); return ORC_E_INVALID; }
    fill_ghosts(h, n, G, P->bc_left, P->bc_right, 1.0, eh);
    fill_ghosts(q, n, G, P->bc_left, P->bc_right, -1.0, eq);
    if (P->b) fill_ghosts(P->b, n, G, P->bc_left, P->bc_right, 1.0, eb);
    int st = ORC_OK;
    for (int i = -G; i < n + G; i++) {
        if (!(eh[i + G] > P->h_min)) st = ORC_E_DRY;
        eu[i + G] = eq[i + G] / eh[i + G];
    }
#define XS(a, i) ((a)[(i) + G])
#define XZ(i) (XS(eh, i) + XS(eb, i))         /* zeta = h + b */
    /* Rusanov fluxes of (q, q^2/h + g h^2/2) at faces f+1/2, f = -1 .. n-1 */
    for (int f = -1; f <= n - 1; f++) {
        double vm[2], vp[2];
        const double *ev[2] = {eh, eq};
        for (int k = 0; k < 2; k++) {
            double v0 = XS(ev[k], f), v1 = XS(ev[k], f + 1);
            if (P->order == 2) {
                double s0 = (XS(ev[k], f + 1) - XS(ev[k], f - 1)) / 2.0;
                double s1 = (XS(ev[k], f + 2) - XS(ev[k], f)) / 2.0;
                vm[k] = v0 + s0 / 2.0;
                vp[k] = v1 - s1 / 2.0;
            } else {
                vm[k] = v0;
                vp[k] = v1;
            }
        }
        double um = vm[1] / vm[0], up_ = vp[1] / vp[0];
        double am = fabs(um) + sqrt(g * vm[0]), ap = fabs(up_) + sqrt(g * vp[0]);
        double a = am > ap ? am : ap;
        double fhm = vm[1], fhp = vp[1];
        double fqm = vm[1] * um + 0.5 * g * vm[0] * vm[0];
        double fqp = vp[1] * up_ + 0.5 * g * vp[0] * vp[0];
        Fh[f + 1] = 0.5 * (fhm + fhp) - 0.5 * a * (vp[0] - vm[0]);
        Fq[f + 1] = 0.5 * (fqm + fqp) - 0.5 * a * (vp[1] - vm[1]);
    }
    /* phi system */
    for (int i = 0; i < n; i++) {
        double hl = 0.5 * (XS(eh, i - 1) + XS(eh, i)), hr = 0.5 * (XS(eh, i) + XS(eh, i + 1));
        double cl = hl * hl * hl / (3.0 * dx * dx), cr = hr * hr * hr / (3.0 * dx * dx);
        double hp = XS(eh, i + 1), hm = XS(eh, i - 1);
        double hp3 = hp * hp * hp, hm3 = hm * hm * hm;
        double up2 = XS(eu, i + 2) - XS(eu, i), um2 = XS(eu, i) - XS(eu, i - 2);
        if (!P->b) {
            rhs[i] = -(1.0 / (6.0 * dx * dx * dx))
                     * (g * hp3 * (XS(eh, i + 2) - 2.0 * hp + XS(eh, i)) + 0.5 * hp3 * up2 * up2
                        - g * hm3 * (XS(eh, i) - 2.0 * hm + XS(eh, i - 2)) - 0.5 * hm3 * um2 * um2);
        } else {
            rhs[i] = -(1.0 / (6.0 * dx * dx * dx))
                     * (g * hp3 * (XZ(i + 2) - 2.0 * XZ(i + 1) + XZ(i)) + 0.5 * hp3 * up2 * up2
                        - g * hm3 * (XZ(i) - 2.0 * XZ(i - 1) + XZ(i - 2)) - 0.5 * hm3 * um2 * um2);
            /* rho at cells j = i -+ 1 and Q at cell i (A26) */
            double rho[2];
            for (int s2 = 0; s2 < 2; s2++) {
                const int j = s2 == 0 ? i - 1 : i + 1;
                const double hj = XS(eh, j), uj = XS(eu, j);
                const double bx = (XS(eb, j + 1) - XS(eb, j - 1)) / (2.0 * dx);
                const double zx = (XZ(j + 1) - XZ(j - 1)) / (2.0 * dx);
                const double bxx = (XS(eb, j + 1) - 2.0 * XS(eb, j) + XS(eb, j - 1)) / (dx * dx);
                rho[s2] = -(hj * hj * bx / 2.0) * g * zx + hj * hj * hj * uj * uj * bxx;
            }
            const double h0 = XS(eh, i), u0 = XS(eu, i);
            const double bx = (XS(eb, i + 1) - XS(eb, i - 1)) / (2.0 * dx);
            const double zx = (XZ(i + 1) - XZ(i - 1)) / (2.0 * dx);
            const double zxx = (XZ(i + 1) - 2.0 * XZ(i) + XZ(i - 1)) / (dx * dx);
            const double bxx = (XS(eb, i + 1) - 2.0 * XS(eb, i) + XS(eb, i - 1)) / (dx * dx);
            const double ux = (XS(eu, i + 1) - XS(eu, i - 1)) / (2.0 * dx);
            const double Q = (h0 / 2.0) * g * zxx - (3.0 * g * bx / 4.0) * zx + h0 * ux * ux
                             + 1.5 * h0 * u0 * u0 * bxx;
            rhs[i] += -(rho[1] - rho[0]) / (2.0 * dx) - h0 * Q * bx;
        }
        lo[i] = -cl;
        up[i] = -cr;
        di[i] = XS(eh, i) + cl + cr;
        if (P->b) {
            const double bx = (XS(eb, i + 1) - XS(eb, i - 1)) / (2.0 * dx);
            const double kap = (hr * hr * (XS(eb, i + 1) - XS(eb, i)) - hl * hl * (XS(eb, i) - XS(eb, i - 1)))
                               / (2.0 * dx * dx)
                               + 0.75 * XS(eh, i) * bx * bx;
            di[i] += kap;
        }
    }
    if (P->bc_left != ORC_BC_PERIODIC) {
        /* phi_{-1} = p phi_0 folds into the diagonal: -cl (p phi_0) */
        double pl = (P->bc_left == ORC_BC_WALL) ? -1.0 : 1.0;
        double pr = (P->bc_right == ORC_BC_WALL) ? -1.0 : 1.0;
        di[0] += lo[0] * pl;
        di[n - 1] += up[n - 1] * pr;
        st = (st == ORC_OK) ? orc_thomas(n, lo, di, up, rhs, phi) : st;
    } else {
        st = (st == ORC_OK) ? (n >= 3 ? orc_cyclic_thomas(n, lo, di, up, rhs, phi) : ORC_E_INVALID) : st;
    }
    for (int i = 0; i < n; i++) {
        Lh[i] = -(Fh[i + 1] - Fh[i]) / dx;
        Lq[i] = -(Fq[i + 1] - Fq[i]) / dx + XS(eh, i) * phi[i];
        if (P->b) Lq[i] -= g * XS(eh, i) * (XS(eb, i + 1) - XS(eb, i - 1)) / (2.0 * dx);   /* A26 */
    }
#undef XZ
#undef XS
    free(phi);
    free(buf);
    return st;
}

int orc_sgn_rhs(const orc_problem *P, const double *h, const double *q, double *Lh, double *Lq)
{
    return sgn_L(P, h, q, Lh, Lq);
}

/* One SGN step: stages 1 forward Euler, 2 Heun; then the optional A19
 * filter (q only is a field of this model; W is carried). */
int orc_sgn_step(const orc_problem *P, int stages, double dt, double *h, double *q)
{
    if (stages != 1 && stages != 2) return ORC_E_INVALID;
    const int n = P->n;
    double *buf = (double *)malloc(sizeof(double) * (size_t)n * 6);
    if (!buf) return ORC_E_INVALID;
    double *h0 = buf, *q0 = h0 + n, *h1 = q0 + n, *q1 = h1 + n, *Lh = q1 + n, *Lq = Lh + n;
    memcpy(h0, h, sizeof(double) * (size_t)n);
    memcpy(q0, q, sizeof(double) * (size_t)n);
    int st = sgn_L(P, h0, q0, Lh, Lq);
    if (st == ORC_OK) {
        for (int i = 0; i < n; i++) { h1[i] = h0[i] + dt * Lh[i]; q1[i] = q0[i] + dt * Lq[i]; }
        if (stages == 1) {
            memcpy(h, h1, sizeof(double) * (size_t)n);
            memcpy(q, q1, sizeof(double) * (size_t)n);
        } else {
            st = sgn_L(P, h1, q1, Lh, Lq);
            if (st == ORC_OK)
                for (int i = 0; i < n; i++) {
                    h[i] = 0.5 * h0[i] + 0.5 * (h1[i] + dt * Lh[i]);
                    q[i] = 0.5 * q0[i] + 0.5 * (q1[i] + dt * Lq[i]);
                }
        }
    }
    if (st == ORC_OK)
        for (int i = 0; i < n; i++)
            if (!(h[i] > P->h_min)) st = ORC_E_DRY;
    if (st == ORC_OK && P->filter_sigma > 0.0 && (P->filter_mask & 2)) {
        double *U[4] = {h, q, NULL, NULL};
        orc_problem Pq = *P;
        Pq.filter_mask = 2;             /* q only */
        st = apply_filter(&Pq, U);
    }
    free(buf);
    return st;
}

/* dt = CFL_SGN dx / max_i (|u_i| + sqrt(g h_i)) */
int orc_sgn_dt(const orc_problem *P, double cfl, const double *h, const double *q, double *dt)
{
    double s = 0.0;
    for (int i = 0; i < P->n; i++) {
        if (!(h[i] > P->h_min)) return ORC_E_DRY;
        double v = fabs(q[i] / h[i]) + sqrt(P->g * h[i]);
        if (v > s) s = v;
    }
    if (!(cfl > 0.0)) return ORC_E_INVALID;
    *dt = cfl * P->dx / s;
    return ORC_OK;
}

int orc_sgn_run(const orc_problem *P, int stages, double cfl, double dt_fixed, double t0,
                double t_end, int64_t max_steps, double *h, double *q, double *t_out,
                int64_t *steps_out)
{
    double t = t0;
    int64_t s = 0;
    int st = ORC_OK;
    int use_tend = (t_end > t0);
    while (s < max_steps) {
        if (use_tend && !(t < t_end)) break;
        double dt;
        if (dt_fixed > 0.0) dt = dt_fixed;
        else {
            st = orc_sgn_dt(P, cfl, h, q, &dt);
            if (st != ORC_OK) break;
        }
        if (use_tend && t + dt >= t_end) dt = t_end - t;
        st = orc_sgn_step(P, stages, dt, h, q);
        if (st != ORC_OK) break;
        t = (use_tend && dt == t_end - t) ? t_end : t + dt;
        s++;
    }
    if (t_out) *t_out = t;
    if (steps_out) *steps_out = s;
    return st;
}

/* total mass sum_i h_i dx */
double orc_mass(int n, double dx, const double *h)
{
    double m = 0.0;
    for (int i = 0; i < n; i++) m += h[i];
    return m * dx;
}
