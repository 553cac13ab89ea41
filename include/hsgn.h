/*
 * hsgn.h -- C ABI of libhsgn.so: the B200 (sm_100a) fp64 implementation of the
 * semi-implicit IMEX Runge-Kutta step of the hyperbolised Serre-Green-Naghdi
 * (hSGN) system of arXiv 2510.07539.
 *
 * Citations: "P:n" = line n of the paper text, "Ak" = reading k of
 * the ambiguity ledger in DESIGN.md section 3.
 *
 * What one step computes (efficient form P:397-403):
 *   U1      = S(U^n, U^n, a^I_11 dt)                       (stage 1)
 *   E2      = (1 - wE) U^n + wE U1,  wE = a^E_21 / a^I_11
 *   R2      = (1 - wR) U^n + wR U1,  wR = a^I_21 / a^I_11
 *   U^{n+1} = S(E2, R2, a^I_22 dt)                          (stage 2)
 * where S(E, R, tau) is the fully discrete SI stage of P:500-517: MUSCL
 * + Rusanov convective predictor on E, coefficients
 * beta1, beta2, beta, delta at E (A2), one tridiagonal depth solve
 * Delta[hbar] = h^dagger (A1), and back-substitution.
 * A 1-stage tableau gives the first-order SI step (P:500-517 literally).
 *
 * Data layout.  All state arrays are fp64, structure-of-arrays, member-major:
 * field[m * n_cells + i] for member m in [0, n_members) and cell i in
 * [0, n_cells).  The state is (h, q = h u, K, W = h w) with K = h eta on a
 * flat bottom and K = h (eta + 3 b / 2) with bathymetry.
 *
 * Memory ownership.  The library never allocates device memory: the caller
 * queries hsgn_workspace_bytes() and hands in one device allocation with
 * hsgn_set_workspace() (the Python binding allocates it with torch).  All
 * arrays passed to set_* / get_* are owned by the caller; they may be device
 * or host pointers (copies use cudaMemcpyDefault, ordered on the context's
 * stream).  The context owns nothing else but host-side bookkeeping and the
 * CUDA graphs it captures.
 *
 * Errors.  Every call returns an hsgn_status.  Device-side failures (kappa <= 0,
 * h <= h_min, non-finite values, insufficient solver overlap) are latched in a
 * device error word; the stage kernels stop computing once it is set, the step
 * that failed is not committed, and the next synchronising call (hsgn_step
 * with dt_used, hsgn_advance_to, hsgn_run_steps, hsgn_get_*, hsgn_sync) returns
 * the status.  After an error the state reads back as the last committed step.
 *
 * Threading.  A context is not thread-safe; use one context per thread.
 * Asynchrony: hsgn_run_steps and hsgn_step (dt_used == NULL) only enqueue work
 * on the context's stream; hsgn_sync() waits and reports device errors.
 */
#ifndef HSGN_H_
#define HSGN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hsgn_ctx hsgn_ctx; /* opaque */

typedef enum {
    HSGN_OK = 0,
    HSGN_E_INVALID = -1,    /* bad argument, extent, tableau or call order */
    HSGN_E_DRY = -2,        /* hbar <= h_min after a stage        */
    HSGN_E_COERCIVITY = -3, /* beta (= kappa) <= 0 at some cell */
    HSGN_E_SINGULAR = -4,   /* zero pivot in the depth solve              */
    HSGN_E_NONFINITE = -5,  /* NaN/Inf produced                           */
    HSGN_E_CUDA = -6,       /* CUDA runtime error                         */
    HSGN_E_OVERLAP = -7,    /* tile overlap too short for the depth solve's
                               decay (solver); result inexact  */
    HSGN_E_NOWORKSPACE = -8,/* workspace missing or too small             */
    HSGN_E_COMM = -9        /* NCCL failure in the slab transport (halo
                               send/recv, dt all-reduce, communicator)   */
} hsgn_status;

typedef enum {
    HSGN_BC_PERIODIC = 0,     /* cyclic (both sides must be periodic)           */
    HSGN_BC_WALL = 1,         /* reflecting: h, K, W even, q odd; Neumann depth rows (A10) */
    HSGN_BC_TRANSMISSIVE = 2, /* zero-order extrapolation; Neumann depth rows */
    HSGN_BC_HALO = 3          /* neighbouring slab of one large domain: w + 3 ghost cells
                                 exchanged before each stage;
                                 requires n_members == 1 and a group or NCCL */
} hsgn_bc;

/* Double Butcher tableau.  Validated by hsgn_set_tableau:
 * stages in {1, 2}; A_E strictly lower triangular; A_I lower triangular with
 * positive diagonal; for 2 stages the implicit tableau must be stiffly
 * accurate (last row == b). */
typedef struct {
    int32_t stages;
    int32_t pad_;
    double a_exp[2][2];
    double a_imp[2][2];
    double b[2];
} hsgn_tableau;

/* Problem description (uniform 1-D grid). */
typedef struct {
    int64_t n_cells;     /* cells per member, >= 4                                  */
    int32_t n_members;   /* independent domains (ensemble), >= 1                    */
    int32_t order;       /* 1: first-order faces, 2: MUSCL              */
    double x_min, x_max; /* dx = (x_max - x_min) / n_cells                         */
    int32_t bc_left;     /* hsgn_bc */
    int32_t bc_right;    /* hsgn_bc */
    int32_t tile_cells;  /* kept cells per CTA tile; 0 = automatic                  */
    int32_t overlap;     /* tile overlap w (cells) for the depth solve; 0 = auto:
                            chosen from CFL_IMEX and the tableau at set_params /
                            set_tableau                       */
} hsgn_desc;

/* Diagnostics (all members): mass = sum_i h_i dx summed over members,
 * min_h, max_abs_u, nu_max = max(|u| + c), t_min/t_max over members,
 * dt_last_min/max = the dt of the next step over members (set from the
 * current state by the rule of P:613-617), rho_max = largest
 * (tau/dx)^2 (beta_i + beta_{i+1})/2 seen (sets the solver overlap),
 * min_kappa = smallest beta = kappa of any cell in any SI
 * stage since hsgn_set_state, rounded toward zero to 2^-20 relative (its
 * high word) -- the coercivity monitor of the proposition at P:297-334 (a
 * value <= 0 also latches HSGN_E_COERCIVITY; +inf before the first SI stage;
 * not updated by the explicit and SGN schemes),
 * cfl_imex / mcfl = the achieved Courant numbers dt nu_max / dx and
 * dt max|u| / dx of the next step (max over members; P:617-643 report the
 * varying CFL), steps = committed steps. */
typedef struct {
    double mass;
    double min_h;
    double max_abs_u;
    double nu_max;
    double t_min;
    double t_max;
    double dt_last_min;
    double dt_last_max;
    double rho_max;      /* max off-diagonal rho of the depth system seen since set_state */
    double min_kappa;    /* min kappa = beta since set_state (coercivity monitor)        */
    double cfl_imex;     /* dt nu_max / dx of the next step (max over members)           */
    double mcfl;         /* dt max|u| / dx of the next step (max over members)           */
    int64_t steps;
    int32_t error_bits;
    int32_t pad_;
} hsgn_diag;

/* ---- lifecycle ---------------------------------------------------------- */

/* Create a context on the current CUDA device.  cuda_stream is a cudaStream_t
 * (NULL = legacy default stream) that every later call enqueues on. */
hsgn_status hsgn_create(const hsgn_desc *desc, void *cuda_stream, hsgn_ctx **out);
/* Synchronises the context's streams (no kernel or copy still uses the
 * workspace when it returns) and frees the context.  NULL is a no-op. */
void hsgn_destroy(hsgn_ctx *ctx);

/* Bytes of device workspace the context needs (3 state buffers of
 * 4 * n_cells * n_members doubles, bathymetry, per-member scalars). */
size_t hsgn_workspace_bytes(const hsgn_ctx *ctx);
/* Hand in a device allocation of at least hsgn_workspace_bytes() bytes,
 * 256-byte aligned.  The caller keeps it alive until hsgn_destroy. */
hsgn_status hsgn_set_workspace(hsgn_ctx *ctx, void *dev_ptr, size_t bytes);

/* ---- parameters -------------------------------------- */

/* g > 0; lambda[n_members] (host array) >= 0 (lambda = 0 allowed: the
 * semi-implicit shallow-water limit); cfl_imex <= 0 disables the CFL rule,
 * mcfl <= 0 disables the material rule; h_min >= 0. */
hsgn_status hsgn_set_params(hsgn_ctx *ctx, double g, const double *lambda, double cfl_imex,
                            double mcfl, double h_min);
/* Default: the paper's tableau, gamma = 1 - 1/sqrt2, c = 1/(2 gamma). */
hsgn_status hsgn_set_tableau(hsgn_ctx *ctx, const hsgn_tableau *tab);
/* b[n_cells] shared by all members (host or device pointer), or NULL = flat.
 * Bathymetric terms follow reading A9 of DESIGN.md. */
hsgn_status hsgn_set_bathymetry(hsgn_ctx *ctx, const double *b);
/* Optional stability filter of reading A19, applied after each
 * step: f_i -= (sigma/16) (f_{i-2} - 4 f_{i-1} + 6 f_i - 4 f_{i+1} + f_{i+2})
 * for f in {q, W}.  sigma = 0 disables it (default).  field_mask must be
 * (1<<1)|(1<<3) (q and W) or 0. */
hsgn_status hsgn_set_filter(hsgn_ctx *ctx, double sigma, uint32_t field_mask);

/* Relaxation zones (A10, cfg4), applied to U^{n+1} after the filter:
 * U -= s(x) (U - U_target(x, t^{n+1})), x_i = x_min + (i + 1/2) dx.
 *   wavemaker x <= gen_x1: s = gen_rate (1 - (x - x_min)/(gen_x1 - x_min))^2,
 *     eta = amp sin(omega t - k (x - x_min)), h = level + eta - b,
 *     q = h cp eta / level, K = h (h + 1.5 b), W = 0;
 *   sponge x >= sp_x0: s = sp_rate ((x - sp_x0)/(x_max - sp_x0))^2, lake at rest
 *     h = level - b, q = 0, K = h (h + 1.5 b), W = 0.
 * A rate <= 0 disables a zone; NULL disables both (default). */
typedef struct {
    double level, gen_x1, gen_rate, amp, omega, k, cp, sp_x0, sp_rate;
} hsgn_relax;
hsgn_status hsgn_set_relaxation(hsgn_ctx *ctx, const hsgn_relax *relax);

/* ---- state -------------------------------------------------------------- */

/* Copy in (h, q, K, W), each n_members * n_cells doubles, host or device
 * pointers; t0 is the start time of every member.  Also (re)computes the
 * max|u| and max(|u|+c) the first step's dt needs, and clears errors. */
hsgn_status hsgn_set_state(hsgn_ctx *ctx, const double *h, const double *q, const double *K,
                           const double *W, double t0);
/* Copy out the last committed state; any pointer may be NULL.  t (host array
 * of n_members, or NULL) receives each member's time.  Synchronises.  Returns a
 * latched device error of a failed step (HSGN_E_COERCIVITY, _DRY, _NONFINITE,
 * _OVERLAP, _INVALID for a bad dt) after making the copy: the data are then the
 * last committed state, which the failed step left untouched. */
hsgn_status hsgn_get_state(hsgn_ctx *ctx, double *h, double *q, double *K, double *W,
                           double *t);
/* Whole ensemble job from and to host memory, pipelined over member chunks
 * (DESIGN.md section 7): the members are split into `chunks` contiguous
 * groups (at most 16 and n_members); for each group, in order, its initial
 * state (h, q, K, W: n_members * n_cells doubles each, member-major, as for
 * hsgn_set_state) is copied in on one copy stream, n_steps steps run on the
 * context's stream or, for odd groups, a second compute stream ordered after
 * the context's earlier work (exactly as hsgn_set_state + hsgn_run_steps would: members
 * are independent, so each member's result is bitwise the same), and its final
 * state and times are copied out on a second copy stream -- group k+1's input
 * and group k-1's output transfers overlap group k's steps.  Use page-locked
 * host buffers for the overlap (pageable ones work, serialised).  t0: start
 * time of every member; t_out (n_members doubles, or NULL) receives the final
 * times.  Synchronises before returning.  Afterwards the context holds no state
 * (call hsgn_set_state before hsgn_step / hsgn_run_steps).  Not for slab
 * contexts or the SGN scheme (its tile geometry depends on the whole state).
 * Errors: HSGN_E_INVALID (null pointer, n_steps < 0, chunks < 1, slab / SGN),
 * HSGN_E_NOWORKSPACE, HSGN_E_CUDA; a device error in a group (dry bed,
 * coercivity, non-finite, overlap) returns that status, and that group's
 * outputs hold its last committed state and times. */
hsgn_status hsgn_run_host(hsgn_ctx *ctx, const double *h, const double *q, const double *K,
                          const double *W, double t0, int64_t n_steps, double *h_out,
                          double *q_out, double *K_out, double *W_out, double *t_out,
                          int32_t chunks);

/* ---- stepping ------------------------------------------------------------ */

/* One SI-IMEX step.  dt > 0: fixed step for every member; dt <= 0: the
 * two-condition rule of P:613-617 per member.  If dt_used (host, n_members)
 * is non-NULL the call synchronises and reports the dt each member took. */
hsgn_status hsgn_step(hsgn_ctx *ctx, double dt, double *dt_used);
/* Enqueue n_steps automatic-dt steps (CUDA-graph replay); asynchronous.
 * Per step: the stage kernels and one commit / next-dt kernel; for small
 * ensembles (at most two waves of stage CTAs, e.g. cfg1 and cfg2) the first
 * stage evaluates the dt rule itself and one commit kernel closes each
 * sequence of steps -- same dt, same results. */
hsgn_status hsgn_run_steps(hsgn_ctx *ctx, int64_t n_steps);
/* Advance every member to t_end (last step clipped), at most max_steps
 * steps; polls the device every `poll` steps.  *steps_done = steps taken. */
hsgn_status hsgn_advance_to(hsgn_ctx *ctx, double t_end, int64_t max_steps,
                            int64_t *steps_done);
/* Run n_steps automatic-dt steps as ONE CUDA graph (captured with event record
 * nodes before, between and after the kernels, then launched once -- the launch
 * mode of hsgn_run_steps), synchronise, and return (ms, device clock) in
 * stage_ms[0] / stage_ms[1] the summed time of the stage-1 / stage-2 kernels
 * (stage_ms[1] = 0 for a 1-stage tableau) and in stage_ms[2] the time of the whole n steps (first to last
 * kernel).  stage_ms: 3 doubles.  Same arithmetic as hsgn_run_steps; used by
 * bench.py for the step time and the per-kernel rooflines.  Needs a
 * non-default stream; not for slab contexts (HSGN_E_INVALID). */
hsgn_status hsgn_run_steps_timed(hsgn_ctx *ctx, int64_t n_steps, double *stage_ms);
/* Wait for the stream; return the latched device status. */
hsgn_status hsgn_sync(hsgn_ctx *ctx);

/* ---- diagnostics ----------------------------------------------------------- */
hsgn_status hsgn_get_diagnostics(hsgn_ctx *ctx, hsgn_diag *out);
/* Number of kernel launches enqueued by this context since creation. */
int64_t hsgn_launch_count(const hsgn_ctx *ctx);
/* Time-stepping scheme.  HSGN_SCHEME_SI (default): the
 * semi-implicit IMEX step of P:500-517.  HSGN_SCHEME_EXPLICIT: the explicit
 * hSGN scheme of P:442-458 -- central D_x for the mass flux and the pressure
 * gradient with a^2, alpha at the cell, Rusanov D^_x on the MUSCL
 * faces for the convective fluxes, relaxation sources -- advanced
 * by forward Euler (stages = 1) or Heun (stages = 2); dt = CFL dx /
 * max(|u| + c) with the CFL of hsgn_set_params (the material MCFL is not
 * used); the A19 filter applies if set.  Explicit runs need a flat bottom, no
 * relaxation zones and no slab sides (HSGN_E_INVALID at the next step
 * otherwise).  Errors: HSGN_E_INVALID (unknown scheme, stages not 1 or 2). */
#define HSGN_SCHEME_SI 0
#define HSGN_SCHEME_EXPLICIT 1
/* HSGN_SCHEME_SGN: the classical SGN equations in elliptic-hyperbolic form
 * on (h, q) -- Rusanov shallow water on MUSCL
 * faces with alpha = max(|u| + sqrt(g h)), a tridiagonal phi system per stage
 * (reading A23: g h^3 in h*), source h phi; Euler or Heun;
 * dt = CFL dx / max(|u| + sqrt(g h)); K, W are carried unchanged.
 * With bathymetry (hsgn_set_bathymetry) the phi system carries the kappa, rho, Q
 * closure of P:562-578 and the momentum the hydrostatic source -g h b_x
 * (reading A26).  No filter, no relaxation zones or slabs.  The phi overlap is
 * chosen from the state (hsgn_set_state / hsgn_set_scheme); HSGN_E_INVALID if
 * dx is too small against h for the tile width. */
#define HSGN_SCHEME_SGN 2
hsgn_status hsgn_set_scheme(hsgn_ctx *ctx, int32_t scheme, int32_t stages);
/* Picard re-linearisation of the depth equation (reading A24, SURVEY 8(f)
 * row f4): after the paper's linearised solve of each SI
 * stage, `passes` more assemble+solve passes with beta1 = 1 + lam tau^2/h^2
 * and beta2 = 2 lam tau^2/(beta1^2 h^3) (hence kappa = beta and delta) at the
 * latest hbar, alpha and a^2 staying at the stage input E.  0 (default) = the
 * paper's scheme.  Runs on the overlapped-tile stage kernels; not with relaxation zones or the
 * explicit / SGN schemes (HSGN_E_INVALID at the next step).  Errors:
 * HSGN_E_INVALID (null context, passes outside 0..16). */
hsgn_status hsgn_set_picard(hsgn_ctx *ctx, int32_t passes);
/* Exactly well-balanced face form of the SI stage (reading A25, SURVEY 8(f)
 * row f4; P:163-171 hSGNb): the depth right-hand side uses the face
 * coefficient dhat_{i+1/2} = -(2 sigma^ - 1)/(3 h~) b1~ (face averages of
 * sigma = H/h^2, h and 1/beta1 at E) in place of (delta_i + delta_{i+1})/2,
 * and qbar = q^dag - tau/(2 dx) (Phi_{i+1/2} + Phi_{i-1/2}) with the face
 * fluxes Phi = beta~ (hbar_R - hbar_L) + lam dhat (H^dag_R - H^dag_L)
 * + g h~ (b_R - b_L).  The lake at rest over any bathymetry is then a fixed
 * point to round-off at lam > 0 (the paper's cell-centred form keeps it to
 * O(dx^2) only, reading A9); the scheme stays conservative and second order.
 * on = 0 (default): the paper's form.  Runs on the one-CTA-per-tile stage
 * kernels; not with Picard passes or the explicit / SGN schemes
 * (HSGN_E_INVALID at the next step).  Drops captured graphs.  Errors:
 * HSGN_E_INVALID (null context). */
hsgn_status hsgn_set_well_balanced(hsgn_ctx *ctx, int32_t on);
/* Exact depth solve across tiles (hsgn_cluster.cuh).
 * Cluster kernels: the C CTAs of a member form one thread-block cluster and
 * solve the depth system of P:509-512 EXACTLY across their tiles (partition
 * method per thread chunk, interior PCR with two spike columns, one DSMEM
 * exchange of 12 doubles per CTA, a C-unknown separator system solved
 * redundantly per CTA; cyclic for periodic members) -- no overlap rows and no
 * decay condition.  They need the member to fit: n_cells % 4 == 0, both sides
 * periodic (C = the smallest power of two with n_cells <= 512 C) or both
 * physical (wall / transmissive, C = ceil(n_cells / 512)), C <= 16.
 * Tile-level SPIKE (members of any size, n_cells % 4 == 0): per stage, the
 * tiles' reduced systems (12 values per tile to global memory), one CTA per
 * member solving the separator system exactly (the same scheme one level up),
 * the tiles recomputed and finished with their separator values, and, with the
 * A19 filter, the two rows at each tile end completed by a small kernel: about
 * 2x the work of a stage on the overlapped tiles, for any decay length.
 * Slab contexts (HSGN_BC_HALO sides, group or NCCL transport; every slab in the
 * same mode): tile-level SPIKE spans all slabs -- each slab solves its
 * separator system for Y and the spike columns V, W of its two outer
 * couplings, the slabs exchange 6 doubles right-to-left and all-gather 6 per
 * slab, and every slab solves the 2P end-separator system (DESIGN.md section
 * 8); halos shrink to the 4-row stencil.  The host-staged transport refuses it.
 * Both: the SI stage without Picard passes or the A25 form; the cluster
 * kernels also not on slab contexts.
 * mode 0: never (overlapped tiles with the decay check); 1: the cluster kernels
 * whenever the member fits; 3: tile-level SPIKE whenever eligible; 2 (default,
 * "auto"): exact paths only when the overlapped tiles cannot bound the decay a
 * priori, i.e. material-CFL-only stepping (cfl_imex <= 0) without a
 * user overlap -- the cluster kernels if the member fits, else tile-level
 * SPIKE -- or when the overlapped tiles solve many redundant rows ((T + 2w) / T
 * >= 1.5 for the cluster kernels, >= 2.4 for SPIKE, e.g. the first-order SI
 * step); the overlapped tiles are faster on B200 when CFL_IMEX bounds rho
 * tightly (the paper's tableau at CFL_IMEX 2: 1.19 rows per kept cell).
 * Drops captured graphs.  Errors: HSGN_E_INVALID (null context, mode outside
 * 0..3). */
hsgn_status hsgn_set_cluster(hsgn_ctx *ctx, int32_t mode);
/* Member-resident stepping (hsgn_multi.cuh): the C CTAs
 * of every member (one cluster, as for the cluster kernels: the member must
 * fit) load its state once, advance it by n_steps full SI-IMEX steps with the
 * dt rule of P:613-617 (per member, the last step clipped to t_end if t_end > 0,
 * S:342; a member at t_end stays there for the remaining steps), keeping the state, the stage inputs E2, R2 and
 * all intermediates in shared memory and exchanging only edge rows,
 * separator data and dt maxima between the CTAs (DSMEM), and store it once.
 * Same arithmetic as hsgn_run_steps on the cluster kernels up to rounding
 * order (E2, R2 formed in the H-form).  Synchronous; *device_ms (or NULL)
 * receives the kernel's device time.  2-stage tableau, SI scheme without
 * Picard passes, the A25 form or slab sides.  On a device error (coercivity,
 * dry bed, non-finite, dt) the call returns it and the state stays at the
 * call's start for every member; otherwise n_steps steps are committed.
 * Errors: HSGN_E_INVALID (not eligible, n_steps < 0), HSGN_E_NOWORKSPACE,
 * HSGN_E_CUDA, device errors as above. */
hsgn_status hsgn_run_resident(hsgn_ctx *ctx, int64_t n_steps, double t_end, double *device_ms);
/* 1 if the next step runs on the cluster kernels, 2 if on tile-level SPIKE
 * (then *ctas = CTAs (tiles) per member and *tile_rows = rows per tile, the last
 * n_cells - (ctas - 1) * tile_rows), 0 for the overlapped tiles (both 0), -1 for
 * a null context.  Either pointer may be NULL. */
int32_t hsgn_get_cluster(const hsgn_ctx *ctx, int32_t *ctas, int32_t *tile_rows);
/* Tile geometry chosen by hsgn_create: kept cells per tile, overlap, tiles per
 * member, threads per CTA, max rows per CTA. */
hsgn_status hsgn_get_geometry(const hsgn_ctx *ctx, int32_t *tile_cells, int32_t *overlap,
                              int32_t *tiles_per_member, int32_t *threads, int32_t *max_rows);

/* ---- slab decomposition of one domain --
 * A domain of N cells split into P contiguous slabs, slab i a context whose
 * interior sides are HSGN_BC_HALO.  Each step: max-reduce the dt maxima across
 * slabs, dt, exchange w + 3 boundary cells of U^n, stage 1, exchange U1,
 * stage 2, commit.  Two transports:
 *   group: all slabs in this process on one device and one stream (device-to-
 *          device copies; ctxs in ring order, ctxs[i-1] left of ctxs[i]);
 *          bathymetry must be set before hsgn_group_create;
 *   NCCL:  one slab per process/GPU, ring by rank (send/recv of the halos,
 *          all-reduce max of the dt maxima), on the context's stream. */
typedef struct hsgn_group hsgn_group;
hsgn_status hsgn_group_create(hsgn_ctx *const *ctxs, int32_t n, hsgn_group **out);
hsgn_status hsgn_group_run_steps(hsgn_group *g, int64_t n_steps);
void hsgn_group_destroy(hsgn_group *g);
/* Development aid: copy `count` doubles of an internal SPIKE array to host
 * memory (which: 0 separators L [members][G], 1 slab Y, V, W [3][members][G],
 * 2 slab end separators (E_{p-1}, F_{p+1}) [members][2], 3 right slab's tile-0
 * relation [members][6], 4 all-gathered end values [P][members][6], 5 tile tips
 * [members][G][12], 6 unfiltered tile-end rows [members][G][16]).  Synchronises.
 * Errors: HSGN_E_INVALID (null pointer, unknown or unallocated array). */
hsgn_status hsgn_debug_copy(hsgn_ctx *ctx, int32_t which, double *host, int64_t count);
/* 128-byte ncclUniqueId (rank 0; the caller broadcasts it, e.g. torch.distributed) */
hsgn_status hsgn_nccl_unique_id(void *id);
/* Collective over the `world` ranks (every rank calls it with the same id).
 * Checks that every rank has the same overlap w and member count (an NCCL
 * max-reduce at attach time) and n_cells >= w + 3; the overlap must then stay
 * as attached (a later hsgn_set_params that changes w makes hsgn_run_steps
 * return HSGN_E_INVALID).  Errors: HSGN_E_INVALID (no BC_HALO side, already
 * attached, slab shorter than its halo, ranks disagree), HSGN_E_COMM, HSGN_E_CUDA. */
hsgn_status hsgn_attach_nccl(hsgn_ctx *ctx, const void *id, int32_t rank, int32_t world);

/* ---- host-staged slab transport (any process-group transport, e.g. gloo) --
 * One slab step of a context with HSGN_BC_HALO sides, neither grouped nor
 * NCCL-attached, in phases; between them the caller moves the data with its
 * own collectives (tests/test_gpu_slab_gloo.py):
 *   1. hsgn_slab_get(MAXIMA) -> max-reduce over the slabs -> hsgn_slab_put(MAXIMA)
 *      (2 n_members uint64: bit patterns of the non-negative max|u|, max(|u|+c)
 *      of U^n; the max of the bit patterns is the max of the values)
 *   2. hsgn_slab_phase(HSGN_PHASE_DT)           dt of the step (clipped to t_end)
 *   3. hsgn_slab_get(UN): [left boundary: 4 x H][right boundary: 4 x H] of U^n
 *      (h, q, K, W; H = overlap + 3 cells), send the left part to the left
 *      neighbour and the right part to the right one; hsgn_slab_put(UN):
 *      [left halo: 4 x H (the left neighbour's right boundary)][right halo]
 *   4. hsgn_slab_phase(HSGN_PHASE_STAGE1)
 *   5. as 3 with U1 (UN -> U1), then hsgn_slab_phase(HSGN_PHASE_STAGE2)
 *      (2-stage tableaux only)
 *   6. hsgn_slab_phase(HSGN_PHASE_COMMIT)
 * With bathymetry, the static b halos are exchanged once the same way (B: 1
 * field) before the first step.  hsgn_slab_xfer_count gives the doubles (or
 * uint64) of one get/put buffer.  get/put synchronise the context's stream;
 * phases only enqueue.  Errors: HSGN_E_INVALID (not a host-staged slab
 * context, unknown transfer or phase, STAGE2 with a 1-stage tableau). */
#define HSGN_XFER_MAXIMA 0
#define HSGN_XFER_UN 1
#define HSGN_XFER_U1 2
#define HSGN_XFER_B 3
#define HSGN_PHASE_DT 0
#define HSGN_PHASE_STAGE1 1
#define HSGN_PHASE_STAGE2 2
#define HSGN_PHASE_COMMIT 3
int64_t hsgn_slab_xfer_count(const hsgn_ctx *ctx, int32_t what);
hsgn_status hsgn_slab_get(hsgn_ctx *ctx, int32_t what, void *host_out);
hsgn_status hsgn_slab_put(hsgn_ctx *ctx, int32_t what, const void *host_in);
hsgn_status hsgn_slab_phase(hsgn_ctx *ctx, int32_t phase);

const char *hsgn_status_string(hsgn_status s);
const char *hsgn_last_error(const hsgn_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* HSGN_H_ */
