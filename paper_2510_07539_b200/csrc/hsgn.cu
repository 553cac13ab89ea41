// hsgn.cu -- C ABI runtime of libhsgn.so (see include/hsgn.h).
//
// Host side: validates the problem, chooses the tile geometry, lays out the
// caller-provided workspace, launches the stage kernels of
// hsgn_kernels.cuh on the caller's stream, and replays CUDA graphs of
// GRAPH_STEPS steps for hsgn_run_steps / hsgn_advance_to.  One step k =
// stage 1, stage 2, dt_commit(k+1) (commit step k, dt of step k+1); every run
// starts with dt_commit(k, no commit).  Never allocates
// device memory and never falls back to the CPU.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hsgn.h"
#include "hsgn_kernels.cuh"
#include "hsgn_cluster.cuh"
#include "hsgn_multi.cuh"

using namespace hsgn;

namespace {

constexpr int GRAPH_STEPS = 18;   // steps per captured graph: a multiple of 6, so the buffer
                                  // parity (k mod 2) and the maxima slot (k mod 3) repeat
constexpr int POLL_STEPS = 256;   // advance_to polls the device every POLL_STEPS
constexpr int T_MIN = 64;         // smallest kept tile (bounds the partials workspace)
constexpr int H_MAX = (LCAP - 2 - T_MIN) / 2 + 3;   // largest slab halo (overlap + stencil)
constexpr int KIDS_MAX = 16;      // member chunks of hsgn_run_host
constexpr int GROUP_MAX_SX = 64;  // slabs of one domain (= GROUP_MAX)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// small per-member arrays of one member chunk of hsgn_run_host
size_t kid_small_bytes(int n, int cnt)
{
    return align256(2 * size_t(cnt) * 8) + 2 * align256(size_t(cnt) * 8) + align256(6 * size_t(cnt) * 8) +
           align256(size_t(cnt) * ((n + T_MIN - 1) / T_MIN + 1) * 4 * 8) + 512;
}

}  // namespace

struct hsgn_ctx {
    hsgn_desc desc{};
    cudaStream_t stream = nullptr;
    int device = 0;
    // geometry
    int n = 0, members = 0, T = 0, w = 0, tiles = 0;
    double dx = 0;
    // parameters
    double g = 9.81, cfl = 2.0, mcfl = 0.5, h_min = 1e-8;
    std::vector<double> lam;
    bool have_params = false, have_state = false, bathy = false;
    hsgn_tableau tab{};
    double aI1 = 0, aI2 = 0, wE = 0, wR = 0;
    double filter_sigma = 0;
    hsgn_relax relax{};
    // workspace
    char *ws = nullptr;
    size_t ws_bytes = 0;
    double *buf[3][4] = {};     // [A, B, U1][field]
    double *b = nullptr, *lamd = nullptr, *t = nullptr, *dt = nullptr, *dt_used = nullptr,
           *partials = nullptr;
    unsigned long long *maxes = nullptr, *rho_obs = nullptr;
    unsigned int *kmin = nullptr;
    unsigned int *err = nullptr, *done = nullptr;
    long long *steps = nullptr;
    Ctrl *ctrl = nullptr;
    // host bookkeeping
    int cur = 0;                  // buffer index holding the state at device step `base_steps`
    long long host_steps = 0;     // steps enqueued since set_state
    long long dev_steps = 0;      // committed device steps at the last reconcile
    Ctrl ctrl_host{0.0, 0.0};
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    long long launches = 0;
    // slab decomposition (BC_HALO sides): halo receive buffers [9][H_MAX] per side
    double *halo_l = nullptr, *halo_r = nullptr;
    bool slab = false;
    // scheme: 0 = SI-IMEX (default), 1 = explicit hSGN (P:442-480,
    // x_stages 1 = Euler, 2 = Heun) on tiles of xT cells
    int scheme = 0, x_stages = 2, xT = 0, xtiles = 0;
    // classical SGN (scheme 2): phi-system overlap and tiles, from the state
    int sw = 0, sT = 0, stiles = 0;
    int picard = 0;               // A24 Picard passes of the SI depth solve (0: the paper's)
    bool wb = false;              // A25 exactly well-balanced face form of the SI stage
    bool ev_ext = false;          // record events as graph nodes (timed capture)
    // cluster stage kernels (exact depth solve across the CTAs of a cluster,
    // hsgn_cluster.cuh): C CTAs of clT rows per member; used whenever the
    // member fits (n <= 16 * 512, n % 4 == 0) and the step is the SI stage
    // without Picard passes, the A25 form, relaxation zones or slab sides
    int cl_mode = 2;              // 0 off, 1 on (when the member fits), 2 auto: on when the
                                  // overlapped tiles cannot bound the decay a priori
                                  // (material-CFL-only stepping); HSGN_CLUSTER overrides
    int clC = 0, clT = 0;
    // tile-level SPIKE (general exact path: any member size): spG tiles of spT
    // rows per member; buffers in the workspace (tips, L, filter rows, scratch)
    int spG = 0, spT = 0;
    double *sp_tips = nullptr, *sp_L = nullptr, *sp_fb = nullptr, *sp_S = nullptr;
    // SPIKE across slabs (slab contexts only; Params::sx_*)
    double *sx_nx = nullptr, *sx_fbl = nullptr, *sx_fbr = nullptr, *sx_elfr = nullptr;
    double *sx_yvw = nullptr, *sx_all = nullptr, *sx_send = nullptr;
    ncclComm_t nccl = nullptr;
    int nrank = 0, nworld = 1;
    int nccl_w = -1;              // overlap w at hsgn_attach_nccl (the halo size every rank agreed on)
    std::string last_error;
    // hsgn_run_host pipeline: member-chunk views of this context (their state
    // buffers are slices of ours, their small arrays live in the workspace tail)
    std::vector<hsgn_ctx *> kids;
    long long gen = 0, kids_gen = -1;   // settings generation (bumped by drop_graphs)
    char *kid_ws = nullptr;
    cudaStream_t cp_in = nullptr, cp_out = nullptr;
    cudaStream_t cs2 = nullptr;         // second compute stream (odd chunks) or null
    cudaEvent_t ev_start = nullptr, ev_in[16] = {}, ev_done[16] = {};
    long long *kstat = nullptr;         // pinned [16][2]: error bits, committed steps
    double *tstage = nullptr;           // pinned [n_members]: final times (a pageable
                                        // destination would block the enqueue loop)
};

namespace {

hsgn_status fail(hsgn_ctx *c, hsgn_status s, const std::string &msg)
{
    if (c) c->last_error = msg;
    return s;
}

#define CUDA_TRY(c, expr)                                                              \
    do {                                                                               \
        cudaError_t e_ = (expr);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail((c), HSGN_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
    } while (0)

hsgn_status status_from_bits(unsigned int bits)
{
    if (!bits) return HSGN_OK;
    if (bits & ERR_COERC) return HSGN_E_COERCIVITY;
    if (bits & ERR_DRY) return HSGN_E_DRY;
    if (bits & ERR_NONFINITE) return HSGN_E_NONFINITE;
    if (bits & ERR_OVERLAP) return HSGN_E_OVERLAP;
    if (bits & ERR_DT) return HSGN_E_INVALID;
    return HSGN_E_INVALID;
}

int slab_H(const hsgn_ctx *c);

Params make_params(hsgn_ctx *c, long long k)
{
    Params P{};
    P.kslot = int(k % 3);
    P.kpar = int(k & 1);
    P.n = c->n; P.members = c->members; P.tiles = c->tiles; P.T = c->T; P.w = c->w;
    P.bcl = c->desc.bc_left; P.bcr = c->desc.bc_right; P.order = c->desc.order;
    P.dx = c->dx; P.idx = 1.0 / c->dx; P.g = c->g; P.h_min = c->h_min; P.cfl = c->cfl; P.mcfl = c->mcfl;
    P.aI1 = c->aI1; P.aI2 = c->aI2; P.wE = c->wE; P.wR = c->wR;
    P.filter_sigma = c->filter_sigma;
    P.x_min = c->desc.x_min; P.x_max = c->desc.x_max;
    P.level = c->relax.level; P.gen_x1 = c->relax.gen_x1; P.gen_rate = c->relax.gen_rate;
    P.amp = c->relax.amp; P.omega = c->relax.omega; P.kw = c->relax.k; P.cp = c->relax.cp;
    P.sp_x0 = c->relax.sp_x0; P.sp_rate = c->relax.sp_rate;
    P.b = c->bathy ? c->b : nullptr;
    P.lam = c->lamd; P.t = c->t; P.dt = c->dt; P.maxes = c->maxes; P.err = c->err;
    P.steps = c->steps; P.done = c->done; P.rho_obs = c->rho_obs; P.kmin = c->kmin; P.ctrl = c->ctrl;
    P.H = slab_H(c);
    if (c->scheme == 1) {            // explicit: its own tiles, dt = CFL_EX dx / mu_max only
        P.T = c->xT;
        P.tiles = c->xtiles;
        P.mcfl = 0.0;
    } else if (c->scheme == 2) {     // classical SGN: phi tiles, dt = CFL_SGN dx / max(|u| + sqrt(g h))
        P.T = c->sT;
        P.tiles = c->stiles;
        P.w = c->sw;
        P.mcfl = 0.0;
    }
    P.inv_tiles = 1.0 / double(c->tiles);
    {   // r = 2 rho/(1 + 2 rho + sqrt(1 + 4 rho)) inverts to rho = r/(1 - r)^2
        const double r = std::exp2(-60.0 / double(std::max(P.w, 1)));
        P.rho_ok = r / ((1.0 - r) * (1.0 - r));
    }
    P.picard = c->picard;
    P.sp_tips = c->sp_tips; P.sp_L = c->sp_L; P.sp_fb = c->sp_fb; P.sp_S = c->sp_S;
    P.sx_nx = c->sx_nx; P.sx_fbl = c->sx_fbl; P.sx_fbr = c->sx_fbr; P.sx_elfr = c->sx_elfr;
    P.sx_yvw = c->sx_yvw; P.sx_all = c->sx_all; P.sx_send = c->sx_send;
    P.sx_rank = c->nrank; P.sx_P = c->nworld;
    for (int k = 0; k < 9; k++) {
        P.halo_l[k] = c->halo_l ? c->halo_l + k * H_MAX : nullptr;
        P.halo_r[k] = c->halo_r ? c->halo_r + k * H_MAX : nullptr;
    }
    return P;
}

// Plain launch on the context's stream (cudaLaunchKernelEx, no attributes).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(hsgn_ctx *c, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

// Event record on the context's stream; inside a timed capture as an event
// record node of the graph (cudaEventRecordExternal), so it times the replay.
cudaError_t rec_ev(hsgn_ctx *c, cudaEvent_t e)
{
    return c->ev_ext ? cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal)
                     : cudaEventRecord(e, c->stream);
}

template <bool S2, bool FIN, bool BATHY>
hsgn_status launch_stage(hsgn_ctx *c, const Params &P, const Bufs &B)
{
    const bool relax = FIN && (c->relax.gen_rate > 0.0 || c->relax.sp_rate > 0.0);
    const size_t sm = BATHY ? SMEM_BYTES_B : SMEM_BYTES;    // one-CTA-per-tile kernels: b in smem
    if (c->picard > 0) {             // A24: one CTA per tile, Picard variant
        dim3 grid(c->tiles, c->members);
        CUDA_TRY(c, launch_k(c, stage_kernel<S2, FIN, BATHY, false, true>, grid, dim3(NT),
                               BATHY ? SMEM_BYTES_PIC_B : SMEM_BYTES_PIC, P, B));
    } else if (c->wb) {              // A25: one CTA per tile, face form
        dim3 grid(c->tiles, c->members);
        if (relax) CUDA_TRY(c, launch_k(c, stage_kernel<S2, FIN, BATHY, true, false, true>, grid, dim3(NT), sm, P, B));
        else CUDA_TRY(c, launch_k(c, stage_kernel<S2, FIN, BATHY, false, false, true>, grid, dim3(NT), sm, P, B));
    } else {
        dim3 grid(c->tiles, c->members);
        if (relax) CUDA_TRY(c, launch_k(c, stage_kernel<S2, FIN, BATHY, true>, grid, dim3(NT), sm, P, B));
        else if (S2 == FIN && P.fuse_dt)     // small ensembles: the latency variants
            CUDA_TRY(c, launch_k(c, stage_kernel<S2, FIN, BATHY, false, false, false, true>, grid, dim3(NT), sm, P, B));
        else CUDA_TRY(c, launch_k(c, stage_kernel<S2, FIN, BATHY, false>, grid, dim3(NT), sm, P, B));
    }
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return HSGN_OK;
}

template <bool S2, bool FIN>
hsgn_status launch_stage_b(hsgn_ctx *c, const Params &P, const Bufs &B)
{
    return c->bathy ? launch_stage<S2, FIN, true>(c, P, B) : launch_stage<S2, FIN, false>(c, P, B);
}

// Cluster path eligibility for the current settings (the geometry clC, clT
// depends only on n and the boundary kinds and is fixed at hsgn_create).
bool exact_eligible(const hsgn_ctx *c)
{
    return c->scheme == 0 && !c->slab && c->picard == 0 && !c->wb;
}

// tile-level SPIKE also runs on slab contexts (across slabs, section 8)
bool spike_eligible(const hsgn_ctx *c)
{
    return c->scheme == 0 && c->picard == 0 && !c->wb;
}

// material-CFL-only stepping without a user overlap: the overlapped tiles
// cannot bound the depth system's decay a priori
bool overlap_unbounded(const hsgn_ctx *c) { return !(c->cfl > 0.0) && c->desc.overlap <= 0; }

// rows the overlapped tiles solve per kept cell, (T + 2w) / T (1 when the caller
// chose the tile geometry: then auto mode keeps the tiles)
double tile_redundancy(const hsgn_ctx *c)
{
    if (c->desc.tile_cells > 0 || c->desc.overlap > 0 || c->T <= 0) return 1.0;
    return double(c->T + 2 * c->w) / c->T;
}

// auto mode (2): the exact paths also win where the overlap tax is high.
// Measured on cfg3: per solved row the cluster kernels
// cost ~1.33x and tile-level SPIKE ~1.9x the overlapped tiles, which solve
// (T + 2w) / T rows per kept cell (1.19 at CFL_IMEX 2 with the paper's
// tableau, 1.91 for the first-order SI step: cluster 27.3 vs tiles 24.4 G)
constexpr double AUTO_CLUSTER_REDUNDANCY = 1.5, AUTO_SPIKE_REDUNDANCY = 2.4;

bool use_cluster(const hsgn_ctx *c)
{
    const bool on = c->cl_mode == 1 ||
                    (c->cl_mode == 2 && (overlap_unbounded(c) || tile_redundancy(c) >= AUTO_CLUSTER_REDUNDANCY));
    return on && c->clC > 0 && exact_eligible(c);
}

bool use_spike(const hsgn_ctx *c)
{
    if (use_cluster(c) || c->spG <= 0 || !spike_eligible(c) || c->sp_tips == nullptr) return false;
    return c->cl_mode == 3 ||
           (c->cl_mode == 2 && (overlap_unbounded(c) || (!c->slab && tile_redundancy(c) >= AUTO_SPIKE_REDUNDANCY)));
}

// ghost cells a BC_HALO side takes from its neighbour per exchange: the
// overlapped tiles need w + 3 (overlap + stencil), SPIKE across slabs only the
// stencil's 4 rows (the depth coupling goes through the separators)
int slab_H(const hsgn_ctx *c) { return use_spike(c) ? 4 : c->w + 3; }

void choose_spike(hsgn_ctx *c)
{
    c->spG = c->spT = 0;
    const int bl = c->desc.bc_left, br = c->desc.bc_right;
    const bool cyc = bl == HSGN_BC_PERIODIC && br == HSGN_BC_PERIODIC;
    // non-periodic sides: physical or slab halo (SPIKE across slabs)
    auto side = [](int b) { return b == HSGN_BC_WALL || b == HSGN_BC_TRANSMISSIVE || b == HSGN_BC_HALO; };
    const bool phys = side(bl) && side(br);
    const int n = c->n;
    if ((!cyc && !phys) || (n % 4) != 0 || n < 8) return;
    const int G = (n + CT_MAX - 1) / CT_MAX;
    int T = G == 1 ? n : CT_MAX;
    if (G > 1 && n - (G - 1) * T < 8) T = CT_MAX - 4;      // last tile 4 rows: shorten the others
    if (G > 1 && (n - (G - 1) * T < 8 || n - (G - 1) * T > CT_MAX)) return;
    c->spG = G;
    c->spT = T;
}

size_t spike_bytes(const hsgn_ctx *c)
{
    // per member and tile: 12 (tips) + 1 (L) + 16 (filter rows) doubles, and the
    // separator solve's scratch (sep_scratch: 3 G, or 6 (G + 1024) for G > 1024)
    const int G = std::max(c->spG, 1);
    const size_t sx = c->slab ? size_t(c->members) * (6 + 8 + 8 + 2 + 16 + 6 * GROUP_MAX_SX + 3 * size_t(G)) : 0;
    return 12 * 256 + (size_t(c->members) * (size_t(G) * 29 + sep_scratch(G)) + sx) * sizeof(double);
}

void choose_cluster(hsgn_ctx *c)
{
    c->clC = c->clT = 0;
    const int bl = c->desc.bc_left, br = c->desc.bc_right;
    const bool cyc = bl == HSGN_BC_PERIODIC && br == HSGN_BC_PERIODIC;
    const bool phys = (bl == HSGN_BC_WALL || bl == HSGN_BC_TRANSMISSIVE) &&
                      (br == HSGN_BC_WALL || br == HSGN_BC_TRANSMISSIVE);
    const int n = c->n;
    if ((!cyc && !phys) || (n % 4) != 0) return;
    int C;
    if (cyc) {                    // cyclic separator PCR: C a power of two
        C = 1;
        while (C * CT_MAX < n) C *= 2;
    } else {
        C = (n + CT_MAX - 1) / CT_MAX;
    }
    if (C > C_MAX) return;
    const int T = (((n + C - 1) / C) + 3) / 4 * 4;
    const int last = n - (C - 1) * T;
    if (T < 8 || T > CT_MAX || last < 8) return;
    c->clC = C;
    c->clT = T;
}

template <bool S2, bool FIN, bool BATHY>
hsgn_status launch_cl(hsgn_ctx *c, Params P, const Bufs &B)
{
    P.T = c->clT;
    P.tiles = c->clC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->clC, c->members);
    cfg.blockDim = dim3(CNT);
    cfg.dynamicSmemBytes = BATHY ? CSMEM_BYTES_B : CSMEM_BYTES;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(c->clC);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(c, cudaLaunchKernelEx(&cfg, cl_stage_kernel<S2, FIN, BATHY>, P, B));
    c->launches++;
    return HSGN_OK;
}

template <bool S2, bool FIN>
hsgn_status launch_cl_b(hsgn_ctx *c, const Params &P, const Bufs &B)
{
    return c->bathy ? launch_cl<S2, FIN, true>(c, P, B) : launch_cl<S2, FIN, false>(c, P, B);
}

template <bool S2, bool FIN, bool BATHY>
hsgn_status launch_spike(hsgn_ctx *c, Params P, const Bufs &B)
{
    P.T = c->spT;
    P.tiles = c->spG;
    P.sp_tips = c->sp_tips; P.sp_L = c->sp_L; P.sp_fb = c->sp_fb; P.sp_S = c->sp_S;
    const dim3 grid(c->spG, c->members);
    if (c->slab) return HSGN_E_INVALID;               // slabs: slab_spike_stage
    const size_t sm = BATHY ? CSMEM_BYTES_B : CSMEM_BYTES;
    CUDA_TRY(c, launch_k(c, cl_stage_kernel<S2, FIN, BATHY, CL_MODE_TIPS>, grid, dim3(CNT), sm, P, B));
    if (c->spG > 1024) {
        CUDA_TRY(c, launch_k(c, sep_coef_kernel, dim3((c->spG + 255) / 256, c->members), dim3(256), 0, P, 0));
        CUDA_TRY(c, launch_k(c, sep_solve_kernel<1024>, dim3(c->members), dim3(1024), sep_smem_bytes(1024), P, 0,
                             (double *)nullptr));
        c->launches++;
    }
    else
        CUDA_TRY(c, launch_k(c, sep_solve_kernel<CNT>, dim3(c->members), dim3(CNT), sep_smem_bytes(CNT), P, 0,
                             (double *)nullptr));
    CUDA_TRY(c, launch_k(c, cl_stage_kernel<S2, FIN, BATHY, CL_MODE_FINISH>, grid, dim3(CNT), sm, P, B));
    c->launches += 3;
    if (FIN && c->filter_sigma > 0.0) {
        CUDA_TRY(c, launch_k(c, filter_fix_kernel, dim3((4 * c->spG + 127) / 128, c->members), dim3(128), 0, P, B));
        c->launches++;
    }
    return HSGN_OK;
}

template <bool S2, bool FIN>
hsgn_status launch_spike_b(hsgn_ctx *c, const Params &P, const Bufs &B)
{
    return c->bathy ? launch_spike<S2, FIN, true>(c, P, B) : launch_spike<S2, FIN, false>(c, P, B);
}

// Small ensembles (at most two waves of stage CTAs: launch-latency bound, e.g.
// cfg1, cfg2) run the step's first stage as stage_kernel<..., FDT>, which
// computes the step's dt itself (Params::fuse_dt): no dt_commit_kernel between
// the steps of a sequence, only after its last step (the commit of that step
// and the next dt).  cfg2: 15.5 -> 14.0 us per step.  Large ensembles keep the
// separate commit kernel (the fused first stage measured 4 % slower on cfg3).
bool fused_dt(const hsgn_ctx *c)
{
    static int wave = 0;
    if (!wave) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        wave = HSGN_MINB * std::max(sms, 1);
    }
    return c->scheme == 0 && !c->slab && c->tab.stages == 2 && c->picard == 0 && !c->wb &&
           !use_cluster(c) && !use_spike(c) && (long long)c->tiles * c->members <= 2LL * wave;
}

// kernels enqueued per step (graph launch accounting)
int launches_per_step(const hsgn_ctx *c)
{
    if (c->scheme != 0) return c->x_stages + 1;
    if (fused_dt(c)) return c->tab.stages;      // + one dt_commit per sequence
    if (use_spike(c)) {
        const int fix = c->filter_sigma > 0.0 ? 1 : 0;
        return (c->spG > 1024 ? 4 : 3) * c->tab.stages + fix + 1;
    }
    return c->tab.stages + 1;
}

template <bool BATHY>
void multi_attrs()
{
    cudaFuncSetAttribute(cl_multi_kernel<BATHY>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cl_multi_kernel<BATHY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(BATHY ? CSMEM_BYTES_B : CSMEM_BYTES));
}

template <bool S2, bool FIN, bool BATHY>
void cl_attrs()
{
    cudaFuncSetAttribute(cl_stage_kernel<S2, FIN, BATHY>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int sm = int(BATHY ? CSMEM_BYTES_B : CSMEM_BYTES);
    cudaFuncSetAttribute(cl_stage_kernel<S2, FIN, BATHY>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(cl_stage_kernel<S2, FIN, BATHY, CL_MODE_TIPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(cl_stage_kernel<S2, FIN, BATHY, CL_MODE_FINISH>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}

hsgn_status launch_dtc(hsgn_ctx *c, long long k, int commit_prev, int compute_dt)
{
    const Params P = make_params(c, k);
    CUDA_TRY(c, launch_k(c, dt_commit_kernel, dim3((c->members + 127) / 128), dim3(128), 0, P, commit_prev,
                           compute_dt));
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return HSGN_OK;
}

// Enqueue step k reading buf[cur], writing buf[cur ^ 1]: the stages, then the
// commit of step k and the dt of step k+1.  ev (optional, 3 events) brackets
// the stage kernels; dt_copy (optional, device) receives the dt step k used.
// first / last: position in a sequence of steps enqueued back to back -- with
// fused_dt the first stage of a non-first step commits the previous one, and
// only the last step ends with dt_commit_kernel.
hsgn_status enqueue_step(hsgn_ctx *c, int cur, long long k, cudaEvent_t *ev = nullptr,
                         double *dt_copy = nullptr, bool first = true, bool last = true)
{
    Params P = make_params(c, k);
    const bool fused = fused_dt(c);
    if (fused) {
        P.fuse_dt = 1;
        P.commit_prev = first ? 0 : 1;
    }
    Bufs B{};
    for (int f = 0; f < 4; f++) {
        B.Un[f] = c->buf[cur][f];
        B.U1[f] = c->buf[2][f];
    }
    hsgn_status st;
    if (ev) CUDA_TRY(c, rec_ev(c, ev[0]));
    if (c->scheme == 2) {
        dim3 grid(c->stiles, c->members);
        if (c->x_stages == 1) {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            if (c->bathy) sgn_kernel<false, true, true><<<grid, SNT, SSMEM_BYTES_B, c->stream>>>(P, B);
            else sgn_kernel<false, true><<<grid, SNT, SSMEM_BYTES, c->stream>>>(P, B);
            c->launches++;
            CUDA_TRY(c, cudaGetLastError());
            if (ev) CUDA_TRY(c, rec_ev(c, ev[1]));
        } else {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[2][f];
            if (c->bathy) sgn_kernel<false, false, true><<<grid, SNT, SSMEM_BYTES_B, c->stream>>>(P, B);
            else sgn_kernel<false, false><<<grid, SNT, SSMEM_BYTES, c->stream>>>(P, B);
            c->launches++;
            CUDA_TRY(c, cudaGetLastError());
            if (ev) CUDA_TRY(c, rec_ev(c, ev[1]));
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            if (c->bathy) sgn_kernel<true, true, true><<<grid, SNT, SSMEM_BYTES_B, c->stream>>>(P, B);
            else sgn_kernel<true, true><<<grid, SNT, SSMEM_BYTES, c->stream>>>(P, B);
            c->launches++;
            CUDA_TRY(c, cudaGetLastError());
        }
        if (ev) CUDA_TRY(c, rec_ev(c, ev[2]));
    } else if (c->scheme == 1) {
        dim3 grid(c->xtiles, c->members);
        const bool filt = c->filter_sigma > 0.0;
        if (c->x_stages == 1) {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            if (filt) explicit_kernel<false, true, true><<<grid, XNT, XSMEM_BYTES, c->stream>>>(P, B);
            else explicit_kernel<false, true, false><<<grid, XNT, XSMEM_BYTES_NF, c->stream>>>(P, B);
            c->launches++;
            CUDA_TRY(c, cudaGetLastError());
            if (ev) CUDA_TRY(c, rec_ev(c, ev[1]));
        } else {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[2][f];
            explicit_kernel<false, false, false><<<grid, XNT, XSMEM_BYTES_NF, c->stream>>>(P, B);
            c->launches++;
            CUDA_TRY(c, cudaGetLastError());
            if (ev) CUDA_TRY(c, rec_ev(c, ev[1]));
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            if (filt) explicit_kernel<true, true, true><<<grid, XNT, XSMEM_BYTES, c->stream>>>(P, B);
            else explicit_kernel<true, true, false><<<grid, XNT, XSMEM_BYTES_NF, c->stream>>>(P, B);
            c->launches++;
            CUDA_TRY(c, cudaGetLastError());
        }
        if (ev) CUDA_TRY(c, rec_ev(c, ev[2]));
    } else if (use_cluster(c)) {
        if (c->tab.stages == 1) {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            st = launch_cl_b<false, true>(c, P, B);
            if (st != HSGN_OK) return st;
            if (ev) {
                CUDA_TRY(c, rec_ev(c, ev[1]));
                CUDA_TRY(c, rec_ev(c, ev[2]));
            }
        } else {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[2][f];
            st = launch_cl_b<false, false>(c, P, B);
            if (st != HSGN_OK) return st;
            if (ev) CUDA_TRY(c, rec_ev(c, ev[1]));
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            st = launch_cl_b<true, true>(c, P, B);
            if (st != HSGN_OK) return st;
            if (ev) CUDA_TRY(c, rec_ev(c, ev[2]));
        }
    } else if (use_spike(c)) {
        if (c->tab.stages == 1) {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            st = launch_spike_b<false, true>(c, P, B);
            if (st != HSGN_OK) return st;
            if (ev) {
                CUDA_TRY(c, rec_ev(c, ev[1]));
                CUDA_TRY(c, rec_ev(c, ev[2]));
            }
        } else {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[2][f];
            st = launch_spike_b<false, false>(c, P, B);
            if (st != HSGN_OK) return st;
            if (ev) CUDA_TRY(c, rec_ev(c, ev[1]));
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
            st = launch_spike_b<true, true>(c, P, B);
            if (st != HSGN_OK) return st;
            if (ev) CUDA_TRY(c, rec_ev(c, ev[2]));
        }
    } else if (c->tab.stages == 1) {
        for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
        st = launch_stage_b<false, true>(c, P, B);
        if (st != HSGN_OK) return st;
        if (ev) {
            CUDA_TRY(c, rec_ev(c, ev[1]));
            CUDA_TRY(c, rec_ev(c, ev[2]));
        }
    } else {
        for (int f = 0; f < 4; f++) B.out[f] = c->buf[2][f];
        st = launch_stage_b<false, false>(c, P, B);
        if (st != HSGN_OK) return st;
        if (ev) CUDA_TRY(c, rec_ev(c, ev[1]));
        for (int f = 0; f < 4; f++) B.out[f] = c->buf[cur ^ 1][f];
        st = launch_stage_b<true, true>(c, P, B);
        if (st != HSGN_OK) return st;
        if (ev) CUDA_TRY(c, rec_ev(c, ev[2]));
    }
    if (dt_copy)
        CUDA_TRY(c, cudaMemcpyAsync(dt_copy, c->dt, c->members * sizeof(double),
                                    cudaMemcpyDeviceToDevice, c->stream));
    if (fused && !last) return HSGN_OK;
    return launch_dtc(c, k + 1, 1, 1);
}

void drop_graphs(hsgn_ctx *c)
{
    for (auto &gx : c->graph)
        if (gx) { cudaGraphExecDestroy(gx); gx = nullptr; }
    c->gen++;                     // every setter passes here: member-chunk views are stale
}

hsgn_status set_ctrl(hsgn_ctx *c, double t_end, double dt_fixed)
{
    if (c->ctrl_host.t_end == t_end && c->ctrl_host.dt_fixed == dt_fixed) return HSGN_OK;
    c->ctrl_host.t_end = t_end;
    c->ctrl_host.dt_fixed = dt_fixed;
    // ctrl_host is read by the copy after this call returns only if the
    // stream is idle; copy from a stable per-context staging location
    CUDA_TRY(c, cudaMemcpyAsync(c->ctrl, &c->ctrl_host, sizeof(Ctrl), cudaMemcpyHostToDevice,
                                c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

// Tile geometry: overlap w from the CFL-implied bound on
// rho = (tau/dx)^2 beta <= 3 (a_ii CFL)^2 (beta <= ~2 nu^2 at rest, margin 1.5),
// r = 2 rho / (1 + 2 rho + sqrt(1 + 4 rho)), w >= 60 ln2 / -ln r.  Every CTA
// re-checks r^w <= 2^-60 with its actual rho_max.
void choose_geometry(hsgn_ctx *c)
{
    int w;
    if (c->desc.overlap > 0) {
        w = c->desc.overlap;
    } else if (c->cfl > 0.0) {
        const double a = std::max(c->aI1, c->aI2);
        const double rho = 3.0 * (a * c->cfl) * (a * c->cfl);
        const double r = 2.0 * rho / (1.0 + 2.0 * rho + std::sqrt(1.0 + 4.0 * rho));
        w = int(std::ceil(41.588830833596716 / -std::log(r))) + 4;
        w = ((w + 7) / 8) * 8;
    } else {
        w = 256;   // material-CFL-only stepping: rho is not bounded a priori
    }
    w = std::max(3, std::min(w, (LCAP - 2 - T_MIN) / 2));
    const int maxT = LCAP - 2 - 2 * w;
    int T;
    if (c->desc.tile_cells > 0) T = std::max(std::min<int>(c->desc.tile_cells, maxT), T_MIN);
    else {
        const int ntiles = (c->n + maxT - 1) / maxT;
        T = (c->n + ntiles - 1) / ntiles;
        if (ntiles > 1) T = ((T + 31) / 32) * 32;
        if (T > maxT) T = (T + 1) & ~1;                 // even: aligned bulk stores
        T = std::max(std::min(T, maxT), std::min(T_MIN, c->n));
    }
    c->T = T;
    c->w = w;
    c->tiles = (c->n + T - 1) / T;
    c->xT = std::min(c->n, XT);
    c->xtiles = (c->n + c->xT - 1) / c->xT;
}

hsgn_status ready(hsgn_ctx *c)
{
    if (!c) return HSGN_E_INVALID;
    if (!c->ws) return fail(c, HSGN_E_NOWORKSPACE, "workspace not set");
    if (!c->have_params) return fail(c, HSGN_E_INVALID, "hsgn_set_params not called");
    if (!c->have_state) return fail(c, HSGN_E_INVALID, "hsgn_set_state not called");
    if (c->scheme != 0 && ((c->bathy && c->scheme == 1) || c->slab || c->relax.gen_rate > 0.0 ||
                           c->relax.sp_rate > 0.0))
        return fail(c, HSGN_E_INVALID, "explicit scheme: flat bottom; explicit / SGN: no relaxation zones, no slabs");
    if (c->picard > 0 && (c->scheme != 0 || c->relax.gen_rate > 0.0 || c->relax.sp_rate > 0.0))
        return fail(c, HSGN_E_INVALID, "Picard passes: SI scheme without relaxation zones");
    if (c->wb && (c->scheme != 0 || c->picard > 0))
        return fail(c, HSGN_E_INVALID, "well-balanced form: SI scheme without Picard passes");
    if (c->scheme == 2 && c->filter_sigma > 0.0)
        return fail(c, HSGN_E_INVALID, "SGN scheme: no A19 filter (its Rusanov speed includes sqrt(g h))");
    if (c->scheme == 2 && c->sT <= 0) return fail(c, HSGN_E_INVALID, "SGN geometry not set");
    return HSGN_OK;
}

hsgn_status slab_step(std::vector<hsgn_ctx *> &g, long long k, bool nccl);

hsgn_status run_steps_impl(hsgn_ctx *c, long long n_steps)
{
    if (n_steps <= 0) return HSGN_OK;
    if (c->slab) {
        if (!c->nccl)
            return fail(c, HSGN_E_INVALID, "BC_HALO sides need hsgn_group_run_steps or hsgn_attach_nccl");
        if (c->n < slab_H(c)) return fail(c, HSGN_E_INVALID, "slab shorter than its halo (n < overlap + 3)");
        if (c->w != c->nccl_w)     // the neighbours' send/recv sizes would no longer match
            return fail(c, HSGN_E_INVALID, "overlap changed since hsgn_attach_nccl (set it with the "
                                           "descriptor's overlap, or re-attach on every rank)");
        std::vector<hsgn_ctx *> g{c};
        for (long long i = 0; i < n_steps; i++) {
            hsgn_status st = slab_step(g, c->host_steps, true);
            if (st != HSGN_OK) return st;
        }
        return HSGN_OK;
    }
    hsgn_status st = HSGN_OK;
    if (!fused_dt(c)) st = launch_dtc(c, c->host_steps, 0, 1);   // dt of the first step
    if (st != HSGN_OK) return st;
    long long done = 0;
    bool seq_first = true;
    while (done < n_steps) {
        if (n_steps - done >= GRAPH_STEPS && c->stream != nullptr && c->host_steps % 6 == 0) {
            cudaGraphExec_t &gx = c->graph[c->cur];
            if (!gx) {
                cudaGraph_t gr;
                CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
                const long long l0 = c->launches;
                int cc = c->cur;
                for (int k = 0; k < GRAPH_STEPS && st == HSGN_OK; k++) {
                    st = enqueue_step(c, cc, c->host_steps + k, nullptr, nullptr, k == 0, k == GRAPH_STEPS - 1);
                    cc ^= 1;
                }
                cudaError_t ce = cudaStreamEndCapture(c->stream, &gr);
                if (st != HSGN_OK) return st;
                if (ce != cudaSuccess) return fail(c, HSGN_E_CUDA, cudaGetErrorString(ce));
                c->launches = l0;   // counted at replay
                CUDA_TRY(c, cudaGraphInstantiate(&gx, gr, 0));
                cudaGraphDestroy(gr);
            }
            CUDA_TRY(c, cudaGraphLaunch(gx, c->stream));
            c->launches += GRAPH_STEPS * launches_per_step(c) + (fused_dt(c) ? 1 : 0);
            done += GRAPH_STEPS;          // even: cur unchanged
            c->host_steps += GRAPH_STEPS;
        } else {
            // eager steps back to back share one closing dt_commit (fused dt):
            // the sequence ends before the last step and before a graph
            const long long left = n_steps - done - 1;
            const bool last = left == 0 || (left >= GRAPH_STEPS && c->stream != nullptr &&
                                            (c->host_steps + 1) % 6 == 0);
            st = enqueue_step(c, c->cur, c->host_steps, nullptr, nullptr, seq_first, last);
            if (st != HSGN_OK) return st;
            seq_first = last;
            c->cur ^= 1;
            c->host_steps++;
            done++;
        }
    }
    return HSGN_OK;
}

// ---------------------------------------------------------------------------
// Slab decomposition: one domain split into
// contiguous slabs whose BC_HALO sides take H = w + 3 ghost cells from the
// neighbour, exchanged before each stage (U^n before stage 1, U1 before stage
// 2); the dt maxima are max-reduced across slabs before each step's dt.
// Transports: in-process loopback group (all slabs on one device and one
// stream, D2D copies) and NCCL (one slab per process / GPU).
// ---------------------------------------------------------------------------
constexpr int GROUP_MAX = 64;
struct MaxPtrs { unsigned long long *p[GROUP_MAX]; };

__global__ void group_max_kernel(MaxPtrs ptrs, int P, int count)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    unsigned long long mx = 0ull;
    for (int k = 0; k < P; k++) mx = max(mx, ptrs.p[k][i]);
    for (int k = 0; k < P; k++) ptrs.p[k][i] = mx;
}

// halo array index: which = 0 (U^n), 1 (U1), 2 (b)
double *halo_dst(hsgn_ctx *c, bool left, int which, int f)
{
    return (left ? c->halo_l : c->halo_r) + (which == 2 ? 8 : which * 4 + f) * H_MAX;
}

const double *bnd_src(hsgn_ctx *c, bool right_end, int which, int f, int H)
{
    const double *base = which == 2 ? c->b : (which == 0 ? c->buf[c->cur][f] : c->buf[2][f]);
    return right_end ? base + (c->n - H) : base;
}

hsgn_status loopback_exchange(std::vector<hsgn_ctx *> &g, int which)
{
    const int P = int(g.size());
    const int nf = which == 2 ? 1 : 4;
    for (int i = 0; i < P; i++) {
        hsgn_ctx *c = g[i];
        const int H = slab_H(c);                      // (equal over the group: checked per run)
        hsgn_ctx *L = g[(i - 1 + P) % P], *R = g[(i + 1) % P];
        for (int f = 0; f < nf; f++) {
            if (c->desc.bc_left == HSGN_BC_HALO)
                CUDA_TRY(c, cudaMemcpyAsync(halo_dst(c, true, which, f), bnd_src(L, true, which, f, H),
                                            H * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
            if (c->desc.bc_right == HSGN_BC_HALO)
                CUDA_TRY(c, cudaMemcpyAsync(halo_dst(c, false, which, f), bnd_src(R, false, which, f, H),
                                            H * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        }
    }
    return HSGN_OK;
}

#define NCCL_TRY(c, expr)                                                             \
    do {                                                                              \
        ncclResult_t r_ = (expr);                                                     \
        if (r_ != ncclSuccess)                                                        \
            return fail((c), HSGN_E_COMM, std::string(#expr ": ") + ncclGetErrorString(r_)); \
    } while (0)

hsgn_status nccl_exchange(hsgn_ctx *c, int which)
{
    const int H = slab_H(c);
    const int left = (c->nrank - 1 + c->nworld) % c->nworld, right = (c->nrank + 1) % c->nworld;
    const int nf = which == 2 ? 1 : 4;
    NCCL_TRY(c, ncclGroupStart());
    for (int f = 0; f < nf; f++) {
        // per peer the order is: my right boundary -> right's left halo, then my
        // left boundary -> left's right halo (matches for a ring of 2 as well)
        if (c->desc.bc_right == HSGN_BC_HALO)
            NCCL_TRY(c, ncclSend(bnd_src(c, true, which, f, H), H, ncclDouble, right, c->nccl, c->stream));
        if (c->desc.bc_left == HSGN_BC_HALO)
            NCCL_TRY(c, ncclRecv(halo_dst(c, true, which, f), H, ncclDouble, left, c->nccl, c->stream));
        if (c->desc.bc_left == HSGN_BC_HALO)
            NCCL_TRY(c, ncclSend(bnd_src(c, false, which, f, H), H, ncclDouble, left, c->nccl, c->stream));
        if (c->desc.bc_right == HSGN_BC_HALO)
            NCCL_TRY(c, ncclRecv(halo_dst(c, false, which, f), H, ncclDouble, right, c->nccl, c->stream));
    }
    NCCL_TRY(c, ncclGroupEnd());
    return HSGN_OK;
}

// Slab step phases (shared by the group, NCCL and host-staged transports).
// b. dt of step k (after the maxima were max-reduced over the slabs)
hsgn_status slab_phase_dt(std::vector<hsgn_ctx *> &g, long long k)
{
    hsgn_status st;
    for (auto *c : g) if ((st = launch_dtc(c, k, 0, 1)) != HSGN_OK) return st;
    return HSGN_OK;
}

hsgn_status slab_spike_stage(std::vector<hsgn_ctx *> &g, long long k, bool s2, bool nccl);

// c/d. stage 1 (s2 = false) or stage 2 (s2 = true) of step k, halos in place
hsgn_status slab_phase_stage(std::vector<hsgn_ctx *> &g, long long k, bool s2, bool nccl = false)
{
    hsgn_status st;
    if (use_spike(g[0])) return slab_spike_stage(g, k, s2, nccl);
    for (auto *c : g) {
        const Params Pm = make_params(c, k);
        Bufs B{};
        for (int f = 0; f < 4; f++) { B.Un[f] = c->buf[c->cur][f]; B.U1[f] = c->buf[2][f]; }
        if (s2) {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[c->cur ^ 1][f];
            if ((st = launch_stage_b<true, true>(c, Pm, B)) != HSGN_OK) return st;
        } else if (c->tab.stages == 1) {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[c->cur ^ 1][f];
            if ((st = launch_stage_b<false, true>(c, Pm, B)) != HSGN_OK) return st;
        } else {
            for (int f = 0; f < 4; f++) B.out[f] = c->buf[2][f];
            if ((st = launch_stage_b<false, false>(c, Pm, B)) != HSGN_OK) return st;
        }
    }
    return HSGN_OK;
}

// e. commit step k
hsgn_status slab_phase_commit(std::vector<hsgn_ctx *> &g, long long k)
{
    hsgn_status st;
    for (auto *c : g) {
        if ((st = launch_dtc(c, k + 1, 1, 0)) != HSGN_OK) return st;
        c->cur ^= 1;
        c->host_steps++;
    }
    return HSGN_OK;
}

// one slab step k for every context of g (lockstep, one shared stream) or for
// the single NCCL-attached context g[0]
hsgn_status slab_step(std::vector<hsgn_ctx *> &g, long long k, bool nccl)
{
    hsgn_status st;
    const int P = int(g.size());
    const int slot = int(k % 3);
    hsgn_ctx *c0 = g[0];
    const int count = 2 * c0->members;
    // a. global max of the dt maxima of U^k
    if (nccl) {
        unsigned long long *mx = c0->maxes + size_t(slot) * 2 * c0->members;
        NCCL_TRY(c0, ncclAllReduce(mx, mx, count, ncclUint64, ncclMax, c0->nccl, c0->stream));
    } else if (P > 1) {
        MaxPtrs mp{};
        for (int i = 0; i < P; i++) mp.p[i] = g[i]->maxes + size_t(slot) * 2 * c0->members;
        group_max_kernel<<<(count + 127) / 128, 128, 0, c0->stream>>>(mp, P, count);
        c0->launches++;
        CUDA_TRY(c0, cudaGetLastError());
    }
    if ((st = slab_phase_dt(g, k)) != HSGN_OK) return st;
    // static b halos (again every step: cheap, and the halo width follows the solve mode)
    if (c0->bathy && (st = nccl ? nccl_exchange(c0, 2) : loopback_exchange(g, 2)) != HSGN_OK) return st;
    // c. U^n halos, stage 1
    if ((st = nccl ? nccl_exchange(c0, 0) : loopback_exchange(g, 0)) != HSGN_OK) return st;
    if ((st = slab_phase_stage(g, k, false, nccl)) != HSGN_OK) return st;
    if (c0->tab.stages == 2) {
        // d. U1 halos, stage 2
        if ((st = nccl ? nccl_exchange(c0, 1) : loopback_exchange(g, 1)) != HSGN_OK) return st;
        if ((st = slab_phase_stage(g, k, true, nccl)) != HSGN_OK) return st;
    }
    return slab_phase_commit(g, k);
}

// One stage of step k with the depth system solved exactly across all slabs
// (tile-level SPIKE per slab + the slab interface system, section 8):
//   TIPS -> [right slab's tile-0 relation] -> sep solves Y, V, W -> [all-gather
//   of the end values] -> interface solve, L -> FINISH -> (final stage with the
//   filter) [neighbouring slabs' unfiltered end rows] -> filter_fix.
// Transports: loopback group (D2D copies on the shared stream) or NCCL.
// HSGN_DEBUG_SYNC=1: synchronise and report after every phase (development aid)
bool dbg_sync(hsgn_ctx *c, const char *what, int k)
{
    static const bool on = std::getenv("HSGN_DEBUG_SYNC") != nullptr;
    if (!on) return false;
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) return false;
    fprintf(stderr, "hsgn: %s %d: %s\n", what, k, cudaGetErrorString(e));
    c->last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return true;
}

template <bool S2, bool FIN, bool BATHY>
hsgn_status slab_spike_kernels(hsgn_ctx *c, Params P, const Bufs &B, int phase)
{
    P.T = c->spT;
    P.tiles = c->spG;
    const dim3 grid(c->spG, c->members);
    const size_t sm = BATHY ? CSMEM_BYTES_B : CSMEM_BYTES;
    const int mb = (c->members + 127) / 128;
    if (phase == 0) {                 // tips, tile-0 relation packed for the left slab
        CUDA_TRY(c, launch_k(c, cl_stage_kernel<S2, FIN, BATHY, CL_MODE_TIPS>, grid, dim3(CNT), sm, P, B));
        CUDA_TRY(c, launch_k(c, slab_pack_kernel, dim3(mb), dim3(128), 0, P, 0));
        c->launches += 2;
    } else if (phase == 1) {          // Y, V, W of the slab's separator system; end values packed
        for (int mode = 0; mode < 3; mode++) {
            double *out = c->sx_yvw + size_t(mode) * c->members * c->spG;
            if (c->spG > 1024) {
                CUDA_TRY(c, launch_k(c, sep_coef_kernel, dim3((c->spG + 255) / 256, c->members), dim3(256), 0, P, mode));
                CUDA_TRY(c, launch_k(c, sep_solve_kernel<1024>, dim3(c->members), dim3(1024), sep_smem_bytes(1024),
                                     P, mode, out));
                c->launches += 2;
            } else {
                CUDA_TRY(c, launch_k(c, sep_solve_kernel<CNT>, dim3(c->members), dim3(CNT), sep_smem_bytes(CNT),
                                     P, mode, out));
                c->launches++;
            }
        }
        CUDA_TRY(c, launch_k(c, slab_pack_kernel, dim3(mb), dim3(128), 0, P, 1));
        c->launches++;
    } else if (phase == 2) {          // interface solve, separators, finish; filter rows packed
        const size_t ism = size_t(2 * P.sx_P) * (2 * P.sx_P + 1) * sizeof(double);
        CUDA_TRY(c, launch_k(c, slab_iface_kernel, dim3(c->members), dim3(128), ism, P));
        CUDA_TRY(c, launch_k(c, cl_stage_kernel<S2, FIN, BATHY, CL_MODE_FINISH>, grid, dim3(CNT), sm, P, B));
        c->launches += 2;
        if (FIN && c->filter_sigma > 0.0) {
            CUDA_TRY(c, launch_k(c, slab_pack_kernel, dim3(mb), dim3(128), 0, P, 2));
            c->launches++;
        }
    } else if (FIN && c->filter_sigma > 0.0) {   // phase 3: filter rows at tile and slab ends
        CUDA_TRY(c, launch_k(c, filter_fix_kernel, dim3((4 * (c->spG + 1) + 127) / 128, c->members), dim3(128), 0, P, B));
        c->launches++;
    }
    return HSGN_OK;
}

template <bool S2, bool FIN>
hsgn_status slab_spike_kernels_b(hsgn_ctx *c, const Params &P, const Bufs &B, int phase)
{
    return c->bathy ? slab_spike_kernels<S2, FIN, true>(c, P, B, phase)
                    : slab_spike_kernels<S2, FIN, false>(c, P, B, phase);
}

// exchange x of the slab SPIKE stage: 0 tile-0 relation (right -> left), 1 end
// values (all-gather), 2 unfiltered end rows (both ways)
hsgn_status slab_spike_xfer(std::vector<hsgn_ctx *> &g, int x, bool nccl)
{
    const int P = int(g.size());
    hsgn_ctx *c0 = g[0];
    const size_t M = c0->members;
    if (nccl) {
        hsgn_ctx *c = c0;
        const int left = (c->nrank - 1 + c->nworld) % c->nworld, right = (c->nrank + 1) % c->nworld;
        const bool hl = c->desc.bc_left == HSGN_BC_HALO, hr = c->desc.bc_right == HSGN_BC_HALO;
        if (x == 1) {
            NCCL_TRY(c, ncclAllGather(c->sx_send, c->sx_all, 6 * M, ncclDouble, c->nccl, c->stream));
            return HSGN_OK;
        }
        NCCL_TRY(c, ncclGroupStart());
        if (x == 0) {
            if (hl) NCCL_TRY(c, ncclSend(c->sx_send, 6 * M, ncclDouble, left, c->nccl, c->stream));
            if (hr) NCCL_TRY(c, ncclRecv(c->sx_nx, 6 * M, ncclDouble, right, c->nccl, c->stream));
        } else {
            if (hl) NCCL_TRY(c, ncclSend(c->sx_send, 8 * M, ncclDouble, left, c->nccl, c->stream));
            if (hr) NCCL_TRY(c, ncclRecv(c->sx_fbr, 8 * M, ncclDouble, right, c->nccl, c->stream));
            if (hr) NCCL_TRY(c, ncclSend(c->sx_send + 8 * M, 8 * M, ncclDouble, right, c->nccl, c->stream));
            if (hl) NCCL_TRY(c, ncclRecv(c->sx_fbl, 8 * M, ncclDouble, left, c->nccl, c->stream));
        }
        NCCL_TRY(c, ncclGroupEnd());
        return HSGN_OK;
    }
    for (int i = 0; i < P; i++) {
        hsgn_ctx *c = g[i], *L = g[(i - 1 + P) % P], *R = g[(i + 1) % P];
        const bool hl = c->desc.bc_left == HSGN_BC_HALO, hr = c->desc.bc_right == HSGN_BC_HALO;
        auto cp = [&](double *dst, const double *src, size_t nd) {
            return cudaMemcpyAsync(dst, src, nd * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
        };
        if (x == 0) {
            if (hr) CUDA_TRY(c, cp(c->sx_nx, R->sx_send, 6 * M));
        } else if (x == 1) {
            for (int q = 0; q < P; q++) CUDA_TRY(c, cp(c->sx_all + size_t(q) * 6 * M, g[q]->sx_send, 6 * M));
        } else {
            if (hr) CUDA_TRY(c, cp(c->sx_fbr, R->sx_send, 8 * M));
            if (hl) CUDA_TRY(c, cp(c->sx_fbl, L->sx_send + 8 * M, 8 * M));
        }
    }
    return HSGN_OK;
}

hsgn_status slab_spike_stage(std::vector<hsgn_ctx *> &g, long long k, bool s2, bool nccl)
{
    const int Pn = int(g.size());
    if (!nccl && Pn > GROUP_MAX_SX) return fail(g[0], HSGN_E_INVALID, "slab SPIKE: too many slabs");
    if (nccl && g[0]->nworld > GROUP_MAX_SX) return fail(g[0], HSGN_E_INVALID, "slab SPIKE: too many ranks");
    const bool fin = s2 || g[0]->tab.stages == 1;
    hsgn_status st;
    for (int phase = 0; phase < 4; phase++) {
        for (int i = 0; i < Pn; i++) {
            hsgn_ctx *c = g[i];
            Params Pm = make_params(c, k);
            if (!nccl) { Pm.sx_rank = i; Pm.sx_P = Pn; }
            Bufs B{};
            for (int f = 0; f < 4; f++) { B.Un[f] = c->buf[c->cur][f]; B.U1[f] = c->buf[2][f]; }
            for (int f = 0; f < 4; f++) B.out[f] = fin ? c->buf[c->cur ^ 1][f] : c->buf[2][f];
            if (s2) st = slab_spike_kernels_b<true, true>(c, Pm, B, phase);
            else if (fin) st = slab_spike_kernels_b<false, true>(c, Pm, B, phase);
            else st = slab_spike_kernels_b<false, false>(c, Pm, B, phase);
            if (st != HSGN_OK) return st;
            if (dbg_sync(c, "slab spike phase", phase)) return HSGN_E_CUDA;
        }
        if (phase < 2 || (phase == 2 && fin && g[0]->filter_sigma > 0.0))
            if ((st = slab_spike_xfer(g, phase, nccl)) != HSGN_OK) return st;
        if (dbg_sync(g[0], "slab spike xfer", phase)) return HSGN_E_CUDA;
    }
    return HSGN_OK;
}

// After a sync: reconcile host buffer parity with the device's committed steps.
hsgn_status reconcile(hsgn_ctx *c, unsigned int *bits_out = nullptr)
{
    unsigned int bits = 0;
    long long dsteps = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&bits, c->err, sizeof(bits), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&dsteps, c->steps, sizeof(dsteps), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (bits_out) *bits_out = bits;
    c->dev_steps = dsteps;
    if (dsteps != c->host_steps) {
        // steps after the failing one did nothing: the committed state is in
        // the buffer reached after dsteps ping-pongs
        const long long extra = c->host_steps - dsteps;
        if (extra & 1) c->cur ^= 1;
        c->host_steps = dsteps;
    }
    hsgn_status st = status_from_bits(bits);
    if (st != HSGN_OK) {
        char msg[160];
        snprintf(msg, sizeof msg, "device error bits 0x%x after %lld committed steps", bits, dsteps);
        c->last_error = msg;
    }
    return st;
}

void free_kids(hsgn_ctx *c)
{
    for (hsgn_ctx *k : c->kids) { drop_graphs(k); delete k; }
    c->kids.clear();
    c->kids_gen = -1;
}

__global__ void fill_kernel(double *p, int count, double v)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}

// Member-chunk views for hsgn_run_host: chunk k = members [m0, m1) with the
// same settings and geometry as c, state buffers = slices of c's, own small
// arrays in the workspace tail, c's stream.  Rebuilt when a setter ran.
hsgn_status make_kids(hsgn_ctx *c, int chunks)
{
    if (int(c->kids.size()) == chunks && c->kids_gen == c->gen) return HSGN_OK;
    free_kids(c);
    char *q = c->kid_ws;
    for (int k = 0; k < chunks; k++) {
        const int m0 = int((long long)c->members * k / chunks), m1 = int((long long)c->members * (k + 1) / chunks);
        const int cnt = m1 - m0;
        hsgn_ctx *kc = new hsgn_ctx();
        kc->desc = c->desc;
        kc->desc.n_members = cnt;
        kc->stream = (c->cs2 && (k & 1)) ? c->cs2 : c->stream;   // chunks alternate compute streams
        kc->device = c->device;
        kc->n = c->n; kc->members = cnt; kc->dx = c->dx;
        kc->g = c->g; kc->cfl = c->cfl; kc->mcfl = c->mcfl; kc->h_min = c->h_min;
        kc->lam.assign(c->lam.begin() + m0, c->lam.begin() + m1);
        kc->have_params = true;
        kc->bathy = c->bathy;
        kc->tab = c->tab; kc->aI1 = c->aI1; kc->aI2 = c->aI2; kc->wE = c->wE; kc->wR = c->wR;
        kc->filter_sigma = c->filter_sigma;
        kc->relax = c->relax;
        kc->scheme = c->scheme; kc->x_stages = c->x_stages;
        kc->picard = c->picard; kc->wb = c->wb;
        kc->cl_mode = c->cl_mode; kc->clC = c->clC; kc->clT = c->clT;
        kc->spG = c->spG; kc->spT = c->spT;
        if (c->sp_tips) {
            const size_t o = size_t(m0) * c->spG;
            kc->sp_tips = c->sp_tips + o * XPUB; kc->sp_L = c->sp_L + o;
            kc->sp_fb = c->sp_fb + o * 16; kc->sp_S = c->sp_S + size_t(m0) * sep_scratch(c->spG);
        }
        kc->ws = c->ws;
        for (int bi = 0; bi < 3; bi++)
            for (int f = 0; f < 4; f++) kc->buf[bi][f] = c->buf[bi][f] + size_t(m0) * c->n;
        kc->b = c->b;
        kc->lamd = c->lamd + m0;
        kc->t = (double *)q; q += align256(2 * size_t(cnt) * 8);
        kc->dt = (double *)q; q += align256(size_t(cnt) * 8);
        kc->dt_used = (double *)q; q += align256(size_t(cnt) * 8);
        kc->maxes = (unsigned long long *)q; q += align256(6 * size_t(cnt) * 8);
        kc->partials = (double *)q; q += align256(size_t(cnt) * ((c->n + T_MIN - 1) / T_MIN + 1) * 4 * 8);
        kc->err = (unsigned int *)q;
        kc->done = (unsigned int *)(q + 4);
        kc->steps = (long long *)(q + 8);
        kc->rho_obs = (unsigned long long *)(q + 16);
        kc->kmin = (unsigned int *)(q + 64);
        q += 256;
        kc->ctrl = (Ctrl *)q;
        q += 256;
        choose_geometry(kc);
        c->kids.push_back(kc);
    }
    c->kids_gen = c->gen;
    return HSGN_OK;
}

// hsgn_set_state's device part for a member-chunk view whose U^n slice was
// copied in on another stream: t = t0, dt/maxima/error words cleared, dt
// maxima of the initial state (no host synchronisation).
hsgn_status kid_state_init(hsgn_ctx *kc, double t0)
{
    fill_kernel<<<(kc->members + 255) / 256, 256, 0, kc->stream>>>(kc->t, kc->members, t0);
    CUDA_TRY(kc, cudaMemsetAsync(kc->dt, 0, kc->members * sizeof(double), kc->stream));
    CUDA_TRY(kc, cudaMemsetAsync(kc->maxes, 0, 6 * size_t(kc->members) * 8, kc->stream));
    CUDA_TRY(kc, cudaMemsetAsync(kc->err, 0, 512, kc->stream));   // scalars + ctrl
    dim3 grid(kc->tiles, kc->members);
    reduce_kernel<<<grid, NT, 0, kc->stream>>>(kc->buf[0][0], kc->buf[0][1], kc->buf[0][2],
                                               kc->bathy ? kc->b : nullptr, kc->lamd, kc->n, kc->T, kc->g,
                                               kc->partials, kc->maxes, kc->members, kc->scheme == 2);
    kc->launches += 2;
    CUDA_TRY(kc, cudaGetLastError());
    kc->cur = 0;
    kc->dev_steps = 0;
    kc->host_steps = 0;
    kc->ctrl_host = Ctrl{0.0, 0.0};
    kc->have_state = true;
    return HSGN_OK;
}

}  // namespace

// Classical SGN (scheme 2): overlap of the phi system from the state.  Rows
// are normalised by h_i, so the off-diagonals are c_{i+-1/2}/h_i <= h_max^3 /
// (3 dx^2 h_min) =: rho; w from the decay bound r^w <= 2^-60 with a 1.25
// margin on rho (the kernel re-checks with its own rho), tiles of up to
// SLCAP - 2 - 2w kept cells (h_min, h_max from a reduction of the state).
hsgn_status sgn_geometry(hsgn_ctx *c)
{
    dim3 grid(c->tiles, c->members);
    reduce_kernel<<<grid, NT, 0, c->stream>>>(c->buf[c->cur][0], c->buf[c->cur][1], c->buf[c->cur][2],
                                              nullptr, c->lamd, c->n, c->T, c->g, c->partials, nullptr,
                                              c->members, 2);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    std::vector<double> part(size_t(c->members) * c->tiles * 4);
    CUDA_TRY(c, cudaMemcpyAsync(part.data(), c->partials, part.size() * sizeof(double),
                                cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    double hmin = 1e300, hmax = 0.0;
    for (size_t i = 0; i < part.size(); i += 4) {
        hmin = std::min(hmin, part[i + 1]);
        hmax = std::max(hmax, part[i + 2]);
    }
    if (!(hmin > 0.0)) return fail(c, HSGN_E_DRY, "SGN geometry: non-positive depth");
    const double rho = 1.25 * hmax * hmax * hmax / (3.0 * c->dx * c->dx * hmin);
    const double r = 2.0 * rho / (1.0 + 2.0 * rho + std::sqrt(1.0 + 4.0 * rho));
    int w = int(std::ceil(41.588830833596716 / -std::log(r))) + 4;
    w = ((w + 7) / 8) * 8;
    const int maxT = SLCAP - 2 - 2 * w;
    if (maxT < 16)
        return fail(c, HSGN_E_INVALID, "SGN: phi decay length too long for the tile (dx too small vs h)");
    const int ntiles = (c->n + maxT - 1) / maxT;
    c->sw = w;
    c->sT = (c->n + ntiles - 1) / ntiles;
    c->stiles = (c->n + c->sT - 1) / c->sT;
    return HSGN_OK;
}

// Re-seed the dt maxima slot of the next step from the current state (after
// a scheme change: the SGN celerity differs from the hSGN one).
hsgn_status reseed_maxima(hsgn_ctx *c)
{
    const int slot = int(c->host_steps % 3);
    unsigned long long *mx = c->maxes + size_t(slot) * 2 * c->members;
    CUDA_TRY(c, cudaMemsetAsync(mx, 0, 2 * size_t(c->members) * 8, c->stream));
    dim3 grid(c->tiles, c->members);
    reduce_kernel<<<grid, NT, 0, c->stream>>>(c->buf[c->cur][0], c->buf[c->cur][1], c->buf[c->cur][2],
                                              c->bathy ? c->b : nullptr, c->lamd, c->n, c->T, c->g,
                                              c->partials, mx, c->members, c->scheme == 2);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return HSGN_OK;
}

extern "C" {

const char *hsgn_status_string(hsgn_status s)
{
    switch (s) {
    case HSGN_OK: return "ok";
    case HSGN_E_INVALID: return "invalid argument or call order";
    case HSGN_E_DRY: return "dry bed: hbar <= h_min";
    case HSGN_E_COERCIVITY: return "coercivity violated: beta (kappa) <= 0";
    case HSGN_E_SINGULAR: return "singular pivot in the depth solve";
    case HSGN_E_NONFINITE: return "non-finite value";
    case HSGN_E_CUDA: return "CUDA error";
    case HSGN_E_OVERLAP: return "tile overlap too short for the depth-solve decay";
    case HSGN_E_NOWORKSPACE: return "workspace missing or too small";
    case HSGN_E_COMM: return "NCCL communication error (slab transport)";
    }
    return "unknown status";
}

const char *hsgn_last_error(const hsgn_ctx *c) { return c ? c->last_error.c_str() : "null context"; }

hsgn_status hsgn_create(const hsgn_desc *d, void *stream, hsgn_ctx **out)
{
    if (!d || !out) return HSGN_E_INVALID;
    *out = nullptr;
    if (d->n_cells < 4 || d->n_cells > (int64_t(1) << 31) - 1 || d->n_members < 1 ||
        d->n_members > 65535 || !(d->x_max > d->x_min) || (d->order != 1 && d->order != 2))
        return HSGN_E_INVALID;
    if (d->bc_left < 0 || d->bc_left > 3 || d->bc_right < 0 || d->bc_right > 3) return HSGN_E_INVALID;
    if ((d->bc_left == HSGN_BC_PERIODIC) != (d->bc_right == HSGN_BC_PERIODIC)) return HSGN_E_INVALID;
    const bool slab = (d->bc_left == HSGN_BC_HALO || d->bc_right == HSGN_BC_HALO);
    if (slab && d->n_members != 1) return HSGN_E_INVALID;   // slabs split one domain
    hsgn_ctx *c = new hsgn_ctx();
    c->desc = *d;
    c->slab = slab;
    c->stream = (cudaStream_t)stream;
    cudaGetDevice(&c->device);
    c->n = int(d->n_cells);
    c->members = d->n_members;
    c->dx = (d->x_max - d->x_min) / double(d->n_cells);
    c->lam.assign(c->members, 0.0);
    // default tableau
    const double gm = 1.0 - 1.0 / std::sqrt(2.0), cc = 1.0 / (2.0 * gm);
    hsgn_tableau tb{};
    tb.stages = 2;
    tb.a_exp[1][0] = cc;
    tb.a_imp[0][0] = gm; tb.a_imp[1][0] = 1.0 - gm; tb.a_imp[1][1] = gm;
    tb.b[0] = 1.0 - gm; tb.b[1] = gm;
    c->tab = tb;
    c->aI1 = gm; c->aI2 = gm; c->wE = cc / gm; c->wR = (1.0 - gm) / gm;
    // kernels need > 48 KiB dynamic smem
    cudaFuncSetAttribute(stage_kernel<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    cudaFuncSetAttribute(stage_kernel<false, false, false, false, false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    cudaFuncSetAttribute(stage_kernel<false, false, true, false, false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_B));
    cudaFuncSetAttribute(stage_kernel<true, true, false, false, false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    cudaFuncSetAttribute(stage_kernel<true, true, true, false, false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_B));
    cudaFuncSetAttribute(stage_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_B));
    cudaFuncSetAttribute(stage_kernel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    cudaFuncSetAttribute(stage_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_B));
    cudaFuncSetAttribute(stage_kernel<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    cudaFuncSetAttribute(stage_kernel<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_B));
    cudaFuncSetAttribute(stage_kernel<true, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    cudaFuncSetAttribute(stage_kernel<true, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_B));
    cudaFuncSetAttribute(stage_kernel<false, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    cudaFuncSetAttribute(stage_kernel<false, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_B));
    cudaFuncSetAttribute(stage_kernel<false, false, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_PIC));
    cudaFuncSetAttribute(stage_kernel<false, false, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_PIC_B));
    cudaFuncSetAttribute(stage_kernel<true, true, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_PIC));
    cudaFuncSetAttribute(stage_kernel<true, true, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_PIC_B));
    cudaFuncSetAttribute(stage_kernel<false, true, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_PIC));
    cudaFuncSetAttribute(stage_kernel<false, true, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES_PIC_B));
    cudaFuncSetAttribute(sgn_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SSMEM_BYTES));
    cudaFuncSetAttribute(sgn_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SSMEM_BYTES));
    cudaFuncSetAttribute(sgn_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SSMEM_BYTES));
    cudaFuncSetAttribute(sgn_kernel<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SSMEM_BYTES_B));
    cudaFuncSetAttribute(sgn_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SSMEM_BYTES_B));
    cudaFuncSetAttribute(sgn_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SSMEM_BYTES_B));
    cudaFuncSetAttribute(explicit_kernel<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(XSMEM_BYTES));
    cudaFuncSetAttribute(explicit_kernel<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(XSMEM_BYTES));
    cudaFuncSetAttribute(explicit_kernel<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(XSMEM_BYTES));
    cudaFuncSetAttribute(explicit_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(XSMEM_BYTES));
    cudaFuncSetAttribute(explicit_kernel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(XSMEM_BYTES));
    cl_attrs<false, false, false>(); cl_attrs<false, false, true>();
    cl_attrs<true, true, false>(); cl_attrs<true, true, true>();
    cl_attrs<false, true, false>(); cl_attrs<false, true, true>();
    multi_attrs<false>(); multi_attrs<true>();
    cudaFuncSetAttribute(sep_solve_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sep_smem_bytes(1024)));
    cudaFuncSetAttribute(slab_iface_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(2 * GROUP_MAX_SX * (2 * GROUP_MAX_SX + 1) * sizeof(double)));
    if (const char *e = std::getenv("HSGN_CLUSTER")) c->cl_mode = std::atoi(e);
    choose_geometry(c);
    if (!slab) choose_cluster(c);
    choose_spike(c);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        delete c;
        return HSGN_E_CUDA;
    }
    *out = c;
    return HSGN_OK;
}

void hsgn_destroy(hsgn_ctx *c)
{
    if (!c) return;
    // the caller frees the workspace after this returns: no kernel or copy of
    // this context may still be using it
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->cs2) cudaStreamSynchronize(c->cs2);
    if (c->cp_in) cudaStreamSynchronize(c->cp_in);
    if (c->cp_out) cudaStreamSynchronize(c->cp_out);
    free_kids(c);
    if (c->cp_in) cudaStreamDestroy(c->cp_in);
    if (c->cp_out) cudaStreamDestroy(c->cp_out);
    if (c->cs2) cudaStreamDestroy(c->cs2);
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    for (int k = 0; k < KIDS_MAX; k++) {
        if (c->ev_in[k]) cudaEventDestroy(c->ev_in[k]);
        if (c->ev_done[k]) cudaEventDestroy(c->ev_done[k]);
    }
    if (c->kstat) cudaFreeHost(c->kstat);
    if (c->tstage) cudaFreeHost(c->tstage);
    drop_graphs(c);
    if (c->nccl) ncclCommDestroy(c->nccl);
    delete c;
}

size_t hsgn_workspace_bytes(const hsgn_ctx *c)
{
    if (!c) return 0;
    const size_t N = size_t(c->n) * c->members;
    size_t s = 0;
    s += 12 * align256(N * sizeof(double));                 // 3 buffers x 4 fields
    s += align256(size_t(c->n) * sizeof(double));           // b
    s += 3 * align256(size_t(c->members) * sizeof(double)); // lam, dt, dt_used
    s += align256(2 * size_t(c->members) * sizeof(double)); // t[2]
    s += align256(6 * size_t(c->members) * 8);              // maxes[3][2]
    s += align256(size_t(c->members) * ((c->n + T_MIN - 1) / T_MIN + 1) * 4 * sizeof(double));  // partials
    s += 256;                                               // scalars
    s += 256;                                               // ctrl
    s += 2 * align256(9 * size_t(H_MAX) * sizeof(double));  // slab halos
    s += kid_small_bytes(c->n, c->members) + KIDS_MAX * kid_small_bytes(c->n, 1);  // hsgn_run_host
    s += spike_bytes(c);                                    // tile-level SPIKE buffers
    return s;
}

hsgn_status hsgn_set_workspace(hsgn_ctx *c, void *p, size_t bytes)
{
    if (!c || !p) return HSGN_E_INVALID;
    if (bytes < hsgn_workspace_bytes(c)) return fail(c, HSGN_E_NOWORKSPACE, "workspace too small");
    if ((uintptr_t)p & 255) return fail(c, HSGN_E_INVALID, "workspace must be 256-byte aligned");
    drop_graphs(c);
    c->ws = (char *)p;
    c->ws_bytes = bytes;
    const size_t N = size_t(c->n) * c->members;
    char *q = c->ws;
    for (int bi = 0; bi < 3; bi++)
        for (int k = 0; k < 4; k++) { c->buf[bi][k] = (double *)q; q += align256(N * sizeof(double)); }
    c->b = (double *)q; q += align256(size_t(c->n) * sizeof(double));
    c->lamd = (double *)q; q += align256(size_t(c->members) * sizeof(double));
    c->t = (double *)q; q += align256(2 * size_t(c->members) * sizeof(double));
    c->dt = (double *)q; q += align256(size_t(c->members) * sizeof(double));
    c->dt_used = (double *)q; q += align256(size_t(c->members) * sizeof(double));
    c->maxes = (unsigned long long *)q; q += align256(6 * size_t(c->members) * 8);
    c->partials = (double *)q; q += align256(size_t(c->members) * ((c->n + T_MIN - 1) / T_MIN + 1) * 4 * sizeof(double));
    c->err = (unsigned int *)q;
    c->done = (unsigned int *)(q + 4);
    c->steps = (long long *)(q + 8);
    c->rho_obs = (unsigned long long *)(q + 16);
    c->kmin = (unsigned int *)(q + 64);
    q += 256;
    c->ctrl = (Ctrl *)q;
    q += 256;
    c->halo_l = (double *)q; q += align256(9 * size_t(H_MAX) * sizeof(double));
    c->halo_r = (double *)q; q += align256(9 * size_t(H_MAX) * sizeof(double));
    if (c->spG > 0) {
        const size_t mg = size_t(c->members) * c->spG;
        c->sp_tips = (double *)q; q += align256(mg * XPUB * sizeof(double));
        c->sp_L = (double *)q; q += align256(mg * sizeof(double));
        c->sp_fb = (double *)q; q += align256(mg * 16 * sizeof(double));
        c->sp_S = (double *)q; q += align256(size_t(c->members) * sep_scratch(c->spG) * sizeof(double));
        if (c->slab) {
            const size_t M = c->members;
            c->sx_nx = (double *)q; q += align256(M * 6 * sizeof(double));
            c->sx_fbl = (double *)q; q += align256(M * 8 * sizeof(double));
            c->sx_fbr = (double *)q; q += align256(M * 8 * sizeof(double));
            c->sx_elfr = (double *)q; q += align256(M * 2 * sizeof(double));
            c->sx_send = (double *)q; q += align256(M * 16 * sizeof(double));
            c->sx_all = (double *)q; q += align256(M * 6 * GROUP_MAX_SX * sizeof(double));
            c->sx_yvw = (double *)q; q += align256(M * 3 * size_t(c->spG) * sizeof(double));
        }
    } else {
        q += spike_bytes(c);
    }
    c->kid_ws = q;
    CUDA_TRY(c, cudaMemsetAsync(c->ws + (size_t)((char *)c->err - c->ws), 0, 512, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->b, 0, size_t(c->n) * sizeof(double), c->stream));
    c->ctrl_host = Ctrl{0.0, 0.0};
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->have_params) {
        CUDA_TRY(c, cudaMemcpy(c->lamd, c->lam.data(), c->members * sizeof(double), cudaMemcpyHostToDevice));
    }
    c->have_state = false;
    return HSGN_OK;
}

hsgn_status hsgn_set_params(hsgn_ctx *c, double g, const double *lambda, double cfl, double mcfl,
                            double h_min)
{
    if (!c || !lambda) return HSGN_E_INVALID;
    if (!(g > 0.0) || !(h_min >= 0.0)) return fail(c, HSGN_E_INVALID, "g must be > 0, h_min >= 0");
    for (int m = 0; m < c->members; m++)
        if (!(lambda[m] >= 0.0) || !std::isfinite(lambda[m]))
            return fail(c, HSGN_E_INVALID, "lambda must be finite and >= 0");
    c->g = g;
    c->cfl = cfl;
    c->mcfl = mcfl;
    c->h_min = h_min;
    c->lam.assign(lambda, lambda + c->members);
    c->have_params = true;
    drop_graphs(c);
    choose_geometry(c);
    if (c->ws) {
        CUDA_TRY(c, cudaMemcpyAsync(c->lamd, c->lam.data(), c->members * sizeof(double),
                                    cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    return HSGN_OK;
}

hsgn_status hsgn_set_tableau(hsgn_ctx *c, const hsgn_tableau *t)
{
    if (!c || !t) return HSGN_E_INVALID;
    if (t->stages == 1) {
        if (!(t->a_imp[0][0] > 0.0)) return fail(c, HSGN_E_INVALID, "a_11 must be > 0");
        c->aI1 = t->a_imp[0][0]; c->aI2 = 0; c->wE = 0; c->wR = 0;
    } else if (t->stages == 2) {
        if (!(t->a_imp[0][0] > 0.0) || !(t->a_imp[1][1] > 0.0) || t->a_exp[0][0] != 0.0 ||
            t->a_exp[0][1] != 0.0 || t->a_exp[1][1] != 0.0 || t->a_imp[0][1] != 0.0)
            return fail(c, HSGN_E_INVALID, "tableau shape");
        if (t->a_imp[1][0] != t->b[0] || t->a_imp[1][1] != t->b[1])
            return fail(c, HSGN_E_INVALID, "implicit tableau must be stiffly accurate (P:368)");
        c->aI1 = t->a_imp[0][0]; c->aI2 = t->a_imp[1][1];
        c->wE = t->a_exp[1][0] / t->a_imp[0][0];
        c->wR = t->a_imp[1][0] / t->a_imp[0][0];
    } else {
        return fail(c, HSGN_E_INVALID, "stages must be 1 or 2");
    }
    c->tab = *t;
    drop_graphs(c);
    choose_geometry(c);
    return HSGN_OK;
}

hsgn_status hsgn_set_bathymetry(hsgn_ctx *c, const double *b)
{
    if (!c) return HSGN_E_INVALID;
    if (!c->ws) return fail(c, HSGN_E_NOWORKSPACE, "workspace not set");
    drop_graphs(c);
    if (!b) {
        c->bathy = false;
        CUDA_TRY(c, cudaMemsetAsync(c->b, 0, size_t(c->n) * sizeof(double), c->stream));
    } else {
        c->bathy = true;
        CUDA_TRY(c, cudaMemcpyAsync(c->b, b, size_t(c->n) * sizeof(double), cudaMemcpyDefault, c->stream));
    }
    if (c->nccl) {
        hsgn_status st = nccl_exchange(c, 2);
        if (st != HSGN_OK) return st;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_set_filter(hsgn_ctx *c, double sigma, uint32_t mask)
{
    if (!c || !(sigma >= 0.0)) return HSGN_E_INVALID;
    if (sigma > 0.0 && mask != ((1u << 1) | (1u << 3)))
        return fail(c, HSGN_E_INVALID, "filter mask must be q|W (0xA)");
    c->filter_sigma = sigma;
    drop_graphs(c);
    return HSGN_OK;
}

hsgn_status hsgn_set_relaxation(hsgn_ctx *c, const hsgn_relax *r)
{
    if (!c) return HSGN_E_INVALID;
    if (!r) { c->relax = hsgn_relax{}; drop_graphs(c); return HSGN_OK; }
    if ((r->gen_rate > 0.0 && !(r->gen_x1 > c->desc.x_min)) ||
        (r->sp_rate > 0.0 && !(r->sp_x0 < c->desc.x_max)) || !(r->gen_rate <= 1.0) ||
        !(r->sp_rate <= 1.0) || ((r->gen_rate > 0.0 || r->sp_rate > 0.0) && !(r->level > 0.0)))
        return fail(c, HSGN_E_INVALID, "relaxation zones: bad extents or rates");
    c->relax = *r;
    drop_graphs(c);
    return HSGN_OK;
}

hsgn_status hsgn_set_state(hsgn_ctx *c, const double *h, const double *q, const double *K,
                           const double *W, double t0)
{
    if (!c || !h || !q || !K || !W) return HSGN_E_INVALID;
    if (!c->ws) return fail(c, HSGN_E_NOWORKSPACE, "workspace not set");
    if (!c->have_params) return fail(c, HSGN_E_INVALID, "hsgn_set_params first");
    const size_t N = size_t(c->n) * c->members;
    const double *src[4] = {h, q, K, W};
    c->cur = 0;
    for (int k = 0; k < 4; k++)
        CUDA_TRY(c, cudaMemcpyAsync(c->buf[0][k], src[k], N * sizeof(double), cudaMemcpyDefault, c->stream));
    std::vector<double> tv(c->members, t0);
    CUDA_TRY(c, cudaMemcpyAsync(c->t, tv.data(), c->members * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    c->dev_steps = 0;
    CUDA_TRY(c, cudaMemsetAsync(c->dt, 0, c->members * sizeof(double), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->maxes, 0, 6 * size_t(c->members) * 8, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->err, 0, 72, c->stream));   // err, done, steps, rho_obs, kmin
    dim3 grid(c->tiles, c->members);
    reduce_kernel<<<grid, NT, 0, c->stream>>>(c->buf[0][0], c->buf[0][1], c->buf[0][2],
                                              c->bathy ? c->b : nullptr, c->lamd, c->n, c->T, c->g,
                                              c->partials, c->maxes, c->members, c->scheme == 2);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));   // tv must outlive the copy
    c->host_steps = 0;
    c->have_state = true;
    if (c->scheme == 2) return sgn_geometry(c);
    return HSGN_OK;
}

hsgn_status hsgn_get_state(hsgn_ctx *c, double *h, double *q, double *K, double *W, double *t)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    st = reconcile(c);
    const size_t N = size_t(c->n) * c->members;
    double *dst[4] = {h, q, K, W};
    for (int k = 0; k < 4; k++)
        if (dst[k])
            CUDA_TRY(c, cudaMemcpyAsync(dst[k], c->buf[c->cur][k], N * sizeof(double), cudaMemcpyDefault, c->stream));
    if (t) CUDA_TRY(c, cudaMemcpyAsync(t, c->t + (c->dev_steps & 1) * c->members, c->members * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return st;
}

hsgn_status hsgn_run_host(hsgn_ctx *c, const double *h, const double *q, const double *K, const double *W,
                          double t0, int64_t n_steps, double *h_out, double *q_out, double *K_out,
                          double *W_out, double *t_out, int32_t chunks)
{
    if (!c || !h || !q || !K || !W || !h_out || !q_out || !K_out || !W_out || n_steps < 0 || chunks < 1)
        return HSGN_E_INVALID;
    if (!c->ws) return fail(c, HSGN_E_NOWORKSPACE, "workspace not set");
    if (!c->have_params) return fail(c, HSGN_E_INVALID, "hsgn_set_params first");
    if (c->slab) return fail(c, HSGN_E_INVALID, "hsgn_run_host: not for slab contexts");
    if (c->scheme == 2)
        return fail(c, HSGN_E_INVALID, "hsgn_run_host: SGN geometry depends on the whole state (use set_state)");
    chunks = std::min(std::min(chunks, KIDS_MAX), c->members);
    hsgn_status st;
    if (!c->cp_in) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cp_in, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cp_out, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
        for (int k = 0; k < KIDS_MAX; k++) {
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming));
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_done[k], cudaEventDisableTiming));
        }
        CUDA_TRY(c, cudaMallocHost(&c->kstat, KIDS_MAX * 2 * sizeof(long long)));
        CUDA_TRY(c, cudaMallocHost(&c->tstage, size_t(c->members) * sizeof(double)));
        // odd chunks run on a second compute stream: two chunks' kernels interleave
        // and fill each other's last-wave tails (HSGN_RH_STREAMS=1: one stream)
        const char *e = std::getenv("HSGN_RH_STREAMS");
        if (!(e && std::atoi(e) == 1)) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cs2, cudaStreamNonBlocking));
    }
    if ((st = make_kids(c, chunks)) != HSGN_OK) return st;
    c->have_state = false;                       // our buffers are the chunks' from here on
    const double *src[4] = {h, q, K, W};
    double *dst[4] = {h_out, q_out, K_out, W_out};
    const size_t n = size_t(c->n);
    CUDA_TRY(c, cudaEventRecord(c->ev_start, c->stream));   // earlier work on our buffers
    CUDA_TRY(c, cudaStreamWaitEvent(c->cp_in, c->ev_start, 0));
    if (c->cs2) CUDA_TRY(c, cudaStreamWaitEvent(c->cs2, c->ev_start, 0));
    long long l0 = 0;
    for (hsgn_ctx *kc : c->kids) l0 += kc->launches;
    size_t m0 = 0;
    for (int k = 0; k < chunks; k++) {
        hsgn_ctx *kc = c->kids[k];
        const size_t cn = size_t(kc->members) * n;
        for (int f = 0; f < 4; f++)
            CUDA_TRY(c, cudaMemcpyAsync(kc->buf[0][f], src[f] + m0 * n, cn * sizeof(double),
                                        cudaMemcpyDefault, c->cp_in));
        CUDA_TRY(c, cudaEventRecord(c->ev_in[k], c->cp_in));
        CUDA_TRY(c, cudaStreamWaitEvent(kc->stream, c->ev_in[k], 0));
        if ((st = kid_state_init(kc, t0)) != HSGN_OK) return fail(c, st, kc->last_error);
        if ((st = run_steps_impl(kc, n_steps)) != HSGN_OK) return fail(c, st, kc->last_error);
        CUDA_TRY(c, cudaEventRecord(c->ev_done[k], kc->stream));
        CUDA_TRY(c, cudaStreamWaitEvent(c->cp_out, c->ev_done[k], 0));
        for (int f = 0; f < 4; f++)
            CUDA_TRY(c, cudaMemcpyAsync(dst[f] + m0 * n, kc->buf[kc->cur][f], cn * sizeof(double),
                                        cudaMemcpyDefault, c->cp_out));
        CUDA_TRY(c, cudaMemcpyAsync(c->tstage + m0, kc->t + (kc->host_steps & 1) * kc->members,
                                    kc->members * sizeof(double), cudaMemcpyDeviceToHost, c->cp_out));
        CUDA_TRY(c, cudaMemcpyAsync(c->kstat + 2 * k, kc->err, 2 * sizeof(long long),
                                    cudaMemcpyDeviceToHost, c->cp_out));
        m0 += kc->members;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->cp_out));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->cs2) CUDA_TRY(c, cudaStreamSynchronize(c->cs2));
    if (t_out) std::memcpy(t_out, c->tstage, size_t(c->members) * sizeof(double));
    long long l1 = 0;
    for (hsgn_ctx *kc : c->kids) l1 += kc->launches;
    c->launches += l1 - l0;
    // a chunk that stopped early (device error): its committed state replaces
    // what was copied out, and the first error is returned
    hsgn_status first = HSGN_OK;
    m0 = 0;
    for (int k = 0; k < chunks; k++) {
        hsgn_ctx *kc = c->kids[k];
        const unsigned bits = unsigned(c->kstat[2 * k] & 0xffffffffll);
        if (bits || c->kstat[2 * k + 1] != n_steps) {
            const hsgn_status ks = reconcile(kc);
            const size_t cn = size_t(kc->members) * n;
            for (int f = 0; f < 4; f++)
                CUDA_TRY(c, cudaMemcpy(dst[f] + m0 * n, kc->buf[kc->cur][f], cn * sizeof(double), cudaMemcpyDefault));
            if (t_out)
                CUDA_TRY(c, cudaMemcpy(t_out + m0, kc->t + (kc->dev_steps & 1) * kc->members,
                                       kc->members * sizeof(double), cudaMemcpyDefault));
            if (first == HSGN_OK) {
                first = ks != HSGN_OK ? ks : HSGN_E_INVALID;
                c->last_error = "member chunk " + std::to_string(k) + ": " + kc->last_error;
            }
        }
        m0 += kc->members;
    }
    return first;
}

hsgn_status hsgn_step(hsgn_ctx *c, double dt, double *dt_used)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    st = set_ctrl(c, c->ctrl_host.t_end, dt > 0.0 ? dt : 0.0);
    if (st != HSGN_OK) return st;
    if (c->slab) {
        st = run_steps_impl(c, 1);
        if (st != HSGN_OK) return st;
        if (dt_used)
            CUDA_TRY(c, cudaMemcpyAsync(c->dt_used, c->dt, c->members * sizeof(double),
                                        cudaMemcpyDeviceToDevice, c->stream));
    } else {
        if (!fused_dt(c)) st = launch_dtc(c, c->host_steps, 0, 1);
        if (st != HSGN_OK) return st;
        st = enqueue_step(c, c->cur, c->host_steps, nullptr, dt_used ? c->dt_used : nullptr);
        if (st != HSGN_OK) return st;
        c->cur ^= 1;
        c->host_steps++;
    }
    if (dt_used) {
        st = reconcile(c);
        CUDA_TRY(c, cudaMemcpy(dt_used, c->dt_used, c->members * sizeof(double), cudaMemcpyDeviceToHost));
        return st;
    }
    return HSGN_OK;
}

hsgn_status hsgn_run_steps(hsgn_ctx *c, int64_t n_steps)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (n_steps < 0) return HSGN_E_INVALID;
    st = set_ctrl(c, c->ctrl_host.t_end, 0.0);
    if (st != HSGN_OK) return st;
    return run_steps_impl(c, n_steps);
}

hsgn_status hsgn_run_steps_timed(hsgn_ctx *c, int64_t n_steps, double *stage_ms)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (n_steps < 0 || !stage_ms) return HSGN_E_INVALID;
    if (c->slab) return fail(c, HSGN_E_INVALID, "hsgn_run_steps_timed: not for slab contexts");
    if (!c->stream) return fail(c, HSGN_E_INVALID, "hsgn_run_steps_timed: needs a non-default stream");
    st = set_ctrl(c, c->ctrl_host.t_end, 0.0);
    if (st != HSGN_OK) return st;
    // the n steps are captured into one CUDA graph with event record nodes
    // before, between and after the kernels, instantiated, then launched once:
    // the same launch mode as hsgn_run_steps, timed on the device
    const size_t ne = size_t(n_steps) * 3 + 2;
    std::vector<cudaEvent_t> ev(ne);
    for (auto &e : ev) CUDA_TRY(c, cudaEventCreate(&e));
    cudaGraph_t gr = nullptr;
    cudaGraphExec_t gx = nullptr;
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->ev_ext = true;
    cudaError_t ce = rec_ev(c, ev[ne - 2]);
    int cc = c->cur;
    if (ce == cudaSuccess && !fused_dt(c)) st = launch_dtc(c, c->host_steps, 0, 1);
    for (int64_t k = 0; k < n_steps && st == HSGN_OK && ce == cudaSuccess; k++) {
        st = enqueue_step(c, cc, c->host_steps + k, &ev[3 * k], nullptr, k == 0, k == n_steps - 1);
        cc ^= 1;
    }
    if (ce == cudaSuccess) ce = rec_ev(c, ev[ne - 1]);
    c->ev_ext = false;
    const cudaError_t ce2 = cudaStreamEndCapture(c->stream, &gr);
    if (st == HSGN_OK && ce == cudaSuccess && ce2 == cudaSuccess) ce = cudaGraphInstantiate(&gx, gr, 0);
    if (st == HSGN_OK && ce == cudaSuccess && ce2 == cudaSuccess) ce = cudaGraphLaunch(gx, c->stream);
    if (st == HSGN_OK && ce == cudaSuccess && ce2 == cudaSuccess) {
        c->cur = cc;
        c->host_steps += n_steps;
        ce = cudaStreamSynchronize(c->stream);
    }
    stage_ms[0] = stage_ms[1] = stage_ms[2] = 0.0;
    if (st == HSGN_OK && ce == cudaSuccess && ce2 == cudaSuccess) {
        for (int64_t k = 0; k < n_steps; k++) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, ev[3 * k], ev[3 * k + 1]);
            cudaEventElapsedTime(&b, ev[3 * k + 1], ev[3 * k + 2]);
            stage_ms[0] += a;
            stage_ms[1] += b;
        }
        float tot = 0.f;
        cudaEventElapsedTime(&tot, ev[ne - 2], ev[ne - 1]);
        stage_ms[2] = tot;
    }
    if (gx) cudaGraphExecDestroy(gx);
    if (gr) cudaGraphDestroy(gr);
    for (auto &e : ev) cudaEventDestroy(e);
    if (st != HSGN_OK) return st;
    if (ce != cudaSuccess || ce2 != cudaSuccess)
        return fail(c, HSGN_E_CUDA, std::string("timed graph: ") + cudaGetErrorString(ce != cudaSuccess ? ce : ce2));
    return reconcile(c);
}

hsgn_status hsgn_sync(hsgn_ctx *c)
{
    if (!c) return HSGN_E_INVALID;
    return reconcile(c);
}

hsgn_status hsgn_advance_to(hsgn_ctx *c, double t_end, int64_t max_steps, int64_t *steps_done)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (!(t_end > 0.0)) return fail(c, HSGN_E_INVALID, "t_end must be > 0");
    st = set_ctrl(c, t_end, 0.0);
    if (st != HSGN_OK) return st;
    std::vector<double> tv(c->members);
    long long taken = 0;
    const long long s0 = c->host_steps;
    while (taken < max_steps) {
        st = reconcile(c);
        CUDA_TRY(c, cudaMemcpy(tv.data(), c->t + (c->dev_steps & 1) * c->members, c->members * sizeof(double), cudaMemcpyDeviceToHost));
        if (st != HSGN_OK) break;
        bool all = true;
        for (double tm : tv) all &= !(tm < t_end);
        if (all) break;
        const long long chunk = std::min<long long>(POLL_STEPS, max_steps - taken);
        st = run_steps_impl(c, chunk);
        if (st != HSGN_OK) break;
        taken += chunk;
    }
    if (st == HSGN_OK) st = reconcile(c);
    // steps that actually advanced some member are not distinguishable from
    // carried no-op steps here; report committed device steps since entry
    if (steps_done) *steps_done = c->host_steps - s0;
    set_ctrl(c, 0.0, 0.0);
    return st;
}

hsgn_status hsgn_get_diagnostics(hsgn_ctx *c, hsgn_diag *o)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (!o) return HSGN_E_INVALID;
    unsigned int bits = 0;
    st = reconcile(c, &bits);
    dim3 grid(c->tiles, c->members);
    reduce_kernel<<<grid, NT, 0, c->stream>>>(c->buf[c->cur][0], c->buf[c->cur][1], c->buf[c->cur][2],
                                              c->bathy ? c->b : nullptr, c->lamd, c->n, c->T, c->g,
                                              c->partials, nullptr, c->members, 0);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    std::vector<double> part(size_t(c->members) * c->tiles * 4), tv(c->members), dv(c->members);
    long long dsteps = 0;
    CUDA_TRY(c, cudaMemcpyAsync(part.data(), c->partials, part.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(tv.data(), c->t + (c->dev_steps & 1) * c->members, c->members * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(dv.data(), c->dt, c->members * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&dsteps, c->steps, sizeof(dsteps), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    hsgn_diag d{};
    d.min_h = 1e300;
    d.t_min = 1e300; d.t_max = -1e300; d.dt_last_min = 1e300; d.dt_last_max = -1e300;
    for (int m = 0; m < c->members; m++) {
        double mass = 0.0, um = 0.0, nm = 0.0;
        for (int j = 0; j < c->tiles; j++) {
            const double *p = &part[(size_t(m) * c->tiles + j) * 4];
            mass += p[0];
            d.min_h = std::min(d.min_h, p[1]);
            um = std::max(um, p[2]);
            nm = std::max(nm, p[3]);
        }
        d.max_abs_u = std::max(d.max_abs_u, um);
        d.nu_max = std::max(d.nu_max, nm);
        // achieved Courant numbers of the step about to be taken:
        // its dt (set from this state) against this state's maxima
        d.cfl_imex = std::max(d.cfl_imex, dv[m] * nm / c->dx);
        d.mcfl = std::max(d.mcfl, dv[m] * um / c->dx);
        d.mass += mass * c->dx;
        d.t_min = std::min(d.t_min, tv[m]); d.t_max = std::max(d.t_max, tv[m]);
        d.dt_last_min = std::min(d.dt_last_min, dv[m]); d.dt_last_max = std::max(d.dt_last_max, dv[m]);
    }
    unsigned long long rb = 0;
    unsigned int kb = 0;
    CUDA_TRY(c, cudaMemcpy(&rb, c->rho_obs, sizeof(rb), cudaMemcpyDeviceToHost));
    CUDA_TRY(c, cudaMemcpy(&kb, c->kmin, sizeof(kb), cudaMemcpyDeviceToHost));
    double rmx;
    memcpy(&rmx, &rb, sizeof(rmx));
    d.rho_max = rmx;
    // min kappa: ~kb is the ordered key of the high word (hsgn_kernels.cuh
    // khi_key); the value is that high word with a zero low word, i.e. the
    // minimum rounded toward zero to 2^-20 relative (0: no SI stage -> +inf)
    if (kb == 0) {
        d.min_kappa = HUGE_VAL;
    } else {
        const int key = int(~kb);
        const int hi = key >= 0 ? key : (key ^ 0x7fffffff);
        const unsigned long long b = (unsigned long long)(unsigned int)hi << 32;
        memcpy(&d.min_kappa, &b, sizeof(b));
    }
    d.steps = dsteps;
    d.error_bits = int32_t(bits);
    *o = d;
    return st;
}

int64_t hsgn_launch_count(const hsgn_ctx *c) { return c ? c->launches : 0; }

hsgn_status hsgn_set_scheme(hsgn_ctx *c, int32_t scheme, int32_t stages)
{
    if (!c) return HSGN_E_INVALID;
    const int prev = c->scheme;
    if (scheme == HSGN_SCHEME_SI) {
        c->scheme = 0;
    } else if (scheme == HSGN_SCHEME_EXPLICIT || scheme == HSGN_SCHEME_SGN) {
        if (stages != 1 && stages != 2) return fail(c, HSGN_E_INVALID, "explicit stages must be 1 or 2");
        c->scheme = scheme == HSGN_SCHEME_EXPLICIT ? 1 : 2;
        c->x_stages = stages;
    } else {
        return fail(c, HSGN_E_INVALID, "unknown scheme");
    }
    drop_graphs(c);
    choose_geometry(c);
    if (c->have_state && c->ws) {
        hsgn_status st = reconcile(c);
        if (st != HSGN_OK) return st;
        if ((prev == 2) != (c->scheme == 2)) {
            st = reseed_maxima(c);      // the SGN celerity differs from hSGN's
            if (st != HSGN_OK) return st;
        }
        if (c->scheme == 2) return sgn_geometry(c);
    }
    return HSGN_OK;
}

hsgn_status hsgn_set_picard(hsgn_ctx *c, int32_t passes)
{
    if (!c || passes < 0 || passes > 16) return HSGN_E_INVALID;
    c->picard = passes;
    drop_graphs(c);
    choose_geometry(c);
    return HSGN_OK;
}

hsgn_status hsgn_set_well_balanced(hsgn_ctx *c, int32_t on)
{
    if (!c) return HSGN_E_INVALID;
    c->wb = on != 0;
    drop_graphs(c);
    choose_geometry(c);
    return HSGN_OK;
}

hsgn_status hsgn_run_resident(hsgn_ctx *c, int64_t n_steps, double t_end, double *device_ms)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (n_steps < 0 || n_steps > (1 << 30)) return fail(c, HSGN_E_INVALID, "run_resident: n_steps out of range");
    if (c->clC <= 0 || !exact_eligible(c) || c->tab.stages != 2)
        return fail(c, HSGN_E_INVALID, "run_resident: member must fit a cluster (n % 4 == 0, <= 16 x 512 cells), "
                                       "SI scheme, 2-stage tableau, no Picard / A25 / slab sides");
    st = reconcile(c);
    if (st != HSGN_OK) return st;
    st = set_ctrl(c, t_end > 0.0 ? t_end : 0.0, 0.0);
    if (st != HSGN_OK) return st;
    if (n_steps == 0) { if (device_ms) *device_ms = 0.0; return HSGN_OK; }
    const long long k0 = c->host_steps;
    Params P = make_params(c, k0);
    P.T = c->clT;
    P.tiles = c->clC;
    Bufs B{};
    for (int f = 0; f < 4; f++) { B.Un[f] = c->buf[c->cur][f]; B.U1[f] = c->buf[2][f]; B.out[f] = c->buf[c->cur ^ 1][f]; }
    CUDA_TRY(c, cudaMemsetAsync(c->maxes, 0, 6 * size_t(c->members) * 8, c->stream));
    if (!c->ev_start) CUDA_TRY(c, cudaEventCreate(&c->ev_start));
    cudaEvent_t e1;
    CUDA_TRY(c, cudaEventCreate(&e1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->clC, c->members);
    cfg.blockDim = dim3(CNT);
    cfg.dynamicSmemBytes = c->bathy ? CSMEM_BYTES_B : CSMEM_BYTES;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(c->clC);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(c, cudaEventRecord(c->ev_start, c->stream));
    if (c->bathy) CUDA_TRY(c, cudaLaunchKernelEx(&cfg, cl_multi_kernel<true>, P, B, int(n_steps), int(k0)));
    else CUDA_TRY(c, cudaLaunchKernelEx(&cfg, cl_multi_kernel<false>, P, B, int(n_steps), int(k0)));
    CUDA_TRY(c, cudaEventRecord(e1, c->stream));
    c->launches++;
    CUDA_TRY(c, cudaEventSynchronize(e1));
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, c->ev_start, e1);
    cudaEventDestroy(e1);
    if (device_ms) *device_ms = ms;
    unsigned int bits = 0;
    CUDA_TRY(c, cudaMemcpy(&bits, c->err, sizeof(bits), cudaMemcpyDeviceToHost));
    if (bits) return fail(c, status_from_bits(bits), "run_resident: device error bits; state kept at the call's start");
    // commit: the output buffer becomes the state, n_steps more steps
    long long ds = 0;
    CUDA_TRY(c, cudaMemcpy(&ds, c->steps, sizeof(ds), cudaMemcpyDeviceToHost));
    ds += n_steps;
    CUDA_TRY(c, cudaMemcpy(c->steps, &ds, sizeof(ds), cudaMemcpyHostToDevice));
    c->cur ^= 1;
    c->host_steps += n_steps;
    c->dev_steps = ds;
    return HSGN_OK;
}

hsgn_status hsgn_set_cluster(hsgn_ctx *c, int32_t mode)
{
    if (!c || mode < 0 || mode > 3) return HSGN_E_INVALID;
    drop_graphs(c);
    c->cl_mode = mode;
    return HSGN_OK;
}

int32_t hsgn_get_cluster(const hsgn_ctx *c, int32_t *ctas, int32_t *tile_rows)
{
    if (!c) return -1;
    if (use_cluster(c)) {
        if (ctas) *ctas = c->clC;
        if (tile_rows) *tile_rows = c->clT;
        return 1;
    }
    if (use_spike(c)) {
        if (ctas) *ctas = c->spG;
        if (tile_rows) *tile_rows = c->spT;
        return 2;
    }
    if (ctas) *ctas = 0;
    if (tile_rows) *tile_rows = 0;
    return 0;
}

#if HSGN_EXP_TIMING
// timing experiments only (not part of the product ABI): per-stage sums of
// CTA clocks [load wait, compute + store issue, epilogue + store drain, CTAs]
int hsgn_cl_counters(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_clt, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(g_clt, z, sizeof(z));
    }
    return 0;
}

int hsgn_exp_counters(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_exp, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_exp, z, sizeof(z));
    }
    return 0;
}
#endif

hsgn_status hsgn_get_geometry(const hsgn_ctx *c, int32_t *T, int32_t *w, int32_t *tiles,
                              int32_t *threads, int32_t *max_rows)
{
    if (!c) return HSGN_E_INVALID;
    if (T) *T = c->T;
    if (w) *w = c->w;
    if (tiles) *tiles = c->tiles;
    if (threads) *threads = NT;
    if (max_rows) *max_rows = LCAP;
    return HSGN_OK;
}


// ---- slab groups and NCCL ---------------------------------

struct hsgn_group {
    std::vector<hsgn_ctx *> ctx;
};

hsgn_status hsgn_group_create(hsgn_ctx *const *ctxs, int32_t n, hsgn_group **out)
{
    if (!ctxs || !out || n < 1 || n > GROUP_MAX) return HSGN_E_INVALID;
    *out = nullptr;
    hsgn_ctx *c0 = ctxs[0];
    for (int i = 0; i < n; i++) {
        hsgn_ctx *c = ctxs[i];
        hsgn_status st = ready(c);
        if (st != HSGN_OK) return st;
        if (c->stream != c0->stream || c->w != c0->w || c->members != c0->members ||
            c->tab.stages != c0->tab.stages || c->host_steps != c0->host_steps || c->nccl)
            return fail(c, HSGN_E_INVALID, "group: contexts must share stream, overlap, tableau and step");
        if (c->n < slab_H(c)) return fail(c, HSGN_E_INVALID, "group: slab shorter than its halo");
    }
    hsgn_group *g = new hsgn_group();
    g->ctx.assign(ctxs, ctxs + n);
    if (c0->bathy) {
        hsgn_status st = loopback_exchange(g->ctx, 2);   // static bathymetry halos
        if (st != HSGN_OK) { delete g; return st; }
    }
    *out = g;
    return HSGN_OK;
}

hsgn_status hsgn_group_run_steps(hsgn_group *g, int64_t n_steps)
{
    if (!g || n_steps < 0) return HSGN_E_INVALID;
    for (auto *c : g->ctx) {
        if (c->w != g->ctx[0]->w || slab_H(c) != slab_H(g->ctx[0]) || use_spike(c) != use_spike(g->ctx[0]) ||
            c->n < slab_H(c))
            return fail(c, HSGN_E_INVALID, "group: the slabs' overlaps or depth-solve modes differ "
                                           "(or a slab is shorter than its halo)");
        hsgn_status st = set_ctrl(c, c->ctrl_host.t_end, 0.0);
        if (st != HSGN_OK) return st;
    }
    for (int64_t i = 0; i < n_steps; i++) {
        hsgn_status st = slab_step(g->ctx, g->ctx[0]->host_steps, false);
        if (st != HSGN_OK) return st;
    }
    return HSGN_OK;
}

void hsgn_group_destroy(hsgn_group *g) { delete g; }

// ---- host-staged slab transport ------------------------------------------
int64_t hsgn_slab_xfer_count(const hsgn_ctx *c, int32_t what)
{
    if (!c || !c->slab) return -1;
    if (what == HSGN_XFER_MAXIMA) return 2 * int64_t(c->members);
    if (what < HSGN_XFER_UN || what > HSGN_XFER_B) return -1;
    const int nf = what == HSGN_XFER_B ? 1 : 4;
    return 2 * int64_t(nf) * (c->w + 3);
}

hsgn_status hsgn_slab_get(hsgn_ctx *c, int32_t what, void *host_out)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (!host_out || !c->slab || c->nccl) return fail(c, HSGN_E_INVALID, "slab_get: host-staged slab contexts only");
    if (what == HSGN_XFER_MAXIMA) {
        const int slot = int(c->host_steps % 3);
        CUDA_TRY(c, cudaMemcpyAsync(host_out, c->maxes + size_t(slot) * 2 * c->members,
                                    2 * size_t(c->members) * 8, cudaMemcpyDeviceToHost, c->stream));
    } else if (what >= HSGN_XFER_UN && what <= HSGN_XFER_B) {
        const int which = what - HSGN_XFER_UN, nf = which == 2 ? 1 : 4, H = c->w + 3;
        double *o = (double *)host_out;
        for (int f = 0; f < nf; f++) {       // [left boundary: nf x H][right boundary: nf x H]
            CUDA_TRY(c, cudaMemcpyAsync(o + f * H, bnd_src(c, false, which, f, H), H * 8, cudaMemcpyDeviceToHost,
                                        c->stream));
            CUDA_TRY(c, cudaMemcpyAsync(o + (nf + f) * H, bnd_src(c, true, which, f, H), H * 8,
                                        cudaMemcpyDeviceToHost, c->stream));
        }
    } else {
        return fail(c, HSGN_E_INVALID, "slab_get: unknown transfer");
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return HSGN_OK;
}

hsgn_status hsgn_slab_put(hsgn_ctx *c, int32_t what, const void *host_in)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (!host_in || !c->slab || c->nccl) return fail(c, HSGN_E_INVALID, "slab_put: host-staged slab contexts only");
    if (what == HSGN_XFER_MAXIMA) {
        const int slot = int(c->host_steps % 3);
        CUDA_TRY(c, cudaMemcpyAsync(c->maxes + size_t(slot) * 2 * c->members, host_in, 2 * size_t(c->members) * 8,
                                    cudaMemcpyHostToDevice, c->stream));
    } else if (what >= HSGN_XFER_UN && what <= HSGN_XFER_B) {
        const int which = what - HSGN_XFER_UN, nf = which == 2 ? 1 : 4, H = c->w + 3;
        const double *in = (const double *)host_in;
        for (int f = 0; f < nf; f++) {       // [left halo: nf x H][right halo: nf x H]
            if (c->desc.bc_left == HSGN_BC_HALO)
                CUDA_TRY(c, cudaMemcpyAsync(halo_dst(c, true, which, f), in + f * H, H * 8, cudaMemcpyHostToDevice,
                                            c->stream));
            if (c->desc.bc_right == HSGN_BC_HALO)
                CUDA_TRY(c, cudaMemcpyAsync(halo_dst(c, false, which, f), in + (nf + f) * H, H * 8,
                                            cudaMemcpyHostToDevice, c->stream));
        }
    } else {
        return fail(c, HSGN_E_INVALID, "slab_put: unknown transfer");
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));   // the host buffer may be reused at return
    return HSGN_OK;
}

hsgn_status hsgn_slab_phase(hsgn_ctx *c, int32_t phase)
{
    hsgn_status st = ready(c);
    if (st != HSGN_OK) return st;
    if (!c->slab || c->nccl) return fail(c, HSGN_E_INVALID, "slab_phase: host-staged slab contexts only");
    if (use_spike(c))
        return fail(c, HSGN_E_INVALID, "slab_phase: SPIKE across slabs needs the group or NCCL transport "
                                       "(set_cluster(0) and a CFL_IMEX bound for the overlapped tiles)");
    if (phase == HSGN_PHASE_DT) {
        st = set_ctrl(c, c->ctrl_host.t_end, 0.0);
        if (st != HSGN_OK) return st;
    }
    std::vector<hsgn_ctx *> g{c};
    const long long k = c->host_steps;
    switch (phase) {
    case HSGN_PHASE_DT: return slab_phase_dt(g, k);
    case HSGN_PHASE_STAGE1: return slab_phase_stage(g, k, false);
    case HSGN_PHASE_STAGE2:
        if (c->tab.stages != 2) return fail(c, HSGN_E_INVALID, "slab_phase: 1-stage tableau has no stage 2");
        return slab_phase_stage(g, k, true);
    case HSGN_PHASE_COMMIT: return slab_phase_commit(g, k);
    default: return fail(c, HSGN_E_INVALID, "slab_phase: unknown phase");
    }
}

hsgn_status hsgn_debug_copy(hsgn_ctx *c, int32_t which, double *host, int64_t count)
{
    if (!c || !host || count < 0) return HSGN_E_INVALID;
    const double *src[7] = {c->sp_L, c->sx_yvw, c->sx_elfr, c->sx_nx, c->sx_all, c->sp_tips, c->sp_fb};
    if (which < 0 || which > 6 || !src[which]) return HSGN_E_INVALID;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    CUDA_TRY(c, cudaMemcpy(host, src[which], size_t(count) * sizeof(double), cudaMemcpyDeviceToHost));
    return HSGN_OK;
}

hsgn_status hsgn_nccl_unique_id(void *id)
{
    if (!id) return HSGN_E_INVALID;
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return HSGN_E_CUDA;
    memcpy(id, &u, sizeof(u));
    return HSGN_OK;
}

hsgn_status hsgn_attach_nccl(hsgn_ctx *c, const void *id, int32_t rank, int32_t world)
{
    if (!c || !id || world < 1 || rank < 0 || rank >= world) return HSGN_E_INVALID;
    if (!c->slab) return fail(c, HSGN_E_INVALID, "attach_nccl: context has no BC_HALO side");
    if (c->nccl) return fail(c, HSGN_E_INVALID, "attach_nccl: already attached");
    if (c->n < slab_H(c)) return fail(c, HSGN_E_INVALID, "attach_nccl: slab shorter than its halo (n < overlap + 3)");
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    NCCL_TRY(c, ncclCommInitRank(&c->nccl, world, u, rank));
    c->nrank = rank;
    c->nworld = world;
    // every rank must exchange halos of the same size (w + 3) for the same
    // members: max over ranks of (w, -w, members, -members)
    {
        long long v[4] = {c->w, -c->w, c->members, -c->members};
        long long *d = nullptr;
        cudaError_t ce = cudaMalloc(&d, sizeof v);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(d, v, sizeof v, cudaMemcpyHostToDevice, c->stream);
        ncclResult_t nr = ncclSuccess;
        if (ce == cudaSuccess) nr = ncclAllReduce(d, d, 4, ncclInt64, ncclMax, c->nccl, c->stream);
        if (ce == cudaSuccess && nr == ncclSuccess) ce = cudaMemcpyAsync(v, d, sizeof v, cudaMemcpyDeviceToHost, c->stream);
        if (ce == cudaSuccess && nr == ncclSuccess) ce = cudaStreamSynchronize(c->stream);
        if (d) cudaFree(d);
        if (ce != cudaSuccess || nr != ncclSuccess) {
            ncclCommDestroy(c->nccl);
            c->nccl = nullptr;
            return fail(c, ce != cudaSuccess ? HSGN_E_CUDA : HSGN_E_COMM,
                        ce != cudaSuccess ? cudaGetErrorString(ce) : ncclGetErrorString(nr));
        }
        if (v[0] != -v[1] || v[2] != -v[3]) {
            ncclCommDestroy(c->nccl);
            c->nccl = nullptr;
            return fail(c, HSGN_E_INVALID, "attach_nccl: ranks disagree on the overlap or the member count");
        }
    }
    c->nccl_w = c->w;
    if (c->bathy) return nccl_exchange(c, 2);
    return HSGN_OK;
}

}  // extern "C"
