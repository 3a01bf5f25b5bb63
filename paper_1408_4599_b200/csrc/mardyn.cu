// mardyn.cu -- host engine and C ABI (include/mardyn.h) of the B200-native
// ls1-mardyn hot path.  Every step of the path runs in the kernels of
// kernels_state.cuh / kernels_force.cuh; this file validates inputs, lays
// out the caller-provided workspace, builds the per-component tables,
// captures one time step per buffer parity as a CUDA graph and replays it.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/mardyn.h"
#include "common.cuh"
#include "decomp.hpp"
#include "nccl_api.hpp"
#include "kernels_force.cuh"
#include "kernels_lj1.cuh"
#include "kernels_rigid3.cuh"
#include "kernels_state.cuh"

// NVTX ranges around the library's host phases (visible in Nsight Systems / ncu --nvtx; a no-op
// without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace {

struct HostComp {
    std::vector<mardyn_lj_site> lj;
    std::vector<mardyn_charge> q;
    std::vector<mardyn_polar> mu, Q;
    double mass;
    double I[3];
};

enum KernelKind { KER_LJ1 = 0, KER_RIGID = 1, KER_GENERIC = 2 };
enum RigidShape { SHAPE_NONE, SHAPE_2CLJQ, SHAPE_TIP4P, SHAPE_GEN };

#ifndef MD_LJ1_WARPS
#define MD_LJ1_WARPS 4
#endif
#ifndef MD_LJ1_CAPP
#define MD_LJ1_CAPP 448
#endif
#ifndef MD_LJ1_MINB
#define MD_LJ1_MINB 4
#endif
constexpr int LJ1_WARPS = MD_LJ1_WARPS;
constexpr int LJ1_CAPP = MD_LJ1_CAPP;
using LJ1 = lj1::Cfg<LJ1_WARPS, LJ1_CAPP>;
#define K_LJ1 lj1::k_force_lj1<LJ1_WARPS, LJ1_CAPP, MD_LJ1_MINB, false>
#define K_LJ1_STEP lj1::k_force_lj1<LJ1_WARPS, LJ1_CAPP, MD_LJ1_MINB, true>
#define K_LJ1_STEP_DD lj1::k_force_lj1<LJ1_WARPS, LJ1_CAPP, MD_LJ1_MINB, true, true>
constexpr int RIG_WARPS = rig3::WARPS;   // load-balanced rigid kernel (kernels_rigid3.cuh), configs 2, 3
constexpr int GEN_WARPS = 1;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct Group;                            // ranks that step together (dist_engine.cuh)
struct mardyn_ctx;
static bool group_is_nccl(const Group* g);
// one rank's entry of the IPC handle all-gather (dist_engine.cuh: nccl_ipc_setup): the
// 64-byte handle of the allocation holding its receive areas, their offsets, the receive
// capacity, a success word and its per-source receive-segment offsets
static size_t ipc_blob_bytes(int p) { return 64 + 5 * 8 + 8 * (size_t)p; }
static int set_molecules_dd(mardyn_ctx* ctx, int64_t n, const int64_t* id, const int32_t* comp, const double* r,
                            const double* v, const double* q, const double* j, int32_t half_step);
static int egress_dd(mardyn_ctx* ctx, double* r, double* v, double* q, double* j, double* F, double* tau,
                     uint32_t* ufix, int32_t* cell, int64_t n_slots, int64_t* n_out, int64_t* ids_out,
                     int32_t* comp_out);
static int group_observables(mardyn_ctx* ctx, std::vector<ObsRec>& ring);
static int group_step(mardyn_ctx* ctx, int32_t nsteps);
static int group_compute_forces(mardyn_ctx* ctx);
static void group_release(mardyn_ctx* ctx);
static int compute_forces_local(mardyn_ctx* ctx);
static std::vector<mardyn_ctx*> group_members(mardyn_ctx* ctx);
static void group_drop_graphs(Group* G);

struct mardyn_ctx {
    std::string err;
    double L[3], rc, dt, eps_rf;
    int lj_shift;
    std::vector<HostComp> comps;
    std::vector<double> eta;
    GridP g;
    DevModel model;
    int kernel = KER_LJ1;
    int shape = SHAPE_NONE;
    bool rigid = false;
    int nslots = 0;
    int force_warps_per_block = LJ1_WARPS;
    int force_blocks = 0;              // occupancy grid (sizes the per-warp partials)
    int force_grid = 0;                // launched grid: the occupancy grid, or fewer CTAs for small systems
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int device = 0;
    int num_sms = 0;
    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0;
    int64_t cap = 0;
    int ncell_pad = 0;
    int ntiles = 0;
    int nkblocks = 0;
    uint4* pos[2] = {nullptr, nullptr};
    float4* vel[2] = {nullptr, nullptr};
    float4* quat[2] = {nullptr, nullptr};
    float4* angm[2] = {nullptr, nullptr};
    float4* xs = nullptr;
    float4* site = nullptr;
    float4* force = nullptr;
    float4* torque = nullptr;
    int* cell_of = nullptr;
    int* rank = nullptr;
    int* count = nullptr;
    int* start = nullptr;
    unsigned long long* scan_flags = nullptr;   // ntiles look-back flags + tile counter
    FinPart* fin_scratch = nullptr;
    int* fin_ticket = nullptr;
    unsigned long long* keys = nullptr;
    int* oldidx = nullptr;
    ForcePartial* fpart = nullptr;     // per-warp partials, then (single-site kernel) per-block partials
    int nfpart = 0;                    // entries k_finalize sums
    int nfw = 0;                       // per-warp entries
    int* blk_ctr = nullptr;
    double* kpart = nullptr;
    ObsRec* hist = nullptr;
    long long* step_ctr = nullptr;
    int* flag = nullptr;
    DevModel* dmodel = nullptr;
    char* stage = nullptr;
    size_t stage_bytes = 0;
    // state
    int cur = 0;
    int64_t n = 0;
    bool loaded = false;
    bool poisoned = false;
    double ndof = 0;
    long long host_step = 0;       // number of completed steps
    long long last_obs = -1;       // history index of the last evaluated time
    std::vector<int64_t> ids;
    std::vector<int32_t> comp_host;    // decomposed runs only (host-side egress merge)
    int64_t* ids_dev = nullptr;        // caller ids, input order
    double T_target = 0.0;             // NVT (A24): 0 = NVE
    int thermo_interval = 0;
    std::vector<int64_t> comp_counts;  // molecules per component (tail corrections)
    int32_t* comp_dev = nullptr;       // components, input order
    // graphs: one time step starting from buffer parity 0 / 1
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int64_t graph_n = -1;              // molecule count and N_dof the step graphs were built for
    double graph_ndof = -1.0;
    cudaEvent_t ev_f0[2] = {nullptr, nullptr}, ev_f1[2] = {nullptr, nullptr};
    cudaEvent_t ev_s0 = nullptr, ev_s1 = nullptr;      // fork / join of the graph's side branch
    cudaEvent_t ev_r[4] = {nullptr, nullptr, nullptr, nullptr};   // decomposed step: this rank's begin / end
    bool rank_timed = false;
    long long dd_glaunch = 0;              // kernel launches of this rank per replay of the group's step graph
    cudaStream_t side_stream = nullptr;
    int last_parity = 0;
    bool profiling = true;
    long long launches = 0;
    double last_total_ms = 0, last_force_ms = 0;
    int last_force_launches = 0;
    // spatial decomposition (§4): this rank's box, cell owners, halos
    Group* grp = nullptr;                  // distributed / loopback group (nullptr: one domain)
    int dd_rank = 0, nranks = 1;
    int rebalance_interval = 0;            // steps between re-partitions (0: static)
    int cost_model = 0;                    // per-cell load of the k-d tree: 0 = Eq. 6, 1 = molecule count
    long long last_rebalance = -1;         // host_step of the last re-partition
    bool seg_ready = false;                // exchange segments sized (else the next step is synchronous)
    bool n_stale = false;                  // asynchronous decomposed steps: host copy of n out of date
    bool side_join = false;                // the step's finalize runs on the side stream until end_step
    int* recv_cnt = nullptr;               // asynchronous exchange: records received per source rank (device)
    DDRec** put_rec = nullptr;             // direct puts: per destination rank, where this rank's records go
    int** put_cnt = nullptr;               //   and where its record count goes (device arrays of addresses)
    bool direct = false;
    bool polar_com = false;                // 2CLJQ with the quadrupole at the centre of mass
    bool sym_linear = false;               //   and both LJ sites on its axis (rig3 SYM)
    float hsym[2] = {0.f, 0.f};
    // NCCL groups: two receive areas (and count arrays, put tables) used by alternate steps
    // (parity = cur), so that a peer storing the next step's records never overwrites the
    // records this rank is still importing; direct puts across processes through CUDA IPC
    DDRec* recv_area[2] = {nullptr, nullptr};
    int* rcnt_area[2] = {nullptr, nullptr};
    DDRec** put_rec_area[2] = {nullptr, nullptr};
    int** put_cnt_area[2] = {nullptr, nullptr};
    char* ipc_blob = nullptr;              // device staging of the handle all-gather
    int* ipc_word = nullptr;               // the one-word all-reduce that orders puts before imports
    int* n_aux = nullptr;                  // [0] unsorted count after the import, [1] n at force time, [2] egress counter
    int64_t seg_max = 0;                   // send segment stride of the workspace layout
    int* seg_tab = nullptr;                // per-peer segments (device): send offsets, send caps, recv offsets, recv caps
    bool peer_segs = false;                // seg_tab in use (else uniform seg_cap segments)
    int64_t recv_span = 0;                 // records of the receive buffer the segments cover
    std::vector<int64_t> send_off, send_caps, recv_off, recv_caps;   // host copies of the segment layout
    std::vector<int32_t> boxes;
    std::vector<uint8_t> h_owner;
    std::vector<uint32_t> h_gmask;
    double ndof_global = -1.0;
    int64_t n_global = 0;                  // molecules of the whole system (decomposed contexts)
    uint8_t* owner = nullptr;
    uint32_t* gmask = nullptr;
    int* gcount = nullptr;                 // per-cell owned counts (rebalance)
    int64_t* cmat = nullptr;               // record-count matrix staging (NCCL allgather)
    ObsRec* obs_all = nullptr;             // allgathered observable rings (NCCL)
    DDRec* sendbuf = nullptr;
    DDRec* recvbuf = nullptr;
    int* send_cnt = nullptr;
    int64_t seg_cap = 0, recv_cap = 0;
    int64_t n_input = 0;
    int64_t n_force = 0;       // molecules (sorted slots) of the buffer the last forces belong to
    int rank_id() const { return dd_rank; }
};

// ------------------------------------------------------------------------
// helpers

static int fail(mardyn_ctx* c, int code, const std::string& msg)
{
    if (c) c->err = msg;
    return code;
}

#define CK(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            ctx->poisoned = true;                                                          \
            return fail(ctx, MARDYN_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
        }                                                                                  \
    } while (0)

// grid and fixed-point lattice, reading A12
static int grid_setup(const double L[3], double rc, double dt, GridP& g, std::string& err)
{
    int nc[3];
    for (int k = 0; k < 3; ++k) {
        nc[k] = (int)std::floor(L[k] / rc);
        if (nc[k] < 3) { err = "box must hold >= 3 cells of edge >= rc per axis"; return MARDYN_EINVAL; }
    }
    double s = 0;
    long long E[3];
    for (int it = 0; it < 4; ++it) {
        double emax = 0;
        for (int k = 0; k < 3; ++k) emax = std::fmax(emax, L[k] / nc[k]);
        int ex = (int)std::ceil(std::log2(emax));
        s = std::ldexp(1.0, ex - 22);
        bool again = false;
        for (int k = 0; k < 3; ++k) {
            E[k] = std::llround(L[k] / (nc[k] * s));
            if ((double)E[k] * s < rc) { nc[k] -= 1; again = true; }
            if (nc[k] < 3) { err = "box must hold >= 3 cells of edge >= rc per axis"; return MARDYN_EINVAL; }
        }
        if (!again) break;
    }
    std::memset(&g, 0, sizeof(g));
    long long ncell = 1;
    for (int k = 0; k < 3; ++k) {
        g.nc[k] = nc[k];
        g.E[k] = (uint32_t)E[k];
        // ceil(2^64 / E) for the multiply-high division (E >= 2, so no overflow)
        g.Einv[k] = (uint64_t)(~0ull / (uint64_t)E[k]) + 1ull;
        uint64_t P = (uint64_t)E[k] * (uint64_t)nc[k];
        if (P > (1ull << 32)) { err = "box too large for 32-bit fixed point"; return MARDYN_EINVAL; }
        g.P64[k] = P;
        g.P[k] = (uint32_t)(P & 0xffffffffu);
        g.edge[k] = (float)((double)E[k] * s);
        ncell *= nc[k];
    }
    if (ncell > (1ll << 30)) { err = "too many cells"; return MARDYN_EINVAL; }
    g.ncell = (int)ncell;
    g.s = (float)s;
    g.inv_s = (float)(1.0 / s);
    double rc2 = rc * rc;
    g.cut2 = (float)rc2;
    g.cut2_lo = std::nextafterf((float)(rc2 * (1.0 - std::ldexp(1.0, -20))), 0.f);
    g.cut2_hi = std::nextafterf((float)(rc2 * (1.0 + std::ldexp(1.0, -20))), INFINITY);
    g.band_mid = 0.5f * (g.cut2_lo + g.cut2_hi);
    g.band_hw = 0.5f * (g.cut2_hi - g.cut2_lo) + 1e-6f * g.cut2_hi;
    g.cut2_q = (long long)std::ceil(rc2 / (s * s));
    g.dt = (float)dt;
    for (int k = 0; k < 3; ++k) { g.hlo[k] = 0; g.hdim[k] = g.nc[k]; g.wlo[k] = 0; g.wn[k] = g.nc[k]; }
    g.nhome = g.ncell;
    g.wncell = g.ncell;
    return MARDYN_OK;
}

static int setup_grid(mardyn_ctx* ctx)
{
    std::string err;
    int rc = grid_setup(ctx->L, ctx->rc, ctx->dt, ctx->g, err);
    return rc ? fail(ctx, rc, err) : MARDYN_OK;
}

static int build_model(mardyn_ctx* ctx)
{
    DevModel& M = ctx->model;
    std::memset(&M, 0, sizeof(M));
    const int nc = (int)ctx->comps.size();
    M.n_comp = nc;
    const double rc = ctx->rc, rc3 = rc * rc * rc;
    double krf, kmm;
    if (std::isinf(ctx->eps_rf)) { krf = 1.0 / (2.0 * rc3); kmm = 1.0 / rc3; }
    else {
        krf = (ctx->eps_rf - 1.0) / ((2.0 * ctx->eps_rf + 1.0) * rc3);
        kmm = 2.0 * (ctx->eps_rf - 1.0) / ((2.0 * ctx->eps_rf + 1.0) * rc3);
    }
    M.krf = (float)krf;
    M.crf = (float)(1.0 / rc + krf * rc * rc);
    M.krf_mumu = (float)kmm;
    int lj_total = 0;
    std::vector<double> ljsig, ljeps;
    std::vector<int> ljcomp;
    ctx->rigid = false;
    ctx->nslots = 0;
    for (int c = 0; c < nc; ++c) {
        const HostComp& H = ctx->comps[c];
        DevComp& D = M.comp[c];
        D.mass = (float)H.mass;
        D.inv_mass = (float)(1.0 / H.mass);
        D.rot = 0;
        for (int k = 0; k < 3; ++k) {
            D.invI[k] = H.I[k] > 0 ? (float)(1.0 / H.I[k]) : 0.f;
            D.rot += H.I[k] > 0;
        }
        D.n_lj = (int)H.lj.size(); D.n_q = (int)H.q.size();
        D.n_mu = (int)H.mu.size(); D.n_Q = (int)H.Q.size();
        D.lj0 = lj_total;
        D.slot_lj = 0; D.slot_q = D.n_lj; D.slot_mu = D.n_lj + D.n_q; D.slot_Q = D.slot_mu + 2 * D.n_mu;
        D.n_slots = D.slot_Q + 2 * D.n_Q;
        ctx->nslots = std::max(ctx->nslots, D.n_slots);
        int s = 0;
        bool offcentre = false;
        for (auto& x : H.lj) {
            for (int k = 0; k < 3; ++k) { D.bpos[s][k] = (float)x.r[k]; offcentre |= x.r[k] != 0; }
            D.mom[s++] = 0.f;
            ljsig.push_back(x.sigma); ljeps.push_back(x.epsilon); ljcomp.push_back(c);
            ++lj_total;
        }
        for (auto& x : H.q) {
            for (int k = 0; k < 3; ++k) { D.bpos[s][k] = (float)x.r[k]; offcentre |= x.r[k] != 0; }
            D.mom[s++] = (float)x.q;
        }
        for (auto* lst : {&H.mu, &H.Q})
            for (auto& x : *lst) {
                double nrm = std::sqrt(x.e[0] * x.e[0] + x.e[1] * x.e[1] + x.e[2] * x.e[2]);
                for (int k = 0; k < 3; ++k) {
                    D.bpos[s][k] = (float)x.r[k];
                    D.baxis[s][k] = (float)(x.e[k] / nrm);
                }
                D.mom[s++] = (float)x.m;
                offcentre = true;
            }
        if (offcentre || D.rot > 0 || D.n_q + D.n_mu + D.n_Q > 0 || D.n_lj != 1) ctx->rigid = true;
    }
    M.n_lj_total = lj_total;
    for (int a = 0; a < lj_total; ++a)
        for (int b = 0; b < lj_total; ++b) {
            double eta = ctx->eta.empty() ? 1.0 : ctx->eta[ljcomp[a] * nc + ljcomp[b]];
            double sig = 0.5 * (ljsig[a] + ljsig[b]);          // Lorentz
            double eps = eta * std::sqrt(ljeps[a] * ljeps[b]); // Berthelot * eta
            double sc6 = std::pow(sig / rc, 6.0);
            int t = a * MD_MAX_LJ_TOTAL + b;
            M.sig2[t] = (float)(sig * sig);
            M.eps24[t] = (float)(24.0 * eps);
            M.eps4[t] = (float)(4.0 * eps);
            M.shift[t] = ctx->lj_shift ? (float)(4.0 * eps * (sc6 * sc6 - sc6)) : 0.f;
        }
    // kernel choice
    if (!ctx->rigid && nc == 1) {
        ctx->kernel = KER_LJ1;
        ctx->shape = SHAPE_NONE;
        ctx->force_warps_per_block = LJ1_WARPS;
    } else if (nc == 1 && M.comp[0].n_lj == 2 && M.comp[0].n_q == 0 && M.comp[0].n_mu == 0 && M.comp[0].n_Q == 1) {
        ctx->kernel = KER_RIGID; ctx->shape = SHAPE_2CLJQ; ctx->force_warps_per_block = RIG_WARPS;
        const float* qp = M.comp[0].bpos[M.comp[0].n_lj + M.comp[0].n_q + M.comp[0].n_mu];   // the Q site
        ctx->polar_com = qp[0] == 0.f && qp[1] == 0.f && qp[2] == 0.f && !std::getenv("MARDYN_NO_POLAR_COM");
        // linear: both LJ sites on the quadrupole axis (body positions h_b * axis exactly)
        const DevComp& C = M.comp[0];
        const int iq = C.n_lj + C.n_q + C.n_mu;
        const float* ax = C.baxis[iq];
        bool lin = ctx->polar_com && !std::getenv("MARDYN_NO_SYM");
        for (int b = 0; b < 2 && lin; ++b) {
            const float h = C.bpos[b][0] * ax[0] + C.bpos[b][1] * ax[1] + C.bpos[b][2] * ax[2];
            for (int k = 0; k < 3; ++k) lin = lin && C.bpos[b][k] == h * ax[k];
            ctx->hsym[b] = h;
        }
        ctx->sym_linear = lin;
    } else if (nc == 1 && M.comp[0].n_lj == 1 && M.comp[0].n_q == 3 && M.comp[0].n_mu == 0 && M.comp[0].n_Q == 0) {
        ctx->kernel = KER_RIGID; ctx->shape = SHAPE_TIP4P; ctx->force_warps_per_block = RIG_WARPS;
    } else {
        ctx->kernel = KER_GENERIC; ctx->shape = SHAPE_GEN; ctx->force_warps_per_block = GEN_WARPS;
        ctx->rigid = true;
    }
    if (ctx->kernel != KER_LJ1) ctx->rigid = true;
    return MARDYN_OK;
}

template <typename K>
static int occupancy_grid(mardyn_ctx* ctx, K kernel, int threads, size_t smem = 0)
{
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    return per_sm * ctx->num_sms;
}

// after asynchronous decomposed steps the molecule count is only in device
// memory (start[ncell] of the last cell rebuild): fetch it before host-side use
static int refresh_n(mardyn_ctx* ctx)
{
    if (ctx->side_join) {              // an asynchronous step's finalize still runs on the side stream
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_s1, 0));
        ctx->side_join = false;
    }
    if (!ctx->n_stale) return MARDYN_OK;
    int kept = 0, nf = 0;
    CK(cudaMemcpyAsync(&kept, ctx->start + ctx->g.wncell, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&nf, ctx->n_aux + 1, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->n = kept;
    ctx->n_force = nf;
    ctx->n_stale = false;
    return MARDYN_OK;
}


// forces at the current state of buffer `buf`; step = true (single-site
// kernel, one domain) also advances the molecules by one leapfrog step and
// bins them for the next cell rebuild (count must be zeroed before)
static int launch_force(mardyn_ctx* ctx, int buf, bool step = false, bool in_graph = false,
                        const DDArgs* dd = nullptr)
{
    ctx->n_force = ctx->n;
    ForceArgs a;
    a.g = ctx->g;
    a.n = (int)ctx->n;
    a.cap = (int)ctx->cap;
    a.start = ctx->start;
    a.xs = ctx->xs;
    a.site = ctx->site;
    a.force = ctx->force;
    a.torque = ctx->torque;
    a.part = ctx->fpart;
    a.flag = ctx->flag;
    a.model = ctx->dmodel;
    const DevComp& C0 = ctx->model.comp[0];
    (void)C0;
    a.sig2 = ctx->model.sig2[0];
    a.eps24 = ctx->model.eps24[0];
    a.eps4 = ctx->model.eps4[0];
    a.shift = ctx->model.shift[0];
    for (int ia = 0; ia < 2; ++ia)
        for (int ib = 0; ib < 2; ++ib) {
            const int t = ia * MD_MAX_LJ_TOTAL + ib;
            a.lj3[2 * ia + ib] = make_float4(ctx->model.sig2[t], ctx->model.eps24[t], ctx->model.eps4[t],
                                             ctx->model.shift[t]);
        }
    a.krf = ctx->model.krf;
    a.crf = ctx->model.crf;
    a.kmm = ctx->model.krf_mumu;
    a.hsym[0] = ctx->hsym[0];
    a.hsym[1] = ctx->hsym[1];
    const int threads = 32 * ctx->force_warps_per_block;
    switch (ctx->shape) {
    case SHAPE_2CLJQ:
        if (ctx->sym_linear)
            rig3::k_force_rigid3<2, 0, 0, 1, true, true><<<ctx->force_grid, threads, rig3::smem_bytes<2, 0, 0, 1>(), ctx->stream>>>(a);
        else if (ctx->polar_com)
            rig3::k_force_rigid3<2, 0, 0, 1, true><<<ctx->force_grid, threads, rig3::smem_bytes<2, 0, 0, 1>(), ctx->stream>>>(a);
        else
            rig3::k_force_rigid3<2, 0, 0, 1><<<ctx->force_grid, threads, rig3::smem_bytes<2, 0, 0, 1>(), ctx->stream>>>(a);
        break;
    case SHAPE_TIP4P:
        rig3::k_force_rigid3<1, 3, 0, 0><<<ctx->force_grid, threads, rig3::smem_bytes<1, 3, 0, 0>(), ctx->stream>>>(a);
        break;
    case SHAPE_GEN:
        k_force_rigid<4, 4, 2, 2, true, GEN_WARPS>
            <<<ctx->force_grid, threads, rigid_smem<4, 4, 2, 2, GEN_WARPS>(), ctx->stream>>>(a);
        break;
    default: {
        lj1::Args b;
        b.g = ctx->g;
        b.start = ctx->start;
        b.pos = ctx->pos[buf];
        b.xs = ctx->xs;
        b.force = ctx->force;
        b.part = ctx->fpart;
        b.bpart = ctx->fpart + ctx->nfw;
        b.nbcap = ctx->nfpart - ctx->nfw;
        b.ctr = ctx->blk_ctr;
        // the block counter is zero whenever no force kernel runs (the scan resets it after a
        // step); calls outside the step graph restore that invariant themselves
        if (!in_graph) CK(cudaMemsetAsync(ctx->blk_ctr, 0, sizeof(int), ctx->stream));
        b.sig2 = a.sig2; b.eps24 = a.eps24; b.eps4 = a.eps4; b.shift = a.shift;
        b.vel = ctx->vel[buf];
        b.cell_of = ctx->cell_of;
        b.rank = ctx->rank;
        b.count = ctx->count;
        b.flag = ctx->flag;
        b.mass = ctx->model.comp[0].mass;
        b.inv_mass = ctx->model.comp[0].inv_mass;
        if (step && dd) {
            b.dd = *dd;
            K_LJ1_STEP_DD<<<ctx->force_grid, threads, LJ1::SMEM, ctx->stream>>>(b);
        } else if (step) {
            K_LJ1_STEP<<<ctx->force_grid, threads, LJ1::SMEM, ctx->stream>>>(b);
        } else {
            K_LJ1<<<ctx->force_grid, threads, LJ1::SMEM, ctx->stream>>>(b);
        }
        if (!in_graph) CK(cudaMemsetAsync(ctx->blk_ctr, 0, sizeof(int), ctx->stream));
    }
    }
    ctx->launches += 1;
    return MARDYN_OK;
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// counting sort of the unsorted buffer `src` (cell_of / rank / count
// filled) into buffer `dst`, canonical in-cell order (A13)
// n_dev: the unsorted count is in device memory (asynchronous decomposed step;
// the grids then cover the capacity)
static int enqueue_sort(mardyn_ctx* ctx, int src, int dst, int64_t n_unsorted = -1, const int* n_dev = nullptr)
{
    // the scan covers the rank-local cell window (the whole grid for one domain)
    const int n = n_dev ? (int)ctx->cap : (int)(n_unsorted < 0 ? ctx->n : n_unsorted), ncell = ctx->g.wncell;
    // count known on the host: one thread per molecule; in device memory only: a grid-stride
    // grid of 8 blocks per SM (independent of the capacity)
    const int gb = n_dev ? std::min(nblk(n, 256), 8 * ctx->num_sms) : nblk(n, 256);
    cudaStream_t s = ctx->stream;
    // (look-back flags carry an epoch, counts are zeroed as read: no memsets per step)
    if (ncell >= SCAN_BIG_GRID)
        k_scan<16><<<(ncell + 16383) / 16384, 1024, 0, s>>>(ncell, ctx->count, ctx->start, ctx->scan_flags,
                                                           reinterpret_cast<unsigned*>(ctx->scan_flags + ctx->ntiles),
                                                           ctx->blk_ctr);
    else
        k_scan<SCAN_PT_SMALL><<<(ncell + 1024 * SCAN_PT_SMALL - 1) / (1024 * SCAN_PT_SMALL), 1024, 0, s>>>(ncell, ctx->count, ctx->start, ctx->scan_flags,
                                                        reinterpret_cast<unsigned*>(ctx->scan_flags + ctx->ntiles),
                                                        ctx->blk_ctr);
    k_scatter<<<gb, 256, 0, s>>>(n, ctx->pos[src], ctx->cell_of, ctx->rank, ctx->start, ctx->keys,
                                            ctx->oldidx, ctx->oldidx + ctx->cap, n_dev);
    if (ctx->rigid)
        k_canon<true><<<gb, 256, 0, s>>>(n, (int)ctx->cap, ctx->g, ctx->keys, ctx->oldidx, ctx->oldidx + ctx->cap, ctx->start,
                                                   ctx->pos[src], ctx->vel[src], ctx->quat[src], ctx->angm[src],
                                                   ctx->pos[dst], ctx->vel[dst], ctx->quat[dst], ctx->angm[dst],
                                                   ctx->xs, ctx->site, ctx->dmodel);
    else
        k_canon<false><<<gb, 256, 0, s>>>(n, (int)ctx->cap, ctx->g, ctx->keys, ctx->oldidx, ctx->oldidx + ctx->cap, ctx->start,
                                                    ctx->pos[src], ctx->vel[src], nullptr, nullptr,
                                                    ctx->pos[dst], ctx->vel[dst], nullptr, nullptr, ctx->xs,
                                                    nullptr, ctx->dmodel);
    ctx->launches += 3;      // scan, scatter, canon
    return MARDYN_OK;
}

// one time step from buffer parity b (A23): forces at t_k, observables of
// t_k, leapfrog + rotation, cell rebuild into parity 1-b
// NVT (reading A24): rescale the half-step velocities of buffer b after the
// finalize of the step (the kernel checks the cadence on the device)
static void enqueue_thermostat(mardyn_ctx* ctx, int b)
{
    if (!(ctx->T_target > 0) || ctx->thermo_interval < 1) return;
    const int n = (int)ctx->n;
    k_rescale<<<nblk(n, 256), 256, 0, ctx->stream>>>(n, ctx->vel[b], ctx->rigid ? ctx->angm[b] : nullptr, ctx->hist,
                                                     ctx->step_ctr, ctx->T_target, ctx->thermo_interval, ctx->flag);
    ctx->launches += 1;
}

static int enqueue_step(mardyn_ctx* ctx, int b, bool timing_events)
{
    cudaStream_t s = ctx->stream;
    const int n = (int)ctx->n;
    const bool fused = ctx->kernel == KER_LJ1 && ctx->nranks == 1;
    // the cell counts are zero here: the previous rebuild's scan cleared them
    if (timing_events) CK(cudaEventRecordWithFlags(ctx->ev_f0[b], s, cudaEventRecordExternal));
    launch_force(ctx, b, fused, true);
    if (timing_events) CK(cudaEventRecordWithFlags(ctx->ev_f1[b], s, cudaEventRecordExternal));
    if (fused) {
        // the single-site kernel has advanced and binned the molecules (kinetic energy in its
        // partials).  Without NVT the observables do not feed the cell rebuild: the finalize
        // runs on a side branch of the graph, concurrently with scan / scatter / canon.
        const bool side = !(ctx->T_target > 0 && ctx->thermo_interval > 0) && ctx->side_stream;
        cudaStream_t fs = side ? ctx->side_stream : s;
        if (side) {
            CK(cudaEventRecord(ctx->ev_s0, s));
            CK(cudaStreamWaitEvent(fs, ctx->ev_s0, 0));
        }
        k_finalize<<<FIN_BLOCKS, FIN_THREADS, 0, fs>>>(ctx->nfpart, ctx->fpart, 0, ctx->kpart, ctx->ndof,
                                                       ctx->step_ctr, 1, ctx->hist, ctx->fin_scratch, ctx->fin_ticket);
        ctx->launches += 1;
        enqueue_thermostat(ctx, b);
        const int rc = enqueue_sort(ctx, b, 1 - b);
        if (side) {                          // join: the next step's force rewrites the partials
            CK(cudaEventRecord(ctx->ev_s1, fs));
            CK(cudaStreamWaitEvent(s, ctx->ev_s1, 0));
        }
        return rc;
    }
    if (ctx->rigid)
        k_integrate<true><<<ctx->nkblocks, 256, 0, s>>>(n, ctx->g, ctx->dmodel, ctx->pos[b], ctx->vel[b],
                                                        ctx->quat[b], ctx->angm[b], ctx->force, ctx->torque,
                                                        ctx->cell_of, ctx->rank, ctx->count, ctx->kpart, ctx->flag);
    else
        k_integrate<false><<<ctx->nkblocks, 256, 0, s>>>(n, ctx->g, ctx->dmodel, ctx->pos[b], ctx->vel[b],
                                                         nullptr, nullptr, ctx->force, ctx->torque, ctx->cell_of,
                                                         ctx->rank, ctx->count, ctx->kpart, ctx->flag);
    k_finalize<<<FIN_BLOCKS, FIN_THREADS, 0, s>>>(ctx->nfpart, ctx->fpart, ctx->nkblocks, ctx->kpart, ctx->ndof,
                                                  ctx->step_ctr, 1, ctx->hist, ctx->fin_scratch, ctx->fin_ticket);
    ctx->launches += 2;
    enqueue_thermostat(ctx, b);
    return enqueue_sort(ctx, b, 1 - b);
}

static int build_graphs(mardyn_ctx* ctx)
{
    for (int b = 0; b < 2; ++b) {
        if (ctx->gexec[b]) { cudaGraphExecDestroy(ctx->gexec[b]); ctx->gexec[b] = nullptr; }
        cudaGraph_t graph;
        long long l0 = ctx->launches;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_step(ctx, b, ctx->profiling);
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
        ctx->launches = l0;   // captured launches are counted at replay
        if (rc != MARDYN_OK) return rc;
        CK(e);
        CK(cudaGraphInstantiate(&ctx->gexec[b], graph, 0));
        CK(cudaGraphDestroy(graph));
    }
    return MARDYN_OK;
}

static int launches_per_step(const mardyn_ctx* ctx)
{   // force (+ integrate unless fused), finalize, (rescale,) scan, scatter, canon
    return ((ctx->kernel == KER_LJ1 && ctx->nranks == 1) ? 5 : 6) +
           ((ctx->T_target > 0 && ctx->thermo_interval > 0) ? 1 : 0);
}

// ------------------------------------------------------------------------
// C ABI

extern "C" {

int mardyn_create(const double box[3], double cutoff, const mardyn_component* comps, int32_t n_comps,
                  const mardyn_options* opt, mardyn_ctx** out)
{
    if (!out) return MARDYN_EINVAL;
    *out = nullptr;
    mardyn_ctx* ctx = new mardyn_ctx();
    auto bad = [&](const char* m) { ctx->err = m; return MARDYN_EINVAL; };
    if (!box || !comps || n_comps < 1 || n_comps > MD_MAX_COMP || !opt) {
        *out = ctx;
        return bad("invalid arguments (box, components 1..8, options required)");
    }
    *out = ctx;
    if (!(cutoff > 0)) return bad("cutoff must be > 0");
    if (!(opt->dt > 0)) return bad("dt must be > 0");
    if (!(opt->eps_rf >= 1.0)) return bad("eps_rf must be >= 1 (INFINITY allowed)");
    for (int k = 0; k < 3; ++k) {
        if (!(box[k] > 0) || !std::isfinite(box[k])) return bad("box must be positive and finite");
        ctx->L[k] = box[k];
    }
    ctx->rc = cutoff;
    ctx->dt = opt->dt;
    ctx->eps_rf = opt->eps_rf;
    ctx->lj_shift = opt->lj_shift;
    if (opt->rebalance_interval < 0) return bad("rebalance_interval must be >= 0");
    ctx->rebalance_interval = opt->rebalance_interval;
    int lj_total = 0;
    for (int c = 0; c < n_comps; ++c) {
        const mardyn_component& C = comps[c];
        if (C.n_lj < 0 || C.n_q < 0 || C.n_mu < 0 || C.n_Q < 0) return bad("negative site count");
        if (C.n_lj > 4 || C.n_q > 4 || C.n_mu > 2 || C.n_Q > 2)
            return bad("component limits: <= 4 LJ sites, <= 4 charges, <= 2 dipoles, <= 2 quadrupoles");
        if (C.n_lj + C.n_q + C.n_mu + C.n_Q == 0) return bad("component without sites");
        if (!(C.mass > 0)) return bad("mass must be > 0");
        for (int k = 0; k < 3; ++k) if (!(C.inertia[k] >= 0)) return bad("inertia must be >= 0");
        HostComp H;
        H.mass = C.mass;
        for (int k = 0; k < 3; ++k) H.I[k] = C.inertia[k];
        if ((C.n_lj && !C.lj) || (C.n_q && !C.q) || (C.n_mu && !C.mu) || (C.n_Q && !C.Q))
            return bad("null site array");
        H.lj.assign(C.lj, C.lj + C.n_lj);
        H.q.assign(C.q, C.q + C.n_q);
        H.mu.assign(C.mu, C.mu + C.n_mu);
        H.Q.assign(C.Q, C.Q + C.n_Q);
        for (auto& x : H.lj) if (!(x.sigma > 0) || !(x.epsilon >= 0)) return bad("LJ sigma > 0, epsilon >= 0");
        for (auto* lst : {&H.mu, &H.Q})
            for (auto& x : *lst)
                if (!(std::fabs(x.e[0] * x.e[0] + x.e[1] * x.e[1] + x.e[2] * x.e[2] - 1.0) < 1e-6))
                    return bad("polar site axis must be a unit vector");
        lj_total += C.n_lj;
        ctx->comps.push_back(H);
    }
    if (lj_total > MD_MAX_LJ_TOTAL) return bad("more than 16 LJ sites over all components");
    if (opt->eta) {
        ctx->eta.assign(opt->eta, opt->eta + n_comps * n_comps);
        for (double e : ctx->eta) if (!(e > 0)) return bad("eta must be > 0");
    }
    int rc = setup_grid(ctx);
    if (rc) return rc;
    rc = build_model(ctx);
    if (rc) return rc;
    CK(cudaGetDevice(&ctx->device));
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    if (opt->cuda_stream) {
        ctx->stream = (cudaStream_t)opt->cuda_stream;
    } else {
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    int threads = 32 * ctx->force_warps_per_block;
    switch (ctx->shape) {
    case SHAPE_2CLJQ: {
        auto k = ctx->sym_linear ? rig3::k_force_rigid3<2, 0, 0, 1, true, true>
                 : ctx->polar_com ? rig3::k_force_rigid3<2, 0, 0, 1, true> : rig3::k_force_rigid3<2, 0, 0, 1>;
        const int sm = rig3::smem_bytes<2, 0, 0, 1>();
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        ctx->force_blocks = occupancy_grid(ctx, k, threads, sm);
        break;
    }
    case SHAPE_TIP4P: {
        auto k = rig3::k_force_rigid3<1, 3, 0, 0>;
        const int sm = rig3::smem_bytes<1, 3, 0, 0>();
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        ctx->force_blocks = occupancy_grid(ctx, k, threads, sm);
        break;
    }
    case SHAPE_GEN: {
        auto k = k_force_rigid<4, 4, 2, 2, true, GEN_WARPS>;
        const int sm = rigid_smem<4, 4, 2, 2, GEN_WARPS>();
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        ctx->force_blocks = occupancy_grid(ctx, k, threads, sm);
        break;
    }
    default:
        CK(cudaFuncSetAttribute(K_LJ1, cudaFuncAttributeMaxDynamicSharedMemorySize, LJ1::SMEM));
        CK(cudaFuncSetAttribute(K_LJ1_STEP, cudaFuncAttributeMaxDynamicSharedMemorySize, LJ1::SMEM));
        CK(cudaFuncSetAttribute(K_LJ1_STEP_DD, cudaFuncAttributeMaxDynamicSharedMemorySize, LJ1::SMEM));
        ctx->force_blocks = occupancy_grid(ctx, K_LJ1, threads, LJ1::SMEM);
    }
    for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreate(&ctx->ev_f0[b]));
        CK(cudaEventCreate(&ctx->ev_f1[b]));
    }
    for (int k = 0; k < 4; ++k) CK(cudaEventCreate(&ctx->ev_r[k]));
    CK(cudaEventCreateWithFlags(&ctx->ev_s0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_s1, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
    return MARDYN_OK;
}

int mardyn_get_grid(const mardyn_ctx* ctx, mardyn_grid* out)
{
    if (!ctx || !out) return MARDYN_EINVAL;
    const GridP& g = ctx->g;
    for (int k = 0; k < 3; ++k) {
        out->ncell[k] = g.nc[k];
        out->period[k] = (int64_t)g.P64[k];
        out->edge[k] = g.E[k];
        out->box[k] = (double)g.P64[k] * (double)g.s;
    }
    out->pad = 0;
    out->quantum = (double)g.s;
    out->cut2_q = g.cut2_q;
    out->kernel = ctx->kernel;
    out->n_slots = ctx->nslots;
    return MARDYN_OK;
}

static size_t layout(mardyn_ctx* ctx, int64_t cap, bool assign)
{
    const size_t A = 256;
    size_t off = 0;
    char* base = ctx->ws;
    auto take = [&](size_t bytes) -> char* {
        char* p = assign ? base + off : nullptr;
        off = align_up(off + bytes, A);
        return p;
    };
    const int ncell = ctx->g.ncell;
    const int ncell_pad = (int)align_up((size_t)ncell, SCAN_TILE);
    const int ntiles = ncell_pad / (1024 * SCAN_PT_SMALL);   // look-back flags: enough for the smallest tiles
    const int nk = std::max(1, nblk(cap, 256));
    const int nfw = std::max(1, ctx->force_blocks * ctx->force_warps_per_block);
    // single-site kernel: one partial per block -- blocks of 32, or (small systems) half blocks
    // of 16 (k_force_lj1: MD_LJ1_HALF)
    const int nbc = ctx->kernel == KER_LJ1 ? nblk(cap, 32) + 1 + MD_LJ1_HALF * nfw : 0;
    uint4* pos0 = (uint4*)take(16 * cap);
    uint4* pos1 = (uint4*)take(16 * cap);
    float4* vel0 = (float4*)take(16 * cap);
    float4* vel1 = (float4*)take(16 * cap);
    float4 *q0 = nullptr, *q1 = nullptr, *j0 = nullptr, *j1 = nullptr, *site = nullptr, *tq = nullptr;
    if (ctx->rigid) {
        q0 = (float4*)take(16 * cap); q1 = (float4*)take(16 * cap);
        j0 = (float4*)take(16 * cap); j1 = (float4*)take(16 * cap);
        site = (float4*)take((size_t)16 * cap * std::max(1, ctx->nslots));
        tq = (float4*)take(16 * cap);
    }
    float4* xs = (float4*)take(16 * cap);
    float4* force = (float4*)take(16 * cap);
    int* cell_of = (int*)take(4 * cap);
    int* rank = (int*)take(4 * cap);
    unsigned long long* keys = (unsigned long long*)take(8 * cap);
    int* oldidx = (int*)take(8 * cap);               // [0, cap) unsorted index, [cap, 2 cap) cell of the slot
    int* count = (int*)take(4 * (size_t)ncell_pad);
    int* start = (int*)take(4 * ((size_t)ncell + 1));
    unsigned long long* scan_flags = (unsigned long long*)take(8 * (size_t)(std::max(ntiles, 1) + 1));
    FinPart* fin_scratch = (FinPart*)take(sizeof(FinPart) * FIN_BLOCKS);
    int* fin_ticket = (int*)take(sizeof(int));
    ForcePartial* fpart = (ForcePartial*)take(sizeof(ForcePartial) * (nfw + nbc));
    int* blk_ctr = (int*)take(sizeof(int));
    double* kpart = (double*)take(16 * (size_t)nk);
    ObsRec* hist = (ObsRec*)take(sizeof(ObsRec) * MD_HISTORY);
    long long* step_ctr = (long long*)take(8);
    int* flag = (int*)take(4);
    DevModel* dmodel = (DevModel*)take(sizeof(DevModel));
    const size_t stage_bytes = (size_t)cap * (24 * 8);   // ingest chunks (108 B), egress (<= 184 B)
    char* stage = take(stage_bytes);
    int64_t* ids_dev = (int64_t*)take(8 * (size_t)cap);
    int32_t* comp_dev = (int32_t*)take(4 * (size_t)cap);
    uint8_t* owner = nullptr;
    uint32_t* gmask = nullptr;
    int* gcount = nullptr;
    int64_t* cmat = nullptr;
    ObsRec* obs_all = nullptr;
    DDRec *sendbuf = nullptr, *recvbuf = nullptr;
    int* send_cnt = nullptr;
    int* recv_cnt = nullptr;
    int* n_aux = nullptr;
    int* seg_tab = nullptr;
    DDRec** put_rec = nullptr;
    int** put_cnt = nullptr;
    char* ipc_blob = nullptr;
    int* ipc_word = nullptr;
    const bool two_areas = ctx->nranks > 1 && ctx->grp && group_is_nccl(ctx->grp);
    const int nar = two_areas ? 2 : 1;
    const int64_t seg_cap = ctx->nranks > 1 ? cap / ctx->nranks + 4096 : 0;
    const int64_t recv_cap = ctx->nranks > 1 ? cap : 0;
    if (ctx->nranks > 1) {
        owner = (uint8_t*)take((size_t)ncell);
        gmask = (uint32_t*)take(4 * (size_t)ncell);
        gcount = (int*)take(4 * (size_t)ncell);
        cmat = (int64_t*)take(8 * ((size_t)ctx->nranks * (ctx->nranks + 1) + 2));   // + group_agree's flag
        sendbuf = (DDRec*)take(sizeof(DDRec) * (size_t)seg_cap * ctx->nranks);
        recvbuf = (DDRec*)take(sizeof(DDRec) * (size_t)recv_cap * nar);
        send_cnt = (int*)take(4 * (size_t)ctx->nranks);
        recv_cnt = (int*)take(4 * (size_t)ctx->nranks * nar);
        n_aux = (int*)take(16);                    // [0] unsorted count after import, [1] n at force time, [2] egress
        seg_tab = (int*)take(16 * (size_t)ctx->nranks);
        put_rec = (DDRec**)take(sizeof(void*) * (size_t)ctx->nranks * nar);
        put_cnt = (int**)take(sizeof(void*) * (size_t)ctx->nranks * nar);
        if (two_areas) {
            ipc_blob = take(ipc_blob_bytes(ctx->nranks) * (size_t)ctx->nranks);
            ipc_word = (int*)take(4);
        }
    }
    if (ctx->grp && group_is_nccl(ctx->grp))
        obs_all = (ObsRec*)take(sizeof(ObsRec) * MD_HISTORY * (size_t)ctx->nranks);
    if (assign) {
        ctx->pos[0] = pos0; ctx->pos[1] = pos1; ctx->vel[0] = vel0; ctx->vel[1] = vel1;
        ctx->quat[0] = q0; ctx->quat[1] = q1; ctx->angm[0] = j0; ctx->angm[1] = j1;
        ctx->site = site; ctx->torque = tq; ctx->xs = xs; ctx->force = force;
        ctx->cell_of = cell_of; ctx->rank = rank; ctx->keys = keys; ctx->oldidx = oldidx; ctx->count = count;
        ctx->start = start; ctx->scan_flags = scan_flags; ctx->fin_scratch = fin_scratch; ctx->fin_ticket = fin_ticket; ctx->fpart = fpart; ctx->kpart = kpart;
        ctx->nfw = nfw; ctx->nfpart = nfw + nbc; ctx->blk_ctr = blk_ctr;
        ctx->hist = hist; ctx->step_ctr = step_ctr; ctx->flag = flag; ctx->dmodel = dmodel;
        ctx->stage = stage; ctx->stage_bytes = stage_bytes;
        ctx->ids_dev = ids_dev; ctx->comp_dev = comp_dev;
        ctx->owner = owner; ctx->gmask = gmask; ctx->gcount = gcount; ctx->cmat = cmat; ctx->obs_all = obs_all;
        ctx->sendbuf = sendbuf;
        ctx->recvbuf = recvbuf; ctx->send_cnt = send_cnt; ctx->seg_cap = seg_cap; ctx->recv_cap = recv_cap;
        ctx->recv_cnt = recv_cnt; ctx->n_aux = n_aux; ctx->seg_max = seg_cap; ctx->n_stale = false;
        ctx->seg_ready = false;
        ctx->seg_tab = seg_tab; ctx->peer_segs = false;
        ctx->put_rec = put_rec; ctx->put_cnt = put_cnt; ctx->direct = false;
        for (int q = 0; q < 2; ++q) {
            const int a = q < nar ? q : 0;
            ctx->recv_area[q] = recvbuf ? recvbuf + (size_t)a * recv_cap : nullptr;
            ctx->rcnt_area[q] = recv_cnt ? recv_cnt + (size_t)a * ctx->nranks : nullptr;
            ctx->put_rec_area[q] = put_rec ? put_rec + (size_t)a * ctx->nranks : nullptr;
            ctx->put_cnt_area[q] = put_cnt ? put_cnt + (size_t)a * ctx->nranks : nullptr;
        }
        ctx->ipc_blob = ipc_blob; ctx->ipc_word = ipc_word;
        ctx->ncell_pad = ncell_pad; ctx->ntiles = ntiles; ctx->nkblocks = nk;
    }
    return off;
}

int mardyn_workspace_bytes(mardyn_ctx* ctx, int64_t n_capacity, size_t* bytes)
{
    if (!ctx || !bytes || n_capacity < 1 || n_capacity > (1ll << 28)) return fail(ctx, MARDYN_EINVAL, "bad capacity");
    *bytes = layout(ctx, n_capacity, false);
    return MARDYN_OK;
}

int mardyn_set_workspace(mardyn_ctx* ctx, void* device_ptr, size_t bytes, int64_t n_capacity)
{
    if (!ctx || !device_ptr || n_capacity < 1) return fail(ctx, MARDYN_EINVAL, "bad workspace");
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (((uintptr_t)device_ptr) % 256) return fail(ctx, MARDYN_EINVAL, "workspace must be 256-byte aligned");
    size_t need = layout(ctx, n_capacity, false);
    if (bytes < need) return fail(ctx, MARDYN_ECAPACITY, "workspace too small");
    ctx->ws = (char*)device_ptr;
    ctx->ws_bytes = bytes;
    ctx->cap = n_capacity;
    layout(ctx, n_capacity, true);
    ctx->loaded = false;
    CK(cudaMemcpyAsync(ctx->dmodel, &ctx->model, sizeof(DevModel), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->step_ctr, 0, 8, ctx->stream));
    CK(cudaMemsetAsync(ctx->flag, 0, 4, ctx->stream));
    CK(cudaMemsetAsync(ctx->fin_ticket, 0, 4, ctx->stream));
    CK(cudaMemsetAsync(ctx->scan_flags, 0, sizeof(unsigned long long) * (ctx->ntiles + 1), ctx->stream));
    CK(cudaMemsetAsync(ctx->count, 0, sizeof(int) * ctx->ncell_pad, ctx->stream));
    if (ctx->blk_ctr) CK(cudaMemsetAsync(ctx->blk_ctr, 0, sizeof(int), ctx->stream));
    CK(cudaMemsetAsync(ctx->hist, 0, sizeof(ObsRec) * MD_HISTORY, ctx->stream));
    if (ctx->nranks > 1 && !ctx->h_owner.empty()) {
        CK(cudaMemcpyAsync(ctx->owner, ctx->h_owner.data(), ctx->g.ncell, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->gmask, ctx->h_gmask.data(), 4 * (size_t)ctx->g.ncell, cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    for (int b = 0; b < 2; ++b)
        if (ctx->gexec[b]) { cudaGraphExecDestroy(ctx->gexec[b]); ctx->gexec[b] = nullptr; }
    return MARDYN_OK;
}

int mardyn_set_molecules(mardyn_ctx* ctx, int64_t n, const int64_t* id, const int32_t* comp, const double* r,
                         const double* v, const double* q, const double* j, int32_t half_step)
{
    NvtxRange nvtx_range("mardyn_set_molecules");
    if (!ctx) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (!ctx->ws) return fail(ctx, MARDYN_ESTATE, "set_workspace must precede set_molecules");
    if (ctx->nranks > 1) return set_molecules_dd(ctx, n, id, comp, r, v, q, j, half_step);
    if (n < 1 || n > ctx->cap) return fail(ctx, MARDYN_EINVAL, "n must be in [1, capacity]");
    if (!comp || !r || !v) return fail(ctx, MARDYN_EINVAL, "comp, r, v are required");
    if (ctx->rigid && (!q || !j)) return fail(ctx, MARDYN_EINVAL, "q and j are required for rigid molecules");
    const int ncomp = (int)ctx->comps.size();
    // per-molecule validation runs on the device (k_ingest); the host keeps copies of
    // ids and components only for the decomposed egress
    ctx->n = n;
    ctx->n_stale = false;
    ctx->comp_counts.assign(ncomp, 0);
    if (ncomp == 1) ctx->comp_counts[0] = n;
    else
        for (int64_t i = 0; i < n; ++i)
            if (comp[i] >= 0 && comp[i] < ncomp) ctx->comp_counts[comp[i]] += 1;
    double ndof = 3.0 * n;
    if (ctx->rigid) {
        if (ncomp == 1) ndof += (double)ctx->model.comp[0].rot * n;
        else
            for (int64_t i = 0; i < n; ++i)
                if (comp[i] >= 0 && comp[i] < ncomp) ndof += ctx->model.comp[comp[i]].rot;
    }
    ctx->ndof = ndof;
    ctx->n_input = n;
    cudaStream_t s = ctx->stream;
    // launched force grid: the occupancy grid, or (one domain) just enough CTAs for a
    // small system -- 1 warp per 32-molecule block (single-site kernel) or per home cell
    // (rigid kernels); the per-warp partials of warps not launched stay zero
    {
        int grid = ctx->force_blocks;
        if (ctx->nranks == 1) {
            // (single-site: half blocks of 16 when there are fewer 32-blocks than warps)
            const int64_t units = ctx->kernel == KER_LJ1 ? (n + 15) / 16 : (int64_t)ctx->g.nhome;
            const int upb = ctx->kernel == KER_RIGID ? 1 : ctx->force_warps_per_block;   // rig3: CTA per cell
            const int64_t need = (units + upb - 1) / upb;
            grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, need));
        }
        const bool regraph = grid != ctx->force_grid || n != ctx->graph_n || ndof != ctx->graph_ndof;
        if (grid != ctx->force_grid) {
            ctx->force_grid = grid;
            CK(cudaMemsetAsync(ctx->fpart, 0, sizeof(ForcePartial) * ctx->nfpart, s));
        }
        ctx->graph_n = n;
        ctx->graph_ndof = ndof;
        // the step graphs hold the launch shape, the molecule count n and N_dof: rebuilt when a
        // reload changes them (a graph of another n would scatter stale or too few molecules)
        if (regraph)
            for (int b = 0; b < 2; ++b)
                if (ctx->gexec[b]) { cudaGraphExecDestroy(ctx->gexec[b]); ctx->gexec[b] = nullptr; }
    }
    // host -> device (the caller's buffers; pinned ones are DMA'd directly)
    double* dr = (double*)ctx->stage;
    double* dv = dr + 3 * n;
    double* dq = dv + 3 * n;
    double* dj = dq + 4 * n;
    CK(cudaMemcpyAsync(dr, r, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dv, v, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    if (ctx->rigid) {
        CK(cudaMemcpyAsync(dq, q, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dj, j, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemcpyAsync(ctx->comp_dev, comp, sizeof(int) * n, cudaMemcpyHostToDevice, s));
    if (id) CK(cudaMemcpyAsync(ctx->ids_dev, id, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    else k_iota64<<<nblk(n, 256), 256, 0, s>>>((int)n, ctx->ids_dev);
    CK(cudaMemsetAsync(ctx->count, 0, sizeof(int) * ctx->ncell_pad, s));
    CK(cudaMemsetAsync(ctx->flag, 0, 4, s));
    const int src = 1, dst = 0;
    k_ingest<<<nblk(n, 256), 256, 0, s>>>((int)n, dr, dv, ctx->rigid ? dq : nullptr, ctx->rigid ? dj : nullptr,
                                           ctx->comp_dev, ctx->g, ctx->pos[src], ctx->vel[src],
                                           ctx->rigid ? ctx->quat[src] : nullptr,
                                           ctx->rigid ? ctx->angm[src] : nullptr, ctx->cell_of, ctx->rank, ctx->count,
                                           ncomp, ctx->flag);
    ctx->launches += 1;
    int rc = enqueue_sort(ctx, src, dst, n);
    if (rc) return rc;
    CK(cudaGetLastError());
    ctx->cur = dst;
    long long step = ctx->host_step;
    CK(cudaMemcpyAsync(ctx->step_ctr, &step, 8, cudaMemcpyHostToDevice, s));
    if (!half_step) {   // A8: backward half kick with F(t0), tau(t0) of the molecules kept (ctx->n)
        launch_force(ctx, ctx->cur);
        const int nk = (int)ctx->n;
        if (ctx->rigid)
            k_half_kick<true><<<nblk(nk, 256), 256, 0, s>>>(nk, ctx->g, ctx->dmodel, ctx->vel[ctx->cur],
                                                            ctx->angm[ctx->cur], ctx->force, ctx->torque);
        else
            k_half_kick<false><<<nblk(nk, 256), 256, 0, s>>>(nk, ctx->g, ctx->dmodel, ctx->vel[ctx->cur],
                                                             nullptr, ctx->force, nullptr);
        ctx->launches += 1;
    }
    CK(cudaGetLastError());
    int hflag = 0;
    CK(cudaMemcpyAsync(&hflag, ctx->flag, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hflag & 512) {
        ctx->loaded = false;
        CK(cudaMemsetAsync(ctx->flag, 0, 4, s));
        return fail(ctx, MARDYN_EINVAL, "invalid input: non-finite position or velocity, component id out of "
                                        "range, or non-unit quaternion");
    }
    ctx->loaded = true;
    ctx->last_obs = -1;
    return MARDYN_OK;
}

int mardyn_compute_forces(mardyn_ctx* ctx)
{
    NvtxRange nvtx_range("mardyn_compute_forces");
    if (!ctx) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (ctx->grp && ctx->nranks > 1) return group_compute_forces(ctx);
    if (!ctx->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules first");
    return compute_forces_local(ctx);
}

}  // extern "C"

static int compute_forces_local(mardyn_ctx* ctx)
{
    if (int rc0 = refresh_n(ctx)) return rc0;
    cudaStream_t s = ctx->stream;
    const int n = (int)ctx->n, b = ctx->cur;
    launch_force(ctx, b);
    if (ctx->rigid)
        k_kinetic<true><<<ctx->nkblocks, 256, 0, s>>>(n, ctx->g, ctx->dmodel, ctx->vel[b], ctx->quat[b], ctx->angm[b],
                                                      ctx->force, ctx->torque, ctx->kpart);
    else
        k_kinetic<false><<<ctx->nkblocks, 256, 0, s>>>(n, ctx->g, ctx->dmodel, ctx->vel[b], nullptr, nullptr,
                                                       ctx->force, nullptr, ctx->kpart);
    // kpart beyond the used blocks stays from earlier steps: same block count
    k_finalize<<<FIN_BLOCKS, FIN_THREADS, 0, s>>>(ctx->nfpart, ctx->fpart, ctx->nkblocks, ctx->kpart, ctx->ndof,
                                                  ctx->step_ctr, 0, ctx->hist, ctx->fin_scratch, ctx->fin_ticket,
                                                  ctx->nranks > 1 ? 0 : 1);
    ctx->launches += 3;
    CK(cudaGetLastError());
    ctx->last_obs = ctx->host_step;
    return MARDYN_OK;
}

extern "C" {

int mardyn_set_thermostat(mardyn_ctx* ctx, double T_target, int32_t interval)
{
    if (!ctx) return MARDYN_EINVAL;
    if (!(T_target >= 0) || !std::isfinite(T_target) || interval < 0)
        return fail(ctx, MARDYN_EINVAL, "T_target must be finite and >= 0, interval >= 0");
    ctx->T_target = T_target;
    ctx->thermo_interval = interval;
    if (ctx->grp && ctx->nranks > 1)      // a decomposed run rescales with the global T: every rank alike
        for (mardyn_ctx* c : group_members(ctx)) { c->T_target = T_target; c->thermo_interval = interval; }
    for (int b = 0; b < 2; ++b)                       // the step graphs change
        if (ctx->gexec[b]) { cudaGraphExecDestroy(ctx->gexec[b]); ctx->gexec[b] = nullptr; }
    return MARDYN_OK;
}

// isotropic LJ tail corrections (reading A3): with g(r) = 1 beyond rc,
//   U = sum_{ci,cj} N_ci N_cj / (2V) sum_{LJ sites a,b} int_rc^inf u_ab 4 pi r^2 dr,
//   W = -sum_{ci,cj} N_ci N_cj / (2V) sum_{a,b} int_rc^inf r u_ab' 4 pi r^2 dr,
// u_ab the plain 12-6 potential with Lorentz-Berthelot * eta parameters
int mardyn_lj_tail(const mardyn_component* comps, int32_t n_comps, const double* eta, const int64_t* counts,
                   double volume, double cutoff, double* U, double* W)
{
    if (!comps || n_comps < 1 || !counts || !U || !W || !(volume > 0) || !(cutoff > 0)) return MARDYN_EINVAL;
    const double pi = 3.14159265358979323846;
    double u = 0.0, w = 0.0;
    for (int a = 0; a < n_comps; ++a)
        for (int b = 0; b < n_comps; ++b) {
            const double e_ab = eta ? eta[a * n_comps + b] : 1.0;
            const double dens = (double)counts[a] * (double)counts[b] / (2.0 * volume);
            for (int i = 0; i < comps[a].n_lj; ++i)
                for (int k = 0; k < comps[b].n_lj; ++k) {
                    const mardyn_lj_site& p = comps[a].lj[i];
                    const mardyn_lj_site& q = comps[b].lj[k];
                    const double sig = 0.5 * (p.sigma + q.sigma), eps = e_ab * std::sqrt(p.epsilon * q.epsilon);
                    const double s3 = (sig / cutoff) * (sig / cutoff) * (sig / cutoff), s9 = s3 * s3 * s3;
                    const double c = 16.0 * pi * eps * sig * sig * sig * dens;
                    u += c * (s9 / 9.0 - s3 / 3.0);
                    w += c * (4.0 / 3.0 * s9 - 2.0 * s3);
                }
        }
    *U = u;
    *W = w;
    return MARDYN_OK;
}

int mardyn_get_tail_corrections(mardyn_ctx* ctx, double* U, double* W)
{
    if (!ctx || !U || !W) return MARDYN_EINVAL;
    if (!ctx->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules first");
    std::vector<mardyn_component> cs(ctx->comps.size());
    for (size_t c = 0; c < cs.size(); ++c) {
        std::memset(&cs[c], 0, sizeof(mardyn_component));
        cs[c].n_lj = (int32_t)ctx->comps[c].lj.size();
        cs[c].lj = ctx->comps[c].lj.data();
    }
    const double V = (double)ctx->g.P64[0] * ctx->g.P64[1] * ctx->g.P64[2] * (double)ctx->g.s * ctx->g.s * ctx->g.s;
    return mardyn_lj_tail(cs.data(), (int32_t)cs.size(), ctx->eta.empty() ? nullptr : ctx->eta.data(),
                          ctx->comp_counts.data(), V, ctx->rc, U, W);
}

int mardyn_step(mardyn_ctx* ctx, int32_t nsteps)
{
    NvtxRange nvtx_range("mardyn_step");
    if (!ctx) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (!ctx->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules first");
    if (nsteps < 0) return fail(ctx, MARDYN_EINVAL, "n must be >= 0");
    if (nsteps == 0) return MARDYN_OK;
    if (ctx->nranks > 1) return group_step(ctx, nsteps);
    if (!ctx->gexec[0]) {
        int rc = build_graphs(ctx);
        if (rc) return rc;
    }
    for (int k = 0; k < nsteps; ++k) {
        CK(cudaGraphLaunch(ctx->gexec[ctx->cur], ctx->stream));
        ctx->last_parity = ctx->cur;
        ctx->cur ^= 1;
        ctx->launches += launches_per_step(ctx);
    }
    ctx->host_step += nsteps;
    ctx->last_obs = ctx->host_step - 1;
    ctx->last_force_launches = nsteps;
    return MARDYN_OK;
}

static int sync_check(mardyn_ctx* ctx)
{
    if (ctx->side_join) CK(cudaStreamSynchronize(ctx->side_stream));
    CK(cudaStreamSynchronize(ctx->stream));
    int flag = 0;
    CK(cudaMemcpy(&flag, ctx->flag, 4, cudaMemcpyDeviceToHost));
    if (flag & 4) return fail(ctx, MARDYN_ECAPACITY, "a row of three cells exceeds the force kernel's shared-memory slab");
    if (flag & 256) return fail(ctx, MARDYN_ECAPACITY, "exchange segment overflow (raise the segment capacity)");
    if (flag & 512) return fail(ctx, MARDYN_ECAPACITY, "owned + received molecules exceed the capacity");
    if (flag & 2) return fail(ctx, MARDYN_EOVERLAP, "two molecule centres coincide");
    if (flag) return fail(ctx, MARDYN_EUNSTABLE, "non-finite force/torque or a molecule moved more than one cell edge in a step");
    return MARDYN_OK;
}

static void to_obs(const ObsRec& o, mardyn_observables* out)
{
    out->step = o.step;
    out->U_pot = o.U;
    out->virial = o.W;
    out->T = o.T;
    out->E_kin_trans = o.KEt;
    out->E_kin_rot = o.KEr;
    out->n_pairs = o.npairs;
    out->n_candidates = o.ncand;
}

int mardyn_get_observables(mardyn_ctx* ctx, mardyn_observables* out)
{
    if (!ctx || !out) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (ctx->last_obs < 0) return fail(ctx, MARDYN_ESTATE, "no force evaluation yet (step or compute_forces)");
    if (ctx->grp) {                           // global values: rank-ordered sums over the group (A23)
        std::vector<ObsRec> ring;
        int rc = group_observables(ctx, ring);
        if (rc) return rc;
        to_obs(ring[ctx->last_obs % MD_HISTORY], out);
        return MARDYN_OK;
    }
    int rc = sync_check(ctx);
    if (rc) return rc;
    ObsRec o;
    CK(cudaMemcpy(&o, ctx->hist + (ctx->last_obs % MD_HISTORY), sizeof(o), cudaMemcpyDeviceToHost));
    to_obs(o, out);
    return MARDYN_OK;
}

int mardyn_get_observable_history(mardyn_ctx* ctx, int32_t cap, int32_t* n, mardyn_observables* out)
{
    if (!ctx || !n || (cap > 0 && !out)) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    long long last = ctx->last_obs;
    long long avail = std::min<long long>(last + 1, MD_HISTORY);
    long long m = std::min<long long>(avail, cap);
    std::vector<ObsRec> h(MD_HISTORY);
    if (ctx->grp) {
        int rc = group_observables(ctx, h);
        if (rc) return rc;
    } else {
        int rc = sync_check(ctx);
        if (rc) return rc;
        CK(cudaMemcpy(h.data(), ctx->hist, sizeof(ObsRec) * MD_HISTORY, cudaMemcpyDeviceToHost));
    }
    for (long long k = 0; k < m; ++k) to_obs(h[(last - m + 1 + k) % MD_HISTORY], out + k);
    *n = (int32_t)m;
    return MARDYN_OK;
}

// Copy molecule data (caller's original order = set_molecules index) to
// host arrays.  Single rank: all n molecules.  Decomposed: the molecules this
// rank owns, compacted in index order; their ids go to ids_out.
static int egress(mardyn_ctx* ctx, double* r, double* v, double* q, double* j, double* F, double* tau,
                  uint32_t* ufix, int32_t* cell, int64_t n_slots = -1, int64_t* n_out = nullptr,
                  int64_t* ids_out = nullptr, int32_t* comp_out = nullptr)
{
    if (ctx->nranks > 1)      // the rank's owned molecules, compacted, with their ids
        return egress_dd(ctx, r, v, q, j, F, tau, ufix, cell, n_slots, n_out, ids_out, comp_out);
    const int64_t n = n_slots < 0 ? ctx->n : n_slots;          // sorted slots to read = molecules
    cudaStream_t s = ctx->stream;
    double* d_r = (double*)ctx->stage;
    double* d_v = d_r + 3 * n;
    double* d_q = d_v + 3 * n;
    double* d_j = d_q + 4 * n;
    double* d_F = d_j + 3 * n;
    double* d_t = d_F + 3 * n;
    uint32_t* d_u = (uint32_t*)(d_t + 3 * n);
    int* d_c = (int*)(d_u + 3 * n);
    const int b = ctx->cur;
    if (ctx->rigid)
        k_egress<true><<<nblk(n, 256), 256, 0, s>>>((int)n, ctx->g, ctx->pos[b], ctx->vel[b], ctx->quat[b],
                                                    ctx->angm[b], ctx->force, ctx->torque, r ? d_r : nullptr,
                                                    v ? d_v : nullptr, q ? d_q : nullptr, j ? d_j : nullptr,
                                                    F ? d_F : nullptr, tau ? d_t : nullptr, ufix ? d_u : nullptr,
                                                    cell ? d_c : nullptr);
    else
        k_egress<false><<<nblk(n, 256), 256, 0, s>>>((int)n, ctx->g, ctx->pos[b], ctx->vel[b], nullptr, nullptr,
                                                     ctx->force, nullptr, r ? d_r : nullptr, v ? d_v : nullptr,
                                                     q ? d_q : nullptr, j ? d_j : nullptr, F ? d_F : nullptr,
                                                     tau ? d_t : nullptr, ufix ? d_u : nullptr, cell ? d_c : nullptr);
    ctx->launches += 1;
    CK(cudaGetLastError());
    if (r) CK(cudaMemcpyAsync(r, d_r, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
    if (v) CK(cudaMemcpyAsync(v, d_v, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
    if (q) CK(cudaMemcpyAsync(q, d_q, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, s));
    if (j) CK(cudaMemcpyAsync(j, d_j, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
    if (F) CK(cudaMemcpyAsync(F, d_F, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
    if (tau) CK(cudaMemcpyAsync(tau, d_t, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
    if (ufix) CK(cudaMemcpyAsync(ufix, d_u, sizeof(uint32_t) * 3 * n, cudaMemcpyDeviceToHost, s));
    if (cell) CK(cudaMemcpyAsync(cell, d_c, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    if (n_out) *n_out = n;
    return sync_check(ctx);
}

int mardyn_get_molecules(mardyn_ctx* ctx, int64_t cap, int64_t* n, int64_t* id, int32_t* comp, double* r,
                         double* v, double* q, double* j)
{
    NvtxRange nvtx_range("mardyn_get_molecules");
    if (!ctx || !n) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (!ctx->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules first");
    if (int rc0 = refresh_n(ctx)) return rc0;
    if (cap < ctx->n) return fail(ctx, MARDYN_EINVAL, "cap < number of molecules");
    if (ctx->nranks > 1)      // the rank's owned molecules, with their ids
        return egress(ctx, r, v, q, j, nullptr, nullptr, nullptr, nullptr, -1, n, id, comp);
    *n = ctx->n;
    if (id) CK(cudaMemcpyAsync(id, ctx->ids_dev, sizeof(int64_t) * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
    if (comp) CK(cudaMemcpyAsync(comp, ctx->comp_dev, sizeof(int32_t) * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
    return egress(ctx, r, v, q, j, nullptr, nullptr, nullptr, nullptr);
}

int mardyn_get_forces(mardyn_ctx* ctx, int64_t cap, double* F, double* tau, int64_t* n_out, int64_t* ids)
{
    if (!ctx) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (!ctx->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules first");
    if (int rc0 = refresh_n(ctx)) return rc0;
    if (cap < ctx->n) return fail(ctx, MARDYN_EINVAL, "cap < number of molecules");
    // forces are indexed by the sorted slots of the buffer they were computed on
    int64_t* idp = nullptr;
    int64_t nn = 0;
    if (ctx->nranks > 1) idp = ids;
    if (ctx->last_obs >= 0 && ctx->last_obs == ctx->host_step - 1 && ctx->host_step > 0) {
        // after a step: F belongs to the previous parity; egress that buffer's ids
        int b = ctx->cur;
        ctx->cur = ctx->last_parity;
        int rc = egress(ctx, nullptr, nullptr, nullptr, nullptr, F, tau, nullptr, nullptr, ctx->n_force, &nn, idp);
        ctx->cur = b;
        if (n_out) *n_out = nn;
        return rc;
    }
    int rc = egress(ctx, nullptr, nullptr, nullptr, nullptr, F, tau, nullptr, nullptr, ctx->n_force, &nn, idp);
    if (n_out) *n_out = nn;
    return rc;
}

int mardyn_get_raw(mardyn_ctx* ctx, int64_t cap, uint32_t* pos_fixed, int32_t* cell, int32_t* cell_count)
{
    if (!ctx) return MARDYN_EINVAL;
    if (ctx->poisoned) return fail(ctx, MARDYN_ECUDA, "context poisoned");
    if (!ctx->loaded) return fail(ctx, MARDYN_ESTATE, "set_molecules first");
    if (int rc0 = refresh_n(ctx)) return rc0;
    if (cap < ctx->n) return fail(ctx, MARDYN_EINVAL, "cap < number of molecules");
    int rc = egress(ctx, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, pos_fixed, cell);
    if (rc) return rc;
    if (cell_count) {
        // counts of the current sorted state = start differences
        // counts of the current sorted state = start differences over the (rank-local) window,
        // reported per global cell (0 outside the window)
        const GridP& g = ctx->g;
        std::vector<int> st(g.wncell + 1);
        CK(cudaMemcpy(st.data(), ctx->start, sizeof(int) * (g.wncell + 1), cudaMemcpyDeviceToHost));
        std::fill(cell_count, cell_count + g.ncell, 0);
        for (int l = 0; l < g.wncell; ++l) {
            const int lx = l % g.wn[0], ly = (l / g.wn[0]) % g.wn[1], lz = l / (g.wn[0] * g.wn[1]);
            cell_count[cell_glob(g, glob_axis(g, 0, lx), glob_axis(g, 1, ly), glob_axis(g, 2, lz))] = st[l + 1] - st[l];
        }
    }
    return MARDYN_OK;
}

int mardyn_last_step_timing(mardyn_ctx* ctx, double* total_ms, double* force_ms, int32_t* force_launches)
{
    if (!ctx) return MARDYN_EINVAL;
    CK(cudaStreamSynchronize(ctx->stream));
    float f = 0.f;
    if (ctx->profiling && (ctx->gexec[0] || ctx->nranks > 1)) {
        cudaError_t e = cudaEventElapsedTime(&f, ctx->ev_f0[ctx->last_parity], ctx->ev_f1[ctx->last_parity]);
        if (e != cudaSuccess) { f = 0.f; cudaGetLastError(); }
    }
    double tot = 0.0;
    if (ctx->rank_timed) {        // decomposed step: this rank's own kernels (begin + end halves)
        float a = 0.f, b = 0.f;
        if (cudaEventElapsedTime(&a, ctx->ev_r[0], ctx->ev_r[1]) == cudaSuccess &&
            cudaEventElapsedTime(&b, ctx->ev_r[2], ctx->ev_r[3]) == cudaSuccess)
            tot = (double)a + (double)b;
        else
            cudaGetLastError();
    }
    if (total_ms) *total_ms = tot;
    if (force_ms) *force_ms = f;
    if (force_launches) *force_launches = 1;
    return MARDYN_OK;
}

int mardyn_set_profiling(mardyn_ctx* ctx, int32_t on)
{
    if (!ctx) return MARDYN_EINVAL;
    if ((bool)on != ctx->profiling) {
        ctx->profiling = on != 0;
        group_drop_graphs(ctx->grp);
        for (int b = 0; b < 2; ++b)
            if (ctx->gexec[b]) { cudaGraphExecDestroy(ctx->gexec[b]); ctx->gexec[b] = nullptr; }
    }
    return MARDYN_OK;
}

int64_t mardyn_launch_count(const mardyn_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"

// spatial decomposition across GPUs: the distributed engine and its C ABI
#include "dist_engine.cuh"

extern "C" {

int mardyn_cell_cost(const int32_t* counts, int32_t nx, int32_t ny, int32_t nz, double* cost)
{
    if (!counts || !cost || nx < 1 || ny < 1 || nz < 1) return MARDYN_EINVAL;
    mdd::cell_cost(counts, nx, ny, nz, cost);
    return MARDYN_OK;
}

int mardyn_kd_decompose(const double* cost, int32_t nx, int32_t ny, int32_t nz, int32_t p, int32_t* boxes,
                        double* loads)
{
    if (!cost || !boxes || p < 1 || nx < 1 || ny < 1 || nz < 1) return MARDYN_EINVAL;
    std::vector<mdd::Box> leaves;
    mdd::Box all;
    all.lo[0] = all.lo[1] = all.lo[2] = 0;
    all.hi[0] = nx; all.hi[1] = ny; all.hi[2] = nz;
    if (!mdd::kd_split(cost, nx, ny, all, p, 0, leaves) || (int)leaves.size() != p) return MARDYN_EINVAL;
    for (int r = 0; r < p; ++r) {
        const mdd::Box& b = leaves[r];
        double l = 0.0;
        for (int z = b.lo[2]; z < b.hi[2]; ++z)
            for (int y = b.lo[1]; y < b.hi[1]; ++y)
                for (int x = b.lo[0]; x < b.hi[0]; ++x) l += cost[x + nx * (y + ny * z)];
        for (int k = 0; k < 3; ++k) { boxes[6 * r + k] = b.lo[k]; boxes[6 * r + 3 + k] = b.hi[k]; }
        if (loads) loads[r] = l;
    }
    return MARDYN_OK;
}

const char* mardyn_last_error(const mardyn_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void mardyn_destroy(mardyn_ctx* ctx)
{
    if (!ctx) return;
#ifdef MD_LJ1_STATS
    if (ctx->flag) {
        unsigned long long st[4] = {0, 0, 0, 0};
        cudaMemcpy(st, ctx->flag + 16, sizeof(st), cudaMemcpyDeviceToHost);
        std::printf("LJ1_STATS useful_pairs %llu slot_pairs %llu balance %.4f subchunk_lanes %llu perlane_lanes %llu\n",
                    st[0], st[1], st[1] ? (double)st[0] / (double)st[1] : 0.0, st[2], st[3]);
    }
#endif
    group_release(ctx);
    for (int b = 0; b < 2; ++b) {
        if (ctx->gexec[b]) cudaGraphExecDestroy(ctx->gexec[b]);
        if (ctx->ev_f0[b]) cudaEventDestroy(ctx->ev_f0[b]);
        if (ctx->ev_f1[b]) cudaEventDestroy(ctx->ev_f1[b]);
    }
    if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
    for (int k = 0; k < 4; ++k)
        if (ctx->ev_r[k]) cudaEventDestroy(ctx->ev_r[k]);
    if (ctx->ev_s0) cudaEventDestroy(ctx->ev_s0);
    if (ctx->ev_s1) cudaEventDestroy(ctx->ev_s1);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

}  // extern "C"
