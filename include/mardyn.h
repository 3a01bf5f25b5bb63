/*
 * mardyn.h -- C ABI of the B200-native ls1-mardyn hot path (arXiv:1408.4599).
 *
 * One context = one simulation box on one GPU: rigid multi-centre molecules
 * interacting through Lennard-Jones 12-6 sites (Eq. 1,
 * P:70-74, truncated and shifted P:75-76), point charges with reaction field
 * (P:39), point dipoles and linear point quadrupoles; forces
 * found by linked cells of edge >= rc rebuilt every step; time
 * integration by leapfrog (Eqs. 2-3) plus the quaternion
 * rotational leapfrog (Eqs. 4-5).  The readings of the paper's
 * silent points are listed in DESIGN.md §2 and cited below as A<k>.
 *
 * Conventions shared by every call
 *  - Every call returns int: MARDYN_OK (0) or a negative MARDYN_E* code;
 *    mardyn_last_error(ctx) gives a one-line message.  After MARDYN_ECUDA the
 *    context is poisoned and must be destroyed.
 *  - Units: any consistent set with k_B = k_C = 1.
 *  - Host arrays passed in are owned by the caller and only read during the
 *    call; output arrays are caller-allocated with the stated capacity.
 *  - Device memory is owned by the caller (PyTorch in the Python binding):
 *    the library reports its need (mardyn_workspace_bytes) and carves the
 *    buffer given to mardyn_set_workspace.  The context owns no device memory
 *    except the workspace pointer it was handed and its CUDA graphs/events.
 *  - All device work is enqueued on the stream given in mardyn_options
 *    (NULL: a private non-blocking stream).  mardyn_step is asynchronous;
 *    every mardyn_get_* call synchronises that stream.
 *  - One context per host thread; calls are not reentrant.
 *
 * Positions (reading A12).  Positions are stored as unsigned fixed point
 * u_k in [0, P_k) with one quantum s = 2^(ceil(log2(max cell edge)) - 22)
 * common to all axes; each cell edge is E_k quanta, P_k = n_k E_k, and the
 * box is snapped to P_k s (a relative change below 1e-6; mardyn_get_grid
 * returns it).  Cell assignment cell_k = floor(u_k / E_k) is exact integer
 * arithmetic; the cutoff test r^2 < rc^2 on the minimum-image separation is
 * decided exactly (integer arithmetic in a guard band around rc).
 */
#ifndef MARDYN_H
#define MARDYN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MARDYN_OK = 0,
    MARDYN_EINVAL = -1,     /* bad input: < 3 cells per axis, rc <= 0, dt <= 0,
                               eps_rf < 1, mass <= 0, inertia < 0, bad component id,
                               |quaternion| far from 1, n > capacity            */
    MARDYN_EOVERLAP = -2,   /* two molecule centres coincide                    */
    MARDYN_EUNSTABLE = -3,  /* non-finite force/torque or a molecule moved more
                               than one cell edge in one step    */
    MARDYN_ECAPACITY = -4,  /* workspace too small for the requested capacity   */
    MARDYN_ECUDA = -5,      /* CUDA runtime error (context poisoned)            */
    MARDYN_ENCCL = -6,      /* NCCL error (multi-GPU transport; context poisoned) */
    MARDYN_ESTATE = -7      /* call order, e.g. step before set_molecules       */
};

/* Sites of a component, body frame, positions relative to the centre of
 * mass.  Dipole/quadrupole axes are unit vectors.                 */
typedef struct { double r[3]; double sigma, epsilon; } mardyn_lj_site;
typedef struct { double r[3]; double q; } mardyn_charge;
typedef struct { double r[3]; double e[3]; double m; } mardyn_polar; /* m = mu or Q */

/* A component (molecule species).  inertia = principal moments; the body
 * axes are the principal axes.  A moment of 0 removes that rotational
 * degree of freedom (linear molecules: 2; single point site: 0).            */
typedef struct {
    int32_t n_lj, n_q, n_mu, n_Q;
    const mardyn_lj_site* lj;
    const mardyn_charge* q;
    const mardyn_polar* mu;
    const mardyn_polar* Q;
    double mass;
    double inertia[3];
} mardyn_component;

typedef struct {
    double dt;                  /* time step (> 0)                               */
    double eps_rf;              /* reaction-field dielectric constant (>= 1;
                                   INFINITY = conducting boundary), A4           */
    int32_t lj_shift;           /* 1 = truncated and shifted LJ (LJTS, A2)       */
    const double* eta;          /* n_comps*n_comps binary parameters or
                                   NULL (all 1); copied                           */
    int32_t rebalance_interval; /* decomposed contexts: re-partition from the
                                   measured cell loads every this many steps
                                   (P:197); 0 = static partition          */
    void* cuda_stream;          /* cudaStream_t or NULL                          */
} mardyn_options;

typedef struct {
    int64_t step;               /* index k of the time t_k these values refer to */
    double U_pot;               /* potential energy U(t_k)                       */
    double virial;              /* molecular virial W = sum_{i<j} (r_i-r_j).F_ij, A6 */
    double T;                   /* 2 (KE_t + KE_r) / N_dof, A9                   */
    double E_kin_trans, E_kin_rot;
    int64_t n_pairs;            /* unique molecule pairs with r_ij < rc          */
    int64_t n_candidates;       /* 27-cell full-shell candidates (i != j)        */
} mardyn_observables;

typedef struct {
    int32_t ncell[3];           /* cells per axis, n_k = floor(L_k / rc)         */
    int32_t pad;
    double quantum;             /* s (a power of two)                            */
    int64_t period[3];          /* P_k in quanta                                 */
    int64_t edge[3];            /* E_k in quanta                                 */
    double box[3];              /* snapped box P_k * s                           */
    int64_t cut2_q;             /* smallest r^2 (in quanta^2) NOT within rc:
                                   ceil(fl64(rc*rc) / s^2)                        */
    int32_t kernel;             /* force kernel in use: 0 = single LJ site fast
                                   path, 1 = rigid (templated shape), 2 = generic */
    int32_t n_slots;            /* float4 site slots per molecule (rigid kernels) */
} mardyn_grid;

/*
 * Create a context for box L[3] (periodic), cutoff rc and the given
 * components (copied).  Requires n_k = floor(L_k / rc) >= 3 on every axis.
 */
int mardyn_create(const double box[3], double cutoff, const mardyn_component* comps,
                  int32_t n_comps, const mardyn_options* opt, struct mardyn_ctx** out);

/* Grid, lattice and kernel choice of a context (reading A12).              */
int mardyn_get_grid(const struct mardyn_ctx* ctx, mardyn_grid* out);

/* Device bytes needed for up to n_capacity molecules.                      */
int mardyn_workspace_bytes(struct mardyn_ctx* ctx, int64_t n_capacity, size_t* bytes);

/* Hand the context a device buffer (256-byte aligned; MARDYN_EINVAL otherwise) of at least
 * mardyn_workspace_bytes(n_capacity) bytes; must precede set_molecules.     */
int mardyn_set_workspace(struct mardyn_ctx* ctx, void* device_ptr, size_t bytes,
                         int64_t n_capacity);

/*
 * Load n molecules from HOST arrays: id (n, may be NULL = 0..n-1), comp (n),
 * r (n*3 positions, wrapped into the box), v (n*3), q (n*4 unit quaternions
 * (w,x,y,z), body->world), j (n*3 world-frame angular momenta; q, j may be
 * NULL for single-site models).  half_step = 0: v, j are on-step values at
 * t0 and the library applies the backward half kick v -= dt/2 F/m,
 * j -= dt/2 tau with F(t0), tau(t0) (A8); 1: v, j are already
 * v(t0 - dt/2), j(t0 - dt/2), as returned by mardyn_get_molecules.
 * The arrays are copied to the device and converted and validated there
 * (pinned host buffers are DMA'd directly).  Errors: MARDYN_EINVAL for n
 * outside [1, capacity], missing arrays, or any molecule with a non-finite
 * r or v, a component id outside [0, n_comps) or |q|^2 off 1 by 1e-5 (the
 * context then holds no molecules); MARDYN_ESTATE before set_workspace.
 */
int mardyn_set_molecules(struct mardyn_ctx* ctx, int64_t n, const int64_t* id,
                         const int32_t* comp, const double* r, const double* v,
                         const double* q, const double* j, int32_t half_step);

/* F(t), tau(t), U, W at the current positions (no integration).           */
int mardyn_compute_forces(struct mardyn_ctx* ctx);

/* n leapfrog steps (asynchronous; per step: forces at t_k, observables of
 * t_k, kick + drift + rotation, (NVT rescaling,) cell rebuild by counting
 * sort).                                                                    */
int mardyn_step(struct mardyn_ctx* ctx, int32_t n);

/*
 * NVT by velocity rescaling ("kept constant by velocity rescaling";
 * reading A24 of DESIGN.md): after every interval-th step k the half-step
 * velocities and angular momenta are scaled by sqrt(T_target / T(t_k)).
 * T_target = 0 or interval = 0: NVE (default).  On a decomposed run T(t_k) is
 * the global temperature.  Errors: MARDYN_EINVAL for a negative or non-finite
 * T_target or a negative interval; a step with T(t_k) = 0 reports
 * MARDYN_EUNSTABLE.
 */
int mardyn_set_thermostat(struct mardyn_ctx* ctx, double T_target, int32_t interval);

/*
 * Isotropic LJ tail corrections beyond the cutoff ("isotropic cut-off
 * corrections", a mean-field integral with g(r) = 1; reading A3: reported
 * beside U_pot and the virial, never added to them):
 *   U = sum_{a,b} N_a N_b / (2V) sum_{LJ sites i of a, k of b} 16 pi eps sig^3 [(sig/rc)^9/9 - (sig/rc)^3/3]
 *   W = sum_{a,b} N_a N_b / (2V) sum_{i,k} 16 pi eps sig^3 [4/3 (sig/rc)^9 - 2 (sig/rc)^3]
 * with sig, eps mixed as in the forces (Lorentz-Berthelot * eta) and
 * W in the convention of the reported virial (pressure correction W/(3V)).
 * mardyn_lj_tail needs no context or GPU: comps as for mardyn_create, eta
 * n_comps^2 or NULL, counts[a] molecules of component a in volume.
 * mardyn_get_tail_corrections evaluates it for a loaded context (global
 * counts, snapped box).  Errors: MARDYN_EINVAL (null pointers, volume or
 * cutoff <= 0), MARDYN_ESTATE (no molecules).
 */
int mardyn_lj_tail(const mardyn_component* comps, int32_t n_comps, const double* eta, const int64_t* counts,
                   double volume, double cutoff, double* U, double* W);
int mardyn_get_tail_corrections(struct mardyn_ctx* ctx, double* U, double* W);

/* Observables of the last evaluated time (A23): after step(n) from t0 this
 * is t_{n-1}; after compute_forces it is the current t.                     */
int mardyn_get_observables(struct mardyn_ctx* ctx, mardyn_observables* out);

/* Up to cap most recent per-step observables, oldest first (ring of 4096). */
int mardyn_get_observable_history(struct mardyn_ctx* ctx, int32_t cap, int32_t* n,
                                  mardyn_observables* out);

/* Molecule state in the caller's original order (index of set_molecules):
 * r (n*3), v (n*3, at t - dt/2), q (n*4), j (n*3, at t - dt/2); any output
 * pointer may be NULL.  cap must be >= n.  For a decomposed context: the
 * molecules this rank owns, compacted in index order, with their ids.     */
int mardyn_get_molecules(struct mardyn_ctx* ctx, int64_t cap, int64_t* n, int64_t* id,
                         int32_t* comp, double* r, double* v, double* q, double* j);

/* Forces F (n*3) and torques tau (n*3) of the last force evaluation, in the
 * caller's original order; *n_out (may be NULL) = molecules written.  For a
 * decomposed context: the rank's owned molecules, compacted, ids in ids.    */
int mardyn_get_forces(struct mardyn_ctx* ctx, int64_t cap, double* F, double* tau, int64_t* n_out,
                      int64_t* ids);

/* Raw parity hook: fixed-point positions u (n*3, original order), cell of
 * each molecule (n) and count per cell (n_cells), as used by the last force
 * evaluation.  Any pointer may be NULL.                                     */
int mardyn_get_raw(struct mardyn_ctx* ctx, int64_t cap, uint32_t* pos_fixed,
                   int32_t* cell, int32_t* cell_count);

/* Device timing of the last step: force_ms = the force kernel (CUDA events on
 * the context stream; 0 if not recorded); total_ms = on a decomposed context
 * after an asynchronous step, this rank's own kernels of the step (its
 * begin and end halves; the exchange wait excluded), else 0.               */
int mardyn_last_step_timing(struct mardyn_ctx* ctx, double* total_ms, double* force_ms,
                            int32_t* force_launches);

/* Enable (1) / disable (0) per-step CUDA event timing of the force kernel. */
int mardyn_set_profiling(struct mardyn_ctx* ctx, int32_t on);

/* Number of device kernel launches enqueued so far by this context.        */
int64_t mardyn_launch_count(const struct mardyn_ctx* ctx);

/*
 * Host-side load model and spatial decomposition (no device work; usable
 * without a GPU).  PAPER.md §4: per-cell cost Eq. 6
 *     n_d(i) = N_i / 2 (N_i + sum_{j in the 26 neighbours} N_j)
 * and the k-d tree: recursive bisection with planes
 * perpendicular to alternating axes (x, y, z by depth; the next axis if the
 * depth's axis cannot be cut), each plane minimising
 * |load_left / p_left - load_right / p_right| over all admissible planes
 * (ties: the more central plane), >= 2 cells per subvolume per axis,
 * child process counts ceil(p/2), floor(p/2).
 * Arrays are x-fastest over (nx, ny, nz) cells, periodic.
 */
int mardyn_cell_cost(const int32_t* counts, int32_t nx, int32_t ny, int32_t nz, double* cost);

/* boxes: p * 6 int32 (lo_x, lo_y, lo_z, hi_x, hi_y, hi_z; half-open) in rank
 * order; loads: p doubles (sum of cost per box) or NULL.  Returns
 * MARDYN_EINVAL if the 2-cell constraint cannot be met.                    */
int mardyn_kd_decompose(const double* cost, int32_t nx, int32_t ny, int32_t nz, int32_t p,
                        int32_t* boxes, double* loads);

/*
 * Spatial decomposition across GPUs (§4).
 * A decomposed run is a group of ranks with the same box, cutoff, components
 * and options, each rank one context on its own GPU:
 *
 *   rank 0:  mardyn_nccl_unique_id(id)     -- 128 bytes, broadcast by the caller
 *   every rank: mardyn_create_distributed(..., id, rank, world, device, &ctx)
 *               mardyn_partition(ctx, N, r_global)          -- k-d tree (below)
 *               mardyn_dd_counts -> size the workspace       -- owned + halo
 *               mardyn_workspace_bytes / set_workspace
 *               mardyn_set_molecules(ctx, N, GLOBAL arrays)  -- keeps owned + halo
 *               mardyn_step(ctx, n) ...                      -- collective
 *               mardyn_get_observables(ctx, &o)              -- collective, global
 *
 * The library owns the NCCL communicator (NCCL is loaded at run time,
 * dlopen("libnccl.so.2"): the copy a host process already loaded, else the
 * system one; the environment variable MARDYN_NCCL_LIB names another library
 * with NCCL's entry points instead -- the tests run several ranks on one GPU
 * through a host-staged stand-in, tests/nccl_shim.c, since NCCL refuses two
 * ranks of a communicator on one device).  Each step: forces on the rank's home box (its k-d box; the
 * halo holds copies of every molecule within one cell layer of edge >= rc,
 * P:220-221), kick / drift / rotation of the owned molecules, then every
 * molecule whose new cell lies in another rank's box (migrant) or halo
 * (halo copy) is packed as a 64-byte record (position, v, q, j) by the same
 * kernel and stored straight into the receiving rank's memory (CUDA IPC
 * mappings of the peers' receive areas, opened after the first step; one
 * one-word ncclAllReduce per step orders the stores before the imports), or,
 * when a rank cannot export or open them or MARDYN_IPC_PUTS=0, moved by NCCL
 * send / recv (fixed per-peer segments with device-side counts); no host
 * synchronisation after the first step.  The receiver imports them and
 * rebuilds its cells.  Every
 * rebalance_interval steps the measured per-cell loads of the last cell
 * rebuild are summed over the ranks (ncclAllReduce), the Eq. 6 cost and the
 * k-d tree are recomputed on every rank (identical host code), and the
 * molecules are re-distributed through the same records.
 * mardyn_get_observables / _history return GLOBAL values (rank-ordered sums
 * of the ranks' partials; ncclAllGather) and are collective calls;
 * mardyn_get_molecules / get_forces / get_raw return the rank's owned
 * molecules (compacted, ordered by input index) with their ids.  NVT
 * rescaling uses the global temperature (an allreduce of the ranks' kinetic
 * energies; set it on every rank, or on rank 0 of a loopback group).
 * world = 1 is allowed: a one-domain context whose observables travel
 * through the communicator.  Errors: MARDYN_ENCCL (NCCL missing or failed;
 * the context is poisoned), MARDYN_ECAPACITY (a rank's owned + halo +
 * received molecules exceed its capacity, or an exchange segment overflows).
 * Before the collectives of the first step after a load or rebalance, of the
 * rebalance and of get_observables the ranks agree on failure: when one rank
 * fails there, it returns its own error and every other rank returns
 * MARDYN_ESTATE ("another rank of the decomposition failed").
 */
int mardyn_nccl_unique_id(void* out128);
int mardyn_create_distributed(const double box[3], double cutoff, const mardyn_component* comps,
                              int32_t n_comps, const mardyn_options* opt, const void* nccl_unique_id,
                              int32_t rank, int32_t world, int32_t device, struct mardyn_ctx** out);

/* p ranks of one decomposition inside this process, on the current device, all
 * enqueued on one stream (opt->cuda_stream, or one the group creates): the
 * single-GPU correctness path.  out[p] receives the ranks' contexts (rank r =
 * out[r]); each needs its own workspace and set_molecules with the global arrays;
 * step / compute_forces / rebalance go through out[0] and advance every rank
 * (records are stored straight into the receiving rank's buffer); get_observables
 * on any rank returns the global values.                                       */
int mardyn_create_loopback(const double box[3], double cutoff, const mardyn_component* comps,
                           int32_t n_comps, const mardyn_options* opt, int32_t p, struct mardyn_ctx** out);

/* k-d partition from the GLOBAL positions r (n*3, any order; host arrays):
 * per-cell molecule counts on the A12 lattice, the Eq. 6 cost, the k-d tree
 * (mardyn_kd_decompose); every rank computes the same boxes.  Before
 * set_molecules.  mardyn_set_partition: explicit boxes (p*6, as
 * mardyn_kd_decompose returns; e.g. static equal-volume boxes), the context then
 * holds no molecules until the next set_molecules.  mardyn_get_partition: the
 * current boxes (p*6).  mardyn_dd_counts: owned + halo molecules of every rank
 * (p int64) for the current partition (host; to size the workspaces).          */
int mardyn_partition(struct mardyn_ctx* ctx, int64_t n, const double* r);
int mardyn_set_partition(struct mardyn_ctx* ctx, const int32_t* boxes);
int mardyn_get_partition(const struct mardyn_ctx* ctx, int32_t* boxes);
int mardyn_dd_counts(struct mardyn_ctx* ctx, int64_t n, const double* r, int64_t* counts);

/* Per-cell load the k-d tree balances (partition and rebalance; every rank of a group):
 * 0 = Eq. 6 (the default: pair-interaction cost N_i/2 (N_i + sum_26 N_j)),
 * 1 = the molecule count N_i.  On a B200 the step time per molecule varies by less than
 * the pair count does (per-molecule work -- staging, window searches, integration, the
 * rebuild -- dominates, and sparse cells take the slower per-lane path), so model 1 balances
 * heterogeneous systems better.  Errors: MARDYN_EINVAL.             */
int mardyn_set_cost_model(struct mardyn_ctx* ctx, int32_t model);

/* Host-only (no context, no GPU): cells per axis of the A12 lattice for box and
 * cutoff (ncell[3]) and, if counts != NULL, the molecules per cell (x fastest) of
 * the n positions r (n*3); and the k-d partition of those positions into p boxes
 * (Eq. 6 cost + mardyn_kd_decompose), as mardyn_partition computes it.         */
int mardyn_grid_counts(const double box[3], double cutoff, int64_t n, const double* r, int32_t ncell[3],
                       int32_t* counts);
int mardyn_kd_partition(const double box[3], double cutoff, int64_t n, const double* r, int32_t p,
                        int32_t* boxes, double* loads);

/* Re-partition now (collective; loopback: through rank 0), as the periodic
 * rebalance of options.rebalance_interval does.                               */
int mardyn_rebalance(struct mardyn_ctx* ctx);

const char* mardyn_last_error(const struct mardyn_ctx* ctx);
void mardyn_destroy(struct mardyn_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MARDYN_H */
