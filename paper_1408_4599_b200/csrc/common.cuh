// common.cuh -- device-side data layout and constants of the B200 hot path.
//
// HBM layout: structure of arrays, one row per molecule,
// sorted by cell (x fastest) and, inside a cell, by internal id (reading
// A13), rebuilt every step by counting sort.  The state is double-buffered
// (cur -> nxt by the canonicalising gather).
//   pos   uint4  (u_x, u_y, u_z, iid)        fixed-point position (A12) + id
//   vel   float4 (v_x, v_y, v_z, comp bits)  v(t - dt/2)
//   quat  float4 (w, x, y, z)                rigid only
//   angm  float4 (j_x, j_y, j_z, 0)          world frame, j(t - dt/2), rigid
//   xs    float4 (x, y, z cell-relative, comp bits | cell x index)  staging copy read by the
//                force kernels; exact multiples of s below 2^24 s
//   site  float4 [n_slots][cap]              world-frame site offsets / axes
//   force float4 (F, 0), torque float4 (tau, 0)
#pragma once

// debug builds (-DMD_DEBUG_CHECKS, profiles/tools/debug_checks.sh): device-side bounds checks of the
// shared-memory lists and slabs and of the sorted-slot indices; a failed check aborts the kernel
// (cudaErrorAssert -> MARDYN_ECUDA).  compute-sanitizer is not available on the GPU pool.
#ifdef MD_DEBUG_CHECKS
#include <cassert>
#define MD_CHECK(c) assert(c)
#else
#define MD_CHECK(c) ((void)0)
#endif
#include <cstdint>
#include <cuda_runtime.h>

#define MD_MAX_COMP 8
#define MD_MAX_SITES 12          // sites per component
#define MD_MAX_LJ_TOTAL 16       // LJ sites over all components (mixing table)
#define MD_MAX_SLOTS 16          // float4 site slots per molecule
#define MD_HISTORY 4096          // observable ring buffer

enum { MD_LJ = 0, MD_CHARGE = 1, MD_DIPOLE = 2, MD_QUAD = 3 };

struct DevComp {
    float mass, inv_mass;
    float invI[3];               // 0 where the moment is 0
    int n_lj, n_q, n_mu, n_Q;
    int lj0;                     // first global LJ index (mixing table)
    int slot_lj, slot_q, slot_mu, slot_Q;   // first slot of each kind; polar
                                             // sites use 2 slots (pos, axis)
    int n_slots;
    int rot;                     // rotational degrees of freedom
    float bpos[MD_MAX_SITES][3]; // body positions in slot order of kinds
    float baxis[MD_MAX_SITES][3];
    float mom[MD_MAX_SITES];     // q / mu / Q per site (LJ: unused)
};

struct DevModel {
    int n_comp;
    int n_lj_total;
    float krf, crf, krf_mumu;    // reaction field (A4)
    DevComp comp[MD_MAX_COMP];
    // LJ mixing table over global LJ site indices (Lorentz-Berthelot * eta)
    float sig2[MD_MAX_LJ_TOTAL * MD_MAX_LJ_TOTAL];
    float eps24[MD_MAX_LJ_TOTAL * MD_MAX_LJ_TOTAL];
    float eps4[MD_MAX_LJ_TOTAL * MD_MAX_LJ_TOTAL];
    float shift[MD_MAX_LJ_TOTAL * MD_MAX_LJ_TOTAL];   // 4 eps [(s/rc)^12 - (s/rc)^6] if LJTS
};

struct GridP {
    int nc[3];
    int ncell;
    uint32_t E[3];               // cell edge in quanta (<= 2^22)
    uint64_t Einv[3];            // ceil(2^64 / E): u / E == __umul64hi(u, Einv) for every u < 2^32
    uint32_t P[3];               // period in quanta (P may be 2^32 - wrap with 64-bit)
    uint64_t P64[3];
    float s, inv_s;              // quantum, 1/s (powers of two)
    float edge[3];               // E * s
    float cut2;                  // rc^2 (fp32)
    float cut2_lo, cut2_hi;      // guard band around rc^2 for the exact test
    float band_mid, band_hw;     // 0.5 (lo + hi), 0.5 (hi - lo) + 1e-6 hi (fp32, set with lo / hi)
    long long cut2_q;            // exact threshold in quanta^2: in range iff r2q < cut2_q
    float dt;
    // Rank-local cell window (spatial decomposition): the cells a rank can hold -- its box plus
    // one halo layer -- numbered locally, x fastest: local l_k = (c_k - wlo_k) mod nc_k in
    // [0, wn_k); an axis the window covers entirely keeps wlo = 0, wn = nc (and its periodic wrap).
    // count[] / start[] / cell_of[] use local indices (the scan runs over wncell cells), the
    // owner / halo maps global ones.  One domain: wlo = 0, wn = nc (identity).
    int wlo[3], wn[3];
    int wncell;
    int hlo[3], hdim[3];         // home cells of this rank, LOCAL: box [hlo, hlo + hdim) (whole grid if 1 rank)
    int nhome;
};

// local coordinate of global cell coordinate c on axis k (c inside the window)
__host__ __device__ __forceinline__ int loc_axis(const GridP& g, int k, int c)
{
    int l = c - g.wlo[k];
    if (l < 0) l += g.nc[k];
    return l;
}
// global cell coordinate of local coordinate l on axis k
__host__ __device__ __forceinline__ int glob_axis(const GridP& g, int k, int l)
{
    int c = g.wlo[k] + l;
    if (c >= g.nc[k]) c -= g.nc[k];
    return c;
}
// local linear index (count / start / cell_of) of a cell given by global coordinates
__host__ __device__ __forceinline__ int cell_loc(const GridP& g, int cx, int cy, int cz)
{
    return loc_axis(g, 0, cx) + g.wn[0] * (loc_axis(g, 1, cy) + g.wn[1] * loc_axis(g, 2, cz));
}
// global linear index (owner / halo maps) of a cell given by global coordinates
__host__ __device__ __forceinline__ int cell_glob(const GridP& g, int cx, int cy, int cz)
{
    return cx + g.nc[0] * (cy + g.nc[1] * cz);
}

// cell index along axis k of a fixed-point coordinate: floor(u / E_k) by a
// multiply-high (exact for u < 2^32, E_k <= 2^23: the rounding excess of
// ceil(2^64 / E) is below 2^-9 / E, smaller than the gap 1 / E to the next integer)
__device__ __forceinline__ int cell_of_u(const GridP& g, int k, uint32_t u)
{
    return (int)__umul64hi((unsigned long long)u, g.Einv[k]);
}

// home cell t (0 <= t < nhome) of the rank's box, x fastest: LOCAL coordinates and index
__device__ __forceinline__ int home_cell(const GridP& g, int t, int& cx, int& cy, int& cz)
{
    cx = g.hlo[0] + t % g.hdim[0];
    cy = g.hlo[1] + (t / g.hdim[0]) % g.hdim[1];
    cz = g.hlo[2] + t / (g.hdim[0] * g.hdim[1]);
    return cx + g.wn[0] * (cy + g.wn[1] * cz);
}

// vel.w carries the component id (bits 0-7) and the ghost flag (bit 8) of
// a molecule held only as a halo copy on this rank (spatial decomposition)
__device__ __forceinline__ int md_comp(float w) { return __float_as_int(w) & 0xff; }
__device__ __forceinline__ bool md_ghost(float w) { return (__float_as_int(w) >> 8) & 1; }

// spatial decomposition: exchange record of one molecule
struct DDRec {
    uint4 pos;                   // global fixed-point position + id
    float4 vel;                  // v(t - dt/2), comp | ghost << 8
    float4 quat, angm;
};

struct DDArgs {
    int rank, nranks;
    const uint8_t* owner;        // owning rank of every global cell
    const uint32_t* gmask;       // bit r: cell is in rank r's halo (and not owned by r)
    DDRec* send;                 // nranks segments of seg_cap records
    int seg_cap;
    int* send_cnt;               // nranks counters
    int* flag;                   // bit 8: send segment overflow
    const int* n_dev;            // asynchronous step: molecule count in device memory (else the kernel's n)
    const int* seg_tab;          // per-peer segments: [0, nranks) offsets, [nranks, 2 nranks) capacities
                                 // (records); nullptr: uniform segments r * seg_cap of seg_cap records
    DDRec* const* put_rec = nullptr;   // direct puts: record k for rank r goes to put_rec[r][k] (this rank's
                                 // segment in r's receive buffer; peer memory), nullptr: own send buffer
    int* const* put_cnt = nullptr;     // direct puts: where this rank's count for rank r goes (fused kernels:
                                 // the last CTA to finish stores them)
    int* done = nullptr;               // fused kernels: CTA completion ticket (zero between launches)
    int* n_force = nullptr;            // fused kernels: the sorted count the forces were computed for
    bool peer_puts = false;            // put_rec points into other devices (CUDA IPC): a system-scope
                                       // fence orders each thread's record stores before it exits
};

// Pack this lane's exchange records (spatial decomposition): one record for every rank in
// dmask -- a halo copy (ghost flag, bit 8 of the component word) for the ranks whose halo
// holds the molecule's new cell, the molecule itself for its new owner `own`.  Warp-collective
// (every lane calls it, dmask = 0 for none): per destination one atomic reserves the warp's
// slots of that segment.  Overflow sets bit 8 of the flag.
__device__ __forceinline__ void dd_pack_warp(const DDArgs& dd, unsigned dmask, int own, uint4 pn, float4 vn,
                                             float4 qn, float4 jn)
{
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    for (int r = 0; r < dd.nranks; ++r) {
        const bool pr = (dmask >> r) & 1u;
        const unsigned b = __ballot_sync(0xffffffffu, pr);
        if (b == 0u) continue;
        const int leader = __ffs(b) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&dd.send_cnt[r], __popc(b));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (pr) {
            const int k = base + __popc(b & below);
            const int cap_r = dd.seg_tab ? dd.seg_tab[dd.nranks + r] : dd.seg_cap;
            const size_t off_r = dd.seg_tab ? (size_t)dd.seg_tab[r] : (size_t)r * dd.seg_cap;
            if (k >= cap_r) {
                atomicOr(dd.flag, 256);
            } else {
                DDRec rec;
                rec.pos = pn;
                rec.vel = r == own ? vn : make_float4(vn.x, vn.y, vn.z, __int_as_float((__float_as_int(vn.w) & 0xff) | 256));
                rec.quat = qn;
                rec.angm = jn;
                if (dd.put_rec) dd.put_rec[r][k] = rec;
                else dd.send[off_r + k] = rec;
            }
        }
    }
}

struct ObsRec {                  // one history entry (matches mardyn_observables order)
    long long step;
    double U, W, T, KEt, KEr;
    long long npairs, ncand;
};

struct ForcePartial {            // per warp / block of a force kernel
    double U, W;
    long long npairs, ncand;
    double K;                    // translational kinetic energy (force kernels that fuse the step)
};

// translational leapfrog of one molecule (Eqs. 2-3 with readings A9, A12):
// KE_t(t) from v(t) = v(t - dt/2) + dt/2 F/m, kick, fixed-point drift with
// periodic wrap, next cell.  Shared by k_integrate and the fused LJ1 step.
struct LeapOut {
    uint4 p;
    float4 v;
    int c[3];
    bool bad;
    double ket;
};
__device__ __forceinline__ LeapOut md_leapfrog(const GridP& g, uint4 p, float4 v, float Fx, float Fy, float Fz,
                                               float mass, float im)
{
    LeapOut o;
    const float dt = g.dt;
    const float vx = v.x + 0.5f * dt * Fx * im, vy = v.y + 0.5f * dt * Fy * im, vz = v.z + 0.5f * dt * Fz * im;
    o.ket = 0.5 * (double)mass * ((double)vx * vx + (double)vy * vy + (double)vz * vz);
    v.x += dt * Fx * im; v.y += dt * Fy * im; v.z += dt * Fz * im;
    const float vv[3] = {v.x, v.y, v.z};
    uint32_t uu[3] = {p.x, p.y, p.z};
    bool bad = !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float d = (dt * vv[k]) * g.inv_s;
        bad |= !(fabsf(d) < (float)g.E[k]);
        const long long du = bad ? 0 : __float2ll_rn(d);
        long long x = (long long)uu[k] + du;
        const long long P = (long long)g.P64[k];
        if (x < 0) x += P;
        else if (x >= P) x -= P;
        uu[k] = (uint32_t)x;
        o.c[k] = (int)__umul64hi((unsigned long long)uu[k], g.Einv[k]);
    }
    o.p = make_uint4(uu[0], uu[1], uu[2], p.w);
    o.v = v;
    o.bad = bad;
    return o;
}

__device__ __forceinline__ int warp_lane() { return threadIdx.x & 31; }

__device__ __forceinline__ double warp_sum_d(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum_f(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// body -> world rotation of vector b by unit quaternion q = (w,x,y,z)
__device__ __forceinline__ float3 qrot(float4 q, float bx, float by, float bz)
{
    const float w = q.x, x = q.y, y = q.z, z = q.w;
    float3 r;
    r.x = (1.f - 2.f * (y * y + z * z)) * bx + 2.f * (x * y - w * z) * by + 2.f * (x * z + w * y) * bz;
    r.y = 2.f * (x * y + w * z) * bx + (1.f - 2.f * (x * x + z * z)) * by + 2.f * (y * z - w * x) * bz;
    r.z = 2.f * (x * z - w * y) * bx + 2.f * (y * z + w * x) * by + (1.f - 2.f * (x * x + y * y)) * bz;
    return r;
}
// world -> body: R^T v
__device__ __forceinline__ float3 qrotT(float4 q, float3 v)
{
    const float w = q.x, x = q.y, y = q.z, z = q.w;
    float3 r;
    r.x = (1.f - 2.f * (y * y + z * z)) * v.x + 2.f * (x * y + w * z) * v.y + 2.f * (x * z - w * y) * v.z;
    r.y = 2.f * (x * y - w * z) * v.x + (1.f - 2.f * (x * x + z * z)) * v.y + 2.f * (y * z + w * x) * v.z;
    r.z = 2.f * (x * z + w * y) * v.x + 2.f * (y * z - w * x) * v.y + (1.f - 2.f * (x * x + y * y)) * v.z;
    return r;
}

// ---- helpers shared by the force kernels
__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// exact cutoff decision in quanta for separations in the guard band
__device__ __forceinline__ bool exact_in_range(float dx, float dy, float dz, const GridP& g)
{
    long long kx = __float2int_rn(dx * g.inv_s);
    long long ky = __float2int_rn(dy * g.inv_s);
    long long kz = __float2int_rn(dz * g.inv_s);
    return kx * kx + ky * ky + kz * kz < g.cut2_q;
}

__device__ __forceinline__ int wrapi(int c, int n) { return c < 0 ? c + n : (c >= n ? c - n : c); }
