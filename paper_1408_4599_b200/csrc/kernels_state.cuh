// kernels_state.cuh -- bandwidth kernels of the hot path: ingest (host
// doubles -> fixed point), per-step cell rebuild by counting sort
// (histogram fused into the integrator, exclusive scan, scatter, canonical
// in-cell order by id), leapfrog + Fincham integrator, deterministic
// reductions, egress.  All of them are HBM-bound.
#pragma once
#include "common.cuh"

// ------------------------------------------------------------------------
// ingest: host arrays (already on the device as doubles) -> state, cell and
// arrival rank (reading A12: u = rint(r/s) mod P, exact in fp64 because s is
// a power of two).
__global__ void k_ingest(int n, const double* __restrict__ r, const double* __restrict__ v,
                         const double* __restrict__ q, const double* __restrict__ j,
                         const int* __restrict__ comp, GridP g, uint4* __restrict__ pos,
                         float4* __restrict__ vel, float4* __restrict__ quat,
                         float4* __restrict__ angm, int* __restrict__ cell_of,
                         int* __restrict__ rank, int* __restrict__ count, int ncomp, int* __restrict__ flag,
                         const uint8_t* __restrict__ owner = nullptr,
                         const uint32_t* __restrict__ gmask = nullptr, int me = 0)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // input validation (mardyn.h: finite r, v; component in range; unit quaternions):
    // an invalid molecule is dropped and flags the call (MARDYN_EINVAL)
    bool ok = comp[i] >= 0 && comp[i] < ncomp;
#pragma unroll
    for (int k = 0; k < 3; ++k) ok = ok && isfinite(r[3 * i + k]) && isfinite(v[3 * i + k]);
    if (q) {
        const double qn = q[4 * i] * q[4 * i] + q[4 * i + 1] * q[4 * i + 1] + q[4 * i + 2] * q[4 * i + 2] +
                          q[4 * i + 3] * q[4 * i + 3];
        ok = ok && fabs(qn - 1.0) < 1e-5;
    }
    if (!ok) {
        atomicOr(flag, 512);
        cell_of[i] = -1;
        return;
    }
    uint32_t u[3];
    int c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        long long P = (long long)g.P64[k];
        long long x = __double2ll_rn(r[3 * i + k] / (double)g.s);
        x %= P;
        if (x < 0) x += P;
        u[k] = (uint32_t)x;
        c[k] = cell_of_u(g, k, u[k]);
    }
    const int cl0 = cell_glob(g, c[0], c[1], c[2]);
    int gflag = 0;
    if (owner) {                            // spatial decomposition: keep owned + halo molecules
        const bool ghost = (gmask[cl0] >> me) & 1u;
        if (owner[cl0] != me && !ghost) { cell_of[i] = -1; return; }
        gflag = ghost ? 256 : 0;
    }
    pos[i] = make_uint4(u[0], u[1], u[2], (uint32_t)i);
    vel[i] = make_float4((float)v[3 * i], (float)v[3 * i + 1], (float)v[3 * i + 2],
                         __int_as_float(comp[i] | gflag));
    if (quat) {
        quat[i] = q ? make_float4((float)q[4 * i], (float)q[4 * i + 1], (float)q[4 * i + 2], (float)q[4 * i + 3])
                    : make_float4(1.f, 0.f, 0.f, 0.f);
        angm[i] = j ? make_float4((float)j[3 * i], (float)j[3 * i + 1], (float)j[3 * i + 2], 0.f)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    int cl = cell_loc(g, c[0], c[1], c[2]);
    cell_of[i] = cl;
    rank[i] = atomicAdd(&count[cl], 1);
}

__global__ void k_iota64(int n, int64_t* __restrict__ a)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

// ------------------------------------------------------------------------
// exclusive scan of the per-cell counts.  Tiles of 1024 threads x PT consecutive
// cells: PT = 16 for large grids (a 4.1 M-cell grid (c4) is 252 tiles, one wave of
// the co-resident CTAs; 4096-cell tiles took four waves, ~80 us; the 0.55 M-cell window
// of a c4 rank at p = 8 is 34 tiles: 3 us less than 134), PT = 4 below 2^18 cells (c1's
// 85 k cells are 21 tiles; 16 k-cell tiles measured 3.5 us slower there)
#define SCAN_PT_MAX 16
#define SCAN_TILE (1024 * SCAN_PT_MAX)          // padding unit of the count array
#ifndef SCAN_PT_SMALL
#define SCAN_PT_SMALL 4
#endif
#ifndef SCAN_BIG_GRID
#define SCAN_BIG_GRID (1 << 18)
#endif

__device__ __forceinline__ int warp_incl_scan(int v)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// block-wide exclusive scan of one int per thread (blockDim = 1024)
__device__ __forceinline__ int block_excl_scan(int v, int* total)
{
    __shared__ int wsum[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = warp_incl_scan(v);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        int x = wsum[lane];
        int xi = warp_incl_scan(x);
        wsum[lane] = xi - x;
        if (lane == 31) *total = xi;
    }
    __syncthreads();
    int res = inc - v + wsum[w];
    __syncthreads();
    return res;
}

// Single-pass exclusive scan with decoupled look-back: tiles are claimed in
// order through a counter that is never reset (tile = ticket mod ntiles,
// epoch = ticket / ntiles + 1); each tile publishes (epoch, status, value),
// status 1 = its aggregate, 2 = its inclusive prefix, and walks back over
// its predecessors' values of the same epoch (an inclusive prefix ends the
// walk).  The counts are zeroed as they are read (the next step's binning
// starts from zero) and blk_ctr (the force kernel's block counter) is reset.
// start[ncell] = total.
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long scan_word(unsigned epoch, unsigned status, int value)
{
    return ((unsigned long long)epoch << 34) | ((unsigned long long)status << 32) | (unsigned)value;
}

template <int SCAN_PT>
__global__ void __launch_bounds__(1024) k_scan(int ncell, int* __restrict__ count, int* __restrict__ start,
                                               unsigned long long* __restrict__ flags,
                                               unsigned* __restrict__ tile_ctr, int* __restrict__ blk_ctr)
{
    __shared__ int tot, excl_s;
    __shared__ unsigned ticket_s;
    constexpr int TILE = 1024 * SCAN_PT;
    const int ntiles = (ncell + TILE - 1) / TILE;
    if (threadIdx.x == 0) ticket_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int tile = (int)(ticket_s % (unsigned)ntiles);
    const unsigned epoch = (ticket_s / (unsigned)ntiles + 1u) & 0x3fffffffu;
    if (tile == 0 && threadIdx.x == 0 && blk_ctr) *blk_ctr = 0;
    const int base = tile * TILE + threadIdx.x * SCAN_PT;
    int a[SCAN_PT];
    // count is padded to whole tiles (ncell_pad), so the vector loads never leave it
    if constexpr (SCAN_PT % 4 == 0) {
#pragma unroll
        for (int v = 0; v < SCAN_PT / 4; ++v) {
            const int4 c4 = *reinterpret_cast<const int4*>(count + base + 4 * v);
            a[4 * v] = c4.x; a[4 * v + 1] = c4.y; a[4 * v + 2] = c4.z; a[4 * v + 3] = c4.w;
        }
#pragma unroll
        for (int v = 0; v < SCAN_PT / 4; ++v) *reinterpret_cast<int4*>(count + base + 4 * v) = make_int4(0, 0, 0, 0);
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_PT; ++k) a[k] = count[base + k];
#pragma unroll
        for (int k = 0; k < SCAN_PT; ++k) count[base + k] = 0;
    }
    int sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PT; ++k) sum += a[k];
    int ex = block_excl_scan(sum, &tot);
    if (threadIdx.x < 32) {                  // warp 0: publish, then look back 32 tiles at a time
        const int lane = threadIdx.x;
        const int agg = tot;
        if (lane == 0) st_release_u64(flags + tile, scan_word(epoch, tile == 0 ? 2u : 1u, agg));
        int prefix = 0;
        for (int j = tile - 1; j >= 0; j -= 32) {
            const int jj = j - lane;                          // lane 0 nearest
            unsigned long long f = scan_word(epoch, 2u, 0);   // beyond tile 0: an empty inclusive prefix
            if (jj >= 0) {
                do { f = ld_acquire_u64(flags + jj); } while ((unsigned)(f >> 34) != epoch || ((f >> 32) & 3u) == 0);
            }
            const unsigned inc = __ballot_sync(0xffffffffu, ((f >> 32) & 3u) == 2u);
            const int stop = inc ? __ffs(inc) - 1 : 31;       // nearest inclusive prefix ends the walk
            int v = lane <= stop ? (int)(unsigned)(f & 0xffffffffu) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            prefix += v;
            if (inc) break;
        }
        if (lane == 0) {
            if (tile > 0) st_release_u64(flags + tile, scan_word(epoch, 2u, prefix + agg));
            excl_s = prefix;
            if (tile == ntiles - 1) start[ncell] = prefix + agg;
        }
    }
    __syncthreads();
    ex += excl_s;
    if (SCAN_PT % 4 == 0 && base + SCAN_PT <= ncell) {
#pragma unroll
        for (int v = 0; v < SCAN_PT / 4; ++v) {
            int4 o;
            o.x = ex; ex += a[4 * v];
            o.y = ex; ex += a[4 * v + 1];
            o.z = ex; ex += a[4 * v + 2];
            o.w = ex; ex += a[4 * v + 3];
            if ((((uintptr_t)(start + base)) & 15) == 0) *reinterpret_cast<int4*>(start + base + 4 * v) = o;
            else { start[base + 4 * v] = o.x; start[base + 4 * v + 1] = o.y; start[base + 4 * v + 2] = o.z; start[base + 4 * v + 3] = o.w; }
        }
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_PT; ++k) {
            if (base + k < ncell) start[base + k] = ex;
            ex += a[k];
        }
    }
}

// ------------------------------------------------------------------------
// scatter: canonical key (u_x << 32 | iid) and the unsorted index at
// start[cell] + arrival rank
__global__ void k_scatter(int n, const uint4* __restrict__ pos, const int* __restrict__ cell_of,
                          const int* __restrict__ rank, const int* __restrict__ start,
                          unsigned long long* __restrict__ keys, int* __restrict__ oldidx,
                          int* __restrict__ slot_cell,
                          const int* __restrict__ n_dev = nullptr)
{
    if (n_dev) n = *n_dev;                  // asynchronous decomposed step: count on the device
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int cl = cell_of[i];
        if (cl < 0) continue;               // dropped ghost or migrant (spatial decomposition)
        int slot = start[cl] + rank[i];
        const uint4 p = pos[i];
        keys[slot] = ((unsigned long long)p.x << 32) | p.w;
        oldidx[slot] = i;
        slot_cell[slot] = cl;               // the gather reads it coalesced (no dependent load)
    }
}

// canonical gather: each sorted slot finds its rank inside its cell in the
// canonical order (x, then id; reading A13 -- deterministic, and rows of
// three x-adjacent cells come out sorted by x, which the force kernels use
// to prune candidates), then gathers the molecule's state from the unsorted arrays
// and writes the staging copy (cell-relative coordinates, exact) and, for
// rigid models, the world-frame site offsets s = R(q) d.
template <bool RIGID>
__device__ __forceinline__ void canon_one(int t, int cap, const GridP& g, const unsigned long long* __restrict__ keys,
                        const int* __restrict__ oldidx, const int* __restrict__ slot_cell,
                        const int* __restrict__ start,
                        const uint4* __restrict__ pos_s, const float4* __restrict__ vel_s,
                        const float4* __restrict__ quat_s, const float4* __restrict__ angm_s,
                        uint4* __restrict__ pos_d, float4* __restrict__ vel_d,
                        float4* __restrict__ quat_d, float4* __restrict__ angm_d,
                        float4* __restrict__ xs, float4* __restrict__ site,
                        const DevModel* __restrict__ model)
{
    const unsigned long long key = keys[t];
    const int old = oldidx[t];
    int c = slot_cell[t];
    int s0 = start[c], s1 = start[c + 1];
    int r = 0;
    for (int m = s0; m < s1; ++m) r += keys[m] < key;
    int dst = s0 + r;
    MD_CHECK(dst >= 0 && dst < cap && old >= 0 && old < cap && r < s1 - s0);
    uint4 p = pos_s[old];
    float4 v = vel_s[old];
    pos_d[dst] = p;
    vel_d[dst] = v;
    // the slot's cell: local (window) coordinates, and the global ones of its origin
    const int lx = c % g.wn[0];
    const int ly = (c / g.wn[0]) % g.wn[1];
    const int lz = c / (g.wn[0] * g.wn[1]);
    const int cx = glob_axis(g, 0, lx), cy = glob_axis(g, 1, ly), cz = glob_axis(g, 2, lz);
    float4 x;
    x.x = (float)(int)(p.x - (uint32_t)cx * g.E[0]) * g.s;    // exact (A12)
    x.y = (float)(int)(p.y - (uint32_t)cy * g.E[1]) * g.s;
    x.z = (float)(int)(p.z - (uint32_t)cz * g.E[2]) * g.s;
    // rigid kernels: component bits; single-site kernel: the cell's local x index
    // (it rebuilds sub-chunk-relative x = xs.x + (cx - c_origin) * edge exactly)
    x.w = RIGID ? __int_as_float(md_comp(v.w)) : (float)lx;
    xs[dst] = x;
    if (RIGID) {
        float4 q = quat_s[old];
        quat_d[dst] = q;
        angm_d[dst] = angm_s[old];
        const DevComp& C = model->comp[md_comp(v.w)];
        int ns = C.n_lj + C.n_q;
        for (int k = 0; k < ns; ++k) {
            float3 w = qrot(q, C.bpos[k][0], C.bpos[k][1], C.bpos[k][2]);
            site[(size_t)k * cap + dst] = make_float4(w.x, w.y, w.z, C.mom[k]);
        }
        int np = C.n_mu + C.n_Q;
        for (int k = 0; k < np; ++k) {
            int sidx = ns + k;
            float3 w = qrot(q, C.bpos[sidx][0], C.bpos[sidx][1], C.bpos[sidx][2]);
            float3 e = qrot(q, C.baxis[sidx][0], C.baxis[sidx][1], C.baxis[sidx][2]);
            site[(size_t)(ns + 2 * k) * cap + dst] = make_float4(w.x, w.y, w.z, C.mom[sidx]);
            site[(size_t)(ns + 2 * k + 1) * cap + dst] = make_float4(e.x, e.y, e.z, 0.f);
        }
    }
}

// grid-stride over the sorted slots (the asynchronous decomposed step launches a
// capacity-independent grid)
template <bool RIGID>
__global__ void k_canon(int n, int cap, GridP g, const unsigned long long* __restrict__ keys,
                        const int* __restrict__ oldidx, const int* __restrict__ slot_cell,
                        const int* __restrict__ start,
                        const uint4* __restrict__ pos_s, const float4* __restrict__ vel_s,
                        const float4* __restrict__ quat_s, const float4* __restrict__ angm_s,
                        uint4* __restrict__ pos_d, float4* __restrict__ vel_d,
                        float4* __restrict__ quat_d, float4* __restrict__ angm_d,
                        float4* __restrict__ xs, float4* __restrict__ site,
                        const DevModel* __restrict__ model)
{
    const int lim = min(n, start[g.wncell]);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < lim; t += gridDim.x * blockDim.x)
        canon_one<RIGID>(t, cap, g, keys, oldidx, slot_cell, start, pos_s, vel_s, quat_s, angm_s, pos_d, vel_d,
                         quat_d, angm_d, xs, site, model);
}

// ------------------------------------------------------------------------
// integrator (Eqs. 2-5 with readings A7, A9, A12), in place on the sorted
// state; fuses the next step's cell binning (histogram + arrival rank) and
// the kinetic-energy partials (per block, fixed order, fp64).
__device__ __forceinline__ float4 qmul(float4 a, float4 b)
{
    return make_float4(a.x * b.x - a.y * b.y - a.z * b.z - a.w * b.w,
                       a.x * b.y + a.y * b.x + a.z * b.w - a.w * b.z,
                       a.x * b.z - a.y * b.w + a.z * b.x + a.w * b.y,
                       a.x * b.w + a.y * b.z - a.z * b.y + a.w * b.x);
}
__device__ __forceinline__ float4 qnormalize(float4 q)
{
    float s = rsqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    return make_float4(q.x * s, q.y * s, q.z * s, q.w * s);
}

template <int NT>
__device__ __forceinline__ void block_sum2_d(double a, double b, double* out_a, double* out_b)
{
    __shared__ double sa[NT / 32], sb[NT / 32];
    a = warp_sum_d(a);
    b = warp_sum_d(b);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sa[w] = a; sb[w] = b; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0, y = 0;
        for (int k = 0; k < NT / 32; ++k) { x += sa[k]; y += sb[k]; }
        *out_a = x; *out_b = y;
    }
}

// DD = spatial decomposition: ghosts are skipped and
// dropped; an owned molecule whose new cell belongs to another rank is
// packed as a migrant for it (and dropped here); an owned molecule whose new
// cell lies in other ranks' halos is also packed as a ghost for each of them.
template <bool RIGID, bool DD = false>
__global__ void __launch_bounds__(256) k_integrate(int n, GridP g, const DevModel* __restrict__ model,
                                                   uint4* __restrict__ pos, float4* __restrict__ vel,
                                                   float4* __restrict__ quat, float4* __restrict__ angm,
                                                   const float4* __restrict__ force,
                                                   const float4* __restrict__ torque,
                                                   int* __restrict__ cell_of, int* __restrict__ rank,
                                                   int* __restrict__ count, double* __restrict__ ke_part,
                                                   int* __restrict__ flag, DDArgs dd = DDArgs())
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (DD && dd.n_dev) n = *dd.n_dev;      // asynchronous decomposed step: count on the device
    double ket = 0.0, ker = 0.0;
    int cl_bin = -1;
    bool ghost = false;
    unsigned dmask = 0;                                // DD: ranks this molecule is sent to
    int own = -1;
    uint4 pn = make_uint4(0, 0, 0, 0);
    float4 vn = make_float4(0.f, 0.f, 0.f, 0.f), qn = vn, jn = vn;
    if (DD && t < n) {
        ghost = md_ghost(vel[t].w);
        if (ghost) cell_of[t] = -1;
    }
    if (t < n && !ghost) {
        uint4 p = pos[t];
        float4 v = vel[t];
        float4 F = force[t];
        const DevComp& C = model->comp[md_comp(v.w)];
        const float dt = g.dt;
        const LeapOut lo = md_leapfrog(g, p, v, F.x, F.y, F.z, C.mass, C.inv_mass);
        ket = lo.ket;
        int c[3] = {lo.c[0], lo.c[1], lo.c[2]};
        if (lo.bad) atomicOr(flag, 1);
        pos[t] = lo.p;
        vel[t] = lo.v;
        if (RIGID && C.rot) {
            // Fincham rotational leapfrog (reading A7 of Eqs. 4-5)
            float4 q = quat[t];
            float4 jh = angm[t];
            float4 tq = torque[t];
            float3 jt = make_float3(jh.x + 0.5f * dt * tq.x, jh.y + 0.5f * dt * tq.y, jh.z + 0.5f * dt * tq.z);
            float3 jb = qrotT(q, jt);
            float3 wb = make_float3(jb.x * C.invI[0], jb.y * C.invI[1], jb.z * C.invI[2]);
            ker = 0.5 * ((double)jb.x * wb.x + (double)jb.y * wb.y + (double)jb.z * wb.z);
            float4 dq = qmul(q, make_float4(0.f, wb.x, wb.y, wb.z));
            float4 qh = qnormalize(make_float4(q.x + 0.25f * dt * dq.x, q.y + 0.25f * dt * dq.y,
                                               q.z + 0.25f * dt * dq.z, q.w + 0.25f * dt * dq.w));
            float3 jn = make_float3(jh.x + dt * tq.x, jh.y + dt * tq.y, jh.z + dt * tq.z);
            float3 jb2 = qrotT(qh, jn);
            float3 wb2 = make_float3(jb2.x * C.invI[0], jb2.y * C.invI[1], jb2.z * C.invI[2]);
            float4 dq2 = qmul(qh, make_float4(0.f, wb2.x, wb2.y, wb2.z));
            float4 qn = qnormalize(make_float4(q.x + 0.5f * dt * dq2.x, q.y + 0.5f * dt * dq2.y,
                                               q.z + 0.5f * dt * dq2.z, q.w + 0.5f * dt * dq2.w));
            quat[t] = qn;
            angm[t] = make_float4(jn.x, jn.y, jn.z, 0.f);
            if (!(isfinite(jn.x) && isfinite(jn.y) && isfinite(jn.z))) atomicOr(flag, 1);
        }
        const int clg = cell_glob(g, c[0], c[1], c[2]);     // owner / halo maps
        int cl = cell_loc(g, c[0], c[1], c[2]);             // count / cell_of (rank-local window)
        if (DD) {
            pn = pos[t];
            vn = vel[t];
            qn = RIGID ? quat[t] : make_float4(1.f, 0.f, 0.f, 0.f);
            jn = RIGID ? angm[t] : make_float4(0.f, 0.f, 0.f, 0.f);
            own = dd.owner[clg];
            // halo copies for the other ranks whose halo holds the new cell; the record for the
            // new owner (migrant) if that is another rank -- packed below, one atomic per warp
            // and destination
            dmask = (dd.gmask[clg] & ~(1u << dd.rank)) | (own != dd.rank ? 1u << own : 0u);
            if (own != dd.rank) {                          // migrant
                if ((dd.gmask[clg] >> dd.rank) & 1u) {     // its new cell is in my halo: keep a copy
                    vel[t] = make_float4(vn.x, vn.y, vn.z, __int_as_float(md_comp(vn.w) | 256));
                } else {
                    cell_of[t] = -1;
                    cl = -1;
                }
            }
        }
        if (cl >= 0) cell_of[t] = cl;
        cl_bin = cl;
    }
    if (DD) {
        dd_pack_warp(dd, dmask, own, pn, vn, qn, jn);   // warp-aggregated (one atomic per destination)
        if (dd.peer_puts) __threadfence_system();       // receivers on other GPUs (IPC puts)
    }
    // next step's cell histogram + arrival rank: molecules are in cell order, so
    // the lanes of a warp share few cells; one atomic per distinct cell (the arrival
    // order only places molecules before the canonical in-cell ordering)
    const unsigned m = __match_any_sync(0xffffffffu, cl_bin);
    if (cl_bin >= 0) {
        const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
        int b = 0;
        if (lane == leader) b = atomicAdd(&count[cl_bin], __popc(m));
        b = __shfl_sync(m, b, leader);
        rank[t] = b + __popc(m & ((1u << lane) - 1u));
    }
    block_sum2_d<256>(ket, ker, &ke_part[2 * blockIdx.x], &ke_part[2 * blockIdx.x + 1]);
}

// import n exchange records (migrants and ghosts) at unsorted slots
// base .. base + n - 1 and bin them
__global__ void k_import(int n, int base, GridP g, const DDRec* __restrict__ recv, uint4* __restrict__ pos,
                         float4* __restrict__ vel, float4* __restrict__ quat, float4* __restrict__ angm,
                         int* __restrict__ cell_of, int* __restrict__ rank, int* __restrict__ count)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const DDRec r = recv[k];
    const int t = base + k;
    pos[t] = r.pos;
    vel[t] = r.vel;
    if (quat) { quat[t] = r.quat; angm[t] = r.angm; }
    const int cl = cell_loc(g, cell_of_u(g, 0, r.pos.x), cell_of_u(g, 1, r.pos.y), cell_of_u(g, 2, r.pos.z));
    cell_of[t] = cl;
    rank[t] = atomicAdd(&count[cl], 1);
}

// asynchronous decomposed step: import the records of the fixed receive
// segments (segment r = records from rank r, recv_cnt[r] of them, at most
// seg_cap) after the n_old = *n_old_dev molecules kept in place, bin them, and
// write the unsorted count for the cell rebuild.  Nothing goes to the host.
// rtab: per-source segments ([0, nranks) offsets, [nranks, 2 nranks) capacities), or
// nullptr for uniform segments r * seg_cap of seg_cap records; the grid covers the
// sum of the capacities
// direct puts: this rank's record counts into the receiving ranks' count arrays (peer memory)
__global__ void k_put_counts(int nranks, const int* __restrict__ send_cnt, int* const* __restrict__ put_cnt)
{
    const int r = threadIdx.x;
    __threadfence_system();                     // receivers on other GPUs (IPC puts)
    if (r < nranks) *put_cnt[r] = send_cnt[r];
}

__global__ void k_import_seg(int nranks, int seg_cap, const int* __restrict__ rtab, const int* __restrict__ recv_cnt,
                             const int* __restrict__ n_old_dev, int cap, GridP g, const DDRec* __restrict__ recv,
                             uint4* __restrict__ pos, float4* __restrict__ vel, float4* __restrict__ quat,
                             float4* __restrict__ angm, int* __restrict__ cell_of, int* __restrict__ rank,
                             int* __restrict__ count, int* __restrict__ n_unsorted, int* __restrict__ flag,
                             int* __restrict__ send_cnt = nullptr)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_old = *n_old_dev;
    if (send_cnt && t < nranks) send_cnt[t] = 0;       // consumed by this step's exchange: ready for the next
    int r = nranks, k = 0, base = n_old, tot = n_old;
    for (int q = 0; q < nranks; ++q) {
        const int off = rtab ? rtab[q] : q * seg_cap, cq = rtab ? rtab[nranks + q] : seg_cap;
        const int c = min(recv_cnt[q], cq);
        if (t >= off && t < off + cq) { r = q; k = t - off; }
        if (r == nranks) base += c;                       // sources before r
        tot += c;
    }
    if (t == 0) {
        if (tot > cap) atomicOr(flag, 512);
        *n_unsorted = min(tot, cap);
    }
    if (r >= nranks) return;
    const int cr = rtab ? rtab[nranks + r] : seg_cap;
    if (k >= min(recv_cnt[r], cr)) return;
    const int slot = base + k;
    if (slot >= cap) return;
    const DDRec rec = recv[(size_t)t];
    pos[slot] = rec.pos;
    vel[slot] = rec.vel;
    if (quat) { quat[slot] = rec.quat; angm[slot] = rec.angm; }
    const int cl = cell_loc(g, cell_of_u(g, 0, rec.pos.x), cell_of_u(g, 1, rec.pos.y), cell_of_u(g, 2, rec.pos.z));
    cell_of[slot] = cl;
    rank[slot] = atomicAdd(&count[cl], 1);
}

// ------------------------------------------------------------------------
// spatial decomposition (§4)

// decomposed ingest of one chunk of the GLOBAL arrays (molecules base .. base + m - 1,
// already on the device): the molecules of this rank's box and halo are kept at compacted
// slots (one atomic per warp), quantised and binned; iid = global index.  Invalid input
// sets bit 512 of the flag, more kept molecules than the capacity bit 1024.
__global__ void k_ingest_dd(int m, int base, const double* __restrict__ r, const double* __restrict__ v,
                            const double* __restrict__ q, const double* __restrict__ j,
                            const int* __restrict__ comp, GridP g, uint4* __restrict__ pos,
                            float4* __restrict__ vel, float4* __restrict__ quat, float4* __restrict__ angm,
                            int* __restrict__ cell_of, int* __restrict__ rank, int* __restrict__ count,
                            int ncomp, int* __restrict__ flag, const uint8_t* __restrict__ owner,
                            const uint32_t* __restrict__ gmask, int me, int* __restrict__ n_kept, int cap)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    bool keep = false, ghost = false;
    uint32_t u[3] = {0, 0, 0};
    int cl = -1;
    if (i < m) {
        bool ok = comp[i] >= 0 && comp[i] < ncomp;
#pragma unroll
        for (int k = 0; k < 3; ++k) ok = ok && isfinite(r[3 * i + k]) && isfinite(v[3 * i + k]);
        if (q) {
            const double qn = q[4 * i] * q[4 * i] + q[4 * i + 1] * q[4 * i + 1] + q[4 * i + 2] * q[4 * i + 2] +
                              q[4 * i + 3] * q[4 * i + 3];
            ok = ok && fabs(qn - 1.0) < 1e-5;
        }
        if (!ok) {
            atomicOr(flag, 512);
        } else {
            int c[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const long long P = (long long)g.P64[k];
                long long x = __double2ll_rn(r[3 * i + k] / (double)g.s);
                x %= P;
                if (x < 0) x += P;
                u[k] = (uint32_t)x;
                c[k] = cell_of_u(g, k, u[k]);
            }
            const int clg = cell_glob(g, c[0], c[1], c[2]);
            ghost = (gmask[clg] >> me) & 1u;
            keep = owner[clg] == me || ghost;
            if (keep) cl = cell_loc(g, c[0], c[1], c[2]);
        }
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    int slot0 = 0;
    if (b && lane == __ffs(b) - 1) slot0 = atomicAdd(n_kept, __popc(b));
    slot0 = __shfl_sync(0xffffffffu, slot0, __ffs(b ? b : 1u) - 1);
    if (!keep) return;
    const int slot = slot0 + __popc(b & ((1u << lane) - 1u));
    if (slot >= cap) { atomicOr(flag, 1024); return; }
    pos[slot] = make_uint4(u[0], u[1], u[2], (uint32_t)(base + i));
    vel[slot] = make_float4((float)v[3 * i], (float)v[3 * i + 1], (float)v[3 * i + 2],
                            __int_as_float(comp[i] | (ghost ? 256 : 0)));
    if (quat) {
        quat[slot] = q ? make_float4((float)q[4 * i], (float)q[4 * i + 1], (float)q[4 * i + 2], (float)q[4 * i + 3])
                       : make_float4(1.f, 0.f, 0.f, 0.f);
        angm[slot] = j ? make_float4((float)j[3 * i], (float)j[3 * i + 1], (float)j[3 * i + 2], 0.f)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    cell_of[slot] = cl;
    rank[slot] = atomicAdd(&count[cl], 1);
}

// per-cell molecule counts of the cells this rank owns (0 elsewhere) from the last cell
// rebuild: the measured load of the rebalance (Eq. 6 input, reading A19)
__global__ void k_owned_counts(GridP g, const int* __restrict__ start, const uint8_t* __restrict__ owner,
                               int me, int* __restrict__ out)
{
    // over the rank-local window (out[] is zero elsewhere), written per global cell
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= g.wncell) return;
    const int lx = l % g.wn[0], ly = (l / g.wn[0]) % g.wn[1], lz = l / (g.wn[0] * g.wn[1]);
    const int c = cell_glob(g, glob_axis(g, 0, lx), glob_axis(g, 1, ly), glob_axis(g, 2, lz));
    if (owner[c] == me) out[c] = start[l + 1] - start[l];
}

// Rebalance: re-distribute the sorted state under the new cell
// owners / halo masks.  Every molecule this rank owned is sent to its new owner (if
// another rank) and as a halo copy to every rank whose new halo holds its cell; it stays
// here as an owned molecule or a halo copy, or leaves.  The old halo copies are dropped
// (their owners send the new ones).  COUNT: records per destination only (send_cnt);
// else the records are packed at the per-destination offsets of dd.seg_tab and the kept
// molecules binned for the cell rebuild.  No time passes (v, j stay at t - dt/2).
template <bool COUNT>
__global__ void k_repartition(int n, GridP g, DDArgs dd, const uint4* __restrict__ pos, float4* __restrict__ vel,
                              const float4* __restrict__ quat, const float4* __restrict__ angm,
                              int* __restrict__ cell_of, int* __restrict__ rank, int* __restrict__ count)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    unsigned dmask = 0;
    int own = -1, cl = -1;
    uint4 p = make_uint4(0, 0, 0, 0);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f), qn = make_float4(1.f, 0.f, 0.f, 0.f), jn = v;
    if (t < n) {
        v = vel[t];
        if (!md_ghost(v.w)) {
            p = pos[t];
            const int gx = cell_of_u(g, 0, p.x), gy = cell_of_u(g, 1, p.y), gz = cell_of_u(g, 2, p.z);
            const int clg = cell_glob(g, gx, gy, gz);
            own = dd.owner[clg];
            const uint32_t gm = dd.gmask[clg];
            dmask = (gm & ~(1u << dd.rank)) | (own != dd.rank ? 1u << own : 0u);
            if (quat) { qn = quat[t]; jn = angm[t]; }
            if (!COUNT) {
                cl = cell_loc(g, gx, gy, gz);                // in the NEW window
                if (own == dd.rank) {
                    vel[t] = make_float4(v.x, v.y, v.z, __int_as_float(md_comp(v.w)));
                } else if ((gm >> dd.rank) & 1u) {
                    vel[t] = make_float4(v.x, v.y, v.z, __int_as_float(md_comp(v.w) | 256));
                } else {
                    cl = -1;
                }
            }
        }
    }
    if (COUNT) {
        for (int r = 0; r < dd.nranks; ++r) {
            const unsigned b = __ballot_sync(0xffffffffu, (dmask >> r) & 1u);
            if (b && lane == 0) atomicAdd(&dd.send_cnt[r], __popc(b));
        }
        return;
    }
    if (t < n) cell_of[t] = cl;
    const float4 vn = make_float4(v.x, v.y, v.z, __int_as_float(md_comp(v.w)));
    dd_pack_warp(dd, dmask, own, p, vn, qn, jn);
    const unsigned m = __match_any_sync(0xffffffffu, cl);
    if (cl >= 0) {
        const int leader = __ffs(m) - 1;
        int b = 0;
        if (lane == leader) b = atomicAdd(&count[cl], __popc(m));
        b = __shfl_sync(m, b, leader);
        rank[t] = b + __popc(m & ((1u << lane) - 1u));
    }
}

// decomposed egress: this rank's owned molecules, compacted (one atomic per warp) into
// records of rec_words doubles: iid, then the requested fields (the host orders by iid)
__global__ void k_egress_dd(int n, GridP g, const uint4* __restrict__ pos, const float4* __restrict__ vel,
                            const float4* __restrict__ quat, const float4* __restrict__ angm,
                            const float4* __restrict__ force, const float4* __restrict__ torque,
                            unsigned fields, int rec_words, double* __restrict__ out, int* __restrict__ ctr)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool on = t < n && !md_ghost(vel[t].w);
    const unsigned b = __ballot_sync(0xffffffffu, on);
    int k0 = 0;
    if (b && lane == __ffs(b) - 1) k0 = atomicAdd(ctr, __popc(b));
    k0 = __shfl_sync(0xffffffffu, k0, __ffs(b ? b : 1u) - 1);
    if (!on) return;
    double* o = out + (size_t)(k0 + __popc(b & ((1u << lane) - 1u))) * rec_words;
    const uint4 p = pos[t];
    int w = 0;
    o[w++] = (double)p.w;
    if (fields & 1) { o[w++] = (double)p.x * g.s; o[w++] = (double)p.y * g.s; o[w++] = (double)p.z * g.s; }
    if (fields & 2) { const float4 x = vel[t]; o[w++] = x.x; o[w++] = x.y; o[w++] = x.z; }
    if (fields & 4) {
        const float4 x = quat ? quat[t] : make_float4(1.f, 0.f, 0.f, 0.f);
        o[w++] = x.x; o[w++] = x.y; o[w++] = x.z; o[w++] = x.w;
    }
    if (fields & 8) { const float4 x = angm ? angm[t] : make_float4(0.f, 0.f, 0.f, 0.f); o[w++] = x.x; o[w++] = x.y; o[w++] = x.z; }
    if (fields & 16) { const float4 x = force[t]; o[w++] = x.x; o[w++] = x.y; o[w++] = x.z; }
    if (fields & 32) { const float4 x = torque ? torque[t] : make_float4(0.f, 0.f, 0.f, 0.f); o[w++] = x.x; o[w++] = x.y; o[w++] = x.z; }
    if (fields & 64) { o[w++] = (double)p.x; o[w++] = (double)p.y; o[w++] = (double)p.z; }
    if (fields & 128)
        o[w++] = (double)(cell_of_u(g, 0, p.x) + g.nc[0] * (cell_of_u(g, 1, p.y) + g.nc[1] * cell_of_u(g, 2, p.z)));
}

// kinetic energy at t without integrating (compute_forces, A9)
template <bool RIGID>
__global__ void __launch_bounds__(256) k_kinetic(int n, GridP g, const DevModel* __restrict__ model,
                                                 const float4* __restrict__ vel,
                                                 const float4* __restrict__ quat,
                                                 const float4* __restrict__ angm,
                                                 const float4* __restrict__ force,
                                                 const float4* __restrict__ torque,
                                                 double* __restrict__ ke_part)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    double ket = 0.0, ker = 0.0;
    if (t < n && !md_ghost(vel[t].w)) {
        float4 v = vel[t];
        float4 F = force[t];
        const DevComp& C = model->comp[md_comp(v.w)];
        const float dt = g.dt, im = C.inv_mass;
        float vx = v.x + 0.5f * dt * F.x * im, vy = v.y + 0.5f * dt * F.y * im,
              vz = v.z + 0.5f * dt * F.z * im;
        ket = 0.5 * (double)C.mass * ((double)vx * vx + (double)vy * vy + (double)vz * vz);
        if (RIGID && C.rot) {
            float4 q = quat[t], jh = angm[t], tq = torque[t];
            float3 jt = make_float3(jh.x + 0.5f * dt * tq.x, jh.y + 0.5f * dt * tq.y, jh.z + 0.5f * dt * tq.z);
            float3 jb = qrotT(q, jt);
            ker = 0.5 * ((double)jb.x * jb.x * C.invI[0] + (double)jb.y * jb.y * C.invI[1] +
                         (double)jb.z * jb.z * C.invI[2]);
        }
    }
    block_sum2_d<256>(ket, ker, &ke_part[2 * blockIdx.x], &ke_part[2 * blockIdx.x + 1]);
}

// backward half kick of the initial on-step velocities (reading A8)
template <bool RIGID>
__global__ void k_half_kick(int n, GridP g, const DevModel* __restrict__ model, float4* __restrict__ vel,
                            float4* __restrict__ angm, const float4* __restrict__ force,
                            const float4* __restrict__ torque)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    float4 v = vel[t];
    float4 F = force[t];
    const DevComp& C = model->comp[md_comp(v.w)];
    const float h = 0.5f * g.dt;
    v.x -= h * F.x * C.inv_mass; v.y -= h * F.y * C.inv_mass; v.z -= h * F.z * C.inv_mass;
    vel[t] = v;
    if (RIGID && C.rot) {
        float4 j = angm[t], tq = torque[t];
        angm[t] = make_float4(j.x - h * tq.x, j.y - h * tq.y, j.z - h * tq.z, 0.f);
    }
}

// observables of one time t_k: fixed-order sums of the per-warp / per-block
// force partials and the per-block kinetic partials, written to the ring
// buffer.  FIN_BLOCKS blocks each sum a fixed contiguous range (fixed
// thread order, fixed tree); the last block to finish (ticket) adds the
// block results in block order -- the result does not depend on timing.
#define FIN_BLOCKS 48
#define FIN_THREADS 256
struct FinPart {
    double U, W, Kt, Kr;
    long long np, nc;
};

__device__ __forceinline__ void block_sum_fin(FinPart& v)
{
    __shared__ FinPart sp[FIN_THREADS / 32];
    v.U = warp_sum_d(v.U); v.W = warp_sum_d(v.W); v.Kt = warp_sum_d(v.Kt); v.Kr = warp_sum_d(v.Kr);
    v.np = warp_sum_ll(v.np); v.nc = warp_sum_ll(v.nc);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sp[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        FinPart o = sp[0];
        for (int k = 1; k < FIN_THREADS / 32; ++k) {
            o.U += sp[k].U; o.W += sp[k].W; o.Kt += sp[k].Kt; o.Kr += sp[k].Kr; o.np += sp[k].np; o.nc += sp[k].nc;
        }
        v = o;
    }
}

__global__ void __launch_bounds__(FIN_THREADS) k_finalize(int nfp, const ForcePartial* __restrict__ fp,
                                                          int nkp, const double* __restrict__ kp,
                                                          double ndof, long long* __restrict__ step_ctr,
                                                          int advance, ObsRec* __restrict__ hist,
                                                          FinPart* __restrict__ scratch, int* __restrict__ ticket,
                                                          int halve = 1)
{
    FinPart v{0, 0, 0, 0, 0, 0};
    const int cf = (nfp + FIN_BLOCKS - 1) / FIN_BLOCKS, ck = (nkp + FIN_BLOCKS - 1) / FIN_BLOCKS;
    const int f0 = blockIdx.x * cf, f1 = min(f0 + cf, nfp), k0 = blockIdx.x * ck, k1 = min(k0 + ck, nkp);
    for (int k = f0 + threadIdx.x; k < f1; k += FIN_THREADS) {
        const ForcePartial f = fp[k];
        v.U += f.U; v.W += f.W; v.np += f.npairs; v.nc += f.ncand; v.Kt += f.K;
    }
    for (int k = k0 + threadIdx.x; k < k1; k += FIN_THREADS) {
        const double2 q = reinterpret_cast<const double2*>(kp)[k];
        v.Kt += q.x; v.Kr += q.y;
    }
    block_sum_fin(v);
    __shared__ int last;
    if (threadIdx.x == 0) {
        scratch[blockIdx.x] = v;
        __threadfence();
        last = atomicAdd(ticket, 1) == FIN_BLOCKS - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    FinPart w{0, 0, 0, 0, 0, 0};
    if (threadIdx.x < FIN_BLOCKS) {
        const volatile FinPart* sv = scratch + threadIdx.x;
        w.U = sv->U; w.W = sv->W; w.Kt = sv->Kt; w.Kr = sv->Kr; w.np = sv->np; w.nc = sv->nc;
    }
    block_sum_fin(w);
    if (threadIdx.x == 0) {
        ObsRec o;
        o.U = w.U; o.W = w.W; o.KEt = w.Kt; o.KEr = w.Kr; o.npairs = w.np; o.ncand = w.nc;
        if (halve) o.npairs /= 2;            // full shell sees every pair twice (a decomposed
                                             // rank reports ordered pairs of its owned molecules)
        o.T = 2.0 * (o.KEt + o.KEr) / ndof;
        const long long st = *step_ctr;
        o.step = st;
        hist[st % MD_HISTORY] = o;
        if (advance) *step_ctr = st + 1;
        *ticket = 0;
    }
}

// NVT velocity rescaling ("kept constant by velocity rescaling";
// reading A24): after the finalize of step k (step_ctr = k + 1), if
// (k + 1) % interval == 0 the half-step velocities and angular momenta are
// scaled by lambda = sqrt(T_target / T(t_k)).
__global__ void k_rescale(int n, float4* __restrict__ vel, float4* __restrict__ angm,
                          const ObsRec* __restrict__ hist, const long long* __restrict__ step_ctr,
                          double T_target, int interval, int* __restrict__ flag)
{
    const long long k = *step_ctr - 1;
    if (k < 0 || (k + 1) % interval != 0) return;
    const double T = hist[k % MD_HISTORY].T;
    if (!(T > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flag, 1);
        return;
    }
    const float lam = (float)sqrt(T_target / T);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    float4 v = vel[t];
    v.x *= lam; v.y *= lam; v.z *= lam;
    vel[t] = v;
    if (angm) {
        float4 j = angm[t];
        j.x *= lam; j.y *= lam; j.z *= lam;
        angm[t] = j;
    }
}

// NVT on a decomposed run (reading A24 with the GLOBAL temperature): ke[0..1] = the
// global KE_t, KE_r of step k (summed over the ranks); every molecule this rank holds
// (owned + halo copies; the copies are refreshed by the next exchange anyway) is scaled
// by lambda = sqrt(T_target / T(t_k)), T = 2 (KE_t + KE_r) / N_dof.
__global__ void k_ke_entry(const ObsRec* __restrict__ hist, long long k, double* __restrict__ ke)
{
    if (threadIdx.x == 0) {
        const ObsRec& o = hist[k % MD_HISTORY];
        ke[0] = o.KEt;
        ke[1] = o.KEr;
    }
}
__global__ void k_ke_sum(int p, const ObsRec* const* __restrict__ hists, long long k, double* __restrict__ ke)
{
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int r = 0; r < p; ++r) {              // rank order: deterministic
            a += hists[r][k % MD_HISTORY].KEt;
            b += hists[r][k % MD_HISTORY].KEr;
        }
        ke[0] = a;
        ke[1] = b;
    }
}
__global__ void k_rescale_global(int cap, const int* __restrict__ n_dev, float4* __restrict__ vel,
                                 float4* __restrict__ angm, const double* __restrict__ ke, double ndof,
                                 double T_target, int* __restrict__ flag)
{
    const double T = 2.0 * (ke[0] + ke[1]) / ndof;
    if (!(T > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flag, 1);
        return;
    }
    const float lam = (float)sqrt(T_target / T);
    const int n = min(*n_dev, cap);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        float4 v = vel[t];
        v.x *= lam; v.y *= lam; v.z *= lam;
        vel[t] = v;
        if (angm) {
            float4 j = angm[t];
            j.x *= lam; j.y *= lam; j.z *= lam;
            angm[t] = j;
        }
    }
}

// ------------------------------------------------------------------------
// egress: sorted state -> caller order (index = iid), doubles
template <bool RIGID>
__global__ void k_egress(int n, GridP g, const uint4* __restrict__ pos, const float4* __restrict__ vel,
                         const float4* __restrict__ quat, const float4* __restrict__ angm,
                         const float4* __restrict__ force, const float4* __restrict__ torque,
                         double* __restrict__ r, double* __restrict__ v, double* __restrict__ q,
                         double* __restrict__ j, double* __restrict__ F, double* __restrict__ tau,
                         uint32_t* __restrict__ ufix, int* __restrict__ cell)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint4 p = pos[t];
    int i = (int)p.w;
    if (r) { r[3 * i] = (double)p.x * g.s; r[3 * i + 1] = (double)p.y * g.s; r[3 * i + 2] = (double)p.z * g.s; }
    if (ufix) { ufix[3 * i] = p.x; ufix[3 * i + 1] = p.y; ufix[3 * i + 2] = p.z; }
    if (cell) {
        int cx = cell_of_u(g, 0, p.x), cy = cell_of_u(g, 1, p.y), cz = cell_of_u(g, 2, p.z);
        cell[i] = cx + g.nc[0] * (cy + g.nc[1] * cz);
    }
    if (v) { float4 x = vel[t]; v[3 * i] = x.x; v[3 * i + 1] = x.y; v[3 * i + 2] = x.z; }
    if (F) { float4 x = force[t]; F[3 * i] = x.x; F[3 * i + 1] = x.y; F[3 * i + 2] = x.z; }
    if (RIGID) {
        if (q) { float4 x = quat[t]; q[4 * i] = x.x; q[4 * i + 1] = x.y; q[4 * i + 2] = x.z; q[4 * i + 3] = x.w; }
        if (j) { float4 x = angm[t]; j[3 * i] = x.x; j[3 * i + 1] = x.y; j[3 * i + 2] = x.z; }
        if (tau) { float4 x = torque[t]; tau[3 * i] = x.x; tau[3 * i + 1] = x.y; tau[3 * i + 2] = x.z; }
    } else {
        if (q) { q[4 * i] = 1; q[4 * i + 1] = 0; q[4 * i + 2] = 0; q[4 * i + 3] = 0; }
        if (j) { j[3 * i] = 0; j[3 * i + 1] = 0; j[3 * i + 2] = 0; }
        if (tau) { tau[3 * i] = 0; tau[3 * i + 1] = 0; tau[3 * i + 2] = 0; }
    }
}
