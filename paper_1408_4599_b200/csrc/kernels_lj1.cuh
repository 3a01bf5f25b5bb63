// kernels_lj1.cuh -- single-site Lennard-Jones force kernel (configs 0, 1, 4):
// the hot loop of the method ("the largest part of the computational cost is
// caused by the force and distance calculations"; linked
// cells of edge >= rc; LJTS P:76).
//
// Work decomposition.  The sorted state is cut into blocks of
// 32 consecutive molecules; a warp takes a block, one lane per home molecule
// (the north_star's thread per site), and splits it into "sub-chunks": runs
// of lanes in one x-row of cells spanning at most KMAX cells.  For a
// sub-chunk the warp stages the 9 neighbour rows (cells cA-1 .. cB+1 of the
// rows dy, dz in {-1, 0, 1}) into shared memory, relative to a common origin
// at the sub-chunk's middle cell.  With the quantum of reading A12 every
// staged coordinate is an exact fp32 multiple of s (|x| < 4 cell edges), so
// every separation is exact.  Rows are sorted by x (canonical in-cell order
// (x, id), A13, and cells in x order), so for row (dy, dz) a molecule only
// needs the x-window |X - x_i| < sqrt(rc^2 - Dy^2 - Dz^2); the window is found
// by binary search and all windows of a lane are concatenated into one
// segment list, so that each lane iterates over exactly its own candidates
// and the warp does not diverge on window lengths.  Candidates are processed
// two at a time with the packed fp32x2 instructions of sm_100 (FADD2 /
// FMUL2 / FFMA2), which halves the issue slots of the arithmetic; the LJ
// force is evaluated branch-free (masked by the cutoff test).
//
// Cutoff (readings A1, A12): strict r < rc on the COM separation; fp32 r^2
// outside the +-2^-20 relative band around rc^2 decides; a pair in the band is
// re-decided exactly in integer quanta by a rare second pass.
// Blocks that would need more than two sub-chunks (sparse gas) take a
// per-lane path that walks the molecule's own 27 cells.
#pragma once
#include "common.cuh"

namespace lj1 {

#ifndef MD_LJ1_UP
#define MD_LJ1_UP 4
#endif
#ifndef MD_LJ1_PREFETCH
#define MD_LJ1_PREFETCH 1
#endif
constexpr int KMAX = 6;          // home cells per sub-chunk: staged |x| < 4 E (A12 quantum)
constexpr int BLOCKS_PER_FETCH = 1;
// small systems (at most MD_LJ1_HALF blocks of 32 per warp of the grid) are taken as half
// blocks of 16 molecules with two lanes per molecule (each lane one half of the neighbour
// rows): a block's latency sets the time of such a launch.  (Half blocks for the last wave
// of a large system only -- the tail -- measured 1 % slower on c1: staging and window
// searches cost a half block as much as a full one.)
#ifndef MD_LJ1_HALF
#define MD_LJ1_HALF 1
#endif

// per-lane segment [begin, end) of staged pairs: packed 16-bit halves (smaller
// shared memory per warp -> more resident warps) or two ints
#ifndef MD_LJ1_SEG16
#define MD_LJ1_SEG16 0
#endif
#if MD_LJ1_SEG16
typedef uint32_t SegT;
constexpr int SEGB = 4;
__device__ __forceinline__ SegT seg_make(int b, int e) { return (uint32_t)b | ((uint32_t)e << 16); }
__device__ __forceinline__ int seg_b(SegT s) { return (int)(s & 0xffffu); }
__device__ __forceinline__ int seg_e(SegT s) { return (int)(s >> 16); }
#else
typedef int2 SegT;
constexpr int SEGB = 8;
__device__ __forceinline__ SegT seg_make(int b, int e) { return make_int2(b, e); }
__device__ __forceinline__ int seg_b(SegT s) { return s.x; }
__device__ __forceinline__ int seg_e(SegT s) { return s.y; }
#endif
constexpr int NSEG = 11;         // per-lane segments: 9 rows + self split + sentinel
constexpr float FAR = 1.0e18f;   // padding coordinate (r^2 ~ 1e36, finite, never a hit)

struct Args {
    GridP g;
    const int* start;            // ncell + 1
    uint4* pos;                  // sorted fixed-point positions (advanced in place by the fused step)
    const float4* xs;            // cell-relative staging copy, w = cell x index (k_canon<false>)
    float4* force;
    ForcePartial* part;          // one per warp of the grid (n_candidates)
    ForcePartial* bpart;         // one per block of 32 sorted molecules (U, W, n_pairs), nbcap entries
    int nbcap;
    int* ctr;                    // block counter (zeroed before the launch): dynamic block scheduling
    float sig2, eps24, eps4, shift;
    // fused leapfrog step (STEP): v(t - dt/2) in / v(t + dt/2) out, next-step binning
    float4* vel;
    int* cell_of;
    int* rank;
    int* count;
    int* flag;
    float mass, inv_mass;
    DDArgs dd;                   // STEP with DD: exchange packing of the decomposed step
};

// origin (in quanta, mod 2^32) to subtract from the stored u of a molecule
// in the cell at unwrapped index cu (0 <= cu + 1, cu - 1 < n) so that the
// result is its coordinate relative to `base` in the image next to base
__device__ __forceinline__ uint32_t img_origin(uint32_t base, int cu, int n, uint32_t P)
{
    return base + (cu < 0 ? P : 0u) - (cu >= n ? P : 0u);
}

// fixed-point difference (u - o) mod 2^32 as an exact float multiple of s
__device__ __forceinline__ float qdiff(uint32_t u, uint32_t o, float s)
{
    return __int2float_rn((int)(u - o)) * s;
}

template <int WARPS, int CAPP>
struct Cfg {
    // per warp: pair arrays xy[CAPP] (x0, x1, y0, y1), z[CAPP] (z0, z1),
    // segments seg[NSEG][32] (pair begin, pair end), row table
    static constexpr int BYTES_PER_WARP = CAPP * 24 + NSEG * 32 * SEGB + 64 * 4;
    static constexpr int SMEM = WARPS * BYTES_PER_WARP;
};

// In terms of p = 1/r^6 (s6 = (sigma/r)^6 = c6 p, c6 = sigma^6): the force prefactor
// s6 (s6 - 1/2) / r^2 = c6^2 p (p - 1/(2 c6)) / r^2, so the sigma^2 scaling of 1/r^2
// costs nothing per pair (the powers of c6 are applied to the per-lane sums)
struct Acc {
    float2 gx, gy, gz;           // sum ir2 p (p - hc) d   (force = -48 eps c6^2 g)
    float2 a, b, h;              // sum p^2, sum p, sum ir2 r2 (= hit count)
    int hits_exact;              // hits found by the exact band pass / scalar paths
    float mb;                    // min |r^2 - mid| over the candidates (guard band iff <= hw)
};

// two lanes of one molecule (half blocks): sum their partial accumulators (commutative
// adds: both lanes hold the same bits afterwards)
__device__ __forceinline__ void acc_pair_sum(Acc& A, unsigned m)
{
    A.gx.x += __shfl_xor_sync(m, A.gx.x, 1); A.gx.y += __shfl_xor_sync(m, A.gx.y, 1);
    A.gy.x += __shfl_xor_sync(m, A.gy.x, 1); A.gy.y += __shfl_xor_sync(m, A.gy.y, 1);
    A.gz.x += __shfl_xor_sync(m, A.gz.x, 1); A.gz.y += __shfl_xor_sync(m, A.gz.y, 1);
    A.a.x += __shfl_xor_sync(m, A.a.x, 1); A.a.y += __shfl_xor_sync(m, A.a.y, 1);
    A.b.x += __shfl_xor_sync(m, A.b.x, 1); A.b.y += __shfl_xor_sync(m, A.b.y, 1);
    A.h.x += __shfl_xor_sync(m, A.h.x, 1); A.h.y += __shfl_xor_sync(m, A.h.y, 1);
    A.hits_exact += __shfl_xor_sync(m, A.hits_exact, 1);
    A.mb = fminf(A.mb, __shfl_xor_sync(m, A.mb, 1));
}

__device__ __forceinline__ void acc_zero(Acc& A)
{
    A.gx = A.gy = A.gz = A.a = A.b = A.h = make_float2(0.f, 0.f);
    A.hits_exact = 0;
    A.mb = 1.0e30f;
}

// one candidate pair (j, j+1) against molecule (xi, yi, zi), fast pass
__device__ __forceinline__ void pair2(const float4 xy, const float2 z, const float2 nxi, const float2 nyi,
                                      const float2 nzi, const float2 nhc, const float lo, const float2 nmid,
                                      Acc& A)
{
    const float2 dx = __fadd2_rn(make_float2(xy.x, xy.y), nxi);
    const float2 dy = __fadd2_rn(make_float2(xy.z, xy.w), nyi);
    const float2 dz = __fadd2_rn(z, nzi);
    float2 r2 = __fmul2_rn(dx, dx);
    r2 = __ffma2_rn(dy, dy, r2);
    r2 = __ffma2_rn(dz, dz, r2);
    const bool h0 = r2.x < lo, h1 = r2.y < lo;
    // guard band lo <= r^2 < hi  =>  |r^2 - mid| <= hw (the difference is exact there)
    const float2 dm = __fadd2_rn(r2, nmid);
    A.mb = fminf(A.mb, fminf(fabsf(dm.x), fabsf(dm.y)));
    float2 ir2;
    ir2.x = h0 ? rcp_approx(r2.x) : 0.f;
    ir2.y = h1 ? rcp_approx(r2.y) : 0.f;
    const float2 i4 = __fmul2_rn(ir2, ir2);
    const float2 p6 = __fmul2_rn(i4, ir2);
    const float2 t = __fadd2_rn(p6, nhc);
    const float2 fr = __fmul2_rn(__fmul2_rn(p6, ir2), t);
    A.gx = __ffma2_rn(fr, dx, A.gx);
    A.gy = __ffma2_rn(fr, dy, A.gy);
    A.gz = __ffma2_rn(fr, dz, A.gz);
    A.a = __ffma2_rn(p6, p6, A.a);
    A.b = __fadd2_rn(p6, A.b);
    A.h = __ffma2_rn(ir2, r2, A.h);
}

// one element in the exact (guard-band) pass or the scalar paths: the same
// fp32 r^2 as the fast pass; BAND_ONLY: only band pairs, decided exactly
template <bool BAND_ONLY>
__device__ __forceinline__ void elem1(float X, float Y, float Z, float xi, float yi, float zi, float hc,
                                      float lo, float hi, const GridP& g, Acc& A)
{
    const float dx = __fadd_rn(X, -xi), dy = __fadd_rn(Y, -yi), dz = __fadd_rn(Z, -zi);
    const float r2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));   // = the packed path's r^2
    bool hit;
    if (BAND_ONLY) {
        hit = (r2 >= lo) && (r2 < hi) && exact_in_range(dx, dy, dz, g);
    } else {
        const bool inband = (r2 >= lo) && (r2 < hi);
        hit = (r2 < lo) || (inband && exact_in_range(dx, dy, dz, g));
    }
    if (!hit) return;
    const float ir2 = rcp_approx(r2);
    const float p6 = ir2 * ir2 * ir2;
    const float fr = p6 * ir2 * (p6 - hc);
    A.gx.x += fr * dx;
    A.gy.x += fr * dy;
    A.gz.x += fr * dz;
    A.a.x += p6 * p6;
    A.b.x += p6;
    A.hits_exact += 1;
}

// lower bound: first pair p in [rb, re) with X[2p + ODD] (>= if !STRICT, > if
// STRICT) v, starting from the guess g (rows are x-sorted; the guess from the
// row's mean pitch is within a pair or two in a liquid)
template <int ODD, bool STRICT>
__device__ __forceinline__ int find_from(const float* __restrict__ sxf, int rb, int re, int g, float v)
{
    auto below = [&](int p) { const float x = sxf[4 * p + ODD]; return STRICT ? (x <= v) : (x < v); };
    if (g < re && below(g)) {
        do { ++g; } while (g < re && below(g));
    } else {
        while (g > rb && !below(g - 1)) --g;
    }
    return g;
}

// STEP: the leapfrog step of the block's home molecules is fused in (one domain: every
// molecule is home).  DD (with STEP, spatial decomposition): the molecules of halo cells are
// dropped and every home molecule's exchange records -- migrant for its new owner, halo
// copies for the ranks whose halo holds its new cell -- are packed here too (reading the
// force kernel's own results: no separate integrator pass over the state)
template <int WARPS, int CAPP, int MINB, bool STEP, bool DD = false>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_force_lj1(Args a)
{
    using C = Cfg<WARPS, CAPP>;
    extern __shared__ float4 smem_lj1[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    char* wbase = reinterpret_cast<char*>(smem_lj1) + wib * C::BYTES_PER_WARP;
    float4* sxy = reinterpret_cast<float4*>(wbase);
    float2* sz = reinterpret_cast<float2*>(wbase + CAPP * 16);
    SegT* sseg = reinterpret_cast<SegT*>(wbase + CAPP * 24);
    int* srow = reinterpret_cast<int*>(wbase + CAPP * 24 + NSEG * 32 * SEGB);   // [0..9] row pair bases
    uint16_t* scb = reinterpret_cast<uint16_t*>(srow + 12);                  // [9][10] staged-cell element offsets
    float* sxf = reinterpret_cast<float*>(sxy);
    float* szf = reinterpret_cast<float*>(sz);

    const GridP& g = a.g;
    const int gw = blockIdx.x * WARPS + wib, nw = gridDim.x * WARPS;
    // cell coordinates in the rank-local window (the whole grid for one domain)
    const int nx = g.wn[0], ny = g.wn[1], nz = g.wn[2];
    const int kmax = min(KMAX, nx - 2);
    const float lo = g.cut2_lo, hi = g.cut2_hi;
    const float c6 = a.sig2 * a.sig2 * a.sig2, hc = 0.5f / c6;     // sigma^6, 1/(2 sigma^6)
    const double c6d = (double)c6;
    const float2 nhc = make_float2(-hc, -hc);
    // band test |r^2 - mid| <= hw (margin >> rounding of mid); host-computed kernel parameters, so
    // that the main loop takes them as constant operands instead of holding or recomputing them
    const float mid = g.band_mid, hw = g.band_hw;
    const float2 nmid = make_float2(-mid, -mid);
    const float rc2w = hi * (1.f + 1.f / 4096.f);       // generous window (necessary condition only)
    const float ex = g.edge[0], inv_ex = 1.f / g.edge[0];
    long long ncw = 0;

    // n_candidates (27-cell full-shell count, reported observable): each home lane
    // adds sum_27 N_c' - 1 for its molecule (from the staged cell table or start[])
    const int nsorted = __ldg(a.start + g.wncell);
    const int nb32 = (nsorted + 31) >> 5;
    const int B1 = nb32 <= MD_LJ1_HALF * nw ? 0 : nb32;       // blocks of 32, or half blocks of 16
    const int nblocks = B1 + max(0, (nsorted - 32 * B1 + 15) >> 4);
    for (int b = nblocks + gw * 32 + lane; b < a.nbcap; b += nw * 32)     // unused block partials
        a.bpart[b] = ForcePartial{0.0, 0.0, 0, 0, 0.0};
    // blocks are handed out in sorted order by an atomic counter (load balance);
    // each block's sums go to its own slot, so totals do not depend on the schedule
    // (two consecutive blocks per fetch: they share most staged cells, which then hit in L1)
    // first fetch static (no start-up contention on the counter), then dynamic
    int nextb = BLOCKS_PER_FETCH * gw;
    int pend_mi = -1, pend_b = 0, pend_r = 0;          // deferred arrival rank (STEP)
    unsigned pend_m = 0;
    for (;;) {
        const int blk0 = __shfl_sync(0xffffffffu, nextb, 0);
        if (blk0 >= nblocks) break;
        if (lane == 0) nextb = BLOCKS_PER_FETCH * nw + atomicAdd(a.ctr, BLOCKS_PER_FETCH);   // in flight meanwhile
        const int blk1 = min(blk0 + BLOCKS_PER_FETCH, nblocks);
    for (int blk = blk0; blk < blk1; ++blk) {
        double Uw = 0.0, Ww = 0.0;
        long long npw = 0;
        float3 Fown = make_float3(0.f, 0.f, 0.f);  // this lane's molecule (STEP)
        const bool lp2 = blk >= B1;                // half block: lanes 2k, 2k+1 share molecule k
        const int sub = lp2 ? (lane & 1) : 0;      // which half of the neighbour rows (parity of r)
        const bool own_lane = sub == 0;            // the lane that writes the molecule's results
        const int mi = lp2 ? 32 * B1 + 16 * (blk - B1) + (lane >> 1) : blk * 32 + lane;
        bool valid = mi < nsorted;
        uint4 pi = valid ? a.pos[mi] : make_uint4(0, 0, 0, 0);
        const float4 vi = (STEP && valid) ? a.vel[mi] : make_float4(0.f, 0.f, 0.f, 0.f);   // in flight during the forces
        const int cx = loc_axis(g, 0, cell_of_u(g, 0, pi.x)), cy = loc_axis(g, 1, cell_of_u(g, 1, pi.y)),
                  cz = loc_axis(g, 2, cell_of_u(g, 2, pi.z));
        const bool home = valid && cx >= g.hlo[0] && cx < g.hlo[0] + g.hdim[0] && cy >= g.hlo[1] &&
                          cy < g.hlo[1] + g.hdim[1] && cz >= g.hlo[2] && cz < g.hlo[2] + g.hdim[2];
        const int row = cy + ny * cz;
        unsigned todo = __ballot_sync(0xffffffffu, home);
        int passes = 0, klim = kmax;
        while (todo) {
            const int leader = __ffs(todo) - 1;
            const int R = __shfl_sync(0xffffffffu, row, leader);
            const int cA = __shfl_sync(0xffffffffu, cx, leader);
            const bool mine = ((todo >> lane) & 1u) && row == R && cx < cA + klim;
            const unsigned members = __ballot_sync(0xffffffffu, mine);
            const int cB = __shfl_sync(0xffffffffu, cx, 31 - __clz(members));
            const int hy = __shfl_sync(0xffffffffu, cy, leader), hz = __shfl_sync(0xffffffffu, cz, leader);
            // ---------------- staging plan: lanes 0..8 own one neighbour row each
            int p_a0 = 0, p_n1 = 0, p_b0 = 0, p_n2 = 0, p_c0 = 0, p_n3 = 0, plen = 0;
            const int cm = (cA + cB + 1) >> 1;           // origin cell (x); y, z: the home row's corner
            if (lane < 9) {
                const int dy = lane % 3 - 1, dz = lane / 3 - 1;
                const int rowc = nx * (wrapi(hy + dy, ny) + ny * wrapi(hz + dz, nz));
                const int mlo = max(cA - 1, 0), mhi = min(cB + 1, nx - 1);
                p_b0 = __ldg(a.start + rowc + mlo);
                p_n2 = __ldg(a.start + rowc + mhi + 1) - p_b0;
                if (cA == 0) { p_a0 = __ldg(a.start + rowc + nx - 1); p_n1 = __ldg(a.start + rowc + nx) - p_a0; }
                if (cB == nx - 1) { p_c0 = __ldg(a.start + rowc); p_n3 = __ldg(a.start + rowc + 1) - p_c0; }
                plen = (p_n1 + p_n2 + p_n3 + 1) >> 1;        // real pairs; the row adds a far pad pair at each end
                // element offset of staged cell k (x-index cA - 1 + k) in the row: the window search
                // only looks inside the cell that holds the bound
#pragma unroll
                for (int k = 0; k <= KMAX + 2; ++k) {
                    const int cu = cA - 1 + k;
                    if (k <= cB - cA + 3) {
                        int off;
                        if (cu < 0) off = 0;
                        else if (cu >= nx) off = p_n1 + p_n2;
                        else if (cu > mhi) off = p_n1 + p_n2;
                        else off = p_n1 + __ldg(a.start + rowc + cu) - p_b0;
                        if (k == cB - cA + 3) off = p_n1 + p_n2 + p_n3;
                        scb[10 * lane + k] = (uint16_t)off;
                    }
                }
            }
            // scan of the row strides (plen + 2) over lanes 0..8 -> row pair bases
            int incl = lane < 9 ? plen + 2 : 0;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 8);
            if (total + 2 > CAPP && cB > cA) {         // over capacity: fewer home cells
                klim = (cB - cA + 1) >> 1;
                continue;
            }
            if (total + 2 > CAPP || passes >= 2) {
#ifdef MD_LJ1_STATS
                if (lane == 0) atomicAdd((unsigned long long*)(a.flag + 22), (unsigned long long)__popc(todo));
#endif
                // sparse or over-full: per-lane path for the remaining lanes
                Acc A;
                acc_zero(A);
                if ((todo >> lane) & 1u) {
                    int ncand_l = own_lane ? -1 : 0;       // the molecule itself is no candidate
                    // cell-relative coordinates of the staging copy (read-only while the fused
                    // step advances pos in place): neighbour cell (dx, dy, dz) adds its offset, exact
                    const float4 xsi = __ldg(a.xs + mi);
                    for (int dz = -1; dz <= 1; ++dz)
                        for (int dy = -1; dy <= 1; ++dy) {
                            if (((dy + 1 + 3 * (dz + 1)) & 1) != sub && lp2) continue;   // the partner lane's row
                            const int rowc = nx * (wrapi(cy + dy, ny) + ny * wrapi(cz + dz, nz));
                            const float oy = (float)dy * g.edge[1], oz = (float)dz * g.edge[2];
                            for (int dx = -1; dx <= 1; ++dx) {
                                const float ox = (float)dx * ex;
                                const int c2 = rowc + wrapi(cx + dx, nx);
                                const int j0 = __ldg(a.start + c2), j1 = __ldg(a.start + c2 + 1);
                                ncand_l += j1 - j0;
                                for (int j = j0; j < j1; ++j) {
                                    if (j == mi) continue;
                                    const float4 xj = __ldg(a.xs + j);
                                    elem1<false>(xj.x + ox, xj.y + oy, xj.z + oz, xsi.x, xsi.y, xsi.z, hc, lo,
                                                 hi, g, A);
                                }
                            }
                        }
                    if (lp2) acc_pair_sum(A, todo);
                    const float f = -2.f * a.eps24 * c6 * c6;
                    Fown = make_float3(f * A.gx.x, f * A.gy.x, f * A.gz.x);
                    ncw += ncand_l;
                    if (own_lane) {
                        a.force[mi] = make_float4(Fown.x, Fown.y, Fown.z, 0.f);
                        const double Ad = c6d * c6d * A.a.x, Bd = c6d * A.b.x;
                        Uw += (double)a.eps4 * (Ad - Bd) - (double)a.shift * A.hits_exact;
                        Ww += (double)a.eps24 * (2.0 * Ad - Bd);
                        npw += A.hits_exact;
                    }
                }
                break;
            }
            const int rbase = incl - plen - 1;         // first real pair of the row (lanes 0..8)
            const float xlo = (float)(cA - 1 - cm) * ex;          // staged x range [xlo, xlo + (cB-cA+3) ex)
            if (lane < 10) srow[lane] = (lane < 9) ? rbase : total + 1;    // real end of row r = srow[r + 1] - 2
            if (lane < 9) {
                sxy[rbase - 1] = make_float4(FAR, FAR, FAR, FAR);
                sz[rbase - 1] = make_float2(FAR, FAR);
                sxy[rbase + plen] = make_float4(FAR, FAR, FAR, FAR);
                sz[rbase + plen] = make_float2(FAR, FAR);
            }
            // ---------------- staging copy: 3 lanes per row (lanes 0..26), 4 loads in flight per lane;
            //                  x = xs.x + (cx - cm') edge exactly (A12), y, z + the row's offsets
            __syncwarp();
            {
                const int r3 = min(lane / 3, 8);
                const int a0 = __shfl_sync(0xffffffffu, p_a0, r3), n1 = __shfl_sync(0xffffffffu, p_n1, r3);
                const int b0 = __shfl_sync(0xffffffffu, p_b0, r3), n2 = __shfl_sync(0xffffffffu, p_n2, r3);
                const int c0 = __shfl_sync(0xffffffffu, p_c0, r3), n3 = __shfl_sync(0xffffffffu, p_n3, r3);
                const int base = __shfl_sync(0xffffffffu, rbase, r3), np = __shfl_sync(0xffffffffu, plen, r3);
                if (lane < 27) {
                    const float offy = (float)(r3 % 3 - 1) * g.edge[1], offz = (float)(r3 / 3 - 1) * g.edge[2];
                    const int len = n1 + n2 + n3;
                    // element e of the row -> xs index e + d(e), origin cell cm'(e) (branch-free)
                    const int d1 = a0, d2 = b0 - n1, d3 = c0 - n1 - n2, n12 = n1 + n2;
                    const float cm1 = (float)(cm + nx), cm2 = (float)cm, cm3 = (float)(cm - nx);
                    auto fetch = [&](int e, float4& v, float& c) {
                        const int ee = min(e, len - 1);          // len >= 1 whenever the row has a pair
                        const int gi = ee + (ee < n1 ? d1 : (ee < n12 ? d2 : d3));
                        c = ee < n1 ? cm1 : (ee < n12 ? cm2 : cm3);
                        v = __ldg(a.xs + gi);
                    };
                    constexpr int UP = MD_LJ1_UP;                 // pairs per lane per round: 2 UP loads in flight
                    for (int q0 = lane - 3 * r3; q0 < np; q0 += 3 * UP) {
                        float4 v[2 * UP];
                        float c[2 * UP];
#pragma unroll
                        for (int u = 0; u < 2 * UP; ++u) fetch(2 * (q0 + 3 * (u >> 1)) + (u & 1), v[u], c[u]);
#pragma unroll
                        for (int k = 0; k < UP; ++k) {
                            const int q = q0 + 3 * k;
                            if (q < np) {
                                float X[2], Y[2], Z[2];
#pragma unroll
                                for (int h = 0; h < 2; ++h) {
                                    const bool real = 2 * q + h < len;
                                    const float4 w = v[2 * k + h];
                                    X[h] = real ? __fmaf_rn(w.w - c[2 * k + h], ex, w.x) : FAR;
                                    Y[h] = real ? w.y + offy : FAR;
                                    Z[h] = real ? w.z + offz : FAR;
                                }
                                MD_CHECK(base + q < CAPP);
                                sxy[base + q] = make_float4(X[0], X[1], Y[0], Y[1]);
                                sz[base + q] = make_float2(Z[0], Z[1]);
                            }
                        }
                    }
                }
            }
            if (lane < 2) {                             // dummy pairs for exhausted lanes
                sxy[total + lane] = make_float4(FAR, FAR, FAR, FAR);
                sz[total + lane] = make_float2(FAR, FAR);
            }
            __syncwarp();
            // ---------------- windows -> segment list
            const int hb0 = __shfl_sync(0xffffffffu, p_b0, 4), hn1 = __shfl_sync(0xffffffffu, p_n1, 4);
            const int hbase = __shfl_sync(0xffffffffu, rbase, 4);
            const int eself = hn1 + (mi - hb0);          // own element in the staged home row
            const int pself = hbase + (eself >> 1);
            const bool act = (members >> lane) & 1u;
            float xi = 0.f, yi = 0.f, zi = 0.f;
            if (act) {
                xi = sxf[4 * pself + (eself & 1)];
                yi = sxf[4 * pself + 2 + (eself & 1)];
                zi = szf[2 * pself + (eself & 1)];
            }
            int nseg = 0, ttot = 0;
            {
                // pass 1 (branch-free, all rows): window half-width, cells holding the bounds
                // (x of staged cell k: [xlo + k ex, xlo + (k+1) ex), exact), initial search ranges
                const float Dyl = yi, Dyh = g.edge[1] - yi, Dzl = zi, Dzh = g.edge[2] - zi;
                const int nsc = cB - cA + 3;
                float wl[9], wh[9];
                int la[9], lb[9], ua[9], ub[9];
#pragma unroll
                for (int r = 0; r < 9; ++r) {
                    const int dy = r % 3 - 1, dz = r / 3 - 1;
                    const float Dy = dy == 0 ? 0.f : (dy > 0 ? Dyh : Dyl);
                    const float Dz = dz == 0 ? 0.f : (dz > 0 ? Dzh : Dzl);
                    const float w2 = rc2w - Dy * Dy - Dz * Dz;
                    float w;                                     // approximate: rc2w is generous by 2^-12
                    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(fmaxf(w2, 0.f)));
                    const bool on = act && w2 > 0.f && (!lp2 || (r & 1) == sub);
                    const float xl = on ? xi - w : FAR, xh = on ? xi + w : -FAR;   // off: empty window
                    // cell of each bound, rounded outward by 1e-3 cell (>> the 1e-6 rounding of the
                    // product): a lower cell for xl / a higher cell for xh only widens the window
                    const int kl = min(max(__float2int_rd(fmaf(xl - xlo, inv_ex, -1e-3f)), 0), nsc - 1);
                    const int kh = min(max(__float2int_rd(fmaf(xh - xlo, inv_ex, 1e-3f)), 0), nsc - 1);
                    const int rb = srow[r];
                    // lower: first pair whose odd element is >= xl, in [floor(off_kl/2), floor(off_kl+1/2)]
                    la[r] = rb + (scb[10 * r + kl] >> 1);
                    lb[r] = rb + (scb[10 * r + kl + 1] >> 1) - la[r];
                    // upper: first pair whose even element is > xh, in [ceil(off_kh/2), ceil(off_kh+1/2)]
                    ua[r] = rb + ((scb[10 * r + kh] + 1) >> 1);
                    ub[r] = rb + ((scb[10 * r + kh + 1] + 1) >> 1) - ua[r];
                    wl[r] = xl;
                    wh[r] = xh;
                }
                // pass 2: the 18 binary searches step by step, interleaved (independent chains)
                int nmax = 0;
#pragma unroll
                for (int r = 0; r < 9; ++r) nmax = max(nmax, max(lb[r], ub[r]));
                nmax = __reduce_max_sync(0xffffffffu, nmax);
                for (int n = nmax; n > 0; n >>= 1) {
#pragma unroll
                    for (int r = 0; r < 9; ++r) {
                        {
                            const int h = lb[r] >> 1;
                            const bool lt = lb[r] > 0 && sxf[4 * (la[r] + h) + 1] < wl[r];
                            la[r] = lt ? la[r] + h + 1 : la[r];
                            lb[r] = lt ? lb[r] - h - 1 : h;
                        }
                        {
                            const int h = ub[r] >> 1;
                            const bool le = ub[r] > 0 && sxf[4 * (ua[r] + h)] <= wh[r];
                            ua[r] = le ? ua[r] + h + 1 : ua[r];
                            ub[r] = le ? ub[r] - h - 1 : h;
                        }
                    }
                }
                // pass 3: segments of even length, so that the main loop takes two pairs per step
                // from one segment: an odd one grows by a pair inside its row (the far pads at
                // both row ends keep it there); the pair holding the self element is excluded
#pragma unroll
                for (int r = 0; r < 9; ++r) {
                    int pa = la[r];
                    const int pb = ua[r];
                    if (r == 4 && act && own_lane) {
                        if (pself > pa) {
                            const int qa = pa - ((pself - pa) & 1);
                            MD_CHECK(nseg < NSEG - 1);
                            sseg[32 * nseg + lane] = seg_make(qa, pself); ++nseg; ttot += pself - qa;
                        }
                        pa = pself + 1;
                    }
                    if (pb > pa) {
                        const int qb = pb + ((pb - pa) & 1);
                        MD_CHECK(nseg < NSEG - 1 && qb <= total);
                        sseg[32 * nseg + lane] = seg_make(pa, qb); ++nseg; ttot += qb - pa;
                    }
                }
            }
            sseg[32 * nseg + lane] = seg_make(total, total + 2);    // sentinel
            const int tmax = __reduce_max_sync(0xffffffffu, ttot);
#ifdef MD_LJ1_STATS
            {   // profiling build (profiles/tools/lj1_stats.py): lane balance of the main loop --
                // useful pairs vs executed pair slots (32 x the longest list) -- and lanes per path
                const int tsum = __reduce_add_sync(0xffffffffu, ttot);
                if (lane == 0) {
                    atomicAdd((unsigned long long*)(a.flag + 16), (unsigned long long)tsum);
                    atomicAdd((unsigned long long*)(a.flag + 18), (unsigned long long)(32 * tmax));
                    atomicAdd((unsigned long long*)(a.flag + 20), (unsigned long long)__popc(members));
                }
            }
#endif
            __syncwarp();
            // ---------------- main loop: each lane walks its own segments, two candidates per pair;
            //                  the next segment is kept in registers so that the pair index never
            //                  waits on a shared-memory load
            Acc A;
            acc_zero(A);
            const float2 nxi = make_float2(-xi, -xi), nyi = make_float2(-yi, -yi), nzi = make_float2(-zi, -zi);
            {
                int si = lane;
                const int siend = 32 * nseg + lane;
                SegT sg = sseg[si];
                int p = seg_b(sg), e = seg_e(sg);
#if MD_LJ1_PREFETCH
                // software pipelined: the next step's pairs are loaded before this step's
                // arithmetic (past the last step the loads fall on the sentinel's far pads)
                float4 xy0 = sxy[p], xy1 = sxy[p + 1];
                float2 z0 = sz[p], z1 = sz[p + 1];
                for (int it = 0; it < tmax; it += 2) {
                    p += 2;
                    if (p == e) {
                        si = min(si + 32, siend);
                        sg = sseg[si];
                        p = seg_b(sg);
                        e = seg_e(sg);
                    }
                    const float4 nxy0 = sxy[p], nxy1 = sxy[p + 1];
                    const float2 nz0 = sz[p], nz1 = sz[p + 1];
                    pair2(xy0, z0, nxi, nyi, nzi, nhc, lo, nmid, A);
                    pair2(xy1, z1, nxi, nyi, nzi, nhc, lo, nmid, A);
                    xy0 = nxy0; xy1 = nxy1; z0 = nz0; z1 = nz1;
                }
#else
                for (int it = 0; it < tmax; it += 2) {
                    const float4 xy0 = sxy[p], xy1 = sxy[p + 1];
                    const float2 z0 = sz[p], z1 = sz[p + 1];
                    p += 2;
                    if (p == e) {                            // next segment (used by the next step)
                        si = min(si + 32, siend);
                        sg = sseg[si];
                        p = seg_b(sg);
                        e = seg_e(sg);
                    }
                    pair2(xy0, z0, nxi, nyi, nzi, nhc, lo, nmid, A);
                    pair2(xy1, z1, nxi, nyi, nzi, nhc, lo, nmid, A);
                }
#endif
            }
            // the other element of the self pair
            if (act && own_lane) {
                const int eo = eself ^ 1;
                elem1<false>(sxf[4 * pself + (eo & 1)], sxf[4 * pself + 2 + (eo & 1)], szf[2 * pself + (eo & 1)],
                             xi, yi, zi, hc, lo, hi, g, A);
            }
            // guard band (rare): exact re-decision of the band pairs of the lanes that saw one
            if (__any_sync(0xffffffffu, A.mb <= hw)) {
                if (A.mb <= hw) {
                    for (int k = 0; k < nseg; ++k) {
                        const SegT sg = sseg[32 * k + lane];
                        for (int p = seg_b(sg); p < seg_e(sg); ++p) {
                            const float4 xy = sxy[p];
                            const float2 zz = sz[p];
                            elem1<true>(xy.x, xy.z, zz.x, xi, yi, zi, hc, lo, hi, g, A);
                            elem1<true>(xy.y, xy.w, zz.y, xi, yi, zi, hc, lo, hi, g, A);
                        }
                    }
                }
            }
            if (lp2) acc_pair_sum(A, 0xffffffffu);
            if (act && own_lane) {
                int nc27 = -1;                             // the molecule itself is no candidate
                const int kk = cx - cA;                    // staged cells kk, kk+1, kk+2 hold its 27-cell rows
#pragma unroll
                for (int r = 0; r < 9; ++r) nc27 += scb[10 * r + kk + 3] - scb[10 * r + kk];
                ncw += nc27;
                const float f = -2.f * a.eps24 * c6 * c6;
                const float gx = A.gx.x + A.gx.y, gy = A.gy.x + A.gy.y, gz = A.gz.x + A.gz.y;
                Fown = make_float3(f * gx, f * gy, f * gz);
                a.force[mi] = make_float4(Fown.x, Fown.y, Fown.z, 0.f);
                const int hits = __float2int_rn(A.h.x + A.h.y) + A.hits_exact;
                const double Ad = c6d * c6d * ((double)A.a.x + (double)A.a.y), Bd = c6d * ((double)A.b.x + (double)A.b.y);
                Uw += (double)a.eps4 * (Ad - Bd) - (double)a.shift * hits;
                Ww += (double)a.eps24 * (2.0 * Ad - Bd);
                npw += hits;
            }
            __syncwarp();
            todo &= ~members;
            ++passes;
            klim = kmax;
        }
        double Kw = 0.0;
        if (STEP) {
            // fused leapfrog (Eqs. 2-3): this block's molecules are only read by this warp
            // (neighbours are staged from xs), so they are advanced in place
            int clb = -1;
            unsigned dmask = 0;
            int own = -1;
            uint4 pn = make_uint4(0, 0, 0, 0);
            float4 vn = make_float4(0.f, 0.f, 0.f, 0.f);
            if (home && own_lane) {
                const LeapOut o = md_leapfrog(g, pi, vi, Fown.x, Fown.y, Fown.z, a.mass, a.inv_mass);
                if (o.bad) atomicOr(a.flag, 1);
                a.pos[mi] = o.p;
                a.vel[mi] = o.v;
                clb = cell_loc(g, o.c[0], o.c[1], o.c[2]);
                if (DD) {
                    pn = o.p;
                    vn = o.v;
                    const int clg = cell_glob(g, o.c[0], o.c[1], o.c[2]);
                    own = a.dd.owner[clg];
                    const uint32_t gm = a.dd.gmask[clg];
                    dmask = (gm & ~(1u << a.dd.rank)) | (own != a.dd.rank ? 1u << own : 0u);
                    if (own != a.dd.rank) {                // migrant: kept as a ghost if in my halo
                        if ((gm >> a.dd.rank) & 1u) a.vel[mi] = make_float4(vn.x, vn.y, vn.z, __int_as_float(md_comp(vn.w) | 256));
                        else clb = -1;
                    }
                }
                a.cell_of[mi] = clb;
                Kw = o.ket;
            } else if (DD && valid && own_lane) {
                a.cell_of[mi] = -1;                        // last step's halo copies are dropped
            }
            if (DD) {
                dd_pack_warp(a.dd, dmask, own, pn, vn, make_float4(1.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f));
                if (a.dd.peer_puts) __threadfence_system();   // receivers on other GPUs (IPC puts)
            }
            // arrival ranks: one atomic per distinct cell; the rank store waits for the
            // atomic's reply, so it is deferred to after the next block's forces
            if (pend_mi >= 0) a.rank[pend_mi] = __shfl_sync(pend_m, pend_b, __ffs(pend_m) - 1) + pend_r;
            const unsigned m = __match_any_sync(0xffffffffu, clb);
            pend_mi = -1;
            if (clb >= 0) {
                const int leader = __ffs(m) - 1;
                pend_b = 0;
                if (lane == leader) pend_b = atomicAdd(a.count + clb, __popc(m));
                pend_m = m;
                pend_r = __popc(m & ((1u << lane) - 1u));
                pend_mi = mi;
            }
            Kw = warp_sum_d(Kw);
        }
        Uw = warp_sum_d(Uw);
        Ww = warp_sum_d(Ww);
        npw = warp_sum_ll(npw);
        if (lane == 0) a.bpart[blk] = ForcePartial{0.5 * Uw, 0.5 * Ww, npw, 0, Kw};
    }
    }
    if (STEP && pend_mi >= 0) a.rank[pend_mi] = __shfl_sync(pend_m, pend_b, __ffs(pend_m) - 1) + pend_r;
    ncw = warp_sum_ll(ncw);
    if (lane == 0) a.part[gw] = ForcePartial{0.0, 0.0, 0, ncw, 0.0};
    if (DD) {
        // the decomposed step's bookkeeping without extra launches: the sorted count of these
        // forces, and (direct puts) this rank's record counts into the receivers' count arrays,
        // stored by the last CTA to finish (all packing atomics are done by then)
        if (blockIdx.x == 0 && threadIdx.x == 0 && a.dd.n_force) *a.dd.n_force = nsorted;
        if (a.dd.put_cnt) {
            __shared__ int last_cta;
            __syncthreads();
            // system scope: the receivers may be other GPUs (IPC puts of a NCCL group)
            if (threadIdx.x == 0) {
                __threadfence_system();
                last_cta = atomicAdd(a.dd.done, 1) == (int)gridDim.x - 1;
            }
            __syncthreads();
            if (last_cta && threadIdx.x < a.dd.nranks) {
                __threadfence_system();
                *a.dd.put_cnt[threadIdx.x] = *(volatile int*)(a.dd.send_cnt + threadIdx.x);
                if (threadIdx.x == 0) *a.dd.done = 0;
            }
        }
    }
}

}  // namespace lj1
