// kernels_rigid3.cuh -- force/torque kernel for rigid multi-centre molecules of
// one component (configs 2 and 3: 2CLJQ, TIP4P, linked
// cells P:134-155; "the largest part of the computational cost is caused by
// the force and distance calculations"), load-balanced form.
//
// Decomposition.  One CTA per home cell at a time (cells
// strided over the persistent grid).  The CTA stages the whole 27-cell
// neighbourhood once into shared memory -- COM relative to the home cell's
// origin (exact multiples of the quantum s, reading A12) and the world-frame
// site slots -- and its half-warps ("groups" of 16 lanes) take the home
// molecules one at a time.  For home molecule i a group
//   1. tests every staged molecule j against the COM cutoff (reading A1; the
//      guard band around rc^2 is decided exactly in integer quanta), two
//      candidates per lane per step, collects the hits as per-lane bits over
//      four steps and appends them to the group's list in shared memory at
//      once (a group prefix of the lanes' counts; deterministic order);
//   2. evaluates the site pairs of its list 32 partners per round (two per
//      lane, packed into the fp32x2 instructions FADD2/FMUL2/FFMA2 of sm_100);
//   3. reduces the 16 lanes' force and torque (tau = sum_a s_a x f_a + tau_a)
//      with butterfly shuffles in fixed order.
// Every lane of a group works on the same molecule, so the partners are spread
// evenly over the lanes: a round is full except for the last one of a
// molecule.  (The per-lane queues of k_force_rigid2, one home molecule per
// lane, idle most lanes while the longest queue drains.)  Full shell: each
// pair is evaluated from both sides, no scatter, no atomics; energies and
// virials are summed per lane in fixed order and per warp in fp64.
#pragma once
#include "common.cuh"
#include "kernels_force.cuh"
#include "packed2.cuh"

namespace rig3 {

#ifndef MD_RIG3_CAP
#define MD_RIG3_CAP 1152
#endif
#ifndef MD_RIG3_WARPS
#define MD_RIG3_WARPS 8
#endif
#ifndef MD_RIG3_SU
#define MD_RIG3_SU 4       // staging: elements per thread with their loads in flight together
#endif
#ifndef MD_RIG3_BITS
#define MD_RIG3_BITS 1
#endif
constexpr int CAP = MD_RIG3_CAP;      // staged molecules per chunk of the neighbourhood
constexpr int WARPS = MD_RIG3_WARPS;
constexpr int HCAP = 256;             // hit-list entries per group
constexpr int NHMAX = 64;             // home molecules per batch (force/torque accumulators)

using pk2::P2;
using pk2::V3;
using pk2::p2;
using pk2::v3zero;
using pk2::bcast;
using pk2::pack;
using pk2::dot;

// charge-charge with reaction field (A4) without the constant c_rf, which the caller
// subtracts per partner as c_rf (sum_a q_a)(sum_b q_b) -- zero for neutral molecules
// SV (site virial, molecules without charges): the site force -fr r is accumulated with one
// FFMA2 per component from nfr = -fr (the _rn packed intrinsics are never contracted, so
// fa - fr * r is an FMUL2 and an FADD2), and there is no partner-pair force fh; the virial is
// summed per site pair as -r_ab . f_ab = fr r^2 and corrected per home molecule by
// -2 sum_a s_a . F_a at the flush (see the flush below: over the full shell the two
// give the same total as -sum_j d_j . F_ij, reading A6)
template <bool SV>
__device__ __forceinline__ void qq_nocrf(V3 r, P2 qq, float krf, P2& u, V3& fa, V3& fh, P2& w)
{
    const P2 r2 = dot(r, r);
    const P2 ir = pk2::rsqrt2(r2);
    const P2 ir2 = ir * ir;
    u = fma(qq, fma(p2(krf), r2, ir), u);
    if (SV) {
        const P2 nfr = pk2::neg(qq) * fma(ir, ir2, p2(-2.f * krf));
        fa.x = fma(nfr, r.x, fa.x); fa.y = fma(nfr, r.y, fa.y); fa.z = fma(nfr, r.z, fa.z);
        w = fma(pk2::neg(nfr), r2, w);
    } else {
        // with charges the molecular force and virial are small differences of the site terms
        // (neutral molecules): the product is rounded once and subtracted from both sums, the
        // rounding the parity tolerances were established with
        const P2 fr = qq * fma(ir, ir2, p2(-2.f * krf));
        fa.x = fa.x - fr * r.x; fa.y = fa.y - fr * r.y; fa.z = fa.z - fr * r.z;
        fh.x = fh.x - fr * r.x; fh.y = fh.y - fr * r.y; fh.z = fh.z - fr * r.z;
    }
}

// LJ 12-6 of a site pair without the LJTS shift (added per partner by the caller), r = x_b - x_a
template <bool SV>
__device__ __forceinline__ void lj_noshift(V3 r, float sig2, float eps24, float eps4, P2& u, V3& fa, V3& fh, P2& w)
{
    const P2 r2 = dot(r, r);
    const P2 ir2 = pk2::rcp2(r2);
    const P2 s2 = sig2 * ir2;
    const P2 s6 = s2 * s2 * s2;
    u = fma(eps4 * s6, s6 - p2(1.f), u);
    if (SV) {
        const P2 nfr = (-eps24 * ir2) * s6 * fma(p2(2.f), s6, p2(-1.f));
        fa.x = fma(nfr, r.x, fa.x); fa.y = fma(nfr, r.y, fa.y); fa.z = fma(nfr, r.z, fa.z);
        w = fma(pk2::neg(nfr), r2, w);
    } else {
        const P2 fr = (eps24 * ir2) * s6 * fma(p2(2.f), s6, p2(-1.f));
        fa.x = fa.x - fr * r.x; fa.y = fa.y - fr * r.y; fa.z = fa.z - fr * r.z;
        fh.x = fh.x - fr * r.x; fh.y = fh.y - fr * r.y; fh.z = fh.z - fr * r.z;
    }
}

template <int NLJ, int NQ, int NMU, int NQQ>
constexpr int smem_bytes()
{
    // COM pairs (CAP/2 + 1 pairs x 24 B, +1: the far dummy pair), NSLOT x (CAP + 1) site float4,
    // hit lists, accumulators, row table
    return (CAP / 2 + 1) * 16 + ((CAP / 2 + 2) & ~1) * 8 + (NLJ + NQ + 2 * NMU + 2 * NQQ) * (CAP + 1) * 16 + WARPS * 2 * 2 * (HCAP + 2) * 2 +
           NHMAX * 8 * 4 + WARPS * 2 * 8 * 4 + 16 * 8 * 4;
}

// PC: every dipole / quadrupole site sits at the centre of mass (2CLJQ, c2): its site-pair
// separation is the COM separation itself, so the partner's polar site position is not loaded
// (bitwise the same result: d + 0 - 0 = d)
// SYM (with PC): a linear molecule whose LJ sites sit at h_b e along the quadrupole axis e
// (2CLJQ): the partner's LJ site offsets are h_b times its staged axis and its quadrupole
// moment is the component's, so a partner costs its COM and axis instead of four site slots
template <int NLJ, int NQ, int NMU, int NQQ, bool PC = false, bool SYM = false>
__global__ void __launch_bounds__(WARPS * 32, 16 / WARPS) k_force_rigid3(ForceArgs a)
{
    using SH = Shape<NLJ, NQ, NMU, NQQ>;
    constexpr int NSLOT = SH::NSLOT;
    // site-pair virial (no charges: the site terms of point charges cancel strongly within a
    // neutral molecule, and fp32 sums of them lose the molecular virial's digits)
#ifndef MD_RIG3_SV
#define MD_RIG3_SV 1       // 0: never, 1: molecules without charges, 2: always
#endif
    constexpr bool SV = MD_RIG3_SV == 2 || (MD_RIG3_SV == 1 && NQ == 0);
    // slots the partner rounds read: SYM reads only the quadrupole axis, the others are not
    // staged (PC still reads the polar moments, kept in the position slots' w)
    auto staged_slot = [](int s) { return !SYM || s == SH::SQQ + 1; };
    constexpr int NPOL = (NMU + NQQ) > 0 ? (NMU + NQQ) : 1;
    constexpr int STRIDE = CAP + 1;
    constexpr int DUMMY = CAP;                                 // far dummy element (pair CAP / 2)
    constexpr unsigned FULL = 0xffffffffu;
    static_assert(CAP % 2 == 0 && CAP < 32768, "CAP");
    extern __shared__ float4 smem_rig3[];
    // COMs as pairs: cxy[p] = (x_2p, x_2p+1, y_2p, y_2p+1), pz[p] = (z_2p, z_2p+1): two candidates
    // are one packed operand without register moves
    float4* cxy = smem_rig3;
    float2* pz = reinterpret_cast<float2*>(cxy + CAP / 2 + 1);
    float* cxf = reinterpret_cast<float*>(cxy);
    float* czf = reinterpret_cast<float*>(pz);
    // site slots as four component arrays per slot (x, y, z, w): the two partners of a
    // packed operand are two scalar loads into a register pair, no moves
    float* sws = reinterpret_cast<float*>(pz + ((CAP / 2 + 2) & ~1));    // sws[(4 slot + c) * STRIDE + j]
    uint16_t* hls = reinterpret_cast<uint16_t*>(sws + 4 * NSLOT * STRIDE);  // [2 * WARPS][HCAP]
    float* acc = reinterpret_cast<float*>(hls + 2 * WARPS * 2 * (HCAP + 2));         // [NHMAX][8]: F, tau
    float* tacc = acc + NHMAX * 8;                                         // [NG][8]: tail slices (F, tau)
    int* rinfo = reinterpret_cast<int*>(tacc + 2 * WARPS * 8);             // [9][8] row table + [72..]: totals
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    const int half = lane >> 4, gl = lane & 15;
    const int grp = 2 * wib + half, NG = 2 * WARPS;
    uint16_t* hlA = hls + grp * 2 * (HCAP + 2);                            // two lists per group (+ spare slots)
    uint16_t* hlB = hlA + (HCAP + 2);
    [[maybe_unused]] const unsigned gmask = 0xffffu << (16 * half);   // the per-step ballots (MD_RIG3_BITS=0)
    const GridP& g = a.g;
    const float krf = a.krf, crf = a.crf, kmm = a.kmm;
    if (tid == 0) {                       // far dummy partner (padding): COM far away, sites at the COM
        cxy[CAP / 2] = make_float4(1.0e4f, 1.0e4f, 1.0e4f, 1.0e4f);
        pz[CAP / 2] = make_float2(1.0e4f, 1.0e4f);
#pragma unroll
        for (int s = 0; s < NSLOT; ++s) {
            sws[(4 * s + 0) * STRIDE + DUMMY] = 0.f;
            sws[(4 * s + 1) * STRIDE + DUMMY] = 0.f;
            sws[(4 * s + 2) * STRIDE + DUMMY] = 1.f;
            sws[(4 * s + 3) * STRIDE + DUMMY] = 0.f;
        }
    }
    double Uw = 0.0, Ww = 0.0;             // per lane (fp32 per home molecule, then fp64)
    long long npw = 0, ncw = 0;
    int nrej = 0;                          // band entries found out of range
    int nself = 0;                         // the home molecules' own list entries

    for (int t = blockIdx.x; t < g.nhome; t += gridDim.x) {
        int cx, cy, cz;
        const int c = home_cell(g, t, cx, cy, cz);
        const int s_i = __ldg(a.start + c);
        const int n_all = __ldg(a.start + c + 1) - s_i;
        if (n_all == 0) continue;
        // row table, built by warp 0 alone: lanes 0..26 read the 27 cells' start / count, lanes
        // 0..8 form the row lengths and their exclusive prefix (rinfo[8 r + 6]) by shuffles
        __syncthreads();                  // previous cell's consumers are done with smem
        if (tid < 32) {
            int st = 0, cnt = 0;
            if (lane < 27) {
                const int r = lane / 3, k = lane % 3;
                const int dy = r % 3 - 1, dz = r / 3 - 1;
                const int cc = wrapi(cx + k - 1, g.wn[0]) + g.wn[0] * (wrapi(cy + dy, g.wn[1]) + g.wn[1] * wrapi(cz + dz, g.wn[2]));
                st = __ldg(a.start + cc);
                cnt = __ldg(a.start + cc + 1) - st;
                rinfo[8 * r + k] = st;
                rinfo[8 * r + 3 + k] = cnt;
            }
            const int r3 = min(3 * lane, 30);
            const int c0 = __shfl_sync(FULL, cnt, r3), c1 = __shfl_sync(FULL, cnt, r3 + 1),
                      c2 = __shfl_sync(FULL, cnt, r3 + 2);
            const int len = lane < 9 ? c0 + c1 + c2 : 0;
            int incl = len;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const int v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            if (lane < 9) rinfo[8 * lane + 6] = incl - len;
            if (lane == 8) rinfo[72] = incl;
        }
        __syncthreads();
        const int mtot = rinfo[72];
        if (tid == 0) ncw += (long long)n_all * (mtot - 1);
        for (int ib = 0; ib < n_all; ib += NHMAX) {
            const int nb = min(NHMAX, n_all - ib);
            if (ib > 0) __syncthreads();          // previous batch written out
            for (int k = tid; k < nb * 8; k += WARPS * 32) acc[k] = 0.f;
            for (int k = tid; k < NG * 8; k += WARPS * 32) tacc[k] = 0.f;
            // work plan: full rounds of two molecules per group; a last round with at most NG
            // molecules is split instead -- each of them over P = NG / rem groups, one slice of
            // the neighbourhood per group (partials summed in slice order at the write-out)
            const int npr = nb / (2 * NG), rem = nb - npr * 2 * NG;
            const bool split = rem > 0 && rem <= NG;
            const int P = split ? NG / rem : 1;
            const int nrounds = npr + (rem > 0 ? 1 : 0);
            for (int k0 = 0; k0 < mtot; k0 += CAP) {
                const int mm = min(CAP, mtot - k0);
                if (k0 > 0) __syncthreads();      // the previous chunk's rounds are done with it
                // ---- stage elements k0 .. k0 + mm - 1 of the neighbourhood (rows in order)
                // SU elements per thread per pass: all their loads are issued before any store,
                // so a pass waits for one memory latency instead of SU
                constexpr int SU = MD_RIG3_SU;
                for (int kb = tid; kb < mm; kb += SU * WARPS * 32) {
                    float4 xv[SU], sv[SU][NSLOT];
                    float ox[SU], oy[SU], oz[SU];
#pragma unroll
                    for (int u = 0; u < SU; ++u) {
                        const int k = kb + u * WARPS * 32;
                        const int kg = k0 + min(k, mm - 1);
                        int r = 0;
#pragma unroll
                        for (int q = 1; q < 9; ++q) r += kg >= rinfo[8 * q + 6] ? 1 : 0;
                        const int* ri = rinfo + 8 * r;
                        const int kk = kg - ri[6];
                        int src;
                        if (kk < ri[3]) { src = ri[0] + kk; ox[u] = -g.edge[0]; }
                        else if (kk < ri[3] + ri[4]) { src = ri[1] + kk - ri[3]; ox[u] = 0.f; }
                        else { src = ri[2] + kk - ri[3] - ri[4]; ox[u] = g.edge[0]; }
                        oy[u] = (float)(r % 3 - 1) * g.edge[1];
                        oz[u] = (float)(r / 3 - 1) * g.edge[2];
                        xv[u] = __ldg(a.xs + src);
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if (staged_slot(s)) sv[u][s] = __ldg(a.site + (size_t)s * a.cap + src);
                    }
#pragma unroll
                    for (int u = 0; u < SU; ++u) {
                        const int k = kb + u * WARPS * 32;
                        if (k >= mm) break;
                        const int ph = k >> 1, od = k & 1;
                        MD_CHECK(k < CAP);
                        cxf[4 * ph + od] = xv[u].x + ox[u];
                        cxf[4 * ph + 2 + od] = xv[u].y + oy[u];
                        czf[2 * ph + od] = xv[u].z + oz[u];
                        if (k == mm - 1 && !od) {                   // odd chunk: far pad element
                            cxf[4 * ph + 1] = 1.0e4f;
                            cxf[4 * ph + 3] = 1.0e4f;
                            czf[2 * ph + 1] = 1.0e4f;
                        }
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s) {
                            if (!staged_slot(s)) continue;
                            sws[(4 * s + 0) * STRIDE + k] = sv[u][s].x;
                            sws[(4 * s + 1) * STRIDE + k] = sv[u][s].y;
                            sws[(4 * s + 2) * STRIDE + k] = sv[u][s].z;
                            sws[(4 * s + 3) * STRIDE + k] = sv[u][s].w;
                        }
                    }
                }
                __syncthreads();
                // ---- home molecules of this batch, two per group at a time (A, B): the distance
                //      phase tests each staged molecule against both (one load, two tests)
                const int npair = (mm + 1) >> 1;
                for (int rr = 0; rr < nrounds; ++rr) {
                    const bool tail = split && rr == npr;
                    int ilA, ilB, p0 = 0, p1 = npair;                    // batch-local home indices, slice
                    bool gA, gB;
                    float *tgtA, *tgtB;
                    if (!tail) {
                        ilA = rr * 2 * NG + grp; ilB = ilA + NG;
                        gA = ilA < nb; gB = ilB < nb;
                        tgtA = acc + 8 * ilA; tgtB = acc + 8 * ilB;
                    } else {
                        const int t = grp / P, sp = grp - t * P;
                        ilA = npr * 2 * NG + t; ilB = 0;
                        gA = t < rem; gB = false;
                        p0 = sp * npair / P; p1 = (sp + 1) * npair / P;
                        tgtA = tacc + 8 * grp; tgtB = acc;
                    }
                    if (!__any_sync(FULL, gA)) break;
                    const int myA = s_i + ib + (gA ? ilA : 0), myB = s_i + ib + (gB ? ilB : 0);
                    const float4 xiA = __ldg(a.xs + myA), xiB = __ldg(a.xs + myB);
                    // the molecules' own elements in the chunk (row 4 = the home row, after cell x - 1)
                    const int self0 = rinfo[8 * 4 + 6] + rinfo[8 * 4 + 3] + ib - k0;
                    const int selfA = self0 + ilA, selfB = self0 + ilB;

                    // force phase over the group's list [0, cnt): entries (k + gl, k + 16 + gl) packed;
                    // then this lane's force and torque, group reduction, accumulation into acc[il].
                    // Self-contained (site offsets, accumulators and LJ table are loaded here), so
                    // that none of it is live during the distance phase
                    auto flush = [&](int cnt, const uint16_t* hl, int my, float4 xi, int self, float* tgt, bool gact) {
                        float4 si[NSLOT];
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s) si[s] = __ldg(a.site + (size_t)s * a.cap + my);
                        static_assert(NLJ <= 2, "rig3: at most two LJ sites (ForceArgs::lj3)");
                        const float4* ljp = a.lj3;             // [2 ia + ib], kernel parameters
                        V3 fs[SH::NS];
                        V3 ts[NPOL];
#pragma unroll
                        for (int s = 0; s < SH::NS; ++s) fs[s] = v3zero();
#pragma unroll
                        for (int s = 0; s < NPOL; ++s) ts[s] = v3zero();
                        P2 uacc = p2(0.f), wacc = p2(0.f);
                        int nval = 0;                          // real partners evaluated by this lane
                        auto slot3 = [&](int sl, int j0, int j1) {
                            const float* b = sws + 4 * sl * STRIDE;
                            return V3{p2(b[j0], b[j1]), p2(b[STRIDE + j0], b[STRIDE + j1]),
                                      p2(b[2 * STRIDE + j0], b[2 * STRIDE + j1])};
                        };
                        auto slotw = [&](int sl, int j0, int j1) {
                            const float* b = sws + (4 * sl + 3) * STRIDE;
                            return p2(b[j0], b[j1]);
                        };
                        const int cmax = max(__shfl_sync(FULL, cnt, 0), __shfl_sync(FULL, cnt, 16));
                        // list entries of the next round are read one round ahead
                        int hn0 = gl < cnt ? hl[gl] : DUMMY, hn1 = 16 + gl < cnt ? hl[16 + gl] : DUMMY;
                        for (int k = 0; k < cmax; k += 32) {
                            const int e0 = k + gl, e1 = k + 16 + gl;
                            const bool v0 = e0 < cnt, v1 = e1 < cnt;
                            // Entries that are not partners -- past the list, the molecule itself (on the
                            // list with r = 0), out of range in the guard band -- are the far dummy: its
                            // site moments are 0 and its LJ terms vanish (~1e-26), so no mask is needed;
                            // the LJTS shifts are subtracted per real partner at the end
                            const int h0 = hn0, h1 = hn1;
                            hn0 = e0 + 32 < cnt ? hl[e0 + 32] : DUMMY;
                            hn1 = e1 + 32 < cnt ? hl[e1 + 32] : DUMMY;
                            const bool s0 = v0 && h0 == self, s1 = v1 && h1 == self;
                            int j0 = s0 ? DUMMY : h0, j1 = s1 ? DUMMY : h1;
                            auto com_of = [&](int j, float& X, float& Y, float& Z) {
                                const int q = 4 * (j >> 1) + (j & 1);
                                X = cxf[q] - xi.x;
                                Y = cxf[q + 2] - xi.y;
                                Z = czf[2 * (j >> 1) + (j & 1)] - xi.z;
                            };
                            V3 d;
                            com_of(j0, d.x.v.x, d.y.v.x, d.z.v.x);
                            com_of(j1, d.x.v.y, d.y.v.y, d.z.v.y);
                            nself += (s0 ? 1 : 0) + (s1 ? 1 : 0);
                            {
                                // guard band (reading A12): the distance phase took r^2 < hi; a pair at
                                // or above lo is decided exactly in integer quanta (rare)
                                const P2 r2 = dot(d, d);
                                const bool b0 = j0 != DUMMY && r2.v.x >= g.cut2_lo, b1 = j1 != DUMMY && r2.v.y >= g.cut2_lo;
                                if (b0 || b1) {
                                    if (b0 && !exact_in_range(d.x.v.x, d.y.v.x, d.z.v.x, g)) {
                                        j0 = DUMMY;
                                        com_of(j0, d.x.v.x, d.y.v.x, d.z.v.x);
                                        ++nrej;
                                    }
                                    if (b1 && !exact_in_range(d.x.v.y, d.y.v.y, d.z.v.y, g)) {
                                        j1 = DUMMY;
                                        com_of(j1, d.x.v.y, d.y.v.y, d.z.v.y);
                                        ++nrej;
                                    }
                                }
                            }
                            nval += (j0 != DUMMY ? 1 : 0) + (j1 != DUMMY ? 1 : 0);
                            V3 fh = v3zero();
                            static_assert(!SYM || (PC && NQQ == 1 && NQ == 0 && NMU == 0), "rig3: SYM");
                            // SYM: the partners' axes (also the quadrupole axes), and the moment
                            // product m^2 for real partners (0 for the far dummy)
                            V3 eBs = v3zero();
                            P2 mm2 = p2(0.f);
                            if (SYM) {
                                eBs = slot3(SH::SQQ + 1, j0, j1);
                                const float m = si[SH::SQQ].w;
                                mm2 = p2(j0 != DUMMY ? m * m : 0.f, j1 != DUMMY ? m * m : 0.f);
                            }
#pragma unroll
                            for (int ia = 0; ia < NLJ; ++ia) {
                                const V3 sa = bcast(si[ia]);
                                const V3 da = V3{d.x - sa.x, d.y - sa.y, d.z - sa.z};
#pragma unroll
                                for (int ibb = 0; ibb < NLJ; ++ibb) {
                                    const V3 sb = SYM ? V3{a.hsym[ibb] * eBs.x, a.hsym[ibb] * eBs.y, a.hsym[ibb] * eBs.z}
                                                      : slot3(ibb, j0, j1);
                                    const V3 rv = V3{da.x + sb.x, da.y + sb.y, da.z + sb.z};
                                    const float4 pp = ljp[2 * ia + ibb];
                                    lj_noshift<SV>(rv, pp.x, pp.y, pp.z, uacc, fs[ia], fh, wacc);
                                }
                            }
#pragma unroll
                            for (int ia = 0; ia < NQ; ++ia) {
                                const float4 sa4 = si[SH::SQ + ia];
                                const V3 sa = bcast(sa4);
                                const V3 da = V3{d.x - sa.x, d.y - sa.y, d.z - sa.z};
#pragma unroll
                                for (int ibb = 0; ibb < NQ; ++ibb) {
                                    const V3 sb = slot3(SH::SQ + ibb, j0, j1);
                                    const V3 rv = V3{da.x + sb.x, da.y + sb.y, da.z + sb.z};
                                    qq_nocrf<SV>(rv, sa4.w * slotw(SH::SQ + ibb, j0, j1), krf, uacc, fs[NLJ + ia], fh, wacc);
                                }
                            }
#define RIG3_POLAR(KA, KB, NA, NB, SLA, SLB, FIDX, TIDX, STA, STB)                                          \
    _Pragma("unroll") for (int ia = 0; ia < NA; ++ia)                                                      \
    {                                                                                                      \
        const float4 pa4 = si[(SLA) + ia * STA];                                                           \
        const V3 pa = bcast(pa4);                                                                          \
        const V3 ea = (STA == 2) ? bcast(si[((SLA) + ia * STA + 1) % NSLOT]) : v3zero();                  \
        _Pragma("unroll") for (int ibb = 0; ibb < NB; ++ibb)                                               \
        {                                                                                                  \
            const int slb = (SLB) + ibb * STB;                                                             \
            const bool pcab = PC && KA != MD_CHARGE && KB != MD_CHARGE;                                   \
            const V3 pb = pcab ? v3zero() : slot3(slb, j0, j1);                                            \
            const V3 eb = SYM ? eBs : (STB == 2) ? slot3((slb + 1) % NSLOT, j0, j1) : v3zero();           \
            const V3 rv = pcab ? d : V3{d.x + pb.x - pa.x, d.y + pb.y - pa.y, d.z + pb.z - pa.z};          \
            V3 tdummy = v3zero();                                                                          \
            pk2::polar2<KA, KB, SV>(rv, ea, eb, SYM ? mm2 : pa4.w * slotw(slb, j0, j1), kmm, uacc,         \
                                     fs[FIDX + ia],                                                        \
                                 (TIDX) >= 0 ? ts[((TIDX) >= 0 ? (TIDX) : 0) + ia] : tdummy, fh, wacc);  \
        }                                                                                                  \
    }
                            if (NQ > 0 && NMU > 0) {
                                RIG3_POLAR(MD_CHARGE, MD_DIPOLE, NQ, NMU, SH::SQ, SH::SMU, NLJ, -1, 1, 2)
                                RIG3_POLAR(MD_DIPOLE, MD_CHARGE, NMU, NQ, SH::SMU, SH::SQ, NLJ + NQ, 0, 2, 1)
                            }
                            if (NQ > 0 && NQQ > 0) {
                                RIG3_POLAR(MD_CHARGE, MD_QUAD, NQ, NQQ, SH::SQ, SH::SQQ, NLJ, -1, 1, 2)
                                RIG3_POLAR(MD_QUAD, MD_CHARGE, NQQ, NQ, SH::SQQ, SH::SQ, NLJ + NQ + NMU, NMU, 2, 1)
                            }
                            if (NMU > 0) {
                                RIG3_POLAR(MD_DIPOLE, MD_DIPOLE, NMU, NMU, SH::SMU, SH::SMU, NLJ + NQ, 0, 2, 2)
                            }
                            if (NMU > 0 && NQQ > 0) {
                                RIG3_POLAR(MD_DIPOLE, MD_QUAD, NMU, NQQ, SH::SMU, SH::SQQ, NLJ + NQ, 0, 2, 2)
                                RIG3_POLAR(MD_QUAD, MD_DIPOLE, NQQ, NMU, SH::SQQ, SH::SMU, NLJ + NQ + NMU, NMU, 2, 2)
                            }
                            if (NQQ > 0) {
                                RIG3_POLAR(MD_QUAD, MD_QUAD, NQQ, NQQ, SH::SQQ, SH::SQQ, NLJ + NQ + NMU, NMU, 2, 2)
                            }
#undef RIG3_POLAR
                            if (!SV) wacc -= dot(d, fh);      // molecular virial (A6): -r_ij . F_ij
                        }
                        // ---- molecule force and torque of this lane's share, group reduction
                        float F[3] = {0.f, 0.f, 0.f}, T[3] = {0.f, 0.f, 0.f};
                        float sdf = 0.f;                       // SV: sum_a s_a . (this lane's F_a)
#pragma unroll
                        for (int k = 0; k < SH::NS; ++k) {
                            int slot;
                            if (k < NLJ) slot = k;
                            else if (k < NLJ + NQ) slot = NLJ + (k - NLJ);
                            else if (k < NLJ + NQ + NMU) slot = SH::SMU + 2 * (k - NLJ - NQ);
                            else slot = SH::SQQ + 2 * (k - NLJ - NQ - NMU);
                            const float4 sp = si[slot < NSLOT ? slot : 0];
                            const float fx = fs[k].x.v.x + fs[k].x.v.y, fy = fs[k].y.v.x + fs[k].y.v.y,
                                        fz = fs[k].z.v.x + fs[k].z.v.y;
                            F[0] += fx; F[1] += fy; F[2] += fz;
                            if (SV) sdf += sp.x * fx + sp.y * fy + sp.z * fz;
                            T[0] += sp.y * fz - sp.z * fy;
                            T[1] += sp.z * fx - sp.x * fz;
                            T[2] += sp.x * fy - sp.y * fx;
                        }
                        if (NMU + NQQ > 0) {
#pragma unroll
                            for (int k = 0; k < NPOL; ++k) {
                                T[0] += ts[k].x.v.x + ts[k].x.v.y;
                                T[1] += ts[k].y.v.x + ts[k].y.v.y;
                                T[2] += ts[k].z.v.x + ts[k].z.v.y;
                            }
                        }
#pragma unroll
                        for (int o = 8; o > 0; o >>= 1)
#pragma unroll
                            for (int q = 0; q < 3; ++q) {
                                F[q] += __shfl_xor_sync(FULL, F[q], o);
                                T[q] += __shfl_xor_sync(FULL, T[q], o);
                            }
                        float shsum = 0.f;                     // LJTS shifts of one molecule pair (A2)
#pragma unroll
                        for (int k = 0; k < NLJ * NLJ; ++k) shsum += ljp[2 * (k / NLJ) + k % NLJ].w;
                        float qtot = 0.f;                      // molecule charge (one component: partners alike)
#pragma unroll
                        for (int k = 0; k < NQ; ++k) qtot += si[SH::SQ + k].w;
                        Uw += (double)uacc.v.x + (double)uacc.v.y - ((double)shsum + (double)crf * qtot * qtot) * nval;
                        Ww += (double)wacc.v.x + (double)wacc.v.y - (SV ? 2.0 * (double)sdf : 0.0);
                        npw += gl == 0 ? cnt : 0;
                        if (gact && gl == 0) {
                            tgt[0] += F[0]; tgt[1] += F[1]; tgt[2] += F[2];
                            tgt[4] += T[0]; tgt[5] += T[1]; tgt[6] += T[2];
                        }
                    };

                    // ---- distance phase: candidate pair p = base + gl (elements 2p, 2p + 1) against A
                    //      and B, compaction into the two lists (fixed order)
                    int cntA = 0, cntB = 0;
                    const float2 nxA = make_float2(-xiA.x, -xiA.x), nyA = make_float2(-xiA.y, -xiA.y),
                                 nzA = make_float2(-xiA.z, -xiA.z);
                    const float2 nxB = make_float2(-xiB.x, -xiB.x), nyB = make_float2(-xiB.y, -xiB.y),
                                 nzB = make_float2(-xiB.z, -xiB.z);
                    const float hiA = gA ? g.cut2_hi : -1.f, hiB = gB ? g.cut2_hi : -1.f;   // idle: no hits
                    const int span = max(__shfl_sync(FULL, p1 - p0, 0), __shfl_sync(FULL, p1 - p0, 16));
#if MD_RIG3_BITS
                    // hits are collected as per-lane bits over up to 4 iterations (16 bits per list:
                    // bit k = 4 it + 2 u + e for element e of pair p0 + b0 + 32 it + 16 u + gl), then
                    // compacted at once: a group prefix of the lanes' counts (one packed scan for both
                    // lists) and each lane writing its own entries -- lane-major order, fixed
                    int base = 0;
                    for (;;) {
                        const int b0 = base;
                        unsigned bA = 0u, bB = 0u;
#pragma unroll
                        for (int it = 0; it < 4; ++it) {
                            if (base >= span) break;
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const int p = p0 + base + 16 * u + gl;
                                const int pp = p < p1 ? p : CAP / 2;
                                const float4 xy = cxy[pp];
                                const float2 zz = pz[pp];
                                const float2 xx = make_float2(xy.x, xy.y), yy = make_float2(xy.z, xy.w);
                                float2 dx = __fadd2_rn(xx, nxA), dy = __fadd2_rn(yy, nyA), dz = __fadd2_rn(zz, nzA);
                                float2 r2 = __fmul2_rn(dx, dx);
                                r2 = __ffma2_rn(dy, dy, r2);
                                r2 = __ffma2_rn(dz, dz, r2);
                                bA |= ((r2.x < hiA ? 1u : 0u) | (r2.y < hiA ? 2u : 0u)) << (4 * it + 2 * u);
                                dx = __fadd2_rn(xx, nxB); dy = __fadd2_rn(yy, nyB); dz = __fadd2_rn(zz, nzB);
                                r2 = __fmul2_rn(dx, dx);
                                r2 = __ffma2_rn(dy, dy, r2);
                                r2 = __ffma2_rn(dz, dz, r2);
                                bB |= ((r2.x < hiB ? 1u : 0u) | (r2.y < hiB ? 2u : 0u)) << (4 * it + 2 * u);
                            }
                            base += 32;
                        }
                        // group prefix of (count A | count B << 16)
                        const int nab = __popc(bA) | (__popc(bB) << 16);
                        int incl = nab;
#pragma unroll
                        for (int o = 1; o < 16; o <<= 1) {
                            const int v = __shfl_up_sync(FULL, incl, o, 16);
                            if (gl >= o) incl += v;
                        }
                        const int tot = __shfl_sync(FULL, incl, 15, 16);
                        const int totA = tot & 0xffff, totB = tot >> 16;
                        if (__any_sync(FULL, cntA + totA > HCAP || cntB + totB > HCAP)) {
                            __syncwarp();                           // a list would overflow: evaluate both now
                            flush(cntA, hlA, myA, xiA, selfA, tgtA, gA);
                            flush(cntB, hlB, myB, xiB, selfB, tgtB, gB);
                            cntA = cntB = 0;
                            __syncwarp();
                        }
                        const int e0 = 2 * (p0 + b0 + gl);
                        int oA = cntA + ((incl - nab) & 0xffff), oB = cntB + ((incl - nab) >> 16);
                        while (bA) {
                            const int k = __ffs(bA) - 1;
                            bA &= bA - 1u;
                            MD_CHECK(oA < HCAP + 2 && e0 + 16 * k - 15 * (k & 1) < CAP);
                            hlA[oA++] = (uint16_t)(e0 + 16 * k - 15 * (k & 1));
                        }
                        while (bB) {
                            const int k = __ffs(bB) - 1;
                            bB &= bB - 1u;
                            MD_CHECK(oB < HCAP + 2 && e0 + 16 * k - 15 * (k & 1) < CAP);
                            hlB[oB++] = (uint16_t)(e0 + 16 * k - 15 * (k & 1));
                        }
                        cntA += totA;
                        cntB += totB;
                        if (base >= span) break;
                    }
#else
                    unsigned below;
                    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(below));
                    auto append = [&](uint16_t* hl, int& cnt, bool h0, bool h1, int pp) {
                        const unsigned b0 = __ballot_sync(FULL, h0) & gmask, b1 = __ballot_sync(FULL, h1) & gmask;
                        const int n0 = __popc(b0);
                        if (h0) hl[cnt + __popc(b0 & below)] = (uint16_t)(2 * pp);
                        if (h1) hl[cnt + n0 + __popc(b1 & below)] = (uint16_t)(2 * pp + 1);
                        cnt += n0 + __popc(b1);
                    };
                    // two steps per iteration; the lists (HCAP - 64 entries free) are evaluated when full
                    int base = 0;
                    for (;;) {
                        for (; base < span; base += 32) {
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const int p = p0 + base + 16 * u + gl;
                                const int pp = p < p1 ? p : CAP / 2;
                                const float4 xy = cxy[pp];
                                const float2 zz = pz[pp];
                                const float2 xx = make_float2(xy.x, xy.y), yy = make_float2(xy.z, xy.w);
                                float2 dx = __fadd2_rn(xx, nxA), dy = __fadd2_rn(yy, nyA), dz = __fadd2_rn(zz, nzA);
                                float2 r2 = __fmul2_rn(dx, dx);
                                r2 = __ffma2_rn(dy, dy, r2);
                                r2 = __ffma2_rn(dz, dz, r2);
                                const bool a0 = r2.x < hiA, a1 = r2.y < hiA;
                                dx = __fadd2_rn(xx, nxB); dy = __fadd2_rn(yy, nyB); dz = __fadd2_rn(zz, nzB);
                                r2 = __fmul2_rn(dx, dx);
                                r2 = __ffma2_rn(dy, dy, r2);
                                r2 = __ffma2_rn(dz, dz, r2);
                                const bool c0 = r2.x < hiB, c1 = r2.y < hiB;
                                append(hlA, cntA, a0, a1, pp);
                                append(hlB, cntB, c0, c1, pp);
                            }
                            if (__any_sync(FULL, cntA > HCAP - 64 || cntB > HCAP - 64)) { base += 32; break; }
                        }
                        if (base >= span) break;
                        __syncwarp();                               // a list is full: evaluate both now
                        flush(cntA, hlA, myA, xiA, selfA, tgtA, gA);
                        flush(cntB, hlB, myB, xiB, selfB, tgtB, gB);
                        cntA = cntB = 0;
                        __syncwarp();
                    }
#endif
                    __syncwarp();
                    flush(cntA, hlA, myA, xiA, selfA, tgtA, gA);
                    flush(cntB, hlB, myB, xiB, selfB, tgtB, gB);
                    __syncwarp();
                }
            }
            __syncthreads();
            for (int k = tid; k < nb; k += WARPS * 32) {
                float A[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) A[q] = acc[8 * k + q];
                const int t = k - npr * 2 * NG;
                if (split && t >= 0)                          // tail molecule: its slices in order
                    for (int sp = 0; sp < P; ++sp)
#pragma unroll
                        for (int q = 0; q < 8; ++q) A[q] += tacc[8 * (t * P + sp) + q];
                a.force[s_i + ib + k] = make_float4(A[0], A[1], A[2], 0.f);
                a.torque[s_i + ib + k] = make_float4(A[4], A[5], A[6], 0.f);
            }
        }
    }
    Uw = warp_sum_d(Uw);
    Ww = warp_sum_d(Ww);
    npw = warp_sum_ll(npw - nrej - nself);
    ncw = warp_sum_ll(ncw);
    if (lane == 0) a.part[blockIdx.x * WARPS + wib] = ForcePartial{0.5 * Uw, 0.5 * Ww, npw, ncw, 0.0};
}

}  // namespace rig3
