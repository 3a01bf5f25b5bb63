// kernels_force.cuh -- the generic rigid-molecule force/torque kernel (mixtures,
// every site kind, runtime site counts; hot loop of the method: "the largest
// part of the computational cost is caused by the force and distance
// calculations"; linked cells P:134-155), and the row helpers
// it shares with the packed single-component kernel (kernels_rigid3.cuh, packed2.cuh).  The
// single-site LJ kernel is in kernels_lj1.cuh.
//
// Work decomposition.  Persistent grid; each warp owns a
// home cell at a time (cells strided over warps, x fastest, so the cells in
// flight at any moment form a few consecutive z-planes that stay in L2).  The
// warp stages the 27-cell neighbourhood (9 rows of 3 cells) into its shared
// memory in chunks with the geometric cell offset already added, so that every
// staged coordinate is relative to the home cell's origin and every
// separation d = X_j - x_i is an EXACT fp32 multiple of the quantum s
// (reading A12).  Lanes are (i-slot, j-phase) pairs: n_i molecules of the
// home cell x P = floor(32 / n_i) phases.  Full shell (no Newton-3 scatter,
// no atomics): each lane accumulates the force and torque on its own molecule
// only; the phases of a molecule are combined with warp shuffles in fixed
// order, energies and virials per warp in fp64 in fixed order (deterministic).
//
// Cutoff (reading A1, A12): COM separation, strict r < rc.  r^2 in fp32 is
// within 3 ulp of the exact value; inside a +-2^-20 relative band around rc^2
// the decision is recomputed exactly in integer quanta.
#pragma once
#include "common.cuh"
#include "sitepair.cuh"

struct ForceArgs {
    GridP g;
    int n, cap;
    const int* start;            // ncell + 1
    const float4* xs;            // staging coordinates
    const float4* site;          // [n_slots][cap] (rigid)
    float4* force;
    float4* torque;
    ForcePartial* part;          // one per warp of the grid
    int* flag;                   // error flags (2 = coincident molecule centres)
    const DevModel* model;
    float sig2, eps24, eps4, shift;   // single-site LJ fast path
    // one-component rigid kernels (rig3): LJ site pairs (ia, ib < 2) as (sigma^2, 24 eps, 4 eps,
    // shift) and the reaction-field constants, as kernel parameters -- constant-bank operands
    // instead of registers
    float4 lj3[4];
    float krf, crf, kmm;
    float hsym[2];               // rig3 SYM: the LJ sites' positions along the molecular axis
};

// Row descriptor of the 27-cell neighbourhood: the 3 cells (dx = -1, 0, 1)
// of row (dy, dz).  Lanes 0..2 fetch start/count, broadcast by shuffles.
struct Row {
    int st0, st1, st2, n0, n1, n2;
};

__device__ __forceinline__ Row load_row(const int* __restrict__ start, const GridP& g, int cx, int cy,
                                        int cz, int dy, int dz)
{
    const int lane = threadIdx.x & 31;
    int ry = wrapi(cy + dy, g.wn[1]), rz = wrapi(cz + dz, g.wn[2]);     // rank-local window
    int st = 0, cn = 0;
    if (lane < 3) {
        int c = wrapi(cx + lane - 1, g.wn[0]) + g.wn[0] * (ry + g.wn[1] * rz);
        st = __ldg(start + c);
        cn = __ldg(start + c + 1) - st;
    }
    Row r;
    r.st0 = __shfl_sync(0xffffffffu, st, 0);
    r.st1 = __shfl_sync(0xffffffffu, st, 1);
    r.st2 = __shfl_sync(0xffffffffu, st, 2);
    r.n0 = __shfl_sync(0xffffffffu, cn, 0);
    r.n1 = __shfl_sync(0xffffffffu, cn, 1);
    r.n2 = __shfl_sync(0xffffffffu, cn, 2);
    return r;
}

// element kk of a row -> source slot and x offset (-edge, 0, +edge)
__device__ __forceinline__ int row_src(const Row& r, int kk, float edge, float& offx)
{
    if (kk < r.n0) { offx = -edge; return r.st0 + kk; }
    if (kk < r.n0 + r.n1) { offx = 0.f; return r.st1 + kk - r.n0; }
    offx = edge;
    return r.st2 + kk - r.n0 - r.n1;
}

// The single-site LJ kernel (configs 0, 1, 4) is in kernels_lj1.cuh.

// =========================================================================
// Rigid multi-centre molecules (configs 2, 3; mixtures and dipoles through
// the generic instantiation).  One thread per home molecule owning all of
// its sites (see DESIGN.md §6 for why not one thread per site); site-pair
// loops are unrolled at compile time for the component shape.
//   NLJ, NQ, NMU, NQQ : site counts (exact, or maxima when GEN)
//   GEN               : several components / runtime counts
// Slot layout per molecule: [LJ pos][charge pos, w = q][dipole pos, axis]
// [quadrupole pos, axis], world frame relative to the COM.
// =========================================================================
#ifndef RIG_CAP
#define RIG_CAP 128
#endif

template <int NLJ, int NQ, int NMU, int NQQ, int WARPS>
constexpr int rigid_smem() { return WARPS * ((1 + NLJ + NQ + 2 * NMU + 2 * NQQ) * RIG_CAP + RIG_CAP * 2) * 16; }

template <int NLJ, int NQ, int NMU, int NQQ>
struct Shape {
    static constexpr int NS = NLJ + NQ + NMU + NQQ;
    static constexpr int NSLOT = NLJ + NQ + 2 * NMU + 2 * NQQ;
    static constexpr int SQ = NLJ, SMU = NLJ + NQ, SQQ = NLJ + NQ + 2 * NMU;
};

template <int NLJ, int NQ, int NMU, int NQQ, bool GEN, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_force_rigid(ForceArgs a)
{
    using SH = Shape<NLJ, NQ, NMU, NQQ>;
    constexpr int NSLOT = SH::NSLOT;
    constexpr int NPOL = (NMU + NQQ) > 0 ? (NMU + NQQ) : 1;
    extern __shared__ float4 smem_rig[];
    constexpr int PER_WARP = (1 + NSLOT) * RIG_CAP + RIG_CAP * 2;     // float4 units (queue: RIG_CAP*32 B)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float4* com = smem_rig + wib * PER_WARP;
    float4* ssw = com + RIG_CAP;                     // ssw[slot * RIG_CAP + j]
    uint8_t* qcol = reinterpret_cast<uint8_t*>(ssw + NSLOT * RIG_CAP) + lane;   // this lane's queue column
    const GridP& g = a.g;
    const DevModel* __restrict__ M = a.model;
    const int gw = blockIdx.x * WARPS + wib, nw = gridDim.x * WARPS;
    const float krf = M->krf, crf = M->crf, kmm = M->krf_mumu;
    // single-component shapes: LJ pair parameters in registers (no per-pair loads)
    float4 ljp[NLJ > 0 ? NLJ * NLJ : 1];
#pragma unroll
    for (int ia = 0; ia < NLJ; ++ia)
#pragma unroll
        for (int ib = 0; ib < NLJ; ++ib) {
            const int t = ia * MD_MAX_LJ_TOTAL + ib;
            ljp[ia * NLJ + ib] = GEN ? make_float4(0.f, 0.f, 0.f, 0.f)
                                     : make_float4(M->sig2[t], M->eps24[t], M->eps4[t], M->shift[t]);
        }
    double Uw = 0.0, Ww = 0.0;
    long long npw = 0, ncw = 0;

    for (int t = gw; t < g.nhome; t += nw) {
        int cx, cy, cz;
        const int c = home_cell(g, t, cx, cy, cz);
        const int s_i = __ldg(a.start + c);
        const int n_all = __ldg(a.start + c + 1) - s_i;
        if (n_all == 0) continue;
        for (int i0 = 0; i0 < n_all; i0 += 32) {
            const int ni = min(32, n_all - i0);
            const int P = 32 / ni;
            const int islot = lane % ni, phase = lane / ni;
            const bool active = phase < P;
            const int my = s_i + i0 + islot;
            const float4 xi = a.xs[my];
            const int ci = __float_as_int(xi.w);
            const DevComp& Ci = M->comp[ci];
            // own sites (positions / axes) in registers
            float4 si[NSLOT];
#pragma unroll
            for (int k = 0; k < NSLOT; ++k)
                si[k] = (GEN && k >= Ci.n_slots) ? make_float4(0.f, 0.f, 0.f, 0.f)
                                                 : a.site[(size_t)k * a.cap + my];
            float3 fs[SH::NS];
            float3 ts[NPOL];
#pragma unroll
            for (int k = 0; k < SH::NS; ++k) fs[k] = make_float3(0.f, 0.f, 0.f);
#pragma unroll
            for (int k = 0; k < NPOL; ++k) ts[k] = make_float3(0.f, 0.f, 0.f);
            float uacc = 0.f, wacc = 0.f;
            int hits = 0, mtot = 0, m = 0;

            auto compute = [&](int mm) {
                // distance phase: COM test (A1) for this lane's candidates,
                // hits appended to the lane's queue column (slab indices)
                int cnt = 0;
                if (active) {
                    for (int j = phase; j < mm; j += P) {
                        const float4 X = com[j];
                        const float dx = X.x - xi.x, dy = X.y - xi.y, dz = X.z - xi.z;
                        const float r2 = dx * dx + dy * dy + dz * dz;
                        bool hit = (r2 < g.cut2_hi) && ((__float_as_int(X.w) >> 3) != my);
                        if (hit && r2 >= g.cut2_lo) hit = exact_in_range(dx, dy, dz, g);   // guard band (rare)
                        qcol[cnt * 32] = (uint8_t)j;         // unconditional; the slot is reused on a miss
                        cnt += hit ? 1 : 0;
                    }
                }
                hits += cnt;
                __syncwarp();
                // force phase: all site pairs of the queued molecule pairs
                const int cmax = __reduce_max_sync(0xffffffffu, cnt);
                for (int k = 0; k < cmax; ++k) {
                    if (k >= cnt) continue;
                    const int j = qcol[k * 32];
                    const float4 X = com[j];
                    const float dx = X.x - xi.x, dy = X.y - xi.y, dz = X.z - xi.z;
                    const int wj = __float_as_int(X.w);
                    const int cj = wj & 7;
                    const DevComp& Cj = M->comp[cj];
                    const float3 d = make_float3(dx, dy, dz);
                    float3 fh = make_float3(0.f, 0.f, 0.f);
                    // ---- LJ x LJ
#pragma unroll
                    for (int ia = 0; ia < NLJ; ++ia) {
                        if (GEN && ia >= Ci.n_lj) break;
#pragma unroll
                        for (int ib = 0; ib < NLJ; ++ib) {
                            if (GEN && ib >= Cj.n_lj) break;
                            const float4 sb = ssw[(ib) * RIG_CAP + (j)];
                            const float3 rv = make_float3(d.x + sb.x - si[ia].x, d.y + sb.y - si[ia].y,
                                                          d.z + sb.z - si[ia].z);
                            if (GEN) {
                                const int t = (Ci.lj0 + ia) * MD_MAX_LJ_TOTAL + Cj.lj0 + ib;
                                pair_lj(rv, M->sig2[t], M->eps24[t], M->eps4[t], M->shift[t], uacc, fs[ia], fh);
                            } else {
                                const float4 pp = ljp[ia * NLJ + ib];
                                pair_lj(rv, pp.x, pp.y, pp.z, pp.w, uacc, fs[ia], fh);
                            }
                        }
                    }
                    // ---- charge x charge
#pragma unroll
                    for (int ia = 0; ia < NQ; ++ia) {
                        if (GEN && ia >= Ci.n_q) break;
                        const float4 sa = GEN ? a.site[(size_t)(Ci.n_lj + ia) * a.cap + my] : si[SH::SQ + ia];
#pragma unroll
                        for (int ib = 0; ib < NQ; ++ib) {
                            if (GEN && ib >= Cj.n_q) break;
                            const float4 sb = ssw[(GEN ? Cj.n_lj + ib : SH::SQ + ib) * RIG_CAP + (j)];
                            const float3 rv = make_float3(d.x + sb.x - sa.x, d.y + sb.y - sa.y, d.z + sb.z - sa.z);
                            pair_qq(rv, sa.w * sb.w, krf, crf, uacc, fs[NLJ + ia], fh);
                        }
                    }
                    // ---- polar kinds (generic (u_r, u_ca, u_cb, u_cab) recipe)
                    if (NMU + NQQ > 0) {
                        // sides: a = home molecule site, b = partner site
#define MD_POLAR_LOOP(KA, KB, NA, NB, SLA, SLB, CNTA, CNTB, FIDX, TIDX, STA, STB)                     \
    _Pragma("unroll") for (int ia = 0; ia < NA; ++ia)                                                  \
    {                                                                                                  \
        if (GEN && ia >= (CNTA)) break;                                                                \
        const int sla = (SLA) + ia * STA;                                                              \
        const float4 pa = GEN ? a.site[(size_t)sla * a.cap + my] : si[(SLA) + ia * STA];               \
        const float4 ea4 = (STA == 2) ? (GEN ? a.site[(size_t)(sla + 1) * a.cap + my]                   \
                                             : si[((SLA) + ia * STA + 1) % NSLOT])                      \
                                      : make_float4(0.f, 0.f, 0.f, 0.f);                               \
        _Pragma("unroll") for (int ib = 0; ib < NB; ++ib)                                              \
        {                                                                                              \
            if (GEN && ib >= (CNTB)) break;                                                            \
            const int slb = (SLB) + ib * STB;                                                          \
            const float4 pb = ssw[(slb) * RIG_CAP + (j)];                                                      \
            const float4 eb4 = (STB == 2) ? ssw[((slb + 1) % NSLOT) * RIG_CAP + (j)] : make_float4(0.f, 0.f, 0.f, 0.f); \
            const float3 rv = make_float3(d.x + pb.x - pa.x, d.y + pb.y - pa.y, d.z + pb.z - pa.z);  \
            float3 tdummy = make_float3(0.f, 0.f, 0.f);                                                \
            pair_polar<KA, KB>(rv, pa.w, f3(ea4), pb.w, f3(eb4), kmm, uacc, fs[FIDX + ia],            \
                               (TIDX) >= 0 ? ts[((TIDX) >= 0 ? (TIDX) : 0) + ia] : tdummy, fh);       \
        }                                                                                              \
    }
                        const int jq = GEN ? Cj.n_lj : SH::SQ;
                        const int jmu = GEN ? Cj.n_lj + Cj.n_q : SH::SMU;
                        const int jqq = GEN ? Cj.n_lj + Cj.n_q + 2 * Cj.n_mu : SH::SQQ;
                        const int imu = GEN ? Ci.n_lj + Ci.n_q : SH::SMU;
                        const int iqq = GEN ? Ci.n_lj + Ci.n_q + 2 * Ci.n_mu : SH::SQQ;
                        const int iq = GEN ? Ci.n_lj : SH::SQ;
                        if (NQ > 0 && NMU > 0) {
                            MD_POLAR_LOOP(MD_CHARGE, MD_DIPOLE, NQ, NMU, iq, jmu, Ci.n_q, Cj.n_mu, NLJ, -1, 1, 2)
                            MD_POLAR_LOOP(MD_DIPOLE, MD_CHARGE, NMU, NQ, imu, jq, Ci.n_mu, Cj.n_q, NLJ + NQ, 0, 2, 1)
                        }
                        if (NQ > 0 && NQQ > 0) {
                            MD_POLAR_LOOP(MD_CHARGE, MD_QUAD, NQ, NQQ, iq, jqq, Ci.n_q, Cj.n_Q, NLJ, -1, 1, 2)
                            MD_POLAR_LOOP(MD_QUAD, MD_CHARGE, NQQ, NQ, iqq, jq, Ci.n_Q, Cj.n_q, NLJ + NQ + NMU, NMU, 2, 1)
                        }
                        if (NMU > 0) {
                            MD_POLAR_LOOP(MD_DIPOLE, MD_DIPOLE, NMU, NMU, imu, jmu, Ci.n_mu, Cj.n_mu, NLJ + NQ, 0, 2, 2)
                        }
                        if (NMU > 0 && NQQ > 0) {
                            MD_POLAR_LOOP(MD_DIPOLE, MD_QUAD, NMU, NQQ, imu, jqq, Ci.n_mu, Cj.n_Q, NLJ + NQ, 0, 2, 2)
                            MD_POLAR_LOOP(MD_QUAD, MD_DIPOLE, NQQ, NMU, iqq, jmu, Ci.n_Q, Cj.n_mu, NLJ + NQ + NMU, NMU, 2, 2)
                        }
                        if (NQQ > 0) {
                            MD_POLAR_LOOP(MD_QUAD, MD_QUAD, NQQ, NQQ, iqq, jqq, Ci.n_Q, Cj.n_Q, NLJ + NQ + NMU, NMU, 2, 2)
                        }
#undef MD_POLAR_LOOP
                    }
                    // molecular virial (A6): -r_ij . F_ij, F_ij = force on i from j
                    wacc -= d.x * fh.x + d.y * fh.y + d.z * fh.z;
                }
            };

            for (int row = 0; row < 9; ++row) {
                const int dy = row % 3 - 1, dz = row / 3 - 1;
                const Row r = load_row(a.start, g, cx, cy, cz, dy, dz);
                const int tot = r.n0 + r.n1 + r.n2;
                mtot += tot;
                const float offy = dy * g.edge[1], offz = dz * g.edge[2];
                int k0 = 0;
                while (k0 < tot) {
                    const int take = min(tot - k0, RIG_CAP - m);
                    for (int k = lane; k < take; k += 32) {
                        float offx;
                        const int src = row_src(r, k0 + k, g.edge[0], offx);
                        const float4 x = a.xs[src];
                        const int cj = __float_as_int(x.w);
                        com[m + k] = make_float4(x.x + offx, x.y + offy, x.z + offz, __int_as_float(src * 8 + cj));
                        const int nsl = GEN ? M->comp[cj].n_slots : NSLOT;
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if (s < nsl) ssw[(s) * RIG_CAP + (m + k)] = a.site[(size_t)s * a.cap + src];
                    }
                    m += take;
                    k0 += take;
                    if (m == RIG_CAP) {
                        __syncwarp();
                        compute(m);
                        __syncwarp();
                        m = 0;
                    }
                }
            }
            __syncwarp();
            compute(m);
            __syncwarp();
            // molecule force and torque: F = sum_a f_a, tau = sum_a s_a x f_a + tau_a
            float3 F = make_float3(0.f, 0.f, 0.f), T = make_float3(0.f, 0.f, 0.f);
#pragma unroll
            for (int k = 0; k < SH::NS; ++k) {
                // site k in kind order -> its position slot
                int slot;
                if (k < NLJ) slot = k;
                else if (k < NLJ + NQ) slot = (GEN ? Ci.n_lj : NLJ) + (k - NLJ);
                else if (k < NLJ + NQ + NMU) slot = (GEN ? Ci.n_lj + Ci.n_q : SH::SMU) + 2 * (k - NLJ - NQ);
                else slot = (GEN ? Ci.n_lj + Ci.n_q + 2 * Ci.n_mu : SH::SQQ) + 2 * (k - NLJ - NQ - NMU);
                float4 sp;
                if (GEN) sp = (slot < Ci.n_slots) ? a.site[(size_t)slot * a.cap + my] : make_float4(0.f, 0.f, 0.f, 0.f);
                else sp = si[slot < NSLOT ? slot : 0];
                F.x += fs[k].x; F.y += fs[k].y; F.z += fs[k].z;
                T.x += sp.y * fs[k].z - sp.z * fs[k].y;
                T.y += sp.z * fs[k].x - sp.x * fs[k].z;
                T.z += sp.x * fs[k].y - sp.y * fs[k].x;
            }
            if (NMU + NQQ > 0) {
#pragma unroll
                for (int k = 0; k < NPOL; ++k) { T.x += ts[k].x; T.y += ts[k].y; T.z += ts[k].z; }
            }
            float3 SF = F, ST = T;
            for (int p = 1; p < P; ++p) {
                const int srcl = (lane + p * ni) & 31;
                SF.x += __shfl_sync(0xffffffffu, F.x, srcl);
                SF.y += __shfl_sync(0xffffffffu, F.y, srcl);
                SF.z += __shfl_sync(0xffffffffu, F.z, srcl);
                ST.x += __shfl_sync(0xffffffffu, T.x, srcl);
                ST.y += __shfl_sync(0xffffffffu, T.y, srcl);
                ST.z += __shfl_sync(0xffffffffu, T.z, srcl);
            }
            if (phase == 0) {
                a.force[my] = make_float4(SF.x, SF.y, SF.z, 0.f);
                a.torque[my] = make_float4(ST.x, ST.y, ST.z, 0.f);
            }
            Uw += (double)uacc;
            Ww += (double)wacc;
            npw += hits;
            if (lane == 0) ncw += (long long)ni * (mtot - 1);
        }
    }
    Uw = warp_sum_d(Uw);
    Ww = warp_sum_d(Ww);
    npw = warp_sum_ll(npw);
    if (lane == 0) {
        ForcePartial p;
        p.U = 0.5 * Uw;
        p.W = 0.5 * Ww;
        p.npairs = npw;
        p.ncand = ncw;
        p.K = 0.0;
        a.part[gw] = p;
    }
}
