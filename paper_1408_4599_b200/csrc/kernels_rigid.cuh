// kernels_rigid.cuh -- force/torque kernel for rigid multi-centre molecules of
// one component (configs 2 and 3: 2CLJQ, TIP4P, linked
// cells P:134-155), packed two molecule pairs at a time.
//
// Decomposition as k_force_rigid (kernels_force.cuh): one warp per home cell,
// lanes are (molecule, phase) pairs, the 27-cell neighbourhood is staged in
// chunks of RIG_CAP molecules (COM + world-frame site slots), a distance
// phase queues the partners within rc (COM cutoff, reading A1) per lane and a
// force phase evaluates all site pairs of the queued molecule pairs.  Both
// phases here take TWO candidates / partners per step in the packed fp32x2
// instructions of sm_100 (FADD2 / FMUL2 / FFMA2): the site-pair arithmetic of
// partners j0 and j1 of the same home molecule is one instruction stream on
// float2 values, which halves the issue slots of the arithmetic.  An odd
// queue is padded with a far dummy slot whose prefactors are masked to zero.
#pragma once
#include "common.cuh"
#include "kernels_force.cuh"

namespace rig2 {

// staged molecules per chunk: 4 CTAs of 4 warps fit one SM's 228 KB with 4-slot shapes
constexpr int R2CAP = 120;

// ---- packed float2 arithmetic (one FADD2 / FMUL2 / FFMA2 each)
struct P2 {
    float2 v;
};
__device__ __forceinline__ P2 p2(float a) { return P2{make_float2(a, a)}; }
__device__ __forceinline__ P2 p2(float a, float b) { return P2{make_float2(a, b)}; }
__device__ __forceinline__ P2 operator+(P2 a, P2 b) { return P2{__fadd2_rn(a.v, b.v)}; }
__device__ __forceinline__ P2 operator-(P2 a, P2 b) { return P2{__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))}; }
__device__ __forceinline__ P2 operator*(P2 a, P2 b) { return P2{__fmul2_rn(a.v, b.v)}; }
__device__ __forceinline__ P2 operator*(float a, P2 b) { return P2{__fmul2_rn(make_float2(a, a), b.v)}; }
__device__ __forceinline__ P2 fma(P2 a, P2 b, P2 c) { return P2{__ffma2_rn(a.v, b.v, c.v)}; }
__device__ __forceinline__ P2& operator+=(P2& a, P2 b) { a = a + b; return a; }
__device__ __forceinline__ P2& operator-=(P2& a, P2 b) { a = a - b; return a; }

struct V3 {
    P2 x, y, z;
};
__device__ __forceinline__ V3 v3zero() { return V3{p2(0.f), p2(0.f), p2(0.f)}; }
__device__ __forceinline__ P2 dot(V3 a, V3 b) { return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x)); }
__device__ __forceinline__ V3 bcast(float4 a) { return V3{p2(a.x), p2(a.y), p2(a.z)}; }
__device__ __forceinline__ V3 pack(float4 a, float4 b) { return V3{p2(a.x, b.x), p2(a.y, b.y), p2(a.z, b.z)}; }

// 1/x and 1/sqrt(x) per component: MUFU + one Newton step on the residual
// (same form as sitepair.cuh: unbiased)
__device__ __forceinline__ P2 rcp2(P2 x)
{
    float a, b;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x.v.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x.v.y));
    const P2 r = p2(a, b);
    return fma(r, fma(P2{make_float2(-x.v.x, -x.v.y)}, r, p2(1.f)), r);
}
__device__ __forceinline__ P2 rsqrt2(P2 x)
{
    float a, b;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x.v.x));
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x.v.y));
    const P2 y = p2(a, b);
    const P2 e = fma(P2{make_float2(-x.v.x, -x.v.y)} * y, y, p2(1.f));
    return fma(p2(0.5f) * y, e, y);
}

// LJ 12-6, energy shifted (LJTS, A2), r = x_b - x_a; m = mask (0 for padding)
__device__ __forceinline__ void lj2(V3 r, float sig2, P2 eps24m, P2 eps4m, P2 shiftm, P2& u, V3& fa, V3& fh)
{
    const P2 r2 = dot(r, r);
    const P2 ir2 = rcp2(r2);
    const P2 s2 = sig2 * ir2;
    const P2 s6 = s2 * s2 * s2;
    const P2 fr = eps24m * ir2 * s6 * fma(p2(2.f), s6, p2(-1.f));
    u = fma(eps4m * s6, s6 - p2(1.f), u) - shiftm;
    fa.x = fa.x - fr * r.x; fa.y = fa.y - fr * r.y; fa.z = fa.z - fr * r.z;
    fh.x = fh.x - fr * r.x; fh.y = fh.y - fr * r.y; fh.z = fh.z - fr * r.z;
}

// charge-charge with reaction field (A4)
__device__ __forceinline__ void qq2(V3 r, P2 qq, float krf, float crf, P2& u, V3& fa, V3& fh)
{
    const P2 r2 = dot(r, r);
    const P2 ir = rsqrt2(r2);
    const P2 ir2 = ir * ir;
    u = fma(qq, fma(p2(krf), r2, ir) - p2(crf), u);
    const P2 fr = qq * fma(ir, ir2, p2(-2.f * krf));
    fa.x = fa.x - fr * r.x; fa.y = fa.y - fr * r.y; fa.z = fa.z - fr * r.z;
    fh.x = fh.x - fr * r.x; fh.y = fh.y - fr * r.y; fh.z = fh.z - fr * r.z;
}

// point multipoles (A5), same closed forms and gradient recipe as
// sitepair.cuh:pair_polar; p = m_a m_b (masked)
template <int KA, int KB>
__device__ __forceinline__ void polar2(V3 r, V3 ea, V3 eb, P2 p, float kmm, P2& u, V3& fa, V3& ta, V3& fh)
{
    const P2 r2 = dot(r, r);
    const P2 ir = rsqrt2(r2);
    const P2 ir2 = ir * ir, ir3 = ir2 * ir;
    const V3 rh = V3{r.x * ir, r.y * ir, r.z * ir};
    const P2 ca = (KA == MD_CHARGE) ? p2(0.f) : dot(ea, rh);
    const P2 cb = (KB == MD_CHARGE) ? p2(0.f) : dot(eb, rh);
    const P2 cab = (KA == MD_CHARGE || KB == MD_CHARGE) ? p2(0.f) : dot(ea, eb);
    P2 uu = p2(0.f), ur = p2(0.f), uca = p2(0.f), ucb = p2(0.f), ucab = p2(0.f);
    if (KA == MD_CHARGE && KB == MD_DIPOLE) {
        uu = p2(-1.f) * p * cb * ir2; ur = p2(2.f) * p * cb * ir3; ucb = p2(-1.f) * p * ir2;
    } else if (KA == MD_DIPOLE && KB == MD_CHARGE) {
        uu = p * ca * ir2; ur = p2(-2.f) * p * ca * ir3; uca = p * ir2;
    } else if (KA == MD_CHARGE && KB == MD_QUAD) {
        uu = p2(0.5f) * p * fma(p2(3.f) * cb, cb, p2(-1.f)) * ir3; ur = p2(-3.f) * uu * ir;
        ucb = p2(3.f) * p * cb * ir3;
    } else if (KA == MD_QUAD && KB == MD_CHARGE) {
        uu = p2(0.5f) * p * fma(p2(3.f) * ca, ca, p2(-1.f)) * ir3; ur = p2(-3.f) * uu * ir;
        uca = p2(3.f) * p * ca * ir3;
    } else if (KA == MD_DIPOLE && KB == MD_DIPOLE) {
        const P2 pi3 = p * ir3;
        uu = pi3 * fma(p2(-3.f) * ca, cb, cab); ur = p2(-3.f) * uu * ir;
        uca = p2(-3.f) * pi3 * cb; ucb = p2(-3.f) * pi3 * ca; ucab = pi3 - p2(kmm) * p;
        uu = uu - p2(kmm) * p * cab;
    } else if (KA == MD_DIPOLE && KB == MD_QUAD) {
        const P2 pp = p2(1.5f) * p * ir2 * ir2;
        const P2 t5 = fma(p2(5.f) * cb, cb, p2(-1.f));
        uu = pp * (ca * t5 - p2(2.f) * cb * cab); ur = p2(-4.f) * uu * ir;
        uca = pp * t5; ucb = pp * (p2(10.f) * ca * cb - p2(2.f) * cab); ucab = p2(-2.f) * pp * cb;
    } else if (KA == MD_QUAD && KB == MD_DIPOLE) {
        const P2 pp = p2(-1.5f) * p * ir2 * ir2;
        const P2 t5 = fma(p2(5.f) * ca, ca, p2(-1.f));
        uu = pp * (cb * t5 - p2(2.f) * ca * cab); ur = p2(-4.f) * uu * ir;
        ucb = pp * t5; uca = pp * (p2(10.f) * ca * cb - p2(2.f) * cab); ucab = p2(-2.f) * pp * ca;
    } else if (KA == MD_QUAD && KB == MD_QUAD) {
        const P2 pp = p2(0.75f) * p * ir3 * ir2;
        const P2 gg = fma(p2(-5.f) * ca, cb, cab);
        const P2 ca2 = ca * ca, cb2 = cb * cb;
        // 1 - 5 ca^2 - 5 cb^2 - 15 ca^2 cb^2 + 2 gg^2
        const P2 poly = fma(p2(2.f) * gg, gg, fma(p2(-15.f) * ca2, cb2, fma(p2(-5.f), ca2 + cb2, p2(1.f))));
        uu = pp * poly;
        ur = p2(-5.f) * uu * ir;
        // -10 ca - 30 ca cb^2 - 20 cb gg, and the mirror
        uca = pp * fma(p2(-20.f) * cb, gg, fma(p2(-30.f) * ca, cb2, p2(-10.f) * ca));
        ucb = pp * fma(p2(-20.f) * ca, gg, fma(p2(-30.f) * cb, ca2, p2(-10.f) * cb));
        ucab = p2(4.f) * pp * gg;
    }
    u += uu;
    // du/dr_vec = ur rhat + (uca (ea - ca rhat) + ucb (eb - cb rhat)) / r ; force on a = +du
    const P2 k0 = ur - fma(uca, ca, ucb * cb) * ir;
    V3 du = V3{k0 * rh.x, k0 * rh.y, k0 * rh.z};
    if (KA != MD_CHARGE) {
        const P2 c = uca * ir;
        du.x = fma(c, ea.x, du.x); du.y = fma(c, ea.y, du.y); du.z = fma(c, ea.z, du.z);
    }
    if (KB != MD_CHARGE) {
        const P2 c = ucb * ir;
        du.x = fma(c, eb.x, du.x); du.y = fma(c, eb.y, du.y); du.z = fma(c, eb.z, du.z);
    }
    fa.x += du.x; fa.y += du.y; fa.z += du.z;
    fh.x += du.x; fh.y += du.y; fh.z += du.z;
    if (KA != MD_CHARGE) {
        V3 gv = V3{uca * rh.x, uca * rh.y, uca * rh.z};
        if (KB != MD_CHARGE) { gv.x = fma(ucab, eb.x, gv.x); gv.y = fma(ucab, eb.y, gv.y); gv.z = fma(ucab, eb.z, gv.z); }
        ta.x -= ea.y * gv.z - ea.z * gv.y;
        ta.y -= ea.z * gv.x - ea.x * gv.z;
        ta.z -= ea.x * gv.y - ea.y * gv.x;
    }
}

template <int NLJ, int NQ, int NMU, int NQQ, int WARPS>
constexpr int smem_bytes()
{
    // per warp: (1 + NSLOT) x (R2CAP + 1) float4 slots (+1: the far dummy), queue R2CAP x 32 bytes
    return WARPS * ((1 + NLJ + NQ + 2 * NMU + 2 * NQQ) * (R2CAP + 1) * 16 + R2CAP * 32);
}

template <int NLJ, int NQ, int NMU, int NQQ, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 4) k_force_rigid2(ForceArgs a)
{
    using SH = Shape<NLJ, NQ, NMU, NQQ>;
    constexpr int NSLOT = SH::NSLOT;
    constexpr int NPOL = (NMU + NQQ) > 0 ? (NMU + NQQ) : 1;
    constexpr int STRIDE = R2CAP + 1;                       // slot stride (dummy at index R2CAP)
    constexpr int DUMMY = R2CAP;
    extern __shared__ float4 smem_rig2[];
    constexpr int PER_WARP = (1 + NSLOT) * STRIDE + R2CAP * 2;     // float4 units
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float4* com = smem_rig2 + wib * PER_WARP;
    float4* ssw = com + STRIDE;                               // ssw[slot * STRIDE + j]
    uint8_t* qcol = reinterpret_cast<uint8_t*>(ssw + NSLOT * STRIDE) + lane;
    const GridP& g = a.g;
    const DevModel* __restrict__ M = a.model;
    const int gw = blockIdx.x * WARPS + wib, nw = gridDim.x * WARPS;
    const float krf = M->krf, crf = M->crf, kmm = M->krf_mumu;
    float4 ljp[NLJ > 0 ? NLJ * NLJ : 1];
#pragma unroll
    for (int ia = 0; ia < NLJ; ++ia)
#pragma unroll
        for (int ib = 0; ib < NLJ; ++ib) {
            const int t = ia * MD_MAX_LJ_TOTAL + ib;
            ljp[ia * NLJ + ib] = make_float4(M->sig2[t], M->eps24[t], M->eps4[t], M->shift[t]);
        }
    // far dummy partner (padding of odd queues): COM far away, sites at the COM
    if (lane == 0) {
        com[DUMMY] = make_float4(1.0e4f, 1.0e4f, 1.0e4f, __int_as_float(-8));
#pragma unroll
        for (int s = 0; s < NSLOT; ++s) ssw[s * STRIDE + DUMMY] = make_float4(0.f, 0.f, 1.f, 0.f);
    }
    __syncwarp();
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
            float4 si[NSLOT];
#pragma unroll
            for (int k = 0; k < NSLOT; ++k) si[k] = a.site[(size_t)k * a.cap + my];
            V3 fs[SH::NS];
            V3 ts[NPOL];
#pragma unroll
            for (int k = 0; k < SH::NS; ++k) fs[k] = v3zero();
#pragma unroll
            for (int k = 0; k < NPOL; ++k) ts[k] = v3zero();
            P2 uacc = p2(0.f), wacc = p2(0.f);
            int hits = 0, mtot = 0, m = 0;

            auto compute = [&](int mm) {
                // ---- distance phase, two candidates per step (COM cutoff A1; guard band exact)
                int cnt = 0;
                if (active) {
                    const float2 nxi = make_float2(-xi.x, -xi.x), nyi = make_float2(-xi.y, -xi.y),
                                 nzi = make_float2(-xi.z, -xi.z);
                    for (int j = phase; j < mm; j += 2 * P) {
                        const int j1 = min(j + P, DUMMY);           // past the chunk: the far dummy
                        const float4 X0 = com[j], X1 = com[j1 < mm ? j1 : DUMMY];
                        const float2 dx = __fadd2_rn(make_float2(X0.x, X1.x), nxi);
                        const float2 dy = __fadd2_rn(make_float2(X0.y, X1.y), nyi);
                        const float2 dz = __fadd2_rn(make_float2(X0.z, X1.z), nzi);
                        float2 r2 = __fmul2_rn(dx, dx);
                        r2 = __ffma2_rn(dy, dy, r2);
                        r2 = __ffma2_rn(dz, dz, r2);
                        bool h0 = (r2.x < g.cut2_hi) && ((__float_as_int(X0.w) >> 3) != my);
                        bool h1 = (r2.y < g.cut2_hi) && ((__float_as_int(X1.w) >> 3) != my);
                        if (h0 && r2.x >= g.cut2_lo) h0 = exact_in_range(dx.x, dy.x, dz.x, g);   // guard band (rare)
                        if (h1 && r2.y >= g.cut2_lo) h1 = exact_in_range(dx.y, dy.y, dz.y, g);
                        qcol[cnt * 32] = (uint8_t)j;                   // unconditional; reused on a miss
                        cnt += h0 ? 1 : 0;
                        qcol[cnt * 32] = (uint8_t)j1;
                        cnt += h1 ? 1 : 0;
                    }
                }
                hits += cnt;
                __syncwarp();
                // ---- force phase: partners q[2k], q[2k+1] packed; a missing second is the masked dummy
                const int cmax = __reduce_max_sync(0xffffffffu, cnt);
                for (int k = 0; k < cmax; k += 2) {
                    const bool v0 = k < cnt, v1 = k + 1 < cnt;
                    const int j0 = v0 ? qcol[k * 32] : DUMMY;
                    const int j1 = v1 ? qcol[(k + 1) * 32] : DUMMY;
                    const P2 msk = p2(v0 ? 1.f : 0.f, v1 ? 1.f : 0.f);
                    const float4 X0 = com[j0], X1 = com[j1];
                    const V3 d = V3{p2(X0.x - xi.x, X1.x - xi.x), p2(X0.y - xi.y, X1.y - xi.y),
                                    p2(X0.z - xi.z, X1.z - xi.z)};
                    V3 fh = v3zero();
                    // LJ x LJ
#pragma unroll
                    for (int ia = 0; ia < NLJ; ++ia) {
                        const V3 sa = bcast(si[ia]);
#pragma unroll
                        for (int ib = 0; ib < NLJ; ++ib) {
                            const V3 sb = pack(ssw[ib * STRIDE + j0], ssw[ib * STRIDE + j1]);
                            const V3 rv = V3{d.x + sb.x - sa.x, d.y + sb.y - sa.y, d.z + sb.z - sa.z};
                            const float4 pp = ljp[ia * NLJ + ib];
                            lj2(rv, pp.x, pp.y * msk, pp.z * msk, pp.w * msk, uacc, fs[ia], fh);
                        }
                    }
                    // charge x charge
#pragma unroll
                    for (int ia = 0; ia < NQ; ++ia) {
                        const float4 sa4 = si[SH::SQ + ia];
                        const V3 sa = bcast(sa4);
#pragma unroll
                        for (int ib = 0; ib < NQ; ++ib) {
                            const float4 b0 = ssw[(SH::SQ + ib) * STRIDE + j0], b1 = ssw[(SH::SQ + ib) * STRIDE + j1];
                            const V3 sb = pack(b0, b1);
                            const V3 rv = V3{d.x + sb.x - sa.x, d.y + sb.y - sa.y, d.z + sb.z - sa.z};
                            qq2(rv, sa4.w * p2(b0.w, b1.w) * msk, krf, crf, uacc, fs[NLJ + ia], fh);
                        }
                    }
                    // polar kinds
#define RIG2_POLAR(KA, KB, NA, NB, SLA, SLB, FIDX, TIDX, STA, STB)                                          \
    _Pragma("unroll") for (int ia = 0; ia < NA; ++ia)                                                      \
    {                                                                                                      \
        const float4 pa4 = si[(SLA) + ia * STA];                                                           \
        const V3 pa = bcast(pa4);                                                                          \
        const V3 ea = (STA == 2) ? bcast(si[((SLA) + ia * STA + 1) % NSLOT]) : v3zero();                  \
        _Pragma("unroll") for (int ib = 0; ib < NB; ++ib)                                                  \
        {                                                                                                  \
            const int slb = (SLB) + ib * STB;                                                              \
            const float4 b0 = ssw[slb * STRIDE + j0], b1 = ssw[slb * STRIDE + j1];                         \
            const V3 pb = pack(b0, b1);                                                                    \
            const V3 eb = (STB == 2) ? pack(ssw[((slb + 1) % NSLOT) * STRIDE + j0],                          \
                                            ssw[((slb + 1) % NSLOT) * STRIDE + j1]) : v3zero();             \
            const V3 rv = V3{d.x + pb.x - pa.x, d.y + pb.y - pa.y, d.z + pb.z - pa.z};                     \
            V3 tdummy = v3zero();                                                                          \
            polar2<KA, KB>(rv, ea, eb, pa4.w * p2(b0.w, b1.w) * msk, kmm, uacc, fs[FIDX + ia],             \
                           (TIDX) >= 0 ? ts[((TIDX) >= 0 ? (TIDX) : 0) + ia] : tdummy, fh);              \
        }                                                                                                  \
    }
                    if (NQ > 0 && NMU > 0) {
                        RIG2_POLAR(MD_CHARGE, MD_DIPOLE, NQ, NMU, SH::SQ, SH::SMU, NLJ, -1, 1, 2)
                        RIG2_POLAR(MD_DIPOLE, MD_CHARGE, NMU, NQ, SH::SMU, SH::SQ, NLJ + NQ, 0, 2, 1)
                    }
                    if (NQ > 0 && NQQ > 0) {
                        RIG2_POLAR(MD_CHARGE, MD_QUAD, NQ, NQQ, SH::SQ, SH::SQQ, NLJ, -1, 1, 2)
                        RIG2_POLAR(MD_QUAD, MD_CHARGE, NQQ, NQ, SH::SQQ, SH::SQ, NLJ + NQ + NMU, NMU, 2, 1)
                    }
                    if (NMU > 0) {
                        RIG2_POLAR(MD_DIPOLE, MD_DIPOLE, NMU, NMU, SH::SMU, SH::SMU, NLJ + NQ, 0, 2, 2)
                    }
                    if (NMU > 0 && NQQ > 0) {
                        RIG2_POLAR(MD_DIPOLE, MD_QUAD, NMU, NQQ, SH::SMU, SH::SQQ, NLJ + NQ, 0, 2, 2)
                        RIG2_POLAR(MD_QUAD, MD_DIPOLE, NQQ, NMU, SH::SQQ, SH::SMU, NLJ + NQ + NMU, NMU, 2, 2)
                    }
                    if (NQQ > 0) {
                        RIG2_POLAR(MD_QUAD, MD_QUAD, NQQ, NQQ, SH::SQQ, SH::SQQ, NLJ + NQ + NMU, NMU, 2, 2)
                    }
#undef RIG2_POLAR
                    // molecular virial (A6): -r_ij . F_ij
                    wacc -= dot(d, fh);
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
                    const int take = min(tot - k0, R2CAP - m);
                    for (int k = lane; k < take; k += 32) {
                        float offx;
                        const int src = row_src(r, k0 + k, g.edge[0], offx);
                        const float4 x = a.xs[src];
                        com[m + k] = make_float4(x.x + offx, x.y + offy, x.z + offz, __int_as_float(src * 8));
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s) ssw[s * STRIDE + (m + k)] = a.site[(size_t)s * a.cap + src];
                    }
                    m += take;
                    k0 += take;
                    if (m == R2CAP) {
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
                int slot;
                if (k < NLJ) slot = k;
                else if (k < NLJ + NQ) slot = NLJ + (k - NLJ);
                else if (k < NLJ + NQ + NMU) slot = SH::SMU + 2 * (k - NLJ - NQ);
                else slot = SH::SQQ + 2 * (k - NLJ - NQ - NMU);
                const float4 sp = si[slot < NSLOT ? slot : 0];
                const float fx = fs[k].x.v.x + fs[k].x.v.y, fy = fs[k].y.v.x + fs[k].y.v.y,
                            fz = fs[k].z.v.x + fs[k].z.v.y;
                F.x += fx; F.y += fy; F.z += fz;
                T.x += sp.y * fz - sp.z * fy;
                T.y += sp.z * fx - sp.x * fz;
                T.z += sp.x * fy - sp.y * fx;
            }
            if (NMU + NQQ > 0) {
#pragma unroll
                for (int k = 0; k < NPOL; ++k) {
                    T.x += ts[k].x.v.x + ts[k].x.v.y;
                    T.y += ts[k].y.v.x + ts[k].y.v.y;
                    T.z += ts[k].z.v.x + ts[k].z.v.y;
                }
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
            Uw += (double)uacc.v.x + (double)uacc.v.y;
            Ww += (double)wacc.v.x + (double)wacc.v.y;
            npw += hits;
            if (lane == 0) ncw += (long long)ni * (mtot - 1);
        }
    }
    Uw = warp_sum_d(Uw);
    Ww = warp_sum_d(Ww);
    npw = warp_sum_ll(npw);
    if (lane == 0) a.part[gw] = ForcePartial{0.5 * Uw, 0.5 * Ww, npw, ncw, 0.0};
}

}  // namespace rig2
