// packed2.cuh -- packed fp32x2 arithmetic (one FADD2 / FMUL2 / FFMA2 per
// operation on sm_100) and the packed point-multipole site pairs (reading A5)
// of the rigid force kernel (kernels_rigid3.cuh, which holds the packed LJ and
// charge-charge terms), for two molecule pairs at a time.
#pragma once
#include "common.cuh"
#include "kernels_force.cuh"

namespace pk2 {


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
__device__ __forceinline__ P2 neg(P2 a) { return P2{make_float2(-a.v.x, -a.v.y)}; }   // folded into the operand
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

// point multipoles (A5), same closed forms and gradient recipe as
// sitepair.cuh:pair_polar; p = m_a m_b (masked)
// SV: no partner-pair force fh; the site virial -r . f_a = -|r| u_r is summed into w instead
// (r . du = |r| u_r exactly: the angular terms are orthogonal to r after the k0 correction)
template <int KA, int KB, bool SV = false>
__device__ __forceinline__ void polar2(V3 r, V3 ea, V3 eb, P2 p, float kmm, P2& u, V3& fa, V3& ta, V3& fh, P2& w)
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
    if (SV) {
        w = fma(neg(r2 * ir), ur, w);
    } else {
        fh.x += du.x; fh.y += du.y; fh.z += du.z;
    }
    if (KA != MD_CHARGE) {
        V3 gv = V3{uca * rh.x, uca * rh.y, uca * rh.z};
        if (KB != MD_CHARGE) { gv.x = fma(ucab, eb.x, gv.x); gv.y = fma(ucab, eb.y, gv.y); gv.z = fma(ucab, eb.z, gv.z); }
        ta.x -= ea.y * gv.z - ea.z * gv.y;
        ta.y -= ea.z * gv.x - ea.x * gv.z;
        ta.z -= ea.x * gv.y - ea.y * gv.x;
    }
}

}  // namespace pk2
