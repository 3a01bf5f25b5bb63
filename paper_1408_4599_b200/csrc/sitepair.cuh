// sitepair.cuh -- fp32 site-site interactions of the force kernels
// (readings A2, A4, A5 of DESIGN.md §2).
//
// Convention: r = x_b - x_a.  Each function ADDS the energy to u, the force
// on site a to fa, the torque on site a (about the site) to ta and the same
// force on a to fhit (the molecule-pair total used for the virial).  Only
// quantities of the home molecule (side a) are accumulated: the kernels run
// the full 27-cell shell, so every pair is also visited from the other side.
#pragma once
#include "common.cuh"

__device__ __forceinline__ float3 f3(float4 v) { return make_float3(v.x, v.y, v.z); }

// 1/x and 1/sqrt(x): MUFU approximation + one Newton step written on the
// small residual e (y + y e / 2), which keeps e at full relative precision:
// nearly correctly rounded and unbiased, cheaper than the IEEE sequences.
// The raw MUFU values (and the y (1.5 - x y^2 / 2) form, whose correction is
// quantised to ulp(1)) bias the water virial by 2-5e-5, because the site
// terms of neutral molecules cancel.
__device__ __forceinline__ float rcp_nr(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return fmaf(r, fmaf(-x, r, 1.f), r);
}
__device__ __forceinline__ float rsqrt_nr(float x)
{
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    const float e = fmaf(-x * y, y, 1.f);
    return fmaf(0.5f * y, e, y);
}
__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// LJ 12-6 (Eq. 1), energy shifted by `shift` (LJTS, A2); force unshifted.
__device__ __forceinline__ void pair_lj(float3 r, float sig2, float eps24, float eps4, float shift,
                                        float& u, float3& fa, float3& fhit)
{
    float r2 = r.x * r.x + r.y * r.y + r.z * r.z;
    float ir2 = rcp_nr(r2);
    float s2 = sig2 * ir2;
    float s6 = s2 * s2 * s2;
    float fr = eps24 * ir2 * s6 * (2.f * s6 - 1.f);          // f_b = fr r
    u += eps4 * s6 * (s6 - 1.f) - shift;
    fa.x -= fr * r.x; fa.y -= fr * r.y; fa.z -= fr * r.z;
    fhit.x -= fr * r.x; fhit.y -= fr * r.y; fhit.z -= fr * r.z;
}

// charge-charge with reaction field (A4): u = qq (1/r + krf r^2 - crf)
__device__ __forceinline__ void pair_qq(float3 r, float qq, float krf, float crf, float& u, float3& fa,
                                        float3& fhit)
{
    float r2 = r.x * r.x + r.y * r.y + r.z * r.z;
    float ir = rsqrt_nr(r2);
    float ir2 = ir * ir;
    u += qq * (ir + krf * r2 - crf);
    float fr = qq * (ir * ir2 - 2.f * krf);
    fa.x -= fr * r.x; fa.y -= fr * r.y; fa.z -= fr * r.z;
    fhit.x -= fr * r.x; fhit.y -= fr * r.y; fhit.z -= fr * r.z;
}

// Point multipoles (A5): u(r, c_a, c_b, c_ab) with c_a = e_a.rhat,
// c_b = e_b.rhat, c_ab = e_a.e_b; KA, KB in {MD_CHARGE, MD_DIPOLE, MD_QUAD},
// at least one polar.  Force on a = +du/dr_vec, torque on a =
// -e_a x (u_ca rhat + u_cab e_b).  kmm = mu-mu reaction-field constant.
template <int KA, int KB>
__device__ __forceinline__ void pair_polar(float3 r, float ma, float3 ea, float mb, float3 eb, float kmm,
                                           float& u, float3& fa, float3& ta, float3& fhit)
{
    float r2 = r.x * r.x + r.y * r.y + r.z * r.z;
    float ir = rsqrt_nr(r2);
    float ir2 = ir * ir, ir3 = ir2 * ir;
    float3 rh = make_float3(r.x * ir, r.y * ir, r.z * ir);
    float ca = (KA == MD_CHARGE) ? 0.f : dot3(ea, rh);
    float cb = (KB == MD_CHARGE) ? 0.f : dot3(eb, rh);
    float cab = (KA == MD_CHARGE || KB == MD_CHARGE) ? 0.f : dot3(ea, eb);
    float p = ma * mb;
    float uu = 0.f, ur = 0.f, uca = 0.f, ucb = 0.f, ucab = 0.f;
    if (KA == MD_CHARGE && KB == MD_DIPOLE) {
        uu = -p * cb * ir2; ur = 2.f * p * cb * ir3; ucb = -p * ir2;
    } else if (KA == MD_DIPOLE && KB == MD_CHARGE) {
        uu = p * ca * ir2; ur = -2.f * p * ca * ir3; uca = p * ir2;
    } else if (KA == MD_CHARGE && KB == MD_QUAD) {
        uu = 0.5f * p * (3.f * cb * cb - 1.f) * ir3; ur = -3.f * uu * ir; ucb = 3.f * p * cb * ir3;
    } else if (KA == MD_QUAD && KB == MD_CHARGE) {
        uu = 0.5f * p * (3.f * ca * ca - 1.f) * ir3; ur = -3.f * uu * ir; uca = 3.f * p * ca * ir3;
    } else if (KA == MD_DIPOLE && KB == MD_DIPOLE) {
        uu = p * (cab - 3.f * ca * cb) * ir3; ur = -3.f * uu * ir;
        uca = -3.f * p * cb * ir3; ucb = -3.f * p * ca * ir3; ucab = p * ir3 - kmm * p;
        uu -= kmm * p * cab;
    } else if (KA == MD_DIPOLE && KB == MD_QUAD) {
        float pp = 1.5f * p * ir2 * ir2;
        uu = pp * (ca * (5.f * cb * cb - 1.f) - 2.f * cb * cab); ur = -4.f * uu * ir;
        uca = pp * (5.f * cb * cb - 1.f); ucb = pp * (10.f * ca * cb - 2.f * cab); ucab = -2.f * pp * cb;
    } else if (KA == MD_QUAD && KB == MD_DIPOLE) {
        float pp = -1.5f * p * ir2 * ir2;
        uu = pp * (cb * (5.f * ca * ca - 1.f) - 2.f * ca * cab); ur = -4.f * uu * ir;
        ucb = pp * (5.f * ca * ca - 1.f); uca = pp * (10.f * ca * cb - 2.f * cab); ucab = -2.f * pp * ca;
    } else if (KA == MD_QUAD && KB == MD_QUAD) {
        float pp = 0.75f * p * ir3 * ir2;
        float gg = cab - 5.f * ca * cb;
        uu = pp * (1.f - 5.f * ca * ca - 5.f * cb * cb - 15.f * ca * ca * cb * cb + 2.f * gg * gg);
        ur = -5.f * uu * ir;
        uca = pp * (-10.f * ca - 30.f * ca * cb * cb - 20.f * cb * gg);
        ucb = pp * (-10.f * cb - 30.f * ca * ca * cb - 20.f * ca * gg);
        ucab = 4.f * pp * gg;
    }
    u += uu;
    // du/dr_vec = ur rhat + (uca (ea - ca rhat) + ucb (eb - cb rhat)) / r ; force on a = +du
    float k0 = ur - (uca * ca + ucb * cb) * ir;
    float3 du = make_float3(k0 * rh.x, k0 * rh.y, k0 * rh.z);
    if (KA != MD_CHARGE) { du.x += uca * ir * ea.x; du.y += uca * ir * ea.y; du.z += uca * ir * ea.z; }
    if (KB != MD_CHARGE) { du.x += ucb * ir * eb.x; du.y += ucb * ir * eb.y; du.z += ucb * ir * eb.z; }
    fa.x += du.x; fa.y += du.y; fa.z += du.z;
    fhit.x += du.x; fhit.y += du.y; fhit.z += du.z;
    if (KA != MD_CHARGE) {
        float3 gv = make_float3(uca * rh.x, uca * rh.y, uca * rh.z);
        if (KB != MD_CHARGE) { gv.x += ucab * eb.x; gv.y += ucab * eb.y; gv.z += ucab * eb.z; }
        ta.x -= ea.y * gv.z - ea.z * gv.y;
        ta.y -= ea.z * gv.x - ea.x * gv.z;
        ta.z -= ea.x * gv.y - ea.y * gv.x;
    }
}
