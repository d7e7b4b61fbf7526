// common.cuh -- shared device helpers for the RepOps kernels (sm_100a).
//
// Every floating-point operation on the canonical path is written with an
// explicit round-to-nearest intrinsic (__fadd_rn, __fmul_rn, __fmaf_rn,
// __fdiv_rn, __fsqrt_rn) AND the library is compiled with -fmad=false
// -ftz=false -prec-div=true -prec-sqrt=true, so ptxas can neither contract a
// separate multiply and add into an FFMA nor flush subnormals.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define RO_DEV __device__ __forceinline__

namespace ro {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SLOTS = 128;   // R4: 32 lanes x float4
constexpr int TILE = 4096;   // R4: elements per CSUM tile

RO_DEV float canon(float x) { return (x != x) ? __uint_as_float(0x7FC00000u) : x; }

RO_DEV bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// TREE128 on slots held as lane l -> slots 4l..4l+3 (p0..p3).  Levels h = 64..4
// pair slot s with s+h, i.e. lane l with lane l^(h/4); IEEE addition is
// commutative, so both partners compute the identical sum.  h = 2, 1 are
// in-lane.  Every lane returns the full result.
RO_DEV float tree128(float p0, float p1, float p2, float p3) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        p0 = __fadd_rn(p0, __shfl_xor_sync(FULL, p0, off));
        p1 = __fadd_rn(p1, __shfl_xor_sync(FULL, p1, off));
        p2 = __fadd_rn(p2, __shfl_xor_sync(FULL, p2, off));
        p3 = __fadd_rn(p3, __shfl_xor_sync(FULL, p3, off));
    }
    p0 = __fadd_rn(p0, p2);
    p1 = __fadd_rn(p1, p3);
    return __fadd_rn(p0, p1);
}

// Warp CSUM of one tile x[0..n), n <= 4096 (R-CSUM).
RO_DEV float warp_csum_tile(const float *__restrict__ x, int n, int lane) {
    float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
    if (aligned16(x)) {
        int full = n & ~127;
        for (int b = 0; b < full; b += 128) {
            float4 v = __ldg(reinterpret_cast<const float4 *>(x + b) + lane);
            p0 = __fadd_rn(p0, v.x); p1 = __fadd_rn(p1, v.y);
            p2 = __fadd_rn(p2, v.z); p3 = __fadd_rn(p3, v.w);
        }
        int i = full + 4 * lane;
        if (i < n) p0 = __fadd_rn(p0, x[i]);
        if (i + 1 < n) p1 = __fadd_rn(p1, x[i + 1]);
        if (i + 2 < n) p2 = __fadd_rn(p2, x[i + 2]);
        if (i + 3 < n) p3 = __fadd_rn(p3, x[i + 3]);
    } else {
        for (int b = 0; b < n; b += 128) {
            int i = b + 4 * lane;
            if (i < n) p0 = __fadd_rn(p0, x[i]);
            if (i + 1 < n) p1 = __fadd_rn(p1, x[i + 1]);
            if (i + 2 < n) p2 = __fadd_rn(p2, x[i + 2]);
            if (i + 3 < n) p3 = __fadd_rn(p3, x[i + 3]);
        }
    }
    return tree128(p0, p1, p2, p3);
}

// ---------------------------------------------------------------- software math
// R5: Cephes single-precision algorithms as fixed IEEE-RN chains.
RO_DEV float pow2i(int k) { return __uint_as_float((uint32_t)(k + 127) << 23); }

RO_DEV float exp_rn(float x) {
    float t = __fmul_rn(x, 1.44269504088896341f);
    float kf = __fsub_rn(__fadd_rn(t, 12582912.0f), 12582912.0f);
    float r = __fmaf_rn(kf, -0.693359375f, x);
    r = __fmaf_rn(kf, 2.12194440e-4f, r);
    float p = 1.9875691500E-4f;
    p = __fmaf_rn(p, r, 1.3981999507E-3f);
    p = __fmaf_rn(p, r, 8.3334519073E-3f);
    p = __fmaf_rn(p, r, 4.1665795894E-2f);
    p = __fmaf_rn(p, r, 1.6666665459E-1f);
    p = __fmaf_rn(p, r, 5.0000001201E-1f);
    float y = __fadd_rn(__fmaf_rn(p, __fmul_rn(r, r), r), 1.0f);
    int k = __float2int_rz(kf);  // kf is integral: exact
    int k1 = k >> 1;
    int k2 = k - k1;
    // clamp the exponent inputs so out-of-range x (selected away below) stay in range
    k1 = max(min(k1, 127), -126);
    k2 = max(min(k2, 127), -126);
    float res = __fmul_rn(__fmul_rn(y, pow2i(k1)), pow2i(k2));
    res = (x < -104.0f) ? 0.0f : res;
    res = (x > 89.0f) ? __uint_as_float(0x7F800000u) : res;
    res = (x != x) ? __uint_as_float(0x7FC00000u) : res;
    return res;
}

RO_DEV float log_rn(float x) {
    bool sub = x < 1.17549435e-38f;
    float xs = sub ? __fmul_rn(x, 8388608.0f) : x;
    uint32_t u = __float_as_uint(xs);
    int e = (int)((u >> 23) & 0xFFu) - 126 - (sub ? 23 : 0);
    float m = __uint_as_float((u & 0x007FFFFFu) | 0x3F000000u);
    bool lo = m < 0.70710678f;
    e -= lo ? 1 : 0;
    m = lo ? __fadd_rn(m, m) : m;
    float f = __fsub_rn(m, 1.0f);
    float z = __fmul_rn(f, f);
    float p = 7.0376836292E-2f;
    p = __fmaf_rn(p, f, -1.1514610310E-1f);
    p = __fmaf_rn(p, f, 1.1676998740E-1f);
    p = __fmaf_rn(p, f, -1.2420140846E-1f);
    p = __fmaf_rn(p, f, 1.4249322787E-1f);
    p = __fmaf_rn(p, f, -1.6668057665E-1f);
    p = __fmaf_rn(p, f, 2.0000714765E-1f);
    p = __fmaf_rn(p, f, -2.4999993993E-1f);
    p = __fmaf_rn(p, f, 3.3333331174E-1f);
    float ef = (float)e;  // exact
    float y = __fmul_rn(__fmul_rn(p, f), z);
    y = __fmaf_rn(ef, -2.12194440e-4f, y);
    y = __fmaf_rn(z, -0.5f, y);
    y = __fadd_rn(f, y);
    y = __fmaf_rn(ef, 0.693359375f, y);
    y = (x == __uint_as_float(0x7F800000u)) ? x : y;
    y = (x == 0.0f) ? __uint_as_float(0xFF800000u) : y;
    y = (x < 0.0f || x != x) ? __uint_as_float(0x7FC00000u) : y;
    return y;
}

RO_DEV float tanh_rn(float u) {
    float a = fabsf(u);
    float t;
    if (a < 0.625f) {
        float z = __fmul_rn(u, u);
        float p = -5.70498872745E-3f;
        p = __fmaf_rn(p, z, 2.06390887954E-2f);
        p = __fmaf_rn(p, z, -5.37397155531E-2f);
        p = __fmaf_rn(p, z, 1.33314422036E-1f);
        p = __fmaf_rn(p, z, -3.33332819422E-1f);
        t = __fmaf_rn(__fmul_rn(p, z), a, a);
    } else {
        float aa = (a < 44.0f) ? a : 44.0f;
        float e = exp_rn(__fadd_rn(aa, aa));
        t = __fsub_rn(1.0f, __fdiv_rn(2.0f, __fadd_rn(e, 1.0f)));
    }
    t = copysignf(t, u);
    return (u != u) ? __uint_as_float(0x7FC00000u) : t;
}

RO_DEV float rsqrt_rn(float x) { return __fdiv_rn(1.0f, __fsqrt_rn(x)); }

// sin / cos (R26): Cephes sinf/cosf.  Octant from trunc(|x| * 4/pi) rounded up to
// even; three-constant Cody-Waite reduction (|x| > 8192: one pi/4 product); sine
// polynomial fma(r z P(z)... , r, r) or cosine 1 - z/2 + z^2 Q(z) by octant; sign by
// octant (and, for sin, by x).  |x| > 16777215 -> +0; inf / NaN -> canonical NaN.
RO_DEV float sc_reduce_rn(float a, int &oct) {
    const float t = __fmul_rn(a, 1.27323954473516f);
    uint32_t j = __float2uint_rz(t);
    float y = __uint2float_rn(j);
    if (j & 1u) {
        j += 1u;
        y = __fadd_rn(y, 1.0f);
    }
    oct = (int)(j & 7u);
    if (a > 8192.0f) return __fsub_rn(a, __fmul_rn(y, 0.7853981633974483096f));
    float r = __fsub_rn(a, __fmul_rn(y, 0.78515625f));
    r = __fsub_rn(r, __fmul_rn(y, 2.4187564849853515625e-4f));
    return __fsub_rn(r, __fmul_rn(y, 3.77489497744594108e-8f));
}
RO_DEV float sc_sin_poly(float r, float z) {
    float p = __fmaf_rn(-1.9515295891E-4f, z, 8.3321608736E-3f);
    p = __fmaf_rn(p, z, -1.6666654611E-1f);
    return __fmaf_rn(__fmul_rn(p, z), r, r);
}
RO_DEV float sc_cos_poly(float z) {
    float p = __fmaf_rn(2.443315711809948E-5f, z, -1.388731625493765E-3f);
    p = __fmaf_rn(p, z, 4.166664568298827E-2f);
    const float v = __fsub_rn(__fmul_rn(p, __fmul_rn(z, z)), __fmul_rn(0.5f, z));
    return __fadd_rn(v, 1.0f);
}
RO_DEV float sincos_rn(float x, bool want_cos) {
    const float a = fabsf(x);
    if (!(a <= 3.4028235e38f)) return __uint_as_float(0x7FC00000u);  // NaN, +-inf
    if (a > 16777215.0f) return 0.0f;
    int j;
    const float r = sc_reduce_rn(a, j);
    bool neg = want_cos ? false : (x < 0.0f);
    if (j > 3) {
        neg = !neg;
        j -= 4;
    }
    if (want_cos && j > 1) neg = !neg;
    const float z = __fmul_rn(r, r);
    const bool sin_branch = (j == 1 || j == 2) == want_cos;
    const float v = sin_branch ? sc_sin_poly(r, z) : sc_cos_poly(z);
    return neg ? -v : v;
}

// erf (R27): Cephes erff / erfcf.  |x| <= 1: a * T(a^2); 1 < |x| < 10: 1 - (exp(-a^2) / a) * P(1/a^2)
// (P on [1, 2), R on [2, 10)); |x| >= 10: 1; sign applied last.  Horner steps are fmaf.
RO_DEV float erf_rn(float x) {
    const float a = fabsf(x);
    float y;
    if (a <= 1.0f) {
        const float z = __fmul_rn(a, a);
        float p = 7.853861353153693E-5f;
        p = __fmaf_rn(p, z, -8.010193625184903E-4f);
        p = __fmaf_rn(p, z, 5.188327685732524E-3f);
        p = __fmaf_rn(p, z, -2.685381193529856E-2f);
        p = __fmaf_rn(p, z, 1.128358514861418E-1f);
        p = __fmaf_rn(p, z, -3.761262582423300E-1f);
        p = __fmaf_rn(p, z, 1.128379165726710E+0f);
        y = __fmul_rn(a, p);
    } else if (a >= 10.0f) {
        y = 1.0f;
    } else {
        const float e = exp_rn(-__fmul_rn(a, a));
        const float q = __fdiv_rn(1.0f, a);
        const float w = __fmul_rn(q, q);
        float p;
        if (a < 2.0f) {
            p = 2.326819970068386E-2f;
            p = __fmaf_rn(p, w, -1.387039388740657E-1f);
            p = __fmaf_rn(p, w, 3.687424674597105E-1f);
            p = __fmaf_rn(p, w, -5.824733027278666E-1f);
            p = __fmaf_rn(p, w, 6.210004621745983E-1f);
            p = __fmaf_rn(p, w, -4.944515323274145E-1f);
            p = __fmaf_rn(p, w, 3.404879937665872E-1f);
            p = __fmaf_rn(p, w, -2.741127028184656E-1f);
            p = __fmaf_rn(p, w, 5.638259427386472E-1f);
        } else {
            p = -1.047766399936249E+1f;
            p = __fmaf_rn(p, w, 1.297719955372516E+1f);
            p = __fmaf_rn(p, w, -7.495518717768503E+0f);
            p = __fmaf_rn(p, w, 2.921019019210786E+0f);
            p = __fmaf_rn(p, w, -1.015265279202700E+0f);
            p = __fmaf_rn(p, w, 4.218463358204948E-1f);
            p = __fmaf_rn(p, w, -2.820767439740514E-1f);
            p = __fmaf_rn(p, w, 5.641895067754075E-1f);
        }
        y = __fsub_rn(1.0f, __fmul_rn(__fmul_rn(e, q), p));
    }
    y = (x < 0.0f) ? -y : y;
    return (x != x) ? __uint_as_float(0x7FC00000u) : y;
}

// exact GELU (R27): y = (0.5 x)(1 + erf(x * 1/sqrt 2)); backward dx = dy (cdf + x pdf),
// cdf = 0.5 (1 + erf(x / sqrt 2)), pdf = exp(-(0.5 x^2)) * 1/sqrt(2 pi)
RO_DEV float gelu_erf_rn(float v) {
    return __fmul_rn(__fmul_rn(0.5f, v), __fadd_rn(1.0f, erf_rn(__fmul_rn(v, 0.70710678118654752f))));
}
RO_DEV float gelu_erf_grad_rn(float v, float dy) {
    const float cdf = __fmul_rn(0.5f, __fadd_rn(1.0f, erf_rn(__fmul_rn(v, 0.70710678118654752f))));
    const float pdf = __fmul_rn(exp_rn(-__fmul_rn(0.5f, __fmul_rn(v, v))), 0.39894228040143268f);
    return __fmul_rn(dy, __fadd_rn(cdf, __fmul_rn(v, pdf)));
}

// GELU (tanh form, R13): u = c*(x + 0.044715 x^3), y = 0.5x(1 + tanh u)
RO_DEV float gelu_rn(float v) {
    float x2 = __fmul_rn(v, v);
    float x3 = __fmul_rn(x2, v);
    float inner = __fmaf_rn(0.044715f, x3, v);
    float u = __fmul_rn(0.7978845608028654f, inner);
    float t = tanh_rn(u);
    return __fmul_rn(__fmul_rn(0.5f, v), __fadd_rn(1.0f, t));
}

RO_DEV float gelu_grad_rn(float v, float dy) {
    float x2 = __fmul_rn(v, v);
    float x3 = __fmul_rn(x2, v);
    float inner = __fmaf_rn(0.044715f, x3, v);
    float u = __fmul_rn(0.7978845608028654f, inner);
    float t = tanh_rn(u);
    float di = __fmaf_rn(0.134145f, x2, 1.0f);
    float s2 = __fsub_rn(1.0f, __fmul_rn(t, t));
    float g = __fadd_rn(__fmul_rn(0.5f, __fadd_rn(1.0f, t)),
                        __fmul_rn(__fmul_rn(__fmul_rn(0.5f, v), s2), __fmul_rn(0.7978845608028654f, di)));
    return __fmul_rn(dy, g);
}

}  // namespace ro

// ---------------------------------------------------------------- launch helpers (host)
namespace ro_host {
int grid_for(int64_t n, int threads, int per_thread = 1);
int num_sms();
}
