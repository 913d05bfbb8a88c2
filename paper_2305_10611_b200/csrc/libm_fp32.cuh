// libm_fp32.cuh — bit-exact device restatements of the two libm calls on the hot path.
//
// The reference evaluates sigmoid as 1/(1+std::exp(-x)) and tanh as std::tanh(x) on floats
// (proj/src/backend.cpp:94-101, proj/src/exec_batched.cpp:10-19), i.e. glibc 2.39's expf and
// tanhf.  To make the FP32 path bit-identical to the reference (not merely within tolerance),
// these are restatements of those published algorithms:
//   * expf: the exp2f-table method (32-entry 2^(i/32) table, cubic polynomial in double) that
//     glibc ships as sysdeps/ieee754/flt-32/e_expf.c; on x86-64 CPUs with FMA (the reference's
//     hosts) glibc dispatches to the FMA build, so the three polynomial steps are fused here.
//   * tanhf: the fdlibm algorithm (s_tanhf.c) over fdlibm expm1f (s_expm1f.c), pure float.
// Every float op is an explicit round-to-nearest intrinsic on the device (no contraction), and
// the header also compiles for the host so tests/ can check it against the system libm over all
// 2^32 inputs (tests/test_libm_exact.py).
#pragma once
#ifndef MBX_NVRTC
#include <stdint.h>
#endif

#if defined(__CUDACC__)
#define MBX_HD __host__ __device__ __forceinline__
#else
#define MBX_HD static inline
#endif

namespace mbx_libm {

#if defined(__CUDA_ARCH__)
MBX_HD float fmul(float a, float b) { return __fmul_rn(a, b); }
MBX_HD float fadd(float a, float b) { return __fadd_rn(a, b); }
MBX_HD float fsub(float a, float b) { return __fsub_rn(a, b); }
MBX_HD float fdiv(float a, float b) { return __fdiv_rn(a, b); }
MBX_HD double dmul(double a, double b) { return __dmul_rn(a, b); }
MBX_HD double dadd(double a, double b) { return __dadd_rn(a, b); }
MBX_HD double dsub(double a, double b) { return __dsub_rn(a, b); }
MBX_HD double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
MBX_HD uint32_t f2u(float f) { return __float_as_uint(f); }
MBX_HD float u2f(uint32_t u) { return __uint_as_float(u); }
MBX_HD uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d); }
MBX_HD double u2d(uint64_t u) { return __longlong_as_double((long long)u); }
#else
}  // namespace mbx_libm
#include <math.h>
#include <string.h>
namespace mbx_libm {
// Host build: the TU must be compiled with -ffp-contract=off so these stay unfused.
MBX_HD float fmul(float a, float b) { return a * b; }
MBX_HD float fadd(float a, float b) { return a + b; }
MBX_HD float fsub(float a, float b) { return a - b; }
MBX_HD float fdiv(float a, float b) { return a / b; }
MBX_HD double dmul(double a, double b) { return a * b; }
MBX_HD double dadd(double a, double b) { return a + b; }
MBX_HD double dsub(double a, double b) { return a - b; }
MBX_HD double dfma(double a, double b, double c) { return fma(a, b, c); }
MBX_HD uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
MBX_HD float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
MBX_HD uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
MBX_HD double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
#endif

// 2^(i/32) as doubles, bit patterns minus (i << 52)/32, as in glibc's __exp2f_data.tab.
// (Global memory read through the L1, not __constant__: the 32 lanes of a warp index it
// divergently, which the constant cache serialises.)
#if defined(__CUDACC__)
__device__
#endif
static const uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

#if defined(__CUDA_ARCH__)
MBX_HD uint64_t exp2f_tab(uint32_t i) { return (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(&kExp2fTab[i])); }
#else
MBX_HD uint64_t exp2f_tab(uint32_t i) { return kExp2fTab[i]; }
#endif

// expf: |x| >= 88 / NaN special cases, then x*32/ln2 = k + r, 2^(k/32) from the table times a
// cubic in r.
MBX_HD float expf_exact(float x) {
  const double kInvLn2N = 0x1.71547652b82fep+0 * 32;
  const double kShift = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
  const double C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
  const double C2 = 0x1.62e42ff0c52d6p-1 / 32;
  uint32_t ux = f2u(x);
  uint32_t abstop = (ux >> 20) & 0x7ff;
  if (abstop >= (f2u(88.0f) >> 20)) {
    if (ux == 0xff800000u) return 0.0f;                  // -inf
    if (abstop >= (0x7f800000u >> 20)) return fadd(x, x);  // inf / nan
    if (x > 0x1.62e42ep6f) return u2f(0x7f800000u);        // overflow -> inf
    if (x < -0x1.9fe368p6f) return 0.0f;                   // underflow -> 0
  }
  double xd = (double)x;
  // GCC's FMA build fuses both uses of z = InvLn2N * x into the following add/sub.
  double kd = dfma(kInvLn2N, xd, kShift);
  uint64_t ki = d2u(kd);
  kd = dsub(kd, kShift);
  double r = dfma(kInvLn2N, xd, -kd);
  uint64_t t = exp2f_tab((uint32_t)(ki % 32));
  t += ki << (52 - 5);
  double s = u2d(t);
  double zz = dfma(C0, r, C1);
  double r2 = dmul(r, r);
  double y = dfma(C2, r, 1.0);
  y = dfma(zz, r2, y);
  y = dmul(y, s);
  return (float)y;
}

// fdlibm expm1f.
MBX_HD float expm1f_exact(float x) {
  const float one = 1.0f, huge = 1.0e+30f, tiny = 1.0e-30f;
  const float o_threshold = 8.8721679688e+01f;
  const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f, invln2 = 1.4426950216e+00f;
  const float Q1 = -3.3333335072e-02f, Q2 = 1.5873016091e-03f, Q3 = -7.9365076090e-05f,
              Q4 = 4.0082177293e-06f, Q5 = -2.0109921195e-07f;
  float y, hi, lo, c = 0.0f, t, e, hxs, hfx, r1;
  int32_t k;
  uint32_t hx = f2u(x);
  uint32_t xsb = hx & 0x80000000u;
  y = xsb == 0 ? x : -x;
  hx &= 0x7fffffffu;
  if (hx >= 0x4195b844u) {
    if (hx >= 0x42b17218u) {
      if (hx > 0x7f800000u) return fadd(x, x);
      if (hx == 0x7f800000u) return xsb == 0 ? x : -1.0f;
      if (x > o_threshold) return fmul(huge, huge);
    }
    if (xsb != 0) return fsub(tiny, one);
  }
  if (hx > 0x3eb17218u) {
    if (hx < 0x3F851592u) {
      if (xsb == 0) { hi = fsub(x, ln2_hi); lo = ln2_lo; k = 1; }
      else { hi = fadd(x, ln2_hi); lo = -ln2_lo; k = -1; }
    } else {
      k = (int32_t)fadd(fmul(invln2, x), xsb == 0 ? 0.5f : -0.5f);
      t = (float)k;
      hi = fsub(x, fmul(t, ln2_hi));
      lo = fmul(t, ln2_lo);
    }
    x = fsub(hi, lo);
    c = fsub(fsub(hi, x), lo);
  } else if (hx < 0x33000000u) {
    t = fadd(huge, x);
    return fsub(x, fsub(t, fadd(huge, x)));
  } else {
    k = 0;
  }
  hfx = fmul(0.5f, x);
  hxs = fmul(x, hfx);
  r1 = fadd(one, fmul(hxs, fadd(Q1, fmul(hxs, fadd(Q2, fmul(hxs, fadd(Q3, fmul(hxs, fadd(Q4, fmul(hxs, Q5))))))))));
  t = fsub(3.0f, fmul(r1, hfx));
  e = fmul(hxs, fdiv(fsub(r1, t), fsub(6.0f, fmul(x, t))));
  if (k == 0) return fsub(x, fsub(fmul(x, e), hxs));
  e = fsub(fmul(x, fsub(e, c)), c);
  e = fsub(e, hxs);
  if (k == -1) return fsub(fmul(0.5f, fsub(x, e)), 0.5f);
  if (k == 1) {
    if (x < -0.25f) return fmul(-2.0f, fsub(e, fadd(x, 0.5f)));
    return fadd(one, fmul(2.0f, fsub(x, e)));
  }
  if (k <= -2 || k > 56) {
    y = fsub(one, fsub(e, x));
    if (k == 128) y = fmul(fmul(y, 2.0f), 0x1p127f);
    else y = u2f(f2u(y) + ((uint32_t)k << 23));
    return fsub(y, one);
  }
  if (k < 23) {
    t = u2f(0x3f800000u - (0x1000000u >> k));
    y = fsub(t, fsub(e, x));
    y = u2f(f2u(y) + ((uint32_t)k << 23));
  } else {
    t = u2f((uint32_t)(0x7f - k) << 23);
    y = fsub(x, fadd(e, t));
    y = fadd(y, one);
    y = u2f(f2u(y) + ((uint32_t)k << 23));
  }
  return y;
}

// fdlibm tanhf.
MBX_HD float tanhf_exact(float x) {
  const float one = 1.0f, two = 2.0f, tiny = 1.0e-30f;
  float t, z;
  uint32_t jx = f2u(x);
  uint32_t ix = jx & 0x7fffffffu;
  if (ix >= 0x7f800000u) {
    if ((jx & 0x80000000u) == 0) return fadd(fdiv(one, x), one);
    return fsub(fdiv(one, x), one);
  }
  if (ix < 0x41b00000u) {
    if (ix == 0) return x;
    if (ix < 0x24000000u) return fmul(x, fadd(one, x));
    if (ix >= 0x3f800000u) {
      t = expm1f_exact(fmul(two, u2f(ix)));
      z = fsub(one, fdiv(two, fadd(t, two)));
    } else {
      t = expm1f_exact(fmul(-two, u2f(ix)));
      z = fdiv(-t, fadd(t, two));
    }
  } else {
    z = fsub(one, tiny);
  }
  return (jx & 0x80000000u) == 0 ? z : -z;
}

MBX_HD float sigmoidf_exact(float x) { return fdiv(1.0f, fadd(1.0f, expf_exact(-x))); }
MBX_HD float reluf_exact(float x) { return x > 0.0f ? x : 0.0f; }

}  // namespace mbx_libm

#if defined(__CUDA_ARCH__)
// Activations of the tensor-core tails (the GEMM is already approximate; these are accurate to a
// few ulp): sigmoid via __expf, tanh via __expf with a series near 0 against cancellation.
__device__ __forceinline__ float mbx_fsig(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float mbx_ftanh(float x) {
  const float a = fabsf(x);
  if (a < 0.0625f) {
    const float x2 = x * x;
    return x * (1.0f + x2 * (-0.333333343f + x2 * (0.133333340f + x2 * -0.0539682540f)));
  }
  const float t = __expf(-2.0f * a);
  return copysignf(__fdividef(1.0f - t, 1.0f + t), x);
}
#endif
