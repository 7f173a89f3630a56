// rfg_expf.cuh — the C library's expf on the device (used by the bilateral
// filter, rfg_view.cu).
#pragma once

#include <cstdint>

namespace rfg {

// ------------------------------------------------ expf, as the reference
// bilateral_filter calls std::exp(float): glibc's expf (x86-64, FMA ifunc
// variant, glibc >= 2.27; the algorithm of ARM optimized-routines with
// N = 32): k = round(x 32/ln2) by the 1.5*2^52 shift trick, r = x 32/ln2 - k,
// 2^(k/32) from a table, degree-3 polynomial, all in double with the same
// fused operations, then rounded to float.  The constants are mathematical:
// T[i] = bits(2^(i/32)) - (i << 52)/32, C = {c3, c2, c1} / 32^{3,2,1} with
// the published coefficients.  Special cases as glibc: x > 88.72 -> inf,
// x < -103.97 -> 0, [-103.97, -103.28) -> 2^-149, -inf -> 0, NaN -> NaN.
// tests/cuda/expf_glibc.cu compares it with the host libm's expf.
__constant__ unsigned long long kExpT[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

__device__ __forceinline__ float expf_glibc(float x) {
  const uint32_t bits = __float_as_uint(x);
  const uint32_t abstop = (bits >> 20) & 0x7ffu;
  if (abstop > 0x42au) {  // |x| >= 88, inf, nan
    if (bits == 0xff800000u) return 0.f;
    // x + x: +inf, or the input NaN quietened with its payload (x86 SSE
    // semantics; the GPU's own NaN arithmetic returns a canonical NaN)
    if (abstop > 0x7f7u) return (bits & 0x7fffffu) ? __uint_as_float(bits | 0x400000u) : x + x;
    if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
    if (x < -0x1.9fe368p6f) return 0.f;
    if (x < -0x1.9d1d9ep6f) return 0x1p-149f;
  }
  const double kInvLn2N = 0x1.71547652b82fep+5, kShift = 0x1.8p+52;
  const double xd = (double)x;
  const double kd0 = __fma_rn(kInvLn2N, xd, kShift);
  const unsigned long long ki = (unsigned long long)__double_as_longlong(kd0);
  const double kd = kd0 - kShift;
  const double r = __fma_rn(kInvLn2N, xd, -kd);
  const double s = __longlong_as_double((long long)(kExpT[ki & 31u] + (ki << 47)));
  const double z = __fma_rn(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
  const double r2 = r * r;
  const double y0 = __fma_rn(0x1.62e42ff0c52d6p-6, r, 1.0);
  const double y = __fma_rn(z, r2, y0) * s;
  return __double2float_rn(y);
}

}  // namespace rfg
