// Exactness of the arithmetic shortcuts in rfg_common.cuh against the IEEE
// operations they replace (bit-for-bit):
//   1. div_fast(a, b, div_rcp(b)) == a / b for every dividend a with |a| in
//      [2^-100, 2^40] and a = +0, exhaustively, for the divisors the kernels
//      use with a fixed divisor (mu values and every integer weight divisor
//      1..256) — the window integration relies on (rfg_integrate.cu);
//   2. the same for 2^33 random (a, b) pairs, |a| in [2^-100, 2^40] and
//      |b| in [2^-40, 2^40] (the projection's x/z, y/z);
//   3. lround_haz(v) == lroundf(v) for every float with |v| < 2^31 and NaN.
#include <cstdio>
#include <cstdint>
#include "../../paper_1708_00783_b200/csrc/rfg_common.cuh"

using rfg::div_fast;
using rfg::div_ok;
using rfg::div_rcp;
using rfg::lround_haz;

// all bit patterns of |a| in [2^-100, 2^40], both signs, and +0
__global__ void k_exhaustive(const float* divisors, int nDiv, unsigned long long* bad) {
  const uint32_t lo = __float_as_uint(0x1p-100f);
  const uint32_t hi = __float_as_uint(0x1p40f);
  const uint64_t n = (uint64_t)(hi - lo + 1) * 2;
  unsigned long long local = 0;
  for (int d = 0; d < nDiv; ++d) {
    const float b = divisors[d];
    const float rb = div_rcp(b);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t bits = lo + (uint32_t)(i >> 1) | ((uint32_t)(i & 1) << 31);
      const float a = __uint_as_float(bits);
      if (__float_as_uint(div_fast(a, b, rb)) != __float_as_uint(__fdiv_rn(a, b))) ++local;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 &&
        __float_as_uint(div_fast(0.f, b, rb)) != __float_as_uint(__fdiv_rn(0.f, b)))
      ++local;
  }
  if (local) atomicAdd(bad, local);
}

__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return (uint32_t)x;
}

__device__ __forceinline__ float in_window(uint32_t r, int lo, int span) {
  // exponent uniform over [2^lo, 2^(lo+span)), random mantissa and sign
  const uint32_t e = 127 + lo + (r % span);
  return __uint_as_float((r & 0x80000000u) | (e << 23) | (mix(r) & 0x7FFFFFu));
}

__global__ void k_random(uint64_t n, unsigned long long* bad) {
  unsigned long long local = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float a = in_window(mix(2 * i + 1), -100, 140);
    const float b = in_window(mix(2 * i + 2), -40, 80);
    if (__float_as_uint(div_fast(a, b, div_rcp(b))) != __float_as_uint(__fdiv_rn(a, b))) ++local;
  }
  if (local) atomicAdd(bad, local);
}

__global__ void k_lround(unsigned long long* bad) {
  unsigned long long local = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (1ull << 32);
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = __uint_as_float((uint32_t)i);
    if (!(fabsf(v) < 0x1p31f) && v == v) continue;
    const long ref = v == v ? lroundf(v) : 0;
    if ((long)lround_haz(v) != ref) ++local;
  }
  if (local) atomicAdd(bad, local);
}

int main() {
  unsigned long long* bad;
  cudaMallocManaged(&bad, 3 * sizeof(unsigned long long));
  bad[0] = bad[1] = bad[2] = 0;
  float divs[300];
  int nd = 0;
  for (float mu : {0.02f, 0.01f, 0.03f, 0.005f, 0.1f, 0.0125f}) divs[nd++] = mu;
  for (int w = 1; w <= 256; ++w) divs[nd++] = (float)w;
  float* dd;
  cudaMalloc(&dd, sizeof(divs));
  cudaMemcpy(dd, divs, sizeof(divs), cudaMemcpyHostToDevice);
  k_exhaustive<<<148 * 16, 256>>>(dd, nd, bad + 0);
  k_random<<<148 * 16, 256>>>(1ull << 33, bad + 1);
  k_lround<<<148 * 16, 256>>>(bad + 2);
  const cudaError_t err = cudaDeviceSynchronize();
  std::printf("divisors %d  exhaustive mismatches %llu  random mismatches %llu  lround mismatches %llu  (%s)\n", nd,
              bad[0], bad[1], bad[2], cudaGetErrorString(err));
  return (err != cudaSuccess || bad[0] || bad[1] || bad[2]) ? 1 : 0;
}
