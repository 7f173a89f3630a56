// Exhaustive check of the ALU-pipe conversions of rfg_common.cuh against the
// hardware conversions: u23_to_float (every v < 2^23), s16_to_float (every
// int16), trunc_pos_to_int (every float in [0, 2^23)) and lround_haz_alu /
// lround_haz_f2i (every float with |v| < 2^22, against lround_haz / lroundf).
#include <cstdio>
#include "../../paper_1708_00783_b200/csrc/rfg_common.cuh"

__global__ void k_int(unsigned long long* bad) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < (1u << 23); v += gridDim.x * blockDim.x) {
    if (__float_as_uint(rfg::u23_to_float(v)) != __float_as_uint((float)v)) atomicAdd(&bad[0], 1ull);
    if (v < 65536u) {
      const int16_t s = (int16_t)(uint16_t)v;
      if (__float_as_uint(rfg::s16_to_float(s)) != __float_as_uint((float)s)) atomicAdd(&bad[1], 1ull);
    }
  }
}

// every float bit pattern with |v| < 2^23 (exponent field < 150)
__global__ void k_float(unsigned long long* bad) {
  const uint32_t lim = 150u << 23;  // bits of 2^23
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < lim; b += gridDim.x * blockDim.x) {
    const float t = __uint_as_float(b);
    if (rfg::trunc_pos_to_int(t) != (int)t) atomicAdd(&bad[2], 1ull);
    if (b < (149u << 23)) {  // |v| < 2^22
      for (int sgn = 0; sgn < 2; ++sgn) {
        const float v = sgn ? -t : t;
        const int ref = (int)lroundf(v);
        if (rfg::lround_haz_alu(v) != ref || rfg::lround_haz(v) != ref || rfg::lround_haz_f2i(v) != ref)
          atomicAdd(&bad[3], 1ull);
      }
    }
  }
}

int main() {
  unsigned long long* bad;
  cudaMallocManaged(&bad, 4 * sizeof(unsigned long long));
  for (int i = 0; i < 4; ++i) bad[i] = 0;
  k_int<<<1024, 256>>>(bad);
  k_float<<<4096, 256>>>(bad);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("u23 %llu s16 %llu trunc %llu lround %llu (%s)\n", bad[0], bad[1], bad[2], bad[3],
              cudaGetErrorString(e));
  const bool ok = e == cudaSuccess && !bad[0] && !bad[1] && !bad[2] && !bad[3];
  std::printf("%s\n", ok ? "magic conversions: mismatches 0" : "MISMATCH");
  return ok ? 0 : 1;
}
