// Exhaustive check: for every int16 s, the FMA-corrected reciprocal product
// used by rfg_common.cuh:sdf_to_logical equals the IEEE quotient s / 32767.f
// (voxel.hpp:16) bit for bit.
#include <cstdio>
#include "../../paper_1708_00783_b200/csrc/rfg_common.cuh"

__global__ void k(int* bad) {
  const int s = (int)(blockIdx.x * blockDim.x + threadIdx.x) - 32768;
  if (s > 32767) return;
  const float ieee = (float)s / 32767.f;
  const float fast = rfg::sdf_to_logical((int16_t)s);
  if (__float_as_uint(ieee) != __float_as_uint(fast)) atomicAdd(bad, 1);
}

int main() {
  int* bad;
  cudaMallocManaged(&bad, sizeof(int));
  *bad = 0;
  k<<<256, 256>>>(bad);
  cudaDeviceSynchronize();
  std::printf("mismatches %d\n", *bad);
  return *bad != 0;
}
