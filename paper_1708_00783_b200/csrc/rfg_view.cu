// rfg_view.cu — build_view depth path (proj/src/view.cpp:100-143):
// raw u16 -> metres (DepthAffine::toMetres, camera.hpp:54; raw == 0 or
// m <= 0 -> invalid -1) and the 2x2 valid-mean pyramid (downsample_depth,
// view.cpp:69-88).  Pure streaming kernels: 2 B in / 4 B out per pixel, then
// 16 B in / 4 B out per coarser pixel.
#include "rfg_common.cuh"

namespace rfg {

__global__ void k_depth_convert(const uint16_t* __restrict__ raw, float* __restrict__ out, int n, float scale,
                                float offset) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i + 1 < n) {
    const ushort2 r = *reinterpret_cast<const ushort2*>(raw + i);
    float2 o;
    const float m0 = (float)r.x * scale + offset, m1 = (float)r.y * scale + offset;
    o.x = (r.x == 0) ? -1.f : (m0 > 0.f ? m0 : -1.f);
    o.y = (r.y == 0) ? -1.f : (m1 > 0.f ? m1 : -1.f);
    *reinterpret_cast<float2*>(out + i) = o;
  } else if (i < n) {
    const uint16_t r = raw[i];
    const float m = (float)r * scale + offset;
    out[i] = (r == 0) ? -1.f : (m > 0.f ? m : -1.f);
  }
}

__global__ void k_downsample(const float* __restrict__ in, int iw, float* __restrict__ out, int ow, int oh) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= ow || y >= oh) return;
  const float* r0 = in + (size_t)(2 * y) * iw + 2 * x;
  const float* r1 = r0 + iw;
  float sum = 0.f;
  int n = 0;
  const float d[4] = {r0[0], r0[1], r1[0], r1[1]};  // dy-major, dx-minor (view.cpp:78-84)
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (d[k] > 0.f) {
      sum += d[k];
      ++n;
    }
  out[(size_t)y * ow + x] = n > 0 ? sum / (float)n : -1.f;
}

cudaError_t launch_build_view(const uint16_t* raw, int w, int h, float scale, float offset, int levels, float* out,
                              cudaStream_t s) {
  const int n = w * h;
  k_depth_convert<<<(n / 2 + 255) / 256 + 1, 256, 0, s>>>(raw, out, n, scale, offset);
  count_launch();
  const float* prev = out;
  float* cur = out + (size_t)n;
  int pw = w, ph = h;
  for (int l = 1; l < levels; ++l) {
    const int ow = pw / 2, oh = ph / 2;
    k_downsample<<<dim3((ow + 127) / 128, oh), 128, 0, s>>>(prev, pw, cur, ow, oh);
    count_launch();
    prev = cur;
    cur += (size_t)ow * oh;
    pw = ow;
    ph = oh;
  }
  return cudaGetLastError();
}

}  // namespace rfg
