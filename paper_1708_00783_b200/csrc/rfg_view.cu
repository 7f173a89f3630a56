// rfg_view.cu — the ViewBuilder (proj/src/view.cpp:8-143):
//   raw u16 -> metres (DepthAffine::toMetres, camera.hpp:54; raw == 0 or
//   m <= 0 -> invalid -1), optionally straight from a PGM16 payload
//   (big-endian, image_io.cpp:96-113: the byte swap is fused here);
//   5x5 bilateral filter (view.cpp:18-44); central-difference normals
//   (:46-67); RGB -> intensity (:8-16); depth and intensity pyramids
//   (:69-98).  Streaming kernels over the frame; bytes per pixel are listed
//   at each kernel.
#include "rfg_common.cuh"
#include "rfg_expf.cuh"

namespace rfg {

// 2 B in / 4 B out per pixel
__global__ void k_depth_convert(const uint16_t* __restrict__ raw, float* __restrict__ out, int n, float scale,
                                float offset, int bigEndian) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i + 1 < n) {
    ushort2 r = *reinterpret_cast<const ushort2*>(raw + i);
    if (bigEndian) {
      r.x = (uint16_t)((r.x >> 8) | (r.x << 8));
      r.y = (uint16_t)((r.y >> 8) | (r.y << 8));
    }
    float2 o;
    const float m0 = (float)r.x * scale + offset, m1 = (float)r.y * scale + offset;
    o.x = (r.x == 0) ? -1.f : (m0 > 0.f ? m0 : -1.f);
    o.y = (r.y == 0) ? -1.f : (m1 > 0.f ? m1 : -1.f);
    *reinterpret_cast<float2*>(out + i) = o;
  } else if (i < n) {
    uint16_t r = raw[i];
    if (bigEndian) r = (uint16_t)((r >> 8) | (r << 8));
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

// The depth-only view (no bilateral filter, normals or intensity) in one
// launch: a CTA converts a 32x16 tile of raw depth (toMetres, camera.hpp:54)
// and reduces it to the 16x8 and 8x4 tiles of pyramid levels 1 and 2 in
// shared memory (downsample_depth, view.cpp:69-88: 2x2 mean of the valid
// samples in dy-major order).  Tile origins are multiples of 4 at level 0,
// so every coarse pixel's 2x2 source lies inside the tile; per-pixel
// arithmetic is k_depth_convert's and k_downsample's.
__device__ __forceinline__ float raw_to_metres(uint16_t r, float scale, float offset, int bigEndian) {
  if (bigEndian) r = (uint16_t)((r >> 8) | (r << 8));
  const float m = (float)r * scale + offset;
  return (r == 0) ? -1.f : (m > 0.f ? m : -1.f);
}
__device__ __forceinline__ float mean_valid4(float a, float b, float c, float d) {
  const float v[4] = {a, b, c, d};
  float sum = 0.f;
  int n = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (v[k] > 0.f) {
      sum += v[k];
      ++n;
    }
  return n > 0 ? sum / (float)n : -1.f;
}

__global__ void __launch_bounds__(256) k_view_pyramid(const uint16_t* __restrict__ raw, int w, int h, float scale,
                                                     float offset, int bigEndian, int levels, float* __restrict__ out) {
  __shared__ float l0[16][32];
  __shared__ float l1[8][16];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int X0 = blockIdx.x * 32, Y0 = blockIdx.y * 16;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int x = X0 + tx, y = Y0 + ty + 8 * r;
    float m = -1.f;
    if (x < w && y < h) {
      m = raw_to_metres(__ldg(raw + (size_t)y * w + x), scale, offset, bigEndian);
      out[(size_t)y * w + x] = m;
    }
    l0[ty + 8 * r][tx] = m;
  }
  if (levels < 2) return;
  __syncthreads();
  const int w1 = w / 2, h1 = h / 2;
  float* out1 = out + (size_t)w * h;
  if (threadIdx.x < 128) {
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int x = X0 / 2 + lx, y = Y0 / 2 + ly;
    const float v = mean_valid4(l0[2 * ly][2 * lx], l0[2 * ly][2 * lx + 1], l0[2 * ly + 1][2 * lx],
                                l0[2 * ly + 1][2 * lx + 1]);
    l1[ly][lx] = v;
    if (x < w1 && y < h1) out1[(size_t)y * w1 + x] = v;
  }
  if (levels < 3) return;
  __syncthreads();
  const int w2 = w1 / 2, h2 = h1 / 2;
  float* out2 = out1 + (size_t)w1 * h1;
  if (threadIdx.x < 32) {
    const int lx = threadIdx.x & 7, ly = threadIdx.x >> 3;
    const int x = X0 / 4 + lx, y = Y0 / 4 + ly;
    if (x < w2 && y < h2)
      out2[(size_t)y * w2 + x] = mean_valid4(l1[2 * ly][2 * lx], l1[2 * ly][2 * lx + 1], l1[2 * ly + 1][2 * lx],
                                            l1[2 * ly + 1][2 * lx + 1]);
  }
  pdl_trigger();  // the tracker (programmatic dependent) may launch
}

// bilateral_filter (view.cpp:18-44): 32x8 pixels per CTA, the 36x12 input
// tile (2-pixel halo) staged in shared memory; the 25 neighbours in the
// reference's dy-major order.  4 B in (+ halo) / 4 B out per pixel.
constexpr int kBilW = 32, kBilH = 8, kBilR = 2;
__global__ void __launch_bounds__(kBilW* kBilH) k_bilateral(const float* __restrict__ in, int w, int h, float invS2,
                                                           float invR2, float* __restrict__ out) {
  __shared__ float tile[kBilH + 2 * kBilR][kBilW + 2 * kBilR];
  const int x0 = blockIdx.x * kBilW - kBilR, y0 = blockIdx.y * kBilH - kBilR;
  for (int t = threadIdx.x; t < (kBilW + 2 * kBilR) * (kBilH + 2 * kBilR); t += blockDim.x) {
    const int tx = t % (kBilW + 2 * kBilR), ty = t / (kBilW + 2 * kBilR);
    const int gx = x0 + tx, gy = y0 + ty;
    // outside the image: a sentinel the window loop treats as "not contained"
    tile[ty][tx] = (gx >= 0 && gy >= 0 && gx < w && gy < h) ? __ldg(in + (size_t)gy * w + gx) : __int_as_float(0x7fc00001);
  }
  __syncthreads();
  const int lx = threadIdx.x % kBilW, ly = threadIdx.x / kBilW;
  const int x = blockIdx.x * kBilW + lx, y = blockIdx.y * kBilH + ly;
  if (x >= w || y >= h) return;
  const float centre = tile[ly + kBilR][lx + kBilR];
  float res = -1.f;
  if (centre > 0.f) {
    float sum = 0.f, wsum = 0.f;
#pragma unroll
    for (int dy = -kBilR; dy <= kBilR; ++dy)
#pragma unroll
      for (int dx = -kBilR; dx <= kBilR; ++dx) {
        const int nx = x + dx, ny = y + dy;
        if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
        const float d = tile[ly + kBilR + dy][lx + kBilR + dx];
        if (d <= 0.f) continue;
        const float dr = d - centre;
        const float wt = expf_glibc((float)(-(dx * dx + dy * dy)) * invS2 - dr * dr * invR2);
        sum += wt * d;
        wsum += wt;
      }
    res = sum / wsum;
  }
  out[(size_t)y * w + x] = res;
}

// compute_normals (view.cpp:46-67); 20 B in / 16 B out per pixel.
__device__ __forceinline__ f3 bp(const Intr& in, float u, float v, float z) {
  return f3{(u - in.cx) / in.fx * z, (v - in.cy) / in.fy * z, z};
}
__global__ void k_view_normals(const float* __restrict__ d, Intr in, float4* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= in.w || y >= in.h) return;
  float4 res = make_float4(0.f, 0.f, 0.f, -1.f);
  if (x >= 1 && y >= 1 && x + 1 < in.w && y + 1 < in.h) {
    const size_t i = (size_t)y * in.w + x;
    const float dc = __ldg(d + i), dxm = __ldg(d + i - 1), dxp = __ldg(d + i + 1);
    const float dym = __ldg(d + i - in.w), dyp = __ldg(d + i + in.w);
    if (!(dc <= 0.f || dxm <= 0.f || dxp <= 0.f || dym <= 0.f || dyp <= 0.f)) {
      const f3 a = bp(in, (float)x + 1.f, (float)y, dxp), b = bp(in, (float)x - 1.f, (float)y, dxm);
      const f3 px{a.x - b.x, a.y - b.y, a.z - b.z};
      const f3 c = bp(in, (float)x, (float)y + 1.f, dyp), e = bp(in, (float)x, (float)y - 1.f, dym);
      const f3 py{c.x - e.x, c.y - e.y, c.z - e.z};
      f3 n = cross3(px, py);
      const float len = sqrtf(sqnorm3(n));
      if (!(len < 1e-12f)) {
        n = f3{n.x / len, n.y / len, n.z / len};
        if (dot3(n, bp(in, (float)x, (float)y, dc)) > 0.f) n = f3{-n.x, -n.y, -n.z};
        res = make_float4(n.x, n.y, n.z, 1.f);
      }
    }
  }
  out[(size_t)y * in.w + x] = res;
}

// rgb_to_intensity (view.cpp:8-16); 3 B in / 4 B out per pixel.
__global__ void k_intensity(const uint8_t* __restrict__ rgb, int n, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* c = rgb + 3 * (size_t)i;
  out[i] = (0.299f * (float)c[0] + 0.587f * (float)c[1] + 0.114f * (float)c[2]) / 255.f;
}

// downsample_intensity (view.cpp:90-98): plain 2x2 box; 16 B in / 4 B out.
__global__ void k_downsample_intensity(const float* __restrict__ in, int iw, float* __restrict__ out, int ow, int oh) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= ow || y >= oh) return;
  const float* r0 = in + (size_t)(2 * y) * iw + 2 * x;
  const float* r1 = r0 + iw;
  out[(size_t)y * ow + x] = 0.25f * (r0[0] + r0[1] + r1[0] + r1[1]);
}

cudaError_t launch_bilateral(const float* in, int w, int h, float spatialSigma, float rangeSigma, float* out,
                             cudaStream_t s) {
  // view.cpp:21-22, in the reference's float arithmetic
  const float invS2 = 1.f / (2.f * spatialSigma * spatialSigma);
  const float invR2 = 1.f / (2.f * rangeSigma * rangeSigma);
  k_bilateral<<<dim3((w + kBilW - 1) / kBilW, (h + kBilH - 1) / kBilH), kBilW * kBilH, 0, s>>>(in, w, h, invS2, invR2,
                                                                                              out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_view_normals(const float* depth, const Intr& in, float4* out, cudaStream_t s) {
  k_view_normals<<<dim3((in.w + 127) / 128, in.h), 128, 0, s>>>(depth, in, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_intensity(const uint8_t* rgb, int w, int h, float* out, cudaStream_t s) {
  const int n = w * h;
  k_intensity<<<(n + 255) / 256, 256, 0, s>>>(rgb, n, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_downsample_intensity(const float* in, int w, int h, float* out, cudaStream_t s) {
  const int ow = w / 2, oh = h / 2;
  if (ow < 1 || oh < 1) return cudaSuccess;
  k_downsample_intensity<<<dim3((ow + 127) / 128, oh), 128, 0, s>>>(in, w, out, ow, oh);
  count_launch();
  return cudaGetLastError();
}

// build_view (view.cpp:100-143) with every option.  scratch (w*h floats) is
// needed when bilateral is set (the filter reads the unfiltered image).
cudaError_t launch_build_view_full(const uint16_t* raw, const uint8_t* rgb, const Intr& in, float scale, float offset,
                                   int bilateral, int levels, int bigEndian, float* depthLevels,
                                   float* intensityLevels, float4* normals, float* scratch, cudaStream_t s) {
  const int w = in.w, h = in.h, n = w * h;
  if (!bilateral && !normals && !(rgb && intensityLevels) && levels <= 3) {
    k_view_pyramid<<<dim3((w + 31) / 32, (h + 15) / 16), 256, 0, s>>>(raw, w, h, scale, offset, bigEndian, levels,
                                                                     depthLevels);
    count_launch();
    return cudaGetLastError();
  }
  float* conv = bilateral ? scratch : depthLevels;
  k_depth_convert<<<(n / 2 + 255) / 256 + 1, 256, 0, s>>>(raw, conv, n, scale, offset, bigEndian);
  count_launch();
  cudaError_t e = cudaSuccess;
  if (bilateral) {
    // range sigma tied to the sensor quantisation step (view.cpp:121-123)
    e = launch_bilateral(scratch, w, h, 2.f, 10.f * fabsf(scale), depthLevels, s);
    if (e != cudaSuccess) return e;
  }
  if (normals) {
    e = launch_view_normals(depthLevels, in, normals, s);
    if (e != cudaSuccess) return e;
  }
  const bool inten = rgb && intensityLevels;
  if (inten) {
    e = launch_intensity(rgb, w, h, intensityLevels, s);
    if (e != cudaSuccess) return e;
  }
  const float* prev = depthLevels;
  float* cur = depthLevels + (size_t)n;
  const float* prevI = intensityLevels;
  float* curI = inten ? intensityLevels + (size_t)n : nullptr;
  int pw = w, ph = h;
  for (int l = 1; l < levels; ++l) {
    const int ow = pw / 2, oh = ph / 2;
    k_downsample<<<dim3((ow + 127) / 128, oh), 128, 0, s>>>(prev, pw, cur, ow, oh);
    count_launch();
    if (inten) {
      e = launch_downsample_intensity(prevI, pw, ph, curI, s);
      if (e != cudaSuccess) return e;
      prevI = curI;
      curI += (size_t)ow * oh;
    }
    prev = cur;
    cur += (size_t)ow * oh;
    pw = ow;
    ph = oh;
  }
  return cudaGetLastError();
}

// The fused depth-view kernel and whether a view configuration uses it (the
// frame graph re-points its raw-frame argument instead of copying frames).
const void* view_pyramid_kernel() { return reinterpret_cast<const void*>(&k_view_pyramid); }
bool view_is_fused(int bilateral, bool normals, bool intensity, int levels) {
  return !bilateral && !normals && !intensity && levels <= 3;
}

cudaError_t launch_build_view(const uint16_t* raw, int w, int h, float scale, float offset, int levels, float* out,
                              cudaStream_t s) {
  const Intr in{w, h, 1.f, 1.f, 0.f, 0.f};
  return launch_build_view_full(raw, nullptr, in, scale, offset, 0, levels, 0, out, nullptr, nullptr, nullptr, s);
}

}  // namespace rfg
