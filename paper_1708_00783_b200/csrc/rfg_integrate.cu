// rfg_integrate.cu — TSDF (+colour) integration over the visible blocks
// (FusionEngine::integrate_frame, proj/src/fusion.cpp:237-263, voxel updates
// :9-70).
//
// One warp per visible 8^3 block: the block's 512 depth voxels (4 B each,
// 2 KiB) are moved as 4 coalesced 128-bit loads and stores per lane, so each
// warp-wide access covers 512 contiguous bytes.  The grid is persistent
// (a multiple of the SM count) and strides over the device-resident visible
// list, so no host round-trip is needed for its length.  HBM bytes per block:
// 2 x 2 KiB (depth plane) [+ 2 x 2 KiB colour plane].
#include "rfg_common.cuh"

namespace rfg {

struct ColourArgs {
  const uint8_t* rgb;  // packed RGB8, nullptr = depth-only
  int rw, rh;
  float fx, fy, cx, cy;
  float extr[12];      // extrinsics_d_to_rgb
};

__device__ __forceinline__ Pose load_pose_i(const FrameArgs& fa) {
  return pose_from12(fa.poseDev ? fa.poseDev : fa.pose);
}

// update_voxel_depth (fusion.cpp:9-36); returns eta, updates the word.
__device__ __forceinline__ float update_depth(uint32_t& word, f3 pt, const Pose& M, const FrameArgs& fa,
                                              const float* __restrict__ depth) {
  const f3 pc = pose_apply(M, pt);
  if (pc.z <= 0.f) return -1.f;
  const float px = fa.fx * pc.x / pc.z + fa.cx;
  const float py = fa.fy * pc.y / pc.z + fa.cy;
  if (px < 1 || px > (float)(fa.w - 2) || py < 1 || py > (float)(fa.h - 2)) return -1.f;
  const float dm = __ldg(depth + (size_t)(int)(py + 0.5f) * fa.w + (int)(px + 0.5f));
  if (dm <= 0.f) return -1.f;
  const float eta = dm - pc.z;
  if (eta < -fa.mu) return eta;
  const float oldF = sdf_to_logical(vox_sdf(word));
  const int oldW = vox_w(word);
  if (fa.stopAtMaxW && oldW >= fa.maxW) return eta;
  const float newF = smin(1.f, eta / fa.mu);
  const int newW = 1;
  const float merged = ((float)oldW * oldF + (float)newW * newF) / (float)(oldW + newW);
  const int w = min(oldW + newW, fa.maxW);
  word = vox_pack(sdf_from_logical(merged), w);
  return eta;
}

// update_voxel_colour (fusion.cpp:38-70)
__device__ __forceinline__ void update_colour(uint32_t& word, f3 pt, const Pose& M, const ColourArgs& ca, int maxW) {
  const f3 pc = pose_apply(M, pt);
  if (pc.z <= 0.f) return;
  const float px = ca.fx * pc.x / pc.z + ca.cx;
  const float py = ca.fy * pc.y / pc.z + ca.cy;
  if (px < 1 || px > (float)(ca.rw - 2) || py < 1 || py > (float)(ca.rh - 2)) return;
  const int x0 = (int)floorf(px), y0 = (int)floorf(py);
  const float fx = px - (float)x0, fy = py - (float)y0;
  const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
  const uint8_t* c00 = ca.rgb + 3 * ((size_t)y0 * ca.rw + x0);
  const uint8_t* c01 = c00 + 3 * (size_t)ca.rw;
  const int oldW = (int)(word >> 24);
  uint32_t out = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float sample = w00 * (float)__ldg(c00 + k) + w10 * (float)__ldg(c00 + 3 + k) +
                         w01 * (float)__ldg(c01 + k) + w11 * (float)__ldg(c01 + 3 + k);
    const float old = (float)((word >> (8 * k)) & 0xFFu);
    const float merged = ((float)oldW * old + sample) / (float)(oldW + 1);
    long r = lroundf(merged);
    r = r < 0 ? 0 : (r > 255 ? 255 : r);
    out |= (uint32_t)r << (8 * k);
  }
  out |= (uint32_t)min(oldW + 1, maxW) << 24;
  word = out;
}

template <bool kColour>
__global__ void __launch_bounds__(256) k_integrate(DevMap m, const float* __restrict__ depth, FrameArgs fa,
                                                   ColourArgs ca) {
  const int lane = threadIdx.x & 31;
  const int warpsPerCta = blockDim.x >> 5;
  const int gw = blockIdx.x * warpsPerCta + (threadIdx.x >> 5);
  const int nw = gridDim.x * warpsPerCta;
  const int nVis = *((volatile int*)&m.state->nVisible);
  const Pose pose = load_pose_i(fa);
  Pose Mrgb;
  if (kColour) Mrgb = pose_compose(pose_from12(ca.extr), pose);
  for (int b = gw; b < nVis; b += nw) {
    const int idx = m.visibleList[b];
    const int4 e = ld_entry(m.entries, idx);
    if (e.w < 0) continue;
    const int ox = entry_x(e) * kBlock, oy = entry_y(e) * kBlock, oz = entry_z(e) * kBlock;
    uint4* blk = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)e.w * kBlock3);
    uint4* cblk = kColour ? reinterpret_cast<uint4*>(m.vbaColour + (size_t)e.w * kBlock3) : nullptr;
    uint4 v[4], c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = blk[q * 32 + lane];
    if (kColour) {
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] = cblk[q * 32 + lane];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int lin = (q * 32 + lane) * 4;
      const int z = lin >> 6, y = (lin >> 3) & 7, x0 = lin & 7;
      uint32_t w[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
      uint32_t cw[4];
      if (kColour) {
        cw[0] = c[q].x;
        cw[1] = c[q].y;
        cw[2] = c[q].z;
        cw[3] = c[q].w;
      }
      const float pz = (float)(oz + z) * fa.voxelSize;
      const float py = (float)(oy + y) * fa.voxelSize;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const f3 pt{(float)(ox + x0 + i) * fa.voxelSize, py, pz};
        const float eta = update_depth(w[i], pt, pose, fa, depth);
        if (kColour && eta >= -fa.mu) update_colour(cw[i], pt, Mrgb, ca, fa.maxW);
      }
      v[q] = make_uint4(w[0], w[1], w[2], w[3]);
      if (kColour) c[q] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) blk[q * 32 + lane] = v[q];
    if (kColour) {
#pragma unroll
      for (int q = 0; q < 4; ++q) cblk[q * 32 + lane] = c[q];
    }
  }
}

int integrate_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms * 8;  // 8 CTAs x 8 warps per SM
  }
  return grid;
}

cudaError_t launch_integrate(const DevMap& m, const float* depth, const uint8_t* rgb, const FrameArgs& fa,
                             const rfg_intrinsics* intrRgb, const float* extr34, cudaStream_t s) {
  ColourArgs ca{};
  ca.rgb = rgb;
  if (rgb) {
    ca.rw = intrRgb->width;
    ca.rh = intrRgb->height;
    ca.fx = intrRgb->fx;
    ca.fy = intrRgb->fy;
    ca.cx = intrRgb->cx;
    ca.cy = intrRgb->cy;
    for (int i = 0; i < 12; ++i) ca.extr[i] = extr34 ? extr34[i] : ((i % 5 == 0) ? 1.f : 0.f);
    k_integrate<true><<<integrate_grid(), 256, 0, s>>>(m, depth, fa, ca);
  } else {
    k_integrate<false><<<integrate_grid(), 256, 0, s>>>(m, depth, fa, ca);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace rfg
