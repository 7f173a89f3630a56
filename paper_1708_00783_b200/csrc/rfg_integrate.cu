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
    int r = lround_haz(merged);
    r = r < 0 ? 0 : (r > 255 ? 255 : r);
    out |= (uint32_t)r << (8 * k);
  }
  out |= (uint32_t)min(oldW + 1, maxW) << 24;
  word = out;
}

// The depth update of one voxel (update_voxel_depth, fusion.cpp:9-36) is
// split into three phases over a lane's 16 voxels so the depth gathers are
// all in flight together:
//   1. project: pc = M p, pixel = round(project(pc)) or -1 (z <= 0, outside
//      [1, W-2] x [1, H-2]);
//   2. gather:  16 predicated depth loads;
//   3. update:  eta = d - pc.z; unless invalid / eta < -mu / weight-capped,
//      F = (w F + min(1, eta/mu)) / (w + 1), w = min(w + 1, maxW), quantise.
// Every division is the IEEE quotient (div_fast inside div_ok's window, `/`
// outside it), every rounding is the reference's, so the result is
// bit-identical to the per-voxel function.
#ifndef RFG_INT_MINB
#define RFG_INT_MINB 4
#endif
#ifndef RFG_INT_QG
#define RFG_INT_QG 2
#endif
constexpr int kQG = RFG_INT_QG;  // rows (of 4 voxels) per project/gather/update group
template <bool kColour>
__global__ void __launch_bounds__(256, RFG_INT_MINB) k_integrate(DevMap m, const float* __restrict__ depth, FrameArgs fa,
                                                   ColourArgs ca) {
  const int lane = threadIdx.x & 31;
  const int warpsPerCta = blockDim.x >> 5;
  const int gw = blockIdx.x * warpsPerCta + (threadIdx.x >> 5);
  const int nw = gridDim.x * warpsPerCta;
  const int nVis = *((volatile int*)&m.state->nVisible);
  const Pose pose = load_pose_i(fa);
  Pose Mrgb;
  if (kColour) Mrgb = pose_compose(pose_from12(ca.extr), pose);
  const float wLim = (float)(fa.w - 2), hLim = (float)(fa.h - 2);
  const float mu = fa.mu;
  const bool muOk = div_ok(mu);
  const float rMu = div_rcp(mu);
  const bool capW = fa.stopAtMaxW != 0;
  for (int b = gw; b < nVis; b += nw) {
    const int idx = m.visibleList[b];
    const int4 e = ld_entry(m.entries, idx);
    if (e.w < 0) continue;
    const int ox = entry_x(e) * kBlock, oy = entry_y(e) * kBlock, oz = entry_z(e) * kBlock;
    uint4* blk = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)e.w * kBlock3);
    uint4* cblk = kColour ? reinterpret_cast<uint4*>(m.vbaColour + (size_t)e.w * kBlock3) : nullptr;
    uint4 v[4], c[4];
#pragma unroll
    for (int g = 0; g < 4; g += kQG) {
    // the group's rows: one coalesced 128-bit load per lane and row (a
    // warp-wide row access is 512 contiguous bytes of the block)
#pragma unroll
    for (int q = g; q < g + kQG; ++q) {
      v[q] = blk[q * 32 + lane];
      if (kColour) c[q] = cblk[q * 32 + lane];
    }
    // ---- phase 1: project the group's voxels (kQG rows of 4 along x)
    float zc[4 * kQG];
    int pix[4 * kQG];
#pragma unroll
    for (int q = g; q < g + kQG; ++q) {
      const int lin = (q * 32 + lane) * 4;
      const int z = lin >> 6, y = (lin >> 3) & 7, x0 = lin & 7;
      const float pz = (float)(oz + z) * fa.voxelSize;
      const float py = (float)(oy + y) * fa.voxelSize;
      // pose_apply's (R1 y + R2 z) terms are shared by the row
      const float r0 = pose.R[1] * py + pose.R[2] * pz;
      const float r1 = pose.R[4] * py + pose.R[5] * pz;
      const float r2 = pose.R[7] * py + pose.R[8] * pz;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = (q - g) * 4 + i;
        const float px = (float)(ox + x0 + i) * fa.voxelSize;
        const float cxw = (pose.R[0] * px + r0) + pose.t[0];
        const float cyw = (pose.R[3] * px + r1) + pose.t[1];
        const float czw = (pose.R[6] * px + r2) + pose.t[2];
        int p = -1;
        if (czw > 0.f) {
          const float ax = fa.fx * cxw, ay = fa.fy * cyw;
          float qx, qy;
          if (div_ok(czw) && div_ok(ax) && div_ok(ay)) {
            const float rz = div_rcp(czw);
            qx = div_fast(ax, czw, rz);
            qy = div_fast(ay, czw, rz);
          } else {
            qx = div_ieee(ax, czw);
            qy = div_ieee(ay, czw);
          }
          const float u = qx + fa.cx, vv = qy + fa.cy;
          if (!(u < 1 || u > wLim || vv < 1 || vv > hLim)) p = (int)(vv + 0.5f) * fa.w + (int)(u + 0.5f);
        }
        pix[k] = p;
        zc[k] = czw;
      }
    }
    // ---- phase 2: gather (all loads issued before any is consumed)
    float dm[4 * kQG];
#pragma unroll
    for (int k = 0; k < 4 * kQG; ++k) dm[k] = pix[k] >= 0 ? __ldg(depth + pix[k]) : -1.f;
    // ---- phase 3: update
#pragma unroll
    for (int q = g; q < g + kQG; ++q) {
      uint32_t w[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
      uint32_t cw[4];
      if (kColour) {
        cw[0] = c[q].x;
        cw[1] = c[q].y;
        cw[2] = c[q].z;
        cw[3] = c[q].w;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = (q - g) * 4 + i;
        float eta = -1.f;  // update_voxel_depth's "invalid" return
        if (pix[k] >= 0 && !(dm[k] <= 0.f)) {
          eta = dm[k] - zc[k];
          const int oldW = vox_w(w[i]);
          if (!(eta < -mu) && !(capW && oldW >= fa.maxW)) {
            const float oldF = sdf_to_logical(vox_sdf(w[i]));
            float newF = (muOk && div_ok(eta)) ? div_fast(eta, mu, rMu) : div_ieee(eta, mu);
            newF = smin(1.f, newF);
            const float num = (float)oldW * oldF + newF;
            const float den = (float)(oldW + 1);
            const float merged = div_ok(num) ? div_fast(num, den, div_rcp(den)) : div_ieee(num, den);
            w[i] = vox_pack(sdf_from_logical(merged), min(oldW + 1, fa.maxW));
          }
        }
        if (kColour && eta >= -mu) {
          const int lin = (q * 32 + lane) * 4;
          const f3 pt{(float)(ox + (lin & 7) + i) * fa.voxelSize, (float)(oy + ((lin >> 3) & 7)) * fa.voxelSize,
                      (float)(oz + (lin >> 6)) * fa.voxelSize};
          update_colour(cw[i], pt, Mrgb, ca, fa.maxW);
        }
      }
      blk[q * 32 + lane] = make_uint4(w[0], w[1], w[2], w[3]);
      if (kColour) cblk[q * 32 + lane] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
    }
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
