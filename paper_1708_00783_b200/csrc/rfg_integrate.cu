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
__global__ void __launch_bounds__(256, 2) k_integrate(DevMap m, const float* __restrict__ depth, FrameArgs fa,
                                                   ColourArgs ca) {
  const int lane = threadIdx.x & 31;
  const int warpsPerCta = blockDim.x >> 5;
  const int gw = blockIdx.x * warpsPerCta + (threadIdx.x >> 5);
  const int nw = gridDim.x * warpsPerCta;
  const int nVis = *((volatile int*)&m.state->nVisible);
  const Pose pose = frame_pose(fa);
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

// ------------------------------------------------- depth-only, branch-free
// The depth-only kernel (the C1/C2 hot path) computes every voxel's
// projection and update unconditionally and selects the result, so a warp
// issues one instruction stream instead of the union of the per-voxel
// branches.  All divisions take the hoisted fast path; its exactness window
// (tests/cuda/divfast.cu: dividends |a| in [2^-100, 2^40] and 0, divisors in
// [2^-40, 2^40]) covers every quotient of a voxel whose camera z lies in
// [2^-40, 2^40] with |fx X|, |fy Y|, |eta| <= 2^40 and mu in [2^-20, 2^20]:
//   x/z, y/z : dividends below 2^-100 give |quotient| < 2^-60, which leaves
//              u = cx (|cx| >= 2^-30) or u < 1 (invalid) either way;
//   eta/mu   : eta = d - z is 0 or >= 2^-64 in magnitude when z >= 2^-40;
//   merge    : (w F + newF) is 0 or >= 2^-84 (newF >= 2^-84, w F a multiple
//              of 1/32767 for w >= 1), and den = w + 1 is in [1, 256].
// Voxels outside the window (never at sane scales) are flagged and redone
// with IEEE division behind one warp-uniform branch per group.
__device__ __forceinline__ void project_exact(const Pose& pose, const FrameArgs& fa, float wLim, float hLim, float px,
                                              float py, float pz, int* pixOut) {
  const f3 pc = pose_apply(pose, f3{px, py, pz});
  int p = -1;
  if (pc.z > 0.f) {
    const float u = div_ieee(fa.fx * pc.x, pc.z) + fa.cx;
    const float v = div_ieee(fa.fy * pc.y, pc.z) + fa.cy;
    if (!(u < 1 || u > wLim || v < 1 || v > hLim)) p = (int)(v + 0.5f) * fa.w + (int)(u + 0.5f);
  }
  *pixOut = p;
}

__device__ __forceinline__ uint32_t update_exact(uint32_t wd, float eta, float mu, int maxW) {
  const int oldW = vox_w(wd);
  const float oldF = sdf_to_logical(vox_sdf(wd));
  const float newF = smin(1.f, div_ieee(eta, mu));
  const float merged = div_ieee((float)oldW * oldF + newF, (float)(oldW + 1));
  return vox_pack(sdf_from_logical(merged), min(oldW + 1, maxW));
}

// One visible block of the depth-only kernel (one warp, 16 voxels per lane).
// kWindowKnown: the block-level test below has proven that every voxel's
// projection quotients are inside div_fast's exactness window, so only the
// eta quotient keeps a per-voxel window test.
template <bool kWindowKnown>
__device__ __forceinline__ void integrate_block_depth(uint4* blk, int lane, int ox, int oy, int oz, const Pose& pose,
                                                      const FrameArgs& fa, const float* __restrict__ depth, float wLim,
                                                      float hLim, float mu, bool muOk, float rMu, bool capW, int maxW) {
  const float vs = fa.voxelSize;
#pragma unroll
  for (int g = 0; g < 4; g += kQG) {
    uint32_t wd[4 * kQG];
#pragma unroll
    for (int q = g; q < g + kQG; ++q) {
      const uint4 r = blk[q * 32 + lane];
      wd[(q - g) * 4 + 0] = r.x;
      wd[(q - g) * 4 + 1] = r.y;
      wd[(q - g) * 4 + 2] = r.z;
      wd[(q - g) * 4 + 3] = r.w;
    }
    // ---- project
    float zc[4 * kQG];
    int pix[4 * kQG];
    unsigned slow = 0u;
#pragma unroll
    for (int q = g; q < g + kQG; ++q) {
      const int lin = (q * 32 + lane) * 4;
      const float pz = (float)(oz + (lin >> 6)) * vs;
      const float py = (float)(oy + ((lin >> 3) & 7)) * vs;
      const float r0 = pose.R[1] * py + pose.R[2] * pz;
      const float r1 = pose.R[4] * py + pose.R[5] * pz;
      const float r2 = pose.R[7] * py + pose.R[8] * pz;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = (q - g) * 4 + i;
        const float px = (float)(ox + (lin & 7) + i) * vs;
        const float cxw = (pose.R[0] * px + r0) + pose.t[0];
        const float cyw = (pose.R[3] * px + r1) + pose.t[1];
        const float czw = (pose.R[6] * px + r2) + pose.t[2];
        const float ax = fa.fx * cxw, ay = fa.fy * cyw;
        const float rz = div_rcp(czw);
        const float u = div_fast(ax, czw, rz) + fa.cx;
        const float v = div_fast(ay, czw, rz) + fa.cy;
        const bool in = czw > 0.f && !(u < 1 || u > wLim || v < 1 || v > hLim);
        pix[k] = in ? (int)(v + 0.5f) * fa.w + (int)(u + 0.5f) : -1;
        zc[k] = czw;
        if (!kWindowKnown) {
          const bool fast = czw >= 0x1p-40f && czw <= 0x1p40f && fabsf(ax) <= 0x1p40f && fabsf(ay) <= 0x1p40f;
          slow |= (czw > 0.f && !fast) ? (1u << k) : 0u;
        }
      }
    }
    if (!kWindowKnown && __any_sync(0xffffffffu, slow != 0u)) {
#pragma unroll
      for (int k = 0; k < 4 * kQG; ++k) {
        if (slow & (1u << k)) {
          const int lin = ((g + (k >> 2)) * 32 + lane) * 4;
          project_exact(pose, fa, wLim, hLim, (float)(ox + (lin & 7) + (k & 3)) * vs,
                        (float)(oy + ((lin >> 3) & 7)) * vs, (float)(oz + (lin >> 6)) * vs, &pix[k]);
        }
      }
    }
    // ---- gather
    float dm[4 * kQG];
#pragma unroll
    for (int k = 0; k < 4 * kQG; ++k) dm[k] = pix[k] >= 0 ? __ldg(depth + pix[k]) : -1.f;
    // ---- update (update_voxel_depth, fusion.cpp:9-36)
    unsigned redo = 0u;
#pragma unroll
    for (int k = 0; k < 4 * kQG; ++k) {
      const uint32_t w0 = wd[k];
      const int oldW = vox_w(w0);
      const float eta = dm[k] - zc[k];
      const bool upd = pix[k] >= 0 && !(dm[k] <= 0.f) && !(eta < -mu) && !(capW && oldW >= maxW);
      const float oldF = sdf_to_logical(vox_sdf(w0));
      const float newF = smin(1.f, div_fast(eta, mu, rMu));
      const float fw = (float)oldW;
      const float num = fw * oldF + newF;
      const float den = fw + 1.f;  // == (float)(oldW + 1): small integers are exact
      const float merged = div_fast(num, den, div_rcp(den));
      const uint32_t w1 = vox_pack(sdf_from_logical(merged), min(oldW + 1, maxW));
      // out-of-window voxels keep w0 here and are redone exactly below
      const bool slowK = kWindowKnown ? (upd && !(muOk && fabsf(eta) <= 0x1p40f))
                                      : (upd && !(muOk && fabsf(eta) <= 0x1p40f && !(slow & (1u << k))));
      wd[k] = (upd && !slowK) ? w1 : w0;
      redo |= slowK ? (1u << k) : 0u;
    }
    if (__any_sync(0xffffffffu, redo != 0u)) {
#pragma unroll
      for (int k = 0; k < 4 * kQG; ++k)
        if (redo & (1u << k)) wd[k] = update_exact(wd[k], dm[k] - zc[k], mu, maxW);
    }
#pragma unroll
    for (int q = g; q < g + kQG; ++q) {
      const int k = (q - g) * 4;
      blk[q * 32 + lane] = make_uint4(wd[k], wd[k + 1], wd[k + 2], wd[k + 3]);
    }
  }
}

// Block-level proof that every voxel of the block at (ox, oy, oz) projects
// inside div_fast's window (camera z in [2^-40, 2^40], |fx X|, |fy Y| <=
// 2^40).  The camera coordinates are affine in the voxel index, so their
// extremes over the block are at its 8 corners (lanes 0-7, one corner each);
// the computed values differ from the exact ones by a few ulp of the largest
// term, which the 2^-20 relative margin covers with room to spare.
__device__ __forceinline__ bool block_window_known(int lane, int ox, int oy, int oz, const Pose& pose,
                                                   const FrameArgs& fa) {
  bool ok = true;
  if (lane < 8) {
    const float vs = fa.voxelSize;
    const float px = (float)(ox + ((lane & 1) ? 7 : 0)) * vs;
    const float py = (float)(oy + ((lane & 2) ? 7 : 0)) * vs;
    const float pz = (float)(oz + ((lane & 4) ? 7 : 0)) * vs;
    const float cx = (pose.R[0] * px + (pose.R[1] * py + pose.R[2] * pz)) + pose.t[0];
    const float cy = (pose.R[3] * px + (pose.R[4] * py + pose.R[5] * pz)) + pose.t[1];
    const float cz = (pose.R[6] * px + (pose.R[7] * py + pose.R[8] * pz)) + pose.t[2];
    const float mag = fabsf(px) + fabsf(py) + fabsf(pz) + fabsf(pose.t[0]) + fabsf(pose.t[1]) + fabsf(pose.t[2]);
    const float f = fmaxf(1.f, fmaxf(fabsf(fa.fx), fabsf(fa.fy)));
    // either the whole block is in front of the camera inside the window, or
    // the whole block is behind it (z <= 0: every voxel is rejected before
    // any quotient is used)
    const bool front = cz > 0x1p-20f * mag + 0x1p-39f && cz < 0x1p38f;
    ok = front && f * fabsf(cx) < 0x1p38f && f * fabsf(cy) < 0x1p38f && f * mag < 0x1p38f;
  }
  return __all_sync(0xffffffffu, ok);
}

__global__ void __launch_bounds__(256, RFG_INT_MINB) k_integrate_depth(DevMap m, const float* __restrict__ depth,
                                                                       FrameArgs fa) {
  const int lane = threadIdx.x & 31;
  const int warpsPerCta = blockDim.x >> 5;
  const int gw = blockIdx.x * warpsPerCta + (threadIdx.x >> 5);
  const int nw = gridDim.x * warpsPerCta;
  const int nVis = *((volatile int*)&m.state->nVisible);
  const Pose pose = frame_pose(fa);
  const float wLim = (float)(fa.w - 2), hLim = (float)(fa.h - 2);
  const float mu = fa.mu;
  const bool muOk = mu >= 0x1p-20f && mu <= 0x1p20f;
  const float rMu = div_rcp(mu);
  const bool capW = fa.stopAtMaxW != 0;
  const int maxW = fa.maxW;
  for (int b = gw; b < nVis; b += nw) {
    const int idx = m.visibleList[b];
    const int4 e = ld_entry(m.entries, idx);
    if (e.w < 0) continue;
    const int ox = entry_x(e) * kBlock, oy = entry_y(e) * kBlock, oz = entry_z(e) * kBlock;
    uint4* blk = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)e.w * kBlock3);
    if (block_window_known(lane, ox, oy, oz, pose, fa))
      integrate_block_depth<true>(blk, lane, ox, oy, oz, pose, fa, depth, wLim, hLim, mu, muOk, rMu, capW, maxW);
    else
      integrate_block_depth<false>(blk, lane, ox, oy, oz, pose, fa, depth, wLim, hLim, mu, muOk, rMu, capW, maxW);
  }
}

#ifndef RFG_INT_GRID_PER_SM
#define RFG_INT_GRID_PER_SM 8
#endif
int integrate_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms * RFG_INT_GRID_PER_SM;  // two waves of 4 resident CTAs x 8 warps per SM
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
    k_integrate_depth<<<integrate_grid(), 256, 0, s>>>(m, depth, fa);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace rfg
