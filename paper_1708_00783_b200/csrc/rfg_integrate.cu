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

#ifndef RFG_INT_MINB
#define RFG_INT_MINB 4
#endif
#ifndef RFG_INT_QG
#define RFG_INT_QG 2
#endif
constexpr int kQG = RFG_INT_QG;  // rows (of 4 voxels) per project/gather/update group

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
// projection quotients are inside div_fast's exactness window, and the frame
// that every eta quotient is (depths below 2^36 m, mu in [2^-20, 2^20]), so
// no voxel needs a per-voxel window test.
#ifndef RFG_INT_DIET
#define RFG_INT_DIET 1
#endif
#ifndef RFG_INT_SKIP
#define RFG_INT_SKIP 1  // warp-uniform skip of the update math of voxel slots no lane updates
#endif
#ifndef RFG_INT_V2
#define RFG_INT_V2 1  // fewer ALU-pipe instructions per voxel (folded pixel index, F2I lround, sentinel depth)
#endif
#ifndef RFG_INT_RCP_HOIST
#define RFG_INT_RCP_HOIST 1  // a group's eight 1/(w+1) table reads before its per-slot skips
#endif
#ifndef RFG_INT_RCP_INLINE
#define RFG_INT_RCP_INLINE 0  // 1/(w+1) by MUFU + 2 FFMA per voxel instead of the shared table
#endif
#ifndef RFG_INT_V2_RANGE
#define RFG_INT_V2_RANGE 0  // the u / v window tests as (u - 1) bit compares
#endif
#ifndef RFG_INT_TMA
#define RFG_INT_TMA 0  // depth integration with TMA-prefetched voxel rows (k_integrate_depth_tma)
#endif
// RFG_INT_DIET: the per-voxel int<->float conversions and roundings on the
// FMA/ALU pipes (rfg_common.cuh magic conversions), the lane's x-column
// products R_0x px, R_3x px, R_6x px hoisted out of the rows (a lane's four
// voxels per row have the same x in every row), and 1/(w+1) from a per-CTA
// table (the exact div_rcp values) instead of a reciprocal per voxel.
__device__ __forceinline__ int16_t sdf_from_logical_alu(float f) {
  float c = f < -1.f ? -1.f : (1.f < f ? 1.f : f);
  return (int16_t)lround_haz_alu(c * (float)kSdfOne);
}

// 1 / (w + 1) as div_rcp computes it, w = 0..255, per CTA (filled by the
// depth kernels' prologue).  A file-scope __shared__ array, so a load is one
// LDS at the symbol's offset (through a pointer parameter the compiler
// re-derives the CTA's shared window base at every use).
__shared__ float s_rcpTab[256];

template <bool kWindowKnown>
__device__ __forceinline__ void integrate_block_depth(const uint4* src, uint4* blk, int lane, int ox, int oy, int oz,
                                                      const Pose& pose,
                                                      const FrameArgs& fa, const float* __restrict__ depth, float wLim,
                                                      float hLim, float mu, bool muOk, float rMu, bool capW, int maxW,
                                                      const float* rcpTab) {
  const float vs = fa.voxelSize;
#if RFG_INT_V2
  const uint32_t pixMagic = 0x4B000000u * ((uint32_t)fa.w + 1u);
  const int capMax = capW ? maxW : 256;  // oldW < capMax <=> !(capW && oldW >= maxW) (oldW <= 255)
#endif
#if RFG_INT_V2_RANGE
  const uint32_t uBound = __float_as_uint(wLim - 1.f), vBound = __float_as_uint(hLim - 1.f);
#endif
#if RFG_INT_DIET
  // this lane's four x columns: the same in all of its rows
  float rx0[4], rx3[4], rx6[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float px = (float)(ox + ((lane * 4) & 7) + i) * vs;
    rx0[i] = pose.R[0] * px;
    rx3[i] = pose.R[3] * px;
    rx6[i] = pose.R[6] * px;
  }
#endif
#pragma unroll
  for (int g = 0; g < 4; g += kQG) {
    uint32_t wd[4 * kQG];
#pragma unroll
    for (int q = g; q < g + kQG; ++q) {
      const uint4 r = src[q * 32 + lane];  // the voxel rows: global memory, or the TMA-staged copy
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
#if RFG_INT_DIET
        const float cxw = (rx0[i] + r0) + pose.t[0];
        const float cyw = (rx3[i] + r1) + pose.t[1];
        const float czw = (rx6[i] + r2) + pose.t[2];
#else
        const float px = (float)(ox + (lin & 7) + i) * vs;
        const float cxw = (pose.R[0] * px + r0) + pose.t[0];
        const float cyw = (pose.R[3] * px + r1) + pose.t[1];
        const float czw = (pose.R[6] * px + r2) + pose.t[2];
#endif
        const float ax = fa.fx * cxw, ay = fa.fy * cyw;
        const float rz = div_rcp(czw);
        const float u = div_fast(ax, czw, rz) + fa.cx;
        const float v = div_fast(ay, czw, rz) + fa.cy;
#if RFG_INT_V2_RANGE
        // 1 <= u <= wLim as one unsigned compare of the bits of u - 1 (exact
        // for u >= 0.5, negative below; negative floats compare above every
        // positive bound)
        const bool in = czw > 0.f && __float_as_uint(u - 1.f) <= uBound && __float_as_uint(v - 1.f) <= vBound;
#elif RFG_INT_V2
        // the reference's window tests (fusion.cpp:15-17) as the sign of one
        // max: 1 - u <= 0 <=> u >= 1 and u - wLim <= 0 <=> u <= wLim exactly
        // (a rounded difference keeps the sign of the exact one, and is zero
        // only when it is), so the projection stays branch-free with one
        // predicate
        const float outside = fmaxf(fmaxf(1.f - u, u - wLim), fmaxf(1.f - v, v - hLim));
        const bool in = (czw > 0.f) & (outside <= 0.f);
#else
        const bool in = czw > 0.f && !(u < 1 || u > wLim || v < 1 || v > hLim);
#endif
#if RFG_INT_V2
        // u, v in [1, W-2] when `in`: the truncations of u + 0.5, v + 0.5
        // (static_cast<int>, fusion.cpp:18) by the 2^23 magic number, with
        // both magic offsets folded into one constant (mod 2^32); computed
        // for every voxel, selected by `in`
        const int pv = (int)(__float_as_uint(__fadd_rz(v + 0.5f, 8388608.0f)) * (uint32_t)fa.w +
                             __float_as_uint(__fadd_rz(u + 0.5f, 8388608.0f)) - pixMagic);
        pix[k] = in ? pv : -1;
#elif RFG_INT_DIET
        // u, v in [1, W-2] when `in`: the truncations of u + 0.5, v + 0.5 (static_cast<int>, fusion.cpp:18)
        pix[k] = in ? trunc_pos_to_int(v + 0.5f) * fa.w + trunc_pos_to_int(u + 0.5f) : -1;
#else
        pix[k] = in ? (int)(v + 0.5f) * fa.w + (int)(u + 0.5f) : -1;
#endif
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
#if RFG_INT_V2 && RFG_INT_RCP_HOIST
    // the group's 1/(w+1) table reads in one block (one shared-window base)
    float rwt[4 * kQG];
#pragma unroll
    for (int k = 0; k < 4 * kQG; ++k) rwt[k] = s_rcpTab[vox_w(wd[k])];
#endif
#pragma unroll
    for (int k = 0; k < 4 * kQG; ++k) {
      const uint32_t w0 = wd[k];
      const int oldW = vox_w(w0);
      const float eta = dm[k] - zc[k];
#if RFG_INT_V2
      // dm = -1 for a voxel outside the image, so the depth test covers it
      const bool upd = !(dm[k] <= 0.f) && !(eta < -mu) && oldW < capMax;
#else
      const bool upd = pix[k] >= 0 && !(dm[k] <= 0.f) && !(eta < -mu) && !(capW && oldW >= maxW);
#endif
#if RFG_INT_SKIP
      // a voxel slot no lane of the warp updates skips the update math
      if (!__any_sync(0xffffffffu, upd)) continue;
#endif
#if RFG_INT_DIET
      const float oldF = sdf_to_logical_alu(vox_sdf(w0));
      const float newF = smin(1.f, div_fast(eta, mu, rMu));
      const float fw = u23_to_float((uint32_t)oldW);
      const float num = fw * oldF + newF;
      const float den = fw + 1.f;  // == (float)(oldW + 1): small integers are exact
#if RFG_INT_V2 && RFG_INT_RCP_INLINE
      const float merged = div_fast(num, den, div_rcp(den));
      (void)rcpTab;
#elif RFG_INT_V2 && RFG_INT_RCP_HOIST
      const float merged = div_fast(num, den, rwt[k]);  // == div_rcp(oldW + 1)
      (void)rcpTab;
#elif RFG_INT_V2
      const float merged = div_fast(num, den, s_rcpTab[oldW]);  // == div_rcp(oldW + 1)
      (void)rcpTab;
#else
      const float merged = div_fast(num, den, rcpTab[oldW]);  // rcpTab[w] == div_rcp(w + 1)
#endif
#if RFG_INT_V2
      // lround (half away from zero) of the clamped value * 32767: the sum
      // with +-0.5 rounded toward zero, then truncated (F2I.TRUNC)
      const float cl = fminf(fmaxf(merged, -1.f), 1.f) * (float)kSdfOne;
      const int sdfI = lround_haz_f2i(cl);
      const uint32_t w1 = ((uint32_t)sdfI & 0xFFFFu) | ((uint32_t)min(oldW + 1, maxW) << 16);
#else
      const uint32_t w1 = vox_pack(sdf_from_logical_alu(merged), min(oldW + 1, maxW));
#endif
#else
      const float oldF = sdf_to_logical(vox_sdf(w0));
      const float newF = smin(1.f, div_fast(eta, mu, rMu));
      const float fw = (float)oldW;
      const float num = fw * oldF + newF;
      const float den = fw + 1.f;  // == (float)(oldW + 1): small integers are exact
      const float merged = div_fast(num, den, div_rcp(den));
      const uint32_t w1 = vox_pack(sdf_from_logical(merged), min(oldW + 1, maxW));
#endif
      if (kWindowKnown) {
        // the block's quotients and the frame's depths, mu are proven inside
        // div_fast's window (integrate_block_depth's caller)
        wd[k] = upd ? w1 : w0;
        continue;
      }
      // out-of-window voxels keep w0 here and are redone exactly below
      const bool slowK = upd && !(muOk && fabsf(eta) <= 0x1p40f && !(slow & (1u << k)));
      wd[k] = (upd && !slowK) ? w1 : w0;
      redo |= slowK ? (1u << k) : 0u;
    }
    if (!kWindowKnown && __any_sync(0xffffffffu, redo != 0u)) {
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
  pdl_wait();
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
  // |eta| = |depth - z| <= 2^36 + 2^38 < 2^40 for every voxel of a block
  // whose projection window is proven, when the frame's depths are bounded
  const bool frameKnown = muOk && fa.depthBounded;
  float* rcpTab = s_rcpTab;  // 1 / (w + 1) as div_rcp computes it, w = 0..255
  rcpTab[threadIdx.x] = div_rcp((float)(threadIdx.x + 1));  // blockDim.x == 256
  __syncthreads();
  for (int b = gw; b < nVis; b += nw) {
    const int idx = m.visibleList[b];
    const int4 e = ld_entry(m.entries, idx);
    if (e.w < 0) continue;
    const int ox = entry_x(e) * kBlock, oy = entry_y(e) * kBlock, oz = entry_z(e) * kBlock;
    uint4* blk = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)e.w * kBlock3);
    if (frameKnown && block_window_known(lane, ox, oy, oz, pose, fa))
      integrate_block_depth<true>(blk, blk, lane, ox, oy, oz, pose, fa, depth, wLim, hLim, mu, muOk, rMu, capW,
                                  maxW, rcpTab);
    else
      integrate_block_depth<false>(blk, blk, lane, ox, oy, oz, pose, fa, depth, wLim, hLim, mu, muOk, rMu, capW,
                                   maxW, rcpTab);
  }
  pdl_trigger();
}

// ---------------------------------------- depth-only, TMA-prefetched rows
// The same per-block update with the block's 2 KiB of depth voxels brought
// into shared memory by the bulk-copy engine (cp.async.bulk, completion on
// an mbarrier) one block ahead of the warp that integrates it: a persistent
// grid (every CTA resident), each warp owning every nw-th visible block; a
// warp's lanes fetch the entries of its next 32 blocks in one batch, lane 0
// issues the bulk copy of block k+1 before integrating block k from its
// staged copy (2 stages per warp), and the results are stored to global
// memory directly.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load_2k(void* dst, const void* src, unsigned long long* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the stage's generic reads before the async write
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(2048u) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(2048u), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kTmaWarps = 8;
__global__ void __launch_bounds__(256, RFG_INT_MINB) k_integrate_depth_tma(DevMap m, const float* __restrict__ depth,
                                                                           FrameArgs fa) {
  __shared__ __align__(128) uint4 stage[kTmaWarps][2][kBlock3 / 4];
  __shared__ __align__(8) unsigned long long bar[kTmaWarps][2];
  float* rcpTab = s_rcpTab;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = blockIdx.x * kTmaWarps + w;
  const int nw = gridDim.x * kTmaWarps;
  const int nVis = *((volatile int*)&m.state->nVisible);
  const Pose pose = frame_pose(fa);
  const float wLim = (float)(fa.w - 2), hLim = (float)(fa.h - 2);
  const float mu = fa.mu;
  const bool muOk = mu >= 0x1p-20f && mu <= 0x1p20f;
  const float rMu = div_rcp(mu);
  const bool capW = fa.stopAtMaxW != 0;
  const int maxW = fa.maxW;
  rcpTab[threadIdx.x] = div_rcp((float)(threadIdx.x + 1));
  if (lane == 0) {
    mbar_init(&bar[w][0], 1);
    mbar_init(&bar[w][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nMine = nVis > gw ? (nVis - gw + nw - 1) / nw : 0;  // this warp's blocks
  unsigned phase = 0u;  // bit s: the parity stage s waits for next
  int4 eb = make_int4(0, 0, 0, -1);  // lane k: the entry of batch block k
  for (int base = 0; base < nMine; base += 32) {
    // one batched round of entry loads for the next 32 blocks
    const int kk = base + lane;
    eb = kk < nMine ? ld_entry(m.entries, m.visibleList[gw + kk * nw]) : make_int4(0, 0, 0, -1);
    const int nb = min(32, nMine - base);
    // prologue: the batch's first block
    {
      const int ptr0 = __shfl_sync(0xffffffffu, eb.w, 0);
      if (lane == 0 && ptr0 >= 0)
        bulk_load_2k(stage[w][base & 1], m.vbaDepth + (size_t)ptr0 * kBlock3, &bar[w][base & 1]);
    }
    for (int k = 0; k < nb; ++k) {
      const int i = base + k, s = i & 1;
      int4 e;
      e.x = __shfl_sync(0xffffffffu, eb.x, k);
      e.y = __shfl_sync(0xffffffffu, eb.y, k);
      e.w = __shfl_sync(0xffffffffu, eb.w, k);
      // the next block of the batch into the other stage (its last reader,
      // block i - 1, finished before the __syncwarp below)
      if (k + 1 < nb) {
        const int pn = __shfl_sync(0xffffffffu, eb.w, k + 1);
        if (lane == 0 && pn >= 0)
          bulk_load_2k(stage[w][s ^ 1], m.vbaDepth + (size_t)pn * kBlock3, &bar[w][s ^ 1]);
      }
      if (e.w >= 0) {
        mbar_wait(&bar[w][s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const int ox = entry_x(e) * kBlock, oy = entry_y(e) * kBlock, oz = entry_z(e) * kBlock;
        uint4* blk = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)e.w * kBlock3);
        if (muOk && fa.depthBounded && block_window_known(lane, ox, oy, oz, pose, fa))
          integrate_block_depth<true>(stage[w][s], blk, lane, ox, oy, oz, pose, fa, depth, wLim, hLim, mu, muOk,
                                      rMu, capW, maxW, rcpTab);
        else
          integrate_block_depth<false>(stage[w][s], blk, lane, ox, oy, oz, pose, fa, depth, wLim, hLim, mu, muOk,
                                       rMu, capW, maxW, rcpTab);
      }
      __syncwarp();
    }
  }
}

// --------------------------------------------------- RGB-D, branch-free
// ITMVoxel_s_rgb: the depth update above plus update_voxel_colour
// (fusion.cpp:38-70) for every voxel whose depth update returned
// eta >= -mu (fusion.cpp:257; update_voxel_depth returns -1 when the voxel
// does not project onto valid depth).  The colour image is read as packed
// RGBA8 words (k_rgb_to_rgba), one 32-bit load per bilinear tap.
struct ColourArgs {
  const uint32_t* rgba;  // RGBA8 words, rw x rh
  int rw, rh;
  float fx, fy, cx, cy;
  float extr[12];        // extrinsics_d_to_rgb
  int sameCamera;        // identity extrinsics + equal intrinsics: M_rgb == pose bitwise
};

// bilinear colour merge of one voxel (fusion.cpp:52-68); px, py inside
// [1, rw-2] x [1, rh-2]
__device__ __forceinline__ uint32_t colour_merge(uint32_t cw, float px, float py, const ColourArgs& ca, int maxW,
                                                 uint32_t c00, uint32_t c10, uint32_t c01, uint32_t c11) {
  const float fx = px - floorf(px), fy = py - floorf(py);
  const float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
  const int oldW = (int)(cw >> 24);
  const float fw = (float)oldW;
  const float den = (float)(oldW + 1);
  const float rden = div_rcp(den);
  uint32_t out = (uint32_t)min(oldW + 1, maxW) << 24;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int sh = 8 * k;
    const float sample = w00 * (float)((c00 >> sh) & 0xFFu) + w10 * (float)((c10 >> sh) & 0xFFu) +
                         w01 * (float)((c01 >> sh) & 0xFFu) + w11 * (float)((c11 >> sh) & 0xFFu);
    const float old = (float)((cw >> sh) & 0xFFu);
    // num in [0, 65535] and den in [1, 256]: inside div_fast's window (or 0)
    const float merged = div_fast(fw * old + sample, den, rden);
    const int r = lround_haz(merged);  // in [0, 255]: merged is a convex combination of bytes
    out |= (uint32_t)(r < 0 ? 0 : (r > 255 ? 255 : r)) << sh;
  }
  return out;
}

// the colour camera's pixel of a voxel (update_voxel_colour's projection,
// fusion.cpp:48-52): false when behind the camera or outside the margin
__device__ __forceinline__ bool colour_pixel(const Pose& M, const ColourArgs& ca, f3 pt, float* px, float* py) {
  const f3 pc = pose_apply(M, pt);
  if (!(pc.z > 0.f)) return false;
  const float ax = ca.fx * pc.x, ay = ca.fy * pc.y;
  float qx, qy;
  if (div_ok(pc.z) && div_ok(ax) && div_ok(ay)) {
    const float rz = div_rcp(pc.z);
    qx = div_fast(ax, pc.z, rz);
    qy = div_fast(ay, pc.z, rz);
  } else {
    qx = div_ieee(ax, pc.z);
    qy = div_ieee(ay, pc.z);
  }
  *px = qx + ca.cx;
  *py = qy + ca.cy;
  return !(*px < 1 || *px > (float)(ca.rw - 2) || *py < 1 || *py > (float)(ca.rh - 2));
}

template <bool kSameCamera>
__device__ __forceinline__ void integrate_block_rgbd(uint4* blk, uint4* cblk, int lane, int ox, int oy, int oz,
                                                     const Pose& pose, const Pose& Mrgb, const FrameArgs& fa,
                                                     const ColourArgs& ca, const float* __restrict__ depth,
                                                     float wLim, float hLim, float mu, bool muOk, float rMu, bool capW,
                                                     int maxW) {
  const float vs = fa.voxelSize;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    const uint4 r = blk[q * 32 + lane];
    const uint4 rc = cblk[q * 32 + lane];
    uint32_t wd[4] = {r.x, r.y, r.z, r.w};
    uint32_t cw[4] = {rc.x, rc.y, rc.z, rc.w};
    const int lin = (q * 32 + lane) * 4;
    const float pz = (float)(oz + (lin >> 6)) * vs;
    const float py = (float)(oy + ((lin >> 3) & 7)) * vs;
    const float r0 = pose.R[1] * py + pose.R[2] * pz;
    const float r1 = pose.R[4] * py + pose.R[5] * pz;
    const float r2 = pose.R[7] * py + pose.R[8] * pz;
    float zc[4], uu[4], vv[4];
    int pix[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float px = (float)(ox + (lin & 7) + i) * vs;
      const float cxw = (pose.R[0] * px + r0) + pose.t[0];
      const float cyw = (pose.R[3] * px + r1) + pose.t[1];
      const float czw = (pose.R[6] * px + r2) + pose.t[2];
      const float ax = fa.fx * cxw, ay = fa.fy * cyw;
      float u, v;
      if (czw > 0.f && !(div_ok(czw) && div_ok(ax) && div_ok(ay))) {
        u = div_ieee(ax, czw) + fa.cx;
        v = div_ieee(ay, czw) + fa.cy;
      } else {
        const float rz = div_rcp(czw);
        u = div_fast(ax, czw, rz) + fa.cx;
        v = div_fast(ay, czw, rz) + fa.cy;
      }
      const bool in = czw > 0.f && !(u < 1 || u > wLim || v < 1 || v > hLim);
      pix[i] = in ? (int)(v + 0.5f) * fa.w + (int)(u + 0.5f) : -1;
      zc[i] = czw;
      uu[i] = u;
      vv[i] = v;
    }
    float dm[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) dm[i] = pix[i] >= 0 ? __ldg(depth + pix[i]) : -1.f;
    bool gate[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t w0 = wd[i];
      const int oldW = vox_w(w0);
      const bool valid = pix[i] >= 0 && !(dm[i] <= 0.f);
      const float eta = dm[i] - zc[i];
      const bool upd = valid && !(eta < -mu) && !(capW && oldW >= maxW);
      if (upd) {
        const float oldF = sdf_to_logical(vox_sdf(w0));
        const float newF = smin(1.f, (muOk && div_ok(eta)) ? div_fast(eta, mu, rMu) : div_ieee(eta, mu));
        const float fw = (float)oldW;
        const float num = fw * oldF + newF;
        const float den = fw + 1.f;
        const float merged = div_ok(num) ? div_fast(num, den, div_rcp(den)) : div_ieee(num, den);
        wd[i] = vox_pack(sdf_from_logical(merged), min(oldW + 1, maxW));
      }
      gate[i] = (valid ? eta : -1.f) >= -mu;  // fusion.cpp:257 on update_voxel_depth's return value
    }
    // colour: the camera pixel, then the four bilinear taps of every gated voxel
    float cx4[4], cy4[4];
    bool cin[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (kSameCamera) {
        cx4[i] = uu[i];
        cy4[i] = vv[i];
        cin[i] = gate[i] && pix[i] >= 0;
      } else {
        cin[i] = false;
        if (gate[i]) {
          const f3 pt{(float)(ox + (lin & 7) + i) * vs, py, pz};
          cin[i] = colour_pixel(Mrgb, ca, pt, &cx4[i], &cy4[i]);
        }
      }
    }
    uint32_t tap[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (cin[i]) {
        const int x0 = (int)floorf(cx4[i]), y0 = (int)floorf(cy4[i]);
        const uint32_t* p0 = ca.rgba + (size_t)y0 * ca.rw + x0;
        tap[i][0] = __ldg(p0);
        tap[i][1] = __ldg(p0 + 1);
        tap[i][2] = __ldg(p0 + ca.rw);
        tap[i][3] = __ldg(p0 + ca.rw + 1);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (cin[i]) cw[i] = colour_merge(cw[i], cx4[i], cy4[i], ca, maxW, tap[i][0], tap[i][1], tap[i][2], tap[i][3]);
    blk[q * 32 + lane] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    cblk[q * 32 + lane] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
  }
}

// The same-camera form (identity extrinsics, equal intrinsics — the
// synthetic C3 stream): one projection serves both updates, and like the
// depth-only kernel every voxel of a row is computed unconditionally and the
// results selected (kWindowKnown: block_window_known proved the projection
// quotients inside div_fast's window).  The colour taps of the gated voxels
// are loaded (predicated) before any is used.
template <bool kWindowKnown>
__device__ __forceinline__ void integrate_block_rgbd_same(uint4* blk, uint4* cblk, int lane, int ox, int oy, int oz,
                                                          const Pose& pose, const FrameArgs& fa, const ColourArgs& ca,
                                                          const float* __restrict__ depth, float wLim, float hLim,
                                                          float mu, bool muOk, float rMu, bool capW, int maxW) {
  const float vs = fa.voxelSize;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    const uint4 r = blk[q * 32 + lane];
    const uint4 rc = cblk[q * 32 + lane];
    uint32_t wd[4] = {r.x, r.y, r.z, r.w};
    uint32_t cw[4] = {rc.x, rc.y, rc.z, rc.w};
    const int lin = (q * 32 + lane) * 4;
    const float pz = (float)(oz + (lin >> 6)) * vs;
    const float py = (float)(oy + ((lin >> 3) & 7)) * vs;
    const float r0 = pose.R[1] * py + pose.R[2] * pz;
    const float r1 = pose.R[4] * py + pose.R[5] * pz;
    const float r2 = pose.R[7] * py + pose.R[8] * pz;
    float zc[4], uu[4], vv[4];
    int pix[4];
    unsigned slow = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float px = (float)(ox + (lin & 7) + i) * vs;
      const float cxw = (pose.R[0] * px + r0) + pose.t[0];
      const float cyw = (pose.R[3] * px + r1) + pose.t[1];
      const float czw = (pose.R[6] * px + r2) + pose.t[2];
      const float ax = fa.fx * cxw, ay = fa.fy * cyw;
      const float rz = div_rcp(czw);
      float u = div_fast(ax, czw, rz) + fa.cx;
      float v = div_fast(ay, czw, rz) + fa.cy;
      if (!kWindowKnown) {
        const bool fast = czw >= 0x1p-40f && czw <= 0x1p40f && fabsf(ax) <= 0x1p40f && fabsf(ay) <= 0x1p40f;
        slow |= (czw > 0.f && !fast) ? (1u << i) : 0u;
      }
      zc[i] = czw;
      uu[i] = u;
      vv[i] = v;
    }
    if (!kWindowKnown && __any_sync(0xffffffffu, slow != 0u)) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (slow & (1u << i)) {
          const float px = (float)(ox + (lin & 7) + i) * vs;
          const f3 pc = pose_apply(pose, f3{px, py, pz});
          uu[i] = div_ieee(fa.fx * pc.x, pc.z) + fa.cx;
          vv[i] = div_ieee(fa.fy * pc.y, pc.z) + fa.cy;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#if RFG_INT_V2
      // as integrate_block_depth: one predicate, the folded magic pixel index
      const float outside = fmaxf(fmaxf(1.f - uu[i], uu[i] - wLim), fmaxf(1.f - vv[i], vv[i] - hLim));
      const bool in = (zc[i] > 0.f) & (outside <= 0.f);
      const int pv = (int)(__float_as_uint(__fadd_rz(vv[i] + 0.5f, 8388608.0f)) * (uint32_t)fa.w +
                           __float_as_uint(__fadd_rz(uu[i] + 0.5f, 8388608.0f)) - 0x4B000000u * ((uint32_t)fa.w + 1u));
      pix[i] = in ? pv : -1;
#else
      const bool in = zc[i] > 0.f && !(uu[i] < 1 || uu[i] > wLim || vv[i] < 1 || vv[i] > hLim);
      pix[i] = in ? (int)(vv[i] + 0.5f) * fa.w + (int)(uu[i] + 0.5f) : -1;
#endif
    }
    float dm[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) dm[i] = pix[i] >= 0 ? __ldg(depth + pix[i]) : -1.f;
    bool cin[4];
    unsigned redo = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t w0 = wd[i];
      const int oldW = vox_w(w0);
      const bool valid = pix[i] >= 0 && !(dm[i] <= 0.f);
      const float eta = dm[i] - zc[i];
      const bool upd = valid && !(eta < -mu) && !(capW && oldW >= maxW);
      // fusion.cpp:257 on update_voxel_depth's return value (-1 when invalid);
      // same camera: the colour pixel is the depth pixel, in the same margin
      cin[i] = ((valid ? eta : -1.f) >= -mu) && pix[i] >= 0;
#if RFG_INT_SKIP
      if (!__any_sync(0xffffffffu, upd)) continue;  // no lane updates this voxel slot
#endif
#if RFG_INT_V2
      const float oldF = sdf_to_logical_alu(vox_sdf(w0));
      const float newF = smin(1.f, div_fast(eta, mu, rMu));
      const float fw = u23_to_float((uint32_t)oldW);
      const float num = fw * oldF + newF;
      const float den = fw + 1.f;
      const float merged = div_fast(num, den, s_rcpTab[oldW]);  // == div_rcp(oldW + 1)
      const float cl = fminf(fmaxf(merged, -1.f), 1.f) * (float)kSdfOne;
      const int sdfI = lround_haz_f2i(cl);
      const uint32_t w1 = ((uint32_t)sdfI & 0xFFFFu) | ((uint32_t)min(oldW + 1, maxW) << 16);
      if (kWindowKnown) {  // window, depths and mu proven (k_integrate_rgbd)
        wd[i] = upd ? w1 : w0;
        continue;
      }
#else
      const float oldF = sdf_to_logical(vox_sdf(w0));
      const float newF = smin(1.f, div_fast(eta, mu, rMu));
      const float fw = (float)oldW;
      const float num = fw * oldF + newF;
      const float den = fw + 1.f;
      const float merged = div_fast(num, den, div_rcp(den));
      const uint32_t w1 = vox_pack(sdf_from_logical(merged), min(oldW + 1, maxW));
#endif
      // (a voxel whose projection left the window may also have a tiny eta:
      // its update is redone exactly too, as in integrate_block_depth)
      const bool slowK = upd && !(muOk && fabsf(eta) <= 0x1p40f && !(slow & (1u << i)));
      wd[i] = (upd && !slowK) ? w1 : w0;
      redo |= slowK ? (1u << i) : 0u;
    }
#if RFG_INT_V2
    if (!kWindowKnown && __any_sync(0xffffffffu, redo != 0u)) {
#else
    if (__any_sync(0xffffffffu, redo != 0u)) {
#endif
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (redo & (1u << i)) wd[i] = update_exact(wd[i], dm[i] - zc[i], mu, maxW);
    }
    uint32_t tap[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int x0 = (int)floorf(uu[i]), y0 = (int)floorf(vv[i]);
      const uint32_t* p0 = ca.rgba + (cin[i] ? (size_t)y0 * ca.rw + x0 : 0);
      tap[i][0] = cin[i] ? __ldg(p0) : 0u;
      tap[i][1] = cin[i] ? __ldg(p0 + 1) : 0u;
      tap[i][2] = cin[i] ? __ldg(p0 + ca.rw) : 0u;
      tap[i][3] = cin[i] ? __ldg(p0 + ca.rw + 1) : 0u;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#if RFG_INT_SKIP
      if (!__any_sync(0xffffffffu, cin[i])) continue;  // no lane colours this voxel slot
#endif
      const uint32_t c1 = colour_merge(cw[i], uu[i], vv[i], ca, maxW, tap[i][0], tap[i][1], tap[i][2], tap[i][3]);
      cw[i] = cin[i] ? c1 : cw[i];
    }
    blk[q * 32 + lane] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    cblk[q * 32 + lane] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
  }
}

#ifndef RFG_RGBD_MINB
#define RFG_RGBD_MINB 3
#endif
template <bool kSameCamera>
__global__ void __launch_bounds__(256, RFG_RGBD_MINB) k_integrate_rgbd(DevMap m, const float* __restrict__ depth, FrameArgs fa,
                                                           ColourArgs ca) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warpsPerCta = blockDim.x >> 5;
  const int gw = blockIdx.x * warpsPerCta + (threadIdx.x >> 5);
  const int nw = gridDim.x * warpsPerCta;
  const int nVis = *((volatile int*)&m.state->nVisible);
  const Pose pose = frame_pose(fa);
  Pose Mrgb = pose;
  if (!kSameCamera) Mrgb = pose_compose(pose_from12(ca.extr), pose);  // extrinsics_d_to_rgb * pose
  const float wLim = (float)(fa.w - 2), hLim = (float)(fa.h - 2);
  const float mu = fa.mu;
  const bool muOk = mu >= 0x1p-20f && mu <= 0x1p20f;
  const float rMu = div_rcp(mu);
  const bool capW = fa.stopAtMaxW != 0;
  const int maxW = fa.maxW;
#if RFG_INT_V2
  const bool frameKnown = muOk && fa.depthBounded;  // see k_integrate_depth
  s_rcpTab[threadIdx.x] = div_rcp((float)(threadIdx.x + 1));  // blockDim.x == 256
  __syncthreads();
#else
  const bool frameKnown = true;
#endif
  for (int b = gw; b < nVis; b += nw) {
    const int idx = m.visibleList[b];
    const int4 e = ld_entry(m.entries, idx);
    if (e.w < 0) continue;
    const int ox = entry_x(e) * kBlock, oy = entry_y(e) * kBlock, oz = entry_z(e) * kBlock;
    uint4* blk = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)e.w * kBlock3);
    uint4* cblk = reinterpret_cast<uint4*>(m.vbaColour + (size_t)e.w * kBlock3);
#ifdef RFG_RGBD_OLD
    if (false) {
#else
    if (kSameCamera) {
#endif
      if (frameKnown && block_window_known(lane, ox, oy, oz, pose, fa))
        integrate_block_rgbd_same<true>(blk, cblk, lane, ox, oy, oz, pose, fa, ca, depth, wLim, hLim, mu, muOk, rMu,
                                        capW, maxW);
      else
        integrate_block_rgbd_same<false>(blk, cblk, lane, ox, oy, oz, pose, fa, ca, depth, wLim, hLim, mu, muOk, rMu,
                                         capW, maxW);
    } else {
      integrate_block_rgbd<kSameCamera>(blk, cblk, lane, ox, oy, oz, pose, Mrgb, fa, ca, depth, wLim, hLim, mu, muOk,
                                        rMu, capW, maxW);
    }
  }
}

// RGB8 (3 bytes per pixel) -> RGBA8 words, 4 pixels per thread (three
// aligned 32-bit loads when the image is 4-byte aligned)
__global__ void k_rgb_to_rgba(const uint8_t* __restrict__ rgb, uint32_t* __restrict__ out, int n) {
  const int i4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i4 >= n) return;
  if (i4 + 4 <= n && (reinterpret_cast<uintptr_t>(rgb) & 3u) == 0) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(rgb + (size_t)i4 * 3);
    const uint32_t a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2);
    // bytes: a = r0 g0 b0 r1, b = g1 b1 r2 g2, c = b2 r3 g3 b3
    uint4 o;
    o.x = a & 0xFFFFFFu;
    o.y = (a >> 24) | ((b & 0xFFFFu) << 8);
    o.z = (b >> 16) | ((c & 0xFFu) << 16);
    o.w = c >> 8;
    *reinterpret_cast<uint4*>(out + i4) = o;
    return;
  }
  for (int i = i4; i < n && i < i4 + 4; ++i) {
    const uint8_t* s = rgb + (size_t)i * 3;
    out[i] = (uint32_t)s[0] | ((uint32_t)s[1] << 8) | ((uint32_t)s[2] << 16);
  }
}

const void* rgb_to_rgba_kernel() { return (const void*)k_rgb_to_rgba; }

cudaError_t launch_rgb_to_rgba(const uint8_t* rgb, uint32_t* out, int n, cudaStream_t s) {
  const int threads = 256, per = threads * 4;
  k_rgb_to_rgba<<<(n + per - 1) / per, threads, 0, s>>>(rgb, out, n);
  count_launch();
  return cudaGetLastError();
}

#ifndef RFG_INT_GRID_PER_SM
#define RFG_INT_GRID_PER_SM 8
#endif
int integrate_grid() {
  return current_sm_count() * RFG_INT_GRID_PER_SM;  // two waves of 4 resident CTAs x 8 warps per SM
}

// Depth-only (rgba == nullptr) or RGB-D integration of the visible blocks.
// extr34 nullptr = identity extrinsics.
cudaError_t launch_integrate(const DevMap& m, const float* depth, const uint32_t* rgba, const FrameArgs& fa,
                             const rfg_intrinsics* intrRgb, const float* extr34, cudaStream_t s) {
  if (rgba) {
    ColourArgs ca{};
    ca.rgba = rgba;
    ca.rw = intrRgb->width;
    ca.rh = intrRgb->height;
    ca.fx = intrRgb->fx;
    ca.fy = intrRgb->fy;
    ca.cx = intrRgb->cx;
    ca.cy = intrRgb->cy;
    bool ident = true;
    for (int i = 0; i < 12; ++i) {
      ca.extr[i] = extr34 ? extr34[i] : ((i % 5 == 0) ? 1.f : 0.f);
      // identity: M_rgb = extr * pose equals pose up to the sign of zero
      // entries, which cannot change a projection or a test downstream
      ident = ident && ca.extr[i] == ((i % 5 == 0) ? 1.f : 0.f);
    }
    ca.sameCamera = ident && ca.rw == fa.w && ca.rh == fa.h && ca.fx == fa.fx && ca.fy == fa.fy && ca.cx == fa.cx &&
                    ca.cy == fa.cy;
    if (ca.sameCamera)
      k_integrate_rgbd<true><<<integrate_grid(), 256, 0, s>>>(m, depth, fa, ca);
    else
      k_integrate_rgbd<false><<<integrate_grid(), 256, 0, s>>>(m, depth, fa, ca);
  } else {
#if RFG_INT_TMA
    k_integrate_depth_tma<<<current_sm_count() * RFG_INT_MINB, 256, 0, s>>>(m, depth, fa);
#else
    // a plain launch (no programmatic overlap with the allocation's tail): the
    // kernel's own duration is the roofline's denominator
    k_integrate_depth<<<integrate_grid(), 256, 0, s>>>(m, depth, fa);
#endif
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace rfg
