// rfg_raycast.cu — expected-range pass and ICP-map raycast
// (render_expected_ranges proj/src/raycast.cpp:86-127;
//  render_maps(kIcpMaps) proj/include/rf/raycast.hpp:157-207 with
//  cast_ray_field :54-112 and field_normal :137-153).
#include "rfg_common.cuh"

#ifndef RFG_RC_ALU
#define RFG_RC_ALU 1  // the march's conversions on the FMA/ALU pipes (0: XU conversions)
#endif
#ifndef RFG_RC_MERGE
#define RFG_RC_MERGE 1  // coarse residency tests and fine reads share one block resolution per step
#endif
#ifndef RFG_RC_F2I
#define RFG_RC_F2I 0  // 1: the nearest read's roundings as RZ add + F2I.TRUNC (measured slower)
#endif
#ifndef RFG_RC_ORDER
#define RFG_RC_ORDER 1  // the frame pipeline's raycast CTAs take the previous frame's heaviest tiles first
#endif
#ifndef RFG_RC_ORDER_K
#define RFG_RC_ORDER_K 2  // ... that many tiles per SM
#endif

namespace rfg {

// ------------------------------------------------------ expected ranges
// The reference covers each visible block's projected pixel rectangle with
// 16x16 fragments (count -> prefix sum -> emit, raycast.cpp:94-115) and
// min/max-merges every fragment into the range image (:118-126).  Min/max is
// exact and commutative, so any partition of the same rectangles gives the
// identical image.  Here the partition is by SCREEN tile instead of by block:
//   k_range_bin  — warp per visible block: lanes 0-7 project the corners
//                  (projectBlock, raycast.cpp:38-71), the warp reduces the
//                  rectangle and clipped z span, writes the block's bounds,
//                  and appends the block to every 32x32-pixel screen tile its
//                  rectangle touches (fixed-capacity bins);
//   k_range_tile — one CTA per screen tile, one thread per pixel: min/max over
//                  the tile's bin in registers, one store per pixel, no
//                  per-pixel atomics.  A tile whose bin overflowed scans the
//                  bounds of every visible block instead (same result).
constexpr int kRangeTile = kRangeTilePx;

__device__ __forceinline__ int4 pack_bounds(int x0, int y0, int x1, int y1, float lo, float hi) {
  return make_int4(x0 | (y0 << 16), x1 | (y1 << 16), __float_as_int(lo), __float_as_int(hi));
}

// The raycast's tile order for this frame (one extra CTA of the pipeline's
// k_range_bin launch, 256 threads): the tiles whose longest march in the
// previous frame (tileCost, steps) is among the K longest come first, the
// rest follow, each group in raster order; the costs are re-zeroed for this
// frame's raycast.  Only the schedule changes — every pixel's march is the
// same whichever CTA runs it.
__device__ void order_tiles(const DevMap& m, int n, int K) {
  __shared__ int hist[256];
  __shared__ int warpHeavy[8], warpLight[8];
  __shared__ int sT, sH;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  hist[tid] = 0;
  if (tid == 0) {
    sT = 1;
    sH = 0;
  }
  __syncthreads();
  for (int t = tid; t < n; t += 256) atomicAdd(&hist[min(m.tileCost[t], 255)], 1);
  __syncthreads();
  // acc = number of tiles with cost >= b for b = 255 - tid (b >= 1): an
  // inclusive scan over the bins in descending order; T = the largest b with
  // acc >= K (1 when fewer than K tiles have a cost)
  int acc = tid < 255 ? hist[255 - tid] : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, acc, o);
    if (lane >= o) acc += v;
  }
  if (lane == 31) warpHeavy[wid] = acc;
  __syncthreads();
  for (int w = 0; w < wid; ++w) acc += warpHeavy[w];
  const bool reach = tid < 255 && acc >= K;
  const bool first = reach && (tid == 0 || !(acc - (tid < 255 ? hist[255 - tid] : 0) >= K));
  if (first) {
    sT = 255 - tid;
    sH = acc;
  }
  if (tid == 254 && acc < K) sH = acc;  // fewer than K tiles with a cost: all of them first (T = 1)
  __syncthreads();
  const int T = sT, H = sH;
  int hBase = 0, lBase = H;
  for (int base = 0; base < n; base += 256) {
    const int t = base + tid;
    const bool in = t < n;
    const int c = in ? m.tileCost[t] : 0;
    const bool heavy = in && min(c, 255) >= T && c > 0;
    const bool light = in && !heavy;
    const unsigned bh = __ballot_sync(0xffffffffu, heavy), bl = __ballot_sync(0xffffffffu, light);
    if (lane == 0) {
      warpHeavy[wid] = __popc(bh);
      warpLight[wid] = __popc(bl);
    }
    __syncthreads();
    int ph = 0, pl = 0, th = 0, tl = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < wid) {
        ph += warpHeavy[w];
        pl += warpLight[w];
      }
      th += warpHeavy[w];
      tl += warpLight[w];
    }
    const unsigned below = (1u << lane) - 1u;
    if (heavy) m.tileOrder[hBase + ph + __popc(bh & below)] = t;
    if (light) m.tileOrder[lBase + pl + __popc(bl & below)] = t;
    if (in) m.tileCost[t] = 0;
    hBase += th;
    lBase += tl;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_range_bin(DevMap m, FrameArgs fa, int orderK) {
  pdl_wait();
  // orderK > 0: CTA 0 (dispatched first) writes the raycast's tile order
  if (orderK > 0 && blockIdx.x == 0) {
    order_tiles(m, m.binTilesX * ((fa.h + kRangeTile - 1) / kRangeTile), orderK);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int warpsPerCta = blockDim.x >> 5;
  const int cta = blockIdx.x - (orderK > 0 ? 1 : 0);
  const int gw = cta * warpsPerCta + (threadIdx.x >> 5);
  const int nw = (gridDim.x - (orderK > 0 ? 1 : 0)) * warpsPerCta;
  const int nVis = *((volatile int*)&m.state->nVisible);
  const Pose pose = frame_pose(fa);
  const float bs = fa.voxelSize * (float)kBlock;
  for (int b = gw; b < nVis; b += nw) {
    const int idx = m.visibleList[b];
    const int4 e = ld_entry(m.entries, idx);
    float x0 = FLT_MAX, y0 = FLT_MAX, x1 = -FLT_MAX, y1 = -FLT_MAX, zMin = FLT_MAX, zMax = 0.f;
    int valid = 0;
    if (lane < 8 && entry_allocated(e)) {
      const int c = lane;
      const f3 corner{((float)entry_x(e) + (float)(c & 1)) * bs, ((float)entry_y(e) + (float)((c >> 1) & 1)) * bs,
                      ((float)entry_z(e) + (float)((c >> 2) & 1)) * bs};
      const f3 pc = pose_apply(pose, corner);
      if (!(pc.z < 1e-6f)) {
        const float px = fa.fx * pc.x / pc.z + fa.cx;
        const float py = fa.fy * pc.y / pc.z + fa.cy;
        x0 = px;
        y0 = py;
        x1 = px;
        y1 = py;
        zMin = pc.z;
        zMax = pc.z;
        valid = 1;
      }
    }
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) {
      x0 = smin(x0, __shfl_xor_sync(0xffffffffu, x0, o));
      y0 = smin(y0, __shfl_xor_sync(0xffffffffu, y0, o));
      x1 = smax(x1, __shfl_xor_sync(0xffffffffu, x1, o));
      y1 = smax(y1, __shfl_xor_sync(0xffffffffu, y1, o));
      zMin = smin(zMin, __shfl_xor_sync(0xffffffffu, zMin, o));
      zMax = smax(zMax, __shfl_xor_sync(0xffffffffu, zMax, o));
      valid += __shfl_xor_sync(0xffffffffu, valid, o);
    }
    // lane 0 holds the reduction over lanes 0-7
    x0 = __shfl_sync(0xffffffffu, x0, 0);
    y0 = __shfl_sync(0xffffffffu, y0, 0);
    x1 = __shfl_sync(0xffffffffu, x1, 0);
    y1 = __shfl_sync(0xffffffffu, y1, 0);
    zMin = __shfl_sync(0xffffffffu, zMin, 0);
    zMax = __shfl_sync(0xffffffffu, zMax, 0);
    valid = __shfl_sync(0xffffffffu, valid, 0);
    int bx0 = 1, by0 = 1, bx1 = 0, by1 = 0;  // empty rectangle unless valid
    float zlo = 0.f, zhi = -1.f;
    if (valid) {
      bx0 = max(0, (int)floorf(x0));
      by0 = max(0, (int)floorf(y0));
      bx1 = min(fa.w - 1, (int)ceilf(x1));
      by1 = min(fa.h - 1, (int)ceilf(y1));
      zlo = smax(zMin, fa.vfMin);
      zhi = smin(zMax, fa.vfMax);
      if (bx0 > bx1 || by0 > by1 || zlo > zhi) {
        bx0 = by0 = 1;
        bx1 = by1 = 0;
      }
    }
    if (lane == 0) m.rangeBounds[b] = pack_bounds(bx0, by0, bx1, by1, zlo, zhi);
    if (bx0 > bx1) continue;
    const int tx0 = bx0 / kRangeTile, tx1 = bx1 / kRangeTile, ty0 = by0 / kRangeTile, ty1 = by1 / kRangeTile;
    const int ntx = tx1 - tx0 + 1, nt = ntx * (ty1 - ty0 + 1);
    for (int k = lane; k < nt; k += 32) {
      const int t = (ty0 + k / ntx) * m.binTilesX + tx0 + k % ntx;
      const int slot = atomicAdd(&m.binCount[t], 1);
      if (slot < m.binCap) m.bins[(size_t)t * m.binCap + slot] = b;
    }
  }
  pdl_trigger();
}

// The expected range (min, max bits) of this thread's pixel of screen tile t
// (blockIdx), from the tile's bin; every thread of the CTA must call it (it
// synchronises the CTA), and it re-zeroes the bin count for the next frame.
__device__ __forceinline__ int2 tile_ranges(const DevMap& m, int t, int tileX, int tileY, int4* sb) {
  const int count = m.binCount[t];
  const bool overflow = count > m.binCap;
  const int n = overflow ? *((volatile int*)&m.state->nVisible) : count;
  int lo = __float_as_int(FLT_MAX), hi = __float_as_int(-1.f);  // unset: (FLT_MAX, -1)
  for (int base = 0; base < n; base += kRangeTile * kRangeTile) {
    const int i = base + threadIdx.x;
    __syncthreads();
    if (i < n) {
      // the block's rectangle clipped to this tile as a column mask (bits
      // 0-15) and a row mask (bits 16-31): pixel (lx, ly) of the tile is
      // covered iff both of its bits are set (0 for an empty clip)
      const int4 bb = m.rangeBounds[overflow ? i : m.bins[(size_t)t * m.binCap + i]];
      const int tx = tileX * kRangeTile, ty = tileY * kRangeTile;
      const int lx0 = max((bb.x & 0xFFFF) - tx, 0), lx1 = min((bb.y & 0xFFFF) - tx, kRangeTile - 1);
      const int ly0 = max((bb.x >> 16) - ty, 0), ly1 = min((bb.y >> 16) - ty, kRangeTile - 1);
      uint32_t mask = 0u;
      if (lx0 <= lx1 && ly0 <= ly1)
        mask = (((2u << lx1) - 1u) & ~((1u << lx0) - 1u)) | ((((2u << ly1) - 1u) & ~((1u << ly0) - 1u)) << 16);
      sb[threadIdx.x] = make_int4((int)mask, bb.z, bb.w, 0);
    }
    __syncthreads();
    const int cnt = min(n - base, kRangeTile * kRangeTile);
    const uint32_t me = (1u << (threadIdx.x & (kRangeTile - 1))) | (1u << (16 + threadIdx.x / kRangeTile));
    for (int j = 0; j < cnt; ++j) {
      const int4 bb = sb[j];
      if (((uint32_t)bb.x & me) == me) {
        lo = min(lo, bb.y);  // positive floats order like their bit patterns
        hi = max(hi, bb.z);  // -1.f (negative int) loses against any z > 0
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) m.binCount[t] = 0;  // ready for the next frame
  return make_int2(lo, hi);
}

__global__ void __launch_bounds__(kRangeTile* kRangeTile) k_range_tile(DevMap m, FrameArgs fa, float2* range) {
  __shared__ int4 sb[kRangeTile * kRangeTile];
  const int t = blockIdx.y * m.binTilesX + blockIdx.x;
  const int x = blockIdx.x * kRangeTile + (threadIdx.x & (kRangeTile - 1));
  const int y = blockIdx.y * kRangeTile + threadIdx.x / kRangeTile;
  const int2 lh = tile_ranges(m, t, blockIdx.x, blockIdx.y, sb);
  if (x < fa.w && y < fa.h) range[(size_t)y * fa.w + x] = make_float2(__int_as_float(lh.x), __int_as_float(lh.y));
}

#if defined(RFG_RC_STATS) || defined(RFG_RC_TIMING)
__device__ unsigned long long g_rc_stats[32];
#endif
#if defined(RFG_RC_TIMING)
constexpr int kRcWarps = 1 << 14;
__device__ unsigned long long g_rc_warp[kRcWarps][16];
#endif
#ifdef RFG_RC_STATS
// debug build only: march statistics {rays, steps, coarse, invalid-fine,
// nearest-valid, trilinear, lookups, -, hist[log2 steps] x 16, max steps}
#define RC_STAT(i, v) atomicAdd(&g_rc_stats[i], (unsigned long long)(v))
#else
#define RC_STAT(i, v)
#endif

// ------------------------------------------------------------ raycast
// TSDF field reader (MapField, raycast.hpp:32-45) with the reference's
// last-block cache.  Voxel offsets inside a block use bit operations
// (v & 7 == v - (v >> 3) * 8 for negative v too).
// The voxels the raycast reads (the depth plane's sdf halves).  (A 2-B sdf
// mirror plane written by the integration — twice the voxels per L1 / L2
// line — was measured: raycast -2 % at C2 / -4 % at C4, integration +2 %,
// frame +1 %; not kept.)
typedef uint32_t FieldVoxel;
#define RFG_FIELD_PLANE(m) ((m).vbaDepth)
__device__ __forceinline__ int16_t field_sdf(uint32_t v) { return vox_sdf(v); }

struct FieldReader {
  const int4* entries;
  const FieldVoxel* vba;
  uint32_t buckets;
  BlockCache cache;
  int nSteps = 0;  // march steps of this ray (the pipeline's tile costs)
#ifdef RFG_RC_TIMING
  // debug build: what one ray did (hash lookups, entry loads of the chain
  // walks, nearest voxel loads, trilinear reads)
  int nLook = 0, nChain = 0, nNear = 0, nTri = 0;
  unsigned long long tseg[5] = {0, 0, 0, 0, 0};  // %globaltimer at steps 0, 16, 32, 48, 64
#define RC_CNT(f) (++(f))
#else
#define RC_CNT(f)
#endif

  // findEntry + ptr (voxel_block_map.cpp:26-34,63-72), uncached
  __device__ __forceinline__ int lookup(int bx, int by, int bz) const {
    RC_STAT(6, 1);
    RC_CNT(const_cast<FieldReader*>(this)->nLook);
    int ptr = -1;
    if (bx >= -32768 && bx <= 32767 && by >= -32768 && by <= 32767 && bz >= -32768 && bz <= 32767) {
      int idx = (int)hash_index(bx, by, bz, buckets - 1);
      const int xy = (int)((uint32_t)(uint16_t)bx | ((uint32_t)(uint16_t)by << 16));
      for (;;) {
        RC_CNT(const_cast<FieldReader*>(this)->nChain);
        const int4 e = __ldg(entries + idx);
        if (e.w >= -1 && e.x == xy && e.y == bz) {
          ptr = e.w;
          break;
        }
        if (e.z < 1) break;
        idx = (int)buckets + e.z - 1;
      }
    }
    return ptr >= 0 ? ptr : -1;
  }

  __device__ __forceinline__ int ptr_of(int bx, int by, int bz) {
    if (cache.bx == bx && cache.by == by && cache.bz == bz) return cache.ptr;
    cache.bx = bx;
    cache.by = by;
    cache.bz = bz;
    cache.ptr = lookup(bx, by, bz);
    return cache.ptr;
  }

  // MapField::resident (raycast.hpp:38-42)
  __device__ __forceinline__ bool resident(f3 p) {
    return ptr_of(((int)floorf(p.x)) >> 3, ((int)floorf(p.y)) >> 3, ((int)floorf(p.z)) >> 3) >= 0;
  }
  // readSdfNearest (voxel_block_map.cpp:178-185)
  __device__ __forceinline__ float nearest(f3 p, bool& ok) {
#if RFG_RC_F2I
    const int vx = lround_haz_f2i(p.x), vy = lround_haz_f2i(p.y), vz = lround_haz_f2i(p.z);
#elif RFG_RC_ALU
    const int vx = lround_haz_alu(p.x), vy = lround_haz_alu(p.y), vz = lround_haz_alu(p.z);
#else
    const int vx = lround_haz(p.x), vy = lround_haz(p.y), vz = lround_haz(p.z);
#endif
    const int ptr = ptr_of(vx >> 3, vy >> 3, vz >> 3);
    ok = ptr >= 0;
    if (!ok) return 1.f;
    RC_CNT(nNear);
    const FieldVoxel w = __ldg(vba + (size_t)ptr * kBlock3 + ((vx & 7) | ((vy & 7) << 3) | ((vz & 7) << 6)));
#if RFG_RC_ALU
    return sdf_to_logical_alu(field_sdf(w));
#else
    return sdf_to_logical(field_sdf(w));
#endif
  }
  // the sdf of voxel (vx, vy, vz) of block ptr (nearest's load and conversion)
  __device__ __forceinline__ float read_voxel(int ptr, int vx, int vy, int vz) {
    RC_CNT(nNear);
    const FieldVoxel w = __ldg(vba + (size_t)ptr * kBlock3 + ((vx & 7) | ((vy & 7) << 3) | ((vz & 7) << 6)));
    return sdf_to_logical_alu(field_sdf(w));
  }
  // readSdfWeightTrilinear (voxel_block_map.cpp:130-156).  Any missing
  // corner invalidates the read, so the corner order only matters for the
  // weighted sum, which is accumulated in the reference's k order.  Each
  // distinct block of the 2x2x2 cell is resolved once (1 lookup when the cell
  // is inside a block, 2 when it straddles one face, ...), through the
  // last-block cache for the base block, then the 8 voxel loads are issued
  // independently.
  __device__ __forceinline__ float trilinear(f3 p, bool& ok) {
    RC_STAT(5, 1);
    RC_CNT(nTri);
    const int bx = (int)floorf(p.x), by = (int)floorf(p.y), bz = (int)floorf(p.z);
    const float fx = p.x - (float)bx, fy = p.y - (float)by, fz = p.z - (float)bz;
    const int lx = bx & 7, ly = by & 7, lz = bz & 7;
    const bool cx = lx == 7, cy = ly == 7, cz = lz == 7;  // cell crosses into the next block along x/y/z
    const int bx0 = bx >> 3, by0 = by >> 3, bz0 = bz >> 3;
    const int q0 = ptr_of(bx0, by0, bz0);
    int qx = q0, qy = q0, qz = q0;
    if (cx) qx = lookup(bx0 + 1, by0, bz0);
    if (cy) qy = lookup(bx0, by0 + 1, bz0);
    if (cz) qz = lookup(bx0, by0, bz0 + 1);
    int qxy = cx ? qx : qy, qxz = cx ? qx : qz, qyz = cy ? qy : qz;
    if (cx && cy) qxy = lookup(bx0 + 1, by0 + 1, bz0);
    if (cx && cz) qxz = lookup(bx0 + 1, by0, bz0 + 1);
    if (cy && cz) qyz = lookup(bx0, by0 + 1, bz0 + 1);
    int qxyz = !cz ? qxy : (!cy ? qxz : (!cx ? qyz : lookup(bx0 + 1, by0 + 1, bz0 + 1)));
    if ((q0 | qx | qy | qz | qxy | qxz | qyz | qxyz) < 0) {
      ok = false;
      return 1.f;
    }
    const int ox0 = lx, ox1 = (lx + 1) & 7, oy0 = ly << 3, oy1 = ((ly + 1) & 7) << 3, oz0 = lz << 6,
              oz1 = ((lz + 1) & 7) << 6;
    FieldVoxel w[8];
    w[0] = __ldg(vba + (size_t)q0 * kBlock3 + (ox0 | oy0 | oz0));
    w[1] = __ldg(vba + (size_t)qx * kBlock3 + (ox1 | oy0 | oz0));
    w[2] = __ldg(vba + (size_t)qy * kBlock3 + (ox0 | oy1 | oz0));
    w[3] = __ldg(vba + (size_t)qxy * kBlock3 + (ox1 | oy1 | oz0));
    w[4] = __ldg(vba + (size_t)qz * kBlock3 + (ox0 | oy0 | oz1));
    w[5] = __ldg(vba + (size_t)qxz * kBlock3 + (ox1 | oy0 | oz1));
    w[6] = __ldg(vba + (size_t)qyz * kBlock3 + (ox0 | oy1 | oz1));
    w[7] = __ldg(vba + (size_t)qxyz * kBlock3 + (ox1 | oy1 | oz1));
    float sdf = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float bw =
          ((k & 1) ? fx : 1.f - fx) * (((k >> 1) & 1) ? fy : 1.f - fy) * (((k >> 2) & 1) ? fz : 1.f - fz);
#if RFG_RC_ALU
      sdf += bw * sdf_to_logical_alu(field_sdf(w[k]));
#else
      sdf += bw * sdf_to_logical(field_sdf(w[k]));
#endif
    }
    ok = true;
    return sdf;
  }
};

__device__ __forceinline__ f3 at_t(f3 o, f3 d, float t) { return f3{o.x + t * d.x, o.y + t * d.y, o.z + t * d.z}; }

// cast_ray_field (raycast.hpp:54-112).  Each fine/surface step first does
// its reads (the nearest voxel, then the trilinear value where the nearest
// one is valid and <= 0.1) and only then branches on the outcome, so the
// lanes of a warp that took different branches in the previous step still
// issue the reads together (18.7 instead of 15.6 active lanes per warp and
// 9 % fewer instructions than branching on the invalid read first).
__device__ bool cast_ray(FieldReader& field, f3 originM, f3 dirUnit, float tMinM, float tMaxM, float mu, float vs,
                         f3* hit) {
  const float coarseStep = (float)kBlock * vs;
  const float fineStep = mu;
  const float stepScale = mu;
  const f3 oV{originM.x / vs, originM.y / vs, originM.z / vs};
  const f3 dV{dirUnit.x / vs, dirUnit.y / vs, dirUnit.z / vs};
  float t = tMinM;
  enum { COARSE, FINE, SURFACE };
  int state = field.resident(at_t(oV, dV, t)) ? FINE : COARSE;
#ifdef RFG_RC_STATS
  int nSteps = 0, nCoarse = 0, nInv = 0, nNear = 0, nVs = 0;
  struct Fin {
    int& a; int& b; int& c; int& d; int& e;
    __device__ ~Fin() {
      RC_STAT(0, 1); RC_STAT(1, a); RC_STAT(2, b); RC_STAT(3, c); RC_STAT(4, d);
      RC_STAT(8 + min(15, 32 - __clz(a)), 1);
      atomicMax(&g_rc_stats[31], (unsigned long long)a);
      if (a >= 64) {  // the long rays: what their steps are
        RC_STAT(24, 1); RC_STAT(25, a); RC_STAT(26, b); RC_STAT(27, c); RC_STAT(28, e); RC_STAT(29, d - e);
      }
    }
  } fin{nSteps, nCoarse, nInv, nNear, nVs};
#endif
  while (t <= tMaxM) {
#ifdef RFG_RC_TIMING
    if ((field.nSteps & 15) == 0 && field.nSteps < 80)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(field.tseg[field.nSteps >> 4]));
#endif
    ++field.nSteps;
#ifdef RFG_RC_STATS
    ++nSteps;
#endif
#if RFG_RC_MERGE
    // the coarse step's residency test and the fine step's nearest read share
    // one block resolution (one lookup pass for a warp whose lanes are in
    // both states): floor-based block for COARSE (MapField::resident),
    // round-based for the reads
    bool ok = false;
    float sdf = 1.f;
    {
      const f3 p = at_t(oV, dV, t);
      const bool coarse = state == COARSE;
      const int vx = lround_haz_alu(p.x), vy = lround_haz_alu(p.y), vz = lround_haz_alu(p.z);
      const int bx = coarse ? (((int)floorf(p.x)) >> 3) : (vx >> 3);
      const int by = coarse ? (((int)floorf(p.y)) >> 3) : (vy >> 3);
      const int bz = coarse ? (((int)floorf(p.z)) >> 3) : (vz >> 3);
      const int ptr = field.ptr_of(bx, by, bz);
      if (coarse) {
#ifdef RFG_RC_STATS
        ++nCoarse;
#endif
        if (ptr >= 0) {
          state = FINE;
          t = smax(tMinM, t - coarseStep);
        } else {
          t += coarseStep;
        }
        continue;
      }
      ok = ptr >= 0;
      if (ok) sdf = field.read_voxel(ptr, vx, vy, vz);
    }
#else
    if (state == COARSE) {
#ifdef RFG_RC_STATS
      ++nCoarse;
#endif
      if (field.resident(at_t(oV, dV, t))) {
        state = FINE;
        t = smax(tMinM, t - coarseStep);
      } else {
        t += coarseStep;
      }
      continue;
    }
    // reads
    bool ok = false;
    float sdf = field.nearest(at_t(oV, dV, t), ok);
#endif
    if (ok && sdf <= 0.1f) {
      bool okTri = false;
      const float tri = field.trilinear(at_t(oV, dV, t), okTri);
      if (okTri) sdf = tri;
    }
    // the reference's state machine on them
    if (!ok) {
#ifdef RFG_RC_STATS
      ++nInv;
#endif
      if (state == SURFACE) state = FINE;
      t += fineStep;
      continue;
    }
#ifdef RFG_RC_STATS
    ++nNear;
#endif
    if (state == FINE) {
      if (sdf < 0.f) return false;  // WRONG_SIDE
      state = SURFACE;
    }
    if (sdf <= 0.f) {
      float tHit = t + sdf * stepScale;
      bool okR = false;
      const float f1 = field.trilinear(at_t(oV, dV, tHit), okR);
      if (okR) tHit += f1 * stepScale;
      *hit = at_t(oV, dV, tHit);
      return true;
    }
#ifdef RFG_RC_STATS
    if (!(vs < sdf * stepScale)) ++nVs;
#endif
    t += smax(sdf * stepScale, vs);
  }
  return false;
}

// field_normal (raycast.hpp:137-153)
__device__ __forceinline__ bool field_normal(FieldReader& field, f3 h, f3* n) {
  // six reads at hit +/- one voxel per axis, as (h + (1,0,0)), (h - (1,0,0)),
  // ... (the +0.f / -0.f components are kept: they are the reference's ops).
  // One rolled loop keeps a single inlined copy of the trilinear read; any
  // invalid read makes the normal invalid, so the loop may stop early.
  f3 g{0.f, 0.f, 0.f};
  float plus = 0.f;
#pragma unroll 1
  for (int d = 0; d < 6; ++d) {
    const int ax = d >> 1;
    const float ex = ax == 0 ? 1.f : 0.f, ey = ax == 1 ? 1.f : 0.f, ez = ax == 2 ? 1.f : 0.f;
    const f3 q = (d & 1) ? f3{h.x - ex, h.y - ey, h.z - ez} : f3{h.x + ex, h.y + ey, h.z + ez};
    bool ok = false;
    const float v = field.trilinear(q, ok);
    if (!ok) return false;
    if (!(d & 1)) {
      plus = v;
    } else {
      const float gd = plus - v;
      if (ax == 0)
        g.x = gd;
      else if (ax == 1)
        g.y = gd;
      else
        g.z = gd;
    }
  }
  const float len = sqrtf(sqnorm3(g));
  if (len < 1e-12f) return false;
  *n = f3{g.x / len, g.y / len, g.z / len};
  return true;
}

// render_maps_field doPixel (raycast.hpp:167-189) without the normal: the
// raycastResult and points of pixel (x, y).
__device__ __forceinline__ void raycast_pixel(const DevMap& m, const FrameArgs& fa, const float2* __restrict__ range,
                                              int x, int y, float4* raycast, float4* points) {
  const size_t i = (size_t)y * fa.w + x;
  const float4 invalid = make_float4(0.f, 0.f, 0.f, -1.f);
  float4 rc = invalid, pt = invalid;
  const float2 r = range[i];
  if (r.y >= r.x) {
    const Pose c2w = pose_inverse(frame_pose(fa));
    const f3 origin{c2w.t[0], c2w.t[1], c2w.t[2]};
    const f3 dirCam{((float)x - fa.cx) / fa.fx, ((float)y - fa.cy) / fa.fy, 1.f};
    const float norm = sqrtf(sqnorm3(dirCam));
    const f3 dw = rot_apply(c2w.R, dirCam);
    const f3 dirW{dw.x / norm, dw.y / norm, dw.z / norm};
    FieldReader field{m.entries, RFG_FIELD_PLANE(m), m.buckets};
    field.cache.reset();
    f3 hit;
    if (cast_ray(field, origin, dirW, r.x * norm, r.y * norm, fa.mu, fa.voxelSize, &hit)) {
      rc = make_float4(hit.x, hit.y, hit.z, 1.f);
      pt = make_float4(hit.x * fa.voxelSize, hit.y * fa.voxelSize, hit.z * fa.voxelSize, 1.f);
    }
  }
  raycast[i] = rc;
  points[i] = pt;
}

// field_normal (raycast.hpp:137-153) at the hit stored in raycast[i].
__device__ __forceinline__ void normal_pixel(const DevMap& m, const float4* __restrict__ raycast, float4* normals,
                                             size_t i) {
  const float4 r = raycast[i];
  float4 nm = make_float4(0.f, 0.f, 0.f, -1.f);
  if (r.w > 0.f) {
    FieldReader field{m.entries, RFG_FIELD_PLANE(m), m.buckets};
    field.cache.reset();
    f3 n;
    if (field_normal(field, f3{r.x, r.y, r.z}, &n)) nm = make_float4(n.x, n.y, n.z, 1.f);
  }
  normals[i] = nm;
}

#ifndef RFG_RC_MINB
#define RFG_RC_MINB 1
#endif
#ifndef RFG_NRM_MINB
#define RFG_NRM_MINB 1
#endif
// One thread per pixel in 16x8 tiles (neighbouring rays share blocks).
__global__ void __launch_bounds__(128, RFG_RC_MINB) k_raycast_icp(DevMap m, FrameArgs fa, const float2* __restrict__ range,
                                                     float4* raycast, float4* points) {
  const int x = blockIdx.x * 16 + (threadIdx.x & 15);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 4);
#if defined(RFG_RC_TIMING)
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) atomicMin(&g_rc_stats[24], t0);
#endif
  if (x < fa.w && y < fa.h) raycast_pixel(m, fa, range, x, y, raycast, points);
#if defined(RFG_RC_TIMING)
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  unsigned long long dur = t1 - t0, end = t1, sum = t1 - t0;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    dur = max(dur, __shfl_xor_sync(0xffffffffu, dur, o));
    end = max(end, __shfl_xor_sync(0xffffffffu, end, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&g_rc_stats[7], dur);  // longest thread (ray) duration, ns
    atomicMax(&g_rc_stats[25], end);
    atomicAdd(&g_rc_stats[26], sum);
    atomicAdd(&g_rc_stats[27], 32ull);
  }
#endif
}

// The march and the normal of each pixel in one kernel.  A lane computes
// its normal after its march returns, i.e. after the warp's lanes have
// reconverged behind the longest march of the warp, so the six trilinear
// reads of the normals run warp-uniform; and a tile's normals are done while
// other SMs still march their long rays (the separate normals kernel could
// only start after the longest ray of the whole image).
__device__ __forceinline__ void raycast_and_normal(const DevMap& m, const FrameArgs& fa, int x, int y, float2 r,
                                                   float4* raycast, float4* points, float4* normals,
                                                   unsigned long long* ctr = nullptr, int* stepsOut = nullptr) {
  const size_t i = (size_t)y * fa.w + x;
  const float4 invalid = make_float4(0.f, 0.f, 0.f, -1.f);
  float4 rc = invalid, pt = invalid, nm = invalid;
  FieldReader field{m.entries, RFG_FIELD_PLANE(m), m.buckets};
  field.cache.reset();
  bool isHit = false;
  f3 hit{0.f, 0.f, 0.f};
  if (r.y >= r.x) {
    const Pose c2w = pose_inverse(frame_pose(fa));
    const f3 origin{c2w.t[0], c2w.t[1], c2w.t[2]};
    const f3 dirCam{((float)x - fa.cx) / fa.fx, ((float)y - fa.cy) / fa.fy, 1.f};
    const float norm = sqrtf(sqnorm3(dirCam));
    const f3 dw = rot_apply(c2w.R, dirCam);
    const f3 dirW{dw.x / norm, dw.y / norm, dw.z / norm};
    isHit = cast_ray(field, origin, dirW, r.x * norm, r.y * norm, fa.mu, fa.voxelSize, &hit);
#ifdef RFG_RC_REMARCH
    // debug experiment: a long ray marches again with its blocks now warm in
    // L1 / L2; ctr[10] = that second march's ns, ctr[11] = its steps
    if (ctr && field.nSteps >= 48) {
      unsigned long long ta, tb;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ta));
      FieldReader f2{m.entries, RFG_FIELD_PLANE(m), m.buckets};
      f2.cache.reset();
      f3 h2;
      const bool again = cast_ray(f2, origin, dirW, r.x * norm, r.y * norm, fa.mu, fa.voxelSize, &h2);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb));
      ctr[10] = (tb - ta) + (again ? 0ull : 0ull);
      ctr[11] = (unsigned long long)f2.nSteps;
    }
#endif
    if (isHit) {
      rc = make_float4(hit.x, hit.y, hit.z, 1.f);
      pt = make_float4(hit.x * fa.voxelSize, hit.y * fa.voxelSize, hit.z * fa.voxelSize, 1.f);
    }
  }
  raycast[i] = rc;
  points[i] = pt;
  if (isHit) {
    f3 n;
    if (field_normal(field, hit, &n)) nm = make_float4(n.x, n.y, n.z, 1.f);
  }
  normals[i] = nm;
  if (stepsOut) *stepsOut = field.nSteps;
#ifdef RFG_RC_TIMING
  if (ctr) {
    ctr[0] = field.nSteps;
    ctr[1] = field.nLook;
    ctr[2] = field.nChain;
    ctr[3] = field.nNear;
    ctr[4] = field.nTri;
    for (int k = 0; k < 5; ++k) ctr[5 + k] = field.tseg[k];
  }
#else
  (void)ctr;
#endif
}

__global__ void __launch_bounds__(128, RFG_RC_MINB) k_raycast_maps(DevMap m, FrameArgs fa,
                                                                   const float2* __restrict__ range,
                                                                   float4* raycast, float4* points, float4* normals) {
  const int x = blockIdx.x * 16 + (threadIdx.x & 15);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 4);
  if (x >= fa.w || y >= fa.h) return;
  raycast_and_normal(m, fa, x, y, range[(size_t)y * fa.w + x], raycast, points, normals);
}

// The frame pipeline's form: one CTA per 16x16 screen tile first reduces the
// tile's expected ranges from its bin (k_range_tile's work, the range stays
// in a register; it is also stored for the caller), then marches its pixels
// (warps of 16x2 pixels, as k_raycast_maps).  One launch and one pass over
// the range image fewer.
#ifndef RFG_RC_TILES_MINB
#define RFG_RC_TILES_MINB 1
#endif
__global__ void __launch_bounds__(kRangeTile* kRangeTile, RFG_RC_TILES_MINB) k_raycast_tiles(DevMap m, FrameArgs fa, float2* range,
                                                                          float4* raycast, float4* points,
                                                                          float4* normals, int ordered) {
  __shared__ int4 sb[kRangeTile * kRangeTile];
  pdl_wait();
  // ordered: a 1-D grid over the tiles in this frame's order (order_tiles)
  const int t = ordered ? m.tileOrder[blockIdx.x] : blockIdx.y * m.binTilesX + blockIdx.x;
  const int tileX = ordered ? t % m.binTilesX : blockIdx.x, tileY = ordered ? t / m.binTilesX : blockIdx.y;
  const int x = tileX * kRangeTile + (threadIdx.x & (kRangeTile - 1));
  const int y = tileY * kRangeTile + threadIdx.x / kRangeTile;
#if defined(RFG_RC_TIMING)
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
  const int2 lh = tile_ranges(m, t, tileX, tileY, sb);
  if (x >= fa.w || y >= fa.h) return;
  const float2 r = make_float2(__int_as_float(lh.x), __int_as_float(lh.y));
  range[(size_t)y * fa.w + x] = r;
#if defined(RFG_RC_TIMING)
  // debug build: per warp, the longest march (+ normal) and what it did:
  // g_rc_warp[warp] = {dur, start, end, steps, lookups, chain loads, nearest
  // loads, trilinear reads, max steps of the warp, sum of ray ns, CTA start}
  unsigned long long tr;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr));
  unsigned long long ctr[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int steps = 0;
  raycast_and_normal(m, fa, x, y, r, raycast, points, normals, ctr, &steps);
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  const unsigned act = __activemask();
  const unsigned long long dur = t1 - tr;
  unsigned long long key = (dur << 5) | (threadIdx.x & 31), sum = dur;
  int ms = (int)ctr[0];
  for (int o = 16; o >= 1; o >>= 1) {
    key = max(key, __shfl_xor_sync(act, key, o));
    sum += __shfl_xor_sync(act, sum, o);
    ms = max(ms, __shfl_xor_sync(act, ms, o));
  }
  if ((threadIdx.x & 31) == (unsigned)(key & 31)) {
    unsigned long long* rec = g_rc_warp[(t * (kRangeTile * kRangeTile / 32) + (threadIdx.x >> 5)) & (kRcWarps - 1)];
    rec[0] = dur;
    rec[1] = tr;
    rec[2] = t1;
    for (int k = 0; k < 5; ++k) rec[3 + k] = (unsigned long long)ctr[k];
    rec[8] = (unsigned long long)ms;
    rec[9] = sum;
    rec[10] = t0;
    for (int k = 0; k < 3; ++k) rec[11 + k] = ctr[5 + k];  // steps 0, 16, 32
    rec[14] = ctr[10];
    rec[15] = ctr[11];
  }
#else
  int steps = 0;
  raycast_and_normal(m, fa, x, y, r, raycast, points, normals, nullptr, &steps);
#endif
  // the tile's cost for the next frame's order: its longest march
  if (ordered) {
    const int ws = __reduce_max_sync(__activemask(), steps);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(__activemask()) - 1)) atomicMax(&m.tileCost[t], ws);
  }
}

// Normals at every hit, in their own kernel: the six trilinear reads are
// uniform work across the warp instead of running behind the divergent march.
__global__ void __launch_bounds__(128, RFG_NRM_MINB) k_raycast_normals(DevMap m, FrameArgs fa, const float4* __restrict__ raycast,
                                                         float4* normals) {
  const int x = blockIdx.x * 16 + (threadIdx.x & 15);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 4);
  if (x >= fa.w || y >= fa.h) return;
  normal_pixel(m, raycast, normals, (size_t)y * fa.w + x);
}

// render_maps(..., missingOnly) (raycast.hpp:200-202): the listed pixels only.
__global__ void __launch_bounds__(128) k_raycast_list(DevMap m, FrameArgs fa, const float2* __restrict__ range,
                                                      const int* __restrict__ list, const int* __restrict__ count,
                                                      float4* raycast, float4* points) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *count) return;
  const int i = list[k];
  raycast_pixel(m, fa, range, i % fa.w, i / fa.w, raycast, points);
}

__global__ void __launch_bounds__(128) k_normals_list(DevMap m, const int* __restrict__ list,
                                                      const int* __restrict__ count, const float4* __restrict__ raycast,
                                                      float4* normals) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *count) return;
  normal_pixel(m, raycast, normals, (size_t)list[k]);
}

// ------------------------------------------------ colour / grey render modes
// render_maps_field's colour (raycast.hpp:169,191-197; colourAt =
// readColourTrilinear clamped and truncated, raycast.cpp:132-137), computed
// from the maps of the same render after the march and the normals:
// mode 1 kColour = trilinear colour at the hit over the corners that exist,
// mode 2 kGrey = |n . dirWorld| clamped to [0, 1] * 255 where the normal is
// valid; (0, 0, 0) elsewhere.  3 B out + 32 B in (+ 8 colour gathers) per px.
__device__ __forceinline__ uint8_t clamp_u8(float v) { return (uint8_t)(v < 0.f ? 0.f : (255.f < v ? 255.f : v)); }

__global__ void __launch_bounds__(128) k_render_colour(DevMap m, FrameArgs fa, int mode,
                                                       const float4* __restrict__ raycast,
                                                       const float4* __restrict__ normals,
                                                       const int* __restrict__ list, const int* __restrict__ count,
                                                       uint8_t* __restrict__ rgb) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (list) {
    if (i >= *count) return;
    i = list[i];
  } else if (i >= fa.w * fa.h) {
    return;
  }
  uint8_t c0 = 0, c1 = 0, c2 = 0;
  const float4 r = raycast[i];
  if (r.w > 0.f) {
    if (mode == 1 && m.vbaColour) {
      FieldReader field{m.entries, RFG_FIELD_PLANE(m), m.buckets};
      field.cache.reset();
      const int bx = (int)floorf(r.x), by = (int)floorf(r.y), bz = (int)floorf(r.z);
      const float fx = r.x - (float)bx, fy = r.y - (float)by, fz = r.z - (float)bz;
      float cr = 0.f, cg = 0.f, cb = 0.f;
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int vx = bx + (k & 1), vy = by + ((k >> 1) & 1), vz = bz + ((k >> 2) & 1);
        const int ptr = field.ptr_of(vx >> 3, vy >> 3, vz >> 3);
        if (ptr < 0) continue;
        const uint32_t w = __ldg(m.vbaColour + (size_t)ptr * kBlock3 + ((vx & 7) | ((vy & 7) << 3) | ((vz & 7) << 6)));
        const float bw = ((k & 1) ? fx : 1.f - fx) * (((k >> 1) & 1) ? fy : 1.f - fy) * (((k >> 2) & 1) ? fz : 1.f - fz);
        cr += bw * (float)(w & 0xFFu);
        cg += bw * (float)((w >> 8) & 0xFFu);
        cb += bw * (float)((w >> 16) & 0xFFu);
      }
      c0 = clamp_u8(cr);
      c1 = clamp_u8(cg);
      c2 = clamp_u8(cb);
    } else if (mode == 2) {
      const float4 n = normals[i];
      if (n.w > 0.f) {
        const int x = i % fa.w, y = i / fa.w;
        const Pose c2w = pose_inverse(frame_pose(fa));
        const f3 dirCam{((float)x - fa.cx) / fa.fx, ((float)y - fa.cy) / fa.fy, 1.f};
        const float norm = sqrtf(sqnorm3(dirCam));
        const f3 dw = rot_apply(c2w.R, dirCam);
        const f3 dirW{dw.x / norm, dw.y / norm, dw.z / norm};
        float shade = fabsf(dot3(f3{n.x, n.y, n.z}, dirW));
        shade = shade < 0.f ? 0.f : (1.f < shade ? 1.f : shade);
        c0 = c1 = c2 = (uint8_t)(shade * 255.f);
      }
    }
  }
  rgb[3 * (size_t)i] = c0;
  rgb[3 * (size_t)i + 1] = c1;
  rgb[3 * (size_t)i + 2] = c2;
}

cudaError_t launch_render_colour(const DevMap& m, const FrameArgs& fa, int mode, const float4* raycast,
                                 const float4* normals, const int* list, const int* count, int maxCount,
                                 uint8_t* rgb, cudaStream_t s) {
  const int n = list ? maxCount : fa.w * fa.h;
  if (n <= 0) return cudaSuccess;
  k_render_colour<<<(n + 127) / 128, 128, 0, s>>>(m, fa, mode, raycast, normals, list, count, rgb);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------ forward projection
// forward_project (raycast.cpp:141-188).  The serial reference visits the
// previous hits in row-major order and keeps a target pixel's first point
// unless a later one is strictly nearer; one 64-bit atomicMin per source
// point on (float bits of camera z << 32 | source index) keeps exactly that
// point (positive floats order like their bits; ties resolve to the smaller,
// i.e. earlier, source index).
__global__ void k_fwd_init(const float4* __restrict__ raycast, float4* prev, unsigned long long* keys, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  prev[i] = raycast[i];
  keys[i] = ~0ull;
}

__global__ void k_fwd_scatter(const float4* __restrict__ prev, unsigned long long* keys, Pose12 pose, int w, int h,
                              float fx, float fy, float cx, float cy, float vs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w * h) return;
  const float4 r = prev[i];
  if (r.w <= 0.f) return;
  const f3 world{r.x * vs, r.y * vs, r.z * vs};
  const f3 pc = pose_apply(pose_from12(pose.v), world);
  if (pc.z <= 0.f) return;
  const float px = fx * pc.x / pc.z + cx;
  const float py = fy * pc.y / pc.z + cy;
  const int ix = (int)lroundf(px), iy = (int)lroundf(py);
  if (ix < 0 || iy < 0 || ix >= w || iy >= h) return;
  const unsigned long long key = ((unsigned long long)__float_as_uint(pc.z) << 32) | (unsigned)i;
  atomicMin(keys + (size_t)iy * w + ix, key);
}

// Writes the forwarded (or invalid) maps and counts missing pixels per
// 1024-pixel tile for the row-major compaction.
__global__ void __launch_bounds__(kTileThreads) k_fwd_gather(const float4* __restrict__ prev,
                                                              const unsigned long long* __restrict__ keys,
                                                              float4* raycast, float4* points, float4* normals, int n,
                                                              float vs, int2* tileCounts) {
  const float4 invalid = make_float4(0.f, 0.f, 0.f, -1.f);
  int miss = 0;
  for (int j = 0; j < 4; ++j) {
    const int t = blockIdx.x * kTile + j * kTileThreads + threadIdx.x;
    if (t >= n) continue;
    const unsigned long long key = keys[t];
    float4 rc = invalid, pt = invalid;
    if (key != ~0ull) {
      rc = prev[(unsigned)(key & 0xffffffffull)];
      pt = make_float4(rc.x * vs, rc.y * vs, rc.z * vs, 1.f);
    }
    raycast[t] = rc;
    points[t] = pt;
    normals[t] = invalid;  // the reference leaves forwarded normals invalid
    miss += rc.w <= 0.f ? 1 : 0;
  }
  __shared__ int total;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  if (miss) atomicAdd(&total, miss);
  __syncthreads();
  if (threadIdx.x == 0) tileCounts[blockIdx.x] = make_int2(total, 0);
}

__global__ void k_pix_scan(const int2* counts, int2* prefix, int nTiles, int* total) {
  if (threadIdx.x != 0) return;
  int s = 0;
  for (int i = 0; i < nTiles; ++i) {
    prefix[i] = make_int2(s, 0);
    s += counts[i].x;
  }
  *total = s;
}

// Row-major compaction of the missing pixels (tile-local order by a CTA scan).
__global__ void __launch_bounds__(kTileThreads) k_fwd_emit(const float4* __restrict__ raycast, int n,
                                                            const int2* __restrict__ prefix, int* list) {
  __shared__ int warpSum[kTileThreads / 32];
  const int base = blockIdx.x * kTile + threadIdx.x * 4;
  int flags = 0, cnt = 0;
  for (int j = 0; j < 4; ++j) {
    const int t = base + j;
    if (t < n && raycast[t].w <= 0.f) {
      flags |= 1 << j;
      ++cnt;
    }
  }
  // block exclusive scan of cnt
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) warpSum[wid] = inc;
  __syncthreads();
  int wbase = 0;
  for (int k = 0; k < wid; ++k) wbase += warpSum[k];
  int o = prefix[blockIdx.x].x + wbase + inc - cnt;
  for (int j = 0; j < 4; ++j)
    if (flags & (1 << j)) list[o++] = base + j;
}

__global__ void k_iota_count(int* list, int n, int* count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) list[i] = i;
  if (i == 0) *count = n;
}

int range_grid() { return current_sm_count() * 8; }

cudaError_t launch_ranges(const DevMap& m, const FrameArgs& fa, float2* range, cudaStream_t s) {
  const int tx = (fa.w + kRangeTile - 1) / kRangeTile, ty = (fa.h + kRangeTile - 1) / kRangeTile;
  if (tx != m.binTilesX || ty > m.binTilesY) return cudaErrorInvalidValue;  // scratch sized by ensure_range_scratch
  k_range_bin<<<range_grid(), 256, 0, s>>>(m, fa, 0);
  k_range_tile<<<dim3(tx, ty), kRangeTile * kRangeTile, 0, s>>>(m, fa, range);
  count_launch(2);
  return cudaGetLastError();
}

// Expected ranges + ICP maps for the frame pipeline: launch_range_bin, then
// launch_raycast_tiles (the range tiles are reduced inside the raycast's CTAs).
cudaError_t launch_range_bin(const DevMap& m, const FrameArgs& fa, cudaStream_t s) {
  const int tx = (fa.w + kRangeTile - 1) / kRangeTile, ty = (fa.h + kRangeTile - 1) / kRangeTile;
  if (tx != m.binTilesX || ty > m.binTilesY) return cudaErrorInvalidValue;  // scratch sized by ensure_range_scratch
  const int orderK = RFG_RC_ORDER ? current_sm_count() * RFG_RC_ORDER_K : 0;
  const cudaError_t e = launch_pdl(k_range_bin, dim3(range_grid() + (orderK > 0 ? 1 : 0)), dim3(256), s, m, fa, orderK);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_raycast_tiles(const DevMap& m, const FrameArgs& fa, float2* range, float4* raycast, float4* points,
                                 float4* normals, cudaStream_t s) {
  const int tx = (fa.w + kRangeTile - 1) / kRangeTile, ty = (fa.h + kRangeTile - 1) / kRangeTile;
  if (tx != m.binTilesX || ty > m.binTilesY || !raycast) return cudaErrorInvalidValue;
  if (RFG_RC_ORDER)  // the CTAs take the tiles in the order k_range_bin's extra CTA wrote
  {
    const cudaError_t e = launch_pdl(k_raycast_tiles, dim3(tx * ty), dim3(kRangeTile * kRangeTile), s, m, fa, range,
                                     raycast, points, normals, 1);
    if (e != cudaSuccess) return e;
  }
  else
    k_raycast_tiles<<<dim3(tx, ty), kRangeTile * kRangeTile, 0, s>>>(m, fa, range, raycast, points, normals, 0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_icp_maps(const DevMap& m, const FrameArgs& fa, const float2* range, float4* raycast,
                            float4* points, float4* normals, cudaStream_t s) {
  if (!raycast) return cudaErrorInvalidValue;  // the normals pass reads the hits
  dim3 g((fa.w + 15) / 16, (fa.h + 7) / 8);
#ifdef RFG_RC_SPLIT
  k_raycast_icp<<<g, 128, 0, s>>>(m, fa, range, raycast, points);
  k_raycast_normals<<<g, 128, 0, s>>>(m, fa, raycast, normals);
  count_launch(2);
#else
  k_raycast_maps<<<g, 128, 0, s>>>(m, fa, range, raycast, points, normals);
  count_launch(1);
#endif
  return cudaGetLastError();
}

cudaError_t launch_icp_maps_list(const DevMap& m, const FrameArgs& fa, const float2* range, const int* list,
                                 const int* count, int maxCount, float4* raycast, float4* points, float4* normals,
                                 cudaStream_t s) {
  const int g = (maxCount + 127) / 128;
  if (g == 0) return cudaSuccess;
  k_raycast_list<<<g, 128, 0, s>>>(m, fa, range, list, count, raycast, points);
  k_normals_list<<<g, 128, 0, s>>>(m, list, count, raycast, normals);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_forward_project(int hasRaycast, float4* raycast, float4* points, float4* normals,
                                   const float* pose34, int w, int h, float fx, float fy, float cx, float cy,
                                   float vs, float4* prev, unsigned long long* keys, int2* tileCounts,
                                   int2* tilePrefix, int* list, int* count, cudaStream_t s) {
  const int n = w * h;
  if (!hasRaycast) {
    k_iota_count<<<(n + 255) / 256, 256, 0, s>>>(list, n, count);
    count_launch();
    return cudaGetLastError();
  }
  Pose12 p;
  for (int i = 0; i < 12; ++i) p.v[i] = pose34[i];
  const int nTiles = (n + kTile - 1) / kTile;
  k_fwd_init<<<(n + 255) / 256, 256, 0, s>>>(raycast, prev, keys, n);
  k_fwd_scatter<<<(n + 255) / 256, 256, 0, s>>>(prev, keys, p, w, h, fx, fy, cx, cy, vs);
  k_fwd_gather<<<nTiles, kTileThreads, 0, s>>>(prev, keys, raycast, points, normals, n, vs, tileCounts);
  k_pix_scan<<<1, 32, 0, s>>>(tileCounts, tilePrefix, nTiles, count);
  k_fwd_emit<<<nTiles, kTileThreads, 0, s>>>(raycast, n, tilePrefix, list);
  count_launch(5);
  return cudaGetLastError();
}

}  // namespace rfg

// ------------------------------------------------ multi-GPU composition
namespace rfg {

__global__ void k_compose_keys(const float4* __restrict__ points, Pose12 pose, const float* __restrict__ poseDev,
                               int rank, int n, long long* __restrict__ keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 p = points[i];
  long long k = 0x7fffffffffffffffLL;
  if (p.w > 0.f) {
    const Pose P = poseDev ? pose_from12(poseDev) : pose_from12(pose.v);
    const float z = pose_apply(P, f3{p.x, p.y, p.z}).z;  // camera depth of the hit (> 0)
    k = ((long long)(uint32_t)__float_as_int(fmaxf(z, 0.f)) << 32) | (long long)(uint32_t)rank;
  }
  keys[i] = k;
}

__global__ void k_compose_select(const long long* __restrict__ keymin, int rank, int n, float4* raycast,
                                 float4* points, float4* normals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k = keymin[i];
  const bool nobody = k == 0x7fffffffffffffffLL;
  const bool mine = !nobody && (int)(k & 0xffffffffLL) == rank;
  if (mine) return;
  const float4 inval = make_float4(0.f, 0.f, 0.f, (nobody && rank == 0) ? -1.f : 0.f);
  if (raycast) raycast[i] = inval;
  points[i] = inval;
  normals[i] = inval;
}

}  // namespace rfg

extern "C" int rfg_compose_keys(const float* points, const float pose34[12], int rank, int n, int64_t* keys,
                                void* stream) {
  if (!points || !pose34 || !keys || n < 0 || rank < 0) {
    rfg::set_error("rfg_compose_keys: invalid argument");
    return RFG_EINVAL;
  }
  rfg::Pose12 p;
  for (int i = 0; i < 12; ++i) p.v[i] = pose34[i];
  rfg::k_compose_keys<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(points), p, nullptr, rank, n, reinterpret_cast<long long*>(keys));
  rfg::count_launch();
  RFG_CK(cudaGetLastError());
  return RFG_OK;
}

extern "C" int rfg_compose_keys_dev(const float* points, const float* poseDev, int rank, int n, int64_t* keys,
                                    void* stream) {
  if (!points || !poseDev || !keys || n < 0 || rank < 0) {
    rfg::set_error("rfg_compose_keys_dev: invalid argument");
    return RFG_EINVAL;
  }
  rfg::Pose12 p{};
  rfg::k_compose_keys<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(points), p, poseDev, rank, n, reinterpret_cast<long long*>(keys));
  rfg::count_launch();
  RFG_CK(cudaGetLastError());
  return RFG_OK;
}

extern "C" int rfg_compose_select(const int64_t* keymin, int rank, int n, float* raycast, float* points,
                                  float* normals, void* stream) {
  if (!keymin || !points || !normals || n < 0 || rank < 0) {
    rfg::set_error("rfg_compose_select: invalid argument");
    return RFG_EINVAL;
  }
  rfg::k_compose_select<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(keymin), rank, n, reinterpret_cast<float4*>(raycast),
      reinterpret_cast<float4*>(points), reinterpret_cast<float4*>(normals));
  rfg::count_launch();
  RFG_CK(cudaGetLastError());
  return RFG_OK;
}

#if defined(RFG_RC_STATS) || defined(RFG_RC_TIMING)
#if defined(RFG_RC_TIMING)
// debug build: the per-warp records of k_raycast_tiles (kRcWarps x 16)
extern "C" int rfg_debug_rc_warps(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, rfg::g_rc_warp, sizeof(rfg::g_rc_warp));
  if (reset) {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, rfg::g_rc_warp);
    cudaMemset(p, 0, sizeof(rfg::g_rc_warp));
  }
  return 0;
}
#endif
extern "C" int rfg_debug_rc_stats(unsigned long long* out32, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out32, rfg::g_rc_stats, sizeof(rfg::g_rc_stats));
  if (reset) {
    unsigned long long z[32] = {};
    z[24] = ~0ull;  // min start time
    cudaMemcpyToSymbol(rfg::g_rc_stats, z, sizeof(z));
  }
  return 0;
}
#endif
