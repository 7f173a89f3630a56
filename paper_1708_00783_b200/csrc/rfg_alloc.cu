// rfg_alloc.cu — voxel-block hash allocation and visible-list construction
// (FusionEngine::allocate_from_depth, proj/src/fusion.cpp:144-235).
//
// Stage 1 (k_alloc_stage1): one thread per depth pixel walks the blocks
//   stabbed by its d±mu segment (Amanatides-Woo DDA, fusion.cpp:72-114) and
//   probes each block's bucket chain.  Found blocks are marked; missing ones
//   request allocation at the bucket or chain tail.  The serial reference
//   resolves intra-frame collisions "last writer wins" in (row-major pixel,
//   DDA ordinal) order (fusion.cpp:168-176); here every request is keyed
//   (pixel << 6 | ordinal) + 1 and an atomicMax per slot keeps the serial
//   winner; visits are first merged per distinct block inside the CTA, so
//   each chain is probed once per block and CTA.
// Stage 2 (k_req_assign, one launch; stage 1 counts each tile's requests):
//   requests are served in
//   ascending entry-index order, exactly as the serial scan (fusion.cpp:190-201):
//   a request succeeds iff it is a bucket request or among the first
//   nFreeExcess excess requests, and its rank among such candidates is below
//   nFreeBlocks.  Ranks come from a tile scan, so the VBA block and excess
//   slot each request pops are the ones the serial free stacks would pop —
//   the resulting hash table is bit-identical, not only set-identical.
// Stage 3 (k_vis_count): candidates = this frame's marks ∪ the previous
//   visible list (its visibility bytes), frustum tested (fusion.cpp:116-130),
//   appended to the list per tile; the reference's ascending order (its
//   std::sort, fusion.cpp:231) is rebuilt on export (k_vis_tilecount /
//   k_scan_tiles / k_vis_emit).
#include "rfg_common.cuh"

namespace rfg {

// Amanatides-Woo traversal (fusion.cpp:72-114).  visit(cell, ordinal) is
// called for each visited cell in order; returning false stops the walk.
// Per-axis DDA setup (fusion.cpp:87-100).
__device__ __forceinline__ void dda_axis(float d, int c, float a, int& step, float& tMax, float& tDelta) {
  if (d > 0.f) {
    step = 1;
    tMax = ((float)(c + 1) - a) / d;
    tDelta = 1.f / d;
  } else if (d < 0.f) {
    step = -1;
    tMax = ((float)c - a) / d;
    tDelta = -1.f / d;
  } else {
    step = 0;
    tMax = FLT_MAX;
    tDelta = FLT_MAX;
  }
}

// Amanatides-Woo traversal (fusion.cpp:72-114).  visit(cell, ordinal) is
// called for each visited cell in order; returning false stops the walk.
// Scalar per-axis state (no indexed arrays, so nothing lives in local memory).
template <class F>
__device__ __forceinline__ void traverse_blocks(f3 a, f3 b, F&& visit) {
  int cx = (int)floorf(a.x), cy = (int)floorf(a.y), cz = (int)floorf(a.z);
  const int ex = (int)floorf(b.x), ey = (int)floorf(b.y), ez = (int)floorf(b.z);
  int ord = 0;
  if (!visit(i3{cx, cy, cz}, ord++)) return;
  if (cx == ex && cy == ey && cz == ez) return;
  int sx, sy, sz;
  float tmx, tmy, tmz, tdx, tdy, tdz;
  dda_axis(b.x - a.x, cx, a.x, sx, tmx, tdx);
  dda_axis(b.y - a.y, cy, a.y, sy, tmy, tdy);
  dda_axis(b.z - a.z, cz, a.z, sz, tmz, tdz);
  const int maxSteps = abs(ex - cx) + abs(ey - cy) + abs(ez - cz) + 8;
  for (int i = 0; i < maxSteps; ++i) {
    // axis of the smallest tMax, ties to the lower axis (strict <, fusion.cpp:103-105)
    const bool yFirst = tmy < tmx;
    const float tm = yFirst ? tmy : tmx;
    if (tmz < tm) {
      if (tmz > 1.f) break;
      cz += sz;
      tmz += tdz;
    } else if (yFirst) {
      if (tmy > 1.f) break;
      cy += sy;
      tmy += tdy;
    } else {
      if (tmx > 1.f) break;
      cx += sx;
      tmx += tdx;
    }
    if (!visit(i3{cx, cy, cz}, ord++)) return;
    if (cx == ex && cy == ey && cz == ez) break;
  }
  if (!(cx == ex && cy == ey && cz == ez)) visit(i3{ex, ey, ez}, ord++);
}

// Segment of pixel (x, y) in block units (fusion.cpp:183-186).
__device__ __forceinline__ bool pixel_segment(const float* depth, const FrameArgs& fa, const Pose& camToWorld,
                                              int x, int y, f3* a, f3* b) {
  const float d = depth[(size_t)y * fa.w + x];
  if (d <= 0.f || d < fa.vfMin || d > fa.vfMax) return false;
  const Intr in{fa.w, fa.h, fa.fx, fa.fy, fa.cx, fa.cy};
  const float invBlock = 1.f / (fa.voxelSize * (float)kBlock);
  const f3 nearP = pose_apply(camToWorld, backproject(in, (float)x, (float)y, d - fa.mu));
  const f3 farP = pose_apply(camToWorld, backproject(in, (float)x, (float)y, d + fa.mu));
  *a = f3{nearP.x * invBlock, nearP.y * invBlock, nearP.z * invBlock};
  *b = f3{farP.x * invBlock, farP.y * invBlock, farP.z * invBlock};
  return true;
}

// Shard filter: block kept on `rank` if any block of its 3x3x3
// neighbourhood is owned by it (owner = hash of the super-tile mod world).
__device__ __forceinline__ bool shard_keeps(const DevMap& m, i3 b) {
  if (m.world <= 1) return true;
  const int s = m.tileShift;
  // distinct super-tiles touched by b-1..b+1 per axis
  const int x0 = (b.x - 1) >> s, x1 = (b.x + 1) >> s;
  const int y0 = (b.y - 1) >> s, y1 = (b.y + 1) >> s;
  const int z0 = (b.z - 1) >> s, z1 = (b.z + 1) >> s;
  for (int tz = z0; tz <= z1; ++tz)
    for (int ty = y0; ty <= y1; ++ty)
      for (int tx = x0; tx <= x1; ++tx)
        if ((int)(hash_index(tx, ty, tz, 0xFFFFFFFFu) % (uint32_t)m.world) == m.rank) return true;
  return false;
}

// ------------------------------------------------------------- stage 1
// markBlock (fusion.cpp:155-177) for one block and the largest request key
// any of its visits carries: mark it if the chain holds it, otherwise
// request it at the bucket / chain tail (serial last writer = max key).
__device__ __forceinline__ void mark_or_request(const DevMap& m, i3 cell, uint32_t key) {
  int idx = (int)hash_index(cell.x, cell.y, cell.z, m.buckets - 1);
  int4 e = ld_entry(m.entries, idx);
  if (entry_allocated(e)) {
    const int xy = pack_xy(cell);
    for (;;) {
      if (e.x == xy && e.y == cell.z) {
        const uint8_t v = e.w >= 0 ? 1 : 2;
        m.marked[idx] = v;  // idempotent: stored without reading the byte first (the probe ends at the entry)
        return;
      }
      if (e.z < 1) break;
      idx = (int)m.buckets + e.z - 1;
      e = ld_entry(m.entries, idx);
    }
  }
  // (no read of the slot first: the atomic's return value is the only round trip)
  if (atomicMax(&m.reqKey[idx], key) == 0u) {
    // the slot's first request this frame: count it for stage 2 (per
    // kTile-entry tile: requests, and those that extend a chain)
    int2* tc = m.tileCounts + idx / kTile;
    atomicAdd(&tc->x, 1);
    if (entry_allocated(e)) atomicAdd(&tc->y, 1);
  }
}

// The pixels of a CTA (a 32x8 tile) stab a handful of distinct blocks many
// times over (a 4 cm block covers ~15x15 pixels at 1.4 m).  Marks are
// idempotent and a request slot keeps only the maximum key, so the visits
// are first merged per distinct block in a shared-memory table (block ->
// max key over the CTA's visits), and the hash chain is probed once per
// distinct block instead of once per visit.  A visit that finds the table
// full takes the direct path; the outcome is the same either way.
constexpr int kCellSlots = 1024;  // power of two; ~30-90 distinct blocks per CTA at C1
// A CTA covers a 32 x kStage1Rows pixel tile (8 rows per pass): 640x480 is
// 600 CTAs, one wave at 5 CTAs per SM (740 slots), instead of 1.35 waves
// of 32x8 tiles.
constexpr int kStage1Rows = 16;
#ifndef RFG_ALLOC_MINB
#define RFG_ALLOC_MINB 5  // stage-1 CTAs per SM (640x480: 600 CTAs in one wave)
#endif

__global__ void __launch_bounds__(256, RFG_ALLOC_MINB) k_alloc_stage1(DevMap m, const float* __restrict__ depth, FrameArgs fa) {
  pdl_wait();  // the pose (the tracker) and the depth
  __shared__ unsigned long long sCell[kCellSlots];  // (x | y << 16 | z << 32 | 1 << 48), 0 = empty
  __shared__ uint32_t sKey[kCellSlots];
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    // stage-2 / stage-3 bookkeeping of this frame (no stage-1 CTA reads it)
    MapState* st = m.state;
    st->snapFreeBlocks = st->nFreeBlocks;
    st->snapFreeExcess = st->nFreeExcess;
    st->succ = 0;
    st->succType2 = 0;
    st->nVisible = 0;  // stage 3 appends to the visible list
  }
  for (int i = threadIdx.x; i < kCellSlots; i += blockDim.x) {
    sCell[i] = 0ull;
    sKey[i] = 0u;
  }
  __syncthreads();
  const Pose camToWorld = pose_inverse(frame_pose(fa));
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
#pragma unroll 1
  for (int row = 0; row < kStage1Rows; row += 8) {
    const int y = blockIdx.y * kStage1Rows + row + (threadIdx.x >> 5);
    const bool inside = x < fa.w && y < fa.h;
    f3 a, b;
    const bool active = inside && pixel_segment(depth, fa, camToWorld, x, y, &a, &b);
    if (active) {
      const uint32_t pixKey = (uint32_t)(y * fa.w + x) << 6;
      traverse_blocks(a, b, [&](i3 cell, int ord) -> bool {
        if (ord >= 64) {
          atomicOr(&m.state->error, 1 << 1);  // ordinal bound (RFG_ERANGE)
          return false;
        }
        if (!shard_keeps(m, cell)) return true;
        if (!in_i16(cell)) {
          atomicOr(&m.state->error, 1 << 0);  // coordinate outside the int16 entry layout
          return true;
        }
        const uint32_t key = (pixKey | (uint32_t)ord) + 1u;
        const unsigned long long packed = (unsigned long long)(uint16_t)cell.x |
                                          ((unsigned long long)(uint16_t)cell.y << 16) |
                                          ((unsigned long long)(uint16_t)cell.z << 32) | (1ull << 48);
        int h = (int)(hash_index(cell.x, cell.y, cell.z, kCellSlots - 1));
  #pragma unroll 1
        for (int probe = 0; probe < 32; ++probe) {
          const unsigned long long old = atomicCAS(&sCell[h], 0ull, packed);
          if (old == 0ull) {
            // first visit of this block in the CTA: start pulling its bucket
            // entry into L2 now, so the probe after the DDA phase hits it
            const int4* bucket = m.entries + hash_index(cell.x, cell.y, cell.z, m.buckets - 1);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(bucket));
          }
          if (old == 0ull || old == packed) {
            atomicMax(&sKey[h], key);
            return true;
          }
          h = (h + 1) & (kCellSlots - 1);
        }
        mark_or_request(m, cell, key);  // table full: direct path
        return true;
      });
    }
  }
  __syncthreads();
  // compact the occupied slots first, so the chain probes are spread one per
  // thread instead of trailing on the threads whose slots happen to be full
  __shared__ int sList[kCellSlots];
  __shared__ int nList;
  if (threadIdx.x == 0) nList = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < kCellSlots; i += blockDim.x)
    if (sCell[i]) sList[atomicAdd(&nList, 1)] = i;
  __syncthreads();
  for (int k = threadIdx.x; k < nList; k += blockDim.x) {
    const int i = sList[k];
    const unsigned long long c = sCell[i];
    const i3 cell{(int)(int16_t)(c & 0xFFFFu), (int)(int16_t)((c >> 16) & 0xFFFFu), (int)(int16_t)((c >> 32) & 0xFFFFu)};
    mark_or_request(m, cell, sKey[i]);
  }
  pdl_trigger();
}

// Recompute the block a request key refers to (pixel, DDA ordinal).
__device__ __forceinline__ i3 decode_request(uint32_t key, const float* depth, const FrameArgs& fa,
                                             const Pose& camToWorld) {
  const uint32_t k = key - 1u;
  const int pixel = (int)(k >> 6), ord = (int)(k & 63u);
  const int x = pixel % fa.w, y = pixel / fa.w;
  f3 a, b;
  i3 out{0, 0, 0};
  if (!pixel_segment(depth, fa, camToWorld, x, y, &a, &b)) return out;
  traverse_blocks(a, b, [&](i3 cell, int o) -> bool {
    if (o == ord) {
      out = cell;
      return false;
    }
    return true;
  });
  return out;
}

// ------------------------------------------------------- block scan util
template <int NT>
__device__ __forceinline__ int2 block_exclusive_scan2(int2 v, int2* total) {
  __shared__ int2 warpSums[NT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int2 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int a = __shfl_up_sync(0xffffffffu, inc.x, o);
    int b = __shfl_up_sync(0xffffffffu, inc.y, o);
    if (lane >= o) {
      inc.x += a;
      inc.y += b;
    }
  }
  if (lane == 31) warpSums[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int2 s = lane < NT / 32 ? warpSums[lane] : make_int2(0, 0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(0xffffffffu, s.x, o);
      int b = __shfl_up_sync(0xffffffffu, s.y, o);
      if (lane >= o) {
        s.x += a;
        s.y += b;
      }
    }
    if (lane < NT / 32) warpSums[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  int2 base = wid > 0 ? warpSums[wid - 1] : make_int2(0, 0);
  *total = warpSums[NT / 32 - 1];
  __syncthreads();
  return make_int2(base.x + inc.x - v.x, base.y + inc.y - v.y);
}

// Exclusive scan of per-tile counts (single CTA).
__global__ void __launch_bounds__(1024) k_scan_tiles(int2* counts, int2* prefix, int n, MapState* st, int mode) {
  const int per = (n + 1023) / 1024;
  const int lo = threadIdx.x * per;
  int2 sum = make_int2(0, 0);
  for (int i = lo; i < min(n, lo + per); ++i) {
    sum.x += counts[i].x;
    sum.y += counts[i].y;
  }
  int2 total;
  int2 ex = block_exclusive_scan2<1024>(sum, &total);
  for (int i = lo; i < min(n, lo + per); ++i) {
    prefix[i] = ex;
    ex.x += counts[i].x;
    ex.y += counts[i].y;
  }
  if (threadIdx.x == 0) {
    prefix[n] = total;
    if (mode == 1) {
      st->nVisible = total.x;
      st->stats[3] = total.x;
    }
  }
}

// --------------------------------------------------------------- stage 2
// Tiles of kTile = 1024 hash entries, 4 consecutive entries per thread (one
// 16-byte load of keys, one 4-byte load of flag bytes), so a tile's threads
// cover it in ascending entry order and a CTA scan gives the serial ranks.

// (The per-tile request counts come from stage 1: mark_or_request counts a
// slot's first request.)

// Exclusive scan of v over the CTA, with the CTA totals of v and of r.
template <int NT>
__device__ __forceinline__ int2 block_scan2_with_sum2(int2 v, int2 r, int2* total, int2* rsum) {
  __shared__ int4 warpSums[NT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int2 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, inc.x, o);
    const int b = __shfl_up_sync(0xffffffffu, inc.y, o);
    if (lane >= o) {
      inc.x += a;
      inc.y += b;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r.x += __shfl_xor_sync(0xffffffffu, r.x, o);
    r.y += __shfl_xor_sync(0xffffffffu, r.y, o);
  }
  if (lane == 31) warpSums[wid] = make_int4(inc.x, inc.y, r.x, r.y);
  __syncthreads();
  int4 base = make_int4(0, 0, 0, 0), all = make_int4(0, 0, 0, 0);
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    const int4 s = warpSums[w];
    if (w < wid) {
      base.x += s.x;
      base.y += s.y;
    }
    all.x += s.x;
    all.y += s.y;
    all.z += s.z;
    all.w += s.w;
  }
  *total = make_int2(all.x, all.y);
  *rsum = make_int2(all.z, all.w);
  return make_int2(base.x + inc.x - v.x, base.y + inc.y - v.y);
}

// Serve requests in ascending index order with serial-equivalent ranks.
// The kernel is a chain of dependent memory round trips, so the loads that
// do not depend on each other are issued together up front: the tile's keys,
// its own stage-1 request count (tiles without requests leave at once, with
// no barrier), the counts of the tiles before it and the free-stack sizes.
// One scan then gives the in-tile ranks and the prefix; the free-stack pops
// are loaded before the request's block is re-derived by the DDA.
__global__ void __launch_bounds__(kTileThreads) k_req_assign(DevMap m, const float* __restrict__ depth, FrameArgs fa) {
  pdl_wait();
  const uint32_t base = blockIdx.x * kTile + threadIdx.x * 4;
  const bool last = blockIdx.x == gridDim.x - 1;
  const uint4 k4 = __ldcg(reinterpret_cast<const uint4*>(m.reqKey + base));
  const int2 own = __ldcg(m.tileCounts + blockIdx.x);  // this tile's requests (stage 1)
  int nB, nE;
  asm volatile("ld.global.cg.v2.s32 {%0, %1}, [%2];" : "=r"(nB), "=r"(nE) : "l"(&m.state->snapFreeBlocks));
  // (volatile loads: issued here, not sunk below the early exit; four tiles
  // per thread per batch, so a map of up to 1,024 tiles is one round trip)
  int2 pre = make_int2(0, 0);
  for (int i0 = threadIdx.x; i0 < (int)blockIdx.x; i0 += 4 * kTileThreads) {
    int2 c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q * kTileThreads;
      c[q] = make_int2(0, 0);
      if (i < (int)blockIdx.x)
        asm volatile("ld.global.cg.v2.s32 {%0, %1}, [%2];" : "=r"(c[q].x), "=r"(c[q].y) : "l"(m.tileCounts + i));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      pre.x += c[q].x;
      pre.y += c[q].y;
    }
  }
  // (nB in the exit test keeps its load ahead of the exit, beside the others;
  // a free-stack size is never negative)
  if (own.x == 0 && !last && nB >= 0) return;  // (CTA-uniform) most tiles hold no request
  const Pose camToWorld = pose_inverse(frame_pose(fa));  // (loaded beside the entries, before the scan)
  const uint32_t keys[4] = {k4.x, k4.y, k4.z, k4.w};
  int n = 0, n2 = 0;
  uint32_t isT2 = 0;
  int keep[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    keep[j] = 0;
    if (keys[j]) {
      ++n;
      const int4 e = ld_entry(m.entries, base + j);
      keep[j] = e.z;
      if (entry_allocated(e)) {
        ++n2;
        isT2 |= 1u << j;
      }
    }
  }
  int2 total, tp;
  const int2 ex = block_scan2_with_sum2<kTileThreads>(make_int2(n, n2), pre, &total, &tp);
  if (last && threadIdx.x == 0) m.state->nRequests = tp.x + total.x;
  if (n == 0) return;
  int before = tp.x + ex.x, before2 = tp.y + ex.y;
  int succ = 0, succ2 = 0;
#pragma unroll 1
  for (int j = 0; j < 4; ++j) {
    const uint32_t key = j == 0 ? keys[0] : (j == 1 ? keys[1] : (j == 2 ? keys[2] : keys[3]));
    if (!key) continue;
    const int idx = (int)(base + j);
    const bool t2 = (isT2 >> j) & 1u;
    const int before1 = before - before2;
    const int r2 = before2;
    const bool cand = !t2 || r2 < nE;
    const int rb = before1 + min(before2, nE);
    m.reqKey[idx] = 0u;  // consume the request slot
    ++before;
    if (t2) ++before2;
    if (!cand || rb >= nB) continue;
    const int blockPtr = __ldcg(m.freeBlocks + (nB - 1 - rb));
    const int excessIdx = t2 ? __ldcg(m.freeExcess + (nE - 1 - r2)) : 0;
    const i3 p = decode_request(key, depth, fa, camToWorld);
    if (!t2) {
      // free bucket slot (voxel_block_map.cpp:96-104)
      const int kz = j == 0 ? keep[0] : (j == 1 ? keep[1] : (j == 2 ? keep[2] : keep[3]));
      m.entries[idx] = make_entry(p.x, p.y, p.z, kz, blockPtr);
      m.marked[idx] = 1;
    } else {
      // chain tail: link a fresh excess slot (voxel_block_map.cpp:84-93)
      const int newIdx = (int)m.buckets + excessIdx;
      m.entries[newIdx] = make_entry(p.x, p.y, p.z, 0, blockPtr);
      m.entries[idx].z = excessIdx + 1;
      m.marked[newIdx] = 1;
      ++succ2;
    }
    ++succ;
  }
  if (succ) atomicAdd(&m.state->succ, succ);
  if (succ2) atomicAdd(&m.state->succType2, succ2);
  pdl_trigger();
}

// --------------------------------------------------------------- stage 3
// proj/src/fusion.cpp:116-130 (marginPx: the swap-in boundary band)
__device__ __forceinline__ bool block_in_frustum(int bx, int by, int bz, const Pose& pose, const FrameArgs& fa,
                                                 float marginPx = 0.f) {
  const float bs = fa.voxelSize * (float)kBlock;
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {
    const f3 corner{((float)bx + (float)(c & 1)) * bs, ((float)by + (float)((c >> 1) & 1)) * bs,
                    ((float)bz + (float)((c >> 2) & 1)) * bs};
    const f3 pc = pose_apply(pose, corner);
    if (pc.z < fa.vfMin || pc.z > fa.vfMax) continue;
    const float px = fa.fx * pc.x / pc.z + fa.cx;
    const float py = fa.fy * pc.y / pc.z + fa.cy;
    if (px >= -marginPx && py >= -marginPx && px <= (float)(fa.w - 1) + marginPx &&
        py <= (float)(fa.h - 1) + marginPx)
      return true;
  }
  return false;
}

// Candidates (this frame's marks | previous visibility bytes) of the tile are
// queued in shared memory and frustum-tested one per thread, so the tests are
// spread over the CTA whatever the hash distribution.
__global__ void __launch_bounds__(kTileThreads) k_vis_count(DevMap m, FrameArgs fa) {
  __shared__ int queue[kTile];
  __shared__ int vis[kTile];
  __shared__ int nq, nvis, listBase;
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // finalise stage 2 (all k_req_assign CTAs have completed)
    MapState* st = m.state;
    st->nFreeBlocks = st->snapFreeBlocks - st->succ;
    st->nFreeExcess = st->snapFreeExcess - st->succType2;
    st->stats[0] = st->nRequests;
    st->stats[1] = st->succ;
    st->stats[2] = st->nRequests - st->succ;
  }
  if (threadIdx.x == 0) {
    nq = 0;
    nvis = 0;
  }
  __syncthreads();
  const uint32_t base = blockIdx.x * kTile + threadIdx.x * 4;
  uint32_t* mp = reinterpret_cast<uint32_t*>(m.marked + base);
  uint32_t* vp = reinterpret_cast<uint32_t*>(m.visibility + base);
  const uint32_t mk = *mp, vk = *vp;
  const Pose pose = frame_pose(fa);  // (loaded with the bytes, not after the barrier)
  const uint32_t cand = mk | vk;
  if (cand) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((cand >> (8 * j)) & 0xFFu) queue[atomicAdd(&nq, 1)] = (int)(base + j);
    *vp = 0u;  // rewritten below for the candidates that stay visible
  }
  if (mk) *mp = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < nq; i += kTileThreads) {
    const int idx = queue[i];
    const int4 e = ld_entry(m.entries, idx);
    if (!entry_allocated(e)) continue;
    // fusion.cpp:219-229: visible (1), visible but swapped out (2), or with
    // swapping enabled inside the swap-in margin (3, kBoundary)
    uint8_t type = 0;
    if (block_in_frustum(entry_x(e), entry_y(e), entry_z(e), pose, fa))
      type = e.w >= 0 ? 1 : 2;
    else if (fa.swapping && block_in_frustum(entry_x(e), entry_y(e), entry_z(e), pose, fa, fa.swapMargin))
      type = 3;
    if (type) {
      m.visibility[idx] = type;
      vis[atomicAdd(&nvis, 1)] = idx;
    }
  }
  __syncthreads();
  // append this tile's visible entries to the list (one global atomic per
  // CTA); the in-frame consumers (integration, expected ranges) do not
  // depend on the order, and rfg_export_visible regenerates the reference's
  // ascending order (fusion.cpp:231) from the visibility bytes
  if (threadIdx.x == 0) {
    listBase = nvis ? atomicAdd(&m.state->nVisible, nvis) : 0;
    m.tileCounts[blockIdx.x] = make_int2(0, 0);  // stage 2 is done with it: ready for the next stage 1
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nvis; i += kTileThreads) m.visibleList[listBase + i] = vis[i];
  pdl_trigger();
}

// Per-tile count of visible entries (visibility bytes), for regenerating the
// ascending visible list (k_scan_tiles mode 1 + k_vis_emit).
__global__ void __launch_bounds__(kTileThreads) k_vis_tilecount(DevMap m) {
  const uint32_t base = blockIdx.x * kTile + threadIdx.x * 4;
  const uint32_t w = *reinterpret_cast<const uint32_t*>(m.visibility + base);
  int n = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) n += ((w >> (8 * j)) & 0xFFu) ? 1 : 0;
  int2 total;
  block_exclusive_scan2<kTileThreads>(make_int2(n, 0), &total);
  if (threadIdx.x == 0) m.tileCounts[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kTileThreads) k_vis_emit(DevMap m) {
  const uint32_t base = blockIdx.x * kTile + threadIdx.x * 4;
  const uint32_t w = *reinterpret_cast<const uint32_t*>(m.visibility + base);
  int n = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) n += ((w >> (8 * j)) & 0xFFu) ? 1 : 0;
  int2 total;
  const int2 ex = block_exclusive_scan2<kTileThreads>(make_int2(n, 0), &total);
  if (threadIdx.x == 0) m.tileCounts[blockIdx.x] = make_int2(0, 0);  // zero again for the next stage 1
  if (n == 0) return;
  int o = m.tilePrefix[blockIdx.x].x + ex.x;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if ((w >> (8 * j)) & 0xFFu) m.visibleList[o++] = (int)(base + j);
}

cudaError_t launch_allocate(const DevMap& m, const float* depth, const FrameArgs& fa, cudaStream_t s) {
  dim3 g1((fa.w + 31) / 32, (fa.h + kStage1Rows - 1) / kStage1Rows);
  cudaError_t e = launch_pdl(k_alloc_stage1, g1, dim3(256), s, m, depth, fa);
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_req_assign, dim3(m.nTiles), dim3(kTileThreads), s, m, depth, fa);
  if (e != cudaSuccess) return e;
  if ((e = launch_pdl(k_vis_count, dim3(m.nTiles), dim3(kTileThreads), s, m, fa)) != cudaSuccess) return e;
  count_launch(3);
  return cudaGetLastError();
}

// The visible list in the reference's ascending entry order (fusion.cpp:231),
// rebuilt from the visibility bytes (the frame's kernels append it unordered).
cudaError_t launch_sort_visible(const DevMap& m, cudaStream_t s) {
  k_vis_tilecount<<<m.nTiles, kTileThreads, 0, s>>>(m);
  k_scan_tiles<<<1, 1024, 0, s>>>(m.tileCounts, m.tilePrefix, m.nTiles, m.state, 1);
  k_vis_emit<<<m.nTiles, kTileThreads, 0, s>>>(m);
  count_launch(3);
  return cudaGetLastError();
}

}  // namespace rfg
