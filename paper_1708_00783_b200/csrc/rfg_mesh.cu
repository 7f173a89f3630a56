// rfg_mesh.cu — marching-cubes mesh extraction (extract_mesh,
// proj/src/meshing.cpp:144-217).
//
// Output is identical to the serial reference — same vertices in the same
// order, same triangles in the same order — not merely the same surface:
//   1. k_mc_count: one warp per hash entry (ascending index, the reference's
//      outer loop); the block's 8^3 voxels plus the +1 halo from its seven
//      upper neighbours are staged in shared memory (9^3 words), every cell
//      (lz, ly, lx order) is classified (all 8 corners allocated and
//      observed, mask of sdf < 0) and the per-entry triangle count is
//      reduced;
//   2. exclusive scan over entries -> each entry's first triangle;
//   3. k_mc_emit: the same classification again; lane prefix + entry offset
//      place every triangle of the serial stream; each of its 3 corners
//      writes the lattice-edge key (meshing.cpp:146-153) and the vertex the
//      reference would create on that edge;
//   4. vertex numbering: the reference numbers a vertex when its edge first
//      appears in the triangle stream (std::unordered_map::find/emplace,
//      meshing.cpp:196-208).  A device hash keeps, per edge key, the minimum
//      stream position (atomicMin); positions that are their key's minimum
//      are first occurrences, and an exclusive scan over those flags gives
//      exactly the reference's vertex ids.
// The triangulation table is built on the host by the reference's rule
// (meshing.cpp:27-118): crossed edges paired per face (ambiguous faces pair
// the edges around each inside corner), cycles walked, oriented by their
// Newell normal against the inside->outside direction and fanned.
#include <mutex>

#include "rfg_common.cuh"

namespace rfg {

constexpr int kMcMaxTris = 16;
__constant__ unsigned char c_mcCount[256];
__constant__ unsigned char c_mcTris[256][kMcMaxTris][3];

// corner c = (x, y, z) offsets; edges as corner pairs; faces as corner loops
static const int kMcCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                    {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
static const int kMcEdge[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                   {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
static const int kMcFace[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};
__constant__ int c_mcCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                     {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
__constant__ int c_mcEdge[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                    {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};

struct McTable {
  int count[256];
  unsigned char tri[256][kMcMaxTris][3];
};

static int mc_edge_of(int a, int b) {
  for (int e = 0; e < 12; ++e)
    if ((kMcEdge[e][0] == a && kMcEdge[e][1] == b) || (kMcEdge[e][0] == b && kMcEdge[e][1] == a)) return e;
  return -1;
}

static void mc_build(McTable& t) {
  for (int mask = 0; mask < 256; ++mask) {
    auto in = [&](int c) { return (mask >> c) & 1; };
    auto crossed = [&](int e) { return in(kMcEdge[e][0]) != in(kMcEdge[e][1]); };
    int nb[12][2];
    for (auto& p : nb) p[0] = p[1] = -1;
    auto join = [&](int a, int b) {
      (nb[a][0] < 0 ? nb[a][0] : nb[a][1]) = b;
      (nb[b][0] < 0 ? nb[b][0] : nb[b][1]) = a;
    };
    for (const auto& f : kMcFace) {
      int ce[4], n = 0;
      for (int i = 0; i < 4; ++i) {
        const int e = mc_edge_of(f[i], f[(i + 1) % 4]);
        if (crossed(e)) ce[n++] = e;
      }
      if (n == 2) {
        join(ce[0], ce[1]);
      } else if (n == 4) {  // ambiguous face: pair the two edges at each inside corner
        for (int i = 0; i < 4; ++i)
          if (in(f[i])) join(mc_edge_of(f[(i + 3) % 4], f[i]), mc_edge_of(f[i], f[(i + 1) % 4]));
      }
    }
    t.count[mask] = 0;
    bool done[12] = {};
    for (int s = 0; s < 12; ++s) {
      if (!crossed(s) || done[s]) continue;
      int cyc[12], len = 0, cur = s, prev = -1;
      for (;;) {
        cyc[len++] = cur;
        done[cur] = true;
        const int nxt = nb[cur][0] != prev ? nb[cur][0] : nb[cur][1];
        prev = cur;
        cur = nxt;
        if (cur == s) break;
      }
      if (len < 3) continue;
      // Newell normal of the edge-midpoint polygon vs the inside->outside
      // direction (all values are halves: exact in float)
      float nw[3] = {0, 0, 0}, dir[3] = {0, 0, 0};
      for (int i = 0; i < len; ++i) {
        float a[3], b[3];
        for (int k = 0; k < 3; ++k) {
          a[k] = 0.5f * (float)(kMcCorner[kMcEdge[cyc[i]][0]][k] + kMcCorner[kMcEdge[cyc[i]][1]][k]);
          b[k] = 0.5f * (float)(kMcCorner[kMcEdge[cyc[(i + 1) % len]][0]][k] +
                                kMcCorner[kMcEdge[cyc[(i + 1) % len]][1]][k]);
        }
        nw[0] += a[1] * b[2] - a[2] * b[1];
        nw[1] += a[2] * b[0] - a[0] * b[2];
        nw[2] += a[0] * b[1] - a[1] * b[0];
        const int c0 = kMcEdge[cyc[i]][0], c1 = kMcEdge[cyc[i]][1];
        const int ci = in(c0) ? c0 : c1, co = in(c0) ? c1 : c0;
        for (int k = 0; k < 3; ++k) dir[k] += (float)(kMcCorner[co][k] - kMcCorner[ci][k]);
      }
      const float d2 = dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2];
      if (d2 > 1e-12f && nw[0] * dir[0] + nw[1] * dir[1] + nw[2] * dir[2] < 0.f)
        for (int i = 0; i < len / 2; ++i) {
          const int x = cyc[i];
          cyc[i] = cyc[len - 1 - i];
          cyc[len - 1 - i] = x;
        }
      for (int i = 1; i + 1 < len; ++i) {
        const int k = t.count[mask]++;
        t.tri[mask][k][0] = (unsigned char)cyc[0];
        t.tri[mask][k][1] = (unsigned char)cyc[i];
        t.tri[mask][k][2] = (unsigned char)cyc[i + 1];
      }
    }
  }
}

static const McTable& mc_table() {
  static McTable t;
  static std::once_flag once;
  std::call_once(once, [] { mc_build(t); });
  return t;
}

static cudaError_t mc_upload() {
  // per device: the constant tables are per-module, uploaded on first use
  static int uploaded[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && uploaded[dev]) return cudaSuccess;
  const McTable& t = mc_table();
  unsigned char cnt[256];
  for (int i = 0; i < 256; ++i) cnt[i] = (unsigned char)t.count[i];
  cudaError_t e = cudaMemcpyToSymbol(c_mcCount, cnt, sizeof(cnt));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mcTris, t.tri, sizeof(t.tri));
  if (e == cudaSuccess && dev < 64) uploaded[dev] = 1;
  return e;
}

int mc_table_export(int* counts256, int* tris256x16x3) {
  const McTable& t = mc_table();
  for (int m = 0; m < 256; ++m) {
    counts256[m] = t.count[m];
    for (int k = 0; k < kMcMaxTris; ++k)
      for (int j = 0; j < 3; ++j) tris256x16x3[(m * kMcMaxTris + k) * 3 + j] = k < t.count[m] ? t.tri[m][k][j] : -1;
  }
  return 0;
}

// ------------------------------------------------------------------ device
constexpr int kMcWarps = 4;       // warps (entries) per CTA
constexpr int kMcG = 9;           // staged grid edge (8 + 1 halo)
constexpr uint32_t kMcNone = 0xFFFFFFFFu;  // voxel of an absent block

// Stage the entry's block + upper halo; returns false if the entry holds no
// in-memory block (meshing.cpp:161 inMemory).
__device__ bool mc_stage(const DevMap& m, int idx, uint32_t* grid, int lane, int3* origin) {
  const int4 e = ld_entry(m.entries, idx);
  if (e.w < 0) return false;
  const int bx = entry_x(e), by = entry_y(e), bz = entry_z(e);
  int p = -1;
  if (lane == 0) p = e.w;
  if (lane >= 1 && lane < 8) {
    const i3 q{bx + (lane & 1), by + ((lane >> 1) & 1), bz + ((lane >> 2) & 1)};
    int4 f;
    if (find_entry(m, q, &f) >= 0) p = f.w >= 0 ? f.w : -1;
  }
  int nb[8];
#pragma unroll
  for (int d = 0; d < 8; ++d) nb[d] = __shfl_sync(0xffffffffu, p, d);
  for (int t = lane; t < kMcG * kMcG * kMcG; t += 32) {
    const int x = t % kMcG, y = (t / kMcG) % kMcG, z = t / (kMcG * kMcG);
    const int d = (x >> 3) | ((y >> 3) << 1) | ((z >> 3) << 2);
    const int ptr = nb[d];
    grid[t] = ptr >= 0 ? __ldg(m.vbaDepth + (size_t)ptr * kBlock3 + ((x & 7) | ((y & 7) << 3) | ((z & 7) << 6)))
                       : kMcNone;
  }
  __syncwarp();
  *origin = make_int3(bx * kBlock, by * kBlock, bz * kBlock);
  return true;
}

// classify cell (lx, ly, lz): mask, or -1 if any corner is unobserved
// (absent block or w_depth == 0, meshing.cpp:166-176)
__device__ __forceinline__ int mc_mask(const uint32_t* grid, int lx, int ly, int lz) {
  int mask = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t w = grid[(lz + c_mcCorner[c][2]) * kMcG * kMcG + (ly + c_mcCorner[c][1]) * kMcG +
                            (lx + c_mcCorner[c][0])];
    if (w == kMcNone || vox_w(w) == 0) return -1;
    if (vox_sdf(w) < 0) mask |= 1 << c;  // logicalSdf < 0 <=> stored sdf < 0
  }
  return mask;
}

__global__ void __launch_bounds__(kMcWarps * 32) k_mc_count(DevMap m, int nEntries, int* counts) {
  __shared__ uint32_t grid[kMcWarps][kMcG * kMcG * kMcG];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int idx = blockIdx.x * kMcWarps + w; idx < nEntries; idx += gridDim.x * kMcWarps) {
    int3 o;
    int n = 0;
    if (mc_stage(m, idx, grid[w], lane, &o)) {
      for (int c = lane * 16; c < lane * 16 + 16; ++c) {
        const int mask = mc_mask(grid[w], c & 7, (c >> 3) & 7, c >> 6);
        if (mask > 0) n += c_mcCount[mask];
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) n += __shfl_down_sync(0xffffffffu, n, off);
    if (lane == 0) counts[idx] = n;
    __syncwarp();
  }
}

// meshing.cpp:146-153
__device__ __forceinline__ unsigned long long mc_edge_key(int x, int y, int z, int axis) {
  const long long kBias = 1 << 19;
  const unsigned long long ux = (unsigned long long)(x + kBias) & 0xFFFFFull;
  const unsigned long long uy = (unsigned long long)(y + kBias) & 0xFFFFFull;
  const unsigned long long uz = (unsigned long long)(z + kBias) & 0xFFFFFull;
  return (((ux << 20) | uy) << 20 | uz) << 2 | (unsigned long long)axis;
}

__global__ void __launch_bounds__(kMcWarps * 32) k_mc_emit(DevMap m, int nEntries, const int* __restrict__ offsets,
                                                           float vs, unsigned long long* keys, float* pos) {
  __shared__ uint32_t grid[kMcWarps][kMcG * kMcG * kMcG];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int idx = blockIdx.x * kMcWarps + w; idx < nEntries; idx += gridDim.x * kMcWarps) {
    int3 o;
    if (!mc_stage(m, idx, grid[w], lane, &o)) {
      __syncwarp();
      continue;
    }
    int masks[16], n = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = lane * 16 + j;
      masks[j] = mc_mask(grid[w], c & 7, (c >> 3) & 7, c >> 6);
      if (masks[j] > 0) n += c_mcCount[masks[j]];
    }
    int ex = n;  // warp inclusive scan -> exclusive
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, ex, off);
      if (lane >= off) ex += v;
    }
    long long t = (long long)offsets[idx] + ex - n;
#pragma unroll 1
    for (int j = 0; j < 16; ++j) {
      const int mask = masks[j];
      if (mask <= 0) continue;
      const int c = lane * 16 + j, lx = c & 7, ly = (c >> 3) & 7, lz = c >> 6;
      for (int k = 0; k < c_mcCount[mask]; ++k, ++t) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int e = c_mcTris[mask][k][q];
          int a = c_mcEdge[e][0], b = c_mcEdge[e][1];
          int ax = lx + c_mcCorner[a][0], ay = ly + c_mcCorner[a][1], az = lz + c_mcCorner[a][2];
          int bx = lx + c_mcCorner[b][0], by = ly + c_mcCorner[b][1], bz = lz + c_mcCorner[b][2];
          float fa = sdf_to_logical(vox_sdf(grid[w][az * kMcG * kMcG + ay * kMcG + ax]));
          float fb = sdf_to_logical(vox_sdf(grid[w][bz * kMcG * kMcG + by * kMcG + bx]));
          const int axis = ax != bx ? 0 : (ay != by ? 1 : 2);
          const int va = axis == 0 ? ax : (axis == 1 ? ay : az), vb = axis == 0 ? bx : (axis == 1 ? by : bz);
          if (va > vb) {  // orient the edge upward (meshing.cpp:191-194)
            int tmp = ax;
            ax = bx;
            bx = tmp;
            tmp = ay;
            ay = by;
            by = tmp;
            tmp = az;
            az = bz;
            bz = tmp;
            const float ft = fa;
            fa = fb;
            fb = ft;
          }
          const int gx = o.x + ax, gy = o.y + ay, gz = o.z + az;
          const float denom = fa - fb;
          const float tt = fabsf(denom) < 1e-12f ? 0.5f : fa / denom;
          float p[3] = {(float)gx, (float)gy, (float)gz};
          p[axis] += tt;
          const long long s = 3 * t + q;
          keys[s] = mc_edge_key(gx, gy, gz, axis);
          pos[3 * s + 0] = p[0] * vs;
          pos[3 * s + 1] = p[1] * vs;
          pos[3 * s + 2] = p[2] * vs;
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------- first occurrence
__device__ __forceinline__ unsigned int mc_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  return (unsigned int)k;
}

__global__ void k_mc_insert(const unsigned long long* __restrict__ keys, long long n, unsigned long long* hkeys,
                            unsigned int* hmin, unsigned int hmask, unsigned int* slotOf) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n; s += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[s];
    unsigned int h = mc_hash(k) & hmask;
    for (;;) {
      const unsigned long long prev = atomicCAS(&hkeys[h], ~0ull, k);
      if (prev == ~0ull || prev == k) break;
      h = (h + 1) & hmask;
    }
    atomicMin(&hmin[h], (unsigned int)s);
    slotOf[s] = h;
  }
}

__global__ void k_mc_first(const unsigned int* __restrict__ slotOf, const unsigned int* __restrict__ hmin, long long n,
                           int* flags) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n; s += (long long)gridDim.x * blockDim.x)
    flags[s] = hmin[slotOf[s]] == (unsigned int)s ? 1 : 0;
}

__global__ void k_mc_finish(const unsigned int* __restrict__ slotOf, const unsigned int* __restrict__ hmin,
                            const int* __restrict__ vid, const int* __restrict__ flags, const float* __restrict__ pos,
                            long long n, unsigned int* tris, float* verts) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n; s += (long long)gridDim.x * blockDim.x) {
    tris[s] = (unsigned int)vid[hmin[slotOf[s]]];
    if (flags[s]) {
      const int v = vid[s];
      verts[3 * (size_t)v + 0] = pos[3 * s + 0];
      verts[3 * (size_t)v + 1] = pos[3 * s + 1];
      verts[3 * (size_t)v + 2] = pos[3 * s + 2];
    }
  }
}

// ------------------------------------------------------------------- scan
// exclusive scan of n ints (tiles of 2048: per-tile sums, one CTA scans the
// tile sums, tiles add their base); total returned in *total (device)
constexpr int kScanTile = 2048;

__device__ __forceinline__ int block_scan_excl(int v, int* total) {
  __shared__ int warpSums[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warpSums[w] = x;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    int s = lane < nw ? warpSums[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, off);
      if (lane >= off) s += y;
    }
    if (lane < nw) warpSums[lane] = s;
  }
  __syncthreads();
  const int base = w > 0 ? warpSums[w - 1] : 0;
  if (total) *total = warpSums[(blockDim.x >> 5) - 1];
  const int r = base + x - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) k_scan_tile_sums(const int* __restrict__ in, long long n, int* tileSums) {
  const long long lo = (long long)blockIdx.x * kScanTile;
  int s = 0;
  for (long long i = lo + threadIdx.x; i < min(n, lo + kScanTile); i += blockDim.x) s += in[i];
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  __shared__ int ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += ws[k];
    tileSums[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_tile_bases(int* tileSums, int nTiles, int* total) {
  const int per = (nTiles + 1023) / 1024;
  const int lo = threadIdx.x * per;
  int s = 0;
  for (int i = lo; i < min(nTiles, lo + per); ++i) s += tileSums[i];
  int tot;
  int ex = block_scan_excl(s, &tot);
  for (int i = lo; i < min(nTiles, lo + per); ++i) {
    const int v = tileSums[i];
    tileSums[i] = ex;
    ex += v;
  }
  if (threadIdx.x == 0) *total = tot;
}

__global__ void __launch_bounds__(1024) k_scan_apply(const int* __restrict__ in, long long n,
                                                     const int* __restrict__ tileBase, int* out) {
  const long long lo = (long long)blockIdx.x * kScanTile;
  // each thread owns 2 consecutive elements of the tile
  const long long i0 = lo + 2 * threadIdx.x;
  const int a = i0 < n ? in[i0] : 0, b = i0 + 1 < n ? in[i0 + 1] : 0;
  const int ex = block_scan_excl(a + b, nullptr) + tileBase[blockIdx.x];
  if (i0 < n) out[i0] = ex;
  if (i0 + 1 < n) out[i0 + 1] = ex + a;
}

long long scan_tile_scratch_ints(long long n) { return (n + kScanTile - 1) / kScanTile + 2; }

cudaError_t scan_exclusive(const int* in, long long n, int* out, int* tileScratch, int* total, cudaStream_t s) {
  const int nTiles = (int)((n + kScanTile - 1) / kScanTile);
  if (nTiles == 0) return cudaMemsetAsync(total, 0, sizeof(int), s);
  k_scan_tile_sums<<<nTiles, 1024, 0, s>>>(in, n, tileScratch);
  k_scan_tile_bases<<<1, 1024, 0, s>>>(tileScratch, nTiles, total);
  k_scan_apply<<<nTiles, 1024, 0, s>>>(in, n, tileScratch, out);
  count_launch(3);
  return cudaGetLastError();
}

// --------------------------------------------------------------- driver
struct MeshBuffers {
  int* counts = nullptr;  // per entry, then exclusive offsets in place
  int* offsets = nullptr;
  int* tiles = nullptr;
  int* total = nullptr;  // device scalar
  long long cap = 0;      // corner slots
  unsigned long long* keys = nullptr;
  float* pos = nullptr;
  unsigned int* slotOf = nullptr;
  int* flags = nullptr;
  int* vid = nullptr;
  unsigned long long* hkeys = nullptr;
  unsigned int* hmin = nullptr;
  unsigned int hsize = 0;
  unsigned int* tris = nullptr;
  float* verts = nullptr;
  long long nTris = 0, nVerts = 0;
  uint32_t entriesCap = 0;
  long long tilesCap = 0;  // ints in `tiles`
};

static cudaError_t ensure_tiles(MeshBuffers* b, long long n) {
  const long long need = (n + kScanTile - 1) / kScanTile + 2;
  if (need <= b->tilesCap) return cudaSuccess;
  cudaFree(b->tiles);
  b->tiles = nullptr;
  const long long c = need + need / 2 + 64;
  cudaError_t e = cudaMalloc(&b->tiles, c * sizeof(int));
  if (e == cudaSuccess) b->tilesCap = c;
  return e;
}

void mesh_free(void* mb) {
  auto* b = static_cast<MeshBuffers*>(mb);
  if (!b) return;
  void* p[] = {b->counts, b->offsets, b->tiles, b->total, b->keys, b->pos, b->slotOf, b->flags,
               b->vid,    b->hkeys,   b->hmin,  b->tris,  b->verts};
  for (void* q : p)
    if (q) cudaFree(q);
  delete b;
}

static int grid_for(long long n, int threads) {
  const long long g = (n + threads - 1) / threads;
  const long long cap = (long long)current_sm_count() * 16;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

// Extracts the mesh into *mbp (allocated / grown as needed); synchronises.
cudaError_t mesh_extract(const DevMap& m, float vs, void** mbp, long long* nVerts, long long* nTris, cudaStream_t s) {
  cudaError_t e = mc_upload();
  if (e != cudaSuccess) return e;
  auto* b = static_cast<MeshBuffers*>(*mbp);
  if (!b) {
    b = new MeshBuffers();
    *mbp = b;
  }
  const uint32_t nE = m.total;
  if (b->entriesCap < nE) {
    cudaFree(b->counts);
    cudaFree(b->offsets);
    cudaFree(b->total);
    b->counts = b->offsets = b->total = nullptr;
    if ((e = cudaMalloc(&b->counts, nE * sizeof(int))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->offsets, nE * sizeof(int))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->total, sizeof(int))) != cudaSuccess) return e;
    b->entriesCap = nE;
  }
  const int g = 148 * 8;
  if ((e = ensure_tiles(b, nE)) != cudaSuccess) return e;
  k_mc_count<<<g, kMcWarps * 32, 0, s>>>(m, (int)nE, b->counts);
  count_launch();
  if ((e = scan_exclusive(b->counts, nE, b->offsets, b->tiles, b->total, s)) != cudaSuccess) return e;
  int hTris = 0;
  if ((e = cudaMemcpyAsync(&hTris, b->total, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  const long long nS = 3ll * hTris;
  if (nS > b->cap) {
    void* p[] = {b->keys, b->pos, b->slotOf, b->flags, b->vid, b->tris, b->verts};
    for (void* q : p)
      if (q) cudaFree(q);
    b->keys = nullptr;
    b->pos = nullptr;
    b->slotOf = nullptr;
    b->flags = b->vid = nullptr;
    b->tris = nullptr;
    b->verts = nullptr;
    const long long c = nS + nS / 4 + 1024;
    if ((e = cudaMalloc(&b->keys, c * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->pos, c * 12)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->slotOf, c * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->flags, c * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->vid, c * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->tris, c * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->verts, c * 12)) != cudaSuccess) return e;
    b->cap = c;
  }
  unsigned int hs = 1024;
  while ((long long)hs < 2 * nS) hs <<= 1;
  if (hs > b->hsize) {
    cudaFree(b->hkeys);
    cudaFree(b->hmin);
    b->hkeys = nullptr;
    b->hmin = nullptr;
    if ((e = cudaMalloc(&b->hkeys, (size_t)hs * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&b->hmin, (size_t)hs * 4)) != cudaSuccess) return e;
    b->hsize = hs;
  }
  long long nV = 0;
  if ((e = ensure_tiles(b, nS)) != cudaSuccess) return e;
  if (nS > 0) {
    k_mc_emit<<<g, kMcWarps * 32, 0, s>>>(m, (int)nE, b->offsets, vs, b->keys, b->pos);
    cudaMemsetAsync(b->hkeys, 0xFF, (size_t)hs * 8, s);
    cudaMemsetAsync(b->hmin, 0xFF, (size_t)hs * 4, s);
    k_mc_insert<<<grid_for(nS, 256), 256, 0, s>>>(b->keys, nS, b->hkeys, b->hmin, hs - 1, b->slotOf);
    k_mc_first<<<grid_for(nS, 256), 256, 0, s>>>(b->slotOf, b->hmin, nS, b->flags);
    count_launch(3);
    if ((e = scan_exclusive(b->flags, nS, b->vid, b->tiles, b->total, s)) != cudaSuccess) return e;
    k_mc_finish<<<grid_for(nS, 256), 256, 0, s>>>(b->slotOf, b->hmin, b->vid, b->flags, b->pos, nS, b->tris, b->verts);
    count_launch();
    int hv = 0;
    if ((e = cudaMemcpyAsync(&hv, b->total, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    nV = hv;
  }
  b->nTris = hTris;
  b->nVerts = nV;
  *nVerts = nV;
  *nTris = hTris;
  return cudaGetLastError();
}

cudaError_t mesh_copy(void* mbp, float* verts, unsigned int* tris, cudaStream_t s) {
  auto* b = static_cast<MeshBuffers*>(mbp);
  if (!b) return cudaErrorInvalidValue;
  cudaError_t e = cudaSuccess;
  if (verts && b->nVerts) e = cudaMemcpyAsync(verts, b->verts, b->nVerts * 12, cudaMemcpyDefault, s);
  if (e == cudaSuccess && tris && b->nTris) e = cudaMemcpyAsync(tris, b->tris, b->nTris * 12, cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e;
}

}  // namespace rfg
