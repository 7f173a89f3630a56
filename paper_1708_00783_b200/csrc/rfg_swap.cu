// rfg_swap.cu — the swapping engine (SPEC.md:407-465,
// PAPER.md:441-478) over the reference's hooks: ptr == -1 "swapped out",
// reserveBlockForEntry / releaseBlock (voxel_block_map.cpp:107-123) and the
// kVisibleSwapped / kBoundary visibility types (fusion.cpp:219-229).
//
// B200 layout: the host tier is a voxel store indexed by hash entry (depth
// plane, + colour plane for colour maps) in host memory; transfers go through
// one pinned host buffer and one device buffer of `capacity` blocks per
// direction per frame (the SPEC's fixed-size transfer buffers).  Everything
// that decides *which* blocks move runs on the device:
//   swap-in  (after allocation, before integration): flags = visibility 2 and
//            stored on the host; an exclusive scan gives ascending-index ranks;
//            the first `capacity` indices go to the host, which gathers their
//            blocks into the pinned buffer (the only host pass over voxel
//            data), one H2D, then one warp per block pops a VBA block in the
//            serial reserveBlockForEntry order and merges the host voxels
//            into it (a fresh block takes the host voxel; SPEC apply_swapped_in);
//   swap-out (after integration): per resident entry the invisible-frame age
//            is updated on the device; entries with age >= 2 are ranked by
//            index, the first `capacity` are copied into the device transfer
//            buffer and released (free-stack pushes in releaseBlock order),
//            one D2H, and the host scatters them into the store.
// The result — entries, free stack, VBA, host store — is bit-identical to the
// serial restatement (oracle/rfo.c:rfo_swap_in / rfo_swap_out).
#include <cstring>
#include <memory>
#include <string>

#include "rfg_common.cuh"

namespace rfg {

constexpr uint8_t kSwapAge = 2;  // not visible for K = 2 consecutive frames

__global__ void k_swapin_flags(DevMap m, const uint8_t* __restrict__ has, int* flags) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.total) return;
  flags[i] = (m.visibility[i] == 2 && has[i]) ? 1 : 0;
}

// swap-out candidates; ages of resident entries advance here (once per frame)
__global__ void k_swapout_flags(DevMap m, uint8_t* age, int* flags) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.total) return;
  const int4 e = ld_entry(m.entries, (int)i);
  int f = 0;
  if (e.w >= 0) {
    uint8_t a = age[i];
    a = m.visibility[i] ? 0 : (a < 255 ? a + 1 : a);
    age[i] = a;
    f = a >= kSwapAge ? 1 : 0;
  }
  flags[i] = f;
}

__global__ void k_swap_select(const int* __restrict__ flags, const int* __restrict__ rank, uint32_t n, int cap,
                              int* idxOut) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  const int r = rank[i];
  if (r < cap) idxOut[r] = (int)i;
}

// one warp per staged block; nFree0 = free-stack size before the swap-in
__global__ void k_swapin_apply(DevMap m, const int* __restrict__ idx, const uint32_t* __restrict__ depthIn,
                               const uint32_t* __restrict__ colourIn, int n, int maxW) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nFree0 = m.state->nFreeBlocks;
  if (k >= n || k >= nFree0) return;  // VBA exhausted: the rest stay queued
  const int ptr = m.freeBlocks[nFree0 - 1 - k];
  uint32_t* dst = m.vbaDepth + (size_t)ptr * kBlock3;
  const uint32_t* src = depthIn + (size_t)k * kBlock3;
  for (int v = lane; v < kBlock3; v += 32) {
    // reserveBlockForEntry resets the block to Voxel{} (w = 0), so the merge
    // (SPEC apply_swapped_in) takes the host voxel
    dst[v] = src[v];
  }
  if (m.vbaColour) {
    uint32_t* cd = m.vbaColour + (size_t)ptr * kBlock3;
    for (int v = lane; v < kBlock3; v += 32) cd[v] = colourIn ? colourIn[(size_t)k * kBlock3 + v] : 0u;
  }
  if (lane == 0) reinterpret_cast<int*>(m.entries + idx[k])[3] = ptr;  // entry.ptr
  (void)maxW;
}

__global__ void k_swapin_commit(DevMap m, int n) {
  MapState* st = m.state;
  st->nFreeBlocks -= min(n, st->nFreeBlocks);
}

// one warp per selected entry: copy out, release (push in index order)
__global__ void k_swapout_gather(DevMap m, const int* __restrict__ idx, const int* __restrict__ total, int cap,
                                 uint32_t* depthOut, uint32_t* colourOut, uint8_t* has) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int n = min(*total, cap);
  if (k >= n) return;
  const int i = idx[k];
  const int ptr = reinterpret_cast<const int*>(m.entries + i)[3];
  // copy out, then reset the block to Voxel{} before it returns to the free
  // stack: allocateBlock does not clear reused blocks (voxel_block_map.cpp:
  // 74-105), and the SPEC's equivalence invariant needs a
  // swapped-out block's memory to come back clean
  uint32_t* src = m.vbaDepth + (size_t)ptr * kBlock3;
  for (int v = lane; v < kBlock3; v += 32) {
    depthOut[(size_t)k * kBlock3 + v] = src[v];
    src[v] = kDefaultDepthVoxel;
  }
  if (m.vbaColour) {
    uint32_t* cs = m.vbaColour + (size_t)ptr * kBlock3;
    for (int v = lane; v < kBlock3; v += 32) {
      if (colourOut) colourOut[(size_t)k * kBlock3 + v] = cs[v];
      cs[v] = 0u;
    }
  }
  if (lane == 0) {
    m.freeBlocks[m.state->nFreeBlocks + k] = ptr;  // releaseBlock: push_back
    reinterpret_cast<int*>(m.entries + i)[3] = -1;
    has[i] = 1;
  }
}

__global__ void k_swapout_commit(DevMap m, const int* __restrict__ total, int cap) {
  m.state->nFreeBlocks += min(*total, cap);
}

// reserveBlockForEntry / releaseBlock on one entry (voxel_block_map.cpp:107-123)
__global__ void k_reserve_one(DevMap m, int idx, int* result) {
  __shared__ int ptr;
  if (threadIdx.x == 0) {
    const int cur = reinterpret_cast<const int*>(m.entries + idx)[3];
    ptr = -1;
    if (cur >= 0) {
      *result = 1;
    } else if (m.state->nFreeBlocks == 0) {
      *result = 0;
    } else {
      ptr = m.freeBlocks[--m.state->nFreeBlocks];
      reinterpret_cast<int*>(m.entries + idx)[3] = ptr;
      *result = 1;
    }
  }
  __syncthreads();
  if (ptr < 0) return;
  for (int v = threadIdx.x; v < kBlock3; v += blockDim.x) {  // Voxel{}: sdf 32767, w 0, colour 0
    m.vbaDepth[(size_t)ptr * kBlock3 + v] = kDefaultDepthVoxel;
    if (m.vbaColour) m.vbaColour[(size_t)ptr * kBlock3 + v] = 0u;
  }
}

__global__ void k_release_one(DevMap m, int idx) {
  int* e = reinterpret_cast<int*>(m.entries + idx);
  if (e[3] < 0) return;
  m.freeBlocks[m.state->nFreeBlocks++] = e[3];
  e[3] = -1;
}

}  // namespace rfg

struct rfg_swap {
  rfg_map* map = nullptr;
  int cap = 0;
  uint32_t total = 0;
  bool colour = false;
  // host tier (indexed by entry; pages are touched only for stored entries)
  std::unique_ptr<uint32_t[]> hostDepth, hostColour;
  std::unique_ptr<uint8_t[]> hostHas;
  // device state
  uint8_t* hasDev = nullptr;
  uint8_t* age = nullptr;
  int* flags = nullptr;
  int* rank = nullptr;
  int* tiles = nullptr;
  int* dTotal = nullptr;
  int* dIdx = nullptr;
  uint32_t* dDepth = nullptr;
  uint32_t* dColour = nullptr;
  // pinned transfer buffers
  int* hIdx = nullptr;
  int* hTotal = nullptr;
  uint32_t* hDepth = nullptr;
  uint32_t* hColour = nullptr;
};

namespace {

#define SW_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) {            \
      rfg::set_error(msg);    \
      return RFG_EINVAL;      \
    }                         \
  } while (0)

void swap_free(rfg_swap* w) {
  void* d[] = {w->hasDev, w->age, w->flags, w->rank, w->tiles, w->dTotal, w->dIdx, w->dDepth, w->dColour};
  for (void* p : d)
    if (p) cudaFree(p);
  void* h[] = {w->hIdx, w->hTotal, w->hDepth, w->hColour};
  for (void* p : h)
    if (p) cudaFreeHost(p);
  delete w;
}

// rank the flagged entries; returns the selected count (synchronises)
int swap_rank(rfg_swap* w, cudaStream_t s, int* nSel) {
  const uint32_t n = w->total;
  RFG_CK(rfg::scan_exclusive(w->flags, n, w->rank, w->tiles, w->dTotal, s));
  rfg::k_swap_select<<<(n + 255) / 256, 256, 0, s>>>(w->flags, w->rank, n, w->cap, w->dIdx);
  rfg::count_launch();
  RFG_CK(cudaMemcpyAsync(w->hTotal, w->dTotal, sizeof(int), cudaMemcpyDeviceToHost, s));
  RFG_CK(cudaMemcpyAsync(w->hIdx, w->dIdx, sizeof(int) * w->cap, cudaMemcpyDeviceToHost, s));
  RFG_CK(cudaMemcpyAsync(w->map->hostState, w->map->d.state, sizeof(rfg::MapState), cudaMemcpyDeviceToHost, s));
  RFG_CK(cudaStreamSynchronize(s));
  *nSel = *w->hTotal < w->cap ? *w->hTotal : w->cap;
  return RFG_OK;
}

}  // namespace

extern "C" {

int rfg_swap_create(rfg_map* m, int capacity, rfg_swap** out) {
  SW_REQUIRE(m && out && capacity > 0, "invalid swap_create arguments");
  *out = nullptr;
  auto* w = new rfg_swap();
  w->map = m;
  w->cap = capacity;
  w->total = m->d.total;
  w->colour = m->d.vbaColour != nullptr;
  const size_t nE = w->total, blk = (size_t)rfg::kBlock3;
  w->hostDepth.reset(new (std::nothrow) uint32_t[nE * blk]);
  if (w->colour) w->hostColour.reset(new (std::nothrow) uint32_t[nE * blk]);
  w->hostHas.reset(new (std::nothrow) uint8_t[nE]());
  bool ok = w->hostDepth && w->hostHas && (!w->colour || w->hostColour);
  const long long tilesN = rfg::scan_tile_scratch_ints(nE);
  ok = ok && cudaMalloc(&w->hasDev, nE) == cudaSuccess && cudaMalloc(&w->age, nE) == cudaSuccess &&
       cudaMalloc(&w->flags, nE * 4) == cudaSuccess && cudaMalloc(&w->rank, nE * 4) == cudaSuccess &&
       cudaMalloc(&w->tiles, tilesN * 4) == cudaSuccess && cudaMalloc(&w->dTotal, 4) == cudaSuccess &&
       cudaMalloc(&w->dIdx, capacity * 4) == cudaSuccess &&
       cudaMalloc(&w->dDepth, (size_t)capacity * blk * 4) == cudaSuccess &&
       (!w->colour || cudaMalloc(&w->dColour, (size_t)capacity * blk * 4) == cudaSuccess) &&
       cudaMallocHost(&w->hIdx, capacity * 4) == cudaSuccess && cudaMallocHost(&w->hTotal, 4) == cudaSuccess &&
       cudaMallocHost(&w->hDepth, (size_t)capacity * blk * 4) == cudaSuccess &&
       (!w->colour || cudaMallocHost(&w->hColour, (size_t)capacity * blk * 4) == cudaSuccess);
  if (!ok) {
    cudaGetLastError();
    swap_free(w);
    rfg::set_error("swap allocation failed");
    return RFG_ENOMEM;
  }
  cudaStream_t s = m->stream;
  if (cudaMemsetAsync(w->hasDev, 0, nE, s) != cudaSuccess || cudaMemsetAsync(w->age, 0, nE, s) != cudaSuccess) {
    swap_free(w);
    rfg::set_error("swap init failed");
    return RFG_ECUDA;
  }
  *out = w;
  return RFG_OK;
}

int rfg_swap_destroy(rfg_swap* w) {
  if (!w) return RFG_OK;
  if (w->map && w->map->stream) cudaStreamSynchronize(w->map->stream);
  swap_free(w);
  return RFG_OK;
}

int rfg_swap_in(rfg_swap* w, int maxW, int* nIn) {
  SW_REQUIRE(w && nIn, "null argument");
  rfg_map* m = w->map;
  cudaStream_t s = m->stream;
  const uint32_t n = w->total;
  rfg::k_swapin_flags<<<(n + 255) / 256, 256, 0, s>>>(m->d, w->hasDev, w->flags);
  rfg::count_launch();
  int sel = 0;
  int rc = swap_rank(w, s, &sel);
  if (rc != RFG_OK) return rc;
  *nIn = 0;
  // the VBA may run out: the entries beyond the free stack stay queued
  const int nFree0 = m->hostState->nFreeBlocks;
  if (sel > nFree0) sel = nFree0;
  if (sel == 0) return RFG_OK;
  // host gather: the only host pass over voxel data
  const size_t blk = (size_t)rfg::kBlock3;
  for (int k = 0; k < sel; ++k) {
    const size_t i = (size_t)w->hIdx[k];
    std::memcpy(w->hDepth + k * blk, w->hostDepth.get() + i * blk, blk * 4);
    if (w->colour) std::memcpy(w->hColour + k * blk, w->hostColour.get() + i * blk, blk * 4);
  }
  RFG_CK(cudaMemcpyAsync(w->dDepth, w->hDepth, sel * blk * 4, cudaMemcpyHostToDevice, s));
  if (w->colour) RFG_CK(cudaMemcpyAsync(w->dColour, w->hColour, sel * blk * 4, cudaMemcpyHostToDevice, s));
  rfg::k_swapin_apply<<<(sel + 7) / 8, 256, 0, s>>>(m->d, w->dIdx, w->dDepth, w->colour ? w->dColour : nullptr,
                                                   sel, maxW);
  rfg::k_swapin_commit<<<1, 1, 0, s>>>(m->d, sel);
  rfg::count_launch(2);
  RFG_CK(cudaGetLastError());
  *nIn = sel;
  return RFG_OK;
}

int rfg_swap_out(rfg_swap* w, int* nOut) {
  SW_REQUIRE(w && nOut, "null argument");
  rfg_map* m = w->map;
  cudaStream_t s = m->stream;
  const uint32_t n = w->total;
  rfg::k_swapout_flags<<<(n + 255) / 256, 256, 0, s>>>(m->d, w->age, w->flags);
  rfg::count_launch();
  int sel = 0;
  int rc = swap_rank(w, s, &sel);
  if (rc != RFG_OK) return rc;
  *nOut = sel;
  if (sel == 0) return RFG_OK;
  rfg::k_swapout_gather<<<(sel + 7) / 8, 256, 0, s>>>(m->d, w->dIdx, w->dTotal, w->cap, w->dDepth,
                                                     w->colour ? w->dColour : nullptr, w->hasDev);
  rfg::k_swapout_commit<<<1, 1, 0, s>>>(m->d, w->dTotal, w->cap);
  rfg::count_launch(2);
  const size_t blk = (size_t)rfg::kBlock3;
  RFG_CK(cudaMemcpyAsync(w->hDepth, w->dDepth, sel * blk * 4, cudaMemcpyDeviceToHost, s));
  if (w->colour) RFG_CK(cudaMemcpyAsync(w->hColour, w->dColour, sel * blk * 4, cudaMemcpyDeviceToHost, s));
  RFG_CK(cudaStreamSynchronize(s));
  for (int k = 0; k < sel; ++k) {  // host scatter into the store
    const size_t i = (size_t)w->hIdx[k];
    std::memcpy(w->hostDepth.get() + i * blk, w->hDepth + k * blk, blk * 4);
    if (w->colour) std::memcpy(w->hostColour.get() + i * blk, w->hColour + k * blk, blk * 4);
    w->hostHas[i] = 1;
  }
  return RFG_OK;
}

int rfg_map_reserve_block(rfg_map* m, int idx) {
  SW_REQUIRE(m && idx >= 0 && (uint32_t)idx < m->d.total, "invalid entry index");
  int* d = nullptr;
  int h = 0;
  RFG_CK(cudaMalloc(&d, sizeof(int)));
  rfg::k_reserve_one<<<1, 256, 0, m->stream>>>(m->d, idx, d);
  rfg::count_launch();
  cudaError_t e = cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, m->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(m->stream);
  cudaFree(d);
  RFG_CK(e);
  return h;  // 1 reserved (or already resident), 0 VBA exhausted
}

int rfg_map_release_block(rfg_map* m, int idx) {
  SW_REQUIRE(m && idx >= 0 && (uint32_t)idx < m->d.total, "invalid entry index");
  rfg::k_release_one<<<1, 1, 0, m->stream>>>(m->d, idx);
  rfg::count_launch();
  RFG_CK(cudaGetLastError());
  return RFG_OK;
}

int rfg_swap_export(rfg_swap* w, uint8_t* hasOut, uint8_t* ageOut) {
  SW_REQUIRE(w, "null swap");
  if (hasOut) std::memcpy(hasOut, w->hostHas.get(), w->total);
  if (ageOut) {
    RFG_CK(cudaMemcpyAsync(ageOut, w->age, w->total, cudaMemcpyDeviceToHost, w->map->stream));
    RFG_CK(cudaStreamSynchronize(w->map->stream));
  }
  return RFG_OK;
}

// the host-tier copy of entry idx as VoxelSRgb bytes (8 per voxel)
int rfg_swap_host_block(rfg_swap* w, int idx, uint8_t* out4096) {
  SW_REQUIRE(w && out4096 && idx >= 0 && (uint32_t)idx < w->total, "invalid swap_host_block arguments");
  SW_REQUIRE(w->hostHas[idx], "entry has no host data");
  const uint32_t* d = w->hostDepth.get() + (size_t)idx * rfg::kBlock3;
  const uint32_t* c = w->colour ? w->hostColour.get() + (size_t)idx * rfg::kBlock3 : nullptr;
  for (int v = 0; v < rfg::kBlock3; ++v) {
    uint8_t* o = out4096 + 8 * v;
    const uint32_t dw = d[v], cw = c ? c[v] : 0u;
    o[0] = (uint8_t)(dw & 0xFF);
    o[1] = (uint8_t)((dw >> 8) & 0xFF);
    o[2] = (uint8_t)((dw >> 16) & 0xFF);
    o[3] = (uint8_t)(cw & 0xFF);
    o[4] = (uint8_t)((cw >> 8) & 0xFF);
    o[5] = (uint8_t)((cw >> 16) & 0xFF);
    o[6] = (uint8_t)((cw >> 24) & 0xFF);
    o[7] = 0;
  }
  return RFG_OK;
}

}  // extern "C"
