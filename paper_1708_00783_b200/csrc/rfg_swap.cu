// rfg_swap.cu — the swapping engine (SPEC.md:407-465,
// PAPER.md:441-478) over the reference's hooks: ptr == -1 "swapped out",
// reserveBlockForEntry / releaseBlock (voxel_block_map.cpp:107-123) and the
// kVisibleSwapped / kBoundary visibility types (fusion.cpp:219-229).
//
// B200 layout: the host tier is a pool of pinned, device-mapped host slots
// (one 2 KiB slot per plane for every entry ever swapped out; the pool grows
// in 4096-slot chunks, so only stored entries cost host memory, and pinned
// pages never fault).  The GPU reads and writes the slots itself over PCIe:
// there is no staging buffer and no host pass over voxel data.  Everything
// that decides *which* blocks move runs on the device:
//   swap-in  (after allocation, before integration): flags = visibility 2 and
//            stored on the host; an exclusive scan gives ascending-index ranks;
//            the first `capacity` indices come back to the host, which looks up
//            their slots (one pointer pair per block, one small H2D), then one
//            warp per block pops a VBA block in the serial reserveBlockForEntry
//            order and reads the host voxels straight into it (a fresh block
//            takes the host voxel; SPEC apply_swapped_in);
//   swap-out (after integration): per resident entry the invisible-frame age
//            is updated on the device; entries with age >= 2 are ranked by
//            index, the host assigns a slot to each of the first `capacity`
//            that has none, and one warp per block writes it straight into its
//            host slot and releases it (free-stack pushes in releaseBlock
//            order).
// The result — entries, free stack, VBA, host store — is bit-identical to the
// serial restatement (oracle/rfo.c:rfo_swap_in / rfo_swap_out).
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

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
__global__ void k_swapin_apply(DevMap m, const int* __restrict__ idx, const uint64_t* __restrict__ src, int n,
                               int maxW) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nFree0 = m.state->nFreeBlocks;
  if (k >= n || k >= nFree0) return;  // VBA exhausted: the rest stay queued
  const int ptr = m.freeBlocks[nFree0 - 1 - k];
  // reserveBlockForEntry resets the block to Voxel{} (w = 0), so the merge
  // (SPEC apply_swapped_in) takes the host voxel: a 16-B copy per lane from
  // the mapped host slot (512 B per warp request over PCIe)
  uint4* dst = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)ptr * kBlock3);
  const uint4* hs = reinterpret_cast<const uint4*>(src[2 * k]);
#pragma unroll
  for (int v = lane; v < kBlock3 / 4; v += 32) {
    const uint4 h = hs[v];
    dst[v] = h;
  }
  if (m.vbaColour) {
    uint4* cd = reinterpret_cast<uint4*>(m.vbaColour + (size_t)ptr * kBlock3);
    const uint4* hc = reinterpret_cast<const uint4*>(src[2 * k + 1]);
#pragma unroll
    for (int v = lane; v < kBlock3 / 4; v += 32) cd[v] = hc ? hc[v] : make_uint4(0u, 0u, 0u, 0u);
  }
  if (lane == 0) reinterpret_cast<int*>(m.entries + idx[k])[3] = ptr;  // entry.ptr
  (void)maxW;
}

__global__ void k_swapin_commit(DevMap m, int n) {
  MapState* st = m.state;
  st->nFreeBlocks -= min(n, st->nFreeBlocks);
}

// one warp per selected entry: copy out into its mapped host slot, release
// (push in index order)
__global__ void k_swapout_gather(DevMap m, const int* __restrict__ idx, const int* __restrict__ total, int cap,
                                 const uint64_t* __restrict__ dstPtr, uint8_t* has) {
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
  const uint4 dflt = make_uint4(kDefaultDepthVoxel, kDefaultDepthVoxel, kDefaultDepthVoxel, kDefaultDepthVoxel);
  uint4* src = reinterpret_cast<uint4*>(m.vbaDepth + (size_t)ptr * kBlock3);
  uint4* hd = reinterpret_cast<uint4*>(dstPtr[2 * k]);
#pragma unroll
  for (int v = lane; v < kBlock3 / 4; v += 32) {
    hd[v] = src[v];
    src[v] = dflt;
  }
  if (m.vbaColour) {
    uint4* cs = reinterpret_cast<uint4*>(m.vbaColour + (size_t)ptr * kBlock3);
    uint4* hc = reinterpret_cast<uint4*>(dstPtr[2 * k + 1]);
#pragma unroll
    for (int v = lane; v < kBlock3 / 4; v += 32) {
      if (hc) hc[v] = cs[v];
      cs[v] = make_uint4(0u, 0u, 0u, 0u);
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
  // host tier: per entry its slot (host pointer, device alias) per plane, or
  // null; slots come from pinned mapped chunks of kSlotChunk blocks
  std::vector<uint32_t*> slotDepth, slotColour;
  std::vector<uint64_t> devDepth, devColour;
  std::vector<void*> chunks;
  uint32_t* chunkHost[2] = {nullptr, nullptr};
  uint64_t chunkDev[2] = {0, 0};
  size_t chunkUsed = 0, chunkCap = 0, chunkSlots = 0;
  std::unique_ptr<uint8_t[]> hostHas;
  // device state
  uint8_t* hasDev = nullptr;
  uint8_t* age = nullptr;
  int* flags = nullptr;
  int* rank = nullptr;
  int* tiles = nullptr;
  int* dTotal = nullptr;
  int* dIdx = nullptr;
  uint64_t* dPtr = nullptr;  // per selected block: {depth slot, colour slot} device addresses
  // pinned
  int* hIdx = nullptr;
  int* hTotal = nullptr;
  uint64_t* hPtr = nullptr;
};

namespace {

#define SW_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) {            \
      rfg::set_error(msg);    \
      return RFG_EINVAL;      \
    }                         \
  } while (0)

// The whole host tier is pinned up front when it fits kSlotUpFront bytes (the
// InfiniTAM global cache is one host array of every entry's block); larger
// maps grow it in chunks of kSlotChunk slots (128 MiB per plane).  Pinning
// costs ~ms per 10 MiB, so it is kept out of the per-frame swap-out.
// Both limits can be lowered through the environment (RFG_SWAP_PIN_UPFRONT
// bytes, RFG_SWAP_CHUNK_SLOTS) so the tests can drive the chunked growth.
constexpr size_t kSlotUpFront = size_t(4) << 30;
constexpr size_t kSlotChunk = 65536;

size_t env_size(const char* name, size_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  char* end = nullptr;
  const unsigned long long x = std::strtoull(v, &end, 10);
  return (end && *end == 0) ? (size_t)x : dflt;
}

int slot_chunk(rfg_swap* w, size_t slots) {
  const size_t bytes = slots * (size_t)rfg::kBlock3 * 4;
  for (int p = 0; p < (w->colour ? 2 : 1); ++p) {
    void* h = nullptr;
    void* dv = nullptr;
    if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess) {
      cudaGetLastError();
      rfg::set_error("swap host slot allocation failed");
      return RFG_ENOMEM;
    }
    w->chunks.push_back(h);
    RFG_CK(cudaHostGetDevicePointer(&dv, h, 0));
    w->chunkHost[p] = static_cast<uint32_t*>(h);
    w->chunkDev[p] = reinterpret_cast<uint64_t>(dv);
  }
  w->chunkUsed = 0;
  w->chunkCap = slots;
  return RFG_OK;
}

void swap_free(rfg_swap* w) {
  void* d[] = {w->hasDev, w->age, w->flags, w->rank, w->tiles, w->dTotal, w->dIdx, w->dPtr};
  for (void* p : d)
    if (p) cudaFree(p);
  void* h[] = {w->hIdx, w->hTotal, w->hPtr};
  for (void* p : h)
    if (p) cudaFreeHost(p);
  for (void* p : w->chunks) cudaFreeHost(p);
  delete w;
}

// the host slot of entry i (assigned on its first swap-out; kept for life)
int slot_for(rfg_swap* w, size_t i) {
  if (w->slotDepth[i]) return RFG_OK;
  const size_t blk = (size_t)rfg::kBlock3;
  if (w->chunkUsed == w->chunkCap) {
    const int rc = slot_chunk(w, w->chunkSlots);
    if (rc != RFG_OK) return rc;
  }
  const size_t off = (size_t)w->chunkUsed++ * blk;
  w->slotDepth[i] = w->chunkHost[0] + off;
  w->devDepth[i] = w->chunkDev[0] + off * 4;
  if (w->colour) {
    w->slotColour[i] = w->chunkHost[1] + off;
    w->devColour[i] = w->chunkDev[1] + off * 4;
  }
  return RFG_OK;
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
  rfg::DeviceGuard dg_(m ? m->device : -1);
  SW_REQUIRE(m && out && capacity > 0, "invalid swap_create arguments");
  *out = nullptr;
  auto* w = new rfg_swap();
  w->map = m;
  w->cap = capacity;
  w->total = m->d.total;
  w->colour = m->d.vbaColour != nullptr;
  const size_t nE = w->total;
  w->slotDepth.assign(nE, nullptr);
  w->devDepth.assign(nE, 0);
  if (w->colour) {
    w->slotColour.assign(nE, nullptr);
    w->devColour.assign(nE, 0);
  }
  w->hostHas.reset(new (std::nothrow) uint8_t[nE]());
  bool ok = w->hostHas != nullptr;
  const long long tilesN = rfg::scan_tile_scratch_ints(nE);
  ok = ok && cudaMalloc(&w->hasDev, nE) == cudaSuccess && cudaMalloc(&w->age, nE) == cudaSuccess &&
       cudaMalloc(&w->flags, nE * 4) == cudaSuccess && cudaMalloc(&w->rank, nE * 4) == cudaSuccess &&
       cudaMalloc(&w->tiles, tilesN * 4) == cudaSuccess && cudaMalloc(&w->dTotal, 4) == cudaSuccess &&
       cudaMalloc(&w->dIdx, capacity * 4) == cudaSuccess && cudaMalloc(&w->dPtr, capacity * 16) == cudaSuccess &&
       cudaMallocHost(&w->hIdx, capacity * 4) == cudaSuccess && cudaMallocHost(&w->hTotal, 4) == cudaSuccess &&
       cudaMallocHost(&w->hPtr, capacity * 16) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    swap_free(w);
    rfg::set_error("swap allocation failed");
    return RFG_ENOMEM;
  }
  w->chunkSlots = env_size("RFG_SWAP_CHUNK_SLOTS", kSlotChunk);
  if (w->chunkSlots == 0) w->chunkSlots = kSlotChunk;
  const size_t upFront = env_size("RFG_SWAP_PIN_UPFRONT", kSlotUpFront);
  if (nE * (size_t)rfg::kBlock3 * 4 * (w->colour ? 2 : 1) <= upFront && slot_chunk(w, nE) != RFG_OK) {
    swap_free(w);
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
  rfg::DeviceGuard dg_(w && w->map ? w->map->device : -1);
  if (!w) return RFG_OK;
  if (w->map && w->map->stream) cudaStreamSynchronize(w->map->stream);
  swap_free(w);
  return RFG_OK;
}

int rfg_swap_in(rfg_swap* w, int maxW, int* nIn) {
  rfg::DeviceGuard dg_(w && w->map ? w->map->device : -1);
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
  // the selected blocks' host slots (no host pass over voxel data)
  for (int k = 0; k < sel; ++k) {
    const size_t i = (size_t)w->hIdx[k];
    w->hPtr[2 * k] = w->devDepth[i];
    w->hPtr[2 * k + 1] = w->colour ? w->devColour[i] : 0;
  }
  RFG_CK(cudaMemcpyAsync(w->dPtr, w->hPtr, (size_t)sel * 16, cudaMemcpyHostToDevice, s));
  rfg::k_swapin_apply<<<(sel + 7) / 8, 256, 0, s>>>(m->d, w->dIdx, w->dPtr, sel, maxW);
  rfg::k_swapin_commit<<<1, 1, 0, s>>>(m->d, sel);
  rfg::count_launch(2);
  RFG_CK(cudaGetLastError());
  *nIn = sel;
  return RFG_OK;
}

int rfg_swap_out(rfg_swap* w, int* nOut) {
  rfg::DeviceGuard dg_(w && w->map ? w->map->device : -1);
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
  // slots for the selected entries; the gather writes straight into them
  for (int k = 0; k < sel; ++k) {  // may fail (ENOMEM) before anything moved
    rc = slot_for(w, (size_t)w->hIdx[k]);
    if (rc != RFG_OK) return rc;
  }
  for (int k = 0; k < sel; ++k) {
    const size_t i = (size_t)w->hIdx[k];
    w->hPtr[2 * k] = w->devDepth[i];
    w->hPtr[2 * k + 1] = w->colour ? w->devColour[i] : 0;
    w->hostHas[i] = 1;
  }
  RFG_CK(cudaMemcpyAsync(w->dPtr, w->hPtr, (size_t)sel * 16, cudaMemcpyHostToDevice, s));
  rfg::k_swapout_gather<<<(sel + 7) / 8, 256, 0, s>>>(m->d, w->dIdx, w->dTotal, w->cap, w->dPtr, w->hasDev);
  rfg::k_swapout_commit<<<1, 1, 0, s>>>(m->d, w->dTotal, w->cap);
  rfg::count_launch(2);
  RFG_CK(cudaGetLastError());
  return RFG_OK;
}

int rfg_map_reserve_block(rfg_map* m, int idx) {
  rfg::DeviceGuard dg_(m ? m->device : -1);
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
  rfg::DeviceGuard dg_(m ? m->device : -1);
  SW_REQUIRE(m && idx >= 0 && (uint32_t)idx < m->d.total, "invalid entry index");
  rfg::k_release_one<<<1, 1, 0, m->stream>>>(m->d, idx);
  rfg::count_launch();
  RFG_CK(cudaGetLastError());
  return RFG_OK;
}

int rfg_swap_export(rfg_swap* w, uint8_t* hasOut, uint8_t* ageOut) {
  rfg::DeviceGuard dg_(w && w->map ? w->map->device : -1);
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
  rfg::DeviceGuard dg_(w && w->map ? w->map->device : -1);
  SW_REQUIRE(w && out4096 && idx >= 0 && (uint32_t)idx < w->total, "invalid swap_host_block arguments");
  SW_REQUIRE(w->hostHas[idx], "entry has no host data");
  RFG_CK(cudaStreamSynchronize(w->map->stream));  // the slot is written by the swap-out kernel
  const uint32_t* d = w->slotDepth[idx];
  const uint32_t* c = w->colour ? w->slotColour[idx] : nullptr;
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
