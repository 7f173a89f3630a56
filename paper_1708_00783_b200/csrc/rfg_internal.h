// rfg_internal.h — device map layout, per-frame kernel arguments, error
// plumbing.  Shared by the .cu translation units of librfg.so.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/rfg.h"

namespace rfg {

// Device-resident mutable scalars of a map.
struct MapState {
  int nFreeBlocks;   // free VBA stack size (freeBlockStack_.size())
  int nFreeExcess;   // free excess stack size
  int nVisible;      // visibleList_.size()
  int error;         // sticky RFG_E* flag set by kernels
  // per-frame allocation bookkeeping
  int snapFreeBlocks, snapFreeExcess;  // stack sizes at the start of stage 2
  int succ, succType2;                 // stage-2 successes (all / excess-linked)
  int stats[4];                        // requested, allocated, allocFailures, (visibleCount = nVisible)
  int nRequests;                       // stage-2 request count
  int pad[5];
};

// Plain-old-data view of a map passed by value to kernels.
struct DevMap {
  uint32_t buckets, excess, capacity, total;
  int4* entries;           // total x 16 B
  uint32_t* vbaDepth;      // capacity x 512 depth voxels (4 B)
  uint32_t* vbaColour;     // capacity x 512 colour voxels (4 B) or nullptr
  int* freeBlocks;         // capacity
  int* freeExcess;         // excess
  int* visibleList;        // total
  uint8_t* visibility;     // total
  uint32_t* reqKey;        // total: stage-1 last-writer key (0 = no request)
  uint8_t* marked;         // total: stage-1/2 marks (0/1/2)
  MapState* state;
  int2* tileCounts;        // per kTile-entry tile
  int2* tilePrefix;        // exclusive prefix (+ total at [nTiles])
  int nTiles;
  int rank, world, tileShift;  // shard filter
  // expected-range scratch (screen-tile bins), sized for the image in use
  int4* rangeBounds;       // per visible block: packed pixel rectangle + z span
  int* binCount;           // per 32x32 screen tile
  int* bins;               // binTilesX * binTilesY * binCap block indices
  int* tileCost;           // per tile: the last raycast's longest march (steps), for the next frame's order
  int* tileOrder;          // per tile: the raycast's CTA -> tile order (heaviest tiles first)
  int binTilesX, binTilesY, binCap;
  unsigned binGen;         // bumped whenever the range scratch is reallocated (captured graphs re-capture)
};

// Per-call frame arguments (camera, scene params, pose).
struct FrameArgs {
  int w, h;
  float fx, fy, cx, cy;
  float voxelSize, mu;
  int maxW;
  float vfMin, vfMax;
  int stopAtMaxW;
  float pose[12];          // world -> camera (used when poseDev == nullptr)
  const float* poseDev;    // device-resident pose (tracking pipeline)
  int swapping;            // FusionEngine::Options::swappingEnabled (fusion.hpp:55)
  float swapMargin;        // Options::swapMarginPx (fusion.hpp:56)
  int depthBounded;        // every depth value is below 2^36 m in magnitude (the pipeline's u16 frames)
};

struct Pose12 {
  float v[12];
};

constexpr int kRangeTilePx = 16;     // expected-range screen tile edge (pixels)
constexpr int kTile = 1024;          // hash entries per scan tile
constexpr int kTileThreads = 256;    // 4 consecutive entries per thread

void set_error(const std::string& msg);
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// Kernel launch with programmatic stream serialisation when the current
// thread is enqueueing a frame graph (g_pdl, rfg_api.cu:enqueue_frame); a
// plain launch otherwise.
extern thread_local bool g_pdl;
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (g_pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// SM count of the current device, cached per device (grid sizes).
int current_sm_count();

// Makes `device` current for the scope of an entry point and restores the
// caller's device afterwards (a map lives on the device it was created on).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (device < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
      return;
    }
    if (prev != device) cudaSetDevice(device);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

FrameArgs make_frame_args(const rfg_intrinsics* intr, const rfg_scene_params* p, const float* pose34,
                          const float* poseDev);

// kernel launchers (return cudaError_t of the launch)
cudaError_t launch_allocate(const DevMap& m, const float* depth, const FrameArgs& fa, cudaStream_t s);
cudaError_t launch_sort_visible(const DevMap& m, cudaStream_t s);
// depth-only (rgba nullptr) or RGB-D integration; rgba = packed RGBA8 colour
// image (launch_rgb_to_rgba), extr34 nullptr = identity extrinsics
cudaError_t launch_integrate(const DevMap& m, const float* depth, const uint32_t* rgba, const FrameArgs& fa,
                             const rfg_intrinsics* intrRgb, const float* extr34, cudaStream_t s);
cudaError_t launch_rgb_to_rgba(const uint8_t* rgb, uint32_t* out, int n, cudaStream_t s);
const void* rgb_to_rgba_kernel();
cudaError_t launch_ranges(const DevMap& m, const FrameArgs& fa, float2* range, cudaStream_t s);
// (Re)allocate the expected-range bins for a width x height image (host call,
// not capturable; done at pipeline creation or on first use of a size).
int ensure_range_scratch(struct ::rfg_map* m, int width, int height);
cudaError_t launch_range_bin(const DevMap& m, const FrameArgs& fa, cudaStream_t s);
cudaError_t launch_raycast_tiles(const DevMap& m, const FrameArgs& fa, float2* range, float4* raycast, float4* points,
                                 float4* normals, cudaStream_t s);
cudaError_t launch_icp_maps(const DevMap& m, const FrameArgs& fa, const float2* range, float4* raycast,
                            float4* points, float4* normals, cudaStream_t s);
cudaError_t launch_icp_maps_list(const DevMap& m, const FrameArgs& fa, const float2* range, const int* list,
                                 const int* count, int maxCount, float4* raycast, float4* points, float4* normals,
                                 cudaStream_t s);
cudaError_t launch_forward_project(int hasRaycast, float4* raycast, float4* points, float4* normals,
                                   const float* pose34, int w, int h, float fx, float fy, float cx, float cy,
                                   float vs, float4* prev, unsigned long long* keys, int2* tileCounts,
                                   int2* tilePrefix, int* list, int* count, cudaStream_t s);
cudaError_t launch_build_view(const uint16_t* raw, int w, int h, float scale, float offset, int levels, float* out,
                              cudaStream_t s);
// exclusive scan of n ints on the device (rfg_mesh.cu); tileScratch holds
// scan_tile_scratch_ints(n) ints, *total (device) receives the sum
long long scan_tile_scratch_ints(long long n);
cudaError_t scan_exclusive(const int* in, long long n, int* out, int* tileScratch, int* total, cudaStream_t s);
cudaError_t mesh_extract(const DevMap& m, float vs, void** mesh, long long* nVerts, long long* nTris, cudaStream_t s);
cudaError_t mesh_copy(void* mesh, float* verts, unsigned int* tris, cudaStream_t s);
void mesh_free(void* mesh);
int mc_table_export(int* counts256, int* tris256x16x3);
cudaError_t launch_render_colour(const DevMap& m, const FrameArgs& fa, int mode, const float4* raycast,
                                 const float4* normals, const int* list, const int* count, int maxCount,
                                 uint8_t* rgb, cudaStream_t s);

}  // namespace rfg

struct rfg_map {
  rfg::DevMap d;
  rfg_map_config cfg;
  int device;
  cudaStream_t stream;
  rfg::MapState* hostState;  // pinned mirror for readback
  size_t metaBytes;          // the hash-metadata allocation (d.entries ... d.state, tileScratch)
  int* tileScratch;          // 64 KiB inside it: the range stage's per-tile counters when they fit
  // ICP scratch
  void* icpOut;              // device: rfg_icp.cu IcpState (sums, solver state, accumulators)
  float* icpPose;            // device: current cam->world (12) + world->cam (12) + render pose (12)
  // forward-projection scratch (approximate raycast), sized for fwdN pixels
  float4* fwdPrev;
  unsigned long long* fwdKeys;
  int2* fwdTileCounts;
  int2* fwdTilePrefix;
  int fwdN;
  void* mesh;  // rfg_mesh.cu MeshBuffers (extract_mesh scratch + result)
  uint32_t* rgbaScratch;  // packed colour image for rfg_integrate (rgbaN pixels)
  int rgbaN;
};

#define RFG_CK(call)                                                                      \
  do {                                                                                    \
    cudaError_t err_ = (call);                                                            \
    if (err_ != cudaSuccess) {                                                            \
      rfg::set_error(std::string(#call) + ": " + cudaGetErrorString(err_));               \
      return RFG_ECUDA;                                                                   \
    }                                                                                     \
  } while (0)
