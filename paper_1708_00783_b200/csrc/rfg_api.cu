// rfg_api.cu — C-ABI entry points of librfg.so (include/rfg.h): map
// lifetime, the reference-mirroring per-stage calls, parity exports and the
// device-resident frame pipeline with CUDA-graph replay.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "rfg_common.cuh"

namespace rfg {

std::atomic<uint64_t> g_launches{0};

int current_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int n = dev < 64 ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
static thread_local std::string t_lastError;
void set_error(const std::string& msg) { t_lastError = msg; }

// rfg_view.cu
cudaError_t launch_build_view_full(const uint16_t* raw, const uint8_t* rgb, const Intr& in, float scale, float offset,
                                   int bilateral, int levels, int bigEndian, float* depthLevels,
                                   float* intensityLevels, float4* normals, float* scratch, cudaStream_t s);
const void* view_pyramid_kernel();
bool view_is_fused(int bilateral, bool normals, bool intensity, int levels);
cudaError_t launch_bilateral(const float* in, int w, int h, float spatialSigma, float rangeSigma, float* out,
                             cudaStream_t s);
cudaError_t launch_view_normals(const float* depth, const Intr& in, float4* out, cudaStream_t s);
cudaError_t launch_intensity(const uint8_t* rgb, int w, int h, float* out, cudaStream_t s);
cudaError_t launch_downsample_intensity(const float* in, int w, int h, float* out, cudaStream_t s);

// rfg_icp.cu
size_t icp_state_bytes();
void icp_warmup();
cudaError_t launch_icp_track(void* state, const float* depthLevels, int levels, const Intr& in0,
                             const float4* points, const float4* normals, const int* iters, const float* dist,
                             int minCount, const float* w2cInit, const float* renderPose, float* w2cOut,
                             float* renderPoseOut, cudaStream_t s);
cudaError_t launch_icp_reduce_once(void* state, const float* depth, int lw, int lh, const float* f4l, const Intr& in0,
                                   const float4* points, const float4* normals, const float* c2w,
                                   const float* renderPose, float dist, cudaStream_t s);
const double* icp_sums_ptr(void* state);
const long long* icp_fixed_ptr(void* state);
unsigned long long* icp_timers_ptr(void* state);
const double* icp_stats_ptr(void* state);
const int* icp_error_ptr(void* state);
const float* icp_w2c_ptr(void* state);

FrameArgs make_frame_args(const rfg_intrinsics* intr, const rfg_scene_params* p, const float* pose34,
                          const float* poseDev) {
  FrameArgs fa;
  fa.w = intr->width;
  fa.h = intr->height;
  fa.fx = intr->fx;
  fa.fy = intr->fy;
  fa.cx = intr->cx;
  fa.cy = intr->cy;
  fa.voxelSize = p->voxelSize;
  fa.mu = p->mu;
  fa.maxW = p->maxW;
  fa.vfMin = p->viewFrustum_min;
  fa.vfMax = p->viewFrustum_max;
  fa.stopAtMaxW = p->stopIntegratingAtMaxW;
  for (int i = 0; i < 12; ++i) fa.pose[i] = pose34 ? pose34[i] : ((i % 5 == 0) ? 1.f : 0.f);
  fa.poseDev = poseDev;
  fa.swapping = 0;
  fa.swapMargin = 8.f;
  fa.depthBounded = 0;
  return fa;
}

__global__ void k_fill_u32(uint32_t* p, uint32_t v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_fill_u4(uint4* p, uint4 v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_iota(int* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__global__ void k_state_init(MapState* st, int nb, int ne) {
  if (threadIdx.x) return;
  memset(st, 0, sizeof(MapState));
  st->nFreeBlocks = nb;
  st->nFreeExcess = ne;
}
__global__ void k_set12(float* dst, Pose12 p) {
  if (threadIdx.x < 12) dst[threadIdx.x] = p.v[threadIdx.x];
}
__global__ void k_copy12(float* dst, const float* src) {
  if (threadIdx.x < 12) dst[threadIdx.x] = src[threadIdx.x];
}
// A frame's results {MapState, pose (12 floats), ICP stats (8 doubles)}
// written straight into mapped pinned host memory: one launch instead of
// three device-to-host copies on the end-to-end path.
struct FrameResult {
  MapState state;
  float pose[12];
  double icp[RFG_ICP_STATS];
  int icpError;
};
__global__ void k_frame_result(FrameResult* out, const MapState* st, const float* pose, const double* icp,
                               const int* icpError) {
  const int t = threadIdx.x;
  const int* s = reinterpret_cast<const int*>(st);
  int* d = reinterpret_cast<int*>(&out->state);
  for (int i = t; i < (int)(sizeof(MapState) / sizeof(int)); i += blockDim.x) d[i] = s[i];
  if (t < 12) out->pose[t] = pose[t];
  if (t < RFG_ICP_STATS) out->icp[t] = icp[t];
  if (t == 0) out->icpError = *icpError;
}
// Gather VBA blocks (depth + colour planes) into VoxelSRgb byte layout.
__global__ void k_export_blocks(const uint32_t* vbaD, const uint32_t* vbaC, const int* ptrs, int n, uint8_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * kBlock3; i += gridDim.x * blockDim.x) {
    const int b = i / kBlock3, v = i % kBlock3;
    const size_t src = (size_t)ptrs[b] * kBlock3 + v;
    const uint32_t d = vbaD[src];
    const uint32_t c = vbaC ? vbaC[src] : 0u;
    uint8_t* o = out + (size_t)i * 8;
    o[0] = d & 0xFF;
    o[1] = (d >> 8) & 0xFF;
    o[2] = (d >> 16) & 0xFF;
    o[3] = c & 0xFF;
    o[4] = (c >> 8) & 0xFF;
    o[5] = (c >> 16) & 0xFF;
    o[6] = (c >> 24) & 0xFF;
    o[7] = 0;
  }
}
__global__ void k_export_entries(const int4* e, int* out5, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int4 v = e[i];
    out5[5 * i] = entry_x(v);
    out5[5 * i + 1] = entry_y(v);
    out5[5 * i + 2] = entry_z(v);
    out5[5 * i + 3] = v.z;
    out5[5 * i + 4] = v.w;
  }
}

constexpr int kBinCap = 2048;  // blocks per 32x32 screen tile before the overflow path
constexpr size_t kTileScratchBytes = 64 << 10;  // [binCount | tileCost | tileOrder] up to 5,461 screen tiles

int ensure_range_scratch(rfg_map* m, int width, int height) {
  DevMap& d = m->d;
  const int tx = (width + kRangeTilePx - 1) / kRangeTilePx, ty = (height + kRangeTilePx - 1) / kRangeTilePx;
  if (d.bins && d.binTilesX == tx && d.binTilesY >= ty) return RFG_OK;
  // a pipeline's captured frame graph may hold the old bins (and binTilesX):
  // wait for all work on the device, and bump the generation so such graphs
  // are re-captured before their next replay (run_frame)
  RFG_CK(cudaDeviceSynchronize());
  ++d.binGen;
  if (d.bins) cudaFree(d.bins);
  if (d.binCount && d.binCount != m->tileScratch) cudaFree(d.binCount);
  d.bins = nullptr;
  d.binCount = nullptr;
  d.tileCost = nullptr;
  d.tileOrder = nullptr;
  // the per-tile counters carried from frame to frame sit in the map's
  // metadata allocation (the persisting L2 window) when they fit
  const size_t counterBytes = (size_t)tx * ty * 3 * sizeof(int);
  if (counterBytes <= kTileScratchBytes) d.binCount = m->tileScratch;
  if (cudaMalloc(&d.bins, (size_t)tx * ty * kBinCap * sizeof(int)) != cudaSuccess ||
      (!d.binCount && cudaMalloc(&d.binCount, counterBytes) != cudaSuccess)) {
    cudaGetLastError();
    set_error("range scratch allocation failed");
    return RFG_ENOMEM;
  }
  // [binCount | tileCost | tileOrder], tx * ty each
  RFG_CK(cudaMemset(d.binCount, 0, (size_t)tx * ty * 3 * sizeof(int)));
  d.tileCost = d.binCount + (size_t)tx * ty;
  d.tileOrder = d.binCount + (size_t)tx * ty * 2;
  d.binTilesX = tx;
  d.binTilesY = ty;
  d.binCap = kBinCap;
  return RFG_OK;
}

}  // namespace rfg

#ifndef RFG_L2_PERSIST
#define RFG_L2_PERSIST 1  // the map's hash metadata as a persisting L2 access-policy window of the pipeline
#endif

#ifndef RFG_PDL
#define RFG_PDL 1  // programmatic dependent launches in the frame graph's chain
#endif
namespace rfg {
thread_local bool g_pdl = false;
}
using namespace rfg;

namespace {

constexpr float kIcpMaxDist = 2.f;  // fixed-point range of the tracker sums (rfg_icp.cu)

bool valid_intr(const rfg_intrinsics* i) { return i && i->width > 0 && i->height > 0; }
// mu / voxelSize < 80 keeps every pixel's near-far DDA walk (fusion.cpp:72-114)
// under the 64 cells a 6-bit request-key ordinal can name (rfg_alloc.cu:
// k_alloc_stage1); the reference walks any length, so larger ratios are
// rejected here instead of being truncated on the device.
bool valid_params(const rfg_scene_params* p) {
  return p && p->voxelSize > 0.f && p->mu > 0.f && p->mu < 80.f * p->voxelSize;
}

#define RFG_REQUIRE(cond, msg)      \
  do {                              \
    if (!(cond)) {                  \
      rfg::set_error(msg);          \
      return RFG_EINVAL;            \
    }                               \
  } while (0)

int check_device_error(rfg_map* m) {
  RFG_CK(cudaMemcpyAsync(m->hostState, m->d.state, sizeof(MapState), cudaMemcpyDeviceToHost, m->stream));
  RFG_CK(cudaStreamSynchronize(m->stream));
  if (m->hostState->error) {
    const int e = m->hostState->error;
    set_error(std::string("device flagged: ") + ((e & 1) ? "block coordinate outside int16 entry layout " : "") +
              ((e & 2) ? "DDA ordinal bound (64) exceeded" : ""));
    return RFG_ERANGE;
  }
  return RFG_OK;
}

}  // namespace

extern "C" {

const char* rfg_last_error(void) { return t_lastError.c_str(); }
uint64_t rfg_kernel_launch_count(void) { return g_launches.load(); }

int rfg_map_create(const rfg_map_config* cfg, int device, rfg_map** out) {
  RFG_REQUIRE(cfg && out, "null argument");
  *out = nullptr;
  // VoxelBlockMap ctor (voxel_block_map.cpp:10-11); bucketCount 0 is also rejected
  RFG_REQUIRE(cfg->bucketCount != 0 && (cfg->bucketCount & (cfg->bucketCount - 1)) == 0,
              "bucketCount must be a power of two");
  RFG_REQUIRE(cfg->blockCapacity > 0, "blockCapacity must be positive");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error("no CUDA device available (librfg has no CPU fallback)");
    return RFG_ECUDA;
  }
  RFG_REQUIRE(device >= 0 && device < ndev, "no such CUDA device");
  DeviceGuard guard(device);  // the caller's current device is restored on return
  rfg_map* m = new rfg_map();
  memset(&m->d, 0, sizeof(DevMap));
  m->cfg = *cfg;
  m->device = device;
  m->stream = nullptr;
  DevMap& d = m->d;
  d.buckets = cfg->bucketCount;
  d.excess = cfg->excessCount;
  d.capacity = cfg->blockCapacity;
  d.total = d.buckets + d.excess;
  d.nTiles = (int)((d.total + kTile - 1) / kTile);
  const size_t padded = (size_t)d.nTiles * kTile;
  d.world = 1;
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (cudaMalloc(p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  };
  // The per-frame hash metadata — entries, request keys, mark and visibility
  // bytes, tile counts, the map state — in ONE allocation, so that one L2
  // access-policy window covers everything the allocation stages probe
  // (RFG_L2_PERSIST); each part 256-B aligned.
  size_t metaBytes = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = metaBytes;
    metaBytes += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t oEntries = carve(padded * sizeof(int4)), oReq = carve(padded * sizeof(uint32_t)),
               oMarked = carve(padded), oVis = carve(padded), oTiles = carve((size_t)d.nTiles * sizeof(int2)),
               oState = carve(sizeof(MapState)), oTileScratch = carve(kTileScratchBytes);
  char* meta = nullptr;
  bool ok = alloc((void**)&meta, metaBytes);
  if (ok) {
    d.entries = reinterpret_cast<int4*>(meta + oEntries);
    d.reqKey = reinterpret_cast<uint32_t*>(meta + oReq);
    d.marked = reinterpret_cast<uint8_t*>(meta + oMarked);
    d.visibility = reinterpret_cast<uint8_t*>(meta + oVis);
    d.tileCounts = reinterpret_cast<int2*>(meta + oTiles);
    d.state = reinterpret_cast<MapState*>(meta + oState);
    m->tileScratch = reinterpret_cast<int*>(meta + oTileScratch);
    m->metaBytes = metaBytes;
  }
  ok = ok && alloc((void**)&d.vbaDepth, (size_t)d.capacity * kBlock3 * sizeof(uint32_t)) &&
            (!cfg->hasColour || alloc((void**)&d.vbaColour, (size_t)d.capacity * kBlock3 * sizeof(uint32_t))) &&
            alloc((void**)&d.freeBlocks, (size_t)d.capacity * sizeof(int)) &&
            alloc((void**)&d.freeExcess, (size_t)(d.excess ? d.excess : 1) * sizeof(int)) &&
            alloc((void**)&d.visibleList, padded * sizeof(int)) &&
            alloc((void**)&d.tilePrefix, (d.nTiles + 1) * sizeof(int2)) &&
            alloc((void**)&d.rangeBounds, padded * sizeof(int4)) &&
            alloc((void**)&m->icpOut, icp_state_bytes()) && alloc((void**)&m->icpPose, 64 * sizeof(float));
  // the tracker's rotating accumulators must start at zero (rfg_icp.cu:IcpState)
  if (ok && cudaMemset(m->icpOut, 0, icp_state_bytes()) != cudaSuccess) ok = false;
  if (ok && cudaMallocHost((void**)&m->hostState, sizeof(MapState)) != cudaSuccess) {
    cudaGetLastError();
    ok = false;
  }
  if (!ok) {
    rfg_map_destroy(m);
    set_error("device allocation failed");
    return RFG_ENOMEM;
  }
  const int rc = rfg_map_clear(m);
  if (rc != RFG_OK) {
    rfg_map_destroy(m);
    return rc;
  }
  *out = m;
  return RFG_OK;
}

int rfg_map_destroy(rfg_map* m) {
  DeviceGuard dg_(m ? m->device : -1);
  if (!m) return RFG_OK;
  DevMap& d = m->d;
  // (d.entries is the metadata allocation: reqKey, marked, visibility,
  // tileCounts, state and the tile scratch live inside it)
  if (d.binCount == m->tileScratch) d.binCount = nullptr;  // inside the metadata allocation
  void* ptrs[] = {d.entries, d.vbaDepth,   d.vbaColour,  d.freeBlocks,     d.freeExcess, d.visibleList,
                  d.tilePrefix,
                  m->icpOut, m->icpPose, d.rangeBounds, d.bins, d.binCount,
                  m->fwdPrev, m->fwdKeys, m->fwdTileCounts, m->fwdTilePrefix, m->rgbaScratch};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (m->hostState) cudaFreeHost(m->hostState);
  mesh_free(m->mesh);
  delete m;
  return RFG_OK;
}

// VoxelBlockMap::clear (voxel_block_map.cpp:15-24)
int rfg_map_clear(rfg_map* m) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m, "null map");
  DevMap& d = m->d;
  cudaStream_t s = m->stream;
  const size_t padded = (size_t)d.nTiles * kTile;
  const int4 e0 = make_entry(0, 0, 0, 0, -2);
  k_fill_u4<<<1024, 256, 0, s>>>(reinterpret_cast<uint4*>(d.entries), make_uint4(e0.x, e0.y, e0.z, e0.w), padded);
  k_fill_u32<<<4096, 256, 0, s>>>(d.vbaDepth, kDefaultDepthVoxel, (size_t)d.capacity * kBlock3);
  if (d.vbaColour) RFG_CK(cudaMemsetAsync(d.vbaColour, 0, (size_t)d.capacity * kBlock3 * 4, s));
  k_iota<<<512, 256, 0, s>>>(d.freeBlocks, (int)d.capacity);
  if (d.excess) k_iota<<<512, 256, 0, s>>>(d.freeExcess, (int)d.excess);
  RFG_CK(cudaMemsetAsync(d.visibility, 0, padded, s));
  RFG_CK(cudaMemsetAsync(d.marked, 0, padded, s));
  RFG_CK(cudaMemsetAsync(d.reqKey, 0, padded * 4, s));
  RFG_CK(cudaMemsetAsync(d.tileCounts, 0, (size_t)d.nTiles * sizeof(int2), s));  // stage-1 request counts
  k_state_init<<<1, 32, 0, s>>>(d.state, (int)d.capacity, (int)d.excess);
  count_launch(5);
  RFG_CK(cudaGetLastError());
  RFG_CK(cudaStreamSynchronize(s));
  return RFG_OK;
}

int rfg_map_set_stream(rfg_map* m, void* stream) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m, "null map");
  m->stream = static_cast<cudaStream_t>(stream);
  return RFG_OK;
}

int rfg_map_sync(rfg_map* m) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m, "null map");
  RFG_CK(cudaStreamSynchronize(m->stream));
  return check_device_error(m);
}

int rfg_map_set_shard(rfg_map* m, int rank, int world, int tileShift) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && world >= 1 && rank >= 0 && rank < world && tileShift >= 0 && tileShift < 16, "bad shard");
  m->d.rank = rank;
  m->d.world = world;
  m->d.tileShift = tileShift;
  return RFG_OK;
}

int rfg_allocate_from_depth(rfg_map* m, const float* depth, const rfg_intrinsics* intr, const float pose34[12],
                            const rfg_scene_params* params, rfg_alloc_stats* stats) {
  DeviceGuard dg_(m ? m->device : -1);
  return rfg_allocate_from_depth_ex(m, depth, intr, pose34, params, nullptr, stats);
}

int rfg_allocate_from_depth_ex(rfg_map* m, const float* depth, const rfg_intrinsics* intr, const float pose34[12],
                               const rfg_scene_params* params, const rfg_fusion_options* opts,
                               rfg_alloc_stats* stats) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && depth && pose34, "null argument");
  RFG_REQUIRE(valid_intr(intr) && valid_params(params), "invalid intrinsics / scene params");
  RFG_REQUIRE((size_t)intr->width * intr->height < (1u << 25), "image too large for the 25-bit pixel key");
  FrameArgs fa = make_frame_args(intr, params, pose34, nullptr);
  if (opts) {
    fa.swapping = opts->swapping_enabled ? 1 : 0;
    fa.swapMargin = opts->swap_margin_px;
  }
  RFG_CK(launch_allocate(m->d, depth, fa, m->stream));
  if (stats) {
    const int rc = check_device_error(m);  // synchronises, refreshes hostState
    if (rc != RFG_OK) return rc;
    memcpy(stats, m->hostState->stats, sizeof(rfg_alloc_stats));
    stats->visibleCount = m->hostState->nVisible;  // stage 3 appends the list; its length is the count
  }
  return RFG_OK;
}

int rfg_integrate(rfg_map* m, const float* depth, const uint8_t* rgb, const rfg_intrinsics* intrD,
                  const rfg_intrinsics* intrRgb, const float extr34[12], const float pose34[12],
                  const rfg_scene_params* params) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && depth && pose34, "null argument");
  RFG_REQUIRE(valid_intr(intrD) && valid_params(params), "invalid intrinsics / scene params");
  RFG_REQUIRE(!rgb || (m->d.vbaColour && valid_intr(intrRgb)), "colour integration needs a colour map + rgb intrinsics");
  const FrameArgs fa = make_frame_args(intrD, params, pose34, nullptr);
  const uint32_t* rgba = nullptr;
  if (rgb) {
    const int n = intrRgb->width * intrRgb->height;
    if (m->rgbaN < n) {
      RFG_CK(cudaStreamSynchronize(m->stream));
      cudaFree(m->rgbaScratch);
      m->rgbaScratch = nullptr;
      m->rgbaN = 0;
      if (cudaMalloc(&m->rgbaScratch, (size_t)n * 4) != cudaSuccess) {
        cudaGetLastError();
        set_error("colour scratch allocation failed");
        return RFG_ENOMEM;
      }
      m->rgbaN = n;
    }
    RFG_CK(launch_rgb_to_rgba(rgb, m->rgbaScratch, n, m->stream));
    rgba = m->rgbaScratch;
  }
  RFG_CK(launch_integrate(m->d, depth, rgba, fa, intrRgb, extr34, m->stream));
  return RFG_OK;
}

int rfg_render_expected_ranges(rfg_map* m, const float pose34[12], const rfg_intrinsics* intr,
                               const rfg_scene_params* params, float* range) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && pose34 && range, "null argument");
  RFG_REQUIRE(valid_intr(intr) && valid_params(params), "invalid intrinsics / scene params");
  const FrameArgs fa = make_frame_args(intr, params, pose34, nullptr);
  const int rc = ensure_range_scratch(m, intr->width, intr->height);
  if (rc != RFG_OK) return rc;
  RFG_CK(launch_ranges(m->d, fa, reinterpret_cast<float2*>(range), m->stream));
  return RFG_OK;
}

int rfg_render_icp_maps(rfg_map* m, const float pose34[12], const rfg_intrinsics* intr,
                        const rfg_scene_params* params, const float* range, float* raycast, float* points,
                        float* normals) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && pose34 && points && normals, "null argument");
  if (!range) {
    set_error("render_icp_maps needs the expected-range image (render_expected_ranges first)");
    return RFG_ESTATE;
  }
  RFG_REQUIRE(valid_intr(intr) && valid_params(params), "invalid intrinsics / scene params");
  const FrameArgs fa = make_frame_args(intr, params, pose34, nullptr);
  RFG_CK(launch_icp_maps(m->d, fa, reinterpret_cast<const float2*>(range), reinterpret_cast<float4*>(raycast),
                         reinterpret_cast<float4*>(points), reinterpret_cast<float4*>(normals), m->stream));
  return RFG_OK;
}

int rfg_forward_project(rfg_map* m, int hasRaycast, float* raycast, float* points, float* normals,
                        const float newPose34[12], const rfg_intrinsics* intr, float voxelSize, int32_t* missing,
                        int32_t* nMissing) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && raycast && points && normals && newPose34 && missing && nMissing, "null argument");
  RFG_REQUIRE(valid_intr(intr) && voxelSize > 0.f, "invalid intrinsics / voxel size");
  const int n = intr->width * intr->height;
  if (m->fwdN < n) {
    RFG_CK(cudaStreamSynchronize(m->stream));
    cudaFree(m->fwdPrev);
    cudaFree(m->fwdKeys);
    cudaFree(m->fwdTileCounts);
    cudaFree(m->fwdTilePrefix);
    m->fwdPrev = nullptr;  // a failed allocation below must not leave freed pointers for rfg_map_destroy
    m->fwdKeys = nullptr;
    m->fwdTileCounts = nullptr;
    m->fwdTilePrefix = nullptr;
    m->fwdN = 0;
    const int tiles = (n + kTile - 1) / kTile;
    if (cudaMalloc(&m->fwdPrev, (size_t)n * sizeof(float4)) != cudaSuccess ||
        cudaMalloc(&m->fwdKeys, (size_t)n * 8) != cudaSuccess ||
        cudaMalloc(&m->fwdTileCounts, tiles * sizeof(int2)) != cudaSuccess ||
        cudaMalloc(&m->fwdTilePrefix, tiles * sizeof(int2)) != cudaSuccess) {
      cudaGetLastError();
      m->fwdN = 0;
      set_error("forward-projection scratch allocation failed");
      return RFG_ENOMEM;
    }
    m->fwdN = n;
  }
  RFG_CK(launch_forward_project(hasRaycast, reinterpret_cast<float4*>(raycast), reinterpret_cast<float4*>(points),
                                reinterpret_cast<float4*>(normals), newPose34, intr->width, intr->height, intr->fx,
                                intr->fy, intr->cx, intr->cy, voxelSize, m->fwdPrev, m->fwdKeys, m->fwdTileCounts,
                                m->fwdTilePrefix, missing, nMissing, m->stream));
  return RFG_OK;
}

int rfg_render_icp_maps_list(rfg_map* m, const float pose34[12], const rfg_intrinsics* intr,
                             const rfg_scene_params* params, const float* range, const int32_t* missing,
                             const int32_t* nMissing, float* raycast, float* points, float* normals) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && pose34 && missing && nMissing && raycast && points && normals, "null argument");
  if (!range) {
    set_error("render_icp_maps_list needs the expected-range image (render_expected_ranges first)");
    return RFG_ESTATE;
  }
  RFG_REQUIRE(valid_intr(intr) && valid_params(params), "invalid intrinsics / scene params");
  const FrameArgs fa = make_frame_args(intr, params, pose34, nullptr);
  RFG_CK(launch_icp_maps_list(m->d, fa, reinterpret_cast<const float2*>(range), missing, nMissing,
                              intr->width * intr->height, reinterpret_cast<float4*>(raycast),
                              reinterpret_cast<float4*>(points), reinterpret_cast<float4*>(normals), m->stream));
  return RFG_OK;
}

int rfg_render_maps(rfg_map* m, const float pose34[12], const rfg_intrinsics* intr, const rfg_scene_params* params,
                    int mode, const float* range, float* raycast, float* points, float* normals, uint8_t* colour) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0 (kIcpMaps), 1 (kColour) or 2 (kGrey)");
  RFG_REQUIRE(mode == 0 || colour, "colour / grey modes need a colour image");
  RFG_REQUIRE(raycast, "render_maps needs the raycast image (the colour pass reads the hits)");
  const int rc = rfg_render_icp_maps(m, pose34, intr, params, range, raycast, points, normals);
  if (rc != RFG_OK || mode == 0) return rc;
  const FrameArgs fa = make_frame_args(intr, params, pose34, nullptr);
  RFG_CK(launch_render_colour(m->d, fa, mode, reinterpret_cast<const float4*>(raycast),
                              reinterpret_cast<const float4*>(normals), nullptr, nullptr, 0, colour, m->stream));
  return RFG_OK;
}

int rfg_render_maps_list(rfg_map* m, const float pose34[12], const rfg_intrinsics* intr,
                         const rfg_scene_params* params, int mode, const float* range, const int32_t* missing,
                         const int32_t* nMissing, float* raycast, float* points, float* normals, uint8_t* colour) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0 (kIcpMaps), 1 (kColour) or 2 (kGrey)");
  RFG_REQUIRE(mode == 0 || colour, "colour / grey modes need a colour image");
  const int rc = rfg_render_icp_maps_list(m, pose34, intr, params, range, missing, nMissing, raycast, points, normals);
  if (rc != RFG_OK || mode == 0) return rc;
  const FrameArgs fa = make_frame_args(intr, params, pose34, nullptr);
  RFG_CK(launch_render_colour(m->d, fa, mode, reinterpret_cast<const float4*>(raycast),
                              reinterpret_cast<const float4*>(normals), missing, nMissing,
                              intr->width * intr->height, colour, m->stream));
  return RFG_OK;
}

int rfg_extract_mesh(rfg_map* m, float voxelSize, int64_t* nVertices, int64_t* nTriangles) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && nVertices && nTriangles && voxelSize > 0.f, "invalid extract_mesh arguments");
  long long nv = 0, nt = 0;
  RFG_CK(mesh_extract(m->d, voxelSize, &m->mesh, &nv, &nt, m->stream));
  *nVertices = nv;
  *nTriangles = nt;
  return RFG_OK;
}

int rfg_mesh_copy(rfg_map* m, float* vertices3, uint32_t* triangles3) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m, "null map");
  if (!m->mesh) {
    set_error("mesh_copy before extract_mesh");
    return RFG_ESTATE;
  }
  RFG_CK(mesh_copy(m->mesh, vertices3, triangles3, m->stream));
  return RFG_OK;
}

int rfg_mc_table(int32_t counts256[256], int32_t tris[256 * 16 * 3]) {
  RFG_REQUIRE(counts256 && tris, "null argument");
  return mc_table_export(counts256, tris);
}

int rfg_build_view_depth(const uint16_t* raw, int w, int h, float scale, float offset, int levels, float* out,
                         void* stream) {
  // build_view (view.cpp:102-106) rejects levels < 1
  RFG_REQUIRE(raw && out && w > 0 && h > 0 && levels >= 1 && levels <= 4, "invalid build_view arguments");
  RFG_CK(launch_build_view(raw, w, h, scale, offset, levels, out, static_cast<cudaStream_t>(stream)));
  return RFG_OK;
}

int rfg_build_view(const uint16_t* raw, const uint8_t* rgb, const rfg_intrinsics* intr, float scale, float offset,
                   int bilateral, int levels, int rawBigEndian, float* depthLevels, float* intensityLevels,
                   float* normals, float* scratch, void* stream) {
  // build_view (view.cpp:102-106) rejects levels < 1
  RFG_REQUIRE(raw && depthLevels && valid_intr(intr) && levels >= 1 && levels <= 4, "invalid build_view arguments");
  RFG_REQUIRE(!bilateral || scratch, "bilateral needs a scratch image (width*height floats)");
  RFG_REQUIRE(!intensityLevels || rgb, "intensity levels need an rgb image");
  const Intr in{intr->width, intr->height, intr->fx, intr->fy, intr->cx, intr->cy};
  RFG_CK(launch_build_view_full(raw, rgb, in, scale, offset, bilateral, levels, rawBigEndian, depthLevels,
                                intensityLevels, reinterpret_cast<float4*>(normals), scratch,
                                static_cast<cudaStream_t>(stream)));
  return RFG_OK;
}

int rfg_bilateral_filter(const float* in, int w, int h, float spatialSigma, float rangeSigma, float* out,
                         void* stream) {
  RFG_REQUIRE(in && out && in != out && w > 0 && h > 0, "invalid bilateral_filter arguments");
  RFG_CK(launch_bilateral(in, w, h, spatialSigma, rangeSigma, out, static_cast<cudaStream_t>(stream)));
  return RFG_OK;
}

int rfg_compute_normals(const float* depth, const rfg_intrinsics* intr, float* normals, void* stream) {
  RFG_REQUIRE(depth && normals && valid_intr(intr), "invalid compute_normals arguments");
  const Intr in{intr->width, intr->height, intr->fx, intr->fy, intr->cx, intr->cy};
  RFG_CK(launch_view_normals(depth, in, reinterpret_cast<float4*>(normals), static_cast<cudaStream_t>(stream)));
  return RFG_OK;
}

int rfg_rgb_to_intensity(const uint8_t* rgb, int w, int h, float* out, void* stream) {
  RFG_REQUIRE(rgb && out && w > 0 && h > 0, "invalid rgb_to_intensity arguments");
  RFG_CK(launch_intensity(rgb, w, h, out, static_cast<cudaStream_t>(stream)));
  return RFG_OK;
}

int rfg_downsample_intensity(const float* in, int w, int h, float* out, void* stream) {
  RFG_REQUIRE(in && out && w > 0 && h > 0, "invalid downsample_intensity arguments");
  RFG_CK(launch_downsample_intensity(in, w, h, out, static_cast<cudaStream_t>(stream)));
  return RFG_OK;
}

int rfg_icp_track(rfg_map* m, const float* depthLevels, int levels, const rfg_intrinsics* intr, const float* points,
                  const float* normals, const float renderPose34[12], const float initPose34[12], const int iters[3],
                  const float dist[3], int minCount, float poseOut34[12], double stats12[RFG_ICP_STATS]) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && depthLevels && points && normals && renderPose34 && initPose34 && iters && dist,
              "null argument");
  RFG_REQUIRE(valid_intr(intr) && levels >= 1 && levels <= 3, "invalid intrinsics / levels");
  for (int l = 0; l < levels; ++l)
    RFG_REQUIRE(dist[l] > 0.f && dist[l] <= kIcpMaxDist, "ICP outlier gates must be in (0, 2] m");
  float host[24];
  memcpy(host, initPose34, 48);
  memcpy(host + 12, renderPose34, 48);
  RFG_CK(cudaMemcpyAsync(m->icpPose, host, sizeof(host), cudaMemcpyHostToDevice, m->stream));
  const Intr in0{intr->width, intr->height, intr->fx, intr->fy, intr->cx, intr->cy};
  RFG_CK(launch_icp_track(m->icpOut, depthLevels, levels, in0, reinterpret_cast<const float4*>(points),
                          reinterpret_cast<const float4*>(normals), iters, dist, minCount, m->icpPose,
                          m->icpPose + 12, m->icpPose + 24, nullptr, m->stream));
  double st[RFG_ICP_STATS];
  float pose[12];
  int err = 0;
  RFG_CK(cudaMemcpyAsync(st, icp_stats_ptr(m->icpOut), sizeof(st), cudaMemcpyDeviceToHost, m->stream));
  RFG_CK(cudaMemcpyAsync(pose, m->icpPose + 24, sizeof(pose), cudaMemcpyDeviceToHost, m->stream));
  RFG_CK(cudaMemcpyAsync(&err, icp_error_ptr(m->icpOut), sizeof(int), cudaMemcpyDeviceToHost, m->stream));
  RFG_CK(cudaStreamSynchronize(m->stream));
  if (err) {
    set_error("ICP: a world point outside the fixed-point range (|p| components >= 128 m)");
    return RFG_ERANGE;
  }
  if (poseOut34) memcpy(poseOut34, pose, sizeof(pose));
  if (stats12) memcpy(stats12, st, sizeof(st));
  return RFG_OK;
}

int rfg_icp_reduce(rfg_map* m, const float* depthLevel, int level, const rfg_intrinsics* intr, const float* points,
                   const float* normals, const float renderPose34[12], const float camToWorld34[12], float dist,
                   int64_t fixed31[RFG_ICP_SUMS], double out31[RFG_ICP_SUMS]) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && depthLevel && points && normals && renderPose34 && camToWorld34, "null argument");
  RFG_REQUIRE(valid_intr(intr) && level >= 0 && level < 4, "invalid intrinsics / level");
  RFG_REQUIRE(dist > 0.f && dist <= kIcpMaxDist, "ICP outlier gate must be in (0, 2] m");
  float host[24];
  memcpy(host, camToWorld34, 48);
  memcpy(host + 12, renderPose34, 48);
  RFG_CK(cudaMemcpyAsync(m->icpPose, host, sizeof(host), cudaMemcpyHostToDevice, m->stream));
  const Intr in0{intr->width, intr->height, intr->fx, intr->fy, intr->cx, intr->cy};
  const float sc = ldexpf(1.f, -level);
  const float f4l[4] = {intr->fx * sc, intr->fy * sc, intr->cx * sc, intr->cy * sc};
  RFG_CK(launch_icp_reduce_once(m->icpOut, depthLevel, intr->width >> level, intr->height >> level, f4l, in0,
                                reinterpret_cast<const float4*>(points), reinterpret_cast<const float4*>(normals),
                                m->icpPose, m->icpPose + 12, dist, m->stream));
  int err = 0;
  if (out31)
    RFG_CK(cudaMemcpyAsync(out31, icp_sums_ptr(m->icpOut), RFG_ICP_SUMS * sizeof(double), cudaMemcpyDeviceToHost,
                           m->stream));
  if (fixed31)
    RFG_CK(cudaMemcpyAsync(fixed31, icp_fixed_ptr(m->icpOut), RFG_ICP_SUMS * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, m->stream));
  RFG_CK(cudaMemcpyAsync(&err, icp_error_ptr(m->icpOut), sizeof(int), cudaMemcpyDeviceToHost, m->stream));
  RFG_CK(cudaStreamSynchronize(m->stream));
  if (err) {
    set_error("ICP: a world point outside the fixed-point range (|p| components >= 128 m)");
    return RFG_ERANGE;
  }
  return RFG_OK;
}

int rfg_icp_timers(rfg_map* m, uint64_t out8[8], int reset) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && out8, "null argument");
  unsigned long long* t = icp_timers_ptr(m->icpOut);
  RFG_CK(cudaMemcpyAsync(out8, t, 64, cudaMemcpyDeviceToHost, m->stream));
  if (reset) RFG_CK(cudaMemsetAsync(t, 0, 64, m->stream));
  RFG_CK(cudaStreamSynchronize(m->stream));
  return RFG_OK;
}

uint32_t rfg_total_entries(const rfg_map* m) { return m ? m->d.total : 0; }

int rfg_export_entries(rfg_map* m, int32_t* out5) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && out5, "null argument");
  int* dbuf = nullptr;
  RFG_CK(cudaMalloc(&dbuf, (size_t)m->d.total * 5 * sizeof(int)));
  k_export_entries<<<1024, 256, 0, m->stream>>>(m->d.entries, dbuf, (int)m->d.total);
  count_launch();
  cudaMemcpyAsync(out5, dbuf, (size_t)m->d.total * 5 * sizeof(int), cudaMemcpyDeviceToHost, m->stream);
  cudaError_t e = cudaStreamSynchronize(m->stream);
  cudaFree(dbuf);
  RFG_CK(e);
  return check_device_error(m);
}

int rfg_export_blocks(rfg_map* m, const int32_t* ptrs, int n, uint8_t* out) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && (n == 0 || (ptrs && out)) && n >= 0, "null argument");
  if (n == 0) return RFG_OK;
  for (int i = 0; i < n; ++i) RFG_REQUIRE(ptrs[i] >= 0 && (uint32_t)ptrs[i] < m->d.capacity, "block ptr out of range");
  int* dptrs = nullptr;
  uint8_t* dout = nullptr;
  RFG_CK(cudaMalloc(&dptrs, n * sizeof(int)));
  if (cudaMalloc(&dout, (size_t)n * kBlock3 * 8) != cudaSuccess) {
    cudaFree(dptrs);
    set_error("export buffer allocation failed");
    return RFG_ENOMEM;
  }
  cudaMemcpyAsync(dptrs, ptrs, n * sizeof(int), cudaMemcpyHostToDevice, m->stream);
  k_export_blocks<<<1024, 256, 0, m->stream>>>(m->d.vbaDepth, m->d.vbaColour, dptrs, n, dout);
  count_launch();
  cudaMemcpyAsync(out, dout, (size_t)n * kBlock3 * 8, cudaMemcpyDeviceToHost, m->stream);
  cudaError_t e = cudaStreamSynchronize(m->stream);
  cudaFree(dptrs);
  cudaFree(dout);
  RFG_CK(e);
  return RFG_OK;
}

int rfg_export_visible(rfg_map* m, int32_t* list, uint8_t* types, int32_t* count) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && count, "null argument");
  const int rc = check_device_error(m);
  if (rc != RFG_OK) return rc;
  const int n = m->hostState->nVisible;
  *count = n;
  if (list && n) {
    RFG_CK(launch_sort_visible(m->d, m->stream));
    RFG_CK(cudaMemcpyAsync(list, m->d.visibleList, n * sizeof(int), cudaMemcpyDeviceToHost, m->stream));
  }
  if (types) RFG_CK(cudaMemcpyAsync(types, m->d.visibility, m->d.total, cudaMemcpyDeviceToHost, m->stream));
  RFG_CK(cudaStreamSynchronize(m->stream));
  return RFG_OK;
}

int rfg_free_counts(rfg_map* m, int32_t* nb, int32_t* ne) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && nb && ne, "null argument");
  const int rc = check_device_error(m);
  if (rc != RFG_OK) return rc;
  *nb = m->hostState->nFreeBlocks;
  *ne = m->hostState->nFreeExcess;
  return RFG_OK;
}

// ------------------------------------------------------------- pipeline
}  // extern "C"

struct rfg_pipeline {
  rfg_map* map;
  rfg_pipeline_config cfg;
  cudaStream_t stream;
  uint16_t* rawDev;
  float* depthLevels;
  float2* range;
  float4* raycast;
  float4* points;
  float4* normals;
  float* poses;  // [0..11] current w2c, [12..23] render pose of the last raycast
  FrameResult* hostResult;  // mapped pinned: k_frame_result's target
  FrameResult* resultDev;   // its device address (the frame graph's last node writes it)
  float* viewScratch;  // unfiltered depth when cfg.bilateral
  void* pgmStage;      // pinned staging for rfg_pipeline_process_pgm
  cudaEvent_t stageFree;  // the last upload out of pgmStage has been read
  cudaEvent_t rawReady;   // producer stream -> pipeline stream (process_raw_stream)
  cudaEvent_t rawRead;    // pipeline stream has copied the caller's frame
  cudaStream_t side;      // the frame's second branch (range binning + results, beside the integration)
  cudaEvent_t fork, join;
  int frames;
  cudaGraphExec_t exec[2];  // [0] no tracking, [1] tracking
  cudaGraph_t graph[2];     // kept for the view node's handle
  cudaGraphNode_t viewNode[2];            // the k_view_pyramid node (fused view only)
  cudaKernelNodeParams viewParams[2];     // its launch shape
  const uint16_t* viewRaw[2];             // the raw frame it reads now
  uint64_t graphKernels[2];
  cudaEvent_t ev[7];        // stage boundaries (profile mode)
  bool tracked;             // last frame ran the tracker
  // colour pipelines: the RGB8 frame is packed to RGBA8 words by the graph's
  // k_rgb_to_rgba node, which reads the caller's image in place (re-pointed
  // like the view node); rgbDev holds copied-in frames
  uint8_t* rgbDev;
  uint32_t* rgba;
  cudaGraphNode_t rgbNode[2];
  cudaKernelNodeParams rgbParams[2];
  const uint8_t* rgbSrc[2];
  unsigned binGen[2];  // the map's range-scratch generation each graph captured
};

namespace {

#ifndef RFG_FRAME_FORK
#define RFG_FRAME_FORK 1  // the frame's results on a second graph branch (range binning there too measured slower)
#endif
#define RFG_TRY(x)                          \
  do {                                      \
    const cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return e_;       \
  } while (0)
cudaError_t launch_frame_result(rfg_pipeline* p, cudaStream_t s);

cudaError_t enqueue_frame(rfg_pipeline* p, bool track) {
  // the chain after the tracker with programmatic dependent launches
  // (not in profile mode: its event nodes sit between the kernels)
  struct PdlScope {
    explicit PdlScope(bool on) { g_pdl = on; }
    ~PdlScope() { g_pdl = false; }
  } pdlScope_(RFG_PDL != 0 && p->cfg.profile == 0);
  rfg_map* m = p->map;
  const rfg_pipeline_config& c = p->cfg;
  cudaStream_t s = p->stream;
  // profile mode: events between the stages; under capture they become
  // event-record nodes of the frame graph, so the stage times are those of
  // the graph replay itself
  const bool prof = c.profile != 0;
  auto mark = [&](int k) {
    if (prof) cudaEventRecordWithFlags(p->ev[k], s, c.use_graph ? cudaEventRecordExternal : cudaEventRecordDefault);
  };
  mark(0);
  const Intr inV{c.intr.width, c.intr.height, c.intr.fx, c.intr.fy, c.intr.cx, c.intr.cy};
  cudaError_t e = launch_build_view_full(p->rawDev, nullptr, inV, c.aff_scale, c.aff_offset, c.bilateral, c.levels,
                                         c.raw_big_endian, p->depthLevels, nullptr, nullptr, p->viewScratch, s);
  if (e != cudaSuccess) return e;
  mark(1);
  if (track) {
    const Intr in0{c.intr.width, c.intr.height, c.intr.fx, c.intr.fy, c.intr.cx, c.intr.cy};
    e = launch_icp_track(m->icpOut, p->depthLevels, c.levels, in0, p->points, p->normals, c.iters,
                         c.dist, c.min_count, p->poses, p->poses + 12, p->poses, p->poses + 12, s);
    if (e != cudaSuccess) return e;
  }
  mark(2);
  FrameArgs fa = make_frame_args(&c.intr, &c.params, nullptr, p->poses);
  // the frame's depths are raw u16 * scale + offset (view kernels): bounded
  fa.depthBounded = 65535.0 * fabs((double)c.aff_scale) + fabs((double)c.aff_offset) < 0x1p36 ? 1 : 0;
  if ((e = launch_allocate(m->d, p->depthLevels, fa, s)) != cudaSuccess) return e;
  mark(3);
#if RFG_FRAME_FORK
  // the frame's results (the map state is final after the allocation) on a
  // second graph branch, off the critical path; the raycast joins it
  if (!prof) {
    RFG_TRY(cudaEventRecord(p->fork, s));
    RFG_TRY(cudaStreamWaitEvent(p->side, p->fork, 0));
    if ((e = launch_frame_result(p, p->side)) != cudaSuccess) return e;
    RFG_TRY(cudaEventRecord(p->join, p->side));
  }
#endif
  if (c.colour) {
    const int nRgb = c.intr_rgb.width * c.intr_rgb.height;
    if ((e = launch_rgb_to_rgba(p->rgbDev, p->rgba, nRgb, s)) != cudaSuccess) return e;
    if ((e = launch_integrate(m->d, p->depthLevels, p->rgba, fa, &c.intr_rgb, c.extr_d_to_rgb, s)) != cudaSuccess)
      return e;
  } else if ((e = launch_integrate(m->d, p->depthLevels, nullptr, fa, nullptr, nullptr, s)) != cudaSuccess) {
    return e;
  }
  mark(4);
  // expected ranges + ICP maps: the range tiles are reduced inside the
  // raycast's CTAs (profile mode: "ranges" = the binning, "raycast" = the rest)
  if ((e = launch_range_bin(m->d, fa, s)) != cudaSuccess) return e;
  mark(5);
  if ((e = launch_raycast_tiles(m->d, fa, p->range, p->raycast, p->points, p->normals, s)) != cudaSuccess) return e;
  if (!track) {  // a tracked frame's next render pose was written by the tracker
    k_copy12<<<1, 32, 0, s>>>(p->poses + 12, p->poses);
    count_launch();
  }
  mark(6);
#if RFG_FRAME_FORK
  if (!prof) {
    RFG_TRY(cudaStreamWaitEvent(s, p->join, 0));
    return cudaGetLastError();
  }
#endif
  return launch_frame_result(p, s);
}

// The frame's results (map state after the allocation, pose, tracker
// summary) into the mapped host buffer: rfg_pipeline_result only waits.
cudaError_t launch_frame_result(rfg_pipeline* p, cudaStream_t s) {
  rfg_map* m = p->map;
  k_frame_result<<<1, 32, 0, s>>>(p->resultDev, m->d.state, p->poses, icp_stats_ptr(m->icpOut),
                                  icp_error_ptr(m->icpOut));
  count_launch();
  return cudaGetLastError();
}

// Point the frame graph's view kernel at a device raw frame (no copy).
cudaError_t set_view_raw(rfg_pipeline* p, int gi, const uint16_t* raw) {
  if (p->viewRaw[gi] == raw) return cudaSuccess;
  const rfg_pipeline_config& c = p->cfg;
  const uint16_t* r = raw;
  int w = c.intr.width, h = c.intr.height, be = c.raw_big_endian, lv = c.levels;
  float sc = c.aff_scale, of = c.aff_offset;
  float* out = p->depthLevels;
  void* args[] = {&r, &w, &h, &sc, &of, &be, &lv, &out};  // k_view_pyramid's parameters
  cudaKernelNodeParams kp = p->viewParams[gi];
  kp.kernelParams = args;
  kp.extra = nullptr;
  const cudaError_t e = cudaGraphExecKernelNodeSetParams(p->exec[gi], p->viewNode[gi], &kp);
  if (e == cudaSuccess) p->viewRaw[gi] = raw;
  return e;
}

// Point the frame graph's colour packing kernel at an RGB8 frame (no copy).
cudaError_t set_rgb_src(rfg_pipeline* p, int gi, const uint8_t* rgb) {
  if (p->rgbSrc[gi] == rgb) return cudaSuccess;
  const uint8_t* r = rgb;
  uint32_t* out = p->rgba;
  int n = p->cfg.intr_rgb.width * p->cfg.intr_rgb.height;
  void* args[] = {&r, &out, &n};  // k_rgb_to_rgba's parameters
  cudaKernelNodeParams kp = p->rgbParams[gi];
  kp.kernelParams = args;
  kp.extra = nullptr;
  const cudaError_t e = cudaGraphExecKernelNodeSetParams(p->exec[gi], p->rgbNode[gi], &kp);
  if (e == cudaSuccess) p->rgbSrc[gi] = rgb;
  return e;
}

int run_frame(rfg_pipeline* p, const float* pose34, const uint16_t* rawSrc, const uint8_t* rgbSrc = nullptr) {
  const bool track = p->cfg.track && p->frames > 0;
  p->tracked = track;
  if (pose34) {
    Pose12 pv;
    memcpy(pv.v, pose34, 48);
    k_set12<<<1, 32, 0, p->stream>>>(p->poses, pv);
    count_launch();
  }
  // the map's range scratch may have been reallocated for another image size
  // (a map-level render): size it for this pipeline again, and re-capture a
  // graph that holds the old scratch (no replay of freed bins)
  if (ensure_range_scratch(p->map, p->cfg.intr.width, p->cfg.intr.height) != RFG_OK) return RFG_ENOMEM;
  for (int k = 0; k < 2; ++k) {
    if (p->exec[k] && p->binGen[k] != p->map->d.binGen) {
      cudaGraphExecDestroy(p->exec[k]);
      cudaGraphDestroy(p->graph[k]);
      p->exec[k] = nullptr;
      p->graph[k] = nullptr;
      p->viewNode[k] = nullptr;
      p->rgbNode[k] = nullptr;
    }
  }
  if (!p->cfg.use_graph) {
    if (p->cfg.colour && rgbSrc && rgbSrc != p->rgbDev)
      RFG_CK(cudaMemcpyAsync(p->rgbDev, rgbSrc, (size_t)p->cfg.intr_rgb.width * p->cfg.intr_rgb.height * 3,
                             cudaMemcpyDefault, p->stream));
    RFG_CK(enqueue_frame(p, track));
  } else {
    const int gi = track ? 1 : 0;
    if (!p->exec[gi]) {
      cudaGraph_t g;
      const uint64_t before = g_launches.load();
      RFG_CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
      cudaError_t e = enqueue_frame(p, track);
      cudaError_t e2 = cudaStreamEndCapture(p->stream, &g);
      RFG_CK(e);
      RFG_CK(e2);
      p->graphKernels[gi] = g_launches.load() - before;
      g_launches.fetch_sub(p->graphKernels[gi]);  // capture does not launch
      RFG_CK(cudaGraphInstantiate(&p->exec[gi], g, 0));
      p->graph[gi] = g;
      p->binGen[gi] = p->map->d.binGen;
      p->viewRaw[gi] = p->rawDev;
      p->rgbSrc[gi] = p->rgbDev;
      const bool fusedView = view_is_fused(p->cfg.bilateral, false, false, p->cfg.levels);
      size_t nn = 0;
      cudaGraphGetNodes(g, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(g, nodes.data(), &nn);
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        cudaKernelNodeParams kp{};
        if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel ||
            cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess)
          continue;
        if (fusedView && kp.func == view_pyramid_kernel()) {
          p->viewNode[gi] = nd;
          p->viewParams[gi] = kp;
        } else if (p->cfg.colour && kp.func == rgb_to_rgba_kernel()) {
          p->rgbNode[gi] = nd;
          p->rgbParams[gi] = kp;
        }
      }
      cudaGetLastError();
    }
    if (p->viewNode[gi]) RFG_CK(set_view_raw(p, gi, rawSrc));
    if (p->rgbNode[gi]) RFG_CK(set_rgb_src(p, gi, rgbSrc ? rgbSrc : p->rgbDev));
    RFG_CK(cudaGraphLaunch(p->exec[gi], p->stream));
    count_launch(p->graphKernels[gi]);
  }
  ++p->frames;
  return RFG_OK;
}

}  // namespace

extern "C" {

int rfg_pipeline_create(rfg_map* m, const rfg_pipeline_config* cfg, rfg_pipeline** out) {
  DeviceGuard dg_(m ? m->device : -1);
  RFG_REQUIRE(m && cfg && out, "null argument");
  RFG_REQUIRE(valid_intr(&cfg->intr) && valid_params(&cfg->params), "invalid intrinsics / scene params");
  RFG_REQUIRE(cfg->levels >= 1 && cfg->levels <= 3, "levels must be 1..3");
  RFG_REQUIRE(!cfg->track || cfg->levels >= 1, "tracking needs a pyramid");
  for (int l = 0; l < cfg->levels; ++l)
    RFG_REQUIRE(!cfg->track || (cfg->dist[l] > 0.f && cfg->dist[l] <= kIcpMaxDist),
                "ICP outlier gates must be in (0, 2] m");
  RFG_REQUIRE((size_t)cfg->intr.width * cfg->intr.height < (1u << 25), "image too large for the 25-bit pixel key");
  RFG_REQUIRE(!cfg->colour || (m->d.vbaColour && valid_intr(&cfg->intr_rgb)),
              "a colour pipeline needs a colour map and valid rgb intrinsics");
  *out = nullptr;
  rfg_pipeline* p = new rfg_pipeline();
  memset(p, 0, sizeof(*p));
  p->map = m;
  p->cfg = *cfg;
  const size_t n = (size_t)cfg->intr.width * cfg->intr.height;
  size_t lv = 0;
  for (int l = 0; l < cfg->levels; ++l) lv += (size_t)(cfg->intr.width >> l) * (cfg->intr.height >> l);
  bool ok = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMalloc(&p->rawDev, n * 2 + 16) == cudaSuccess &&
            cudaMalloc(&p->depthLevels, lv * 4 + 16) == cudaSuccess &&
            cudaMalloc(&p->range, n * sizeof(float2)) == cudaSuccess &&
            // raycast | points | normals in one allocation, so a sharded
            // rank composes all three with one in-place collective
            cudaMalloc(&p->raycast, 3 * n * sizeof(float4)) == cudaSuccess &&
            cudaMalloc(&p->poses, 32 * sizeof(float)) == cudaSuccess &&
            cudaHostAlloc(&p->hostResult, sizeof(FrameResult), cudaHostAllocMapped) == cudaSuccess &&
            cudaMallocHost(&p->pgmStage, n * 2 + 16) == cudaSuccess &&
            (!cfg->bilateral || cudaMalloc(&p->viewScratch, n * 4 + 16) == cudaSuccess) &&
            (!cfg->colour ||
             (cudaMalloc(&p->rgbDev, (size_t)cfg->intr_rgb.width * cfg->intr_rgb.height * 3 + 16) == cudaSuccess &&
              cudaMalloc(&p->rgba, (size_t)cfg->intr_rgb.width * cfg->intr_rgb.height * 4 + 16) == cudaSuccess));
  if (!ok) {
    cudaGetLastError();
    rfg_pipeline_destroy(p);
    set_error("pipeline allocation failed");
    return RFG_ENOMEM;
  }
  p->points = p->raycast + n;
  p->normals = p->raycast + 2 * n;
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->resultDev), p->hostResult, 0) != cudaSuccess) ok = false;
  memset(p->hostResult, 0, sizeof(FrameResult));  // result() before any frame: zeros
  for (int k = 0; k < 7; ++k)
    if (cudaEventCreate(&p->ev[k]) != cudaSuccess) ok = false;
  if (cudaEventCreateWithFlags(&p->stageFree, cudaEventDisableTiming) != cudaSuccess) ok = false;
  if (cudaEventCreateWithFlags(&p->rawReady, cudaEventDisableTiming) != cudaSuccess) ok = false;
  if (cudaEventCreateWithFlags(&p->rawRead, cudaEventDisableTiming) != cudaSuccess) ok = false;
  if (cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming) != cudaSuccess) ok = false;
  if (cudaEventCreateWithFlags(&p->join, cudaEventDisableTiming) != cudaSuccess) ok = false;
  if (cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking) != cudaSuccess) ok = false;
  if (!ok) {
    cudaGetLastError();
    rfg_pipeline_destroy(p);
    set_error("pipeline event creation failed");
    return RFG_ECUDA;
  }
  m->stream = p->stream;
  icp_warmup();
#if RFG_L2_PERSIST
  // L2 residency control: the map's hash metadata (entries: every stage's
  // lookups and probes; request keys, mark / visibility bytes, tile counts,
  // state: the allocation stages) as a persisting access-policy window on the
  // pipeline's stream
  // (captured into the frame graph's kernel nodes), within the device's
  // persisting set-aside
  {
    int maxPersist = 0, maxWindow = 0;
    cudaDeviceGetAttribute(&maxPersist, cudaDevAttrMaxPersistingL2CacheSize, m->device);
    cudaDeviceGetAttribute(&maxWindow, cudaDevAttrMaxAccessPolicyWindowSize, m->device);
    const size_t bytes = m->metaBytes;  // entries first, then the other per-frame metadata
    if (maxPersist > 0 && maxWindow > 0) {
      const size_t setAside = bytes < (size_t)maxPersist ? bytes : (size_t)maxPersist;
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setAside);
      cudaStreamAttrValue av{};
      av.accessPolicyWindow.base_ptr = m->d.entries;
      av.accessPolicyWindow.num_bytes = bytes < (size_t)maxWindow ? bytes : (size_t)maxWindow;
      av.accessPolicyWindow.hitRatio = (float)setAside / (float)av.accessPolicyWindow.num_bytes;
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(p->stream, cudaStreamAttributeAccessPolicyWindow, &av);
      cudaStreamSetAttribute(p->side, cudaStreamAttributeAccessPolicyWindow, &av);
    }
    cudaGetLastError();
  }
#endif
  if (ensure_range_scratch(m, cfg->intr.width, cfg->intr.height) != RFG_OK) {
    rfg_pipeline_destroy(p);
    return RFG_ENOMEM;
  }
  const int rc = rfg_pipeline_reset(p);
  if (rc != RFG_OK) {
    rfg_pipeline_destroy(p);
    return rc;
  }
  *out = p;
  return RFG_OK;
}

int rfg_pipeline_destroy(rfg_pipeline* p) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  if (!p) return RFG_OK;
  if (p->stream) cudaStreamSynchronize(p->stream);
#if RFG_L2_PERSIST
  cudaCtxResetPersistingL2Cache();  // the window's lines back to normal
#endif
  for (int i = 0; i < 2; ++i)
    if (p->exec[i]) cudaGraphExecDestroy(p->exec[i]);
  for (int i = 0; i < 2; ++i)
    if (p->graph[i]) cudaGraphDestroy(p->graph[i]);
  void* ptrs[] = {p->rawDev, p->depthLevels, p->range, p->raycast, p->poses, p->viewScratch, p->rgbDev, p->rgba};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (int k = 0; k < 7; ++k)
    if (p->ev[k]) cudaEventDestroy(p->ev[k]);
  if (p->stageFree) cudaEventDestroy(p->stageFree);
  if (p->rawReady) cudaEventDestroy(p->rawReady);
  if (p->rawRead) cudaEventDestroy(p->rawRead);
  if (p->fork) cudaEventDestroy(p->fork);
  if (p->join) cudaEventDestroy(p->join);
  if (p->side) {
    cudaStreamSynchronize(p->side);
    cudaStreamDestroy(p->side);
  }
  if (p->hostResult) cudaFreeHost(p->hostResult);
  if (p->pgmStage) cudaFreeHost(p->pgmStage);
  if (p->map && p->map->stream == p->stream) p->map->stream = nullptr;
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
  return RFG_OK;
}

int rfg_pipeline_reset(rfg_pipeline* p) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p, "null pipeline");
  Pose12 id{};
  id.v[0] = id.v[5] = id.v[10] = 1.f;
  k_set12<<<1, 32, 0, p->stream>>>(p->poses, id);
  k_set12<<<1, 32, 0, p->stream>>>(p->poses + 12, id);
  count_launch(2);
  RFG_CK(cudaGetLastError());
  RFG_CK(cudaStreamSynchronize(p->stream));
  p->frames = 0;
  return RFG_OK;
}

int rfg_pipeline_process_raw(rfg_pipeline* p, const uint16_t* raw, const float* pose34) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && raw, "null argument");
  RFG_REQUIRE(!p->cfg.colour, "a colour pipeline takes RGB-D frames (rfg_pipeline_process_rgbd_*)");
  const size_t n = (size_t)p->cfg.intr.width * p->cfg.intr.height;
  if (raw != p->rawDev) RFG_CK(cudaMemcpyAsync(p->rawDev, raw, n * 2, cudaMemcpyDeviceToDevice, p->stream));
  return run_frame(p, pose34, p->rawDev);
}

int rfg_pipeline_process_raw_stream(rfg_pipeline* p, const uint16_t* raw, const float* pose34, void* producer) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && raw, "null argument");
  RFG_REQUIRE(!p->cfg.colour, "a colour pipeline takes RGB-D frames (rfg_pipeline_process_rgbd_*)");
  cudaStream_t ps = static_cast<cudaStream_t>(producer);
  const size_t n = (size_t)p->cfg.intr.width * p->cfg.intr.height;
  // the frame is read after the producer's pending work (its upload) ...
  RFG_CK(cudaEventRecord(p->rawReady, ps));
  RFG_CK(cudaStreamWaitEvent(p->stream, p->rawReady, 0));
  // a captured frame graph with the fused view reads the caller's frame in
  // place (its view node is re-pointed); otherwise the frame is copied in
  const int gi = (p->cfg.track && p->frames > 0) ? 1 : 0;
  const bool direct = p->cfg.use_graph && p->exec[gi] && p->viewNode[gi];
  if (!direct && raw != p->rawDev)
    RFG_CK(cudaMemcpyAsync(p->rawDev, raw, n * 2, cudaMemcpyDeviceToDevice, p->stream));
  const int rc = run_frame(p, pose34, direct ? raw : p->rawDev);
  // ... and the producer's later work (e.g. reusing the buffer) waits until
  // the frame has been read
  RFG_CK(cudaEventRecord(p->rawRead, p->stream));
  RFG_CK(cudaStreamWaitEvent(ps, p->rawRead, 0));
  return rc;
}

#ifndef RFG_HOST_ZEROCOPY
#define RFG_HOST_ZEROCOPY 0  // 1: pinned host frames read in place by the graph's view kernel (measured no faster than the copy)
#endif
int rfg_pipeline_process_host(rfg_pipeline* p, const uint16_t* rawHost, const float* pose34) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && rawHost, "null argument");
  RFG_REQUIRE(!p->cfg.colour, "a colour pipeline takes RGB-D frames (rfg_pipeline_process_rgbd_*)");
  const size_t n = (size_t)p->cfg.intr.width * p->cfg.intr.height;
  // a pinned (device-mapped) host frame is read over PCIe by the captured
  // graph's view kernel itself — no separate DMA and no copy->graph gap;
  // pageable frames, and frames before the graph exists, are copied in
  const int gi = (p->cfg.track && p->frames > 0) ? 1 : 0;
  if (RFG_HOST_ZEROCOPY && p->cfg.use_graph && p->exec[gi] && p->viewNode[gi]) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, rawHost) == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer)
      return run_frame(p, pose34, static_cast<const uint16_t*>(a.devicePointer));
    cudaGetLastError();
  }
  RFG_CK(cudaMemcpyAsync(p->rawDev, rawHost, n * 2, cudaMemcpyHostToDevice, p->stream));
  return run_frame(p, pose34, p->rawDev);
}

int rfg_pipeline_process_rgbd_stream(rfg_pipeline* p, const uint16_t* raw, const uint8_t* rgb, const float* pose34,
                                     void* producer) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && raw && rgb, "null argument");
  RFG_REQUIRE(p->cfg.colour, "rgbd frames need a colour pipeline (cfg.colour = 1)");
  cudaStream_t ps = static_cast<cudaStream_t>(producer);
  const size_t n = (size_t)p->cfg.intr.width * p->cfg.intr.height;
  RFG_CK(cudaEventRecord(p->rawReady, ps));
  RFG_CK(cudaStreamWaitEvent(p->stream, p->rawReady, 0));
  const int gi = (p->cfg.track && p->frames > 0) ? 1 : 0;
  const bool direct = p->cfg.use_graph && p->exec[gi] && p->viewNode[gi] && p->rgbNode[gi];
  if (!direct) {
    if (raw != p->rawDev) RFG_CK(cudaMemcpyAsync(p->rawDev, raw, n * 2, cudaMemcpyDeviceToDevice, p->stream));
    if (rgb != p->rgbDev)
      RFG_CK(cudaMemcpyAsync(p->rgbDev, rgb, (size_t)p->cfg.intr_rgb.width * p->cfg.intr_rgb.height * 3,
                             cudaMemcpyDeviceToDevice, p->stream));
  }
  const int rc = direct ? run_frame(p, pose34, raw, rgb) : run_frame(p, pose34, p->rawDev, p->rgbDev);
  RFG_CK(cudaEventRecord(p->rawRead, p->stream));
  RFG_CK(cudaStreamWaitEvent(ps, p->rawRead, 0));
  return rc;
}

int rfg_pipeline_process_rgbd_host(rfg_pipeline* p, const uint16_t* rawHost, const uint8_t* rgbHost,
                                   const float* pose34) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && rawHost && rgbHost, "null argument");
  RFG_REQUIRE(p->cfg.colour, "rgbd frames need a colour pipeline (cfg.colour = 1)");
  const size_t n = (size_t)p->cfg.intr.width * p->cfg.intr.height;
  const size_t nRgb = (size_t)p->cfg.intr_rgb.width * p->cfg.intr_rgb.height * 3;
  // pinned (device-mapped) host frames are read in place by the graph's view
  // and colour packing kernels; anything else is copied in
  const int gi = (p->cfg.track && p->frames > 0) ? 1 : 0;
  if (RFG_HOST_ZEROCOPY && p->cfg.use_graph && p->exec[gi] && p->viewNode[gi] && p->rgbNode[gi]) {
    cudaPointerAttributes a{}, b{};
    if (cudaPointerGetAttributes(&a, rawHost) == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer &&
        cudaPointerGetAttributes(&b, rgbHost) == cudaSuccess && b.type == cudaMemoryTypeHost && b.devicePointer)
      return run_frame(p, pose34, static_cast<const uint16_t*>(a.devicePointer),
                       static_cast<const uint8_t*>(b.devicePointer));
    cudaGetLastError();
  }
  RFG_CK(cudaMemcpyAsync(p->rawDev, rawHost, n * 2, cudaMemcpyHostToDevice, p->stream));
  RFG_CK(cudaMemcpyAsync(p->rgbDev, rgbHost, nRgb, cudaMemcpyHostToDevice, p->stream));
  return run_frame(p, pose34, p->rawDev, p->rgbDev);
}

int rfg_pipeline_process_pgm(rfg_pipeline* p, const char* path, const float* pose34) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && path, "null argument");
  RFG_REQUIRE(!p->cfg.colour, "a colour pipeline takes RGB-D frames (rfg_pipeline_process_rgbd_*)");
  const int64_t n = (int64_t)p->cfg.intr.width * p->cfg.intr.height;
  int w = 0, h = 0;
  // the previous frame's upload may still be reading the staging buffer
  RFG_CK(cudaEventSynchronize(p->stageFree));
  // the payload goes to the device as stored; the GPU view stage decodes it
  // (cfg.raw_big_endian = 1) — with raw_big_endian = 0 it is swapped here
  int rc = p->cfg.raw_big_endian ? rfg_read_pgm16_payload(path, p->pgmStage, n, &w, &h)
                                 : rfg_read_pgm16(path, static_cast<uint16_t*>(p->pgmStage), n, &w, &h);
  if (rc != RFG_OK) return rc;
  RFG_REQUIRE(w == p->cfg.intr.width && h == p->cfg.intr.height,
              "build_view: depth image size does not match calibration");
  RFG_CK(cudaMemcpyAsync(p->rawDev, p->pgmStage, (size_t)n * 2, cudaMemcpyHostToDevice, p->stream));
  RFG_CK(cudaEventRecord(p->stageFree, p->stream));
  return run_frame(p, pose34, p->rawDev);
}

int rfg_pipeline_result(rfg_pipeline* p, rfg_alloc_stats* stats, float poseOut34[12],
                        double icpStats[RFG_ICP_STATS]) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p, "null pipeline");
  rfg_map* m = p->map;
  // the frame graph's last node wrote the results (enqueue_frame)
  RFG_CK(cudaStreamSynchronize(p->stream));
  const MapState& ms = p->hostResult->state;
  if (ms.error) return check_device_error(m);
  if (stats) {
    memcpy(stats, ms.stats, sizeof(rfg_alloc_stats));
    stats->visibleCount = ms.nVisible;  // stage 3 appends the list; its length is the count
  }
  if (p->hostResult->icpError) {
    set_error("ICP: a world point outside the fixed-point range (|p| components >= 128 m)");
    return RFG_ERANGE;
  }
  if (poseOut34) memcpy(poseOut34, p->hostResult->pose, 48);
  if (icpStats) memcpy(icpStats, p->hostResult->icp, sizeof(p->hostResult->icp));
  return RFG_OK;
}

int rfg_pipeline_stage_times(rfg_pipeline* p, float ms7[7]) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && ms7, "null argument");
  RFG_REQUIRE(p->cfg.profile, "stage times need profile = 1");
  RFG_CK(cudaEventSynchronize(p->ev[6]));
  for (int k = 0; k < 6; ++k) RFG_CK(cudaEventElapsedTime(&ms7[k], p->ev[k], p->ev[k + 1]));
  RFG_CK(cudaEventElapsedTime(&ms7[6], p->ev[0], p->ev[6]));
  if (!p->tracked) ms7[1] = 0.f;
  return RFG_OK;
}

void* rfg_pipeline_stream(rfg_pipeline* p) { return p ? (void*)p->stream : nullptr; }

int rfg_pipeline_pose_buffer(rfg_pipeline* p, float** poseDev) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p && poseDev, "null argument");
  *poseDev = p->poses;
  return RFG_OK;
}

int rfg_pipeline_buffers(rfg_pipeline* p, float** depthLevels, float** range, float** raycast, float** points,
                         float** normals) {
  DeviceGuard dg_(p && p->map ? p->map->device : -1);
  RFG_REQUIRE(p, "null pipeline");
  if (depthLevels) *depthLevels = p->depthLevels;
  if (range) *range = reinterpret_cast<float*>(p->range);
  if (raycast) *raycast = reinterpret_cast<float*>(p->raycast);
  if (points) *points = reinterpret_cast<float*>(p->points);
  if (normals) *normals = reinterpret_cast<float*>(p->normals);
  return RFG_OK;
}

}  // extern "C"
