// rfg.hpp — header-only C++ adapter over the librfg.so C ABI (rfg.h) that
// re-exposes the reference's engine interface under its own names, so a
// maintainer can swap the CPU engine for the B200 one call by call:
//
//   rf::VoxelBlockMapConfig / VoxelBlockMap   proj/include/rf/voxel_block_map.hpp:36-144
//   rf::SceneParams / AllocationStats         proj/include/rf/fusion.hpp:11-27
//   rf::FusionEngine::allocate_from_depth /
//                     integrate_frame         proj/include/rf/fusion.hpp:52-79
//   rf::render_expected_ranges / render_maps  proj/include/rf/raycast.hpp:122-129
//   rf::build_view + view elements            proj/include/rf/view.hpp:12-62
//   rf::extract_mesh / Mesh                   proj/include/rf/meshing.hpp:12-23
//   rf::read_pgm16 / read_ppm / write_*       proj/include/rf/image_io.hpp:10-17
//   FusionEngine::Options, reserve/release    proj/include/rf/fusion.hpp:54-57,
//                                             voxel_block_map.hpp:104-109
//   SwappingEngine (the reference has only the hooks)
//
// Images are device pointers (the reference's View/RenderState hold host
// Images; here the GPU owns them).  Errors follow the reference: an invalid
// bucketCount throws std::invalid_argument (voxel_block_map.cpp:10-11); every
// other failure throws rfg::Error carrying the C status code.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rfg.h"

namespace rfg {

using Pose34 = std::array<float, 12>;  // row-major [R | t], world -> camera

inline Pose34 identity_pose() { return {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0}; }

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

inline void check(int rc) {
  if (rc == RFG_OK) return;
  if (rc == RFG_EINVAL) throw std::invalid_argument(rfg_last_error());
  throw Error(rc, std::string("librfg: ") + rfg_last_error());
}

struct VoxelBlockMapConfig {
  std::uint32_t bucketCount = 1u << 20;
  std::uint32_t excessCount = 1u << 17;
  std::uint32_t blockCapacity = 1u << 18;
  static VoxelBlockMapConfig small() { return {1u << 14, 1u << 11, 1u << 13}; }
};

struct Intrinsics {
  int width = 0, height = 0;
  float fx = 0, fy = 0, cx = 0, cy = 0;
  rfg_intrinsics c() const { return {width, height, fx, fy, cx, cy}; }
};

struct SceneParams {
  float voxelSize = 0.005f;
  float mu = 0.02f;
  int maxW = 100;
  float viewFrustum_min = 0.2f;
  float viewFrustum_max = 6.f;
  bool stopIntegratingAtMaxW = false;
  float blockSizeMetres() const { return voxelSize * 8; }
  rfg_scene_params c() const {
    return {voxelSize, mu, maxW, viewFrustum_min, viewFrustum_max, stopIntegratingAtMaxW ? 1 : 0};
  }
};

struct AllocationStats {
  int requested = 0, allocated = 0, allocFailures = 0, visibleCount = 0;
};

struct HashEntry {
  int x, y, z, offset, ptr;
  bool allocated() const { return ptr >= -1; }
  bool inMemory() const { return ptr >= 0; }
};

class VoxelBlockMap {
 public:
  explicit VoxelBlockMap(const VoxelBlockMapConfig& cfg = VoxelBlockMapConfig::small(), bool colour = false,
                         int device = 0)
      : config_(cfg) {
    rfg_map_config c{cfg.bucketCount, cfg.excessCount, cfg.blockCapacity, colour ? 1 : 0};
    check(rfg_map_create(&c, device, &map_));
  }
  ~VoxelBlockMap() { rfg_map_destroy(map_); }
  VoxelBlockMap(const VoxelBlockMap&) = delete;
  VoxelBlockMap& operator=(const VoxelBlockMap&) = delete;

  rfg_map* handle() const { return map_; }
  const VoxelBlockMapConfig& config() const { return config_; }
  std::uint32_t bucketCount() const { return config_.bucketCount; }
  std::uint32_t totalEntries() const { return config_.bucketCount + config_.excessCount; }
  std::uint32_t hashMask() const { return config_.bucketCount - 1; }
  void clear() { check(rfg_map_clear(map_)); }
  void setStream(void* cudaStream) { check(rfg_map_set_stream(map_, cudaStream)); }

  std::vector<HashEntry> entries() const {
    std::vector<HashEntry> out(totalEntries());
    check(rfg_export_entries(map_, reinterpret_cast<int32_t*>(out.data())));
    return out;
  }
  std::vector<int> visibleList() const {
    std::int32_t n = 0;
    check(rfg_export_visible(map_, nullptr, nullptr, &n));
    std::vector<int> out(n);
    check(rfg_export_visible(map_, out.data(), nullptr, &n));
    return out;
  }
  int freeBlockCount() const {
    std::int32_t nb = 0, ne = 0;
    check(rfg_free_counts(map_, &nb, &ne));
    return nb;
  }
  int allocatedBlockCount() const { return static_cast<int>(config_.blockCapacity) - freeBlockCount(); }
  // voxel_block_map.cpp:107-123
  bool reserveBlockForEntry(int entryIdx) {
    const int rc = rfg_map_reserve_block(map_, entryIdx);
    if (rc < 0) check(rc);
    return rc == 1;
  }
  void releaseBlock(int entryIdx) { check(rfg_map_release_block(map_, entryIdx)); }

 private:
  VoxelBlockMapConfig config_;
  rfg_map* map_ = nullptr;
};

struct FusionOptions {  // FusionEngine::Options, fusion.hpp:54-57
  bool swappingEnabled = false;
  float swapMarginPx = 8.f;
};

class FusionEngine {
 public:
  using Options = FusionOptions;
  AllocationStats allocate_from_depth(VoxelBlockMap& map, const float* depthDev, const Intrinsics& intr,
                                      const Pose34& pose, const SceneParams& params, const Options& opts = Options()) {
    const rfg_intrinsics i = intr.c();
    const rfg_scene_params p = params.c();
    const rfg_fusion_options o{opts.swappingEnabled ? 1 : 0, opts.swapMarginPx};
    rfg_alloc_stats s{};
    check(rfg_allocate_from_depth_ex(map.handle(), depthDev, &i, pose.data(), &p, &o, &s));
    return {s.requested, s.allocated, s.allocFailures, s.visibleCount};
  }
  void integrate_frame(VoxelBlockMap& map, const float* depthDev, const Intrinsics& intr, const Pose34& pose,
                       const SceneParams& params, const std::uint8_t* rgbDev = nullptr,
                       const Intrinsics* intrRgb = nullptr, const Pose34* extrinsics = nullptr) {
    const rfg_intrinsics i = intr.c();
    const rfg_intrinsics ir = intrRgb ? intrRgb->c() : i;
    const rfg_scene_params p = params.c();
    check(rfg_integrate(map.handle(), depthDev, rgbDev, &i, &ir, extrinsics ? extrinsics->data() : nullptr,
                        pose.data(), &p));
  }
};

enum class RenderMode { kIcpMaps, kColour, kGrey };

inline void render_expected_ranges(const VoxelBlockMap& map, const Pose34& pose, const Intrinsics& intr,
                                   const SceneParams& params, float* rangeDev) {
  const rfg_intrinsics i = intr.c();
  const rfg_scene_params p = params.c();
  check(rfg_render_expected_ranges(map.handle(), pose.data(), &i, &p, rangeDev));
}

// raycast.cpp:129-139; colourDev (RGB8 per pixel) is written in kColour /
// kGrey mode and may be null in kIcpMaps mode.
inline void render_maps(const VoxelBlockMap& map, const Pose34& pose, const Intrinsics& intr,
                        const SceneParams& params, RenderMode mode, const float* rangeDev, float* raycastDev,
                        float* pointsDev, float* normalsDev, std::uint8_t* colourDev = nullptr) {
  const rfg_intrinsics i = intr.c();
  const rfg_scene_params p = params.c();
  check(rfg_render_maps(map.handle(), pose.data(), &i, &p, static_cast<int>(mode), rangeDev, raycastDev, pointsDev,
                        normalsDev, colourDev));
}

// ------------------------------------------------------------ view
struct ViewBuildOptions {  // view.hpp:12-15
  bool bilateral = false;
  int levels = 3;
};

// build_view (view.cpp:100-143) on device images: depthLevelsDev receives the
// depth pyramid back to back; intensityLevelsDev (needs rgbDev) and
// normalsDev (float4 per pixel) may be null; scratchDev (width*height floats)
// is needed with bilateral.  rawBigEndian: raw is a PGM16 payload.
inline void build_view(const std::uint16_t* rawDev, const std::uint8_t* rgbDev, const Intrinsics& intrD,
                       float affScale, float affOffset, const ViewBuildOptions& opts, float* depthLevelsDev,
                       float* intensityLevelsDev = nullptr, float* normalsDev = nullptr, float* scratchDev = nullptr,
                       void* cudaStream = nullptr, bool rawBigEndian = false) {
  const rfg_intrinsics i = intrD.c();
  const int rc = rfg_build_view(rawDev, rgbDev, &i, affScale, affOffset, opts.bilateral ? 1 : 0, opts.levels,
                                rawBigEndian ? 1 : 0, depthLevelsDev, intensityLevelsDev, normalsDev, scratchDev,
                                cudaStream);
  if (rc == RFG_EINVAL) throw std::invalid_argument(rfg_last_error());  // view.cpp:102-106
  check(rc);
}
inline void bilateral_filter(const float* inDev, int w, int h, float spatialSigma, float rangeSigma, float* outDev,
                             void* cudaStream = nullptr) {
  check(rfg_bilateral_filter(inDev, w, h, spatialSigma, rangeSigma, outDev, cudaStream));
}
inline void compute_normals(const float* depthDev, const Intrinsics& intr, float* normalsDev,
                            void* cudaStream = nullptr) {
  const rfg_intrinsics i = intr.c();
  check(rfg_compute_normals(depthDev, &i, normalsDev, cudaStream));
}

// ------------------------------------------------------------ mesh
struct Mesh {  // meshing.hpp:12-15 (metres; normals toward positive sdf)
  std::vector<std::array<float, 3>> vertices;
  std::vector<std::array<std::uint32_t, 3>> triangles;
};
inline Mesh extract_mesh(const VoxelBlockMap& map, float voxelSize) {
  std::int64_t nv = 0, nt = 0;
  check(rfg_extract_mesh(map.handle(), voxelSize, &nv, &nt));
  Mesh m;
  m.vertices.resize(static_cast<std::size_t>(nv));
  m.triangles.resize(static_cast<std::size_t>(nt));
  check(rfg_mesh_copy(map.handle(), nv ? m.vertices[0].data() : nullptr, nt ? m.triangles[0].data() : nullptr));
  return m;
}

// ------------------------------------------------------------ image IO
template <class T>
struct HostImage {
  int width = 0, height = 0;
  std::vector<T> data;  // row-major; 3 bytes per pixel for RGB8
};
inline HostImage<std::uint16_t> read_pgm16(const std::string& path) {
  HostImage<std::uint16_t> img;
  int rc = rfg_read_pgm16(path.c_str(), nullptr, 0, &img.width, &img.height);
  if (rc == RFG_EINVAL) throw std::runtime_error(rfg_last_error());  // image_io.cpp messages
  img.data.resize(static_cast<std::size_t>(img.width) * img.height);
  check(rfg_read_pgm16(path.c_str(), img.data.data(), static_cast<int64_t>(img.data.size()), &img.width,
                       &img.height));
  return img;
}
inline HostImage<std::uint8_t> read_ppm(const std::string& path) {
  HostImage<std::uint8_t> img;
  int rc = rfg_read_ppm(path.c_str(), nullptr, 0, &img.width, &img.height);
  if (rc == RFG_EINVAL) throw std::runtime_error(rfg_last_error());
  img.data.resize(static_cast<std::size_t>(img.width) * img.height * 3);
  check(rfg_read_ppm(path.c_str(), img.data.data(), static_cast<int64_t>(img.width) * img.height, &img.width,
                     &img.height));
  return img;
}
inline void write_pgm16(const HostImage<std::uint16_t>& img, const std::string& path) {
  check(rfg_write_pgm16(path.c_str(), img.data.data(), img.width, img.height));
}
inline void write_ppm(const HostImage<std::uint8_t>& img, const std::string& path) {
  check(rfg_write_ppm(path.c_str(), img.data.data(), img.width, img.height));
}

// ------------------------------------------------------------ swapping
// SPEC.md:407-465 over the reference's hooks; per frame:
// allocate_from_depth(..., Options{true}) -> swapIn() -> integrate_frame ->
// render -> swapOut().
class SwappingEngine {
 public:
  SwappingEngine(VoxelBlockMap& map, int capacityBlocks = 512) {
    check(rfg_swap_create(map.handle(), capacityBlocks, &s_));
  }
  ~SwappingEngine() { rfg_swap_destroy(s_); }
  SwappingEngine(const SwappingEngine&) = delete;
  SwappingEngine& operator=(const SwappingEngine&) = delete;
  int swapIn(int maxW = 100) {
    int n = 0;
    check(rfg_swap_in(s_, maxW, &n));
    return n;
  }
  int swapOut() {
    int n = 0;
    check(rfg_swap_out(s_, &n));
    return n;
  }

 private:
  rfg_swap* s_ = nullptr;
};

// TrackerIterationSummary of a track's last evaluation,
// plus the run's outcome (rfg_icp_track's RFG_ICP_* values).
struct TrackerIterationSummary {
  int iterations = 0, inliers = 0;
  double residualSum = 0.0;
  bool converged = false, ok = false;
  int perLevel[3] = {0, 0, 0};
  double inlierFraction = 0.0, hessianDet = 0.0, residualMean = 0.0;
  int validPixels = 0;
  static TrackerIterationSummary from(const double* st) {
    TrackerIterationSummary t;
    t.iterations = (int)st[RFG_ICP_ITERATIONS];
    t.inliers = (int)st[RFG_ICP_COUNT];
    t.residualSum = st[RFG_ICP_RESIDUAL_SUM];
    t.converged = st[RFG_ICP_CONVERGED] != 0.0;
    for (int l = 0; l < 3; ++l) t.perLevel[l] = (int)st[RFG_ICP_IT_L0 + l];
    t.ok = st[RFG_ICP_OK] != 0.0;
    t.inlierFraction = st[RFG_ICP_INLIER_FRACTION];
    t.hessianDet = st[RFG_ICP_HESSIAN_DET];
    t.residualMean = st[RFG_ICP_RESIDUAL_MEAN];
    t.validPixels = (int)st[RFG_ICP_VALID];
    return t;
  }
};

// ITMMainEngine::ProcessFrame-style driver (absent in the reference).  With
// colour = true the map needs a colour plane and frames come with RGB8
// images (processRgbdHost); intrRgb / extrinsics default to the depth
// camera / identity.
class Pipeline {
 public:
  Pipeline(VoxelBlockMap& map, const Intrinsics& intr, const SceneParams& params, float affScale, float affOffset,
           int levels = 3, bool track = true, bool colour = false, const Intrinsics* intrRgb = nullptr,
           const Pose34* extrDToRgb = nullptr) {
    rfg_pipeline_config c{};
    c.intr = intr.c();
    c.params = params.c();
    c.aff_scale = affScale;
    c.aff_offset = affOffset;
    c.levels = levels;
    c.track = track ? 1 : 0;
    c.iters[0] = 6;
    c.iters[1] = 10;
    c.iters[2] = 20;
    c.dist[0] = 0.01f;
    c.dist[1] = 0.02f;
    c.dist[2] = 0.04f;
    c.min_count = 10;
    c.use_graph = 1;
    c.colour = colour ? 1 : 0;
    if (colour) {
      c.intr_rgb = (intrRgb ? *intrRgb : intr).c();
      for (int i = 0; i < 12; ++i) c.extr_d_to_rgb[i] = extrDToRgb ? (*extrDToRgb)[i] : ((i % 5 == 0) ? 1.f : 0.f);
    }
    check(rfg_pipeline_create(map.handle(), &c, &p_));
  }
  ~Pipeline() { rfg_pipeline_destroy(p_); }
  Pipeline(const Pipeline&) = delete;
  Pipeline& operator=(const Pipeline&) = delete;

  void processHost(const std::uint16_t* rawHost, const Pose34* pose = nullptr) {
    check(rfg_pipeline_process_host(p_, rawHost, pose ? pose->data() : nullptr));
  }
  // one frame from a PGM16 file (image_io.cpp:96-113)
  void processPgm(const std::string& path, const Pose34* pose = nullptr) {
    check(rfg_pipeline_process_pgm(p_, path.c_str(), pose ? pose->data() : nullptr));
  }
  // one RGB-D frame of a colour pipeline (RGB8, intrRgb's size)
  void processRgbdHost(const std::uint16_t* rawHost, const std::uint8_t* rgbHost, const Pose34* pose = nullptr) {
    check(rfg_pipeline_process_rgbd_host(p_, rawHost, rgbHost, pose ? pose->data() : nullptr));
  }
  AllocationStats result(Pose34* poseOut = nullptr, TrackerIterationSummary* tracker = nullptr) {
    rfg_alloc_stats s{};
    Pose34 tmp;
    double st[RFG_ICP_STATS] = {};
    check(rfg_pipeline_result(p_, &s, poseOut ? poseOut->data() : tmp.data(), st));
    if (tracker) *tracker = TrackerIterationSummary::from(st);
    return {s.requested, s.allocated, s.allocFailures, s.visibleCount};
  }

 private:
  rfg_pipeline* p_ = nullptr;
};

// Synthetic frame source (proj/src/synth.cpp).
inline std::vector<Pose34> orbit_trajectory(std::array<float, 3> target, float distance, int frames,
                                            float maxAngle = 0.5f) {
  std::vector<Pose34> out(frames);
  check(rfg_synth_orbit_poses(target.data(), distance, frames, maxAngle, out.empty() ? nullptr : out[0].data()));
  return out;
}

}  // namespace rfg
