// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp compiled against oracle/shim/), built by
// oracle/Makefile into oracle/_ref/librfref.so.  It exists to (1) pin the C
// restatement oracle (oracle/rfo.c) against the reference's own code, (2)
// generate the committed golden fixtures under tests/golden/, and (3) serve as
// the timed CPU baseline (`bench.py --impl reference`).  Nothing in the
// product package may load it.
//
// Every entry point calls straight into rf:: functions:
//   FusionEngine::allocate_from_depth / integrate_frame  proj/src/fusion.cpp:225-344
//   render_expected_ranges / render_maps               proj/src/raycast.cpp:86-139
//   build_view                                          proj/src/view.cpp:100-143
//   synth_render_depth / orbit_trajectory               proj/src/synth.cpp:136-195
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>

#include "rf/fusion.hpp"
#include "rf/image_io.hpp"
#include "rf/meshing.hpp"
#include "rf/raycast.hpp"
#include "rf/synth.hpp"
#include "rf/view.hpp"
#include "rf/voxel_block_map.hpp"

using namespace rf;

namespace {

Pose poseFrom12(const float* p) {
  // row-major 3x4 [R | t], world -> camera
  Eigen::Matrix3f R;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R(r, c) = p[r * 4 + c];
  return Pose(R, Eigen::Vector3f(p[3], p[7], p[11]));
}

void poseTo12(const Pose& pose, float* p) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) p[r * 4 + c] = pose.rotation()(r, c);
    p[r * 4 + 3] = pose.translation()[r];
  }
}

Intrinsics intrFrom(const int* wh, const float* f4) {
  Intrinsics i;
  i.width = wh[0];
  i.height = wh[1];
  i.fx = f4[0];
  i.fy = f4[1];
  i.cx = f4[2];
  i.cy = f4[3];
  return i;
}

// params: voxelSize, mu, maxW, vfMin, vfMax, stopAtMaxW
SceneParams paramsFrom(const float* p) {
  SceneParams s;
  s.voxelSize = p[0];
  s.mu = p[1];
  s.maxW = static_cast<int>(p[2]);
  s.viewFrustum_min = p[3];
  s.viewFrustum_max = p[4];
  s.stopIntegratingAtMaxW = p[5] != 0.f;
  return s;
}

// Builder-defined C4 scene (open decision 5): three 4 m
// rooms along +x separated by 0.1 m walls with 1 m doorways, a floor plane,
// a ceiling plane, and furniture (boxes + spheres).  Boxes are one-sided
// (hit from outside only, proj/src/synth.cpp:92-100), so walls are thin boxes.
SyntheticScene makeMultiRoom() {
  SyntheticScene s;
  s.planes.push_back({{0, -1, 0}, -0.45f, Rgb8{150, 170, 150}, false, 0.1f, Rgb8{0, 0, 0}});   // floor y=0.45
  s.planes.push_back({{0, 1, 0}, -2.05f, Rgb8{210, 210, 210}, false, 0.1f, Rgb8{0, 0, 0}});    // ceiling y=-2.05
  const float wallT = 0.05f;
  // outer long walls z = -2 and z = +2 spanning x in [-2, 10]
  s.boxes.push_back({{4.f, -0.8f, -2.f}, {6.f, 1.25f, wallT}, Rgb8{190, 180, 170}});
  s.boxes.push_back({{4.f, -0.8f, 2.f}, {6.f, 1.25f, wallT}, Rgb8{170, 180, 190}});
  // end walls x = -2 and x = 10
  s.boxes.push_back({{-2.f, -0.8f, 0.f}, {wallT, 1.25f, 2.f}, Rgb8{200, 160, 160}});
  s.boxes.push_back({{10.f, -0.8f, 0.f}, {wallT, 1.25f, 2.f}, Rgb8{160, 200, 160}});
  // partition walls at x = 2 and x = 6 with a 1 m doorway centred at z = 0
  for (float x : {2.f, 6.f}) {
    s.boxes.push_back({{x, -0.8f, -1.25f}, {wallT, 1.25f, 0.75f}, Rgb8{180, 180, 200}});
    s.boxes.push_back({{x, -0.8f, 1.25f}, {wallT, 1.25f, 0.75f}, Rgb8{180, 200, 180}});
    s.boxes.push_back({{x, -1.5f, 0.f}, {wallT, 0.55f, 0.5f}, Rgb8{200, 200, 180}});  // lintel
  }
  // furniture
  s.boxes.push_back({{0.5f, 0.2f, 1.2f}, {0.5f, 0.25f, 0.4f}, Rgb8{120, 90, 60}});
  s.boxes.push_back({{4.f, 0.05f, -1.3f}, {0.8f, 0.4f, 0.3f}, Rgb8{90, 120, 60}});
  s.boxes.push_back({{8.3f, 0.15f, 1.f}, {0.4f, 0.3f, 0.6f}, Rgb8{60, 90, 120}});
  s.spheres.push_back({{-0.8f, 0.1f, -1.f}, 0.35f, Rgb8{180, 120, 80}});
  s.spheres.push_back({{3.2f, -0.2f, 1.1f}, 0.5f, Rgb8{80, 120, 180}});
  s.spheres.push_back({{7.5f, 0.f, -0.9f}, 0.45f, Rgb8{160, 80, 160}});
  return s;
}

SyntheticScene sceneOf(int kind) {
  switch (kind) {
    case 0:
      return make_sphere_in_room_scene();
    case 1:
      return makeMultiRoom();
    case 2:
      return make_checker_wall_scene();
    default:
      return make_sphere_scene();
  }
}

struct Engine {
  explicit Engine(const VoxelBlockMapConfig& c) : map(c) {}
  VoxelBlockMap map;
  FusionEngine fusion;
  RenderState render;
  Mesh mesh;
  FusionEngine::Options opts;
};

View makeView(const float* depth, const std::uint8_t* rgb, const Intrinsics& intrD, const Intrinsics& intrRgb,
              const float* extr12) {
  View v;
  v.calib.intrinsics_d = intrD;
  v.calib.intrinsics_rgb = intrRgb;
  if (extr12) v.calib.extrinsics_d_to_rgb = poseFrom12(extr12);
  v.depth_m = Image<float>(intrD.width, intrD.height);
  std::memcpy(v.depth_m.data(), depth, sizeof(float) * intrD.width * intrD.height);
  if (rgb) {
    v.rgb = Image<Rgb8>(intrRgb.width, intrRgb.height);
    for (int i = 0; i < intrRgb.width * intrRgb.height; ++i)
      v.rgb.data()[i] = Rgb8{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
  }
  return v;
}

double nowMs() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- synthetic
int rr_orbit_poses(const float* target3, float distance, int frames, float maxAngle, float* out12) {
  const auto poses = orbit_trajectory(Eigen::Vector3f(target3[0], target3[1], target3[2]), distance, frames, maxAngle);
  for (int i = 0; i < frames; ++i) poseTo12(poses[i], out12 + 12 * i);
  return 0;
}

int rr_render(int sceneKind, const float* pose12, const int* wh, const float* f4, float affScale, float affOffset,
              int renderRgb, std::uint16_t* rawOut, float* depthOut, std::uint8_t* rgbOut) {
  const SyntheticScene scene = sceneOf(sceneKind);
  const Intrinsics intr = intrFrom(wh, f4);
  DepthAffine aff;
  aff.scale = affScale;
  aff.offset = affOffset;
  const SynthRender r = synth_render_depth(scene, poseFrom12(pose12), intr, aff, 0.f, 0, renderRgb != 0);
  const int n = intr.width * intr.height;
  if (rawOut) std::memcpy(rawOut, r.depth_raw.data(), sizeof(std::uint16_t) * n);
  if (depthOut) std::memcpy(depthOut, r.depth_m.data(), sizeof(float) * n);
  if (rgbOut && renderRgb)
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) rgbOut[3 * i + k] = r.rgb.data()[i][k];
  return 0;
}

float rr_scene_sdf(int sceneKind, const float* p3) {
  return sceneOf(sceneKind).signedDistance(Eigen::Vector3f(p3[0], p3[1], p3[2]));
}

// ----------------------------------------------------------------- view
// depthLevels receives level 0 (w*h) followed by each pyramid level.
int rr_build_view(const std::uint16_t* raw, const int* wh, const float* f4, float affScale, float affOffset,
                  int levels, float* depthLevels) {
  RgbdCalib calib;
  calib.intrinsics_d = intrFrom(wh, f4);
  calib.intrinsics_rgb = calib.intrinsics_d;
  calib.depth_affine.scale = affScale;
  calib.depth_affine.offset = affOffset;
  Image<std::uint16_t> img(wh[0], wh[1]);
  std::memcpy(img.data(), raw, sizeof(std::uint16_t) * wh[0] * wh[1]);
  ViewBuildOptions opts;
  opts.levels = levels;
  const View v = build_view(img, {}, calib, opts);
  float* out = depthLevels;
  for (int l = 0; l < levels; ++l) {
    const auto& d = v.pyramid[l].depth;
    std::memcpy(out, d.data(), sizeof(float) * d.size());
    out += d.size();
  }
  return 0;
}

// full ViewBuilder (view.cpp:8-143): every option; outputs packed per level,
// intensity / normals may be null
int rr_build_view_full(const std::uint16_t* raw, const std::uint8_t* rgb, const int* wh, const float* f4,
                       float affScale, float affOffset, int bilateral, int levels, float* depthLevels,
                       float* intensityLevels, float* normals4) {
  RgbdCalib calib;
  calib.intrinsics_d = intrFrom(wh, f4);
  calib.intrinsics_rgb = calib.intrinsics_d;
  calib.depth_affine.scale = affScale;
  calib.depth_affine.offset = affOffset;
  Image<std::uint16_t> img(wh[0], wh[1]);
  std::memcpy(img.data(), raw, sizeof(std::uint16_t) * wh[0] * wh[1]);
  Image<Rgb8> col;
  if (rgb) {
    col = Image<Rgb8>(wh[0], wh[1]);
    std::memcpy(col.data(), rgb, 3 * (size_t)wh[0] * wh[1]);
  }
  ViewBuildOptions opts;
  opts.levels = levels;
  opts.bilateral = bilateral != 0;
  View v;
  try {
    v = build_view(img, col, calib, opts);
  } catch (const std::exception&) {
    return -1;
  }
  float* out = depthLevels;
  float* outI = intensityLevels;
  for (int l = 0; l < levels; ++l) {
    const auto& d = v.pyramid[l].depth;
    std::memcpy(out, d.data(), sizeof(float) * d.size());
    out += d.size();
    if (rgb && outI) {
      const auto& it = v.pyramid[l].intensity;
      std::memcpy(outI, it.data(), sizeof(float) * it.size());
      outI += it.size();
    }
  }
  if (normals4) std::memcpy(normals4, v.normals.data(), sizeof(float) * 4 * v.normals.size());
  return 0;
}

int rr_bilateral_filter(const float* in, int w, int h, float spatialSigma, float rangeSigma, float* out) {
  Image<float> img(w, h);
  std::memcpy(img.data(), in, sizeof(float) * (size_t)w * h);
  const Image<float> o = bilateral_filter(img, spatialSigma, rangeSigma);
  std::memcpy(out, o.data(), sizeof(float) * (size_t)w * h);
  return 0;
}

int rr_compute_normals(const float* in, const int* wh, const float* f4, float* out4) {
  Image<float> img(wh[0], wh[1]);
  std::memcpy(img.data(), in, sizeof(float) * (size_t)wh[0] * wh[1]);
  const auto o = compute_normals(img, intrFrom(wh, f4));
  std::memcpy(out4, o.data(), sizeof(float) * 4 * o.size());
  return 0;
}

// image_io.cpp: Netpbm readers / writers (0 ok, -1 on the reference's exception)
int rr_read_pgm16(const char* path, std::uint16_t* out, int capacity, int* w, int* h) {
  try {
    const auto img = read_pgm16(path);
    *w = img.width();
    *h = img.height();
    if ((long)img.size() > capacity) return -2;
    std::memcpy(out, img.data(), sizeof(std::uint16_t) * img.size());
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}
int rr_read_ppm(const char* path, std::uint8_t* out, int capacity, int* w, int* h) {
  try {
    const auto img = read_ppm(path);
    *w = img.width();
    *h = img.height();
    if ((long)img.size() * 3 > capacity) return -2;
    std::memcpy(out, img.data(), 3 * img.size());
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}
int rr_write_pgm16(const char* path, const std::uint16_t* in, int w, int h) {
  try {
    Image<std::uint16_t> img(w, h);
    std::memcpy(img.data(), in, sizeof(std::uint16_t) * (size_t)w * h);
    write_pgm16(img, path);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}
int rr_write_ppm(const char* path, const std::uint8_t* in, int w, int h) {
  try {
    Image<Rgb8> img(w, h);
    std::memcpy(img.data(), in, 3 * (size_t)w * h);
    write_ppm(img, path);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// -------------------------------------------------------------- elements
std::uint32_t rr_hash_index(const int* pos3, std::uint32_t mask) {
  return hash_index(Eigen::Vector3i(pos3[0], pos3[1], pos3[2]), mask);
}

int rr_traverse_blocks(const float* a3, const float* b3, int* cellsOut, int maxCells) {
  int n = 0;
  traverse_blocks(Eigen::Vector3f(a3[0], a3[1], a3[2]), Eigen::Vector3f(b3[0], b3[1], b3[2]),
                  [&](const Eigen::Vector3i& c) {
                    if (n < maxCells) {
                      cellsOut[3 * n] = c.x();
                      cellsOut[3 * n + 1] = c.y();
                      cellsOut[3 * n + 2] = c.z();
                    }
                    ++n;
                  });
  return n;
}

int rr_block_in_frustum(const int* pos3, const float* pose12, const int* wh, const float* f4, const float* params) {
  return block_in_frustum(Eigen::Vector3i(pos3[0], pos3[1], pos3[2]), poseFrom12(pose12), intrFrom(wh, f4),
                          paramsFrom(params))
             ? 1
             : 0;
}

// voxel8: VoxelSRgb bytes {sdf lo, sdf hi, w_depth, r, g, b, w_color, pad}
float rr_update_voxel_depth(std::uint8_t* voxel8, const float* pt3, const float* pose12, const int* wh,
                            const float* f4, float mu, int maxW, const float* depth, int stopAtMaxW) {
  VoxelSRgb v;
  std::memcpy(&v.sdf, voxel8, 2);
  v.w_depth = voxel8[2];
  Image<float> img(wh[0], wh[1]);
  std::memcpy(img.data(), depth, sizeof(float) * wh[0] * wh[1]);
  const float eta = update_voxel_depth(v, Eigen::Vector3f(pt3[0], pt3[1], pt3[2]), poseFrom12(pose12),
                                       intrFrom(wh, f4), mu, maxW, img, stopAtMaxW != 0);
  std::memcpy(voxel8, &v.sdf, 2);
  voxel8[2] = v.w_depth;
  return eta;
}

// ----------------------------------------------------------------- engine
void* rr_create(std::uint32_t buckets, std::uint32_t excess, std::uint32_t capacity) {
  try {
    return new Engine(VoxelBlockMapConfig{buckets, excess, capacity});
  } catch (...) {
    return nullptr;
  }
}

void rr_destroy(void* h) { delete static_cast<Engine*>(h); }

int rr_allocate(void* h, const float* depth, const int* wh, const float* f4, const float* pose12, const float* params,
                int* stats4, double* ms) {
  auto* e = static_cast<Engine*>(h);
  const Intrinsics intr = intrFrom(wh, f4);
  const View v = makeView(depth, nullptr, intr, intr, nullptr);
  const double t0 = nowMs();
  const AllocationStats s = e->fusion.allocate_from_depth(e->map, v, poseFrom12(pose12), paramsFrom(params), e->opts);
  if (ms) *ms = nowMs() - t0;
  stats4[0] = s.requested;
  stats4[1] = s.allocated;
  stats4[2] = s.allocFailures;
  stats4[3] = s.visibleCount;
  return 0;
}

// FusionEngine::Options (fusion.hpp:54-57) for the engine's allocate calls
int rr_set_fusion_options(void* h, int swappingEnabled, float swapMarginPx) {
  auto* e = static_cast<Engine*>(h);
  e->opts.swappingEnabled = swappingEnabled != 0;
  e->opts.swapMarginPx = swapMarginPx;
  return 0;
}
// VoxelBlockMap::reserveBlockForEntry / releaseBlock (voxel_block_map.cpp:107-123)
int rr_reserve_block(void* h, int idx) { return static_cast<Engine*>(h)->map.reserveBlockForEntry(idx) ? 1 : 0; }
int rr_release_block(void* h, int idx) {
  static_cast<Engine*>(h)->map.releaseBlock(idx);
  return 0;
}

int rr_integrate(void* h, const float* depth, const std::uint8_t* rgb, const int* whD, const float* f4D,
                 const int* whRgb, const float* f4Rgb, const float* extr12, const float* pose12, const float* params,
                 double* ms) {
  auto* e = static_cast<Engine*>(h);
  const Intrinsics intrD = intrFrom(whD, f4D);
  const Intrinsics intrRgb = whRgb ? intrFrom(whRgb, f4Rgb) : intrD;
  const View v = makeView(depth, rgb, intrD, intrRgb, extr12);
  const double t0 = nowMs();
  e->fusion.integrate_frame(e->map, v, poseFrom12(pose12), paramsFrom(params));
  if (ms) *ms = nowMs() - t0;
  return 0;
}

int rr_render_ranges(void* h, const float* pose12, const int* wh, const float* f4, const float* params,
                     float* rangeOut, double* ms) {
  auto* e = static_cast<Engine*>(h);
  const double t0 = nowMs();
  render_expected_ranges(e->map, poseFrom12(pose12), intrFrom(wh, f4), paramsFrom(params), e->render);
  if (ms) *ms = nowMs() - t0;
  if (rangeOut)
    for (std::size_t i = 0; i < e->render.expectedRange.size(); ++i) {
      rangeOut[2 * i] = e->render.expectedRange.data()[i].x();
      rangeOut[2 * i + 1] = e->render.expectedRange.data()[i].y();
    }
  return 0;
}

int rr_render_icp(void* h, const float* pose12, const int* wh, const float* f4, const float* params, float* raycastOut,
                  float* pointsOut, float* normalsOut, double* ms) {
  auto* e = static_cast<Engine*>(h);
  const double t0 = nowMs();
  render_maps(e->map, poseFrom12(pose12), intrFrom(wh, f4), paramsFrom(params), RenderMode::kIcpMaps, e->render);
  if (ms) *ms = nowMs() - t0;
  const std::size_t n = e->render.points.size();
  for (std::size_t i = 0; i < n; ++i)
    for (int k = 0; k < 4; ++k) {
      if (raycastOut) raycastOut[4 * i + k] = e->render.raycastResult.data()[i][k];
      if (pointsOut) pointsOut[4 * i + k] = e->render.points.data()[i][k];
      if (normalsOut) normalsOut[4 * i + k] = e->render.normals.data()[i][k];
    }
  return 0;
}

// render_maps with any RenderMode (raycast.cpp:129-139): 0 kIcpMaps,
// 1 kColour, 2 kGrey; the three float4 maps plus the RGB8 colour image.
int rr_render_maps(void* h, int mode, const float* pose12, const int* wh, const float* f4, const float* params,
                   float* raycastOut, float* pointsOut, float* normalsOut, std::uint8_t* colourOut) {
  auto* e = static_cast<Engine*>(h);
  const RenderMode rm = mode == 1 ? RenderMode::kColour : (mode == 2 ? RenderMode::kGrey : RenderMode::kIcpMaps);
  render_maps(e->map, poseFrom12(pose12), intrFrom(wh, f4), paramsFrom(params), rm, e->render);
  const std::size_t n = e->render.points.size();
  for (std::size_t i = 0; i < n; ++i) {
    for (int k = 0; k < 4; ++k) {
      if (raycastOut) raycastOut[4 * i + k] = e->render.raycastResult.data()[i][k];
      if (pointsOut) pointsOut[4 * i + k] = e->render.points.data()[i][k];
      if (normalsOut) normalsOut[4 * i + k] = e->render.normals.data()[i][k];
    }
    if (colourOut)
      for (int k = 0; k < 3; ++k) colourOut[3 * i + k] = e->render.colour.data()[i][k];
  }
  return 0;
}

// extract_mesh (meshing.cpp:144-217): keeps the mesh in the engine; counts out
int rr_extract_mesh(void* h, float voxelSize, long long* nV, long long* nT) {
  auto* e = static_cast<Engine*>(h);
  e->mesh = extract_mesh(e->map, voxelSize);
  *nV = (long long)e->mesh.vertices.size();
  *nT = (long long)e->mesh.triangles.size();
  return 0;
}
int rr_mesh_copy(void* h, float* v3, std::uint32_t* t3) {
  auto* e = static_cast<Engine*>(h);
  for (std::size_t i = 0; i < e->mesh.vertices.size(); ++i)
    for (int k = 0; k < 3; ++k) v3[3 * i + k] = e->mesh.vertices[i][k];
  for (std::size_t i = 0; i < e->mesh.triangles.size(); ++i)
    for (int k = 0; k < 3; ++k) t3[3 * i + k] = e->mesh.triangles[i][k];
  return 0;
}
// detail::marchingCubesTable (meshing.cpp:27-118): counts + edge triples
int rr_mc_table(int* counts256, int* tris) {
  const auto& t = detail::marchingCubesTable();
  for (int m = 0; m < 256; ++m) {
    counts256[m] = (int)t[m].size();
    for (int k = 0; k < 16; ++k)
      for (int j = 0; j < 3; ++j) tris[(m * 16 + k) * 3 + j] = k < (int)t[m].size() ? t[m][k][j] : -1;
  }
  return 0;
}
// direct voxel writes (test support: analytic TSDFs as the reference's
// meshing tests build them, test_voxelmap.cpp:231-280)
int rr_set_block(void* h, const int* pos3, const std::int16_t* sdf512, const std::uint8_t* w512) {
  auto* e = static_cast<Engine*>(h);
  const auto idx = e->map.allocateBlock(Eigen::Vector3i(pos3[0], pos3[1], pos3[2]));
  if (!idx) return -1;
  Voxel* b = e->map.blockData(e->map.entry(*idx).ptr);
  for (int i = 0; i < kBlockSize3; ++i) {
    b[i].sdf = sdf512[i];
    b[i].w_depth = w512[i];
  }
  return 0;
}

// forward_project (proj/src/raycast.cpp:141-188) on the engine's RenderState:
// returns the number of missing pixels and writes them as (x, y) pairs.
int rr_forward_project(void* h, const float* pose12, const int* wh, const float* f4, float voxelSize,
                       int* missingXY) {
  auto* e = static_cast<Engine*>(h);
  const auto missing = forward_project(e->render, poseFrom12(pose12), intrFrom(wh, f4), voxelSize);
  for (std::size_t i = 0; i < missing.size(); ++i) {
    missingXY[2 * i] = missing[i].x();
    missingXY[2 * i + 1] = missing[i].y();
  }
  return static_cast<int>(missing.size());
}

// render_maps(kIcpMaps, missingOnly) (raycast.hpp:200-202); outputs the full
// state images afterwards.
int rr_render_icp_missing(void* h, const float* pose12, const int* wh, const float* f4, const float* params,
                          const int* missingXY, int n, float* raycastOut, float* pointsOut, float* normalsOut) {
  auto* e = static_cast<Engine*>(h);
  std::vector<Eigen::Vector2i> missing(n);
  for (int i = 0; i < n; ++i) missing[i] = Eigen::Vector2i(missingXY[2 * i], missingXY[2 * i + 1]);
  render_maps(e->map, poseFrom12(pose12), intrFrom(wh, f4), paramsFrom(params), RenderMode::kIcpMaps, e->render,
              &missing);
  const std::size_t np = e->render.points.size();
  for (std::size_t i = 0; i < np; ++i)
    for (int k = 0; k < 4; ++k) {
      raycastOut[4 * i + k] = e->render.raycastResult.data()[i][k];
      pointsOut[4 * i + k] = e->render.points.data()[i][k];
      normalsOut[4 * i + k] = e->render.normals.data()[i][k];
    }
  return 0;
}

// Set the expected-range image directly (used to drive render_icp from a
// range image produced elsewhere).
int rr_set_ranges(void* h, const int* wh, const float* f4, const float* rangeIn) {
  auto* e = static_cast<Engine*>(h);
  e->render.resize(intrFrom(wh, f4));
  for (std::size_t i = 0; i < e->render.expectedRange.size(); ++i)
    e->render.expectedRange.data()[i] = Eigen::Vector2f(rangeIn[2 * i], rangeIn[2 * i + 1]);
  return 0;
}

std::uint32_t rr_total_entries(void* h) { return static_cast<Engine*>(h)->map.totalEntries(); }

// entries: 5 int32 per entry {x, y, z, offset, ptr}
int rr_export_entries(void* h, int* out5) {
  auto* e = static_cast<Engine*>(h);
  const auto& ents = e->map.entries();
  for (std::size_t i = 0; i < ents.size(); ++i) {
    out5[5 * i] = ents[i].pos.x();
    out5[5 * i + 1] = ents[i].pos.y();
    out5[5 * i + 2] = ents[i].pos.z();
    out5[5 * i + 3] = ents[i].offset;
    out5[5 * i + 4] = ents[i].ptr;
  }
  return static_cast<int>(ents.size());
}

// VoxelSRgb blocks for the given VBA pointers: 512 * 8 bytes each.
int rr_export_blocks(void* h, const int* ptrs, int n, std::uint8_t* out) {
  auto* e = static_cast<Engine*>(h);
  for (int b = 0; b < n; ++b) {
    const Voxel* blk = e->map.blockData(ptrs[b]);
    for (int v = 0; v < kBlockSize3; ++v) {
      std::uint8_t* o = out + (std::size_t(b) * kBlockSize3 + v) * 8;
      std::memcpy(o, &blk[v].sdf, 2);
      o[2] = blk[v].w_depth;
      o[3] = blk[v].clr[0];
      o[4] = blk[v].clr[1];
      o[5] = blk[v].clr[2];
      o[6] = blk[v].w_color;
      o[7] = 0;
    }
  }
  return 0;
}

int rr_export_visible(void* h, int* listOut, std::uint8_t* typesOut) {
  auto* e = static_cast<Engine*>(h);
  const auto& vl = e->map.visibleList();
  if (listOut) std::memcpy(listOut, vl.data(), sizeof(int) * vl.size());
  if (typesOut) std::memcpy(typesOut, e->map.visibilityTypes().data(), e->map.visibilityTypes().size());
  return static_cast<int>(vl.size());
}

int rr_free_counts(void* h, int* nb, int* ne) {
  auto* e = static_cast<Engine*>(h);
  *nb = e->map.freeBlockCount();
  *ne = e->map.freeExcessCount();
  return 0;
}

}  // extern "C"
