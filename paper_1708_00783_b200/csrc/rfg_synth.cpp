// rfg_synth.cpp — synthetic frame source for benchmarks and parity runs.
//
// Re-implements the reference's analytic scene renderer (proj/src/synth.cpp,
// proj/include/rf/synth.hpp) on the host so that the product can generate
// the benchmark sequences without the reference: exact ray/plane/sphere/box
// intersections (synth.cpp:43-113), z-depth + Lambert RGB rendering
// (:136-171) and the orbit trajectory (:173-195).  Float expressions keep
// the reference's (Eigen) association order and the library is compiled with
// -ffp-contract=off, so frames are bit-identical to the reference's
// (tests/test_synth.py).  Scene 1 is the builder-defined multi-room scene of
// config C4 (open decision 5), mirrored in
// oracle/ref_driver.cpp:makeMultiRoom.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <vector>

#include "../../include/rfg.h"

namespace {

struct V3 {
  float x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 mul(float s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 mulr(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
inline float dot(V3 a, V3 b) { return a.x * b.x + (a.y * b.y + a.z * b.z); }
inline float sqn(V3 a) { return a.x * a.x + (a.y * a.y + a.z * a.z); }
inline float norm(V3 a) { return std::sqrt(sqn(a)); }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline V3 normalized(V3 a) {  // Eigen MatrixBase::normalized
  const float z = sqn(a);
  if (z > 0.f) {
    const float s = std::sqrt(z);
    return {a.x / s, a.y / s, a.z / s};
  }
  return a;
}
// Eigen unitOrthogonal_selector<.,3> (float precision 1e-5)
inline V3 unitOrthogonal(V3 s) {
  auto muchSmaller = [](float a, float b) { return std::abs(a) <= std::abs(b) * 1e-5f; };
  if (!muchSmaller(s.x, s.z) || !muchSmaller(s.y, s.z)) {
    const float invnm = 1.f / std::sqrt(s.x * s.x + s.y * s.y);
    return {-s.y * invnm, s.x * invnm, 0.f};
  }
  const float invnm = 1.f / std::sqrt(s.y * s.y + s.z * s.z);
  return {0.f, -s.z * invnm, s.y * invnm};
}

struct Rgb {
  uint8_t c[3];
};
struct Plane {
  V3 n;
  float d;
  Rgb colour;
  bool checker;
  float checkerSize;
  Rgb colour2;
};
struct Sphere {
  V3 c;
  float r;
  Rgb colour;
};
struct Box {
  V3 c, h;
  Rgb colour;
};
struct Scene {
  std::vector<Plane> planes;
  std::vector<Sphere> spheres;
  std::vector<Box> boxes;
};

Scene sphereInRoom() {  // synth.cpp:121-128
  Scene s;
  s.spheres.push_back({{0.f, 0.15f, 1.4f}, 0.3f, {{180, 120, 80}}});
  s.planes.push_back({{0, 0, -1}, -2.2f, {{190, 190, 190}}, true, 0.25f, {{90, 90, 90}}});
  s.planes.push_back({{0, -1, 0}, -0.45f, {{150, 170, 150}}, false, 0.1f, {{0, 0, 0}}});
  return s;
}
Scene multiRoom() {  // mirrors oracle/ref_driver.cpp:makeMultiRoom
  Scene s;
  s.planes.push_back({{0, -1, 0}, -0.45f, {{150, 170, 150}}, false, 0.1f, {{0, 0, 0}}});
  s.planes.push_back({{0, 1, 0}, -2.05f, {{210, 210, 210}}, false, 0.1f, {{0, 0, 0}}});
  const float wallT = 0.05f;
  s.boxes.push_back({{4.f, -0.8f, -2.f}, {6.f, 1.25f, wallT}, {{190, 180, 170}}});
  s.boxes.push_back({{4.f, -0.8f, 2.f}, {6.f, 1.25f, wallT}, {{170, 180, 190}}});
  s.boxes.push_back({{-2.f, -0.8f, 0.f}, {wallT, 1.25f, 2.f}, {{200, 160, 160}}});
  s.boxes.push_back({{10.f, -0.8f, 0.f}, {wallT, 1.25f, 2.f}, {{160, 200, 160}}});
  for (float x : {2.f, 6.f}) {
    s.boxes.push_back({{x, -0.8f, -1.25f}, {wallT, 1.25f, 0.75f}, {{180, 180, 200}}});
    s.boxes.push_back({{x, -0.8f, 1.25f}, {wallT, 1.25f, 0.75f}, {{180, 200, 180}}});
    s.boxes.push_back({{x, -1.5f, 0.f}, {wallT, 0.55f, 0.5f}, {{200, 200, 180}}});
  }
  s.boxes.push_back({{0.5f, 0.2f, 1.2f}, {0.5f, 0.25f, 0.4f}, {{120, 90, 60}}});
  s.boxes.push_back({{4.f, 0.05f, -1.3f}, {0.8f, 0.4f, 0.3f}, {{90, 120, 60}}});
  s.boxes.push_back({{8.3f, 0.15f, 1.f}, {0.4f, 0.3f, 0.6f}, {{60, 90, 120}}});
  s.spheres.push_back({{-0.8f, 0.1f, -1.f}, 0.35f, {{180, 120, 80}}});
  s.spheres.push_back({{3.2f, -0.2f, 1.1f}, 0.5f, {{80, 120, 180}}});
  s.spheres.push_back({{7.5f, 0.f, -0.9f}, 0.45f, {{160, 80, 160}}});
  return s;
}
Scene checkerWall() {  // synth.cpp:130-134
  Scene s;
  s.planes.push_back({{0, 0, -1}, -1.f, {{230, 230, 230}}, true, 0.1f, {{30, 30, 30}}});
  return s;
}

Rgb planeColour(const Plane& pl, V3 p) {  // synth.cpp:27-35
  if (!pl.checker) return pl.colour;
  const V3 u = unitOrthogonal(pl.n);
  const V3 v = cross(pl.n, u);
  const int iu = static_cast<int>(std::floor(dot(u, p) / pl.checkerSize));
  const int iv = static_cast<int>(std::floor(dot(v, p) / pl.checkerSize));
  return ((iu + iv) & 1) ? pl.colour2 : pl.colour;
}

// SyntheticScene::raycast (synth.cpp:43-113)
std::optional<float> raycast(const Scene& sc, V3 origin, V3 dir, float tMin, float tMax, Rgb* colour, V3* normal) {
  float best = tMax;
  bool hit = false;
  Rgb bestColour{{0, 0, 0}};
  V3 bestNormal{0, 0, 0};
  for (const auto& pl : sc.planes) {
    const float denom = dot(pl.n, dir);
    if (std::abs(denom) < 1e-12f) continue;
    const float t = (pl.d - dot(pl.n, origin)) / denom;
    if (t > tMin && t < best) {
      best = t;
      hit = true;
      bestColour = planeColour(pl, add(origin, mul(t, dir)));
      bestNormal = pl.n;
    }
  }
  for (const auto& s : sc.spheres) {
    const V3 oc = sub(origin, s.c);
    const float a = sqn(dir);
    const float b = 2.f * dot(oc, dir);
    const float c = sqn(oc) - s.r * s.r;
    const float disc = b * b - 4.f * a * c;
    if (disc < 0.f) continue;
    const float sq = std::sqrt(disc);
    const float ts[2] = {(-b - sq) / (2.f * a), (-b + sq) / (2.f * a)};
    for (const float t : ts) {
      if (t > tMin && t < best) {
        best = t;
        hit = true;
        bestColour = s.colour;
        bestNormal = normalized(sub(add(origin, mul(t, dir)), s.c));
        break;
      }
    }
  }
  for (const auto& bx : sc.boxes) {
    float t0 = tMin, t1 = best;
    bool ok = true;
    int hitAxis = -1;
    const float cA[3] = {bx.c.x, bx.c.y, bx.c.z}, hA[3] = {bx.h.x, bx.h.y, bx.h.z};
    const float oA[3] = {origin.x, origin.y, origin.z}, dA[3] = {dir.x, dir.y, dir.z};
    for (int a = 0; a < 3 && ok; ++a) {
      const float lo = cA[a] - hA[a], hi = cA[a] + hA[a];
      if (std::abs(dA[a]) < 1e-12f) {
        ok = oA[a] >= lo && oA[a] <= hi;
      } else {
        float ta = (lo - oA[a]) / dA[a];
        float tb = (hi - oA[a]) / dA[a];
        if (ta > tb) std::swap(ta, tb);
        if (ta > t0) {
          t0 = ta;
          hitAxis = a;
        }
        t1 = std::min(t1, tb);
        ok = t0 <= t1;
      }
    }
    if (ok && t0 > tMin && t0 < best && hitAxis >= 0) {
      best = t0;
      hit = true;
      bestColour = bx.colour;
      float n[3] = {0.f, 0.f, 0.f};
      n[hitAxis] = dA[hitAxis] > 0 ? -1.f : 1.f;
      bestNormal = {n[0], n[1], n[2]};
    }
  }
  if (!hit) return std::nullopt;
  if (colour) *colour = bestColour;
  if (normal) *normal = bestNormal;
  return best;
}

struct PoseF {
  float R[9];  // row-major
  float t[3];
};
PoseF inverse(const PoseF& p) {  // pose.hpp:33-36
  PoseF q;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) q.R[r * 3 + c] = p.R[c * 3 + r];
  for (int r = 0; r < 3; ++r) q.t[r] = -(q.R[r * 3] * p.t[0] + (q.R[r * 3 + 1] * p.t[1] + q.R[r * 3 + 2] * p.t[2]));
  return q;
}
V3 rot(const float* R, V3 x) {
  return {R[0] * x.x + (R[1] * x.y + R[2] * x.z), R[3] * x.x + (R[4] * x.y + R[5] * x.z),
          R[6] * x.x + (R[7] * x.y + R[8] * x.z)};
}
void to34(const PoseF& p, float* out) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) out[r * 4 + c] = p.R[r * 3 + c];
    out[r * 4 + 3] = p.t[r];
  }
}

// Look-at camera (y down), as orbit_trajectory (synth.cpp:181-193).
PoseF lookAt(V3 camPos, V3 target) {
  const V3 zAxis = normalized(sub(target, camPos));
  V3 up{0, 1, 0};
  if (std::abs(dot(up, zAxis)) > 0.99f) up = {1, 0, 0};
  const V3 xAxis = mulr(normalized(cross(up, zAxis)), -1.f);
  const V3 yAxis = cross(zAxis, xAxis);
  PoseF camToWorld;
  const V3 cols[3] = {xAxis, yAxis, zAxis};
  for (int c = 0; c < 3; ++c) {
    camToWorld.R[0 * 3 + c] = cols[c].x;
    camToWorld.R[1 * 3 + c] = cols[c].y;
    camToWorld.R[2 * 3 + c] = cols[c].z;
  }
  camToWorld.t[0] = camPos.x;
  camToWorld.t[1] = camPos.y;
  camToWorld.t[2] = camPos.z;
  return inverse(camToWorld);
}

}  // namespace

extern "C" {

int rfg_synth_orbit_poses(const float target3[3], float distance, int frames, float maxAngleRad, float* out34) {
  if (!target3 || !out34 || frames < 0) return RFG_EINVAL;
  const V3 target{target3[0], target3[1], target3[2]};
  for (int i = 0; i < frames; ++i) {
    const float a = frames > 1 ? maxAngleRad * (2.f * i / (frames - 1) - 1.f) : 0.f;
    const float b = frames > 1 ? 0.4f * maxAngleRad * std::sin(3.f * float(i) / frames) : 0.f;
    const V3 offset{std::sin(a) * std::cos(b), std::sin(b), -std::cos(a) * std::cos(b)};
    const V3 camPos = add(target, mul(distance, offset));
    to34(lookAt(camPos, target), out34 + 12 * i);
  }
  return RFG_OK;
}

// Builder-defined C4 trajectory: a walk along +x through both doorways with
// a slow yaw sweep (mirrors oracle/ref_driver.cpp:rr_multiroom_poses).
int rfg_synth_multiroom_poses(int frames, float* out34) {
  if (!out34 || frames < 0) return RFG_EINVAL;
  for (int i = 0; i < frames; ++i) {
    const float s = frames > 1 ? float(i) / float(frames - 1) : 0.f;
    const float x = -1.2f + 10.4f * s;
    const float z = 0.3f * std::sin(12.566371f * s);
    const float yaw = 0.6f * std::sin(18.849556f * s);
    const V3 camPos{x, -0.6f, z};
    const V3 fwd{std::cos(yaw), 0.1f, std::sin(yaw)};
    to34(lookAt(camPos, add(camPos, fwd)), out34 + 12 * i);
  }
  return RFG_OK;
}

// synth_render_depth (synth.cpp:136-171), noise 0.
int rfg_synth_render(int scene, const float pose34[12], const rfg_intrinsics* intr, float affScale, float affOffset,
                     int renderRgb, uint16_t* rawOut, float* depthOut, uint8_t* rgbOut) {
  if (!pose34 || !intr || intr->width <= 0 || intr->height <= 0) return RFG_EINVAL;
  const Scene sc = scene == 0 ? sphereInRoom() : (scene == 1 ? multiRoom() : checkerWall());
  PoseF pose;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) pose.R[r * 3 + c] = pose34[r * 4 + c];
    pose.t[r] = pose34[r * 4 + 3];
  }
  const PoseF camToWorld = inverse(pose);
  const V3 origin{camToWorld.t[0], camToWorld.t[1], camToWorld.t[2]};
  const int w = intr->width, h = intr->height;
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      if (rawOut) rawOut[i] = 0;
      if (depthOut) depthOut[i] = -1.f;
      if (rgbOut && renderRgb) rgbOut[3 * i] = rgbOut[3 * i + 1] = rgbOut[3 * i + 2] = 0;
      const V3 rd{(float(x) - intr->cx) / intr->fx, (float(y) - intr->cy) / intr->fy, 1.f};
      const V3 dirWorld = rot(camToWorld.R, rd);
      Rgb colour{{0, 0, 0}};
      V3 n{0, 0, 0};
      const auto t = raycast(sc, origin, dirWorld, 1e-4f, 100.f, &colour, &n);
      if (!t) continue;
      const float z = *t;
      if (depthOut) depthOut[i] = z;
      if (rawOut) {  // DepthAffine::toRaw (camera.hpp:56-61)
        const float r = std::round((z - affOffset) / affScale);
        rawOut[i] = !(r > 0.f) ? 0 : (r > 65535.f ? 65535 : static_cast<uint16_t>(r));
      }
      if (rgbOut && renderRgb) {
        const float lambert = std::abs(dot(n, normalized(dirWorld)));
        const float shade = 0.35f + 0.65f * lambert;
        for (int k = 0; k < 3; ++k) rgbOut[3 * i + k] = static_cast<uint8_t>(std::min(255.f, colour.c[k] * shade));
      }
    }
  }
  return RFG_OK;
}

}  // extern "C"
