// C++ use of the drop-in adapter (include/rfg.hpp), written like the
// reference's own doctest cases.  Without a GPU it checks the error contract
// and exits 0; with one it fuses a short synthetic sequence through the
// public pipeline and checks the reference's frame-0 statistics.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "rfg.hpp"

static int failures = 0;
#define CHECK(x)                                                   \
  do {                                                             \
    if (!(x)) {                                                    \
      std::fprintf(stderr, "%s:%d: FAILED %s\n", __FILE__, __LINE__, #x); \
      ++failures;                                                  \
    }                                                              \
  } while (0)

int main() {
  // voxel_block_map.cpp:10-11 — non-power-of-two bucket count throws
  bool threw = false;
  try {
    rfg::VoxelBlockMap bad({1000, 16, 16});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);

  // image_io.cpp round trip + the reference's error messages (host only)
  {
    rfg::HostImage<std::uint16_t> img;
    img.width = 37;
    img.height = 23;
    for (int i = 0; i < 37 * 23; ++i) img.data.push_back(static_cast<std::uint16_t>(i * 977));
    rfg::write_pgm16(img, "/tmp/rfg_adapter_test.pgm");
    const auto back = rfg::read_pgm16("/tmp/rfg_adapter_test.pgm");
    CHECK(back.width == 37 && back.height == 23 && back.data == img.data);
    bool missing = false;
    try {
      (void)rfg::read_pgm16("/tmp/rfg_adapter_test_missing.pgm");
    } catch (const std::runtime_error& e) {
      missing = std::string(e.what()).find("cannot open") != std::string::npos;
    }
    CHECK(missing);
  }

  try {
    rfg::VoxelBlockMap map({0x40000, 0x20000, 0x40000});
    const rfg::Intrinsics intr{640, 480, 525.f, 525.f, 319.5f, 239.5f};
    const rfg::SceneParams params;
    const auto poses = rfg::orbit_trajectory({0.f, 0.15f, 1.4f}, 1.4f, 100);
    rfg::Pipeline pipe(map, intr, params, 1.f / 5000.f, 0.f, 3, /*track=*/false);
    std::vector<std::uint16_t> raw(640 * 480);
    std::vector<float> depth(640 * 480);
    const rfg_intrinsics ci = intr.c();
    rfg_synth_render(0, poses[0].data(), &ci, 1.f / 5000.f, 0.f, 0, raw.data(), depth.data(), nullptr);
    pipe.processHost(raw.data(), &poses[0]);
    const rfg::AllocationStats st = pipe.result();
    // the reference's frame-0 statistics on C1 (tests/golden/c1_frames.json)
    CHECK(st.requested == 8349 && st.allocated == 8349 && st.allocFailures == 0 && st.visibleCount == 8349);
    CHECK(map.allocatedBlockCount() == 8349);
    // marching cubes on the fused map (meshing.cpp:144-217)
    const rfg::Mesh mesh = rfg::extract_mesh(map, params.voxelSize);
    CHECK(mesh.triangles.size() > 10000 && mesh.vertices.size() > 5000);
    for (const auto& t : mesh.triangles) CHECK(t[0] < mesh.vertices.size() && t[2] < mesh.vertices.size());
    // releaseBlock / reserveBlockForEntry (voxel_block_map.cpp:107-123)
    const auto ents = map.entries();
    int idx = -1;
    for (int i = 0; i < static_cast<int>(ents.size()) && idx < 0; ++i)
      if (ents[i].inMemory()) idx = i;
    map.releaseBlock(idx);
    CHECK(map.entries()[idx].ptr == -1 && map.allocatedBlockCount() == 8348);
    CHECK(map.reserveBlockForEntry(idx) && map.entries()[idx].inMemory());
    // the tracked pipeline (C2): frame 0 at its pose, then tracking; the
    // summary of the last evaluation
    {
      rfg::VoxelBlockMap tmap({0x40000, 0x20000, 0x40000});
      rfg::Pipeline tp(tmap, intr, params, 1.f / 5000.f, 0.f, 3, /*track=*/true);
      rfg::TrackerIterationSummary ts;
      for (int f = 0; f < 4; ++f) {
        rfg_synth_render(0, poses[f].data(), &ci, 1.f / 5000.f, 0.f, 0, raw.data(), depth.data(), nullptr);
        tp.processHost(raw.data(), f == 0 ? &poses[0] : nullptr);
        rfg::Pose34 pose;
        tp.result(&pose, &ts);
        if (f > 0) {
          CHECK(ts.ok && ts.iterations > 0 && ts.inlierFraction > 0.5 && ts.inlierFraction <= 1.0);
          CHECK(ts.hessianDet > 1e-12);
          float err = 0.f;
          for (int r = 0; r < 3; ++r) err = std::max(err, std::abs(pose[r * 4 + 3] - poses[f][r * 4 + 3]));
          CHECK(err < 2e-3f);  // tracks the synthetic orbit
        }
      }
    }
    // colour fusion (C3): a colour map, RGB-D frames
    {
      rfg::VoxelBlockMap cmap({0x40000, 0x20000, 0x40000}, /*colour=*/true);
      rfg::SceneParams p4;
      p4.voxelSize = 0.004f;
      rfg::Pipeline cp(cmap, intr, p4, 1.f / 5000.f, 0.f, 1, /*track=*/false, /*colour=*/true);
      std::vector<std::uint8_t> rgb(640 * 480 * 3);
      rfg_synth_render(0, poses[0].data(), &ci, 1.f / 5000.f, 0.f, 1, raw.data(), depth.data(), rgb.data());
      cp.processRgbdHost(raw.data(), rgb.data(), &poses[0]);
      const rfg::AllocationStats cs = cp.result();
      CHECK(cs.allocated > 10000 && cs.allocFailures == 0);
    }
    std::printf("adapter_test: GPU sequence ok\n");
  } catch (const rfg::Error& e) {
    CHECK(e.code() == RFG_ECUDA);  // no device: fail loudly, no CPU fallback
    std::printf("adapter_test: no GPU (%s)\n", e.what());
  }
  return failures ? 1 : 0;
}
