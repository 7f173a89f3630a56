/* oracle/rfo.h — CPU restatement oracle of the dense-fusion hot path.
 *
 * TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load oracle/_build/librfo.so, and only as the checker.
 *
 * Plain C11, compiled with -ffp-contract=off.  Every function restates the
 * reference (/root/reference/proj) at the file:line cited beside it, with the
 * float association order of the reference's Eigen expressions
 * (oracle/shim/Eigen/Core documents the order: 3-term sums are e0+(e1+e2)).
 * It is pinned bit-for-bit against the reference itself compiled here
 * (oracle/_ref/librfref.so) by tests/test_oracle_pin.py.
 *
 * Conventions shared with the product C-ABI (include/rfg.h):
 *   pose12  row-major 3x4 [R|t], world -> camera (proj/include/rf/raycast.hpp:21)
 *   wh[2]   image width, height;  f4[4] = fx, fy, cx, cy
 *   params6 voxelSize, mu, maxW, viewFrustum_min, viewFrustum_max, stopIntegratingAtMaxW
 *   voxel   8 bytes = VoxelSRgb {int16 sdf, u8 w_depth, u8 clr[3], u8 w_color, pad}
 *   entry   5 int32 = HashEntry {x, y, z, offset, ptr}
 */
#ifndef RFO_H
#define RFO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rfo_map rfo_map;

/* threads for the per-pixel raycast loops (default 1; output is independent of it) */
void rfo_set_threads(int n);

uint32_t rfo_hash_index(const int* pos3, uint32_t mask);
int rfo_traverse_blocks(const float* a3, const float* b3, int* cellsOut, int maxCells);
int rfo_block_in_frustum(const int* pos3, const float* pose12, const int* wh, const float* f4, const float* params6);
float rfo_update_voxel_depth(uint8_t* voxel8, const float* pt3, const float* pose12, const int* wh, const float* f4,
                             float mu, int maxW, const float* depth, int stopAtMaxW);

rfo_map* rfo_create(uint32_t buckets, uint32_t excess, uint32_t capacity);
void rfo_destroy(rfo_map* m);
void rfo_clear(rfo_map* m);
/* Spatial sharding filter (multi-GPU parity oracle):
 * a block is kept on `rank` when any block of its 3x3x3 neighbourhood is
 * owned by `rank`; owner = hash of the (block >> tileShift) super-tile mod world.
 * world <= 1 disables the filter. */
void rfo_set_shard(rfo_map* m, int rank, int world, int tileShift);

int rfo_allocate(rfo_map* m, const float* depth, const int* wh, const float* f4, const float* pose12,
                 const float* params6, int* stats4);
int rfo_integrate(rfo_map* m, const float* depth, const uint8_t* rgb, const int* whD, const float* f4D,
                  const int* whRgb, const float* f4Rgb, const float* extr12, const float* pose12,
                  const float* params6);
int rfo_render_ranges(rfo_map* m, const float* pose12, const int* wh, const float* f4, const float* params6,
                      float* rangeOut);
int rfo_set_ranges(rfo_map* m, const int* wh, const float* rangeIn);
int rfo_render_icp(rfo_map* m, const float* pose12, const int* wh, const float* f4, const float* params6,
                   float* raycastOut, float* pointsOut, float* normalsOut);

/* Approximate raycast (useApproximateRaycast): forward_project
 * (proj/src/raycast.cpp:141-188) and render_maps(kIcpMaps, missingOnly)
 * (proj/include/rf/raycast.hpp:200-202).  Images are caller-owned in/out. */
int rfo_forward_project(int hasRaycast, float* raycast, float* points, float* normals, const float* newPose12,
                        const int* wh, const float* f4, float voxelSize, int* missingXY);
int rfo_render_icp_list(rfo_map* m, const float* pose12, const int* wh, const float* f4, const float* params6,
                        const int* missingXY, int n, float* raycastOut, float* pointsOut, float* normalsOut);

/* build_view depth path (proj/src/view.cpp:112-119,134-142): level 0 then each
 * pyramid level, concatenated into depthLevels. */
int rfo_build_view(const uint16_t* raw, const int* wh, float affScale, float affOffset, int levels,
                   float* depthLevels);
int rfo_render_colour(const rfo_map* m, int mode, const float* pose12, const int* wh, const float* f4,
                      const float* raycast, const float* normals, const int* list, int nList, uint8_t* rgbOut);
/* swapping: reference hooks + the SPEC's engine */
void rfo_set_fusion_options(rfo_map* m, int swappingEnabled, float swapMarginPx);
int rfo_reserve_block(rfo_map* m, int idx);
void rfo_release_block(rfo_map* m, int idx);
/* marching cubes (meshing.cpp) */
int rfo_mc_table(int* counts256, int* tris);
int rfo_extract_mesh(const rfo_map* m, float voxelSize, float** vOut, uint32_t** tOut, long long* nV, long long* nT);
void rfo_free(void* p);
int rfo_set_block(rfo_map* m, const int* pos3, const int16_t* sdf512, const uint8_t* w512);
/* full ViewBuilder (view.cpp:8-143) */
void rfo_rgb_to_intensity(const uint8_t* rgb, int w, int h, float* out);
void rfo_bilateral_filter(const float* in, int w, int h, float spatialSigma, float rangeSigma, float* out);
void rfo_compute_normals(const float* depth, int w, int h, const float* f4, float* out4);
void rfo_downsample_intensity(const float* in, int w, int h, float* out);
int rfo_build_view_full(const uint16_t* raw, const uint8_t* rgb, const int* wh, const float* f4, float affScale,
                        float affOffset, int bilateral, int levels, float* depthLevels, float* intensityLevels,
                        float* normals4);

/* ICP point-to-plane depth tracker (absent in the reference; restated from
 * see DESIGN.md "ICP oracle").
 *   depthLevels: pyramid as produced by rfo_build_view, level 0 is wh
 *   points/normals: last render (float4 per pixel, w > 0 valid), renderPose12
 *   and renderF4 describe that render (resolution wh).
 *   icp6 = {levels, iters_l0, iters_l1, iters_l2, minCount, reserved}
 *   dist3 = outlier distance gate per level (metres, <= 2)
 *   poseOut12 = tracked world->camera pose; statsOut12 = TrackerIterationSummary
 *   {iterations run, inliers, sum r^2, converged, per-level iterations x3, ok,
 *    inlier_fraction, hessian_det = det(H/n), residual_mean = sum|r|/n, valid px}
 * Returns 0, or -2 when a world point is outside the fixed-point range. */
int rfo_icp_track(const float* depthLevels, const int* wh, const float* f4, const float* points,
                  const float* normals, const float* renderPose12, const float* renderF4, const float* initPose12,
                  const int* icp6, const float* dist3, float* poseOut12, double* statsOut12);
/* One ICP evaluation at a given level and float pose: the 31 fixed-point sums
 * (sums31, int64) and their decoded doubles (out31): H upper (21, row-major),
 * g (6), sum r^2, n, sum |r|, valid pixels.  Either output may be NULL. */
int rfo_icp_reduce(const float* depth, int lw, int lh, const float* f4l, const float* points, const float* normals,
                   const int* wh, const float* renderPose12, const float* renderF4, const float* camToWorld12,
                   float dist, int64_t* sums31, double* out31);

/* the Rodrigues coefficients sin t/t, (1-cos t)/t^2, (t-sin t)/t^3 at th2 = t^2 */
void rfo_se3_coeffs(double th2, double* abc3);
/* LDL^T solve of H delta = -g from the decoded sums; det(H/n) to *det;
 * -1 when degenerate. */
int rfo_solve6(const double* sums31, double* x, double* det);

uint32_t rfo_total_entries(const rfo_map* m);
int rfo_export_entries(const rfo_map* m, int* out5);
int rfo_export_blocks(const rfo_map* m, const int* ptrs, int n, uint8_t* out);
int rfo_export_visible(const rfo_map* m, int* listOut, uint8_t* typesOut);
int rfo_free_counts(const rfo_map* m, int* nb, int* ne);

#ifdef __cplusplus
}
#endif
#endif
