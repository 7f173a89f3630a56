/* rfg.h — C ABI of the B200-native dense-fusion hot path (librfg.so).
 *
 * Drop-in replacement for the reference's per-frame engine calls
 * (/root/reference/proj).  The reference has no plugin/FFI layer: its
 * boundary is the concrete C++ API listed beside each entry point.  A C++
 * adapter with the reference's own names sits on top of this ABI in
 * include/rfg.hpp; Python binds it with ctypes (paper_1708_00783_b200/_lib.py).
 *
 * Conventions
 *  - Every call returns an int status (RFG_OK = 0, negative on error) and never
 *    throws; rfg_last_error() returns the message of the last failure on the
 *    calling thread.
 *  - Poses are row-major 3x4 [R | t] float arrays, world -> camera
 *    (proj/include/rf/raycast.hpp:21, proj/include/rf/synth.hpp:62).
 *  - Pointers named *_dev are device pointers owned by the caller; the map
 *    owns its hash table, voxel block array, free stacks, visible list and
 *    scratch in device memory.
 *  - Work is enqueued on the map's stream (rfg_map_set_stream); calls are
 *    asynchronous unless they return host data (stats, exports), which
 *    synchronise the stream.
 *  - A CUDA error or an invalid argument fails loudly with a status code;
 *    there is no CPU fallback.
 */
#ifndef RFG_H
#define RFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RFG_OK 0
#define RFG_EINVAL (-1)   /* invalid argument (e.g. non-power-of-two bucketCount) */
#define RFG_ECUDA (-2)    /* CUDA runtime error / no device */
#define RFG_ENOMEM (-3)   /* device allocation failed */
#define RFG_ERANGE (-4)   /* block coordinate outside the int16 entry layout, or DDA ordinal bound exceeded */
#define RFG_ESTATE (-5)   /* call order violated (e.g. ICP maps before expected ranges) */

typedef struct rfg_map rfg_map;

/* VoxelBlockMapConfig, proj/include/rf/voxel_block_map.hpp:36-45.
 * hasColour allocates the colour plane (ITMVoxel_s_rgb); 0 = depth-only
 * (ITMVoxel_s: 4-byte {sdf, w_depth} voxels). */
typedef struct {
  uint32_t bucketCount;
  uint32_t excessCount;
  uint32_t blockCapacity;
  int32_t hasColour;
} rfg_map_config;

/* Intrinsics, proj/include/rf/camera.hpp:13-47 */
typedef struct {
  int32_t width, height;
  float fx, fy, cx, cy;
} rfg_intrinsics;

/* SceneParams, proj/include/rf/fusion.hpp:11-20 */
typedef struct {
  float voxelSize;
  float mu;
  int32_t maxW;
  float viewFrustum_min;
  float viewFrustum_max;
  int32_t stopIntegratingAtMaxW;
} rfg_scene_params;

/* AllocationStats, proj/include/rf/fusion.hpp:22-27 */
typedef struct {
  int32_t requested, allocated, allocFailures, visibleCount;
} rfg_alloc_stats;

/* ------------------------------------------------------------------ map */
/* VoxelBlockMap::VoxelBlockMap(const VoxelBlockMapConfig&)
 * (proj/src/voxel_block_map.cpp:9-13): RFG_EINVAL when bucketCount is not a
 * power of two (the reference throws std::invalid_argument). */
int rfg_map_create(const rfg_map_config* cfg, int device, rfg_map** out);
int rfg_map_destroy(rfg_map* map);
/* VoxelBlockMap::clear (proj/src/voxel_block_map.cpp:15-24) */
int rfg_map_clear(rfg_map* map);
/* cudaStream_t to enqueue on (NULL = legacy default stream). */
int rfg_map_set_stream(rfg_map* map, void* cuda_stream);
int rfg_map_sync(rfg_map* map);
/* Multi-GPU spatial shard filter; world <= 1 disables. */
int rfg_map_set_shard(rfg_map* map, int rank, int world, int tile_shift);
const char* rfg_last_error(void);
/* Number of kernels this library has launched in the process. */
uint64_t rfg_kernel_launch_count(void);

/* ---------------------------------------------------------- fusion engine */
/* FusionEngine::allocate_from_depth (proj/src/fusion.cpp:144-235,
 * proj/include/rf/fusion.hpp:63-68).  depth_dev: level-0 metres (View::depth_m),
 * width*height floats, invalid <= 0.  stats may be NULL (fully asynchronous);
 * otherwise the call synchronises and fills it. */
int rfg_allocate_from_depth(rfg_map* map, const float* depth_dev, const rfg_intrinsics* intr, const float pose34[12],
                            const rfg_scene_params* params, rfg_alloc_stats* stats);

/* FusionEngine::integrate_frame (proj/src/fusion.cpp:237-263).  rgb_dev
 * (packed RGB8, intr_rgb sized) may be NULL for depth-only fusion;
 * extr34 = extrinsics_d_to_rgb (NULL = identity). */
int rfg_integrate(rfg_map* map, const float* depth_dev, const uint8_t* rgb_dev, const rfg_intrinsics* intr_d,
                  const rfg_intrinsics* intr_rgb, const float extr34[12], const float pose34[12],
                  const rfg_scene_params* params);

/* ------------------------------------------------------------- raycast */
/* render_expected_ranges (proj/src/raycast.cpp:86-127): range_dev receives
 * width*height float2 (min, max); unset pixels keep (FLT_MAX, -1). */
int rfg_render_expected_ranges(rfg_map* map, const float pose34[12], const rfg_intrinsics* intr,
                               const rfg_scene_params* params, float* range_dev);

/* render_maps(..., RenderMode::kIcpMaps, ...) (proj/src/raycast.cpp:129-139,
 * proj/include/rf/raycast.hpp:157-207).  Outputs are width*height float4
 * images: raycastResult (voxel coords, w = 1 hit), points (world metres),
 * normals (world unit normals); invalid = (0,0,0,-1). */
int rfg_render_icp_maps(rfg_map* map, const float pose34[12], const rfg_intrinsics* intr,
                        const rfg_scene_params* params, const float* range_dev, float* raycast_dev, float* points_dev,
                        float* normals_dev);

/* Approximate raycast (useApproximateRaycast).
 * forward_project (proj/src/raycast.cpp:141-188): the previous raycastResult
 * in raycast_dev is re-projected into new_pose34 (nearest point per pixel,
 * ties keep the first in row-major source order); points are set for the
 * forwarded pixels and normals left invalid, exactly as the reference.
 * has_raycast = 0 (no previous raycast) marks every pixel missing.  The
 * row-major linear indices (y * width + x) of the missing pixels go to
 * missing_dev (capacity width*height) and their count to *n_missing_dev. */
int rfg_forward_project(rfg_map* map, int has_raycast, float* raycast_dev, float* points_dev, float* normals_dev,
                        const float new_pose34[12], const rfg_intrinsics* intr, float voxel_size, int32_t* missing_dev,
                        int32_t* n_missing_dev);
/* render_maps(kIcpMaps, missingOnly) (proj/include/rf/raycast.hpp:200-202):
 * raycast only the listed pixels (device list and device count). */
int rfg_render_icp_maps_list(rfg_map* map, const float pose34[12], const rfg_intrinsics* intr,
                             const rfg_scene_params* params, const float* range_dev, const int32_t* missing_dev,
                             const int32_t* n_missing_dev, float* raycast_dev, float* points_dev, float* normals_dev);

/* render_maps with any RenderMode (raycast.hpp:28,157-207): mode 0 kIcpMaps
 * (= rfg_render_icp_maps), 1 kColour (colour_dev: RGB8 per pixel, the
 * trilinear colour at the hit — zero for depth-only maps, like an
 * un-coloured VoxelSRgb map), 2 kGrey (|n . ray| shading).  The _list form
 * is render_maps(..., missingOnly). */
int rfg_render_maps(rfg_map* map, const float pose34[12], const rfg_intrinsics* intr, const rfg_scene_params* params,
                    int mode, const float* range_dev, float* raycast_dev, float* points_dev, float* normals_dev,
                    uint8_t* colour_dev);
int rfg_render_maps_list(rfg_map* map, const float pose34[12], const rfg_intrinsics* intr,
                         const rfg_scene_params* params, int mode, const float* range_dev, const int32_t* missing_dev,
                         const int32_t* n_missing_dev, float* raycast_dev, float* points_dev, float* normals_dev,
                         uint8_t* colour_dev);

/* --------------------------------------------------------- swapping */
/* FusionEngine::Options (proj/include/rf/fusion.hpp:54-57). */
typedef struct {
  int32_t swapping_enabled;  /* visible list also keeps blocks within the margin (kBoundary = 3) */
  float swap_margin_px;      /* default 8 */
} rfg_fusion_options;
/* allocate_from_depth(..., const Options&) (fusion.hpp:63-66). */
int rfg_allocate_from_depth_ex(rfg_map* map, const float* depth_dev, const rfg_intrinsics* intr,
                               const float pose34[12], const rfg_scene_params* params,
                               const rfg_fusion_options* opts, rfg_alloc_stats* stats);
/* VoxelBlockMap::reserveBlockForEntry (returns 1 reserved / already
 * resident, 0 VBA exhausted) and releaseBlock (voxel_block_map.cpp:107-123). */
int rfg_map_reserve_block(rfg_map* map, int entry_index);
int rfg_map_release_block(rfg_map* map, int entry_index);
/* The swapping engine (rfg_swap.cu): a pinned, device-mapped
 * host slot per stored entry (the whole host tier is pinned at create when it
 * fits 4 GiB), at most `capacity` blocks per frame and direction, copied by
 * the GPU straight between VBA and host slots.  Larger host tiers grow in
 * pinned chunks of 65,536 slots; the environment variables
 * RFG_SWAP_PIN_UPFRONT (bytes) and RFG_SWAP_CHUNK_SLOTS, read at create,
 * lower both limits.
 * Per frame: rfg_allocate_from_depth_ex(swapping_enabled = 1) ->
 * rfg_swap_in (blocks visible but swapped out come back, ascending entry
 * index, merged into fresh VBA blocks) -> integrate / render ->
 * rfg_swap_out (blocks invisible for 2 frames go to the host, ascending
 * index).  Both wait for the device-side selection (one small readback);
 * the block copies stay queued on the map's stream (rfg_swap_host_block
 * synchronises before reading a slot). */
typedef struct rfg_swap rfg_swap;
int rfg_swap_create(rfg_map* map, int capacity_blocks, rfg_swap** out);
int rfg_swap_destroy(rfg_swap* swap);
int rfg_swap_in(rfg_swap* swap, int max_w, int* n_swapped_in);
int rfg_swap_out(rfg_swap* swap, int* n_swapped_out);
/* host tier export (tests): per-entry stored flags and invisible-frame ages
 * (totalEntries bytes each, either may be NULL); one stored block as
 * VoxelSRgb bytes */
int rfg_swap_export(rfg_swap* swap, uint8_t* has_out, uint8_t* age_out);
int rfg_swap_host_block(rfg_swap* swap, int entry_index, uint8_t* voxels_srgb_4096);

/* ---------------------------------------------------------------- mesh */
/* extract_mesh (proj/src/meshing.cpp:144-217): marching cubes over the
 * in-memory blocks of the map.  Vertices (metres) and triangles come out in
 * exactly the reference's order (entry index, cell order, table order; a
 * vertex numbered where its cell edge first appears).  The result stays in
 * map-owned device memory until the next extraction; rfg_mesh_copy copies it
 * to host or device buffers (3 floats per vertex, 3 uint32 per triangle).
 * Synchronous (the sizes are read back). */
int rfg_extract_mesh(rfg_map* map, float voxel_size, int64_t* n_vertices, int64_t* n_triangles);
int rfg_mesh_copy(rfg_map* map, float* vertices3, uint32_t* triangles3);
/* The 256-case triangulation table (meshing.cpp:27-118 marchingCubesTable):
 * counts[m] triangles of cell-edge triples, tris[(m*16 + k)*3 + j], -1 pad. */
int rfg_mc_table(int32_t counts256[256], int32_t tris[256 * 16 * 3]);

/* ---------------------------------------------------------------- view */
/* build_view depth path (proj/src/view.cpp:100-143): raw u16 -> metres
 * (m = raw*scale + offset, raw == 0 or m <= 0 -> -1) and `levels` pyramid
 * levels by 2x2 valid-mean (downsample_depth, view.cpp:69-88), written
 * back to back into depth_levels_dev. */
int rfg_build_view_depth(const uint16_t* raw_dev, int width, int height, float aff_scale, float aff_offset, int levels,
                         float* depth_levels_dev, void* cuda_stream);

/* Full ViewBuilder (proj/src/view.cpp:8-143, build_view with every option):
 * raw u16 depth (host byte order, or the big-endian payload of a PGM16 file
 * when raw_big_endian = 1, image_io.cpp:96-113) -> metres; bilateral = 1
 * applies bilateral_filter(depth, 2, 10 |aff_scale|) (needs scratch_dev,
 * width*height floats); normals_dev (float4 per pixel, may be NULL) =
 * compute_normals of the level-0 depth; with rgb_dev (packed RGB8, may be
 * NULL) intensity_levels_dev gets rgb_to_intensity + downsample_intensity
 * levels.  Depth / intensity levels are written back to back.  The filter's
 * std::exp is reproduced bit-for-bit (glibc expf, see rfg_view.cu). */
int rfg_build_view(const uint16_t* raw_dev, const uint8_t* rgb_dev, const rfg_intrinsics* intr_d, float aff_scale,
                   float aff_offset, int bilateral, int levels, int raw_big_endian, float* depth_levels_dev,
                   float* intensity_levels_dev, float* normals_dev, float* scratch_dev, void* cuda_stream);
/* The ViewBuilder's elements (view.hpp:44-62), device images. */
int rfg_bilateral_filter(const float* depth_dev, int width, int height, float spatial_sigma, float range_sigma,
                         float* out_dev, void* cuda_stream);
int rfg_compute_normals(const float* depth_dev, const rfg_intrinsics* intr, float* normals_dev, void* cuda_stream);
int rfg_rgb_to_intensity(const uint8_t* rgb_dev, int width, int height, float* out_dev, void* cuda_stream);
int rfg_downsample_intensity(const float* in_dev, int width, int height, float* out_dev, void* cuda_stream);

/* ------------------------------------------------------------ image IO */
/* Netpbm IO (proj/src/image_io.cpp, host memory).  The readers return
 * RFG_EINVAL with the reference's exception message (rfg_last_error) on a
 * missing file, wrong magic / maxval or truncated data, and RFG_ERANGE when
 * capacity (pixels) is too small; *width / *height are set either way when
 * the header parsed.  read_pgm16 returns host-order values;
 * read_pgm16_payload returns the pixel bytes as stored (big-endian), to be
 * uploaded as-is and decoded on the GPU (rfg_build_view raw_big_endian = 1,
 * rfg_pipeline_process_pgm). */
int rfg_read_pgm16(const char* path, uint16_t* out, int64_t capacity, int* width, int* height);
int rfg_read_pgm16_payload(const char* path, void* out, int64_t capacity, int* width, int* height);
int rfg_read_ppm(const char* path, uint8_t* out_rgb, int64_t capacity, int* width, int* height);
int rfg_write_pgm16(const char* path, const uint16_t* img, int width, int height);
int rfg_write_ppm(const char* path, const uint8_t* rgb, int width, int height);

/* ----------------------------------------------------------------- ICP */
/* Point-to-plane ICP tracker (ITMDepthTracker; absent in the reference, see
 * DESIGN.md "ICP oracle" and SPEC.md:333-356).  depth_levels_dev as produced
 * by rfg_build_view_depth; points/normals_dev and render_pose34 describe the
 * previous ICP-map render at level-0 resolution.  iters[3] per level (level 0
 * = finest), dist[3] outlier gates (m, in (0, 2]).  pose_out34 = tracked
 * world->camera; a degenerate Hessian (det(H/n) < 1e-12) returns
 * init_pose34 with ok = 0.  stats12 = TrackerIterationSummary
 * of the last evaluation, indexed by RFG_ICP_*: iterations, inliers,
 * sum r^2, converged, iterations per level x3, ok, inlier_fraction,
 * hessian_det (det(H/n)), residual_mean (sum |r| / inliers), valid pixels.
 * The sums are fixed-point integers (bit-identical to the CPU oracle); a
 * world point with a coordinate beyond +-128 m returns RFG_ERANGE. */
#define RFG_ICP_STATS 12
#define RFG_ICP_SUMS 31
enum {
  RFG_ICP_ITERATIONS = 0, RFG_ICP_COUNT = 1, RFG_ICP_RESIDUAL_SUM = 2, RFG_ICP_CONVERGED = 3, RFG_ICP_IT_L0 = 4,
  RFG_ICP_IT_L1 = 5, RFG_ICP_IT_L2 = 6, RFG_ICP_OK = 7, RFG_ICP_INLIER_FRACTION = 8, RFG_ICP_HESSIAN_DET = 9,
  RFG_ICP_RESIDUAL_MEAN = 10, RFG_ICP_VALID = 11
};
int rfg_icp_track(rfg_map* map, const float* depth_levels_dev, int levels, const rfg_intrinsics* intr,
                  const float* points_dev, const float* normals_dev, const float render_pose34[12],
                  const float init_pose34[12], const int iters[3], const float dist[3], int min_count,
                  float pose_out34[12], double stats12[RFG_ICP_STATS]);
/* One evaluation of the 31 normal-equation sums (H upper 21, g 6, sum r^2,
 * inliers, sum |r|, valid pixels) at pyramid level `level` for camera->world
 * pose cam_to_world34: fixed31 = the fixed-point integers (H 2^-32, g 2^-38,
 * r^2 and |r| 2^-44 units, counts), out31 = decoded doubles; either may be
 * NULL. */
int rfg_icp_reduce(rfg_map* map, const float* depth_level_dev, int level, const rfg_intrinsics* intr,
                   const float* points_dev, const float* normals_dev, const float render_pose34[12],
                   const float cam_to_world34[12], float dist, int64_t fixed31[RFG_ICP_SUMS],
                   double out31[RFG_ICP_SUMS]);

/* Tracker phase timers of CTA 0 (ns, accumulated since the last reset):
 * {associate + block reduce + atomics, grid barrier wait, read totals, solve,
 *  iterations, 0, 0, 0}.  Synchronises the map's stream. */
int rfg_icp_timers(rfg_map* map, uint64_t out8[8], int reset);

/* ------------------------------------------------------ frame pipeline */
/* The per-frame driver (ITMMainEngine::ProcessFrame order):
 * [track] -> allocate -> integrate -> expected ranges -> ICP-map raycast,
 * device resident, capturable in a CUDA graph.  The pose of each frame
 * lives on the device (tracked or supplied). */
typedef struct rfg_pipeline rfg_pipeline;
typedef struct {
  rfg_intrinsics intr;     /* depth camera, level 0 */
  rfg_scene_params params;
  float aff_scale, aff_offset;  /* DepthAffine */
  int32_t levels;          /* pyramid levels (1..3) */
  int32_t track;           /* 1 = ICP tracking from the previous render */
  int32_t iters[3];
  float dist[3];
  int32_t min_count;
  int32_t use_graph;       /* capture the frame into a CUDA graph */
  int32_t profile;         /* record CUDA events between stages (graph mode: event-record nodes) */
  int32_t bilateral;       /* ViewBuildOptions::bilateral (view.hpp:13) */
  int32_t raw_big_endian;  /* raw frames are PGM16 payloads (decoded in the view stage) */
  /* ITMVoxel_s_rgb colour fusion (BASELINE configs[2]): the map must have a
   * colour plane and frames come with an RGB8 image (rfg_pipeline_process_rgbd_*) */
  int32_t colour;
  rfg_intrinsics intr_rgb;        /* RgbdCalib::intrinsics_rgb */
  float extr_d_to_rgb[12];        /* RgbdCalib::extrinsics_d_to_rgb (row-major 3x4) */
} rfg_pipeline_config;

int rfg_pipeline_create(rfg_map* map, const rfg_pipeline_config* cfg, rfg_pipeline** out);
int rfg_pipeline_destroy(rfg_pipeline* p);
/* Enqueue one frame from raw depth already on the device.  pose34 (host) is
 * used when tracking is off or for the first frame; NULL keeps the device
 * pose.  Asynchronous. */
int rfg_pipeline_process_raw(rfg_pipeline* p, const uint16_t* raw_dev, const float* pose34);
/* As rfg_pipeline_process_raw for a frame produced on another CUDA stream:
 * the pipeline reads it after the producer stream's pending work, and the
 * producer stream's later work waits until the frame has been read.  Once
 * the frame graph is captured, the frame is read in place (its view kernel
 * is re-pointed at raw_dev) instead of being copied. */
int rfg_pipeline_process_raw_stream(rfg_pipeline* p, const uint16_t* raw_dev, const float pose34[12],
                                    void* producer_cuda_stream);
/* Enqueue one frame from HOST raw depth, copied H2D on the pipeline's
 * stream.  A pageable frame's buffer may be reused once the call returns; a
 * pinned (cudaHostAlloc / cudaHostRegister) frame is copied asynchronously,
 * so — as with any asynchronous copy from pinned memory — the caller keeps
 * the buffer unchanged until rfg_pipeline_result returns. */
int rfg_pipeline_process_host(rfg_pipeline* p, const uint16_t* raw_host, const float* pose34);
/* RGB-D frames of a colour pipeline (cfg.colour = 1): depth as in
 * rfg_pipeline_process_raw_stream / _host plus the RGB8 image (width x height
 * x 3 bytes, intr_rgb's size): a device image is read in place by the
 * captured graph's colour packing kernel, a host image is copied H2D with
 * the depth (pinned: asynchronously, kept unchanged until the result). */
int rfg_pipeline_process_rgbd_stream(rfg_pipeline* p, const uint16_t* raw_dev, const uint8_t* rgb_dev,
                                     const float pose34[12], void* producer_cuda_stream);
int rfg_pipeline_process_rgbd_host(rfg_pipeline* p, const uint16_t* raw_host, const uint8_t* rgb_host,
                                   const float pose34[12]);
/* One frame straight from a PGM16 file (image_io.cpp:96-113): the payload is
 * read into pinned staging and uploaded as stored; with raw_big_endian = 1
 * the GPU view stage decodes it (no host pass over the pixels). */
int rfg_pipeline_process_pgm(rfg_pipeline* p, const char* path, const float pose34[12]);
/* Read back the last frame's stats, pose and tracker summary (RFG_ICP_STATS
 * doubles, see rfg_icp_track): the frame graph itself writes them into mapped
 * pinned host memory (the map state as the frame's allocation left it), so
 * this only synchronises the pipeline's stream. */
int rfg_pipeline_result(rfg_pipeline* p, rfg_alloc_stats* stats, float pose_out34[12],
                        double icp_stats[RFG_ICP_STATS]);
/* Device pointers of the pipeline's buffers (for parity checks). */
int rfg_pipeline_buffers(rfg_pipeline* p, float** depth_levels, float** range, float** raycast, float** points,
                         float** normals);
/* Reset the device pose / tracking state (not the map). */
int rfg_pipeline_reset(rfg_pipeline* p);
/* Per-stage device times (ms) of the last frame when cfg.profile = 1:
 * {view, icp, allocate, integrate, ranges, raycast, total}.  Synchronises. */
int rfg_pipeline_stage_times(rfg_pipeline* p, float ms7[7]);
/* The pipeline's stream (cudaStream_t) for event timing by the caller. */
void* rfg_pipeline_stream(rfg_pipeline* p);
/* Device pointer to the pipeline's current world->camera pose (12 floats,
 * row-major 3x4; written by the tracker or rfg_pipeline_process*'s pose34),
 * valid for work ordered after the frame on the pipeline's stream.  The
 * three maps of rfg_pipeline_buffers are one allocation, in the order
 * raycast | points | normals (3 x width x height float4). */
int rfg_pipeline_pose_buffer(rfg_pipeline* p, float** pose_dev);

/* --------------------------------------------- multi-GPU composition */
/* Per-pixel nearest-hit composition of spatially sharded renders
 * (SURVEY.md §8(e)).  keys_dev[i] = (float bits of the hit's camera z) << 32
 * | rank for a hit pixel, INT64_MAX for a miss; after an all-reduce MIN of
 * the keys, rfg_compose_select zeroes every pixel this rank did not win (rank
 * 0 keeps the invalid marker on pixels nobody hit), so an all-reduce SUM of
 * the three maps yields the composed render exactly. */
int rfg_compose_keys(const float* points_dev, const float pose34[12], int rank, int n, int64_t* keys_dev,
                     void* cuda_stream);
/* Same, with the pose read on the device (e.g. rfg_pipeline_pose_buffer). */
int rfg_compose_keys_dev(const float* points_dev, const float* pose34_dev, int rank, int n, int64_t* keys_dev,
                         void* cuda_stream);
int rfg_compose_select(const int64_t* keymin_dev, int rank, int n, float* raycast_dev, float* points_dev,
                       float* normals_dev, void* cuda_stream);

/* --------------------------------------------------------------- export */
uint32_t rfg_total_entries(const rfg_map* map);
/* Host copies for parity: entries as 5 int32 {x, y, z, offset, ptr}
 * (HashEntry, voxel_block_map.hpp:17-27) */
int rfg_export_entries(rfg_map* map, int32_t* out5_host);
/* VoxelSRgb bytes {sdf lo, sdf hi, w_depth, r, g, b, w_color, 0} of the given
 * VBA blocks (512 voxels each) */
int rfg_export_blocks(rfg_map* map, const int32_t* ptrs_host, int n, uint8_t* out_host);
/* visibleList in the reference's ascending entry order (fusion.cpp:231;
 * the frame's kernels append it unordered, and this call rebuilds the order
 * on the device from the visibility bytes) and per-entry visibility bytes
 * (nullable); returns the count in *count */
int rfg_export_visible(rfg_map* map, int32_t* list_host, uint8_t* types_host, int32_t* count);
int rfg_free_counts(rfg_map* map, int32_t* free_blocks, int32_t* free_excess);

/* ------------------------------------------------------------ synthetic */
/* Synthetic analytic scenes (the reference's synth module,
 * proj/src/synth.cpp, re-implemented as a frame source for benchmarks):
 * scene 0 = make_sphere_in_room_scene, 1 = multi-room (C4), 2 = checker wall. */
int rfg_synth_orbit_poses(const float target3[3], float distance, int frames, float max_angle, float* out34);
int rfg_synth_multiroom_poses(int frames, float* out34);
int rfg_synth_render(int scene, const float pose34[12], const rfg_intrinsics* intr, float aff_scale, float aff_offset,
                     int render_rgb, uint16_t* raw_out, float* depth_out, uint8_t* rgb_out);

#ifdef __cplusplus
}
#endif
#endif /* RFG_H */
