/* oracle/rfo.c — CPU restatement oracle (TEST INFRASTRUCTURE ONLY; see rfo.h).
 *
 * Float association follows the reference's Eigen expressions
 * (3-term reductions e0 + (e1 + e2); mat*vec row i = R_i0 x0 + (R_i1 x1 + R_i2 x2)).
 * Compiled with -ffp-contract=off, so no FMA contraction.
 */
#include "rfo.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Threads for the per-pixel raycast loops (rfo_set_threads).  Default 1: the
 * oracle is a single-threaded restatement; tests may raise it to shorten long
 * parity runs.  Every pixel is independent and reads the map only, so the
 * output does not depend on the thread count. */
static int g_threads = 1;
void rfo_set_threads(int n) { g_threads = n > 0 ? n : 1; }

typedef struct {
  float x, y, z;
} v3;
typedef struct {
  int x, y, z;
} i3;
typedef struct {
  float R[9]; /* row-major */
  float t[3];
} pose_t;
typedef struct {
  int w, h;
  float fx, fy, cx, cy;
} intr_t;
typedef struct {
  float voxelSize, mu;
  int maxW;
  float vfMin, vfMax;
  int stopAtMaxW;
} params_t;
typedef struct {
  int x, y, z, offset, ptr;
} entry_t;
typedef struct {
  int16_t sdf;
  uint8_t w;
  uint8_t clr[3];
  uint8_t wc;
  uint8_t pad;
} voxel_t;

#define BS 8
#define BS3 512
#define SDF_ONE 32767

struct rfo_map {
  uint32_t buckets, excess, capacity;
  entry_t* entries;
  voxel_t* vba;
  int* freeBlocks;
  int nFreeBlocks;
  int* freeExcess;
  int nFreeExcess;
  int* visible;
  int nVisible;
  uint8_t* visibility;
  /* FusionEngine scratch (proj/include/rf/fusion.hpp:76-78) */
  uint8_t* allocType;
  i3* blockCoords;
  uint8_t* marked;
  /* RenderState.expectedRange (proj/include/rf/raycast.hpp:16) */
  float* range;
  int rangeW, rangeH;
  /* shard filter */
  int rank, world, tileShift;
  /* FusionEngine::Options (proj/include/rf/fusion.hpp:54-57) */
  int swapping;
  float swapMargin;
};

/* ------------------------------------------------------------ core math */
/* proj/include/rf/pose.hpp:29 apply = R*x + t; Eigen lazy-product order */
static v3 pose_apply(const pose_t* p, v3 x) {
  v3 o;
  o.x = (p->R[0] * x.x + (p->R[1] * x.y + p->R[2] * x.z)) + p->t[0];
  o.y = (p->R[3] * x.x + (p->R[4] * x.y + p->R[5] * x.z)) + p->t[1];
  o.z = (p->R[6] * x.x + (p->R[7] * x.y + p->R[8] * x.z)) + p->t[2];
  return o;
}
/* R * x without translation */
static v3 rot_apply(const float* R, v3 x) {
  v3 o;
  o.x = R[0] * x.x + (R[1] * x.y + R[2] * x.z);
  o.y = R[3] * x.x + (R[4] * x.y + R[5] * x.z);
  o.z = R[6] * x.x + (R[7] * x.y + R[8] * x.z);
  return o;
}
/* proj/include/rf/pose.hpp:33-36 inverse = (R^T, -(R^T t)) */
static pose_t pose_inverse(const pose_t* p) {
  pose_t q;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) q.R[r * 3 + c] = p->R[c * 3 + r];
  v3 t = {p->t[0], p->t[1], p->t[2]};
  v3 rt = rot_apply(q.R, t);
  q.t[0] = -rt.x;
  q.t[1] = -rt.y;
  q.t[2] = -rt.z;
  return q;
}
/* proj/include/rf/pose.hpp:31 compose = (R R', R t' + t) */
static pose_t pose_compose(const pose_t* a, const pose_t* b) {
  pose_t q;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      q.R[r * 3 + c] = a->R[r * 3 + 0] * b->R[0 * 3 + c] + (a->R[r * 3 + 1] * b->R[1 * 3 + c] + a->R[r * 3 + 2] * b->R[2 * 3 + c]);
  v3 t = {b->t[0], b->t[1], b->t[2]};
  v3 rt = rot_apply(a->R, t);
  q.t[0] = rt.x + a->t[0];
  q.t[1] = rt.y + a->t[1];
  q.t[2] = rt.z + a->t[2];
  return q;
}
static pose_t pose_from12(const float* p) {
  pose_t q;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) q.R[r * 3 + c] = p[r * 4 + c];
    q.t[r] = p[r * 4 + 3];
  }
  return q;
}
static intr_t intr_from(const int* wh, const float* f4) {
  intr_t i = {wh[0], wh[1], f4[0], f4[1], f4[2], f4[3]};
  return i;
}
static params_t params_from(const float* p) {
  params_t s = {p[0], p[1], (int)p[2], p[3], p[4], p[5] != 0.f};
  return s;
}
/* proj/include/rf/camera.hpp:23-25 */
static v3 backproject(const intr_t* in, float u, float v, float z) {
  v3 o = {(u - in->cx) / in->fx * z, (v - in->cy) / in->fy * z, z};
  return o;
}
static float dot3(v3 a, v3 b) { return a.x * b.x + (a.y * b.y + a.z * b.z); }
static float sqnorm3(v3 a) { return a.x * a.x + (a.y * a.y + a.z * a.z); }
static v3 cross3(v3 a, v3 b) {
  v3 o = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
  return o;
}
/* std::min / std::max semantics: min(a,b) = (b < a) ? b : a */
static float smin(float a, float b) { return (b < a) ? b : a; }
static float smax(float a, float b) { return (a < b) ? b : a; }

/* proj/include/rf/voxel.hpp:16-21 */
static float sdf_to_logical(int16_t s) { return (float)s / (float)SDF_ONE; }
static int16_t sdf_from_logical(float f) {
  float c = f < -1.f ? -1.f : (1.f < f ? 1.f : f); /* std::clamp */
  return (int16_t)lroundf(c * (float)SDF_ONE);
}

/* ---------------------------------------------------------- hash map */
/* proj/include/rf/voxel_block_map.hpp:47-52 */
static uint32_t hash_index(i3 p, uint32_t mask) {
  return (((uint32_t)p.x * 73856093u) ^ ((uint32_t)p.y * 19349669u) ^ ((uint32_t)p.z * 83492791u)) & mask;
}
uint32_t rfo_hash_index(const int* pos3, uint32_t mask) {
  i3 p = {pos3[0], pos3[1], pos3[2]};
  return hash_index(p, mask);
}
static int allocated(const entry_t* e) { return e->ptr >= -1; }
static int same_pos(const entry_t* e, i3 p) { return e->x == p.x && e->y == p.y && e->z == p.z; }

/* proj/src/voxel_block_map.cpp:26-34 */
static int find_entry(const rfo_map* m, i3 p) {
  int idx = (int)hash_index(p, m->buckets - 1);
  for (;;) {
    const entry_t* e = &m->entries[idx];
    if (allocated(e) && same_pos(e, p)) return idx;
    if (e->offset < 1) return -1;
    idx = (int)m->buckets + e->offset - 1;
  }
}
/* proj/src/voxel_block_map.cpp:36-61 (the BlockCache never changes results,
 * proj/tests/unit/test_voxelmap.cpp:183-198, so it is omitted) */
static const voxel_t* find_voxel(const rfo_map* m, i3 v) {
  i3 b = {v.x >> 3, v.y >> 3, v.z >> 3};
  int idx = find_entry(m, b);
  int ptr = idx >= 0 ? m->entries[idx].ptr : -1;
  if (ptr < 0) return NULL;
  int lin = (v.x - b.x * BS) + (v.y - b.y * BS) * BS + (v.z - b.z * BS) * BS * BS;
  return &m->vba[(size_t)ptr * BS3 + lin];
}
/* proj/src/voxel_block_map.cpp:74-105; returns entry idx or -1 */
static int allocate_block(rfo_map* m, i3 p) {
  int idx = (int)hash_index(p, m->buckets - 1);
  if (allocated(&m->entries[idx])) {
    for (;;) {
      entry_t* e = &m->entries[idx];
      if (same_pos(e, p) && allocated(e)) return idx;
      if (e->offset < 1) break;
      idx = (int)m->buckets + e->offset - 1;
    }
    if (m->nFreeExcess == 0 || m->nFreeBlocks == 0) return -1;
    int excessIdx = m->freeExcess[--m->nFreeExcess];
    int blockPtr = m->freeBlocks[--m->nFreeBlocks];
    int newIdx = (int)m->buckets + excessIdx;
    entry_t ne = {p.x, p.y, p.z, 0, blockPtr};
    m->entries[newIdx] = ne;
    m->entries[idx].offset = excessIdx + 1;
    return newIdx;
  }
  if (m->nFreeBlocks == 0) return -1;
  int blockPtr = m->freeBlocks[--m->nFreeBlocks];
  int keep = m->entries[idx].offset;
  entry_t ne = {p.x, p.y, p.z, keep, blockPtr};
  m->entries[idx] = ne;
  return idx;
}

rfo_map* rfo_create(uint32_t buckets, uint32_t excess, uint32_t capacity) {
  if (buckets == 0 || (buckets & (buckets - 1)) != 0) return NULL; /* voxel_block_map.cpp:10-11 */
  rfo_map* m = (rfo_map*)calloc(1, sizeof(rfo_map));
  m->buckets = buckets;
  m->excess = excess;
  m->capacity = capacity;
  size_t total = (size_t)buckets + excess;
  m->entries = (entry_t*)malloc(sizeof(entry_t) * total);
  m->vba = (voxel_t*)malloc(sizeof(voxel_t) * (size_t)capacity * BS3);
  m->freeBlocks = (int*)malloc(sizeof(int) * (capacity ? capacity : 1));
  m->freeExcess = (int*)malloc(sizeof(int) * (excess ? excess : 1));
  m->visible = (int*)malloc(sizeof(int) * total);
  m->visibility = (uint8_t*)malloc(total);
  m->allocType = (uint8_t*)malloc(total);
  m->blockCoords = (i3*)malloc(sizeof(i3) * total);
  m->marked = (uint8_t*)malloc(total);
  m->world = 1;
  rfo_clear(m);
  return m;
}

void rfo_destroy(rfo_map* m) {
  if (!m) return;
  free(m->entries);
  free(m->vba);
  free(m->freeBlocks);
  free(m->freeExcess);
  free(m->visible);
  free(m->visibility);
  free(m->allocType);
  free(m->blockCoords);
  free(m->marked);
  free(m->range);
  free(m);
}

/* proj/src/voxel_block_map.cpp:15-24 */
void rfo_clear(rfo_map* m) {
  size_t total = (size_t)m->buckets + m->excess;
  entry_t e0 = {0, 0, 0, 0, -2};
  for (size_t i = 0; i < total; ++i) m->entries[i] = e0;
  voxel_t v0;
  memset(&v0, 0, sizeof v0);
  v0.sdf = SDF_ONE;
  for (size_t i = 0; i < (size_t)m->capacity * BS3; ++i) m->vba[i] = v0;
  for (uint32_t i = 0; i < m->capacity; ++i) m->freeBlocks[i] = (int)i;
  m->nFreeBlocks = (int)m->capacity;
  for (uint32_t i = 0; i < m->excess; ++i) m->freeExcess[i] = (int)i;
  m->nFreeExcess = (int)m->excess;
  m->nVisible = 0;
  memset(m->visibility, 0, total);
  memset(m->allocType, 0, total);
  memset(m->marked, 0, total);
}

void rfo_set_shard(rfo_map* m, int rank, int world, int tileShift) {
  m->rank = rank;
  m->world = world;
  m->tileShift = tileShift;
}

static int owner_of(i3 b, int world, int shift) {
  i3 t = {b.x >> shift, b.y >> shift, b.z >> shift};
  return (int)(hash_index(t, 0xFFFFFFFFu) % (uint32_t)world);
}
static int shard_keeps(const rfo_map* m, i3 b) {
  if (m->world <= 1) return 1;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        i3 n = {b.x + dx, b.y + dy, b.z + dz};
        if (owner_of(n, m->world, m->tileShift) == m->rank) return 1;
      }
  return 0;
}

/* ------------------------------------------------------------- fusion */
/* proj/src/fusion.cpp:72-114 — Amanatides-Woo DDA in block units */
typedef void (*visit_fn)(void* ctx, i3 cell);
static void traverse_blocks(v3 a, v3 b, visit_fn visit, void* ctx) {
  i3 cell = {(int)floorf(a.x), (int)floorf(a.y), (int)floorf(a.z)};
  i3 endCell = {(int)floorf(b.x), (int)floorf(b.y), (int)floorf(b.z)};
  visit(ctx, cell);
  if (cell.x == endCell.x && cell.y == endCell.y && cell.z == endCell.z) return;
  float d[3] = {b.x - a.x, b.y - a.y, b.z - a.z};
  float av[3] = {a.x, a.y, a.z};
  int c[3] = {cell.x, cell.y, cell.z};
  int e[3] = {endCell.x, endCell.y, endCell.z};
  int step[3];
  float tMax[3], tDelta[3];
  for (int k = 0; k < 3; ++k) {
    if (d[k] > 0.f) {
      step[k] = 1;
      tMax[k] = ((float)(c[k] + 1) - av[k]) / d[k];
      tDelta[k] = 1.f / d[k];
    } else if (d[k] < 0.f) {
      step[k] = -1;
      tMax[k] = ((float)c[k] - av[k]) / d[k];
      tDelta[k] = -1.f / d[k];
    } else {
      step[k] = 0;
      tMax[k] = FLT_MAX;
      tDelta[k] = FLT_MAX;
    }
  }
  int maxSteps = abs(e[0] - c[0]) + abs(e[1] - c[1]) + abs(e[2] - c[2]) + 8;
  for (int i = 0; i < maxSteps; ++i) {
    int axis = 0;
    if (tMax[1] < tMax[0]) axis = 1;
    if (tMax[2] < tMax[axis]) axis = 2;
    if (tMax[axis] > 1.f) break;
    c[axis] += step[axis];
    tMax[axis] += tDelta[axis];
    i3 cc = {c[0], c[1], c[2]};
    visit(ctx, cc);
    if (c[0] == e[0] && c[1] == e[1] && c[2] == e[2]) break;
  }
  if (!(c[0] == e[0] && c[1] == e[1] && c[2] == e[2])) visit(ctx, endCell);
}

typedef struct {
  int* out;
  int n, max;
} collect_ctx;
static void collect_visit(void* ctx, i3 c) {
  collect_ctx* cc = (collect_ctx*)ctx;
  if (cc->n < cc->max) {
    cc->out[3 * cc->n] = c.x;
    cc->out[3 * cc->n + 1] = c.y;
    cc->out[3 * cc->n + 2] = c.z;
  }
  cc->n++;
}
int rfo_traverse_blocks(const float* a3, const float* b3, int* cellsOut, int maxCells) {
  v3 a = {a3[0], a3[1], a3[2]}, b = {b3[0], b3[1], b3[2]};
  collect_ctx cc = {cellsOut, 0, maxCells};
  traverse_blocks(a, b, collect_visit, &cc);
  return cc.n;
}

/* proj/src/fusion.cpp:116-130 */
static int block_in_frustum(i3 p, const pose_t* pose, const intr_t* in, const params_t* s, float marginPx) {
  const float bs = s->voxelSize * (float)BS;
  for (int c = 0; c < 8; ++c) {
    v3 corner = {((float)p.x + (float)(c & 1)) * bs, ((float)p.y + (float)((c >> 1) & 1)) * bs,
                 ((float)p.z + (float)((c >> 2) & 1)) * bs};
    v3 pc = pose_apply(pose, corner);
    if (pc.z < s->vfMin || pc.z > s->vfMax) continue;
    float px = in->fx * pc.x / pc.z + in->cx;
    float py = in->fy * pc.y / pc.z + in->cy;
    if (px >= -marginPx && py >= -marginPx && px <= (float)(in->w - 1) + marginPx &&
        py <= (float)(in->h - 1) + marginPx)
      return 1;
  }
  return 0;
}
int rfo_block_in_frustum(const int* pos3, const float* pose12, const int* wh, const float* f4, const float* params6) {
  i3 p = {pos3[0], pos3[1], pos3[2]};
  pose_t pose = pose_from12(pose12);
  intr_t in = intr_from(wh, f4);
  params_t s = params_from(params6);
  return block_in_frustum(p, &pose, &in, &s, 0.f);
}

/* proj/src/fusion.cpp:9-36 */
static float update_voxel_depth(voxel_t* vx, v3 pt, const pose_t* M, const intr_t* in, float mu, int maxW,
                                const float* depth, int dw, int dh, int stopAtMaxW) {
  v3 pc = pose_apply(M, pt);
  if (pc.z <= 0.f) return -1.f;
  float px = in->fx * pc.x / pc.z + in->cx;
  float py = in->fy * pc.y / pc.z + in->cy;
  if (px < 1 || px > (float)(dw - 2) || py < 1 || py > (float)(dh - 2)) return -1.f;
  float dm = depth[(size_t)(int)(py + 0.5f) * dw + (int)(px + 0.5f)];
  if (dm <= 0.f) return -1.f;
  float eta = dm - pc.z;
  if (eta < -mu) return eta;
  float oldF = sdf_to_logical(vx->sdf);
  int oldW = vx->w;
  if (stopAtMaxW && oldW >= maxW) return eta;
  float newF = smin(1.f, eta / mu);
  int newW = 1;
  float merged = ((float)oldW * oldF + (float)newW * newF) / (float)(oldW + newW);
  newW = (oldW + newW) < maxW ? (oldW + newW) : maxW;
  vx->sdf = sdf_from_logical(merged);
  vx->w = (uint8_t)newW;
  return eta;
}
float rfo_update_voxel_depth(uint8_t* voxel8, const float* pt3, const float* pose12, const int* wh, const float* f4,
                             float mu, int maxW, const float* depth, int stopAtMaxW) {
  voxel_t v;
  memcpy(&v, voxel8, 8);
  v3 pt = {pt3[0], pt3[1], pt3[2]};
  pose_t pose = pose_from12(pose12);
  intr_t in = intr_from(wh, f4);
  float eta = update_voxel_depth(&v, pt, &pose, &in, mu, maxW, depth, wh[0], wh[1], stopAtMaxW);
  memcpy(voxel8, &v, 8);
  return eta;
}

/* proj/src/fusion.cpp:38-70 */
static void update_voxel_colour(voxel_t* vx, v3 pt, const pose_t* M, const intr_t* in, int maxW, const uint8_t* rgb,
                                int rw, int rh) {
  v3 pc = pose_apply(M, pt);
  if (pc.z <= 0.f) return;
  float px = in->fx * pc.x / pc.z + in->cx;
  float py = in->fy * pc.y / pc.z + in->cy;
  if (px < 1 || px > (float)(rw - 2) || py < 1 || py > (float)(rh - 2)) return;
  int x0 = (int)floorf(px), y0 = (int)floorf(py);
  float fx = px - (float)x0, fy = py - (float)y0;
  float w00 = (1.f - fx) * (1.f - fy), w10 = fx * (1.f - fy), w01 = (1.f - fx) * fy, w11 = fx * fy;
  const uint8_t* c00 = rgb + 3 * ((size_t)y0 * rw + x0);
  const uint8_t* c10 = rgb + 3 * ((size_t)y0 * rw + x0 + 1);
  const uint8_t* c01 = rgb + 3 * ((size_t)(y0 + 1) * rw + x0);
  const uint8_t* c11 = rgb + 3 * ((size_t)(y0 + 1) * rw + x0 + 1);
  int oldW = vx->wc;
  for (int k = 0; k < 3; ++k) {
    float sample = w00 * (float)c00[k] + w10 * (float)c10[k] + w01 * (float)c01[k] + w11 * (float)c11[k];
    float merged = ((float)oldW * (float)vx->clr[k] + sample) / (float)(oldW + 1);
    long r = lroundf(merged);
    vx->clr[k] = (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
  }
  vx->wc = (uint8_t)((oldW + 1) < maxW ? (oldW + 1) : maxW);
}

typedef struct {
  rfo_map* m;
} mark_ctx;
/* proj/src/fusion.cpp:155-177 (markBlock) */
static void mark_visit(void* ctx, i3 p) {
  rfo_map* m = ((mark_ctx*)ctx)->m;
  if (!shard_keeps(m, p)) return;
  int idx = (int)hash_index(p, m->buckets - 1);
  const entry_t* e = &m->entries[idx];
  if (allocated(e)) {
    for (;;) {
      if (same_pos(e, p)) {
        m->marked[idx] = e->ptr >= 0 ? 1 : 2;
        return;
      }
      if (e->offset < 1) break;
      idx = (int)m->buckets + e->offset - 1;
      e = &m->entries[idx];
    }
    m->allocType[idx] = 2;
    m->blockCoords[idx] = p;
  } else {
    m->allocType[idx] = 1;
    m->blockCoords[idx] = p;
  }
}

/* proj/src/fusion.cpp:144-235 */
int rfo_allocate(rfo_map* m, const float* depth, const int* wh, const float* f4, const float* pose12,
                 const float* params6, int* stats4) {
  const size_t total = (size_t)m->buckets + m->excess;
  memset(m->allocType, 0, total); /* ensureScratch :132-142 */
  memset(m->marked, 0, total);
  intr_t in = intr_from(wh, f4);
  params_t s = params_from(params6);
  pose_t pose = pose_from12(pose12);
  pose_t camToWorld = pose_inverse(&pose);
  const float invBlock = 1.f / (s.voxelSize * (float)BS);
  int requested = 0, allocatedN = 0, failures = 0;

  /* stage 1 :179-187 */
  mark_ctx ctx = {m};
  for (int y = 0; y < in.h; ++y)
    for (int x = 0; x < in.w; ++x) {
      float d = depth[(size_t)y * in.w + x];
      if (d <= 0.f || d < s.vfMin || d > s.vfMax) continue;
      v3 nearP = pose_apply(&camToWorld, backproject(&in, (float)x, (float)y, d - s.mu));
      v3 farP = pose_apply(&camToWorld, backproject(&in, (float)x, (float)y, d + s.mu));
      v3 a = {nearP.x * invBlock, nearP.y * invBlock, nearP.z * invBlock};
      v3 b = {farP.x * invBlock, farP.y * invBlock, farP.z * invBlock};
      traverse_blocks(a, b, mark_visit, &ctx);
    }

  /* stage 2 :190-201 */
  for (size_t idx = 0; idx < total; ++idx) {
    if (m->allocType[idx] == 0) continue;
    ++requested;
    int e = allocate_block(m, m->blockCoords[idx]);
    if (e < 0) {
      ++failures;
      continue;
    }
    ++allocatedN;
    m->marked[e] = 1;
  }

  /* stage 3 :205-233 — candidates = marked ∪ previous visible, frustum
   * tested, sorted by idx.  Candidate indices are unique, so an ascending scan
   * of the candidate flags yields the same sorted list. */
  for (int i = 0; i < m->nVisible; ++i)
    if (!m->marked[m->visible[i]]) m->marked[m->visible[i]] = 3; /* prev-visible candidate */
  memset(m->visibility, 0, total);
  int nv = 0;
  for (size_t idx = 0; idx < total; ++idx) {
    if (!m->marked[idx]) continue;
    const entry_t* e = &m->entries[idx];
    if (!allocated(e)) continue;
    i3 p = {e->x, e->y, e->z};
    uint8_t type = 0;
    if (block_in_frustum(p, &pose, &in, &s, 0.f))
      type = e->ptr >= 0 ? 1 : 2;
    else if (m->swapping && block_in_frustum(p, &pose, &in, &s, m->swapMargin))
      type = 3; /* kBoundary, fusion.cpp:223-224 */
    if (type) {
      m->visibility[idx] = type;
      m->visible[nv++] = (int)idx;
    }
  }
  m->nVisible = nv;
  stats4[0] = requested;
  stats4[1] = allocatedN;
  stats4[2] = failures;
  stats4[3] = nv;
  return 0;
}

/* proj/src/fusion.cpp:237-263 */
int rfo_integrate(rfo_map* m, const float* depth, const uint8_t* rgb, const int* whD, const float* f4D,
                  const int* whRgb, const float* f4Rgb, const float* extr12, const float* pose12,
                  const float* params6) {
  intr_t inD = intr_from(whD, f4D);
  intr_t inRgb = whRgb ? intr_from(whRgb, f4Rgb) : inD;
  params_t s = params_from(params6);
  pose_t pose = pose_from12(pose12);
  pose_t extr;
  if (extr12) {
    extr = pose_from12(extr12);
  } else {
    memset(&extr, 0, sizeof extr);
    extr.R[0] = extr.R[4] = extr.R[8] = 1.f;
  }
  pose_t Mrgb = pose_compose(&extr, &pose);
  for (int i = 0; i < m->nVisible; ++i) {
    const entry_t* e = &m->entries[m->visible[i]];
    if (e->ptr < 0) continue;
    voxel_t* blk = &m->vba[(size_t)e->ptr * BS3];
    int ox = e->x * BS, oy = e->y * BS, oz = e->z * BS;
    for (int z = 0; z < BS; ++z)
      for (int y = 0; y < BS; ++y)
        for (int x = 0; x < BS; ++x) {
          voxel_t* v = &blk[x + y * BS + z * BS * BS];
          v3 pt = {(float)(ox + x) * s.voxelSize, (float)(oy + y) * s.voxelSize, (float)(oz + z) * s.voxelSize};
          float eta = update_voxel_depth(v, pt, &pose, &inD, s.mu, s.maxW, depth, inD.w, inD.h, s.stopAtMaxW);
          if (rgb && eta >= -s.mu) update_voxel_colour(v, pt, &Mrgb, &inRgb, s.maxW, rgb, inRgb.w, inRgb.h);
        }
  }
  return 0;
}

/* ------------------------------------------------------------ raycast */
static void ensure_range(rfo_map* m, int w, int h) {
  if (m->rangeW != w || m->rangeH != h) {
    free(m->range);
    m->range = (float*)malloc(sizeof(float) * 2 * (size_t)w * h);
    m->rangeW = w;
    m->rangeH = h;
  }
}

/* proj/src/raycast.cpp:38-71 (projectBlock), :86-127 (render_expected_ranges).
 * The 16x16 fragment split of each block's pixel rectangle only partitions
 * the min/max merge (commutative), so merging the rectangle directly yields
 * identical ranges. */
int rfo_render_ranges(rfo_map* m, const float* pose12, const int* wh, const float* f4, const float* params6,
                      float* rangeOut) {
  intr_t in = intr_from(wh, f4);
  params_t s = params_from(params6);
  pose_t pose = pose_from12(pose12);
  ensure_range(m, in.w, in.h);
  for (size_t i = 0; i < (size_t)in.w * in.h; ++i) {
    m->range[2 * i] = FLT_MAX;
    m->range[2 * i + 1] = -1.f;
  }
  const float bs = s.voxelSize * (float)BS;
  for (int vi = 0; vi < m->nVisible; ++vi) {
    const entry_t* e = &m->entries[m->visible[vi]];
    if (!allocated(e)) continue;
    float x0 = FLT_MAX, y0 = FLT_MAX, x1 = -FLT_MAX, y1 = -FLT_MAX, zMin = FLT_MAX, zMax = 0.f;
    int valid = 0;
    for (int c = 0; c < 8; ++c) {
      v3 corner = {((float)e->x + (float)(c & 1)) * bs, ((float)e->y + (float)((c >> 1) & 1)) * bs,
                   ((float)e->z + (float)((c >> 2) & 1)) * bs};
      v3 pc = pose_apply(&pose, corner);
      if (pc.z < 1e-6f) continue;
      float px = in.fx * pc.x / pc.z + in.cx;
      float py = in.fy * pc.y / pc.z + in.cy;
      x0 = smin(x0, px);
      y0 = smin(y0, py);
      x1 = smax(x1, px);
      y1 = smax(y1, py);
      zMin = smin(zMin, pc.z);
      zMax = smax(zMax, pc.z);
      ++valid;
    }
    if (valid == 0) continue;
    int bx0 = (int)floorf(x0), by0 = (int)floorf(y0), bx1 = (int)ceilf(x1), by1 = (int)ceilf(y1);
    bx0 = bx0 > 0 ? bx0 : 0;
    by0 = by0 > 0 ? by0 : 0;
    bx1 = bx1 < in.w - 1 ? bx1 : in.w - 1;
    by1 = by1 < in.h - 1 ? by1 : in.h - 1;
    if (bx0 > bx1 || by0 > by1) continue;
    float zlo = smax(zMin, s.vfMin), zhi = smin(zMax, s.vfMax);
    if (zlo > zhi) continue;
    for (int y = by0; y <= by1; ++y)
      for (int x = bx0; x <= bx1; ++x) {
        float* r = &m->range[2 * ((size_t)y * in.w + x)];
        r[0] = smin(r[0], zlo);
        r[1] = smax(r[1], zhi);
      }
  }
  if (rangeOut) memcpy(rangeOut, m->range, sizeof(float) * 2 * (size_t)in.w * in.h);
  return 0;
}

int rfo_set_ranges(rfo_map* m, const int* wh, const float* rangeIn) {
  ensure_range(m, wh[0], wh[1]);
  memcpy(m->range, rangeIn, sizeof(float) * 2 * (size_t)wh[0] * wh[1]);
  return 0;
}

/* MapField (proj/include/rf/raycast.hpp:32-45) */
static int field_resident(const rfo_map* m, v3 p) {
  i3 b = {((int)floorf(p.x)) >> 3, ((int)floorf(p.y)) >> 3, ((int)floorf(p.z)) >> 3};
  int idx = find_entry(m, b);
  return idx >= 0 && m->entries[idx].ptr >= 0; /* blockResident voxel_block_map.cpp:63-72 */
}
/* readSdfNearest voxel_block_map.cpp:178-185 */
static float sdf_nearest(const rfo_map* m, v3 p, int* ok) {
  i3 v = {(int)lroundf(p.x), (int)lroundf(p.y), (int)lroundf(p.z)};
  const voxel_t* vx = find_voxel(m, v);
  *ok = vx != NULL;
  return vx ? sdf_to_logical(vx->sdf) : 1.f;
}
/* readSdfWeightTrilinear voxel_block_map.cpp:130-156 */
static float sdf_trilinear(const rfo_map* m, v3 p, int* ok) {
  int bx = (int)floorf(p.x), by = (int)floorf(p.y), bz = (int)floorf(p.z);
  float fx = p.x - (float)bx, fy = p.y - (float)by, fz = p.z - (float)bz;
  float sdf = 0.f;
  for (int k = 0; k < 8; ++k) {
    i3 c = {bx + (k & 1), by + ((k >> 1) & 1), bz + ((k >> 2) & 1)};
    const voxel_t* vx = find_voxel(m, c);
    if (!vx) {
      *ok = 0;
      return 1.f;
    }
    float bw = ((k & 1) ? fx : 1.f - fx) * (((k >> 1) & 1) ? fy : 1.f - fy) * (((k >> 2) & 1) ? fz : 1.f - fz);
    sdf += bw * sdf_to_logical(vx->sdf);
  }
  *ok = 1;
  return sdf;
}

static v3 at_t(v3 o, v3 d, float t) {
  v3 r = {o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
  return r;
}

/* cast_ray_field proj/include/rf/raycast.hpp:54-112; returns 1 on hit */
static int cast_ray(const rfo_map* m, v3 originM, v3 dirUnit, float tMinM, float tMaxM, float mu, float vs,
                    v3* hit) {
  const float coarseStep = (float)BS * vs;
  const float fineStep = mu;
  const float stepScale = mu;
  v3 oV = {originM.x / vs, originM.y / vs, originM.z / vs};
  v3 dV = {dirUnit.x / vs, dirUnit.y / vs, dirUnit.z / vs};
  float t = tMinM;
  enum { COARSE, FINE, SURFACE } state = field_resident(m, at_t(oV, dV, t)) ? FINE : COARSE;
  while (t <= tMaxM) {
    v3 p = at_t(oV, dV, t);
    if (state == COARSE) {
      if (field_resident(m, p)) {
        state = FINE;
        t = smax(tMinM, t - coarseStep);
      } else {
        t += coarseStep;
      }
      continue;
    }
    int ok = 0;
    float sdf = sdf_nearest(m, p, &ok);
    if (!ok) {
      if (state == SURFACE) state = FINE;
      t += fineStep;
      continue;
    }
    if (sdf <= 0.1f) {
      int okTri = 0;
      float tri = sdf_trilinear(m, p, &okTri);
      if (okTri) sdf = tri;
    }
    if (state == FINE) {
      if (sdf < 0.f) return 0; /* WRONG_SIDE */
      state = SURFACE;
    }
    if (sdf <= 0.f) {
      float tHit = t + sdf * stepScale;
      int okR = 0;
      float f1 = sdf_trilinear(m, at_t(oV, dV, tHit), &okR);
      if (okR) tHit += f1 * stepScale;
      *hit = at_t(oV, dV, tHit);
      return 1;
    }
    t += smax(sdf * stepScale, vs);
  }
  return 0;
}

/* field_normal proj/include/rf/raycast.hpp:137-153 */
static int field_normal(const rfo_map* m, v3 h, v3* n) {
  int ok[6];
  v3 px = {h.x + 1.f, h.y + 0.f, h.z + 0.f}, mx = {h.x - 1.f, h.y - 0.f, h.z - 0.f};
  v3 py = {h.x + 0.f, h.y + 1.f, h.z + 0.f}, my = {h.x - 0.f, h.y - 1.f, h.z - 0.f};
  v3 pz = {h.x + 0.f, h.y + 0.f, h.z + 1.f}, mz = {h.x - 0.f, h.y - 0.f, h.z - 1.f};
  v3 g;
  g.x = sdf_trilinear(m, px, &ok[0]) - sdf_trilinear(m, mx, &ok[1]);
  g.y = sdf_trilinear(m, py, &ok[2]) - sdf_trilinear(m, my, &ok[3]);
  g.z = sdf_trilinear(m, pz, &ok[4]) - sdf_trilinear(m, mz, &ok[5]);
  if (!(ok[0] && ok[1] && ok[2] && ok[3] && ok[4] && ok[5])) return 0;
  float len = sqrtf(sqnorm3(g));
  if (len < 1e-12f) return 0;
  n->x = g.x / len;
  n->y = g.y / len;
  n->z = g.z / len;
  return 1;
}

/* One pixel of render_maps_field (proj/include/rf/raycast.hpp:157-207, mode
 * kIcpMaps): the doPixel lambda. */
typedef struct {
  const rfo_map* m;
  intr_t in;
  params_t s;
  pose_t c2w;
  v3 origin;
  const int* list; /* NULL: every pixel, row-major; else (x, y) pairs */
  float *raycast, *points, *normals;
} icp_job_t;

static void icp_pixel(const icp_job_t* j, int x, int y) {
  const rfo_map* m = j->m;
  const intr_t in = j->in;
  size_t i = (size_t)y * in.w + x;
  float* rc = j->raycast + 4 * i;
  float* pt = j->points + 4 * i;
  float* nm = j->normals + 4 * i;
  rc[0] = rc[1] = rc[2] = 0.f;
  rc[3] = -1.f;
  pt[0] = pt[1] = pt[2] = 0.f;
  pt[3] = -1.f;
  nm[0] = nm[1] = nm[2] = 0.f;
  nm[3] = -1.f;
  float r0 = m->range[2 * i], r1 = m->range[2 * i + 1];
  if (!(r1 >= r0)) return;
  v3 dirCam = {((float)x - in.cx) / in.fx, ((float)y - in.cy) / in.fy, 1.f};
  float norm = sqrtf(sqnorm3(dirCam));
  v3 dw = rot_apply(j->c2w.R, dirCam);
  v3 dirW = {dw.x / norm, dw.y / norm, dw.z / norm};
  v3 hit;
  if (!cast_ray(m, j->origin, dirW, r0 * norm, r1 * norm, j->s.mu, j->s.voxelSize, &hit)) return;
  rc[0] = hit.x;
  rc[1] = hit.y;
  rc[2] = hit.z;
  rc[3] = 1.f;
  pt[0] = hit.x * j->s.voxelSize;
  pt[1] = hit.y * j->s.voxelSize;
  pt[2] = hit.z * j->s.voxelSize;
  pt[3] = 1.f;
  v3 n;
  if (field_normal(m, hit, &n)) {
    nm[0] = n.x;
    nm[1] = n.y;
    nm[2] = n.z;
    nm[3] = 1.f;
  }
}

/* The pixels are split into chunks handed out by an atomic counter to
 * g_threads workers (each pixel is independent and reads the map only). */
typedef struct {
  const icp_job_t* job;
  int n, chunk;
  int next; /* atomic */
} icp_pool_t;

static void icp_run_item(const icp_job_t* j, int k) {
  if (j->list)
    icp_pixel(j, j->list[2 * k], j->list[2 * k + 1]);
  else
    icp_pixel(j, k % j->in.w, k / j->in.w);
}

static void* icp_worker(void* arg) {
  icp_pool_t* p = (icp_pool_t*)arg;
  for (;;) {
    const int k0 = __atomic_fetch_add(&p->next, p->chunk, __ATOMIC_RELAXED);
    if (k0 >= p->n) break;
    const int k1 = k0 + p->chunk < p->n ? k0 + p->chunk : p->n;
    for (int k = k0; k < k1; ++k) icp_run_item(p->job, k);
  }
  return NULL;
}

static void icp_run(const icp_job_t* j, int n) {
  if (g_threads <= 1) {
    for (int k = 0; k < n; ++k) icp_run_item(j, k);
    return;
  }
  icp_pool_t pool = {j, n, 256, 0};
  pthread_t th[256];
  const int nt = g_threads < 256 ? g_threads : 256;
  int started = 0;
  for (int t = 1; t < nt; ++t)
    if (pthread_create(&th[started], NULL, icp_worker, &pool) == 0) ++started;
  icp_worker(&pool);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* render_maps_field proj/include/rf/raycast.hpp:157-207, mode kIcpMaps */
int rfo_render_icp(rfo_map* m, const float* pose12, const int* wh, const float* f4, const float* params6,
                   float* raycastOut, float* pointsOut, float* normalsOut) {
  icp_job_t j;
  j.m = m;
  j.in = intr_from(wh, f4);
  j.s = params_from(params6);
  pose_t pose = pose_from12(pose12);
  j.c2w = pose_inverse(&pose);
  j.origin = (v3){j.c2w.t[0], j.c2w.t[1], j.c2w.t[2]};
  j.list = NULL;
  j.raycast = raycastOut;
  j.points = pointsOut;
  j.normals = normalsOut;
  if (m->rangeW != j.in.w || m->rangeH != j.in.h) return -1;
  icp_run(&j, j.in.w * j.in.h);
  return 0;
}

/* render_maps(kIcpMaps, missingOnly) (raycast.hpp:200-202): doPixel for the
 * listed (x, y) pixels only; the other pixels of the in/out images keep their
 * values. */
int rfo_render_icp_list(rfo_map* m, const float* pose12, const int* wh, const float* f4, const float* params6,
                        const int* missingXY, int n, float* raycastOut, float* pointsOut, float* normalsOut) {
  icp_job_t j;
  j.m = m;
  j.in = intr_from(wh, f4);
  j.s = params_from(params6);
  pose_t pose = pose_from12(pose12);
  j.c2w = pose_inverse(&pose);
  j.origin = (v3){j.c2w.t[0], j.c2w.t[1], j.c2w.t[2]};
  j.list = missingXY;
  j.raycast = raycastOut;
  j.points = pointsOut;
  j.normals = normalsOut;
  if (m->rangeW != j.in.w || m->rangeH != j.in.h) return -1;
  icp_run(&j, n);
  return 0;
}

/* forward_project (proj/src/raycast.cpp:141-188).  hasRaycast = 0: every
 * pixel is missing.  Otherwise the previous raycastResult (in/out) is
 * re-projected into newPose keeping the nearest point per pixel (strictly
 * nearer replaces, so ties keep the first in row-major source order);
 * points are set for the forwarded pixels, normals stay invalid.  Returns the
 * number of missing pixels, written row-major as (x, y) pairs. */
int rfo_forward_project(int hasRaycast, float* raycast, float* points, float* normals, const float* newPose12,
                        const int* wh, const float* f4, float voxelSize, int* missingXY) {
  intr_t in = intr_from(wh, f4);
  const size_t n = (size_t)in.w * in.h;
  int nm = 0;
  if (!hasRaycast) {
    for (int y = 0; y < in.h; ++y)
      for (int x = 0; x < in.w; ++x) {
        missingXY[2 * nm] = x;
        missingXY[2 * nm + 1] = y;
        ++nm;
      }
    return nm;
  }
  pose_t pose = pose_from12(newPose12);
  float* prev = (float*)malloc(sizeof(float) * 4 * n);
  float* depthBuf = (float*)malloc(sizeof(float) * n);
  memcpy(prev, raycast, sizeof(float) * 4 * n);
  for (size_t i = 0; i < n; ++i) {
    depthBuf[i] = FLT_MAX;
    for (int k = 0; k < 3; ++k) raycast[4 * i + k] = points[4 * i + k] = normals[4 * i + k] = 0.f;
    raycast[4 * i + 3] = points[4 * i + 3] = normals[4 * i + 3] = -1.f;
  }
  for (size_t i = 0; i < n; ++i) {
    const float* r = prev + 4 * i;
    if (r[3] <= 0.f) continue;
    v3 world = {r[0] * voxelSize, r[1] * voxelSize, r[2] * voxelSize};
    v3 pc = pose_apply(&pose, world);
    if (pc.z <= 0.f) continue;
    float px = in.fx * pc.x / pc.z + in.cx;
    float py = in.fy * pc.y / pc.z + in.cy;
    int ix = (int)lroundf(px), iy = (int)lroundf(py);
    if (ix < 0 || iy < 0 || ix >= in.w || iy >= in.h) continue;
    size_t t = (size_t)iy * in.w + ix;
    if (pc.z >= depthBuf[t]) continue;
    depthBuf[t] = pc.z;
    memcpy(raycast + 4 * t, r, sizeof(float) * 4);
    points[4 * t] = world.x;
    points[4 * t + 1] = world.y;
    points[4 * t + 2] = world.z;
    points[4 * t + 3] = 1.f;
  }
  for (int y = 0; y < in.h; ++y)
    for (int x = 0; x < in.w; ++x)
      if (raycast[4 * ((size_t)y * in.w + x) + 3] <= 0.f) {
        missingXY[2 * nm] = x;
        missingXY[2 * nm + 1] = y;
        ++nm;
      }
  free(prev);
  free(depthBuf);
  return nm;
}

/* --------------------------------------------------------------- view */
/* proj/src/view.cpp:112-119 depth conversion, :69-88 downsample_depth */
int rfo_build_view(const uint16_t* raw, const int* wh, float affScale, float affOffset, int levels,
                   float* depthLevels) {
  if (levels < 1) return -1;
  int w = wh[0], h = wh[1];
  float* out = depthLevels;
  for (int i = 0; i < w * h; ++i) {
    out[i] = -1.f;
    if (raw[i] == 0) continue;
    float mtr = (float)raw[i] * affScale + affOffset;
    out[i] = mtr > 0.f ? mtr : -1.f;
  }
  const float* prev = out;
  int pw = w, ph = h;
  out += (size_t)w * h;
  for (int l = 1; l < levels; ++l) {
    int lw = pw / 2, lh = ph / 2;
    for (int y = 0; y < lh; ++y)
      for (int x = 0; x < lw; ++x) {
        float sum = 0.f;
        int n = 0;
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            float d = prev[(size_t)(2 * y + dy) * pw + 2 * x + dx];
            if (d > 0.f) {
              sum += d;
              ++n;
            }
          }
        out[(size_t)y * lw + x] = n > 0 ? sum / (float)n : -1.f;
      }
    prev = out;
    out += (size_t)lw * lh;
    pw = lw;
    ph = lh;
  }
  return 0;
}

/* ------------------------------------------------- colour / grey modes */
/* readColourTrilinear (voxel_block_map.cpp:158-175): missing corners are
 * skipped, clr += bw * (r, g, b) per component. */
static v3 colour_trilinear(const rfo_map* m, v3 p) {
  int bx = (int)floorf(p.x), by = (int)floorf(p.y), bz = (int)floorf(p.z);
  float fx = p.x - (float)bx, fy = p.y - (float)by, fz = p.z - (float)bz;
  v3 c = {0.f, 0.f, 0.f};
  for (int k = 0; k < 8; ++k) {
    i3 q = {bx + (k & 1), by + ((k >> 1) & 1), bz + ((k >> 2) & 1)};
    const voxel_t* vx = find_voxel(m, q);
    if (!vx) continue;
    float bw = ((k & 1) ? fx : 1.f - fx) * (((k >> 1) & 1) ? fy : 1.f - fy) * (((k >> 2) & 1) ? fz : 1.f - fz);
    c.x += bw * (float)vx->clr[0];
    c.y += bw * (float)vx->clr[1];
    c.z += bw * (float)vx->clr[2];
  }
  return c;
}
static uint8_t clamp_u8(float v) { return (uint8_t)(v < 0.f ? 0.f : (255.f < v ? 255.f : v)); }

/* render_maps_field's colour (raycast.hpp:169,191-197, raycast.cpp:132-137)
 * from the ICP maps of the same render: mode 1 = kColour (trilinear colour at
 * the hit, clamped and truncated), 2 = kGrey (|n . dirWorld| clamped to
 * [0, 1] * 255, only where the normal is valid); (0,0,0) elsewhere.  list /
 * nList restrict it to the listed pixels (missingOnly), like the maps. */
int rfo_render_colour(const rfo_map* m, int mode, const float* pose12, const int* wh, const float* f4,
                      const float* raycast, const float* normals, const int* list, int nList, uint8_t* rgbOut) {
  intr_t in = intr_from(wh, f4);
  pose_t pose = pose_from12(pose12);
  pose_t c2w = pose_inverse(&pose);
  const int n = list ? nList : in.w * in.h;
  for (int k = 0; k < n; ++k) {
    const int i = list ? list[k] : k;
    const int x = i % in.w, y = i / in.w;
    uint8_t* o = rgbOut + 3 * (size_t)i;
    o[0] = o[1] = o[2] = 0;
    const float* rc = raycast + 4 * (size_t)i;
    if (!(rc[3] > 0.f)) continue;
    if (mode == 1) {
      v3 h = {rc[0], rc[1], rc[2]};
      v3 c = colour_trilinear(m, h);
      o[0] = clamp_u8(c.x);
      o[1] = clamp_u8(c.y);
      o[2] = clamp_u8(c.z);
    } else if (mode == 2) {
      const float* nm = normals + 4 * (size_t)i;
      if (!(nm[3] > 0.f)) continue;
      v3 dirCam = {((float)x - in.cx) / in.fx, ((float)y - in.cy) / in.fy, 1.f};
      float norm = sqrtf(sqnorm3(dirCam));
      v3 dw = rot_apply(c2w.R, dirCam);
      v3 dirW = {dw.x / norm, dw.y / norm, dw.z / norm};
      float shade = fabsf(nm[0] * dirW.x + (nm[1] * dirW.y + nm[2] * dirW.z));
      shade = shade < 0.f ? 0.f : (1.f < shade ? 1.f : shade);
      const uint8_t g = (uint8_t)(shade * 255.f);
      o[0] = o[1] = o[2] = g;
    }
  }
  return 0;
}

/* ----------------------------------------------------------- swapping */
/* FusionEngine::Options (fusion.hpp:54-57) */
void rfo_set_fusion_options(rfo_map* m, int swappingEnabled, float swapMarginPx) {
  m->swapping = swappingEnabled;
  m->swapMargin = swapMarginPx;
}

/* VoxelBlockMap::reserveBlockForEntry (voxel_block_map.cpp:107-116): pop a
 * VBA block, reset it to Voxel{} and attach it. */
int rfo_reserve_block(rfo_map* m, int idx) {
  entry_t* e = &m->entries[idx];
  if (e->ptr >= 0) return 1;
  if (m->nFreeBlocks == 0) return 0;
  const int ptr = m->freeBlocks[--m->nFreeBlocks];
  voxel_t* b = &m->vba[(size_t)ptr * BS3];
  for (int i = 0; i < BS3; ++i) {
    memset(&b[i], 0, sizeof(voxel_t));
    b[i].sdf = 32767;
  }
  e->ptr = ptr;
  return 1;
}
/* VoxelBlockMap::releaseBlock (voxel_block_map.cpp:118-123): push the block
 * back (contents kept) and mark the entry swapped out. */
void rfo_release_block(rfo_map* m, int idx) {
  entry_t* e = &m->entries[idx];
  if (e->ptr < 0) return;
  m->freeBlocks[m->nFreeBlocks++] = e->ptr;
  e->ptr = -1;
}

/* The swapping engine (the reference has only the hooks
 * above, so this restatement is the oracle): a host voxel store indexed by
 * entry, transfer capacity C blocks per frame and direction.
 *   swap-in (after allocation, before integration): entries with visibility
 *     2 (visible, swapped out) that have host data, ascending index, at most
 *     C: reserve a block (reserveBlockForEntry order) and merge the host
 *     voxels into the fresh block (w = 0 device voxel -> host voxel;
 *     otherwise the running-average merge); stops when the VBA is exhausted
 *     (the rest stay queued).
 *   swap-out (after integration): per resident entry, age = 0 if it has a
 *     visibility type this frame, else age + 1 (saturating); entries with
 *     age >= 2, ascending index, at most C: copy the block to the host
 *     store, reset it to Voxel{} and release it. */
typedef struct {
  int capacity;
  voxel_t* host;  /* total entries x 512 */
  uint8_t* has;
  uint8_t* age;
} rfo_swap;

rfo_swap* rfo_swap_create(const rfo_map* m, int capacity) {
  const size_t total = (size_t)m->buckets + m->excess;
  rfo_swap* w = (rfo_swap*)calloc(1, sizeof(rfo_swap));
  w->capacity = capacity;
  w->host = (voxel_t*)calloc(total * BS3, sizeof(voxel_t));
  w->has = (uint8_t*)calloc(total, 1);
  w->age = (uint8_t*)calloc(total, 1);
  return w;
}
void rfo_swap_destroy(rfo_swap* w) {
  if (!w) return;
  free(w->host);
  free(w->has);
  free(w->age);
  free(w);
}

static void merge_voxel(voxel_t* d, const voxel_t* h, int maxW) {
  if (d->w == 0) {
    *d = *h;
    return;
  }
  if (h->w == 0) return;
  const float fd = sdf_to_logical(d->sdf), fh = sdf_to_logical(h->sdf);
  const float merged = ((float)d->w * fd + (float)h->w * fh) / (float)(d->w + h->w);
  const int w = d->w + h->w;
  d->sdf = sdf_from_logical(merged);
  d->w = (uint8_t)(w < maxW ? w : maxW);
}

int rfo_swap_in(rfo_map* m, rfo_swap* w, int maxW) {
  const size_t total = (size_t)m->buckets + m->excess;
  int n = 0;
  for (size_t idx = 0; idx < total && n < w->capacity; ++idx) {
    if (m->visibility[idx] != 2 || !w->has[idx]) continue;
    if (!rfo_reserve_block(m, (int)idx)) break; /* VBA exhausted: left queued */
    voxel_t* b = &m->vba[(size_t)m->entries[idx].ptr * BS3];
    for (int i = 0; i < BS3; ++i) merge_voxel(&b[i], &w->host[idx * BS3 + i], maxW);
    ++n;
  }
  return n;
}

int rfo_swap_out(rfo_map* m, rfo_swap* w) {
  const size_t total = (size_t)m->buckets + m->excess;
  int n = 0;
  for (size_t idx = 0; idx < total; ++idx) {
    const entry_t* e = &m->entries[idx];
    if (e->ptr < 0) continue;
    if (m->visibility[idx])
      w->age[idx] = 0;
    else if (w->age[idx] < 255)
      w->age[idx]++;
    if (w->age[idx] >= 2 && n < w->capacity) {
      voxel_t* b = &m->vba[(size_t)e->ptr * BS3];
      memcpy(&w->host[idx * BS3], b, sizeof(voxel_t) * BS3);
      w->has[idx] = 1;
      /* the released block comes back clean (allocateBlock does not clear
       * reused blocks; SPEC.md:444 equivalence) */
      for (int i = 0; i < BS3; ++i) {
        memset(&b[i], 0, sizeof(voxel_t));
        b[i].sdf = 32767;
      }
      rfo_release_block(m, (int)idx);
      ++n;
    }
  }
  return n;
}

/* host store export (tests): has flags and the stored block of an entry */
int rfo_swap_export(const rfo_swap* w, size_t total, uint8_t* hasOut, uint8_t* ageOut) {
  if (hasOut) memcpy(hasOut, w->has, total);
  if (ageOut) memcpy(ageOut, w->age, total);
  return 0;
}
int rfo_swap_host_block(const rfo_swap* w, int idx, uint8_t* out4096) {
  memcpy(out4096, &w->host[(size_t)idx * BS3], sizeof(voxel_t) * BS3);
  return 0;
}

/* ------------------------------------------------------ marching cubes */
/* The triangulation table by the reference's rule (meshing.cpp:27-118):
 * pair the crossed edges on each face (ambiguous faces: the two edges at
 * each inside corner), walk the cycles, orient each by its Newell normal
 * against the inside->outside direction, fan it. */
static const int MC_C[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
static const int MC_E[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
static const int MC_F[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};
static int mc_cnt[256];
static int mc_tri[256][16][3];
static int mc_ready = 0;

static int mc_edge(int a, int b) {
  for (int e = 0; e < 12; ++e)
    if ((MC_E[e][0] == a && MC_E[e][1] == b) || (MC_E[e][0] == b && MC_E[e][1] == a)) return e;
  return -1;
}
static void mc_link(int nb[12][2], int a, int b) {
  if (nb[a][0] < 0) nb[a][0] = b; else nb[a][1] = b;
  if (nb[b][0] < 0) nb[b][0] = a; else nb[b][1] = a;
}
static void mc_build_table(void) {
  if (mc_ready) return;
  for (int mask = 0; mask < 256; ++mask) {
    int nb[12][2];
    for (int e = 0; e < 12; ++e) nb[e][0] = nb[e][1] = -1;
    for (int f = 0; f < 6; ++f) {
      int ce[4], n = 0;
      for (int i = 0; i < 4; ++i) {
        int e = mc_edge(MC_F[f][i], MC_F[f][(i + 1) % 4]);
        if (((mask >> MC_E[e][0]) & 1) != ((mask >> MC_E[e][1]) & 1)) ce[n++] = e;
      }
      if (n == 2) {
        mc_link(nb, ce[0], ce[1]);
      } else if (n == 4) {
        for (int i = 0; i < 4; ++i) {
          int c = MC_F[f][i];
          if ((mask >> c) & 1) mc_link(nb, mc_edge(MC_F[f][(i + 3) % 4], c), mc_edge(c, MC_F[f][(i + 1) % 4]));
        }
      }
    }
    mc_cnt[mask] = 0;
    int used[12] = {0};
    for (int st = 0; st < 12; ++st) {
      int crossed = ((mask >> MC_E[st][0]) & 1) != ((mask >> MC_E[st][1]) & 1);
      if (!crossed || used[st]) continue;
      int cyc[12], len = 0, cur = st, prev = -1;
      for (;;) {
        cyc[len++] = cur;
        used[cur] = 1;
        int nxt = nb[cur][0] != prev ? nb[cur][0] : nb[cur][1];
        prev = cur;
        cur = nxt;
        if (cur == st) break;
      }
      if (len < 3) continue;
      float nw[3] = {0, 0, 0}, rf[3] = {0, 0, 0};
      for (int i = 0; i < len; ++i) {
        float a[3], b[3];
        int ea = cyc[i], eb = cyc[(i + 1) % len];
        for (int k = 0; k < 3; ++k) {
          a[k] = 0.5f * (float)(MC_C[MC_E[ea][0]][k] + MC_C[MC_E[ea][1]][k]);
          b[k] = 0.5f * (float)(MC_C[MC_E[eb][0]][k] + MC_C[MC_E[eb][1]][k]);
        }
        nw[0] += a[1] * b[2] - a[2] * b[1];
        nw[1] += a[2] * b[0] - a[0] * b[2];
        nw[2] += a[0] * b[1] - a[1] * b[0];
        int c0 = MC_E[ea][0], c1 = MC_E[ea][1];
        int in = ((mask >> c0) & 1) ? c0 : c1, out = ((mask >> c0) & 1) ? c1 : c0;
        for (int k = 0; k < 3; ++k) rf[k] += (float)(MC_C[out][k] - MC_C[in][k]);
      }
      if (rf[0] * rf[0] + rf[1] * rf[1] + rf[2] * rf[2] > 1e-12f && nw[0] * rf[0] + nw[1] * rf[1] + nw[2] * rf[2] < 0.f)
        for (int i = 0; i < len / 2; ++i) {
          int t = cyc[i];
          cyc[i] = cyc[len - 1 - i];
          cyc[len - 1 - i] = t;
        }
      for (int i = 1; i + 1 < len; ++i) {
        int k = mc_cnt[mask]++;
        mc_tri[mask][k][0] = cyc[0];
        mc_tri[mask][k][1] = cyc[i];
        mc_tri[mask][k][2] = cyc[i + 1];
      }
    }
  }
  mc_ready = 1;
}

int rfo_mc_table(int* counts256, int* tris) {
  mc_build_table();
  for (int m = 0; m < 256; ++m) {
    counts256[m] = mc_cnt[m];
    for (int k = 0; k < 16; ++k)
      for (int j = 0; j < 3; ++j) tris[(m * 16 + k) * 3 + j] = k < mc_cnt[m] ? mc_tri[m][k][j] : -1;
  }
  return 0;
}

/* meshing.cpp:146-153 */
static uint64_t mc_key(int x, int y, int z, int axis) {
  const int64_t kBias = 1 << 19;
  uint64_t ux = (uint64_t)(x + kBias) & 0xFFFFF, uy = (uint64_t)(y + kBias) & 0xFFFFF;
  uint64_t uz = (uint64_t)(z + kBias) & 0xFFFFF;
  return (((ux << 20) | uy) << 20 | uz) << 2 | (uint64_t)axis;
}

typedef struct {
  uint64_t* keys; /* ~0 = empty */
  uint32_t* vals;
  size_t cap, n;
} mc_map;
static uint32_t mc_map_get_or_add(mc_map* h, uint64_t k, uint32_t v, int* added) {
  if (2 * (h->n + 1) > h->cap) { /* grow */
    size_t nc = h->cap ? 2 * h->cap : 1 << 16;
    uint64_t* nk = (uint64_t*)malloc(nc * 8);
    uint32_t* nv = (uint32_t*)malloc(nc * 4);
    memset(nk, 0xFF, nc * 8);
    for (size_t i = 0; i < h->cap; ++i)
      if (h->keys[i] != ~(uint64_t)0) {
        size_t j = (size_t)((h->keys[i] * 0x9E3779B97F4A7C15ull) >> 20) & (nc - 1);
        while (nk[j] != ~(uint64_t)0) j = (j + 1) & (nc - 1);
        nk[j] = h->keys[i];
        nv[j] = h->vals[i];
      }
    free(h->keys);
    free(h->vals);
    h->keys = nk;
    h->vals = nv;
    h->cap = nc;
  }
  size_t j = (size_t)((k * 0x9E3779B97F4A7C15ull) >> 20) & (h->cap - 1);
  while (h->keys[j] != ~(uint64_t)0) {
    if (h->keys[j] == k) {
      *added = 0;
      return h->vals[j];
    }
    j = (j + 1) & (h->cap - 1);
  }
  h->keys[j] = k;
  h->vals[j] = v;
  h->n++;
  *added = 1;
  return v;
}

/* extract_mesh (meshing.cpp:156-217): entries in index order, cells lz/ly/lx,
 * a cell is skipped unless all 8 corners are allocated with w_depth > 0;
 * a vertex is created the first time its lattice edge is met.  Outputs are
 * malloc'ed (free with rfo_free). */
int rfo_extract_mesh(const rfo_map* m, float voxelSize, float** vOut, uint32_t** tOut, long long* nV,
                     long long* nT) {
  mc_build_table();
  size_t vcap = 1 << 16, tcap = 1 << 16, nv = 0, nt = 0;
  float* V = (float*)malloc(vcap * 12);
  uint32_t* T = (uint32_t*)malloc(tcap * 12);
  mc_map h = {NULL, NULL, 0, 0};
  const uint32_t total = m->buckets + m->excess;
  for (uint32_t idx = 0; idx < total; ++idx) {
    const entry_t* e = &m->entries[idx];
    if (e->ptr < 0) continue;
    for (int lz = 0; lz < BS; ++lz)
      for (int ly = 0; ly < BS; ++ly)
        for (int lx = 0; lx < BS; ++lx) {
          const int cx = e->x * BS + lx, cy = e->y * BS + ly, cz = e->z * BS + lz;
          float sdf[8];
          int observed = 1;
          for (int c = 0; c < 8 && observed; ++c) {
            i3 v = {cx + MC_C[c][0], cy + MC_C[c][1], cz + MC_C[c][2]};
            const voxel_t* vx = find_voxel(m, v);
            observed = vx != NULL && vx->w > 0;
            sdf[c] = vx ? sdf_to_logical(vx->sdf) : 1.f;
          }
          if (!observed) continue;
          int mask = 0;
          for (int c = 0; c < 8; ++c)
            if (sdf[c] < 0.f) mask |= 1 << c;
          for (int k = 0; k < mc_cnt[mask]; ++k) {
            uint32_t id[3];
            for (int q = 0; q < 3; ++q) {
              const int ed = mc_tri[mask][k][q];
              int a = MC_E[ed][0], b = MC_E[ed][1];
              int va[3] = {cx + MC_C[a][0], cy + MC_C[a][1], cz + MC_C[a][2]};
              int vb[3] = {cx + MC_C[b][0], cy + MC_C[b][1], cz + MC_C[b][2]};
              float fa = sdf[a], fb = sdf[b];
              int axis = va[0] != vb[0] ? 0 : (va[1] != vb[1] ? 1 : 2);
              if (va[axis] > vb[axis]) {
                for (int t = 0; t < 3; ++t) {
                  int x = va[t];
                  va[t] = vb[t];
                  vb[t] = x;
                }
                float ft = fa;
                fa = fb;
                fb = ft;
              }
              int added = 0;
              id[q] = mc_map_get_or_add(&h, mc_key(va[0], va[1], va[2], axis), (uint32_t)nv, &added);
              if (added) {
                const float denom = fa - fb;
                const float t = fabsf(denom) < 1e-12f ? 0.5f : fa / denom;
                float p[3] = {(float)va[0], (float)va[1], (float)va[2]};
                p[axis] += t;
                if (nv == vcap) V = (float*)realloc(V, (vcap *= 2) * 12);
                V[3 * nv + 0] = p[0] * voxelSize;
                V[3 * nv + 1] = p[1] * voxelSize;
                V[3 * nv + 2] = p[2] * voxelSize;
                ++nv;
              }
            }
            if (nt == tcap) T = (uint32_t*)realloc(T, (tcap *= 2) * 12);
            T[3 * nt + 0] = id[0];
            T[3 * nt + 1] = id[1];
            T[3 * nt + 2] = id[2];
            ++nt;
          }
        }
  }
  free(h.keys);
  free(h.vals);
  *vOut = V;
  *tOut = T;
  *nV = (long long)nv;
  *nT = (long long)nt;
  return 0;
}
void rfo_free(void* p) { free(p); }

/* direct voxel writes (analytic TSDF test maps, as the reference's meshing
 * tests build them) */
int rfo_set_block(rfo_map* m, const int* pos3, const int16_t* sdf512, const uint8_t* w512) {
  i3 p = {pos3[0], pos3[1], pos3[2]};
  int idx = allocate_block(m, p);
  if (idx < 0) return -1;
  voxel_t* b = &m->vba[(size_t)m->entries[idx].ptr * BS3];
  for (int i = 0; i < BS3; ++i) {
    b[i].sdf = sdf512[i];
    b[i].w = w512[i];
  }
  return 0;
}

/* ------------------------------------------------- full ViewBuilder */
/* rgb_to_intensity (P/src/view.cpp:8-16): (0.299 r + 0.587 g + 0.114 b) / 255,
 * C++ left-to-right evaluation, the channels promoted to float. */
void rfo_rgb_to_intensity(const uint8_t* rgb, int w, int h, float* out) {
  for (int i = 0; i < w * h; ++i) {
    const uint8_t* c = rgb + 3 * (size_t)i;
    out[i] = (0.299f * (float)c[0] + 0.587f * (float)c[1] + 0.114f * (float)c[2]) / 255.f;
  }
}

/* bilateral_filter (view.cpp:18-44): 5x5 window, invalid (<= 0) centre and
 * neighbours skipped, w = exp(-(dx^2 + dy^2) invS2 - dr^2 invR2) with the C
 * library's expf (the reference calls std::exp(float)); out = sum / wsum. */
void rfo_bilateral_filter(const float* in, int w, int h, float spatialSigma, float rangeSigma, float* out) {
  const int radius = 2;
  const float invS2 = 1.f / (2.f * spatialSigma * spatialSigma);
  const float invR2 = 1.f / (2.f * rangeSigma * rangeSigma);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const float centre = in[(size_t)y * w + x];
      out[(size_t)y * w + x] = -1.f;
      if (centre <= 0.f) continue;
      float sum = 0.f, wsum = 0.f;
      for (int dy = -radius; dy <= radius; ++dy)
        for (int dx = -radius; dx <= radius; ++dx) {
          const int nx = x + dx, ny = y + dy;
          if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
          const float d = in[(size_t)ny * w + nx];
          if (d <= 0.f) continue;
          const float dr = d - centre;
          const float wt = expf((float)(-(dx * dx + dy * dy)) * invS2 - dr * dr * invR2);
          sum += wt * d;
          wsum += wt;
        }
      out[(size_t)y * w + x] = sum / wsum;
    }
}

/* compute_normals (view.cpp:46-67): central differences of backprojected
 * points, n = px x py / |px x py| (Eigen: cross components as written, norm =
 * sqrt(x^2 + (y^2 + z^2)), per-coefficient division), oriented toward the
 * camera; (0,0,0,-1) where invalid, on the border, or |n| < 1e-12. */
static void bp3(const intr_t* in, float u, float v, float z, float* o) {
  o[0] = (u - in->cx) / in->fx * z;
  o[1] = (v - in->cy) / in->fy * z;
  o[2] = z;
}
void rfo_compute_normals(const float* d, int w, int h, const float* f4, float* out4) {
  const intr_t in = {w, h, f4[0], f4[1], f4[2], f4[3]};
  for (int i = 0; i < w * h; ++i) {
    out4[4 * i + 0] = 0.f;
    out4[4 * i + 1] = 0.f;
    out4[4 * i + 2] = 0.f;
    out4[4 * i + 3] = -1.f;
  }
  for (int y = 1; y + 1 < h; ++y)
    for (int x = 1; x + 1 < w; ++x) {
      const float dc = d[(size_t)y * w + x];
      const float dxm = d[(size_t)y * w + x - 1], dxp = d[(size_t)y * w + x + 1];
      const float dym = d[(size_t)(y - 1) * w + x], dyp = d[(size_t)(y + 1) * w + x];
      if (dc <= 0.f || dxm <= 0.f || dxp <= 0.f || dym <= 0.f || dyp <= 0.f) continue;
      float a[3], b[3], px[3], py[3], n[3], c[3];
      bp3(&in, (float)x + 1.f, (float)y, dxp, a);
      bp3(&in, (float)x - 1.f, (float)y, dxm, b);
      for (int k = 0; k < 3; ++k) px[k] = a[k] - b[k];
      bp3(&in, (float)x, (float)y + 1.f, dyp, a);
      bp3(&in, (float)x, (float)y - 1.f, dym, b);
      for (int k = 0; k < 3; ++k) py[k] = a[k] - b[k];
      n[0] = px[1] * py[2] - px[2] * py[1];
      n[1] = px[2] * py[0] - px[0] * py[2];
      n[2] = px[0] * py[1] - px[1] * py[0];
      const float len = sqrtf(n[0] * n[0] + (n[1] * n[1] + n[2] * n[2]));
      if (len < 1e-12f) continue;
      for (int k = 0; k < 3; ++k) n[k] /= len;
      bp3(&in, (float)x, (float)y, dc, c);
      if (n[0] * c[0] + (n[1] * c[1] + n[2] * c[2]) > 0.f)
        for (int k = 0; k < 3; ++k) n[k] = -n[k];
      float* o = out4 + 4 * ((size_t)y * w + x);
      o[0] = n[0];
      o[1] = n[1];
      o[2] = n[2];
      o[3] = 1.f;
    }
}

/* downsample_intensity (view.cpp:90-98): 0.25 * (((a + b) + c) + d). */
void rfo_downsample_intensity(const float* in, int w, int h, float* out) {
  const int lw = w / 2, lh = h / 2;
  for (int y = 0; y < lh; ++y)
    for (int x = 0; x < lw; ++x)
      out[(size_t)y * lw + x] = 0.25f * (in[(size_t)(2 * y) * w + 2 * x] + in[(size_t)(2 * y) * w + 2 * x + 1] +
                                         in[(size_t)(2 * y + 1) * w + 2 * x] +
                                         in[(size_t)(2 * y + 1) * w + 2 * x + 1]);
}

/* build_view (view.cpp:100-143) with every option: depth conversion,
 * optional bilateral (spatial sigma 2, range sigma 10 |scale|), intensity
 * when rgb is given, level-0 normals, depth (+ intensity) pyramids.
 * Outputs are packed level after level; intensity / normals may be NULL. */
int rfo_build_view_full(const uint16_t* raw, const uint8_t* rgb, const int* wh, const float* f4, float affScale,
                        float affOffset, int bilateral, int levels, float* depthLevels, float* intensityLevels,
                        float* normals4) {
  const int w = wh[0], h = wh[1];
  if (levels < 1) return -1;
  if (rfo_build_view(raw, wh, affScale, affOffset, 1, depthLevels) != 0) return -1;
  if (bilateral) {
    float* tmp = (float*)malloc(sizeof(float) * (size_t)w * h);
    if (!tmp) return -1;
    memcpy(tmp, depthLevels, sizeof(float) * (size_t)w * h);
    rfo_bilateral_filter(tmp, w, h, 2.f, 10.f * fabsf(affScale), depthLevels);
    free(tmp);
  }
  if (normals4) rfo_compute_normals(depthLevels, w, h, f4, normals4);
  if (rgb && intensityLevels) rfo_rgb_to_intensity(rgb, w, h, intensityLevels);
  const float* prev = depthLevels;
  const float* prevI = intensityLevels;
  float* out = depthLevels + (size_t)w * h;
  float* outI = intensityLevels ? intensityLevels + (size_t)w * h : NULL;
  int pw = w, ph = h;
  for (int l = 1; l < levels; ++l) {
    const int lw = pw / 2, lh = ph / 2;
    for (int y = 0; y < lh; ++y)
      for (int x = 0; x < lw; ++x) {
        float sum = 0.f;
        int n = 0;
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            const float dd = prev[(size_t)(2 * y + dy) * pw + 2 * x + dx];
            if (dd > 0.f) {
              sum += dd;
              ++n;
            }
          }
        out[(size_t)y * lw + x] = n > 0 ? sum / (float)n : -1.f;
      }
    if (rgb && outI) {
      rfo_downsample_intensity(prevI, pw, ph, outI);
      prevI = outI;
      outI += (size_t)lw * lh;
    }
    prev = out;
    out += (size_t)lw * lh;
    pw = lw;
    ph = lh;
  }
  return 0;
}

/* ---------------------------------------------------------------- ICP */
/* Point-to-plane ICP depth tracker (absent in the reference; restated from
 * DESIGN.md §5 "ICP oracle").
 *
 * One evaluation of the normal equations: per valid pixel p
 * of the level, p_w = T_cw p_cam; project p_w into the last render (nearest
 * pixel); V, N = render point/normal; reject invalid maps and
 * |p_w - V| > dist; r = (p_w - V).N; J = [p_w x N; N] (left-multiplied
 * world-frame twist [omega; nu]).
 *
 * The sums are FIXED-POINT integers: every per-pixel term (a product of two
 * floats, exact in double) is scaled by a power of two and floored to an
 * int64, and the int64 terms are summed.  Integer addition is associative, so
 * the sums do not depend on the summation order: the GPU's tree/atomic
 * reduction yields exactly these sums, and the whole tracker (solve, SE(3)
 * update, convergence test) is bit-identical between this oracle and the B200.
 *   S[0..20]  H upper, row-major   floor(J_a J_b 2^32)
 *   S[21..26] g                    floor(J_a r   2^38)
 *   S[27]     sum r^2              floor(r^2     2^44)
 *   S[28]     inliers (count)
 *   S[29]     sum |r|              floor(|r|     2^44)
 *   S[30]     valid depth pixels of the level
 * Range: |p_w| components < 128 m (so |J_a J_b| < 2^16) and gates <= 2 m;
 * a term outside the range fails the evaluation (RFO_ICP_ERANGE). */
#define ICP_SUMS 31
#define RFO_ICP_ERANGE (-2)
static const int kIcpShift[ICP_SUMS] = {32, 32, 32, 32, 32, 32, 32, 32, 32, 32, 32, 32, 32, 32, 32, 32,
                                        32, 32, 32, 32, 32, 38, 38, 38, 38, 38, 38, 44, 0,  44, 0};

static int64_t icp_fixed(double x, int shift) { return (int64_t)floor(ldexp(x, shift)); }

static int icp_accumulate(const float* depth, int lw, int lh, const intr_t* inl, const float* points,
                          const float* normals, const intr_t* inr, const pose_t* renderPose, const pose_t* c2w,
                          float dist, int64_t* S) {
  memset(S, 0, sizeof(int64_t) * ICP_SUMS);
  const float dist2 = dist * dist;
  int err = 0;
  for (int y = 0; y < lh; ++y)
    for (int x = 0; x < lw; ++x) {
      float d = depth[(size_t)y * lw + x];
      if (!(d > 0.f)) continue;
      S[30] += 1;
      v3 pc = backproject(inl, (float)x, (float)y, d);
      v3 pw = pose_apply(c2w, pc);
      v3 q = pose_apply(renderPose, pw);
      if (!(q.z > 0.f)) continue;
      float u = inr->fx * q.x / q.z + inr->cx;
      float v = inr->fy * q.y / q.z + inr->cy;
      if (!(u >= 0.f && v >= 0.f && u <= (float)(inr->w - 1) && v <= (float)(inr->h - 1))) continue;
      int iu = (int)(u + 0.5f), iv = (int)(v + 0.5f);
      const float* V = points + 4 * ((size_t)iv * inr->w + iu);
      const float* N = normals + 4 * ((size_t)iv * inr->w + iu);
      if (!(V[3] > 0.f) || !(N[3] > 0.f)) continue;
      v3 diff = {pw.x - V[0], pw.y - V[1], pw.z - V[2]};
      if (sqnorm3(diff) > dist2) continue;
      if (!(fabsf(pw.x) < 128.f && fabsf(pw.y) < 128.f && fabsf(pw.z) < 128.f)) err = 1;
      v3 n = {N[0], N[1], N[2]};
      float r = dot3(diff, n);
      v3 pxn = cross3(pw, n);
      double J[6] = {pxn.x, pxn.y, pxn.z, n.x, n.y, n.z};
      double rd = r;
      int k = 0;
      for (int a = 0; a < 6; ++a)
        for (int b = a; b < 6; ++b, ++k) S[k] += icp_fixed(J[a] * J[b], 32);
      for (int a = 0; a < 6; ++a) S[21 + a] += icp_fixed(J[a] * rd, 38);
      S[27] += icp_fixed(rd * rd, 44);
      S[28] += 1;
      S[29] += icp_fixed(fabs(rd), 44);
    }
  return err ? RFO_ICP_ERANGE : 0;
}

/* The fixed-point sums as doubles (round to nearest, exact power-of-two scaling). */
static void icp_decode(const int64_t* S, double* out) {
  for (int k = 0; k < ICP_SUMS; ++k) out[k] = ldexp((double)S[k], -kIcpShift[k]);
}

int rfo_icp_reduce(const float* depth, int lw, int lh, const float* f4l, const float* points, const float* normals,
                   const int* wh, const float* renderPose12, const float* renderF4, const float* camToWorld12,
                   float dist, int64_t* sums31, double* out31) {
  int lwh[2] = {lw, lh};
  intr_t inl = intr_from(lwh, f4l);
  intr_t inr = intr_from(wh, renderF4);
  pose_t rp = pose_from12(renderPose12);
  pose_t c2w = pose_from12(camToWorld12);
  int64_t S[ICP_SUMS];
  const int rc = icp_accumulate(depth, lw, lh, &inl, points, normals, &inr, &rp, &c2w, dist, S);
  if (sums31) memcpy(sums31, S, sizeof(S));
  if (out31) icp_decode(S, out31);
  return rc;
}

/* double-precision SE(3) helpers (proj/include/rf/pose.hpp:38-60, S = double) */
typedef struct {
  double R[9];
  double t[3];
} posed_t;
static void matmul3d(const double* A, const double* B, double* C) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) C[r * 3 + c] = A[r * 3 + 0] * B[c] + (A[r * 3 + 1] * B[3 + c] + A[r * 3 + 2] * B[6 + c]);
}
/* sin(x)/x, (1 - cos x)/x^2, (x - sin x)/x^3 for t = x^2 < 1 by their Taylor
 * series, nested, with as many terms as t needs: the first dropped term is
 * below 2^-64 of the value (t < 2^-40: 2 terms; < 2^-20: 3; < 2^-8: 6;
 * else 10).  Basic IEEE operations only, so the B200
 * (rfg_icp.cu:se3_series) evaluates them bit-identically. */
static void se3_series(double t, double* a, double* b, double* c) {
  if (t < 0x1p-40) {
    *a = 1.0 - t * (1.0 / 6.0);
    *b = 0.5 * (1.0 - t * (1.0 / 12.0));
    *c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0));
  } else if (t < 0x1p-20) {
    *a = 1.0 - t * (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0));
    *b = 0.5 * (1.0 - t * (1.0 / 12.0) * (1.0 - t * (1.0 / 30.0)));
    *c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0)));
  } else if (t < 0x1p-8) {
    *a = 1.0 - t * (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0)))));
    *b = 0.5 * (1.0 - t * (1.0 / 12.0) * (1.0 - t * (1.0 / 30.0) * (1.0 - t * (1.0 / 56.0) * (1.0 - t * (1.0 / 90.0) *
         (1.0 - t * (1.0 / 132.0))))));
    *c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0) * (1.0 - t * (1.0 / 156.0))))));
  } else {
    *a = 1.0 - t * (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0) * (1.0 - t * (1.0 / 156.0) * (1.0 - t * (1.0 / 210.0) * (1.0 - t * (1.0 / 272.0) *
         (1.0 - t * (1.0 / 342.0) * (1.0 - t * (1.0 / 420.0))))))))));
    *b = 0.5 * (1.0 - t * (1.0 / 12.0) * (1.0 - t * (1.0 / 30.0) * (1.0 - t * (1.0 / 56.0) * (1.0 - t * (1.0 / 90.0) *
         (1.0 - t * (1.0 / 132.0) * (1.0 - t * (1.0 / 182.0) * (1.0 - t * (1.0 / 240.0) * (1.0 - t * (1.0 / 306.0) *
         (1.0 - t * (1.0 / 380.0))))))))));
    *c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0) * (1.0 - t * (1.0 / 156.0) * (1.0 - t * (1.0 / 210.0) * (1.0 - t * (1.0 / 272.0) *
         (1.0 - t * (1.0 / 342.0) * (1.0 - t * (1.0 / 420.0))))))))));
  }
}
/* Rodrigues coefficients of exp([omega]x) for th2 = |omega|^2: the series
 * below 1 rad; above, sin/cos of theta / 2^k by the series and k exact
 * double-angle steps (no libm: bit-identical on the B200). */
static void se3_coeffs(double th2, double* a, double* b, double* c) {
  if (th2 < 1.0) {
    se3_series(th2, a, b, c);
    return;
  }
  const double theta = sqrt(th2);
  double h = theta;
  int k = 0;
  while (h >= 1.0) {
    h *= 0.5;
    ++k;
  }
  double sa, sb, sc;
  se3_series(h * h, &sa, &sb, &sc);
  double s = h * sa, co = 1.0 - (h * h) * sb;
  for (int i = 0; i < k; ++i) {
    const double s2 = 2.0 * s * co;
    co = 1.0 - 2.0 * s * s;
    s = s2;
  }
  *a = s / theta;
  *b = (1.0 - co) / th2;
  *c = (theta - s) / (theta * th2);
}
/* test hook: the three Rodrigues coefficients for th2 */
void rfo_se3_coeffs(double th2, double* abc) { se3_coeffs(th2, &abc[0], &abc[1], &abc[2]); }

static posed_t se3_exp(const double* tau) {
  const double* w = tau;
  const double* v = tau + 3;
  const double th2 = w[0] * w[0] + (w[1] * w[1] + w[2] * w[2]);
  double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double WW[9];
  matmul3d(W, W, WW);
  double a, b, c;
  se3_coeffs(th2, &a, &b, &c);
  posed_t p;
  double V[9];
  for (int i = 0; i < 9; ++i) {
    double I = (i % 4 == 0) ? 1.0 : 0.0;
    p.R[i] = I + a * W[i] + b * WW[i];
    V[i] = I + b * W[i] + c * WW[i];
  }
  for (int r = 0; r < 3; ++r) p.t[r] = V[r * 3] * v[0] + (V[r * 3 + 1] * v[1] + V[r * 3 + 2] * v[2]);
  return p;
}
static posed_t posed_compose(const posed_t* a, const posed_t* b) {
  posed_t q;
  matmul3d(a->R, b->R, q.R);
  for (int r = 0; r < 3; ++r)
    q.t[r] = (a->R[r * 3] * b->t[0] + (a->R[r * 3 + 1] * b->t[1] + a->R[r * 3 + 2] * b->t[2])) + a->t[r];
  return q;
}
static posed_t posed_inverse(const posed_t* p) {
  posed_t q;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) q.R[r * 3 + c] = p->R[c * 3 + r];
  for (int r = 0; r < 3; ++r) q.t[r] = -(q.R[r * 3] * p->t[0] + (q.R[r * 3 + 1] * p->t[1] + q.R[r * 3 + 2] * p->t[2]));
  return q;
}
static pose_t posed_to_f(const posed_t* p) {
  pose_t q;
  for (int i = 0; i < 9; ++i) q.R[i] = (float)p->R[i];
  for (int i = 0; i < 3; ++i) q.t[i] = (float)p->t[i];
  return q;
}

/* Solve H x = -g from the decoded sums by an LDL^T factorisation (no square
 * roots; one IEEE reciprocal per pivot), in a fixed operation order that the
 * B200 solver (rfg_icp.cu:solve6) repeats:
 *   D_j  = H_jj - sum_{p<j} (L_jp L_jp) D_p,   inv_j = 1 / D_j
 *   L_ij = (H_ij - sum_{p<j} (L_ip L_jp) D_p) inv_j          (i > j)
 *   y_i  = -g_i - sum_{p<i} L_ip y_p  (p ascending)
 *   x_i  = y_i inv_i - sum_{p>i} L_pi x_p  (p descending, i.e. as the x_p appear)
 * *detOut = det(H / n) = prod_j (D_j * (1/n)), the Hessian determinant
 * "after scaling" by the inlier count n; 0 when H is not
 * positive definite.  Returns 0, or -1 when H is not positive definite or
 * det(H / n) < 1e-12 (degenerate). */
static int sym6(int a, int b) { /* index of H_ab in the row-major upper triangle */
  if (a > b) {
    int t = a;
    a = b;
    b = t;
  }
  return a * 6 - a * (a - 1) / 2 + (b - a);
}
int rfo_solve6(const double* sums, double* x, double* detOut) {
  const double n = sums[28];
  double L[36] = {0};
  double D[6], inv[6];
  *detOut = 0.0;
  for (int j = 0; j < 6; ++j) {
    double d = sums[sym6(j, j)];
    for (int p = 0; p < j; ++p) d -= (L[j * 6 + p] * L[j * 6 + p]) * D[p];
    if (!(d > 0.0)) return -1;
    D[j] = d;
    inv[j] = 1.0 / d;
    for (int i = j + 1; i < 6; ++i) {
      double t = sums[sym6(i, j)];
      for (int p = 0; p < j; ++p) t -= (L[i * 6 + p] * L[j * 6 + p]) * D[p];
      L[i * 6 + j] = t * inv[j];
    }
  }
  const double ninv = 1.0 / n;
  double det = 1.0;
  for (int j = 0; j < 6; ++j) det *= D[j] * ninv;
  *detOut = det;
  if (!(det >= 1e-12)) return -1; /* SPEC.md:352 degenerate Hessian */
  double y[6];
  for (int i = 0; i < 6; ++i) {
    double t = -sums[21 + i];
    for (int p = 0; p < i; ++p) t -= L[i * 6 + p] * y[p];
    y[i] = t;
  }
  for (int i = 5; i >= 0; --i) {
    double t = y[i] * inv[i];
    for (int p = 5; p > i; --p) t -= L[p * 6 + i] * x[p];
    x[i] = t;
  }
  return 0;
}

/* Coarse-to-fine tracking loop: levels
 * coarse -> fine, at most iters[l] iterations per level, stop a level when
 * ||delta|| < 1e-4; a level with fewer than minCount inliers is skipped
 * (ok = 0, the pose so far is kept); a degenerate Hessian ends the track and
 * returns the INIT pose, as does a track that never updated
 * the pose.  T_cw <- exp(delta) T_cw.
 * statsOut12 (TrackerIterationSummary, of the last
 * evaluation): {iterations run, inliers, sum r^2, converged, iterations per
 * level x3, ok, inlier_fraction, hessian_det (det(H/n)), residual_mean
 * (sum |r| / n), valid pixels}.  Returns 0, or RFO_ICP_ERANGE. */
int rfo_icp_track(const float* depthLevels, const int* wh, const float* f4, const float* points,
                  const float* normals, const float* renderPose12, const float* renderF4, const float* initPose12,
                  const int* icp6, const float* dist3, float* poseOut12, double* statsOut12) {
  const int levels = icp6[0];
  const int minCount = icp6[4];
  intr_t in0 = intr_from(wh, f4);
  intr_t inr = intr_from(wh, renderF4);
  pose_t rp = pose_from12(renderPose12);
  pose_t init = pose_from12(initPose12);
  pose_t c2wf = pose_inverse(&init);
  posed_t c2w, c2wInit;
  for (int i = 0; i < 9; ++i) c2w.R[i] = c2wf.R[i];
  for (int i = 0; i < 3; ++i) c2w.t[i] = c2wf.t[i];
  c2wInit = c2w;
  /* level offsets inside depthLevels */
  size_t off[8];
  size_t o = 0;
  for (int l = 0; l < levels; ++l) {
    off[l] = o;
    o += (size_t)(in0.w >> l) * (in0.h >> l);
  }
  int64_t S[ICP_SUMS];
  double acc[ICP_SUMS];
  int totalIt = 0, converged = 0, rc = 0, failed = 0;
  double* st = statsOut12;
  memset(st, 0, sizeof(double) * 12);
  st[7] = 1;
  for (int l = levels - 1; l >= 0 && !failed; --l) {
    intr_t inl = in0;
    float sc = ldexpf(1.f, -l);
    inl.w = in0.w >> l;
    inl.h = in0.h >> l;
    inl.fx = in0.fx * sc;
    inl.fy = in0.fy * sc;
    inl.cx = in0.cx * sc;
    inl.cy = in0.cy * sc;
    int it;
    for (it = 0; it < icp6[1 + l]; ++it) {
      pose_t c2wF = posed_to_f(&c2w);
      if (icp_accumulate(depthLevels + off[l], inl.w, inl.h, &inl, points, normals, &inr, &rp, &c2wF, dist3[l], S))
        rc = RFO_ICP_ERANGE;
      icp_decode(S, acc);
      st[1] = acc[28];
      st[2] = acc[27];
      st[8] = acc[30] > 0.0 ? acc[28] / acc[30] : 0.0;
      st[9] = 0.0;
      st[10] = acc[28] > 0.0 ? acc[29] / acc[28] : 0.0;
      st[11] = acc[30];
      if (acc[28] < (double)minCount) {
        st[7] = 0;
        break;
      }
      double delta[6];
      if (rfo_solve6(acc, delta, &st[9]) != 0) {
        st[7] = 0;
        failed = 1;
        c2w = c2wInit;
        break;
      }
      posed_t inc = se3_exp(delta);
      c2w = posed_compose(&inc, &c2w);
      ++totalIt;
      /* ||delta|| < 1e-4, compared squared */
      double nrm2 = delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2] + delta[3] * delta[3] +
                    delta[4] * delta[4] + delta[5] * delta[5];
      if (nrm2 < 1e-8) {
        converged = 1;
        ++it;
        break;
      }
    }
    st[4 + l] = it;
  }
  st[0] = totalIt;
  st[3] = converged && !failed;
  if (failed || totalIt == 0) {
    /* never updated (or degenerate): the init pose itself */
    memcpy(poseOut12, initPose12, 12 * sizeof(float));
    return rc;
  }
  posed_t w2c = posed_inverse(&c2w);
  pose_t outp = posed_to_f(&w2c);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) poseOut12[r * 4 + c] = outp.R[r * 3 + c];
    poseOut12[r * 4 + 3] = outp.t[r];
  }
  return rc;
}

/* ------------------------------------------------------------- export */
uint32_t rfo_total_entries(const rfo_map* m) { return m->buckets + m->excess; }
int rfo_export_entries(const rfo_map* m, int* out5) {
  size_t total = (size_t)m->buckets + m->excess;
  for (size_t i = 0; i < total; ++i) {
    out5[5 * i] = m->entries[i].x;
    out5[5 * i + 1] = m->entries[i].y;
    out5[5 * i + 2] = m->entries[i].z;
    out5[5 * i + 3] = m->entries[i].offset;
    out5[5 * i + 4] = m->entries[i].ptr;
  }
  return (int)total;
}
int rfo_export_blocks(const rfo_map* m, const int* ptrs, int n, uint8_t* out) {
  for (int b = 0; b < n; ++b) memcpy(out + (size_t)b * BS3 * 8, &m->vba[(size_t)ptrs[b] * BS3], BS3 * 8);
  return 0;
}
int rfo_export_visible(const rfo_map* m, int* listOut, uint8_t* typesOut) {
  if (listOut) memcpy(listOut, m->visible, sizeof(int) * m->nVisible);
  if (typesOut) memcpy(typesOut, m->visibility, (size_t)m->buckets + m->excess);
  return m->nVisible;
}
int rfo_free_counts(const rfo_map* m, int* nb, int* ne) {
  *nb = m->nFreeBlocks;
  *ne = m->nFreeExcess;
  return 0;
}
