// rfg_icp.cu — point-to-plane ICP depth tracker (ITMDepthTracker).
//
// The reference has no tracker; the algorithm is restated
// from SPEC.md:333-356,390-395 and fixed by the CPU oracle
// oracle/rfo.c:rfo_icp_track (DESIGN.md §5 "ICP oracle").
//
// Bit-exact with the oracle.  The per-pixel terms of the normal equations
// (products of floats, exact in double) are accumulated as FIXED-POINT
// integers (each term scaled by 2^32 / 2^38 / 2^44 and floored, oracle
// rfo.c:icp_accumulate), and integer sums do not depend on the order of
// summation: the per-thread, warp-shuffle, CTA and cross-CTA (64-bit atomic)
// reductions below yield exactly the oracle's serial sums.  The solve, the
// SE(3) update and the convergence test then run the oracle's IEEE double
// operation sequence (no FMA contraction, IEEE sqrt/division, no libm), so
// the tracked pose is bit-identical.
//
// Per thread the floor-to-grid accumulation costs one add per term: an
// accumulator offset by M = 1.5 * 2^(52-s) lies in [2^(52-s), 2^(53-s)),
// whose doubles are exactly the multiples of 2^-s, so adding a term with
// round-toward-zero (__dadd_rz; the sum is positive) adds floor(term * 2^s)
// * 2^-s exactly, independent of the order; the accumulator's bits minus
// M's bits are the integer sum.
//
// A frame's whole tracker is ONE cooperative launch (k_icp_track: seed from
// the device pose, levels coarse to fine, output pose) with one grid barrier
// per iteration: each CTA adds its 31 partial sums to a global accumulator
// with 64-bit atomics, and after the barrier every CTA reads the totals and
// runs the same solve, so all CTAs hold the identical new estimate without a
// second barrier.  The launch is capturable in the frame's CUDA graph.
#include <cooperative_groups.h>

#include "rfg_common.cuh"

namespace cg = cooperative_groups;

namespace rfg {

#ifndef RFG_ICP_THREADS
#define RFG_ICP_THREADS 512
#endif
#ifndef RFG_ICP_CPS
#define RFG_ICP_CPS 1  // resident tracker CTAs per SM
#endif
constexpr int kIcpThreads = RFG_ICP_THREADS;  // 16 warps: more would cap the registers at 96 (5 warps per SM sub-partition)
constexpr int kIcpSums = 31;   // H upper 21, g 6, sum r^2, inliers, sum |r|, valid pixels
constexpr int kIcpStats = 12;  // TrackerIterationSummary (include/rfg.h)
// fixed-point scale (log2) per sum; 0 = plain integer count (rfo.c:kIcpShift)
__host__ __device__ constexpr int icp_shift(int k) { return k < 21 ? 32 : (k < 27 ? 38 : (k == 28 || k == 30 ? 0 : 44)); }

#ifndef RFG_ICP_SOLVE_PRELOAD
#define RFG_ICP_SOLVE_PRELOAD 1  // the solve's 28 inputs loaded into registers before the factorisation
#endif

// Device tracking state (rfg_map::icpOut).
struct IcpState {
  double c2w[12];                 // current camera->world estimate (row-major 3x4)
  double sums[kIcpSums];          // last evaluation, decoded
  long long fixed[kIcpSums];      // last evaluation, fixed-point
  double stats[kIcpStats];        // TrackerIterationSummary
  float c2wF[12];                 // float cast of c2w
  float w2cF[12];                 // tracked world->camera (output pose)
  float renderPose[12];           // world->camera of the render being tracked against
  int done[4];                    // per-level stop flags (single evaluations)
  unsigned gen;                   // iterations so far: rotates the accumulators
  int error;                      // sticky: a world point outside the fixed-point range
  // hand-off of the coarse level (k_icp_coarse) to k_icp_track
  double c2wInit[12];
  int failed;
  // phase timers of CTA 0 (ns, %globaltimer), accumulated over iterations:
  // {associate+reduce, grid barrier, read totals, solve, iterations,
  //  level-0 total, level-1 total, level-2 total}
  unsigned long long timers[8];
  // three rotating cross-CTA accumulators: iteration i adds into [i % 3]
  // and zeroes [(i + 1) % 3], which iteration i - 2 used and every CTA has
  // read before the barrier of iteration i - 1 (all zero between launches)
  unsigned long long acc[3][32];
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifdef RFG_ICP_SUB
// debug build: sub-phases of an evaluation as CTA 0 thread 0 sees them, per
// level: {fill, associate+gather+accumulate, warp reduce, wait for the CTA's
// warps, CTA sum + atomics, slowest CTA's evaluation, -, iterations}
__device__ unsigned long long g_icp_sub[3][8];
__device__ unsigned long long g_icp_maxev;
#define ICP_SUB(k) \
  if (blockIdx.x == 0 && threadIdx.x == 0) subT[k] = gtimer()
#else
#define ICP_SUB(k)
#endif

struct IcpLevelArgs {
  const float* depth;   // pyramid level
  int lw, lh;
  float fx, fy, cx, cy; // level intrinsics (Intrinsics::atLevel, camera.hpp:35-45)
  const float4* points;
  const float4* normals;
  int rw, rh;           // render size (level 0)
  float rfx, rfy, rcx, rcy;
  float dist;           // outlier gate |p_w - V| (m)
  int level;
  int iters;
  int minCount;
  int evalOnly;         // 1: record the sums, never update the pose
};

// Per-CTA copy of the Gauss-Newton state (identical in every CTA).
struct GnShared {
  double c2w[12];
  double c2wInit[12];
  double sums[kIcpSums];
  long long fixed[kIcpSums];
  double stats[kIcpStats];
  float c2wF[12];
  float rp[12];
  int done;
  int failed;  // degenerate Hessian: the track returns the init pose
};

// ------------------------------------------------------------- the solve
// double-precision SE(3) (proj/include/rf/pose.hpp:45-60 with S = double);
// every function is the oracle's operation sequence (rfo.c), IEEE ops only
__device__ __forceinline__ void matmul3d(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C[r * 3 + c] = A[r * 3 + 0] * B[c] + (A[r * 3 + 1] * B[3 + c] + A[r * 3 + 2] * B[6 + c]);
}

__device__ void c2w_to_float(const double* c, float* f) {
  for (int i = 0; i < 12; ++i) f[i] = (float)c[i];
}

// rfo.c:se3_series — sin(x)/x, (1 - cos x)/x^2, (x - sin x)/x^3 for t = x^2 < 1,
// as many Taylor terms as t needs (the same tiers as the oracle)
// (returned by value: the coefficients stay in registers — through reference
// parameters across the noinline call they went through local memory)
struct Se3C {
  double a, b, c;
};
__device__ __forceinline__ Se3C se3_series(double t) {
  double a, b, c;
  if (t < 0x1p-40) {
    a = 1.0 - t * (1.0 / 6.0);
    b = 0.5 * (1.0 - t * (1.0 / 12.0));
    c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0));
  } else if (t < 0x1p-20) {
    a = 1.0 - t * (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0));
    b = 0.5 * (1.0 - t * (1.0 / 12.0) * (1.0 - t * (1.0 / 30.0)));
    c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0)));
  } else if (t < 0x1p-8) {
    a = 1.0 - t * (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0)))));
    b = 0.5 * (1.0 - t * (1.0 / 12.0) * (1.0 - t * (1.0 / 30.0) * (1.0 - t * (1.0 / 56.0) * (1.0 - t * (1.0 / 90.0) *
         (1.0 - t * (1.0 / 132.0))))));
    c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0) * (1.0 - t * (1.0 / 156.0))))));
  } else {
    a = 1.0 - t * (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0) * (1.0 - t * (1.0 / 156.0) * (1.0 - t * (1.0 / 210.0) * (1.0 - t * (1.0 / 272.0) *
         (1.0 - t * (1.0 / 342.0) * (1.0 - t * (1.0 / 420.0))))))))));
    b = 0.5 * (1.0 - t * (1.0 / 12.0) * (1.0 - t * (1.0 / 30.0) * (1.0 - t * (1.0 / 56.0) * (1.0 - t * (1.0 / 90.0) *
         (1.0 - t * (1.0 / 132.0) * (1.0 - t * (1.0 / 182.0) * (1.0 - t * (1.0 / 240.0) * (1.0 - t * (1.0 / 306.0) *
         (1.0 - t * (1.0 / 380.0))))))))));
    c = (1.0 / 6.0) * (1.0 - t * (1.0 / 20.0) * (1.0 - t * (1.0 / 42.0) * (1.0 - t * (1.0 / 72.0) *
         (1.0 - t * (1.0 / 110.0) * (1.0 - t * (1.0 / 156.0) * (1.0 - t * (1.0 / 210.0) * (1.0 - t * (1.0 / 272.0) *
         (1.0 - t * (1.0 / 342.0) * (1.0 - t * (1.0 / 420.0))))))))));
  }
  return Se3C{a, b, c};
}

// rfo.c:se3_coeffs — the series below 1 rad, else halving + double angles
__device__ __noinline__ Se3C se3_coeffs_large(double th2) {
  const double theta = sqrt(th2);
  double h = theta;
  int k = 0;
  while (h >= 1.0) {
    h *= 0.5;
    ++k;
  }
  const Se3C ser = se3_series(h * h);
  double s = h * ser.a, co = 1.0 - (h * h) * ser.b;
  for (int i = 0; i < k; ++i) {
    const double s2 = 2.0 * s * co;
    co = 1.0 - 2.0 * s * s;
    s = s2;
  }
  return Se3C{s / theta, (1.0 - co) / th2, (theta - s) / (theta * th2)};
}
__device__ __forceinline__ Se3C se3_coeffs(double th2) {
  return th2 < 1.0 ? se3_series(th2) : se3_coeffs_large(th2);
}

// rfo.c:rfo_solve6 — LDL^T of H (no square roots), det(H / n) = prod D_j (1/n),
// forward substitution (p ascending), back substitution (p descending).
// Every loop has constant bounds and is fully unrolled, so the factorisation
// lives in registers; a non-positive pivot raises `bad` (and is replaced by 1
// so the rest stays finite) instead of leaving the unrolled code early.
// 1/D_j is the correctly rounded reciprocal (__drcp_rn == the oracle's 1.0/d).
__host__ __device__ constexpr int sym6(int a, int b) {
  return a <= b ? a * 6 - a * (a - 1) / 2 + (b - a) : b * 6 - b * (b - 1) / 2 + (a - b);
}
__device__ __forceinline__ int solve6(const double* sumsIn, double* x, double* detOut) {
#if RFG_ICP_SOLVE_PRELOAD
  // the 28 inputs into registers up front: the reciprocals' slow-path
  // branches would otherwise keep each column's shared-memory loads behind
  // the previous column's reciprocal
  double sums[29];
#pragma unroll
  for (int k = 0; k < 29; ++k) sums[k] = sumsIn[k];
#pragma unroll
  for (int k = 0; k < 29; ++k) asm volatile("" ::"d"(sums[k]));
#else
  const double* sums = sumsIn;
#endif
  const double n = sums[28];
  double L[36];
  double D[6], inv[6];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double d = sums[sym6(j, j)];
#pragma unroll
    for (int p = 0; p < 6; ++p)
      if (p < j) d -= __dmul_rn(__dmul_rn(L[j * 6 + p], L[j * 6 + p]), D[p]);
    if (!(d > 0.0)) {
      bad = true;
      d = 1.0;
    }
    D[j] = d;
    inv[j] = __drcp_rn(d);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      if (i > j) {
        double t = sums[sym6(i, j)];
#pragma unroll
        for (int p = 0; p < 6; ++p)
          if (p < j) t -= __dmul_rn(__dmul_rn(L[i * 6 + p], L[j * 6 + p]), D[p]);
        L[i * 6 + j] = __dmul_rn(t, inv[j]);
      }
    }
  }
  // (x is computed unconditionally: the degeneracy test is not on the
  // substitution's dependency chain)
  const double ninv = __drcp_rn(n);
  double det = 1.0;
#pragma unroll
  for (int j = 0; j < 6; ++j) det = __dmul_rn(det, __dmul_rn(D[j], ninv));
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double t = -sums[21 + i];
#pragma unroll
    for (int p = 0; p < 6; ++p)
      if (p < i) t -= __dmul_rn(L[i * 6 + p], y[p]);
    y[i] = t;
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double t = __dmul_rn(y[i], inv[i]);
#pragma unroll
    for (int p = 5; p >= 0; --p)
      if (p > i) t -= __dmul_rn(L[p * 6 + i], x[p]);
    x[i] = t;
  }
  *detOut = bad ? 0.0 : det;
  return (bad || !(det >= 1e-12)) ? -1 : 0;  // SPEC.md:352 degenerate Hessian
}

// The evaluation's summary ratios (rfo_icp_track: inlier_fraction,
// residual_mean, valid pixels); off the solve's path.
__device__ __forceinline__ void icp_summary(GnShared& g) {
  const double* acc = g.sums;
  g.stats[8] = acc[30] > 0.0 ? acc[28] / acc[30] : 0.0;
  g.stats[10] = acc[28] > 0.0 ? acc[29] / acc[28] : 0.0;
  g.stats[11] = acc[30];
}

// One Gauss-Newton step on the CTA-local state (oracle: rfo_icp_track loop
// body): summary, count gate, solve, T_cw <- exp(delta) T_cw, convergence.
__device__ void gn_step(GnShared& g, int level, int minCount) {
  const double* acc = g.sums;
  double* st = g.stats;
  // (st[8], st[10], st[11]: icp_summary, on another warp)
  st[1] = acc[28];
  st[2] = acc[27];
  st[9] = 0.0;
  if (acc[28] < (double)minCount) {
    st[7] = 0.0;
    g.done = 1;
    return;
  }
  double delta[6];
  if (solve6(acc, delta, &st[9]) != 0) {
    st[7] = 0.0;
    g.done = 1;
    g.failed = 1;
    for (int i = 0; i < 12; ++i) g.c2w[i] = g.c2wInit[i];
    c2w_to_float(g.c2w, g.c2wF);
    return;
  }
  const double* w = delta;
  const double* v = delta + 3;
  const double th2 = w[0] * w[0] + (w[1] * w[1] + w[2] * w[2]);
  const double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double WW[9];
  matmul3d(W, W, WW);
  const Se3C co = se3_coeffs(th2);
  const double ca = co.a, cb = co.b, cc = co.c;
  double ER[9], V[9], Et[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    if (i % 4 == 0) {
      // diagonal: W[i] = 0, and 1 + (a * 0) == 1 exactly for any finite a,
      // so the oracle's (I + a W) + b WW is 1 + b WW here
      ER[i] = 1.0 + cb * WW[i];
      V[i] = 1.0 + cc * WW[i];
    } else {
      ER[i] = 0.0 + ca * W[i] + cb * WW[i];
      V[i] = 0.0 + cb * W[i] + cc * WW[i];
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) Et[r] = V[r * 3] * v[0] + (V[r * 3 + 1] * v[1] + V[r * 3 + 2] * v[2]);
  double CR[9], Ct[3], NR[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c) CR[r * 3 + c] = g.c2w[r * 4 + c];
    Ct[r] = g.c2w[r * 4 + 3];
  }
  matmul3d(ER, CR, NR);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c) g.c2w[r * 4 + c] = NR[r * 3 + c];
    g.c2w[r * 4 + 3] = (ER[r * 3] * Ct[0] + (ER[r * 3 + 1] * Ct[1] + ER[r * 3 + 2] * Ct[2])) + Et[r];
  }
  c2w_to_float(g.c2w, g.c2wF);
  st[0] += 1.0;
  st[4 + level] += 1.0;
  // ||delta|| < 1e-4, compared squared (rfo.c)
  const double nrm2 = delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2] + delta[3] * delta[3] +
                      delta[4] * delta[4] + delta[5] * delta[5];
  if (nrm2 < 1e-8) {
    st[3] = 1.0;
    g.done = 1;
  }
}

// ------------------------------------------------------ the reduction
// Pixels per thread and round; a level's first round keeps each thread's
// camera-space points (pose-independent) in shared memory for the level's
// later iterations.  Level 0 at 640x480 on 148 CTAs is 4.05 pixels per
// thread: one cached round plus a few uncached pixels.
constexpr int kIcpPx = 5;  // 148 x 512 x 5 >= 640 x 480: one cached round at C1/C2
constexpr int kIcpGroup = 2;  // projections + gathers issued 2 pixels at a time
// pixels per thread between flushes of the per-thread fixed-point
// accumulators (|term| < 2^16 H units, so 8 terms stay inside the 2^19 range)
constexpr int kIcpFlush = 8;

// fixed-point offsets M = 1.5 * 2^(52 - s)
__device__ __forceinline__ double icp_offset(int k) {
  return icp_shift(k) == 32 ? 1572864.0 : (icp_shift(k) == 38 ? 24576.0 : 384.0);
}

// Per-thread accumulators: offset doubles for the 29 fixed-point sums (slots
// 28 and 30 unused) and the two counts.
struct IcpAcc {
  double a[kIcpSums];
  int count, valid;
};

__device__ __forceinline__ void acc_reset(IcpAcc& s) {
#pragma unroll
  for (int k = 0; k < kIcpSums; ++k) s.a[k] = icp_offset(k);
  s.count = 0;
  s.valid = 0;
}

// J J^T, J r, r^2, |r| and the count of one associated pixel (the oracle's
// per-pixel body, rfo.c:icp_accumulate); false when the world point is
// outside the fixed-point range (|p_w| components < 128 m).
__device__ __forceinline__ bool icp_add(IcpAcc& s, f3 pw, float4 V, float4 N, float dist2) {
  if (!(V.w > 0.f) || !(N.w > 0.f)) return true;
  const f3 diff{pw.x - V.x, pw.y - V.y, pw.z - V.z};
  if (sqnorm3(diff) > dist2) return true;
  const bool inRange = fabsf(pw.x) < 128.f && fabsf(pw.y) < 128.f && fabsf(pw.z) < 128.f;
  const f3 nn{N.x, N.y, N.z};
  const float r = dot3(diff, nn);
  const f3 pxn = cross3(pw, nn);
  const double J[6] = {pxn.x, pxn.y, pxn.z, nn.x, nn.y, nn.z};
  const double rd = r;
  int k = 0;
  // the products of two floats are exact in double, so one fused
  // multiply-add rounded toward zero (DFMA.RZ) is exactly the exact product
  // added with the floor at the accumulator's 2^-s ulp (rfo.c icp_fixed)
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i; j < 6; ++j, ++k) s.a[k] = __fma_rz(J[i], J[j], s.a[k]);
#pragma unroll
  for (int i = 0; i < 6; ++i) s.a[21 + i] = __fma_rz(J[i], rd, s.a[21 + i]);
  s.a[27] = __fma_rz(rd, rd, s.a[27]);
  s.a[29] = __dadd_rz(s.a[29], fabs(rd));
  s.count += 1;
  return inRange;
}

// nearest-pixel association in the last render: pixel index or -1
__device__ __forceinline__ int icp_associate(const IcpLevelArgs& a, const Pose& rp, f3 pw) {
  const f3 q = pose_apply(rp, pw);
  if (!(q.z > 0.f)) return -1;
  const float u = a.rfx * q.x / q.z + a.rcx;
  const float v = a.rfy * q.y / q.z + a.rcy;
  if (!(u >= 0.f && v >= 0.f && u <= (float)(a.rw - 1) && v <= (float)(a.rh - 1))) return -1;
  const int iu = (int)(u + 0.5f), iv = (int)(v + 0.5f);
  return iv * a.rw + iu;
}

// The CTA's fixed-point sums of the thread accumulators, added to the global
// accumulator `dst` (64-bit atomics; integer sums, so the order is
// irrelevant).  Warp: recursive halving (lane l ends with sum l: 31
// shuffles of 64 bits instead of 31 x 5); CTA: shared memory.
__device__ __forceinline__ void icp_cta_flush(const IcpAcc& s, long long (*sh)[32], unsigned long long* dst,
                                              int activeWarps, unsigned long long* subT = nullptr) {
  (void)subT;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid < activeWarps) {  // warps without pixels hold zeros: skip their reduction
  long long v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k == 28)
      v[k] = s.count;
    else if (k == 30)
      v[k] = s.valid;
    else if (k < kIcpSums)
      v[k] = __double_as_longlong(s.a[k]) - __double_as_longlong(icp_offset(k));
    else
      v[k] = 0;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const long long send = hi ? v[i] : v[i + o];
      const long long keep = hi ? v[i + o] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  sh[wid][lane] = v[0];
  }
#ifdef RFG_ICP_SUB
  if (subT) ICP_SUB(3);
#endif
  __syncthreads();
#ifdef RFG_ICP_SUB
  if (subT) ICP_SUB(4);
#endif
  if (threadIdx.x < kIcpSums) {
    long long t = 0;
#pragma unroll
    for (int w = 0; w < kIcpThreads / 32; ++w)
      if (w < activeWarps) t += sh[w][threadIdx.x];
    if (t) atomicAdd(dst + threadIdx.x, (unsigned long long)t);
  }
  __syncthreads();  // sh is reused by the next round
#ifdef RFG_ICP_SUB
  if (subT) ICP_SUB(5);
#endif
}

// One evaluation's contribution of this CTA, added to dst.  The level's
// pixels are dealt in 32-pixel chunks round-robin over the CTAs and their
// warps: warp w of CTA c takes chunks c + nCta (w + 16 k), k = 0, 1, ...
// (k < kIcpPx: camera points cached when `fill`; the rest uncached), so
// every CTA samples the whole image (balanced work before the grid barrier)
// and a coarse level still reaches every SM.  Returns false when a world
// point was outside the fixed-point range.  (The sums are order-independent
// integers, so the pixel-to-thread mapping does not change them.)
__device__ __forceinline__ bool icp_cta_eval(const IcpLevelArgs& a, const GnShared& g, const Pose& rp,
                                             const Intr& inl, float dist2, int n, int nCta, long long (*sh)[32],
                                             float4* pcs, bool fill, unsigned long long* dst) {
  const Pose c2w = pose_from12(g.c2wF);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int kWarps = kIcpThreads / 32;
  const int nChunks = (n + 31) >> 5;
  const int c = blockIdx.x;
  // warps with at least one chunk (CTA-uniform), and the CTA's rounds
  const int myChunks = nChunks > c ? (nChunks - c + nCta - 1) / nCta : 0;
  const int activeWarps = min(kWarps, myChunks);
  const int rounds = (myChunks + kWarps - 1) / kWarps;
  auto pixel = [&](int k) -> int {
    const int chunk = c + nCta * (wid + kWarps * k);
    const int p = chunk * 32 + lane;
    return (chunk < nChunks && p < n) ? p : -1;
  };
  bool ok = true;
  IcpAcc s;
  acc_reset(s);
#ifdef RFG_ICP_SUB
  unsigned long long subT[6] = {0, 0, 0, 0, 0, 0};
  ICP_SUB(0);
#else
  unsigned long long* subT = nullptr;
#endif
  if (fill) {
#pragma unroll
    for (int k = 0; k < kIcpPx; ++k) {
      const int p = pixel(k);
      float4 cp = make_float4(0.f, 0.f, 0.f, -1.f);
      if (p >= 0) {
        const float d = __ldg(a.depth + p);
        if (d > 0.f) {
          const int x = p % a.lw, y = p / a.lw;
          const f3 pc = backproject(inl, (float)x, (float)y, d);
          cp = make_float4(pc.x, pc.y, pc.z, 1.f);
        }
      }
      pcs[k * kIcpThreads + t] = cp;  // each thread reads back only its own slots
    }
  }
  ICP_SUB(1);
#pragma unroll
  for (int kb = 0; kb < kIcpPx; kb += kIcpGroup) {
    if (kb >= rounds) break;  // CTA-uniform
    f3 pw[kIcpGroup];
    int pix[kIcpGroup];
#pragma unroll
    for (int j = 0; j < kIcpGroup; ++j) {
      pix[j] = -1;
      if (kb + j >= kIcpPx) continue;
      const float4 cp = pcs[(kb + j) * kIcpThreads + t];
      pw[j] = f3{0.f, 0.f, 0.f};
      if (cp.w > 0.f) {
        s.valid += 1;
        pw[j] = pose_apply(c2w, f3{cp.x, cp.y, cp.z});
        pix[j] = icp_associate(a, rp, pw[j]);
      }
    }
    float4 V[kIcpGroup], N[kIcpGroup];
#pragma unroll
    for (int j = 0; j < kIcpGroup; ++j) {
      if (pix[j] >= 0) {
        V[j] = __ldg(a.points + pix[j]);
        N[j] = __ldg(a.normals + pix[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kIcpGroup; ++j)
      if (pix[j] >= 0) ok &= icp_add(s, pw[j], V[j], N[j], dist2);
  }
  // rounds beyond the cached slots (large images), uncached, flushed every
  // kIcpFlush pixels (the fixed-point accumulators' range)
  for (int k = kIcpPx; k < rounds; ++k) {
    if (k % kIcpFlush == 0) {
      icp_cta_flush(s, sh, dst, activeWarps);
      acc_reset(s);
    }
    const int p = pixel(k);
    if (p < 0) continue;
    const float d = __ldg(a.depth + p);
    if (!(d > 0.f)) continue;
    s.valid += 1;
    const int x = p % a.lw, y = p / a.lw;
    const f3 pc = backproject(inl, (float)x, (float)y, d);
    const f3 pw = pose_apply(c2w, pc);
    const int pix = icp_associate(a, rp, pw);
    if (pix < 0) continue;
    ok &= icp_add(s, pw, __ldg(a.points + pix), __ldg(a.normals + pix), dist2);
  }
  ICP_SUB(2);
  icp_cta_flush(s, sh, dst, activeWarps, subT);
#ifdef RFG_ICP_SUB
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < 5; ++k) g_icp_sub[a.level][k] += subT[k + 1] - subT[k];
    g_icp_sub[a.level][7] += 1;
  }
#endif
  return ok;
}

// One level's Gauss-Newton loop on the CTA-local state g.  CTAs with
// blockIdx.x < nCta own the level's pixels (icp_cta_eval's chunks); the
// others only join the barriers and run the same solve.  `gi` counts
// iterations across levels (accumulator rotation, with the launch's `gen`).
__device__ __forceinline__ void icp_run_level(IcpState* st, const IcpLevelArgs& a, int nCta, GnShared& g,
                                              long long (*sh)[32], float4* pcs, unsigned gen, int& gi,
                                              unsigned long long* tacc) {
  const Intr inl{a.lw, a.lh, a.fx, a.fy, a.cx, a.cy};
  const float dist2 = a.dist * a.dist;
  const int n = a.lw * a.lh;
  const Pose rp = pose_from12(g.rp);
  const bool timed = blockIdx.x == 0 && threadIdx.x == 0;
  const bool owner = (int)blockIdx.x < nCta;
  cg::grid_group grid = cg::this_grid();
  for (int it = 0; it < a.iters && !g.done; ++it, ++gi) {
    unsigned long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    if (timed) t0 = gtimer();
    unsigned long long* buf = st->acc[(gen + gi) % 3];
#ifdef RFG_ICP_SUB
    const unsigned long long tEv = gtimer();
#endif
    if (owner) {
      const bool ok = icp_cta_eval(a, g, rp, inl, dist2, n, nCta, sh, pcs, it == 0, buf);
      if (!ok) st->error = 1;
    }
#ifdef RFG_ICP_SUB
    if (threadIdx.x == 0) atomicMax(&g_icp_maxev, gtimer() - tEv);
#endif
    if (blockIdx.x == 0 && threadIdx.x < 32) st->acc[(gen + gi + 1) % 3][threadIdx.x] = 0ull;
    if (timed) t1 = gtimer();
    grid.sync();
    if (timed) t2 = gtimer();
#ifdef RFG_ICP_SUB
    if (timed && a.level < 3) {
      g_icp_sub[a.level][5] += *((volatile unsigned long long*)&g_icp_maxev);
      g_icp_maxev = 0;
    }
#endif
    if (threadIdx.x < kIcpSums) {
      const long long v = (long long)__ldcg(buf + threadIdx.x);
      g.fixed[threadIdx.x] = v;
      g.sums[threadIdx.x] = ldexp((double)v, -icp_shift(threadIdx.x));
    }
    __syncthreads();
    if (timed) t3 = gtimer();
    if (threadIdx.x == 0) {
      if (a.evalOnly)
        g.done = 1;
      else
        gn_step(g, a.level, a.minCount);
    } else if (threadIdx.x == 32) {
      icp_summary(g);
    }
    __syncthreads();
#ifdef RFG_ICP_LEVEL_ONLY
    if (timed && a.level == RFG_ICP_LEVEL_ONLY) {  // debug: phases of one level only
#else
    if (timed) {  // in registers; flushed once at the end of the kernel
#endif
      const unsigned long long t4 = gtimer();
      tacc[0] += t1 - t0;
      tacc[1] += t2 - t1;
      tacc[2] += t3 - t2;
      tacc[3] += t4 - t3;
      tacc[4] += 1;
      if (a.level < 3) tacc[5 + a.level] += t4 - t0;
    }
  }
}

__device__ __forceinline__ void icp_publish(IcpState* st, const GnShared& g, const unsigned long long* tacc,
                                            unsigned gen, int gi) {
#pragma unroll
  for (int i = 0; i < 8; ++i) st->timers[i] += tacc[i];
  for (int i = 0; i < 12; ++i) {
    st->c2w[i] = g.c2w[i];
    st->c2wF[i] = g.c2wF[i];
  }
  for (int k = 0; k < kIcpSums; ++k) {
    st->sums[k] = g.sums[k];
    st->fixed[k] = g.fixed[k];
  }
  for (int i = 0; i < kIcpStats; ++i) st->stats[i] = g.stats[i];
  st->gen = (gen + (unsigned)gi) % 3u;
}

// Single evaluation / single level on the state in `st` (rfg_icp_reduce).
__global__ void __launch_bounds__(kIcpThreads, RFG_ICP_CPS) k_icp_level(IcpState* st, IcpLevelArgs a) {
  __shared__ long long sh[kIcpThreads / 32][32];
  __shared__ GnShared g;
  __shared__ float4 pcs[kIcpPx * kIcpThreads];
  const unsigned gen = __ldcg(&st->gen);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) {
      g.c2w[i] = __ldcg(&st->c2w[i]);
      g.c2wInit[i] = g.c2w[i];
      g.c2wF[i] = __ldcg(&st->c2wF[i]);
      g.rp[i] = __ldcg(&st->renderPose[i]);
    }
    for (int i = 0; i < kIcpStats; ++i) g.stats[i] = __ldcg(&st->stats[i]);
    g.done = __ldcg(&st->done[a.level]);
    g.failed = 0;
  }
  __syncthreads();
  int gi = 0;
  unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  icp_run_level(st, a, gridDim.x, g, sh, pcs, gen, gi, tacc);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    icp_publish(st, g, tacc, gen, gi);
    st->done[a.level] = g.done;
  }
}

// The whole coarse-to-fine track of a frame in ONE cooperative launch:
// every CTA seeds its state from the device-resident pose, runs the levels
// coarse to fine with the same per-level pixel partition as a per-level
// launch, and CTA 0 publishes the result.
struct IcpTrackArgs {
  IcpLevelArgs lv[3];
  int nCta[3];
  int levels;
  const float* w2cInit;
  const float* renderPose;
  float* w2cOut;
  float* renderPoseOut;  // nullable: the next frame's render pose := the output pose
  int fromState;         // 1: continue the track k_icp_coarse left in the state (its level skipped here)
};

// The track's seed: inverse of the float init pose, widened to double (as
// the oracle).
__device__ __forceinline__ void icp_seed(const IcpTrackArgs& ta, GnShared& g) {
  const Pose q = pose_inverse(pose_from12(ta.w2cInit));
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) g.c2w[r * 4 + c] = (double)q.R[r * 3 + c];
    g.c2w[r * 4 + 3] = (double)q.t[r];
  }
  for (int i = 0; i < 12; ++i) g.c2wInit[i] = g.c2w[i];
  c2w_to_float(g.c2w, g.c2wF);
  for (int i = 0; i < kIcpStats; ++i) g.stats[i] = 0.0;
  g.stats[7] = 1.0;
  for (int k = 0; k < kIcpSums; ++k) {
    g.sums[k] = 0.0;
    g.fixed[k] = 0;
  }
  g.failed = 0;
}
// The track as k_icp_coarse left it.
__device__ __forceinline__ void icp_seed_from_state(IcpState* st, GnShared& g) {
  for (int i = 0; i < 12; ++i) {
    g.c2w[i] = __ldcg(&st->c2w[i]);
    g.c2wInit[i] = __ldcg(&st->c2wInit[i]);
    g.c2wF[i] = __ldcg(&st->c2wF[i]);
  }
  for (int i = 0; i < kIcpStats; ++i) g.stats[i] = __ldcg(&st->stats[i]);
  for (int k = 0; k < kIcpSums; ++k) {
    g.sums[k] = __ldcg(&st->sums[k]);
    g.fixed[k] = __ldcg(&st->fixed[k]);
  }
  g.failed = __ldcg(&st->failed);
}

// The coarsest level on ONE thread-block cluster (kIcpCluster CTAs, one per
// SM of a GPC): the CTAs add their partial sums into CTA rank 0's shared
// memory over DSMEM (64-bit atomics: integer sums, order-free), a cluster
// barrier (~0.25 us) replaces the grid barrier (~1.2 us), and every CTA reads
// the totals from rank 0's shared memory.  The coarse level has few pixels
// (19,200 at 640x480), so 16 SMs hold it; its iterations are the most
// numerous of the track.  k_icp_track then continues from the state.
constexpr int kIcpCluster = 16;
__global__ void __launch_bounds__(kIcpThreads, RFG_ICP_CPS) k_icp_coarse(IcpState* st, IcpTrackArgs ta) {
  __shared__ long long sh[kIcpThreads / 32][32];
  __shared__ GnShared g;
  __shared__ float4 pcs[kIcpPx * kIcpThreads];
  __shared__ unsigned long long cacc[3][32];  // rank 0's are the cluster's accumulators
  cg::cluster_group cl = cg::this_cluster();
  const int l = ta.levels - 1;
  const IcpLevelArgs& a = ta.lv[l];
  if (threadIdx.x < 96) (&cacc[0][0])[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) {
    icp_seed(ta, g);
    for (int i = 0; i < 12; ++i) g.rp[i] = ta.renderPose[i];
    g.done = 0;
  }
  cl.sync();  // zeroed accumulators before any CTA adds into rank 0's
  const Intr inl{a.lw, a.lh, a.fx, a.fy, a.cx, a.cy};
  const float dist2 = a.dist * a.dist;
  const int n = a.lw * a.lh;
  const Pose rp = pose_from12(g.rp);
  const int nCta = (int)gridDim.x;
  const bool rank0 = cl.block_rank() == 0;
  const bool timed = rank0 && threadIdx.x == 0;
  unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool ok = true;
  for (int it = 0; it < a.iters && !g.done; ++it) {
    unsigned long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    if (timed) t0 = gtimer();
    unsigned long long* dst = cl.map_shared_rank(&cacc[it % 3][0], 0);
    ok &= icp_cta_eval(a, g, rp, inl, dist2, n, nCta, sh, pcs, it == 0, dst);
    if (rank0 && threadIdx.x < 32) cacc[(it + 1) % 3][threadIdx.x] = 0ull;  // read by no CTA since it - 2
    if (timed) t1 = gtimer();
    cl.sync();
    if (timed) t2 = gtimer();
    if (threadIdx.x < kIcpSums) {
      const long long v = (long long)dst[threadIdx.x];
      g.fixed[threadIdx.x] = v;
      g.sums[threadIdx.x] = ldexp((double)v, -icp_shift(threadIdx.x));
    }
    __syncthreads();
    if (timed) t3 = gtimer();
    if (threadIdx.x == 0)
      gn_step(g, a.level, a.minCount);
    else if (threadIdx.x == 32)
      icp_summary(g);
    __syncthreads();
    if (timed) {
      const unsigned long long t4 = gtimer();
      tacc[0] += t1 - t0;
      tacc[1] += t2 - t1;
      tacc[2] += t3 - t2;
      tacc[3] += t4 - t3;
      tacc[4] += 1;
      tacc[5 + (a.level < 3 ? a.level : 0)] += t4 - t0;
    }
  }
  if (!ok) st->error = 1;
  if (timed) {
    icp_publish(st, g, tacc, __ldcg(&st->gen), 0);  // the global accumulators were not used
    for (int i = 0; i < 12; ++i) st->c2wInit[i] = g.c2wInit[i];
    st->failed = g.failed;
  }
  cl.sync();  // rank 0's shared memory stays alive until every CTA has read it
}

#ifndef RFG_ICP_PREFETCH
#define RFG_ICP_PREFETCH 1  // render maps prefetched into L2 before the wait for the view kernel
#endif
__global__ void __launch_bounds__(kIcpThreads, RFG_ICP_CPS) k_icp_track(IcpState* st, IcpTrackArgs ta) {
  __shared__ long long sh[kIcpThreads / 32][32];
  __shared__ GnShared g;
  __shared__ float4 pcs[kIcpPx * kIcpThreads];
#if RFG_ICP_PREFETCH
  {
    // the render maps the association gathers from (the previous frame's
    // raycast, long complete) into L2 while the view kernel finishes: the
    // first evaluation of each level would otherwise wait on DRAM for them
    const IcpLevelArgs& l0 = ta.lv[0];
    const size_t lines = ((size_t)l0.rw * l0.rh * sizeof(float4)) >> 7;
    const char* pts = reinterpret_cast<const char*>(l0.points);
    const char* nrm = reinterpret_cast<const char*>(l0.normals);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < lines; i += (size_t)gridDim.x * blockDim.x) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pts + (i << 7)));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(nrm + (i << 7)));
    }
  }
#endif
  pdl_wait();  // the depth pyramid (programmatic dependency on the view kernel)
#ifdef RFG_ICP_PHASES
  const unsigned long long tEntry = gtimer();
#endif
  const unsigned gen = __ldcg(&st->gen);
  if (threadIdx.x == 0) {
    if (ta.fromState) {
      icp_seed_from_state(st, g);
    } else {
      icp_seed(ta, g);
    }
    for (int i = 0; i < 12; ++i) g.rp[i] = ta.renderPose[i];
  }
  __syncthreads();
  int gi = 0;
  unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int l = ta.levels - 1; l >= 0; --l) {
    if (g.failed) break;  // identical in every CTA
    if (ta.lv[l].iters <= 0) continue;
    if (threadIdx.x == 0) g.done = 0;
    __syncthreads();
    icp_run_level(st, ta.lv[l], ta.nCta[l], g, sh, pcs, gen, gi, tacc);
  }
  // every CTA read renderPose before its first grid barrier; with no
  // iteration at all (every level capped at 0) there was none, so one is
  // needed before CTA 0 may overwrite it below (gi is the same in every CTA)
  if (gi == 0 && ta.renderPoseOut) cg::this_grid().sync();
#ifdef RFG_ICP_PHASES
  // kernel entry -> exit of CTA 0 (replaces the per-level slots)
  tacc[5] = gtimer() - tEntry;
  tacc[6] = tacc[7] = 0;
#endif
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (g.failed) g.stats[3] = 0.0;
    icp_publish(st, g, tacc, gen, gi);
    for (int i = 0; i < 12; ++i) st->renderPose[i] = g.rp[i];
    if (g.failed || g.stats[0] == 0.0) {
      // never updated (or degenerate): the init pose itself
      for (int i = 0; i < 12; ++i) st->w2cF[i] = ta.w2cInit[i];
    } else {
      // world->camera output = inverse(c2w) (double) cast to float
      double R[9], t[3];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) R[r * 3 + c] = g.c2w[c * 4 + r];
      for (int r = 0; r < 3; ++r) t[r] = -(R[r * 3] * g.c2w[3] + (R[r * 3 + 1] * g.c2w[7] + R[r * 3 + 2] * g.c2w[11]));
      for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) st->w2cF[r * 4 + c] = (float)R[r * 3 + c];
        st->w2cF[r * 4 + 3] = (float)t[r];
      }
    }
    if (ta.w2cOut)
      for (int i = 0; i < 12; ++i) ta.w2cOut[i] = st->w2cF[i];
    // every CTA read renderPose before the first grid barrier, so it may be
    // overwritten now (the frame's maps are rendered at the output pose)
    if (ta.renderPoseOut)
      for (int i = 0; i < 12; ++i) ta.renderPoseOut[i] = st->w2cF[i];
  }
  pdl_trigger();  // the allocation (programmatic dependent) may launch
}

// CTAs for a level of n pixels: about one pixel per thread, at most one CTA
// per SM (co-residency for grid.sync).  Fixed per (device, level size).
static int icp_grid(int n) {
  static int fits[64] = {};  // per device: 1 fits one CTA per SM, -1 does not
  int dev = 0;
  cudaGetDevice(&dev);
  int f = dev < 64 ? fits[dev] : 0;
  if (!f) {
    int perSm = 0, perSmTrack = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm, k_icp_level, kIcpThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSmTrack, k_icp_track, kIcpThreads, 0);
    f = (perSm < 1 || perSmTrack < 1) ? -1 : 1;
    if (dev < 64) fits[dev] = f;
  }
  if (f < 0) return 0;
  const int sms = current_sm_count() * RFG_ICP_CPS;
  // every SM takes a part of every level (at least a warp of pixels per CTA):
  // spreading a coarse level over all SMs leaves fewer busy warps per SM for
  // the accumulation and the CTA reduction
  const int want = (n + 31) / 32;
  return want < 1 ? 1 : (want < sms ? want : sms);
}

size_t icp_state_bytes() { return sizeof(IcpState); }

#ifndef RFG_ICP_COARSE_CLUSTER
#define RFG_ICP_COARSE_CLUSTER 0  // 1: the coarsest level on one 16-CTA cluster (k_icp_coarse; measured slower)
#endif
// Whether a 16-CTA cluster of k_icp_coarse fits this device (one GPC with 16
// free SMs); cached per device.
static bool coarse_cluster_ok() {
  static int ok[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int v = dev < 64 ? ok[dev] : 0;
  if (!v) {
    v = -1;
    if (cudaFuncSetAttribute(k_icp_coarse, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kIcpCluster);
      cfg.blockDim = dim3(kIcpThreads);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kIcpCluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_icp_coarse, &cfg) == cudaSuccess && n >= 1) v = 1;
    }
    cudaGetLastError();
    if (dev < 64) ok[dev] = v;
  }
  return v > 0;
}

static IcpLevelArgs level_args(const float* depthLevels, int level, const Intr& in0, const float4* points,
                               const float4* normals) {
  IcpLevelArgs a{};
  size_t off = 0;
  for (int l = 0; l < level; ++l) off += (size_t)(in0.w >> l) * (in0.h >> l);
  const float sc = ldexpf(1.f, -level);
  a.depth = depthLevels + off;
  a.lw = in0.w >> level;
  a.lh = in0.h >> level;
  a.fx = in0.fx * sc;
  a.fy = in0.fy * sc;
  a.cx = in0.cx * sc;
  a.cy = in0.cy * sc;
  a.points = points;
  a.normals = normals;
  a.rw = in0.w;
  a.rh = in0.h;
  a.rfx = in0.fx;
  a.rfy = in0.fy;
  a.rcx = in0.cx;
  a.rcy = in0.cy;
  a.level = level;
  return a;
}

// Enqueue a complete coarse-to-fine track: init from (w2c, renderPose) device
// pointers, ONE cooperative launch, final pose to w2cOut (device).
cudaError_t launch_icp_track(void* state, const float* depthLevels, int levels, const Intr& in0,
                             const float4* points, const float4* normals, const int* iters, const float* dist,
                             int minCount, const float* w2cInit, const float* renderPose, float* w2cOut,
                             float* renderPoseOut, cudaStream_t s) {
  IcpState* st = static_cast<IcpState*>(state);
  IcpTrackArgs ta{};
  ta.renderPoseOut = renderPoseOut;
  ta.levels = levels;
  ta.w2cInit = w2cInit;
  ta.renderPose = renderPose;
  ta.w2cOut = w2cOut;
  int grid = 1;
  for (int l = 0; l < levels; ++l) {
    ta.lv[l] = level_args(depthLevels, l, in0, points, normals);
    ta.lv[l].dist = dist[l];
    ta.lv[l].iters = iters[l];
    ta.lv[l].minCount = minCount;
    ta.lv[l].evalOnly = 0;
    ta.nCta[l] = icp_grid(ta.lv[l].lw * ta.lv[l].lh);
    if (ta.nCta[l] <= 0) return cudaErrorCooperativeLaunchTooLarge;
    if (iters[l] > 0 && ta.nCta[l] > grid) grid = ta.nCta[l];
  }
  IcpState* stp = st;
  const int lc = levels - 1;
  if (RFG_ICP_COARSE_CLUSTER && levels >= 2 && iters[lc] > 0 && coarse_cluster_ok()) {
    // the coarsest level on one cluster, then the rest of the track
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kIcpCluster);
    cfg.blockDim = dim3(kIcpThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kIcpCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    count_launch();
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_icp_coarse, stp, ta);
    if (e != cudaSuccess) return e;
    ta.fromState = 1;
    ta.lv[lc].iters = 0;
    grid = 1;
    for (int l = 0; l < lc; ++l)
      if (iters[l] > 0 && ta.nCta[l] > grid) grid = ta.nCta[l];
  }
  void* args[] = {&stp, &ta};
  count_launch();
  if (!g_pdl) return cudaLaunchCooperativeKernel((const void*)k_icp_track, dim3(grid), dim3(kIcpThreads), args, 0, s);
  // a cooperative launch that is also a programmatic dependent of the view kernel
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kIcpThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_icp_track, stp, ta);
}

__global__ void k_icp_set_c2w(IcpState* st, const float* c2w, const float* renderPose) {
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 12; ++i) {
    st->c2wF[i] = c2w[i];
    st->c2w[i] = c2w[i];
    st->renderPose[i] = renderPose[i];
  }
  for (int i = 0; i < 4; ++i) st->done[i] = 0;
}

cudaError_t launch_icp_reduce_once(void* state, const float* depth, int lw, int lh, const float* f4l, const Intr& in0,
                                   const float4* points, const float4* normals, const float* c2w,
                                   const float* renderPose, float dist, cudaStream_t s) {
  IcpState* st = static_cast<IcpState*>(state);
  k_icp_set_c2w<<<1, 32, 0, s>>>(st, c2w, renderPose);
  count_launch();
  IcpLevelArgs a = level_args(depth, 0, in0, points, normals);
  a.depth = depth;
  a.lw = lw;
  a.lh = lh;
  a.fx = f4l[0];
  a.fy = f4l[1];
  a.cx = f4l[2];
  a.cy = f4l[3];
  a.dist = dist;
  a.level = 3;
  a.iters = 1;
  a.minCount = 0;
  a.evalOnly = 1;
  const int grid = icp_grid(a.lw * a.lh);
  if (grid <= 0) return cudaErrorCooperativeLaunchTooLarge;
  IcpState* stp = st;
  void* args[] = {&stp, &a};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)k_icp_level, dim3(grid), dim3(kIcpThreads), args, 0, s);
}

// Device queries the launches need, made outside any stream capture.
void icp_warmup() {
  coarse_cluster_ok();
  icp_grid(1);
}

unsigned long long* icp_timers_ptr(void* state) { return static_cast<IcpState*>(state)->timers; }
const double* icp_sums_ptr(void* state) { return static_cast<IcpState*>(state)->sums; }
const long long* icp_fixed_ptr(void* state) { return static_cast<IcpState*>(state)->fixed; }
const double* icp_stats_ptr(void* state) { return static_cast<IcpState*>(state)->stats; }
const int* icp_error_ptr(void* state) { return &static_cast<IcpState*>(state)->error; }
const float* icp_w2c_ptr(void* state) { return static_cast<IcpState*>(state)->w2cF; }

}  // namespace rfg

#ifdef RFG_ICP_SUB
extern "C" int rfg_debug_icp_sub(unsigned long long* out24, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out24, rfg::g_icp_sub, sizeof(rfg::g_icp_sub));
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(rfg::g_icp_sub, z, sizeof(z));
  }
  return 0;
}
#endif
