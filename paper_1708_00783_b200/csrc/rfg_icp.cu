// rfg_icp.cu — point-to-plane ICP depth tracker (ITMDepthTracker).
//
// The reference has no tracker; the algorithm is restated
// from SPEC.md:348-356,390-395 and fixed by the CPU oracle
// oracle/rfo.c:rfo_icp_track.
//
// One cooperative kernel per pyramid level runs that level's whole
// Gauss-Newton loop on the device.  Per iteration:
//   reduce  — every valid pyramid pixel is backprojected, moved to the world
//             by the current estimate, projected into the last ICP-map render
//             (nearest pixel) and, if associated and within the level's
//             distance gate, adds J J^T (21), J r (6), r^2 and 1 to double
//             accumulators; warp-shuffle tree + shared-memory reduction to one
//             partial per CTA (partials double-buffered by iteration parity);
//   grid.sync();
//   solve   — EVERY CTA sums all partials in the same fixed order and runs
//             the same Cholesky solve and SE(3) update, so all CTAs hold the
//             identical new estimate without a second grid barrier; CTA 0
//             publishes it (pose, stats, done flag) to global memory.
// A frame's whole tracker is ONE cooperative launch (k_icp_track: seed,
// levels coarse to fine, output pose) with one grid barrier per iteration;
// nothing is enqueued for iterations that are not needed, and the launch is
// capturable in the frame's CUDA graph.  The
// grid size is fixed per level, so the reduction order — and the result — is
// run-to-run deterministic.
#include <cooperative_groups.h>

#include "rfg_common.cuh"

namespace cg = cooperative_groups;

namespace rfg {

constexpr int kIcpThreads = 512;
constexpr int kIcpMaxCtas = 512;

// Device tracking state (rfg_map::icpOut).
struct IcpState {
  double c2w[12];       // current camera->world estimate (row-major 3x4)
  double sums[29];      // last evaluation
  double stats[8];      // {iterations, count, E, converged, it_l0, it_l1, it_l2, ok}
  float c2wF[12];       // float cast of c2w
  float w2cF[12];       // tracked world->camera (output pose)
  float renderPose[12]; // world->camera of the render being tracked against
  int done[4];          // per-level stop flags
  int pad[4];
  // phase timers of CTA 0 (ns, %globaltimer), accumulated over iterations:
  // {associate+reduce, grid barrier, final sum, solve, iterations,
  //  level-0 total, level-1 total, level-2 total}
  unsigned long long timers[8];
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

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
  double sums[29];
  double stats[8];
  float c2wF[12];
  float rp[12];
  int done;
};

// double-precision SE(3) (proj/include/rf/pose.hpp:45-60 with S = double)
// (all small-matrix loops are fully unrolled so the solver state stays in
// registers instead of local memory)
__device__ __forceinline__ void matmul3d(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C[r * 3 + c] = A[r * 3 + 0] * B[c] + (A[r * 3 + 1] * B[3 + c] + A[r * 3 + 2] * B[6 + c]);
}

__device__ void c2w_to_float(const double* c, float* f) {
  for (int i = 0; i < 12; ++i) f[i] = (float)c[i];
}

// Load an explicit float camera->world pose (single evaluations).
__global__ void k_icp_set_c2w(IcpState* st, const float* c2w, const float* renderPose) {
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 12; ++i) {
    st->c2wF[i] = c2w[i];
    st->c2w[i] = c2w[i];
    st->renderPose[i] = renderPose[i];
  }
  for (int i = 0; i < 4; ++i) st->done[i] = 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// 1/sqrt(s) for s > 0: MUFU seed + two Newton steps (within ~1 ulp of the
// correctly rounded value).  Inline, unlike the IEEE sqrt/rcp, whose
// out-of-line slow paths made ptxas spill the whole factorisation.
__device__ __forceinline__ double rsqrt_nr(double s) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double e = __fma_rn(-__dmul_rn(s, r), r, 1.0);  // 1 - s r^2
    r = __fma_rn(__dmul_rn(r, 0.5), e, r);
  }
  return r;
}

// Cholesky solve (same operation order as oracle/rfo.c:rfo_solve6; the
// pivot's 1/sqrt comes from rsqrt_nr, so the solution agrees with the oracle
// to rounding — the tracker's pose tolerance is 1e-5).
__device__ __forceinline__ int solve6(const double* acc, double* x) {
  // every loop has constant bounds (guards instead of j-dependent limits) so
  // the whole factorisation unrolls into registers
  double A[36];
  int k = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b) {
      A[a * 6 + b] = acc[k];
      A[b * 6 + a] = acc[k];
      ++k;
    }
  double L[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  // no early exits either: a non-positive pivot raises `bad`, is replaced by
  // 1 so the rest stays finite, and the solve reports failure at the end
  double inv[6];
  double det = 1.0;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double s = A[j * 6 + j];
#pragma unroll
    for (int p = 0; p < 6; ++p)
      if (p < j) s -= L[j * 6 + p] * L[j * 6 + p];
    if (!(s > 0.0)) {
      bad = true;
      s = 1.0;
    }
    det *= s;
    inv[j] = rsqrt_nr(s);
    L[j * 6 + j] = s * inv[j];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      if (i > j) {
        double t = A[i * 6 + j];
#pragma unroll
        for (int p = 0; p < 6; ++p)
          if (p < j) t -= L[i * 6 + p] * L[j * 6 + p];
        L[i * 6 + j] = t * inv[j];
      }
    }
  }
  bad = bad || det < 1e-12;
  double yv[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double t = -acc[21 + i];
#pragma unroll
    for (int p = 0; p < 6; ++p)
      if (p < i) t -= L[i * 6 + p] * yv[p];
    yv[i] = t * inv[i];
  }
  double xv[6];
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double t = yv[i];
#pragma unroll
    for (int p = 0; p < 6; ++p)
      if (p > i) t -= L[p * 6 + i] * xv[p];
    xv[i] = t * inv[i];
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = xv[i];
  return bad ? -1 : 0;
}

// One Gauss-Newton step on the CTA-local state (oracle: rfo_icp_track loop
// body): count gate, Cholesky solve, T_cw <- exp(delta) T_cw, convergence.
__device__ void gn_step(GnShared& g, int level, int minCount) {
  g.stats[1] = g.sums[28];
  g.stats[2] = g.sums[27];
  if (g.sums[28] < (double)minCount) {
    g.stats[7] = 0.0;
    g.done = 1;
    return;
  }
  double delta[6];
  if (solve6(g.sums, delta) != 0) {
    g.stats[7] = 0.0;
    g.done = 1;
    return;
  }
  const double* w = delta;
  const double* v = delta + 3;
  const double th2 = w[0] * w[0] + (w[1] * w[1] + w[2] * w[2]);
  const double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double WW[9];
  matmul3d(W, W, WW);
  double ca, cb, cc;
  if (th2 < 0.0625 * 0.0625) {
    // sin(t)/t, (1 - cos t)/t^2, (t - sin t)/t^3 by their Taylor series
    // (nested to t^10; the truncation error is below 1e-19 for t < 1/16):
    // no sincos, no divisions on the solver's serial path, and no
    // cancellation in 1 - cos t and t - sin t at small angles
    const double t2 = th2;
    ca = 1.0 - t2 * (1.0 / 6.0) * (1.0 - t2 * (1.0 / 20.0) * (1.0 - t2 * (1.0 / 42.0) * (1.0 - t2 * (1.0 / 72.0) * (1.0 - t2 * (1.0 / 110.0)))));
    cb = 0.5 * (1.0 - t2 * (1.0 / 12.0) * (1.0 - t2 * (1.0 / 30.0) * (1.0 - t2 * (1.0 / 56.0) * (1.0 - t2 * (1.0 / 90.0) * (1.0 - t2 * (1.0 / 132.0))))));
    cc = (1.0 / 6.0) * (1.0 - t2 * (1.0 / 20.0) * (1.0 - t2 * (1.0 / 42.0) * (1.0 - t2 * (1.0 / 72.0) * (1.0 - t2 * (1.0 / 110.0) * (1.0 - t2 * (1.0 / 156.0))))));
  } else {
    const double theta = sqrt(th2);
    double s, co;
    sincos(theta, &s, &co);
    ca = s / theta;
    cb = (1.0 - co) / (theta * theta);
    cc = (theta - s) / (theta * theta * theta);
  }
  double ER[9], V[9], Et[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double I = (i % 4 == 0) ? 1.0 : 0.0;
    ER[i] = I + ca * W[i] + cb * WW[i];
    V[i] = I + cb * W[i] + cc * WW[i];
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
  g.stats[0] += 1.0;
  g.stats[4 + level] += 1.0;
  const double nrm = sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2] + delta[3] * delta[3] +
                          delta[4] * delta[4] + delta[5] * delta[5]);
  if (nrm < 1e-4) {
    g.stats[3] = 1.0;
    g.done = 1;
  }
}

// One evaluation's per-CTA partial: every valid level pixel p (grid stride)
// is associated and accumulated in double (J J^T, J r, r^2, count), reduced
// per warp by recursive halving and over the CTA's warps; on return thread k
// < 29 of the CTA holds sum k of its pixels (returned), the others 0.
// Pixels per thread whose camera-space point is kept in shared memory for
// the whole level (computed at the level's first iteration; the depth and the
// backprojection do not depend on the pose).  Level 0 at 640x480 on 148 CTAs
// is 4.05 pixels per thread; pixels beyond the cached slots take the
// uncached path.  Projection + gathers are issued kIcpGroup pixels at a
// time so their loads are in flight together; pixels are accumulated in
// the same order as a plain loop, so the sums do not depend on kIcpGroup.
constexpr int kIcpPxCache = 4;
constexpr int kIcpGroup = 2;  // 1 and 4 measured no faster

// J J^T, J r, r^2, count of one associated pixel (the oracle's per-pixel
// body, rfo_icp_track).
__device__ __forceinline__ void icp_accumulate(double* acc, f3 pw, float4 V, float4 N, float dist2) {
  if (!(V.w > 0.f) || !(N.w > 0.f)) return;
  const f3 diff{pw.x - V.x, pw.y - V.y, pw.z - V.z};
  if (sqnorm3(diff) > dist2) return;
  const f3 nn{N.x, N.y, N.z};
  const float r = dot3(diff, nn);
  const f3 pxn = cross3(pw, nn);
  const double J[6] = {pxn.x, pxn.y, pxn.z, nn.x, nn.y, nn.z};
  const double rd = r;
  int k = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i; j < 6; ++j) acc[k++] += J[i] * J[j];
#pragma unroll
  for (int i = 0; i < 6; ++i) acc[21 + i] += J[i] * rd;
  acc[27] += rd * rd;
  acc[28] += 1.0;
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

// One evaluation's per-CTA partial: every valid level pixel p (grid stride)
// is associated and accumulated in double (J J^T, J r, r^2, count), reduced
// per warp by recursive halving and over the CTA's warps; on return thread k
// < 29 of the CTA holds sum k of its pixels (returned), the others 0.
__device__ __forceinline__ double icp_cta_partial(const IcpLevelArgs& a, const GnShared& g, const Pose& rp,
                                                  const Intr& inl, float dist2, int n, int p0, int pstride,
                                                  double (*sh)[29], float4* pcs, bool fill) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double out = 0.0;
  const Pose c2w = pose_from12(g.c2wF);
  double acc[29];
#pragma unroll
  for (int k = 0; k < 29; ++k) acc[k] = 0.0;
  if (fill) {
#pragma unroll
    for (int k = 0; k < kIcpPxCache; ++k) {
      const int p = p0 + k * pstride;
      float4 c = make_float4(0.f, 0.f, 0.f, -1.f);
      if (p < n) {
        const float d = __ldg(a.depth + p);
        if (d > 0.f) {
          const int x = p % a.lw, y = p / a.lw;
          const f3 pc = backproject(inl, (float)x, (float)y, d);
          c = make_float4(pc.x, pc.y, pc.z, 1.f);
        }
      }
      pcs[k * kIcpThreads + threadIdx.x] = c;  // each thread reads back only its own slots
    }
  }
#pragma unroll
  for (int kb = 0; kb < kIcpPxCache; kb += kIcpGroup) {
    f3 pw[kIcpGroup];
    int pix[kIcpGroup];
#pragma unroll
    for (int j = 0; j < kIcpGroup; ++j) {
      const float4 c = pcs[(kb + j) * kIcpThreads + threadIdx.x];
      pix[j] = -1;
      pw[j] = f3{0.f, 0.f, 0.f};
      if (c.w > 0.f) {
        pw[j] = pose_apply(c2w, f3{c.x, c.y, c.z});
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
      if (pix[j] >= 0) icp_accumulate(acc, pw[j], V[j], N[j], dist2);
  }
  // pixels beyond the cached slots
  for (int p = p0 + kIcpPxCache * pstride; p < n; p += pstride) {
    const float d = __ldg(a.depth + p);
    if (!(d > 0.f)) continue;
    const int x = p % a.lw, y = p / a.lw;
    const f3 pc = backproject(inl, (float)x, (float)y, d);
    const f3 pw = pose_apply(c2w, pc);
    const int pix = icp_associate(a, rp, pw);
    if (pix < 0) continue;
    icp_accumulate(acc, pw, __ldg(a.points + pix), __ldg(a.normals + pix), dist2);
  }
  {
    // multi-value warp reduction by recursive halving: at offset o every
    // lane keeps one half of its live values and sends the other half to
    // lane^o, so 32 (29 + 3 zero) sums take 16+8+4+2+1 = 31 shuffles
    // instead of 29 x 5.  Lane l ends with sum number l.
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = k < 29 ? acc[k] : 0.0;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < o; ++i) {
        const double send = hi ? v[i] : v[i + o];
        const double keep = hi ? v[i + o] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if (lane < 29) sh[wid][lane] = v[0];
  }
  __syncthreads();
  if (threadIdx.x < 29) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kIcpThreads / 32; ++w) s += sh[w][threadIdx.x];
    out = s;
  }
  return out;
}

// One level's Gauss-Newton loop on the CTA-local state g.  CTAs with
// blockIdx.x < nCta own the level's pixels (grid stride nCta x kIcpThreads);
// the others only join the barriers, sum the same partials and run the same
// solve.  `gi` counts iterations across levels so the partial buffers
// alternate without a second barrier.
__device__ __forceinline__ void icp_run_level(const IcpLevelArgs& a, double* partials, int nCta, GnShared& g,
                                              double (*sh)[29], float4* pcs, int& gi, unsigned long long* tacc) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
    double* part = partials + (size_t)(gi & 1) * kIcpMaxCtas * 29;
    if (owner) {
      const double ps = icp_cta_partial(a, g, rp, inl, dist2, n, blockIdx.x * blockDim.x + threadIdx.x,
                                        nCta * blockDim.x, sh, pcs, it == 0);
      if (threadIdx.x < 29) part[threadIdx.x * kIcpMaxCtas + blockIdx.x] = ps;  // [sum][cta]: coalesced final sum
    }
    if (timed) t1 = gtimer();
    grid.sync();
    if (timed) t2 = gtimer();
    // every CTA: fixed-order final sum over the owners (warp w owns sums w,
    // w+16; lanes stride the CTAs; shuffle tree) and the identical solve
    for (int k = wid; k < 29; k += kIcpThreads / 32) {
      // issue all of this lane's loads before the dependent adds
      double v[kIcpMaxCtas / 32];
#pragma unroll
      for (int j = 0; j < kIcpMaxCtas / 32; ++j) {
        const int c = lane + 32 * j;
        v[j] = c < nCta ? __ldcg(part + k * kIcpMaxCtas + c) : 0.0;
      }
      double sum = 0.0;
#pragma unroll
      for (int j = 0; j < kIcpMaxCtas / 32; ++j) sum += v[j];
      sum = warp_sum(sum);
      if (lane == 0) g.sums[k] = sum;
    }
    __syncthreads();
    if (timed) t3 = gtimer();
    if (threadIdx.x == 0) {
      if (a.evalOnly)
        g.done = 1;
      else
        gn_step(g, a.level, a.minCount);
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

__device__ __forceinline__ void icp_publish(IcpState* st, const GnShared& g, const unsigned long long* tacc) {
#pragma unroll
  for (int i = 0; i < 8; ++i) st->timers[i] += tacc[i];
  for (int i = 0; i < 12; ++i) {
    st->c2w[i] = g.c2w[i];
    st->c2wF[i] = g.c2wF[i];
  }
  for (int k = 0; k < 29; ++k) st->sums[k] = g.sums[k];
  for (int i = 0; i < 8; ++i) st->stats[i] = g.stats[i];
}

// Single evaluation / single level on the state in `st` (rfg_icp_reduce).
__global__ void __launch_bounds__(kIcpThreads) k_icp_level(IcpState* st, IcpLevelArgs a, double* partials) {
  __shared__ double sh[kIcpThreads / 32][29];
  __shared__ GnShared g;
  __shared__ float4 pcs[kIcpPxCache * kIcpThreads];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) {
      g.c2w[i] = __ldcg(&st->c2w[i]);
      g.c2wF[i] = __ldcg(&st->c2wF[i]);
      g.rp[i] = __ldcg(&st->renderPose[i]);
    }
    for (int i = 0; i < 8; ++i) g.stats[i] = __ldcg(&st->stats[i]);
    g.done = __ldcg(&st->done[a.level]);
  }
  __syncthreads();
  int gi = 0;
  unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  icp_run_level(a, partials, gridDim.x, g, sh, pcs, gi, tacc);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    icp_publish(st, g, tacc);
    st->done[a.level] = g.done;
  }
}

// The whole coarse-to-fine track of a frame in ONE cooperative launch
// (k_icp_init + a launch per level + k_icp_final before): every CTA seeds
// its state from the device-resident pose, runs the levels coarse to fine
// with the same per-level pixel partition as a per-level launch (so the sums
// and the pose are identical), and CTA 0 publishes the result.
struct IcpTrackArgs {
  IcpLevelArgs lv[3];
  int nCta[3];
  int levels;
  const float* w2cInit;
  const float* renderPose;
  float* w2cOut;
  float* renderPoseOut;  // nullable: the next frame's render pose := the output pose
};

__global__ void __launch_bounds__(kIcpThreads) k_icp_track(IcpState* st, IcpTrackArgs ta, double* partials) {
  __shared__ double sh[kIcpThreads / 32][29];
  __shared__ GnShared g;
  __shared__ float4 pcs[kIcpPxCache * kIcpThreads];
#ifdef RFG_ICP_PHASES
  const unsigned long long tEntry = gtimer();
#endif
  if (threadIdx.x == 0) {
    // k_icp_init: inverse of the float pose, widened to double (as the oracle)
    const Pose q = pose_inverse(pose_from12(ta.w2cInit));
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) g.c2w[r * 4 + c] = (double)q.R[r * 3 + c];
      g.c2w[r * 4 + 3] = (double)q.t[r];
    }
    c2w_to_float(g.c2w, g.c2wF);
    for (int i = 0; i < 12; ++i) g.rp[i] = ta.renderPose[i];
    for (int i = 0; i < 8; ++i) g.stats[i] = 0.0;
    g.stats[7] = 1.0;
    for (int k = 0; k < 29; ++k) g.sums[k] = 0.0;
  }
  __syncthreads();
  int gi = 0;
  unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int l = ta.levels - 1; l >= 0; --l) {
    if (ta.lv[l].iters <= 0) continue;
    if (threadIdx.x == 0) g.done = 0;
    __syncthreads();
    icp_run_level(ta.lv[l], partials, ta.nCta[l], g, sh, pcs, gi, tacc);
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
    icp_publish(st, g, tacc);
    for (int i = 0; i < 12; ++i) st->renderPose[i] = g.rp[i];
    // k_icp_final: world->camera output = inverse(c2w) cast to float
    double R[9], t[3];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) R[r * 3 + c] = g.c2w[c * 4 + r];
    for (int r = 0; r < 3; ++r) t[r] = -(R[r * 3] * g.c2w[3] + (R[r * 3 + 1] * g.c2w[7] + R[r * 3 + 2] * g.c2w[11]));
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) st->w2cF[r * 4 + c] = (float)R[r * 3 + c];
      st->w2cF[r * 4 + 3] = (float)t[r];
    }
    if (ta.w2cOut)
      for (int i = 0; i < 12; ++i) ta.w2cOut[i] = st->w2cF[i];
    // every CTA read renderPose before the first grid barrier, so it may be
    // overwritten now (the frame's maps are rendered at the output pose)
    if (ta.renderPoseOut)
      for (int i = 0; i < 12; ++i) ta.renderPoseOut[i] = st->w2cF[i];
  }
}

// CTAs for a level of n pixels: about one pixel per thread, at most one CTA
// per SM (co-residency for grid.sync).  Fixed per (device, level size).
static int icp_grid(int n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0, perSm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm, k_icp_level, kIcpThreads, 0);
    int perSmTrack = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSmTrack, k_icp_track, kIcpThreads, 0);
    if (perSm < 1 || perSmTrack < 1) sms = -1;
  }
  if (sms <= 0) return 0;
  const int want = (n + kIcpThreads - 1) / kIcpThreads;
  return want < 1 ? 1 : (want < sms ? want : sms);
}

size_t icp_state_bytes() { return sizeof(IcpState); }
int icp_partial_slots() { return 2 * kIcpMaxCtas; }

static cudaError_t launch_level(IcpState* st, const IcpLevelArgs& a, double* partials, cudaStream_t s) {
  const int grid = icp_grid(a.lw * a.lh);
  if (grid <= 0) return cudaErrorCooperativeLaunchTooLarge;
  IcpState* stp = st;
  IcpLevelArgs ap = a;
  double* pp = partials;
  void* args[] = {&stp, &ap, &pp};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)k_icp_level, dim3(grid), dim3(kIcpThreads), args, 0, s);
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
// pointers, one cooperative launch per level, final pose to w2cOut (device).
cudaError_t launch_icp_track(void* state, double* partials, const float* depthLevels, int levels, const Intr& in0,
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
  double* pp = partials;
  void* args[] = {&stp, &ta, &pp};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)k_icp_track, dim3(grid), dim3(kIcpThreads), args, 0, s);
}

cudaError_t launch_icp_reduce_once(void* state, double* partials, const float* depth, int lw, int lh, const float* f4l,
                                   const Intr& in0, const float4* points, const float4* normals, const float* c2w,
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
  return launch_level(st, a, partials, s);
}

unsigned long long* icp_timers_ptr(void* state) { return static_cast<IcpState*>(state)->timers; }
const double* icp_sums_ptr(void* state) { return static_cast<IcpState*>(state)->sums; }
const double* icp_stats_ptr(void* state) { return static_cast<IcpState*>(state)->stats; }
const float* icp_w2c_ptr(void* state) { return static_cast<IcpState*>(state)->w2cF; }

}  // namespace rfg
