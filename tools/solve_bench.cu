// Latency of the tracker's per-iteration solve (rfg_icp.cu:gn_step) on one
// thread, in clock cycles: LDL^T + substitution + SE(3) update, timed with
// clock64 over repeated calls on the same SPD system (tools only).
#include <cstdio>
#include "../paper_1708_00783_b200/csrc/rfg_icp.cu"
namespace rfg {
std::atomic<uint64_t> g_launches{0};
int current_sm_count() { return 148; }
}  // namespace rfg

__global__ void k_bench(const double* sums, unsigned long long* out, int reps) {
  __shared__ rfg::GnShared g;
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 12; ++i) g.c2w[i] = (i % 5 == 0) ? 1.0 : 0.0;
  for (int k = 0; k < 31; ++k) g.sums[k] = sums[k];
  for (int i = 0; i < 12; ++i) g.stats[i] = 0.0;
  unsigned long long best = ~0ull;
  for (int r = 0; r < reps; ++r) {
    g.done = 0;
    g.failed = 0;
    __threadfence_block();
    const unsigned long long t0 = clock64();
    rfg::gn_step(g, 0, 10);
    __threadfence_block();
    const unsigned long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  out[0] = best;
  out[1] = (unsigned long long)(g.c2w[3] * 1e9);
}

int main() {
  // an SPD system like the tracker's: H = J^T J over random J, n = 1e5
  double h[31] = {0};
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (double)(s >> 8) / (1 << 24) - 0.5; };
  for (int p = 0; p < 2000; ++p) {
    double J[6];
    for (int i = 0; i < 6; ++i) J[i] = rnd();
    double r = 1e-3 * rnd();
    int k = 0;
    for (int i = 0; i < 6; ++i)
      for (int j = i; j < 6; ++j) h[k++] += J[i] * J[j];
    for (int i = 0; i < 6; ++i) h[21 + i] += J[i] * r;
    h[28] += 1.0;
  }
  double* d;
  unsigned long long* o;
  cudaMalloc(&d, sizeof(h));
  cudaMallocManaged(&o, 16);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  k_bench<<<1, 32>>>(d, o, 50);
  cudaDeviceSynchronize();
  std::printf("gn_step: %llu cycles (best of 50)  [%llu]\n", o[0], o[1]);
  return 0;
}
