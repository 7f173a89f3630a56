#include <cstdio>
#define REP(op) _Pragma("unroll 1") for (int i = 0; i < 125; ++i) { op; op; op; op; op; op; op; op; }
__global__ void k(double* io, unsigned long long* out) {
  double x = io[0], y = io[1];
  float f = (float)x, g = (float)y;
  unsigned long long t[8];
  REP(f = __fadd_rn(f, g));  // warm-up
  t[0] = clock64();
  REP(x = __dadd_rn(x, y));
  t[1] = clock64();
  REP(x = __dmul_rn(x, y));
  t[2] = clock64();
  REP(x = __drcp_rn(x));
  t[3] = clock64();
  REP(f = __fadd_rn(f, g));
  t[4] = clock64();
  REP(x = __ddiv_rn(x, y));
  t[5] = clock64();
  REP(x = __fma_rn(x, y, y));
  t[6] = clock64();
  io[2] = x + f;
  for (int i = 0; i < 6; ++i) out[i] = t[i + 1] - t[i];
}
int main() {
  double* io; unsigned long long* o;
  cudaMallocManaged(&io, 32); cudaMallocManaged(&o, 64);
  io[0] = 1.0; io[1] = 1.0000001;
  k<<<1, 1>>>(io, o); cudaDeviceSynchronize();
  std::printf("dependent-chain cycles per op: dadd %.1f dmul %.1f drcp %.1f fadd %.1f ddiv %.1f dfma %.1f\n",
              o[0] / 1000.0, o[1] / 1000.0, o[2] / 1000.0, o[3] / 1000.0, o[4] / 1000.0, o[5] / 1000.0);
}
