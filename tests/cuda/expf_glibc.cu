// rfg_view.cu:expf_glibc against the host C library's expf, bit for bit:
// every float in [-110, 0] (all arguments the bilateral filter can produce
// that do not flush to 0 — it only evaluates exp of non-positive numbers), a
// strided sweep of (0, 89] and the special values.  The reference calls
// std::exp(float) = glibc expf; on x86-64 hosts with FMA glibc selects the
// FMA variant, which is the sequence expf_glibc reproduces.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../paper_1708_00783_b200/csrc/rfg_expf.cuh"

__global__ void k_eval(const uint32_t* in, uint32_t* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = __float_as_uint(rfg::expf_glibc(__uint_as_float(in[i])));
}

static uint32_t bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}
static float flt(uint32_t u) {
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

int main() {
  std::vector<uint32_t> args;
  const uint32_t lo = bits(-0.0f), hi = bits(-110.0f);  // negative floats grow in bits with magnitude
  const size_t chunk = 1u << 26;
  uint32_t *dIn, *dOut;
  cudaMalloc(&dIn, chunk * 4);
  cudaMalloc(&dOut, chunk * 4);
  std::vector<uint32_t> hIn(chunk), hOut(chunk);
  unsigned long long checked = 0, bad = 0;
  auto run = [&](size_t n) {
    cudaMemcpy(dIn, hIn.data(), n * 4, cudaMemcpyHostToDevice);
    k_eval<<<148 * 8, 256>>>(dIn, dOut, n);
    cudaMemcpy(hOut.data(), dOut, n * 4, cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < n; ++i) {
      const uint32_t want = bits(std::exp(flt(hIn[i])));
      if (hOut[i] != want) {
        if (bad < 5) std::printf("mismatch x=%a host=%08x gpu=%08x\n", flt(hIn[i]), want, hOut[i]);
        ++bad;
      }
    }
    checked += n;
  };
  size_t n = 0;
  for (uint64_t u = lo; u <= hi; ++u) {
    hIn[n++] = (uint32_t)u;
    if (n == chunk) {
      run(n);
      n = 0;
    }
  }
  // positive side (strided) and the special values
  for (uint32_t u = bits(0x1p-149f); u <= bits(89.0f); u += 97) {
    hIn[n++] = u;
    if (n == chunk) {
      run(n);
      n = 0;
    }
  }
  const float specials[] = {0.0f, -0.0f, INFINITY, -INFINITY, NAN, -103.97f, -103.972f, -103.28f, -103.279f,
                            -0x1.9fe368p6f, -0x1.9d1d9ep6f, 0x1.62e42ep6f, 0x1.62e430p6f, -87.9f, -88.0f, -88.1f};
  for (float f : specials) hIn[n++] = bits(f);
  for (uint32_t nan : {0x7fc00000u, 0xffc00000u, 0x7f800001u, 0xff812345u, 0x7fa5a5a5u}) hIn[n++] = nan;
  run(n);
  std::printf("checked %llu  mismatches %llu\n", checked, bad);
  return bad ? 1 : 0;
}
