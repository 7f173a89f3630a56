// Launch overhead: empty kernel, normal vs cooperative, stream vs CUDA graph.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
__global__ void k_empty(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 100000) *p = 1; }
__global__ void k_sync(int* p) { cooperative_groups::this_grid().sync(); if (p && threadIdx.x == 0 && blockIdx.x == 100000) *p = 1; }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int* p = nullptr; void* args[] = {&p};
  const int N = 200;
  for (int mode = 0; mode < 6; ++mode) {
    auto enqueue = [&]() {
      for (int i = 0; i < N; ++i) {
        if (mode % 3 == 0) k_empty<<<148, 1024, 0, s>>>(p);
        else if (mode % 3 == 1) cudaLaunchCooperativeKernel((void*)k_empty, 148, 1024, args, 0, s);
        else cudaLaunchCooperativeKernel((void*)k_sync, 148, 1024, args, 0, s);
      }
    };
    float ms = 0;
    if (mode < 3) {
      enqueue(); cudaStreamSynchronize(s);
      cudaEventRecord(a, s); enqueue(); cudaEventRecord(b, s); cudaEventSynchronize(b);
    } else {
      cudaGraph_t g; cudaGraphExec_t e;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal); enqueue(); cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&e, g, 0); cudaGraphLaunch(e, s); cudaStreamSynchronize(s);
      cudaEventRecord(a, s); cudaGraphLaunch(e, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    const char* names[] = {"normal", "cooperative", "cooperative+grid.sync"};
    printf("%s %-24s %.2f us per launch (%s)\n", mode < 3 ? "stream" : "graph ", names[mode % 3], ms * 1e3 / N,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
