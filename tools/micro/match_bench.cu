// Throughput of __match_any_sync vs __shfl_sync on this GPU (warp instructions per SM-cycle).
#include <cstdio>
__global__ void k_match(unsigned* out, int iters) {
  unsigned v = threadIdx.x * 2654435761u, acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += __match_any_sync(0xffffffffu, v & 0x3ff);
    v = v * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_shfl(unsigned* out, int iters) {
  unsigned v = threadIdx.x * 2654435761u, acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += __shfl_sync(0xffffffffu, v, acc & 31);
    v = v * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  unsigned* d;
  cudaMalloc(&d, 148 * 1024 * 4 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a);
    k_match<<<148 * 8, 256>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double winst = 148.0 * 8 * 8 * iters;
    printf("match_any: %.3f ms, %.2f warp-instr/ns total, %.3f per SM per cycle(1.9GHz)\n", ms, winst / (ms * 1e6),
           winst / (ms * 1e-3) / 148 / 1.9e9);
    cudaEventRecord(a);
    k_shfl<<<148 * 8, 256>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("shfl:      %.3f ms, %.2f warp-instr/ns total, %.3f per SM per cycle(1.9GHz)\n", ms, winst / (ms * 1e6),
           winst / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
