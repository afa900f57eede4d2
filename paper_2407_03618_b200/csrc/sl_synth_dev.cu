// sl_synth_dev.cu — device side of the seeded synthetic-corpus generator (libsl_synth.so).
//
// Input generation for bench.py and the tests only: token i of the corpus is the Zipf token
// at global position begin + i, bit-identical to the host generator (sl_synth.h). It lives
// in the synth library, not in libsparselex_b200.so, so the product ABI carries no test
// input machinery.
#include <cuda_runtime.h>

#include "sl_synth.h"

namespace {
__global__ void k_synth_tokens(const double* __restrict__ cdf, uint32_t V, uint32_t seed, uint64_t begin,
                               uint64_t count, uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = sl_corpus_token(cdf, V, seed, begin + i);
}
}  // namespace

extern "C" {
/* token_ids_dev[i] = Zipf token at global position begin + i using the f64 CDF `cdf` (host
 * memory when cdf_on_device == 0). Returns 0, or a cudaError_t value. Synchronous. */
int32_t sl_synth_tokens_device(const double* cdf, uint32_t vocab, uint32_t seed, uint64_t begin, uint64_t count,
                               int32_t cdf_on_device, uint32_t* token_ids_dev) {
  if (!cdf || !token_ids_dev || vocab == 0) return (int32_t)cudaErrorInvalidValue;
  const double* dcdf = cdf;
  double* tmp = nullptr;
  cudaError_t e = cudaSuccess;
  if (!cdf_on_device) {
    e = cudaMalloc(&tmp, (uint64_t)vocab * 8);
    if (e == cudaSuccess) e = cudaMemcpy(tmp, cdf, (uint64_t)vocab * 8, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      if (tmp) cudaFree(tmp);
      return (int32_t)e;
    }
    dcdf = tmp;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 64ull * sms) blocks = 64ull * sms;
  if (blocks == 0) blocks = 1;
  k_synth_tokens<<<(unsigned)blocks, 256>>>(dcdf, vocab, seed, begin, count, token_ids_dev);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (tmp) cudaFree(tmp);
  return (int32_t)e;
}
}  // extern "C"
