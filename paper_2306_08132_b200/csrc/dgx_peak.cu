// dgx_peak.cu — FP64 CUDA-core (DFMA) throughput microbenchmark: the roofline
// denominator for the fused kernel (MEASURED_PEAKS.json carries only HBM and
// bf16 tensor peaks). 8 independent FMA chains per thread, full-chip grid.
#include <cuda_runtime.h>

#include "../../include/dgx.h"

namespace {
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace

extern "C" int dgx_fp64_peak(int device, double* tflops, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return DGX_E_CUDA;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return DGX_E_CUDA;
  const double flops = 2.0 * 64.0 * iters * double(blocks) * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms) *ms = best;
  return DGX_OK;
}
