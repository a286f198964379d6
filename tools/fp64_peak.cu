// fp64_peak.cu — DFMA throughput microbenchmark (the FP64-ALU roofline peak for bench.py).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void dfma_loop(double* out, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; c++) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; c++) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; r++) {
    cudaEventRecord(e0);
    for (int k = 0; k < 10; k++) dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = 2.0 * CHAINS * ITERS * (double)threads * blocks * 10;
  printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"how\": \"dfma_loop %d chains x %d iters, %d blocks x %d threads, "
         "best of 10 x 10 launches (CUDA events)\"}\n",
         flops / (best * 1e-3) / 1e12, sms, CHAINS, ITERS, blocks, threads);
  return 0;
}
