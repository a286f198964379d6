// fp64_latency.cu — DFMA pipe utilisation vs independent chains per warp and
// warps per SM (how much ILP x TLP the FP64 pipe needs on this B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_latency.cu -o /tmp/fp64_lat && /tmp/fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int CHAINS>
__global__ void dfma_chains(double* out, double a, double b) {
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
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
void run(int warps_per_sm, int sms, double* out) {
  const int threads = 32 * warps_per_sm, blocks = sms;  // one block per SM
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<CHAINS><<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(e0);
    dfma_chains<CHAINS><<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * CHAINS * ITERS * (double)threads * blocks;
  const double peak = 148 * 64 * 2 * 1.965e9;
  printf("chains %d warps/SM %2d (per SMSP %2d): %.2f TF/s = %.0f%% of nominal\n", CHAINS, warps_per_sm,
         warps_per_sm / 4, flops / (best * 1e-3) / 1e12, 100 * flops / (best * 1e-3) / peak);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1>(w, sms, out);
    run<2>(w, sms, out);
    run<4>(w, sms, out);
  }
  return 0;
}
