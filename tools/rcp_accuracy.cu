// rcp_accuracy.cu — accuracy of the MUFU seeds (rcp/rsqrt.approx.ftz.f64) and of
// the refinements used in echo_dev.cuh, against correctly rounded 1/x, 1/sqrt(x).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/rcp_accuracy.cu -o /tmp/rcp && /tmp/rcp
#include <cstdio>
#include <cuda_runtime.h>

__device__ double seed_rcp(double x) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ double seed_rsq(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ double rcp2(double x) {  // two Newton steps
  double y = seed_rcp(x);
  double e = fma(-x, y, 1.0); y = fma(y, e, y);
  e = fma(-x, y, 1.0); return fma(y, e, y);
}
__device__ double rcp3(double x) {  // one step, cubic: y (1 + e + e^2)
  double y = seed_rcp(x);
  double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
__device__ double rsq2(double x) {
  double y = seed_rsq(x);
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5); y = fma(y, e, y);
  e = fma(-h * y, y, 0.5); return fma(y, e, y);
}
__device__ double rsq3(double x) {  // one step, y (1 + r/2 + 3r^2/8), r = 1 - x y^2
  double y = seed_rsq(x);
  double r = fma(-x * y, y, 1.0);
  return fma(y * r, fma(0.375, r, 0.5), y);
}

__device__ double ulps(double a, double ref) {
  double u = fabs(ref) * 2.220446049250313e-16;
  return fabs(a - ref) / u;
}

__global__ void k(unsigned long long seed, double* out) {
  double m[7] = {0, 0, 0, 0, 0, 0, 0};
  unsigned long long s = seed + blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < 4096; it++) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    double u = (double)(s >> 11) * (1.0 / 9007199254740992.0);
    double x = exp2(-40.0 + 80.0 * u);
    double r = 1.0 / x, q = 1.0 / sqrt(x);
    m[0] = fmax(m[0], fabs(seed_rcp(x) * x - 1.0));
    m[1] = fmax(m[1], fabs(seed_rsq(x) * sqrt(x) - 1.0));
    m[2] = fmax(m[2], ulps(rcp2(x), r));
    m[3] = fmax(m[3], ulps(rcp3(x), r));
    m[4] = fmax(m[4], ulps(rsq2(x), q));
    m[5] = fmax(m[5], ulps(rsq3(x), q));
  }
  for (int i = 0; i < 6; i++) {
    unsigned long long* o = (unsigned long long*)out + i;
    atomicMax(o, (unsigned long long)__double_as_longlong(m[i]));
  }
}

int main() {
  double* d;
  cudaMalloc(&d, 8 * 8);
  cudaMemset(d, 0, 64);
  k<<<1184, 256>>>(12345, d);
  double h[8];
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("{\"seed_rcp_rel\": %.3e, \"seed_rsqrt_rel\": %.3e, \"rcp_2newton_ulp\": %.3f, \"rcp_cubic_ulp\": %.3f, "
         "\"rsqrt_2newton_ulp\": %.3f, \"rsqrt_quadratic_ulp\": %.3f, \"samples\": %d}\n",
         h[0], h[1], h[2], h[3], h[4], h[5], 1184 * 256 * 4096);
  return 0;
}
