// Microbenchmark: does DMMA throughput depend on which operand changes between
// consecutive instructions? The FDM stages issue 3 tiles x 3 products per k step
// with the factor fragment stationary: as the A operand (stages 1, 3) or as the B
// operand (stages 2, 4).
//   mode 0: A stationary per group of 3, B moving;  mode 1: A moving, B stationary;
//   mode 2: both fixed;  mode 3: both moving.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* out, int iters) {
  double s[3], v[9];
#pragma unroll
  for (int t = 0; t < 3; ++t) s[t] = 1.0 + (threadIdx.x + t) * 1e-9;
#pragma unroll
  for (int t = 0; t < 9; ++t) v[t] = 1.0 - (threadIdx.x + 3 * t) * 1e-9;
  double c[9][2];
#pragma unroll
  for (int t = 0; t < 9; ++t) c[t][0] = c[t][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int t = p * 3 + j;
        if (MODE == 0) dmma(c[t][0], c[t][1], s[p], v[t]);
        if (MODE == 1) dmma(c[t][0], c[t][1], v[t], s[p]);
        if (MODE == 2) dmma(c[t][0], c[t][1], s[0], s[1]);
        if (MODE == 3) dmma(c[t][0], c[t][1], v[t], v[(t + 4) % 9]);
      }
  }
  double r = 0;
#pragma unroll
  for (int t = 0; t < 9; ++t) r += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE>
void run(int sms, double* out, int threads) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048;
  k<MODE><<<sms, threads>>>(out, 8);
  cudaEventRecord(e0);
  k<MODE><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double wps = threads / 128.0;
  printf("mode %d, %g warps/SMSP: %.2f cycles per DMMA per SMSP, %.2f TFLOP/s\n", MODE, wps,
         1.965e6 * ms / (iters * 9.0 * wps), double(sms) * (threads / 32) * iters * 9 * 512.0 / ms / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 24);
  for (int th : {128, 512}) { run<0>(sms, out, th); run<1>(sms, out, th); run<2>(sms, out, th); run<3>(sms, out, th); }
  return 0;
}
