// Microbenchmark: cost of DADDs interleaved with DMMAs in the same warp
// (the 3M complex product needs one pre-add per operand fragment).
#include <cstdio>
#include <cuda_runtime.h>
template <int NA>
__global__ void k(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[12][2], x[8];
#pragma unroll
  for (int t = 0; t < 12; ++t) c[t][0] = c[t][1] = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = t * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 12; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
      if (t < NA) asm volatile("add.f64 %0, %0, %1;" : "+d"(x[t & 7]) : "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 12; ++t) s += c[t][0] + c[t][1];
#pragma unroll
  for (int t = 0; t < 8; ++t) s += x[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NA>
void run(int sms, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, iters = 1024;
  k<NA><<<sms, threads>>>(out, 8);
  cudaEventRecord(e0);
  k<NA><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double clk_per_iter_smsp = 1.965e6 * ms / (iters * 4.0);  // 4 warps per SMSP
  printf("12 DMMA + %2d DADD per iteration: %.1f cycles per iteration per SMSP (DMMA only: 192), DMMA %.2f TFLOP/s\n",
         NA, clk_per_iter_smsp, double(sms) * 16 * iters * 12 * 512.0 / ms / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 24);
  run<0>(sms, out); run<2>(sms, out); run<4>(sms, out); run<6>(sms, out); run<8>(sms, out); run<12>(sms, out);
  return 0;
}
