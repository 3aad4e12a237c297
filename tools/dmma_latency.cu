// Microbenchmark: DMMA (mma.sync m8n8k4 f64) dependent-chain latency and the
// number of independent chains per warp / warps per SM sub-partition needed
// to saturate the FP64 tensor pipe.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void chains(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[C][2];
#pragma unroll
  for (int t = 0; t < C; ++t) c[t][0] = c[t][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < C; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < C; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C>
void run(int sms, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wps : {1, 2, 4}) {  // warps per SM sub-partition
    const int threads = 32 * 4 * wps, iters = 2048;
    chains<C><<<sms, threads>>>(out, 16);
    cudaEventRecord(e0);
    chains<C><<<sms, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double clk = 1.965e6 * ms;  // cycles at 1965 MHz
    const double per_dmma_smsp = clk / (double(iters) * C * wps);
    printf("chains=%2d warps/SMSP=%d: %.1f cycles per DMMA per SMSP (dep. latency <= %.1f), %.2f TFLOP/s\n", C, wps,
           per_dmma_smsp, per_dmma_smsp * C * wps, double(sms) * 4 * wps * iters * C * 512.0 / ms / 1e9);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 24);
  run<1>(sms, out); run<2>(sms, out); run<3>(sms, out); run<4>(sms, out); run<6>(sms, out); run<8>(sms, out);
  run<12>(sms, out);
  return 0;
}
