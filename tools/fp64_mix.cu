// Do DMMA (tensor) and DFMA (fp64 pipe) overlap? Half the warps run each.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mix(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 ? true : (mode == 1 ? false : (warp & 1));
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
  double d[16];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
#pragma unroll
  for (int t = 0; t < 16; ++t) d[t] = t;
  if (do_mma) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  } else {
    for (int i = 0; i < iters * 8; ++i) {
#pragma unroll
      for (int t = 0; t < 16; ++t) d[t] = fma(d[t], a, b);
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  for (int t = 0; t < 16; ++t) s += d[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 2, threads = 512, iters = 2048;
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<blocks, threads>>>(out, 16, mode);
    cudaEventRecord(e0);
    mix<<<blocks, threads>>>(out, iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double wm = mode == 0 ? 16 : (mode == 1 ? 0 : 8);  // mma warps per block
    double wf = 16 - wm;
    double fl = blocks * (wm * iters * 8 * 512.0 + wf * 32 * iters * 8 * 16 * 2.0);
    printf("mode %d (%s): %.2f TFLOP/s in %.3f ms\n", mode, mode == 0 ? "dmma" : mode == 1 ? "dfma" : "mixed", fl / ms / 1e9, ms);
  }
  return 0;
}
