// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) and DFMA peak on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) c[t] = t;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = fma(c[t], a, b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb, iters = 4096;
    dmma_loop<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * (threads / 32) * iters * 8 * 512.0;
    printf("DMMA m8n8k4 warps/blk=%d: %.2f TFLOP/s\n", wpb, flops / ms / 1e9);
  }
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb, iters = 4096;
    dfma_loop<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * threads * iters * 16 * 2.0;
    printf("DFMA warps/blk=%d: %.2f TFLOP/s\n", wpb, flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 4 GiB per buffer as double4? 2^27*32B = 4 GiB
  double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32);
  cudaMemset(a, 0, n * 32);
  copy_k<<<sms * 8, 512>>>(a, b, n);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) copy_k<<<sms * 8, 512>>>(a, b, n);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("copy: %.1f GB/s\n", 5.0 * 2 * n * 32 / ms / 1e6);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
