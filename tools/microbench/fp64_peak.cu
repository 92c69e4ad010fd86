// FP64 peak probe for B200 (sm_100a): DFMA vs DMMA (mma.sync m8n8k4 f64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.9999999;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 4096;
    dfma_kernel<<<blocks, tpb>>>(d, 16, 1.000001, 1e-7);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, tpb>>>(d, iters, 1.000001, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * tpb;
    printf("DFMA tpb=%d blocks=%d: %.3f ms  %.2f TFLOP/s\n", tpb, blocks, ms, flops / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (2048 / tpb);
    int iters = 2048;
    dmma_kernel<<<blocks, tpb>>>(d, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, tpb>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * iters * (double)blocks * (tpb / 32);
    printf("DMMA m8n8k4 tpb=%d blocks=%d: %.3f ms  %.2f TFLOP/s\n", tpb, blocks, ms, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
