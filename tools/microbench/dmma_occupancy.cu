// DMMA (mma.sync m8n8k4 f64) throughput vs resident warps per SM and
// independent accumulator chains per warp, one CTA per SM (forced with a
// large dynamic shared-memory request). Sizes the Z-Bus kernel's warp layout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_occupancy dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  extern __shared__ double pad[];
  double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.9999999;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s + pad[0];
}

template <int CHAINS>
void run(int sms, double* d, int warps) {
  const int tpb = 32 * warps, iters = 4096 / (CHAINS / 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(dmma_kernel<CHAINS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_kernel<CHAINS><<<sms, tpb, smem>>>(d, 16);
  cudaEventRecord(e0);
  dmma_kernel<CHAINS><<<sms, tpb, smem>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * CHAINS * (double)iters * sms * warps;
  printf("warps/SM=%2d chains=%2d: %.3f ms %6.2f TFLOP/s\n", warps, CHAINS, ms, flops / ms / 1e9);
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<8>(sms, d, w);
    run<16>(sms, d, w);
    run<32>(sms, d, w);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
