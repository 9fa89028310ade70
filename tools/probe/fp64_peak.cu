// FP64 peak probe: DFMA throughput and DMMA (mma.sync f64) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 - a;
  double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  double a4[2] = {a, a + 1}, b2[2] = {b, b + 1};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c0[0]), "+d"(c0[1]), "+d"(c0[2]), "+d"(c0[3]) : "d"(a4[0]), "d"(a4[1]), "d"(b2[0]));
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c1[0]), "+d"(c1[1]), "+d"(c1[2]), "+d"(c1[3]) : "d"(a4[1]), "d"(a4[0]), "d"(b2[1]));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c0[1] + c0[2] + c0[3] + c1[0] + c1[1] + c1[2] + c1[3];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("name=%s sms=%d smem_optin=%zu smem_per_sm=%zu l2=%d regs_per_sm=%d clock_khz=%d memclk_khz=%d buswidth=%d\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.l2CacheSize,
         p.regsPerMultiprocessor, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    const int iters = 4000;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("DFMA: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  for (int rep = 0; rep < 3; ++rep) {
    const int iters = 2000;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per warp mma m16n8k4: 2*16*8*4 flops
    double flops = 2.0 * 16 * 8 * 4 * 16.0 * (double)iters * blocks * (threads / 32);
    printf("DMMA m16n8k4: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
