// Store-path and FP64-pipe probes for the pair-kernel design (B200, sm_100a).
//  (1) per-SM streaming store rate with G active CTAs (one per SM): is the
//      window-store phase bound by the SM's own store path or by HBM?
//      patterns: 16 B coalesced, 8 B coalesced, 16 B at 32 B stride (two
//      interleaved writers per 32 B sector, written by two different warps)
//  (2) DFMA and DMMA issued concurrently by different warps of one SM:
//      separate pipes (sum > either alone) or one FP64 datapath?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_probe store_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void store_kernel(double* out, long long per_cta, int mode, int iters) {
  double* base = out + (long long)blockIdx.x * per_cta;
  const int T = blockDim.x;
  double2 v = make_double2(threadIdx.x * 1.0, blockIdx.x * 1.0);
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {  // 16 B coalesced
      double2* p = reinterpret_cast<double2*>(base);
      for (long long i = threadIdx.x; i < per_cta / 2; i += T) __stcs(p + i, v);
    } else if (mode == 1) {  // 8 B coalesced
      for (long long i = threadIdx.x; i < per_cta; i += T) __stcs(base + i, v.x);
    } else if (mode == 3) {  // one lane writes 32 B as two back-to-back 16 B stores (lanes at 32 B stride)
      double2* p = reinterpret_cast<double2*>(base);
      for (long long i = threadIdx.x; 2 * i + 1 < per_cta / 2; i += T) {
        __stcs(p + 2 * i, v);
        __stcs(p + 2 * i + 1, v);
      }
    } else if (mode == 4) {  // one lane writes 32 B as four 8 B stores, column base 8 B (not 16 B) aligned
      double* q = base + 1;
      for (long long i = threadIdx.x; 4 * i + 3 < per_cta - 1; i += T) {
        __stcs(q + 4 * i, v.x);
        __stcs(q + 4 * i + 1, v.y);
        __stcs(q + 4 * i + 2, v.x);
        __stcs(q + 4 * i + 3, v.y);
      }
    } else {  // 16 B at 32 B stride; warps 2w and 2w+1 fill the two halves of each sector
      double2* p = reinterpret_cast<double2*>(base);
      const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, half = w & 1, wp = w >> 1, nwp = T / 64;
      for (long long i = wp * 32 + lane; 2 * i + 1 < per_cta / 2; i += nwp * 32) __stcs(p + 2 * i + half, v);
    }
    v.x += 1.0;
  }
}

__global__ void mixed_fp64(double* out, int iters, int dmma_warps) {
  const int w = threadIdx.x >> 5;
  double r = 0;
  if (w < dmma_warps) {
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
    r = c0[0] + c0[1] + c0[2] + c0[3] + c1[0] + c1[1] + c1[2] + c1[3];
  } else {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < 8 * iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
      }
    }
    r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const double clk = p.clockRate * 1e3;
  const long long per_cta = 4ll << 20;  // 32 MB of doubles per CTA
  double* out;
  cudaMalloc(&out, sizeof(double) * per_cta * sms);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[5] = {"16B coalesced", "8B coalesced", "16B @32B stride, 2 warps/sector",
                          "32B/lane as 2x16B (same warp)", "32B/lane as 4x8B, 8B-aligned base"};
  for (int mode : {0, 2, 3, 4}) {
    for (int g : {sms, sms / 4}) {
      for (int threads : {384}) {
        store_kernel<<<g, threads>>>(out, per_cta, mode, 1);
        cudaEventRecord(e0);
        store_kernel<<<g, threads>>>(out, per_cta, mode, 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 2.0 * per_cta * 8 * g * (mode == 2 ? 0.5 : 1.0) * 2.0 / 2.0;
        const double bps = (mode == 2 ? 2.0 * per_cta * 8 * g * 0.5 : 2.0 * per_cta * 8 * g) / (ms * 1e-3);
        (void)bytes;
        printf("store %-34s CTAs %3d x %4d thr: %8.1f GB/s total, %6.1f B/clk per SM\n", names[mode], g, threads,
               bps / 1e9, bps / g / clk);
      }
    }
  }
  // mixed FP64 pipes: 8 warps per CTA, 4 CTAs/SM-equivalent grid
  double* o2;
  cudaMalloc(&o2, sizeof(double) * sms * 8 * 256);
  for (int dw : {0}) {
    const int iters = 2000;
    mixed_fp64<<<sms * 8, 256>>>(o2, iters, dw);
    cudaEventRecord(e0);
    mixed_fp64<<<sms * 8, 256>>>(o2, iters, dw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = sms * 8.0 * 8;
    const double fl_dmma = 2.0 * 16 * 8 * 4 * 16.0 * iters * (warps * dw / 8.0);
    const double fl_dfma = 2.0 * 8 * 16 * 8.0 * (double)iters * 32 * (warps * (8 - dw) / 8.0);
    printf("mixed fp64: %d of 8 warps DMMA: %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", dw, ms,
           fl_dmma / ms / 1e9, fl_dfma / ms / 1e9, (fl_dmma + fl_dfma) / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
