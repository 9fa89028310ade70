// Bulk-copy (cp.async.bulk shared -> global) store-rate probe for the pair-kernel design (B200, sm_100a):
// per-SM rate by op size, destination alignment, cache hint, number of active SMs, and with
// load/store-unit streaming stores running alongside (do the two paths share one egress?).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_store_probe bulk_store_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes, uint64_t pol, bool hint) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(src));
  if (hint)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                     __cvta_generic_to_global(dst)), "r"(sa), "r"(bytes), "l"(pol) : "memory");
  else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(__cvta_generic_to_global(dst)),
                 "r"(sa), "r"(bytes) : "memory");
}

// mode bit 0: cache hint; lsu_warps: warps 1.. also stream 16 B coalesced stores of the same volume elsewhere
__global__ void probe(char* out, long long per_cta, int opbytes, int misalign, int hint, int iters, int lsu,
                      long long* cyc, int W) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = make_double2(i, blockIdx.x);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  char* base = out + (long long)blockIdx.x * per_cta * 2 + misalign;
  const long long t0 = clock64();
  if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < W && !(lsu & 2)) {
    for (int it = 0; it < iters; ++it)
      for (long long o = (threadIdx.x >> 5) * (long long)opbytes; o + opbytes <= per_cta - 128; o += (long long)W * opbytes)
        bulk_store(base + o, reinterpret_cast<char*>(sm) + (o % (131072 - opbytes + 16)) / 16 * 16 % 65536, opbytes, pol, hint);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  if ((lsu & 1) && threadIdx.x >= 32) {
    double2* p = reinterpret_cast<double2*>(base + per_cta - misalign);
    const int T = blockDim.x - 32, t = threadIdx.x - 32;
    if (W > 1) return;
    double2 v = make_double2(t, 1.0);
    for (int it = 0; it < iters; ++it)
      for (long long i = t; i < per_cta / 16; i += T) __stcs(p + i, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const long long per_cta = 4 << 20;  // 4 MiB per path per CTA per iteration
  char* out;
  cudaMalloc(&out, 148LL * per_cta * 2 + 4096);
  long long* cyc;
  cudaMallocManaged(&cyc, 148 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int iters = 4;
  printf("%8s %8s %5s %5s %4s | %10s %10s\n", "ctas", "opbytes", "misal", "hint", "lsu", "B/clk/SM", "GB/s tot");
  for (int W : {1, 2, 4, 12})
    for (int opbytes : {512, 2048, 4096, 8192}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      probe<<<37, 384, 131072>>>(out, per_cta, opbytes, 0, 1, 1, 0, cyc, W);
      cudaEventRecord(e0);
      probe<<<37, 384, 131072>>>(out, per_cta, opbytes, 0, 1, iters, 0, cyc, W);
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      double c = 0;
      for (int i = 0; i < 37; ++i) c += cyc[i];
      c /= 37;
      printf("issuers %2d opbytes %5d : %6.2f B/clk/SM\n", W, opbytes, iters * (double)per_cta / c);
    }
  for (int ctas : {37, 148})
    for (int lsu : {0, 1, 3})
      for (int opbytes : {256, 2048, 16384})
        for (int misalign : {0, 16})
          for (int hint : {0, 1}) {
            if (lsu == 3 && (opbytes != 2048 || misalign || hint)) continue;
            if (lsu == 1 && (opbytes == 256 || misalign)) continue;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            probe<<<ctas, 384, 131072>>>(out, per_cta, opbytes, misalign, hint, 1, lsu, cyc, 1);
            cudaEventRecord(e0);
            probe<<<ctas, 384, 131072>>>(out, per_cta, opbytes, misalign, hint, iters, lsu, cyc, 1);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double c = 0;
            for (int i = 0; i < ctas; ++i) c += cyc[i];
            c /= ctas;
            const double paths = lsu == 1 ? 2.0 : 1.0;
            const double bytes = paths * iters * (double)(per_cta - (lsu == 3 ? 0 : 128));
            printf("%8d %8d %5d %5d %4d | %10.2f %10.1f   %s\n", ctas, opbytes, misalign, hint, lsu, bytes / c,
                   bytes * ctas / ms * 1e-6, cudaGetErrorString(cudaGetLastError()));
          }
  return 0;
}
