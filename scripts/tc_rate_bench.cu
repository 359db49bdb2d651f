// tc_rate_bench.cu -- tcgen05 issue-rate microbenchmark (VERDICT r1 "settle
// the tensor-pipe question"): FLOP per clock per SM of back-to-back
// kind::f16 MMAs (N = 256, K = 16, fp32 accumulate in TMEM, operands in
// 128B-swizzled shared memory) for the tile shapes a split-precision decoder
// could use:
//   cg2 M=128 : cta_group::2, 64 rows per SM   (the shipped k_tc_mlp / k_tc_heads shape)
//   cg2 M=256 : cta_group::2, 128 rows per SM
//   cg1 M=128 : cta_group::1, 128 rows per SM
//   cg1 M=64  : cta_group::1, 64 rows per SM
// Every SM runs one CTA (grid = SM count, clusters of 2 for cta_group::2);
// one thread per CTA (the leader's, for cta_group::2) issues ITER MMAs into one
// accumulator, commits once and waits.  Operand values are irrelevant (zeros).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1911_13225_b200/csrc \
//        scripts/tc_rate_bench.cu -o scripts/tc_rate_bench && scripts/tc_rate_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_core.cuh"

using namespace dist::tc;

constexpr int ITER = 8192;

template <int CG, int M>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b) {
  constexpr uint32_t idesc = (1u << 4) | ((256u >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if constexpr (CG == 2)
    asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b),
                 "n"(idesc));
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b),
                 "n"(idesc));
}

template <int CG, int M>
__global__ void __launch_bounds__(128, 1) k_rate(unsigned long long *cycles) {
  extern __shared__ __align__(1024) char smem_raw[];
  char *smem = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if constexpr (CG == 2) rank = cta_rank();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0u;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (warp == 0) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0 && rank == 0) {
    const uint64_t a = sdesc(smem_u32(smem)), b = sdesc(smem_u32(smem + 32768));
    const unsigned long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < ITER; ++i) mma<CG, M>(tmem, a, b);
    if constexpr (CG == 2)
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)0x3)
          : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  } else if constexpr (CG == 2) {
    if (threadIdx.x == 0) mbar_wait(&bar, 0);   // the multicast commit arrives here too
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (warp == 0) {
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int CG, int M>
static void run(const char *name, int nsm) {
  const int smem = 65536 + 2048;
  auto fn = k_rate<CG, M>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * nsm);
  cudaMemset(cyc, 0, sizeof(unsigned long long) * nsm);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(nsm - (nsm % CG));
  lc.blockDim = dim3(128);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&lc, fn, cyc);   // warm-up (clocks ramp)
  cudaEventRecord(e0);
  const int reps = 10;
  for (int rep = 0; rep < reps; ++rep) cudaLaunchKernelEx(&lc, fn, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[256] = {0};
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
  double cmax = 0;
  int nlead = 0;
  for (int i = 0; i < nsm; ++i)
    if (h[i]) {
      cmax = cmax > h[i] ? cmax : (double)h[i];
      ++nlead;
    }
  const double flop_per_mma = 2.0 * M * 256 * 16;
  const double flop = flop_per_mma * ITER * nlead * reps;
  const double per_sm_clk = flop_per_mma * ITER / (double)CG / cmax;   // one launch, the slowest issuer
  printf("{\"shape\": \"%s\", \"rows_per_sm\": %d, \"issuers\": %d, \"ms\": %.3f, \"tflops\": %.1f, "
         "\"flop_per_clk_per_sm\": %.0f, \"cycles_per_mma\": %.1f, \"err\": \"%s\"}\n",
         name, M / CG, nlead, ms, flop / (ms * 1e-3) / 1e12, per_sm_clk, cmax / ITER, cudaGetErrorString(err));
  cudaFree(cyc);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<2, 128>("cta_group::2 M=128 N=256 K=16", nsm);
  run<2, 256>("cta_group::2 M=256 N=256 K=16", nsm);
  run<1, 128>("cta_group::1 M=128 N=256 K=16", nsm);
  run<1, 64>("cta_group::1 M=64 N=256 K=16", nsm);
  run<2, 128>("cta_group::2 M=128 N=256 K=16 (again)", nsm);
  return 0;
}
