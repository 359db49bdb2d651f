// tc_pattern_bench.cu -- why does k_tc_mlp's MMA phase run at ~55% of the
// tcgen05 issue rate even with the weight stream switched off
// (scripts/tc_debug_timing.py, DIST_TC_DEBUG=4)?  Replays the kernel's exact
// MMA issue pattern (cta_group::2 M=128 N=256 K=16, operands in 128B-swizzled
// shared memory laid out as in tc_core.cuh: A_hi 64 KB, A_lo 64 KB, a 3-stage
// B ring of 32 KB) without any barrier waits, and variants of it:
//   0 const   : one accumulator, constant descriptors (the rate benchmark)
//   1 kernel  : mode 3 -- per K block 4 x hi*hi into D, then 4 x (hi*lo, lo*hi) into D2
//   2 one-acc : the same 12 MMAs per K block, all into D
//   3 hihi    : only the 4 hi*hi per K block (varying descriptors)
//   4 kernel+commit : 1 plus a tcgen05.commit per K block (as the kernel's empty barriers)
//   5 D2-only : only the 8 corrections per K block into D2
//   6 ring    : 1 fed through the kernel's 3-stage full/empty mbarrier ring (a
//               producer thread per CTA waits on empty, rank 0's arrives on
//               full; no TMA: DIST_TC_DEBUG=4's pipeline)
//   7 ring6   : 6 with a 6-stage ring (the same stage size)
//   8 ring-nofence : 6 without the tcgen05.fence::after_thread_sync after each wait
//   9 fence   : 1 (no ring) with a tcgen05.fence::after_thread_sync per K block
//  10 ring-spin  : 6 with every barrier wait a mbarrier.test_wait spin
//  11 ring-nohint: 6 with try_wait without a suspend-time hint
//  12/13/14 self : no producer; before K block it the MMA thread waits on the
//               commit barrier of K block it-RS itself (RS = 3 / 6 / 12)
//  15 self-relaxed : 13 with mbarrier.try_wait.relaxed.cta
//  16 self-lookahead : 13 with the wait for K block it+1 placed after the
//               first 8 MMAs of K block it (4 MMAs still queued while it waits)
//  17 self-sparse : 14 (12 deep) waiting only every 4th K block
//  18 done-wait : 1 plus, per K block, a wait on a barrier completed before the loop
//  21 done-test : 18 with mbarrier.test_wait
//  22 flag-poll : 1 plus, per K block, a volatile shared-memory flag read (and branch)
//  23 named-bar : warp 0 runs the loop (lane 0 issues), per K block bar.sync with warp 1
//  24 warp-loop : 23 without the named barrier
//  25/26 done-wait sparse : 18 with the wait every 2nd / 4th K block
//  27 done-wait unrolled : 18 with the K-block loop fully unrolled (the compiler
//               puts a YIELD on the back-edge of a loop that waits on a barrier)
//  28 +tmem-ld : 27 (no waits) while 8 other warps stream tcgen05.ld from TMEM
//               columns the MMAs do not write (the epilogue's D reads)
//  29 +st.shared : 27 while 8 warps stream 16-byte shared stores into A_lo
//  30 +both   : 28 and 29 together
//  31/32 ring unrolled : 6 / 7 (3- / 6-stage full/empty ring with a producer
//               thread) with the MMA issuer's K loop unrolled
//  33 ring, both unrolled : 31 with the producer's loop unrolled by 8 too
//  34/35 ring pairs : 31/32 waiting for two stages at once on even K blocks
//  36 ring, local arrive : 31 with the producer arriving by mbarrier.arrive.shared::cta
//  37 ring, leader-only  : 36 with only the leader's producer (rank 1's idles)
//  38/39/40 self, unrolled : 12/13/14 (the MMA thread waits on its own commit
//               of K block it-RS, RS = 3 / 6 / 12) with the K loop unrolled
//  41 ring, spin producer : 31 with the producer's empty-wait a test_wait spin
//  42 ring, spin both     : 41 with the MMA thread's full-wait a test_wait spin too
//  43/44 ring, lazy producer : 31 with the producer polling empty by test_wait
//               + __nanosleep(200 / 1000) between polls
//  45 merged  : no producer thread: before K block it the MMA thread waits on
//               its own commit of it-1 (the slot of it+2), arrives on that
//               slot's full barrier itself (where the TMA issue would go), then
//               waits on full[it] -- the producer role folded into the issuer
// FLOP per clock per SM of the slowest issuer; operand values are zeros.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1911_13225_b200/csrc \
//        scripts/tc_pattern_bench.cu -o scripts/tc_pattern_bench && scripts/tc_pattern_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_core.cuh"

using namespace dist::tc;

__device__ __forceinline__ void mma_m256(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  constexpr uint32_t idesc = (1u << 4) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(acc), "n"(idesc));
}

template <int W>
__device__ __forceinline__ void wait_w(uint64_t *b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  if constexpr (W == 5 || W == 6) {
    for (;;) {
      uint32_t ok;
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(a), "r"(parity)
          : "memory");
      if (ok) break;
      __nanosleep(W == 5 ? 200 : 1000);
    }
  } else if constexpr (W == 0) {
    mbar_wait(b, parity);
  } else if constexpr (W == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT1:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT1;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
  } else if constexpr (W == 3) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT3:\n\t"
        "mbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT3;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT2:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT2;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
  }
}

constexpr int TILES = 24;   // x 7 layers x 2 N halves x 8 K blocks

template <int PAT>
__global__ void __launch_bounds__(320, 1) k_pat(unsigned long long *cycles, unsigned long long *nmma) {
  extern __shared__ __align__(1024) char smem_raw[];
  char *smem = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int RS = PAT == 7 || PAT == 13 || PAT == 15 || PAT == 16 || PAT == 32 || PAT == 35 || PAT == 39 ? 6
                     : (PAT == 14 || PAT == 17 || PAT == 40 ? 12 : STAGES);
  constexpr bool SELF = (PAT >= 12 && PAT <= 17) || (PAT >= 38 && PAT <= 40);
  constexpr int WF = PAT == 10 || PAT == 41 || PAT == 42 ? 1 : (PAT == 11 ? 2 : (PAT == 43 ? 5 : (PAT == 44 ? 6 : 0)));
  constexpr bool RING = (PAT >= 6 && PAT <= 8) || PAT == 10 || PAT == 11 || SELF || PAT == 31 || PAT == 32 || PAT == 33 || PAT == 34 || PAT == 35 || PAT == 36 || PAT == 37 ||
                       PAT == 41 || PAT == 42 || PAT == 43 || PAT == 44 || PAT == 45;
  __shared__ uint64_t bar, sbar, full[16], empty[16];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cta_rank();
  for (int i = threadIdx.x; i < (OFF_B + STAGES * STAGE_BYTES) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&sbar, 1);
    for (int i = 0; i < 16; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  constexpr int NIT = TILES * 7 * 2 * NKB;
  if ((PAT == 23 || PAT == 24) && rank == 0 && warp < 2) {
    if (warp == 1) {
      if (PAT == 23)
        for (int it = 0; it < NIT; ++it) asm volatile("bar.sync 2, 64;" ::: "memory");
    } else {
      const int lane = threadIdx.x & 31;
      const uint32_t a_hi = smem_u32(smem + OFF_AHI), a_lo = smem_u32(smem + OFF_ALO);
      const unsigned long long t0 = clock64();
      uint32_t it = 0;
      for (int t = 0; t < TILES; ++t)
        for (int l = 0; l < 7; ++l)
          for (int nh = 0; nh < 2; ++nh) {
            const uint32_t d = tmem + nh * 128;
            for (int kc = 0; kc < NKB; ++kc, ++it) {
              if (PAT == 23) asm volatile("bar.sync 2, 64;" ::: "memory");
              const int s = it % STAGES;
              const uint32_t b_hi = smem_u32(smem + OFF_B + s * STAGE_BYTES), b_lo = b_hi + B_TILE;
              if (lane == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t ak = kc * (ROWS * 128) + q * 32;
                  mma_2sm<true>(d, sdesc(a_hi + ak), sdesc(b_hi + q * 32), (kc | q) ? 1u : 0u);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t ak = kc * (ROWS * 128) + q * 32;
                  mma_2sm<true>(d + 256u, sdesc(a_hi + ak), sdesc(b_lo + q * 32), 1u);
                  mma_2sm<true>(d + 256u, sdesc(a_lo + ak), sdesc(b_hi + q * 32), 1u);
                }
              }
              __syncwarp();
            }
          }
      if (lane == 0) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)0x3)
            : "memory");
        mbar_wait(&bar, 0);
        cycles[blockIdx.x] = clock64() - t0;
        nmma[blockIdx.x] = (unsigned long long)NIT * 12;
      }
    }
  } else if ((PAT == 23 || PAT == 24) && rank == 1 && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  __shared__ volatile int s_stop;
  if (threadIdx.x == 0) s_stop = 0;
  __syncthreads();
  if (PAT >= 28 && PAT <= 30 && warp >= 2) {   // load generators: until the MMA thread is done
    const int q = warp & 3;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + 128u;   // D nh1 columns
    float acc = 0.f;
    int n = 0;
    while (!s_stop) {
      if (PAT == 28 || PAT == 30) {
        float v[32];
        tmem_ld32(tq + ((n & 3) * 32u), v);
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += v[e];
      }
      if (PAT == 29 || PAT == 30) {
        uint4 *dst = reinterpret_cast<uint4 *>(smem + OFF_ALO) + ((threadIdx.x - 64) + (n & 15) * 256) % 4096;
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[e * 1024 % 4096] = make_uint4(0u, 0u, 0u, 0u);
      }
      ++n;
    }
    if (acc == 12345.f) cycles[0] = 1;   // keep the loads
  }
  if ((PAT == 27 || (PAT >= 28 && PAT <= 30)) && threadIdx.x == 0 && rank == 0) {
    if (PAT == 27) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sbar)) : "memory");
    const uint32_t a_hi = smem_u32(smem + OFF_AHI), a_lo = smem_u32(smem + OFF_ALO);
    uint32_t it = 0;
    const unsigned long long t0 = clock64();
    for (int t = 0; t < TILES; ++t)
      for (int l = 0; l < 7; ++l)
        for (int nh = 0; nh < 2; ++nh) {
          const uint32_t d = tmem + nh * 128;
#pragma unroll
          for (int kc = 0; kc < NKB; ++kc, ++it) {
            const int s = it % STAGES;
            const uint32_t b_hi = smem_u32(smem + OFF_B + s * STAGE_BYTES), b_lo = b_hi + B_TILE;
            if (PAT == 27) mbar_wait(&sbar, 0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t ak = kc * (ROWS * 128) + q * 32;
              mma_2sm<true>(d, sdesc(a_hi + ak), sdesc(b_hi + q * 32), (kc | q) ? 1u : 0u);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t ak = kc * (ROWS * 128) + q * 32;
              mma_2sm<true>(d + 256u, sdesc(a_hi + ak), sdesc(b_lo + q * 32), 1u);
              mma_2sm<true>(d + 256u, sdesc(a_lo + ak), sdesc(b_hi + q * 32), 1u);
            }
          }
        }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)0x3)
        : "memory");
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
    nmma[blockIdx.x] = (unsigned long long)NIT * 12;
  } else if ((PAT == 27 || (PAT >= 28 && PAT <= 30)) && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  if (PAT >= 28 && PAT <= 30 && threadIdx.x == 0) s_stop = 1;
  if (RING && !SELF && PAT != 45 && threadIdx.x == 32) {   // producer (both CTAs)
    if constexpr (PAT == 33) {
      for (int i0 = 0; i0 < NIT; i0 += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int it = i0 + j;
          const int s = it % RS;
          wait_w<WF>(&empty[s], ((it / RS) & 1) ^ 1);
          if (rank == 0) mbar_arrive_cluster(&full[s], 0);
        }
      }
    } else if constexpr (PAT == 36 || PAT == 37) {
      if (PAT == 36 || rank == 0)
        for (int it = 0; it < NIT; ++it) {
          const int s = it % RS;
          wait_w<WF>(&empty[s], ((it / RS) & 1) ^ 1);
          if (rank == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        }
    } else {
      for (int it = 0; it < NIT; ++it) {
        const int s = it % RS;
        wait_w<WF>(&empty[s], ((it / RS) & 1) ^ 1);
        if (rank == 0) mbar_arrive_cluster(&full[s], 0);
      }
    }
  }
  if (RING && threadIdx.x == 0 && rank == 0) {   // MMA issuer through the ring
    const uint32_t a_hi = smem_u32(smem + OFF_AHI), a_lo = smem_u32(smem + OFF_ALO);
    const unsigned long long t0 = clock64();
    uint32_t it = 0;
    for (int t = 0; t < TILES; ++t)
      for (int l = 0; l < 7; ++l)
        for (int nh = 0; nh < 2; ++nh) {
          const uint32_t d = tmem + nh * 128;
#pragma unroll (PAT >= 31 ? 8 : 1)
          for (int kc = 0; kc < NKB; ++kc, ++it) {
            const int s = it % RS;
            if constexpr (PAT == 45) {
              // refill the slot of K block it+2 (freed by the commit of it-1)
              const uint32_t nx = it + 2;
              if (nx >= (uint32_t)RS) wait_w<0>(&empty[nx % RS], ((nx / RS) - 1) & 1);
              asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[nx % RS])) : "memory");
              if (it == 0) {   // the first two slots
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[0])) : "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[1])) : "memory");
              }
              wait_w<0>(&full[s], (it / RS) & 1);
            } else if constexpr (PAT == 16) {
              if (it == 0) {}   // K block 0's wait: none (nothing committed yet)
            } else if constexpr (PAT == 17) {
              if (it >= (uint32_t)RS && (it & 3) == 0) wait_w<0>(&empty[s], ((it / RS) - 1) & 1);
            } else if constexpr (SELF) {
              if (it >= (uint32_t)RS) wait_w<PAT == 15 ? 3 : 0>(&empty[s], ((it / RS) - 1) & 1);
            } else if constexpr (PAT == 34 || PAT == 35) {
              if (!(kc & 1)) {
                wait_w<0>(&full[s], (it / RS) & 1);
                wait_w<0>(&full[(it + 1) % RS], ((it + 1) / RS) & 1);
              }
            } else {
              wait_w<PAT == 41 || PAT == 43 || PAT == 44 ? 0 : WF>(&full[s], (it / RS) & 1);
            }
            if (PAT != 8) tc_fence_after();
            const uint32_t b_hi = smem_u32(smem + OFF_B + (s % STAGES) * STAGE_BYTES), b_lo = b_hi + B_TILE;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t ak = kc * (ROWS * 128) + q * 32;
              mma_2sm<true>(d, sdesc(a_hi + ak), sdesc(b_hi + q * 32), (kc | q) ? 1u : 0u);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t ak = kc * (ROWS * 128) + q * 32;
              mma_2sm<true>(d + 256u, sdesc(a_hi + ak), sdesc(b_lo + q * 32), 1u);
              mma_2sm<true>(d + 256u, sdesc(a_lo + ak), sdesc(b_hi + q * 32), 1u);
              if (PAT == 16 && q == 1) {   // the next K block's wait, 4 MMAs still to issue
                const uint32_t nx = it + 1;
                if (nx >= (uint32_t)RS) wait_w<0>(&empty[nx % RS], ((nx / RS) - 1) & 1);
              }
            }
            commit_2sm(&empty[s]);
          }
        }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)0x3)
        : "memory");
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
    nmma[blockIdx.x] = (unsigned long long)NIT * 12;
  } else if (RING && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  } else if ((PAT < 6 || PAT == 9 || (PAT >= 18 && PAT <= 22) || PAT == 25 || PAT == 26) && threadIdx.x == 0 && rank == 0) {
    if (PAT == 18 || PAT == 19 || PAT == 21 || PAT == 25 || PAT == 26) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sbar)) : "memory");
    const uint32_t a_hi = smem_u32(smem + OFF_AHI), a_lo = smem_u32(smem + OFF_ALO);
    unsigned long long n = 0;
    uint32_t it = 0;
    const unsigned long long t0 = clock64();
    for (int t = 0; t < TILES; ++t)
      for (int l = 0; l < 7; ++l)
        for (int nh = 0; nh < 2; ++nh) {
          const uint32_t d = tmem + nh * 128;
          for (int kc = 0; kc < NKB; ++kc, ++it) {
            const int s = it % STAGES;
            const uint32_t b_hi = smem_u32(smem + OFF_B + s * STAGE_BYTES), b_lo = b_hi + B_TILE;
            if (PAT == 0) {
#pragma unroll
              for (int q = 0; q < 12; ++q) mma_2sm<true>(tmem, sdesc(a_hi), sdesc(b_hi), 1u);
              n += 12;
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t ak = kc * (ROWS * 128) + q * 32;
                if (PAT == 19 || PAT == 20) mma_m256(d, sdesc(a_hi + ak), sdesc(b_hi + q * 32), (kc | q) ? 1u : 0u);
                else if (PAT != 5) mma_2sm<true>(d, sdesc(a_hi + ak), sdesc(b_hi + q * 32), (kc | q) ? 1u : 0u);
              }
              if (PAT != 3) {
                const uint32_t d2 = PAT == 2 ? d : d + 256u;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t ak = kc * (ROWS * 128) + q * 32;
                  if (PAT == 19 || PAT == 20) {
                    mma_m256(d2, sdesc(a_hi + ak), sdesc(b_lo + q * 32), 1u);
                    mma_m256(d2, sdesc(a_lo + ak), sdesc(b_hi + q * 32), 1u);
                  } else {
                    mma_2sm<true>(d2, sdesc(a_hi + ak), sdesc(b_lo + q * 32), 1u);
                    mma_2sm<true>(d2, sdesc(a_lo + ak), sdesc(b_hi + q * 32), 1u);
                  }
                }
              }
              n += PAT == 3 ? 4 : (PAT == 5 ? 8 : 12);
              if (PAT == 4) commit_2sm(&sbar);
              if (PAT == 9) tc_fence_after();
              if (PAT == 18 || PAT == 19) mbar_wait(&sbar, 0);
              if (PAT == 25 && !(kc & 1)) mbar_wait(&sbar, 0);
              if (PAT == 26 && !(kc & 3)) mbar_wait(&sbar, 0);
              if (PAT == 21) wait_w<1>(&sbar, 0);
              if (PAT == 22) {
                while (*(volatile uint32_t *)&tmem_base == 0xFFFFFFFFu) {}
              }
            }
          }
        }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)0x3)
        : "memory");
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
    nmma[blockIdx.x] = n;
  } else if ((PAT < 6 || PAT == 9 || (PAT >= 18 && PAT <= 22) || PAT == 25 || PAT == 26) && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int PAT>
static void run(const char *name, int nsm) {
  const int smem = OFF_B + STAGES * STAGE_BYTES + 2048;
  auto fn = k_pat<PAT>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *cyc, *nm;
  cudaMalloc(&cyc, sizeof(unsigned long long) * nsm);
  cudaMalloc(&nm, sizeof(unsigned long long) * nsm);
  cudaMemset(cyc, 0, sizeof(unsigned long long) * nsm);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(nsm - (nsm % 2));
  lc.blockDim = dim3(PAT >= 28 && PAT <= 30 ? 320 : 128);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&lc, fn, cyc, nm);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[256] = {0}, hn[256] = {0};
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
  cudaMemcpy(hn, nm, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
  double cmax = 0, n = 0;
  for (int i = 0; i < nsm; ++i)
    if (h[i] && (double)h[i] > cmax) {
      cmax = (double)h[i];
      n = (double)hn[i];
    }
  const double flop_per_mma = 2.0 * (PAT == 19 || PAT == 20 ? 256 : 128) * 256 * 16;
  printf("{\"pattern\": \"%s\", \"mmas\": %.0f, \"cycles\": %.0f, \"cycles_per_mma\": %.1f, "
         "\"flop_per_clk_per_sm\": %.0f, \"err\": \"%s\"}\n",
         name, n, cmax, cmax / n, flop_per_mma * n / 2.0 / cmax, cudaGetErrorString(err));
  fflush(stdout);
  cudaFree(cyc);
  cudaFree(nm);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<0>("const", nsm);
  run<1>("kernel (mode 3)", nsm);
  run<2>("one accumulator", nsm);
  run<3>("hi*hi only", nsm);
  run<4>("kernel + commit per K block", nsm);
  run<5>("corrections only (D2)", nsm);
  run<6>("kernel through the 3-stage mbarrier ring", nsm);
  run<7>("kernel through a 6-stage mbarrier ring", nsm);
  run<8>("ring without the after_thread_sync fence", nsm);
  run<9>("no ring, fence per K block", nsm);
  run<10>("ring, test_wait spin", nsm);
  run<11>("ring, try_wait without a hint", nsm);
  run<12>("self-throttled on its own commits, 3 deep", nsm);
  run<13>("self-throttled on its own commits, 6 deep", nsm);
  run<14>("self-throttled on its own commits, 12 deep", nsm);
  run<15>("self-throttled 6 deep, relaxed try_wait", nsm);
  run<16>("self-throttled 6 deep, wait issued 4 MMAs early", nsm);
  run<17>("self-throttled 12 deep, waits every 4th K block", nsm);
  run<18>("no ring, a completed-barrier wait per K block", nsm);
  run<21>("no ring, a completed-barrier test_wait per K block", nsm);
  run<22>("no ring, a volatile smem flag poll per K block", nsm);
  run<23>("warp loop, named barrier with a helper warp per K block", nsm);
  run<24>("warp loop, no barrier", nsm);
  run<25>("no ring, a completed-barrier wait every 2nd K block", nsm);
  run<26>("no ring, a completed-barrier wait every 4th K block", nsm);
  run<27>("no ring, completed-barrier wait per K block, K loop unrolled", nsm);
  run<28>("MMA stream + 8 warps of tcgen05.ld on other columns", nsm);
  run<29>("MMA stream + 8 warps of shared stores", nsm);
  run<30>("MMA stream + both", nsm);
  run<31>("3-stage ring, K loop unrolled", nsm);
  run<32>("6-stage ring, K loop unrolled", nsm);
  run<33>("3-stage ring, MMA and producer loops unrolled", nsm);
  run<34>("3-stage ring, unrolled, waits in pairs", nsm);
  run<35>("6-stage ring, unrolled, waits in pairs", nsm);
  run<36>("3-stage ring, unrolled, producer arrives CTA-locally", nsm);
  run<37>("3-stage ring, unrolled, local arrive, leader producer only", nsm);
  run<38>("self-throttled 3 deep, unrolled", nsm);
  run<39>("self-throttled 6 deep, unrolled", nsm);
  run<40>("self-throttled 12 deep, unrolled", nsm);
  run<41>("3-stage ring, unrolled, producer spins on test_wait", nsm);
  run<42>("3-stage ring, unrolled, both spin on test_wait", nsm);
  run<43>("3-stage ring, unrolled, producer polls every 200 ns", nsm);
  run<44>("3-stage ring, unrolled, producer polls every 1000 ns", nsm);
  run<45>("producer folded into the MMA thread (3 slots)", nsm);
  run<1>("kernel (mode 3) again", nsm);
  return 0;
}
