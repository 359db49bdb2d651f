// scan.cuh -- stable device-wide stream compaction (predicate -> ascending
// indices), the np.nonzero of tracer.py:158 / shading.py:67,171.
//
// Two passes over 1024-item blocks: per-block counts, then each block sums
// the counts of the blocks before it (L2-resident, a few KB) and ranks its
// own items with a warp-ballot + block scan.  Order is ascending, so the
// result is identical to np.nonzero.  HBM-bound: reads the predicate inputs
// twice and writes 4 B per selected item.
#pragma once
#include "common.cuh"

namespace dist {

constexpr int kScanBlock = 1024;

template <class Pred>
__global__ void k_compact_count(Pred pred, int64_t n, int32_t *__restrict__ bcount) {
  __shared__ int s_w[32];
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const bool f = i < n && pred(i);
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = __popc(m);
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = s_w[threadIdx.x];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) bcount[blockIdx.x] = v;
  }
}

template <class Pred>
__global__ void k_compact_write(Pred pred, int64_t n, const int32_t *__restrict__ bcount,
                                int32_t *__restrict__ out, int32_t *__restrict__ total) {
  __shared__ int s_w[32];
  __shared__ int s_base;
  __shared__ long long s_red[32];
  // prefix of earlier blocks
  long long acc = 0;
  for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) acc += bcount[b];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) s += s_red[w];
    s_base = (int)s;
  }
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const bool f = i < n && pred(i);
  const unsigned m = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_w[warp] = __popc(m);
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = s_w[threadIdx.x];
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (threadIdx.x >= o) incl += t;
    }
    s_w[threadIdx.x] = incl - v;  // exclusive warp offsets
  }
  __syncthreads();
  if (f) out[s_base + s_w[warp] + __popc(m & ((1u << lane) - 1u))] = (int32_t)i;
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    *total = s_base + bcount[blockIdx.x];
  }
}

inline size_t compact_ws(int64_t n) { return sizeof(int32_t) * (size_t)ceil_div(n, kScanBlock) + 256; }

// out[0..count) = ascending i with pred(i); *total (device) = count.
template <class Pred>
int compact(Pred pred, int64_t n, int32_t *out, int32_t *total, int32_t *bcount, cudaStream_t st) {
  if (n <= 0) {
    cudaError_t e = cudaMemsetAsync(total, 0, sizeof(int32_t), st);
    return e == cudaSuccess ? DIST_OK : cuda_fail(e, "compact memset");
  }
  const int nb = (int)ceil_div(n, kScanBlock);
  k_compact_count<<<nb, kScanBlock, 0, st>>>(pred, n, bcount);
  DIST_CHECK_LAUNCH("k_compact_count");
  k_compact_write<<<nb, kScanBlock, 0, st>>>(pred, n, bcount, out, total);
  DIST_CHECK_LAUNCH("k_compact_write");
  return DIST_OK;
}

}  // namespace dist
