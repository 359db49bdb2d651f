// scan.cuh -- stable device-wide stream compaction (predicate -> ascending
// indices), the np.nonzero of tracer.py:158 / shading.py:67,171.
//
// Two passes over 4096-item blocks (4 items per thread): per-block counts, then each block sums
// the counts of the blocks before it (L2-resident, a few KB) and ranks its
// own items with a warp-ballot + block scan.  Order is ascending, so the
// result is identical to np.nonzero.  HBM-bound: reads the predicate inputs
// twice and writes 4 B per selected item.
#pragma once
#include "common.cuh"

namespace dist {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;                         // items per thread
constexpr int kScanBlock = kScanThreads * kScanItems; // items per block

// Item (u, t) of block b is b*kScanBlock + u*kScanThreads + t: every u is one
// coalesced sweep, and (u, warp, lane) order is ascending item order.  The
// kScanItems predicates of a thread are evaluated before any is used, so each
// thread keeps that many loads in flight.
template <class Pred>
__device__ __forceinline__ void scan_ballots(Pred pred, int64_t n, unsigned (&m)[kScanItems]) {
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  bool f[kScanItems];
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    const int64_t i = base + (int64_t)u * kScanThreads;
    f[u] = i < n && pred(i);
  }
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) m[u] = __ballot_sync(0xffffffffu, f[u]);
}

template <class Pred>
__global__ void __launch_bounds__(kScanThreads) k_compact_count(Pred pred, int64_t n, int32_t *__restrict__ bcount) {
  __shared__ int s_w[32];
  unsigned m[kScanItems];
  scan_ballots(pred, n, m);
  int c = 0;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) c += __popc(m[u]);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = s_w[threadIdx.x];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) bcount[blockIdx.x] = v;
  }
}

template <class Pred>
__global__ void __launch_bounds__(kScanThreads) k_compact_write(Pred pred, int64_t n, const int32_t *__restrict__ bcount,
                                int32_t *__restrict__ out, int32_t *__restrict__ total,
                                int32_t *__restrict__ inv) {
  __shared__ int s_w[kScanItems * 32];   // (u, warp) counts -> exclusive offsets
  __shared__ int s_base;
  __shared__ long long s_red[32];
  unsigned m[kScanItems];
  scan_ballots(pred, n, m);   // loads in flight while the block prefix is summed
  // prefix of earlier blocks
  long long acc = 0;
  for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) acc += bcount[b];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_red[warp] = acc;
#pragma unroll
    for (int u = 0; u < kScanItems; ++u) s_w[u * 32 + warp] = __popc(m[u]);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    long long s = s_red[lane];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_base = (int)s;
    // exclusive scan of the kScanItems*32 (u, warp) counts, u-major
    int carry = 0;
#pragma unroll
    for (int u = 0; u < kScanItems; ++u) {
      const int v = s_w[u * 32 + lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      s_w[u * 32 + lane] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const unsigned below = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    if (m[u] >> lane & 1u) {
      const int64_t i = base + (int64_t)u * kScanThreads;
      const int pos = s_base + s_w[u * 32 + warp] + __popc(m[u] & below);
      out[pos] = (int32_t)i;
      if (inv) inv[i] = pos;   // rank of item i among the selected (unselected: untouched)
    }
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    *total = s_base + bcount[blockIdx.x];
  }
}

inline size_t compact_ws(int64_t n) { return sizeof(int32_t) * (size_t)ceil_div(n, kScanBlock) + 256; }

// out[0..count) = ascending i with pred(i); *total (device) = count; if inv
// is given, inv[out[r]] = r (the inverse map, written only for selected i).
template <class Pred>
int compact(Pred pred, int64_t n, int32_t *out, int32_t *total, int32_t *bcount, cudaStream_t st,
            int32_t *inv = nullptr) {
  if (n <= 0) {
    cudaError_t e = cudaMemsetAsync(total, 0, sizeof(int32_t), st);
    return e == cudaSuccess ? DIST_OK : cuda_fail(e, "compact memset");
  }
  const int nb = (int)ceil_div(n, kScanBlock);
  k_compact_count<<<nb, kScanThreads, 0, st>>>(pred, n, bcount);
  DIST_CHECK_LAUNCH("k_compact_count");
  k_compact_write<<<nb, kScanThreads, 0, st>>>(pred, n, bcount, out, total, inv);
  DIST_CHECK_LAUNCH("k_compact_write");
  return DIST_OK;
}

}  // namespace dist
