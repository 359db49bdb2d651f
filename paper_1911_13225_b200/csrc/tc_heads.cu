// tc_heads.cu -- the memory-light backward on tensor cores: ONE fused
// tcgen05 kernel per tile of 128 frozen head samples (64 per CTA of a pair)
// that runs the taped decoder forward (shading.py:185-206), forms each
// sample's loss seed from its own f (losses.py:54-91, via the generator of
// heads.cuh) and sweeps the gradient back through the hidden layers
// (autodiff.py:220-255) down to the layer-0 pre-activation, whose per-column
// row sums are the only gradient output (the code gradient is their product
// with W0[:D], done once per shape in k_reduce_code_grad).
//
//   * forward phases: as tc_mlp.cu (bf16x3, W^T streamed by TMA), plus the
//     ReLU mask bits of every layer kept in TMEM (columns 256..319) -- the
//     activations themselves are never stored;
//   * backward phases: fp16x2, A = g as ONE fp16 term, each row scaled by a
//     power of two (max in [2^14, 2^15)), B = W (untransposed, fp16 hi + lo,
//     power-of-two layer scale) streamed by a second TMA map, D = g W^T in
//     TMEM (two MMAs per K step instead of three); the epilogue unscales,
//     multiplies by the stored masks and picks the next row scale.  The
//     rounding of g (2^-12) bounds the latent-gradient error at ~4e-4 with
//     random-sign seeds and ~3e-5 with coherent ones (emulated);
//   * the last backward epilogue converts g to exact 128-bit fixed point
//     (common.cuh fx_t), reduces it over the CTA's 64 rows with a warp
//     butterfly and adds the column sums into this CTA's slice of part0: the
//     sums are independent of how rows are partitioned.
#include <cmath>
#include <type_traits>
#include <cstring>

#include "common.cuh"
#include "heads.cuh"
#include "kernels.cuh"
#include "mlp_eval.cuh"
#include "tc_core.cuh"

namespace dist {
namespace tc {

struct HParams {
  DecView dv;
  const double *c0;
  const float *c0f;    // fp32 copy of c0 (kernels.cuh c0_f32)
  const float *bias;   // [G][512]
  const float *w_out;  // [512]
  const float *winv_b; // [G] inverse power-of-two scales of the backward pack
  const float *nrm_b;  // [G] max row l1 norm of each backward W: |g W^T| <= max|g| * nrm
  // nrm_b[G] = max |w_out|: |first backward operand| <= |gout| * max |w_out|
  int n_gemm;
  int S;
  int timeline;        // DIST_TC_TIMELINE: CTA 0 / thread 64 records %globaltimer marks
  fx_t *part0;         // [grid][S][512] exact fixed-point column sums (common.cuh)
  fx_t *parts;         // [grid][S][512] the same for the skip layer's pre-activation (DeepSDF)
  int *bad;            // set on a non-finite / out-of-range contribution
  // DeepSDF skip layer: forward GEMM skipg adds the code part cskf[s] and p . Wsp
  // to its bias; backward phase skipl produces the skip layer's pre-activation
  // gradient, whose column sums (code) and . Wsp (points) it takes
  int skipg, skipl;
  const float *cskf;   // [S][512] fp32 (kernels.cuh c0 layout of cskip)
  double *gpts;        // [n][3] seed * df/dp per row, or null
};

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Mask words indexed by a run-time nh: selects keep the array in registers
// (a dynamic subscript would put it in local memory).
__device__ __forceinline__ uint32_t get4(const uint32_t (&a)[4], int i) {
  return i == 0 ? a[0] : (i == 1 ? a[1] : (i == 2 ? a[2] : a[3]));
}
__device__ __forceinline__ void set4(uint32_t (&a)[4], int i, uint32_t v) {
  a[0] = i == 0 ? v : a[0];
  a[1] = i == 1 ? v : a[1];
  a[2] = i == 2 ? v : a[2];
  a[3] = i == 3 ? v : a[3];
}

// fp64 butterfly over a 16-column chunk (exact when the caller checked the
// binade span); afterwards lanes 2c, 2c+1 both hold the sum of column c
__device__ __forceinline__ void warp_colsum16d(double (&v)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16, n = 8; o >= 2; o >>= 1, n >>= 1) {
    const bool upper = lane & o;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const double send = upper ? v[j] : v[j + n];
      const double keep = upper ? v[j + n] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// exact column sums of a 16-column chunk over the warp's 32 rows (values v in
// true units, zero for rows not counted): the fp64 butterfly when the warp's
// nonzero values span at most 24 binades inside the fixed-point range (then
// exact), else the 128-bit integer butterfly.  Lanes 2c, 2c+1 return the sum of
// column c; nb is set on an out-of-range value.
__device__ __forceinline__ fx_t chunk_sum16(const float (&v)[16], int &nb);

__device__ __forceinline__ void fx_atomic_add(fx_t *dst, fx_t v) {
  // two 64-bit atomics with an explicit carry: exact modulo 2^128 whatever the
  // interleaving of concurrent adders
  unsigned long long *w = reinterpret_cast<unsigned long long *>(dst);
  const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)((unsigned __int128)v >> 64);
  const unsigned long long old = atomicAdd(w, lo);
  atomicAdd(w + 1, hi + ((old + lo < old) ? 1ull : 0ull));
}

// The butterfly on exact fixed-point integers (common.cuh fx_t) over a
// 16-column chunk (registers: 64 per chunk): afterwards lanes 2c and 2c+1
// both hold the sum of column c over the warp's 32 rows.
__device__ __forceinline__ void warp_colsum16x(fx_t (&v)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16, n = 8; o >= 2; o >>= 1, n >>= 1) {
    const bool upper = lane & o;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const fx_t send = upper ? v[j] : v[j + n];
      const fx_t keep = upper ? v[j + n] : v[j];
      v[j] = keep + fx_shfl_xor(send, o);
    }
  }
  v[0] += fx_shfl_xor(v[0], 1);
}

__device__ __forceinline__ fx_t chunk_sum16(const float (&v)[16], int &nb) {
  uint32_t emin = 255u, emax = 0u;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const uint32_t ex = (__float_as_uint(v[e]) >> 23) & 0xffu;
    if (v[e] != 0.f) {
      emin = min(emin, ex);
      emax = max(emax, ex);
    }
  }
  emin = __reduce_min_sync(0xffffffffu, emin);
  emax = __reduce_max_sync(0xffffffffu, emax);
  if (emax < emin || (emax - emin <= 24u && emin >= 55u && emax <= 151u)) {
    double w[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) w[e] = (double)v[e];
    warp_colsum16d(w);
    return fx_from_double(w[0], &nb);
  }
  fx_t w[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) w[e] = fx_from_float(v[e], nb);
  warp_colsum16x(w);
  return w[0];
}

// Sum v[0..63] over the 32 lanes of the warp; afterwards lane l holds the
// column sums of columns 2l and 2l+1 in v[0], v[1].
__device__ __forceinline__ void warp_colsum64(float (&v)[64]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16, n = 32; o >= 1; o >>= 1, n >>= 1) {
    const bool upper = lane & o;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const float send = upper ? v[j] : v[j + n];
      const float keep = upper ? v[j + n] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// debug timeline (DIST_TC_TIMELINE=1): (mark id, %globaltimer) pairs of CTA 0's
// first epilogue thread; read with dist_debug_heads_timeline
static __device__ unsigned long long g_heads_tl[4096];
#define TL(id) DIST_TL_MARK(g_heads_tl, id)

// BWD: backward-only rows (the ReLU-mask record, include/dist.h): f and the
// masks of every layer come from the march's own query of the sample, so the
// forward phases are skipped and a tile is the G backward GEMMs alone.
template <class Gen, bool BWD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_tc_heads(const __grid_constant__ CUtensorMap wfwd, const __grid_constant__ CUtensorMap wbwd,
               HParams P, Gen gen) {
  extern __shared__ __align__(16) char smem_raw[];
  char *smem = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Misc &m = *reinterpret_cast<Misc *>(smem + OFF_MISC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int64_t nrows = gen.count();
  if (nrows <= 0) return;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&m.full[s], 1);
      mbar_init(&m.empty[s], 1);
    }
    mbar_init(&m.dfull[0], 1);
    mbar_init(&m.dfull[1], 1);
    mbar_init(&m.aready, 2);
    mbar_init(&m.aready2, 2);
    mbar_init(&m.afree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&m.tmem_base)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = m.tmem_base;

  const int64_t ntiles = ceil_div(nrows, 2 * ROWS);
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int G = P.n_gemm;
  const int NPH = 2 * G;  // forward GEMM phases, then backward phases

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = cluster; t < ntiles; t += nclusters)
        for (int ph = BWD ? G : 0; ph < NPH; ++ph) {
          const bool fwd = !BWD && ph < G;   // compile-time false in the backward-only kernel
          const int l = fwd ? ph : 2 * G - 1 - ph;
          const CUtensorMap *map = fwd ? &wfwd : &wbwd;
          for (int nh = 0; nh < 2; ++nh)
            for (int kc = 0; kc < NKB; ++kc, ++it) {
              const int s = it % STAGES;
              mbar_wait(&m.empty[s], ((it / STAGES) & 1) ^ 1);
              if (rank == 0) mbar_arrive_expect_tx(&m.full[s], 2 * STAGE_BYTES);
              const uint32_t dst = smem_u32(smem + OFF_B + s * STAGE_BYTES);
              const int y = nh * 256 + (int)rank * 128;
              tma_load_2sm(dst, map, &m.full[s], kc * 64, (l * 2 + 0) * KDIM + y);
              tma_load_2sm(dst + B_TILE, map, &m.full[s], kc * 64, (l * 2 + 1) * KDIM + y);
            }
        }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA) =====
    if (rank == 0 && lane == 0) {
      uint32_t it = 0, phase = 0;
      const uint32_t a_hi = smem_u32(smem + OFF_AHI), a_lo = smem_u32(smem + OFF_ALO);
      for (int64_t t = cluster; t < ntiles; t += nclusters)
        for (int ph = BWD ? G : 0; ph < NPH; ++ph, ++phase) {
          mbar_wait(&m.aready, phase & 1);
          tc_fence_after();
          // One GEMM: the N-half and K loops fully unrolled (a loop that waits
          // on a barrier gets a YIELD on its back-edge, which costs the MMA
          // issue ~25% of the tensor pipe: scripts/tc_pattern_bench.cu), one
          // copy per product scheme so each phase's issue code is contiguous
          // (the forward and backward variants interleaved per stage doubled
          // the instruction footprint of either).
          auto gemm = [&](auto fwd_tag) {
            constexpr bool FWD = decltype(fwd_tag)::value;
            // BWD: a tile's first operand is built in A_lo (parked there during
            // the previous tile's last GEMM); every later one in A_hi
            const uint32_t ab = (!FWD && BWD && ph == G) ? a_lo : a_hi;
#pragma unroll
            for (int nh = 0; nh < 2; ++nh) {
              const uint32_t d = tmem + nh * 128;
#pragma unroll
              for (int kc = 0; kc < NKB; ++kc, ++it) {
                if (nh == 0 && kc == NKB / 2) {   // second half of A: written after the first
                  mbar_wait(&m.aready2, phase & 1);
                  tc_fence_after();
                }
                const int s = it % STAGES;
                mbar_wait(&m.full[s], (it / STAGES) & 1);
                tc_fence_after();
                const uint32_t b_hi = smem_u32(smem + OFF_B + s * STAGE_BYTES), b_lo = b_hi + B_TILE;
                if constexpr (FWD) {   // forward: bf16x3
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const uint32_t ak = kc * (ROWS * 128) + q * 32;
                    const uint64_t dah = sdesc(a_hi + ak), dal = sdesc(a_lo + ak);
                    const uint64_t dbh = sdesc(b_hi + q * 32), dbl = sdesc(b_lo + q * 32);
                    mma_2sm<false>(d, dah, dbh, (kc | q) ? 1u : 0u);
                    mma_2sm<false>(d, dah, dbl, 1u);
                    mma_2sm<false>(d, dal, dbh, 1u);
                  }
                } else {               // backward: fp16x2, g x (W_hi + W_lo)
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const uint64_t dah = sdesc(ab + kc * (ROWS * 128) + q * 32);
                    mma_2sm<true>(d, dah, sdesc(b_hi + q * 32), (kc | q) ? 1u : 0u);
                    mma_2sm<true>(d, dah, sdesc(b_lo + q * 32), 1u);
                  }
                }
                commit_2sm(&m.empty[s]);
                // phases that write the next operand: A's K blocks 0..3 are free
                // once the nh = 1 MMAs are past them (tc_mlp.cu, same barrier)
                if (nh == 1 && kc == NKB / 2 - 1 && (ph < G - 1 || (ph >= G && ph < 2 * G - 1)))
                  commit_2sm(&m.afree);
              }
              commit_2sm(&m.dfull[nh]);
            }
          };
          if (!BWD && ph < G) gemm(std::true_type{});   // never in the backward-only kernel
          else gemm(std::false_type{});
        }
    }
  } else {
    // ===== epilogue warps =====
    // DIST_TC_TIMELINE bit 0 records the full kernel, bit 1 the backward-only one
    const bool tl_on = (P.timeline & (BWD ? 2 : 1)) && blockIdx.x == 0 && threadIdx.x == 64;
    int tl_i = 0;
    const int q = warp & 3;
    const int sub = (warp - 2) >> 2;
    const int row = (q & 1) * 32 + lane;
    const int half = q >> 1;
    const bool row_thread = (sub == 0 && half == 0);
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    // the next GEMM's A is announced in two halves (K blocks 0..3, 4..7): the MMA
    // warp starts its first N half while the epilogue writes the second
    auto a_ready_lo = [&] { if (warp == 2 && lane == 0) mbar_arrive_cluster(&m.aready, 0); };
    auto a_ready_hi = [&] { if (warp == 2 && lane == 0) mbar_arrive_cluster(&m.aready2, 0); };
    auto a_ready_all = [&] { a_ready_lo(); a_ready_hi(); };
    auto announce_lo = [&] {
      fence_proxy_async();
      tc_fence_before();
      epi_sync();
      a_ready_lo();
    };
    // mask bits of layer output ml, this thread's 2 x 64 columns: TMEM cols 256 + 8 ml + 4 sub
    auto mask_addr = [&](int ml) { return tq + 256 + ml * 8 + sub * 4; };
    const int n0 = P.dv.np[0];
    uint32_t phase = 0;
    uint32_t afree_n = 0;   // afree phases consumed (phases that write the next operand)
    // [64] per-row head gradient; m.ray is unused by this kernel, so gout does
    // not alias the m.xch row exchange
    float *gout = reinterpret_cast<float *>(&m.ray[0]);
    // the next tile's sample point is fetched during the current tile's last
    // backward GEMM (a dependent chain of global loads)
    // backward-only rows: this thread's 4 words of each layer's mask record
    // (tc_mlp.cu put_mask: words 4 q4 .. 4 q4 + 3, q4 = 2 half + sub)
    const int mq = 4 * (2 * half + sub);
    auto fetch = [&](int64_t tt, double (&q)[3], int &ss, const uint32_t *&mr) {
      const int64_t g2 = tt * (2 * ROWS) + (int64_t)rank * ROWS + row;
      q[0] = q[1] = q[2] = 0.0;
      ss = -1;
      mr = nullptr;
      if (tt < ntiles && g2 < nrows && !gen.point(g2, q, ss)) ss = -1;
      if constexpr (BWD) {
        if (ss >= 0) mr = gen.masks_rec(g2);
      }
    };
    double nxp[3];
    int nxs;
    const uint32_t *nxm;
    fetch(cluster, nxp, nxs, nxm);
    // BWD: the first backward operand is mask_G * w_out alone -- the row's seed
    // scales the first backward epilogue instead (one fp32 rounding) -- so the
    // next tile's operand is built during this tile's last GEMM, into A_lo
    // (unused by backward GEMMs), which that tile's first GEMM reads
    const float sc0 = BWD ? pow2_scale(P.nrm_b[G]) : 1.f;   // |w_out| <= nrm_b[G]
    bool have_park = false;
    // this thread's 64 fp16 operand columns of N half nh (32 packed words)
    auto a0_words = [&](uint32_t wlo, uint32_t whi, int nh, uint32_t (&w)[32]) {
      const int cb = nh * 256 + half * 128 + sub * 64;
#pragma unroll
      for (int j = 0; j < 64; j += 8) {
        float wo[8];
        ldg8(P.w_out + cb + j, wo);
        const uint32_t wb = (j < 32 ? wlo : whi) >> (j & 31);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float x0 = ((wb >> (2 * i)) & 1u) ? wo[2 * i] * sc0 : 0.f;
          const float x1 = ((wb >> (2 * i + 1)) & 1u) ? wo[2 * i + 1] * sc0 : 0.f;
          const __half2 hv = __floats2half2_rn(x0, x1);
          w[j / 2 + i] = *reinterpret_cast<const uint32_t *>(&hv);
        }
      }
    };
    auto a0_store = [&](int nh, const uint32_t (&w)[32]) {   // -> A_lo (the BWD first operand)
      const int cb = nh * 256 + half * 128 + sub * 64;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<uint4 *>(smem + OFF_ALO + a_off(row, cb + 8 * j)) =
            make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
    };
    // masks of layers 0..G of a record into this thread's TMEM mask columns;
    // returns mask G's words (lo, hi of N half 0, lo, hi of N half 1)
    auto load_masks = [&](const uint32_t *mr, uint32_t (&mg)[4]) {
#pragma unroll 1
      for (int m0 = 0; m0 <= G; m0 += 4) {
        uint4 a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[i] = make_uint4(0u, 0u, 0u, 0u);
          if (mr && m0 + i <= G) a[i] = __ldg(reinterpret_cast<const uint4 *>(mr + (m0 + i) * 16 + mq));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (m0 + i > G) break;
          const uint32_t mk[4] = {a[i].x, a[i].y, a[i].z, a[i].w};
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(mask_addr(m0 + i)),
                       "r"(mk[0]), "r"(mk[1]), "r"(mk[2]), "r"(mk[3])
                       : "memory");
          if (m0 + i == G) {
            mg[0] = mk[0]; mg[1] = mk[1]; mg[2] = mk[2]; mg[3] = mk[3];
          }
        }
      }
      tmem_wait_st();
    };
    for (int64_t t = cluster; t < ntiles; t += nclusters) {
      TL(1);
      const int64_t gi = t * (2 * ROWS) + (int64_t)rank * ROWS + row;
      double p[3] = {nxp[0], nxp[1], nxp[2]};
      const int s = nxs;
      const uint32_t *const mrec = nxm;

      if (row_thread) m.shape[row] = s;
      const float px = (float)p[0], py = (float)p[1], pz = (float)p[2];
      // the DeepSDF skip layer's extra input terms (code part + p . Wsp) for n
      // consecutive columns, added to the bias of forward GEMM P.skipg
      auto skip_terms = [&](int col, float *bb, int n) {
        const int ns = P.dv.nskip;
        const float *cf = P.cskf + (size_t)(s < 0 ? 0 : s) * ns + col;
        for (int e0 = 0; e0 < n; e0 += 8) {
          float w0[8], w1[8], w2[8], c8[8];
          ldg8(P.dv.Wspf + col + e0, w0);
          ldg8(P.dv.Wspf + ns + col + e0, w1);
          ldg8(P.dv.Wspf + 2 * ns + col + e0, w2);
          ldg8(cf + e0, c8);
#pragma unroll
          for (int e = 0; e < 8; ++e) bb[e0 + e] += fmaf(pz, w2[e], fmaf(py, w1[e], fmaf(px, w0[e], c8[e])));
        }
      };
      float head = 0.f;
      typename Gen::Prep sp{};
      float gr_b = 0.f;    // BWD: this row's seed, applied in the first backward epilogue
      if constexpr (BWD) {
        if (!have_park) {   // else: built in A_lo during the previous tile's last GEMM
          uint32_t mg[4];
          load_masks(mrec, mg);
#pragma unroll 1
          for (int nh = 0; nh < 2; ++nh) {
            uint32_t w[32];
            a0_words(nh ? mg[2] : mg[0], nh ? mg[3] : mg[1], nh, w);
            a0_store(nh, w);
          }
        }
        fence_proxy_async();
        tc_fence_before();
        epi_sync();
        named_arrive(2, 2 * N_EPI_WARPS * 32);   // pairs with phase G-1's post (no A0 max exchange)
        a_ready_all();
        TL(6);
        // the seed: its loads overlap the first backward GEMM
        double go = 0.0;
        if (row_thread && gi < nrows && s >= 0) {
          sp = gen.prep(gi);
          const double fv = gen.f_rec(gi);
          gen.store(gi, fv);
          go = gen.apply(sp, fv) * head_dact(P.dv.final_act, fv);
        }
        if (row_thread) gout[row] = (float)go;
        epi_sync();
        TL(5);
        gr_b = gout[row];
      } else {
      // ---- layer 0 (folded bias + p . W0p, fp32) + mask 0 ----
      {
        const float *c0f = P.c0f + (size_t)(s < 0 ? 0 : s) * n0;
        uint32_t mk[4] = {0, 0, 0, 0};
        for (int nh = 0; nh < 2; ++nh) {
          const int cb = nh * 256 + half * 128 + sub * 64;
#pragma unroll 2
          for (int j = 0; j < 64; j += 8) {
            float x[8], w0[8], w1[8], w2[8], cf[8];
            ldg8(P.dv.W0pf + cb + j, w0);
            ldg8(P.dv.W0pf + n0 + cb + j, w1);
            ldg8(P.dv.W0pf + 2 * n0 + cb + j, w2);
            ldg8(c0f + cb + j, cf);
            uint32_t bits = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float v = fmaf(pz, w2[e], fmaf(py, w1[e], fmaf(px, w0[e], cf[e])));
              const bool on = s >= 0 && v > 0.f;
              x[e] = on ? v : 0.f;
              bits |= (on ? 1u : 0u) << e;
            }
            set4(mk, nh * 2 + (j >> 5), get4(mk, nh * 2 + (j >> 5)) | (bits << (j & 31)));
            put8<false>(smem, row, cb + j, x);
          }
        }
        tmem_st4(mask_addr(0), mk);
      }
      fence_proxy_async();
      tc_fence_before();
      epi_sync();
      a_ready_all();
      TL(2);
      // the seed's loads, issued once layer 0 is handed to the MMA warp so
      // they land during the forward GEMMs
      if (row_thread && gi < nrows && s >= 0) sp = gen.prep(gi);
      // ---- forward hidden layers ----
      // The nh = 0 half of each forward GEMM is processed while the nh = 1
      // MMAs run: its packed A words are parked in the TMEM columns just read
      // and copied to A once the GEMM is done (tc_mlp.cu, same scheme).
      for (int l = 0; l < G; ++l, ++phase) {
        const bool last = (l == G - 1);
        const float *bias = P.bias + (size_t)l * KDIM;
        uint32_t mk[4] = {0, 0, 0, 0};
        // early half (nh = 0): bias loaded per 8 columns (latency hidden under
        // the nh = 1 MMAs), packed words returned in r for parking
        auto fwd_early = [&](int c, uint32_t (&r)[32]) -> uint32_t {
          const int cb = half * 128 + sub * 64;
          float v[32];
          tmem_ld32(tq + sub * 64 + c * 32, v);
          uint32_t bits = 0;
#pragma unroll
          for (int g8 = 0; g8 < 4; ++g8) {
            float x[8], bb[8];
            ldg8(bias + cb + c * 32 + g8 * 8, bb);
            if (l == P.skipg) skip_terms(cb + c * 32 + g8 * 8, bb, 8);
            if (last) {
              float wo[8];
              ldg8(P.w_out + cb + c * 32 + g8 * 8, wo);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float y = v[g8 * 8 + e] + bb[e];
                bits |= (y > 0.f ? 1u : 0u) << (g8 * 8 + e);
                head = fmaf(y > 0.f ? y : 0.f, wo[e], head);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float y = v[g8 * 8 + e] + bb[e];
                x[e] = y > 0.f ? y : 0.f;
                bits |= (y > 0.f ? 1u : 0u) << (g8 * 8 + e);
              }
              uint32_t hi[4], lo[4];
              pack8<false>(x, hi, lo);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                r[g8 * 4 + i] = hi[i];
                r[16 + g8 * 4 + i] = lo[i];
              }
            }
          }
          return bits;
        };
        // late half (nh = 1): on the critical path, bias loads issued ahead
        auto fwd_late = [&](int c) -> uint32_t {
          const int cb = 256 + half * 128 + sub * 64;
          float v[32], bbc[32];
          ldg32(bias + cb + c * 32, bbc);
          if (l == P.skipg) skip_terms(cb + c * 32, bbc, 32);
          tmem_ld32(tq + 128 + sub * 64 + c * 32, v);
          uint32_t bits = 0;
#pragma unroll
          for (int g8 = 0; g8 < 4; ++g8) {
            float x[8], wo[8];
            const float *bb = bbc + g8 * 8;
            if (last) ldg8(P.w_out + cb + c * 32 + g8 * 8, wo);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float y = v[g8 * 8 + e] + bb[e];
              x[e] = y > 0.f ? y : 0.f;
              bits |= (y > 0.f ? 1u : 0u) << (g8 * 8 + e);
              if (last) head = fmaf(x[e], wo[e], head);
            }
            if (!last) put8<false>(smem, row, cb + c * 32 + g8 * 8, x);
          }
          return bits;
        };
        mbar_wait(&m.dfull[0], phase & 1);
        TL(3);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {   // early half (nh = 0)
          uint32_t r[32];
          set4(mk, c, fwd_early(c, r));
          if (!last) tmem_st32(tq + sub * 64 + c * 32, r);
        }
        if (!last) {
          tmem_wait_st();
          mbar_wait(&m.afree, afree_n & 1);
          ++afree_n;
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {   // parked words -> A (K blocks 0..3)
            float v[32];
            tmem_ld32(tq + sub * 64 + c * 32, v);
            const int k0 = half * 128 + sub * 64 + c * 32;
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8) {
              uint32_t hi[4], lo[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                hi[i] = __float_as_uint(v[g8 * 4 + i]);
                lo[i] = __float_as_uint(v[16 + g8 * 4 + i]);
              }
              st8(smem, row, k0 + g8 * 8, hi, lo);
            }
          }
          announce_lo();
        }
        mbar_wait(&m.dfull[1], phase & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 2; ++c) set4(mk, 2 + c, fwd_late(c));   // nh = 1
        tmem_st4(mask_addr(l + 1), mk);
        tc_fence_before();
        if (!last) {
          fence_proxy_async();
          epi_sync();
          a_ready_hi();
          TL(4);
        }
      }
      // ---- head: the four partial dot products of each row ----
      m.xch[half * 2 + sub][row] = head;
      epi_sync();
      }   // !BWD
      float rinv = BWD ? 1.f / sc0 : 1.f;   // 1 / (this row's scale of the A operand now in smem)
      float amax = BWD ? P.nrm_b[G] : 0.f;  // max |g| of this row's A operand (true units; BWD: before the seed)
      if constexpr (!BWD) {
      // ---- seed, d loss / d h_G ----
      double go = 0.0;
      if (row_thread) {
        const double sum = (double)m.xch[0][row] + (double)m.xch[1][row] +
                           (double)m.xch[2][row] + (double)m.xch[3][row] + P.dv.b_out;
        const double fv = head_act(P.dv.final_act, sum);
        if (gi < nrows && s >= 0) {
          gen.store(gi, fv);
          const double sd = gen.apply(sp, fv);
          go = sd * head_dact(P.dv.final_act, fv);
        }
      }
      if (row_thread) gout[row] = (float)go;   // gout does not alias m.xch: no barrier before
      epi_sync();
      TL(5);
      {
        // one pass: the scale comes from the bound |gout| * max|w_out|; the true
        // row max of what is written feeds the first backward phase's bound
        const float gr = gout[row];
        uint32_t mk[4];
        tmem_ld4(mask_addr(G), mk);
        const float sc = pow2_scale(fabsf(gr) * P.nrm_b[G]);
        rinv = 1.f / sc;
        float part = 0.f;
        for (int nh = 0; nh < 2; ++nh) {
          const int cb = nh * 256 + half * 128 + sub * 64;
#pragma unroll 2
          for (int j = 0; j < 64; j += 8) {
            float x[8], wo[8];
            ldg8(P.w_out + cb + j, wo);
            const uint32_t wb = get4(mk, nh * 2 + (j >> 5)) >> (j & 31);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              x[e] = ((wb >> e) & 1u) ? (gr * sc) * wo[e] : 0.f;
              part = fmaxf(part, fabsf(x[e]));
            }
            put8h(smem, row, cb + j, x);
          }
        }
        m.xch[half * 2 + sub][row] = part * rinv;
      }
      fence_proxy_async();
      tc_fence_before();
      epi_sync();
      amax = fmaxf(fmaxf(m.xch[0][row], m.xch[1][row]), fmaxf(m.xch[2][row], m.xch[3][row]));
      named_arrive(2, 2 * N_EPI_WARPS * 32);   // this read happens before phase G-1 posts its maxima
      a_ready_all();
      TL(6);
      }   // !BWD
      // The DeepSDF skip layer's share of the backward: its pre-activation
      // gradient g_{z_skip} (the operand phase P.skipl just wrote to A, true
      // units x * rinv) feeds the code gradient through W_skip's code rows
      // (exact column sums into P.parts, per shape) and the sample points
      // through its xyz rows (gps, added to d/dp with the layer-0 term).
      float gps[3] = {0.f, 0.f, 0.f};
      auto skip_backward = [&](float ri) {
        const int ns = P.dv.nskip;
        int nb = 0;
        int shapes_done = 0;
        for (int guard = 0; guard < ROWS; ++guard) {
          int next = 0x7fffffff;
          for (int r = 0; r < ROWS; ++r) {
            const int sr = m.shape[r];
            if (sr >= 0 && sr >= shapes_done && sr < next) next = sr;
          }
          if (next == 0x7fffffff) break;
          const bool mine = (s == next);
          for (int nh = 0; nh < 2; ++nh) {
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              const int cb = nh * 256 + half * 128 + sub * 64 + c * 16;
              float v[16];
#pragma unroll
              for (int g2 = 0; g2 < 2; ++g2) {
                const uint4 q4 = *reinterpret_cast<const uint4 *>(smem + OFF_AHI + a_off(row, cb + g2 * 8));
                const uint32_t wds[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 f2 = __half22float2(*reinterpret_cast<const __half2 *>(&wds[i]));
                  v[g2 * 8 + 2 * i] = mine ? f2.x * ri : 0.f;
                  v[g2 * 8 + 2 * i + 1] = mine ? f2.y * ri : 0.f;
                }
              }
              if (P.gpts && mine) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  gps[0] = fmaf(v[e], __ldg(P.dv.Wspf + cb + e), gps[0]);
                  gps[1] = fmaf(v[e], __ldg(P.dv.Wspf + ns + cb + e), gps[1]);
                  gps[2] = fmaf(v[e], __ldg(P.dv.Wspf + 2 * ns + cb + e), gps[2]);
                }
              }
              const fx_t r = chunk_sum16(v, nb);
              if (!(lane & 1)) fx_atomic_add(P.parts + ((size_t)blockIdx.x * P.S + next) * ns + cb + (lane >> 1), r);
            }
          }
          shapes_done = next + 1;
        }
        if (nb) atomicOr(P.bad, 1);
      };
      // ---- backward through GEMM layers G-1 .. 0 ----
      for (int gl = G - 1; gl >= 0; --gl, ++phase) {
        if (gl == 0) fetch(t + nclusters, nxp, nxs, nxm);
        uint32_t mk[4];
        tmem_ld4(mask_addr(gl), mk);   // written in the forward, readable now
        // BWD: the first backward GEMM ran on mask_G * w_out; the seed enters here
        const float gfac = (BWD && gl == G - 1) ? gr_b : 1.f;
        if constexpr (BWD) {
          if (gl == 0) {
            // this tile's masks are in mk / done: the next tile's go to TMEM and
            // its first operand is parked while the last GEMM runs
            have_park = false;
            if (t + nclusters < ntiles) {
              uint32_t mg[4];
              load_masks(nxm, mg);
#pragma unroll 1
              for (int nh = 0; nh < 2; ++nh) {
                uint32_t w[32];
                a0_words(nh ? mg[2] : mg[0], nh ? mg[3] : mg[1], nh, w);
                a0_store(nh, w);
              }
              have_park = true;
            }
          }
        }
        // D = (g / rinv) (W / winv_b): true dgrad = D * unscale
        const float unscale = rinv * P.winv_b[gl] * gfac;
        if (gl > 0) {
          // One pass: the scale comes from a rigorous bound, |g_next| <= amax *
          // nrm_b[gl], so the fp16 operand cannot overflow; the true row max
          // of what is written becomes the next phase's amax.
          const float sc = pow2_scale(amax * fabsf(gfac) * P.nrm_b[gl]);
          const float f = unscale * sc;   // exact (powers of two) except the BWD seed factor
          rinv = 1.f / sc;
          float part = 0.f;
          // 8 masked, scaled values of chunk (nh, c) -> 4 packed fp16 words
          auto bwd8 = [&](const float (&v)[32], uint32_t bits, int g8, uint32_t (&h)[4]) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int e = g8 * 8 + 2 * i;
              const float x0 = ((bits >> e) & 1u) ? v[e] * f : 0.f;
              const float x1 = ((bits >> (e + 1)) & 1u) ? v[e + 1] * f : 0.f;
              part = fmaxf(part, fmaxf(fabsf(x0), fabsf(x1)));
              const __half2 hv = __floats2half2_rn(x0, x1);
              h[i] = *reinterpret_cast<const uint32_t *>(&hv);
            }
          };
          mbar_wait(&m.dfull[0], phase & 1);
          TL(7);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {   // early half (nh = 0), parked in TMEM
            float v[32];
            tmem_ld32(tq + sub * 64 + c * 32, v);
            const uint32_t bits = get4(mk, c);
            uint32_t r[32];
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8) {
              uint32_t h[4];
              bwd8(v, bits, g8, h);
#pragma unroll
              for (int i = 0; i < 4; ++i) r[g8 * 4 + i] = h[i];
            }
#pragma unroll
            for (int i = 16; i < 32; ++i) r[i] = 0u;
            tmem_st32(tq + sub * 64 + c * 32, r);
          }
          tmem_wait_st();
          mbar_wait(&m.afree, afree_n & 1);
          ++afree_n;
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {   // parked words -> A (K blocks 0..3)
            float v[32];
            tmem_ld32(tq + sub * 64 + c * 32, v);
            const int k0 = half * 128 + sub * 64 + c * 32;
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8)
              *reinterpret_cast<uint4 *>(smem + OFF_AHI + a_off(row, k0 + g8 * 8)) =
                  make_uint4(__float_as_uint(v[g8 * 4]), __float_as_uint(v[g8 * 4 + 1]),
                             __float_as_uint(v[g8 * 4 + 2]), __float_as_uint(v[g8 * 4 + 3]));
          }
          announce_lo();
          mbar_wait(&m.dfull[1], phase & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {   // nh = 1
            float v[32];
            tmem_ld32(tq + 128 + sub * 64 + c * 32, v);
            const uint32_t bits = get4(mk, 2 + c);
            const int k0 = 256 + half * 128 + sub * 64 + c * 32;
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8) {
              uint32_t h[4];
              bwd8(v, bits, g8, h);
              *reinterpret_cast<uint4 *>(smem + OFF_AHI + a_off(row, k0 + g8 * 8)) =
                  make_uint4(h[0], h[1], h[2], h[3]);
            }
          }
          // post this warp's part max; barrier 2 orders it after every warp's
          // read of the previous phase's maxima (bar.arrive there, below)
          named_sync(2, 2 * N_EPI_WARPS * 32);
          m.xch[half * 2 + sub][row] = part * rinv;
          tc_fence_before();
          fence_proxy_async();
          epi_sync();
          amax = fmaxf(fmaxf(m.xch[0][row], m.xch[1][row]), fmaxf(m.xch[2][row], m.xch[3][row]));
          if (gl >= 2) named_arrive(2, 2 * N_EPI_WARPS * 32);
          a_ready_hi();
          TL(8);
          if (gl == P.skipl) skip_backward(rinv);
        } else {
          mbar_wait(&m.dfull[1], phase & 1);
          TL(7);
          mbar_wait(&m.dfull[0], phase & 1);
          tc_fence_after();
          // g_pre0 = D * mask0 * unscale; column sums over the CTA's rows, per
          // shape.  TMEM is read inside the shape loop (usually one pass), so no
          // per-thread copy of the 128 values is kept (it lived in local memory).
          float *red = reinterpret_cast<float *>(smem + OFF_AHI);  // A is free now: [2][512] fx_t
          if (P.gpts) {
            // d loss / d p = g_pre0 . W0p^T per row: this thread's 128 columns,
            // then the row's four part sums through smem (after `red`)
            float *gp = red + 8 * KDIM;   // [3][4][64], after the [2][512] fixed-point column sums
            float acc[3] = {gps[0], gps[1], gps[2]};   // + the skip layer's xyz rows (skip_backward)
            for (int nh = 0; nh < 2; ++nh) {
              const int cb = nh * 256 + half * 128 + sub * 64;
#pragma unroll 1
              for (int c = 0; c < 2; ++c) {
                float v[32];
                tmem_ld32(tq + nh * 128 + sub * 64 + c * 32, v);
                const uint32_t bits = get4(mk, nh * 2 + c);
#pragma unroll
                for (int g8 = 0; g8 < 4; ++g8) {
                  float w0[8], w1[8], w2[8];
                  const int col = cb + c * 32 + g8 * 8;
                  ldg8(P.dv.W0pf + col, w0);
                  ldg8(P.dv.W0pf + n0 + col, w1);
                  ldg8(P.dv.W0pf + 2 * n0 + col, w2);
#pragma unroll
                  for (int e = 0; e < 8; ++e) {
                    const float g = ((bits >> (g8 * 8 + e)) & 1u) ? v[g8 * 8 + e] * unscale : 0.f;
                    acc[0] = fmaf(g, w0[e], acc[0]);
                    acc[1] = fmaf(g, w1[e], acc[1]);
                    acc[2] = fmaf(g, w2[e], acc[2]);
                  }
                }
              }
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) gp[(a * 4 + half * 2 + sub) * ROWS + row] = acc[a];
            tc_fence_before();
            epi_sync();
            if (row_thread && gi < nrows && s >= 0)
#pragma unroll
              for (int a = 0; a < 3; ++a)
                P.gpts[gi * 3 + a] = (double)gp[(a * 4) * ROWS + row] + (double)gp[(a * 4 + 1) * ROWS + row] +
                                     (double)gp[(a * 4 + 2) * ROWS + row] + (double)gp[(a * 4 + 3) * ROWS + row];
          }
          int shapes_done = 0;
          fx_t *redx = reinterpret_cast<fx_t *>(red);   // [2][512] fixed point
          for (int guard = 0; guard < ROWS; ++guard) {
            // next shape = smallest shape id > previous (uniform across threads)
            int next = 0x7fffffff;
            for (int r = 0; r < ROWS; ++r) {
              const int sr = m.shape[r];
              if (sr >= 0 && sr >= shapes_done && sr < next) next = sr;
            }
            if (next == 0x7fffffff) break;
            const bool mine = (s == next);
            int nb = 0;
            for (int nh = 0; nh < 2; ++nh) {
#pragma unroll 1
              for (int c = 0; c < 4; ++c) {
                // The column sums must be exact (common.cuh fx_t) so that they
                // do not depend on which rows share a tile, a CTA or a rank.
                // Fast path: when the warp's nonzero values of this 16-column
                // chunk span at most 24 binades (and sit inside the fixed-point
                // range) their fp64 sums are exact, so one fp64 butterfly and
                // one conversion per column give the exact integer; otherwise
                // every value is converted and summed as a 128-bit integer.
                float v[16];
                tmem_ld16(tq + nh * 128 + sub * 64 + c * 16, v);
                const uint32_t bits = mine ? (get4(mk, nh * 2 + (c >> 1)) >> ((c & 1) * 16)) : 0u;
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = ((bits >> e) & 1u) ? v[e] * unscale : 0.f;
                // lanes 2c', 2c'+1 end up holding column c' of the chunk; the
                // two row-warps (q&1 = 0, 1) of the chunk combine in smem below
                const int col = nh * 256 + half * 128 + sub * 64 + c * 16 + (lane >> 1);
                const fx_t r = chunk_sum16(v, nb);
                if (!(lane & 1)) redx[(q & 1) * 512 + col] = r;
              }
            }
            if (nb) atomicOr(P.bad, 1);
            tc_fence_before();
            epi_sync();
            TL(10);
            fx_t *dst = P.part0 + ((size_t)blockIdx.x * P.S + next) * n0;
            for (int col = threadIdx.x - 64; col < KDIM; col += N_EPI_WARPS * 32)
              dst[col] += redx[col] + redx[512 + col];
            epi_sync();
            shapes_done = next + 1;
            TL(9);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
}

}  // namespace tc

// ---------------------------------------------------------------------------
bool tc_heads_supported(const DecView &dv) {
  // the head kernel's forward is bf16x3 in both split modes: slot 0 of a bf16x3
  // decoder, slot 3 of an fp16x3 one (tc_mlp.cu packs)
  const int fs = dv.prec == DIST_PREC_FP16X3 ? 3 : 0;
  return tc_supported(dv) && dv.tc_w[1] != nullptr && dv.tc_w[fs] != nullptr;
}


template <class Gen, bool BWD>
static int launch_heads_impl(const DecView &dv, const double *c0, const double *cs, const Gen &gen,
                             int64_t n_bound, int S, fx_t *part0, fx_t *parts, int *bad, int grid_cap,
                             int *grid_out, cudaStream_t st, double *gpts) {
  CUtensorMap mf, mb;
  const int fs = dv.prec == DIST_PREC_FP16X3 ? 3 : 0;   // bf16x3 forward pack
  int rc = tc_make_map(dv, fs, &mf);
  if (!rc) rc = tc_make_map(dv, 1, &mb);
  if (rc) return rc;
  tc::HParams P;
  P.dv = dv;
  P.c0 = c0;
  P.c0f = c0_f32(c0, S, dv.np[0]);
  P.bias = dv.tc_bias[fs];
  P.w_out = dv.tc_bias[fs] + (size_t)(dv.n_layers - 2) * tc::KDIM;
  P.winv_b = dv.tc_bias[1];
  P.nrm_b = dv.tc_bias[1] + (dv.n_layers - 2);

  P.n_gemm = dv.n_layers - 2;
  P.S = S;
  {
    const char *tl = getenv("DIST_TC_TIMELINE");
    P.timeline = tl ? atoi(tl) : 0;
  }
  P.part0 = part0;
  P.parts = parts;
  P.bad = bad;
  P.skipg = dv.skip > 0 ? dv.skip - 1 : -1;
  P.skipl = dv.skip > 0 ? dv.skip : -1;
  P.cskf = dv.skip > 0 ? c0_f32(cs, S, dv.nskip) : nullptr;
  P.gpts = gpts;
  const void *fn = (const void *)tc::k_tc_heads<Gen, BWD>;
  static int attr_dev = -1;   // per instantiation: set once per device
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  if (attr_dev != cur_dev) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BYTES);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc heads)");
    attr_dev = cur_dev;
  }
  int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_bound, 128), sm_count() / 2));
  pairs = std::min(pairs, grid_cap / 2);
  *grid_out = 2 * pairs;
  tc::k_tc_heads<Gen, BWD><<<2 * pairs, tc::THREADS, tc::SMEM_BYTES, st>>>(mf, mb, P, gen);
  DIST_CHECK_LAUNCH("k_tc_heads");
  return DIST_OK;
}

template <class Gen>
int launch_tc_heads(const DecView &dv, const double *c0, const double *cs, const Gen &gen, int64_t n_bound,
                    int S, fx_t *part0, fx_t *parts, int *bad, int grid_cap, int *grid_out, cudaStream_t st,
                    double *gpts) {
  return launch_heads_impl<Gen, false>(dv, c0, cs, gen, n_bound, S, part0, parts, bad, grid_cap, grid_out, st,
                                       gpts);
}

int launch_tc_heads_bwd(const DecView &dv, const double *c0, const double *cs, const ObjGen &gen,
                        int64_t n_bound, int S, fx_t *part0, fx_t *parts, int *bad, int grid_cap,
                        int *grid_out, cudaStream_t st) {
  return launch_heads_impl<ObjGen, true>(dv, c0, cs, gen, n_bound, S, part0, parts, bad, grid_cap, grid_out, st,
                                         nullptr);
}

extern "C" DIST_API int dist_debug_heads_timeline(unsigned long long *out, int n) {
  return cudaMemcpyFromSymbol(out, tc::g_heads_tl, sizeof(unsigned long long) * (size_t)std::min(n, 4096)) ==
                 cudaSuccess ? 0 : -1;
}

template int launch_tc_heads<ObjGen>(const DecView &, const double *, const double *, const ObjGen &, int64_t,
                                     int, fx_t *, fx_t *, int *, int, int *, cudaStream_t, double *);
template int launch_tc_heads<ArrayGen>(const DecView &, const double *, const double *, const ArrayGen &,
                                       int64_t, int, fx_t *, fx_t *, int *, int, int *, cudaStream_t, double *);

}  // namespace dist
