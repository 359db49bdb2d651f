// tc_core.cuh -- tcgen05 / TMEM / TMA building blocks shared by the
// split-precision decoder kernels (tc_mlp.cu forward, tc_heads.cu fused
// forward + backward).  See tc_mlp.cu for the design.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace dist {
namespace tc {

constexpr int ROWS = 64;                     // rows per CTA (128 per pair)
constexpr int KDIM = 512;
constexpr int NKB = KDIM / 64;               // 64-element K blocks (128 B swizzle rows)
constexpr int A_PART = NKB * ROWS * 128;     // 64 KB per hi / lo
constexpr int B_TILE = 128 * 128;            // 128 n-rows x 64 k bf16 = 16 KB
constexpr int STAGE_BYTES = 2 * B_TILE;      // hi + lo
constexpr int STAGES = 3;
constexpr int OFF_AHI = 0;
constexpr int OFF_ALO = A_PART;
constexpr int OFF_B = 2 * A_PART;
constexpr int OFF_MISC = OFF_B + STAGES * STAGE_BYTES;   // 229376
constexpr int N_EPI_WARPS = 8;
constexpr int THREADS = (2 + N_EPI_WARPS) * 32;          // producer, MMA, 8 epilogue warps
// k_tc_mlp adds two "finish" warps that apply each tile's row results (the
// march update, survivor append; the eval store) off the epilogue's critical
// path.  12 warps keep the register cap of 10 (3 warps per SM sub-partition).
constexpr int FIN0 = 2 + N_EPI_WARPS;
constexpr int THREADS_MLP = (FIN0 + 2) * 32;
constexpr int TMEM_COLS = 512;

struct Misc {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t dfull[2];
  uint64_t aready;    // next layer's A, K blocks 0..3 (output columns 0..255) written
  uint64_t aready2;   // ... and K blocks 4..7
  uint64_t afree;     // the GEMM's nh = 1 MMAs have consumed A's K blocks 0..3
  uint64_t tk_bar[2]; // fluid march: tile ticket k is in tk_base/tk_cnt[k & 1]
  int64_t tk_base[2]; //   (published by CTA 0's scheduler thread into both CTAs)
  int32_t tk_cnt[2];  //   rows in the tile; 0 = no more tiles
  uint64_t fin_full;  // k_tc_mlp: a tile's row results posted (g_fin) ...
  uint64_t fin_empty; // ... and read by the finish warps
  int32_t fin_stop;   // no more tiles
  uint64_t nx_full;   // k_tc_mlp: the next tile's rows are in g_next (finish warps) ...
  uint64_t nx_empty;  // ... and were read by the epilogue
  uint32_t tmem_base;
  int32_t go, cur, cnt, nan;
  int32_t ray[ROWS];
  int32_t shape[ROWS];
  float xch[4][ROWS];   // per-row exchange: row max (scaling), then head partial sums
};
constexpr int SMEM_BYTES = OFF_MISC + (int)sizeof(Misc) + 1024;  // + alignment slack
static_assert(SMEM_BYTES <= 232448, "shared memory budget");

// ---- PTX helpers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx)
               : "memory");
}
// arrive on the barrier at the same offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *b, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(b)), "r"(rank));
  // default semantics (release, CTA scope) as CUTLASS's ClusterBarrier::arrive:
  // .release.cluster compiles to MEMBAR.ALL.GPU, which waits for every
  // outstanding global store (the march update) on the operand hand-off path.
  // The operand writes reach the tensor core through fence.proxy.async.
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void epi_sync() {  // named barrier over the epilogue warps
  asm volatile("bar.sync 1, %0;" ::"n"(N_EPI_WARPS * 32) : "memory");
}
// producer / consumer named barriers (count = arriving + syncing threads)
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_load_2sm(uint32_t dst, const CUtensorMap *map, uint64_t *bar,
                                             int x, int y) {
  const uint32_t mb = smem_u32(bar) & 0xFEFFFFFFu;  // leader CTA's barrier
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mb), "r"(x), "r"(y)
      : "memory");
}
// K-major, 128B-swizzled UMMA shared-memory descriptor (SBO = 1024 B).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8-row core-matrix groups 1024 B apart
  d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptors: {BF16|F16} x {BF16|F16} -> F32, K-major A/B,
// M=128 (cta_group::2), N=256.
constexpr uint32_t IDESC_BF16 =
    (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t IDESC_F16 = (1u << 4) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

template <bool F16>
__device__ __forceinline__ void mma_2sm(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(a), "l"(b), "n"(F16 ? IDESC_F16 : IDESC_BF16), "r"(acc));
}
__device__ __forceinline__ void commit_2sm(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
          "r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Two 32-column TMEM loads in flight, one wait (the accumulator and the
// correction accumulator of the same columns).
__device__ __forceinline__ void tmem_ld32x2(uint32_t ta, uint32_t tb, float (&v)[32], float (&w)[32]) {
  uint32_t r[32], s[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]),
        "=r"(s[7]), "=r"(s[8]), "=r"(s[9]), "=r"(s[10]), "=r"(s[11]), "=r"(s[12]), "=r"(s[13]),
        "=r"(s[14]), "=r"(s[15]), "=r"(s[16]), "=r"(s[17]), "=r"(s[18]), "=r"(s[19]),
        "=r"(s[20]), "=r"(s[21]), "=r"(s[22]), "=r"(s[23]), "=r"(s[24]), "=r"(s[25]),
        "=r"(s[26]), "=r"(s[27]), "=r"(s[28]), "=r"(s[29]), "=r"(s[30]), "=r"(s[31])
      : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = __uint_as_float(r[i]);
    w[i] = __uint_as_float(s[i]);
  }
}

// 8 consecutive fp32 constants (32-byte aligned) through the read-only path
__device__ __forceinline__ void ldg8(const float *p, float (&x)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
  const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
  x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}

// 32 consecutive fp32 constants (128-byte aligned), issued ahead of a TMEM load
__device__ __forceinline__ void ldg32(const float *p, float (&x)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p) + i);
    x[4 * i] = a.x; x[4 * i + 1] = a.y; x[4 * i + 2] = a.z; x[4 * i + 3] = a.w;
  }
}

// Debug phase timeline (DIST_TC_TIMELINE=1): CTA 0's first epilogue thread
// appends (mark id << 56 | %globaltimer) to a per-kernel device buffer.
#define DIST_TL_MARK(buf, id)                                                          \
  do {                                                                                \
    if (tl_on && tl_i < 4096) {                                                       \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      buf[tl_i++] = ((unsigned long long)(id) << 56) | (t_ & 0xFFFFFFFFFFFFFFull);    \
    }                                                                                 \
  } while (0)

// byte offset of A[row][k] (bf16) inside one 64 KB hi/lo part
__device__ __forceinline__ uint32_t a_off(int row, int k) {
  const int kb = k >> 6, kk = k & 63;
  const int chunk = (kk >> 3) ^ (row & 7);
  return (uint32_t)(kb * (ROWS * 128) + row * 128 + chunk * 16 + (kk & 7) * 2);
}

// split x into hi + lo of the MMA element type (x - hi is exact in fp32)
template <bool F16>
__device__ __forceinline__ void split2(float x, uint16_t &h, uint16_t &l) {
  if constexpr (F16) {
    const __half hh = __float2half_rn(x);
    h = __half_as_ushort(hh);
    l = __half_as_ushort(__float2half_rn(x - __half2float(hh)));
  } else {
    const __nv_bfloat16 hh = __float2bfloat16_rn(x);
    h = __bfloat16_as_ushort(hh);
    l = __bfloat16_as_ushort(__float2bfloat16_rn(x - __bfloat162float(hh)));
  }
}

// split 8 activations into packed hi / lo 16-bit pairs of the MMA element type
template <bool F16>
__device__ __forceinline__ void pack8(const float (&x)[8], uint32_t (&hi)[4], uint32_t (&lo)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (F16) {
      // packed: one cvt.rn.f16x2.f32 for hi, one back to f32x2, one for lo
      const __half2 h = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
      const float2 hf = __half22float2(h);
      const __half2 l = __floats2half2_rn(x[2 * i] - hf.x, x[2 * i + 1] - hf.y);
      hi[i] = *reinterpret_cast<const uint32_t *>(&h);
      lo[i] = *reinterpret_cast<const uint32_t *>(&l);
    } else {
      // one cvt.rn.bf16x2 per pair; bf16 -> f32 is a 16-bit shift
      const __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
      const uint32_t hu = *reinterpret_cast<const uint32_t *>(&h);
      const float r0 = x[2 * i] - __uint_as_float(hu << 16);
      const float r1 = x[2 * i + 1] - __uint_as_float(hu & 0xFFFF0000u);
      const __nv_bfloat162 l = __floats2bfloat162_rn(r0, r1);
      hi[i] = hu;
      lo[i] = *reinterpret_cast<const uint32_t *>(&l);
    }
  }
}

// store packed hi / lo words of 8 consecutive activations (k0 % 8 == 0) of `row`
__device__ __forceinline__ void st8(char *smem, int row, int k0, const uint32_t *hi, const uint32_t *lo) {
  const uint32_t off = a_off(row, k0);
  *reinterpret_cast<uint4 *>(smem + OFF_AHI + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4 *>(smem + OFF_ALO + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

// write 8 consecutive activations (k0..k0+7, k0 % 8 == 0) of `row` as hi/lo
template <bool F16>
__device__ __forceinline__ void put8(char *smem, int row, int k0, const float (&x)[8]) {
  uint32_t hi[4], lo[4];
  pack8<F16>(x, hi, lo);
  st8(smem, row, k0, hi, lo);
}

// ReLU mask bits of 8 non-negative values from their packed hi halves (element
// 2i low / 2i+1 high half of hi[i]): bit e = (high byte of element e's half
// != 0).  That is x > 0 except below 2^-16 of the fp16 scale (row maxima sit
// near 2^14) or 2^-125 in bf16 -- far under the split arithmetic's own
// resolution of the ReLU kink.  Gathered with byte permutes and a multiply
// instead of 8 compares and selects.
__device__ __forceinline__ uint32_t nz_bits8(const uint32_t (&hi)[4]) {
  const uint32_t a = (__byte_perm(hi[0], hi[1], 0x7531) + 0x7f7f7f7fu) & 0x80808080u;
  const uint32_t b = (__byte_perm(hi[2], hi[3], 0x7531) + 0x7f7f7f7fu) & 0x80808080u;
  // (w * 0x00204081) moves bit 7 of byte k to bit 28 + k (no carries); the
  // high words place the 4 flags of a at bits 0..3 and of b at bits 4..7
  return (__umulhi(a, 0x00204081u << 4) | __umulhi(b, 0x00204081u << 8)) & 0xffu;
}

template <bool F16>
__device__ __forceinline__ uint32_t put8m(char *smem, int row, int k0, const float (&x)[8]) {
  uint32_t hi[4], lo[4];
  pack8<F16>(x, hi, lo);
  st8(smem, row, k0, hi, lo);
  return nz_bits8(hi);
}

// 32 columns of this warp's TMEM lanes <- 32 registers (the early half's
// packed A words parked in the accumulator columns they came from)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&h)[4], const uint32_t (&l)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// write 8 consecutive values (k0 % 8 == 0) of `row` as fp16 into A_hi only
// (the single-term fp16 activation operand of the backward GEMMs)
__device__ __forceinline__ void put8h(char *smem, int row, int k0, const float (&x)[8]) {
  uint32_t h[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 v = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
    h[i] = *reinterpret_cast<const uint32_t *>(&v);
  }
  *reinterpret_cast<uint4 *>(smem + OFF_AHI + a_off(row, k0)) = make_uint4(h[0], h[1], h[2], h[3]);
}

// power of two that puts a row maximum `mx` in [2^14, 2^15) (fp16 operands)
__device__ __forceinline__ float pow2_scale(float mx) {
  return mx > 0.f ? ldexpf(1.f, min(max(14 - ilogbf(mx), -126), 126)) : 1.f;
}

}  // namespace tc
}  // namespace dist
