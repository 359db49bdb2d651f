// mlp_eval.cuh -- persistent point-evaluation kernels over a point generator.
//
// A generator `Gen` supplies, on the device:
//   int64_t count() const                  rows to evaluate (may read a device counter)
//   bool point(int64_t i, double p[3], int &shape) const
//   double seed(int64_t i, double f) const (vjp only: the seed of row i given f)
//   void store(int64_t i, double f) const  (where the value goes)
// so the same tile code serves NeuralField.evaluate (explicit points), the
// normal probes of shading.py:84-87 and the frozen head samples of
// shading.py:185-206 without materialising point arrays in HBM.
#pragma once
#include "common.cuh"
#include "mlp_simt.cuh"

namespace dist {

template <typename T, class Gen, bool PAIR = false>
__global__ void __launch_bounds__(SimtTile<T>::NT)
    k_eval_gen(DecView dv, const double *__restrict__ c0, const double *__restrict__ cskip, Gen gen) {
  extern __shared__ __align__(16) char smem[];
  using Tile = SimtTile<T>;
  Tile tile(smem);
  const int64_t n = gen.count();
  const int64_t ntiles = ceil_div(n, Tile::TM);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * Tile::TM;
    if (threadIdx.x < Tile::TM) {
      const int64_t i = base + threadIdx.x;
      double p[3] = {0.0, 0.0, 0.0};
      int s = -1;
      if (i < n && !gen.point(i, p, s)) s = -1;
      tile.shape[threadIdx.x] = s;
      for (int a = 0; a < 3; ++a) tile.pts[threadIdx.x * 3 + a] = p[a];
    }
    __syncthreads();
    if constexpr (PAIR) tile.forward_pair(dv, c0);
    else tile.forward(dv, c0, cskip, false);
    if (threadIdx.x < Tile::TM && base + threadIdx.x < n) gen.store(base + threadIdx.x, tile.f[threadIdx.x]);
    __syncthreads();
  }
}

// Taped forward + reverse sweep per tile.  Column sums of the layer-0 / skip
// pre-activation gradients accumulate into part0[cta][S][np0] /
// parts[cta][S][nskip] as exact fixed-point integers (common.cuh fx_t), so
// the result does not depend on how rows fall into tiles or CTAs; `bad` is
// set on a non-finite contribution.  gpts[i][3] receives seed * df/dp.
template <typename T, class Gen>
__global__ void __launch_bounds__(SimtTile<T>::NT)
    k_vjp_gen(DecView dv, const double *__restrict__ c0, const double *__restrict__ cskip, Gen gen,
              int S, fx_t *__restrict__ part0, fx_t *__restrict__ parts,
              double *__restrict__ gpts, int *__restrict__ bad) {
  extern __shared__ __align__(16) char smem[];
  using Tile = SimtTile<T>;
  Tile tile(smem);
  __shared__ double s_seed[Tile::TM];
  __shared__ double s_seedm[Tile::TM];
  __shared__ double s_gp[Tile::TM * 3];
  __shared__ fx_t s_sum0[kMaxWidth];
  __shared__ fx_t s_sums[kMaxWidth];
  __shared__ int s_shapes[Tile::TM];
  __shared__ int s_nsh;
  const int n0 = dv.np[0];
  const int ns = dv.nskip;
  const int64_t n = gen.count();
  const int64_t ntiles = ceil_div(n, Tile::TM);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * Tile::TM;
    if (threadIdx.x < Tile::TM) {
      const int64_t i = base + threadIdx.x;
      double p[3] = {0.0, 0.0, 0.0};
      int s = -1;
      if (i < n && !gen.point(i, p, s)) s = -1;
      tile.shape[threadIdx.x] = s;
      for (int a = 0; a < 3; ++a) tile.pts[threadIdx.x * 3 + a] = p[a];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int cnt = 0;
      for (int r = 0; r < Tile::TM; ++r) {
        const int s = tile.shape[r];
        if (s < 0) continue;
        bool seen = false;
        for (int q = 0; q < cnt; ++q) seen |= (s_shapes[q] == s);
        if (!seen) s_shapes[cnt++] = s;
      }
      s_nsh = cnt;
    }
    tile.forward(dv, c0, cskip, true);
    if (threadIdx.x < Tile::TM) {
      const int64_t i = base + threadIdx.x;
      const bool ok = i < n && tile.shape[threadIdx.x] >= 0;
      const double fv = tile.f[threadIdx.x];
      s_seed[threadIdx.x] = ok ? gen.seed(i, fv) : 0.0;
      if (i < n) gen.store(i, fv);
    }
    __syncthreads();
    const int nsh = s_nsh;
    for (int q = 0; q < nsh; ++q) {
      const int s = s_shapes[q];
      if (threadIdx.x < Tile::TM) {
        s_seedm[threadIdx.x] = (tile.shape[threadIdx.x] == s) ? s_seed[threadIdx.x] : 0.0;
        for (int a = 0; a < 3; ++a) s_gp[threadIdx.x * 3 + a] = 0.0;
      }
      for (int j = threadIdx.x; j < kMaxWidth; j += blockDim.x) s_sum0[j] = s_sums[j] = 0;
      __syncthreads();
      tile.backward(dv, s_seedm, s_sum0, s_sums, s_gp, bad);
      fx_t *p0 = part0 + ((size_t)blockIdx.x * S + s) * n0;
      for (int j = threadIdx.x; j < n0; j += blockDim.x) p0[j] += s_sum0[j];
      if (ns) {
        fx_t *ps = parts + ((size_t)blockIdx.x * S + s) * ns;
        for (int j = threadIdx.x; j < ns; j += blockDim.x) ps[j] += s_sums[j];
      }
      if (gpts && threadIdx.x < Tile::TM && base + threadIdx.x < n && tile.shape[threadIdx.x] == s)
        for (int a = 0; a < 3; ++a) gpts[(base + threadIdx.x) * 3 + a] = s_gp[threadIdx.x * 3 + a];
      __syncthreads();
    }
  }
}

// explicit arrays (NeuralField.evaluate / HeadBundle.backward with seeds)
struct ArrayGen {
  const double *pts;
  const int32_t *shape;
  const double *seeds;
  double *f;
  int64_t n;
  __device__ int64_t count() const { return n; }
  __device__ bool point(int64_t i, double p[3], int &s) const {
    p[0] = pts[i * 3];
    p[1] = pts[i * 3 + 1];
    p[2] = pts[i * 3 + 2];
    s = shape ? shape[i] : 0;
    return true;
  }
  __device__ double seed(int64_t i, double) const { return seeds[i]; }
  __device__ void store(int64_t i, double v) const {
    if (f) f[i] = v;
  }
  // the tensor-core head kernel's seed interface (heads.cuh ObjGen): the seed
  // is given, so prep() loads it and apply() ignores f
  struct Prep {
    double seed;
  };
  __device__ Prep prep(int64_t i) const { return Prep{seeds ? seeds[i] : 0.0}; }
  __device__ double apply(const Prep &p, double) const { return p.seed; }
};

int sm_count();

// Heads of up to kMaxHeads decoders that share every layer but the last
// (AttributeField's channels, fields.py:332-338): the hidden stack runs once
// per tile, then each head; out[i * m + c].
constexpr int kMaxHeads = 8;
struct HeadSet {
  const void *w[kMaxHeads];   // head weights in the tile's arithmetic type
  double b[kMaxHeads];
  int m;
};

template <typename T>
__global__ void __launch_bounds__(SimtTile<T>::NT)
    k_eval_channels(DecView dv, const double *__restrict__ c0, const double *__restrict__ cskip,
                    ArrayGen gen, HeadSet hs, double *__restrict__ out) {
  extern __shared__ __align__(16) char smem[];
  using Tile = SimtTile<T>;
  Tile tile(smem);
  const int64_t n = gen.count();
  const int64_t ntiles = ceil_div(n, Tile::TM);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * Tile::TM;
    if (threadIdx.x < Tile::TM) {
      const int64_t i = base + threadIdx.x;
      double p[3] = {0.0, 0.0, 0.0};
      int s = -1;
      if (i < n && !gen.point(i, p, s)) s = -1;
      tile.shape[threadIdx.x] = s;
      for (int a = 0; a < 3; ++a) tile.pts[threadIdx.x * 3 + a] = p[a];
    }
    __syncthreads();
    tile.layer0(dv, c0, false);
    for (int l = 1; l <= dv.n_layers - 2; ++l) tile.hidden(dv, l, cskip, false);
    for (int c = 0; c < hs.m; ++c) {
      tile.output_head(dv, reinterpret_cast<const T *>(hs.w[c]), hs.b[c]);
      if (threadIdx.x < Tile::TM && base + threadIdx.x < n) out[(base + threadIdx.x) * hs.m + c] = tile.f[threadIdx.x];
    }
    __syncthreads();
  }
}

template <typename T>
int launch_eval_channels(const DecView &dv, const double *c0, const double *cskip, const ArrayGen &gen,
                         const HeadSet &hs, double *out, cudaStream_t st) {
  using Tile = SimtTile<T>;
  const void *fn = (const void *)k_eval_channels<T>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Tile::fwd_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(eval_channels)");
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, Tile::NT, Tile::fwd_bytes);
  const int64_t tiles = std::max<int64_t>(1, ceil_div(gen.n, Tile::TM));
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)std::max(per_sm, 1) * sm_count());
  k_eval_channels<T><<<grid, Tile::NT, Tile::fwd_bytes, st>>>(dv, c0, cskip, gen, hs, out);
  DIST_CHECK_LAUNCH("k_eval_channels");
  return DIST_OK;
}

template <typename T, class Gen, bool PAIR = false>
int launch_eval_gen(const DecView &dv, const double *c0, const double *cskip, const Gen &gen,
                    int64_t n_bound, cudaStream_t st) {
  using Tile = SimtTile<T>;
  const void *fn = (const void *)k_eval_gen<T, Gen, PAIR>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Tile::fwd_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(eval)");
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, Tile::NT, Tile::fwd_bytes);
  const int64_t tiles = std::max<int64_t>(1, ceil_div(n_bound, Tile::TM));
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)std::max(per_sm, 1) * sm_count());
  k_eval_gen<T, Gen, PAIR><<<grid, Tile::NT, Tile::fwd_bytes, st>>>(dv, c0, cskip, gen);
  DIST_CHECK_LAUNCH("k_eval_gen");
  return DIST_OK;
}

template <typename T, class Gen>
int launch_vjp_gen(const DecView &dv, const double *c0, const double *cskip, const Gen &gen,
                   int64_t n_bound, int S, fx_t *part0, fx_t *parts, double *gpts, int *bad,
                   int grid_cap, int *grid_out, cudaStream_t st) {
  using Tile = SimtTile<T>;
  const void *fn = (const void *)k_vjp_gen<T, Gen>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Tile::vjp_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(vjp)");
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, Tile::NT, Tile::vjp_bytes);
  const int64_t tiles = std::max<int64_t>(1, ceil_div(n_bound, Tile::TM));
  int grid = (int)std::min<int64_t>(tiles, (int64_t)std::max(per_sm, 1) * sm_count());
  grid = std::min(grid, grid_cap);
  *grid_out = grid;
  k_vjp_gen<T, Gen><<<grid, Tile::NT, Tile::vjp_bytes, st>>>(dv, c0, cskip, gen, S, part0, parts,
                                                             gpts, bad);
  DIST_CHECK_LAUNCH("k_vjp_gen");
  return DIST_OK;
}

}  // namespace dist
