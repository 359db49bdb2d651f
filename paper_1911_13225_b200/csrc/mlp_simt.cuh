// mlp_simt.cuh -- CTA-tile SIMT evaluation of the latent-conditioned decoder.
//
// Restates NeuralField._forward (fields.py:239-247) and the reverse sweep of
// autodiff.backward over affine/relu/tanh (autodiff.py:95-129, 220-255) for a
// tile of TM query rows, in fp64 (the reference's arithmetic) or
// fp32.  Activations of the tile stay in shared memory, k-major
// (Ht[k][row]), for all layers; the latent half of layer 0 is folded into a
// per-shape bias (SURVEY 0 finding 8) computed once per call in fp64.
//
// Thread (rg, cg) of NT = TM/8*64 threads owns rows rg*8..rg*8+7 and columns
// cg + 64c, c < N/64: weight loads of a warp are 128-byte coalesced rows of
// W[k][:], activation loads are warp-broadcasts, and the column-strided
// ownership makes the k-major stores bank-conflict free.
#pragma once
#include "common.cuh"

namespace dist {

template <typename T>
struct SimtTraits;
template <>
struct SimtTraits<float> {
  static constexpr int TM = 32;
  static constexpr int PAD = 4;
};
template <>
struct SimtTraits<double> {
  static constexpr int TM = 16;
  static constexpr int PAD = 2;
};

template <typename T>
struct SimtTile {
  static constexpr int WI = sizeof(T) == 4 ? 1 : 0;  // DecView copy index
  static constexpr int TM = SimtTraits<T>::TM;
  static constexpr int NT = TM / 8 * 64;
  static constexpr int LD = TM + SimtTraits<T>::PAD;
  static constexpr int MB = TM / 8;  // mask bytes per column

  // shared memory layout (bytes)
  static constexpr size_t off_H = 0;
  static constexpr size_t off_pts = off_H + sizeof(T) * kMaxWidth * LD;
  static constexpr size_t off_shape = off_pts + sizeof(double) * TM * 3;
  static constexpr size_t off_f = off_shape + sizeof(int) * TM;
  static constexpr size_t off_red = off_f + sizeof(double) * TM;
  static constexpr size_t off_mask = off_red + sizeof(double) * NT;
  static constexpr size_t fwd_bytes = off_mask;
  static constexpr size_t vjp_bytes = off_mask + (size_t)kMaxLayers * kMaxWidth * MB;

  T *H;
  double *pts;   // [TM][3]
  int *shape;    // [TM]  (-1 = empty row)
  double *f;     // [TM]
  double *red;   // [NT]
  uint8_t *mask; // [L][512][MB]

  __device__ explicit SimtTile(char *smem) {
    H = reinterpret_cast<T *>(smem + off_H);
    pts = reinterpret_cast<double *>(smem + off_pts);
    shape = reinterpret_cast<int *>(smem + off_shape);
    f = reinterpret_cast<double *>(smem + off_f);
    red = reinterpret_cast<double *>(smem + off_red);
    mask = reinterpret_cast<uint8_t *>(smem + off_mask);
  }

  // Layer 0 with the latent part folded: pre = c0[shape] + p . W0p; relu.
  __device__ void layer0(const DecView &dv, const double *__restrict__ c0, bool keep_mask) {
    const int tid = threadIdx.x, cg = tid & 63, rg = tid >> 6;
    const int n0 = dv.np[0];
    for (int c = 0; c < kMaxWidth / 64; ++c) {
      const int col = cg + 64 * c;
      if (col >= n0) break;
      const double w0 = dv.W0p[col], w1 = dv.W0p[n0 + col], w2 = dv.W0p[2 * n0 + col];
      uint32_t bits = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int row = rg * 8 + r;
        const int s = shape[row];
        double v = 0.0;
        if (s >= 0) {
          v = c0[(size_t)s * n0 + col];
          v = fma(pts[row * 3 + 0], w0, v);
          v = fma(pts[row * 3 + 1], w1, v);
          v = fma(pts[row * 3 + 2], w2, v);
        }
        bits |= (v > 0.0 ? 1u : 0u) << r;
        H[col * LD + row] = (T)(!(v <= 0.0) ? v : 0.0);   // np.maximum: NaN propagates
      }
      if (keep_mask) mask[(size_t)col * MB + rg] = (uint8_t)bits;
    }
    __syncthreads();
  }

  // acc[c][r] = sum_k H[k][rg*8+r] * W[k][cg+64c]
  __device__ __forceinline__ void gemm(const T *__restrict__ W, int K, int N, T (&acc)[8][8]) {
    const int tid = threadIdx.x, cg = tid & 63, rg = tid >> 6;
    const int nc = N >> 6;
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[c][r] = (T)0;
    const T *hrow = H + rg * 8;
    const T *wcol = W + cg;
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
      T a[8], w[8];
      if constexpr (sizeof(T) == 4) {
        const float4 *p = reinterpret_cast<const float4 *>(hrow + k * LD);
        float4 x0 = p[0], x1 = p[1];
        a[0] = x0.x; a[1] = x0.y; a[2] = x0.z; a[3] = x0.w;
        a[4] = x1.x; a[5] = x1.y; a[6] = x1.z; a[7] = x1.w;
      } else {
        const double2 *p = reinterpret_cast<const double2 *>(hrow + k * LD);
        double2 x0 = p[0], x1 = p[1], x2 = p[2], x3 = p[3];
        a[0] = x0.x; a[1] = x0.y; a[2] = x1.x; a[3] = x1.y;
        a[4] = x2.x; a[5] = x2.y; a[6] = x3.x; a[7] = x3.y;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) w[c] = (c < nc) ? __ldg(wcol + (size_t)k * N + 64 * c) : (T)0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[c][r] = fma(a[r], w[c], acc[c][r]);
    }
    __syncthreads();  // every thread is done reading H before it is overwritten
  }

  // hidden layer l forward: H <- relu(H @ W_l + b_l)  (+ skip input terms)
  __device__ void hidden(const DecView &dv, int l, const double *__restrict__ cskip,
                         bool keep_mask) {
    const int tid = threadIdx.x, cg = tid & 63, rg = tid >> 6;
    const int K = dv.kp[l], N = dv.np[l];
    T acc[8][8];
    gemm(reinterpret_cast<const T *>(dv.W[WI][l]), K, N, acc);
    const T *bias = reinterpret_cast<const T *>(dv.bias[WI][l]);
    const bool is_skip = (l == dv.skip);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = cg + 64 * c;
      if (col < N) {
        const T bb = bias[col];
        uint32_t bits = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int row = rg * 8 + r;
          T v = acc[c][r] + bb;
          if (is_skip) {
            const int s = shape[row];
            double e = 0.0;
            if (s >= 0) {
              e = cskip[(size_t)s * N + col];
              e = fma(pts[row * 3 + 0], dv.Wsp[col], e);
              e = fma(pts[row * 3 + 1], dv.Wsp[N + col], e);
              e = fma(pts[row * 3 + 2], dv.Wsp[2 * N + col], e);
            }
            v = (T)((double)v + e);
          }
          bits |= (v > (T)0 ? 1u : 0u) << r;
          acc[c][r] = !(v <= (T)0) ? v : (T)0;   // np.maximum: NaN propagates
        }
        if (keep_mask) mask[((size_t)l * kMaxWidth + col) * MB + rg] = (uint8_t)bits;
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = cg + 64 * c;
      if (col < N) {
        T *dst = H + col * LD + rg * 8;
#pragma unroll
        for (int r = 0; r < 8; ++r) dst[r] = acc[c][r];
      }
    }
    __syncthreads();
  }

  // Output layer: f[row] = head(H[:,row] . w_out + b_out).
  __device__ void output(const DecView &dv) {
    output_head(dv, reinterpret_cast<const T *>(dv.w_out[WI]), dv.b_out);
  }
  // the same with another head (w, b_out) on this decoder's last hidden layer
  // (AttributeField channels, dist_eval_channels)
  __device__ void output_head(const DecView &dv, const T *w, double b_out) {
    const int tid = threadIdx.x;
    const int K = dv.np[dv.n_layers - 2];
    constexpr int P = NT / TM;  // threads per row
    const int row = tid % TM, part = tid / TM;
    T acc = (T)0;
    for (int k = part; k < K; k += P) acc = fma(H[k * LD + row], w[k], acc);
    red[tid] = (double)acc;
    __syncthreads();
    if (tid < TM) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < P; ++p) s += red[p * TM + tid];
      s += b_out;
      f[tid] = head_act(dv.final_act, s);
    }
    __syncthreads();
  }

  // Full forward for rows already staged in pts/shape; result in f[].
  __device__ void forward(const DecView &dv, const double *c0, const double *cskip,
                          bool keep_mask) {
    layer0(dv, c0, keep_mask);
    for (int l = 1; l <= dv.n_layers - 2; ++l) hidden(dv, l, cskip, keep_mask);
    output(dv);
  }

  // ---- (mid, diff) pair mode: rows 2i / 2i+1 hold the probes p+ / p- of one
  // central difference (shading.py:84-87).  They are carried through the
  // network as m = (h+ + h-)/2 and d = (h+ - h-)/2, so the difference never
  // cancels; the result row 2i+1 receives f+ - f-.
  __device__ static __forceinline__ void relu_pair(double m, double d, double &mo, double &dd) {
    const double ad = fabs(d);
    if (m - ad > 0.0) {          // both probes active: exact pass-through
      mo = m;
      dd = d;
    } else if (m + ad <= 0.0) {  // both inactive
      mo = 0.0;
      dd = 0.0;
    } else {                     // straddles the kink
      const double a = fmax(m + d, 0.0), b = fmax(m - d, 0.0);
      mo = 0.5 * (a + b);
      dd = 0.5 * (a - b);
    }
  }

  __device__ void layer0_pair(const DecView &dv, const double *__restrict__ c0) {
    const int tid = threadIdx.x, cg = tid & 63, rg = tid >> 6;
    const int n0 = dv.np[0];
    for (int c = 0; c < kMaxWidth / 64; ++c) {
      const int col = cg + 64 * c;
      if (col >= n0) break;
      const double w0 = dv.W0p[col], w1 = dv.W0p[n0 + col], w2 = dv.W0p[2 * n0 + col];
#pragma unroll
      for (int r = 0; r < 8; r += 2) {
        const int row = rg * 8 + r;
        const int s = shape[row];
        double m = 0.0, d = 0.0;
        if (s >= 0) {
          double vp = c0[(size_t)s * n0 + col], vm = vp;
          vp = fma(pts[row * 3 + 0], w0, vp);
          vp = fma(pts[row * 3 + 1], w1, vp);
          vp = fma(pts[row * 3 + 2], w2, vp);
          vm = fma(pts[row * 3 + 3], w0, vm);
          vm = fma(pts[row * 3 + 4], w1, vm);
          vm = fma(pts[row * 3 + 5], w2, vm);
          const double a = vp > 0.0 ? vp : 0.0, b = vm > 0.0 ? vm : 0.0;
          m = 0.5 * (a + b);
          d = 0.5 * (a - b);
        }
        H[col * LD + row] = (T)m;
        H[col * LD + row + 1] = (T)d;
      }
    }
    __syncthreads();
  }

  __device__ void hidden_pair(const DecView &dv, int l) {
    const int tid = threadIdx.x, cg = tid & 63, rg = tid >> 6;
    const int K = dv.kp[l], N = dv.np[l];
    T acc[8][8];
    gemm(reinterpret_cast<const T *>(dv.W[WI][l]), K, N, acc);
    const T *bias = reinterpret_cast<const T *>(dv.bias[WI][l]);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = cg + 64 * c;
      if (col < N) {
        const double bb = (double)bias[col];
#pragma unroll
        for (int r = 0; r < 8; r += 2) {
          double mo, dd;
          relu_pair((double)acc[c][r] + bb, (double)acc[c][r + 1], mo, dd);
          acc[c][r] = (T)mo;
          acc[c][r + 1] = (T)dd;
        }
        T *dst = H + col * LD + rg * 8;
#pragma unroll
        for (int r = 0; r < 8; ++r) dst[r] = acc[c][r];
      }
    }
    __syncthreads();
  }

  __device__ void output_pair(const DecView &dv) {
    const int tid = threadIdx.x;
    const int K = dv.np[dv.n_layers - 2];
    const T *w = reinterpret_cast<const T *>(dv.w_out[WI]);
    constexpr int P = NT / TM;
    const int row = tid % TM, part = tid / TM;
    T acc = (T)0;
    for (int k = part; k < K; k += P) acc = fma(H[k * LD + row], w[k], acc);
    red[tid] = (double)acc;
    __syncthreads();
    if (tid < TM) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < P; ++p) s += red[p * TM + tid];
      f[tid] = s;
    }
    __syncthreads();
    if (tid < TM && (tid & 1)) {
      const double om = f[tid - 1] + dv.b_out, od = f[tid];
      // f+ - f- without cancellation: tanh(a) - tanh(b) = sinh(a - b) / (cosh a cosh b)
      if (dv.final_act == 0)
        f[tid] = sinh(2.0 * od) / (cosh(om + od) * cosh(om - od));
      else if (dv.final_act == 1)
        f[tid] = 2.0 * od;
      else
        f[tid] = head_act(2, om + od) - head_act(2, om - od);
      f[tid - 1] = head_act(dv.final_act, om);
    }
    __syncthreads();
  }

  __device__ void forward_pair(const DecView &dv, const double *c0) {
    layer0_pair(dv, c0);
    for (int l = 1; l <= dv.n_layers - 2; ++l) hidden_pair(dv, l);
    output_pair(dv);
  }

  // Reverse sweep after forward(keep_mask=true).  seed[row] (shared, TM
  // entries, 0 for empty rows) multiplies f.  Accumulates the column sums of
  // the layer-0 (and skip-layer) pre-activation gradients into gsum0/gsums
  // (shared double[512] each) and writes d f/d p * seed to gpts[row][3].
  __device__ void backward(const DecView &dv, const double *seed, fx_t *gsum0,
                           fx_t *gsums, double *gpts, int *bad) {
    const int tid = threadIdx.x, cg = tid & 63, rg = tid >> 6;
    const int L = dv.n_layers;
    // head: g[row][k] = seed * (1 - f^2) * w_out[k], masked by layer L-2
    {
      const int K = dv.np[L - 2];
      const T *w = reinterpret_cast<const T *>(dv.w_out[WI]);
      for (int c = 0; c < 8; ++c) {
        const int col = cg + 64 * c;
        if (col >= K) break;
        const uint32_t bits = mask[((size_t)(L - 2) * kMaxWidth + col) * MB + rg];
        const T wk = w[col];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int row = rg * 8 + r;
          const double fr = f[row];
          const double gh = seed[row] * head_dact(dv.final_act, fr);
          H[col * LD + row] = ((bits >> r) & 1u) ? (T)(gh * (double)wk) : (T)0;
        }
      }
      __syncthreads();
    }
    for (int l = L - 2; l >= 1; --l) {
      if (l == dv.skip) colsum(dv.np[l], gsums, gpts, dv.Wsp, dv.np[l], bad);
      // g_in[row][k] = sum_n G[row][n] * W_l[k][n]  -> GEMM with Wt [np][kp]
      const int K = dv.np[l], N = dv.kp[l];
      T acc[8][8];
      gemm(reinterpret_cast<const T *>(dv.Wt[WI][l]), K, N, acc);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = cg + 64 * c;
        if (col < N) {
          const uint32_t bits = mask[((size_t)(l - 1) * kMaxWidth + col) * MB + rg];
          T *dst = H + col * LD + rg * 8;
#pragma unroll
          for (int r = 0; r < 8; ++r) dst[r] = ((bits >> r) & 1u) ? acc[c][r] : (T)0;
        }
      }
      __syncthreads();
    }
    colsum(dv.np[0], gsum0, gpts, dv.W0p, dv.np[0], bad);
  }

  // gsum[col] += sum_rows G[col][row] (exact fixed point, common.cuh);
  // gpts[row][a] += sum_col G[col][row] * Wp[a][col]
  __device__ void colsum(int N, fx_t *gsum, double *gpts, const double *Wp, int ldp, int *bad) {
    const int tid = threadIdx.x;
    int nb = 0;
    for (int col = tid; col < N; col += NT) {
      fx_t s = 0;
#pragma unroll 4
      for (int r = 0; r < TM; ++r) s += fx_from_double((double)H[col * LD + r], &nb);
      gsum[col] += s;
    }
    if (nb) atomicOr(bad, 1);
    if (gpts) {
      constexpr int P = NT / TM;
      const int row = tid % TM, part = tid / TM;
      double a0 = 0, a1 = 0, a2 = 0;
      for (int col = part; col < N; col += P) {
        const double g = (double)H[col * LD + row];
        a0 = fma(g, Wp[col], a0);
        a1 = fma(g, Wp[ldp + col], a1);
        a2 = fma(g, Wp[2 * ldp + col], a2);
      }
      __syncthreads();
      red[tid] = a0;
      __syncthreads();
      if (tid < TM) {
        double s = 0;
        for (int p = 0; p < P; ++p) s += red[p * TM + tid];
        gpts[tid * 3 + 0] += s;
      }
      __syncthreads();
      red[tid] = a1;
      __syncthreads();
      if (tid < TM) {
        double s = 0;
        for (int p = 0; p < P; ++p) s += red[p * TM + tid];
        gpts[tid * 3 + 1] += s;
      }
      __syncthreads();
      red[tid] = a2;
      __syncthreads();
      if (tid < TM) {
        double s = 0;
        for (int p = 0; p < P; ++p) s += red[p * TM + tid];
        gpts[tid * 3 + 2] += s;
      }
    }
    __syncthreads();
  }
};

}  // namespace dist
