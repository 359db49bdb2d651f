// mlp_small.cuh -- one-ray-per-thread SIMT evaluation of NARROW decoders
// (every hidden layer <= kSmallWidth wide: the reference's tiny_net
// 5-16-16-1 of conftest.py:33-39, C1).
//
// The CTA-tile kernel of mlp_simt.cuh pads every layer to 64 columns and
// spreads one 16-row tile over 128 threads; for a 16-wide network that is 32x
// the necessary FMAs, and a step of a few thousand rays costs ~25 us.  Here
// the whole decoder (true widths, no padding) is staged in shared memory once
// per launch and each thread evaluates its own ray with its activations in a
// private shared-memory column ([width][NT], conflict-free).
//
// Arithmetic is the tile kernel's, operation for operation, so results are
// bit-identical to it: layer 0 in fp64 (c0 + p.W0p, fma in a fixed order)
// then cast to T; hidden layers acc = fma(h_k, W[k][n], acc) over k ascending
// from (T)0, + bias, the skip layer's fp64 (cskip + p.Wsp) term; the head as
// 8 interleaved partial sums (k = p mod 8) added in order, + b_out.  The
// padded rows/columns the tile kernel also visits add exact zeros.
#pragma once
#include "common.cuh"

namespace dist {

constexpr int kSmallWidth = 64;   // widest hidden layer of the narrow path
constexpr int kSmallNT = 64;      // threads (rays) per CTA

template <typename T>
struct SmallNet {
  static constexpr int WI = sizeof(T) == 4 ? 1 : 0;
  static constexpr int NT = kSmallNT;

  // shared-memory bytes of the staged decoder (0: not a narrow decoder)
  __host__ __device__ static size_t weight_bytes(const DecView &dv) {
    const int L = dv.n_layers;
    if (L < 2) return 0;
    for (int l = 0; l <= L - 2; ++l)
      if (dv.nr[l] > kSmallWidth) return 0;
    size_t b = al8(sizeof(double) * 3 * dv.nr[0]);   // W0p
    for (int l = 1; l <= L - 2; ++l) {
      b += al8(sizeof(T) * (size_t)dv.nr[l - 1] * dv.nr[l]) + al8(sizeof(T) * dv.nr[l]);
      if (l == dv.skip) b += al8(sizeof(double) * 3 * dv.nr[l]);
    }
    b += al8(sizeof(T) * dv.nr[L - 2]);
    return round_up((int64_t)b, 16);
  }
  __host__ static size_t smem_bytes(const DecView &dv) {
    const size_t w = weight_bytes(dv);
    return w ? w + 2 * sizeof(T) * kSmallWidth * NT : 0;
  }

  // staged arrays in shared memory, in this order (8-byte aligned each):
  // W0p [3][n0] f64; per hidden layer l: W [K][N] T, b [N] T, (skip layer:
  // Wsp [3][N] f64); w_out [K_out] T; then the two activation buffers.  The
  // per-layer pointers are re-derived while walking the layers (an indexed
  // pointer table would live in local memory).
  const double *W0p;
  const char *layers;   // first hidden layer's W
  const T *wout;
  T *act0, *act1;

  __host__ __device__ static size_t al8(size_t x) { return (x + 7) & ~size_t(7); }

  // Every thread of the CTA calls stage(); a __syncthreads() follows.
  __device__ void stage(const DecView &dv, char *smem) {
    const int L = dv.n_layers, tid = threadIdx.x, nt = blockDim.x;
    char *q = smem;
    auto take = [&](size_t bytes) {
      char *r = q;
      q += al8(bytes);
      return r;
    };
    const int n0 = dv.nr[0], s0 = dv.np[0];
    double *w0 = reinterpret_cast<double *>(take(sizeof(double) * 3 * n0));
    for (int i = tid; i < 3 * n0; i += nt) w0[i] = dv.W0p[(i / n0) * s0 + i % n0];
    W0p = w0;
    layers = q;
    for (int l = 1; l <= L - 2; ++l) {
      const int K = dv.nr[l - 1], N = dv.nr[l], ldw = dv.np[l];
      T *w = reinterpret_cast<T *>(take(sizeof(T) * K * N));
      T *bb = reinterpret_cast<T *>(take(sizeof(T) * N));
      const T *gw = reinterpret_cast<const T *>(dv.W[WI][l]);
      const T *gb = reinterpret_cast<const T *>(dv.bias[WI][l]);
      for (int i = tid; i < K * N; i += nt) w[i] = gw[(size_t)(i / N) * ldw + i % N];
      for (int i = tid; i < N; i += nt) bb[i] = gb[i];
      if (l == dv.skip) {
        double *ws = reinterpret_cast<double *>(take(sizeof(double) * 3 * N));
        for (int i = tid; i < 3 * N; i += nt) ws[i] = dv.Wsp[(size_t)(i / N) * ldw + i % N];
      }
    }
    const int Ko = dv.nr[L - 2];
    T *wo = reinterpret_cast<T *>(take(sizeof(T) * Ko));
    const T *gwo = reinterpret_cast<const T *>(dv.w_out[WI]);
    for (int i = tid; i < Ko; i += nt) wo[i] = gwo[i];
    wout = wo;
    q = smem + weight_bytes(dv);
    act0 = reinterpret_cast<T *>(q);
    act1 = act0 + kSmallWidth * NT;
  }

  // f(p) of shape s for this thread's ray (s >= 0).
  __device__ double eval(const DecView &dv, const double *__restrict__ c0,
                         const double *__restrict__ cskip, const double p[3], int s) const {
    const int L = dv.n_layers, tid = threadIdx.x;
    T *A = act0 + tid, *B = act1 + tid;
    {
      const int n0 = dv.nr[0], s0 = dv.np[0];
      const double *cz = c0 + (size_t)s * s0;
      for (int n = 0; n < n0; ++n) {
        double v = __ldg(cz + n);
        v = fma(p[0], W0p[n], v);
        v = fma(p[1], W0p[n0 + n], v);
        v = fma(p[2], W0p[2 * n0 + n], v);
        A[n * NT] = (T)(!(v <= 0.0) ? v : 0.0);   // np.maximum: NaN propagates
      }
    }
    const char *q = layers;
    for (int l = 1; l <= L - 2; ++l) {
      const int K = dv.nr[l - 1], N = dv.nr[l];
      const T *w = reinterpret_cast<const T *>(q);
      q += al8(sizeof(T) * K * N);
      const T *bb = reinterpret_cast<const T *>(q);
      q += al8(sizeof(T) * N);
      const bool is_skip = (l == dv.skip);
      const double *Wsp = reinterpret_cast<const double *>(q);
      if (is_skip) q += al8(sizeof(double) * 3 * N);
      int n = 0;
      for (; n + 4 <= N; n += 4) {
        T a0 = (T)0, a1 = (T)0, a2 = (T)0, a3 = (T)0;
        for (int k = 0; k < K; ++k) {
          const T h = A[k * NT];
          const T *wr = w + k * N + n;
          a0 = fma(h, wr[0], a0);
          a1 = fma(h, wr[1], a1);
          a2 = fma(h, wr[2], a2);
          a3 = fma(h, wr[3], a3);
        }
        T acc[4] = {a0, a1, a2, a3};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          B[(n + j) * NT] = finish(dv, acc[j] + bb[n + j], is_skip, Wsp, cskip, p, s, n + j);
      }
      for (; n < N; ++n) {
        T a0 = (T)0;
        for (int k = 0; k < K; ++k) a0 = fma(A[k * NT], w[k * N + n], a0);
        B[n * NT] = finish(dv, a0 + bb[n], is_skip, Wsp, cskip, p, s, n);
      }
      T *t = A;
      A = B;
      B = t;
    }
    const int Ko = dv.nr[L - 2];
    T part[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) part[j] = (T)0;
    int k = 0;
    for (; k + 8 <= Ko; k += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) part[j] = fma(A[(k + j) * NT], wout[k + j], part[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (k + j < Ko) part[j] = fma(A[(k + j) * NT], wout[k + j], part[j]);
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) sum += (double)part[j];
    sum += dv.b_out;
    return head_act(dv.final_act, sum);
  }

  __host__ static int width_bucket(const DecView &dv) {
    int w = 0;
    for (int l = 0; l <= dv.n_layers - 2; ++l) w = w > dv.nr[l] ? w : dv.nr[l];
    return w <= 16 ? 16 : (w <= 32 ? 32 : 64);
  }

  __device__ __forceinline__ T finish(const DecView &dv, T v, bool is_skip, const double *Wsp,
                                      const double *__restrict__ cskip, const double p[3], int s,
                                      int col) const {
    if (is_skip) {
      const int N = dv.nr[dv.skip];
      double e = __ldg(cskip + (size_t)s * dv.np[dv.skip] + col);
      e = fma(p[0], Wsp[col], e);
      e = fma(p[1], Wsp[N + col], e);
      e = fma(p[2], Wsp[2 * N + col], e);
      v = (T)((double)v + e);
    }
    return !(v <= (T)0) ? v : (T)0;
  }
};

// The same arithmetic with the activations in registers, for decoders whose
// every width is <= WB (16 or 32): the decoder is staged zero-padded to
// WB x WB per layer, so the fully unrolled loops need no width guards and
// read weight rows as 16-byte broadcasts.  The padding adds exact zeros
// (h = 0 past a layer's width, w = 0 past its rows/columns; an accumulator
// starting at +0 never becomes -0), so results equal SmallNet::eval's bits.
// k outer / n inner: each h_k feeds WB independent FMA chains, each summed
// over k ascending from (T)0.
template <typename T, int WB>
struct RegNet {
  static constexpr int WI = sizeof(T) == 4 ? 1 : 0;

  // staged layout: W0p [3][WB] f64; per hidden layer: W [WB][WB] T, b [WB] T,
  // Wsp [3][WB] f64 (every layer: keeps the stride uniform); w_out [WB] T
  __host__ __device__ static size_t layer_bytes() {
    return sizeof(T) * (WB * WB + WB) + sizeof(double) * 3 * WB;
  }
  __host__ __device__ static size_t weight_bytes(const DecView &dv) {
    return sizeof(double) * 3 * WB + (size_t)(dv.n_layers - 2) * layer_bytes() + sizeof(T) * WB;
  }

  const char *base;

  __device__ void stage(const DecView &dv, char *smem) {
    const int L = dv.n_layers, tid = threadIdx.x, nt = blockDim.x;
    base = smem;
    double *w0 = reinterpret_cast<double *>(smem);
    const int n0 = dv.nr[0], s0 = dv.np[0];
    for (int i = tid; i < 3 * WB; i += nt) {
      const int a = i / WB, n = i % WB;
      w0[i] = n < n0 ? dv.W0p[a * s0 + n] : 0.0;
    }
    char *q = smem + sizeof(double) * 3 * WB;
    for (int l = 1; l <= L - 2; ++l, q += layer_bytes()) {
      const int K = dv.nr[l - 1], N = dv.nr[l], ldw = dv.np[l];
      T *w = reinterpret_cast<T *>(q);
      T *bb = w + WB * WB;
      double *ws = reinterpret_cast<double *>(bb + WB);
      const T *gw = reinterpret_cast<const T *>(dv.W[WI][l]);
      const T *gb = reinterpret_cast<const T *>(dv.bias[WI][l]);
      for (int i = tid; i < WB * WB; i += nt) {
        const int k = i / WB, n = i % WB;
        w[i] = (k < K && n < N) ? gw[(size_t)k * ldw + n] : (T)0;
      }
      for (int i = tid; i < WB; i += nt) bb[i] = i < N ? gb[i] : (T)0;
      for (int i = tid; i < 3 * WB; i += nt) {
        const int a = i / WB, n = i % WB;
        ws[i] = (l == dv.skip && n < N) ? dv.Wsp[(size_t)a * ldw + n] : 0.0;
      }
    }
    T *wo = reinterpret_cast<T *>(q);
    const int Ko = dv.nr[L - 2];
    const T *gwo = reinterpret_cast<const T *>(dv.w_out[WI]);
    for (int i = tid; i < WB; i += nt) wo[i] = i < Ko ? gwo[i] : (T)0;
  }

  // cz / cs: this ray's shape rows of c0 and cskip, zero past the widths
  // (>= WB readable entries each)
  __device__ __forceinline__ double eval(const DecView &dv, const double *cz, const double *cs,
                                         const double p[3]) const {
    const int L = dv.n_layers;
    const double *W0p = reinterpret_cast<const double *>(base);
    T h[WB], o[WB];
#pragma unroll
    for (int n = 0; n < WB; ++n) {
      double v = cz[n];
      v = fma(p[0], W0p[n], v);
      v = fma(p[1], W0p[WB + n], v);
      v = fma(p[2], W0p[2 * WB + n], v);
      h[n] = (T)(!(v <= 0.0) ? v : 0.0);   // np.maximum: NaN propagates
    }
    const char *q = base + sizeof(double) * 3 * WB;
    for (int l = 1; l <= L - 2; ++l, q += layer_bytes()) {
      const T *w = reinterpret_cast<const T *>(q);
      const T *bb = w + WB * WB;
      const double *Wsp = reinterpret_cast<const double *>(bb + WB);
#pragma unroll
      for (int n = 0; n < WB; ++n) o[n] = (T)0;
#pragma unroll
      for (int k = 0; k < WB; ++k) {
        const T hk = h[k];
#pragma unroll
        for (int n = 0; n < WB; ++n) o[n] = fma(hk, w[k * WB + n], o[n]);
      }
      if (l == dv.skip) {
#pragma unroll
        for (int n = 0; n < WB; ++n) {
          T v = o[n] + bb[n];
          double e = cs[n];
          e = fma(p[0], Wsp[n], e);
          e = fma(p[1], Wsp[WB + n], e);
          e = fma(p[2], Wsp[2 * WB + n], e);
          v = (T)((double)v + e);
          h[n] = !(v <= (T)0) ? v : (T)0;
        }
      } else {
#pragma unroll
        for (int n = 0; n < WB; ++n) {
          const T v = o[n] + bb[n];
          h[n] = !(v <= (T)0) ? v : (T)0;
        }
      }
    }
    const T *wout = reinterpret_cast<const T *>(q);
    T part[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) part[j] = (T)0;
#pragma unroll
    for (int k = 0; k < WB; ++k) part[k & 7] = fma(h[k], wout[k], part[k & 7]);
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) sum += (double)part[j];
    sum += dv.b_out;
    return head_act(dv.final_act, sum);
  }
};

}  // namespace dist
