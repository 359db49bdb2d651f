// decoder.cu -- NeuralField on the device: weight packing, per-shape code
// bias, point evaluation (NeuralField.evaluate, fields.py:233-247) and the
// taped evaluation + reverse sweep (fields.py:260-291, autodiff.py:220-255).
#include <cmath>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "mlp_eval.cuh"

namespace dist {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { g_err = msg; }
int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return DIST_ERR_CUDA;
}
void count_launch(int n) { g_launches += n; }

// ---------------------------------------------------------------------------
// acc + sum_{k<n} a[k*as] * b[k*bs] as one fma chain in ascending k (the same
// rounding as the plain loop), with the operands of U steps loaded ahead so
// the chain waits on one round of L2/HBM latency per U steps, not per step.
template <int U>
__device__ __forceinline__ double dot_ordered(const double *__restrict__ a, int64_t as,
                                              const double *__restrict__ b, int64_t bs, int n,
                                              double acc) {
  int k = 0;
  for (; k + U <= n; k += U) {
    double x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = __ldg(a + (int64_t)(k + u) * as);
      y[u] = __ldg(b + (int64_t)(k + u) * bs);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fma(x[u], y[u], acc);
  }
  for (; k < n; ++k) acc = fma(__ldg(a + (int64_t)k * as), __ldg(b + (int64_t)k * bs), acc);
  return acc;
}

// per-shape folded biases: c0[s][j] = b0[j] + sum_k z[s][k] W0z[k][j]  (fp64)
// and the skip layer's code part cskip[s][j] = sum_k z[s][k] Wsz[k][j].
// One thread per output (64-thread blocks: S x 512 outputs spread over many
// SMs); each output is a latency-bound 256-step chain, so loads run 16 ahead.
__global__ void k_code_bias(DecView dv, const double *__restrict__ codes, int S,
                            double *__restrict__ c0, double *__restrict__ cskip) {
  const int n0 = dv.np[0];
  const int D = dv.latent_dim;
  const int total = S * n0;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += gridDim.x * blockDim.x) {
    const int s = idx / n0, j = idx % n0;
    const double v = dot_ordered<16>(codes + (size_t)s * D, 1, dv.W0z + j, n0, D, dv.b0[j]);
    c0[idx] = v;
    reinterpret_cast<float *>(c0 + total)[idx] = (float)v;   // fp32 copy (kernels.cuh c0_f32)
    // per-shape max |c0| (kernels.cuh c0_absmax): non-negative floats order as ints
    atomicMax(reinterpret_cast<int *>(c0 + total) + total + s, __float_as_int(fabsf((float)v)));
  }
  if (dv.skip > 0) {
    // the skip layer's code part, laid out like c0 (fp64, fp32 copy, per-shape max |.|)
    const int ns = dv.nskip;
    const int tot2 = S * ns;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < tot2;
         idx += gridDim.x * blockDim.x) {
      const int s = idx / ns, j = idx % ns;
      const double v = codes ? dot_ordered<16>(codes + (size_t)s * D, 1, dv.Wsz + j, ns, D, 0.0) : 0.0;
      cskip[idx] = v;
      reinterpret_cast<float *>(cskip + tot2)[idx] = (float)v;
      atomicMax(reinterpret_cast<int *>(cskip + tot2) + tot2 + s, __float_as_int(fabsf((float)v)));
    }
  }
}

int launch_code_bias(const DecView &dv, const double *codes, int S, double *c0, double *cskip,
                     cudaStream_t st) {
  if (S <= 0) return DIST_OK;
  const int n = S * dv.np[0];
  cudaError_t e = cudaMemsetAsync(const_cast<float *>(c0_absmax(c0, S, dv.np[0])), 0, sizeof(float) * S, st);
  if (e == cudaSuccess && dv.skip > 0)
    e = cudaMemsetAsync(const_cast<float *>(c0_absmax(cskip, S, dv.nskip)), 0, sizeof(float) * S, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(c0 max)");
  const int nmax = std::max(n, S * std::max(dv.nskip, 0));
  k_code_bias<<<(int)std::min<int64_t>(ceil_div(nmax, 64), 4096), 64, 0, st>>>(dv, codes, S, c0, cskip);
  DIST_CHECK_LAUNCH("k_code_bias");
  return DIST_OK;
}

// grad[s][k] = sum_j (sum_cta part0[cta][s][j]) W0z[k][j] + skip part.
// The partials are exact fixed-point integers (common.cuh fx_t): their sum is
// the same whatever the order or the number of slots, then it is rounded once
// to fp64 and contracted with W0z in a fixed order.
__global__ void k_reduce_colsums(DecView dv, int S, int G, const fx_t *__restrict__ part0,
                                 const fx_t *__restrict__ parts, fx_t *__restrict__ colsum0,
                                 fx_t *__restrict__ colsums) {
  const int n0 = dv.np[0], ns = dv.nskip;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_all = (int64_t)S * (n0 + ns);
  if (t >= n_all) return;
  constexpr int U = 8;
  const bool main_part = t < (int64_t)S * n0;
  const int64_t q = main_part ? t : t - (int64_t)S * n0;
  const int w = main_part ? n0 : ns;
  const int s = (int)(q / w), j = (int)(q - (int64_t)s * w);
  const fx_t *src = (main_part ? part0 : parts) + (size_t)s * w + j;
  const int64_t stride = (int64_t)S * w;
  fx_t acc = 0;
  int c = 0;
  for (; c + U <= G; c += U) {
    fx_t x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = src[(c + u) * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) acc += x[u];
  }
  for (; c < G; ++c) acc += src[c * stride];
  (main_part ? colsum0 : colsums)[q] = acc;
}

__device__ __forceinline__ double dot_fixed(const fx_t *__restrict__ a, const double *__restrict__ b,
                                            int n, double acc) {
  for (int k = 0; k < n; ++k) acc = fma(fx_to_double(a[k]), __ldg(b + k), acc);
  return acc;
}

__global__ void k_reduce_code_grad(DecView dv, int S, const fx_t *__restrict__ colsum0,
                                   const fx_t *__restrict__ colsums, const int *__restrict__ bad,
                                   double *__restrict__ grad) {
  const int n0 = dv.np[0], ns = dv.nskip, D = dv.latent_dim;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S * D) return;
  const int s = t / D, k = t - s * D;
  double acc = dot_fixed(colsum0 + (size_t)s * n0, dv.W0z + (size_t)k * n0, n0, 0.0);
  if (ns > 0) acc = dot_fixed(colsums + (size_t)s * ns, dv.Wsz + (size_t)k * ns, ns, acc);
  grad[t] = (bad && *bad) ? __longlong_as_double(0x7ff8000000000000ll) : acc;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int vjp_grid_cap(int prec) {
  // fixed upper bound on the vjp grid so partial buffers can be sized up front
  (void)prec;
  return 4 * sm_count();
}

int eval_points(const DecView &dv, const double *c0, const double *cskip, int S, const double *pts,
                const int32_t *shape, int64_t n, double *f, cudaStream_t st) {
  if (n <= 0) return DIST_OK;
  ArrayGen g{pts, shape, nullptr, f, n};
  if (dv.prec == DIST_PREC_FP64) return launch_eval_gen<double>(dv, c0, cskip, g, n, st);
  if (dv.prec >= DIST_PREC_BF16X3) return tc_eval_points(dv, c0, cskip, S, pts, shape, n, f, st);
  return launch_eval_gen<float>(dv, c0, cskip, g, n, st);
}

int vjp_points(const DecView &dv, const double *c0, const double *cskip, const double *pts,
               const int32_t *shape, int64_t n, const double *seed, int S, double *f,
               fx_t *part0, fx_t *parts, int *bad, double *gpts, int grid_cap, int *grid_out,
               cudaStream_t st) {
  *grid_out = 0;
  if (n <= 0) return DIST_OK;
  ArrayGen g{pts, shape, seed, f, n};
  if (dv.prec == DIST_PREC_FP64)
    return launch_vjp_gen<double>(dv, c0, cskip, g, n, S, part0, parts, gpts, bad, grid_cap, grid_out, st);
  // bf16x3: the fused tensor-core head kernel (forward, given seeds, fp16x2 dgrad)
  if (tc_heads_supported(dv))
    return launch_tc_heads<ArrayGen>(dv, c0, cskip, g, n, S, part0, parts, bad, grid_cap, grid_out, st, gpts);
  return launch_vjp_gen<float>(dv, c0, cskip, g, n, S, part0, parts, gpts, bad, grid_cap, grid_out, st);
}

int reduce_code_grad(const DecView &dv, int S, int G, const fx_t *part0, const fx_t *parts,
                     const int *bad, fx_t *colsum0, fx_t *colsums, double *grad, cudaStream_t st) {
  if (S <= 0 || dv.latent_dim == 0) return DIST_OK;
  const int64_t nc = (int64_t)S * (dv.np[0] + std::max(dv.nskip, 0));
  if (G > 0) {
    k_reduce_colsums<<<(int)ceil_div(nc, 64), 64, 0, st>>>(dv, S, G, part0, parts, colsum0, colsums);
    DIST_CHECK_LAUNCH("k_reduce_colsums");
  }
  if (grad) {
    k_reduce_code_grad<<<(int)ceil_div((int64_t)S * dv.latent_dim, 64), 64, 0, st>>>(dv, S, colsum0, colsums,
                                                                                     bad, grad);
    DIST_CHECK_LAUNCH("k_reduce_code_grad");
  }
  return DIST_OK;
}

size_t eval_ws(const DecView &dv, int64_t n, int S, bool vjp) {
  Carve cv{nullptr, 0, ~size_t(0)};
  const int s1 = std::max(S, 1);
  cv.take<double>(c0_doubles(s1, dv.np[0]));
  cv.take<double>(c0_doubles(s1, std::max(dv.nskip, 1)));
  if (vjp) {
    const int G = vjp_grid_cap(dv.prec);
    cv.take<fx_t>((size_t)G * s1 * dv.np[0]);
    cv.take<fx_t>((size_t)G * s1 * std::max(dv.nskip, 1));
    cv.take<fx_t>((size_t)s1 * dv.np[0]);
    cv.take<fx_t>((size_t)s1 * std::max(dv.nskip, 1));
    cv.take<int>(4);
  }
  (void)n;
  return cv.off + 256;
}

}  // namespace dist

using namespace dist;

// ===========================================================================
// C ABI
extern "C" {

const char *dist_last_error(void) { return g_err.c_str(); }

int64_t dist_launch_count(void) { return g_launches.load(); }

int dist_device_info(int *sm, int *major, int *minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  cudaDeviceGetAttribute(sm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev);
  return DIST_OK;
}

int dist_decoder_create(const double *const *W, const double *const *b, int L,
                        const int32_t *dims, int D, int skip, int final_linear, int prec,
                        dist_decoder **out) {
  if (!out || !W || !b || !dims) return fail(DIST_ERR_CONFIG, "null argument");
  *out = nullptr;
  if (L < 2 || L > kMaxLayers) return fail(DIST_ERR_CONFIG, "n_layers must be in [2, 16]");
  if (D < 0) return fail(DIST_ERR_CONFIG, "latent_dim must be >= 0");
  if (prec < DIST_PREC_FP64 || prec > DIST_PREC_FP16X3)
    return fail(DIST_ERR_CONFIG, "unknown precision");
  if (dims[L] != 1) return fail(DIST_ERR_CONFIG, "final layer must map to one output");
  if (skip < 0) skip = -1;
  else if (skip == 0 || skip >= L - 1)
    return fail(DIST_ERR_CONFIG, "skip layer must be in [1, L-2]");
  if (dims[0] != D + 3) return fail(DIST_ERR_CONFIG, "first layer width must be latent_dim + 3");
  for (int l = 1; l < L; ++l)
    if (dims[l] < 1 || dims[l] > kMaxWidth)
      return fail(DIST_ERR_CONFIG, "hidden widths must be in [1, 512]");
  int cc_major = 0, cc_minor = 0, nsm = 0;
  if (dist_device_info(&nsm, &cc_major, &cc_minor)) return DIST_ERR_CUDA;
  if (cc_major != 10) return fail(DIST_ERR_CUDA, "libdist_b200 requires an sm_100 (B200) device");

  DecView v{};
  v.n_layers = L;
  v.latent_dim = D;
  v.skip = skip;
  if (final_linear < 0 || final_linear > 2) return fail(DIST_ERR_CONFIG, "final activation must be 0 (tanh), 1 (linear) or 2 (sigmoid)");
  v.final_act = final_linear;
  v.prec = prec;
  for (int l = 0; l < L - 1; ++l) v.np[l] = (int)round_up(dims[l + 1], 64);
  v.np[L - 1] = 1;
  for (int l = 0; l < L; ++l) v.nr[l] = dims[l + 1];
  for (int l = 1; l < L; ++l) v.kp[l] = v.np[l - 1];
  v.nskip = skip > 0 ? v.np[skip] : 0;
  if (prec >= DIST_PREC_BF16X3 && !tc_shape_ok(v))
    // any other shape would silently run SIMT fp32 -- refuse instead
    return fail(DIST_ERR_CONFIG,
                "tensor-core precisions (bf16x3, fp16x3) need >= 2 hidden layers, a 512-wide first "
                "hidden layer (and skip layer), and a skip layer below the top hidden layer; use "
                "precision fp32 or fp64 for this decoder");

  // host staging of every packed array, then one device blob
  std::vector<char> host;
  auto put = [&](size_t bytes) {
    size_t off = (size_t)round_up((int64_t)host.size(), 256);
    host.resize(off + bytes, 0);
    return off;
  };
  const int n0 = v.np[0];
  size_t o_W0z = put(sizeof(double) * std::max(D, 1) * n0);
  size_t o_W0p = put(sizeof(double) * 3 * n0);
  size_t o_W0pf = put(sizeof(float) * 3 * n0);
  size_t o_b0 = put(sizeof(double) * n0);
  {
    double *W0z = (double *)(host.data() + o_W0z);
    double *W0p = (double *)(host.data() + o_W0p);
    double *b0 = (double *)(host.data() + o_b0);
    for (int k = 0; k < D; ++k)
      for (int j = 0; j < dims[1]; ++j) W0z[(size_t)k * n0 + j] = W[0][(size_t)k * dims[1] + j];
    for (int a = 0; a < 3; ++a)
      for (int j = 0; j < dims[1]; ++j) W0p[(size_t)a * n0 + j] = W[0][(size_t)(D + a) * dims[1] + j];
    float *W0pf = (float *)(host.data() + o_W0pf);
    for (int i = 0; i < 3 * n0; ++i) W0pf[i] = (float)W0p[i];
    for (int j = 0; j < dims[1]; ++j) b0[j] = b[0][j];
  }
  size_t o_W[2][kMaxLayers] = {}, o_Wt[2][kMaxLayers] = {}, o_b[2][kMaxLayers] = {};
  size_t o_Wsz = 0, o_Wsp = 0, o_Wspf = 0;
  for (int l = 1; l <= L - 2; ++l) {
    const int K = v.kp[l], N = v.np[l];
    const int kin = dims[l], nout = dims[l + 1];  // true h-part input width and output width
    const int rowsW = kin + (l == skip ? D + 3 : 0);
    (void)rowsW;
    for (int c = 0; c < 2; ++c) {
      const size_t es = c == 0 ? sizeof(double) : sizeof(float);
      o_W[c][l] = put(es * K * N);
      o_Wt[c][l] = put(es * K * N);
      o_b[c][l] = put(es * N);
      for (int k = 0; k < kin; ++k)
        for (int j = 0; j < nout; ++j) {
          const double w = W[l][(size_t)k * nout + j];
          if (c == 0) {
            ((double *)(host.data() + o_W[c][l]))[(size_t)k * N + j] = w;
            ((double *)(host.data() + o_Wt[c][l]))[(size_t)j * K + k] = w;
          } else {
            ((float *)(host.data() + o_W[c][l]))[(size_t)k * N + j] = (float)w;
            ((float *)(host.data() + o_Wt[c][l]))[(size_t)j * K + k] = (float)w;
          }
        }
      for (int j = 0; j < nout; ++j) {
        if (c == 0) ((double *)(host.data() + o_b[c][l]))[j] = b[l][j];
        else ((float *)(host.data() + o_b[c][l]))[j] = (float)b[l][j];
      }
    }
    if (l == skip) {
      o_Wsz = put(sizeof(double) * std::max(D, 1) * N);
      o_Wsp = put(sizeof(double) * 3 * N);
      o_Wspf = put(sizeof(float) * 3 * N);
      double *Wsz = (double *)(host.data() + o_Wsz);
      double *Wsp = (double *)(host.data() + o_Wsp);
      float *Wspf = (float *)(host.data() + o_Wspf);
      for (int k = 0; k < D; ++k)
        for (int j = 0; j < nout; ++j) Wsz[(size_t)k * N + j] = W[l][(size_t)(kin + k) * nout + j];
      for (int a = 0; a < 3; ++a) {
        double m = 0.0;
        for (int j = 0; j < nout; ++j) {
          const double w = W[l][(size_t)(kin + D + a) * nout + j];
          Wsp[(size_t)a * N + j] = w;
          Wspf[(size_t)a * N + j] = (float)w;
          m = std::max(m, std::fabs(w));
        }
        v.wsm[a] = (float)(m * (1.0 + 1e-6));   // rounded up: a bound
      }
    }
  }
  const int Ko = v.np[L - 2];
  size_t o_wo[2];
  o_wo[0] = put(sizeof(double) * Ko);
  o_wo[1] = put(sizeof(float) * Ko);
  for (int k = 0; k < dims[L - 1]; ++k) {
    ((double *)(host.data() + o_wo[0]))[k] = W[L - 1][k];
    ((float *)(host.data() + o_wo[1]))[k] = (float)W[L - 1][k];
  }
  v.b_out = b[L - 1][0];
  if (skip > 0 && skip == L - 1) return fail(DIST_ERR_CONFIG, "skip cannot be the output layer");

  // tensor-core packs (bf16 hi/lo) for the split-precision path
  size_t o_tc[kMaxLayers] = {}, o_tcb[kMaxLayers] = {};
  if (prec >= DIST_PREC_BF16X3) tc_pack_sizes(v, [&](int l, size_t wbytes, size_t bbytes) {
      o_tc[l] = put(wbytes);
      o_tcb[l] = put(bbytes);
    });

  void *blob = nullptr;
  cudaError_t e = cudaMalloc(&blob, host.size());
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(decoder)");
  if (prec >= DIST_PREC_BF16X3)
    tc_pack_fill(v, W, b, dims, [&](int l) { return (void *)(host.data() + o_tc[l]); },
                 [&](int l) { return (float *)(host.data() + o_tcb[l]); });
  e = cudaMemcpy(blob, host.data(), host.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(blob);
    return cuda_fail(e, "cudaMemcpy(decoder)");
  }
  char *base = (char *)blob;
  v.W0z = (const double *)(base + o_W0z);
  v.W0p = (const double *)(base + o_W0p);
  v.W0pf = (const float *)(base + o_W0pf);
  v.b0 = (const double *)(base + o_b0);
  for (int l = 1; l <= L - 2; ++l)
    for (int c = 0; c < 2; ++c) {
      v.W[c][l] = base + o_W[c][l];
      v.Wt[c][l] = base + o_Wt[c][l];
      v.bias[c][l] = base + o_b[c][l];
    }
  v.Wsz = skip > 0 ? (const double *)(base + o_Wsz) : nullptr;
  v.Wsp = skip > 0 ? (const double *)(base + o_Wsp) : nullptr;
  v.Wspf = skip > 0 ? (const float *)(base + o_Wspf) : nullptr;
  v.w_out[0] = base + o_wo[0];
  v.w_out[1] = base + o_wo[1];
  if (prec >= DIST_PREC_BF16X3)
    for (int l = 0; l < kMaxLayers; ++l)
      if (o_tc[l]) {
        v.tc_w[l] = base + o_tc[l];
        v.tc_bias[l] = (const float *)(base + o_tcb[l]);
      }
  v.tc_gain[0] = v.tc_gain[1] = 1.0;
  if (prec >= DIST_PREC_BF16X3) {
    const int rc = tc_calibrate(v);
    if (rc) {
      cudaFree(blob);
      return rc;
    }
  }
  dist_decoder *d = new dist_decoder;
  d->view = v;
  d->blob = blob;
  d->blob_bytes = host.size();
  for (int l = 0; l <= L; ++l) d->dims[l] = dims[l];
  *out = d;
  return DIST_OK;
}

int dist_decoder_destroy(dist_decoder *dec) {
  if (!dec) return DIST_OK;
  if (dec->view.prec >= DIST_PREC_BF16X3) tc_forget_maps(dec->view);
  cudaFree(dec->blob);
  delete dec;
  return DIST_OK;
}

int dist_decoder_precision(const dist_decoder *dec) { return dec ? dec->view.prec : -1; }

int dist_decoder_colsum_width(const dist_decoder *dec) {
  return dec ? dec->view.np[0] + std::max(dec->view.nskip, 0) : -1;
}

int dist_decoder_head_gain(const dist_decoder *dec, double *gain2) {
  if (!dec || !gain2) return fail(DIST_ERR_CONFIG, "null argument");
  gain2[0] = dec->view.tc_gain[0];
  gain2[1] = dec->view.tc_gain[1];
  return DIST_OK;
}

size_t dist_eval_workspace_size(const dist_decoder *dec, int64_t n, int S) {
  return dec ? eval_ws(dec->view, n, S, true) : 0;
}

int dist_eval(const dist_decoder *dec, const double *codes, int S, const double *pts,
              const int32_t *shape, int64_t n, double *f, void *ws, size_t ws_bytes,
              void *stream) {
  if (!dec) return fail(DIST_ERR_CONFIG, "null decoder");
  const DecView &dv = dec->view;
  if (dv.latent_dim > 0 && (!codes || S < 1)) return fail(DIST_ERR_CONFIG, "field expects a latent code");
  cudaStream_t st = (cudaStream_t)stream;
  Carve cv{(char *)ws, 0, ws_bytes};
  const int s1 = std::max(S, 1);
  double *c0 = cv.take<double>(c0_doubles(s1, dv.np[0]));
  double *cs = cv.take<double>(c0_doubles(s1, std::max(dv.nskip, 1)));
  if (!cv.ok) return fail(DIST_ERR_CONFIG, "workspace too small");
  int rc;
  if (dv.latent_dim > 0) {
    rc = launch_code_bias(dv, codes, S, c0, cs, st);
  } else {
    rc = launch_code_bias(dv, nullptr, 1, c0, cs, st);
  }
  if (rc) return rc;
  return eval_points(dv, c0, cs, s1, pts, shape, n, f, st);
}

int dist_eval_channels(const dist_decoder *const *decs, int m, const double *codes, int S,
                       const double *pts, const int32_t *shape, int64_t n, double *out, void *ws,
                       size_t ws_bytes, void *stream) {
  if (!decs || !decs[0] || !out) return fail(DIST_ERR_CONFIG, "null argument");
  if (m < 1 || m > kMaxHeads) return fail(DIST_ERR_CONFIG, "channel count must be in [1, 8]");
  const dist_decoder *d0 = decs[0];
  const DecView &dv = d0->view;
  if (dv.prec >= DIST_PREC_BF16X3)
    return fail(DIST_ERR_CONFIG, "dist_eval_channels takes the SIMT precisions (fp64, fp32)");
  HeadSet hs{};
  hs.m = m;
  const int wi = dv.prec == DIST_PREC_FP64 ? 0 : 1;
  for (int c = 0; c < m; ++c) {
    const dist_decoder *dc = decs[c];
    if (!dc) return fail(DIST_ERR_CONFIG, "null decoder");
    const DecView &v = dc->view;
    bool same = v.n_layers == dv.n_layers && v.latent_dim == dv.latent_dim && v.skip == dv.skip &&
                v.prec == dv.prec && v.final_act == dv.final_act;
    for (int l = 0; same && l <= dv.n_layers; ++l) same = dc->dims[l] == d0->dims[l];
    if (!same) return fail(DIST_ERR_CONFIG, "channel decoders must share layout, precision and head activation");
    hs.w[c] = v.w_out[wi];
    hs.b[c] = v.b_out;
  }
  if (dv.latent_dim > 0 && (!codes || S < 1)) return fail(DIST_ERR_CONFIG, "field expects a latent code");
  if (n <= 0) return DIST_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Carve cv{(char *)ws, 0, ws_bytes};
  const int s1 = std::max(S, 1);
  double *c0 = cv.take<double>(c0_doubles(s1, dv.np[0]));
  double *cs = cv.take<double>(c0_doubles(s1, std::max(dv.nskip, 1)));
  if (!cv.ok) return fail(DIST_ERR_CONFIG, "workspace too small");
  int rc = launch_code_bias(dv, dv.latent_dim > 0 ? codes : nullptr, s1, c0, cs, st);
  if (rc) return rc;
  ArrayGen g{pts, shape, nullptr, nullptr, n};
  if (dv.prec == DIST_PREC_FP64) return launch_eval_channels<double>(dv, c0, cs, g, hs, out, st);
  return launch_eval_channels<float>(dv, c0, cs, g, hs, out, st);
}

int dist_eval_vjp(const dist_decoder *dec, const double *codes, int S, const double *pts,
                  const int32_t *shape, int64_t n, const double *seed, double *f,
                  double *grad_codes, double *gpts, void *ws, size_t ws_bytes, void *stream) {
  if (!dec) return fail(DIST_ERR_CONFIG, "null decoder");
  const DecView &dv = dec->view;
  if (dv.latent_dim > 0 && (!codes || S < 1)) return fail(DIST_ERR_CONFIG, "field expects a latent code");
  cudaStream_t st = (cudaStream_t)stream;
  const int s1 = std::max(S, 1);
  Carve cv{(char *)ws, 0, ws_bytes};
  double *c0 = cv.take<double>(c0_doubles(s1, dv.np[0]));
  double *cs = cv.take<double>(c0_doubles(s1, std::max(dv.nskip, 1)));
  const int G = vjp_grid_cap(dv.prec);
  fx_t *part0 = cv.take<fx_t>((size_t)G * s1 * dv.np[0]);
  fx_t *parts = cv.take<fx_t>((size_t)G * s1 * std::max(dv.nskip, 1));
  fx_t *col0 = cv.take<fx_t>((size_t)s1 * dv.np[0]);
  fx_t *cols = cv.take<fx_t>((size_t)s1 * std::max(dv.nskip, 1));
  int *bad = cv.take<int>(4);
  if (!cv.ok) return fail(DIST_ERR_CONFIG, "workspace too small");
  int rc = launch_code_bias(dv, dv.latent_dim > 0 ? codes : nullptr, s1, c0, cs, st);
  if (rc) return rc;
  cudaError_t e = cudaMemsetAsync(part0, 0, sizeof(fx_t) * G * s1 * dv.np[0], st);
  if (e == cudaSuccess && dv.nskip)
    e = cudaMemsetAsync(parts, 0, sizeof(fx_t) * G * s1 * dv.nskip, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (e == cudaSuccess && gpts) e = cudaMemsetAsync(gpts, 0, sizeof(double) * 3 * n, st);
  if (e == cudaSuccess && grad_codes && dv.latent_dim)
    e = cudaMemsetAsync(grad_codes, 0, sizeof(double) * s1 * dv.latent_dim, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  int grid = 0;
  rc = vjp_points(dv, c0, cs, pts, shape, n, seed, s1, f, part0, parts, bad, gpts, G, &grid, st);
  if (rc) return rc;
  if (grad_codes && grid > 0)
    return reduce_code_grad(dv, s1, grid, part0, parts, bad, col0, cols, grad_codes, st);
  return DIST_OK;
}

}  // extern "C"
