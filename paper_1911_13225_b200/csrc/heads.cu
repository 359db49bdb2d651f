// heads.cu -- the memory-light backward of one latent-optimisation iterate,
// fully on the device (optimize.py:102-138 with shading.py:156-281 and
// losses.py:54-117), plus the bias-corrected Adam step (optimize.py:47-63).
//
// Pipeline per iterate, all stream-ordered, no host synchronisation:
//   1. sample list over the frozen record: recorded rays (finite
//      topk_absf[:,0]) and every finite top-K slot, both in ascending order
//      exactly as np.nonzero/np.repeat build them (shading.py:171-183);
//   2. per-view loss preparation: n_px (converged & observed), n_conv, the
//      silhouette hinge loss and its per-pixel gradient (losses.py:78-91);
//   3. ONE fused kernel per tile of samples: taped decoder forward at the
//      frozen points c + d_k v, the depth seed w*sign(r)*scale computed from
//      the tile's own f (losses.py:70-75) plus the silhouette seed on slot 0,
//      then the reverse sweep -- activations and ReLU masks never leave
//      shared memory; per-CTA column sums of the layer-0 gradient are the
//      only output besides f;
//   4. per-view depth loss from f, a fixed-order reduction of the column
//      sums into d/dz, the latent regulariser added once per shape.
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"
#include "march.cuh"
#include "mlp_eval.cuh"
#include "scan.cuh"
#include "heads.cuh"

namespace dist {

// rec_rank[g] = index of recorded ray g in h.rec (written by the rec
// compaction); every sample's ray is recorded (finite slot 0: topk_absf is
// sorted ascending), so the lookup is one gather instead of a binary search.
__global__ void k_heads_index(HeadsDev h, const int32_t *__restrict__ rec_rank, int K, int V,
                              int64_t WH) {
  const int64_t nrec = h.counts[0], nsamp = h.counts[1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nsamp;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t flat = h.samp[i];
    const int64_t g = flat / K;
    const int64_t r = rec_rank[g];
    h.samp_pix[i] = (int32_t)r;
    if (flat - g * K == 0) h.best[r] = (int32_t)i;
  }
  if (blockIdx.x == 0)
    for (int v = threadIdx.x; v <= V; v += blockDim.x) {
      h.view_rec[v] = (int32_t)lower_bound_i32(h.rec, nrec, (int64_t)v * WH);
      h.view_samp[v] = (int32_t)lower_bound_i32(h.samp, nsamp, (int64_t)v * WH * K);
    }
}

__device__ __forceinline__ double block_sum(double v, double *red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;  // valid in thread 0
}

// one block per view: n_px, n_conv, silhouette loss + per-pixel seed
// gridDim.y blocks per view sum fixed pixel chunks into part[v][b][3];
// k_view_prep_finish adds them in order (deterministic)
constexpr int kPrepBlocks = 32;
__global__ void k_view_prep(const dist_camera *__restrict__ cams, LevelState ls, int K, double eps,
                            ObjIn in, const double *__restrict__ view_norm, double *part,
                            double *sil_seed) {
  __shared__ double red[32];
  const int v = blockIdx.x, b = blockIdx.y, nb = gridDim.y;
  const int64_t WH = (int64_t)ls.lw * ls.lh;
  const int64_t g0 = v * WH;
  const int64_t chunk = (WH + nb - 1) / nb;
  const int64_t q0 = b * chunk, q1 = min(WH, q0 + chunk);
  double n_px = 0, n_conv = 0, sl = 0;
  // silhouette_loss is a mean over the view's pixels (losses.py:78-91); a
  // pixel tile of a sharded view divides by the whole view's pixel count
  const double inv_n = 1.0 / (view_norm ? view_norm[v * 3 + 1] : (double)WH);
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int64_t g = g0 + q;
    const bool conv = ls.status[g] == DIST_CONVERGED;
    const bool rec = isfinite(ls.tk_a[g * K]);
    n_conv += (conv && rec) ? 1.0 : 0.0;
    if (conv && rec && depth_valid(in, g)) n_px += 1.0;
    if (in.obs_sil) {
      double s;
      if (rec) {
        s = ls.tk_a[g * K] - eps;
      } else {
        const int j = (int)(q / ls.lw), i = (int)(q - (int64_t)j * ls.lw);
        double dir[3];
        pixel_ray(cams[v], i, j, 1, dir, nullptr);
        const double *o = cams[v].origin;
        const double m = dir[0] * o[0] + dir[1] * o[1] + dir[2] * o[2];
        const double c2 = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
        s = sqrt(fmax(c2 - m * m, 0.0)) - 1.0;
      }
      const double t = in.obs_sil[g];
      sl += t * fmax(s, 0.0) + (1.0 - t) * fmax(-s, 0.0);
      const double gr = (t * (s > 0.0 ? 1.0 : 0.0) - (1.0 - t) * (s < 0.0 ? 1.0 : 0.0)) * inv_n;
      sil_seed[g] = in.w_sil * gr;
    }
  }
  const double a = block_sum(n_px, red);
  const double bc = block_sum(n_conv, red);
  const double c = block_sum(sl, red);
  if (threadIdx.x == 0) {
    double *o = part + ((size_t)v * nb + b) * 3;
    o[0] = a;
    o[1] = bc;
    o[2] = c;
  }
}

__global__ void k_view_prep_finish(int V, int nb, int64_t WH, const double *__restrict__ part,
                                   bool sil, const double *__restrict__ view_norm, int32_t *npx,
                                   double *terms) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    double a = 0.0, bc = 0.0, c = 0.0;
    for (int b = 0; b < nb; ++b) {
      const double *o = part + ((size_t)v * nb + b) * 3;
      a += o[0];
      bc += o[1];
      c += o[2];
    }
    // the depth term normalises by the view's n_px (losses.py:61-72): the
    // whole view's count when this is a tile of a sharded view
    npx[v] = (int32_t)(view_norm ? view_norm[v * 3 + 0] : a);
    terms[v * kViewTerms + 0] = 0.0;
    terms[v * kViewTerms + 1] = sil ? c / (view_norm ? view_norm[v * 3 + 1] : (double)WH) : 0.0;
    terms[v * kViewTerms + 2] = a;
    terms[v * kViewTerms + 3] = bc;
  }
}

// --- normal term (losses.py:94-111; seeds shading.py:259-269) ----------------
// valid = converged & non-degenerate rendered normal & finite, trusted observation
__device__ __forceinline__ bool normal_valid(const LevelState &ls, const NormIn &nn, int64_t g) {
  if (ls.status[g] != DIST_CONVERGED || !(nn.rawnorm[g] > 0.0)) return false;
  const double *o = nn.obs + g * 3;
  bool ok = isfinite(o[0]) && isfinite(o[1]) && isfinite(o[2]);
  if (nn.mask) ok = ok && nn.mask[g];
  return ok;
}

// per view: n valid pixels and sum of n_hat . n_obs (fixed chunks, in order)
__global__ void k_view_normal(LevelState ls, NormIn nn, double *part) {
  __shared__ double red[32];
  const int v = blockIdx.x, b = blockIdx.y, nb = gridDim.y;
  const int64_t WH = (int64_t)ls.lw * ls.lh;
  const int64_t chunk = (WH + nb - 1) / nb;
  const int64_t q0 = b * chunk, q1 = min(WH, q0 + chunk);
  double cnt = 0.0, dot = 0.0;
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int64_t g = v * WH + q;
    if (!normal_valid(ls, nn, g)) continue;
    cnt += 1.0;
    const double *u = nn.unit + g * 3, *o = nn.obs + g * 3;
    dot += u[0] * o[0] + u[1] * o[1] + u[2] * o[2];
  }
  const double a = block_sum(cnt, red);
  const double c = block_sum(dot, red);
  if (threadIdx.x == 0) {
    double *o = part + ((size_t)v * nb + b) * 2;
    o[0] = a;
    o[1] = c;
  }
}

__global__ void k_view_normal_finish(int V, int nb, const double *__restrict__ part,
                                     const double *__restrict__ view_norm, double *nnorm,
                                     double *terms) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    double a = 0.0, c = 0.0;
    for (int b = 0; b < nb; ++b) {
      a += part[((size_t)v * nb + b) * 2 + 0];
      c += part[((size_t)v * nb + b) * 2 + 1];
    }
    const double n = view_norm ? view_norm[v * 3 + 2] : a;
    nnorm[v] = n;
    terms[v * kViewTerms + 4] = n > 0.0 ? -c / n : 0.0;
    terms[v * kViewTerms + 5] = a;
  }
}

// depth loss = sum_i w_i |r_i| over each view's samples: gridDim.y blocks per
// view sum fixed chunks into part[v][b]; k_view_loss_finish adds them in order
constexpr int kLossBlocks = 64;
__global__ void k_view_depth_loss(const dist_camera *__restrict__ cams, LevelState ls, int K,
                                  HeadsDev h, ObjIn in, const int32_t *npx, double *part) {
  __shared__ double red[32];
  const int v = blockIdx.x, b = blockIdx.y, nb = gridDim.y;
  const int64_t WH = (int64_t)ls.lw * ls.lh;
  const int64_t v0 = h.view_samp[v], v1 = h.view_samp[v + 1];
  const int64_t chunk = (v1 - v0 + nb - 1) / nb;
  const int64_t s0 = v0 + b * chunk, s1 = min(v1, s0 + chunk);
  double acc = 0.0;
  if (in.obs_depth && npx[v] > 0) {
    for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
      const int64_t flat = h.samp[i];
      const int64_t g = flat / K;
      if (ls.status[g] != DIST_CONVERGED || !depth_valid(in, g)) continue;
      int cnt = 0;
      for (int k = 0; k < K; ++k) cnt += isfinite(ls.tk_a[g * K + k]) ? 1 : 0;
      const int64_t q = g - v * WH;
      const int j = (int)(q / ls.lw), ii = (int)(q - (int64_t)j * ls.lw);
      double dir[3], scale;
      pixel_ray(cams[v], ii, j, 1, dir, &scale);
      const double w = (1.0 / cnt) / (double)npx[v];
      const double r = __dmul_rn(__dadd_rn(ls.tk_d[flat], h.f[i]), scale) - in.obs_depth[g];
      acc += w * fabs(r);
    }
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[(size_t)v * nb + b] = s;
}

__global__ void k_view_loss_finish(int V, int nb, const double *__restrict__ part, double *terms) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[(size_t)v * nb + b];
    terms[v * kViewTerms + 0] = s;
  }
}

// per shape: grad += w_lat * 2 z; total = sum_views(w_d L_d + w_s L_s) + w_lat |z|^2
__global__ void k_shape_finish(const dist_camera *__restrict__ cams, int V, int S, int D,
                               const double *__restrict__ codes, const double *__restrict__ terms,
                               ObjIn in, double *grad, double *shape_terms) {
  __shared__ double red[32];
  const int s = blockIdx.x;
  double zz = 0.0;
  for (int k = threadIdx.x; k < D; k += blockDim.x) {
    const double z = codes[(size_t)s * D + k];
    zz += z * z;
    grad[(size_t)s * D + k] += in.w_lat * (2.0 * z);
  }
  const double reg = block_sum(zz, red);
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int v = 0; v < V; ++v)
      if (cams[v].shape == s)
        tot += in.w_depth * terms[v * kViewTerms + 0] + in.w_sil * terms[v * kViewTerms + 1] +
               in.w_normal * terms[v * kViewTerms + 4];
    shape_terms[s * 2 + 0] = tot + in.w_lat * reg;
    shape_terms[s * 2 + 1] = reg;
  }
}

// Adam (optimize.py:47-63) per shape, with the best-iterate bookkeeping of
// complete_shape (optimize.py:170-176) and the loss history.
__global__ void k_adam(int S, int D, double *params, const double *grad, double *m, double *v,
                       int32_t *t, int32_t *skipped, const double *shape_terms, double *best_loss,
                       double *best_params, int32_t *best_iter, int iter_host, const int32_t *iter_dev,
                       double *hist, dist_adam_config cfg) {
  __shared__ int s_bad;
  __shared__ int s_best;
  const int s = blockIdx.x;
  const int iter = iter_dev ? *iter_dev : iter_host;
  if (threadIdx.x == 0) {
    s_bad = 0;
    s_best = 0;
    if (shape_terms) {
      const double tot = shape_terms[s * 2];
      if (hist) hist[(size_t)iter * S + s] = tot;
      if (best_loss && tot < best_loss[s]) {
        best_loss[s] = tot;
        best_iter[s] = iter;
        s_best = 1;
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < D; k += blockDim.x) {
    if (s_best) best_params[(size_t)s * D + k] = params[(size_t)s * D + k];
    if (!isfinite(grad[(size_t)s * D + k])) atomicOr(&s_bad, 1);
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) skipped[s] += 1;
    return;
  }
  const int tt = t[s] + 1;
  const double c1 = 1.0 - pow(cfg.beta1, (double)tt), c2 = 1.0 - pow(cfg.beta2, (double)tt);
  for (int k = threadIdx.x; k < D; k += blockDim.x) {
    const size_t i = (size_t)s * D + k;
    const double g = grad[i];
    const double mm = cfg.beta1 * m[i] + (1.0 - cfg.beta1) * g;
    const double vv = cfg.beta2 * v[i] + (1.0 - cfg.beta2) * g * g;
    m[i] = mm;
    v[i] = vv;
    params[i] = params[i] - cfg.lr * (mm / c1) / (sqrt(vv / c2) + cfg.eps);
  }
  __syncthreads();
  if (threadIdx.x == 0) t[s] = tt;
}

// grad += w_lat * 2 z (latent_reg, losses.py:114-117), once per shape
__global__ void k_add_reg(int S, int D, const double *__restrict__ codes, double w_lat, double *grad) {
  const int s = blockIdx.x;
  for (int k = threadIdx.x; k < D; k += blockDim.x)
    grad[(size_t)s * D + k] += w_lat * (2.0 * codes[(size_t)s * D + k]);
}

__global__ void k_iter_inc(int32_t *it) { *it += 1; }

struct ObjLayout {
  HeadsDev h;
  double *c0, *cs, *sil_seed, *gdotv, *probe_f, *loss_part;
  fx_t *part0, *parts, *col0, *cols;          // exact fixed-point column sums (common.cuh)
  int *bad;                                   // non-finite gradient contribution seen
  int32_t *npx, *bcount, *conv, *conv_count;
  int32_t *sel_own, *sel_oth, *sel_counts;   // samples with / without a ReLU-mask record
  int32_t *rec_rank;                          // [n] index of a recorded ray in h.rec
  // normal term
  double *nunit, *nraw, *nnorm, *npart;
  int32_t *nlist, *ncount;
  size_t bytes;
};

// flags of dist_objective_workspace_size
constexpr int kObjNormals = 1;

static ObjLayout obj_layout(const DecView &dv, int V, int W, int H, int K, int S, int mode,
                            int flags, char *ws, size_t cap) {
  ObjLayout L{};
  Carve cv{ws, 0, cap};
  const int64_t n = (int64_t)V * W * H;
  const int s1 = std::max(S, 1);
  const bool probes = mode >= 1 || (flags & kObjNormals);
  const bool normals = flags & kObjNormals;
  L.h.rec = cv.take<int32_t>(n);
  L.rec_rank = cv.take<int32_t>(n);
  L.h.best = cv.take<int32_t>(n);
  L.h.samp = cv.take<int32_t>(n * K);
  L.h.samp_pix = cv.take<int32_t>(n * K);
  L.h.f = cv.take<double>(n * K);
  L.h.view_rec = cv.take<int32_t>(V + 1);
  L.h.view_samp = cv.take<int32_t>(V + 1);
  L.h.counts = cv.take<int32_t>(4);
  L.sel_own = cv.take<int32_t>(n * K);
  L.sel_oth = cv.take<int32_t>(n * K);
  L.sel_counts = cv.take<int32_t>(4);
  L.sil_seed = cv.take<double>(n);
  L.gdotv = cv.take<double>(mode >= 1 ? n : 1);
  L.probe_f = cv.take<double>(probes ? n * 6 : 1);   // implicit modes and the normal term
  L.conv = cv.take<int32_t>(probes ? n : 1);
  L.conv_count = cv.take<int32_t>(4);
  L.nunit = cv.take<double>(normals ? n * 3 : 1);
  L.nraw = cv.take<double>(normals ? n : 1);
  L.nlist = cv.take<int32_t>(normals ? n : 1);
  L.ncount = cv.take<int32_t>(4);
  L.nnorm = cv.take<double>(V);
  L.npart = cv.take<double>((size_t)V * kPrepBlocks * 2);
  L.npx = cv.take<int32_t>(V);
  L.loss_part = cv.take<double>((size_t)V * std::max(kLossBlocks, 3 * kPrepBlocks));
  L.bcount = cv.take<int32_t>(ceil_div(n * K, kScanBlock) + 1);
  L.c0 = cv.take<double>(c0_doubles(s1, dv.np[0]));
  L.cs = cv.take<double>(c0_doubles(s1, std::max(dv.nskip, 1)));
  const int G = vjp_grid_cap(dv.prec);
  L.part0 = cv.take<fx_t>((size_t)G * s1 * dv.np[0]);
  L.parts = cv.take<fx_t>((size_t)G * s1 * std::max(dv.nskip, 1));
  L.col0 = cv.take<fx_t>((size_t)s1 * dv.np[0]);
  L.cols = cv.take<fx_t>((size_t)s1 * std::max(dv.nskip, 1));
  L.bad = cv.take<int>(4);
  L.bytes = cv.off + 256;
  return L;
}

}  // namespace dist

using namespace dist;

extern "C" {

size_t dist_objective_workspace_size(const dist_decoder *dec, int V, int W, int H, int K, int S,
                                     int mode, int flags) {
  if (!dec) return 0;
  return obj_layout(dec->view, V, W, H, K, S, mode, flags, nullptr, ~size_t(0)).bytes;
}

int dist_objective(const dist_decoder *dec, const double *codes, int S, const dist_camera *cams,
                   int V, int W, int H, const dist_trace_config *cfg, const dist_ray_state *st,
                   const dist_objective_io *io, void *ws, size_t ws_bytes, void *stream) {
  if (!dec || !cams || !cfg || !st || !io || !io->grad || !io->view_terms || !io->shape_terms)
    return fail(DIST_ERR_CONFIG, "null argument");
  const DecView &dv = dec->view;
  if (dv.latent_dim > 0 && (!codes || S < 1)) return fail(DIST_ERR_CONFIG, "field expects a latent code");
  if (io->phase < 0 || io->phase > 2) return fail(DIST_ERR_CONFIG, "phase must be 0, 1 or 2");
  if (io->grad_mode < 0 || io->grad_mode > 2)
    return fail(DIST_ERR_CONFIG, "grad_mode must be 0 (surrogate), 1 (implicit) or 2 (implicit, unit normal)");
  const int K = cfg->k_samples;
  if (K < 1 || K > 16) return fail(DIST_ERR_CONFIG, "k_samples must be in [1, 16]");
  if (V < 1 || W < 1 || H < 1) return fail(DIST_ERR_CONFIG, "resolution must be positive");
  // sample ids g*K + k are int32 (h.samp, the selection lists, the scan)
  if ((int64_t)V * W * H * K >= ((int64_t)1 << 31))
    return fail(DIST_ERR_CONFIG, "too many samples (views x pixels x k_samples) for one objective call");
  cudaStream_t sm = (cudaStream_t)stream;
  const int s1 = std::max(S, 1);
  const bool want_n = io->obs_normal != nullptr;
  ObjLayout L = obj_layout(dv, V, W, H, K, S, io->grad_mode, want_n ? kObjNormals : 0, (char *)ws, ws_bytes);
  if (L.bytes > ws_bytes) return fail(DIST_ERR_CONFIG, "objective workspace too small");
  const int64_t n = (int64_t)V * W * H, WH = (int64_t)W * H;
  LevelState ls{st->d, st->b, st->status, st->steps, st->topk_d, st->topk_f, st->topk_absf, W, H, 1, n};
  // the march's ReLU-mask record (include/dist.h): samples its own queries
  // wrote skip the taped forward
  const bool use_masks = st->relu_masks && st->topk_slot && tc_heads_supported(dv);
  if (use_masks) {
    ls.masks = st->relu_masks;
    ls.tk_p = st->topk_slot;
    ls.nmask = dv.n_layers - 1;
  }
  ObjIn in{io->obs_depth, io->obs_depth_mask, io->obs_sil, io->w_depth, io->w_sil, io->w_latent,
           want_n ? io->w_normal : 0.0};
  NormIn nin{L.nunit, L.nraw, io->obs_normal, io->obs_normal_mask};
  const double *vnorm = io->phase == 2 ? io->view_norm : nullptr;
  int rc = DIST_OK;
  cudaError_t e;

  if (io->phase != 2) {
    // 1. sample list
    const double *ta = st->topk_absf;
    const int Kc = K;
    rc = compact([ta, Kc] __device__(int64_t g) { return (bool)isfinite(ta[g * Kc]); }, n, L.h.rec,
                 L.h.counts + 0, L.bcount, sm, L.rec_rank);
    if (rc) return rc;
    // Only samples that carry a seed enter the fused kernel: slot 0 of every
    // recorded ray when a silhouette term is present, and every sample of a
    // converged pixel with a valid depth observation (losses.py:60-75).  The
    // others contribute neither loss nor gradient (~60% of K=3
    // samples remain in the depth-only C3 objective).
    const uint8_t *status = st->status;
    const bool has_sil = io->obs_sil != nullptr;
    const ObjIn inq = in;
    rc = compact(
        [ta, Kc, status, has_sil, inq] __device__(int64_t q) {
          if (!isfinite(ta[q])) return false;
          const int64_t g = q / Kc;
          if (has_sil && q - g * Kc == 0) return true;
          return status[g] == DIST_CONVERGED && depth_valid(inq, g);
        },
        n * K, L.h.samp, L.h.counts + 1, L.bcount, sm);
    if (rc) return rc;
    const int gi = (int)std::min<int64_t>(ceil_div(n * K, 256), (int64_t)sm_count() * 16);
    k_heads_index<<<std::max(gi, 1), 256, 0, sm>>>(L.h, L.rec_rank, K, V, WH);
    DIST_CHECK_LAUNCH("k_heads_index");
    // the decoder's per-shape code bias, shared by the probe pass and the heads
    rc = launch_code_bias(dv, dv.latent_dim > 0 ? codes : nullptr, s1, L.c0, L.cs, sm);
    if (rc) return rc;
    // normal probes at the converged pixels: implicit-gradient factors and/or
    // the rendered normals of the normal term (shading.py:190-225)
    if (io->grad_mode >= 1 || want_n) {
      rc = normals_pass(dv, L.c0, L.cs, s1, cams, ls, cfg, want_n ? L.nunit : nullptr,
                        io->grad_mode >= 1 ? L.gdotv : nullptr, L.conv, L.conv_count, L.bcount,
                        L.probe_f, sm, io->grad_mode == 2, want_n ? L.nraw : nullptr);
      if (rc) return rc;
    }
  }
  // 2. per-view loss preparation (phase 2: again, with the whole views' normalisers)
  // blocks per view: fixed by the view size only, so a view's (or a tile's)
  // partial sums do not depend on what else is in the batch
  const int nb_prep = (int)std::min<int64_t>(kPrepBlocks, std::max<int64_t>(1, ceil_div(WH, 2048)));
  const int nb_loss = (int)std::min<int64_t>(kLossBlocks, std::max<int64_t>(1, ceil_div(WH * K, 8192)));
  k_view_prep<<<dim3(V, nb_prep), 256, 0, sm>>>(cams, ls, K, cfg->epsilon, in, vnorm, L.loss_part,
                                                L.sil_seed);
  DIST_CHECK_LAUNCH("k_view_prep");
  k_view_prep_finish<<<(int)ceil_div(V, 128), 128, 0, sm>>>(V, nb_prep, (int64_t)W * H, L.loss_part,
                                                            in.obs_sil != nullptr, vnorm, L.npx,
                                                            io->view_terms);
  DIST_CHECK_LAUNCH("k_view_prep_finish");
  if (want_n) {
    k_view_normal<<<dim3(V, nb_prep), 256, 0, sm>>>(ls, nin, L.npart);
    DIST_CHECK_LAUNCH("k_view_normal");
    k_view_normal_finish<<<(int)ceil_div(V, 128), 128, 0, sm>>>(V, nb_prep, L.npart, vnorm, L.nnorm,
                                                                io->view_terms);
    DIST_CHECK_LAUNCH("k_view_normal_finish");
    if (io->phase != 2) {
      const LevelState lsq = ls;
      const NormIn nq = nin;
      rc = compact([lsq, nq] __device__(int64_t g) { return normal_valid(lsq, nq, g); }, n, L.nlist,
                   L.ncount, L.bcount, sm);
      if (rc) return rc;
    }
  } else {
    e = cudaMemsetAsync(L.nnorm, 0, sizeof(double) * V, sm);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(nnorm)");
    // view_terms[4..5] = 0: no normal term
    k_view_normal_finish<<<(int)ceil_div(V, 128), 128, 0, sm>>>(V, 0, L.npart, nullptr, L.nnorm,
                                                                io->view_terms);
    DIST_CHECK_LAUNCH("k_view_normal_finish");
  }
  if (io->phase == 1) return DIST_OK;

  // 3. fused forward -> seed -> backward
  const int G = vjp_grid_cap(dv.prec);
  e = cudaMemsetAsync(L.part0, 0, sizeof(fx_t) * G * s1 * dv.np[0], sm);
  if (e == cudaSuccess && dv.nskip) e = cudaMemsetAsync(L.parts, 0, sizeof(fx_t) * G * s1 * dv.nskip, sm);
  if (e == cudaSuccess) e = cudaMemsetAsync(L.bad, 0, sizeof(int), sm);
  if (e == cudaSuccess) e = cudaMemsetAsync(io->grad, 0, sizeof(double) * s1 * std::max(dv.latent_dim, 1), sm);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(objective)");
  ObjGen gen{cams, ls, K, WH, L.h, in, L.npx, io->obs_sil ? L.sil_seed : nullptr,
             io->grad_mode >= 1 ? L.gdotv : nullptr};
  int grid = 0;
  if (use_masks) {
    // split the sample list: rows with a mask record -> backward-only kernel
    const int32_t *samp = L.h.samp, *nsamp = L.h.counts + 1;
    const uint8_t *tkp = st->topk_slot;
    const int Kc = K;
    for (int want = 1; want >= 0 && !rc; --want)
      rc = compact(
          [samp, nsamp, tkp, Kc, want] __device__(int64_t i) {
            if (i >= *nsamp) return false;
            const int64_t flat = samp[i];
            const int64_t g = flat / Kc;
            return (int)((tkp[g * (Kc + 1) + (flat - g * Kc)] & 0x80) != 0) == want;
          },
          n * K, want ? L.sel_own : L.sel_oth, L.sel_counts + (want ? 0 : 1), L.bcount, sm);
    if (rc) return rc;
    ObjGen gown = gen, goth = gen;
    gown.sel = L.sel_own;
    gown.sel_count = L.sel_counts + 0;
    goth.sel = L.sel_oth;
    goth.sel_count = L.sel_counts + 1;
    int grid2 = 0;
    rc = launch_tc_heads_bwd(dv, L.c0, L.cs, gown, n * K, s1, L.part0, L.parts, L.bad, G, &grid, sm);
    if (!rc) rc = launch_tc_heads<ObjGen>(dv, L.c0, L.cs, goth, n * K, s1, L.part0, L.parts, L.bad, G, &grid2, sm);
    grid = std::max(grid, grid2);
  } else if (tc_heads_supported(dv))
    rc = launch_tc_heads<ObjGen>(dv, L.c0, L.cs, gen, n * K, s1, L.part0, L.parts, L.bad, G, &grid, sm);
  else if (dv.prec == DIST_PREC_FP64)
    rc = launch_vjp_gen<double>(dv, L.c0, L.cs, gen, n * K, s1, L.part0, L.parts, nullptr, L.bad, G, &grid, sm);
  else
    rc = launch_vjp_gen<float>(dv, L.c0, L.cs, gen, n * K, s1, L.part0, L.parts, nullptr, L.bad, G, &grid, sm);
  if (rc) return rc;
  if (want_n) {
    // normal-loss probe rows: taped forward + reverse sweep on the SIMT path
    // (fp32 for the tensor-core decoders): the +-1/(2 delta) seeds difference
    // two nearly equal gradients, which the head kernel's fp16 backward
    // operand could not resolve (the x500 conditioning of SURVEY 0 finding 3)
    NormalGen ng{cams, ls, L.nlist, L.ncount, cfg->alpha, cfg->normal_delta, in.w_normal, nin, L.nnorm};
    int gridn = 0;
    if (dv.prec == DIST_PREC_FP64)
      rc = launch_vjp_gen<double>(dv, L.c0, L.cs, ng, n * 6, s1, L.part0, L.parts, nullptr, L.bad, G, &gridn, sm);
    else
      rc = launch_vjp_gen<float>(dv, L.c0, L.cs, ng, n * 6, s1, L.part0, L.parts, nullptr, L.bad, G, &gridn, sm);
    if (rc) return rc;
    grid = std::max(grid, gridn);
  }
  // 4. losses, code gradient, regulariser
  k_view_depth_loss<<<dim3(V, nb_loss), 256, 0, sm>>>(cams, ls, K, L.h, in, L.npx, L.loss_part);
  DIST_CHECK_LAUNCH("k_view_depth_loss");
  k_view_loss_finish<<<(int)ceil_div(V, 128), 128, 0, sm>>>(V, nb_loss, L.loss_part, io->view_terms);
  DIST_CHECK_LAUNCH("k_view_loss_finish");
  if (dv.latent_dim > 0) {
    // the caller may take the exact column sums (cross-rank reduction, then
    // dist_code_grad_fixed); grad is always formed from the local sums
    // layout [S][np0] then (skip decoders) [S][nskip]
    fx_t *col0 = io->colsum_fixed ? reinterpret_cast<fx_t *>(io->colsum_fixed) : L.col0;
    fx_t *cols = io->colsum_fixed ? col0 + (size_t)s1 * dv.np[0] : L.cols;
    if (grid == 0) {   // no seeded sample anywhere: zero sums
      e = cudaMemsetAsync(col0, 0, sizeof(fx_t) * s1 * dv.np[0], sm);
      if (e == cudaSuccess && dv.nskip) e = cudaMemsetAsync(cols, 0, sizeof(fx_t) * s1 * dv.nskip, sm);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(colsum)");
    }
    rc = reduce_code_grad(dv, s1, grid, L.part0, L.parts, L.bad, col0, cols, io->grad, sm);
    if (rc) return rc;
  }
  if (io->counts_out) {
    e = cudaMemcpyAsync(io->counts_out, L.h.counts, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, sm);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(counts)");
  }
  k_shape_finish<<<s1, 256, 0, sm>>>(cams, V, s1, dv.latent_dim, codes, io->view_terms, in, io->grad,
                                      io->shape_terms);
  DIST_CHECK_LAUNCH("k_shape_finish");
  return DIST_OK;
}

// Code gradient from exact column sums summed across ranks: every
// rank passes the same [S][np0] fixed-point totals and gets the same bits.
int dist_code_grad_fixed(const dist_decoder *dec, int S, const void *colsum_fixed,
                         const double *codes, double w_latent, double *grad, void *stream) {
  if (!dec || !colsum_fixed || !grad) return fail(DIST_ERR_CONFIG, "null argument");
  const DecView &dv = dec->view;
  if (S < 1) return fail(DIST_ERR_CONFIG, "S must be >= 1");
  if (dv.latent_dim == 0) return DIST_OK;
  cudaStream_t sm = (cudaStream_t)stream;
  fx_t *col0 = const_cast<fx_t *>(reinterpret_cast<const fx_t *>(colsum_fixed));
  int rc = reduce_code_grad(dv, S, 0, nullptr, nullptr, nullptr, col0,
                            dv.nskip ? col0 + (size_t)S * dv.np[0] : nullptr, grad, sm);
  if (rc) return rc;
  if (codes && w_latent != 0.0) {
    k_add_reg<<<S, 256, 0, sm>>>(S, dv.latent_dim, codes, w_latent, grad);
    DIST_CHECK_LAUNCH("k_add_reg");
  }
  return DIST_OK;
}

int dist_adam_step(int S, int D, double *params, const double *grad, double *m, double *v,
                   int32_t *t, int32_t *skipped, const double *shape_terms, double *best_loss,
                   double *best_params, int32_t *best_iter, int iter, double *hist,
                   const dist_adam_config *cfg, int32_t *iter_dev, void *stream) {
  if (!params || !grad || !m || !v || !t || !skipped || !cfg) return fail(DIST_ERR_CONFIG, "null argument");
  if (S < 1 || D < 0) return fail(DIST_ERR_CONFIG, "bad Adam shape");
  if (D == 0) return DIST_OK;
  cudaStream_t st = (cudaStream_t)stream;
  k_adam<<<S, 256, 0, st>>>(S, D, params, grad, m, v, t, skipped, shape_terms, best_loss, best_params,
                            best_iter, iter, iter_dev, hist, *cfg);
  DIST_CHECK_LAUNCH("k_adam");
  if (iter_dev) {   // the iteration index lives on the device (a captured iterate replays as is)
    k_iter_inc<<<1, 1, 0, st>>>(iter_dev);
    DIST_CHECK_LAUNCH("k_iter_inc");
  }
  return DIST_OK;
}

}  // extern "C"
