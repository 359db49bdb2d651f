// heads.cuh -- frozen-sample head list and the per-sample seed generator of
// the fused objective (shading.py:166-206, losses.py:54-91), shared by the
// SIMT (mlp_eval.cuh) and tcgen05 (tc_heads.cu) backward kernels.
#pragma once
#include "common.cuh"
#include "march.cuh"

namespace dist {

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *a, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

struct HeadsDev {
  int32_t *rec, *samp, *samp_pix, *best, *view_rec, *view_samp, *counts;
  double *f;
};

struct ObjIn {
  const double *obs_depth;
  const uint8_t *obs_mask;
  const double *obs_sil;
  double w_depth, w_sil, w_lat, w_normal;
};

// per-view terms written by dist_objective (include/dist.h view_terms)
constexpr int kViewTerms = 6;

// Implicit-gradient modes: pixels with grad f . v >= -0.1 (within ~6 degrees
// of grazing, where -1/(grad f . v) exceeds 10 and amplifies the surface
// point's own error) carry no depth gradient.  The same rule is restated in
// oracle/sdf_oracle.py implicit_depth_seeds.
constexpr double kImplicitGrazing = 0.1;

// normal term inputs: rendered unit normals and |raw| of the Eq. 3 difference
// vector (from the probe pass), the observation and its mask
struct NormIn {
  const double *unit;     // [n][3]
  const double *rawnorm;  // [n]
  const double *obs;      // [n][3]
  const uint8_t *mask;    // [n] or null
};

// Probe rows of the normal loss: row 6r + a is probe a of valid pixel
// list[r], in the reference's order (shading.py:196-197: +e_x, +e_y, +e_z,
// -e_x, -e_y, -e_z around the surface point c + (d + (1-alpha) b) v).  The
// seed of a probe is +-raw_seed/(2 delta) with raw_seed = (I - n n^T) ns /
// |raw| and ns = w_normal * (-n_obs / n_valid) (losses.py:107-111,
// shading.py:259-269); it does not depend on f.
struct NormalGen {
  const dist_camera *cams;
  LevelState ls;
  const int32_t *list;
  const int32_t *cnt;
  double alpha, delta, w_normal;
  NormIn nn;
  const double *nnorm;   // [V] n_valid of each view (the whole view's when sharded)
  __device__ int64_t count() const { return (int64_t)*cnt * 6; }
  __device__ bool point(int64_t i, double p[3], int &s) const {
    const int64_t r = i / 6;
    const int a = (int)(i - r * 6);
    const int64_t g = list[r];
    const int64_t per = (int64_t)ls.lw * ls.lh;
    const int v = (int)(g / per);
    const int64_t pix = g - (int64_t)v * per;
    const int j = (int)(pix / ls.lw), ii = (int)(pix - (int64_t)j * ls.lw);
    double dir[3];
    pixel_ray(cams[v], ii, j, 1, dir, nullptr);
    const double ds = __dadd_rn(ls.d[g], __dmul_rn(1.0 - alpha, ls.b[g]));
    for (int q = 0; q < 3; ++q) p[q] = __dadd_rn(cams[v].origin[q], __dmul_rn(ds, dir[q]));
    const int axis = a % 3;
    p[axis] = __dadd_rn(p[axis], a < 3 ? delta : -delta);
    s = cams[v].shape;
    return true;
  }
  __device__ double seed(int64_t i, double) const {
    const int64_t r = i / 6;
    const int a = (int)(i - r * 6);
    const int64_t g = list[r];
    const int v = (int)(g / ((int64_t)ls.lw * ls.lh));
    const double n = nnorm[v];
    const double *o = nn.obs + g * 3, *u = nn.unit + g * 3;
    double ns[3];
    for (int c = 0; c < 3; ++c) ns[c] = w_normal * (-o[c] / n);
    const double un = u[0] * ns[0] + u[1] * ns[1] + u[2] * ns[2];
    const int axis = a % 3;
    const double rs = (ns[axis] - u[axis] * un) / nn.rawnorm[g];
    const double pp = rs / (2.0 * delta);
    return a < 3 ? pp : -pp;
  }
  __device__ void store(int64_t, double) const {}
};

__device__ __forceinline__ bool depth_valid(const ObjIn &in, int64_t g) {
  if (!in.obs_depth) return false;
  const double z = in.obs_depth[g];
  bool ok = isfinite(z);
  if (in.obs_mask) ok = ok && in.obs_mask[g];
  return ok;
}

// Generator for the fused forward -> seed -> backward over head samples.
struct ObjGen {
  const dist_camera *cams;
  LevelState ls;
  int K;
  int64_t WH;
  HeadsDev h;
  ObjIn in;
  const int32_t *npx;
  const double *sil_seed;
  const double *gdotv;   // implicit mode: grad f . v per ray (raw Eq. 3 vector), else null
  // optional row -> sample map: the samples split by the ReLU-mask record
  // (rows of the backward-only head kernel / of the full one)
  const int32_t *sel = nullptr;
  const int32_t *sel_count = nullptr;
  __device__ int64_t at(int64_t r) const { return sel ? (int64_t)sel[r] : r; }
  __device__ int64_t count() const { return sel ? (int64_t)*sel_count : (int64_t)h.counts[1]; }
  // backward-only rows: the march's f at the sample (tracer.py:141 records it)
  // and the ReLU masks its query left in the ray's record (march.cuh)
  __device__ double f_rec(int64_t r) const { return ls.tk_f[h.samp[at(r)]]; }
  __device__ const uint32_t *masks_rec(int64_t r) const {
    const int64_t flat = h.samp[at(r)];
    const int64_t g = flat / K;
    return mask_record(ls, K, g, ls.tk_p[g * (K + 1) + (flat - g * K)] & 0x7f);
  }
  __device__ bool point(int64_t i, double p[3], int &s) const {
    const int64_t flat = h.samp[at(i)];
    const int64_t g = flat / K;
    const int v = (int)(g / WH);
    const int64_t q = g - v * WH;
    const int j = (int)(q / ls.lw), ii = (int)(q - (int64_t)j * ls.lw);
    double dir[3];
    pixel_ray(cams[v], ii, j, 1, dir, nullptr);
    const double dk = ls.tk_d[flat];
    for (int a = 0; a < 3; ++a) p[a] = __dadd_rn(cams[v].origin[a], __dmul_rn(dk, dir[a]));
    s = cams[v].shape;
    return true;
  }
  __device__ double seed(int64_t i, double f) const {
    const int64_t flat = h.samp[at(i)];
    const int64_t g = flat / K;
    const int v = (int)(g / WH);
    double sd = 0.0;
    if (in.obs_depth && ls.status[g] == DIST_CONVERGED && depth_valid(in, g) && npx[v] > 0) {
      int cnt = 0;
      for (int k = 0; k < K; ++k) cnt += isfinite(ls.tk_a[g * K + k]) ? 1 : 0;
      const int64_t q = g - v * WH;
      const int j = (int)(q / ls.lw), ii = (int)(q - (int64_t)j * ls.lw);
      double dir[3], scale;
      pixel_ray(cams[v], ii, j, 1, dir, &scale);
      const double w = (1.0 / cnt) / (double)npx[v];
      const double r = __dmul_rn(__dadd_rn(ls.tk_d[flat], f), scale) - in.obs_depth[g];
      const double sg = r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0);
      sd = in.w_depth * __dmul_rn(__dmul_rn(w, sg), scale);
      if (gdotv) {  // implicit gradient: scale by -1/(grad f . v), drop grazing
        const double gv = gdotv[g];
        sd = gv < -kImplicitGrazing ? sd * (-1.0 / gv) : 0.0;
      }
    }
    if (sil_seed && flat - g * K == 0) sd = __dadd_rn(sd, sil_seed[g]);
    return sd;
  }
  __device__ void store(int64_t i, double v) const { h.f[at(i)] = v; }

  // seed(i, f) split in two for the tensor-core head kernel: prep() does every
  // load at tile start (overlapping the forward GEMMs), apply() needs only f.
  // Bit-identical to seed(): the +-1 sign factor commutes exactly with the
  // roundings it is moved across.
  struct Prep {
    double d, scale, obs, c1, ginv, sil;   // c1 = w_depth * (w * scale); 0 if no depth term
  };
  __device__ Prep prep(int64_t i) const {
    Prep r{0.0, 0.0, 0.0, 0.0, 1.0, 0.0};
    const int64_t flat = h.samp[at(i)];
    const int64_t g = flat / K;
    const int v = (int)(g / WH);
    if (in.obs_depth && ls.status[g] == DIST_CONVERGED && depth_valid(in, g) && npx[v] > 0) {
      int cnt = 0;
      for (int k = 0; k < K; ++k) cnt += isfinite(ls.tk_a[g * K + k]) ? 1 : 0;
      const int64_t q = g - v * WH;
      const int j = (int)(q / ls.lw), ii = (int)(q - (int64_t)j * ls.lw);
      double dir[3], scale;
      pixel_ray(cams[v], ii, j, 1, dir, &scale);
      const double w = (1.0 / cnt) / (double)npx[v];
      r.d = ls.tk_d[flat];
      r.scale = scale;
      r.obs = in.obs_depth[g];
      r.c1 = in.w_depth * __dmul_rn(w, scale);
      if (gdotv) {
        const double gv = gdotv[g];
        r.ginv = gv < -kImplicitGrazing ? (-1.0 / gv) : 0.0;
      }
    }
    if (sil_seed && flat - g * K == 0) r.sil = sil_seed[g];
    return r;
  }
  __device__ double apply(const Prep &p, double f) const {
    double sd = 0.0;
    if (p.c1 != 0.0) {
      const double r = __dmul_rn(__dadd_rn(p.d, f), p.scale) - p.obs;
      const double sg = r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0);
      sd = sg * p.c1;
      if (gdotv) sd = sd * p.ginv;
    }
    if (sil_seed) sd = __dadd_rn(sd, p.sil);
    return sd;
  }
};

}  // namespace dist
