// pose.cu -- pose recovery's objective on the device:
// pose_objective (optimize.py:185-233) with the frozen marching record of one
// traced view.  The rows are dense, K per pixel (ray id g, top-K slot k): row
// (g, k) is a head sample when pixel g is recorded (top-K slot 0 finite) and
// slot k is finite (HeadBundle, shading.py:156-281); any other row has the
// origin as its point and seed 0.
//
//   dist_pose_samples : the sample points origin + topk_d * dir;
//   dist_pose_seeds   : depth_loss (losses.py:54-75: each valid pixel's samples
//                       share one unit, L1 on camera z) and silhouette_loss
//                       (losses.py:78-91: hinge on the soft silhouette) -- the
//                       loss values (one block, fixed order) and the per-row
//                       seeds w_depth * s + w_sil * gimg (best sample);
//   dist_pose_grad    : the chain rule of camera.py:255-278 with the distances
//                       frozen, p_m = c + d_m v_m, over the head rows (point
//                       gradients from dist_eval_vjp) and the unrecorded
//                       pixels' silhouette term (the closest point of the ray
//                       to the origin, optimize.py:220-229): 6 numbers, one
//                       block, fixed order.
// Memory-light single-view work: a few reads per row.
#include <cmath>

#include "common.cuh"

namespace dist {

struct PoseView {
  const dist_camera *cam;
  int W, H, K;
  const uint8_t *status;
  const double *topk_d, *topk_absf;
  __device__ bool recorded(int64_t g) const { return isfinite(topk_absf[g * K]); }
  __device__ bool sample(int64_t g, int k) const { return recorded(g) && isfinite(topk_absf[g * K + k]); }
  __device__ int count(int64_t g) const {
    int c = 0;
    for (int k = 0; k < K; ++k) c += isfinite(topk_absf[g * K + k]) ? 1 : 0;
    return c;
  }
};

__device__ __forceinline__ void pose_ray(const PoseView &pv, int64_t g, double dir[3], double *scale) {
  const int j = (int)(g / pv.W), i = (int)(g - (int64_t)j * pv.W);
  pixel_ray(*pv.cam, i, j, 1, dir, scale);
}

__global__ void k_pose_samples(PoseView pv, double *__restrict__ pts) {
  const int64_t n = (int64_t)pv.W * pv.H * pv.K;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = r / pv.K;
    const int k = (int)(r - g * pv.K);
    const bool ok = pv.sample(g, k);
    double dir[3], sc;
    pose_ray(pv, g, dir, &sc);
    const double d = pv.topk_d[r];
    const double *o = pv.cam->origin;
    for (int a = 0; a < 3; ++a) pts[r * 3 + a] = ok ? __dadd_rn(o[a], __dmul_rn(d, dir[a])) : 0.0;
  }
}

// silhouette gradient image value of pixel g: (t (s > 0) - (1 - t) (s < 0)) / n
__device__ __forceinline__ double sil_grad(const double *soft, const double *target, int64_t g, double inv_n) {
  const double s = soft[g], t = target[g];
  return (t * (s > 0.0 ? 1.0 : 0.0) - (1.0 - t) * (s < 0.0 ? 1.0 : 0.0)) * inv_n;
}

__device__ __forceinline__ bool depth_valid(const PoseView &pv, const uint8_t *obs_valid, int64_t g) {
  return pv.status[g] == DIST_CONVERGED && pv.recorded(g) && obs_valid[g];
}

// one block: out[0] = depth loss, out[1] = silhouette loss, out[2] = n_px
__global__ void k_pose_loss(PoseView pv, const double *__restrict__ f, const double *__restrict__ obs_depth,
                            const uint8_t *__restrict__ obs_valid, const double *__restrict__ soft,
                            const double *__restrict__ target, double *__restrict__ out) {
  __shared__ double sa[1024], sb[1024];
  __shared__ long long sn[1024];
  const int64_t n = (int64_t)pv.W * pv.H;
  long long c = 0;
  if (obs_depth)
    for (int64_t g = threadIdx.x; g < n; g += blockDim.x) c += depth_valid(pv, obs_valid, g) ? 1 : 0;
  sn[threadIdx.x] = c;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sn[threadIdx.x] += sn[threadIdx.x + s];
    __syncthreads();
  }
  const long long npx = sn[0];
  double a = 0.0, b = 0.0;
  for (int64_t g = threadIdx.x; g < n; g += blockDim.x) {
    if (obs_depth && npx > 0 && depth_valid(pv, obs_valid, g)) {
      double dir[3], sc;
      pose_ray(pv, g, dir, &sc);
      const double w = (1.0 / pv.count(g)) / (double)npx;   // sample_weight / n_px
      for (int k = 0; k < pv.K; ++k) {
        const int64_t r = g * pv.K + k;
        if (!isfinite(pv.topk_absf[r])) continue;
        const double res = __dmul_rn(__dadd_rn(pv.topk_d[r], f[r]), sc) - obs_depth[g];
        a += w * fabs(res);
      }
    }
    if (soft) {
      const double s = soft[g], t = target[g];
      b += t * fmax(s, 0.0) + (1.0 - t) * fmax(-s, 0.0);
    }
  }
  __syncthreads();
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      sa[threadIdx.x] += sa[threadIdx.x + s];
      sb[threadIdx.x] += sb[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sa[0];
    out[1] = soft ? sb[0] / (double)n : 0.0;
    out[2] = (double)npx;
  }
}

__global__ void k_pose_seeds(PoseView pv, const double *__restrict__ f, const double *__restrict__ obs_depth,
                             const uint8_t *__restrict__ obs_valid, const double *__restrict__ soft,
                             const double *__restrict__ target, double w_depth, double w_sil,
                             const double *__restrict__ loss, double *__restrict__ seed) {
  const int64_t npix = (int64_t)pv.W * pv.H, n = npix * pv.K;
  const double npx = loss[2], inv_n = 1.0 / (double)npix;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = r / pv.K;
    const int k = (int)(r - g * pv.K);
    double sd = 0.0;
    if (pv.sample(g, k)) {
      if (obs_depth && npx > 0.0 && depth_valid(pv, obs_valid, g)) {
        double dir[3], sc;
        pose_ray(pv, g, dir, &sc);
        const double w = (1.0 / pv.count(g)) / npx;
        const double res = __dmul_rn(__dadd_rn(pv.topk_d[r], f[r]), sc) - obs_depth[g];
        const double sg = res > 0.0 ? 1.0 : (res < 0.0 ? -1.0 : 0.0);
        sd = w_depth * (w * sg * sc);
      }
      if (soft && k == 0) sd += w_sil * sil_grad(soft, target, g, inv_n);   // the best sample
    }
    seed[r] = sd;
  }
}

// one block: out[0..2] = dL/d omega, out[3..5] = dL/d t.  mats = R, dR_0, dR_1,
// dR_2 (row-major 3x3 each), t.
__global__ void k_pose_grad(PoseView pv, const double *__restrict__ gp, const double *__restrict__ soft,
                            const double *__restrict__ target, double w_sil,
                            const double *__restrict__ mats, double *__restrict__ out) {
  __shared__ double red[6][256];
  const int64_t npix = (int64_t)pv.W * pv.H;
  const double inv_n = 1.0 / (double)npix;
  const double *R = mats, *t = mats + 36;
  double acc[6] = {0, 0, 0, 0, 0, 0};   // gs[3], T[3]
  auto add = [&](const double u[3], double d, const double gm[3]) {
    for (int b = 0; b < 3; ++b) acc[b] += gm[b];
    for (int q = 0; q < 3; ++q) {
      const double *dR = mats + 9 * (q + 1);
      double s = 0.0;
      for (int b = 0; b < 3; ++b) s += gm[b] * (u[0] * dR[0 * 3 + b] + u[1] * dR[1 * 3 + b] + u[2] * dR[2 * 3 + b]);
      acc[3 + q] += d * s;
    }
  };
  for (int64_t g = threadIdx.x; g < npix; g += blockDim.x) {
    const int j = (int)(g / pv.W), i = (int)(g - (int64_t)j * pv.W);
    double dir[3], sc;
    pixel_ray(*pv.cam, i, j, 1, dir, &sc);
    // unit camera-frame direction (camera.py pixel_dirs_cam)
    const dist_camera &c = *pv.cam;
    const double x = ((i + 0.5) - c.cx) / c.fx, y = ((j + 0.5) - c.cy) / c.fy;
    const double nn = sqrt(x * x + y * y + 1.0);
    const double u[3] = {x / nn, y / nn, 1.0 / nn};
    if (pv.recorded(g)) {
      for (int k = 0; k < pv.K; ++k) {
        const int64_t r = g * pv.K + k;
        if (!isfinite(pv.topk_absf[r])) continue;
        const double gm[3] = {gp[r * 3], gp[r * 3 + 1], gp[r * 3 + 2]};
        add(u, pv.topk_d[r], gm);
      }
    } else if (soft) {
      // d loss / d p at the ray's closest point to the origin (optimize.py:220-229)
      const double sd = w_sil * sil_grad(soft, target, g, inv_n);
      const double *o = c.origin;
      const double dstar = -(dir[0] * o[0] + dir[1] * o[1] + dir[2] * o[2]);
      const double ps[3] = {o[0] + dstar * dir[0], o[1] + dstar * dir[1], o[2] + dstar * dir[2]};
      const double nrm = sqrt(ps[0] * ps[0] + ps[1] * ps[1] + ps[2] * ps[2]);
      const double gm[3] = {nrm > 0.0 ? sd * (ps[0] / nrm) : 0.0, nrm > 0.0 ? sd * (ps[1] / nrm) : 0.0,
                            nrm > 0.0 ? sd * (ps[2] / nrm) : 0.0};
      add(u, dstar, gm);
    }
  }
  for (int q = 0; q < 6; ++q) red[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int q = 0; q < 6; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double gs[3] = {red[0][0], red[1][0], red[2][0]};
    for (int q = 0; q < 3; ++q) {
      const double *dR = mats + 9 * (q + 1);
      double v = 0.0;
      for (int b = 0; b < 3; ++b) v += gs[b] * -(dR[0 * 3 + b] * t[0] + dR[1 * 3 + b] * t[1] + dR[2 * 3 + b] * t[2]);
      out[q] = v + red[3 + q][0];
    }
    for (int a = 0; a < 3; ++a) out[3 + a] = -(R[a * 3 + 0] * gs[0] + R[a * 3 + 1] * gs[1] + R[a * 3 + 2] * gs[2]);
  }
}

static PoseView pose_view(const dist_camera *cam, int W, int H, int K, const dist_ray_state *st) {
  return PoseView{cam, W, H, K, st->status, st->topk_d, st->topk_absf};
}

}  // namespace dist

using namespace dist;

extern "C" {

int dist_pose_samples(const dist_camera *cam_dev, int width, int height, int k_samples,
                      const dist_ray_state *st, double *points_dev, void *stream) {
  if (!cam_dev || !st || !st->status || !st->topk_d || !st->topk_absf || !points_dev)
    return fail(DIST_ERR_CONFIG, "null argument");
  if (width <= 0 || height <= 0 || k_samples <= 0 || k_samples > 16) return fail(DIST_ERR_CONFIG, "bad shape");
  const int64_t n = (int64_t)width * height * k_samples;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4096);
  k_pose_samples<<<grid, 256, 0, (cudaStream_t)stream>>>(pose_view(cam_dev, width, height, k_samples, st),
                                                         points_dev);
  DIST_CHECK_LAUNCH("k_pose_samples");
  return DIST_OK;
}

int dist_pose_seeds(const dist_camera *cam_dev, int width, int height, int k_samples,
                    const dist_ray_state *st, const double *f_dev, const double *obs_depth,
                    const uint8_t *obs_valid, const double *soft_sil, const double *obs_sil,
                    double w_depth, double w_sil, double *loss_dev, double *seed_dev, void *stream) {
  if (!cam_dev || !st || !f_dev || !loss_dev || !seed_dev) return fail(DIST_ERR_CONFIG, "null argument");
  if ((obs_depth && !obs_valid) || (!soft_sil != !obs_sil)) return fail(DIST_ERR_CONFIG, "incomplete observation");
  if (width <= 0 || height <= 0 || k_samples <= 0 || k_samples > 16) return fail(DIST_ERR_CONFIG, "bad shape");
  cudaStream_t s = (cudaStream_t)stream;
  const PoseView pv = pose_view(cam_dev, width, height, k_samples, st);
  k_pose_loss<<<1, 1024, 0, s>>>(pv, f_dev, obs_depth, obs_valid, soft_sil, obs_sil, loss_dev);
  DIST_CHECK_LAUNCH("k_pose_loss");
  const int64_t n = (int64_t)width * height * k_samples;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4096);
  k_pose_seeds<<<grid, 256, 0, s>>>(pv, f_dev, obs_depth, obs_valid, soft_sil, obs_sil, w_depth, w_sil,
                                    loss_dev, seed_dev);
  DIST_CHECK_LAUNCH("k_pose_seeds");
  return DIST_OK;
}

int dist_pose_grad(const dist_camera *cam_dev, int width, int height, int k_samples,
                   const dist_ray_state *st, const double *point_grads_dev, const double *soft_sil,
                   const double *obs_sil, double w_sil, const double *mats_dev, double *grad_dev,
                   void *stream) {
  if (!cam_dev || !st || !point_grads_dev || !mats_dev || !grad_dev) return fail(DIST_ERR_CONFIG, "null argument");
  if (!soft_sil != !obs_sil) return fail(DIST_ERR_CONFIG, "incomplete observation");
  if (width <= 0 || height <= 0 || k_samples <= 0 || k_samples > 16) return fail(DIST_ERR_CONFIG, "bad shape");
  k_pose_grad<<<1, 256, 0, (cudaStream_t)stream>>>(pose_view(cam_dev, width, height, k_samples, st),
                                                   point_grads_dev, soft_sil, obs_sil, w_sil, mats_dev,
                                                   grad_dev);
  DIST_CHECK_LAUNCH("k_pose_grad");
  return DIST_OK;
}

}  // extern "C"
