// photometric.cu -- multi-view photometric consistency:
// visibility_mask, bilinear_sample and photometric_loss of losses.py:128-222
// as per-pixel device kernels.  View i's depth is unprojected, projected into
// view j, visibility-tested against j's depth (squared depth gap < thresh),
// j's gray image is bilinearly sampled and the L1 residual's gradient is
// pushed back to i's depth through the warp (losses.py:210-221).
//
// Three launches: per-pixel residual / raw gradient, a single-block
// fixed-order reduction (n visible, sum |r|), and the 1/n normalisation, so
// the loss is deterministic.  HBM-bound: 3 x 8 B reads + a 4-pixel gather per
// pixel.
#include <cmath>

#include "common.cuh"

namespace dist {

struct PhotoCam {
  double R[9], t[3];
  double fx, fy, cx, cy;
};

__device__ __forceinline__ PhotoCam photo_cam(const dist_camera &c) {
  PhotoCam p;
  for (int i = 0; i < 9; ++i) p.R[i] = c.R[i];
  // t = -R c (camera.py:157-172 inverted)
  for (int r = 0; r < 3; ++r)
    p.t[r] = -(c.R[r * 3 + 0] * c.origin[0] + c.R[r * 3 + 1] * c.origin[1] + c.R[r * 3 + 2] * c.origin[2]);
  p.fx = c.fx;
  p.fy = c.fy;
  p.cx = c.cx;
  p.cy = c.cy;
  return p;
}

__global__ void k_photo_pixels(const dist_camera *__restrict__ cams, int H, int W, int Hj, int Wj,
                               const double *__restrict__ zi, const double *__restrict__ gi,
                               const double *__restrict__ gj, const double *__restrict__ zj,
                               double thresh, double *__restrict__ absr, double *__restrict__ graw,
                               uint8_t *__restrict__ vis) {
  const PhotoCam ci = photo_cam(cams[0]), cj = photo_cam(cams[1]);
  const int64_t n = (int64_t)H * W;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    absr[p] = 0.0;
    graw[p] = 0.0;
    vis[p] = 0;
    const double z = zi[p];
    if (!isfinite(z)) continue;
    const int y = (int)(p / W), x = (int)(p - (int64_t)y * W);
    const double u = x + 0.5, v = y + 0.5;
    // unproject (losses.py:171; camera.py:232-240): world = R_i^T (p_c - t_i)
    const double pc[3] = {(u - ci.cx) / ci.fx * z, (v - ci.cy) / ci.fy * z, z};
    double w[3];
    for (int a = 0; a < 3; ++a)
      w[a] = (pc[0] - ci.t[0]) * ci.R[0 * 3 + a] + (pc[1] - ci.t[1]) * ci.R[1 * 3 + a] +
             (pc[2] - ci.t[2]) * ci.R[2 * 3 + a];
    // project into j (camera.py:219-229)
    double q[3];
    for (int r = 0; r < 3; ++r)
      q[r] = cj.R[r * 3 + 0] * w[0] + cj.R[r * 3 + 1] * w[1] + cj.R[r * 3 + 2] * w[2] + cj.t[r];
    const double uj = cj.fx * q[0] / q[2] + cj.cx, vj = cj.fy * q[1] / q[2] + cj.cy;
    // visibility (losses.py:159-183)
    const double sx = uj - 0.5, sy = vj - 0.5;
    const bool inb = sx >= 0.0 && sx <= Wj - 1.0 && sy >= 0.0 && sy <= Hj - 1.0 && q[2] > 0.0;
    if (!inb) continue;
    const int xi = min(max((int)rint(sx), 0), Wj - 1), yi = min(max((int)rint(sy), 0), Hj - 1);
    const double zs = zj[(int64_t)yi * Wj + xi];
    if (!isfinite(zs) || !((q[2] - zs) * (q[2] - zs) < thresh)) continue;
    vis[p] = 1;
    // bilinear sample of gray_j at (uj, vj) and its derivatives (losses.py:128-150)
    const double xs = fmin(fmax(uj - 0.5, 0.0), Wj - 1.0), ys = fmin(fmax(vj - 0.5, 0.0), Hj - 1.0);
    const int x0 = Wj > 1 ? min(max((int)floor(xs), 0), Wj - 2) : 0;
    const int y0 = Hj > 1 ? min(max((int)floor(ys), 0), Hj - 2) : 0;
    const int x1 = min(x0 + 1, Wj - 1), y1 = min(y0 + 1, Hj - 1);
    const double fx = xs - x0, fy = ys - y0;
    const double v00 = gj[(int64_t)y0 * Wj + x0], v10 = gj[(int64_t)y0 * Wj + x1];
    const double v01 = gj[(int64_t)y1 * Wj + x0], v11 = gj[(int64_t)y1 * Wj + x1];
    const double val = (v00 * (1 - fx) + v10 * fx) * (1 - fy) + (v01 * (1 - fx) + v11 * fx) * fy;
    const double gu = (v10 - v00) * (1 - fy) + (v11 - v01) * fy;
    const double gv = (v01 - v00) * (1 - fx) + (v11 - v10) * fx;
    const double r = gi[p] - val;
    absr[p] = fabs(r);
    // d(warp uv)/dz: the unprojected point slides along the pixel's ray (losses.py:210-221)
    const double ray_c[3] = {(u - ci.cx) / ci.fx, (v - ci.cy) / ci.fy, 1.0};
    double ray[3];
    for (int a = 0; a < 3; ++a)
      ray[a] = ray_c[0] * ci.R[0 * 3 + a] + ray_c[1] * ci.R[1 * 3 + a] + ray_c[2] * ci.R[2 * 3 + a];
    double dX[3];
    for (int r2 = 0; r2 < 3; ++r2)
      dX[r2] = cj.R[r2 * 3 + 0] * ray[0] + cj.R[r2 * 3 + 1] * ray[1] + cj.R[r2 * 3 + 2] * ray[2];
    const double Z = q[2];
    const double du = cj.fx * (dX[0] / Z - q[0] * dX[2] / (Z * Z));
    const double dv = cj.fy * (dX[1] / Z - q[1] * dX[2] / (Z * Z));
    const double sg = r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0);
    graw[p] = -sg * (gu * du + gv * dv);
  }
}

// single block: n = #visible, loss = sum |r| / n (fixed order)
__global__ void k_photo_reduce(int64_t n, const double *__restrict__ absr,
                               const uint8_t *__restrict__ vis, double *__restrict__ out) {
  __shared__ double sa[1024];
  __shared__ long long sn[1024];
  double a = 0.0;
  long long c = 0;
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x) {
    a += absr[p];
    c += vis[p];
  }
  sa[threadIdx.x] = a;
  sn[threadIdx.x] = c;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      sa[threadIdx.x] += sa[threadIdx.x + s];
      sn[threadIdx.x] += sn[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sn[0] ? sa[0] / (double)sn[0] : 0.0;
    out[1] = (double)sn[0];
  }
}

__global__ void k_photo_scale(int64_t n, const double *__restrict__ graw,
                              const double *__restrict__ red, double *__restrict__ dz) {
  const double cnt = red[1];
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    dz[p] = cnt > 0.0 ? graw[p] / cnt : 0.0;
}

// --- reconstruct_multiview's depth heads on the device (optimize.py:272-358) --
// The photometric iterate only reads, per converged recorded pixel, the depth
// head of its best sample (top-K slot 0): HeadBundle.depth_image
// (shading.py:156-281) -> photometric_loss -> seed at that sample.  One dense
// row per pixel: a pixel without a converged sample has scale 0 (its point is
// the origin, its seed 0), so the reverse sweep needs no compaction.
__global__ void k_photo_heads(const dist_camera *__restrict__ cams, int W, int H, int64_t n, int K,
                              const uint8_t *__restrict__ status, const double *__restrict__ topk_d,
                              const double *__restrict__ topk_absf, double *__restrict__ pts,
                              double *__restrict__ scale) {
  const int64_t per = (int64_t)W * H;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(g / per);
    const int64_t pix = g - (int64_t)v * per;
    const int j = (int)(pix / W), i = (int)(pix - (int64_t)j * W);
    const bool ok = status[g] == DIST_CONVERGED && isfinite(topk_absf[g * K]);
    double dir[3], sc;
    pixel_ray(cams[v], i, j, 1, dir, &sc);
    const double d = topk_d[g * K];
    const double *o = cams[v].origin;
    // origin + d * dir, rounded as numpy does (shading.py HeadBundle points)
    for (int a = 0; a < 3; ++a) pts[g * 3 + a] = ok ? __dadd_rn(o[a], __dmul_rn(d, dir[a])) : 0.0;
    scale[g] = ok ? sc : 0.0;
  }
}

// z = (d + f) * scale at converged pixels, +inf elsewhere (depth_image)
__global__ void k_photo_depth(int64_t n, int K, const double *__restrict__ topk_d,
                              const double *__restrict__ f, const double *__restrict__ scale,
                              double *__restrict__ z) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x)
    z[g] = scale[g] > 0.0 ? __dmul_rn(__dadd_rn(topk_d[g * K], f[g]), scale[g])
                          : __longlong_as_double(0x7ff0000000000000ll);
}

// depth seed of the best sample: w_photo * dL/dz * scale (optimize.py:340-341)
__global__ void k_photo_seeds(int64_t n, const double *__restrict__ dz, const double *__restrict__ scale,
                              double w, double *__restrict__ seed) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x)
    seed[g] = scale[g] > 0.0 ? __dmul_rn(__dmul_rn(w, dz[g]), scale[g]) : 0.0;
}

}  // namespace dist

using namespace dist;

extern "C" {

size_t dist_photometric_workspace_size(int height, int width) {
  return (size_t)height * width * (2 * sizeof(double)) + 1024;
}

int dist_photometric(const dist_camera *cams_dev, int H, int W, int Hj, int Wj, const double *z_i,
                     const double *gray_i, const double *gray_j, const double *z_j, double thresh,
                     double *loss_dev, double *dz_dev, uint8_t *vis_dev, void *ws, size_t ws_bytes,
                     void *stream) {
  if (!cams_dev || !z_i || !gray_i || !gray_j || !z_j || !loss_dev || !dz_dev || !vis_dev)
    return fail(DIST_ERR_CONFIG, "null argument");
  if (H <= 0 || W <= 0 || Hj <= 0 || Wj <= 0) return fail(DIST_ERR_CONFIG, "empty image");
  const int64_t n = (int64_t)H * W;
  Carve cv{(char *)ws, 0, ws_bytes};
  double *absr = cv.take<double>(n);
  double *graw = cv.take<double>(n);
  if (!cv.ok) return fail(DIST_ERR_CONFIG, "photometric workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4096);
  k_photo_pixels<<<grid, 256, 0, st>>>(cams_dev, H, W, Hj, Wj, z_i, gray_i, gray_j, z_j, thresh, absr,
                                       graw, vis_dev);
  DIST_CHECK_LAUNCH("k_photo_pixels");
  k_photo_reduce<<<1, 1024, 0, st>>>(n, absr, vis_dev, loss_dev);
  DIST_CHECK_LAUNCH("k_photo_reduce");
  k_photo_scale<<<grid, 256, 0, st>>>(n, graw, loss_dev, dz_dev);
  DIST_CHECK_LAUNCH("k_photo_scale");
  return DIST_OK;
}

int dist_photo_heads(const dist_camera *cams_dev, int n_views, int width, int height, int k_samples,
                     const dist_ray_state *st, double *points_dev, double *scale_dev, void *stream) {
  if (!cams_dev || !st || !st->status || !st->topk_d || !st->topk_absf || !points_dev || !scale_dev)
    return fail(DIST_ERR_CONFIG, "null argument");
  if (n_views <= 0 || width <= 0 || height <= 0 || k_samples <= 0) return fail(DIST_ERR_CONFIG, "empty trace");
  const int64_t n = (int64_t)n_views * width * height;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4096);
  k_photo_heads<<<grid, 256, 0, (cudaStream_t)stream>>>(cams_dev, width, height, n, k_samples, st->status,
                                                        st->topk_d, st->topk_absf, points_dev, scale_dev);
  DIST_CHECK_LAUNCH("k_photo_heads");
  return DIST_OK;
}

int dist_photo_depth(int64_t n, int k_samples, const double *topk_d, const double *f_dev,
                     const double *scale_dev, double *z_dev, void *stream) {
  if (!topk_d || !f_dev || !scale_dev || !z_dev || k_samples <= 0) return fail(DIST_ERR_CONFIG, "null argument");
  if (n <= 0) return DIST_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4096);
  k_photo_depth<<<grid, 256, 0, (cudaStream_t)stream>>>(n, k_samples, topk_d, f_dev, scale_dev, z_dev);
  DIST_CHECK_LAUNCH("k_photo_depth");
  return DIST_OK;
}

int dist_photo_seeds(int64_t n, const double *dz_dev, const double *scale_dev, double w_photo,
                     double *seed_dev, void *stream) {
  if (!dz_dev || !scale_dev || !seed_dev) return fail(DIST_ERR_CONFIG, "null argument");
  if (n <= 0) return DIST_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), 4096);
  k_photo_seeds<<<grid, 256, 0, (cudaStream_t)stream>>>(n, dz_dev, scale_dev, w_photo, seed_dev);
  DIST_CHECK_LAUNCH("k_photo_seeds");
  return DIST_OK;
}

}  // extern "C"
