/*
 * dist.h -- C ABI of the B200-native DIST sphere-tracing hot path.
 *
 * One shared library (libdist_b200.so, sm_100a) exports these entry points.
 * They are the drop-in boundary for the reference package `sdftrace`
 * (/root/reference/pkg/src/sdftrace): every function below replaces one
 * reference interface, cited as file:line.  All pointers named *_dev are
 * device pointers owned by the caller (PyTorch allocates them); the library
 * never allocates per call.  Every call is stream-ordered on `stream` and does
 * not synchronise the host.  Return codes:
 *   DIST_OK            0
 *   DIST_ERR_CONFIG    2  -> ValueError            (bad shape / config)
 *   DIST_ERR_NUMERIC   3  -> FloatingPointError    (non-finite gradient)
 *   DIST_ERR_CUDA      4  -> RuntimeError          (CUDA / no device)
 * dist_last_error() returns a thread-local message for the last failure.
 * Handles are immutable after creation and safe to share across threads and
 * streams ("fields are immutable; eval is pure").
 */
#ifndef DIST_B200_H
#define DIST_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DIST_API __attribute__((visibility("default")))
#else
#define DIST_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DIST_OK 0
#define DIST_ERR_CONFIG 2
#define DIST_ERR_NUMERIC 3
#define DIST_ERR_CUDA 4

/* ray status codes, tracer.py:24 */
#define DIST_MARCHING 0
#define DIST_CONVERGED 1
#define DIST_ESCAPED 2
#define DIST_EXHAUSTED 3

/* arithmetic of the decoder evaluation */
#define DIST_PREC_FP64 0   /* SIMT fp64: the reference's own precision */
#define DIST_PREC_FP32 1   /* SIMT fp32 */
#define DIST_PREC_BF16X3 2 /* tcgen05 bf16 hi/lo 3-pass, fp32 accumulate in TMEM */
#define DIST_PREC_FP16X3 3 /* tcgen05 fp16 hi/lo 3-pass with power-of-2 row/layer scaling */

/* warning bits in stats[3] */
#define DIST_WARN_CAMERA_INSIDE 1   /* tracer.py:100-102 */

typedef struct dist_decoder dist_decoder;

/* Pinhole camera of one view: camera.py:25-61 (intrinsics) and 157-172
 * (pose).  R is the world-to-camera rotation (row-major), origin the camera
 * centre -R^T t.  `shape` selects the latent code (row of codes_dev). */
typedef struct dist_camera {
  double R[9];
  double origin[3];
  double fx, fy, cx, cy;
  int32_t width, height;
  int32_t shape;
  int32_t reserved;
} dist_camera;

/* TraceConfig, tracer.py:27-50 (validated by the library as in :41-50). */
typedef struct dist_trace_config {
  double alpha, epsilon, normal_delta;
  int32_t max_steps, k_samples, coarse_start_scale, split_interval;
  int32_t use_dynamic_mask;
  int32_t reserved;
} dist_trace_config;

/* Full-resolution SoA ray state, RayState of tracer.py:53-73, for V views of
 * H x W rays, ray index = (view * H + j) * W + i.  topk_* are [n][K].
 *
 * Optional (both NULL = off; honoured by the tensor-core precisions): the
 * ReLU masks of every recorded sample, written by the full-resolution march
 * as it queries, so that dist_objective runs only the backward sweep for
 * them instead of re-evaluating the taped forward at the frozen points
 * (shading.py:185-206 recomputes exactly the values the march computed).
 *   relu_masks  [n][K+1][n_layers-1][16] uint32 (512 bits per layer of 512,
 *               word order internal to the library)
 *   topk_slot   [n][K+1] uint8: physical mask slot of logical record k
 *               (bit 7 set when this ray's own query wrote it), slot K spare. */
typedef struct dist_ray_state {
  double *d, *b;
  uint8_t *status;
  int32_t *steps;
  double *topk_d, *topk_f, *topk_absf;
  uint32_t *relu_masks;
  uint8_t *topk_slot;
} dist_ray_state;

/* ---- library ---------------------------------------------------------- */
DIST_API const char *dist_last_error(void);
DIST_API int dist_device_info(int *sm_count, int *cc_major, int *cc_minor);
/* number of kernel launches the library enqueued since load (bench audit) */
DIST_API int64_t dist_launch_count(void);

/* Debug: per-phase timeline of the last k_tc_mlp / k_tc_heads launch, recorded
 * when DIST_TC_TIMELINE=1 (entries: mark id << 56 | %globaltimer ns of CTA 0's
 * first epilogue thread; scripts/tile_timeline.py). Copies up to n entries. */
DIST_API int dist_debug_mlp_timeline(unsigned long long *out, int n);
/* DIST_TC_TIMELINE=4: one row per CTA of the fluid march's slot grids,
 * {slot | block << 32, start ns, end ns, first rows ns | tiles << 48};
 * copies up to n (<= 16384) rows. */
DIST_API int dist_debug_fluid_timeline(unsigned long long *out, int n);
DIST_API int dist_debug_heads_timeline(unsigned long long *out, int n);

/* ---- decoder (NeuralField, fields.py:185-247) -------------------------- */
/* W[l] is the reference's row-major W[in,out] float64 (fields.py:195-196),
 * b[l] its bias; dims has n_layers+1 entries (dims[0] = latent_dim + 3 +
 * 0, dims[n_layers] = 1).  skip_layer >= 0 selects the DeepSDF layout where
 * layer `skip_layer` consumes concat(h, code, xyz);
 * -1 is the reference's plain stack.  The tensor-core precisions take
 * skip_layer <= n_layers - 3 (a hidden layer follows the skip layer) with
 * 512-wide hidden layers (the pre-skip layer may be narrower: it is
 * zero-padded to 512) and return DIST_ERR_CONFIG for any other shape.  final_linear selects the head: 0 = tanh,
 * 1 = linear (fields.py:200-201, 245-246), 2 = sigmoid (AttributeField,
 * fields.py:332-338).  Hidden activation is ReLU. */
DIST_API int dist_decoder_create(const double *const *W, const double *const *b, int n_layers,
                        const int32_t *dims, int latent_dim, int skip_layer,
                        int final_linear, int precision, dist_decoder **out);
DIST_API int dist_decoder_destroy(dist_decoder *dec);
DIST_API int dist_decoder_precision(const dist_decoder *dec);

/* Workspace needed by dist_eval / dist_eval_vjp for n points and S shapes. */
DIST_API size_t dist_eval_workspace_size(const dist_decoder *dec, int64_t n, int n_shapes);

/* NeuralField.evaluate (fields.py:233-247): f[i] = field(points[i], codes[shape[i]]).
 * shape_dev may be NULL (all rows use code 0); codes_dev may be NULL when
 * latent_dim == 0. */
DIST_API int dist_eval(const dist_decoder *dec, const double *codes_dev, int n_shapes,
              const double *points_dev, const int32_t *shape_dev, int64_t n,
              double *f_dev, void *ws, size_t ws_bytes, void *stream);

/* AttributeField.evaluate (fields.py:332-338): m <= 8 decoders that share
 * every layer but the last (the attribute field's channels, each a
 * single-output sigmoid-head decoder over the same hidden stack), evaluated
 * with the hidden stack of decs[0] computed once: out[i*m + c] = channel c at
 * points[i], bit-identical to dist_eval of decs[c].  SIMT precisions only;
 * the workspace is dist_eval_workspace_size(decs[0], n, n_shapes). */
DIST_API int dist_eval_channels(const dist_decoder *const *decs, int m, const double *codes_dev,
                                int n_shapes, const double *points_dev, const int32_t *shape_dev,
                                int64_t n, double *out_dev, void *ws, size_t ws_bytes, void *stream);

/* Taped evaluation + reverse sweep (fields.py:260-291 with
 * autodiff.py:220-255): f, d(sum seed*f)/d code [S,D] and d/d points [n,3]
 * (grad_points_dev may be NULL). */
DIST_API int dist_eval_vjp(const dist_decoder *dec, const double *codes_dev, int n_shapes,
                  const double *points_dev, const int32_t *shape_dev, int64_t n,
                  const double *seed_dev, double *f_dev, double *grad_codes_dev,
                  double *grad_points_dev, void *ws, size_t ws_bytes, void *stream);

/* ---- tracing (trace, tracer.py:221-252) --------------------------------- */
DIST_API size_t dist_trace_workspace_size(const dist_decoder *dec, const dist_trace_config *cfg,
                                 int n_views, int width, int height, int n_shapes);

/* Coarse-to-fine, dynamic-mask, aggressive sphere tracing of V views that
 * share one resolution.  Each view keeps the reference's own step budget and
 * level progression (tracer.py:236-252 traces one view at a time: a view
 * whose coarse level empties early moves on with its own steps_done).
 * Outputs: the final-level ray state, per-view per-step query counts
 * live_counts_dev[V][max_steps] (TraceResult.live_counts of view v: the
 * nonzero prefix of row v), and stats_dev[4] = {total_queries (all views),
 * nan_count, the largest per-view step count, warning bits}. */
DIST_API int dist_trace(const dist_decoder *dec, const double *codes_dev, int n_shapes,
               const dist_camera *cams_dev, int n_views, int width, int height,
               const dist_trace_config *cfg, const dist_ray_state *out,
               int64_t *live_counts_dev, int64_t *stats_dev, void *ws, size_t ws_bytes,
               void *stream);

/* ---- the plugin seam: a caller-evaluated field ------------------------------
 * The reference's trace accepts any duck-typed field with evaluate(points,
 * code) (tracer.py:165; analytic fields, test fakes such as NanField,
 * test_tracer.py:172-178).  dist_trace_external runs the same march -- init,
 * dynamic mask, top-K record, update, splits, audit counters -- on the device
 * and calls `field` once per step with the step's query points in host memory
 * (points_host [n][3], caller-allocated for V*W*H rows); the callback writes
 * f_host[n] and returns 0 (non-zero aborts with DIST_ERR_CONFIG).  The
 * library synchronises the stream once per step.  Non-finite values exhaust
 * their rays (tracer.py:170-176). */
typedef int (*dist_field_fn)(const double *points_host, int64_t n, double *f_host, void *user);
DIST_API size_t dist_trace_external_workspace_size(const dist_trace_config *cfg, int n_views,
                                                   int width, int height);
DIST_API int dist_trace_external(dist_field_fn field, void *user, const dist_camera *cams_dev,
                                 int n_views, int width, int height, const dist_trace_config *cfg,
                                 const dist_ray_state *out, int64_t *live_counts_dev,
                                 int64_t *stats_dev, double *points_host, double *f_host, void *ws,
                                 size_t ws_bytes, void *stream);

/* ---- maps (shading.py:48-113) ------------------------------------------ */
/* depth_map (+inf background), hard_mask, soft_silhouette for all V views,
 * images [V,H,W].  Any output pointer may be NULL. */
DIST_API int dist_maps(const dist_camera *cams_dev, int n_views, int width, int height,
              const dist_trace_config *cfg, const dist_ray_state *st, double *depth_dev,
              uint8_t *mask_dev, double *silhouette_dev, void *stream);

/* normal_map (shading.py:73-94): six-probe central differences at every
 * converged pixel, zero elsewhere; normals_dev [V,H,W,3]. */
DIST_API size_t dist_normals_workspace_size(const dist_decoder *dec, int n_views, int width,
                                   int height, int n_shapes);
DIST_API int dist_normals(const dist_decoder *dec, const double *codes_dev, int n_shapes,
                 const dist_camera *cams_dev, int n_views, int width, int height,
                 const dist_trace_config *cfg, const dist_ray_state *st, double *normals_dev,
                 void *ws, size_t ws_bytes, void *stream);

/* ---- one latent-optimisation iterate (completion_objective,
 *      optimize.py:102-138; HeadBundle shading.py:156-281; losses.py:54-117) */
typedef struct dist_objective_io {
  const double *obs_depth;       /* [V*H*W] observed camera z, +inf background; NULL = no depth term */
  const uint8_t *obs_depth_mask; /* [V*H*W] trusted pixels or NULL (Observation.mask, losses.py:38-42) */
  const double *obs_sil;         /* [V*H*W] binary silhouette target; NULL = no silhouette term */
  double w_depth, w_sil, w_latent; /* LossWeights, losses.py:45-51 */
  double *grad;                  /* out [S*D]: d total / d code (device) */
  double *view_terms;            /* out [V*6]: depth loss, silhouette loss, n_px, n_converged,
                                    normal loss, n_normal (valid normal pixels) */
  double *shape_terms;           /* out [S*2]: total objective, |z|^2 */
  int32_t grad_mode;             /* 0: the reference's frozen-sample surrogate (shading.py:9-11);
                                    1: implicit gradient -(df/dz)/(grad f . v) at converged pixels;
                                    2: the paper's literal -(df/dz)/(n . v), n the unit Eq. 3 normal */
  int32_t reserved;
  int32_t *counts_out;           /* optional out [2]: recorded rays, seeded head samples (device) */
  /* normal term (normal_loss, losses.py:94-111; seeds shading.py:259-269) */
  const double *obs_normal;      /* [V*H*W*3] observed unit normals; NULL = no normal term */
  const uint8_t *obs_normal_mask;/* [V*H*W] trusted pixels or NULL */
  double w_normal;               /* LossWeights.normal */
  /* Split iterate for views sharded over ranks as pixel tiles.
   * phase 0: the whole iterate.  phase 1: sample lists, probes and the
   * per-view counts only (view_terms[2], [3], [5]).  phase 2 (same workspace,
   * after phase 1): the rest, with view_norm[v*3 + {0,1,2}] = the whole
   * view's n_px, pixel count and n_normal replacing the tile's own (the
   * normalisers of losses.py:61-111), so every term is the tile's exact share
   * of its view's term. */
  int32_t phase;
  int32_t reserved2;
  const double *view_norm;       /* [V*3] (phase 2) or NULL */
  void *colsum_fixed;            /* optional out [S*w] (w = dist_decoder_colsum_width) 16-byte
                                    two's-complement integers: the layer-0 gradient column sums
                                    * 2^95 as [S][np0], then for a skip decoder the skip layer's
                                    as [S][nskip] (exact, so ranks can add them in any order);
                                    see dist_code_grad_fixed */
} dist_objective_io;

/* flags: bit 0 = a normal term will be requested (reserves its buffers) */
DIST_API size_t dist_objective_workspace_size(const dist_decoder *dec, int n_views, int width,
                                              int height, int k_samples, int n_shapes,
                                              int grad_mode, int flags);
/* After dist_trace: frozen-sample heads, loss seeds, the fused taped forward
 * -> seed -> reverse sweep per tile of samples, and the code gradient with the
 * latent regulariser added once per shape.  Views contribute their own
 * per-view-normalised depth term, as Sum_v completion_objective(view v). */
DIST_API int dist_objective(const dist_decoder *dec, const double *codes_dev, int n_shapes,
                            const dist_camera *cams_dev, int n_views, int width, int height,
                            const dist_trace_config *cfg, const dist_ray_state *st,
                            const dist_objective_io *io, void *ws, size_t ws_bytes, void *stream);

/* d/dz = W0[:D] colsum (+ W_skip[code rows] colsum_skip) + w_latent * 2 z from exact column sums (the element-
 * wise integer sum of every rank's dist_objective_io.colsum_fixed): the
 * reduction step of optimize.py:340-341 ("g += hg['code']", regulariser once)
 * with a result that is bit-identical for any number of ranks. */
DIST_API int dist_code_grad_fixed(const dist_decoder *dec, int n_shapes, const void *colsum_fixed,
                                  const double *codes_dev, double w_latent, double *grad_dev,
                                  void *stream);
/* fixed-point column sums per shape: padded width of layer 0 (+ that of the
 * skip layer for a skip decoder) -- colsum_fixed holds S times this many */
DIST_API int dist_decoder_colsum_width(const dist_decoder *dec);
/* The tensor-core decoders' calibrated head gain (measured at creation):
 * tcgen05 accumulates fp32 in TMEM with truncation toward zero, which shrinks
 * every hidden pre-activation by a nearly constant relative amount; the
 * 512 -> 1 head dot is scaled by g = sum(d64^2)/sum(dtc d64) fitted on 65,536
 * fixed quasi-random points of the unit ball (code 0).  gain2[0]: the
 * march/eval pack; gain2[1]: the fp16 probe pack.  1.0 for fp64/fp32. */
DIST_API int dist_decoder_head_gain(const dist_decoder *dec, double *gain2);

/* ---- photometric consistency (losses.py:128-222) ------- */
/* cams_dev[0] = view i, cams_dev[1] = view j.  Images are row-major doubles
 * (depth: +inf background).  Outputs: loss_dev[2] = {mean |r| over visible
 * pixels, n visible}, dz_dev[H*W] = d loss / d z_i, vis_dev[H*W] = visibility
 * of i's pixels in j (visibility_mask, losses.py:159-183). */
DIST_API size_t dist_photometric_workspace_size(int height, int width);
DIST_API int dist_photometric(const dist_camera *cams_dev, int height, int width, int height_j,
                              int width_j, const double *z_i, const double *gray_i,
                              const double *gray_j, const double *z_j, double thresh,
                              double *loss_dev, double *dz_dev, uint8_t *vis_dev, void *ws,
                              size_t ws_bytes, void *stream);

/* reconstruct_multiview on the device (optimize.py:272-358): the depth head
 * of each converged recorded pixel's best sample (top-K slot 0;
 * HeadBundle.depth_image, shading.py:156-281), one dense row per pixel of the
 * V traced views (ray id (v*H + j)*W + i).
 * dist_photo_heads: points_dev[g] = origin + topk_d[g][0] * dir, scale_dev[g]
 *   = the ray's distance -> camera-z factor; a pixel without a converged
 *   sample gets scale 0 and the origin as its point.
 * dist_photo_depth: z_dev[g] = (topk_d[g][0] + f[g]) * scale, +inf where
 *   scale is 0 (f = dist_eval at points_dev).
 * dist_photo_seeds: seed_dev[g] = w_photo * dz[g] * scale (0 where scale is 0),
 *   the depth seeds of optimize.py:340-341 for dist_eval_vjp. */
DIST_API int dist_photo_heads(const dist_camera *cams_dev, int n_views, int width, int height,
                              int k_samples, const dist_ray_state *st, double *points_dev,
                              double *scale_dev, void *stream);
DIST_API int dist_photo_depth(int64_t n, int k_samples, const double *topk_d, const double *f_dev,
                              const double *scale_dev, double *z_dev, void *stream);
DIST_API int dist_photo_seeds(int64_t n, const double *dz_dev, const double *scale_dev,
                              double w_photo, double *seed_dev, void *stream);

/* pose_objective on the device (optimize.py:185-233): one
 * traced view, dense rows K per pixel (row g*K + k is a head sample when pixel
 * g is recorded and top-K slot k is finite; other rows: origin, seed 0).
 * dist_pose_samples: points_dev[row] = origin + topk_d * dir.
 * dist_pose_seeds: loss_dev[0] = depth_loss (losses.py:54-75; obs_depth [H*W]
 *   camera z with obs_valid [H*W] = finite & trusted, or NULL for no depth
 *   term), loss_dev[1] = silhouette_loss (losses.py:78-91; soft_sil = the
 *   dist_maps silhouette, obs_sil the target, both NULL for no term),
 *   loss_dev[2] = n_px; seed_dev[row] = w_depth * depth seed + w_sil *
 *   silhouette seed (best sample), f_dev = dist_eval at points_dev.
 * dist_pose_grad: grad_dev[6] = (dL/d omega, dL/d t) by camera.py:255-278 from
 *   the rows' point gradients (dist_eval_vjp) and the unrecorded pixels'
 *   silhouette term at the ray's closest point to the origin
 *   (optimize.py:220-229); mats_dev = R, dR/d omega_0..2 (row-major 3x3) and t
 *   (39 doubles, camera.rotation_derivatives). */
DIST_API int dist_pose_samples(const dist_camera *cam_dev, int width, int height, int k_samples,
                               const dist_ray_state *st, double *points_dev, void *stream);
DIST_API int dist_pose_seeds(const dist_camera *cam_dev, int width, int height, int k_samples,
                             const dist_ray_state *st, const double *f_dev, const double *obs_depth,
                             const uint8_t *obs_valid, const double *soft_sil, const double *obs_sil,
                             double w_depth, double w_sil, double *loss_dev, double *seed_dev,
                             void *stream);
DIST_API int dist_pose_grad(const dist_camera *cam_dev, int width, int height, int k_samples,
                            const dist_ray_state *st, const double *point_grads_dev,
                            const double *soft_sil, const double *obs_sil, double w_sil,
                            const double *mats_dev, double *grad_dev, void *stream);

/* ---- Adam (AdamState/adam_step, optimize.py:35-63) ------------------------ */
typedef struct dist_adam_config {
  double lr, beta1, beta2, eps;
} dist_adam_config;
/* One bias-corrected step per shape; a shape whose gradient has a non-finite
 * entry is skipped and counted.  With shape_terms/best_*: records the loss
 * history hist[iter*S + s] and keeps the best-loss iterate (optimize.py:170-176)
 * before updating.  iter_dev (optional device int32): the iteration index is
 * read from it instead of `iter` and incremented after the step, so a
 * captured iterate (CUDA graph) replays correctly. */
DIST_API int dist_adam_step(int n_shapes, int dim, double *params_dev, const double *grad_dev,
                            double *m_dev, double *v_dev, int32_t *t_dev, int32_t *skipped_dev,
                            const double *shape_terms_dev, double *best_loss_dev,
                            double *best_params_dev, int32_t *best_iter_dev, int iter,
                            double *hist_dev, const dist_adam_config *cfg, int32_t *iter_dev,
                            void *stream);

#ifdef __cplusplus
}
#endif
#endif
