// kernels.cuh -- cross-translation-unit entry points inside libdist_b200.
#pragma once
#include <functional>

#include "common.cuh"

namespace dist {

int sm_count();
// c0 buffers hold [s1][np0] fp64 followed by the same values in fp32 (read by
// the tensor-core prologues, which would otherwise convert per row and column)
// and then [s1] per-shape max |c0| (bounds the fp16 row scale of layer 0)
inline size_t c0_doubles(int s1, int np0) {
  const size_t n = (size_t)s1 * np0;
  return n + (n + 1) / 2 + ((size_t)s1 + 1) / 2;
}
inline const float *c0_f32(const double *c0, int s1, int np0) {
  return reinterpret_cast<const float *>(c0 + (size_t)s1 * np0);
}
inline const float *c0_absmax(const double *c0, int s1, int np0) {
  return c0_f32(c0, s1, np0) + (size_t)s1 * np0;
}
int launch_code_bias(const DecView &dv, const double *codes, int S, double *c0, double *cskip,
                     cudaStream_t st);
int eval_points(const DecView &dv, const double *c0, const double *cskip, int S, const double *pts,
                const int32_t *shape, int64_t n, double *f, cudaStream_t st);
int vjp_points(const DecView &dv, const double *c0, const double *cskip, const double *pts,
               const int32_t *shape, int64_t n, const double *seed, int S, double *f,
               fx_t *part0, fx_t *parts, int *bad, double *gpts, int grid_cap, int *grid_out,
               cudaStream_t st);
// sums the per-CTA fixed-point partials (G slots) into colsum0/colsums
// (fixed point) and forms d/dz = W0z^T colsum (+ skip part); NaN when *bad
int reduce_code_grad(const DecView &dv, int S, int G, const fx_t *part0, const fx_t *parts,
                     const int *bad, fx_t *colsum0, fx_t *colsums, double *grad, cudaStream_t st);
int vjp_grid_cap(int prec);
size_t eval_ws(const DecView &dv, int64_t n, int S, bool vjp);

// tensor-core (tcgen05) split-precision decoder, tc_mlp.cu
int tc_eval_points(const DecView &dv, const double *c0, const double *cskip, int S, const double *pts,
                   const int32_t *shape, int64_t n, double *f, cudaStream_t st);
void tc_pack_sizes(const DecView &dv, const std::function<void(int, size_t, size_t)> &put);
void tc_pack_fill(const DecView &dv, const double *const *W, const double *const *b,
                  const int32_t *dims, const std::function<void *(int)> &wdst,
                  const std::function<float *(int)> &bdst);
bool tc_supported(const DecView &dv);
bool tc_shape_ok(const DecView &dv);
// measures DecView.tc_gain (the accumulator-bias gain of the head dot)
int tc_calibrate(DecView &dv);
bool tc_heads_supported(const DecView &dv);
}  // namespace dist
#include <cuda.h>
namespace dist {
int tc_make_map(const DecView &dv, int slot, CUtensorMap *map);
void tc_forget_maps(const DecView &dv);
template <class Gen>
int launch_tc_heads(const DecView &dv, const double *c0, const double *cs, const Gen &gen, int64_t n_bound,
                    int S, fx_t *part0, fx_t *parts, int *bad, int grid_cap, int *grid_out, cudaStream_t st,
                    double *gpts = nullptr);

struct LevelState;
struct ProbeGen;
struct ObjGen;
// backward-only head rows (f and ReLU masks from the march's mask record)
int launch_tc_heads_bwd(const DecView &dv, const double *c0, const double *cs, const ObjGen &gen,
                        int64_t n_bound, int S, fx_t *part0, fx_t *parts, int *bad, int grid_cap,
                        int *grid_out, cudaStream_t st);
int tc_eval_probes(const DecView &dv, const double *c0, const double *cs, int S, const ProbeGen &gen, int64_t n_bound,
                   cudaStream_t st);
int normals_pass(const DecView &dv, const double *c0, const double *cs, int S, const dist_camera *cams,
                 const LevelState &ls, const dist_trace_config *cfg, double *normals, double *gdotv,
                 int32_t *conv, int32_t *count, int32_t *bcount, double *f, cudaStream_t st,
                 int gdotv_unit = 0, double *rawnorm = nullptr);

// stable device-wide compaction of flags -> ascending indices (scan.cu)
size_t compact_ws_bytes(int64_t n);

}  // namespace dist
