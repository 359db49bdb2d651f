// tc_mlp.cu -- tcgen05/TMEM split-precision decoder (placeholder until the
// tensor-core kernel lands; BF16X3 decoders run the fp32 SIMT tiles).
#include "common.cuh"
#include "kernels.cuh"
#include "march.cuh"
#include "mlp_eval.cuh"

namespace dist {

bool tc_supported(const DecView &) { return false; }

int tc_eval_points(const DecView &dv, const double *c0, const double *cskip, const double *pts,
                   const int32_t *shape, int64_t n, double *f, cudaStream_t st) {
  ArrayGen g{pts, shape, nullptr, f, n};
  return launch_eval_gen<float>(dv, c0, cskip, g, n, st);
}

void tc_pack_sizes(const DecView &, const std::function<void(int, size_t, size_t)> &) {}
void tc_pack_fill(const DecView &, const double *const *, const double *const *, const int32_t *,
                  const std::function<void *(int)> &, const std::function<float *(int)> &) {}

int tc_run_steps(const DecView &, const double *, const double *, const dist_camera *,
                 const LevelState &, Ctl *, int32_t *, int32_t *, const MarchArgs &, int, int64_t *,
                 int64_t *, cudaStream_t) {
  return fail(DIST_ERR_CONFIG, "tcgen05 step kernel not built");
}

}  // namespace dist
