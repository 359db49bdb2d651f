// march.cuh -- ray state, the march update (tracer.py:132-193) and the
// step-slot bookkeeping shared by the SIMT and tcgen05 step kernels.
#pragma once
#include "common.cuh"

namespace dist {

struct LevelState {
  double *d, *b;
  uint8_t *status;
  int32_t *steps;
  double *tk_d, *tk_f, *tk_a;
  int lw, lh, level;
  int64_t n;  // V * lw * lh
  // Optional ReLU-mask record (full resolution, tensor-core march only;
  // include/dist.h dist_ray_state.relu_masks): tk_p[g][k] is the physical mask
  // slot of logical record k (bit 7: the masks were written by this ray's own
  // query), tk_p[g][K] the spare slot the current query's masks go to.
  uint32_t *masks;   // [n][K+1][nmask][16]
  uint8_t *tk_p;     // [n][K+1]
  int nmask;         // ReLU layers (hidden GEMMs + 1)
};

// words of one (ray, physical slot) mask record
__device__ __forceinline__ uint32_t *mask_record(const LevelState &ls, int K, int64_t g, int slot) {
  return ls.masks + ((size_t)g * (K + 1) + slot) * ls.nmask * 16;
}

struct Ctl {
  int32_t cnt[2];
  int32_t cur;
  uint32_t done;
  int32_t steps_done;
  int32_t pad[3];
};

struct MarchArgs {
  double alpha, eps;
  int K, max_steps, dynamic, V;
};

// Per-view step budget and live counts.  The reference traces one view at a
// time (tracer.py:236-252): each view has its own steps_done, leaves a coarse
// level as soon as it has no live ray, and records its own live_counts.  In a
// batched trace every step slot gates each ray by its view's budget, counts
// the queried rows per view, and the slot's last CTA advances exactly the
// views that stepped (vb_close).
struct ViewBudget {
  int32_t *steps;   // [V] steps the view has taken
  int32_t *cnt;     // [V] this slot's queried live rows of the view
  int64_t *live;    // [V][max_steps] out: the view's own live_counts
  int64_t per;      // rays per view at the current level
};

__device__ __forceinline__ int vb_view(const ViewBudget &vb, int64_t g) { return (int)(g / vb.per); }
__device__ __forceinline__ bool vb_active(const ViewBudget &vb, const MarchArgs &a, int64_t g) {
  return vb.steps[vb_view(vb, g)] < a.max_steps;
}
// the ray's view still steps after this slot (its survivors go to the next list)
__device__ __forceinline__ bool vb_continues(const ViewBudget &vb, const MarchArgs &a, int64_t g) {
  return vb.steps[vb_view(vb, g)] + 1 < a.max_steps;
}
// count one queried live row of view v (v < 0: none); every lane of the warp calls
__device__ __forceinline__ void vb_count(const ViewBudget &vb, int v) {
  const unsigned peers = __match_any_sync(0xffffffffu, v);
  const int lane = threadIdx.x & 31;
  if (v >= 0 && lane == __ffs(peers) - 1) atomicAdd(&vb.cnt[v], __popc(peers));
}

__device__ __forceinline__ void ray_of(const dist_camera *__restrict__ cams, const LevelState &ls,
                                       int64_t g, double dir[3], const dist_camera **cam) {
  const int64_t per = (int64_t)ls.lw * ls.lh;
  const int v = (int)(g / per);
  const int64_t pix = g - (int64_t)v * per;
  const int j = (int)(pix / ls.lw), i = (int)(pix - (int64_t)j * ls.lw);
  *cam = cams + v;
  pixel_ray(**cam, i, j, ls.level, dir, nullptr);
}

// warp-aggregated append of `value` when keep; every lane of the warp must call.
__device__ __forceinline__ void warp_append(bool keep, int32_t value, int32_t *list, int32_t *cnt) {
  const unsigned m = __ballot_sync(0xffffffffu, keep);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(cnt, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (keep) list[base + __popc(m & ((1u << lane) - 1u))] = value;
}

// --- the march update for one queried ray (tracer.py:170-192) -----------------
// One ray's state, wherever it lives: the level arrays in HBM (stride 1 for
// the top-K lists) or a CTA's shared-memory copy (k_march_resident: stride NT).
struct RayRef {
  double *d, *b;
  uint8_t *status;
  int32_t *steps;
  double *ta, *tf, *td;   // top-K |f|, f, d; entry k at [k * ks]
  int ks;
  uint8_t *tp;            // ReLU-mask record slots [K+1] or nullptr
};

__device__ __forceinline__ RayRef ray_ref(const LevelState &ls, int K, int64_t g) {
  return RayRef{ls.d + g, ls.b + g, ls.status + g, ls.steps + g, ls.tk_a + g * K, ls.tk_f + g * K,
                ls.tk_d + g * K, 1, ls.tk_p ? ls.tk_p + g * (K + 1) : nullptr};
}

// Returns true if the ray is still marching.  Arithmetic is kept
// uncontracted so that d' = d + alpha*f rounds exactly like numpy.
__device__ __forceinline__ bool march_update_at(const RayRef &r, const MarchArgs &a, const double dir[3],
                                                const double *o, double f, int *nan_count) {
  if (!isfinite(f)) {
    *r.status = DIST_EXHAUSTED;
    *r.b = __longlong_as_double(0x7ff8000000000000ll);
    *r.steps += 1;
    ++*nan_count;
    return false;
  }
  const double dk = *r.d;
  const double av = fabs(f);
  const int K = a.K, ks = r.ks;
  double *ta = r.ta, *tf = r.tf, *td = r.td;
  if (av < ta[(K - 1) * ks]) {  // strict: the earliest query wins ties (tracer.py:133-134)
    uint8_t *tp = r.tp;
    const uint8_t evicted = tp ? tp[K - 1] : 0;
    int pos = K - 1;
    while (pos > 0 && ta[(pos - 1) * ks] > av) {
      ta[pos * ks] = ta[(pos - 1) * ks];
      tf[pos * ks] = tf[(pos - 1) * ks];
      td[pos * ks] = td[(pos - 1) * ks];
      if (tp) tp[pos] = tp[pos - 1];
      --pos;
    }
    ta[pos * ks] = av;
    tf[pos * ks] = f;
    td[pos * ks] = dk;
    if (tp) {  // this query's masks sit in the spare slot; the evicted one's becomes spare
      tp[pos] = tp[K] | 0x80;
      tp[K] = evicted & 0x7f;
    }
  }
  *r.steps += 1;
  *r.b = f;
  const double dn = __dadd_rn(dk, __dmul_rn(a.alpha, f));
  *r.d = dn;
  if (av < a.eps) {
    *r.status = DIST_CONVERGED;
    return false;
  }
  double p[3];
  for (int i = 0; i < 3; ++i) p[i] = __dadd_rn(o[i], __dmul_rn(dn, dir[i]));
  const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(p[0], p[0]), __dmul_rn(p[1], p[1])), __dmul_rn(p[2], p[2]));
  const double vp = __dadd_rn(__dadd_rn(__dmul_rn(dir[0], p[0]), __dmul_rn(dir[1], p[1])), __dmul_rn(dir[2], p[2]));
  if (r2 > 1.0 && f > 0.0 && vp > 0.0) {
    *r.status = DIST_ESCAPED;
    return false;
  }
  return true;
}

__device__ __forceinline__ bool march_update(const LevelState &ls, const MarchArgs &a, int64_t g,
                                             const double dir[3], const double *o, double f,
                                             int *nan_count) {
  return march_update_at(ray_ref(ls, a.K, g), a, dir, o, f, nan_count);
}

// Last CTA of a step slot records every stepping view's query count
// (dynamic mask: its live rows; without it the whole view, tracer.py:158-163),
// advances those views' steps, and flips the live lists.  Every thread of the
// CTA calls it.
__device__ __forceinline__ void step_epilogue(Ctl *ctl, int cur, const ViewBudget &vb, const MarchArgs &a,
                                              int nan_block, int64_t *stats) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (nan_block) atomicAdd((unsigned long long *)&stats[1], (unsigned long long)nan_block);
    __threadfence();
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  unsigned long long q = 0;
  int smax = 0;
  for (int v = threadIdx.x; v < a.V; v += blockDim.x) {
    const int c = vb.cnt[v];
    if (!c) continue;
    const int s = vb.steps[v];
    const int64_t n = a.dynamic ? (int64_t)c : vb.per;
    vb.live[(int64_t)v * a.max_steps + s] = n;
    q += (unsigned long long)n;
    vb.steps[v] = s + 1;
    smax = max(smax, s + 1);
    vb.cnt[v] = 0;
  }
  if (q) atomicAdd((unsigned long long *)&stats[0], q);
  if (smax) atomicMax((unsigned long long *)&stats[2], (unsigned long long)smax);
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl->steps_done += 1;   // slots executed (all views)
    ctl->cnt[cur] = 0;
    ctl->cur = cur ^ 1;
    ctl->done = 0;
    __threadfence();
  }
}

// Buffers of the fluid tensor-core march (tc_mlp.cu MarchFluid): a third
// live list and [4 (max_steps + 2)] per-slot counters; null disables it.
struct FluidBufs {
  int32_t *list2;
  int32_t *ctr;
};

int tc_run_steps(const DecView &dv, const double *c0, const double *cskip, int S,
                 const dist_camera *cams, const LevelState &ls, Ctl *ctl, int32_t *l0, int32_t *l1,
                 const MarchArgs &a, int slots, const ViewBudget &vb, int64_t *stats, cudaStream_t st,
                 const FluidBufs &fb = FluidBufs{nullptr, nullptr});

// Normal probes of the converged rays (shading.py:73-94): row 6r + 2a (+1)
// is p +/- delta e_a of converged ray r, so consecutive rows form the
// (p+, p-) pairs of the (mid, diff) evaluation.
struct ProbeGen {
  const dist_camera *cams;
  LevelState ls;
  const int32_t *conv;   // converged ray ids
  const int32_t *cnt_ptr;  // device count
  double alpha, delta;
  double *f;
  __device__ int64_t count() const { return (int64_t)*cnt_ptr * 6; }
  __device__ bool point(int64_t i, double p[3], int &s) const {
    const int64_t r = i / 6;
    const int a = (int)(i - r * 6);
    const int64_t g = conv[r];
    double dir[3];
    const int64_t per = (int64_t)ls.lw * ls.lh;
    const int v = (int)(g / per);
    const int64_t pix = g - (int64_t)v * per;
    const int j = (int)(pix / ls.lw), ii = (int)(pix - (int64_t)j * ls.lw);
    pixel_ray(cams[v], ii, j, 1, dir, nullptr);
    const double ds = __dadd_rn(ls.d[g], __dmul_rn(1.0 - alpha, ls.b[g]));
    for (int q = 0; q < 3; ++q) p[q] = __dadd_rn(cams[v].origin[q], __dmul_rn(ds, dir[q]));
    // probe order (+x, -x, +y, -y, +z, -z): consecutive rows form the
    // (p + delta e_a, p - delta e_a) pairs of the (mid, diff) evaluation
    const int axis = a >> 1;
    p[axis] = __dadd_rn(p[axis], (a & 1) ? -delta : delta);
    s = cams[v].shape;
    return true;
  }
  __device__ double seed(int64_t, double) const { return 0.0; }
  __device__ void store(int64_t i, double v) const { f[i] = v; }
};

}  // namespace dist
