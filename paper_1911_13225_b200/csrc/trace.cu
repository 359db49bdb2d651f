// trace.cu -- device-resident sphere tracing (tracer.py:88-252) and the maps
// of shading.py:48-113.
//
// The march runs as a fixed schedule of launches that the host enqueues up
// front (no host synchronisation per step): init, split_interval step slots
// per coarse level, a split, and max_steps slots at full resolution.  Each
// slot is one persistent kernel that reads the live count and the global step
// budget from a device controller and exits immediately when the reference
// loop would have broken (tracer.py:242-245: budget spent or nothing live), so
// the executed steps equal the reference's exactly.  Inside a slot every CTA
// takes TM-row tiles of the current live list, evaluates the decoder, applies
// the march update (NaN -> EXHAUSTED, top-K record, d += alpha f, converge /
// escape tests) in the tile epilogue, and appends surviving rays to the next
// live list with warp-aggregated atomics; the last CTA to finish records the
// step's query count (TraceResult.live_counts) and flips the lists.  The
// SIMT precisions run all slots of a level as ONE cooperative launch instead
// (k_march_coop: the same step body, a grid barrier between steps).
#include <cooperative_groups.h>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "mlp_eval.cuh"
#include "mlp_small.cuh"
#include "scan.cuh"
#include "march.cuh"

namespace dist {

namespace cg = cooperative_groups;

// --- init (tracer.py:88-119) ----------------------------------------------
__global__ void k_init(const dist_camera *__restrict__ cams, LevelState ls, int K,
                       int32_t *__restrict__ list, Ctl *ctl, int64_t *stats) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ls.n; base += stride) {
    const int64_t g = base + threadIdx.x;
    bool live = false;
    if (g < ls.n) {
      double v[3];
      const dist_camera *c;
      ray_of(cams, ls, g, v, &c);
      const double *o = c->origin;
      const double c2 = __dadd_rn(__dadd_rn(__dmul_rn(o[0], o[0]), __dmul_rn(o[1], o[1])),
                                  __dmul_rn(o[2], o[2]));
      double d0 = 0.0;
      uint8_t stt = DIST_MARCHING;
      if (c2 <= 1.0) {
        if (g == 0 || (g % ((int64_t)ls.lw * ls.lh)) == 0) atomicOr((unsigned long long *)&stats[3], (unsigned long long)DIST_WARN_CAMERA_INSIDE);
      } else {
        const double m = __dadd_rn(__dadd_rn(__dmul_rn(v[0], o[0]), __dmul_rn(v[1], o[1])),
                                   __dmul_rn(v[2], o[2]));
        const double disc = __dsub_rn(__dmul_rn(m, m), __dsub_rn(c2, 1.0));
        if (disc >= 0.0 && m < 0.0) d0 = __dsub_rn(-m, sqrt(disc));
        else stt = DIST_ESCAPED;
      }
      ls.d[g] = d0;
      ls.b[g] = __longlong_as_double(0x7ff8000000000000ll);
      ls.status[g] = stt;
      ls.steps[g] = 0;
      for (int k = 0; k < K; ++k) {
        ls.tk_d[g * K + k] = 0.0;
        ls.tk_f[g * K + k] = 0.0;
        ls.tk_a[g * K + k] = __longlong_as_double(0x7ff0000000000000ll);
      }
      if (ls.tk_p)
        for (int k = 0; k <= K; ++k) ls.tk_p[g * (K + 1) + k] = (uint8_t)k;
      live = stt == DIST_MARCHING;
    }
    warp_append(live, (int32_t)g, list, &ctl->cnt[0]);
  }
}

// --- 4-way split (tracer.py:196-218) ---------------------------------------
__global__ void k_split(LevelState par, LevelState ch, int K, int32_t *__restrict__ list, Ctl *ctl,
                        const int32_t *__restrict__ vsteps, int max_steps) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t per_c = (int64_t)ch.lw * ch.lh, per_p = (int64_t)par.lw * par.lh;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ch.n; base += stride) {
    const int64_t g = base + threadIdx.x;
    bool live = false;
    if (g < ch.n) {
      const int64_t v = g / per_c, pix = g - v * per_c;
      const int j = (int)(pix / ch.lw), i = (int)(pix - (int64_t)j * ch.lw);
      const int64_t p = v * per_p + (int64_t)(j / 2) * par.lw + (i / 2);
      uint8_t s = par.status[p];
      if (s == DIST_CONVERGED) s = DIST_MARCHING;
      ch.status[g] = s;
      ch.d[g] = par.d[p];
      ch.b[g] = par.b[p];
      ch.steps[g] = par.steps[p];
      for (int k = 0; k < K; ++k) {
        ch.tk_d[g * K + k] = par.tk_d[p * K + k];
        ch.tk_f[g * K + k] = par.tk_f[p * K + k];
        ch.tk_a[g * K + k] = par.tk_a[p * K + k];
      }
      // inherited records carry no masks of this ray (own bit clear)
      if (ch.tk_p)
        for (int k = 0; k <= K; ++k) ch.tk_p[g * (K + 1) + k] = (uint8_t)k;
      // a view whose budget is spent marches no more (tracer.py:243)
      live = s == DIST_MARCHING && vsteps[v] < max_steps;
    }
    warp_append(live, (int32_t)g, list, &ctl->cnt[0]);
  }
}

// The same split, one thread per PARENT: the parent's state is read once and
// written to its 2 x 2 children with paired stores (children 2i, 2i+1 of a row
// are adjacent, so every child array gets 2-element vector stores; a warp
// writes whole 32 B sectors of each array).  Used when the child arrays are
// aligned for those stores (run_trace checks) and K <= kSplitMaxK.
constexpr int kSplitMaxK = 8;
__global__ void k_split_quad(LevelState par, LevelState ch, int K, int32_t *__restrict__ list, Ctl *ctl,
                             const int32_t *__restrict__ vsteps, int max_steps) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t per_c = (int64_t)ch.lw * ch.lh, per_p = (int64_t)par.lw * par.lh;
  const bool tkp4 = ch.tk_p && K == 3;   // one 8-byte store per child row
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < par.n; base += stride) {
    const int64_t p = base + threadIdx.x;
    bool live = false;
    int64_t g0 = 0;
    if (p < par.n) {
      const int64_t v = p / per_p, pix = p - v * per_p;
      const int j = (int)(pix / par.lw), i = (int)(pix - (int64_t)j * par.lw);
      g0 = v * per_c + (int64_t)(2 * j) * ch.lw + 2 * i;
      uint8_t s = par.status[p];
      if (s == DIST_CONVERGED) s = DIST_MARCHING;
      const double d = par.d[p], b = par.b[p];
      const int32_t stp = par.steps[p];
      double pd[kSplitMaxK], pf[kSplitMaxK], pa[kSplitMaxK];
      for (int k = 0; k < K; ++k) {
        pd[k] = par.tk_d[p * K + k];
        pf[k] = par.tk_f[p * K + k];
        pa[k] = par.tk_a[p * K + k];
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int64_t g = g0 + (int64_t)r * ch.lw;
        *reinterpret_cast<uchar2 *>(ch.status + g) = make_uchar2(s, s);
        *reinterpret_cast<double2 *>(ch.d + g) = make_double2(d, d);
        *reinterpret_cast<double2 *>(ch.b + g) = make_double2(b, b);
        *reinterpret_cast<int2 *>(ch.steps + g) = make_int2(stp, stp);
        // [child 2i: k = 0..K-1][child 2i+1: k = 0..K-1] = element e -> record e % K
        double2 *od = reinterpret_cast<double2 *>(ch.tk_d + g * K);
        double2 *of = reinterpret_cast<double2 *>(ch.tk_f + g * K);
        double2 *oa = reinterpret_cast<double2 *>(ch.tk_a + g * K);
        for (int e = 0; e < K; ++e) {
          const int k0 = (2 * e) % K, k1 = (2 * e + 1) % K;
          od[e] = make_double2(pd[k0], pd[k1]);
          of[e] = make_double2(pf[k0], pf[k1]);
          oa[e] = make_double2(pa[k0], pa[k1]);
        }
        // inherited records carry no masks of this ray (own bit clear)
        if (tkp4) {
          *reinterpret_cast<uint2 *>(ch.tk_p + g * 4) = make_uint2(0x03020100u, 0x03020100u);
        } else if (ch.tk_p) {
          for (int c = 0; c < 2; ++c)
            for (int k = 0; k <= K; ++k) ch.tk_p[(g + c) * (K + 1) + k] = (uint8_t)k;
        }
      }
      live = s == DIST_MARCHING && vsteps[v] < max_steps;
    }
    // the four children join the live list together (its order is free: every
    // row of a tile is evaluated independently)
    const unsigned m = __ballot_sync(0xffffffffu, live);
    if (m) {
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(m) - 1;
      int lb = 0;
      if (lane == leader) lb = atomicAdd(&ctl->cnt[0], 4 * __popc(m));
      lb = __shfl_sync(0xffffffffu, lb, leader);
      if (live) {
        int32_t *o = list + lb + 4 * __popc(m & ((1u << lane) - 1u));
        o[0] = (int32_t)g0;
        o[1] = (int32_t)(g0 + 1);
        o[2] = (int32_t)(g0 + ch.lw);
        o[3] = (int32_t)(g0 + ch.lw + 1);
      }
    }
  }
}

static bool split_quad_ok(const LevelState &par, const LevelState &ch, int K) {
  auto al = [](const void *q, uintptr_t a) { return q == nullptr || ((uintptr_t)q & (a - 1)) == 0; };
  return K <= kSplitMaxK && ch.lw == 2 * par.lw && ch.lh == 2 * par.lh && al(ch.status, 2) &&
         al(ch.d, 16) && al(ch.b, 16) && al(ch.steps, 8) && al(ch.tk_d, 16) && al(ch.tk_f, 16) &&
         al(ch.tk_a, 16) && al(ch.tk_p, 8);
}

__global__ void k_finalize(LevelState ls) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ls.n;
       g += (int64_t)gridDim.x * blockDim.x)
    if (ls.status[g] == DIST_MARCHING) ls.status[g] = DIST_EXHAUSTED;
}

// --- one step slot, SIMT decoder --------------------------------------------
// Returns false (block-uniform) when the live list is empty: the slot is a
// no-op and so is every later slot of the level.
template <typename T>
__device__ __forceinline__ bool simt_step(char *smem, const DecView &dv, const double *__restrict__ c0,
                                          const double *__restrict__ cskip,
                                          const dist_camera *__restrict__ cams, const LevelState &ls,
                                          Ctl *ctl, int32_t *list0, int32_t *list1, const MarchArgs &a,
                                          const ViewBudget &vb, int64_t *stats) {
  using Tile = SimtTile<T>;
  Tile tile(smem);
  __shared__ int s_cur, s_cnt, s_go, s_nan;
  if (threadIdx.x == 0) {
    s_cur = *(volatile int *)&ctl->cur;
    s_cnt = *(volatile int *)&ctl->cnt[s_cur];
    s_go = s_cnt > 0;   // per-view budgets gate the rays (ViewBudget)
    s_nan = 0;
  }
  __syncthreads();
  if (!s_go) return false;
  const int cur = s_cur;
  const int32_t *in = cur ? list1 : list0;
  int32_t *out = cur ? list0 : list1;
  int32_t *out_cnt = &ctl->cnt[cur ^ 1];
  const int64_t rows = a.dynamic ? (int64_t)s_cnt : ls.n;
  const int64_t ntiles = ceil_div(rows, Tile::TM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t g = -1;
    double dir[3] = {0, 0, 0};
    const dist_camera *cam = cams;
    if (threadIdx.x < Tile::TM) {
      const int64_t idx = t * Tile::TM + threadIdx.x;
      double p[3] = {0, 0, 0};
      int s = -1;
      if (idx < rows) {
        g = a.dynamic ? in[idx] : idx;
        ray_of(cams, ls, g, dir, &cam);
        const double dg = ls.d[g];
        for (int i = 0; i < 3; ++i) p[i] = __dadd_rn(cam->origin[i], __dmul_rn(dg, dir[i]));
        s = cam->shape;
      }
      tile.shape[threadIdx.x] = s;
      for (int i = 0; i < 3; ++i) tile.pts[threadIdx.x * 3 + i] = p[i];
    }
    __syncthreads();
    tile.forward(dv, c0, cskip, false);
    if (warp == 0) {
      bool keep = false;
      int v = -1;
      if (threadIdx.x < Tile::TM && g >= 0 && ls.status[g] == DIST_MARCHING && vb_active(vb, a, g)) {
        int nn = 0;
        v = vb_view(vb, g);
        keep = march_update(ls, a, g, dir, cam->origin, tile.f[threadIdx.x], &nn) && vb_continues(vb, a, g);
        if (nn) atomicAdd(&s_nan, nn);
      }
      vb_count(vb, v);
      warp_append(keep, (int32_t)g, out, out_cnt);
    }
    (void)lane;
    __syncthreads();
  }
  step_epilogue(ctl, cur, vb, a, s_nan, stats);
  return true;
}

template <typename T>
__global__ void __launch_bounds__(SimtTile<T>::NT)
    k_step(DecView dv, const double *__restrict__ c0, const double *__restrict__ cskip,
           const dist_camera *__restrict__ cams, LevelState ls, Ctl *ctl, int32_t *list0,
           int32_t *list1, MarchArgs a, ViewBudget vb, int64_t *stats) {
  extern __shared__ __align__(16) char smem[];
  simt_step<T>(smem, dv, c0, cskip, cams, ls, ctl, list0, list1, a, vb, stats);
}

// All `slots` steps of a level in one cooperative launch (every CTA
// co-resident): a grid barrier after each step's epilogue publishes the
// flipped live list.  The same per-step code as k_step, without a launch per
// slot -- what bounds small workloads (C1: ~100 slots of a few thousand rays).
template <typename T>
__global__ void __launch_bounds__(SimtTile<T>::NT)
    k_march_coop(DecView dv, const double *__restrict__ c0, const double *__restrict__ cskip,
                 const dist_camera *__restrict__ cams, LevelState ls, Ctl *ctl, int32_t *list0,
                 int32_t *list1, MarchArgs a, ViewBudget vb, int64_t *stats, int slots) {
  extern __shared__ __align__(16) char smem[];
  cg::grid_group grid = cg::this_grid();
  for (int s = 0; s < slots; ++s) {
    if (!simt_step<T>(smem, dv, c0, cskip, cams, ls, ctl, list0, list1, a, vb, stats)) break;
    grid.sync();
  }
}

// All slots of a level for a NARROW decoder (mlp_small.cuh): one ray per
// thread, the decoder staged in shared memory once, one cooperative launch
// with a grid barrier after each step.  Same march update, compaction and
// step bookkeeping as k_step.
template <typename T>
__global__ void __launch_bounds__(kSmallNT)
    k_march_small(DecView dv, const double *__restrict__ c0, const double *__restrict__ cskip,
                  const dist_camera *__restrict__ cams, LevelState ls, Ctl *ctl, int32_t *list0,
                  int32_t *list1, MarchArgs a, ViewBudget vb, int64_t *stats, int slots) {
  extern __shared__ __align__(16) char smem[];
  cg::grid_group grid = cg::this_grid();
  SmallNet<T> net;
  net.stage(dv, smem);
  __syncthreads();
  __shared__ int s_cur, s_cnt, s_nan;
  for (int sl = 0; sl < slots; ++sl) {
    if (threadIdx.x == 0) {
      s_cur = *(volatile int *)&ctl->cur;
      s_cnt = *(volatile int *)&ctl->cnt[s_cur];
      s_nan = 0;
    }
    __syncthreads();
    if (s_cnt <= 0) break;   // grid-uniform: every CTA read the same controller
    const int cur = s_cur;
    const int32_t *in = cur ? list1 : list0;
    int32_t *out = cur ? list0 : list1;
    int32_t *out_cnt = &ctl->cnt[cur ^ 1];
    const int64_t rows = a.dynamic ? (int64_t)s_cnt : ls.n;
    for (int64_t base = (int64_t)blockIdx.x * kSmallNT; base < rows; base += (int64_t)gridDim.x * kSmallNT) {
      const int64_t idx = base + threadIdx.x;
      bool keep = false;
      int v = -1;
      int64_t g = -1;
      if (idx < rows) {
        g = a.dynamic ? in[idx] : idx;
        if (ls.status[g] == DIST_MARCHING && vb_active(vb, a, g)) {
          double dir[3], p[3];
          const dist_camera *cam;
          ray_of(cams, ls, g, dir, &cam);
          const double dg = ls.d[g];
          for (int i = 0; i < 3; ++i) p[i] = __dadd_rn(cam->origin[i], __dmul_rn(dg, dir[i]));
          const double f = net.eval(dv, c0, cskip, p, cam->shape);
          int nn = 0;
          v = vb_view(vb, g);
          keep = march_update(ls, a, g, dir, cam->origin, f, &nn) && vb_continues(vb, a, g);
          if (nn) atomicAdd(&s_nan, nn);
        }
      }
      vb_count(vb, v);
      warp_append(keep, (int32_t)g, out, out_cnt);
    }
    step_epilogue(ctl, cur, vb, a, s_nan, stats);
    grid.sync();
  }
}

// Narrow decoder, level small enough for every ray to have a home thread
// (<= kResidentR rays per thread over a co-resident grid): the level's ray
// state is copied into shared memory at the start, each thread marches its
// own rays for all slots (no live list: a ray is live while it is MARCHING and
// its view has budget), and the state is written back once at the end.
//
// One grid barrier per step and no last-CTA hand-off: the step's per-view
// query counts and its survivor count go to one of three rotating counter
// rows (rcnt[3][V+1]); after the barrier every CTA reads the row and advances
// its own shared copy of the per-view step counters identically, CTA 0
// records live_counts and clears the row two steps ahead (read by everyone
// before the previous barrier, written again only after the next).  The
// bookkeeping is step_epilogue's (march.cuh), so the executed steps, the
// per-view live_counts and the audit counters equal k_step's.
constexpr int kResidentR = 4;
constexpr int kResidentMaxViews = 1024;
constexpr size_t kResidentCodeBytes = 48 * 1024;   // c0/cskip rows staged up to this size

struct ResidentLayout {
  int R, S, wb;          // rays per thread, shapes, register width bucket (64: shared activations)
  int code_in_smem;      // c0 / cskip rows staged in shared memory
  size_t off_vsteps, off_code, off_state, bytes;
  // bytes per resident ray: d, b, top-K (3K), dir, origin (f64); steps, shape, view (i32); status
  __host__ __device__ static size_t per_ray(int K) { return 8 * (2 + 3 * (size_t)K + 6) + 12 + 1; }
};

template <typename T, int WB>
__global__ void __launch_bounds__(kSmallNT)
    k_march_resident(DecView dv, const double *__restrict__ c0, const double *__restrict__ cskip,
                     const dist_camera *__restrict__ cams, LevelState ls, Ctl *ctl, MarchArgs a,
                     ViewBudget vb, int64_t *stats, int slots, ResidentLayout rl, int32_t *rcnt) {
  extern __shared__ __align__(16) char smem[];
  constexpr int NT = kSmallNT;
  cg::grid_group grid = cg::this_grid();
  SmallNet<T> net;
  RegNet<T, WB < 64 ? WB : 16> rnet;
  if constexpr (WB < 64) rnet.stage(dv, smem);
  else net.stage(dv, smem);
  const int K = a.K, R = rl.R, t = threadIdx.x, V = a.V;
  // staged code rows: [S][cw] of c0 then [S][cw] of cskip (zero-padded to WB
  // for the register path, the true widths otherwise)
  const int n0 = dv.nr[0], ns = dv.skip > 0 ? dv.nr[dv.skip] : 0;
  const int cw0 = WB < 64 ? WB : n0, cws = WB < 64 ? (ns ? WB : 0) : ns;
  // shared ray state, [field][R * NT] (slot i = r * NT + t)
  const int M = R * NT;
  double *sd = reinterpret_cast<double *>(smem + rl.off_state);
  double *sb = sd + M;
  double *sta = sb + M, *stf = sta + (size_t)K * M, *std_ = stf + (size_t)K * M;
  double *sdir = std_ + (size_t)K * M, *sorg = sdir + 3 * M;
  int32_t *ssteps = reinterpret_cast<int32_t *>(sorg + 3 * M);
  int32_t *sshape = ssteps + M, *sview = sshape + M;
  uint8_t *sstat = reinterpret_cast<uint8_t *>(sview + M);
  int32_t *vsteps = reinterpret_cast<int32_t *>(smem + rl.off_vsteps);   // [V] this CTA's copy
  double *scode = reinterpret_cast<double *>(smem + rl.off_code);       // [S][n0] then [S][ns]
  if (rl.code_in_smem) {   // the blob's rows are zero-padded to np >= 64 >= cw
    for (int i = t; i < rl.S * cw0; i += NT) scode[i] = c0[(size_t)(i / cw0) * dv.np[0] + i % cw0];
    for (int i = t; i < rl.S * cws; i += NT)
      scode[rl.S * cw0 + i] = cskip[(size_t)(i / cws) * dv.np[dv.skip] + i % cws];
  }
  const int64_t g0 = (int64_t)blockIdx.x * M;
  for (int i = t; i < M; i += NT) {
    const int64_t g = g0 + i;
    if (g < ls.n) {
      sd[i] = ls.d[g];
      sb[i] = ls.b[g];
      ssteps[i] = ls.steps[g];
      sstat[i] = ls.status[g];
      for (int k = 0; k < K; ++k) {
        sta[k * M + i] = ls.tk_a[g * K + k];
        stf[k * M + i] = ls.tk_f[g * K + k];
        std_[k * M + i] = ls.tk_d[g * K + k];
      }
      double dir[3];
      const dist_camera *cam;
      ray_of(cams, ls, g, dir, &cam);   // fixed for the level: once, not per step
      for (int c = 0; c < 3; ++c) {
        sdir[c * M + i] = dir[c];
        sorg[c * M + i] = cam->origin[c];
      }
      sshape[i] = cam->shape;
      sview[i] = vb_view(vb, g);
    } else {
      sstat[i] = DIST_CONVERGED;   // no ray: never live
    }
  }
  for (int v = t; v < V; v += NT) vsteps[v] = vb.steps[v];
  const int W = V + 1;   // counter row: [V] queried rows per view, [V] survivors
  if (blockIdx.x == 0)
    for (int i = t; i < 3 * W; i += NT) rcnt[i] = 0;
  __shared__ int s_live, s_keep, s_nan, s_smax;
  __shared__ unsigned long long s_q;
  if (t == 0) {
    s_live = ctl->cnt[ctl->cur];   // the level's initial live list (k_init / k_split)
    s_q = 0;
    s_smax = 0;
  }
  grid.sync();
  int executed = 0;
  for (int sl = 0; sl < slots; ++sl) {
    if (s_live <= 0) break;   // grid-uniform: every CTA read the same row
    int32_t *row = rcnt + (sl % 3) * W;
    if (t == 0) {
      s_keep = 0;
      s_nan = 0;
    }
    __syncthreads();
    int kept = 0;
    for (int r = 0; r < R; ++r) {
      const int i = r * NT + t;
      int v = -1;
      if (sstat[i] == DIST_MARCHING) {
        const int vv = sview[i];
        if (vsteps[vv] < a.max_steps) {
          const double dir[3] = {sdir[i], sdir[M + i], sdir[2 * M + i]};
          const double org[3] = {sorg[i], sorg[M + i], sorg[2 * M + i]};
          const double dg = sd[i];
          double p[3];
          for (int c = 0; c < 3; ++c) p[c] = __dadd_rn(org[c], __dmul_rn(dg, dir[c]));
          const int sh = sshape[i];
          double f;
          if constexpr (WB < 64) {
            const double *cz = rl.code_in_smem ? scode + (size_t)sh * cw0 : c0 + (size_t)sh * dv.np[0];
            const double *cs = rl.code_in_smem ? scode + (size_t)rl.S * cw0 + (size_t)sh * cws
                                               : (ns ? cskip + (size_t)sh * dv.np[dv.skip] : nullptr);
            f = rnet.eval(dv, cz, cs, p);
          } else {
            f = net.eval(dv, c0, cskip, p, sh);
          }
          int nn = 0;
          v = vv;
          const RayRef ref{sd + i, sb + i, sstat + i, ssteps + i, sta + i, stf + i, std_ + i, M, nullptr};
          kept += (march_update_at(ref, a, dir, org, f, &nn) && vsteps[vv] + 1 < a.max_steps) ? 1 : 0;
          if (nn) atomicAdd(&s_nan, nn);
        }
      }
      const unsigned peers = __match_any_sync(0xffffffffu, v);
      if (v >= 0 && (t & 31) == __ffs(peers) - 1) atomicAdd(&row[v], __popc(peers));
    }
    kept = __reduce_add_sync(0xffffffffu, kept);
    if ((t & 31) == 0 && kept) atomicAdd(&s_keep, kept);
    __syncthreads();
    if (t == 0) {
      if (s_keep) atomicAdd(&row[V], s_keep);
      if (s_nan) atomicAdd((unsigned long long *)&stats[1], (unsigned long long)s_nan);
    }
    grid.sync();
    // every CTA: advance its view step copies from the row
    for (int v = t; v < V; v += NT) {
      const int c = *(volatile int32_t *)&row[v];
      if (!c) continue;
      const int sv = vsteps[v];
      if (blockIdx.x == 0) {
        const int64_t n = a.dynamic ? (int64_t)c : vb.per;
        vb.live[(int64_t)v * a.max_steps + sv] = n;
        atomicAdd(&s_q, (unsigned long long)n);
        atomicMax(&s_smax, sv + 1);
      }
      vsteps[v] = sv + 1;
    }
    if (t == 0) s_live = *(volatile int32_t *)&row[V];
    if (blockIdx.x == 0) {   // the row two steps ahead: read by all before this barrier
      int32_t *nxt = rcnt + ((sl + 2) % 3) * W;
      for (int i = t; i < W; i += NT) nxt[i] = 0;
    }
    ++executed;
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    for (int v = t; v < V; v += NT) vb.steps[v] = vsteps[v];
    if (t == 0) {
      ctl->steps_done += executed;
      if (s_q) atomicAdd((unsigned long long *)&stats[0], s_q);
      if (s_smax) atomicMax((unsigned long long *)&stats[2], (unsigned long long)s_smax);
    }
  }
  for (int i = t; i < M; i += NT) {
    const int64_t g = g0 + i;
    if (g < ls.n) {
      ls.d[g] = sd[i];
      ls.b[g] = sb[i];
      ls.steps[g] = ssteps[i];
      ls.status[g] = sstat[i];
      for (int k = 0; k < K; ++k) {
        ls.tk_a[g * K + k] = sta[k * M + i];
        ls.tk_f[g * K + k] = stf[k * M + i];
        ls.tk_d[g * K + k] = std_[k * M + i];
      }
    }
  }
}

template <typename T, int WB>
static int launch_resident(const DecView &dv, const double *c0, const double *cskip,
                           const dist_camera *cams, const LevelState &ls, Ctl *ctl, const MarchArgs &a,
                           int slots, const ViewBudget &vb, int64_t *stats, int32_t *rcnt, int S,
                           cudaStream_t st, bool *launched) {
  *launched = false;
  const int K = a.K;
  const size_t wbytes = WB < 64 ? RegNet<T, WB < 64 ? WB : 16>::weight_bytes(dv) : SmallNet<T>::weight_bytes(dv);
  const size_t act = WB < 64 ? 0 : 2 * sizeof(T) * kSmallWidth * kSmallNT;
  const int n0 = dv.nr[0], ns = dv.skip > 0 ? dv.nr[dv.skip] : 0;
  const size_t code = sizeof(double) * (size_t)S * (WB < 64 ? WB + (ns ? WB : 0) : n0 + ns);
  ResidentLayout rl{};
  rl.S = S;
  rl.wb = WB;
  rl.off_vsteps = round_up((int64_t)(wbytes + act), 16);
  rl.off_code = round_up((int64_t)(rl.off_vsteps + sizeof(int32_t) * a.V), 16);
  rl.code_in_smem = code <= kResidentCodeBytes;
  rl.off_state = round_up((int64_t)(rl.off_code + (rl.code_in_smem ? code : 0)), 16);
  for (int R = 1; R <= kResidentR; ++R) {
    const size_t bytes = rl.off_state + (size_t)R * kSmallNT * ResidentLayout::per_ray(K);
    if (bytes > 200 * 1024) break;
    const void *rf = (const void *)k_march_resident<T, WB>;
    cudaError_t e = cudaFuncSetAttribute(rf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(march_resident)");
    int cap_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cap_sm, rf, kSmallNT, bytes);
    const int64_t grid = ceil_div(ls.n, (int64_t)R * kSmallNT);
    if (cap_sm < 1 || grid > (int64_t)cap_sm * sm_count()) continue;
    rl.R = R;
    rl.bytes = bytes;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3(kSmallNT);
    lc.dynamicSmemBytes = bytes;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelEx(&lc, k_march_resident<T, WB>, dv, c0, cskip, cams, ls, ctl, a, vb, stats, slots,
                           rl, rcnt);
    if (e != cudaSuccess) return cuda_fail(e, "k_march_resident");
    DIST_CHECK_LAUNCH("k_march_resident");
    *launched = true;
    return DIST_OK;
  }
  return DIST_OK;
}

// --- maps (shading.py:48-61, 97-113) ------------------------------------------
__global__ void k_maps(const dist_camera *__restrict__ cams, LevelState ls, double alpha, double eps,
                       int K, double *depth, uint8_t *mask, double *sil) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ls.n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t s = ls.status[g];
    const bool conv = s == DIST_CONVERGED;
    double dir[3], scale;
    const int64_t per = (int64_t)ls.lw * ls.lh;
    const int v = (int)(g / per);
    const int64_t pix = g - (int64_t)v * per;
    const int j = (int)(pix / ls.lw), i = (int)(pix - (int64_t)j * ls.lw);
    pixel_ray(cams[v], i, j, 1, dir, &scale);
    if (depth) {
      const double ds = __dadd_rn(ls.d[g], __dmul_rn(1.0 - alpha, ls.b[g]));
      depth[g] = conv ? __dmul_rn(ds, scale) : __longlong_as_double(0x7ff0000000000000ll);
    }
    if (mask) mask[g] = conv ? 1 : 0;
    if (sil) {
      const double a0 = ls.tk_a[g * K];
      if (isfinite(a0)) {
        sil[g] = a0 - eps;
      } else {
        const double *o = cams[v].origin;
        const double m = dir[0] * o[0] + dir[1] * o[1] + dir[2] * o[2];
        const double c2 = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
        sil[g] = sqrt(fmax(c2 - m * m, 0.0)) - 1.0;
      }
    }
  }
}

static int grid_for(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), (int64_t)sm_count() * 16));
}

// --- normals (shading.py:73-94) ----------------------------------------------

__global__ void k_normals_assemble(const dist_camera *__restrict__ cams, LevelState ls,
                                   const int32_t *__restrict__ conv,
                                   const int32_t *__restrict__ count, const double *__restrict__ f,
                                   double delta, int pair, double *__restrict__ normals,
                                   double *__restrict__ gdotv, int gdotv_unit,
                                   double *__restrict__ rawnorm) {
  const int64_t n = *count;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = conv[r];
    double raw[3];
    for (int a = 0; a < 3; ++a)  // row 2a+1 of the pair holds f(p + d e_a) - f(p - d e_a)
      raw[a] = pair ? f[r * 6 + 2 * a + 1] / (2.0 * delta)
                    : (f[r * 6 + 2 * a] - f[r * 6 + 2 * a + 1]) / (2.0 * delta);
    const double nrm = sqrt(raw[0] * raw[0] + raw[1] * raw[1] + raw[2] * raw[2]);
    if (rawnorm) rawnorm[g] = nrm;
    if (normals)
      for (int a = 0; a < 3; ++a) normals[g * 3 + a] = nrm > 0.0 ? raw[a] / nrm : 0.0;
    if (gdotv) {  // grad f . v (raw Eq. 3 vector, or n . v with the unit normal) for the implicit gradient
      const int64_t per = (int64_t)ls.lw * ls.lh;
      const int v = (int)(g / per);
      const int64_t pix = g - (int64_t)v * per;
      const int j = (int)(pix / ls.lw), i = (int)(pix - (int64_t)j * ls.lw);
      double dir[3];
      pixel_ray(cams[v], i, j, 1, dir, nullptr);
      const double dot = raw[0] * dir[0] + raw[1] * dir[1] + raw[2] * dir[2];
      gdotv[g] = !gdotv_unit ? dot : (nrm > 0.0 ? dot / nrm : 0.0);
    }
  }
}

// Normal probes at every converged ray (shading.py:73-94): compaction, probe
// evaluation ((mid, diff) pairs except in fp64), assembly of unit normals
// and/or grad f . v.
int normals_pass(const DecView &dv, const double *c0, const double *cs, int S, const dist_camera *cams,
                 const LevelState &ls, const dist_trace_config *cfg, double *normals, double *gdotv,
                 int32_t *conv, int32_t *count, int32_t *bcount, double *f, cudaStream_t st,
                 int gdotv_unit, double *rawnorm) {
  const int64_t n = ls.n;
  const uint8_t *status = ls.status;
  int rc = compact([status] __device__(int64_t i) { return status[i] == DIST_CONVERGED; }, n, conv,
                   count, bcount, st);
  if (rc) return rc;
  ProbeGen gen{cams, ls, conv, count, cfg->alpha, cfg->normal_delta, f};
  // fp64: plain probes (the reference's own arithmetic); every other mode
  // evaluates the probe pairs as (mid, diff) in fp32 so that the 1/(2 delta)
  // amplification does not act on rounding error (SURVEY 0 finding 3).
  // On tensor-core decoders the pairs run through k_tc_mlp's pair mode.
  const int pair = dv.prec == DIST_PREC_FP64 ? 0 : 1;
  if (!pair) rc = launch_eval_gen<double>(dv, c0, cs, gen, n * 6, st);
  else if (tc_supported(dv)) rc = tc_eval_probes(dv, c0, cs, S, gen, n * 6, st);
  else rc = launch_eval_gen<float, ProbeGen, true>(dv, c0, cs, gen, n * 6, st);
  if (rc) return rc;
  k_normals_assemble<<<grid_for(n, 256), 256, 0, st>>>(cams, ls, conv, count, f, cfg->normal_delta,
                                                       pair, normals, gdotv, gdotv_unit, rawnorm);
  DIST_CHECK_LAUNCH("k_normals_assemble");
  return DIST_OK;
}

// --- the plugin seam: a field evaluated by the caller (tracer.py:165) ----------
// One step of the march for a field the library cannot evaluate (a duck-typed
// Python field, an analytic SDF): the device gathers the query points of the
// step, the caller's callback evaluates them, the device applies the update.
__global__ void k_ext_points(const dist_camera *__restrict__ cams, LevelState ls, const Ctl *ctl,
                             const int32_t *__restrict__ list0, const int32_t *__restrict__ list1,
                             int dynamic, double *__restrict__ pts) {
  const int cur = ctl->cur;
  const int64_t rows = dynamic ? (int64_t)ctl->cnt[cur] : ls.n;
  const int32_t *in = cur ? list1 : list0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = dynamic ? in[i] : i;
    double dir[3];
    const dist_camera *cam;
    ray_of(cams, ls, g, dir, &cam);
    const double dg = ls.d[g];
    for (int a = 0; a < 3; ++a) pts[i * 3 + a] = __dadd_rn(cam->origin[a], __dmul_rn(dg, dir[a]));
  }
}

// With the dynamic mask off the whole grid is queried and dead rays' values
// discarded (tracer.py:158-168), exactly as march_step does.
__global__ void k_ext_apply(const dist_camera *__restrict__ cams, LevelState ls, Ctl *ctl,
                            int32_t *list0, int32_t *list1, MarchArgs a, const double *__restrict__ f,
                            ViewBudget vb, int64_t *stats) {
  __shared__ int s_nan;
  const int cur = ctl->cur;
  const int64_t rows = a.dynamic ? (int64_t)ctl->cnt[cur] : ls.n;
  const int32_t *in = cur ? list1 : list0;
  int32_t *out = cur ? list0 : list1;
  if (threadIdx.x == 0) s_nan = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < rows; base += stride) {
    const int64_t i = base + threadIdx.x;
    bool keep = false;
    int64_t g = -1;
    int v = -1;
    if (i < rows) {
      g = a.dynamic ? in[i] : i;
      if (ls.status[g] == DIST_MARCHING && vb_active(vb, a, g)) {
        double dir[3];
        const dist_camera *cam;
        ray_of(cams, ls, g, dir, &cam);
        int nn = 0;
        v = vb_view(vb, g);
        keep = march_update(ls, a, g, dir, cam->origin, f[i], &nn) && vb_continues(vb, a, g);
        if (nn) atomicAdd(&s_nan, nn);
      }
    }
    vb_count(vb, v);
    warp_append(keep, (int32_t)g, out, &ctl->cnt[cur ^ 1]);
  }
  __syncthreads();   // every warp's NaN count is in s_nan before thread 0 reads it
  step_epilogue(ctl, cur, vb, a, s_nan, stats);
}

// --- host side --------------------------------------------------------------
static int check_cfg(const dist_trace_config *c, int width, int height, int V) {
  if (!c) return fail(DIST_ERR_CONFIG, "null config");
  if (!(c->alpha > 0.0 && c->alpha < 2.0)) return fail(DIST_ERR_CONFIG, "alpha must be in (0, 2)");
  if (!(c->epsilon > 0.0)) return fail(DIST_ERR_CONFIG, "epsilon must be positive");
  if (c->max_steps < 1) return fail(DIST_ERR_CONFIG, "max_steps must be at least 1");
  if (c->k_samples < 1 || c->k_samples > 16) return fail(DIST_ERR_CONFIG, "k_samples must be in [1, 16]");
  if (c->coarse_start_scale != 1 && c->coarse_start_scale != 2 && c->coarse_start_scale != 4)
    return fail(DIST_ERR_CONFIG, "coarse_start_scale must be 1, 2, or 4");
  if (c->split_interval < 1) return fail(DIST_ERR_CONFIG, "split_interval must be at least 1");
  if (width <= 0 || height <= 0 || V <= 0) return fail(DIST_ERR_CONFIG, "resolution must be positive");
  if (width % c->coarse_start_scale || height % c->coarse_start_scale)
    return fail(DIST_ERR_CONFIG, "resolution not divisible by coarse_start_scale");
  if ((int64_t)V * width * height >= (int64_t)1 << 31)
    return fail(DIST_ERR_CONFIG, "too many rays for one trace call");
  return DIST_OK;
}

struct TraceLayout {
  double *c0, *cskip;
  LevelState lv[3];
  int n_levels;
  int32_t *list0, *list1, *bcount;
  int32_t *vsteps, *vcnt;   // ViewBudget: per-view steps and this slot's counts
  int32_t *rcnt;            // k_march_resident: three rotating [V+1] counter rows
  FluidBufs fluid;          // the fluid tensor-core march (tc_mlp.cu), or nulls
  Ctl *ctl;
  size_t bytes;
};

static TraceLayout layout(const DecView &dv, const dist_trace_config *cfg, int V, int W, int H,
                          int S, char *ws, size_t cap, const dist_ray_state *out) {
  TraceLayout L{};
  Carve cv{ws, 0, cap};
  const int s1 = std::max(S, 1);
  L.c0 = cv.take<double>(c0_doubles(s1, dv.np[0]));
  L.cskip = cv.take<double>(c0_doubles(s1, std::max(dv.nskip, 1)));
  int levels[3], nl = 0;
  for (int s = cfg->coarse_start_scale; s >= 1; s /= 2) levels[nl++] = s;
  L.n_levels = nl;
  const int K = cfg->k_samples;
  for (int li = 0; li < nl; ++li) {
    LevelState &ls = L.lv[li];
    ls.level = levels[li];
    ls.lw = W / ls.level;
    ls.lh = H / ls.level;
    ls.n = (int64_t)V * ls.lw * ls.lh;
    if (ls.level == 1) {
      if (out) {
        ls.d = out->d; ls.b = out->b; ls.status = out->status; ls.steps = out->steps;
        ls.tk_d = out->topk_d; ls.tk_f = out->topk_f; ls.tk_a = out->topk_absf;
        if (out->relu_masks && out->topk_slot && tc_heads_supported(dv)) {
          ls.masks = out->relu_masks;
          ls.tk_p = out->topk_slot;
          ls.nmask = dv.n_layers - 1;
        }
      }
    } else {
      ls.d = cv.take<double>(ls.n);
      ls.b = cv.take<double>(ls.n);
      ls.status = cv.take<uint8_t>(ls.n);
      ls.steps = cv.take<int32_t>(ls.n);
      ls.tk_d = cv.take<double>(ls.n * K);
      ls.tk_f = cv.take<double>(ls.n * K);
      ls.tk_a = cv.take<double>(ls.n * K);
    }
  }
  const int64_t nmax = (int64_t)V * W * H;
  L.list0 = cv.take<int32_t>(nmax);
  L.list1 = cv.take<int32_t>(nmax);
  if (tc_supported(dv) && cfg->use_dynamic_mask) {   // the fluid march's third list and counters
    L.fluid.list2 = cv.take<int32_t>(nmax);
    L.fluid.ctr = cv.take<int32_t>(4 * ((size_t)cfg->max_steps + 2));
  }
  L.bcount = cv.take<int32_t>(ceil_div(nmax * 6, kScanBlock) + 1);
  L.vsteps = cv.take<int32_t>(2 * (size_t)V);
  L.vcnt = L.vsteps ? L.vsteps + V : nullptr;
  L.rcnt = cv.take<int32_t>(3 * ((size_t)V + 1));
  L.ctl = cv.take<Ctl>(1);
  L.bytes = cv.off + 256;
  return L;
}

template <typename T>
static int run_steps(const DecView &dv, const double *c0, const double *cskip,
                     const dist_camera *cams, const LevelState &ls, Ctl *ctl, int32_t *l0,
                     int32_t *l1, const MarchArgs &a, int slots, const ViewBudget &vb, int64_t *stats,
                     int32_t *rcnt, int S, cudaStream_t st) {
  using Tile = SimtTile<T>;
  const size_t small = SmallNet<T>::smem_bytes(dv);
  if (small && !ls.tk_p && rcnt && a.V <= kResidentMaxViews) {
    // every ray resident in shared memory for the whole level?
    bool done = false;
    const int wb = SmallNet<T>::width_bucket(dv);
    int rc = wb == 16 ? launch_resident<T, 16>(dv, c0, cskip, cams, ls, ctl, a, slots, vb, stats, rcnt, S, st, &done)
           : wb == 32 ? launch_resident<T, 32>(dv, c0, cskip, cams, ls, ctl, a, slots, vb, stats, rcnt, S, st, &done)
                      : launch_resident<T, 64>(dv, c0, cskip, cams, ls, ctl, a, slots, vb, stats, rcnt, S, st, &done);
    if (rc || done) return rc;
  }
  if (small && small <= 200 * 1024) {
    // narrow decoder: one ray per thread, the whole level in one cooperative launch
    const void *sf = (const void *)k_march_small<T>;
    cudaError_t e = cudaFuncSetAttribute(sf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(march_small)");
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sf, kSmallNT, small);
    if (per >= 1) {
      const int64_t need = ceil_div(ls.n, kSmallNT);
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)per * sm_count()));
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(kSmallNT);
      lc.dynamicSmemBytes = small;
      lc.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      e = cudaLaunchKernelEx(&lc, k_march_small<T>, dv, c0, cskip, cams, ls, ctl, l0, l1, a, vb, stats, slots);
      if (e != cudaSuccess) return cuda_fail(e, "k_march_small");
      DIST_CHECK_LAUNCH("k_march_small");
      return DIST_OK;
    }
  }
  const void *fn = (const void *)k_step<T>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Tile::fwd_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(step)");
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, Tile::NT, Tile::fwd_bytes);
  const int64_t tiles = ceil_div(ls.n, Tile::TM);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)std::max(per_sm, 1) * sm_count()));
  if (slots > 1 && per_sm >= 1) {
    // one cooperative launch for the level (grid <= co-resident CTAs)
    const void *cf = (const void *)k_march_coop<T>;
    e = cudaFuncSetAttribute(cf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Tile::fwd_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(march_coop)");
    int coop_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&coop_sm, cf, Tile::NT, Tile::fwd_bytes);
    const int cgrid = std::min(grid, std::max(coop_sm, 1) * sm_count());
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(cgrid);
    lc.blockDim = dim3(Tile::NT);
    lc.dynamicSmemBytes = Tile::fwd_bytes;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelEx(&lc, k_march_coop<T>, dv, c0, cskip, cams, ls, ctl, l0, l1, a, vb, stats, slots);
    if (e != cudaSuccess) return cuda_fail(e, "k_march_coop");
    DIST_CHECK_LAUNCH("k_march_coop");
    return DIST_OK;
  }
  for (int s = 0; s < slots; ++s) {
    k_step<T><<<grid, Tile::NT, Tile::fwd_bytes, st>>>(dv, c0, cskip, cams, ls, ctl, l0, l1, a, vb,
                                                      stats);
    DIST_CHECK_LAUNCH("k_step");
  }
  return DIST_OK;
}


}  // namespace dist

using namespace dist;

extern "C" {

size_t dist_trace_workspace_size(const dist_decoder *dec, const dist_trace_config *cfg, int V,
                                 int W, int H, int S) {
  if (!dec || !cfg || cfg->coarse_start_scale < 1) return 0;
  return layout(dec->view, cfg, V, W, H, S, nullptr, ~size_t(0), nullptr).bytes;
}

int dist_trace(const dist_decoder *dec, const double *codes, int S, const dist_camera *cams,
               int V, int W, int H, const dist_trace_config *cfg, const dist_ray_state *out,
               int64_t *live, int64_t *stats, void *ws, size_t ws_bytes, void *stream) {
  if (!dec || !out || !cams || !live || !stats) return fail(DIST_ERR_CONFIG, "null argument");
  int rc = check_cfg(cfg, W, H, V);
  if (rc) return rc;
  const DecView &dv = dec->view;
  if (dv.latent_dim > 0 && (!codes || S < 1)) return fail(DIST_ERR_CONFIG, "field expects a latent code");
  cudaStream_t st = (cudaStream_t)stream;
  TraceLayout L = layout(dv, cfg, V, W, H, S, (char *)ws, ws_bytes, out);
  if (L.bytes > ws_bytes) return fail(DIST_ERR_CONFIG, "trace workspace too small");
  cudaError_t e = cudaMemsetAsync(L.ctl, 0, sizeof(Ctl), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(stats, 0, 4 * sizeof(int64_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(live, 0, (size_t)V * cfg->max_steps * sizeof(int64_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(L.vsteps, 0, 2 * sizeof(int32_t) * V, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(trace)");
  rc = launch_code_bias(dv, dv.latent_dim > 0 ? codes : nullptr, std::max(S, 1), L.c0, L.cskip, st);
  if (rc) return rc;
  MarchArgs a{cfg->alpha, cfg->epsilon, cfg->k_samples, cfg->max_steps,
              cfg->use_dynamic_mask ? 1 : 0, V};
  const int K = cfg->k_samples;
  k_init<<<grid_for(L.lv[0].n, 256), 256, 0, st>>>(cams, L.lv[0], K, L.list0, L.ctl, stats);
  DIST_CHECK_LAUNCH("k_init");
  for (int li = 0; li < L.n_levels; ++li) {
    const LevelState &ls = L.lv[li];
    if (li > 0) {
      // fresh lists for the new level; steps_done (offset 16) persists
      e = cudaMemsetAsync(L.ctl, 0, 16, st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(ctl)");
      if (split_quad_ok(L.lv[li - 1], ls, K)) {
        k_split_quad<<<grid_for(L.lv[li - 1].n, 256), 256, 0, st>>>(L.lv[li - 1], ls, K, L.list0, L.ctl,
                                                                     L.vsteps, cfg->max_steps);
        DIST_CHECK_LAUNCH("k_split_quad");
      } else {
        k_split<<<grid_for(ls.n, 256), 256, 0, st>>>(L.lv[li - 1], ls, K, L.list0, L.ctl, L.vsteps,
                                                     cfg->max_steps);
        DIST_CHECK_LAUNCH("k_split");
      }
    }
    const int slots = std::min(ls.level > 1 ? cfg->split_interval : cfg->max_steps, cfg->max_steps);
    const ViewBudget vb{L.vsteps, L.vcnt, live, (int64_t)ls.lw * ls.lh};
    if (dv.prec == DIST_PREC_FP64)
      rc = run_steps<double>(dv, L.c0, L.cskip, cams, ls, L.ctl, L.list0, L.list1, a, slots, vb, stats, L.rcnt, std::max(S, 1), st);
    else if (tc_supported(dv))
      rc = tc_run_steps(dv, L.c0, L.cskip, std::max(S, 1), cams, ls, L.ctl, L.list0, L.list1, a, slots, vb, stats, st,
                        L.fluid);
    else
      rc = run_steps<float>(dv, L.c0, L.cskip, cams, ls, L.ctl, L.list0, L.list1, a, slots, vb, stats, L.rcnt, std::max(S, 1), st);
    if (rc) return rc;
  }
  const LevelState &fin = L.lv[L.n_levels - 1];
  k_finalize<<<grid_for(fin.n, 256), 256, 0, st>>>(fin);
  DIST_CHECK_LAUNCH("k_finalize");
  return DIST_OK;
}

size_t dist_trace_external_workspace_size(const dist_trace_config *cfg, int V, int W, int H) {
  if (!cfg || cfg->coarse_start_scale < 1) return 0;
  DecView dv{};
  dv.np[0] = 64;
  const int64_t n = (int64_t)V * W * H;
  Carve cv{nullptr, 0, ~size_t(0)};
  cv.off = layout(dv, cfg, V, W, H, 1, nullptr, ~size_t(0), nullptr).bytes;
  cv.take<double>(n * 3);
  cv.take<double>(n);
  return cv.off + 256;
}

int dist_trace_external(dist_field_fn field, void *user, const dist_camera *cams, int V, int W, int H,
                        const dist_trace_config *cfg, const dist_ray_state *out, int64_t *live,
                        int64_t *stats, double *points_host, double *f_host, void *ws, size_t ws_bytes,
                        void *stream) {
  if (!field || !out || !cams || !live || !stats || !points_host || !f_host)
    return fail(DIST_ERR_CONFIG, "null argument");
  int rc = check_cfg(cfg, W, H, V);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  DecView dv{};
  dv.np[0] = 64;
  dist_ray_state o = *out;
  o.relu_masks = nullptr;
  o.topk_slot = nullptr;
  TraceLayout L = layout(dv, cfg, V, W, H, 1, (char *)ws, ws_bytes, &o);
  Carve cv{(char *)ws, L.bytes - 256, ws_bytes};
  const int64_t nmax = (int64_t)V * W * H;
  double *pts = cv.take<double>(nmax * 3);
  double *fd = cv.take<double>(nmax);
  if (!cv.ok || L.bytes > ws_bytes) return fail(DIST_ERR_CONFIG, "trace workspace too small");
  cudaError_t e = cudaMemsetAsync(L.ctl, 0, sizeof(Ctl), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(stats, 0, 4 * sizeof(int64_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(live, 0, (size_t)V * cfg->max_steps * sizeof(int64_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(L.vsteps, 0, 2 * sizeof(int32_t) * V, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(trace)");
  MarchArgs a{cfg->alpha, cfg->epsilon, cfg->k_samples, cfg->max_steps, cfg->use_dynamic_mask ? 1 : 0, V};
  const int K = cfg->k_samples;
  k_init<<<grid_for(L.lv[0].n, 256), 256, 0, st>>>(cams, L.lv[0], K, L.list0, L.ctl, stats);
  DIST_CHECK_LAUNCH("k_init");
  for (int li = 0; li < L.n_levels; ++li) {
    const LevelState &ls = L.lv[li];
    if (li > 0) {
      e = cudaMemsetAsync(L.ctl, 0, 16, st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(ctl)");
      k_split<<<grid_for(ls.n, 256), 256, 0, st>>>(L.lv[li - 1], ls, K, L.list0, L.ctl, L.vsteps,
                                                   cfg->max_steps);
      DIST_CHECK_LAUNCH("k_split");
    }
    const int budget = ls.level > 1 ? cfg->split_interval : cfg->max_steps;
    const ViewBudget vb{L.vsteps, L.vcnt, live, (int64_t)ls.lw * ls.lh};
    for (int step = 0; step < budget; ++step) {
      // the reference loop's own test, on the host (tracer.py:242-245); the
      // per-view budgets are applied on the device (ViewBudget)
      Ctl c;
      e = cudaMemcpyAsync(&c, L.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return cuda_fail(e, "controller read");
      if (c.cnt[c.cur] <= 0) break;
      const int64_t rows = a.dynamic ? (int64_t)c.cnt[c.cur] : ls.n;
      k_ext_points<<<grid_for(rows, 256), 256, 0, st>>>(cams, ls, L.ctl, L.list0, L.list1, a.dynamic, pts);
      DIST_CHECK_LAUNCH("k_ext_points");
      e = cudaMemcpyAsync(points_host, pts, sizeof(double) * 3 * rows, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return cuda_fail(e, "points to host");
      if (field(points_host, rows, f_host, user) != 0)
        return fail(DIST_ERR_CONFIG, "field callback failed");
      e = cudaMemcpyAsync(fd, f_host, sizeof(double) * rows, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "values to device");
      k_ext_apply<<<grid_for(rows, 256), 256, 0, st>>>(cams, ls, L.ctl, L.list0, L.list1, a, fd, vb, stats);
      DIST_CHECK_LAUNCH("k_ext_apply");
    }
  }
  const LevelState &fin = L.lv[L.n_levels - 1];
  k_finalize<<<grid_for(fin.n, 256), 256, 0, st>>>(fin);
  DIST_CHECK_LAUNCH("k_finalize");
  return DIST_OK;
}

int dist_maps(const dist_camera *cams, int V, int W, int H, const dist_trace_config *cfg,
              const dist_ray_state *stt, double *depth, uint8_t *mask, double *sil, void *stream) {
  if (!cams || !cfg || !stt) return fail(DIST_ERR_CONFIG, "null argument");
  LevelState ls{stt->d, stt->b, stt->status, stt->steps, stt->topk_d, stt->topk_f, stt->topk_absf,
                W, H, 1, (int64_t)V * W * H};
  k_maps<<<grid_for(ls.n, 256), 256, 0, (cudaStream_t)stream>>>(cams, ls, cfg->alpha, cfg->epsilon,
                                                                 cfg->k_samples, depth, mask, sil);
  DIST_CHECK_LAUNCH("k_maps");
  return DIST_OK;
}

size_t dist_normals_workspace_size(const dist_decoder *dec, int V, int W, int H, int S) {
  if (!dec) return 0;
  const int64_t n = (int64_t)V * W * H;
  Carve cv{nullptr, 0, ~size_t(0)};
  const int s1 = std::max(S, 1);
  cv.take<double>(c0_doubles(s1, dec->view.np[0]));
  cv.take<double>(c0_doubles(s1, std::max(dec->view.nskip, 1)));
  cv.take<int32_t>(n);
  cv.take<int32_t>(4);
  cv.take<int32_t>(ceil_div(n, kScanBlock) + 1);
  cv.take<double>(n * 6);
  return cv.off + 256;
}

int dist_normals(const dist_decoder *dec, const double *codes, int S, const dist_camera *cams,
                 int V, int W, int H, const dist_trace_config *cfg, const dist_ray_state *stt,
                 double *normals, void *ws, size_t ws_bytes, void *stream) {
  if (!dec || !cams || !cfg || !stt || !normals) return fail(DIST_ERR_CONFIG, "null argument");
  const DecView &dv = dec->view;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = (int64_t)V * W * H;
  const int s1 = std::max(S, 1);
  Carve cv{(char *)ws, 0, ws_bytes};
  double *c0 = cv.take<double>(c0_doubles(s1, dv.np[0]));
  double *cs = cv.take<double>(c0_doubles(s1, std::max(dv.nskip, 1)));
  int32_t *conv = cv.take<int32_t>(n);
  int32_t *count = cv.take<int32_t>(4);
  int32_t *bcount = cv.take<int32_t>(ceil_div(n, kScanBlock) + 1);
  double *f = cv.take<double>(n * 6);
  if (!cv.ok) return fail(DIST_ERR_CONFIG, "normals workspace too small");
  cudaError_t e = cudaMemsetAsync(normals, 0, sizeof(double) * 3 * n, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(normals)");
  int rc = launch_code_bias(dv, dv.latent_dim > 0 ? codes : nullptr, s1, c0, cs, st);
  if (rc) return rc;
  LevelState ls{stt->d, stt->b, stt->status, stt->steps, stt->topk_d, stt->topk_f, stt->topk_absf,
                W, H, 1, n};
  return normals_pass(dv, c0, cs, s1, cams, ls, cfg, normals, nullptr, conv, count, bcount, f, st);
}

}  // extern "C"
