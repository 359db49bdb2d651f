// common.cuh -- shared device/host helpers for libdist_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/dist.h"

namespace dist {

constexpr int kMaxLayers = 16;
constexpr int kMaxWidth = 512;          // widest hidden layer the kernels tile
constexpr int kSampleAlign = 128;       // per-view sample segment alignment (tcgen05 tile M)

// error plumbing ----------------------------------------------------------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *where);
void count_launch(int n = 1);

#define DIST_CHECK_LAUNCH(where)                                   \
  do {                                                             \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return ::dist::cuda_fail(_e, where);    \
    ::dist::count_launch();                                        \
  } while (0)

// decoder -------------------------------------------------------------------
// Device view of a decoder, passed to kernels by value.  Widths are padded to
// multiples of 64 (np[l]); padded units carry zero weights and bias so they
// stay exactly zero through ReLU.
struct DecView {
  int n_layers;           // L weight matrices
  int latent_dim;         // D
  int skip;               // -1 or skip layer index
  int final_act;          // head activation: 0 tanh, 1 linear, 2 sigmoid (AttributeField)
  int prec;
  int np[kMaxLayers + 1]; // padded output width of layer l (np[L-1] = 1)
  int kp[kMaxLayers + 1]; // padded input width of hidden layer l (GEMM K)
  // layer 0 in fp64: W0z [D][np0], W0p [3][np0], b0 [np0]
  const double *W0z, *W0p, *b0;
  const float *W0pf;       // fp32 copy of W0p for the tensor-core prologue
  // hidden GEMM layers 1..L-2, [0] = fp64 copy, [1] = fp32 copy:
  // W [kp][np] (row-major, the reference's x@W layout), Wt [np][kp], bias [np]
  const void *W[2][kMaxLayers], *Wt[2][kMaxLayers], *bias[2][kMaxLayers];
  // skip layer extra input rows (code+xyz part) kept in fp64: Wsz [D][np], Wsp [3][np]
  const double *Wsz, *Wsp;
  int nskip;              // np[skip] (0 if no skip)
  // output layer: w_out [kp_out] (fp64 / fp32 copies), b_out
  const void *w_out[2];
  double b_out;
  // split-precision packs for the tensor-core path (bf16 hi/lo, K-major tiles)
  const void *tc_w[kMaxLayers];
  const float *tc_bias[kMaxLayers];
};

}  // namespace dist

struct dist_decoder {
  dist::DecView view;
  void *blob;          // single device allocation holding every array
  size_t blob_bytes;
  int dims[dist::kMaxLayers + 1];
};

namespace dist {

// Head activation and its derivative written in terms of the output f
// (fields.py:245-246 tanh/linear; fields.py:332-338 sigmoid of AttributeField).
__host__ __device__ inline double head_act(int act, double s) {
  return act == 0 ? tanh(s) : (act == 1 ? s : 1.0 / (1.0 + exp(-s)));
}
__host__ __device__ inline double head_dact(int act, double f) {
  return act == 0 ? 1.0 - f * f : (act == 1 ? 1.0 : f * (1.0 - f));
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Pixel-centre ray of pixel (i, j) at `level` (camera.py:190-212):
// v_cam = (((i+.5)L - cx)/fx, ((j+.5)L - cy)/fy, 1); dir = R^T v_cam/|v_cam|;
// scale = 1/|v_cam| converts ray distance to camera z.
__device__ __forceinline__ void pixel_ray(const dist_camera &c, int i, int j, int level,
                                          double dir[3], double *scale) {
  double x = ((i + 0.5) * level - c.cx) / c.fx;
  double y = ((j + 0.5) * level - c.cy) / c.fy;
  double n = sqrt(x * x + y * y + 1.0);
  double ux = x / n, uy = y / n, uz = 1.0 / n;
  dir[0] = ux * c.R[0] + uy * c.R[3] + uz * c.R[6];
  dir[1] = ux * c.R[1] + uy * c.R[4] + uz * c.R[7];
  dir[2] = ux * c.R[2] + uy * c.R[5] + uz * c.R[8];
  if (scale) *scale = 1.0 / n;
}

// Workspace carving: bump allocator over a caller-provided buffer.
struct Carve {
  char *base;
  size_t off, cap;
  bool ok = true;
  template <typename T>
  T *take(size_t count, size_t align = 256) {
    off = (size_t)round_up((int64_t)off, (int64_t)align);
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += count * sizeof(T);
    if (off > cap) ok = false;
    return p;
  }
};

}  // namespace dist
