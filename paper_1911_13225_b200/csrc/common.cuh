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
  int nr[kMaxLayers + 1]; // true output width of layer l (dims[l + 1]; the h part for the skip input)
  // layer 0 in fp64: W0z [D][np0], W0p [3][np0], b0 [np0]
  const double *W0z, *W0p, *b0;
  const float *W0pf;       // fp32 copy of W0p for the tensor-core prologue
  // hidden GEMM layers 1..L-2, [0] = fp64 copy, [1] = fp32 copy:
  // W [kp][np] (row-major, the reference's x@W layout), Wt [np][kp], bias [np]
  const void *W[2][kMaxLayers], *Wt[2][kMaxLayers], *bias[2][kMaxLayers];
  // skip layer extra input rows (code+xyz part) kept in fp64: Wsz [D][np], Wsp [3][np]
  const double *Wsz, *Wsp;
  const float *Wspf;      // fp32 copy of Wsp for the tensor-core epilogues
  float wsm[3];           // max |Wsp row a| (bounds the fp16 row scale of the skip layer)
  int nskip;              // np[skip] (0 if no skip)
  // output layer: w_out [kp_out] (fp64 / fp32 copies), b_out
  const void *w_out[2];
  double b_out;
  // split-precision packs for the tensor-core path (bf16 hi/lo, K-major tiles)
  const void *tc_w[kMaxLayers];
  const float *tc_bias[kMaxLayers];
  // Calibrated gain of the 512 -> 1 head dot in the tensor-core forward
  // (tc_mlp.cu tc_calibrate): [0] for pack slot 0, [1] for the fp16 probe
  // pack of a bf16x3 decoder (slot 2).  1 for the SIMT precisions.
  double tc_gain[2];
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

// Exact gradient column sums.  Every per-row contribution to the layer-0
// column sums (the code gradient is W0[:D] times them, autodiff.py:175-185) is
// converted to a 128-bit two's-complement fixed-point integer, value * 2^95,
// and summed as an integer.  Integer addition is associative, so the sums --
// and the code gradient -- are the same bit pattern whatever the partition of
// samples into tiles, CTAs or ranks (identical iterates for any GPU
// count), and no rounding accumulates with the sample count.  Range +-2^31;
// resolution 2^-95 (a double with |x| >= 2^-42 converts exactly).  A
// non-finite or out-of-range contribution sets a flag that turns the gradient
// into NaN (the reference raises on a non-finite gradient, autodiff.py:253-254).
typedef __int128 fx_t;
constexpr int kFxShift = 95;

__device__ __forceinline__ fx_t fx_from_double(double x, int *bad) {
  if (!(fabs(x) < 2147483648.0)) {  // also catches NaN
    *bad = 1;
    return 0;
  }
  const double a = x * 4294967296.0;                 // x * 2^32, exact
  const long long A = (long long)a;                  // toward zero, |A| < 2^63
  const double r = a - (double)A;                    // exact fractional part, |r| < 1
  const long long B = (long long)(r * 9223372036854775808.0);   // r * 2^63, toward zero
  return (fx_t)((unsigned __int128)(fx_t)A << 63) + (fx_t)B;
}

// fp32 -> fx_t from the bit pattern (the tensor-core kernels' rows):
// x = m 2^(e-150) -> m << (e - 55), truncated toward zero below 2^-95
__device__ __forceinline__ fx_t fx_from_float(float x, int &bad) {
  const uint32_t u = __float_as_uint(x);
  const int e = (int)((u >> 23) & 0xffu);
  if (e >= 158) {   // |x| >= 2^31, inf or NaN
    bad = 1;
    return 0;
  }
  const uint32_t m = (u & 0x7fffffu) | (e ? 0x800000u : 0u);
  const int sh = (e ? e : 1) - 55;
  const fx_t mag = sh >= 0 ? (fx_t)((unsigned __int128)m << sh) : (sh > -24 ? (fx_t)(m >> -sh) : (fx_t)0);
  return (u >> 31) ? -mag : mag;
}

__device__ __forceinline__ fx_t fx_shfl_xor(fx_t v, int o) {
  const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, o);
  const unsigned long long hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
  return (fx_t)(((unsigned __int128)hi2 << 64) | lo2);
}

// correctly rounded (one rounding, to nearest): the top 64 significant bits
// with a sticky bit for the rest convert exactly like the full value, so
// scaling the sums by a power of two scales the result exactly
__device__ inline double fx_to_double(fx_t v) {
  if (v == 0) return 0.0;
  const bool neg = v < 0;
  unsigned __int128 m = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
  const unsigned long long hi = (unsigned long long)(m >> 64);
  const int lz = hi ? __clzll(hi) : 64 + __clzll((unsigned long long)m);
  m <<= lz;
  unsigned long long t = (unsigned long long)(m >> 64);
  t |= ((unsigned long long)m != 0ull) ? 1ull : 0ull;
  const double r = ldexp((double)t, 64 - lz - kFxShift);
  return neg ? -r : r;
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
