// Standalone host program over the C ABI only (include/dist.h): no Python, no
// torch.  It loads a decoder + one view from a flat binary "job" file, runs
// dist_trace -> dist_maps -> dist_normals on the GPU and writes the depth map,
// status, normals and the trace statistics back to a flat binary file.  This
// is the call sequence a non-Python integrator of the reference's render path
// (tracer.py:221-252 trace, shading.py:48-113 depth_map / normal_map) would
// write.  tests/test_cabi_example.py writes the job from a NeuralField and
// checks the output against the Python package bit for bit.
//
// Build:  make -C examples        (links ../paper_1911_13225_b200/libdist_b200.so)
// Run:    examples/trace_cabi job.bin out.bin
//
// Job file (little endian):
//   int32 n_layers, latent_dim, skip_layer, final_linear, precision
//   int32 dims[n_layers + 1]
//   per layer: float64 W[dims[l] * dims[l+1]] (row-major [in,out]), float64 b[dims[l+1]]
//   float64 code[latent_dim]
//   dist_camera (raw struct), dist_trace_config (raw struct)
// Output file:
//   int64 stats[4], int64 live_counts[max_steps]
//   float64 depth[H*W], uint8 status[H*W], float64 normals[H*W*3]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dist.h"

#define CK_DIST(x)                                                              \
  do {                                                                          \
    int rc_ = (x);                                                              \
    if (rc_ != DIST_OK) {                                                       \
      std::fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, dist_last_error()); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)
#define CK_CUDA(x)                                                                   \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));           \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

template <class T>
static void get(FILE* f, T* dst, size_t n) {
  if (std::fread(dst, sizeof(T), n, f) != n) {
    std::fprintf(stderr, "truncated job file\n");
    std::exit(1);
  }
}

template <class T>
static T* dev_alloc(size_t n) {
  void* p = nullptr;
  CK_CUDA(cudaMalloc(&p, n * sizeof(T) + 16));
  return static_cast<T*>(p);
}

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: %s job.bin out.bin\n", argv[0]);
    return 2;
  }
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) {
    std::perror(argv[1]);
    return 1;
  }
  int32_t hdr[5];
  get(f, hdr, 5);
  const int L = hdr[0], latent = hdr[1], skip = hdr[2], final_linear = hdr[3], prec = hdr[4];
  std::vector<int32_t> dims(L + 1);
  get(f, dims.data(), dims.size());
  std::vector<std::vector<double>> W(L), b(L);
  std::vector<const double*> Wp(L), bp(L);
  for (int l = 0; l < L; ++l) {
    W[l].resize(size_t(dims[l]) * dims[l + 1]);
    b[l].resize(dims[l + 1]);
    get(f, W[l].data(), W[l].size());
    get(f, b[l].data(), b[l].size());
    Wp[l] = W[l].data();
    bp[l] = b[l].data();
  }
  std::vector<double> code(latent);
  get(f, code.data(), code.size());
  dist_camera cam;
  dist_trace_config cfg;
  get(f, &cam, 1);
  get(f, &cfg, 1);
  std::fclose(f);

  int sms = 0, ccM = 0, ccm = 0;
  CK_DIST(dist_device_info(&sms, &ccM, &ccm));

  dist_decoder* dec = nullptr;
  CK_DIST(dist_decoder_create(Wp.data(), bp.data(), L, dims.data(), latent, skip, final_linear,
                              prec, &dec));

  const int Wd = cam.width, Ht = cam.height, K = cfg.k_samples;
  const size_t n = size_t(Wd) * Ht;
  cudaStream_t stream;
  CK_CUDA(cudaStreamCreate(&stream));

  double* codes_dev = latent ? dev_alloc<double>(latent) : nullptr;
  if (latent)
    CK_CUDA(cudaMemcpy(codes_dev, code.data(), latent * sizeof(double), cudaMemcpyHostToDevice));
  dist_camera* cam_dev = dev_alloc<dist_camera>(1);
  CK_CUDA(cudaMemcpy(cam_dev, &cam, sizeof cam, cudaMemcpyHostToDevice));

  dist_ray_state rs;
  rs.d = dev_alloc<double>(n);
  rs.b = dev_alloc<double>(n);
  rs.status = dev_alloc<uint8_t>(n);
  rs.steps = dev_alloc<int32_t>(n);
  rs.topk_d = dev_alloc<double>(n * K);
  rs.topk_f = dev_alloc<double>(n * K);
  rs.topk_absf = dev_alloc<double>(n * K);
  rs.relu_masks = nullptr;   // no objective here: the mask record stays off
  rs.topk_slot = nullptr;
  int64_t* live_dev = dev_alloc<int64_t>(cfg.max_steps);
  int64_t* stats_dev = dev_alloc<int64_t>(4);

  // one workspace big enough for the trace and the normal probes
  size_t ws_trace = dist_trace_workspace_size(dec, &cfg, 1, Wd, Ht, 1);
  size_t ws_norm = dist_normals_workspace_size(dec, 1, Wd, Ht, 1);
  size_t ws_bytes = ws_trace > ws_norm ? ws_trace : ws_norm;
  void* ws = dev_alloc<uint8_t>(ws_bytes);

  double* depth_dev = dev_alloc<double>(n);
  double* normals_dev = dev_alloc<double>(n * 3);

  CK_DIST(dist_trace(dec, codes_dev, 1, cam_dev, 1, Wd, Ht, &cfg, &rs, live_dev, stats_dev, ws,
                     ws_bytes, stream));
  CK_DIST(dist_maps(cam_dev, 1, Wd, Ht, &cfg, &rs, depth_dev, nullptr, nullptr, stream));
  CK_DIST(dist_normals(dec, codes_dev, 1, cam_dev, 1, Wd, Ht, &cfg, &rs, normals_dev, ws,
                       ws_bytes, stream));
  CK_CUDA(cudaStreamSynchronize(stream));

  std::vector<int64_t> stats(4), live(cfg.max_steps);
  std::vector<double> depth(n), normals(n * 3);
  std::vector<uint8_t> status(n);
  CK_CUDA(cudaMemcpy(stats.data(), stats_dev, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  CK_CUDA(cudaMemcpy(live.data(), live_dev, cfg.max_steps * sizeof(int64_t), cudaMemcpyDeviceToHost));
  CK_CUDA(cudaMemcpy(depth.data(), depth_dev, n * sizeof(double), cudaMemcpyDeviceToHost));
  CK_CUDA(cudaMemcpy(status.data(), rs.status, n, cudaMemcpyDeviceToHost));
  CK_CUDA(cudaMemcpy(normals.data(), normals_dev, n * 3 * sizeof(double), cudaMemcpyDeviceToHost));

  FILE* o = std::fopen(argv[2], "wb");
  if (!o) {
    std::perror(argv[2]);
    return 1;
  }
  std::fwrite(stats.data(), sizeof(int64_t), 4, o);
  std::fwrite(live.data(), sizeof(int64_t), live.size(), o);
  std::fwrite(depth.data(), sizeof(double), n, o);
  std::fwrite(status.data(), 1, n, o);
  std::fwrite(normals.data(), sizeof(double), n * 3, o);
  std::fclose(o);

  size_t hits = 0;
  for (uint8_t s : status) hits += s == DIST_CONVERGED;
  std::printf("{\"sm_count\": %d, \"cc\": \"%d.%d\", \"rays\": %zu, \"converged\": %zu, "
              "\"queries\": %lld, \"steps\": %lld, \"launches\": %lld}\n",
              sms, ccM, ccm, n, hits, (long long)stats[0], (long long)stats[2],
              (long long)dist_launch_count());

  CK_DIST(dist_decoder_destroy(dec));
  for (void* p : {(void*)codes_dev, (void*)cam_dev, (void*)rs.d, (void*)rs.b, (void*)rs.status,
                  (void*)rs.steps, (void*)rs.topk_d, (void*)rs.topk_f, (void*)rs.topk_absf,
                  (void*)live_dev, (void*)stats_dev, ws, (void*)depth_dev, (void*)normals_dev})
    if (p) CK_CUDA(cudaFree(p));
  CK_CUDA(cudaStreamDestroy(stream));
  return 0;
}
