// dcnv4_launch.h -- internal host-side launch description shared by the API and the
// per-dtype instantiation units (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>

namespace dcnv4 {

struct Geo;

struct Launch {
  int nch;          // 16-B chunks per (pixel, group) = D*sizeof(T)/16
  int cpl;          // chunks per lane
  int lanes;        // nch / cpl lanes per (pixel, group)
  int ppc;          // output pixels per CTA
  int threads;      // CTA size (multiple of 32)
  long long ctas;   // tiles (CTA work units); persistent grid = min(tiles, SMs x occupancy)
  bool persistent;  // false: one CTA per tile (ablation)
  size_t smem;      // dynamic shared memory bytes
  bool k33;         // compile-time 3x3 path
  bool unit;        // offset_scale == 1 exact-split path
  cudaStream_t stream;
  bool halo;        // forward: TMA halo kernel (else the global-gather kernel)
  CUtensorMap xmap; // TMA descriptor of x for the halo kernels
  CUtensorMap gymap;  // TMA descriptor of grad_output (backward halo kernel)
  bool det;         // backward: deterministic int64 grad_input accumulation
};

#define DCNV4_DECLARE(SUFFIX)                                                              \
  cudaError_t launch_fwd_##SUFFIX(const Launch& lc, const Geo& g, const void* x,          \
                                  const void* om, void* y);                                \
  cudaError_t launch_bwd_##SUFFIX(const Launch& lc, const Geo& g, const void* x,          \
                                  const void* om, const void* gy, void* gxacc, void* gom); \
  cudaError_t launch_fwd_group_##SUFFIX(const Launch& lc, const Geo& g,                    \
                                        const void* grp /* Fwd33Group */);                 \
  cudaError_t launch_convert_##SUFFIX(const float* src, void* dst, long long nchunk,      \
                                      cudaStream_t stream);                                \
  cudaError_t launch_detmax_##SUFFIX(const void* gy, const void* om, long long N, int npix, \
                                     int C, int S, int G, int K, int softmax, unsigned* mx, \
                                     cudaStream_t stream);                                 \
  cudaError_t launch_detconv_##SUFFIX(const long long* src, const unsigned* mx, int lc,     \
                                      long long per_image, void* dst, long long nchunk,     \
                                      cudaStream_t stream);

DCNV4_DECLARE(f32)
DCNV4_DECLARE(f16)
DCNV4_DECLARE(bf16)

}  // namespace dcnv4
