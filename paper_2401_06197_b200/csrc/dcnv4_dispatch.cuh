// dcnv4_dispatch.cuh -- template instantiation table for one storage type.
// Included once per dtype translation unit (dcnv4_f32.cu / _f16.cu / _bf16.cu) so the
// three sets compile in parallel.  Defines launch_fwd_<SUFFIX> / launch_bwd_<SUFFIX> /
// launch_convert_<SUFFIX>.
#pragma once
#include "dcnv4_kernels.cuh"
#include "dcnv4_launch.h"

namespace dcnv4 {

// Persistent grid: as many CTAs as fit on the device at once (never more than tiles).
// The occupancy query costs tens of microseconds of host time; its answer depends only on
// (device, kernel, threads, shared memory), so it is memoised per host thread.
static unsigned grid_size(const Launch& lc, const void* kern) {
  if (!lc.persistent) return (unsigned)lc.ctas;
  struct Memo {
    const void* kern;
    int dev, threads, sms, per_sm;
    size_t smem;
  };
  thread_local Memo memo[16];
  thread_local int memo_n = 0;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  for (int i = 0; i < memo_n; ++i) {
    const Memo& m = memo[i];
    if (m.kern == kern && m.dev == dev && m.threads == lc.threads && m.smem == lc.smem) {
      const long long g = (long long)m.sms * m.per_sm;
      return (unsigned)(g < lc.ctas ? g : lc.ctas);
    }
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, lc.threads, lc.smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  memo[memo_n % 16] = Memo{kern, dev, lc.threads, sms, per_sm, lc.smem};
  memo_n = memo_n < 16 ? memo_n + 1 : 16;
  const long long g = (long long)sms * per_sm;
  return (unsigned)(g < lc.ctas ? g : lc.ctas);
}

template <typename T, int NCH, int CPL>
static cudaError_t fwd_variant(const Launch& lc, const Geo& g, const void* x, const void* om,
                               void* y) {
  const T* xp = static_cast<const T*>(x);
  const T* op = static_cast<const T*>(om);
  T* yp = static_cast<T*>(y);
  if (lc.halo) {  // 3x3 / stride 1 / dilation 1: TMA halo kernel
    void (*hk)(const __grid_constant__ Fwd33Prob);
    if (lc.unit) hk = fwd33_kernel<T, NCH, CPL, true>;
    else hk = fwd33_kernel<T, NCH, CPL, false>;
    if (lc.smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)lc.smem);
      if (e != cudaSuccess) return e;
    }
    cudaFuncSetAttribute(hk, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    Fwd33Prob prob;
    prob.xmap = lc.xmap;
    prob.g = g;
    prob.x = xp;
    prob.om = op;
    prob.y = yp;
    prob.t0 = 0;
    hk<<<grid_size(lc, (const void*)hk), lc.threads, lc.smem, lc.stream>>>(prob);
    return cudaGetLastError();
  }
  void (*kern)(Geo, const T*, const T*, T*);
  if (lc.k33 && lc.unit) kern = fwd_kernel<T, NCH, CPL, 3, 3, true>;
  else if (lc.k33) kern = fwd_kernel<T, NCH, CPL, 3, 3, false>;
  else kern = fwd_kernel<T, NCH, CPL, 0, 0, false>;
  if (lc.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lc.smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid_size(lc, (const void*)kern), lc.threads, lc.smem, lc.stream>>>(g, xp, op, yp);
  return cudaGetLastError();
}

template <typename T, int NCH, int CPL>
static cudaError_t bwd_variant(const Launch& lc, const Geo& g, const void* x, const void* om,
                               const void* gy, void* gxacc, void* gom) {
  const T* xp = static_cast<const T*>(x);
  const T* op = static_cast<const T*>(om);
  const T* gyp = static_cast<const T*>(gy);
  T* gomp = static_cast<T*>(gom);
  if (lc.halo) {  // 3x3 / stride 1 / dilation 1: TMA halo + binned scatter
    void (*hk)(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, Geo,
               const T*, const T*, void*, T*);
    if (lc.det) hk = lc.unit ? bwd33_kernel<T, NCH, CPL, true, true> : bwd33_kernel<T, NCH, CPL, false, true>;
    else hk = lc.unit ? bwd33_kernel<T, NCH, CPL, true, false> : bwd33_kernel<T, NCH, CPL, false, false>;
    if (lc.smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)lc.smem);
      if (e != cudaSuccess) return e;
    }
    // the largest shared-memory carveout, so the occupancy the tile was sized for is reached
    cudaFuncSetAttribute(hk, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    hk<<<grid_size(lc, (const void*)hk), lc.threads, lc.smem, lc.stream>>>(lc.xmap, lc.gymap, g, xp,
                                                                            op, gxacc, gomp);
    return cudaGetLastError();
  }
  void (*kern)(Geo, const T*, const T*, const T*, void*, T*);
  if (lc.det) {
    if (lc.k33 && lc.unit) kern = bwd_kernel<T, NCH, CPL, 3, 3, true, true>;
    else if (lc.k33) kern = bwd_kernel<T, NCH, CPL, 3, 3, false, true>;
    else kern = bwd_kernel<T, NCH, CPL, 0, 0, false, true>;
  } else {
    if (lc.k33 && lc.unit) kern = bwd_kernel<T, NCH, CPL, 3, 3, true, false>;
    else if (lc.k33) kern = bwd_kernel<T, NCH, CPL, 3, 3, false, false>;
    else kern = bwd_kernel<T, NCH, CPL, 0, 0, false, false>;
  }
  if (lc.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lc.smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid_size(lc, (const void*)kern), lc.threads, lc.smem, lc.stream>>>(g, xp, op, gyp, gxacc, gomp);
  return cudaGetLastError();
}

// Several fwd33 problems in one persistent launch (dcnv4_forward_grouped).
template <typename T, int NCH, int CPL>
static cudaError_t fwd_group_variant(const Launch& lc, const Geo&, const void* grp) {
  void (*hk)(const __grid_constant__ Fwd33Group);
  if (lc.unit) hk = fwd33_group_kernel<T, NCH, CPL, true>;
  else hk = fwd33_group_kernel<T, NCH, CPL, false>;
  if (lc.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.smem);
    if (e != cudaSuccess) return e;
  }
  cudaFuncSetAttribute(hk, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  hk<<<grid_size(lc, (const void*)hk), lc.threads, lc.smem, lc.stream>>>(
      *static_cast<const Fwd33Group*>(grp));
  return cudaGetLastError();
}

static inline unsigned flat_blocks(long long n) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  return (unsigned)(blocks < 1 ? 1 : blocks);
}

#ifdef DCNV4_VARIANT_MIN  // A/B variant builds (scripts/build_variant.py): D = 16 only
#define DCNV4_TABLE(FN, T, ...)                                        \
  switch (lc.nch * 100 + lc.cpl) {                                     \
    case 202: return FN<T, 2, 2>(lc, g, __VA_ARGS__);                  \
    case 402: return FN<T, 4, 2>(lc, g, __VA_ARGS__);                  \
    default: return cudaErrorInvalidConfiguration;                     \
  }
#else
#define DCNV4_TABLE(FN, T, ...)                                        \
  switch (lc.nch * 100 + lc.cpl) {                                     \
    case 101: return FN<T, 1, 1>(lc, g, __VA_ARGS__);                  \
    case 201: return FN<T, 2, 1>(lc, g, __VA_ARGS__);                  \
    case 202: return FN<T, 2, 2>(lc, g, __VA_ARGS__);                  \
    case 401: return FN<T, 4, 1>(lc, g, __VA_ARGS__);                  \
    case 402: return FN<T, 4, 2>(lc, g, __VA_ARGS__);                  \
    case 404: return FN<T, 4, 4>(lc, g, __VA_ARGS__);                  \
    case 802: return FN<T, 8, 2>(lc, g, __VA_ARGS__);                  \
    case 804: return FN<T, 8, 4>(lc, g, __VA_ARGS__);                  \
    case 1602: return FN<T, 16, 2>(lc, g, __VA_ARGS__);                \
    case 1604: return FN<T, 16, 4>(lc, g, __VA_ARGS__);                \
    default: return cudaErrorInvalidConfiguration;                     \
  }
#endif

// One storage type's launchers (used by dcnv4_f32.cu / _f16.cu / _bf16.cu).
#define DCNV4_DEFINE(SUFFIX, T)                                                                 \
  cudaError_t launch_fwd_##SUFFIX(const Launch& lc, const Geo& g, const void* x, const void* om, \
                                  void* y) {                                                    \
    DCNV4_TABLE(fwd_variant, T, x, om, y)                                                      \
  }                                                                                             \
  cudaError_t launch_bwd_##SUFFIX(const Launch& lc, const Geo& g, const void* x, const void* om, \
                                  const void* gy, void* gxacc, void* gom) {                     \
    DCNV4_TABLE(bwd_variant, T, x, om, gy, gxacc, gom)                                         \
  }                                                                                             \
  cudaError_t launch_fwd_group_##SUFFIX(const Launch& lc, const Geo& g, const void* grp) {     \
    DCNV4_TABLE(fwd_group_variant, T, grp)                                                      \
  }                                                                                             \
  cudaError_t launch_convert_##SUFFIX(const float* src, void* dst, long long nchunk,            \
                                      cudaStream_t stream) {                                    \
    if (nchunk <= 0) return cudaSuccess;                                                        \
    convert_kernel<T><<<flat_blocks(nchunk), 256, 0, stream>>>(src, static_cast<T*>(dst), nchunk); \
    return cudaGetLastError();                                                                  \
  }                                                                                             \
  cudaError_t launch_detmax_##SUFFIX(const void* gy, const void* om, long long N, int npix,     \
                                     int C, int S, int G, int K, int softmax, unsigned* mx,     \
                                     cudaStream_t stream) {                                     \
    if (N <= 0) return cudaSuccess;                                                             \
    const long long chunks = (long long)npix * C / Elem<T>::E;                                 \
    /* images on grid.y, at most 65535 per launch */                                         \
    for (long long n0 = 0; n0 < N; n0 += 65535) {                                               \
      const long long nb = N - n0 < 65535 ? N - n0 : 65535;                                     \
      long long per = (chunks + 255) / 256;                                                     \
      const long long want = (148LL * 8 + nb - 1) / nb;                                         \
      if (per > want) per = want;                                                               \
      dim3 grid((unsigned)(per < 1 ? 1 : per), (unsigned)nb);                                   \
      det_scale_kernel<T><<<grid, 256, 0, stream>>>(static_cast<const T*>(gy),                  \
                                                    static_cast<const T*>(om), chunks, npix, S, G, \
                                                    K, softmax, mx, n0);                        \
    }                                                                                           \
    return cudaGetLastError();                                                                  \
  }                                                                                             \
  cudaError_t launch_detconv_##SUFFIX(const long long* src, const unsigned* mx, int lc,         \
                                      long long per_image, void* dst, long long nchunk,         \
                                      cudaStream_t stream) {                                    \
    if (nchunk <= 0) return cudaSuccess;                                                        \
    det_convert_kernel<T><<<flat_blocks(nchunk), 256, 0, stream>>>(src, mx, lc, per_image,     \
                                                                  static_cast<T*>(dst), nchunk); \
    return cudaGetLastError();                                                                  \
  }

}  // namespace dcnv4
