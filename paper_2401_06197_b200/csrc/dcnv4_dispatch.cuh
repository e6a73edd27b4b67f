// dcnv4_dispatch.cuh -- template instantiation table for one storage type.
// Included once per dtype translation unit (dcnv4_f32.cu / _f16.cu / _bf16.cu) so the
// three sets compile in parallel.  Defines launch_fwd_<SUFFIX> / launch_bwd_<SUFFIX> /
// launch_convert_<SUFFIX>.
#pragma once
#include "dcnv4_kernels.cuh"
#include "dcnv4_launch.h"

namespace dcnv4 {

// Persistent grid: as many CTAs as fit on the device at once (never more than tiles).
static unsigned grid_size(const Launch& lc, const void* kern) {
  if (!lc.persistent) return (unsigned)lc.ctas;
  int dev = 0, sms = 148, per_sm = 1;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, lc.threads, lc.smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
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
    void (*hk)(const __grid_constant__ CUtensorMap, Geo, const T*, const T*, T*);
    if (lc.unit) hk = fwd33_kernel<T, NCH, CPL, true>;
    else hk = fwd33_kernel<T, NCH, CPL, false>;
    if (lc.smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)lc.smem);
      if (e != cudaSuccess) return e;
    }
    hk<<<grid_size(lc, (const void*)hk), lc.threads, lc.smem, lc.stream>>>(lc.xmap, g, xp, op, yp);
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
                               const void* gy, float* gx32, void* gom) {
  const T* xp = static_cast<const T*>(x);
  const T* op = static_cast<const T*>(om);
  const T* gyp = static_cast<const T*>(gy);
  T* gomp = static_cast<T*>(gom);
  if (lc.halo) {  // 3x3 / stride 1 / dilation 1: TMA halo + binned scatter
    void (*hk)(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, Geo,
               const T*, const T*, float*, T*);
    if (lc.unit) hk = bwd33_kernel<T, NCH, CPL, true>;
    else hk = bwd33_kernel<T, NCH, CPL, false>;
    if (lc.smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)lc.smem);
      if (e != cudaSuccess) return e;
    }
    hk<<<grid_size(lc, (const void*)hk), lc.threads, lc.smem, lc.stream>>>(lc.xmap, lc.gymap, g, xp,
                                                                            op, gx32, gomp);
    return cudaGetLastError();
  }
  void (*kern)(Geo, const T*, const T*, const T*, float*, T*);
  if (lc.k33 && lc.unit) kern = bwd_kernel<T, NCH, CPL, 3, 3, true>;
  else if (lc.k33) kern = bwd_kernel<T, NCH, CPL, 3, 3, false>;
  else kern = bwd_kernel<T, NCH, CPL, 0, 0, false>;
  if (lc.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lc.smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid_size(lc, (const void*)kern), lc.threads, lc.smem, lc.stream>>>(g, xp, op, gyp, gx32, gomp);
  return cudaGetLastError();
}

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

}  // namespace dcnv4
