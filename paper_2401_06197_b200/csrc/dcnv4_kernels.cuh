// dcnv4_kernels.cuh -- sm_100a kernels of the DCNv4 spatial aggregation.
//
// PAPER.md Eq. (1)-(2), softmax removed:
//   y_g(p0) = sum_k m_gk * x_g(p0 + p_k + dp_gk)
// B200 design:
//   * work item = one lane covering CPL 16-byte channel chunks of one (pixel, group);
//     L = NCH/CPL lanes share a (pixel, group) (NCH = D*sizeof(T)/16).  Offsets and m
//     are read once per (pixel, group) from shared memory and the bilinear coefficients
//     are computed once per (pixel, group, k) and reused across the lane's channels
//     (P:318-324);
//   * the CTA's offset_mask rows are one contiguous byte range; it is staged into
//     shared memory with one TMA bulk copy (cp.async.bulk + mbarrier) -- the 16-B
//     aligned body -- plus a few plain loads for the unaligned head/tail;
//   * corner gathers are 16-byte read-only vector loads (LDG.E.128.CONSTANT), predicated
//     off outside the image ("128-bit packed value");
//   * fp32 accumulation for every storage type, RN-even store (P:329 half precision);
//   * backward: grad_offset/grad_mask partials reduced across the L lanes with warp
//     shuffles, staged in shared memory and written coalesced; grad_input is a bilinear
//     scatter with 16-byte vector reductions (red.global.add.v4.f32) into fp32.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dcnv4 {

// Geometry handed to every kernel by value (validated on the host; per-image element
// counts fit in int32).
struct Geo {
  int H, W, Ho, Wo, G, D, C, S, K;
  int kh, kw, sh, sw, ph, pw, dh, dw, cy, cx;
  float s;
  int softmax;
  long long P;  // N*Ho*Wo output pixels
  int ppc;      // output pixels per CTA
};

// ------------------------------------------------------------------ element types
template <typename T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int E = 4;  // elements per 16-byte chunk
  __device__ __forceinline__ static float f(float v) { return v; }
  __device__ __forceinline__ static void unpack(const uint4& u, float* o) {
    o[0] = __uint_as_float(u.x); o[1] = __uint_as_float(u.y);
    o[2] = __uint_as_float(u.z); o[3] = __uint_as_float(u.w);
  }
  __device__ __forceinline__ static uint4 pack(const float* v) {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
  }
  __device__ __forceinline__ static float from_f32(float v) { return v; }
};
template <>
struct Elem<__half> {
  static constexpr int E = 8;
  __device__ __forceinline__ static float f(__half v) { return __half2float(v); }
  __device__ __forceinline__ static void unpack(const uint4& u, float* o) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 f2 = __half22float2(h);
      o[2 * i] = f2.x; o[2 * i + 1] = f2.y;
    }
  }
  __device__ __forceinline__ static uint4 pack(const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ static __half from_f32(float v) { return __float2half_rn(v); }
};
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int E = 8;
  __device__ __forceinline__ static float f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static void unpack(const uint4& u, float* o) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[2 * i] = __uint_as_float(w[i] << 16);
      o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ __forceinline__ static uint4 pack(const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ static __nv_bfloat16 from_f32(float v) { return __float2bfloat16_rn(v); }
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint4 ldg16(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

// Stage `count` elements of T starting at global `src` into shared memory.  The 16-B
// aligned body goes through one TMA bulk copy (UBLKCP) completing on an mbarrier; the
// unaligned head/tail (< 16 B each) is copied by threads.  Returns the shared-memory
// address of element 0.  Every thread of the CTA must call it.
template <typename T>
__device__ __forceinline__ const T* stage_rows(unsigned char* smem, uint64_t* bar,
                                              const T* src, int count) {
  const uintptr_t g0 = reinterpret_cast<uintptr_t>(src);
  const uintptr_t g1 = g0 + (uintptr_t)count * sizeof(T);
  const uintptr_t a0 = (g0 + 15) & ~uintptr_t(15);
  const uintptr_t a1 = g1 & ~uintptr_t(15);
  const uintptr_t gbase = g0 & ~uintptr_t(15);          // maps to smem offset 0
  T* tile = reinterpret_cast<T*>(smem + (g0 - gbase));
  const bool bulk = a1 > a0;
  if (threadIdx.x == 0 && bulk) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t bytes = (uint32_t)(a1 - a0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(smem + (a0 - gbase))),
        "l"(a0), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
  }
  // head [g0, min(a0, g1)) and tail [max(a1, a0), g1) by plain loads
  const int head = bulk ? (int)((a0 - g0) / sizeof(T)) : count;
  const int tail0 = bulk ? (int)((a1 - g0) / sizeof(T)) : count;
  for (int e = threadIdx.x; e < head; e += blockDim.x) tile[e] = src[e];
  for (int e = tail0 + threadIdx.x; e < count; e += blockDim.x) tile[e] = src[e];
  __syncthreads();  // head/tail visible; mbarrier init visible to the waiters
  if (bulk) {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(bar))
          : "memory");
    }
  }
  return tile;
}

// Sampling coordinate along one axis (R5, R11, R12):
//   p = base + s*(tap + d),  i0 = floor(p),  f = p - i0.
// With s == 1 the split is exact: floor and fraction of d alone, integer tap added
// to the integer part.  Returns false (drop the sample) for NaN or |s*(tap+d)| > 2^20.
template <bool UNIT>
__device__ __forceinline__ bool locate(float s, int base, int tap, float d, int& i0, float& f) {
  const float t = UNIT ? d : s * ((float)tap + d);
  if (!(fabsf(t) <= 1048576.f)) return false;
  const float fl = floorf(t);
  f = t - fl;
  i0 = base + (UNIT ? tap : 0) + (int)fl;
  return true;
}

// The K modulation scalars of one (pixel, group): raw (DCNv4) or the softmax
// over K (DCNv3; max-shifted).
template <typename T, int KC>
__device__ __forceinline__ void load_m(const T* row, int K, int softmax, float* m) {
#pragma unroll
  for (int k = 0; k < KC; ++k) m[k] = Elem<T>::f(row[2 * K + k]);
  if (softmax) {
    float mx = m[0];
#pragma unroll
    for (int k = 1; k < KC; ++k) mx = fmaxf(mx, m[k]);
    float den = 0.f;
#pragma unroll
    for (int k = 0; k < KC; ++k) { m[k] = __expf(m[k] - mx); den += m[k]; }
    const float inv = 1.f / den;
#pragma unroll
    for (int k = 0; k < KC; ++k) m[k] *= inv;
  }
}

// Generic-K version: softmax statistics (max, 1/sum) of one row.
template <typename T>
__device__ __forceinline__ void softmax_stats(const T* row, int K, float& mx, float& inv) {
  mx = Elem<T>::f(row[2 * K]);
  for (int k = 1; k < K; ++k) mx = fmaxf(mx, Elem<T>::f(row[2 * K + k]));
  float den = 0.f;
  for (int k = 0; k < K; ++k) den += __expf(Elem<T>::f(row[2 * K + k]) - mx);
  inv = 1.f / den;
}

// Bilinear corners of one sample: element offsets (relative to the image base, group
// base already added) and weights; out-of-image corners get weight 0 and valid=false.
struct Corners {
  int off[4];
  float w[4];
  bool ok[4];
  float fy, fx;
};

template <bool UNIT>
__device__ __forceinline__ void corners(const Geo& g, int yb, int xb, int tapy, int tapx,
                                        float dx, float dy, int gbase, Corners& c) {
  int y0, x0;
  float fy, fx;
  const bool oky = locate<UNIT>(g.s, yb, tapy, dy, y0, fy);
  const bool okx = locate<UNIT>(g.s, xb, tapx, dx, x0, fx);
  const bool ok = oky && okx;
  if (!ok) { y0 = -2; x0 = -2; fy = 0.f; fx = 0.f; }
  const bool vy0 = (unsigned)y0 < (unsigned)g.H, vy1 = (unsigned)(y0 + 1) < (unsigned)g.H;
  const bool vx0 = (unsigned)x0 < (unsigned)g.W, vx1 = (unsigned)(x0 + 1) < (unsigned)g.W;
  const float hy = 1.f - fy, hx = 1.f - fx;
  c.fy = fy; c.fx = fx;
  c.w[0] = hy * hx; c.w[1] = hy * fx; c.w[2] = fy * hx; c.w[3] = fy * fx;
  c.ok[0] = vy0 && vx0; c.ok[1] = vy0 && vx1; c.ok[2] = vy1 && vx0; c.ok[3] = vy1 && vx1;
  const int o = (y0 * g.W + x0) * g.C + gbase;
  c.off[0] = o; c.off[1] = o + g.C; c.off[2] = o + g.W * g.C; c.off[3] = o + g.W * g.C + g.C;
}

// ------------------------------------------------------------------ forward
// KH = KW = 0: runtime kernel size; otherwise compile-time (3x3 is the paper's grid).
template <typename T, int NCH, int CPL, int KH, int KW, bool UNIT>
__global__ void __launch_bounds__(256) fwd_kernel(Geo g, const T* __restrict__ x,
                                                  const T* __restrict__ om,
                                                  T* __restrict__ y) {
  constexpr int L = NCH / CPL;
  constexpr int E = Elem<T>::E;
  constexpr int KC = KH * KW;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t bar;

  const long long p_first = (long long)blockIdx.x * g.ppc;
  const int npix = (int)min((long long)g.ppc, g.P - p_first);
  const T* tile = stage_rows<T>(smem, &bar, om + p_first * g.S, npix * g.S);

  const int GL = g.G * L;
  const int t = threadIdx.x;
  const int pl = t / GL;
  if (pl >= npix) return;
  const int rem = t - pl * GL;
  const int grp = rem / L;
  const int lg = rem - grp * L;
  const long long pix = p_first + pl;
  const int HWo = g.Ho * g.Wo;
  const int n = (int)(pix / HWo);
  const int hw = (int)(pix - (long long)n * HWo);
  const int ho = hw / g.Wo, wo = hw - (hw / g.Wo) * g.Wo;
  const int yb = ho * g.sh - g.ph + g.cy;
  const int xb = wo * g.sw - g.pw + g.cx;
  const T* ximg = x + (long long)n * g.H * g.W * g.C;
  const int K = KC ? KC : g.K;
  const T* row = tile + pl * g.S + grp * 3 * K;
  const int cbase = grp * g.D + lg * CPL * E;

  float acc[CPL * E];
#pragma unroll
  for (int e = 0; e < CPL * E; ++e) acc[e] = 0.f;

  auto do_point = [&](int i, int j, int k, float m) {
    Corners c;
    corners<UNIT>(g, yb, xb, j * g.dh - g.cy, i * g.dw - g.cx, Elem<T>::f(row[2 * k]),
                  Elem<T>::f(row[2 * k + 1]), cbase, c);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = c.ok[q] ? m * c.w[q] : 0.f;
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        uint4 u = make_uint4(0, 0, 0, 0);
        if (c.ok[q]) u = ldg16(ximg + c.off[q] + h * E);
        float v[E];
        Elem<T>::unpack(u, v);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[h * E + e] = fmaf(a, v[e], acc[h * E + e]);
      }
    }
  };

  if constexpr (KC > 0) {
    float m[KC];
    load_m<T, KC>(row, KC, g.softmax, m);
#pragma unroll
    for (int i = 0; i < KW; ++i)
#pragma unroll
      for (int j = 0; j < KH; ++j) do_point(i, j, i * KH + j, m[i * KH + j]);
  } else {
    float mx = 0.f, inv = 1.f;
    if (g.softmax) softmax_stats<T>(row, K, mx, inv);
    for (int i = 0; i < g.kw; ++i)
      for (int j = 0; j < g.kh; ++j) {
        const int k = i * g.kh + j;
        float m = Elem<T>::f(row[2 * K + k]);
        if (g.softmax) m = __expf(m - mx) * inv;
        do_point(i, j, k, m);
      }
  }

  T* yo = y + pix * g.C + cbase;
#pragma unroll
  for (int h = 0; h < CPL; ++h)
    *reinterpret_cast<uint4*>(yo + h * E) = Elem<T>::pack(acc + h * E);
}

// ------------------------------------------------------------------ backward
// gx32: fp32 accumulator [N][H][W][C], zeroed by the host before launch.
template <typename T, int NCH, int CPL, int KH, int KW, bool UNIT>
__global__ void __launch_bounds__(256) bwd_kernel(Geo g, const T* __restrict__ x,
                                                  const T* __restrict__ om,
                                                  const T* __restrict__ gy,
                                                  float* __restrict__ gx32,
                                                  T* __restrict__ gom) {
  constexpr int L = NCH / CPL;
  constexpr int E = Elem<T>::E;
  constexpr int KC = KH * KW;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t bar;

  const long long p_first = (long long)blockIdx.x * g.ppc;
  const int npix = (int)min((long long)g.ppc, g.P - p_first);
  // shared memory: [om tile (+16 B slack)] [fp32 grad tile, ppc*S]
  const int om_bytes = ((g.ppc * g.S * (int)sizeof(T) + 16) + 15) & ~15;
  float* gtile = reinterpret_cast<float*>(smem + om_bytes);
  for (int e = threadIdx.x; e < npix * g.S; e += blockDim.x) gtile[e] = 0.f;
  const T* tile = stage_rows<T>(smem, &bar, om + p_first * g.S, npix * g.S);

  const int GL = g.G * L;
  const int t = threadIdx.x;
  const int pl0 = t / GL;
  const bool active = pl0 < npix;  // inactive lanes still take part in the shuffles
  const int pl = active ? pl0 : 0;
  const int rem = t - pl0 * GL;
  const int grp = rem / L;
  const int lg = rem - grp * L;
  const long long pix = p_first + pl;
  const int HWo = g.Ho * g.Wo;
  const int n = (int)(pix / HWo);
  const int hw = (int)(pix - (long long)n * HWo);
  const int ho = hw / g.Wo, wo = hw - (hw / g.Wo) * g.Wo;
  const int yb = ho * g.sh - g.ph + g.cy;
  const int xb = wo * g.sw - g.pw + g.cx;
  const long long img = (long long)n * g.H * g.W * g.C;
  const T* ximg = x + img;
  float* gximg = gx32 + img;
  const int K = KC ? KC : g.K;
  const T* row = tile + pl * g.S + grp * 3 * K;
  float* grow = gtile + pl * g.S + grp * 3 * K;
  const int cbase = grp * g.D + lg * CPL * E;

  float gyv[CPL * E];
  {
    const T* gyo = gy + pix * g.C + cbase;
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      uint4 u = make_uint4(0, 0, 0, 0);
      if (active) u = ldg16(gyo + h * E);
      Elem<T>::unpack(u, gyv + h * E);
    }
  }

  auto do_point = [&](int i, int j, int k, float m) {
    Corners c;
    corners<UNIT>(g, yb, xb, j * g.dh - g.cy, i * g.dw - g.cx, Elem<T>::f(row[2 * k]),
                  Elem<T>::f(row[2 * k + 1]), cbase, c);
    float sgm = 0.f, sgy = 0.f, sgx = 0.f;
    const float hy = 1.f - c.fy, hx = 1.f - c.fx;
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      float v[4][E];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = make_uint4(0, 0, 0, 0);
        if (active && c.ok[q]) u = ldg16(ximg + c.off[q] + h * E);
        Elem<T>::unpack(u, v[q]);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float gye = gyv[h * E + e];
        const float val = c.w[0] * v[0][e] + c.w[1] * v[1][e] + c.w[2] * v[2][e] + c.w[3] * v[3][e];
        const float dvy = hx * (v[2][e] - v[0][e]) + c.fx * (v[3][e] - v[1][e]);
        const float dvx = hy * (v[1][e] - v[0][e]) + c.fy * (v[3][e] - v[2][e]);
        sgm = fmaf(gye, val, sgm);
        sgy = fmaf(gye, dvy, sgy);
        sgx = fmaf(gye, dvx, sgx);
      }
      // bilinear scatter of m*w*gy into the in-bounds corners
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (active && c.ok[q]) {
          const float a = m * c.w[q];
          float* dst = gximg + c.off[q] + h * E;
#pragma unroll
          for (int e = 0; e < E; e += 4)
            red_add_v4(dst + e, a * gyv[h * E + e], a * gyv[h * E + e + 1],
                       a * gyv[h * E + e + 2], a * gyv[h * E + e + 3]);
        }
      }
    }
    // reduce the three partial dot products over the L lanes of this (pixel, group)
#pragma unroll
    for (int o = 1; o < L; o <<= 1) {
      sgm += __shfl_xor_sync(0xffffffffu, sgm, o);
      sgy += __shfl_xor_sync(0xffffffffu, sgy, o);
      sgx += __shfl_xor_sync(0xffffffffu, sgx, o);
    }
    if (active && lg == 0) {
      grow[2 * k] = g.s * m * sgx;      // d/d dx_k
      grow[2 * k + 1] = g.s * m * sgy;  // d/d dy_k
      grow[2 * K + k] = sgm;            // d/d m_k
    }
  };

  if constexpr (KC > 0) {
    float m[KC];
    load_m<T, KC>(row, KC, g.softmax, m);
#pragma unroll
    for (int i = 0; i < KW; ++i)
#pragma unroll
      for (int j = 0; j < KH; ++j) do_point(i, j, i * KH + j, m[i * KH + j]);
    if (g.softmax && active && lg == 0) {  // dL/dz_k = p_k (gm_k - sum_j p_j gm_j)
      float dot = 0.f;
#pragma unroll
      for (int k = 0; k < KC; ++k) dot += m[k] * grow[2 * KC + k];
#pragma unroll
      for (int k = 0; k < KC; ++k) grow[2 * KC + k] = m[k] * (grow[2 * KC + k] - dot);
    }
  } else {
    float mx = 0.f, inv = 1.f;
    if (g.softmax) softmax_stats<T>(row, K, mx, inv);
    for (int i = 0; i < g.kw; ++i)
      for (int j = 0; j < g.kh; ++j) {
        const int k = i * g.kh + j;
        float m = Elem<T>::f(row[2 * K + k]);
        if (g.softmax) m = __expf(m - mx) * inv;
        do_point(i, j, k, m);
      }
    if (g.softmax && active && lg == 0) {
      float dot = 0.f;
      for (int k = 0; k < K; ++k) dot += __expf(Elem<T>::f(row[2 * K + k]) - mx) * inv * grow[2 * K + k];
      for (int k = 0; k < K; ++k) {
        const float p = __expf(Elem<T>::f(row[2 * K + k]) - mx) * inv;
        grow[2 * K + k] = p * (grow[2 * K + k] - dot);
      }
    }
  }
  __syncthreads();
  // coalesced write of the CTA's grad_offset_mask rows (padding channels stay 0)
  T* gdst = gom + p_first * g.S;
  for (int e = threadIdx.x; e < npix * g.S; e += blockDim.x) gdst[e] = Elem<T>::from_f32(gtile[e]);
}

// fp32 accumulator -> grad_input in T (half dtypes only); n16 = number of 16-B T chunks.
template <typename T>
__global__ void __launch_bounds__(256) convert_kernel(const float* __restrict__ src,
                                                      T* __restrict__ dst, long long nchunk) {
  constexpr int E = Elem<T>::E;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nchunk;
       i += (long long)gridDim.x * blockDim.x) {
    float v[E];
    const float4* s4 = reinterpret_cast<const float4*>(src + i * E);
#pragma unroll
    for (int q = 0; q < E / 4; ++q) {
      float4 f = __ldcs(s4 + q);
      v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
    }
    reinterpret_cast<uint4*>(dst)[i] = Elem<T>::pack(v);
  }
}

}  // namespace dcnv4
