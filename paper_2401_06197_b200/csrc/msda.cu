// msda.cu -- multi-scale deformable attention on sm_100a: the C ABI of
// include/msda.h, validation, launch and the kernels for fp32 / fp16 / bf16.
//
// The operator (R20; PAPER.md P:143 names it, P:329 says the DCNv4 kernel
// techniques carry over):  out[n,q,m,:] = sum_{l,p} attn * V_l(phi_l(loc)),
// phi_l(x, y) = (x*W_l - 1/2, y*H_l - 1/2), bilinear with per-corner zero padding.
// B200 design, the DCNv4 gather-kernel techniques of P:318-329:
//   * work item = (n, q, m); L_ = D*sizeof(T)/16/CPL lanes share it, each lane owning CPL
//     16-B channel chunks, so one corner vector of an item is read by its lanes as whole
//     128-B lines (CPL = 1 for D*b <= 128 B) -- loc/attn and the bilinear coefficients are
//     computed once per (item, level, point) per lane and reused across its channels;
//   * corner gathers are 16-B read-only vector loads (value stays L2-resident: 20 MB per
//     image at the Deformable-DETR encoder shape), fp32 accumulation (FFMA2 / FHFMA);
//   * sampling coordinates split exactly into integer and fraction (x*W - 1/2 is exact in
//     fp64), so the fp32 fraction has relative error <= 2^-24 at any level size (R11 analog);
//   * backward: <gy, v_corner> dot products reduced over the L_ lanes with shuffles give
//     grad_attn / grad_loc; grad_value is a bilinear scatter of 16-B vector reductions
//     (red.global.add.v4.f32) into an fp32 accumulator.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/msda.h"
#include "ablation.h"
#include "dcnv4_kernels.cuh"

void dcnv4_internal_set_error(const char* msg);  // dcnv4_api.cu (not exported)

namespace msda {

using dcnv4::Elem;

struct MGeo {
  int Lq, M, D, L, P;
  int S;                     // value tokens per image
  int H[MSDA_MAX_LEVELS], W[MSDA_MAX_LEVELS], start[MSDA_MAX_LEVELS];
  long long items;           // N * Lq * M
  long long chunk;           // persistent schedule: slots per CTA per image (0 = flat launch)
  long long nimg;            // N
  int qfast;                 // slot order: 1 = queries fastest (see slot_item)
};

// One sample: the four corner element offsets (token*M*D, relative to the item's value
// base) and bilinear weights (0 for corners outside the level), plus fractions.
struct Corners {
  unsigned o[4];
  float w[4];
  float fh, fw;  // fractions
  float hh, hw;  // 1 - fractions (each rounded once from the exact fp64 value)
  bool ok[4];
};

// floor / fraction of v*n - 1/2 for v in fp32 and integer n.  v*n - 1/2 is exact in fp64
// (24 + 13 significant bits), so the fraction is the exact one rounded once to fp32: its
// RELATIVE error is <= 2^-24 even when it is tiny (a sample just inside the level edge
// whose only in-level corner carries weight ~fraction; an fp32 TwoProd split leaves an
// absolute 2^-25 there, i.e. 3e-5 relative at fraction 1e-3).
__device__ __forceinline__ void split_coord(float v, int n, int& i0, float& f, float& f1) {
  const double w = fma((double)v, (double)n, -0.5);
  const double fl = floor(w);
  i0 = (int)fl;
  f = (float)(w - fl);
  f1 = (float)((fl + 1.0) - w);  // 1 - fraction, also rounded once from the exact value
}

// a[l] for a runtime level l without dynamic indexing (which would copy the parameter
// arrays to local memory): a select chain over the MSDA_MAX_LEVELS entries
__device__ __forceinline__ int lvl(const int (&a)[MSDA_MAX_LEVELS], int l) {
  int v = a[0];
#pragma unroll
  for (int i = 1; i < MSDA_MAX_LEVELS; ++i) v = l == i ? a[i] : v;
  return v;
}

__device__ __forceinline__ void corners(const MGeo& g, int l, float x, float y, Corners& c) {
  const int H = lvl(g.H, l), W = lvl(g.W, l);
  const bool fin = fabsf(x) <= 4096.f && fabsf(y) <= 4096.f;  // NaN / huge: dropped
  int x0, y0;
  float fw, fh, hw, hh;
  split_coord(fin ? x : 0.f, W, x0, fw, hw);
  split_coord(fin ? y : 0.f, H, y0, fh, hh);
  c.fh = fh;
  c.fw = fw;
  c.hh = hh;
  c.hw = hw;
  const bool vy0 = fin && (unsigned)y0 < (unsigned)H, vy1 = fin && (unsigned)(y0 + 1) < (unsigned)H;
  const bool vx0 = fin && (unsigned)x0 < (unsigned)W, vx1 = fin && (unsigned)(x0 + 1) < (unsigned)W;
  c.ok[0] = vy0 && vx0;
  c.ok[1] = vy0 && vx1;
  c.ok[2] = vy1 && vx0;
  c.ok[3] = vy1 && vx1;
  const float w[4] = {hh * hw, hh * fw, fh * hw, fh * fw};
  const int ys[4] = {y0, y0, y0 + 1, y0 + 1}, xs[4] = {x0, x0 + 1, x0, x0 + 1};
  const unsigned MD = (unsigned)(g.M * g.D);
  const int st = lvl(g.start, l);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    c.w[q] = c.ok[q] ? w[q] : 0.f;
    c.o[q] = c.ok[q] ? (unsigned)(st + ys[q] * W + xs[q]) * MD : 0u;
  }
}

// The L*P sampling records (x, y, attn) of one item.  LP = L*P > 0 (compile time): read
// once with 16-B streaming loads (ld.global.cs: loc / attn are touched once, so they
// should not evict the L2-resident value tensor) and kept in registers; LP = 0: scalar
// loads at the point of use (any L*P, T-aligned pointers).
template <typename T, int LP>
struct ItemSamples {
  static constexpr int NLV = LP > 0 ? LP * 2 * (int)sizeof(T) / 16 : 1;
  static constexpr int NAV = LP > 0 ? LP * (int)sizeof(T) / 16 : 1;
  uint4 lv[NLV], av[NAV];
  const T* lp;
  const T* ap;
  __device__ __forceinline__ void load(const T* l, const T* a) {
    lp = l;
    ap = a;
    if constexpr (LP > 0) {
#pragma unroll
      for (int i = 0; i < NLV; ++i) lv[i] = __ldcs(reinterpret_cast<const uint4*>(l) + i);
#pragma unroll
      for (int i = 0; i < NAV; ++i) av[i] = __ldcs(reinterpret_cast<const uint4*>(a) + i);
    }
  }
  __device__ __forceinline__ float x(int i) const {
    if constexpr (LP > 0) return Elem<T>::f(reinterpret_cast<const T*>(lv)[2 * i]);
    else return Elem<T>::f(lp[2 * i]);
  }
  __device__ __forceinline__ float y(int i) const {
    if constexpr (LP > 0) return Elem<T>::f(reinterpret_cast<const T*>(lv)[2 * i + 1]);
    else return Elem<T>::f(lp[2 * i + 1]);
  }
  __device__ __forceinline__ float a(int i) const {
    if constexpr (LP > 0) return Elem<T>::f(reinterpret_cast<const T*>(av)[i]);
    else return Elem<T>::f(ap[i]);
  }
};

// Slot -> work item.  g.qfast = 0: items in memory order (n, q, m), heads fastest.
// g.qfast = 1: (n, m, q), queries fastest -- the 32 items of a 256-thread CTA are 32
// neighbouring queries of ONE head, whose samples land on neighbouring tokens of the same
// head's value slice (one 128-B line per (token, head) at D*b = 128 B), so the CTA's
// corner gathers share L1 lines.  Outputs stay whole 128-B lines per item.
__device__ __forceinline__ void slot_item(const MGeo& g, long long slot, long long& n, int& m,
                                          long long& item) {
  if (g.qfast) {
    const long long per = (long long)g.Lq * g.M;
    n = slot / per;
    const long long r = slot - n * per;
    m = (int)(r / g.Lq);
    const long long q = r - (long long)m * g.Lq;
    item = (n * g.Lq + q) * g.M + m;
  } else {
    item = slot;
    m = (int)(slot % g.M);
    n = slot / ((long long)g.M * g.Lq);
  }
}

template <typename T, int NCH, int CPL, int LP>
__global__ void __launch_bounds__(256) msda_fwd_kernel(MGeo g, const T* __restrict__ value,
                                                       const T* __restrict__ loc,
                                                       const T* __restrict__ attn,
                                                       T* __restrict__ out) {
  constexpr int LN = NCH / CPL;  // lanes per item
  constexpr int E = Elem<T>::E;
  const long long total = g.items * LN;
  const long long stride = (long long)gridDim.x * blockDim.x;
  auto body = [&](long long t) {
    const long long slot = t / LN;
    const int lg = (int)(t - slot * LN);
    int m;
    long long n, item;
    slot_item(g, slot, n, m, item);
    int co[CPL];
#pragma unroll
    for (int h = 0; h < CPL; ++h) co[h] = (h * LN + lg) * E;
    const T* vb = value + ((long long)n * g.S * g.M + m) * g.D;
    ItemSamples<T, LP> smp;
    smp.load(loc + item * g.L * g.P * 2, attn + item * g.L * g.P);
    float acc[CPL * E];
#pragma unroll
    for (int e = 0; e < CPL * E; ++e) acc[e] = 0.f;
    auto point = [&](int l, int i) {
      Corners c;
      corners(g, l, smp.x(i), smp.y(i), c);
      const float a = smp.a(i);
      uint4 u[4][CPL];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < CPL; ++h) u[q][h] = dcnv4::ldg16_idx<sizeof(T)>(vb + co[h], c.o[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < CPL; ++h) dcnv4::fma_chunk<T>(acc + h * E, a * c.w[q], u[q][h]);
    };
    if constexpr (LP > 0) {
#pragma unroll
      for (int i = 0; i < LP; ++i) point(i / g.P, i);
    } else {
      for (int l = 0; l < g.L; ++l) {
#pragma unroll 2
        for (int p = 0; p < g.P; ++p) point(l, l * g.P + p);
      }
    }
    T* o = out + item * g.D;
#pragma unroll
    for (int h = 0; h < CPL; ++h) __stcs(reinterpret_cast<uint4*>(o + co[h]), Elem<T>::pack(acc + h * E));
  };
  if (g.chunk == 0) {  // flat launch: one (item, lane) slot per thread, blocks in index order
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) body(t);
  } else {  // persistent: image by image, CTA b owns the contiguous slot range b of each image
    const long long per_img = total / g.nimg;
    const long long lo = (long long)blockIdx.x * g.chunk;
    const long long hi = lo + g.chunk < per_img ? lo + g.chunk : per_img;
    for (long long n = 0; n < g.nimg; ++n)
      for (long long b = lo + threadIdx.x; b < hi; b += blockDim.x) body(n * per_img + b);
  }
}

// Backward for fp16 / bf16 with 8-byte channel chunks (4 channels per lane): twice the
// lanes per (query, head) of the 16-B layout, so twice the threads in flight for the
// latency-bound gather / dot / vector-reduction chain, with the same bytes and the same
// number of 16-B fp32 reductions per corner (one per lane).  LN = D / 4 lanes per item.
template <typename T, int LN>
__global__ void __launch_bounds__(256) msda_bwd8_kernel(MGeo g, const T* __restrict__ value,
                                                        const T* __restrict__ loc,
                                                        const T* __restrict__ attn,
                                                        const T* __restrict__ gout,
                                                        float* __restrict__ gv32,
                                                        T* __restrict__ gloc,
                                                        T* __restrict__ gattn) {
  const long long total = g.items * LN;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (LN >= 32 ? 0xffffffffu : ((1u << LN) - 1u)) << (lane & ~(LN - 1));
  auto body = [&](long long t) {
    const long long slot = t / LN;
    const int lg = (int)(t - slot * LN);
    int m;
    long long n, item;
    slot_item(g, slot, n, m, item);
    const int co = lg * 4;
    const long long vbase = ((long long)n * g.S * g.M + m) * g.D;
    const T* vb = value + vbase + co;
    float* gb = gv32 + vbase + co;
    ItemSamples<T, 0> smp;
    smp.load(loc + item * g.L * g.P * 2, attn + item * g.L * g.P);
    const uint2 gu = __ldcs(reinterpret_cast<const uint2*>(gout + item * g.D + co));
    float gy[4];
    {
      const T* gh = reinterpret_cast<const T*>(&gu);
#pragma unroll
      for (int e = 0; e < 4; ++e) gy[e] = Elem<T>::f(gh[e]);
    }
    for (int l = 0; l < g.L; ++l) {
      const float Wl = (float)lvl(g.W, l), Hl = (float)lvl(g.H, l);
      for (int p = 0; p < g.P; ++p) {
        const int i = l * g.P + p;
        Corners c;
        corners(g, l, smp.x(i), smp.y(i), c);
        const float a = smp.a(i);
        uint2 u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = __ldg(reinterpret_cast<const uint2*>(vb + c.o[q]));
        float S[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const T* xh = reinterpret_cast<const T*>(&u[q]);
          float s0 = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) s0 = fmaf(gy[e], Elem<T>::f(xh[e]), s0);
          S[q] = c.ok[q] ? s0 : 0.f;
        }
        const float hh = c.hh, hw = c.hw;
        float sa = hh * hw * S[0] + hh * c.fw * S[1] + c.fh * hw * S[2] + c.fh * c.fw * S[3];
        float sw = hh * (S[1] - S[0]) + c.fh * (S[3] - S[2]);  // d/dw
        float sh = hw * (S[2] - S[0]) + c.fw * (S[3] - S[1]);  // d/dh
#pragma unroll
        for (int o = 1; o < LN; o <<= 1) {
          sa += __shfl_xor_sync(gmask, sa, o);
          sw += __shfl_xor_sync(gmask, sw, o);
          sh += __shfl_xor_sync(gmask, sh, o);
        }
        if (lg == 0) {
          gattn[item * g.L * g.P + i] = Elem<T>::from_f32(sa);
          gloc[(item * g.L * g.P + i) * 2] = Elem<T>::from_f32(a * Wl * sw);
          gloc[(item * g.L * g.P + i) * 2 + 1] = Elem<T>::from_f32(a * Hl * sh);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float aw = a * c.w[q];
          if (aw != 0.f) dcnv4::red_add_v4_idx(gb, c.o[q], aw * gy[0], aw * gy[1], aw * gy[2], aw * gy[3]);
        }
      }
    }
  };
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) body(t);
}

template <typename T, int NCH, int CPL, int LP>
__global__ void __launch_bounds__(256) msda_bwd_kernel(MGeo g, const T* __restrict__ value,
                                                       const T* __restrict__ loc,
                                                       const T* __restrict__ attn,
                                                       const T* __restrict__ gout,
                                                       float* __restrict__ gv32,
                                                       T* __restrict__ gloc,
                                                       T* __restrict__ gattn) {
  constexpr int LN = NCH / CPL;
  constexpr int E = Elem<T>::E;
  const long long total = g.items * LN;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = (LN >= 32 ? 0xffffffffu : ((1u << LN) - 1u)) << (lane & ~(LN - 1));
  auto body = [&](long long t) {
    const long long slot = t / LN;
    const int lg = (int)(t - slot * LN);
    int m;
    long long n, item;
    slot_item(g, slot, n, m, item);
    int co[CPL];
#pragma unroll
    for (int h = 0; h < CPL; ++h) co[h] = (h * LN + lg) * E;
    const long long vbase = ((long long)n * g.S * g.M + m) * g.D;
    const T* vb = value + vbase;
    float* gb = gv32 + vbase;
    ItemSamples<T, LP> smp;
    smp.load(loc + item * g.L * g.P * 2, attn + item * g.L * g.P);
    uint4 gyu[CPL];
    float gyv[CPL * E];
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      gyu[h] = dcnv4::ld_stream(reinterpret_cast<const uint4*>(gout + item * g.D + co[h]));
      Elem<T>::unpack(gyu[h], gyv + h * E);
    }
    auto point = [&](int l, int i) {
        const float Wl = (float)lvl(g.W, l), Hl = (float)lvl(g.H, l);
        Corners c;
        corners(g, l, smp.x(i), smp.y(i), c);
        const float a = smp.a(i);
        float S[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int h = 0; h < CPL; ++h)
            dcnv4::dot_chunk<T>(s2, gyu[h], dcnv4::ldg16_idx<sizeof(T)>(vb + co[h], c.o[q]));
          S[q] = c.ok[q] ? s2.x + s2.y : 0.f;
        }
        const float hh = c.hh, hw = c.hw;
        float sa = hh * hw * S[0] + hh * c.fw * S[1] + c.fh * hw * S[2] + c.fh * c.fw * S[3];
        float sw = hh * (S[1] - S[0]) + c.fh * (S[3] - S[2]);  // d/dw
        float sh = hw * (S[2] - S[0]) + c.fw * (S[3] - S[1]);  // d/dh
#pragma unroll
        for (int o = 1; o < LN; o <<= 1) {
          sa += __shfl_xor_sync(gmask, sa, o);
          sw += __shfl_xor_sync(gmask, sw, o);
          sh += __shfl_xor_sync(gmask, sh, o);
        }
        if (lg == 0) {
          gattn[item * g.L * g.P + i] = Elem<T>::from_f32(sa);
          gloc[(item * g.L * g.P + i) * 2] = Elem<T>::from_f32(a * Wl * sw);
          gloc[(item * g.L * g.P + i) * 2 + 1] = Elem<T>::from_f32(a * Hl * sh);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float aw = a * c.w[q];
          if (aw != 0.f) {
#pragma unroll
            for (int h = 0; h < CPL; ++h)
#pragma unroll
              for (int e = 0; e < E; e += 4)
                dcnv4::red_add_v4_idx(gb + co[h] + e, c.o[q], aw * gyv[h * E + e], aw * gyv[h * E + e + 1],
                                      aw * gyv[h * E + e + 2], aw * gyv[h * E + e + 3]);
          }
        }
    };
    if constexpr (LP > 0) {
#pragma unroll
      for (int i = 0; i < LP; ++i) point(i / g.P, i);
    } else {
      for (int l = 0; l < g.L; ++l)
        for (int p = 0; p < g.P; ++p) point(l, l * g.P + p);
    }
  };
  if (g.chunk == 0) {  // flat launch: one (item, lane) slot per thread, blocks in index order
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) body(t);
  } else {  // persistent: image by image, CTA b owns the contiguous slot range b of each image
    const long long per_img = total / g.nimg;
    const long long lo = (long long)blockIdx.x * g.chunk;
    const long long hi = lo + g.chunk < per_img ? lo + g.chunk : per_img;
    for (long long n = 0; n < g.nimg; ++n)
      for (long long b = lo + threadIdx.x; b < hi; b += blockDim.x) body(n * per_img + b);
  }
}

namespace {

// errors go to the library's one thread-local message (dcnv4_last_error)
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  dcnv4_internal_set_error(buf);
  return code;
}

int esize(int dtype) { return dtype == DCNV4_F32 ? 4 : 2; }

int validate(const msda_params* p, int dtype, long long* S) {
  dcnv4_internal_set_error("");
  if (!p) return fail(DCNV4_ERR_INVALID_ARG, "params is NULL");
  if (dtype != DCNV4_F32 && dtype != DCNV4_F16 && dtype != DCNV4_BF16)
    return fail(DCNV4_ERR_INVALID_ARG, "dtype %d is not DCNV4_F32/F16/BF16", dtype);
  if (p->N < 0) return fail(DCNV4_ERR_INVALID_ARG, "N = %lld < 0", (long long)p->N);
  if (p->Lq < 0) return fail(DCNV4_ERR_INVALID_ARG, "Lq = %lld < 0", (long long)p->Lq);
  if (p->M <= 0) return fail(DCNV4_ERR_INVALID_ARG, "M = %d <= 0 (heads axis)", p->M);
  if (p->D <= 0) return fail(DCNV4_ERR_INVALID_ARG, "D = %d <= 0 (channel axis)", p->D);
  if (p->P <= 0) return fail(DCNV4_ERR_INVALID_ARG, "P = %d <= 0 (points axis)", p->P);
  if (p->L <= 0 || p->L > MSDA_MAX_LEVELS)
    return fail(DCNV4_ERR_INVALID_ARG, "L = %d outside [1, %d] (levels axis)", p->L, MSDA_MAX_LEVELS);
  long long s = 0;
  for (int l = 0; l < p->L; ++l) {
    if (p->H[l] <= 0 || p->W[l] <= 0)
      return fail(DCNV4_ERR_INVALID_ARG, "level %d shape %dx%d must be positive", l, p->H[l], p->W[l]);
    if (p->H[l] > 4096 || p->W[l] > 4096)
      return fail(DCNV4_ERR_SHAPE, "level %d shape %dx%d exceeds 4096", l, p->H[l], p->W[l]);
    s += (long long)p->H[l] * p->W[l];
  }
  *S = s;
  const long long lim = 1LL << 31;
  if (s * p->M * p->D >= lim) return fail(DCNV4_ERR_SHAPE, "per-image value S*M*D must be < 2^31");
  if (p->Lq * p->M * (long long)p->L * p->P * 2 >= lim)
    return fail(DCNV4_ERR_SHAPE, "per-image loc Lq*M*L*P*2 must be < 2^31");
  const int b = esize(dtype);
  if (((long long)p->D * b) % 16 || (long long)p->D * b > 256)
    return fail(DCNV4_ERR_UNSUPPORTED, "D*sizeof(dtype) = %lld bytes must be a multiple of 16 and <= 256",
                (long long)p->D * b);
  const int nch = p->D * b / 16;
  if (nch & (nch - 1))
    return fail(DCNV4_ERR_UNSUPPORTED, "D*sizeof(dtype) = %d bytes is not 16 B times a power of two",
                p->D * b);
  return DCNV4_OK;
}

MGeo make_geo(const msda_params* p, long long S) {
  MGeo g;
  g.Lq = (int)p->Lq; g.M = p->M; g.D = p->D; g.L = p->L; g.P = p->P; g.S = (int)S;
  int st = 0;
  for (int l = 0; l < MSDA_MAX_LEVELS; ++l) {
    g.H[l] = l < p->L ? p->H[l] : 1;
    g.W[l] = l < p->L ? p->W[l] : 1;
    g.start[l] = st;
    if (l < p->L) st += p->H[l] * p->W[l];
  }
  g.items = p->N * p->Lq * p->M;
  g.chunk = 0;
  g.nimg = p->N;
  const char* ord = dcnv4::ablation(dcnv4::kAblMsdaOrder);
  g.qfast = (ord && ord[0] == 'q') ? 1 : 0;  // ablation only: measured no better
  return g;
}

// chunks per lane: whole 128-B corner lines per item when possible (env MSDA_CPL overrides)
int pick_cpl(int nch) {
  int cpl = nch <= 8 ? 1 : nch / 8;
  const char* env = dcnv4::ablation(dcnv4::kAblMsdaCpl);
  if (env && *env) {
    const int v = atoi(env);
    if (v >= 1 && v <= nch && (v & (v - 1)) == 0 && nch / v <= 32) cpl = v;
  }
  return cpl;
}

// One thread per (item, lane) slot: blocks are dispatched in index order, so the
// resident CTAs sweep the images in order and each image's value tensor (20 MB at the
// Deformable-DETR shape) is read from HBM about once and then hit in L2 by all four
// query-level segments of the image.  (A capped grid-stride launch keeps eight images in
// flight and re-reads value from HBM: 2.8x the algorithmic bytes.)  MSDA_GRID_CAP=1
// restores the capped launch (ablation).
unsigned grid_for(long long threads) {
  long long b = (threads + 255) / 256;
  const char* env = dcnv4::ablation(dcnv4::kAblMsdaGridCap);
  const long long cap = (env && *env == '1') ? 148LL * 8 * 4 : 0x7fffffffLL;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

// Launch `k` over thr (item, lane) slots.  MSDA_SCHED=persist (ablation): a resident grid
// (SMs x occupancy) sweeping the images in order, CTA b owning the contiguous slot range b
// of every image (spatially adjacent queries on one SM share L1 lines); default: the flat
// launch (grid_for).
template <typename K, typename... A>
cudaError_t launch_sched(K k, MGeo g, long long thr, cudaStream_t st, A... args) {
  const char* env = dcnv4::ablation(dcnv4::kAblMsdaSched);
  unsigned grid;
  g.chunk = 0;
  g.nimg = 1;
  if (env && env[0] == 'p' && g.items > 0) {
    int dev = 0, sms = 148, per_sm = 1;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
    g.nimg = g.items / ((long long)g.Lq * g.M);
    const long long per_img = thr / g.nimg;
    const long long ctas = (long long)sms * per_sm;
    long long chunk = (per_img + ctas - 1) / ctas;
    chunk = (chunk + 255) / 256 * 256;
    g.chunk = chunk;
    grid = (unsigned)((per_img + chunk - 1) / chunk);
  } else {
    grid = grid_for(thr);
  }
  k<<<grid, 256, 0, st>>>(g, args...);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fwd(const MGeo& g, int nch, int cpl, const void* v, const void* lo,
                       const void* at, void* out, cudaStream_t st) {
  // vectorised sample records (L*P = 16, 16-B aligned loc / attn): opt-in, MSDA_VEC=1 --
  // measured slower than scalar loads (f32 fwd 757 -> 965 us: 80-90 registers)
  const bool v16 = g.L * g.P == 16 && ((reinterpret_cast<uintptr_t>(lo) | reinterpret_cast<uintptr_t>(at)) & 15) == 0 &&
                   (*dcnv4::ablation(dcnv4::kAblMsdaVec) == '1');
  const T* vp = static_cast<const T*>(v);
  const T* lp = static_cast<const T*>(lo);
  const T* ap = static_cast<const T*>(at);
  T* op = static_cast<T*>(out);
  const long long thr = g.items * (nch / cpl);
#define MSDA_FWD(NC, CP)                                                                  \
  case NC * 100 + CP:                                                                     \
    return v16 ? launch_sched(msda_fwd_kernel<T, NC, CP, 16>, g, thr, st, vp, lp, ap, op)  \
               : launch_sched(msda_fwd_kernel<T, NC, CP, 0>, g, thr, st, vp, lp, ap, op);
  switch (nch * 100 + cpl) {
    MSDA_FWD(1, 1) MSDA_FWD(2, 1) MSDA_FWD(2, 2) MSDA_FWD(4, 1) MSDA_FWD(4, 2) MSDA_FWD(4, 4)
    MSDA_FWD(8, 1) MSDA_FWD(8, 2) MSDA_FWD(8, 4) MSDA_FWD(16, 1) MSDA_FWD(16, 2) MSDA_FWD(16, 4)
    default: return cudaErrorInvalidConfiguration;
  }
#undef MSDA_FWD
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_bwd(const MGeo& g, int nch, int cpl, const void* v, const void* lo,
                       const void* at, const void* go, float* gv, void* gl, void* ga,
                       cudaStream_t st) {
  const T* vp = static_cast<const T*>(v);
  const T* lp = static_cast<const T*>(lo);
  const T* ap = static_cast<const T*>(at);
  const T* gp = static_cast<const T*>(go);
  T* glp = static_cast<T*>(gl);
  T* gap = static_cast<T*>(ga);
  if (sizeof(T) == 2 && *dcnv4::ablation(dcnv4::kAblMsdaBwd8) != '0') {
    const long long thr8 = g.items * (g.D / 4);
    switch (g.D / 4) {
      case 4: return launch_sched(msda_bwd8_kernel<T, 4>, g, thr8, st, vp, lp, ap, gp, gv, glp, gap);
      case 8: return launch_sched(msda_bwd8_kernel<T, 8>, g, thr8, st, vp, lp, ap, gp, gv, glp, gap);
      case 16: return launch_sched(msda_bwd8_kernel<T, 16>, g, thr8, st, vp, lp, ap, gp, gv, glp, gap);
      case 32: return launch_sched(msda_bwd8_kernel<T, 32>, g, thr8, st, vp, lp, ap, gp, gv, glp, gap);
      default: break;
    }
  }
  const long long thr = g.items * (nch / cpl);
  const bool v16 = g.L * g.P == 16 && ((reinterpret_cast<uintptr_t>(lo) | reinterpret_cast<uintptr_t>(at)) & 15) == 0 &&
                   (*dcnv4::ablation(dcnv4::kAblMsdaVec) == '1');
#define MSDA_BWD(NC, CP)                                                                          \
  case NC * 100 + CP:                                                                             \
    return v16 ? launch_sched(msda_bwd_kernel<T, NC, CP, 16>, g, thr, st, vp, lp, ap, gp, gv, glp, gap) \
               : launch_sched(msda_bwd_kernel<T, NC, CP, 0>, g, thr, st, vp, lp, ap, gp, gv, glp, gap);
  switch (nch * 100 + cpl) {
    MSDA_BWD(1, 1) MSDA_BWD(2, 1) MSDA_BWD(2, 2) MSDA_BWD(4, 1) MSDA_BWD(4, 2) MSDA_BWD(4, 4)
    MSDA_BWD(8, 1) MSDA_BWD(8, 2) MSDA_BWD(8, 4) MSDA_BWD(16, 1) MSDA_BWD(16, 2) MSDA_BWD(16, 4)
    default: return cudaErrorInvalidConfiguration;
  }
#undef MSDA_BWD
  return cudaGetLastError();
}

template <typename T>
__global__ void __launch_bounds__(256) convert(const float* __restrict__ src, T* __restrict__ dst,
                                               long long nchunk) {
  constexpr int E = Elem<T>::E;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nchunk;
       i += (long long)gridDim.x * blockDim.x) {
    float v[E];
    const float4* s4 = reinterpret_cast<const float4*>(src + i * E);
#pragma unroll
    for (int q = 0; q < E / 4; ++q) {
      const float4 f = __ldcs(s4 + q);
      v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
    }
    reinterpret_cast<uint4*>(dst)[i] = Elem<T>::pack(v);
  }
}

bool al16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

}  // namespace
}  // namespace msda

using namespace msda;

extern "C" {

int msda_value_tokens(const msda_params* p, int64_t* S) {
  long long s = 0;
  if (!S) return fail(DCNV4_ERR_INVALID_ARG, "S is NULL");
  const int rc = validate(p, DCNV4_F32, &s);
  if (rc && rc != DCNV4_ERR_UNSUPPORTED) return rc;
  *S = s;
  return DCNV4_OK;
}

int msda_forward(const msda_params* p, dcnv4_dtype dtype, const void* value, const void* loc,
                 const void* attn, void* out, void* stream) {
  long long S = 0;
  int rc = validate(p, dtype, &S);
  if (rc) return rc;
  if (p->N * p->Lq == 0) return DCNV4_OK;
  if (!value || !loc || !attn || !out)
    return fail(DCNV4_ERR_INVALID_ARG, "%s is NULL", !value ? "value" : !loc ? "loc" : !attn ? "attn" : "out");
  if (!al16(value) || !al16(out)) return fail(DCNV4_ERR_MISALIGNED, "value / out must be 16-byte aligned");
  const int b = esize(dtype);
  if (reinterpret_cast<uintptr_t>(loc) % b || reinterpret_cast<uintptr_t>(attn) % b)
    return fail(DCNV4_ERR_MISALIGNED, "loc / attn are not element aligned");
  const MGeo g = make_geo(p, S);
  const int nch = p->D * b / 16, cpl = pick_cpl(nch);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (dtype) {
    case DCNV4_F32: e = launch_fwd<float>(g, nch, cpl, value, loc, attn, out, st); break;
    case DCNV4_F16: e = launch_fwd<__half>(g, nch, cpl, value, loc, attn, out, st); break;
    default: e = launch_fwd<__nv_bfloat16>(g, nch, cpl, value, loc, attn, out, st); break;
  }
  if (e != cudaSuccess) return fail(DCNV4_ERR_CUDA, "msda_forward launch: %s", cudaGetErrorString(e));
  return DCNV4_OK;
}

size_t msda_backward_workspace_bytes(const msda_params* p, dcnv4_dtype dtype) {
  long long S = 0;
  if (validate(p, dtype, &S)) return 0;
  if (dtype == DCNV4_F32) return 0;
  return (size_t)p->N * S * p->M * p->D * sizeof(float);
}

int msda_backward(const msda_params* p, dcnv4_dtype dtype, const void* value, const void* loc,
                  const void* attn, const void* grad_out, void* grad_value, void* grad_loc,
                  void* grad_attn, void* workspace, size_t workspace_bytes, void* stream) {
  long long S = 0;
  int rc = validate(p, dtype, &S);
  if (rc) return rc;
  const size_t nval = (size_t)p->N * S * p->M * p->D;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->N * p->Lq == 0) {  // no queries: grad_value is zero
    if (p->N && grad_value) {
      cudaError_t e = cudaMemsetAsync(grad_value, 0, nval * esize(dtype), st);
      if (e != cudaSuccess) return fail(DCNV4_ERR_CUDA, "msda_backward zero: %s", cudaGetErrorString(e));
    }
    return DCNV4_OK;
  }
  if (!value || !loc || !attn || !grad_out || !grad_value || !grad_loc || !grad_attn)
    return fail(DCNV4_ERR_INVALID_ARG, "a tensor argument is NULL");
  if (!al16(value) || !al16(grad_out) || !al16(grad_value))
    return fail(DCNV4_ERR_MISALIGNED, "value / grad_out / grad_value must be 16-byte aligned");
  const int b = esize(dtype);
  if (reinterpret_cast<uintptr_t>(loc) % b || reinterpret_cast<uintptr_t>(attn) % b ||
      reinterpret_cast<uintptr_t>(grad_loc) % b || reinterpret_cast<uintptr_t>(grad_attn) % b)
    return fail(DCNV4_ERR_MISALIGNED, "loc / attn / grad_loc / grad_attn are not element aligned");
  const size_t need = msda_backward_workspace_bytes(p, dtype);
  if (need && (!workspace || workspace_bytes < need))
    return fail(DCNV4_ERR_WORKSPACE, "workspace of %zu bytes required, got %zu", need,
                workspace ? workspace_bytes : (size_t)0);
  if (need && !al16(workspace)) return fail(DCNV4_ERR_MISALIGNED, "workspace is not 16-byte aligned");
  const MGeo g = make_geo(p, S);
  const int nch = p->D * b / 16, cpl = pick_cpl(nch);
  float* gv32 = dtype == DCNV4_F32 ? static_cast<float*>(grad_value) : static_cast<float*>(workspace);
  cudaError_t e = cudaMemsetAsync(gv32, 0, nval * sizeof(float), st);
  if (e != cudaSuccess) return fail(DCNV4_ERR_CUDA, "msda_backward zero: %s", cudaGetErrorString(e));
  switch (dtype) {
    case DCNV4_F32: e = launch_bwd<float>(g, nch, cpl, value, loc, attn, grad_out, gv32, grad_loc, grad_attn, st); break;
    case DCNV4_F16: e = launch_bwd<__half>(g, nch, cpl, value, loc, attn, grad_out, gv32, grad_loc, grad_attn, st); break;
    default: e = launch_bwd<__nv_bfloat16>(g, nch, cpl, value, loc, attn, grad_out, gv32, grad_loc, grad_attn, st); break;
  }
  if (e != cudaSuccess) return fail(DCNV4_ERR_CUDA, "msda_backward launch: %s", cudaGetErrorString(e));
  if (dtype != DCNV4_F32) {
    const long long nchunk = (long long)(nval / 8);
    const unsigned grid = grid_for(nchunk);
    if (dtype == DCNV4_F16)
      convert<__half><<<grid, 256, 0, st>>>(gv32, static_cast<__half*>(grad_value), nchunk);
    else
      convert<__nv_bfloat16><<<grid, 256, 0, st>>>(gv32, static_cast<__nv_bfloat16*>(grad_value), nchunk);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(DCNV4_ERR_CUDA, "msda_backward convert: %s", cudaGetErrorString(e));
  }
  return DCNV4_OK;
}

}  // extern "C"
