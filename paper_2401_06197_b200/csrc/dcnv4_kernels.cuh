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
//   * CTA = a 2-D tile of output pixels x a run of Gc groups of one image, so the
//     CTA's corner footprint (tile + 7-pixel halo) stays L1-resident and x is fetched
//     from L2 ~2-3x instead of ~17x (ncu, profiles/r01_v1_*);
//   * persistent CTAs: the next tile's offset_mask segments are copied into a second
//     shared-memory buffer with cp.async while the current tile is computed;
//   * lanes are ordered (pixel, group, lane) and each lane's chunk order is rotated so
//     the eight lanes of a 128-bit load phase hit eight distinct bank quads (microbench:
//     115 vs 57-81 B/clk/SM, profiles/r01_microbench_l1_red.jsonl);
//   * corner gathers are 16-byte read-only vector loads (LDG.E.128.CONSTANT), predicated
//     off outside the image ("128-bit packed value");
//   * fp32 accumulation for every storage type, RN-even store (P:329 half precision);
//   * backward: grad_offset/grad_mask partials reduced across the L lanes with warp
//     shuffles, staged in shared memory and written coalesced; grad_input is a bilinear
//     scatter with 16-byte vector reductions (red.global.add.v4.f32) into fp32.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

// Compile-time experiment knobs (scripts/build_variant.py builds A/B libraries with -D;
// never set in the product build).
// bwd33 P4 pair-loop unroll depth (fp32 1, half 2: measured best of 1/2/4/8, c4 step
// 4651 / 4706 / 4803 / 4966 us, c5 1454 / 1450 / 1463 / 1481 us;
// profiles/r02_bwd_p4_unroll.jsonl), and two accumulator sets (even / odd entries)
#ifndef DCNV4_P4_UNROLL
#define DCNV4_P4_UNROLL (sizeof(T) == 4 ? 1 : 2)
#endif
#ifndef DCNV4_P4_ACC2
#define DCNV4_P4_ACC2 0
#endif
// fwd33 software-pipeline depth (gathers issued DEPTH-1 samples ahead of their FMAs; 2 is
// best: depth 3 / 4 are 1-4% slower on c4 fp32 and c2/c3 fp16, profiles/r02_fwd_pipe_depth.jsonl)
#ifndef DCNV4_FWD_PIPE
#define DCNV4_FWD_PIPE 2
#endif
// bwd33 P4: 16-B chunks per pull lane (NCH / PC lanes per (halo pixel, group))
#ifndef DCNV4_P4_PC
#define DCNV4_P4_PC (NCH >= 2 ? 2 : 1)
#endif
// bwd33 P1 (count) loop unroll depth
#ifndef DCNV4_P1_UNROLL
#define DCNV4_P1_UNROLL 1
#endif
// DCNV4_BWD_ABL: timing-only phase ablation of bwd33 (wrong results): bit 0 skips the P4
// pull, bit 1 the P3 corner gathers and dots, bit 2 the P1 count, P3 filing and P4 pull,
// bit 3 the P3 grad_offset_mask stores (profiles/r02_bwd_blockpull_rejected.jsonl).
#ifndef DCNV4_BWD_ABL
#define DCNV4_BWD_ABL 0
#endif

namespace dcnv4 {

// Geometry handed to every kernel by value (validated on the host; per-image element
// counts fit in int32).
// Division by a runtime constant d for n < 2^31: q = (umulhi(n, m) + n) >> l
// (m = ceil(2^(32+l)/d) - 2^32, l = ceil(log2 d); set up on the host).
struct FastDiv {
  unsigned m, l;
};
__device__ __forceinline__ unsigned fdiv(unsigned n, FastDiv f) { return (__umulhi(n, f.m) + n) >> f.l; }

struct Geo {
  int H, W, Ho, Wo, G, D, C, S, K;
  int kh, kw, sh, sw, ph, pw, dh, dw, cy, cx;
  float s;
  int softmax;
  // CTA tiling (chosen on the host, see dcnv4_api.cu make_launch)
  int TH, TW, Gc;                  // output-pixel tile and groups per CTA
  int tiles_h, tiles_w, gblocks;   // grid = N * tiles_h * tiles_w * gblocks
  int rot_shift;                   // chunk-order stagger: rot = (pg_in_warp >> s) & (CPL-1)
  int seg;                         // shared-memory elements per tile pixel (om segment)
  int tiles_total;                 // N * tiles_h * tiles_w * gblocks (< 2^31)
  // TMA halo path (forward): halo box = HH x HW pixels x Gc*D channels
  int HH, HW;                      // halo rows / cols
  int halo_bytes;                  // shared-memory bytes per halo buffer (128-B multiple)
  int halo_box_bytes;              // bytes one TMA box delivers
  int upp, unit;                   // om staging: units per tile pixel, unit bytes (8 or 4)
  FastDiv fd_gb, fd_tw, fd_th, fd_upp;
  // backward (bwd33) shared-memory carve-up (byte offsets) and TMA box of the gy tile
  int gy_box_bytes;
  int o_gy, o_om, o_gom, o_cnt, o_slot, o_ent, o_wsum, o_bar;
  // deterministic grad_input (params.deterministic): ceil(log2(Ho*Wo*K)) and the
  // per-image maxima {max|gy|, max|m|} (float bits) written by det_scale_kernel
  int det_lc;
  int ent_cap;  // bwd33: bin-entry capacity of the tile (fp32 keeps a and src in two arrays)
  const unsigned* detmax;
  // bwd33 P4: halo bins in descending order of their expected entry count (so the lanes of
  // a warp get bins of similar size and wait less on each other); identity if disabled
  unsigned char p4ord[200];
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
  __device__ __forceinline__ static unsigned short bits(float) { return 0; }  // unused (8-B entries)
  __device__ __forceinline__ static float from_bits(unsigned short) { return 0.f; }
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
  __device__ __forceinline__ static unsigned short bits(float v) { return __half_as_ushort(__float2half_rn(v)); }
  __device__ __forceinline__ static float from_bits(unsigned short b) { return __half2float(__ushort_as_half(b)); }
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
  __device__ __forceinline__ static unsigned short bits(float v) { return __bfloat16_as_ushort(__float2bfloat16_rn(v)); }
  __device__ __forceinline__ static float from_bits(unsigned short b) { return __uint_as_float((unsigned)b << 16); }
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint4 ldg16(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// 16-B read-only gather at base + idx*ES (one IMAD.WIDE.U32 for the address: idx is a
// 32-bit element index inside one image, base a per-thread 64-bit pointer).
template <int ES>
__device__ __forceinline__ uint4 ldg16_idx(const void* base, unsigned idx) {
  uint4 r;
  asm("{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %4, %6, %5;\n\t"
      "ld.global.nc.v4.u32 {%0, %1, %2, %3}, [a];\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "r"(idx), "l"(base), "n"(ES));
  return r;
}

// 16-B vector reduction into fp32 at base + idx*4.
__device__ __forceinline__ void red_add_v4_idx(float* base, unsigned idx, float a, float b, float c,
                                               float d) {
  asm volatile("{\n\t.reg .u64 p;\n\tmad.wide.u32 p, %0, 4, %1;\n\t"
               "red.global.add.v4.f32 [p], {%2, %3, %4, %5};\n\t}" ::"r"(idx), "l"(base), "f"(a),
               "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}


// ------------------------------------------------------------------ deterministic grad_input
// DESIGN.md R19.  Every contribution m*w*gy_c of image n is rounded once to the integer
// grid 2^-F_n and summed in int64 (shared-memory bins and global reductions alike), so
// the sum is independent of the order the atomics land in.  F_n is fixed per image from
// M_g = max|gy|, M_m = max|m| and lc = ceil(log2(Ho*Wo*K)) (an input element receives at
// most Ho*Wo*K contributions, each < 2^eg * 2^em):  F = 62 - lc - eg - em, so every
// partial sum stays below 2^62.  Images whose maxima are non-finite or outside
// [2^-64, 2^64) are flagged and their grad_input is written as NaN.
struct DetScale {
  float s1, s2;  // 2^F = s1 * s2 (each a normal float)
  int F;
  bool bad;
};

__device__ __forceinline__ int det_exp(unsigned bits) {  // smallest e with |v| < 2^e
  const int E = (int)(bits >> 23);
  return (E < 1 ? 1 : E) - 126;
}

__device__ __forceinline__ DetScale det_scale(const unsigned* mx, int n, int lc) {
  DetScale d = {0.f, 0.f, 0, false};
  const unsigned gb = mx[2 * n], mb = mx[2 * n + 1];
  if (gb >= 0x7f800000u || mb >= 0x7f800000u) { d.bad = true; return d; }
  if (gb == 0u || mb == 0u) return d;  // every contribution is exactly 0
  const int eg = det_exp(gb), em = det_exp(mb);
  if (eg < -63 || eg > 64 || em < -63 || em > 64) { d.bad = true; return d; }
  d.F = 62 - lc - eg - em;  // in [-66 - lc, 188 - lc]
  const int F1 = d.F / 2, F2 = d.F - F1;
  d.s1 = __int_as_float((F1 + 127) << 23);
  d.s2 = __int_as_float((F2 + 127) << 23);
  return d;
}

// 64-bit integer reduction (RED.E.ADD.64): order-independent
__device__ __forceinline__ void red_add_s64(long long* p, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Asynchronous global -> shared copies (LDGSTS): the CTA's next offset_mask tile is
// fetched while the current one is computed.
template <int B>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  if constexpr (B == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(B) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ------------------------------------------------------------------ tiles
// A tile = one image n, a TH x TW block of output pixels and a run of Gc groups from g0.
// Tile index = ((n * tiles_h + th) * tiles_w + tw) * gblocks + gb.  The grid is
// persistent: CTA b processes tiles b, b + gridDim.x, ...
struct Tile {
  int n, h0, w0, g0;
};

__device__ __forceinline__ Tile decode_tile(const Geo& g, int t) {
  Tile r;
  const int gb = t % g.gblocks; t /= g.gblocks;
  const int tw = t % g.tiles_w; t /= g.tiles_w;
  const int th = t % g.tiles_h;
  r.n = t / g.tiles_h;
  r.h0 = th * g.TH;
  r.w0 = tw * g.TW;
  r.g0 = gb * g.Gc;
  return r;
}

// Issue the copies of one tile's offset_mask rows into `buf`: per tile pixel the Gc*3K
// contiguous values of groups [g0, g0+Gc), one segment per pixel (g.seg elements apart,
// 16-B aligned).  One warp per pixel segment, widest unit the source alignment allows.
template <typename T>
__device__ __forceinline__ void stage_tile(const Geo& g, int t, const T* __restrict__ om,
                                           T* buf) {
  const Tile tl = decode_tile(g, t);
  const int nbytes = g.Gc * 3 * g.K * (int)sizeof(T);
  const int npix = g.TH * g.TW;
  const int lane = threadIdx.x & 31;
  for (int p = threadIdx.x >> 5; p < npix; p += blockDim.x >> 5) {
    const int ho = tl.h0 + p / g.TW, wo = tl.w0 + p % g.TW;
    if (ho >= g.Ho || wo >= g.Wo) continue;
    const char* src = reinterpret_cast<const char*>(
        om + ((long long)(tl.n * g.Ho + ho) * g.Wo + wo) * g.S + tl.g0 * 3 * g.K);
    char* dst = reinterpret_cast<char*>(buf + p * g.seg);
    const unsigned a = (unsigned)reinterpret_cast<uintptr_t>(src) | (unsigned)nbytes;
    if ((a & 15) == 0) {
      for (int i = lane * 16; i < nbytes; i += 512) cp_async<16>(dst + i, src + i);
    } else if ((a & 7) == 0) {
      for (int i = lane * 8; i < nbytes; i += 256) cp_async<8>(dst + i, src + i);
    } else if ((a & 3) == 0) {
      for (int i = lane * 4; i < nbytes; i += 128) cp_async<4>(dst + i, src + i);
    } else {  // 2-byte aligned half rows: synchronous copy
      const unsigned short* s2 = reinterpret_cast<const unsigned short*>(src);
      unsigned short* d2 = reinterpret_cast<unsigned short*>(dst);
      for (int i = lane; i < nbytes / 2; i += 32) d2[i] = s2[i];
    }
  }
}

// The bilinear sample of one point (R5-R7, R11, R12).  Coordinates are split
// into an integer base and an fp32 fraction; with s == 1 the split is exact.  A NaN or
// |s*(tap+d)| > 2^20 offset drops the sample.  Corner offsets are clamped into the image
// so the four 16-B gathers are unconditional (no divergence, no register zeroing); an
// out-of-image corner gets weight 0 and ok = false.
struct Samp {
  unsigned o[4]; // element offsets of the corners (image base excluded, group base included)
  float w[4];    // bilinear weights, 0 for out-of-image corners
  bool ok[4];    // corner inside the image
  float fy, fx;  // fractional parts
  float hy, hx;  // 1 - fractional parts (R11: exact or rounded once)
};

// Reading R11: the sample offset t = s*(tap + d) (UNIT, s = 1: t = d, the tap is added as an
// integer by the caller) split into floor, fraction f and complement 1 - f, each with
// relative error <= 2^-24 even when tiny (an edge sample whose only in-image corner has
// weight ~f must not lose it).  UNIT: d - floor(d) and (floor(d) + 1) - d are exact
// (Sterbenz).  Otherwise s*(tap + d) is formed exactly in fp64 (24 x 26 significant bits)
// and f, 1 - f are rounded once from it.  |t| > 2^20 or NaN: fin = false (sample dropped).
template <bool UNIT>
__device__ __forceinline__ void split_t(float s, int tap, float d, bool& fin, int& fl, float& f,
                                        float& f1) {
  if constexpr (UNIT) {
    fin = fabsf(d) <= 1048576.f;
    const float t = fin ? d : 0.f;
    const float flf = floorf(t);
    fl = (int)flf;
    f = t - flf;
    f1 = (flf + 1.f) - t;
  } else {
    const double t = (double)s * ((double)tap + (double)d);
    fin = fabs(t) <= 1048576.0;
    const double tt = fin ? t : 0.0;
    const double fld = floor(tt);
    fl = (int)fld;
    f = (float)(tt - fld);
    f1 = (float)((fld + 1.0) - tt);
  }
}

template <bool UNIT>
__device__ __forceinline__ void sample(int H, int W, unsigned C, float s, int yb, int xb, int tapy,
                                       int tapx, float dx, float dy, unsigned gbase, Samp& c) {
  bool finy, finx;
  int fly, flx;
  float hy, hx;
  split_t<UNIT>(s, tapy, dy, finy, fly, c.fy, hy);
  split_t<UNIT>(s, tapx, dx, finx, flx, c.fx, hx);
  const bool fin = finy && finx;
  const int y0 = yb + (UNIT ? tapy : 0) + fly;
  const int x0 = xb + (UNIT ? tapx : 0) + flx;
  const bool vy0 = fin && (unsigned)y0 < (unsigned)H, vy1 = fin && (unsigned)(y0 + 1) < (unsigned)H;
  const bool vx0 = (unsigned)x0 < (unsigned)W, vx1 = (unsigned)(x0 + 1) < (unsigned)W;
  const int y0c = min(max(y0, 0), H - 1), y1c = min(max(y0 + 1, 0), H - 1);
  const int x0c = min(max(x0, 0), W - 1), x1c = min(max(x0 + 1, 0), W - 1);
  const unsigned r0 = (unsigned)(y0c * W), r1 = (unsigned)(y1c * W);
  c.o[0] = (r0 + x0c) * C + gbase;
  c.o[1] = (r0 + x1c) * C + gbase;
  c.o[2] = (r1 + x0c) * C + gbase;
  c.o[3] = (r1 + x1c) * C + gbase;
  c.ok[0] = vy0 && vx0; c.ok[1] = vy0 && vx1; c.ok[2] = vy1 && vx0; c.ok[3] = vy1 && vx1;
  c.hy = hy;
  c.hx = hx;
  c.w[0] = c.ok[0] ? hy * hx : 0.f;
  c.w[1] = c.ok[1] ? hy * c.fx : 0.f;
  c.w[2] = c.ok[2] ? c.fy * hx : 0.f;
  c.w[3] = c.ok[3] ? c.fy * c.fx : 0.f;
}

// The K modulation scalars of one (pixel, group): raw (DCNv4) or the softmax
// over K (DCNv3; max-shifted).
template <typename T, int KC>
__device__ __forceinline__ void load_m(const T* row, int softmax, float* m) {
#pragma unroll
  for (int k = 0; k < KC; ++k) m[k] = Elem<T>::f(row[2 * KC + k]);
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

// Per-thread slot inside every tile (the tile shape is fixed for the launch): threads
// are ordered (pixel, group, lane) -- lane fastest, then group, then pixel (x fastest) --
// so a warp covers consecutive groups of neighbouring pixels.  The lane's 16-B chunks are
// dealt round-robin over the L lanes (L x 16 B contiguous per instruction) and their order
// is rotated so an 8-lane phase of a 128-bit load touches 8 distinct bank quads
// (microbench: 115 vs 57-81 B/clk/SM, profiles/r01_microbench_l1_red.jsonl).
template <int L, int CPL, int E>
struct Slot {
  int p, py, px, gl, lg;
  int co[CPL];  // element offset of the lane's h-th chunk inside the group vector
  __device__ __forceinline__ Slot(const Geo& g) {
    const int t = threadIdx.x;
    lg = t % L;
    const int q = t / L;
    gl = q % g.Gc;
    p = q / g.Gc;
    py = p / g.TW;
    px = p - py * g.TW;
    const int rot = g.rot_shift < 0 ? 0 : (((t & 31) / L) >> g.rot_shift) & (CPL - 1);
#pragma unroll
    for (int h = 0; h < CPL; ++h) co[h] = (((h + rot) & (CPL - 1)) * L + lg) * E;
  }
};

// ------------------------------------------------------------------ forward
// KH = KW = 0: runtime kernel size; otherwise compile-time (3x3 is the paper's grid).
template <typename T, int NCH, int CPL, int KH, int KW, bool UNIT>
__global__ void __launch_bounds__(256) fwd_kernel(Geo g, const T* __restrict__ x,
                                                  const T* __restrict__ om,
                                                  T* __restrict__ y) {
  constexpr int L = NCH / CPL;
  constexpr int E = Elem<T>::E;
  constexpr int KC = KH * KW;
  extern __shared__ __align__(128) unsigned char smem[];
  T* const bufs0 = reinterpret_cast<T*>(smem);
  const int bstride = g.TH * g.TW * g.seg;
  const Slot<L, CPL, E> sl(g);
  const bool slot_ok = sl.p < g.TH * g.TW;
  const int H = g.H, W = g.W, C = g.C, K = KC ? KC : g.K;
  const float s = g.s;

  int t = blockIdx.x;
  stage_tile<T>(g, t, om, bufs0);
  cp_async_commit();
  for (int it = 0; t < g.tiles_total; t += gridDim.x, ++it) {
    const int tn = t + gridDim.x;
    if (tn < g.tiles_total) stage_tile<T>(g, tn, om, bufs0 + ((it + 1) & 1) * bstride);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const Tile tl = decode_tile(g, t);
    const int ho = tl.h0 + sl.py, wo = tl.w0 + sl.px;
    if (slot_ok && ho < g.Ho && wo < g.Wo) {
      const T* row = bufs0 + (it & 1) * bstride + sl.p * g.seg + sl.gl * 3 * K;
      const int grp = tl.g0 + sl.gl;
      const unsigned gbase = grp * g.D;
      const int yb = ho * g.sh - g.ph + g.cy;
      const int xb = wo * g.sw - g.pw + g.cx;
      const T* ximg = x + (long long)tl.n * H * W * C;
      const T* xh[CPL];  // per-chunk base pointers: one IMAD.WIDE per gather address
#pragma unroll
      for (int h = 0; h < CPL; ++h) xh[h] = ximg + sl.co[h];
      float acc[CPL * E];
#pragma unroll
      for (int e = 0; e < CPL * E; ++e) acc[e] = 0.f;
      auto point = [&](int i, int j, int k, float m) {
        Samp c;
        sample<UNIT>(H, W, C, s, yb, xb, j * g.dh - g.cy, i * g.dw - g.cx,
                     Elem<T>::f(row[2 * k]), Elem<T>::f(row[2 * k + 1]), gbase, c);
        uint4 u[4][CPL];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < CPL; ++h) u[q][h] = ldg16_idx<sizeof(T)>(xh[h], c.o[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float a = m * c.w[q];
#pragma unroll
          for (int h = 0; h < CPL; ++h) {
            float v[E];
            Elem<T>::unpack(u[q][h], v);
#pragma unroll
            for (int e = 0; e < E; ++e) acc[h * E + e] = fmaf(a, v[e], acc[h * E + e]);
          }
        }
      };
      if constexpr (KC > 0) {
        float m[KC];
        load_m<T, KC>(row, g.softmax, m);
#pragma unroll
        for (int i = 0; i < KW; ++i)
#pragma unroll
          for (int j = 0; j < KH; ++j) point(i, j, i * KH + j, m[i * KH + j]);
      } else {
        float mx = 0.f, inv = 1.f;
        if (g.softmax) softmax_stats<T>(row, K, mx, inv);
        for (int i = 0; i < g.kw; ++i)
          for (int j = 0; j < g.kh; ++j) {
            const int k = i * g.kh + j;
            float m = Elem<T>::f(row[2 * K + k]);
            if (g.softmax) m = __expf(m - mx) * inv;
            point(i, j, k, m);
          }
      }
      T* yo = y + ((long long)(tl.n * g.Ho + ho) * g.Wo + wo) * C + gbase;
#pragma unroll
      for (int h = 0; h < CPL; ++h)
        *reinterpret_cast<uint4*>(yo + sl.co[h]) = Elem<T>::pack(acc + h * E);
    }
    __syncthreads();  // everyone is done with bufs[it & 1] before it is refilled
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ forward, TMA halo path
// The CTA's input footprint -- the tile plus a 2-pixel margin around the conv window,
// HH x HW pixels x Gc*D channels -- is fetched into shared memory by ONE TMA tensor
// copy (cp.async.bulk.tensor.4d, UTMALDG) that also zero-fills out-of-image pixels, so
// in-halo samples need no bounds checks, no clamping and only 32-bit shared addresses.
// Samples that leave the halo (|offset| >= 2 px) are recorded in a bit mask and added
// after the main loop with bounds-checked global gathers (rare; the main loop is
// branch-free).
// Halo and offset_mask tiles are double-buffered: the next tile's copies are in flight
// while the current tile is computed (persistent CTAs).
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
          "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint4 lds16(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}

// acc[0..E) += a * v (fp32 pairs through FFMA2)
template <int E>
__device__ __forceinline__ void axpy2(float* acc, float a, const float* v) {
  const float2 a2 = make_float2(a, a);
#pragma unroll
  for (int e = 0; e < E; e += 2) {
    float2 r = __ffma2_rn(a2, make_float2(v[e], v[e + 1]), make_float2(acc[e], acc[e + 1]));
    acc[e] = r.x;
    acc[e + 1] = r.y;
  }
}

// acc[0..E) += a * chunk, the chunk being one 16-byte vector of T:
//   fp32      -> 2 FFMA2 (packed fp32 pairs)
//   fp16/bf16 -> 8 FHFMA (sm_100 mixed-precision fma.rn.f32.{f16,bf16}: half x half + f32,
//                reading both halves of each register with no unpack); the weight a is
//                rounded to T once (relative error <= 2^-11 / 2^-8 per term, within the
//                1e-2 half-precision tolerance; R10)
template <typename T>
__device__ __forceinline__ void fma_chunk(float* acc, float a, const uint4& u);
template <>
__device__ __forceinline__ void fma_chunk<float>(float* acc, float a, const uint4& u) {
  float v[4];
  Elem<float>::unpack(u, v);
  axpy2<4>(acc, a, v);
}
template <>
__device__ __forceinline__ void fma_chunk<__half>(float* acc, float a, const uint4& u) {
  const unsigned short ah = __half_as_ushort(__float2half_rn(a));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "fma.rn.f32.f16 %0, %3, l, %0;\n\tfma.rn.f32.f16 %1, %3, h, %1;\n\t}"
        : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1])
        : "r"(w[i]), "h"(ah));
}
template <>
__device__ __forceinline__ void fma_chunk<__nv_bfloat16>(float* acc, float a, const uint4& u) {
  const unsigned short ah = __bfloat16_as_ushort(__float2bfloat16_rn(a));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "fma.rn.f32.bf16 %0, %3, l, %0;\n\tfma.rn.f32.bf16 %1, %3, h, %1;\n\t}"
        : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1])
        : "r"(w[i]), "h"(ah));
}

// S += <g, x> over one 16-byte chunk (two partial sums).  For fp16/bf16 both operands stay
// packed and FHFMA multiplies half x half exactly into the fp32 accumulator.
template <typename T>
__device__ __forceinline__ void dot_chunk(float2& S, const uint4& g, const uint4& x);
template <>
__device__ __forceinline__ void dot_chunk<float>(float2& S, const uint4& g, const uint4& x) {
  S = __ffma2_rn(make_float2(__uint_as_float(g.x), __uint_as_float(g.y)),
                 make_float2(__uint_as_float(x.x), __uint_as_float(x.y)), S);
  S = __ffma2_rn(make_float2(__uint_as_float(g.z), __uint_as_float(g.w)),
                 make_float2(__uint_as_float(x.z), __uint_as_float(x.w)), S);
}
#define DCNV4_DOT_HALF(TY, PTXT)                                                                  \
  template <>                                                                                     \
  __device__ __forceinline__ void dot_chunk<TY>(float2& S, const uint4& g, const uint4& x) {      \
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w}, xw[4] = {x.x, x.y, x.z, x.w};                    \
    _Pragma("unroll") for (int i = 0; i < 4; ++i)                                                 \
      asm("{\n\t.reg .b16 gl, gh, xl, xh;\n\tmov.b32 {gl, gh}, %2;\n\tmov.b32 {xl, xh}, %3;\n\t" \
          "fma.rn.f32." PTXT " %0, gl, xl, %0;\n\tfma.rn.f32." PTXT " %1, gh, xh, %1;\n\t}"        \
          : "+f"(S.x), "+f"(S.y)                                                                  \
          : "r"(gw[i]), "r"(xw[i]));                                                              \
  }
DCNV4_DOT_HALF(__half, "f16")
DCNV4_DOT_HALF(__nv_bfloat16, "bf16")
#undef DCNV4_DOT_HALF

// One fwd33 problem: its TMA map, geometry, tensors and first tile in the launch's tile
// space.  A launch covers one problem (fwd33_kernel) or several with the same storage
// type, channel layout and tile shape (fwd33_group_kernel, dcnv4_forward_grouped): the
// persistent CTAs then sweep the concatenated tile ranges, so the tails of small problems
// (late stages, batch 1) overlap the next problem instead of idling the SMs.
struct Fwd33Prob {
  CUtensorMap xmap;
  Geo g;
  const void* x;
  const void* om;
  void* y;
  int t0;  // first tile of this problem
};
constexpr int kMaxGroup = 8;
struct Fwd33Group {
  Fwd33Prob p[kMaxGroup];
  int count;
  int tiles_total;
};

// Problem owning global tile t (count <= kMaxGroup, ranges ascending)
template <typename Src>
__device__ __forceinline__ int find_prob(const Src& src, int t) {
  int pi = 0;
#pragma unroll
  for (int i = 1; i < kMaxGroup; ++i)
    if (i < src.count() && t >= src.prob(i).t0) pi = i;
  return pi;
}

// fwd33 body over a problem source: src.count(), src.prob(i) -> const Fwd33Prob&,
// src.tiles_total().  Fields used uniformly (TH, halo sizes, seg, rot_shift, softmax, s)
// are equal across the problems of one launch (checked on the host).
template <typename T, int NCH, int CPL, bool UNIT, typename Src>
__device__ __forceinline__ void fwd33_body(const Src& src) {
  const Geo& g = src.prob(0).g;  // uniform fields
  // Specialised for the paper's grid (3x3, stride 1, dilation 1; any padding):
  //   TW = 8 output columns, GC groups per CTA so one halo pixel is PB = GC*D*b >= 128 B,
  //   halo = (TH + 6) x 14 pixels, all strides compile-time (shift/immediate addressing).
  constexpr int L = NCH / CPL;
  constexpr int E = Elem<T>::E;
  constexpr int GC = NCH >= 8 ? 1 : 8 / NCH;
  constexpr int PB = GC * NCH * 16;
  constexpr int TW = 8, HWC = TW + 6, ROWB = HWC * PB;
  constexpr int K = 9;
  extern __shared__ __align__(128) unsigned char smem[];
  const int TH = g.TH, HH = TH + 6;
  const int npix = TH * TW;
  T* const ombase = reinterpret_cast<T*>(smem + 2 * g.halo_bytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(
      smem + 2 * g.halo_bytes + ((2 * npix * g.seg * (int)sizeof(T) + 7) & ~7));
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // thread slot: (pixel row, pixel col, group, lane) -- all powers of two
  const int tid = threadIdx.x;
  const int lg = tid % L;
  const int gl = (tid / L) % GC;
  const int px = (tid / (L * GC)) % TW;
  const int py = tid / (L * GC * TW);
  const bool slot_ok = py < TH;
  const int rot = g.rot_shift < 0 ? 0 : (((tid & 31) / L) >> g.rot_shift) & (CPL - 1);
  int co[CPL];
  uint32_t hb0[CPL];
#pragma unroll
  for (int h = 0; h < CPL; ++h) {
    co[h] = (((h + rot) & (CPL - 1)) * L + lg) * E;
    hb0[h] = smem_u32(smem) + (uint32_t)(gl * NCH * 16 + co[h] * (int)sizeof(T));
  }
  const float s = g.s;
  const unsigned segB = (unsigned)g.seg * sizeof(T);

  // global tile -> (problem, image, tile origin, group block)
  auto decode = [&](int t, int& pi, int& n, int& h0, int& w0, int& g0) {
    pi = find_prob(src, t);
    const Geo& q = src.prob(pi).g;
    t -= src.prob(pi).t0;
    const unsigned q1 = fdiv((unsigned)t, q.fd_gb);
    g0 = (t - (int)q1 * q.gblocks) * GC;
    const unsigned q2 = fdiv(q1, q.fd_tw);
    w0 = ((int)q1 - (int)q2 * q.tiles_w) * TW;
    const unsigned q3 = fdiv(q2, q.fd_th);
    h0 = ((int)q2 - (int)q3 * q.tiles_h) * TH;
    n = (int)q3;
  };
  auto issue = [&](int t, int b) {
    int pi, n, h0, w0, g0;
    decode(t, pi, n, h0, w0, g0);
    const Fwd33Prob& P = src.prob(pi);
    const Geo& g = P.g;
    const T* om = static_cast<const T*>(P.om);
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bar[b], (uint32_t)g.halo_box_bytes);
      tma_load_4d(smem + b * g.halo_bytes, &P.xmap, g0 * g.D, w0 - g.pw - 2, h0 - g.ph - 2, n, &bar[b]);
    }
    // offset_mask: GC*3K values per tile pixel, as upp units of g.unit bytes
    const char* src0 = reinterpret_cast<const char*>(
        om + ((long long)(n * g.Ho + h0) * g.Wo + w0) * g.S + g0 * 3 * K);
    unsigned char* dst0 = reinterpret_cast<unsigned char*>(ombase + b * npix * g.seg);
    const unsigned rowS = (unsigned)g.Wo * g.S * sizeof(T), pixS = (unsigned)g.S * sizeof(T);
    for (int f = tid; f < npix * g.upp; f += blockDim.x) {
      const int pix = (int)fdiv((unsigned)f, g.fd_upp);
      const int u = f - pix * g.upp;
      const int ppy = pix / TW, ppx = pix % TW;
      if (h0 + ppy >= g.Ho || w0 + ppx >= g.Wo) continue;
      const char* src = src0 + (ppy * rowS + ppx * pixS + (unsigned)(u * g.unit));
      unsigned char* dst = dst0 + pix * segB + u * g.unit;
      if (g.unit == 8) cp_async<8>(dst, src);
      else cp_async<4>(dst, src);
    }
  };

  const int tiles_total = src.tiles_total();
  int t = blockIdx.x;
  issue(t, 0);
  cp_async_commit();
  for (int it = 0; t < tiles_total; t += gridDim.x, ++it) {
    const int b = it & 1;
    const int tn = t + gridDim.x;
    if (tn < tiles_total) issue(tn, b ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    mbar_wait(&bar[b], (uint32_t)((it >> 1) & 1));
    __syncthreads();
    int pi, n, h0, w0, g0;
    decode(t, pi, n, h0, w0, g0);
    const Fwd33Prob& P = src.prob(pi);
    const Geo& g = P.g;
    const T* x = static_cast<const T*>(P.x);
    T* y = static_cast<T*>(P.y);
    const int H = g.H, W = g.W, C = g.C;
    const int ho = h0 + py, wo = w0 + px;
    if (slot_ok && ho < g.Ho && wo < g.Wo) {
      const T* row = ombase + b * npix * g.seg + (py * TW + px) * g.seg + gl * 3 * K;
      const unsigned gbase = (g0 + gl) * g.D;
      uint32_t hb[CPL];
#pragma unroll
      for (int h = 0; h < CPL; ++h) hb[h] = hb0[h] + (uint32_t)(b * g.halo_bytes);
      float m[K];
      load_m<T, K>(row, g.softmax, m);
      float acc[CPL * E];
#pragma unroll
      for (int e = 0; e < CPL * E; ++e) acc[e] = 0.f;
      unsigned outside = 0;  // samples that left the halo (handled after the main loop)
      struct Fetched {
        uint4 u[4][CPL];
        float a[4];
      };
      auto fetch = [&](int k, Fetched& F) {
        const int i = k / 3, j = k % 3;
        const float dx = Elem<T>::f(row[2 * k]), dy = Elem<T>::f(row[2 * k + 1]);
        bool finy, finx;
        int fly, flx;
        float fy, fx, hy, hx;
        split_t<UNIT>(s, j - 1, dy, finy, fly, fy, hy);
        split_t<UNIT>(s, i - 1, dx, finx, flx, fx, hx);
        const bool fin = finy && finx;
        // local halo coordinates: halo origin = (h0 - ph - 2, w0 - pw - 2)
        const int yl = py + (UNIT ? j + 2 : 3) + fly;
        const int xl = px + (UNIT ? i + 2 : 3) + flx;
        const bool in = (unsigned)yl <= (unsigned)(HH - 2) && (unsigned)xl <= (unsigned)(HWC - 2);
        outside |= (fin && !in) ? (1u << k) : 0u;
        const float mk = (fin && in) ? m[k] : 0.f;
        const uint32_t off = (uint32_t)((in ? yl : 0) * ROWB + (in ? xl : 0) * PB);
#pragma unroll
        for (int h = 0; h < CPL; ++h) {
          const uint32_t a0 = hb[h] + off;
          F.u[0][h] = lds16(a0);
          F.u[1][h] = lds16(a0 + PB);
          F.u[2][h] = lds16(a0 + ROWB);
          F.u[3][h] = lds16(a0 + ROWB + PB);
        }
        const float my = mk * hy, ny = mk * fy;
        F.a[0] = my * hx; F.a[1] = my * fx; F.a[2] = ny * hx; F.a[3] = ny * fx;
      };
      auto accum = [&](const Fetched& F) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < CPL; ++h) fma_chunk<T>(acc + h * E, F.a[q], F.u[q][h]);
      };
      // software pipeline: the gathers of point k+DEPTH-1 are issued before the FMAs of k
      constexpr int DEPTH = DCNV4_FWD_PIPE;
      Fetched F[DEPTH];
#pragma unroll
      for (int k = 0; k < DEPTH - 1; ++k) fetch(k, F[k]);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (k + DEPTH - 1 < K) fetch(k + DEPTH - 1, F[(k + DEPTH - 1) % DEPTH]);
        accum(F[k % DEPTH]);
      }
      if (outside) {  // rare: |offset| >= 2 px -- bounds-checked global gathers
        const T* ximg = x + (long long)n * H * W * C;
        float smx = 0.f, sinv = 1.f;
        if (g.softmax) softmax_stats<T>(row, K, smx, sinv);
#pragma unroll 1
        for (int k = 0; k < K; ++k) {
          if (!((outside >> k) & 1u)) continue;
          float mk = Elem<T>::f(row[2 * K + k]);  // re-read: m[] must stay in registers
          if (g.softmax) mk = __expf(mk - smx) * sinv;
          const int i = k / 3, j = k % 3;
          Samp c;
          sample<UNIT>(H, W, C, s, ho - g.ph + 1, wo - g.pw + 1, j - 1, i - 1,
                       Elem<T>::f(row[2 * k]), Elem<T>::f(row[2 * k + 1]), gbase, c);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < CPL; ++h) {
              float v[E];
              Elem<T>::unpack(ldg16_idx<sizeof(T)>(ximg + co[h], c.o[q]), v);
              axpy2<E>(acc + h * E, mk * c.w[q], v);
            }
        }
      }
      T* yo = y + ((long long)(n * g.Ho + ho) * g.Wo + wo) * C + gbase;
#pragma unroll
      for (int h = 0; h < CPL; ++h)
        *reinterpret_cast<uint4*>(yo + co[h]) = Elem<T>::pack(acc + h * E);
    }
    __syncthreads();  // everyone is done with halo[b] / om[b] before they are refilled
  }
  cp_async_wait<0>();
}

template <typename T, int NCH, int CPL, bool UNIT>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 0 : 2) fwd33_kernel(const __grid_constant__ Fwd33Prob prob) {
  struct One {
    const Fwd33Prob& p;
    __device__ int count() const { return 1; }
    __device__ const Fwd33Prob& prob(int) const { return p; }
    __device__ int tiles_total() const { return p.g.tiles_total; }
  } src{prob};
  fwd33_body<T, NCH, CPL, UNIT>(src);
}

template <typename T, int NCH, int CPL, bool UNIT>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 0 : 2) fwd33_group_kernel(const __grid_constant__ Fwd33Group grp) {
  struct Many {
    const Fwd33Group& q;
    __device__ int count() const { return q.count; }
    __device__ const Fwd33Prob& prob(int i) const { return q.p[i]; }
    __device__ int tiles_total() const { return q.tiles_total; }
  } src{grp};
  fwd33_body<T, NCH, CPL, UNIT>(src);
}

// ------------------------------------------------------------------ backward
// gx32: fp32 accumulator [N][H][W][C], zeroed by the host before launch.
// Per (pixel, group, k) with corner vectors v_q and this lane's gy:
//   S_q = sum_c gy_c v_qc          (4 dot products, the only per-channel work)
//   grad_m  partial = sum_q w_q S_q
//   grad_dy partial = (1-fx)(S_2 - S_0) + fx (S_3 - S_1)     [times s*m]
//   grad_dx partial = (1-fy)(S_1 - S_0) + fy (S_3 - S_2)     [times s*m]
// (S_q of out-of-image corners is 0) reduced over the L lanes with shuffles;
// grad_input += m w_q gy by 16-B vector reductions.
template <typename T, int NCH, int CPL, int KH, int KW, bool UNIT, bool DET>
__global__ void __launch_bounds__(256) bwd_kernel(Geo g, const T* __restrict__ x,
                                                  const T* __restrict__ om,
                                                  const T* __restrict__ gy,
                                                  void* __restrict__ gxacc,
                                                  T* __restrict__ gom) {
  float* const gx32 = static_cast<float*>(gxacc);       // DET = false
  long long* const gx64 = static_cast<long long*>(gxacc);  // DET = true
  constexpr int L = NCH / CPL;
  constexpr int E = Elem<T>::E;
  constexpr int KC = KH * KW;
  extern __shared__ __align__(128) unsigned char smem[];
  const int npix = g.TH * g.TW;
  T* const bufs0 = reinterpret_cast<T*>(smem);
  const int bstride = npix * g.seg;
  const int K = KC ? KC : g.K;
  const int seg32 = g.Gc * 3 * K;
  float* gtile = reinterpret_cast<float*>(smem + (((size_t)2 * npix * g.seg * sizeof(T) + 15) & ~(size_t)15));
  const Slot<L, CPL, E> sl(g);
  const bool slot_ok = sl.p < npix;
  const int H = g.H, W = g.W, C = g.C;
  const float s = g.s;
  const int lane = threadIdx.x & 31;

  int t = blockIdx.x;
  stage_tile<T>(g, t, om, bufs0);
  cp_async_commit();
  for (int it = 0; t < g.tiles_total; t += gridDim.x, ++it) {
    const int tn = t + gridDim.x;
    if (tn < g.tiles_total) stage_tile<T>(g, tn, om, bufs0 + ((it + 1) & 1) * bstride);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const Tile tl = decode_tile(g, t);
    const int ho0 = tl.h0 + sl.py, wo0 = tl.w0 + sl.px;
    const bool active = slot_ok && ho0 < g.Ho && wo0 < g.Wo;  // inactive lanes still shuffle
    const int ho = active ? ho0 : tl.h0, wo = active ? wo0 : tl.w0;
    const int pp = active ? sl.p : 0;
    const T* row = bufs0 + (it & 1) * bstride + pp * g.seg + sl.gl * 3 * K;
    float* grow = gtile + pp * seg32 + sl.gl * 3 * K;
    const int grp = tl.g0 + sl.gl;
    const unsigned gbase = grp * g.D;
    const int yb = ho * g.sh - g.ph + g.cy;
    const int xb = wo * g.sw - g.pw + g.cx;
    const long long img = (long long)tl.n * H * W * C;
    const T* xh[CPL];
    float* gxh[CPL];
    long long* gxq[CPL];
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      xh[h] = x + img + sl.co[h];
      gxh[h] = gx32 + img + sl.co[h];
      gxq[h] = gx64 + img + sl.co[h];
    }
    DetScale ds = {0.f, 0.f, 0, false};
    if constexpr (DET) ds = det_scale(g.detmax, tl.n, g.det_lc);

    float gyv[CPL * E];
    {
      const T* gyo = gy + ((long long)(tl.n * g.Ho + ho) * g.Wo + wo) * C + gbase;
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        uint4 u = ld_stream(reinterpret_cast<const uint4*>(gyo + sl.co[h]));
        Elem<T>::unpack(u, gyv + h * E);
      }
    }

    auto point = [&](int i, int j, int k, float m) {
      Samp c;
      sample<UNIT>(H, W, C, s, yb, xb, j * g.dh - g.cy, i * g.dw - g.cx,
                   Elem<T>::f(row[2 * k]), Elem<T>::f(row[2 * k + 1]), gbase, c);
      uint4 u[4][CPL];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < CPL; ++h) u[q][h] = ldg16_idx<sizeof(T)>(xh[h], c.o[q]);
      float S[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < CPL; ++h) {
          float v[E];
          Elem<T>::unpack(u[q][h], v);
#pragma unroll
          for (int e = 0; e < E; ++e) S[q] = fmaf(gyv[h * E + e], v[e], S[q]);
        }
#pragma unroll
      for (int q = 0; q < 4; ++q) S[q] = (active && c.ok[q]) ? S[q] : 0.f;
      // bilinear scatter of m*w*gy into the in-image corners
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a = m * c.w[q];
        if (active && a != 0.f) {
          if constexpr (DET) {
            const float ap = (a * ds.s1) * ds.s2;
#pragma unroll
            for (int h = 0; h < CPL; ++h)
#pragma unroll
              for (int e = 0; e < E; ++e) red_add_s64(gxq[h] + c.o[q] + e, __float2ll_rn(ap * gyv[h * E + e]));
          } else {
#pragma unroll
            for (int h = 0; h < CPL; ++h) {
#pragma unroll
              for (int e = 0; e < E; e += 4)
                red_add_v4_idx(gxh[h] + e, c.o[q], a * gyv[h * E + e], a * gyv[h * E + e + 1],
                               a * gyv[h * E + e + 2], a * gyv[h * E + e + 3]);
            }
          }
        }
      }
      const float hy = c.hy, hx = c.hx;
      float sgm = c.w[0] * S[0] + c.w[1] * S[1] + c.w[2] * S[2] + c.w[3] * S[3];
      float sgy = hx * (S[2] - S[0]) + c.fx * (S[3] - S[1]);
      float sgx = hy * (S[1] - S[0]) + c.fy * (S[3] - S[2]);
#pragma unroll
      for (int o = 1; o < L; o <<= 1) {
        sgm += __shfl_xor_sync(0xffffffffu, sgm, o);
        sgy += __shfl_xor_sync(0xffffffffu, sgy, o);
        sgx += __shfl_xor_sync(0xffffffffu, sgx, o);
      }
      if (active && sl.lg == 0) {
        grow[2 * k] = s * m * sgx;      // d/d dx_k
        grow[2 * k + 1] = s * m * sgy;  // d/d dy_k
        grow[2 * K + k] = sgm;          // d/d m_k
      }
    };

    if constexpr (KC > 0) {
      float m[KC];
      load_m<T, KC>(row, g.softmax, m);
#pragma unroll
      for (int i = 0; i < KW; ++i)
#pragma unroll
        for (int j = 0; j < KH; ++j) point(i, j, i * KH + j, m[i * KH + j]);
      if (g.softmax && active && sl.lg == 0) {  // dL/dz_k = p_k (gm_k - sum_j p_j gm_j)
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
          point(i, j, k, m);
        }
      if (g.softmax && active && sl.lg == 0) {
        float dot = 0.f;
        for (int k = 0; k < K; ++k) dot += __expf(Elem<T>::f(row[2 * K + k]) - mx) * inv * grow[2 * K + k];
        for (int k = 0; k < K; ++k) {
          const float p = __expf(Elem<T>::f(row[2 * K + k]) - mx) * inv;
          grow[2 * K + k] = p * (grow[2 * K + k] - dot);
        }
      }
    }
    __syncthreads();
    // write the tile's grad_offset_mask segments (warp per pixel, coalesced); the last
    // group run also zeroes the padding channels [3GK, S)
    const bool last = tl.g0 + g.Gc == g.G;
    for (int p = threadIdx.x >> 5; p < npix; p += blockDim.x >> 5) {
      const int pho = tl.h0 + p / g.TW, pwo = tl.w0 + p % g.TW;
      if (pho >= g.Ho || pwo >= g.Wo) continue;
      T* dst = gom + ((long long)(tl.n * g.Ho + pho) * g.Wo + pwo) * g.S;
      for (int e = lane; e < seg32; e += 32) dst[tl.g0 * 3 * K + e] = Elem<T>::from_f32(gtile[p * seg32 + e]);
      if (last)
        for (int e = g.G * 3 * K + lane; e < g.S; e += 32) dst[e] = Elem<T>::from_f32(0.f);
    }
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ backward, 3x3 halo + binned scatter
// One CTA tile (TH x 8 output pixels x GC groups) per iteration, persistent grid:
//  P0  TMA: x halo ((TH+6) x 14 px) and the gy tile; cp.async: offset_mask rows
//  P1  coordinates only: every in-image corner contribution a = m*w_q (the bilinear
//      scatter weight) is counted into its halo target bin (native shared-memory integer
//      reduction; fp32 shared atomics would be CAS loops)
//  P2  exclusive scan of the bin counts (padded to even: 16-B aligned bins) -> fill pointers
//  P3  per (pixel, group) lane group, the 9 samples from the shared-memory halo:
//        S_q = <gy, x_q> (4 dot products per sample), grad_m / grad_offset partials
//        reduced over the L lanes -> grad_om tile; each contribution is filed as
//        (a, source pixel) at its bin's fill pointer (counting sort, one ATOMS each)
//  P4  per (halo pixel, group, 16-B chunk): gx = sum_bin a * gy[source] from shared
//      memory, then ONE 16-B vector reduction into the fp32 grad_input accumulator --
//      ~3x the tile's pixels instead of 36 per (pixel, group) (the v3 kernel was bound
//      by L2 reduction throughput, profiles/r01_v1_*).
// Samples leaving the halo (|offset| >= 2 px) take a bounds-checked global path with
// direct vector reductions.
// v[q] for a runtime q in [0, 4) without dynamic register-array indexing (no local memory)
template <typename V>
__device__ __forceinline__ V pick4(const V* v, int q) {
  const V lo = (q & 1) ? v[1] : v[0];
  const V hi = (q & 1) ? v[3] : v[2];
  return (q & 2) ? hi : lo;
}

// PAD2: every count is rounded up to even (bins start 16-B aligned for paired entry loads)
// and the parity of the true count is kept in bit 0 of the (even) offset.
template <bool PAD2>
__device__ __forceinline__ int block_exclusive_scan(int* data, int n, int* warp_sums) {
  // in-place exclusive prefix sum of data[0..n) by the whole CTA; returns the total
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + nt - 1) / nt;
  const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
  int local = 0;
  for (int i = b0; i < b1; ++i) local += PAD2 ? (data[i] + 1) & ~1 : data[i];
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = nt >> 5;
    int ws = lane < nw ? warp_sums[lane] : 0;
    int wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    if (lane < nw) warp_sums[lane] = wi - ws;  // exclusive per warp
    if (lane == nw - 1) warp_sums[32] = wi;    // total
  }
  __syncthreads();
  int run = warp_sums[warp] + incl - local;
  for (int i = b0; i < b1; ++i) {
    const int v = data[i];
    data[i] = PAD2 ? run | (v & 1) : run;
    run += PAD2 ? (v + 1) & ~1 : v;
  }
  const int total = warp_sums[32];
  __syncthreads();
  return total;
}

template <typename T, int NCH, int CPL, bool UNIT, bool DET>
__global__ void __launch_bounds__(sizeof(T) == 4 ? 224 : 256, sizeof(T) == 4 ? 3 : 2) bwd33_kernel(const __grid_constant__ CUtensorMap xmap,
                                                    const __grid_constant__ CUtensorMap gymap, Geo g,
                                                    const T* __restrict__ x,
                                                    const T* __restrict__ om,
                                                    void* __restrict__ gxacc,
                                                    T* __restrict__ gom) {
  float* const gx32 = static_cast<float*>(gxacc);       // DET = false
  long long* const gx64 = static_cast<long long*>(gxacc);  // DET = true
  constexpr int L = NCH / CPL;
  constexpr int E = Elem<T>::E;
  constexpr int GC = NCH >= 8 ? 1 : 8 / NCH;
  constexpr int DG = NCH * E;  // channels per group (compile-time)
  constexpr int PB = GC * DG * (int)sizeof(T);
  constexpr int TW = 8, HWC = 14, ROWB = HWC * PB;
  constexpr int K = 9;
  constexpr int QPL = L >= 4 ? 1 : 4 / L;  // corners whose scatter this lane owns
  extern __shared__ __align__(128) unsigned char smem[];
  const int TH = g.TH, HH = TH + 6, NT = HH * HWC;
  const int npix = TH * TW;
  const T* gyt = reinterpret_cast<const T*>(smem + g.o_gy);
  T* const omt = reinterpret_cast<T*>(smem + g.o_om);
  int* const cnt = reinterpret_cast<int*>(smem + g.o_cnt);
  int* const fill = reinterpret_cast<int*>(smem + g.o_slot);  // per-bin fill pointers (P3)
  // bin entries (a, source pixel): fp32 -> 8 B {a, src}; fp16/bf16 -> 4 B {a rounded to T |
  // src << 16} (the pull's FHFMA rounds a to T anyway, fma_chunk), half the shared memory
  // fp32: 5 B per entry in two arrays, a (fp32) and the source pixel (u8), so the tile fits
  // three CTAs per SM
  constexpr bool ENT8 = sizeof(T) == 4;
  uint32_t* const ent = reinterpret_cast<uint32_t*>(smem + g.o_ent);   // half: {a_T | src << 16}
  float* const ent_a = reinterpret_cast<float*>(smem + g.o_ent);        // fp32: a
  unsigned char* const ent_s = reinterpret_cast<unsigned char*>(smem + g.o_ent) + 4 * g.ent_cap;  // fp32: src
  int* const wsum = reinterpret_cast<int*>(smem + g.o_wsum);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + g.o_bar);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31;
  const int lg = tid % L;
  const int gl = (tid / L) % GC;
  const int px = (tid / (L * GC)) % TW;
  const int py = tid / (L * GC * TW);
  const bool slot_ok = py < TH;
  const unsigned gmask = (L >= 32 ? 0xffffffffu : ((1u << L) - 1u)) << (lane & ~(L - 1));
  const int rot = g.rot_shift < 0 ? 0 : (((tid & 31) / L) >> g.rot_shift) & (CPL - 1);
  int co[CPL];
  uint32_t hb[CPL];
#pragma unroll
  for (int h = 0; h < CPL; ++h) {
    co[h] = (((h + rot) & (CPL - 1)) * L + lg) * E;
    hb[h] = smem_u32(smem) + (uint32_t)(gl * DG * (int)sizeof(T) + co[h] * (int)sizeof(T));
  }
  const int H = g.H, W = g.W, C = g.C;
  const float s = g.s;
  const unsigned segB = (unsigned)g.seg * sizeof(T);

  for (int t = blockIdx.x, it = 0; t < g.tiles_total; t += gridDim.x, ++it) {
    int n, h0, w0, g0;
    {
      const unsigned q1 = fdiv((unsigned)t, g.fd_gb);
      g0 = (t - (int)q1 * g.gblocks) * GC;
      const unsigned q2 = fdiv(q1, g.fd_tw);
      w0 = ((int)q1 - (int)q2 * g.tiles_w) * TW;
      const unsigned q3 = fdiv(q2, g.fd_th);
      h0 = ((int)q2 - (int)q3 * g.tiles_h) * TH;
      n = (int)q3;
    }
    const int hy0 = h0 - g.ph - 2, hx0 = w0 - g.pw - 2;  // halo origin in input pixels
    DetScale ds = {0.f, 0.f, 0, false};
    if constexpr (DET) ds = det_scale(g.detmax, n, g.det_lc);
    // ---- P0: loads
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, (uint32_t)(g.halo_box_bytes + g.gy_box_bytes));
      tma_load_4d(smem, &xmap, g0 * DG, hx0, hy0, n, bar);
      tma_load_4d(smem + g.o_gy, &gymap, g0 * DG, w0, h0, n, bar);
    }
    {
      const char* src0 = reinterpret_cast<const char*>(
          om + ((long long)(n * g.Ho + h0) * g.Wo + w0) * g.S + g0 * 3 * K);
      unsigned char* dst0 = reinterpret_cast<unsigned char*>(omt);
      const unsigned rowS = (unsigned)g.Wo * g.S * sizeof(T), pixS = (unsigned)g.S * sizeof(T);
      for (int f = tid; f < npix * g.upp; f += blockDim.x) {
        const int pix = (int)fdiv((unsigned)f, g.fd_upp);
        const int u = f - pix * g.upp;
        const int ppy = pix / TW, ppx = pix % TW;
        if (h0 + ppy >= g.Ho || w0 + ppx >= g.Wo) continue;
        const char* src = src0 + (ppy * rowS + ppx * pixS + (unsigned)(u * g.unit));
        unsigned char* dst = dst0 + pix * segB + u * g.unit;
        if (g.unit == 8) cp_async<8>(dst, src);
        else cp_async<4>(dst, src);
      }
      cp_async_commit();
    }
    for (int i = tid; i < GC * NT; i += blockDim.x) cnt[i] = 0;
    cp_async_wait<0>();
    mbar_wait(bar, (uint32_t)(it & 1));
    __syncthreads();

    const int ho = h0 + py, wo = w0 + px;
    const bool active = slot_ok && ho < g.Ho && wo < g.Wo;  // uniform over the L-lane group
    const T* row = omt + (py * TW + px) * g.seg + gl * 3 * K;
    float m[K];
    unsigned outside = 0;
    // Sample k of the item at tile position (qy, qx) whose offset_mask row is `rw`: halo-
    // local floor corner (yl, xl), fractions, whether it lies inside the halo, and the
    // in-image corners.  P1 and P3 both call this, so the contributions P1 counts are
    // exactly the ones P3 files.
    struct Pt {
      int yl, xl;
      float fy, fx, hy, hx;  // fractions and 1 - fractions (R11)
      bool fin, in, ok[4];
    };
    auto point_at = [&](const T* rw, int qy, int qx, int k) {
      Pt P;
      const int i = k / 3, j = k % 3;
      const float dx = Elem<T>::f(rw[2 * k]), dy = Elem<T>::f(rw[2 * k + 1]);
      bool finy, finx;
      int fly, flx;
      split_t<UNIT>(s, j - 1, dy, finy, fly, P.fy, P.hy);
      split_t<UNIT>(s, i - 1, dx, finx, flx, P.fx, P.hx);
      P.fin = finy && finx;
      const int yl = qy + (UNIT ? j + 2 : 3) + fly;
      const int xl = qx + (UNIT ? i + 2 : 3) + flx;
      P.in = P.fin && (unsigned)yl <= (unsigned)(HH - 2) && (unsigned)xl <= (unsigned)(HWC - 2);
      P.yl = P.in ? yl : 0;
      P.xl = P.in ? xl : 0;
      const int yy = hy0 + P.yl, xx = hx0 + P.xl;
      const bool vy0 = (unsigned)yy < (unsigned)H, vy1 = (unsigned)(yy + 1) < (unsigned)H;
      const bool vx0 = (unsigned)xx < (unsigned)W, vx1 = (unsigned)(xx + 1) < (unsigned)W;
      P.ok[0] = P.in && vy0 && vx0;
      P.ok[1] = P.in && vy0 && vx1;
      P.ok[2] = P.in && vy1 && vx0;
      P.ok[3] = P.in && vy1 && vx1;
      return P;
    };
    auto point = [&](int k) { return point_at(row, py, px, k); };
    if (active) load_m<T, K>(row, g.softmax, m);
    // ---- P1: bin counts only (coordinates, no data): shared-memory integer reductions.
    // DCNv4: one thread per (item, sample) over the whole tile (the L lanes of an item do
    // not repeat each other's coordinate work); DCNv3 softmax: each item's lanes (m needs
    // the softmax over all K of the item).
    if (DCNV4_BWD_ABL & 4) {
    } else if (!g.softmax && L >= 2) {
      const int nsamp = npix * GC * K;
      constexpr int P1U = DCNV4_P1_UNROLL;
#pragma unroll P1U
      for (int sidx = tid; sidx < nsamp; sidx += blockDim.x) {
        const int it9 = (sidx * 7282) >> 16;  // sidx / 9 (exact for sidx < 9216)
        const int k = sidx - it9 * 9;
        const int sgl = it9 % GC, spix = it9 / GC;
        const int sy = spix / TW, sx = spix % TW;
        if (h0 + sy >= g.Ho || w0 + sx >= g.Wo) continue;
        const T* rw = omt + spix * g.seg + sgl * 3 * K;
        const Pt P = point_at(rw, sy, sx, k);
        const float mk = Elem<T>::f(rw[2 * K + k]);
        const float w[4] = {P.hy * P.hx, P.hy * P.fx, P.fy * P.hx, P.fy * P.fx};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (P.ok[q] && mk * w[q] != 0.f)
            atomicAdd(&cnt[sgl * NT + (P.yl + (q >> 1)) * HWC + P.xl + (q & 1)], 1);
      }
    } else if (active) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const Pt P = point(k);
        const float w[4] = {P.hy * P.hx, P.hy * P.fx, P.fy * P.hx, P.fy * P.fx};
#pragma unroll
        for (int r = 0; r < QPL; ++r) {
          const int q = (lg % 4) + r * L;
          if (lg < 4 && q < 4 && pick4(P.ok, q) && m[k] * pick4(w, q) != 0.f) {
            const int tt = (P.yl + (q >> 1)) * HWC + P.xl + (q & 1);
            atomicAdd(&cnt[gl * NT + tt], 1);
          }
        }
      }
    }
    __syncthreads();
    // ---- P2: bin offsets (one in-place exclusive scan over all groups' bins, counts padded
    // to even; bin i holds entries [offs[i] & ~1, offs[i+1] & ~1)) and fill pointers
    int* const offs = cnt;
    {
      const int total = block_exclusive_scan<true>(offs, GC * NT, wsum);
      if (tid == 0) offs[GC * NT] = total;
      for (int i = tid; i < GC * NT; i += blockDim.x) fill[i] = offs[i] & ~1;
      __syncthreads();
    }
    // ---- P3: gathers from the x halo, grad_om (written straight to memory from the
    // lanes), and filing of the contributions
    if (active) {
      // this item's grad_offset_mask row: lane 0 writes d/d dx and d/d m, lane 1 d/d dy
      T* const grow = gom + ((long long)(n * g.Ho + ho) * g.Wo + wo) * g.S + (g0 + gl) * 3 * K;
      float gmv[K];
      float gyv[CPL * E];
      uint4 gyu[CPL];  // the lane's gy chunks, packed (dot products)
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        uint4 u = *reinterpret_cast<const uint4*>(gyt + (py * TW + px) * GC * DG + gl * DG + co[h]);
        gyu[h] = u;
        Elem<T>::unpack(u, gyv + h * E);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const Pt P = point(k);
        outside |= (P.fin && !P.in) ? (1u << k) : 0u;
        const uint32_t off = (uint32_t)(P.yl * ROWB + P.xl * PB);
        float S[4];
        float2 S2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < CPL; ++h) {
          if (DCNV4_BWD_ABL & 2) break;
          const uint32_t a0 = hb[h] + off;
          uint4 u[4] = {lds16(a0), lds16(a0 + PB), lds16(a0 + ROWB), lds16(a0 + ROWB + PB)};
#pragma unroll
          for (int q = 0; q < 4; ++q) dot_chunk<T>(S2[q], gyu[h], u[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) S[q] = S2[q].x + S2[q].y;
        // halo pixels outside the image hold zeros, so S needs no validity mask
        const float hy = P.hy, hx = P.hx;
        const float w[4] = {hy * hx, hy * P.fx, P.fy * hx, P.fy * P.fx};
        float sgm = w[0] * S[0] + w[1] * S[1] + w[2] * S[2] + w[3] * S[3];
        float sgy = hx * (S[2] - S[0]) + P.fx * (S[3] - S[1]);
        float sgx = hy * (S[1] - S[0]) + P.fy * (S[3] - S[2]);
#pragma unroll
        for (int o = 1; o < L; o <<= 1) {
          sgm += __shfl_xor_sync(gmask, sgm, o);
          sgy += __shfl_xor_sync(gmask, sgy, o);
          sgx += __shfl_xor_sync(gmask, sgx, o);
        }
        gmv[k] = P.in ? sgm : 0.f;
        // d/d dx_k, d/d dy_k (samples beyond the halo are written by the global path below)
        if (DCNV4_BWD_ABL & 8) {
        } else if (L >= 2) {
          if (lg < 2 && !(P.fin && !P.in))
            grow[2 * k + lg] = Elem<T>::from_f32(P.in ? s * m[k] * (lg ? sgy : sgx) : 0.f);
        } else if (!(P.fin && !P.in)) {
          grow[2 * k] = Elem<T>::from_f32(P.in ? s * m[k] * sgx : 0.f);
          grow[2 * k + 1] = Elem<T>::from_f32(P.in ? s * m[k] * sgy : 0.f);
        }
        // file this lane's scatter contributions into their bins
#pragma unroll
        for (int r = 0; r < QPL; ++r) {
          const int q = (lg % 4) + r * L;
          const float a = m[k] * pick4(w, q);
          if (!(DCNV4_BWD_ABL & 4) && lg < 4 && q < 4 && pick4(P.ok, q) && a != 0.f) {
            const int tt = (P.yl + (q >> 1)) * HWC + P.xl + (q & 1);
            const int e = atomicAdd(&fill[gl * NT + tt], 1);
            if constexpr (ENT8) {
              ent_a[e] = a;
              ent_s[e] = (unsigned char)(py * TW + px);
            } else {
              ent[e] = (uint32_t)Elem<T>::bits(a) | ((uint32_t)(py * TW + px) << 16);
            }
          }
        }
      }
      if (outside) {  // rare: samples beyond the halo -- global gathers and reductions
        const T* ximg = x + (long long)n * H * W * C;
        float* gximg = gx32 + (long long)n * H * W * C;
        long long* gxqimg = gx64 + (long long)n * H * W * C;
        const unsigned gbase = (g0 + gl) * DG;
        float smx = 0.f, sinv = 1.f;
        if (g.softmax) softmax_stats<T>(row, K, smx, sinv);
#pragma unroll 1
        for (int k = 0; k < K; ++k) {
          if (!((outside >> k) & 1u)) continue;
          const int i = k / 3, j = k % 3;
          float mk = Elem<T>::f(row[2 * K + k]);
          if (g.softmax) mk = __expf(mk - smx) * sinv;
          Samp c;
          sample<UNIT>(H, W, C, s, ho - g.ph + 1, wo - g.pw + 1, j - 1, i - 1,
                       Elem<T>::f(row[2 * k]), Elem<T>::f(row[2 * k + 1]), gbase, c);
          float S[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < CPL; ++h) {
              float v[E];
              Elem<T>::unpack(ldg16_idx<sizeof(T)>(ximg + co[h], c.o[q]), v);
#pragma unroll
              for (int e = 0; e < E; ++e) S[q] = fmaf(gyv[h * E + e], v[e], S[q]);
            }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!c.ok[q]) S[q] = 0.f;
            const float a = mk * c.w[q];
            if (a != 0.f) {
              if constexpr (DET) {
                const float ap = (a * ds.s1) * ds.s2;
#pragma unroll
                for (int h = 0; h < CPL; ++h)
#pragma unroll
                  for (int e = 0; e < E; ++e)
                    red_add_s64(gxqimg + c.o[q] + co[h] + e, __float2ll_rn(ap * gyv[h * E + e]));
              } else {
#pragma unroll
                for (int h = 0; h < CPL; ++h)
#pragma unroll
                  for (int e = 0; e < E; e += 4)
                    red_add_v4_idx(gximg + co[h] + e, c.o[q], a * gyv[h * E + e], a * gyv[h * E + e + 1],
                                   a * gyv[h * E + e + 2], a * gyv[h * E + e + 3]);
              }
            }
          }
          const float hy = c.hy, hx = c.hx;
          float sgm = c.w[0] * S[0] + c.w[1] * S[1] + c.w[2] * S[2] + c.w[3] * S[3];
          float sgy = hx * (S[2] - S[0]) + c.fx * (S[3] - S[1]);
          float sgx = hy * (S[1] - S[0]) + c.fy * (S[3] - S[2]);
#pragma unroll
          for (int o = 1; o < L; o <<= 1) {
            sgm += __shfl_xor_sync(gmask, sgm, o);
            sgy += __shfl_xor_sync(gmask, sgy, o);
            sgx += __shfl_xor_sync(gmask, sgx, o);
          }
          if (lg == 0) {  // the same thread reads these back below (program order)
            grow[2 * k] = Elem<T>::from_f32(s * mk * sgx);
            grow[2 * k + 1] = Elem<T>::from_f32(s * mk * sgy);
            grow[2 * K + k] = Elem<T>::from_f32(sgm);
          }
        }
      }
      if (lg == 0) {  // d/d m_k (DCNv3: w.r.t. the logits, dL/dz_k = p_k (gm_k - sum_j p_j gm_j))
        if (outside) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            if ((outside >> k) & 1u) gmv[k] = Elem<T>::f(grow[2 * K + k]);
        }
        if (g.softmax) {
          float dot = 0.f;
#pragma unroll
          for (int k = 0; k < K; ++k) dot += m[k] * gmv[k];
#pragma unroll
          for (int k = 0; k < K; ++k) gmv[k] = m[k] * (gmv[k] - dot);
        }
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (!(DCNV4_BWD_ABL & 8)) grow[2 * K + k] = Elem<T>::from_f32(gmv[k]);
      }
    }
    // padding channels [3GK, S) of grad_offset_mask: written 0 by the last group run
    if (g0 + GC == g.G && g.S > g.G * 3 * K) {
      const int npad = g.S - g.G * 3 * K;
      for (int f = tid; f < npix * npad; f += blockDim.x) {
        const int p = f / npad, e = f - p * npad;
        const int pho = h0 + p / TW, pwo = w0 + p % TW;
        if (pho < g.Ho && pwo < g.Wo)
          gom[((long long)(n * g.Ho + pho) * g.Wo + pwo) * g.S + g.G * 3 * K + e] = Elem<T>::from_f32(0.f);
      }
    }
    __syncthreads();
    // ---- P4: pull per (halo pixel, group, PC chunks) and one vector reduction per chunk;
    // PC = 2 chunks per lane amortise the entry loads; the chunk order alternates with
    // the halo pixel so an 8-lane phase still touches 8 distinct bank quads
    {
      constexpr int PC = DCNV4_P4_PC;
      constexpr int NCL = NCH / PC;  // lanes per (halo pixel, group)
      float* gximg = gx32 + (long long)n * H * W * C;
      long long* gxqimg = gx64 + (long long)n * H * W * C;
      const int ntask = (DCNV4_BWD_ABL & 5) ? 0 : NT * GC * NCL;
      for (int f = tid; f < ntask; f += blockDim.x) {
        const int cl = f % NCL;
        const int gg = (f / NCL) % GC;
        const int rk = f / (NCL * GC);
        const int tt = g.p4ord[rk];
        const int o0 = offs[gg * NT + tt];
        const int b0 = o0 & ~1;
        const int np = ((offs[gg * NT + tt + 1] & ~1) - b0) >> 1;  // entry pairs (last may be half)
        if (np == 0) continue;
        const bool odd = o0 & 1;
        const uint2* bh = reinterpret_cast<const uint2*>(ent + b0);       // half: entry pairs
        const float2* ba = reinterpret_cast<const float2*>(ent_a + b0);   // fp32: weight pairs
        const unsigned short* bs = reinterpret_cast<const unsigned short*>(ent_s + b0);  // fp32: source pairs
        // decoded entry pair: weights and source pixels
        struct Dec { float a0, a1; unsigned s0, s1; };
        auto dec = [&](int q) {
          Dec d;
          if constexpr (ENT8) {
            const float2 a2 = ba[q];
            const unsigned s2 = bs[q];
            d.a0 = a2.x; d.s0 = s2 & 0xffu; d.a1 = a2.y; d.s1 = s2 >> 8;
          } else {
            const uint2 en = bh[q];
            d.a0 = Elem<T>::from_bits((unsigned short)(en.x & 0xffffu)); d.s0 = en.x >> 16;
            d.a1 = Elem<T>::from_bits((unsigned short)(en.y & 0xffffu)); d.s1 = en.y >> 16;
          }
          return d;
        };
        int cc[PC];
#pragma unroll
        for (int h = 0; h < PC; ++h) cc[h] = (cl * PC + ((h + rk) & (PC - 1))) * E;
        const T* gyg = gyt + gg * DG;
        const int yy = hy0 + tt / HWC, xx = hx0 + tt % HWC;
        const unsigned dsto = (unsigned)(yy * W + xx) * C + (g0 + gg) * DG;
        if constexpr (DET) {  // per-contribution rounding to the 2^-F grid, int64 sums
          long long acc[PC * E];
#pragma unroll
          for (int e = 0; e < PC * E; ++e) acc[e] = 0;
          for (int q = 0; q < np; ++q) {
            const Dec en = dec(q);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              if (r == 1 && odd && q == np - 1) break;
              const T* src = gyg + (r ? en.s1 : en.s0) * (GC * DG);
              const float ap = ((r ? en.a1 : en.a0) * ds.s1) * ds.s2;
#pragma unroll
              for (int h = 0; h < PC; ++h) {
                float v[E];
                Elem<T>::unpack(*reinterpret_cast<const uint4*>(src + cc[h]), v);
#pragma unroll
                for (int e = 0; e < E; ++e) acc[h * E + e] += __float2ll_rn(ap * v[e]);
              }
            }
          }
          long long* dst = gxqimg + dsto;
#pragma unroll
          for (int h = 0; h < PC; ++h)
#pragma unroll
            for (int e = 0; e < E; ++e) red_add_s64(dst + cc[h] + e, acc[h * E + e]);
        } else {
          float acc[PC * E];
#pragma unroll
          for (int e = 0; e < PC * E; ++e) acc[e] = 0.f;
          // full pairs (branch-free; unrolled so the entry and gy loads of several pairs
          // are in flight together), then the last pair
#if DCNV4_P4_ACC2
          float acc2[PC * E];
#pragma unroll
          for (int e = 0; e < PC * E; ++e) acc2[e] = 0.f;
#endif
          constexpr int P4U = DCNV4_P4_UNROLL;
#pragma unroll P4U
          for (int q = 0; q < np - 1; ++q) {
            const Dec en = dec(q);
            const T* src0 = gyg + en.s0 * (GC * DG);
            const T* src1 = gyg + en.s1 * (GC * DG);
#pragma unroll
            for (int h = 0; h < PC; ++h) {
              fma_chunk<T>(acc + h * E, en.a0, *reinterpret_cast<const uint4*>(src0 + cc[h]));
#if DCNV4_P4_ACC2
              fma_chunk<T>(acc2 + h * E, en.a1, *reinterpret_cast<const uint4*>(src1 + cc[h]));
#else
              fma_chunk<T>(acc + h * E, en.a1, *reinterpret_cast<const uint4*>(src1 + cc[h]));
#endif
            }
          }
#if DCNV4_P4_ACC2
#pragma unroll
          for (int e = 0; e < PC * E; ++e) acc[e] += acc2[e];
#endif
          {
            const Dec en = dec(np - 1);
            const T* src0 = gyg + en.s0 * (GC * DG);
            const T* src1 = gyg + (odd ? 0u : en.s1) * (GC * DG);
            const float a1 = odd ? 0.f : en.a1;
#pragma unroll
            for (int h = 0; h < PC; ++h) {
              fma_chunk<T>(acc + h * E, en.a0, *reinterpret_cast<const uint4*>(src0 + cc[h]));
              fma_chunk<T>(acc + h * E, a1, *reinterpret_cast<const uint4*>(src1 + cc[h]));
            }
          }
          float* dst = gximg + dsto;
#pragma unroll
          for (int h = 0; h < PC; ++h)
#pragma unroll
            for (int e = 0; e < E; e += 4)
              red_add_v4(dst + cc[h] + e, acc[h * E + e], acc[h * E + e + 1], acc[h * E + e + 2],
                         acc[h * E + e + 3]);
        }
      }
    }
    __syncthreads();  // shared memory is reused by the next tile
  }
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

// Deterministic mode, pass 1: per-image maxima {max|gy|, max|m|} as float bits
// (non-negative floats order as unsigned integers; NaN sorts above +inf).  grid =
// (blocks per image, images of this launch), image n = n0 + blockIdx.y; mx must be zeroed.  softmax: the mask bound is 1 (softmax
// outputs), unless a logit is non-finite.
template <typename T>
__global__ void __launch_bounds__(256) det_scale_kernel(const T* __restrict__ gy,
                                                        const T* __restrict__ om, long long gy_chunks,
                                                        int npix, int S, int G, int K, int softmax,
                                                        unsigned* __restrict__ mx, long long n0) {
  constexpr int E = Elem<T>::E;
  const long long n = n0 + blockIdx.y;
  const int nt = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned vg = 0u, vm = 0u;
  const uint4* g4 = reinterpret_cast<const uint4*>(gy) + (long long)n * gy_chunks;
  for (long long i = t0; i < gy_chunks; i += nt) {
    float v[E];
    Elem<T>::unpack(ld_stream(g4 + i), v);
#pragma unroll
    for (int e = 0; e < E; ++e) vg = max(vg, __float_as_uint(v[e]) & 0x7fffffffu);
  }
  const T* o = om + (long long)n * npix * S;
  const long long nm = (long long)npix * G * K;
  for (long long i = t0; i < nm; i += nt) {
    const long long pix = i / (G * K);
    const int r = (int)(i - pix * (G * K));
    const int gg = r / K, k = r - gg * K;
    vm = max(vm, __float_as_uint(Elem<T>::f(o[pix * S + gg * 3 * K + 2 * K + k])) & 0x7fffffffu);
  }
  if (softmax) vm = vm >= 0x7f800000u ? vm : 0x3f800000u;
  vg = __reduce_max_sync(0xffffffffu, vg);
  vm = __reduce_max_sync(0xffffffffu, vm);
  if ((threadIdx.x & 31) == 0) {
    if (vg) atomicMax(mx + 2 * n, vg);
    if (vm) atomicMax(mx + 2 * n + 1, vm);
  }
}

// Deterministic mode, pass 3: int64 accumulator -> grad_input in T (RN), NaN for flagged
// images.  nchunk = number of E-element chunks; per_image = H*W*C.
template <typename T>
__global__ void __launch_bounds__(256) det_convert_kernel(const long long* __restrict__ src,
                                                          const unsigned* __restrict__ mx, int lc,
                                                          long long per_image, T* __restrict__ dst,
                                                          long long nchunk) {
  constexpr int E = Elem<T>::E;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nchunk;
       i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)((i * E) / per_image);
    const DetScale d = det_scale(mx, n, lc);
    float v[E];
    const longlong2* s2 = reinterpret_cast<const longlong2*>(src + i * E);
#pragma unroll
    for (int q = 0; q < E / 2; ++q) {
      const longlong2 w = __ldcs(s2 + q);
      v[2 * q] = d.bad ? __int_as_float(0x7fc00000) : (float)ldexp((double)w.x, -d.F);
      v[2 * q + 1] = d.bad ? __int_as_float(0x7fc00000) : (float)ldexp((double)w.y, -d.F);
    }
    reinterpret_cast<uint4*>(dst)[i] = Elem<T>::pack(v);
  }
}

}  // namespace dcnv4
