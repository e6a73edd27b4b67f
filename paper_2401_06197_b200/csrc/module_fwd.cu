// module_fwd.cu -- the fused lightweight-module forward of include/dcnv4_module.h.
// ======================================================================================
// Fused lightweight-module forward (include/dcnv4_module.h dcnv4_module_forward):
//   y = DCNv4(x, RN_T(x . W^T + b))  -- P:334 (one linear layer for offsets and weights)
//   and P:1003-1009 (the lightweight module samples x itself) -- with the offset_mask
//   computed per tile on the tensor cores and consumed from shared memory: it never
//   reaches HBM or L2.
// CTA tile = 16 output rows x 8 output columns (128 pixels = the MMA's M) x GC groups
// (GC * D * sizeof(T) = 128 B).  Per tile:
//   thread 0   TMA: the x halo (22 x 14 pixels x GC*D channels, zero-filled outside the
//              image) and, per 64-channel k block, the A box x[16 rows][8 cols][64 ch]
//              (128-B swizzle: row m = 8*row + col is the canonical K-major layout) and
//              the B box W[GC*27 rows of this group block][64 ch];
//   thread 32  tcgen05.mma (M=128, N=BN >= GC*27, K=16) x 4 per k block into TMEM;
//   all warps  tcgen05.ld (warp w: TMEM lanes 32(w%4).., column chunks of parity w/4),
//              + bias, RN to T, into the tile's offset_mask rows in shared memory --
//              the same [pixel][group][dx0,dy0,...,m8] segment layout fwd33 stages;
//   all warps  the fwd33 aggregation (2 passes of 8 rows; halo gathers, FHFMA).
// Single-buffered; two or more CTAs per SM overlap each other's loads and MMAs.
// ======================================================================================
#include "../../include/dcnv4_module.h"
#include "dcnv4_kernels.cuh"
#include "sm100_tc.cuh"
#include "ablation.h"

namespace oml {

struct FGeo {
  int H, W, C, G, D, J;        // J = 3*G*9
  int ph, pw;
  float s;
  int softmax;
  int BN, kb, stages;
  int tiles_h, tiles_w, gblocks, tiles_total;
  dcnv4::FastDiv fd_gb, fd_tw, fd_th;
  int halo_bytes, halo_box_bytes, seg;  // seg: om_s elements per pixel
  uint32_t idesc, tmem_cols;
};

template <typename T, int NCH, int CPL, bool UNIT>
__global__ void __launch_bounds__(256, 3) module_fwd_kernel(const __grid_constant__ CUtensorMap hmap,
                                                         const __grid_constant__ CUtensorMap amap,
                                                         const __grid_constant__ CUtensorMap bmap,
                                                         FGeo g, const T* __restrict__ x,
                                                         const T* __restrict__ bias, T* __restrict__ y) {
  using dcnv4::Elem;
  constexpr int L = NCH / CPL;
  constexpr int E = Elem<T>::E;
  constexpr int GC = NCH >= 8 ? 1 : 8 / NCH;
  constexpr int PB = GC * NCH * 16;
  constexpr int TH = 16, TW = 8, HH = TH + 6, HWC = TW + 6, ROWB = HWC * PB, K = 9;
  constexpr int RPP = 256 / (TW * GC * L);  // tile rows per aggregation pass
  static_assert(TW * GC * L == 32, "one warp per tile row");
  constexpr int JB = GC * 3 * K;            // om columns of this group block
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int stages = g.stages;
  const uint32_t B_BYTES = (uint32_t)g.BN * 128u;
  // the tile's offset_mask rows alias the A/B ring: they are written after the tile's
  // MMAs completed (tfull) and dead before the next tile's TMA loads (end-of-tile barrier)
  const uint32_t sA = base, sB = sA + stages * A_BYTES, sH = sB + stages * B_BYTES;
  T* om_s = reinterpret_cast<T*>(gbase);
  const uint32_t sBias = sH + (uint32_t)g.halo_bytes;
  float* bias_s = reinterpret_cast<float*>(gbase + (sBias - base));
  const uint32_t sBar = (sBias + (JB + 1) * 4 + 7u) & ~7u;
  const uint32_t full = sBar, empty = sBar + 8 * stages, hbar = sBar + 16 * stages, tfull = hbar + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (tfull + 8 - base));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    mbar_init(hbar, 1);
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(g.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  // aggregation slot: (tile row within the pass, column, group, lane)
  const int lg = tid % L;
  const int gl = (tid / L) % GC;
  const int px = (tid / (L * GC)) % TW;
  const int pyl = tid / (L * GC * TW);
  // chunk order alternates with the column parity: an 8-lane phase of a 128-bit shared
  // load (two columns) then covers all eight 16-B bank quads of the 128-B halo pixels
  const int rot = px & (CPL - 1);
  int co[CPL];
#pragma unroll
  for (int h = 0; h < CPL; ++h) co[h] = (((h + rot) & (CPL - 1)) * L + lg) * E;
  const float s = g.s;
  int sp = 0, sm = 0;
  uint32_t php = 0, phm = 0;

  for (int it = 0, t = blockIdx.x; t < g.tiles_total; t += gridDim.x, ++it) {
    const unsigned q1 = dcnv4::fdiv((unsigned)t, g.fd_gb);
    const int g0 = (t - (int)q1 * g.gblocks) * GC;
    const unsigned q2 = dcnv4::fdiv(q1, g.fd_tw);
    const int w0 = ((int)q1 - (int)q2 * g.tiles_w) * TW;
    const unsigned q3 = dcnv4::fdiv(q2, g.fd_th);
    const int h0 = ((int)q2 - (int)q3 * g.tiles_h) * TH;
    const int n = (int)q3;
    for (int i = tid; i <= JB; i += 256)  // one zero pad entry (odd JB, packed pairs)
      bias_s[i] = (bias != nullptr && i < JB) ? Elem<T>::f(bias[g0 * 3 * K + i]) : 0.f;
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(hbar, (uint32_t)g.halo_box_bytes);
      tma_load_4d_u(sH, &hmap, g0 * g.D, w0 - g.pw - 2, h0 - g.ph - 2, n, hbar);
      for (int k = 0; k < g.kb; ++k) {
        mbar_wait(empty + 8 * sp, php ^ 1);
        mbar_expect_tx(full + 8 * sp, A_BYTES + B_BYTES);
        tma_load_4d_u(sA + sp * A_BYTES, &amap, k * BK, w0, h0, n, full + 8 * sp);
        tma_load_2d(sB + sp * B_BYTES, &bmap, k * BK, g0 * 3 * K, full + 8 * sp);
        if (++sp == stages) {
          sp = 0;
          php ^= 1;
        }
      }
    } else if (tid == 32) {
      fence_after();
      for (int k = 0; k < g.kb; ++k) {
        mbar_wait(full + 8 * sm, phm);
        fence_after();
        const uint64_t ad = sdesc(sA + sm * A_BYTES), bd = sdesc(sB + sm * B_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) mma_f16(tmem, ad + 2 * kk, bd + 2 * kk, g.idesc, (k | kk) != 0);
        mma_commit(empty + 8 * sm);
        if (++sm == stages) {
          sm = 0;
          phm ^= 1;
        }
      }
      mma_commit(tfull);
    }
    __syncthreads();  // bias_s written
    // ---- om epilogue: TMEM -> (+bias, RN_T) -> om_s[pixel][JB]
    mbar_wait(tfull, (uint32_t)(it & 1));
    fence_after();
    {
      const int q = warp & 3, half = warp >> 2;
      const int p = q * 32 + lane;  // tile pixel = 8 * row + col (A box order)
      T* orow = om_s + p * g.seg;
#pragma unroll
      for (int c = 0; c < (JB + 31) / 32; ++c) {
        if ((c & 1) != half) continue;
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t* orow2 = reinterpret_cast<uint32_t*>(orow);  // seg and JB are even
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int j = c * 32 + e;
          if (j < JB)
            orow2[j >> 1] = Cvt<T>::pack(__uint_as_float(r[e]) + bias_s[j], __uint_as_float(r[e + 1]) + bias_s[j + 1]);
        }
      }
    }
    fence_before();
    mbar_wait(hbar, (uint32_t)(it & 1));
    __syncthreads();  // om_s complete, halo landed, TMEM drained
    // ---- aggregation (fwd33 body on the 16-row tile, RPP rows per pass)
    const uint32_t hb0 = sH + (uint32_t)(gl * NCH * 16);
    const unsigned gbase_c = (unsigned)(g0 + gl) * g.D;
#pragma unroll 1
    for (int pass = 0; pass < TH / RPP; ++pass) {
      const int py = pass * RPP + pyl;
      const int ho = h0 + py, wo = w0 + px;
      if (ho >= g.H || wo >= g.W) continue;
      const T* row = om_s + (py * TW + px) * g.seg + gl * 3 * K;
      uint32_t hb[CPL];
#pragma unroll
      for (int h = 0; h < CPL; ++h) hb[h] = hb0 + (uint32_t)(co[h] * (int)sizeof(T));
      float m[K];
      dcnv4::load_m<T, K>(row, g.softmax, m);
      float acc[CPL * E];
#pragma unroll
      for (int e = 0; e < CPL * E; ++e) acc[e] = 0.f;
      unsigned outside = 0;
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
        dcnv4::split_t<UNIT>(s, j - 1, dy, finy, fly, fy, hy);
        dcnv4::split_t<UNIT>(s, i - 1, dx, finx, flx, fx, hx);
        const bool fin = finy && finx;
        const int yl = py + (UNIT ? j + 2 : 3) + fly;
        const int xl = px + (UNIT ? i + 2 : 3) + flx;
        const bool in = (unsigned)yl <= (unsigned)(HH - 2) && (unsigned)xl <= (unsigned)(HWC - 2);
        outside |= (fin && !in) ? (1u << k) : 0u;
        const float mk = (fin && in) ? m[k] : 0.f;
        const uint32_t off = (uint32_t)((in ? yl : 0) * ROWB + (in ? xl : 0) * PB);
#pragma unroll
        for (int h = 0; h < CPL; ++h) {
          const uint32_t a0 = hb[h] + off;
          F.u[0][h] = dcnv4::lds16(a0);
          F.u[1][h] = dcnv4::lds16(a0 + PB);
          F.u[2][h] = dcnv4::lds16(a0 + ROWB);
          F.u[3][h] = dcnv4::lds16(a0 + ROWB + PB);
        }
        const float my = mk * hy, ny = mk * fy;
        F.a[0] = my * hx;
        F.a[1] = my * fx;
        F.a[2] = ny * hx;
        F.a[3] = ny * fx;
      };
      auto accum = [&](const Fetched& F) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < CPL; ++h) dcnv4::fma_chunk<T>(acc + h * E, F.a[q], F.u[q][h]);
      };
      // software pipeline (as fwd33): the gathers of point k+1 issue before the FMAs of k
      Fetched F0, F1;
      fetch(0, F0);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (k + 1 < K) fetch(k + 1, (k & 1) ? F0 : F1);
        accum((k & 1) ? F1 : F0);
      }
      if (outside) {  // |offset| >= 2 px: bounds-checked global gathers
        const T* ximg = x + (long long)n * g.H * g.W * g.C;
        float smx = 0.f, sinv = 1.f;
        if (g.softmax) dcnv4::softmax_stats<T>(row, K, smx, sinv);
#pragma unroll 1
        for (int k = 0; k < K; ++k) {
          if (!((outside >> k) & 1u)) continue;
          float mk = Elem<T>::f(row[2 * K + k]);
          if (g.softmax) mk = __expf(mk - smx) * sinv;
          const int i = k / 3, j = k % 3;
          dcnv4::Samp c;
          dcnv4::sample<UNIT>(g.H, g.W, (unsigned)g.C, s, ho - g.ph + 1, wo - g.pw + 1, j - 1, i - 1,
                              Elem<T>::f(row[2 * k]), Elem<T>::f(row[2 * k + 1]), gbase_c, c);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < CPL; ++h) {
              float v[E];
              Elem<T>::unpack(dcnv4::ldg16_idx<sizeof(T)>(ximg + co[h], c.o[q]), v);
              dcnv4::axpy2<E>(acc + h * E, mk * c.w[q], v);
            }
        }
      }
      T* yo = y + ((long long)(n * g.H + ho) * g.W + wo) * g.C + gbase_c;
#pragma unroll
      for (int h = 0; h < CPL; ++h) *reinterpret_cast<uint4*>(yo + co[h]) = Elem<T>::pack(acc + h * E);
    }
    fence_before();
    __syncthreads();  // halo, om_s and TMEM free for the next tile
    fence_after();
  }
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(g.tmem_cols)
                 : "memory");
}

dcnv4::FastDiv fastdiv(unsigned d) {  // n / d == (umulhi(n, m) + n) >> l (as dcnv4_api.cu)
  unsigned l = 0;
  while ((1ull << l) < d) ++l;
  const unsigned long long mf = ((1ull << (32 + l)) + d - 1) / d;
  return {(unsigned)(mf - (1ull << 32)), l};
}

// Row pitch (bytes) of the fused kernel's shared-memory offset_mask tile for GC groups of
// 27 halves per pixel: the 4-B multiple minimising the worst bank-conflict degree of the
// epilogue stores (lane = pixel, one u32 each) plus that of the aggregation's reads.
int seg_pitch(int GC) {
  const int JB = GC * 27, b = 2;
  auto ways = [](const int* words, int n) {  // max distinct words mapping to one bank
    int w = 1;
    for (int bank = 0; bank < 32; ++bank) {
      int distinct[32], nd = 0;
      for (int i = 0; i < n; ++i) {
        if (words[i] % 32 != bank) continue;
        bool seen = false;
        for (int k = 0; k < nd; ++k) seen |= distinct[k] == words[i];
        if (!seen) distinct[nd++] = words[i];
      }
      w = nd > w ? nd : w;
    }
    return w;
  };
  int best = 1 << 30, pitch = 0;
  for (int sw = (JB * b + 3) / 4; sw < (JB * b + 3) / 4 + 16; ++sw) {
    int words[32], cost = 0;
    for (int j = 0; j < 4; ++j) {
      for (int q = 0; q < 32; ++q) words[q] = q * sw + j;
      const int w = ways(words, 32);
      cost = cost > w ? cost : w;
    }
    int rc = 0;
    const int Lg = 32 / (8 * GC);
    for (int k = 0; k < 27; ++k) {
      int n = 0;
      for (int px = 0; px < 8; ++px)
        for (int gl = 0; gl < GC; ++gl)
          for (int lg = 0; lg < Lg; ++lg) words[n++] = (px * sw * 4 + gl * 54 + 2 * k) / 4;
      const int w = ways(words, n);
      rc = rc > w ? rc : w;
    }
    if (cost + rc < best) {
      best = cost + rc;
      pitch = sw * 4;
    }
  }
  return pitch;
}

template <typename T, int NCH, int CPL>
cudaError_t launch_module(const CUtensorMap& hm, const CUtensorMap& am, const CUtensorMap& bm, const FGeo& g,
                          bool unit, size_t smem, const void* x, const void* bias, void* y, cudaStream_t st) {
  void (*k)(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
            const __grid_constant__ CUtensorMap, FGeo, const T*, const T*, T*) =
      unit ? module_fwd_kernel<T, NCH, CPL, true> : module_fwd_kernel<T, NCH, CPL, false>;
  // per-kernel setup (attributes, register count) once per host thread and device
  struct Memo {
    const void* k;
    int dev, regs, sms;
    size_t smem;
  };
  thread_local Memo memo[8];
  thread_local int memo_n = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int regs_used = -1, sms = 148;
  for (int i = 0; i < memo_n; ++i)
    if (memo[i].k == (const void*)k && memo[i].dev == dev && memo[i].smem >= smem) {
      regs_used = memo[i].regs;
      sms = memo[i].sms;
    }
  cudaError_t e = cudaSuccess;
  if (regs_used < 0) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa0;
    e = cudaFuncGetAttributes(&fa0, k);
    if (e != cudaSuccess) return e;
    regs_used = fa0.numRegs;
    sms = num_sms();
    memo[memo_n % 8] = Memo{(const void*)k, dev, regs_used, sms, smem};
    memo_n = memo_n < 8 ? memo_n + 1 : 8;
  }
  // CTAs per SM from registers, shared memory and TMEM columns.  (The occupancy query
  // reports 1 for this kernel; co-residency of 2-3 CTAs was measured to run and to pay:
  // c2 stage 1 143 -> 98 us.)
  const int regs = ((regs_used + 7) / 8) * 8 * 256;
  int per_sm = 65536 / (regs > 0 ? regs : 65536);
  const int by_smem = (int)((228 * 1024) / (smem + 1024));
  if (by_smem < per_sm) per_sm = by_smem;
  if ((int)(512 / g.tmem_cols) < per_sm) per_sm = (int)(512 / g.tmem_cols);
  if (dcnv4::ablation_set(dcnv4::kAblModulePerSm)) per_sm = atoi(dcnv4::ablation(dcnv4::kAblModulePerSm));  // ablation only
  if (per_sm < 1) per_sm = 1;
  const long long cap = (long long)sms * per_sm;
  const unsigned grid = (unsigned)(g.tiles_total < cap ? g.tiles_total : cap);
  k<<<grid, 256, smem, st>>>(hm, am, bm, g, static_cast<const T*>(x), static_cast<const T*>(bias),
                             static_cast<T*>(y));
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_module_t(int nch, const CUtensorMap& hm, const CUtensorMap& am, const CUtensorMap& bm,
                            const FGeo& g, bool unit, size_t smem, const void* x, const void* bias, void* y,
                            cudaStream_t st) {
  switch (nch) {
    case 2: return launch_module<T, 2, 2>(hm, am, bm, g, unit, smem, x, bias, y, st);
    case 4: return launch_module<T, 4, 2>(hm, am, bm, g, unit, smem, x, bias, y, st);
    default: return launch_module<T, 8, 2>(hm, am, bm, g, unit, smem, x, bias, y, st);
  }
}

}  // namespace oml

namespace oml {
// y = DCNv4(value, RN_T(input . W^T + b)): the offset_mask from `input`, the samples from
// `value` (the lightweight module: value == input)
static int module_forward_impl(const dcnv4_params* p, dcnv4_dtype dtype, const void* input, const void* value,
                               const void* weight, const void* bias, void* output, void* stream) {
  using namespace oml;
  int64_t Ho = 0, Wo = 0;
  int rc = dcnv4_output_size(p, &Ho, &Wo);
  if (rc != DCNV4_OK) return rc;
  dcnv4_internal_set_error("");
  if (dtype != DCNV4_F32 && dtype != DCNV4_F16 && dtype != DCNV4_BF16)
    return fail(DCNV4_ERR_INVALID_ARG, "dtype %d is not DCNV4_F32/F16/BF16", (int)dtype);
  if (dtype == DCNV4_F32)
    return fail(DCNV4_ERR_UNSUPPORTED, "dtype DCNV4_F32: the tcgen05 linear takes F16/BF16 operands");
  if (p->kernel_h != 3 || p->kernel_w != 3 || p->stride_h != 1 || p->stride_w != 1 || p->pad_h != 1 ||
      p->pad_w != 1 || p->dilation_h != 1 || p->dilation_w != 1)
    return fail(DCNV4_ERR_UNSUPPORTED, "the fused module needs kernel 3x3, stride 1, pad 1, dilation 1");
  const int b = 2;
  const int nch = p->D * b / 16;
  if (p->D * b % 16 || (nch != 2 && nch != 4 && nch != 8))
    return fail(DCNV4_ERR_UNSUPPORTED, "D*sizeof(dtype) = %d B must be 32, 64 or 128", p->D * b);
  const int GC = nch >= 8 ? 1 : 8 / nch;
  if (p->G % GC) return fail(DCNV4_ERR_UNSUPPORTED, "G = %d must be a multiple of %d", p->G, GC);
  const long long C = (long long)p->G * p->D;
  const long long J = 27LL * p->G;
  if (p->N * p->H * p->W * C >= (1LL << 31) * 8)
    return fail(DCNV4_ERR_SHAPE, "input too large");
  if (p->H * p->W * C >= (1LL << 31)) return fail(DCNV4_ERR_SHAPE, "per-image size H*W*C must be < 2^31");
  if (p->N == 0) return DCNV4_OK;
  if (!input || !value || !weight || !output)
    return fail(DCNV4_ERR_INVALID_ARG, "%s is NULL", !input ? "input" : !value ? "value" : !weight ? "weight" : "output");
  if (((uintptr_t)input | (uintptr_t)value | (uintptr_t)weight | (uintptr_t)output) & 15)
    return fail(DCNV4_ERR_MISALIGNED, "%s is not 16-B aligned",
                ((uintptr_t)input & 15) ? "input" : ((uintptr_t)weight & 15) ? "weight" : "output");
  if ((uintptr_t)bias & 1) return fail(DCNV4_ERR_MISALIGNED, "bias is not 2-B aligned");
  FGeo g;
  g.H = (int)p->H;
  g.W = (int)p->W;
  g.C = (int)C;
  g.G = p->G;
  g.D = p->D;
  g.J = (int)J;
  g.ph = p->pad_h;
  g.pw = p->pad_w;
  g.s = p->offset_scale;
  g.softmax = p->softmax;
  const int JB = GC * 27;
  g.BN = (JB + 15) / 16 * 16;
  g.kb = (int)((C + BK - 1) / BK);
  g.tiles_h = (int)((p->H + 15) / 16);
  g.tiles_w = (int)((p->W + 7) / 8);
  g.gblocks = p->G / GC;
  // operand ring: one stage (72 KB of shared memory -> 3 CTAs/SM, other CTAs hide the
  // k-block loads) up to 4 k blocks (C <= 256).  Beyond that a tile's 8 sequential k-block
  // rounds dominate and two stages pay -- but only when there are enough tiles for every
  // SM to hold two (c2 C=512, 512 tiles: 28.7 vs 32.6 us); with fewer tiles than that
  // each CTA runs ~one tile and the extra shared memory only costs (c3 batch 1 C=512,
  // 80 tiles: one stage 44.96 vs two 47.14 us; profiles/r01b_module_stages_ab.txt).
  // DCNV4_MODULE_STAGES=1|2 overrides (ablation).
  {
    const long long ntiles = p->N * g.tiles_h * g.tiles_w * (long long)g.gblocks;
    g.stages = (g.kb > 4 && ntiles >= 2LL * num_sms()) ? 2 : 1;
  }
  if (dcnv4::ablation_set(dcnv4::kAblModuleStages)) {
    const char* se = dcnv4::ablation(dcnv4::kAblModuleStages);
    const int v = atoi(se);
    if (v == 1 || v == 2) g.stages = v <= g.kb ? v : g.stages;
  }
  const long long tiles = p->N * g.tiles_h * g.tiles_w * (long long)g.gblocks;
  if (tiles >= (1LL << 31)) return fail(DCNV4_ERR_SHAPE, "too many tiles");
  g.tiles_total = (int)tiles;
  g.fd_gb = fastdiv((unsigned)g.gblocks);
  g.fd_tw = fastdiv((unsigned)g.tiles_w);
  g.fd_th = fastdiv((unsigned)g.tiles_h);
  const int PB = 128;
  g.halo_box_bytes = 22 * 14 * PB;
  g.halo_bytes = (g.halo_box_bytes + 1023) & ~1023;
  // om_s row pitch (4-B multiple) minimising simulated bank conflicts of the epilogue's
  // row-per-lane u32 stores (32 consecutive pixels) plus the aggregation's scalar reads
  // (a warp = 8 columns x GC groups x L lanes of one tile row); computed once per GC
  static const int kSegBytes[3] = {seg_pitch(1), seg_pitch(2), seg_pitch(4)};
  const int seg_bytes = kSegBytes[GC == 1 ? 0 : GC == 2 ? 1 : 2];
  g.seg = seg_bytes / b;
  g.idesc = (1u << 4) | ((dtype == DCNV4_BF16 ? 1u : 0u) << 7) | ((dtype == DCNV4_BF16 ? 1u : 0u) << 10) |
            ((uint32_t)(g.BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  g.tmem_cols = g.BN <= 32 ? 32 : g.BN <= 64 ? 64 : 128;
  if (128 * (size_t)seg_bytes > (size_t)g.stages * (A_BYTES + g.BN * 128))
    return fail(DCNV4_ERR_UNSUPPORTED, "offset_mask tile does not fit the operand ring");
  const size_t smem = 1024 + (size_t)g.stages * (A_BYTES + g.BN * 128) + g.halo_bytes + (JB + 1) * 4 + 8 +
                      8 * (2 * g.stages + 2) + 16;
  if (smem > 227 * 1024) return fail(DCNV4_ERR_UNSUPPORTED, "shared-memory plan exceeds 227 KB");
  CUtensorMap hm, am, bm;
  CUresult e1 = encode4d(&hm, dtype, value, p->N, p->H, p->W, C, GC * p->D, 14, 22, false);
  CUresult e2 = encode4d(&am, dtype, input, p->N, p->H, p->W, C, BK, 8, 16, true);
  CUresult e3 = encode2d(&bm, dtype, weight, J, C, BK, g.BN);
  if (e1 != CUDA_SUCCESS || e2 != CUDA_SUCCESS || e3 != CUDA_SUCCESS)
    return fail(DCNV4_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d/%d/%d)", (int)e1, (int)e2, (int)e3);
  const bool unit = p->offset_scale == 1.0f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t err = dtype == DCNV4_F16
                        ? launch_module_t<__half>(nch, hm, am, bm, g, unit, smem, value, bias, output, st)
                        : launch_module_t<__nv_bfloat16>(nch, hm, am, bm, g, unit, smem, value, bias, output, st);
  if (err != cudaSuccess) return fail(DCNV4_ERR_CUDA, "module_fwd launch: %s", cudaGetErrorString(err));
  return DCNV4_OK;
}
}  // namespace oml

extern "C" {

int dcnv4_module_forward(const dcnv4_params* p, dcnv4_dtype dtype, const void* input, const void* weight,
                         const void* bias, void* output, void* stream) {
  return oml::module_forward_impl(p, dtype, input, input, weight, bias, output, stream);
}

int dcnv4_module_core_forward(const dcnv4_params* p, dcnv4_dtype dtype, const void* input, const void* value,
                              const void* weight, const void* bias, void* output, void* stream) {
  if (value == output && value) {
    dcnv4_internal_set_error("dcnv4_module_core_forward: output must not alias value");
    return DCNV4_ERR_INVALID_ARG;
  }
  return oml::module_forward_impl(p, dtype, input, value, weight, bias, output, stream);
}

}  // extern "C"
