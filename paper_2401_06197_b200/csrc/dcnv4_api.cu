// dcnv4_api.cu -- the C ABI of include/dcnv4.h: validation, launch configuration,
// dispatch.  Stateless apart from the thread-local error string; never allocates,
// synchronises or changes the device.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include <cudaTypedefs.h>

#include "../../include/dcnv4.h"
#include "dcnv4_kernels.cuh"
#include "dcnv4_launch.h"
#include "ablation.h"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int elem_size(int dtype) { return dtype == DCNV4_F32 ? 4 : 2; }

constexpr int kMaxK = 64;           // largest kernel_h*kernel_w supported
constexpr int kMaxThreads = 256;    // CTA size bound (__launch_bounds__)

// Default chunks-per-lane for a given chunk count; the harness may override it with the
// env vars DCNV4_FWD_CPL / DCNV4_BWD_CPL (ablation only).
int default_cpl(int nch, int pass) {
  (void)pass;
  if (nch <= 2) return nch;
  if (nch <= 8) return 2;
  return 4;
}

bool cpl_supported(int nch, int cpl) {
  switch (nch * 100 + cpl) {
    case 101: case 201: case 202: case 401: case 402: case 404: case 802: case 804:
    case 1602: case 1604: return true;
    default: return false;
  }
}

int validate_geometry(const dcnv4_params* p, int dtype, int64_t* Ho, int64_t* Wo) {
  if (!p) return fail(DCNV4_ERR_INVALID_ARG, "params is NULL");
  if (dtype != DCNV4_F32 && dtype != DCNV4_F16 && dtype != DCNV4_BF16)
    return fail(DCNV4_ERR_INVALID_ARG, "dtype %d is not DCNV4_F32/F16/BF16", dtype);
  if (p->N < 0) return fail(DCNV4_ERR_INVALID_ARG, "N = %lld < 0", (long long)p->N);
  if (p->H <= 0) return fail(DCNV4_ERR_INVALID_ARG, "H = %lld <= 0", (long long)p->H);
  if (p->W <= 0) return fail(DCNV4_ERR_INVALID_ARG, "W = %lld <= 0", (long long)p->W);
  if (p->G <= 0) return fail(DCNV4_ERR_INVALID_ARG, "G = %d <= 0", p->G);
  if (p->D <= 0) return fail(DCNV4_ERR_INVALID_ARG, "D = %d <= 0", p->D);
  if (p->kernel_h <= 0 || p->kernel_w <= 0)
    return fail(DCNV4_ERR_INVALID_ARG, "kernel %dx%d must be positive", p->kernel_h, p->kernel_w);
  if (p->stride_h <= 0 || p->stride_w <= 0)
    return fail(DCNV4_ERR_INVALID_ARG, "stride %dx%d must be positive", p->stride_h, p->stride_w);
  if (p->pad_h < 0 || p->pad_w < 0)
    return fail(DCNV4_ERR_INVALID_ARG, "pad %dx%d must be >= 0", p->pad_h, p->pad_w);
  if (p->dilation_h <= 0 || p->dilation_w <= 0)
    return fail(DCNV4_ERR_INVALID_ARG, "dilation %dx%d must be positive", p->dilation_h,
                p->dilation_w);
  if (!isfinite(p->offset_scale))
    return fail(DCNV4_ERR_INVALID_ARG, "offset_scale is not finite");
  if (p->softmax != 0 && p->softmax != 1)
    return fail(DCNV4_ERR_INVALID_ARG, "softmax flag %d is not 0 or 1", p->softmax);
  if (p->deterministic != 0 && p->deterministic != 1)
    return fail(DCNV4_ERR_INVALID_ARG, "deterministic flag %d is not 0 or 1", p->deterministic);
  const int64_t K = (int64_t)p->kernel_h * p->kernel_w;
  if (K > kMaxK)
    return fail(DCNV4_ERR_UNSUPPORTED, "K = kernel_h*kernel_w = %lld exceeds %d", (long long)K, kMaxK);
  const int64_t h = p->H + 2 * (int64_t)p->pad_h - (int64_t)p->dilation_h * (p->kernel_h - 1) - 1;
  const int64_t w = p->W + 2 * (int64_t)p->pad_w - (int64_t)p->dilation_w * (p->kernel_w - 1) - 1;
  if (h < 0) return fail(DCNV4_ERR_SHAPE, "output height is empty (H axis)");
  if (w < 0) return fail(DCNV4_ERR_SHAPE, "output width is empty (W axis)");
  *Ho = h / p->stride_h + 1;
  *Wo = w / p->stride_w + 1;
  const int64_t S = p->om_stride ? p->om_stride : 3 * (int64_t)p->G * K;
  if (S < 3 * (int64_t)p->G * K)
    return fail(DCNV4_ERR_SHAPE, "om_stride = %d < 3*G*K = %lld (offset_mask channel axis)",
                p->om_stride, (long long)(3 * p->G * K));
  const int64_t C = (int64_t)p->G * p->D;
  const int64_t lim = (int64_t)1 << 31;
  if (p->H * p->W * C >= lim)
    return fail(DCNV4_ERR_SHAPE, "per-image input H*W*C = %lld must be < 2^31",
                (long long)(p->H * p->W * C));
  if (*Ho * *Wo * C >= lim || *Ho * *Wo * S >= lim)
    return fail(DCNV4_ERR_SHAPE, "per-image output/offset_mask size must be < 2^31");
  if (p->H + 2 > (1 << 20) || p->W + 2 > (1 << 20))
    return fail(DCNV4_ERR_SHAPE, "H and W must be < 2^20");
  const int b = elem_size(dtype);
  if (((int64_t)p->D * b) % 16 != 0)
    return fail(DCNV4_ERR_UNSUPPORTED,
                "D*sizeof(dtype) = %lld bytes is not a multiple of 16 (group channel axis)",
                (long long)p->D * b);
  if ((int64_t)p->D * b > 256)
    return fail(DCNV4_ERR_UNSUPPORTED, "D*sizeof(dtype) = %lld bytes exceeds 256",
                (long long)p->D * b);
  const int64_t nch = (int64_t)p->D * b / 16;
  if (nch & (nch - 1))
    return fail(DCNV4_ERR_UNSUPPORTED,
                "D*sizeof(dtype) = %lld bytes is not 16 B times a power of two (group channel axis)",
                (long long)p->D * b);
  return DCNV4_OK;
}

// Average 128-bit load wavefronts per 8-lane phase relative to the ideal (1.0 = every
// phase hits 8 distinct bank quads) for a CTA whose threads are ordered
// (pixel, group, lane) with Gc groups and L lanes per (pixel, group); tries the chunk
// stagger shifts and returns the best (rot = (pg_in_warp >> shift) & (CPL-1)).
double conflict_factor(int Gc, int L, int cpl, int nch, int threads, int* best_shift) {
  double best = 1e30;
  *best_shift = -1;
  for (int rs = -1; rs <= 4; ++rs) {
    double wf = 0, ideal = 0;
    for (int t0 = 0; t0 < threads; t0 += 8) {
      for (int c = 0; c < cpl; ++c) {
        int count[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int active = 0, mx = 0;
        for (int l = 0; l < 8 && t0 + l < threads; ++l) {
          const int t = t0 + l;
          const int lg = t % L, q = t / L, gl = q % Gc;
          const int pg = (t & 31) / L;
          const int rot = rs < 0 ? 0 : (pg >> rs) & (cpl - 1);
          const int ch = ((c + rot) & (cpl - 1)) * L + lg;
          const int quad = (gl * nch + ch) & 7;
          mx = ++count[quad] > mx ? count[quad] : mx;
          ++active;
        }
        if (active) { wf += mx; ideal += (active + 7) / 8; }
      }
    }
    const double f = wf / ideal;
    if (f < best - 1e-9) { best = f; *best_shift = rs; }
  }
  return best;
}

struct TileChoice {
  int TH, TW, Gc, rot_shift;
};

// CTA tile: minimise (L2->L1 footprint traffic) + (bank-conflict excess) + (idle lanes)
// + (per-CTA overhead), all in bytes-equivalent.  DESIGN.md "Tiling".
dcnv4::FastDiv make_fastdiv(unsigned d) {
  unsigned l = 0;
  while ((1ull << l) < d) ++l;
  const unsigned long long mf = ((1ull << (32 + l)) + d - 1) / d;
  return {(unsigned)(mf - (1ull << 32)), l};
}

// Halo box (TMA path): rows/cols of input the tile's samples need with |offset| < 2 px.
inline int halo_rows(const dcnv4_params* p, int TH) {
  return (TH - 1) * p->stride_h + (p->kernel_h - 1) * p->dilation_h + 5;
}
inline int halo_cols(const dcnv4_params* p, int TW) {
  return (TW - 1) * p->stride_w + (p->kernel_w - 1) * p->dilation_w + 5;
}
constexpr size_t kHaloSmemBudget = 110 * 1024;  // two CTAs per SM

size_t seg_bytes_for(int Gc, int K, int b) {
  int sb = ((Gc * 3 * K * b) + 15) & ~15;
  if ((sb / 16) % 2 == 0) sb += 16;
  return (size_t)sb;
}

size_t halo_smem(const dcnv4_params* p, int TH, int TW, int Gc, int b) {
  const size_t PB = (size_t)Gc * p->D * b;
  const size_t hb = ((size_t)halo_rows(p, TH) * halo_cols(p, TW) * PB + 127) & ~(size_t)127;
  return 2 * hb + 2 * (size_t)TH * TW * seg_bytes_for(Gc, p->kernel_h * p->kernel_w, b) + 16;
}

TileChoice choose_tile_search(const dcnv4_params* p, int b, int nch, int cpl, int64_t Ho,
                              int64_t Wo, bool halo);

// The tile search costs tens of microseconds of host time per call and depends only on
// the geometry and the chunking (the DCNV4_TILE ablation is fixed at first use): memoised
// per host thread.
TileChoice choose_tile(const dcnv4_params* p, int b, int nch, int cpl, int64_t Ho, int64_t Wo,
                       bool halo) {
  struct Memo {
    dcnv4_params p;
    int b, nch, cpl, halo;
    TileChoice tc;
  };
  thread_local Memo memo[32];
  thread_local int memo_n = 0, memo_next = 0;
  for (int i = 0; i < memo_n; ++i) {
    const Memo& m = memo[i];
    if (m.b == b && m.nch == nch && m.cpl == cpl && m.halo == (int)halo &&
        memcmp(&m.p, p, sizeof(dcnv4_params)) == 0)
      return m.tc;
  }
  const TileChoice tc = choose_tile_search(p, b, nch, cpl, Ho, Wo, halo);
  Memo& m = memo[memo_next];
  memcpy(&m.p, p, sizeof(dcnv4_params));
  m.b = b; m.nch = nch; m.cpl = cpl; m.halo = (int)halo;
  m.tc = tc;
  memo_next = (memo_next + 1) % 32;
  memo_n = memo_n < 32 ? memo_n + 1 : 32;
  return tc;
}

TileChoice choose_tile_search(const dcnv4_params* p, int b, int nch, int cpl, int64_t Ho,
                              int64_t Wo, bool halo) {
  const int L = nch / cpl;
  const int G = p->G;
  const double V = nch * 16.0;  // bytes of one (pixel, group) channel vector
  const double K = (double)p->kernel_h * p->kernel_w;
  const double kappa = 3.0;     // L2->L1 byte vs L1-hit byte
  TileChoice best = {1, 1, G, -1};
  double best_cost = 1e300;
  const char* env = dcnv4::ablation(dcnv4::kAblTile);
  int fth = 0, ftw = 0, fgc = 0;
  if (env && *env) sscanf(env, "%d,%d,%d", &fth, &ftw, &fgc);
  const int cand[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 20, 24, 25, 28, 32, 40, 50, 56, 64};
  const double total_pg = (double)p->N * Ho * Wo * G;
  for (int Gc = 1; Gc <= G; ++Gc) {
    if (G % Gc || Gc * L > kMaxThreads) continue;
    if (fgc && Gc != fgc) continue;
    int shift;
    const double cf = conflict_factor(Gc, L, cpl, nch, 128 > Gc * L ? 128 : Gc * L, &shift);
    for (int TH : cand) {
      if (TH > Ho || (fth && TH != fth)) continue;
      for (int TW : cand) {
        if (TW > Wo || (ftw && TW != ftw)) continue;
        const int thr = TH * TW * Gc * L;
        if (thr > kMaxThreads) break;
        const bool whole = TH == Ho && TW == Wo;
        if (thr < 64 && !whole && !(fth && ftw)) continue;
        const double tiles = (double)((Ho + TH - 1) / TH) * ((Wo + TW - 1) / TW) * (G / Gc) * p->N;
        double fh = halo_rows(p, TH), fw = halo_cols(p, TW);
        double cfe = cf;
        if (halo) {  // the whole box is fetched (zero-filled outside the image)
          if (fh > 256 || fw > 256 || halo_smem(p, TH, TW, Gc, b) > kHaloSmemBudget) continue;
          if (((size_t)Gc * p->D * b) % 128) cfe += 0.5;  // pixel pitch breaks the quad pattern
        } else {
          fh = std::min<double>(fh, p->H);
          fw = std::min<double>(fw, p->W);
        }
        const double idle = tiles * TH * TW * Gc - total_pg;
        const double l1 = total_pg * 4.0 * K * V;
        const double cost = tiles * kappa * fh * fw * Gc * V + (cfe - 1.0) * l1 +
                            idle * 4.0 * K * V * 0.25 + tiles * 4096.0 +
                            (thr % 32 ? (32 - thr % 32) : 0) * tiles * 64.0;
        if (cost < best_cost) {
          best_cost = cost;
          best = {TH, TW, Gc, shift};
        }
      }
    }
  }
  (void)b;
  return best;
}

// TMA descriptor of x as a 4-D tensor {C, W, H, N} (innermost first) with a
// {Gc*D, HW, HH, 1} box; out-of-image elements are zero-filled by the hardware.
bool encode_nhwc_map(int dtype, const void* ptr, int64_t N, int64_t Hh, int64_t Ww, int64_t C,
                     int box_c, int box_w, int box_h, CUtensorMap* map);

bool encode_x_map(const dcnv4_params* p, int dtype, const void* x, int box_c, int box_w,
                  int box_h, CUtensorMap* map) {
  return encode_nhwc_map(dtype, x, p->N, p->H, p->W, (int64_t)p->G * p->D, box_c, box_w, box_h, map);
}

bool encode_nhwc_map(int dtype, const void* ptr, int64_t N, int64_t Hh, int64_t Ww, int64_t Cc,
                     int box_c, int box_w, int box_h, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const int b = elem_size(dtype);
  const cuuint64_t C = (cuuint64_t)Cc;
  const cuuint64_t dims[4] = {C, (cuuint64_t)Ww, (cuuint64_t)Hh, (cuuint64_t)N};
  const cuuint64_t strides[3] = {C * b, C * b * Ww, C * b * Ww * Hh};
  const cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapDataType dt = dtype == DCNV4_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : dtype == DCNV4_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                      : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  auto run = [&] {
    return encode(map, dt, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUresult r = run();
  if (r == CUDA_ERROR_INVALID_CONTEXT) {
    // a thread that has not touched the runtime yet (e.g. torch's autograd worker) has
    // no current context: bind the current device's primary context (same device)
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) r = run();
  }
  return r == CUDA_SUCCESS;
}

// Forward on the paper's grid (3x3, stride 1, dilation 1): the TMA halo kernel with
// compile-time strides (dcnv4_kernels.cuh fwd33_kernel).  Fills lc/g and returns true
// when the geometry, alignment and shared-memory budget allow it; the caller otherwise
// keeps the global-gather kernel.  `x` may be NULL (planning only, lc->halo stays false).
bool plan_fwd33(const dcnv4_params* p, int dtype, int64_t Ho, int64_t Wo, const void* x,
                dcnv4::Launch* lc, dcnv4::Geo* g, int th_force = 0) {
  const char* path = dcnv4::ablation(dcnv4::kAblFwdPath);
  if (path && path[0] == 'g') return false;
  if (p->kernel_h != 3 || p->kernel_w != 3 || p->stride_h != 1 || p->stride_w != 1 ||
      p->dilation_h != 1 || p->dilation_w != 1)
    return false;
  const int b = elem_size(dtype);
  const int nch = lc->nch, cpl = lc->cpl, L = lc->lanes;
  const int GC = nch >= 8 ? 1 : 8 / nch;
  if (p->G % GC) return false;
  const int PB = GC * nch * 16;
  const int per_row = 8 * GC * L;  // threads per tile row
  // 128-thread CTAs (TH = 4 at D = 16): four CTAs per SM overlap their per-tile halo waits
  // better than two 256-thread ones; measured best or within 2% on every c2/c3 stage
  // (profiles/r01_fwd_th_sweep.jsonl)
  int TH = std::max(1, 128 / per_row);
  if (TH < 1) return false;
  const char* th_env = dcnv4::ablation(dcnv4::kAblFwd33TH);
  if (th_env && *th_env) TH = std::max(1, std::min(TH, atoi(th_env)));
  if (TH > Ho) TH = (int)Ho;
  if (th_force) TH = th_force;  // grouped launch: one tile shape for every problem
  const int K = 9;
  const int S = p->om_stride ? p->om_stride : 3 * p->G * K;
  const int segB_raw = GC * 3 * K * b;
  int unit = 0;
  for (int u : {8, 4})
    if ((S * b) % u == 0 && segB_raw % u == 0) { unit = u; break; }
  if (!unit) return false;
  // the kernels form a tile pixel's offset_mask source offset (row * Wo*S*b + col * S*b)
  // in 32-bit unsigned arithmetic
  if ((long long)(TH + 1) * std::max<int64_t>(Wo, 8) * S * b >= (1LL << 32)) return false;
  int seg_bytes = (segB_raw + 15) & ~15;
  if ((seg_bytes / 16) % 2 == 0) seg_bytes += 16;
  const int HH = TH + 6, HWc = 14;
  const int halo_box = HH * HWc * PB;
  const int halo_bytes = (halo_box + 127) & ~127;
  const size_t smem = 2 * (size_t)halo_bytes + 2 * (size_t)TH * 8 * seg_bytes + 16;
  if (smem > 227 * 1024) return false;
  const long long tiles_h = (Ho + TH - 1) / TH, tiles_w = (Wo + 7) / 8, gblocks = p->G / GC;
  const long long tiles = (long long)p->N * tiles_h * tiles_w * gblocks;
  if (tiles > 0x7fffffffLL) return false;
  if (x == nullptr) return false;
  if (reinterpret_cast<uintptr_t>(x) % 16) return false;
  dcnv4::Launch l2 = *lc;
  dcnv4::Geo g2 = *g;
  if (!encode_x_map(p, dtype, x, GC * p->D, HWc, HH, &l2.xmap)) return false;
  int shift;
  conflict_factor(GC, L, cpl, nch, per_row * TH, &shift);
  g2.TH = TH; g2.TW = 8; g2.Gc = GC;
  g2.tiles_h = (int)tiles_h; g2.tiles_w = (int)tiles_w; g2.gblocks = (int)gblocks;
  g2.tiles_total = (int)tiles;
  g2.rot_shift = shift;
  g2.seg = seg_bytes / b;
  g2.HH = HH; g2.HW = HWc;
  g2.halo_box_bytes = halo_box;
  g2.halo_bytes = halo_bytes;
  g2.unit = unit;
  g2.upp = segB_raw / unit;
  g2.fd_gb = make_fastdiv((unsigned)gblocks);
  g2.fd_tw = make_fastdiv((unsigned)tiles_w);
  g2.fd_th = make_fastdiv((unsigned)tiles_h);
  g2.fd_upp = make_fastdiv((unsigned)g2.upp);
  l2.halo = true;
  l2.ppc = TH * 8;
  l2.threads = per_row * TH;
  l2.ctas = tiles;
  l2.smem = smem;
  *lc = l2;
  *g = g2;
  return true;
}

// Backward on the paper's grid: TMA halo + binned (counting-sort) grad_input scatter
// (bwd33_kernel).  Same tile as the forward; shared memory is single-buffered (two CTAs
// per SM overlap each other's loads).  Needs x and gy pointers for the TMA maps.
bool plan_bwd33(const dcnv4_params* p, int dtype, int64_t Ho, int64_t Wo, const void* x,
                const void* gy, dcnv4::Launch* lc, dcnv4::Geo* g) {
  const char* path = dcnv4::ablation(dcnv4::kAblBwdPath);
  if (path && path[0] == 'g') return false;
  if (p->kernel_h != 3 || p->kernel_w != 3 || p->stride_h != 1 || p->stride_w != 1 ||
      p->dilation_h != 1 || p->dilation_w != 1)
    return false;
  const int b = elem_size(dtype);
  const int nch = lc->nch, cpl = lc->cpl, L = lc->lanes;
  const int GC = nch >= 8 ? 1 : 8 / nch;
  if (p->G % GC) return false;
  const int DG = p->D;
  const int PB = GC * DG * b;
  const int per_row = 8 * GC * L;
  // fp32: 224-thread tiles (TH = 7 at 32 threads per tile row) whose shared memory (5-B bin
  // entries) and registers fit three CTAs per SM; fp16/bf16: 256 threads, two CTAs
  int TH = (b == 4 ? 224 : 256) / per_row;
  if (TH < 1) return false;
  const char* th_env = dcnv4::ablation(dcnv4::kAblBwd33TH);
  if (th_env && *th_env) TH = std::max(1, std::min(TH, atoi(th_env)));
  if (TH > Ho) TH = (int)Ho;
  const int K = 9;
  const int S = p->om_stride ? p->om_stride : 3 * p->G * K;
  const int segB_raw = GC * 3 * K * b;
  int unit = 0;
  for (int u : {8, 4})
    if ((S * b) % u == 0 && segB_raw % u == 0) { unit = u; break; }
  if (!unit) return false;
  // the kernels form a tile pixel's offset_mask source offset (row * Wo*S*b + col * S*b)
  // in 32-bit unsigned arithmetic
  if ((long long)(TH + 1) * std::max<int64_t>(Wo, 8) * S * b >= (1LL << 32)) return false;
  int seg_bytes = (segB_raw + 15) & ~15;
  if ((seg_bytes / 16) % 2 == 0) seg_bytes += 16;
  const int npix = TH * 8, HH = TH + 6, NT = HH * 14;
  if (NT > (int)sizeof(g->p4ord)) return false;
  auto up = [](size_t v, size_t a) { return (v + a - 1) / a * a; };
  size_t o = 0;
  const int halo_box = HH * 14 * PB;
  o = up((size_t)halo_box, 128);
  const int o_gy = (int)o;
  const int gy_box = npix * GC * DG * b;
  o = up(o + gy_box, 128);
  const int o_om = (int)o;
  o = up(o + (size_t)npix * seg_bytes, 16);
  const int o_gom = -1;  // grad_offset_mask goes straight from registers to memory
  const int o_cnt = (int)o;
  o = up(o + ((size_t)GC * NT + 1) * 4, 16);
  const int o_slot = (int)o;
  o = up(o + (size_t)GC * NT * 4, 16);  // fill pointers
  const int o_ent = (int)o;
  // bin entries (+ one pad slot per bin): fp32 5 B {a fp32} + {src u8} in two arrays,
  // half 4 B {a in T | src << 16}
  const size_t ent_cap = (size_t)GC * npix * 36 + (size_t)GC * NT;
  o = up(o + ent_cap * (b == 4 ? 5 : 4), 16);
  const int o_wsum = (int)o;
  o = up(o + 33 * 4, 16);
  const int o_bar = (int)o;
  const size_t smem = o + 16;
  if (smem > 227 * 1024) return false;
  const long long tiles_h = (Ho + TH - 1) / TH, tiles_w = (Wo + 7) / 8, gblocks = p->G / GC;
  const long long tiles = (long long)p->N * tiles_h * tiles_w * gblocks;
  if (tiles > 0x7fffffffLL) return false;
  if (!x || !gy || reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(gy) % 16)
    return false;
  dcnv4::Launch l2 = *lc;
  dcnv4::Geo g2 = *g;
  if (!encode_x_map(p, dtype, x, GC * DG, 14, HH, &l2.xmap)) return false;
  if (!encode_nhwc_map(dtype, gy, p->N, Ho, Wo, (int64_t)p->G * DG, GC * DG, 8, TH, &l2.gymap))
    return false;
  int shift;
  conflict_factor(GC, L, cpl, nch, per_row * TH, &shift);
  g2.TH = TH; g2.TW = 8; g2.Gc = GC;
  g2.tiles_h = (int)tiles_h; g2.tiles_w = (int)tiles_w; g2.gblocks = (int)gblocks;
  g2.tiles_total = (int)tiles;
  g2.rot_shift = shift;
  g2.seg = seg_bytes / b;
  g2.HH = HH; g2.HW = 14;
  g2.halo_box_bytes = halo_box;
  g2.halo_bytes = (int)up((size_t)halo_box, 128);
  g2.gy_box_bytes = gy_box;
  g2.o_gy = o_gy; g2.o_om = o_om; g2.o_gom = o_gom; g2.o_cnt = o_cnt; g2.o_slot = o_slot;
  g2.o_ent = o_ent; g2.o_wsum = o_wsum; g2.o_bar = o_bar;
  g2.ent_cap = (int)ent_cap;
  {  // P4 bin order: expected entry count for U(-2,2)-like offsets, separable in y and x.
    // A sample of output row py lands (floor) on halo row py + j + 2 + floor(dy), j in
    // {0,1,2}, floor(dy) in {-2..1}; its corners cover that row and the next.
    auto profile = [](int n_out, int n_halo, double* prof) {
      double w[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int j = 0; j < 3; ++j)
        for (int f = 0; f < 4; ++f) { w[j + f] += 0.5; w[j + f + 1] += 0.5; }
      for (int r = 0; r < n_halo; ++r) {
        prof[r] = 0;
        for (int q = 0; q < n_out; ++q)
          if (r - q >= 0 && r - q < 7) prof[r] += w[r - q];
      }
    };
    double py_[32], px_[32];
    profile(TH, HH, py_);
    profile(8, 14, px_);
    int idx[200];
    for (int i = 0; i < NT; ++i) idx[i] = i;
    const char* ord = dcnv4::ablation(dcnv4::kAblP4Order);
    if (!(ord && *ord == '0'))
      std::stable_sort(idx, idx + NT, [&](int a, int b2) {
        return py_[a / 14] * px_[a % 14] > py_[b2 / 14] * px_[b2 % 14];
      });
    for (int i = 0; i < NT; ++i) g2.p4ord[i] = (unsigned char)idx[i];
  }
  g2.unit = unit;
  g2.upp = segB_raw / unit;
  g2.fd_gb = make_fastdiv((unsigned)gblocks);
  g2.fd_tw = make_fastdiv((unsigned)tiles_w);
  g2.fd_th = make_fastdiv((unsigned)tiles_h);
  g2.fd_upp = make_fastdiv((unsigned)g2.upp);
  l2.halo = true;
  l2.ppc = npix;
  l2.threads = per_row * TH;
  l2.ctas = tiles;
  l2.smem = smem;
  *lc = l2;
  *g = g2;
  return true;
}

int make_launch(const dcnv4_params* p, int dtype, int pass, int64_t Ho, int64_t Wo,
                dcnv4::Launch* lc, dcnv4::Geo* g, const void* x = nullptr,
                const void* gy = nullptr, int th_force = 0) {
  const int b = elem_size(dtype);
  const int nch = p->D * b / 16;
  int cpl = default_cpl(nch, pass);
  const char* env = dcnv4::ablation(pass == 0 ? dcnv4::kAblFwdCpl : dcnv4::kAblBwdCpl);
  if (env && *env) {
    int v = atoi(env);
    if (cpl_supported(nch, v)) cpl = v;
  }
  const int lanes = nch / cpl;
  const int K = p->kernel_h * p->kernel_w;
  const int S = p->om_stride ? p->om_stride : 3 * p->G * K;
  const TileChoice tc = choose_tile(p, b, nch, cpl, Ho, Wo, false);
  const int npix = tc.TH * tc.TW;
  // per-pixel om segment in shared memory: 16-B aligned, and an odd number of 16-B
  // units so the rows of the <= 8 pixels a warp covers fall in distinct bank quads
  int seg_bytes = ((tc.Gc * 3 * K * b) + 15) & ~15;
  if ((seg_bytes / 16) % 2 == 0) seg_bytes += 16;
  lc->nch = nch;
  lc->cpl = cpl;
  lc->lanes = lanes;
  lc->ppc = npix;
  lc->threads = ((npix * tc.Gc * lanes + 31) / 32) * 32;
  const long long tiles_h = (Ho + tc.TH - 1) / tc.TH, tiles_w = (Wo + tc.TW - 1) / tc.TW;
  lc->ctas = (long long)p->N * tiles_h * tiles_w * (p->G / tc.Gc);
  lc->smem = (size_t)2 * npix * seg_bytes;  // double-buffered om tile
  if (pass == 1) lc->smem = ((lc->smem + 15) & ~(size_t)15) + (size_t)npix * tc.Gc * 3 * K * sizeof(float);
  lc->k33 = p->kernel_h == 3 && p->kernel_w == 3;
  lc->unit = p->offset_scale == 1.0f;
  if (lc->threads > kMaxThreads)
    return fail(DCNV4_ERR_UNSUPPORTED, "CTA of %d threads exceeds %d", lc->threads, kMaxThreads);
  if (lc->smem > 227 * 1024)
    return fail(DCNV4_ERR_UNSUPPORTED, "offset_mask tile needs %zu B of shared memory", lc->smem);
  if (lc->ctas > 0x7fffffffLL)
    return fail(DCNV4_ERR_SHAPE, "too many CTAs (N*Ho*Wo too large)");
  g->H = (int)p->H; g->W = (int)p->W; g->Ho = (int)Ho; g->Wo = (int)Wo;
  g->G = p->G; g->D = p->D; g->C = p->G * p->D; g->S = S; g->K = K;
  g->kh = p->kernel_h; g->kw = p->kernel_w; g->sh = p->stride_h; g->sw = p->stride_w;
  g->ph = p->pad_h; g->pw = p->pad_w; g->dh = p->dilation_h; g->dw = p->dilation_w;
  g->cy = p->dilation_h * (p->kernel_h - 1) / 2;
  g->cx = p->dilation_w * (p->kernel_w - 1) / 2;
  g->s = p->offset_scale;
  g->softmax = p->softmax;
  g->TH = tc.TH; g->TW = tc.TW; g->Gc = tc.Gc;
  g->tiles_h = (int)tiles_h; g->tiles_w = (int)tiles_w; g->gblocks = p->G / tc.Gc;
  g->rot_shift = tc.rot_shift;
  g->seg = seg_bytes / b;
  lc->halo = false;
  if (pass == 0) plan_fwd33(p, dtype, Ho, Wo, x, lc, g, th_force);
  else plan_bwd33(p, dtype, Ho, Wo, x, gy, lc, g);
  g->tiles_total = (int)lc->ctas;
  lc->persistent = dcnv4::ablation(dcnv4::kAblNonPersistent)[0] != '1';
  lc->det = pass == 1 && p->deterministic;
  {  // ceil(log2(Ho*Wo*K)): bound on the contributions one input element receives
    const long long cnt = (long long)Ho * Wo * K;
    int lcnt = 0;
    while ((1LL << lcnt) < cnt) ++lcnt;
    g->det_lc = lcnt;
  }
  g->detmax = nullptr;
  return DCNV4_OK;
}

bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

int cuda_fail(cudaError_t e, const char* what) {
  return fail(DCNV4_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace

// shared with msda.cu: one thread-local message for every entry point of the library
void dcnv4_internal_set_error(const char* msg) { snprintf(g_err, sizeof(g_err), "%s", msg); }

extern "C" {

int dcnv4_version(void) { return DCNV4_VERSION; }

const char* dcnv4_last_error(void) { return g_err; }

int dcnv4_output_size(const dcnv4_params* p, int64_t* H_out, int64_t* W_out) {
  g_err[0] = 0;
  if (!H_out || !W_out) return fail(DCNV4_ERR_INVALID_ARG, "H_out/W_out is NULL");
  int64_t Ho, Wo;
  int rc = validate_geometry(p, DCNV4_F32, &Ho, &Wo);
  if (rc != DCNV4_OK && rc != DCNV4_ERR_UNSUPPORTED) return rc;
  if (rc == DCNV4_ERR_UNSUPPORTED) g_err[0] = 0;  // size is defined even if unsupported
  const int64_t h = p->H + 2 * (int64_t)p->pad_h - (int64_t)p->dilation_h * (p->kernel_h - 1) - 1;
  const int64_t w = p->W + 2 * (int64_t)p->pad_w - (int64_t)p->dilation_w * (p->kernel_w - 1) - 1;
  if (h < 0 || w < 0) return fail(DCNV4_ERR_SHAPE, "output is empty");
  *H_out = h / p->stride_h + 1;
  *W_out = w / p->stride_w + 1;
  return DCNV4_OK;
}

int dcnv4_launch_info(const dcnv4_params* p, dcnv4_dtype dtype, int pass, int32_t* lanes,
                      int32_t* chunks_per_lane, int32_t* pixels_per_cta,
                      int32_t* threads_per_cta, int64_t* ctas) {
  g_err[0] = 0;
  int64_t Ho, Wo;
  int rc = validate_geometry(p, dtype, &Ho, &Wo);
  if (rc) return rc;
  dcnv4::Launch lc;
  dcnv4::Geo g;
  rc = make_launch(p, dtype, pass ? 1 : 0, Ho, Wo, &lc, &g, reinterpret_cast<const void*>(256),
                   reinterpret_cast<const void*>(256));
  if (rc) return rc;
  if (lanes) *lanes = lc.lanes;
  if (chunks_per_lane) *chunks_per_lane = lc.cpl;
  if (pixels_per_cta) *pixels_per_cta = lc.ppc;
  if (threads_per_cta) *threads_per_cta = lc.threads;
  if (ctas) *ctas = lc.ctas;
  return DCNV4_OK;
}

int dcnv4_forward(const dcnv4_params* p, dcnv4_dtype dtype, const void* input,
                  const void* offset_mask, void* output, void* stream) {
  g_err[0] = 0;
  int64_t Ho, Wo;
  int rc = validate_geometry(p, dtype, &Ho, &Wo);
  if (rc) return rc;
  if (p->N == 0) return DCNV4_OK;
  if (!input) return fail(DCNV4_ERR_INVALID_ARG, "input is NULL");
  if (!offset_mask) return fail(DCNV4_ERR_INVALID_ARG, "offset_mask is NULL");
  if (!output) return fail(DCNV4_ERR_INVALID_ARG, "output is NULL");
  if (!aligned16(input)) return fail(DCNV4_ERR_MISALIGNED, "input is not 16-byte aligned");
  if (!aligned16(output)) return fail(DCNV4_ERR_MISALIGNED, "output is not 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(offset_mask) % elem_size(dtype))
    return fail(DCNV4_ERR_MISALIGNED, "offset_mask is not element aligned");
  dcnv4::Launch lc;
  dcnv4::Geo g;
  rc = make_launch(p, dtype, 0, Ho, Wo, &lc, &g, input);
  if (rc) return rc;
  lc.stream = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (dtype) {
    case DCNV4_F32: e = dcnv4::launch_fwd_f32(lc, g, input, offset_mask, output); break;
    case DCNV4_F16: e = dcnv4::launch_fwd_f16(lc, g, input, offset_mask, output); break;
    default: e = dcnv4::launch_fwd_bf16(lc, g, input, offset_mask, output); break;
  }
  if (e != cudaSuccess) return cuda_fail(e, "dcnv4_forward launch");
  return DCNV4_OK;
}

static_assert(sizeof(dcnv4::Fwd33Group) <= 32000, "grouped-forward kernel parameters exceed 32 KB");

int dcnv4_forward_grouped(const dcnv4_params* const* params, int32_t count, dcnv4_dtype dtype,
                          const void* const* inputs, const void* const* offset_masks, void* const* outputs,
                          void* stream) {
  g_err[0] = 0;
  if (count < 1 || count > dcnv4::kMaxGroup)
    return fail(DCNV4_ERR_INVALID_ARG, "count = %d must be in [1, %d]", count, dcnv4::kMaxGroup);
  if (!params || !inputs || !offset_masks || !outputs)
    return fail(DCNV4_ERR_INVALID_ARG, "params/inputs/offset_masks/outputs array is NULL");
  int64_t Ho[dcnv4::kMaxGroup], Wo[dcnv4::kMaxGroup];
  for (int i = 0; i < count; ++i) {  // validate every problem before launching anything
    const dcnv4_params* p = params[i];
    int rc = validate_geometry(p, dtype, &Ho[i], &Wo[i]);
    if (rc) {
      char m[512];
      snprintf(m, sizeof(m), "problem %d: %s", i, g_err);
      return fail(rc, "%s", m);
    }
    if (p->N == 0) continue;
    if (!inputs[i] || !offset_masks[i] || !outputs[i])
      return fail(DCNV4_ERR_INVALID_ARG, "problem %d: input/offset_mask/output is NULL", i);
    if (!aligned16(inputs[i]) || !aligned16(outputs[i]))
      return fail(DCNV4_ERR_MISALIGNED, "problem %d: input/output not 16-byte aligned", i);
    if (reinterpret_cast<uintptr_t>(offset_masks[i]) % elem_size(dtype))
      return fail(DCNV4_ERR_MISALIGNED, "problem %d: offset_mask is not element aligned", i);
  }
  // one launch when every non-empty problem takes the TMA-halo kernel with the same
  // template instantiation and tile shape; otherwise one dcnv4_forward per problem
  dcnv4::Fwd33Group grp;
  grp.count = 0;
  dcnv4::Launch l0;
  bool one = true;
  int th = 0;
  long long tiles = 0;
  for (int i = 0; i < count && one; ++i) {
    const dcnv4_params* p = params[i];
    if (p->N == 0) continue;
    dcnv4::Launch lc;
    dcnv4::Geo g;
    if (make_launch(p, dtype, 0, Ho[i], Wo[i], &lc, &g, inputs[i], nullptr, th) != DCNV4_OK || !lc.halo) {
      one = false;
      break;
    }
    if (grp.count == 0) {
      l0 = lc;
      th = g.TH;
      // re-plan the first problem without its own tile-height clamp only if needed below
    }
    const dcnv4::Geo& g0 = grp.count ? grp.p[0].g : g;
    if (lc.nch != l0.nch || lc.cpl != l0.cpl || lc.unit != l0.unit || g.TH != th || g.seg != g0.seg ||
        g.halo_bytes != g0.halo_bytes || g.rot_shift != g0.rot_shift || lc.threads != l0.threads ||
        lc.smem != l0.smem) {
      one = false;
      break;
    }
    dcnv4::Fwd33Prob& q = grp.p[grp.count++];
    q.xmap = lc.xmap;
    q.g = g;
    q.x = inputs[i];
    q.om = offset_masks[i];
    q.y = outputs[i];
    q.t0 = (int)tiles;
    tiles += lc.ctas;
  }
  if (one && tiles >= 0x7fffffffLL) one = false;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!one) {
    for (int i = 0; i < count; ++i) {
      const int rc = dcnv4_forward(params[i], dtype, inputs[i], offset_masks[i], outputs[i], stream);
      if (rc) return rc;
    }
    return DCNV4_OK;
  }
  if (grp.count == 0) return DCNV4_OK;
  grp.tiles_total = (int)tiles;
  l0.ctas = tiles;
  l0.stream = st;
  cudaError_t e;
  switch (dtype) {
    case DCNV4_F32: e = dcnv4::launch_fwd_group_f32(l0, grp.p[0].g, &grp); break;
    case DCNV4_F16: e = dcnv4::launch_fwd_group_f16(l0, grp.p[0].g, &grp); break;
    default: e = dcnv4::launch_fwd_group_bf16(l0, grp.p[0].g, &grp); break;
  }
  if (e != cudaSuccess) return cuda_fail(e, "dcnv4_forward_grouped launch");
  return DCNV4_OK;
}

size_t dcnv4_backward_workspace_bytes(const dcnv4_params* p, dcnv4_dtype dtype) {
  int64_t Ho, Wo;
  if (validate_geometry(p, dtype, &Ho, &Wo)) return 0;
  const size_t nelem = (size_t)p->N * p->H * p->W * p->G * p->D;
  if (p->deterministic)  // int64 accumulator + per-image {max|gy|, max|m|}
    return nelem * sizeof(long long) + (((size_t)p->N * 2 * sizeof(unsigned) + 15) & ~(size_t)15);
  if (dtype == DCNV4_F32) return 0;
  return nelem * sizeof(float);
}

int dcnv4_backward(const dcnv4_params* p, dcnv4_dtype dtype, const void* input,
                   const void* offset_mask, const void* grad_output, void* grad_input,
                   void* grad_offset_mask, void* workspace, size_t workspace_bytes,
                   void* stream) {
  g_err[0] = 0;
  int64_t Ho, Wo;
  int rc = validate_geometry(p, dtype, &Ho, &Wo);
  if (rc) return rc;
  if (p->N == 0) return DCNV4_OK;
  if (!input) return fail(DCNV4_ERR_INVALID_ARG, "input is NULL");
  if (!offset_mask) return fail(DCNV4_ERR_INVALID_ARG, "offset_mask is NULL");
  if (!grad_output) return fail(DCNV4_ERR_INVALID_ARG, "grad_output is NULL");
  if (!grad_input) return fail(DCNV4_ERR_INVALID_ARG, "grad_input is NULL");
  if (!grad_offset_mask) return fail(DCNV4_ERR_INVALID_ARG, "grad_offset_mask is NULL");
  if (!aligned16(input)) return fail(DCNV4_ERR_MISALIGNED, "input is not 16-byte aligned");
  if (!aligned16(grad_output)) return fail(DCNV4_ERR_MISALIGNED, "grad_output is not 16-byte aligned");
  if (!aligned16(grad_input)) return fail(DCNV4_ERR_MISALIGNED, "grad_input is not 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(offset_mask) % elem_size(dtype))
    return fail(DCNV4_ERR_MISALIGNED, "offset_mask is not element aligned");
  if (reinterpret_cast<uintptr_t>(grad_offset_mask) % elem_size(dtype))
    return fail(DCNV4_ERR_MISALIGNED, "grad_offset_mask is not element aligned");
  const size_t need = dcnv4_backward_workspace_bytes(p, dtype);
  if (need) {
    if (!workspace || workspace_bytes < need)
      return fail(DCNV4_ERR_WORKSPACE, "workspace of %zu bytes required, got %zu", need,
                  workspace ? workspace_bytes : (size_t)0);
    if (!aligned16(workspace)) return fail(DCNV4_ERR_MISALIGNED, "workspace is not 16-byte aligned");
  }
  dcnv4::Launch lc;
  dcnv4::Geo g;
  rc = make_launch(p, dtype, 1, Ho, Wo, &lc, &g, input, grad_output);
  if (rc) return rc;
  lc.stream = static_cast<cudaStream_t>(stream);
  const size_t nelem = (size_t)p->N * p->H * p->W * p->G * p->D;
  const int K = p->kernel_h * p->kernel_w;
  const int S = p->om_stride ? p->om_stride : 3 * p->G * K;
  cudaError_t e;
  if (p->deterministic) {
    // int64 fixed point (R19): maxima pass, backward, int64 -> T conversion
    long long* acc = static_cast<long long*>(workspace);
    unsigned* mx = reinterpret_cast<unsigned*>(acc + nelem);
    g.detmax = mx;
    e = cudaMemsetAsync(workspace, 0, need, lc.stream);
    if (e != cudaSuccess) return cuda_fail(e, "dcnv4_backward zero workspace");
    const int npix = (int)(Ho * Wo), C = p->G * p->D;
    switch (dtype) {
      case DCNV4_F32:
        e = dcnv4::launch_detmax_f32(grad_output, offset_mask, p->N, npix, C, S, p->G, K, p->softmax, mx, lc.stream);
        break;
      case DCNV4_F16:
        e = dcnv4::launch_detmax_f16(grad_output, offset_mask, p->N, npix, C, S, p->G, K, p->softmax, mx, lc.stream);
        break;
      default:
        e = dcnv4::launch_detmax_bf16(grad_output, offset_mask, p->N, npix, C, S, p->G, K, p->softmax, mx, lc.stream);
        break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "dcnv4_backward maxima");
    switch (dtype) {
      case DCNV4_F32: e = dcnv4::launch_bwd_f32(lc, g, input, offset_mask, grad_output, acc, grad_offset_mask); break;
      case DCNV4_F16: e = dcnv4::launch_bwd_f16(lc, g, input, offset_mask, grad_output, acc, grad_offset_mask); break;
      default: e = dcnv4::launch_bwd_bf16(lc, g, input, offset_mask, grad_output, acc, grad_offset_mask); break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "dcnv4_backward launch");
    const long long per_image = (long long)p->H * p->W * C;
    const long long nchunk = (long long)(nelem * elem_size(dtype) / 16);
    switch (dtype) {
      case DCNV4_F32: e = dcnv4::launch_detconv_f32(acc, mx, g.det_lc, per_image, grad_input, nchunk, lc.stream); break;
      case DCNV4_F16: e = dcnv4::launch_detconv_f16(acc, mx, g.det_lc, per_image, grad_input, nchunk, lc.stream); break;
      default: e = dcnv4::launch_detconv_bf16(acc, mx, g.det_lc, per_image, grad_input, nchunk, lc.stream); break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "dcnv4_backward convert");
    return DCNV4_OK;
  }
  float* gx32 = dtype == DCNV4_F32 ? static_cast<float*>(grad_input) : static_cast<float*>(workspace);
  e = cudaMemsetAsync(gx32, 0, nelem * sizeof(float), lc.stream);
  if (e != cudaSuccess) return cuda_fail(e, "dcnv4_backward zero grad_input");
  switch (dtype) {
    case DCNV4_F32:
      e = dcnv4::launch_bwd_f32(lc, g, input, offset_mask, grad_output, gx32, grad_offset_mask);
      break;
    case DCNV4_F16:
      e = dcnv4::launch_bwd_f16(lc, g, input, offset_mask, grad_output, gx32, grad_offset_mask);
      break;
    default:
      e = dcnv4::launch_bwd_bf16(lc, g, input, offset_mask, grad_output, gx32, grad_offset_mask);
      break;
  }
  if (e != cudaSuccess) return cuda_fail(e, "dcnv4_backward launch");
  if (dtype != DCNV4_F32) {
    const long long nchunk = (long long)(nelem / 8);
    e = dtype == DCNV4_F16 ? dcnv4::launch_convert_f16(gx32, grad_input, nchunk, lc.stream)
                           : dcnv4::launch_convert_bf16(gx32, grad_input, nchunk, lc.stream);
    if (e != cudaSuccess) return cuda_fail(e, "dcnv4_backward convert");
  }
  return DCNV4_OK;
}

}  // extern "C"
