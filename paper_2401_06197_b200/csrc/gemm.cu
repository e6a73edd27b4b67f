// gemm.cu -- the dense contractions of the full DCNv4 module (include/dcnv4_module.h,
// SURVEY 8(f) NEXT-2): its 1x1 input/output projections ("a 1x1 point-wise
// convolution on x and y can be applied before and after", the full module
// of the rest of the models) and the backward of every linear layer of the module
// (grad_input and grad_weight), as one persistent tcgen05 GEMM for sm_100a:
//
//   C[M][N] = sum over two K segments of A_s[M][K_s] . B_s[N][K_s]^T
//
// Each operand is read by TMA in whichever orientation it has in memory:
//   K-major  (the contraction index is contiguous: activations in a forward linear,
//             weights in nn.Linear layout) -- box {64 k, 128 m} / {64 k, BN n};
//   MN-major (the output index is contiguous: weights in a grad_input product, every
//             operand of a grad_weight product, which contracts over pixels) -- boxes
//             {64 mn, 64 k}, 1024-B atoms of 8 k rows x 128 B, 8 KB per 64-wide mn block.
// Both are 128-B swizzled; the tcgen05 shared-memory descriptor says which (K-major: SBO
// 1024 B between 8-row groups; MN-major: LBO 8 KB between 64-wide mn blocks, SBO 1024 B
// between 8-k groups) and the instruction descriptor carries the a/b major bits.
//
// Warp roles as om_linear.cu (warp 0 lane 0 TMA producer into a `stages`-deep ring,
// warp 1 lane 0 MMA issuer into two TMEM accumulators, warp 2 TMEM allocator, warps 4-7
// epilogue).  Epilogues:
//   EPI_STORE  RN_T(acc + bias) -> 128-B swizzled staging -> TMA store (clipped to M x N);
//   EPI_RED    fp32 16-B vector reductions into a caller-zeroed fp32 [M][N] buffer: the
//              K range is split over CTAs (grad_weight contracts over all pixels).
// fp32 operands (the fp32 module path) run on the tf32 tensor cores as 3xTF32: warps 2-3
// split every staged tile into hi = x with the low 13 mantissa bits cleared (exactly
// tf32) and lo = x - hi (exact), and the MMA warp accumulates hi.hi + hi.lo + lo.hi --
// the dropped lo.lo term and lo's own tf32 rounding are <= ~2^-20 of each product, so
// the result meets the fp32 parity bar (1e-5) that a single tf32 pass (2^-11) misses.
#include "../../include/dcnv4_module.h"
#include "sm100_tc.cuh"

namespace oml {

enum { EPI_STORE = 0, EPI_RED = 1 };

struct GArgs {
  int M, N;            // output rows / columns
  int kb0, kb1;        // 64-wide k blocks of segment 0 / 1
  int kpb;             // k blocks per split
  int ksplit;          // K splits (EPI_RED); 1 otherwise
  int mb, nb;          // m / n tiles
  int BN, stages;
  long long tiles;     // mb * nb * ksplit
  uint32_t idesc, tmem_cols;
};

// MN-major swizzled operand: 128-B-wide mn blocks `lbo` bytes apart (LBO; one block =
// the stage's k rows x 128 B), k-row groups `sbo` bytes apart (SBO), descriptor version 1.
// 16-bit types: SWIZZLE_128B (16-B chunks within 128 B, 8-row atoms, SBO 1024 B).
// tf32: SWIZZLE_128B_BASE32B (32-B chunks within 128 B, 4-row atoms, SBO 512 B) -- the
// only MN-major layout the tf32 MMA reads; TMA writes it with SWIZZLE_128B_ATOM_32B.
template <bool TF32>
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t addr, uint32_t lbo) {
  constexpr uint64_t sbo = TF32 ? 512 : 1024, layout = TF32 ? 1 : 2;
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((sbo >> 4) << 32) |
         ((uint64_t)1 << 46) | (layout << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <typename T>
__device__ __forceinline__ float ld_bias(const T* p) { return Cvt<T>::f(p); }
template <>
__device__ __forceinline__ float ld_bias<float>(const float* p) { return *p; }

template <typename T, bool AMN, bool BMN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap amap0, const __grid_constant__ CUtensorMap bmap0,
                const __grid_constant__ CUtensorMap amap1, const __grid_constant__ CUtensorMap bmap1,
                const __grid_constant__ CUtensorMap omap, const T* __restrict__ bias,
                float* __restrict__ out32, void* __restrict__ out_t, GArgs a) {
  constexpr bool X3 = sizeof(T) == 4;           // fp32: 3xTF32 on the tf32 tensor cores
  constexpr int BKE = 128 / (int)sizeof(T);       // k (K-major) or mn (MN-major) per 128-B row
  constexpr int KI = X3 ? 8 : 16;                 // k per MMA instruction
  constexpr uint32_t MNBLK = (uint32_t)BKE * 128u;  // bytes of one 128-B-wide mn block of a stage
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int BN = a.BN, stages = a.stages;
  const uint32_t B_BYTES = (uint32_t)BN * 128u;
  const uint32_t sA = base;
  const uint32_t sB = sA + stages * A_BYTES;
  const uint32_t sAl = sB + stages * B_BYTES;                 // X3: lo parts
  const uint32_t sBl = sAl + (X3 ? stages * A_BYTES : 0u);
  const uint32_t sStg = sBl + (X3 ? stages * B_BYTES : 0u);
  const uint32_t stg_bytes = (EPI == EPI_STORE && !X3) ? 8 * STG_BYTES : 0u;
  const uint32_t nbias = EPI == EPI_STORE ? (uint32_t)a.nb * BN : 0u;
  float* sBias = reinterpret_cast<float*>(gbase + (sStg + stg_bytes - base));
  const uint32_t sBar = (sStg + stg_bytes + nbias * 4 + 7u) & ~7u;
  const uint32_t full = sBar, empty = sBar + 8 * stages, split = sBar + 16 * stages,
                 tfull = sBar + 24 * stages, tempty = tfull + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (tempty + 16 - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t i = threadIdx.x; i < nbias; i += kThreads)
    sBias[i] = (bias != nullptr && (int)i < a.N) ? ld_bias<T>(bias + i) : 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
      mbar_init(split + 8 * s, 2);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull + 8 * s, 1);
      mbar_init(tempty + 8 * s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int kbt = a.kb0 + a.kb1;

  // tile t -> (m, n, split); the split's k blocks [k0, k1)
  auto tile_of = [&](long long t, int& m, int& n, int& k0, int& k1) {
    const int ks = (int)(t % a.ksplit);
    const long long mn = t / a.ksplit;
    n = (int)(mn % a.nb);
    m = (int)(mn / a.nb);
    k0 = ks * a.kpb;
    k1 = k0 + a.kpb < kbt ? k0 + a.kpb : kbt;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        int m, n, k0, k1;
        tile_of(t, m, n, k0, k1);
        for (int kk = k0; kk < k1; ++kk) {
          const bool s1 = kk >= a.kb0;
          const CUtensorMap* am = s1 ? &amap1 : &amap0;
          const CUtensorMap* bm = s1 ? &bmap1 : &bmap0;
          const int kc = (s1 ? kk - a.kb0 : kk) * BKE;
          mbar_wait(empty + 8 * s, ph ^ 1);
          mbar_expect_tx(full + 8 * s, A_BYTES + B_BYTES);
          const uint32_t dA = sA + s * A_BYTES, dB = sB + s * B_BYTES;
          if constexpr (AMN) {  // [K][M] in memory: 128-B-wide m blocks of BKE k rows
#pragma unroll
            for (int j = 0; j < BM / BKE; ++j) tma_load_2d(dA + j * MNBLK, am, m * BM + j * BKE, kc, full + 8 * s);
          } else {
            tma_load_2d(dA, am, kc, m * BM, full + 8 * s);
          }
          if constexpr (BMN) {  // [K][N] in memory: BN / BKE blocks of BKE k rows
            for (int j = 0; j < BN / BKE; ++j) tma_load_2d(dB + j * MNBLK, bm, n * BN + j * BKE, kc, full + 8 * s);
          } else {
            tma_load_2d(dB, bm, kc, n * BN, full + 8 * s);
          }
          if (++s == stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        int m, n, k0, k1;
        tile_of(t, m, n, k0, k1);
        mbar_wait(tempty + 8 * acc, aph ^ 1);
        fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int kk = k0; kk < k1; ++kk) {
          mbar_wait((X3 ? split : full) + 8 * s, ph);
          fence_after();
          const uint64_t ad = AMN ? sdesc_mn<X3>(sA + s * A_BYTES, MNBLK) : sdesc(sA + s * A_BYTES);
          const uint64_t bd = BMN ? sdesc_mn<X3>(sB + s * B_BYTES, MNBLK) : sdesc(sB + s * B_BYTES);
          // advance per MMA: K-major +32 B inside the atom; MN-major +KI k rows (KI*128 B)
          constexpr uint64_t AST = AMN ? (KI * 128) >> 4 : 2, BST = BMN ? (KI * 128) >> 4 : 2;
          if constexpr (X3) {
            const uint64_t adl = AMN ? sdesc_mn<X3>(sAl + s * A_BYTES, MNBLK) : sdesc(sAl + s * A_BYTES);
            const uint64_t bdl = BMN ? sdesc_mn<X3>(sBl + s * B_BYTES, MNBLK) : sdesc(sBl + s * B_BYTES);
#pragma unroll
            for (int q = 0; q < BKE / KI; ++q) {
              const uint32_t first = (kk > k0 || q) ? 1u : 0u;
              mma_tf32(d, adl + AST * q, bd + BST * q, a.idesc, first);   // lo . hi
              mma_tf32(d, ad + AST * q, bdl + BST * q, a.idesc, 1u);      // hi . lo
              mma_tf32(d, ad + AST * q, bd + BST * q, a.idesc, 1u);       // hi . hi
            }
          } else {
#pragma unroll
            for (int q = 0; q < BKE / KI; ++q)
              mma_f16(d, ad + AST * q, bd + BST * q, a.idesc, (kk > k0 || q) ? 1u : 0u);
          }
          mma_commit(empty + 8 * s);
          if (++s == stages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(tfull + 8 * acc);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else if (X3 && (warp == 2 || warp == 3)) {  // ---- 3xTF32 split of each staged tile
    const int ct = threadIdx.x - 64;             // 64 threads
    int s = 0;
    uint32_t ph = 0;
    for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      int m, n, k0, k1;
      tile_of(t, m, n, k0, k1);
      for (int kk = k0; kk < k1; ++kk) {
        mbar_wait(full + 8 * s, ph);
        auto split16 = [&](uint32_t src, uint32_t lo) {
          uint4 v;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(src));
          const uint4 h = make_uint4(v.x & 0xffffe000u, v.y & 0xffffe000u, v.z & 0xffffe000u, v.w & 0xffffe000u);
          const float l0 = __uint_as_float(v.x) - __uint_as_float(h.x), l1 = __uint_as_float(v.y) - __uint_as_float(h.y);
          const float l2 = __uint_as_float(v.z) - __uint_as_float(h.z), l3 = __uint_as_float(v.w) - __uint_as_float(h.w);
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(src), "r"(h.x), "r"(h.y), "r"(h.z), "r"(h.w)
                       : "memory");
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(lo), "f"(l0), "f"(l1), "f"(l2), "f"(l3)
                       : "memory");
        };
        for (uint32_t o = (uint32_t)ct * 16; o < (uint32_t)A_BYTES; o += 64 * 16)
          split16(sA + s * A_BYTES + o, sAl + s * A_BYTES + o);
        for (uint32_t o = (uint32_t)ct * 16; o < B_BYTES; o += 64 * 16)
          split16(sB + s * B_BYTES + o, sBl + s * B_BYTES + o);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(split + 8 * s);
        if (++s == stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ---- epilogue
    const int q = warp - 4;
    const uint32_t stg0 = sStg + (uint32_t)q * 2 * STG_BYTES;
    const int row = lane;
    int acc = 0, slab = 0;
    uint32_t aph = 0;
    for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      int m, n, k0, k1;
      tile_of(t, m, n, k0, k1);
      mbar_wait(tfull + 8 * acc, aph);
      fence_after();
      const int grow = m * BM + q * 32 + row;
      for (int j = 0; j < BN / 64; ++j) {
        const int col = n * BN + j * 64;
        if (col >= a.N) break;
        uint32_t r[64];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + j * 64);
        tmem_ld32(ta, r);
        tmem_ld32(ta + 32, r + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if constexpr (EPI == EPI_RED) {
          if (grow < a.M) {
            float* dst = out32 + (long long)grow * a.N + col;
#pragma unroll
            for (int e = 0; e < 64; e += 4)
              if (col + e < a.N)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + e),
                             "f"(__uint_as_float(r[e])), "f"(__uint_as_float(r[e + 1])),
                             "f"(__uint_as_float(r[e + 2])), "f"(__uint_as_float(r[e + 3]))
                             : "memory");
          }
        } else if constexpr (X3) {  // fp32 output: the thread's row segment, 16-B stores
          if (grow < a.M) {
            float* dst = reinterpret_cast<float*>(const_cast<T*>(static_cast<const T*>(out_t))) +
                         (long long)grow * a.N + col;
#pragma unroll
            for (int e = 0; e < 64; e += 4)
              if (col + e < a.N)
                *reinterpret_cast<float4*>(dst + e) =
                    make_float4(__uint_as_float(r[e]) + sBias[col + e], __uint_as_float(r[e + 1]) + sBias[col + e + 1],
                                __uint_as_float(r[e + 2]) + sBias[col + e + 2],
                                __uint_as_float(r[e + 3]) + sBias[col + e + 3]);
          }
        } else {
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e)
            pk[e] = Cvt<T>::pack(__uint_as_float(r[2 * e]) + sBias[col + 2 * e],
                                 __uint_as_float(r[2 * e + 1]) + sBias[col + 2 * e + 1]);
          const uint32_t buf = stg0 + (uint32_t)(slab & 1) * STG_BYTES;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t dst = buf + (uint32_t)row * 128u + (uint32_t)((c ^ (row & 7)) * 16);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(pk[4 * c]),
                         "r"(pk[4 * c + 1]), "r"(pk[4 * c + 2]), "r"(pk[4 * c + 3])
                         : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&omap, buf, col, m * BM + q * 32);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++slab;
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + 8 * acc);
      acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
    if (EPI == EPI_STORE && !X3 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols)
                 : "memory");
  }
}

__device__ __forceinline__ void store_t(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_t(__half* p, float v) { *p = __float2half_rn(v); }
__device__ __forceinline__ void store_t(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// fp32 accumulator -> T (round to nearest even)
template <typename T>
__global__ void __launch_bounds__(256) f32_to_t_kernel(const float* __restrict__ src, T* __restrict__ dst,
                                                       long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    store_t(dst + i, src[i]);
}

// Column sums of a [rows][ld] T matrix over its first `cols` columns, fp32, accumulated
// into colsum[cols] (zeroed by the caller): the bias gradient of a linear layer.
// Block = 32 x 8 threads: x over 32 consecutive columns, y over row slices.
template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ g, long long rows, int ld, int cols,
                                                     int rows_per_block, float* __restrict__ colsum) {
  const int c = blockIdx.x * 32 + threadIdx.x;
  const long long r0 = (long long)blockIdx.y * rows_per_block;
  long long r1 = r0 + rows_per_block;
  if (r1 > rows) r1 = rows;
  float s = 0.f;
  if (c < cols)
    for (long long r = r0 + threadIdx.y; r < r1; r += 8) s += ld_bias<T>(g + r * ld + c);
  __shared__ float red[8][33];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    atomicAdd(colsum + c, t);
  }
}

// ---------------------------------------------------------------------------- host side

struct Operand {
  const void* ptr;
  long long rows, cols;  // as stored: row-major [rows][cols], cols contiguous
  bool mn;               // MN-major: rows index K (else rows index M or N, cols index K)
};

// 2-D map of an operand as stored; one 128-B row per box row (64 halves / 32 floats):
// K-major boxes {BKE, box_rows}, MN-major boxes {BKE, BKE}
inline CUresult encode_operand(CUtensorMap* map, int dtype, const Operand& o, int box_rows) {
  const int bke = dtype == DCNV4_F32 ? 32 : 64;
  const CUtensorMapSwizzle swz =
      (o.mn && dtype == DCNV4_F32) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  return encode2d(map, dtype, o.ptr, o.rows, o.cols, bke, o.mn ? bke : box_rows, swz);
}

size_t gemm_smem(int BN, int stages, int N, bool store, bool x3) {
  const int nb = (N + BN - 1) / BN;
  const size_t stage = (A_BYTES + (size_t)BN * 128) * (x3 ? 2 : 1);  // + lo parts (3xTF32)
  return 1024 + (size_t)stages * stage + (store && !x3 ? 8 * STG_BYTES : 0) +
         (store ? (size_t)nb * BN * 4 : 0) + 24 * (size_t)stages + 64 + 16;
}

template <typename T, bool AMN, bool BMN, int EPI>
cudaError_t launch_gemm(const CUtensorMap* m4, const CUtensorMap& om, const void* bias, float* out32, void* C,
                        const GArgs& a, size_t smem, unsigned grid, cudaStream_t st) {
  auto k = gemm_kernel<T, AMN, BMN, EPI>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kThreads, smem, st>>>(m4[0], m4[1], m4[2], m4[3], om, static_cast<const T*>(bias), out32, C, a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_gemm(bool amn, bool bmn, int epi, const CUtensorMap* m4, const CUtensorMap& om,
                          const void* bias, float* out32, void* C, const GArgs& a, size_t smem, unsigned grid,
                          cudaStream_t st) {
#define GEMM_CASE(A_, B_, E_)                                                                     \
  if (amn == A_ && bmn == B_ && epi == E_)                                                         \
    return launch_gemm<T, A_, B_, E_>(m4, om, bias, out32, C, a, smem, grid, st);
  GEMM_CASE(false, false, EPI_STORE)
  GEMM_CASE(false, true, EPI_STORE)
  GEMM_CASE(true, true, EPI_RED)
  GEMM_CASE(false, false, EPI_RED)
#undef GEMM_CASE
  return cudaErrorInvalidConfiguration;
}

// C[M][N] = A0 . B0^T (+ A1 . B1^T) (+ bias) as described at the top of the file.
// epi = EPI_STORE: C is T [M][N] row-major (16-B rows), bias [N] T or NULL.
// epi = EPI_RED:   out32 [M][N] fp32 += the product (zeroed by the caller).
int run_gemm(int dtype, long long M, long long N, const Operand& a0, const Operand& b0, long long K0,
             const Operand* a1, const Operand* b1, long long K1, int epi, void* C, const void* bias,
             float* out32, cudaStream_t st) {
  if (M <= 0 || N <= 0) return DCNV4_OK;
  const bool x3 = dtype == DCNV4_F32;
  const int bke = x3 ? 32 : 64;
  GArgs g;
  g.M = (int)M;
  g.N = (int)N;
  const int BN = N <= 64 ? 64 : N <= 128 ? 128 : 256;
  g.BN = BN;
  g.kb0 = (int)((K0 + bke - 1) / bke);
  g.kb1 = a1 ? (int)((K1 + bke - 1) / bke) : 0;
  g.mb = (int)((M + BM - 1) / BM);
  g.nb = (int)((N + BN - 1) / BN);
  const int kbt = g.kb0 + g.kb1;
  const int sms = num_sms();
  g.ksplit = 1;
  if (epi == EPI_RED) {  // split K so the output tiles x splits fill the SMs
    const long long mn = (long long)g.mb * g.nb;
    long long ks = (sms + mn - 1) / mn;
    if (ks > kbt) ks = kbt;
    g.ksplit = (int)(ks < 1 ? 1 : ks);
  }
  g.kpb = (kbt + g.ksplit - 1) / g.ksplit;
  g.ksplit = (kbt + g.kpb - 1) / g.kpb;
  g.tiles = (long long)g.mb * g.nb * g.ksplit;
  const bool amn = a0.mn, bmn = b0.mn;
  const uint32_t fmt = x3 ? 2u : (dtype == DCNV4_BF16 ? 1u : 0u);  // TF32 / BF16 / F16
  g.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  g.tmem_cols = BN * 2 <= 128 ? 128 : BN * 2 <= 256 ? 256 : 512;
  int stages = 4;
  while (stages > 2 && gemm_smem(BN, stages, (int)N, epi == EPI_STORE, x3) > 227 * 1024) --stages;
  g.stages = stages;
  const size_t smem = gemm_smem(BN, stages, (int)N, epi == EPI_STORE, x3);
  if (smem > 227 * 1024) return fail(DCNV4_ERR_UNSUPPORTED, "GEMM N = %lld: bias table exceeds shared memory", N);
  CUtensorMap m4[4], om;
  CUresult e[6] = {CUDA_SUCCESS, CUDA_SUCCESS, CUDA_SUCCESS, CUDA_SUCCESS, CUDA_SUCCESS, CUDA_SUCCESS};
  e[0] = encode_operand(&m4[0], dtype, a0, BM);
  e[1] = encode_operand(&m4[1], dtype, b0, BN);
  e[2] = encode_operand(&m4[2], dtype, a1 ? *a1 : a0, BM);
  e[3] = encode_operand(&m4[3], dtype, b1 ? *b1 : b0, BN);
  if (epi == EPI_STORE && !x3) e[4] = encode2d(&om, dtype, C, M, N, 64, 32);
  else om = m4[0];
  for (int i = 0; i < 5; ++i)
    if (e[i] != CUDA_SUCCESS) return fail(DCNV4_ERR_CUDA, "cuTensorMapEncodeTiled failed (operand %d: %d)", i, (int)e[i]);
  const unsigned grid = (unsigned)(g.tiles < sms ? g.tiles : sms);
  cudaError_t err =
      x3 ? dispatch_gemm<float>(amn, bmn, epi, m4, om, bias, out32, C, g, smem, grid, st)
      : dtype == DCNV4_F16
          ? dispatch_gemm<__half>(amn, bmn, epi, m4, om, bias, out32, C, g, smem, grid, st)
          : dispatch_gemm<__nv_bfloat16>(amn, bmn, epi, m4, om, bias, out32, C, g, smem, grid, st);
  if (err != cudaSuccess) return fail(DCNV4_ERR_CUDA, "gemm launch: %s", cudaGetErrorString(err));
  return DCNV4_OK;
}

int check_common(dcnv4_dtype dtype, const char* what) {
  if (dtype != DCNV4_F32 && dtype != DCNV4_F16 && dtype != DCNV4_BF16)
    return fail(DCNV4_ERR_INVALID_ARG, "%s: dtype %d is not DCNV4_F32/F16/BF16", what, (int)dtype);
  return DCNV4_OK;
}

// elements per 16 B (row pitches must be 16-B multiples for TMA)
int epv(dcnv4_dtype dtype) { return dtype == DCNV4_F32 ? 4 : 8; }

bool a16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace oml

extern "C" {

int dcnv4_linear(dcnv4_dtype dtype, int64_t M, int32_t K, int32_t N, const void* x, const void* weight,
                 const void* bias, void* y, void* stream) {
  using namespace oml;
  dcnv4_internal_set_error("");
  int rc = check_common(dtype, "dcnv4_linear");
  if (rc) return rc;
  if (M < 0 || K <= 0 || N <= 0) return fail(DCNV4_ERR_INVALID_ARG, "dcnv4_linear: M=%lld K=%d N=%d", (long long)M, K, N);
  if (K % epv(dtype) || N % epv(dtype))
    return fail(DCNV4_ERR_UNSUPPORTED, "dcnv4_linear: K = %d and N = %d must be multiples of %d (16-B rows)", K, N,
                epv(dtype));
  if (M >= (1LL << 31)) return fail(DCNV4_ERR_SHAPE, "dcnv4_linear: M = %lld must be < 2^31", (long long)M);
  if (M == 0) return DCNV4_OK;
  if (!x || !weight || !y) return fail(DCNV4_ERR_INVALID_ARG, "dcnv4_linear: %s is NULL", !x ? "x" : !weight ? "weight" : "y");
  if (!a16(x) || !a16(weight) || !a16(y)) return fail(DCNV4_ERR_MISALIGNED, "dcnv4_linear: x/weight/y must be 16-B aligned");
  if ((uintptr_t)bias % (dtype == DCNV4_F32 ? 4 : 2))
    return fail(DCNV4_ERR_MISALIGNED, "dcnv4_linear: bias is not element aligned");
  Operand a0{x, M, K, false}, b0{weight, N, K, false};
  return run_gemm(dtype, M, N, a0, b0, K, nullptr, nullptr, 0, EPI_STORE, y, bias, nullptr,
                  static_cast<cudaStream_t>(stream));
}

int dcnv4_linear_grad_input(dcnv4_dtype dtype, int64_t M, int32_t K, int32_t N0, const void* gy0, int32_t ld0,
                            const void* weight0, int32_t N1, const void* gy1, const void* weight1, void* gx,
                            void* stream) {
  using namespace oml;
  dcnv4_internal_set_error("");
  int rc = check_common(dtype, "dcnv4_linear_grad_input");
  if (rc) return rc;
  if (M < 0 || K <= 0 || N0 <= 0 || N1 < 0 || ld0 < N0)
    return fail(DCNV4_ERR_INVALID_ARG, "dcnv4_linear_grad_input: M=%lld K=%d N0=%d ld0=%d N1=%d", (long long)M, K, N0, ld0, N1);
  if (K % epv(dtype) || ld0 % epv(dtype) || N1 % epv(dtype))
    return fail(DCNV4_ERR_UNSUPPORTED, "dcnv4_linear_grad_input: K, ld0, N1 must be multiples of %d", epv(dtype));
  if (M >= (1LL << 31)) return fail(DCNV4_ERR_SHAPE, "dcnv4_linear_grad_input: M must be < 2^31");
  if (M == 0) return DCNV4_OK;
  if (!gy0 || !weight0 || !gx || (N1 && (!gy1 || !weight1)))
    return fail(DCNV4_ERR_INVALID_ARG, "dcnv4_linear_grad_input: NULL operand");
  if (!a16(gy0) || !a16(weight0) || !a16(gx) || (N1 && (!a16(gy1) || !a16(weight1))))
    return fail(DCNV4_ERR_MISALIGNED, "dcnv4_linear_grad_input: operands must be 16-B aligned");
  // gx[M][K] = gy0[M][:N0] . W0[N0][K] (+ gy1[M][N1] . W1[N1][K]): the weights are read
  // MN-major (output index K contiguous); columns N0..ld0 of gy0 meet zero-filled rows
  Operand a0{gy0, M, ld0, false}, b0{weight0, N0, K, true};
  Operand a1{gy1, M, N1, false}, b1{weight1, N1, K, true};
  return run_gemm(dtype, M, K, a0, b0, N0, N1 ? &a1 : nullptr, N1 ? &b1 : nullptr, N1, EPI_STORE, gx, nullptr,
                  nullptr, static_cast<cudaStream_t>(stream));
}

size_t dcnv4_linear_grad_weight_workspace_bytes(int32_t K, int32_t N) {
  return ((size_t)N * K + (size_t)N) * sizeof(float);
}

int dcnv4_linear_grad_weight(dcnv4_dtype dtype, int64_t M, int32_t K, int32_t N, const void* x, const void* gy,
                             int32_t ld_gy, void* grad_weight, void* grad_bias, void* workspace,
                             size_t workspace_bytes, void* stream) {
  using namespace oml;
  dcnv4_internal_set_error("");
  int rc = check_common(dtype, "dcnv4_linear_grad_weight");
  if (rc) return rc;
  if (M < 0 || K <= 0 || N <= 0 || ld_gy < N)
    return fail(DCNV4_ERR_INVALID_ARG, "dcnv4_linear_grad_weight: M=%lld K=%d N=%d ld_gy=%d", (long long)M, K, N, ld_gy);
  if (K % epv(dtype) || ld_gy % epv(dtype))
    return fail(DCNV4_ERR_UNSUPPORTED, "dcnv4_linear_grad_weight: K and ld_gy must be multiples of %d", epv(dtype));
  if (M >= (1LL << 31)) return fail(DCNV4_ERR_SHAPE, "dcnv4_linear_grad_weight: M must be < 2^31");
  if (!x || !gy || !grad_weight) return fail(DCNV4_ERR_INVALID_ARG, "dcnv4_linear_grad_weight: NULL operand");
  if (!a16(x) || !a16(gy) || !a16(grad_weight) || !a16(workspace))
    return fail(DCNV4_ERR_MISALIGNED, "dcnv4_linear_grad_weight: operands and workspace must be 16-B aligned");
  if ((uintptr_t)grad_bias % (dtype == DCNV4_F32 ? 4 : 2))
    return fail(DCNV4_ERR_MISALIGNED, "dcnv4_linear_grad_weight: grad_bias not element aligned");
  const size_t need = dcnv4_linear_grad_weight_workspace_bytes(K, N);
  if (!workspace || workspace_bytes < need)
    return fail(DCNV4_ERR_WORKSPACE, "dcnv4_linear_grad_weight: workspace of %zu bytes required, got %zu", need,
                workspace ? workspace_bytes : (size_t)0);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* acc = static_cast<float*>(workspace);
  float* bsum = acc + (size_t)N * K;
  cudaError_t e = cudaMemsetAsync(workspace, 0, need, st);
  if (e != cudaSuccess) return fail(DCNV4_ERR_CUDA, "dcnv4_linear_grad_weight memset: %s", cudaGetErrorString(e));
  if (M > 0) {
    // dW[N][K] = gy^T . x: both operands MN-major (the contraction runs over the M rows)
    Operand a0{gy, M, ld_gy, true}, b0{x, M, K, true};
    rc = run_gemm(dtype, N, K, a0, b0, M, nullptr, nullptr, 0, EPI_RED, nullptr, nullptr, acc, st);
    if (rc) return rc;
    if (grad_bias) {
      const int rpb = 4096;
      dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + rpb - 1) / rpb));
      if (dtype == DCNV4_F32)
        colsum_kernel<float><<<grid, dim3(32, 8), 0, st>>>(static_cast<const float*>(gy), M, ld_gy, N, rpb, bsum);
      else if (dtype == DCNV4_F16)
        colsum_kernel<__half><<<grid, dim3(32, 8), 0, st>>>(static_cast<const __half*>(gy), M, ld_gy, N, rpb, bsum);
      else
        colsum_kernel<__nv_bfloat16><<<grid, dim3(32, 8), 0, st>>>(static_cast<const __nv_bfloat16*>(gy), M, ld_gy, N,
                                                                    rpb, bsum);
    }
  }
  const long long n1 = (long long)N * K;
  const unsigned blocks = (unsigned)((n1 + 255) / 256 < 148 * 8 ? (n1 + 255) / 256 : 148 * 8);
  if (dtype == DCNV4_F32) {
    f32_to_t_kernel<float><<<blocks, 256, 0, st>>>(acc, static_cast<float*>(grad_weight), n1);
    if (grad_bias) f32_to_t_kernel<float><<<1, 256, 0, st>>>(bsum, static_cast<float*>(grad_bias), N);
  } else if (dtype == DCNV4_F16) {
    f32_to_t_kernel<__half><<<blocks, 256, 0, st>>>(acc, static_cast<__half*>(grad_weight), n1);
    if (grad_bias) f32_to_t_kernel<__half><<<1, 256, 0, st>>>(bsum, static_cast<__half*>(grad_bias), N);
  } else {
    f32_to_t_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(acc, static_cast<__nv_bfloat16*>(grad_weight), n1);
    if (grad_bias) f32_to_t_kernel<__nv_bfloat16><<<1, 256, 0, st>>>(bsum, static_cast<__nv_bfloat16*>(grad_bias), N);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DCNV4_ERR_CUDA, "dcnv4_linear_grad_weight launch: %s", cudaGetErrorString(e));
  return DCNV4_OK;
}

}  // extern "C"
