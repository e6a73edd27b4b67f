// om_linear.cu -- the fused offset/mask linear layer of the DCNv4 module (
// include/dcnv4_module.h) as a persistent tcgen05 GEMM for sm_100a:
//
//   om[R][S] = feat[R][C_in] . weight[J][C_in]^T + bias   (columns >= J written 0)
//
// Both operands are K-major ("TN"), the native tcgen05 operand order.  One CTA per SM
// loops over 128 x BN output tiles (n fastest, so the CTAs working on one 128-row block
// of feat share it through L2).  Warp roles:
//   warp 0 (one lane)  TMA producer: A (128 x 64) and B (BN x 64) boxes, 128-B swizzle,
//                      into a `stages`-deep shared-memory ring (full/empty mbarriers);
//   warp 1 (one lane)  MMA issuer: 4 x tcgen05.mma.kind::f16 (M=128, N=BN, K=16) per
//                      64-wide k block into one of two TMEM accumulators (BN fp32
//                      columns each), tcgen05.commit frees the smem slot / signals the
//                      epilogue;
//   warp 2             TMEM allocator (2*BN columns, power of two);
//   warps 4-7          epilogue: warp q reads TMEM lanes 32q..32q+31 (one output row per
//                      thread) with tcgen05.ld.32x32b, adds the bias (fp32, from smem),
//                      rounds to T, writes 64-column slabs into a 128-B-swizzled staging
//                      buffer (conflict-free) and stores them with a TMA bulk tensor
//                      store (rows >= R and columns >= S are clipped by the hardware).
// The accumulators are double-buffered, so the epilogue of tile i overlaps the MMAs of
// tile i+1 and the TMA loads of tiles i+1..i+stages.
#include "../../include/dcnv4_module.h"
#include "sm100_tc.cuh"

namespace oml {

struct Args {
  int R;        // rows
  int S;        // om row stride (columns written)
  int J;        // real output columns (3GK)
  int BN;       // tile width (64..256, multiple of 64)
  int nb;       // column tiles
  int kb;       // k blocks = ceil(C_in / 64)
  int stages;
  long long tiles;
  uint32_t idesc;  // tcgen05 instruction descriptor
  uint32_t tmem_cols;
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    om_linear_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                     const __grid_constant__ CUtensorMap omap, const T* __restrict__ bias, Args a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int BN = a.BN, stages = a.stages;
  const uint32_t B_BYTES = (uint32_t)BN * 128u;
  // carve: A ring | B ring | epilogue staging (4 warps x 2 slabs) | bias | barriers
  const uint32_t sA = base;
  const uint32_t sB = sA + stages * A_BYTES;
  const uint32_t sStg = sB + stages * B_BYTES;
  float* sBias = reinterpret_cast<float*>(gbase + (sStg + 8 * STG_BYTES - base));
  const uint32_t nbias = (uint32_t)a.nb * BN;
  const uint32_t sBar = (sStg + 8 * STG_BYTES + nbias * 4 + 7u) & ~7u;
  const uint32_t full = sBar, empty = sBar + 8 * stages, tfull = sBar + 16 * stages,
                 tempty = tfull + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (tempty + 16 - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t i = threadIdx.x; i < nbias; i += kThreads)
    sBias[i] = (bias != nullptr && (int)i < a.J) ? Cvt<T>::f(bias + i) : 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull + 8 * s, 1);
      mbar_init(tempty + 8 * s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&omap)) : "memory");
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

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        const int m = (int)(t / a.nb), n = (int)(t % a.nb);
        for (int k = 0; k < a.kb; ++k) {
          mbar_wait(empty + 8 * s, ph ^ 1);
          mbar_expect_tx(full + 8 * s, A_BYTES + B_BYTES);
          tma_load_2d(sA + s * A_BYTES, &amap, k * BK, m * BM, full + 8 * s);
          tma_load_2d(sB + s * B_BYTES, &bmap, k * BK, n * BN, full + 8 * s);
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
        mbar_wait(tempty + 8 * acc, aph ^ 1);
        fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int k = 0; k < a.kb; ++k) {
          mbar_wait(full + 8 * s, ph);
          fence_after();
          const uint64_t ad = sdesc(sA + s * A_BYTES), bd = sdesc(sB + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)  // +32 B along K inside the swizzle atom
            mma_f16(d, ad + 2 * kk, bd + 2 * kk, a.idesc, (k | kk) != 0);
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
  } else if (warp >= 4) {  // ---- epilogue
    const int q = warp - 4;
    const uint32_t stg0 = sStg + (uint32_t)q * 2 * STG_BYTES;
    const int row = lane;
    int acc = 0, slab = 0;
    uint32_t aph = 0;
    for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      const int m = (int)(t / a.nb), n = (int)(t % a.nb);
      mbar_wait(tfull + 8 * acc, aph);
      fence_after();
      for (int j = 0; j < BN / 64; ++j) {
        const int col = n * BN + j * 64;
        if (col >= a.S) break;
        uint32_t r[64];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + j * 64);
        tmem_ld32(ta, r);
        tmem_ld32(ta + 32, r + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e)
          pk[e] = Cvt<T>::pack(__uint_as_float(r[2 * e]) + sBias[col + 2 * e],
                               __uint_as_float(r[2 * e + 1]) + sBias[col + 2 * e + 1]);
        const uint32_t buf = stg0 + (uint32_t)(slab & 1) * STG_BYTES;
        // the TMA store issued from this buffer two slabs ago must have read it
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
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + 8 * acc);
      acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------- host side

// Tile plan: BN = min(256, S rounded up to 64), nb = ceil(S / BN); stages fill the
// shared-memory budget (<= 4).
bool plan(int S, int J, int C_in, long long R, int dtype, Args* a, size_t* smem) {
  a->R = (int)R;
  a->S = S;
  a->J = J;
  int s64 = (S + 63) / 64 * 64;
  a->BN = s64 < 256 ? s64 : 256;
  a->nb = (S + a->BN - 1) / a->BN;
  a->kb = (C_in + BK - 1) / BK;
  a->tiles = (R + BM - 1) / BM * (long long)a->nb;
  a->idesc = (1u << 4) | ((dtype == DCNV4_BF16 ? 1u : 0u) << 7) | ((dtype == DCNV4_BF16 ? 1u : 0u) << 10) |
             ((uint32_t)(a->BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  a->tmem_cols = a->BN * 2 <= 256 ? (a->BN * 2 <= 128 ? 128 : 256) : 512;
  const size_t fixed = 1024 + 8 * STG_BYTES + (size_t)a->nb * a->BN * 4 + 16 * 6 + 64;
  const size_t per = A_BYTES + (size_t)a->BN * 128;
  const size_t budget = 227 * 1024;
  int st = (int)((budget - fixed) / per);
  if (st > 4) st = 4;
  if (st < 2) return false;
  a->stages = st;
  *smem = fixed + (size_t)st * per + 16 * (size_t)st;
  return *smem <= budget;
}


}  // namespace oml

extern "C" {

int dcnv4_offset_mask_linear(const dcnv4_params* p, dcnv4_dtype dtype, int32_t C_in, const void* feat,
                             const void* weight, const void* bias, void* offset_mask, void* stream) {
  using namespace oml;
  int64_t Ho = 0, Wo = 0;
  int rc = dcnv4_output_size(p, &Ho, &Wo);  // validates p, sets last_error
  if (rc != DCNV4_OK) return rc;
  dcnv4_internal_set_error("");
  if (dtype != DCNV4_F32 && dtype != DCNV4_F16 && dtype != DCNV4_BF16)
    return fail(DCNV4_ERR_INVALID_ARG, "dtype %d is not DCNV4_F32/F16/BF16", (int)dtype);
  if (dtype == DCNV4_F32)
    return fail(DCNV4_ERR_UNSUPPORTED, "dtype DCNV4_F32: the tcgen05 linear takes F16/BF16 operands");
  const long long J = 3LL * p->G * p->kernel_h * p->kernel_w;
  const long long S = p->om_stride ? p->om_stride : J;
  if (S < J) return fail(DCNV4_ERR_SHAPE, "om_stride %lld < 3*G*K = %lld", S, J);
  if (C_in < 8 || C_in % 8)
    return fail(DCNV4_ERR_UNSUPPORTED, "C_in = %d must be a positive multiple of 8 (16-B rows)", C_in);
  if (S % 8) return fail(DCNV4_ERR_UNSUPPORTED, "om_stride S = %lld must be a multiple of 8 (16-B rows)", S);
  if (J > (1 << 20)) return fail(DCNV4_ERR_UNSUPPORTED, "3*G*K = %lld too large", J);
  const long long R = p->N * Ho * Wo;
  if (R >= (1LL << 31)) return fail(DCNV4_ERR_SHAPE, "rows N*Ho*Wo = %lld must be < 2^31", R);
  if (R == 0) return DCNV4_OK;
  if (!feat || !weight || !offset_mask)
    return fail(DCNV4_ERR_INVALID_ARG, "%s is NULL", !feat ? "feat" : !weight ? "weight" : "offset_mask");
  if (((uintptr_t)feat | (uintptr_t)weight | (uintptr_t)offset_mask) & 15)
    return fail(DCNV4_ERR_MISALIGNED, "%s is not 16-B aligned",
                ((uintptr_t)feat & 15) ? "feat" : ((uintptr_t)weight & 15) ? "weight" : "offset_mask");
  if ((uintptr_t)bias & 1) return fail(DCNV4_ERR_MISALIGNED, "bias is not 2-B aligned");
  Args a;
  size_t smem = 0;
  if (!plan((int)S, (int)J, C_in, R, dtype, &a, &smem))
    return fail(DCNV4_ERR_UNSUPPORTED, "om_stride %lld: bias table exceeds shared memory", S);
  CUtensorMap am, bm, om;
  CUresult e1 = encode2d(&am, dtype, feat, R, C_in, BK, BM);
  CUresult e2 = encode2d(&bm, dtype, weight, J, C_in, BK, a.BN);
  CUresult e3 = encode2d(&om, dtype, offset_mask, R, S, 64, 32);
  if (e1 != CUDA_SUCCESS || e2 != CUDA_SUCCESS || e3 != CUDA_SUCCESS)
    return fail(DCNV4_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d/%d/%d)", (int)e1, (int)e2, (int)e3);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long grid = a.tiles < num_sms() ? a.tiles : num_sms();
  cudaError_t err;
  if (dtype == DCNV4_F16) {
    auto k = om_linear_kernel<__half>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)grid, kThreads, smem, st>>>(am, bm, om, static_cast<const __half*>(bias), a);
  } else {
    auto k = om_linear_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)grid, kThreads, smem, st>>>(am, bm, om, static_cast<const __nv_bfloat16*>(bias), a);
  }
  err = cudaGetLastError();
  if (err != cudaSuccess) return fail(DCNV4_ERR_CUDA, "om_linear launch: %s", cudaGetErrorString(err));
  return DCNV4_OK;
}

}  // extern "C"
