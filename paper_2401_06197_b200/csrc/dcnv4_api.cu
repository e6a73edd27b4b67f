// dcnv4_api.cu -- the C ABI of include/dcnv4.h: validation, launch configuration,
// dispatch.  Stateless apart from the thread-local error string; never allocates,
// synchronises or changes the device.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/dcnv4.h"
#include "dcnv4_kernels.cuh"
#include "dcnv4_launch.h"

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
constexpr int kTargetThreads = 256;

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

int make_launch(const dcnv4_params* p, int dtype, int pass, int64_t Ho, int64_t Wo,
                dcnv4::Launch* lc, dcnv4::Geo* g) {
  const int b = elem_size(dtype);
  const int nch = p->D * b / 16;
  int cpl = default_cpl(nch, pass);
  const char* env = getenv(pass == 0 ? "DCNV4_FWD_CPL" : "DCNV4_BWD_CPL");
  if (env && *env) {
    int v = atoi(env);
    if (cpl_supported(nch, v)) cpl = v;
  }
  // keep a pixel's G*lanes threads inside one CTA
  while (p->G * (nch / cpl) > kMaxThreads && cpl < nch && cpl_supported(nch, cpl * 2)) cpl *= 2;
  const int lanes = nch / cpl;
  const int gl = p->G * lanes;
  if (gl > kMaxThreads)
    return fail(DCNV4_ERR_UNSUPPORTED, "G*lanes = %d exceeds %d threads (G axis too large)", gl,
                kMaxThreads);
  const int K = p->kernel_h * p->kernel_w;
  const int S = p->om_stride ? p->om_stride : 3 * p->G * K;
  int ppc = kTargetThreads / gl;
  if (ppc < 1) ppc = 1;
  const long long P = (long long)p->N * Ho * Wo;
  lc->nch = nch;
  lc->cpl = cpl;
  lc->lanes = lanes;
  lc->ppc = ppc;
  lc->threads = ((ppc * gl + 31) / 32) * 32;
  lc->ctas = (P + ppc - 1) / ppc;
  size_t om_bytes = (((size_t)ppc * S * b + 16) + 15) & ~(size_t)15;
  lc->smem = om_bytes + (pass == 1 ? (size_t)ppc * S * 4 : 0);
  lc->k33 = p->kernel_h == 3 && p->kernel_w == 3;
  lc->unit = p->offset_scale == 1.0f;
  if (lc->smem > 227 * 1024)
    return fail(DCNV4_ERR_UNSUPPORTED, "offset_mask tile needs %zu B of shared memory", lc->smem);
  if (lc->ctas > 0x7fffffffLL)
    return fail(DCNV4_ERR_SHAPE, "too many output pixels (N*Ho*Wo)");
  g->H = (int)p->H; g->W = (int)p->W; g->Ho = (int)Ho; g->Wo = (int)Wo;
  g->G = p->G; g->D = p->D; g->C = p->G * p->D; g->S = S; g->K = K;
  g->kh = p->kernel_h; g->kw = p->kernel_w; g->sh = p->stride_h; g->sw = p->stride_w;
  g->ph = p->pad_h; g->pw = p->pad_w; g->dh = p->dilation_h; g->dw = p->dilation_w;
  g->cy = p->dilation_h * (p->kernel_h - 1) / 2;
  g->cx = p->dilation_w * (p->kernel_w - 1) / 2;
  g->s = p->offset_scale;
  g->softmax = p->softmax;
  g->P = P;
  g->ppc = ppc;
  return DCNV4_OK;
}

bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

int cuda_fail(cudaError_t e, const char* what) {
  return fail(DCNV4_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace

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
  rc = make_launch(p, dtype, pass ? 1 : 0, Ho, Wo, &lc, &g);
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
  rc = make_launch(p, dtype, 0, Ho, Wo, &lc, &g);
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

size_t dcnv4_backward_workspace_bytes(const dcnv4_params* p, dcnv4_dtype dtype) {
  int64_t Ho, Wo;
  if (validate_geometry(p, dtype, &Ho, &Wo)) return 0;
  if (dtype == DCNV4_F32) return 0;
  return (size_t)p->N * p->H * p->W * p->G * p->D * sizeof(float);
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
  rc = make_launch(p, dtype, 1, Ho, Wo, &lc, &g);
  if (rc) return rc;
  lc.stream = static_cast<cudaStream_t>(stream);
  const size_t nelem = (size_t)p->N * p->H * p->W * p->G * p->D;
  float* gx32 = dtype == DCNV4_F32 ? static_cast<float*>(grad_input) : static_cast<float*>(workspace);
  cudaError_t e = cudaMemsetAsync(gx32, 0, nelem * sizeof(float), lc.stream);
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
