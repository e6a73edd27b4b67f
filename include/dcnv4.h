/*
 * dcnv4.h -- C ABI of the B200 (sm_100a) DCNv4 spatial-aggregation library (libdcnv4.so).
 *
 * The operation (PAPER.md = arxiv 2401.06197 LaTeX source; "P:n" = line n):
 *   Eq. (1)-(2):  y_g(p0) = sum_{k=1..K} m_gk * x_g(p0 + p_k + dp_gk),
 *                            y = concat_g y_g,
 *   DCNv4 removes the softmax over K, so m is an unbounded raw scalar.
 *   Channel-last layout (P:319 footnote); the offset and modulation linear layers are
 *   fused into one tensor, read once per (pixel, group) and reused across the
 *   D = C/G channels of the group.
 * The backward (grad_input, grad_offset, grad_mask) is not in the paper; it is Eq. (1)
 * differentiated, right derivative at integer coordinates.
 *
 * Conventions (DESIGN.md "Readings" R1-R17 gives the reason for each):
 *   input        x   [N][H][W][G*D]            dtype T, NHWC, contiguous
 *   offset_mask  om  [N][Ho][Wo][S]            dtype T, S = om_stride (0 => 3*G*K)
 *                for group g, channels g*3K .. g*3K+3K-1 hold
 *                [dx_0, dy_0, dx_1, dy_1, ..., dx_{K-1}, dy_{K-1}, m_0, ..., m_{K-1}];
 *                channels [3GK, S) are padding and are ignored.
 *   output       y   [N][Ho][Wo][G*D]          dtype T
 *   K = kernel_h*kernel_w; point k = i*kernel_h + j, i = x-tap (outer), j = y-tap (inner)
 *   Ho = floor((H + 2*pad_h - dilation_h*(kernel_h-1) - 1)/stride_h) + 1 (Wo likewise)
 *   cy = floor(dilation_h*(kernel_h-1)/2), cx likewise
 *   sampling point: py = (ho*stride_h - pad_h + cy) + s*(j*dilation_h - cy + dy_k)
 *                   px = (wo*stride_w - pad_w + cx) + s*(i*dilation_w - cx + dx_k)
 *   bilinear with integer coordinates at pixel centres, zero outside [0,H)x[0,W) per
 *   corner; an offset whose scaled value is NaN or exceeds 2^20 in magnitude drops the
 *   sample (its output is unspecified, memory stays safe).
 *   Arithmetic: fp32 for coordinates and accumulation in every dtype; results are
 *   rounded to T (round-to-nearest-even).
 *
 * Ownership and threading: the caller owns every buffer and the stream.  The library
 * never allocates, frees, synchronises or changes the current device; all pointers are
 * device pointers on the current device.  Calls are asynchronous on `stream` (a
 * cudaStream_t passed as void*, NULL = legacy default stream) and capturable into CUDA
 * graphs.  The library is stateless apart from the thread-local error string, and
 * re-entrant: concurrent calls on different streams are fine.
 * Errors: every entry point returns a dcnv4_status and never aborts, prints or throws;
 * dcnv4_last_error() returns a thread-local message naming the offending argument/axis.
 */
#ifndef DCNV4_H_
#define DCNV4_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DCNV4_API __attribute__((visibility("default")))
#else
#define DCNV4_API
#endif

#define DCNV4_VERSION 130 /* 1.3.0: dcnv4_forward_grouped, full-module GEMMs (dcnv4_module.h); 1.2.0: module path; 1.1.0: dcnv4_params.deterministic */

typedef enum { DCNV4_F32 = 0, DCNV4_F16 = 1, DCNV4_BF16 = 2 } dcnv4_dtype;

typedef enum {
  DCNV4_OK = 0,
  DCNV4_ERR_INVALID_ARG = 1, /* NULL pointer, non-positive size, bad enum, bad flag     */
  DCNV4_ERR_SHAPE = 2,       /* empty output, om_stride < 3GK, per-image size >= 2^31   */
  DCNV4_ERR_UNSUPPORTED = 3, /* D*sizeof(T) not 16 B x a power of two or > 256 B, K > 64,
                                offset_mask tile larger than shared memory              */
  DCNV4_ERR_MISALIGNED = 4,  /* x / y / grad pointers not 16-B aligned, om not T-aligned */
  DCNV4_ERR_WORKSPACE = 5,   /* backward workspace missing or too small                 */
  DCNV4_ERR_CUDA = 6         /* a launch failed; the CUDA error string is in last_error */
} dcnv4_status;

/* Problem geometry.  P:187-198 states the problem as x in R^{HxWxC}, G groups and K
 * points on the regular conv grid; stride/pad/dilation follow conv2d ("as in
 * regular convolutions"); offset_scale s scales tap + offset (R5).          */
typedef struct {
  int64_t N, H, W;       /* batch, input height, input width (N may be 0: no-op)      */
  int32_t G, D;          /* groups, channels per group; C = G*D                        */
  int32_t kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w, dilation_h, dilation_w;
  float offset_scale;    /* s; finite                                                  */
  int32_t om_stride;     /* S, channels per offset_mask pixel; 0 => 3*G*K              */
  int32_t softmax;       /* 0 = DCNv4 (raw m, the paper's operator);
                            1 = DCNv3 normalisation, m <- softmax_K(m)         */
  int32_t deterministic; /* backward only. 0 = grad_input summed with fp32 atomics
                            (run-to-run differences at rounding level);
                            1 = bit-reproducible grad_input: every contribution is
                            rounded once to a per-image fixed-point grid 2^-F and summed
                            in int64, F from the image's max|gy| and max|m| (DESIGN.md
                            R19).  Adds |error| <= n * 2^-(F+1) for an element with n
                            contributions; an image whose max|gy| or max|m| is
                            non-finite or outside [2^-64, 2^64) gets NaN grad_input.   */
} dcnv4_params;

/* Library version (DCNV4_VERSION). */
DCNV4_API int dcnv4_version(void);

/* Thread-local description of the last failed call on this thread ("" if none). */
DCNV4_API const char *dcnv4_last_error(void);

/* Output spatial size (conv2d arithmetic, see above).  Host-only; no CUDA call.
 * Returns DCNV4_OK or INVALID_ARG/SHAPE with last_error naming the axis.             */
DCNV4_API int dcnv4_output_size(const dcnv4_params *p, int64_t *H_out, int64_t *W_out);

/* Forward, Eq. (1)-(2): y = DCNv4(x, om).  Reads x and om, fully overwrites y
 * (y must not alias x or om).  Bit-deterministic.  One kernel launch (none if N = 0). */
DCNV4_API int dcnv4_forward(const dcnv4_params *p, dcnv4_dtype dtype, const void *input,
                  const void *offset_mask, void *output, void *stream);

/* Several independent forwards in ONE launch (e.g. the four stages of a backbone, or a
 * batch-1 pyramid whose late stages are too small to fill the GPU on their own):
 * output i = DCNv4(inputs[i], offset_masks[i]) with params[i], exactly as dcnv4_forward
 * computes it (bit-identical).  1 <= count <= 8; all problems share dtype.  When every
 * non-empty problem runs the TMA-halo kernel (3x3, stride 1, dilation 1) with the same
 * channel layout (D * sizeof(T)) and tile shape, a single persistent grid sweeps the
 * concatenated tile ranges, so the tail of one problem overlaps the next; otherwise the
 * problems are launched one after another on `stream`.  Every problem is validated
 * before anything is launched (errors name the problem index).                        */
DCNV4_API int dcnv4_forward_grouped(const dcnv4_params *const *params, int32_t count,
                                    dcnv4_dtype dtype, const void *const *inputs,
                                    const void *const *offset_masks, void *const *outputs,
                                    void *stream);

/* Workspace bytes dcnv4_backward needs: 0 for DCNV4_F32; N*H*W*C*4 (an fp32
 * grad_input accumulator) for DCNV4_F16 / DCNV4_BF16; with deterministic = 1, for every
 * dtype, N*H*W*C*8 (int64 accumulator) + 8*N rounded up to 16 (per-image maxima).     */
DCNV4_API size_t dcnv4_backward_workspace_bytes(const dcnv4_params *p, dcnv4_dtype dtype);

/* Backward of Eq. (1) given grad_output gy [N][Ho][Wo][C]:
 *   grad_input  [N][H][W][C]  gx = sum over samples and in-bounds corners of m*w*gy
 *   grad_offset_mask [N][Ho][Wo][S], same layout as om:
 *     d/d dx_k = s*m_k*sum_c gy_c dv_kc/dpx,  d/d dy_k = s*m_k*sum_c gy_c dv_kc/dpy,
 *     d/d m_k  = sum_c gy_c v_kc  (softmax = 1: w.r.t. the pre-softmax logits),
 *     padding channels [3GK, S) are written 0.
 * Both outputs are fully overwritten (nothing accumulates into caller data).
 * grad_offset_mask is bit-deterministic; grad_input is summed with fp32 atomics and is
 * deterministic only up to rounding order, unless p->deterministic = 1 (bit-identical
 * across runs, grids and batch splits).  workspace: >= the size returned by
 * dcnv4_backward_workspace_bytes, 16-B aligned, scratch owned by the caller (may be NULL
 * when that size is 0).  Launches: a memset of the fp32 accumulator, the backward
 * kernel, and (half dtypes) one fp32 -> T conversion kernel; deterministic = 1: a
 * memset of the workspace, a per-image maxima kernel, the backward kernel and one
 * int64 -> T conversion kernel.                                                        */
DCNV4_API int dcnv4_backward(const dcnv4_params *p, dcnv4_dtype dtype, const void *input,
                   const void *offset_mask, const void *grad_output, void *grad_input,
                   void *grad_offset_mask, void *workspace, size_t workspace_bytes,
                   void *stream);

/* Launch-shape introspection used by the harness (lanes per (pixel, group), 16-B chunks
 * per lane, output pixels per CTA tile, threads per CTA, CTAs) for forward (pass = 0) or backward
 * (pass = 1).  Host-only.                                                             */
DCNV4_API int dcnv4_launch_info(const dcnv4_params *p, dcnv4_dtype dtype, int pass, int32_t *lanes,
                      int32_t *chunks_per_lane, int32_t *pixels_per_cta,
                      int32_t *threads_per_cta, int64_t *ctas);

#ifdef __cplusplus
}
#endif

#endif /* DCNV4_H_ */
