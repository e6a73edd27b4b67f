/*
 * msda.h -- C ABI of multi-scale deformable attention (MSDA) in libdcnv4.so
 * (SURVEY.md 8(f) NEXT-3).
 *
 * The operation.  PAPER.md names deformable attention as the operator that "enables each
 * query to concentrate on a select number of key sampling points, with dynamically
 * determined locations and weights" and states that the DCNv4 kernel techniques
 * "can also be applied to ... deformable attention, as they share a similar performance
 * bottleneck".  The sampling core of its multi-scale form (R20):
 *
 *   out[n,q,m,:] = sum_{l<L} sum_{p<P} attn[n,q,m,l,p] * V_l[n,:,m,:](phi_l(loc[n,q,m,l,p]))
 *
 *   value  [N][S][M][D]         dtype T; S = sum_l H_l*W_l tokens, level l occupying
 *                               tokens [start_l, start_l + H_l*W_l) in row-major (h, w)
 *   loc    [N][Lq][M][L][P][2]  dtype T; normalised (x, y) in [0, 1] over the level
 *   attn   [N][Lq][M][L][P]     dtype T; used as given (no softmax inside)
 *   out    [N][Lq][M][D]        dtype T
 *   phi_l(x, y) = (w, h) = (x*W_l - 1/2, y*H_l - 1/2) (grid_sample align_corners=False);
 *   bilinear over the four integer neighbours with per-corner zero padding outside
 *   [0, H_l) x [0, W_l); right derivative at integer coordinates.
 *   Arithmetic: fp32 coordinates and accumulation in every dtype, RN-even results.
 *
 * Ownership, threading and errors as in dcnv4.h (caller-owned device buffers and stream,
 * asynchronous, capturable, stateless; every call returns a dcnv4_status and
 * dcnv4_last_error() names the offending argument).
 */
#ifndef MSDA_H_
#define MSDA_H_

#include "dcnv4.h"

#ifdef __cplusplus
extern "C" {
#endif

#define MSDA_MAX_LEVELS 8

typedef struct {
  int64_t N, Lq;           /* batch, queries per image (either may be 0: no-op)           */
  int32_t M, D;            /* heads, channels per head (D*sizeof(T) = 16 B x 2^k <= 256 B) */
  int32_t L, P;            /* levels (1..MSDA_MAX_LEVELS), points per level and head       */
  int32_t H[MSDA_MAX_LEVELS], W[MSDA_MAX_LEVELS];  /* level shapes, entries >= L ignored  */
} msda_params;

/* Total value tokens S = sum_l H_l*W_l (host-only).                                   */
DCNV4_API int msda_value_tokens(const msda_params *p, int64_t *S);

/* Forward: reads value, loc, attn; fully overwrites out.  Bit-deterministic.  One
 * kernel launch (none if N*Lq = 0).  value/out 16-B aligned; loc, attn T-aligned.      */
DCNV4_API int msda_forward(const msda_params *p, dcnv4_dtype dtype, const void *value,
                           const void *loc, const void *attn, void *out, void *stream);

/* Workspace: 0 for DCNV4_F32; N*S*M*D*4 (fp32 grad_value accumulator) for half types. */
DCNV4_API size_t msda_backward_workspace_bytes(const msda_params *p, dcnv4_dtype dtype);

/* Backward given grad_out [N][Lq][M][D]:
 *   grad_value [N][S][M][D]      = sum over samples and in-level corners of attn*w*grad_out
 *                                  (fp32 vector reductions; order unspecified)
 *   grad_loc   [N][Lq][M][L][P][2] = attn * (W_l, H_l) * <grad_out, dV/d(w, h)>
 *   grad_attn  [N][Lq][M][L][P]    = <grad_out, V_l(phi_l(loc))>
 * All three are fully overwritten; grad_loc and grad_attn are bit-deterministic.
 * Launches: a memset of the fp32 accumulator, the backward kernel, and (half dtypes)
 * one fp32 -> T conversion kernel.                                                     */
DCNV4_API int msda_backward(const msda_params *p, dcnv4_dtype dtype, const void *value,
                            const void *loc, const void *attn, const void *grad_out,
                            void *grad_value, void *grad_loc, void *grad_attn,
                            void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* MSDA_H_ */
