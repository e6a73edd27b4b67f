/*
 * dcnv4_module.h -- C ABI of the DCNv4 module path in libdcnv4.so.
 *
 * The operation.  PAPER.md P:334 ("Micro design in DCN module"): "the linear layers for
 * computing offset and dynamic weights can actually be combined into one linear layer",
 * and the depthwise conv in front of it "can also be removed with only a minor
 * performance sacrifice" when latency comes first.  P:1003-1009: the "lightweight"
 * DCNv4 module has no input/output projections, i.e. the operator samples the module
 * input itself.  So the module's offset/mask branch is one linear layer
 *
 *     om[r][j] = sum_{c < C_in} feat[r][c] * weight[j][c] + bias[j],   j < J = 3*G*K,
 *
 * over every output pixel r = (n, ho, wo), producing the fused offset_mask that
 * include/dcnv4.h's dcnv4_forward reads (layout there: per group
 * [dx_0, dy_0, ..., dx_{K-1}, dy_{K-1}, m_0, ..., m_{K-1}]).
 *
 * Reading R21: the linear's result is rounded once to the storage dtype T
 * (round-to-nearest-even) before the operator reads it -- exactly what an unfused module
 * stores between its two layers -- so dcnv4_module_forward and the two-call path
 * (dcnv4_offset_mask_linear + dcnv4_forward) compute the same function.
 *
 * Arithmetic: the contraction runs on the sm_100a 5th-generation tensor cores
 * (tcgen05.mma kind::f16, operands staged in shared memory by TMA, fp32 accumulators in
 * tensor memory); the bias is added in fp32 and the sum rounded to T.  Only DCNV4_F16
 * and DCNV4_BF16 are supported (DCNV4_F32 returns DCNV4_ERR_UNSUPPORTED: fp32 operands
 * would need the tf32 kind, which does not meet the fp32 parity bar).
 *
 * Conventions shared with dcnv4.h: the caller owns every buffer and the stream; the
 * library never allocates, frees, synchronises or changes the device; pointers are
 * device pointers on the current device; calls are asynchronous on `stream` and
 * capturable into CUDA graphs; errors are returned as dcnv4_status with
 * dcnv4_last_error() naming the argument, never printed or thrown.
 */
#ifndef DCNV4_MODULE_H_
#define DCNV4_MODULE_H_

#include "dcnv4.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Fused offset/mask linear layer on tcgen05 tensor cores.
 *   p        geometry; rows R = N*Ho*Wo (Ho, Wo from dcnv4_output_size), J = 3*G*K,
 *            S = p->om_stride (0 => J).
 *   feat     [R][C_in]  T, row-major (for the lightweight module at stride 1 with
 *            "same" padding this is x itself: feat[(n*H + h)*W + w][c] = x[n][h][w][c]).
 *   weight   [J][C_in]  T, row-major (nn.Linear layout: out_features x in_features).
 *   bias     [J]        T, or NULL for no bias.
 *   offset_mask [R][S]  T, fully overwritten: om[r][j] = RN_T(sum_c feat*weight + bias)
 *            for j < J, 0 for J <= j < S.
 * Requirements: dtype F16 or BF16 (else UNSUPPORTED); C_in >= 8 and C_in % 8 == 0,
 * S % 8 == 0 (16-B row pitches; else UNSUPPORTED); feat, weight, offset_mask 16-B
 * aligned, bias 2-B aligned (else MISALIGNED); R < 2^31 (else SHAPE).  N = 0: no-op.
 * One kernel launch (persistent grid, one CTA per SM).  Bit-deterministic.            */
DCNV4_API int dcnv4_offset_mask_linear(const dcnv4_params *p, dcnv4_dtype dtype, int32_t C_in,
                                       const void *feat, const void *weight, const void *bias,
                                       void *offset_mask, void *stream);

/* Fused lightweight-module forward (P:334 + P:1003-1009), one kernel launch:
 *   y = DCNv4(x, RN_T(x . weight^T + bias))     (Eq. (1)-(2) with the om of R21)
 * The offset_mask of each 16 x 8-pixel tile is computed on the tensor cores (tcgen05,
 * fp32 accumulation in TMEM), rounded to T, and consumed from shared memory by the
 * aggregation in the same CTA: it is never written to memory.  The result equals
 * dcnv4_offset_mask_linear followed by dcnv4_forward (same rounding of om, same
 * aggregation arithmetic) up to the fp32 summation order of the linear.
 *   p        geometry: kernel 3x3, stride 1, pad 1, dilation 1 (else UNSUPPORTED);
 *            p->om_stride and p->deterministic are ignored; p->softmax and
 *            p->offset_scale apply as in dcnv4_forward.
 *   input    x [N][H][W][G*D] T;  weight [3GK][G*D] T;  bias [3GK] T or NULL;
 *   output   y [N][H][W][G*D] T, fully overwritten (must not alias input).
 * Requirements: dtype F16/BF16 (F32 -> UNSUPPORTED); D*sizeof(T) in {32, 64, 128} B and
 * G a multiple of 128 / (D*sizeof(T)) (UNSUPPORTED otherwise); input, weight, output
 * 16-B aligned, bias 2-B aligned (MISALIGNED).  Bit-deterministic.  N = 0: no-op.     */
DCNV4_API int dcnv4_module_forward(const dcnv4_params *p, dcnv4_dtype dtype, const void *input,
                                   const void *weight, const void *bias, void *output,
                                   void *stream);


/* Module core forward with a separate value tensor (the full module, P:198 / P:1006-1009:
 * a 1x1 input projection produces the value the operator samples, while the offset/mask
 * linear reads the module input -- reading R22):
 *   y = DCNv4(value, RN_T(input . weight^T + bias))
 * Same kernel, requirements and arithmetic as dcnv4_module_forward (which is this call
 * with value = input); value [N][H][W][G*D] T, 16-B aligned; output must not alias value
 * (INVALID_ARG) or input.                                                               */
DCNV4_API int dcnv4_module_core_forward(const dcnv4_params *p, dcnv4_dtype dtype, const void *input,
                                        const void *value, const void *weight, const void *bias,
                                        void *output, void *stream);

/* ------------------------------------------------------------------------------------
 * Dense layers of the full module and their backward (tcgen05 GEMMs, csrc/gemm.cu).
 * All three take row-major T matrices, fp32 accumulation in tensor memory, one
 * persistent launch (+ the small launches noted).  F16/BF16: kind::f16 MMAs.  F32: 3xTF32
 * on kind::tf32 (each operand split into an exact tf32 high part and its remainder;
 * hi.hi + hi.lo + lo.hi, relative error ~2^-20 per product, within the fp32 parity bar).
 * Every pointer 16-B aligned (bias / grad_bias element-aligned) else MISALIGNED; every
 * channel count and leading dimension a multiple of 16 B (8 halves / 4 floats) else
 * UNSUPPORTED; M < 2^31.
 * Bit-deterministic except dcnv4_linear_grad_weight (fp32 reductions over K splits).    */

/* y[M][N] = RN_T(x[M][K] . weight[N][K]^T + bias[N])  (nn.Linear layout; the module's
 * 1x1 input / output projections).  bias may be NULL.               */
DCNV4_API int dcnv4_linear(dcnv4_dtype dtype, int64_t M, int32_t K, int32_t N, const void *x,
                           const void *weight, const void *bias, void *y, void *stream);

/* grad_input of one or two linear layers that read the same input (the module's input
 * feeds both the input projection and the offset/mask linear):
 *   gx[M][K] = RN_T( gy0[M][0:N0] . weight0[N0][K]  +  gy1[M][N1] . weight1[N1][K] )
 * gy0 has leading dimension ld0 >= N0 (e.g. grad_offset_mask [R][S], S >= 3GK, whose
 * padding columns must be finite: they meet zero rows); N1 = 0 drops the second term
 * (gy1, weight1 ignored).  The weights are read in their stored [N][K] layout (MN-major
 * operands of the tensor-core MMA), no transposed copy.                                 */
DCNV4_API int dcnv4_linear_grad_input(dcnv4_dtype dtype, int64_t M, int32_t K, int32_t N0,
                                      const void *gy0, int32_t ld0, const void *weight0, int32_t N1,
                                      const void *gy1, const void *weight1, void *gx, void *stream);

/* Workspace (fp32 accumulators) dcnv4_linear_grad_weight needs: (N*K + N) * 4 bytes.     */
DCNV4_API size_t dcnv4_linear_grad_weight_workspace_bytes(int32_t K, int32_t N);

/* grad_weight and grad_bias of y = x . weight^T + bias over M rows:
 *   grad_weight[N][K] = RN_T(sum_m gy[m][n] x[m][k]),  grad_bias[N] = RN_T(sum_m gy[m][n])
 * gy [M][ld_gy] (first N columns used; N need not be a multiple of 8, e.g. N = 3GK of the
 * offset/mask linear with gy = grad_offset_mask of row stride S), x [M][K].  The
 * contraction over all M rows is
 * split across CTAs and summed in fp32 (16-B vector reductions) into the workspace, then
 * rounded once to T.  grad_bias may be NULL.  Launches: a workspace memset, the GEMM,
 * a column-sum kernel (grad_bias) and the fp32 -> T conversion(s).                      */
DCNV4_API int dcnv4_linear_grad_weight(dcnv4_dtype dtype, int64_t M, int32_t K, int32_t N, const void *x,
                                       const void *gy, int32_t ld_gy, void *grad_weight, void *grad_bias,
                                       void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* DCNV4_MODULE_H_ */
