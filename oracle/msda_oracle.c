/*
 * msda_oracle.c -- plain, slow, fp64 CPU oracle for multi-scale deformable attention
 * (SURVEY.md 8(f) NEXT-3).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no source,
 * header, table or helper with the CUDA path (paper_2401_06197_b200/csrc/), and the
 * CUDA path never calls it.
 *
 * What it computes.  PAPER.md (arXiv 2401.06197) names deformable attention as the
 * operator "that enables each query to concentrate on a select number of key sampling
 * points, with dynamically determined locations and weights" and states that
 * the DCNv4 kernel optimisations "can also be applied to ... deformable attention, as
 * they share a similar performance bottleneck".  The paper does not write the
 * operator out; reading R20 takes the multi-scale form of its citation
 * (zhu2020deformable), the sampling core without the value / output projections:
 *
 *   out[n,q,m,:] = sum_{l<L} sum_{p<P} A[n,q,m,l,p] * V_l[n,m](phi_l(loc[n,q,m,l,p]))
 *
 *   value  V [N][S][M][D], S = sum_l H_l*W_l, level l occupying tokens
 *          [start_l, start_l + H_l*W_l) in row-major (h, w) order;
 *   loc    [N][Lq][M][L][P][2] = (x, y), normalised to [0, 1] over the level;
 *   A      [N][Lq][M][L][P]    attention weights, used as given (R20: the caller's
 *          softmax, as in the prior-art operator);
 *   phi_l(x, y) = (w, h) = (x*W_l - 1/2, y*H_l - 1/2)   (pixel centres at integers +
 *          1/2 in normalised units: the grid_sample align_corners=False convention);
 *   V_l(h, w) bilinear over the four integer neighbours, zero outside [0,H_l)x[0,W_l)
 *          per corner (as R6/R7 for DCNv4).
 *
 * Backward (the operator differentiated; right derivative at integer coordinates, R8):
 *   gV_l[corner] += A * w_corner * gout
 *   gA  = <gout, V_l(phi_l(loc))>
 *   gx  = A * W_l * <gout, dV/dw>,   gy = A * H_l * <gout, dV/dh>
 *
 * Arithmetic: fp64 throughout; loops in the order n, q, m, l, p, corner, c.  OpenMP
 * runs over (n, m): each (n, m) owns disjoint slices of out, grad_value, grad_loc and
 * grad_attn, so the result does not depend on the thread count.
 *
 * Pins (tests/test_oracle_msda.py): torch grid_sample (align_corners=False, zeros) per
 * level plus autograd for all three gradients; closed forms (constant value, pixel
 * centres, affine ramp value); linearity; the adjoint identity.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* shape vector: N, Lq, M, D, L, P, then H_0, W_0, ..., H_{L-1}, W_{L-1} */
enum { MN, MLQ, MM, MD, ML, MP, MSHAPES };

static int64_t total_tokens(const int64_t *g) {
  int64_t s = 0;
  for (int64_t l = 0; l < g[ML]; ++l) s += g[MSHAPES + 2 * l] * g[MSHAPES + 2 * l + 1];
  return s;
}

static int64_t level_start(const int64_t *g, int64_t l) {
  int64_t s = 0;
  for (int64_t i = 0; i < l; ++i) s += g[MSHAPES + 2 * i] * g[MSHAPES + 2 * i + 1];
  return s;
}

/* V[n][start + h*W + w][m][c], zero outside the level (per-corner zero padding) */
static double Vat(const double *v, const int64_t *g, int64_t S, int64_t n, int64_t m,
                  int64_t start, int64_t H, int64_t W, int64_t h, int64_t w, int64_t c) {
  if (h < 0 || h >= H || w < 0 || w >= W) return 0.0;
  const int64_t M = g[MM], D = g[MD];
  return v[(((n * S) + start + h * W + w) * M + m) * D + c];
}

/* phi_l: normalised (x, y) -> pixel coordinates (w, h), align_corners=False */
static void phi(double x, double y, int64_t H, int64_t W, double *h, double *w) {
  *w = x * (double)W - 0.5;
  *h = y * (double)H - 0.5;
}

int msda_oracle_forward(const int64_t *g, const double *value, const double *loc,
                        const double *attn, double *out, double *out_abs) {
  const int64_t N = g[MN], Lq = g[MLQ], M = g[MM], D = g[MD], L = g[ML], P = g[MP];
  const int64_t S = total_tokens(g);
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t m = 0; m < M; ++m)
      for (int64_t q = 0; q < Lq; ++q) {
        double *o = out + ((n * Lq + q) * M + m) * D;
        double *oa = out_abs ? out_abs + ((n * Lq + q) * M + m) * D : 0;
        for (int64_t c = 0; c < D; ++c) {
          o[c] = 0.0;
          if (oa) oa[c] = 0.0;
        }
        for (int64_t l = 0; l < L; ++l) {
          const int64_t H = g[MSHAPES + 2 * l], W = g[MSHAPES + 2 * l + 1];
          const int64_t start = level_start(g, l);
          for (int64_t p = 0; p < P; ++p) {
            const int64_t i = (((n * Lq + q) * M + m) * L + l) * P + p;
            const double a = attn[i];
            double h, w;
            phi(loc[2 * i], loc[2 * i + 1], H, W, &h, &w);
            const double h0 = floor(h), w0 = floor(w);
            const double fh = h - h0, fw = w - w0;
            const int64_t y0 = (int64_t)h0, x0 = (int64_t)w0;
            const double wt[4] = {(1 - fh) * (1 - fw), (1 - fh) * fw, fh * (1 - fw), fh * fw};
            const int64_t cy[4] = {y0, y0, y0 + 1, y0 + 1}, cx[4] = {x0, x0 + 1, x0, x0 + 1};
            for (int corner = 0; corner < 4; ++corner)
              for (int64_t c = 0; c < D; ++c) {
                const double v = Vat(value, g, S, n, m, start, H, W, cy[corner], cx[corner], c);
                o[c] += a * wt[corner] * v;
                if (oa) oa[c] += fabs(a) * wt[corner] * fabs(v);
              }
          }
        }
      }
  return 0;
}

/* grad_value is written (zeroed first); with_abs arrays (may be NULL) receive the
 * magnitude scales of each output for the abs-scaled error metric. */
int msda_oracle_backward(const int64_t *g, const double *value, const double *loc,
                         const double *attn, const double *gout, double *gvalue,
                         double *gloc, double *gattn, double *gvalue_abs, double *gloc_abs,
                         double *gattn_abs) {
  const int64_t N = g[MN], Lq = g[MLQ], M = g[MM], D = g[MD], L = g[ML], P = g[MP];
  const int64_t S = total_tokens(g);
  memset(gvalue, 0, sizeof(double) * (size_t)(N * S * M * D));
  if (gvalue_abs) memset(gvalue_abs, 0, sizeof(double) * (size_t)(N * S * M * D));
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t m = 0; m < M; ++m)
      for (int64_t q = 0; q < Lq; ++q) {
        const double *go = gout + ((n * Lq + q) * M + m) * D;
        for (int64_t l = 0; l < L; ++l) {
          const int64_t H = g[MSHAPES + 2 * l], W = g[MSHAPES + 2 * l + 1];
          const int64_t start = level_start(g, l);
          for (int64_t p = 0; p < P; ++p) {
            const int64_t i = (((n * Lq + q) * M + m) * L + l) * P + p;
            const double a = attn[i];
            double h, w;
            phi(loc[2 * i], loc[2 * i + 1], H, W, &h, &w);
            const double h0 = floor(h), w0 = floor(w);
            const double fh = h - h0, fw = w - w0;
            const int64_t y0 = (int64_t)h0, x0 = (int64_t)w0;
            const double wt[4] = {(1 - fh) * (1 - fw), (1 - fh) * fw, fh * (1 - fw), fh * fw};
            /* d wt / d h and d wt / d w */
            const double dh[4] = {-(1 - fw), -fw, (1 - fw), fw};
            const double dw[4] = {-(1 - fh), (1 - fh), -fh, fh};
            const int64_t cy[4] = {y0, y0, y0 + 1, y0 + 1}, cx[4] = {x0, x0 + 1, x0, x0 + 1};
            double sa = 0, sh = 0, sw = 0, saa = 0, sha = 0, swa = 0;
            for (int corner = 0; corner < 4; ++corner) {
              const int inb = cy[corner] >= 0 && cy[corner] < H && cx[corner] >= 0 && cx[corner] < W;
              for (int64_t c = 0; c < D; ++c) {
                const double v = Vat(value, g, S, n, m, start, H, W, cy[corner], cx[corner], c);
                sa += go[c] * wt[corner] * v;
                sh += go[c] * dh[corner] * v;
                sw += go[c] * dw[corner] * v;
                saa += fabs(go[c]) * wt[corner] * fabs(v);
                sha += fabs(go[c]) * fabs(dh[corner]) * fabs(v);
                swa += fabs(go[c]) * fabs(dw[corner]) * fabs(v);
                if (inb) {
                  const int64_t t = (((n * S) + start + cy[corner] * W + cx[corner]) * M + m) * D + c;
                  gvalue[t] += a * wt[corner] * go[c];
                  if (gvalue_abs) gvalue_abs[t] += fabs(a) * wt[corner] * fabs(go[c]);
                }
              }
            }
            gattn[i] = sa;
            gloc[2 * i] = a * (double)W * sw;
            gloc[2 * i + 1] = a * (double)H * sh;
            if (gattn_abs) gattn_abs[i] = saa;
            if (gloc_abs) {
              gloc_abs[2 * i] = fabs(a) * (double)W * swa;
              gloc_abs[2 * i + 1] = fabs(a) * (double)H * sha;
            }
          }
        }
      }
  return 0;
}
