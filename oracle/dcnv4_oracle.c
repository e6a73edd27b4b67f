/*
 * dcnv4_oracle.c -- plain, slow, fp64 CPU oracle for the DCNv4 spatial aggregation.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no source,
 * header, table or helper with the CUDA path (paper_2401_06197_b200/csrc/), and the
 * CUDA path never calls it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   Eq. (1)-(2):   y_g = sum_{k=1..K} m_gk * x_g(p0 + p_k + dp_gk),
 *                             y   = concat_g y_g        (channel-last, P:319 footnote)
 *   DCNv4 = Eq. (1) with the softmax over K removed; m is used raw.
 *   The DCNv3 form (softmax over K) is available behind `softmax` != 0.
 *   The backward is not in the paper; it is Eq. (1) differentiated.
 *
 * Readings of the paper that this file fixes (DESIGN.md "Readings" R1..R17 lists
 * them with reasons; SURVEY.md 8(c).2 is the source):
 *   R1  K = kh*kw points (P:187 vs P:319 notation clash).
 *   R2  point k = i*kh + j with i the x-tap (outer) and j the y-tap (inner);
 *       offsets are stored as (dx, dy) pairs.
 *   R3  fused offset_mask row per pixel: for group g, [dx_0,dy_0,...,dx_{K-1},dy_{K-1},
 *       m_0..m_{K-1}] at channels g*3K .. g*3K+3K-1; row stride S >= 3*G*K.
 *   R4  output size and tap geometry are conv2d's ("as in regular convolutions").
 *   R5  offset_scale s:  p = p0 + s*(p_k + dp), p0 the window centre.
 *   R6  per-corner zero padding outside [0,H)x[0,W).
 *   R7  integer coordinates are pixel centres; y0 = floor(py).
 *   R8  gradient at integer coordinates = right derivative of the floor convention.
 *
 * Arithmetic: every value is fp64; loops follow the order n, g, ho, wo, i, j, corner, c.
 * OpenMP runs over (n, g); each (n, g) owns disjoint slices of y, grad_x and grad_om,
 * so the result does not depend on the thread count.
 *
 * Parity pins (tests/test_oracle_pins.py): conv2d reduction, grid_sample + autograd
 * equivalence, closed forms (constant, affine ramp, shift, out-of-bounds, 1x1
 * identity), the bilinear examples of SPEC S:122-124, finite differences, the adjoint
 * and Euler identities, and the softmax examples of SPEC S:113-115.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* geometry vector, in this order (index: meaning):
 *  0 N   1 H   2 W   3 G   4 D   5 kh  6 kw  7 sh  8 sw  9 ph  10 pw  11 dh  12 dw
 *  13 S (offset_mask channels per pixel)  14 softmax flag (0 = DCNv4, 1 = DCNv3) */
enum { GN, GH, GW, GG, GD, GKH, GKW, GSH, GSW, GPH, GPW, GDH, GDW, GS, GSOFT, GEOM_LEN };

int oracle_geom_len(void) { return GEOM_LEN; }

/* Output size: PyTorch conv2d arithmetic (reading R4). Returns 0 on success. */
int oracle_output_size(const int64_t *g, int64_t *Ho, int64_t *Wo) {
  int64_t h = (g[GH] + 2 * g[GPH] - g[GDH] * (g[GKH] - 1) - 1);
  int64_t w = (g[GW] + 2 * g[GPW] - g[GDW] * (g[GKW] - 1) - 1);
  if (g[GSH] <= 0 || g[GSW] <= 0 || h < 0 || w < 0) return 1;
  *Ho = h / g[GSH] + 1;
  *Wo = w / g[GSW] + 1;
  return 0;
}

/* x[n][yy][xx][g*D + c] with zero outside the image (reading R6). */
static double X(const double *x, const int64_t *g, int64_t n, int64_t yy, int64_t xx,
                int64_t grp, int64_t c) {
  if (yy < 0 || yy >= g[GH] || xx < 0 || xx >= g[GW]) return 0.0;
  int64_t C = g[GG] * g[GD];
  return x[((n * g[GH] + yy) * g[GW] + xx) * C + grp * g[GD] + c];
}

/* Sampling location of point (i, j) for output (ho, wo) (readings R2, R4, R5):
 *   py = (ho*sh - ph + cy) + s*(j*dh - cy + dy),  cy = floor(dh*(kh-1)/2)
 *   px = (wo*sw - pw + cx) + s*(i*dw - cx + dx),  cx = floor(dw*(kw-1)/2)        */
static void location(const int64_t *g, double s, int64_t ho, int64_t wo, int64_t i,
                     int64_t j, double dx, double dy, double *py, double *px) {
  int64_t cy = g[GDH] * (g[GKH] - 1) / 2;
  int64_t cx = g[GDW] * (g[GKW] - 1) / 2;
  *py = (double)(ho * g[GSH] - g[GPH] + cy) + s * ((double)(j * g[GDH] - cy) + dy);
  *px = (double)(wo * g[GSW] - g[GPW] + cx) + s * ((double)(i * g[GDW] - cx) + dx);
}

/* Modulation scalars of one (n, ho, wo, g): raw m (DCNv4) or softmax over K
 * (DCNv3) with the max subtracted. */
static void modulation(const double *row, int64_t K, int softmax, double *m) {
  for (int64_t k = 0; k < K; ++k) m[k] = row[2 * K + k];
  if (!softmax) return;
  double mx = m[0];
  for (int64_t k = 1; k < K; ++k) mx = m[k] > mx ? m[k] : mx;
  double den = 0.0;
  for (int64_t k = 0; k < K; ++k) { m[k] = exp(m[k] - mx); den += m[k]; }
  for (int64_t k = 0; k < K; ++k) m[k] /= den;
}

#define KMAX 1024

/* Forward, Eq. (1)-(2).  y and y_abs are [N][Ho][Wo][G*D]; y_abs (may be NULL) is the
 * same sum taken over |m|, |x| (the magnitude scale of the error metric).
 * Returns 0, or 1 on bad geometry, or 2 on a non-finite offset/mask value. */
int oracle_forward(const int64_t *g, double s, const double *x, const double *om, double *y,
                   double *y_abs) {
  int64_t Ho, Wo;
  if (oracle_output_size(g, &Ho, &Wo)) return 1;
  const int64_t N = g[GN], G = g[GG], D = g[GD], C = G * D, K = g[GKH] * g[GKW];
  if (K > KMAX || g[GS] < 3 * G * K) return 1;
  for (int64_t q = 0; q < N * Ho * Wo * g[GS]; ++q)
    if (!isfinite(om[q])) return 2;
  int64_t n;
#pragma omp parallel for collapse(2) schedule(static)
  for (n = 0; n < N; ++n) {
    for (int64_t grp = 0; grp < G; ++grp) {
      double m[KMAX];
      for (int64_t ho = 0; ho < Ho; ++ho) {
        for (int64_t wo = 0; wo < Wo; ++wo) {
          const double *row = om + ((n * Ho + ho) * Wo + wo) * g[GS] + grp * 3 * K;
          double *yo = y + ((n * Ho + ho) * Wo + wo) * C + grp * D;
          double *ya = y_abs ? y_abs + ((n * Ho + ho) * Wo + wo) * C + grp * D : 0;
          modulation(row, K, (int)g[GSOFT], m);
          for (int64_t c = 0; c < D; ++c) { yo[c] = 0.0; if (ya) ya[c] = 0.0; }
          for (int64_t i = 0; i < g[GKW]; ++i) {
            for (int64_t j = 0; j < g[GKH]; ++j) {
              int64_t k = i * g[GKH] + j;
              double py, px;
              location(g, s, ho, wo, i, j, row[2 * k], row[2 * k + 1], &py, &px);
              double fy0 = floor(py), fx0 = floor(px);
              int64_t y0 = (int64_t)fy0, x0 = (int64_t)fx0;
              double fy = py - fy0, fx = px - fx0;
              /* the four corners and their bilinear weights (reading R7) */
              int64_t cyy[4] = {y0, y0, y0 + 1, y0 + 1};
              int64_t cxx[4] = {x0, x0 + 1, x0, x0 + 1};
              double cw[4] = {(1 - fy) * (1 - fx), (1 - fy) * fx, fy * (1 - fx), fy * fx};
              for (int corner = 0; corner < 4; ++corner) {
                for (int64_t c = 0; c < D; ++c) {
                  double v = X(x, g, n, cyy[corner], cxx[corner], grp, c);
                  yo[c] += m[k] * cw[corner] * v;
                  if (ya) ya[c] += fabs(m[k]) * cw[corner] * fabs(v);
                }
              }
            }
          }
        }
      }
    }
  }
  return 0;
}

/* Backward of Eq. (1) (SPEC S:135-143 derivation; reading R8 at kinks).
 * Inputs x, om, gy.  Outputs (fully overwritten): gx [N][H][W][C], gom [N][Ho][Wo][S]
 * (padding channels [3GK, S) are 0).  With softmax, gom's m-channels hold the gradient
 * w.r.t. the raw (pre-softmax) logits.
 * Optional magnitude scales (NULL to skip): gx_abs like gx, gom_abs like gom:
 *   gx_abs  = sum |m| w |gy|,   gm_abs = sum_c |gy_c| sum_corner w |X|,
 *   gd*_abs = |s m| sum_c |gy_c| (bilinear-derivative weights) (|X_a| + |X_b|).      */
int oracle_backward(const int64_t *g, double s, const double *x, const double *om,
                    const double *gy, double *gx, double *gom, double *gx_abs,
                    double *gom_abs) {
  int64_t Ho, Wo;
  if (oracle_output_size(g, &Ho, &Wo)) return 1;
  const int64_t N = g[GN], H = g[GH], W = g[GW], G = g[GG], D = g[GD], C = G * D;
  const int64_t K = g[GKH] * g[GKW], S = g[GS];
  if (K > KMAX || S < 3 * G * K) return 1;
  for (int64_t q = 0; q < N * Ho * Wo * S; ++q)
    if (!isfinite(om[q])) return 2;
  memset(gx, 0, sizeof(double) * (size_t)(N * H * W * C));
  memset(gom, 0, sizeof(double) * (size_t)(N * Ho * Wo * S));
  if (gx_abs) memset(gx_abs, 0, sizeof(double) * (size_t)(N * H * W * C));
  if (gom_abs) memset(gom_abs, 0, sizeof(double) * (size_t)(N * Ho * Wo * S));
  int64_t n;
#pragma omp parallel for collapse(2) schedule(static)
  for (n = 0; n < N; ++n) {
    for (int64_t grp = 0; grp < G; ++grp) {
      double m[KMAX], gm[KMAX], gma[KMAX];
      for (int64_t ho = 0; ho < Ho; ++ho) {
        for (int64_t wo = 0; wo < Wo; ++wo) {
          const int64_t pix = (n * Ho + ho) * Wo + wo;
          const double *row = om + pix * S + grp * 3 * K;
          const double *g_y = gy + pix * C + grp * D;
          double *grow = gom + pix * S + grp * 3 * K;
          double *garow = gom_abs ? gom_abs + pix * S + grp * 3 * K : 0;
          modulation(row, K, (int)g[GSOFT], m);
          for (int64_t i = 0; i < g[GKW]; ++i) {
            for (int64_t j = 0; j < g[GKH]; ++j) {
              int64_t k = i * g[GKH] + j;
              double py, px;
              location(g, s, ho, wo, i, j, row[2 * k], row[2 * k + 1], &py, &px);
              double fy0 = floor(py), fx0 = floor(px);
              int64_t y0 = (int64_t)fy0, x0 = (int64_t)fx0;
              double fy = py - fy0, fx = px - fx0;
              int64_t cyy[4] = {y0, y0, y0 + 1, y0 + 1};
              int64_t cxx[4] = {x0, x0 + 1, x0, x0 + 1};
              double cw[4] = {(1 - fy) * (1 - fx), (1 - fy) * fx, fy * (1 - fx), fy * fx};
              /* d(weight)/d(py) and d(weight)/d(px) of each corner (right derivative) */
              double dwy[4] = {-(1 - fx), -fx, (1 - fx), fx};
              double dwx[4] = {-(1 - fy), (1 - fy), -fy, fy};
              double sgm = 0.0, sgy = 0.0, sgx = 0.0, agm = 0.0, agy = 0.0, agx = 0.0;
              for (int corner = 0; corner < 4; ++corner) {
                int inb = cyy[corner] >= 0 && cyy[corner] < H && cxx[corner] >= 0 &&
                          cxx[corner] < W;
                for (int64_t c = 0; c < D; ++c) {
                  double v = X(x, g, n, cyy[corner], cxx[corner], grp, c);
                  sgm += g_y[c] * cw[corner] * v;
                  sgy += g_y[c] * dwy[corner] * v;
                  sgx += g_y[c] * dwx[corner] * v;
                  agm += fabs(g_y[c]) * cw[corner] * fabs(v);
                  agy += fabs(g_y[c]) * fabs(dwy[corner]) * fabs(v);
                  agx += fabs(g_y[c]) * fabs(dwx[corner]) * fabs(v);
                  if (inb) {
                    int64_t q = ((n * H + cyy[corner]) * W + cxx[corner]) * C + grp * D + c;
                    gx[q] += m[k] * cw[corner] * g_y[c];
                    if (gx_abs) gx_abs[q] += fabs(m[k]) * cw[corner] * fabs(g_y[c]);
                  }
                }
              }
              gm[k] = sgm;
              gma[k] = agm;
              grow[2 * k + 1] = s * m[k] * sgy; /* d/d(dy): py = ... + s*dy */
              grow[2 * k] = s * m[k] * sgx;     /* d/d(dx) */
              if (garow) {
                garow[2 * k + 1] = fabs(s * m[k]) * agy;
                garow[2 * k] = fabs(s * m[k]) * agx;
              }
            }
          }
          if (!g[GSOFT]) {
            for (int64_t k = 0; k < K; ++k) {
              grow[2 * K + k] = gm[k];
              if (garow) garow[2 * K + k] = gma[k];
            }
          } else {
            /* softmax Jacobian: dL/dz_k = p_k (gm_k - sum_j p_j gm_j) */
            double dot = 0.0, adot = 0.0;
            for (int64_t k = 0; k < K; ++k) { dot += m[k] * gm[k]; adot += m[k] * gma[k]; }
            for (int64_t k = 0; k < K; ++k) {
              grow[2 * K + k] = m[k] * (gm[k] - dot);
              if (garow) garow[2 * K + k] = m[k] * (gma[k] + adot);
            }
          }
        }
      }
    }
  }
  return 0;
}
