/*
 * oracle_kernels.c -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * CPU restatement of the reference's compiled kernels, /root/reference/pkg/src/
 * deformtrack/kernels.py, in plain C. The row arithmetic is written in the same
 * operation order and the rows are carved into the same n_chunks contiguous chunks,
 * each accumulated into a private slab and folded in chunk order (kernels.py:9-13),
 * compiled with -ffp-contract=off like numba's fastmath-off LLVM build, so results are
 * expected to agree with the numba kernels bit for bit (pinned in
 * tests/test_oracle_golden.py against fixtures generated from the reference).
 *
 *   or_warp_and_rasterize   kernels.py:483-569
 *   or_icp_reduce           kernels.py:148-220  (+ _blend_at 55-78, _apply_blend 81-101,
 *                                               _blend_gradient 104-145, _fold_row 47-53)
 *   or_feature_reduce       kernels.py:222-284
 *   or_arap_reduce          kernels.py:341-467  (+ _angle_fold 287-338, _fold_quad 470-480)
 *   or_hamming_match        north-star part 3a (no reference twin): argmin popcount(a^b),
 *                           ties to the lowest frame index
 *
 * OpenMP parallelizes over chunks only, so the thread count never changes the bits.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NC 27
#define KM 16
static const double A_MIN_NORM = 1e-6;   /* energy.py:45 */
static const double A_COLL_EPS = 1e-14;  /* energy.py:46 */

static int tri(int i, int j) { return 6 * i - i * (i + 1) / 2 + j; }

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

static void chunk_range(int64_t n, int nch, int c, int64_t *lo, int64_t *hi) {
  *lo = n * c / nch;
  *hi = n * (c + 1) / nch;
}

static void fold(double *slab, int64_t ci, const double J[6], double wv) {
  double *p = slab + ci * NC;
  for (int i = 0; i < 6; ++i) {
    for (int j = i; j < 6; ++j) p[tri(i, j)] += J[i] * J[j];
    p[21 + i] += J[i] * wv;
  }
}

/* sign-aligned blend of row c against its first bound control */
static void blend(const double *W, const int64_t *idx, const double *al, int k, double B[8],
                  double sg[]) {
  const double *r = W + 8 * idx[0];
  const double rw = r[0], rx = r[1], ry = r[2], rz = r[3];
  for (int e = 0; e < 8; ++e) B[e] = 0.0;
  for (int s = 0; s < k; ++s) {
    const double *w = W + 8 * idx[s];
    const double dot = w[0] * rw + w[1] * rx + w[2] * ry + w[3] * rz;
    const double sgn = dot < 0.0 ? -1.0 : 1.0;
    sg[s] = sgn;
    const double cf = al[s] * sgn;
    for (int e = 0; e < 8; ++e) B[e] += cf * w[e];
  }
}

static void act(const double B[8], double px, double py, double pz, double *x0, double *x1,
                double *x2, double *s2o) {
  const double qw = B[0], qx = B[1], qy = B[2], qz = B[3];
  const double dw = B[4], dx = B[5], dy = B[6], dz = B[7];
  const double s2 = qw * qw + qx * qx + qy * qy + qz * qz;
  const double uu = qx * qx + qy * qy + qz * qz;
  const double qup = qx * px + qy * py + qz * pz;
  const double cx = qy * pz - qz * py, cy = qz * px - qx * pz, cz = qx * py - qy * px;
  const double tx = dy * qz - dz * qy, ty = dz * qx - dx * qz, tz = dx * qy - dy * qx;
  *x0 = ((qw * qw - uu) * px + 2.0 * qup * qx + 2.0 * qw * cx + 2.0 * (qw * dx - dw * qx - tx)) / s2;
  *x1 = ((qw * qw - uu) * py + 2.0 * qup * qy + 2.0 * qw * cy + 2.0 * (qw * dy - dw * qy - ty)) / s2;
  *x2 = ((qw * qw - uu) * pz + 2.0 * qup * qz + 2.0 * qw * cz + 2.0 * (qw * dz - dw * qz - tz)) / s2;
  *s2o = s2;
}

static void grad(const double B[8], double px, double py, double pz, double x0, double x1,
                 double x2, double s2, double G[3][8]) {
  const double qw = B[0], qx = B[1], qy = B[2], qz = B[3];
  const double dw = B[4], dx = B[5], dy = B[6], dz = B[7];
  const double qup = qx * px + qy * py + qz * pz;
  G[0][0] = (2.0 * qw * px + 2.0 * (qy * pz - qz * py) + 2.0 * dx - 2.0 * x0 * qw) / s2;
  G[1][0] = (2.0 * qw * py + 2.0 * (qz * px - qx * pz) + 2.0 * dy - 2.0 * x1 * qw) / s2;
  G[2][0] = (2.0 * qw * pz + 2.0 * (qx * py - qy * px) + 2.0 * dz - 2.0 * x2 * qw) / s2;
  G[0][1] = (-2.0 * px * qx + 2.0 * qx * px + 2.0 * qup - 2.0 * dw - 2.0 * x0 * qx) / s2;
  G[1][1] = (-2.0 * py * qx + 2.0 * qy * px - 2.0 * qw * pz - 2.0 * dz - 2.0 * x1 * qx) / s2;
  G[2][1] = (-2.0 * pz * qx + 2.0 * qz * px + 2.0 * qw * py + 2.0 * dy - 2.0 * x2 * qx) / s2;
  G[0][2] = (-2.0 * px * qy + 2.0 * qx * py + 2.0 * qw * pz + 2.0 * dz - 2.0 * x0 * qy) / s2;
  G[1][2] = (-2.0 * py * qy + 2.0 * qy * py + 2.0 * qup - 2.0 * dw - 2.0 * x1 * qy) / s2;
  G[2][2] = (-2.0 * pz * qy + 2.0 * qz * py - 2.0 * qw * px - 2.0 * dx - 2.0 * x2 * qy) / s2;
  G[0][3] = (-2.0 * px * qz + 2.0 * qx * pz - 2.0 * qw * py - 2.0 * dy - 2.0 * x0 * qz) / s2;
  G[1][3] = (-2.0 * py * qz + 2.0 * qy * pz + 2.0 * qw * px + 2.0 * dx - 2.0 * x1 * qz) / s2;
  G[2][3] = (-2.0 * pz * qz + 2.0 * qz * pz + 2.0 * qup - 2.0 * dw - 2.0 * x2 * qz) / s2;
  G[0][4] = -2.0 * qx / s2;
  G[1][4] = -2.0 * qy / s2;
  G[2][4] = -2.0 * qz / s2;
  G[0][5] = 2.0 * qw / s2;
  G[1][5] = 2.0 * qz / s2;
  G[2][5] = -2.0 * qy / s2;
  G[0][6] = -2.0 * qz / s2;
  G[1][6] = 2.0 * qw / s2;
  G[2][6] = 2.0 * qx / s2;
  G[0][7] = 2.0 * qy / s2;
  G[1][7] = -2.0 * qx / s2;
  G[2][7] = 2.0 * qw / s2;
}

/* fold chunk slabs in chunk order: out = ((0 + s0) + s1) + ... */
static void fold_slabs(const double *slabs, int nch, int64_t len, double *out) {
  for (int64_t i = 0; i < len; ++i) out[i] = 0.0;
  for (int c = 0; c < nch; ++c) {
    const double *s = slabs + (int64_t)c * len;
    for (int64_t i = 0; i < len; ++i) out[i] += s[i];
  }
}

/* ---------------------------------------------------------------------------- */
int or_icp_reduce(const double *pts, const double *onrm, const double *obs, const int64_t *bidx,
                  const double *alpha, int64_t n, int k, const double *W, const double *basis,
                  double tukey, const double *frozen, int use_frozen, int want_jac, int nch,
                  int64_t m, double *partial, double *support, double *cost, double *r_out) {
  if (k > KM || nch < 1) return 1;
  double *sp = calloc((size_t)nch * m * NC, sizeof(double));
  double *ss = calloc((size_t)nch * m, sizeof(double));
  double *sc = calloc((size_t)nch * m, sizeof(double));
  if (!sp || !ss || !sc) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int ch = 0; ch < nch; ++ch) {
    int64_t lo, hi;
    chunk_range(n, nch, ch, &lo, &hi);
    double *P = sp + (int64_t)ch * m * NC, *S = ss + (int64_t)ch * m, *Co = sc + (int64_t)ch * m;
    double B[8], sg[KM], G[3][8], gn[8], J[6];
    for (int64_t c = lo; c < hi; ++c) {
      blend(W, bidx + c * k, alpha + c * k, k, B, sg);
      const double px = pts[3 * c], py = pts[3 * c + 1], pz = pts[3 * c + 2];
      double x0, x1, x2, s2;
      act(B, px, py, pz, &x0, &x1, &x2, &s2);
      const double n0 = onrm[3 * c], n1 = onrm[3 * c + 1], n2 = onrm[3 * c + 2];
      const double r = n0 * (x0 - obs[3 * c]) + n1 * (x1 - obs[3 * c + 1]) + n2 * (x2 - obs[3 * c + 2]);
      r_out[c] = r;
      double rs;
      if (use_frozen) {
        rs = frozen[c];
      } else {
        const double u = r / tukey;
        if (fabs(u) < 1.0) {
          const double w = 1.0 - u * u;
          rs = sqrt(w * w);
        } else {
          rs = 0.0;
        }
      }
      const double rs2 = rs * rs;
      if (want_jac) {
        grad(B, px, py, pz, x0, x1, x2, s2, G);
        for (int e = 0; e < 8; ++e) gn[e] = n0 * G[0][e] + n1 * G[1][e] + n2 * G[2][e];
      }
      for (int s = 0; s < k; ++s) {
        const int64_t ci = bidx[c * k + s];
        const double a = alpha[c * k + s];
        S[ci] += rs2 * a;
        const double sw = rs * sqrt(a);
        const double wv = sw * r;
        Co[ci] += wv * wv;
        if (want_jac) {
          const double cf = sw * a * sg[s];
          const double *K = basis + ci * 48;
          for (int d = 0; d < 6; ++d) {
            double acc = 0.0;
            for (int e = 0; e < 8; ++e) acc += gn[e] * K[e * 6 + d];
            J[d] = cf * acc;
          }
          fold(P, ci, J, wv);
        }
      }
    }
  }
  fold_slabs(sp, nch, m * NC, partial);
  fold_slabs(ss, nch, m, support);
  fold_slabs(sc, nch, m, cost);
  free(sp);
  free(ss);
  free(sc);
  return 0;
}

int or_feature_reduce(const double *pts, const double *obs, const double *mw, const int64_t *bidx,
                      const double *alpha, int64_t n, int k, const double *W, const double *basis,
                      double fw, int want_jac, int nch, int64_t m, double *partial,
                      double *support, double *cost) {
  if (k > KM || nch < 1) return 1;
  double *sp = calloc((size_t)nch * m * NC, sizeof(double));
  double *ss = calloc((size_t)nch * m, sizeof(double));
  double *sc = calloc((size_t)nch * m, sizeof(double));
  if (!sp || !ss || !sc) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int ch = 0; ch < nch; ++ch) {
    int64_t lo, hi;
    chunk_range(n, nch, ch, &lo, &hi);
    double *P = sp + (int64_t)ch * m * NC, *S = ss + (int64_t)ch * m, *Co = sc + (int64_t)ch * m;
    double B[8], sg[KM], G[3][8], GK[3][6];
    for (int64_t c = lo; c < hi; ++c) {
      blend(W, bidx + c * k, alpha + c * k, k, B, sg);
      const double px = pts[3 * c], py = pts[3 * c + 1], pz = pts[3 * c + 2];
      double x0, x1, x2, s2;
      act(B, px, py, pz, &x0, &x1, &x2, &s2);
      const double r0 = x0 - obs[3 * c], r1 = x1 - obs[3 * c + 1], r2 = x2 - obs[3 * c + 2];
      if (want_jac) grad(B, px, py, pz, x0, x1, x2, s2, G);
      for (int s = 0; s < k; ++s) {
        const int64_t ci = bidx[c * k + s];
        const double a = alpha[c * k + s];
        const double wp = fw * mw[c] * a;
        S[ci] += wp;
        const double sw = sqrt(wp);
        const double v0 = sw * r0, v1 = sw * r1, v2 = sw * r2;
        Co[ci] += v0 * v0 + v1 * v1 + v2 * v2;
        if (want_jac) {
          const double cf = sw * a * sg[s];
          const double *K = basis + ci * 48;
          for (int cmp = 0; cmp < 3; ++cmp)
            for (int d = 0; d < 6; ++d) {
              double acc = 0.0;
              for (int e = 0; e < 8; ++e) acc += G[cmp][e] * K[e * 6 + d];
              GK[cmp][d] = cf * acc;
            }
          double *p = P + ci * NC;
          for (int i = 0; i < 6; ++i) {
            for (int j = i; j < 6; ++j)
              p[tri(i, j)] += GK[0][i] * GK[0][j] + GK[1][i] * GK[1][j] + GK[2][i] * GK[2][j];
            p[21 + i] += GK[0][i] * v0 + GK[1][i] * v1 + GK[2][i] * v2;
          }
        }
      }
    }
  }
  fold_slabs(sp, nch, m * NC, partial);
  fold_slabs(ss, nch, m, support);
  fold_slabs(sc, nch, m, cost);
  free(sp);
  free(ss);
  free(sc);
  return 0;
}

/* one bending-angle row (kernels.py:287-338) folded into bins ia (a side) and ib */
static void angle_row(int64_t ia, int64_t ib, double ax, double ay, double az, double bx,
                      double by, double bz, double patx, double paty, double patz, double pbtx,
                      double pbty, double pbtz, double sw, double *P, double *Co, int jac) {
  const double na = sqrt(ax * ax + ay * ay + az * az);
  const double nb = sqrt(bx * bx + by * by + bz * bz);
  const int ok = na > A_MIN_NORM && nb > A_MIN_NORM;
  const double nas = ok ? na : 1.0, nbs = ok ? nb : 1.0;
  const double ahx = ax / nas, ahy = ay / nas, ahz = az / nas;
  const double bhx = bx / nbs, bhy = by / nbs, bhz = bz / nbs;
  double c = ahx * bhx + ahy * bhy + ahz * bhz;
  if (c > 1.0) c = 1.0;
  else if (c < -1.0) c = -1.0;
  const int nz = (1.0 - c) < A_COLL_EPS;
  const int np_ = (1.0 + c) < A_COLL_EPS;
  const double val = (ok && !nz) ? acos(c) : 0.0;
  const double wv = sw * val;
  Co[ia] += wv * wv;
  Co[ib] += wv * wv;
  if (!jac) return;
  double is = 0.0;
  if (ok && !nz && !np_) {
    const double q = 1.0 - c * c;
    is = -1.0 / sqrt(q > 1e-300 ? q : 1e-300);
  }
  const double gax = is * (bhx - c * ahx) / nas, gay = is * (bhy - c * ahy) / nas,
               gaz = is * (bhz - c * ahz) / nas;
  const double gbx = is * (ahx - c * bhx) / nbs, gby = is * (ahy - c * bhy) / nbs,
               gbz = is * (ahz - c * bhz) / nbs;
  double J[6];
  J[0] = sw * ((ay * gaz - az * gay) - (paty * gbz - patz * gby));
  J[1] = sw * ((az * gax - ax * gaz) - (patz * gbx - patx * gbz));
  J[2] = sw * ((ax * gay - ay * gax) - (patx * gby - paty * gbx));
  J[3] = sw * (-gbx);
  J[4] = sw * (-gby);
  J[5] = sw * (-gbz);
  fold(P, ia, J, wv);
  J[0] = sw * (pbty * gbz - pbtz * gby);
  J[1] = sw * (pbtz * gbx - pbtx * gbz);
  J[2] = sw * (pbtx * gby - pbty * gbx);
  J[3] = sw * gbx;
  J[4] = sw * gby;
  J[5] = sw * gbz;
  fold(P, ib, J, wv);
}

static void quad(double *P, int64_t ci, const double J4[4][3], double d0, double d1, double d2,
                 double d3, double sw) {
  double *p = P + ci * NC;
  for (int i = 0; i < 3; ++i) {
    for (int j = i; j < 3; ++j) {
      const double acc = J4[0][i] * J4[0][j] + J4[1][i] * J4[1][j] + J4[2][i] * J4[2][j] +
                         J4[3][i] * J4[3][j];
      p[tri(i, j)] += sw * sw * acc;
    }
    p[21 + i] += sw * sw * (J4[0][i] * d0 + J4[1][i] * d1 + J4[2][i] * d2 + J4[3][i] * d3);
  }
}

static void tf(const double *R, const double *t, double x, double y, double z, double o[3]) {
  o[0] = R[0] * x + R[1] * y + R[2] * z + t[0];
  o[1] = R[3] * x + R[4] * y + R[5] * z + t[1];
  o[2] = R[6] * x + R[7] * y + R[8] * z + t[2];
}

int or_arap_reduce(const double *cp, const double *R, const double *t, const double *W,
                   const int64_t *edges, const double *ew, int64_t ne, const double *wa,
                   double aw, double rw, int jac, int nch, int64_t m, double *partial,
                   double *cost) {
  if (nch < 1) return 1;
  double *sp = calloc((size_t)nch * m * NC, sizeof(double));
  double *sc = calloc((size_t)nch * m, sizeof(double));
  if (!sp || !sc) return 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int ch = 0; ch < nch; ++ch) {
    int64_t lo, hi;
    chunk_range(ne, nch, ch, &lo, &hi);
    double *P = sp + (int64_t)ch * m * NC, *Co = sc + (int64_t)ch * m;
    double J[6], J4[4][3];
    for (int64_t e = lo; e < hi; ++e) {
      const int64_t i0 = edges[2 * e], i1 = edges[2 * e + 1];
      const double base = ew[e] * 0.5 * (wa[i0] + wa[i1]);
      const double *p0 = cp + 3 * i0, *p1 = cp + 3 * i1;
      const double *R0 = R + 9 * i0, *R1 = R + 9 * i1, *t0 = t + 3 * i0, *t1 = t + 3 * i1;
      double a0[3], a1[3];
      tf(R0, t0, p0[0], p0[1], p0[2], a0);
      tf(R1, t1, p1[0], p1[1], p1[2], a1);
      /* length */
      const double rx = p1[0] - p0[0], ry = p1[1] - p0[1], rz = p1[2] - p0[2];
      const double rest = sqrt(rx * rx + ry * ry + rz * rz);
      const double bx = a1[0] - a0[0], by = a1[1] - a0[1], bz = a1[2] - a0[2];
      const double ln = sqrt(bx * bx + by * by + bz * bz);
      const double val = ln - rest;
      const double sw = sqrt(0.5 * base);
      const double wv = sw * val;
      Co[i0] += wv * wv;
      Co[i1] += wv * wv;
      if (jac) {
        double hx = 0.0, hy = 0.0, hz = 0.0;
        if (ln > 1e-9) {
          hx = bx / ln;
          hy = by / ln;
          hz = bz / ln;
        }
        J[0] = sw * (a0[1] * (-hz) - a0[2] * (-hy));
        J[1] = sw * (a0[2] * (-hx) - a0[0] * (-hz));
        J[2] = sw * (a0[0] * (-hy) - a0[1] * (-hx));
        J[3] = sw * (-hx);
        J[4] = sw * (-hy);
        J[5] = sw * (-hz);
        fold(P, i0, J, wv);
        J[0] = sw * (a1[1] * hz - a1[2] * hy);
        J[1] = sw * (a1[2] * hx - a1[0] * hz);
        J[2] = sw * (a1[0] * hy - a1[1] * hx);
        J[3] = sw * hx;
        J[4] = sw * hy;
        J[5] = sw * hz;
        fold(P, i1, J, wv);
      }
      /* bending angle, both directions */
      const double swa = sqrt(0.5 * base * aw);
      double c01[3], c10[3];
      tf(R0, t0, p1[0], p1[1], p1[2], c01);
      angle_row(i0, i1, c01[0] - a0[0], c01[1] - a0[1], c01[2] - a0[2], a1[0] - a0[0],
                a1[1] - a0[1], a1[2] - a0[2], a0[0], a0[1], a0[2], a1[0], a1[1], a1[2], swa, P, Co,
                jac);
      tf(R1, t1, p0[0], p0[1], p0[2], c10);
      angle_row(i1, i0, c10[0] - a1[0], c10[1] - a1[1], c10[2] - a1[2], a0[0] - a1[0],
                a0[1] - a1[1], a0[2] - a1[2], a1[0], a1[1], a1[2], a0[0], a0[1], a0[2], swa, P, Co,
                jac);
      /* rotation consistency */
      const double swr = sqrt(0.5 * base * rw);
      const double *q0 = W + 8 * i0, *q1 = W + 8 * i1;
      const double dq = q0[0] * q1[0] + q0[1] * q1[1] + q0[2] * q1[2] + q0[3] * q1[3];
      const double sg = dq < 0.0 ? -1.0 : 1.0;
      const double d0 = q0[0] - sg * q1[0], d1 = q0[1] - sg * q1[1], d2 = q0[2] - sg * q1[2],
                   d3 = q0[3] - sg * q1[3];
      const double cc = swr * swr * (d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3);
      Co[i0] += cc;
      Co[i1] += cc;
      if (jac) {
        J4[0][0] = -0.5 * q0[1]; J4[0][1] = -0.5 * q0[2]; J4[0][2] = -0.5 * q0[3];
        J4[1][0] = 0.5 * q0[0];  J4[1][1] = 0.5 * q0[3];  J4[1][2] = -0.5 * q0[2];
        J4[2][0] = -0.5 * q0[3]; J4[2][1] = 0.5 * q0[0];  J4[2][2] = 0.5 * q0[1];
        J4[3][0] = 0.5 * q0[2];  J4[3][1] = -0.5 * q0[1]; J4[3][2] = 0.5 * q0[0];
        quad(P, i0, J4, d0, d1, d2, d3, swr);
        const double h = -sg * 0.5;
        J4[0][0] = h * q1[1] * -1.0; J4[0][1] = h * q1[2] * -1.0; J4[0][2] = h * q1[3] * -1.0;
        J4[1][0] = h * q1[0];        J4[1][1] = h * q1[3];        J4[1][2] = h * -q1[2];
        J4[2][0] = h * -q1[3];       J4[2][1] = h * q1[0];        J4[2][2] = h * q1[1];
        J4[3][0] = h * q1[2];        J4[3][1] = h * -q1[1];       J4[3][2] = h * q1[0];
        quad(P, i1, J4, d0, d1, d2, d3, swr);
      }
    }
  }
  fold_slabs(sp, nch, m * NC, partial);
  fold_slabs(sc, nch, m, cost);
  free(sp);
  free(sc);
  return 0;
}

/* ---------------------------------------------------------------------------- */
int or_warp_and_rasterize(const double *pts, const double *nrm, const int64_t *bidx,
                          const double *alpha, int64_t n, int k, const double *W,
                          const double *depth, const uint8_t *dvalid, const double *onrm,
                          int64_t height, int64_t width, double fx, double fy, double cx,
                          double cy, double gate, double cos_gate, int nch, double *out_p,
                          double *out_n, uint8_t *valid, double *obs_p, double *obs_n,
                          int64_t *pixels) {
  if (k > KM || nch < 1) return 1;
  memset(valid, 0, (size_t)n);
  memset(obs_p, 0, sizeof(double) * 3 * n);
  memset(obs_n, 0, sizeof(double) * 3 * n);
  for (int64_t i = 0; i < 2 * n; ++i) pixels[i] = -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int ch = 0; ch < nch; ++ch) {
    int64_t lo, hi;
    chunk_range(n, nch, ch, &lo, &hi);
    double B[8], sg[KM];
    for (int64_t c = lo; c < hi; ++c) {
      blend(W, bidx + c * k, alpha + c * k, k, B, sg);
      double x0, x1, x2, s2u;
      act(B, pts[3 * c], pts[3 * c + 1], pts[3 * c + 2], &x0, &x1, &x2, &s2u);
      out_p[3 * c] = x0;
      out_p[3 * c + 1] = x1;
      out_p[3 * c + 2] = x2;
      const double qw = B[0], qx = B[1], qy = B[2], qz = B[3];
      const double s2 = qw * qw + qx * qx + qy * qy + qz * qz;
      const double uu = qx * qx + qy * qy + qz * qz;
      const double vx = nrm[3 * c], vy = nrm[3 * c + 1], vz = nrm[3 * c + 2];
      const double quv = qx * vx + qy * vy + qz * vz;
      double r0 = ((qw * qw - uu) * vx + 2.0 * quv * qx + 2.0 * qw * (qy * vz - qz * vy)) / s2;
      double r1 = ((qw * qw - uu) * vy + 2.0 * quv * qy + 2.0 * qw * (qz * vx - qx * vz)) / s2;
      double r2 = ((qw * qw - uu) * vz + 2.0 * quv * qz + 2.0 * qw * (qx * vy - qy * vx)) / s2;
      const double ln = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
      if (ln > 0.0) {
        r0 /= ln;
        r1 /= ln;
        r2 /= ln;
      }
      out_n[3 * c] = r0;
      out_n[3 * c + 1] = r1;
      out_n[3 * c + 2] = r2;
      if (x2 <= 0.0) continue;
      const double uf = rint(fx * x0 / x2 + cx);
      const double vf = rint(fy * x1 / x2 + cy);
      if (!(uf >= 0.0 && uf < (double)width && vf >= 0.0 && vf < (double)height)) continue;
      const int64_t ui = (int64_t)uf, vi = (int64_t)vf;
      const int64_t pix = vi * width + ui;
      if (!dvalid[pix]) continue;
      const double d = depth[pix];
      const double ox = ((double)ui - cx) / fx * d;
      const double oy = ((double)vi - cy) / fy * d;
      const double gx = onrm[3 * pix], gy = onrm[3 * pix + 1], gz = onrm[3 * pix + 2];
      if (gx * gx + gy * gy + gz * gz <= 0.25) continue;
      const double dx = ox - x0, dy = oy - x1, dz = d - x2;
      if (sqrt(dx * dx + dy * dy + dz * dz) >= gate) continue;
      if (gx * r0 + gy * r1 + gz * r2 <= cos_gate) continue;
      valid[c] = 1;
      obs_p[3 * c] = ox;
      obs_p[3 * c + 1] = oy;
      obs_p[3 * c + 2] = d;
      obs_n[3 * c] = gx;
      obs_n[3 * c + 1] = gy;
      obs_n[3 * c + 2] = gz;
      pixels[2 * c] = ui;
      pixels[2 * c + 1] = vi;
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------------- */
int or_hamming_match(const uint8_t *td, int64_t nt, const uint8_t *fd, int64_t nf, int32_t *idx,
                     int32_t *dist) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < nt; ++t) {
    const uint64_t *a = (const uint64_t *)(td + 32 * t);
    int best = 257, bi = -1;
    for (int64_t f = 0; f < nf; ++f) {
      const uint64_t *b = (const uint64_t *)(fd + 32 * f);
      const int d = __builtin_popcountll(a[0] ^ b[0]) + __builtin_popcountll(a[1] ^ b[1]) +
                    __builtin_popcountll(a[2] ^ b[2]) + __builtin_popcountll(a[3] ^ b[3]);
      if (d < best) {
        best = d;
        bi = (int)f;
      }
    }
    idx[t] = bi;
    dist[t] = best;
  }
  return 0;
}
