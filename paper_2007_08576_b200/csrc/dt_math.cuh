// dt_math.cuh -- per-row device math of the deformation-tracking hot path.
//
// Every function restates one piece of the reference's row arithmetic with the same
// operation order (the library is compiled with -fmad=false, so the device evaluates
// the same IEEE sequence as numba with fastmath off, kernels.py:9-13). Citations are
// to /root/reference/pkg/src/deformtrack/<file>:<line>.
#pragma once

#include <cstdint>
#include <math.h>

#include "dt_common.cuh"

namespace dt {

constexpr int KMAX = 8;                       // largest bind_k the device path handles
constexpr int NCOLS = 27;                     // 21 triu(J^T J) + 6 J^T r, kernels.py:15-21
constexpr double ANGLE_MIN_NORM = 1e-6;       // energy.py:45
constexpr double ANGLE_COLLINEAR_EPS = 1e-14; // energy.py:46

__host__ __device__ __forceinline__ int triu_col(int i, int j) {
  // row-major upper-triangle index of (i, j), i <= j (kernels.py:41-44)
  return 6 * i - i * (i + 1) / 2 + j;
}

// Sign-aligned weighted warp sum (kernels.py:55-78, warpfield.py:213-233): every bound
// warp is flipped into the hemisphere of the FIRST (nearest) bound control, then the
// weighted 8-vectors are summed without normalization.
template <typename IndexT>
__device__ __forceinline__ void blend_at(const double* __restrict__ warps, const IndexT* idx,
                                         const double* w, int k, double B[8], double sgn[KMAX]) {
  const double* r = warps + 8 * (int64_t)idx[0];
  const double rw = r[0], rx = r[1], ry = r[2], rz = r[3];
#pragma unroll
  for (int e = 0; e < 8; ++e) B[e] = 0.0;
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    if (s < k) {
      const double* W = warps + 8 * (int64_t)idx[s];
      const double dot = W[0] * rw + W[1] * rx + W[2] * ry + W[3] * rz;
      const double sg = dot < 0.0 ? -1.0 : 1.0;
      sgn[s] = sg;
      const double coef = w[s] * sg;
#pragma unroll
      for (int e = 0; e < 8; ++e) B[e] += coef * W[e];
    }
  }
}

// blend_at with a compile-time slot bound KM (k <= KM)
template <int KM, typename IndexT>
__device__ __forceinline__ void blend_at_k(const double* __restrict__ warps, const IndexT* idx,
                                         const double* w, int k, double B[8], double sgn[KM]) {
  const double* r = warps + 8 * (int64_t)idx[0];
  const double rw = r[0], rx = r[1], ry = r[2], rz = r[3];
#pragma unroll
  for (int e = 0; e < 8; ++e) B[e] = 0.0;
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    DT_DCHECK(s >= k || idx[s] >= 0);
    if (s < k) {
      const double* W = warps + 8 * (int64_t)idx[s];
      const double dot = W[0] * rw + W[1] * rx + W[2] * ry + W[3] * rz;
      const double sg = dot < 0.0 ? -1.0 : 1.0;
      sgn[s] = sg;
      const double coef = w[s] * sg;
#pragma unroll
      for (int e = 0; e < 8; ++e) B[e] += coef * W[e];
    }
  }
}

// Normalized dual-quaternion action of an unnormalized sum B on point p
// (kernels.py:81-101, geometry.dq_apply_batch geometry.py:215-235):
// x = (q p q* + 2 vec(d q*)) / |q|^2.
__device__ __forceinline__ void apply_blend(const double B[8], double px, double py, double pz,
                                            double& x0, double& x1, double& x2, double& s2) {
  const double qw = B[0], qx = B[1], qy = B[2], qz = B[3];
  const double dw = B[4], dx = B[5], dy = B[6], dz = B[7];
  s2 = qw * qw + qx * qx + qy * qy + qz * qz;
  const double uu = qx * qx + qy * qy + qz * qz;
  const double qup = qx * px + qy * py + qz * pz;
  const double cx = qy * pz - qz * py;
  const double cy = qz * px - qx * pz;
  const double cz = qx * py - qy * px;
  const double tx = dy * qz - dz * qy;
  const double ty = dz * qx - dx * qz;
  const double tz = dx * qy - dy * qx;
  const double a = qw * qw - uu;
  x0 = (a * px + 2.0 * qup * qx + 2.0 * qw * cx + 2.0 * (qw * dx - dw * qx - tx)) / s2;
  x1 = (a * py + 2.0 * qup * qy + 2.0 * qw * cy + 2.0 * (qw * dy - dw * qy - ty)) / s2;
  x2 = (a * pz + 2.0 * qup * qz + 2.0 * qw * cz + 2.0 * (qw * dz - dw * qz - tz)) / s2;
}

// Rotation of a direction by the real part of B, then renormalized
// (kernels.py:518-536; geometry.dq_rotate_batch + warpfield.warp_all normalization).
__device__ __forceinline__ void rotate_normal(const double B[8], double vx, double vy, double vz,
                                              double& r0, double& r1, double& r2) {
  const double qw = B[0], qx = B[1], qy = B[2], qz = B[3];
  const double s2 = qw * qw + qx * qx + qy * qy + qz * qz;
  const double uu = qx * qx + qy * qy + qz * qz;
  const double quv = qx * vx + qy * vy + qz * vz;
  const double a = qw * qw - uu;
  r0 = (a * vx + 2.0 * quv * qx + 2.0 * qw * (qy * vz - qz * vy)) / s2;
  r1 = (a * vy + 2.0 * quv * qy + 2.0 * qw * (qz * vx - qx * vz)) / s2;
  r2 = (a * vz + 2.0 * quv * qz + 2.0 * qw * (qx * vy - qy * vx)) / s2;
  const double ln = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
  if (ln > 0.0) {
    r0 /= ln;
    r1 /= ln;
    r2 /= ln;
  }
}

// d(action)/dB by the quotient rule, G (3 x 8) row-major (kernels.py:104-145,
// energy.blend_apply_jacobian energy.py:222-266).
__device__ __forceinline__ void blend_gradient(const double B[8], double px, double py, double pz,
                                               double x0, double x1, double x2, double s2,
                                               double G[24]) {
  const double qw = B[0], qx = B[1], qy = B[2], qz = B[3];
  const double dw = B[4], dx = B[5], dy = B[6], dz = B[7];
  const double qup = qx * px + qy * py + qz * pz;
  // column 0: d/dqw
  G[0 * 8 + 0] = (2.0 * qw * px + 2.0 * (qy * pz - qz * py) + 2.0 * dx - 2.0 * x0 * qw) / s2;
  G[1 * 8 + 0] = (2.0 * qw * py + 2.0 * (qz * px - qx * pz) + 2.0 * dy - 2.0 * x1 * qw) / s2;
  G[2 * 8 + 0] = (2.0 * qw * pz + 2.0 * (qx * py - qy * px) + 2.0 * dz - 2.0 * x2 * qw) / s2;
  // column 1: d/dqx
  G[0 * 8 + 1] = (-2.0 * px * qx + 2.0 * qx * px + 2.0 * qup - 2.0 * dw - 2.0 * x0 * qx) / s2;
  G[1 * 8 + 1] = (-2.0 * py * qx + 2.0 * qy * px - 2.0 * qw * pz - 2.0 * dz - 2.0 * x1 * qx) / s2;
  G[2 * 8 + 1] = (-2.0 * pz * qx + 2.0 * qz * px + 2.0 * qw * py + 2.0 * dy - 2.0 * x2 * qx) / s2;
  // column 2: d/dqy
  G[0 * 8 + 2] = (-2.0 * px * qy + 2.0 * qx * py + 2.0 * qw * pz + 2.0 * dz - 2.0 * x0 * qy) / s2;
  G[1 * 8 + 2] = (-2.0 * py * qy + 2.0 * qy * py + 2.0 * qup - 2.0 * dw - 2.0 * x1 * qy) / s2;
  G[2 * 8 + 2] = (-2.0 * pz * qy + 2.0 * qz * py - 2.0 * qw * px - 2.0 * dx - 2.0 * x2 * qy) / s2;
  // column 3: d/dqz
  G[0 * 8 + 3] = (-2.0 * px * qz + 2.0 * qx * pz - 2.0 * qw * py - 2.0 * dy - 2.0 * x0 * qz) / s2;
  G[1 * 8 + 3] = (-2.0 * py * qz + 2.0 * qy * pz + 2.0 * qw * px + 2.0 * dx - 2.0 * x1 * qz) / s2;
  G[2 * 8 + 3] = (-2.0 * pz * qz + 2.0 * qz * pz + 2.0 * qup - 2.0 * dw - 2.0 * x2 * qz) / s2;
  // columns 4..7: d/d(dual)
  G[0 * 8 + 4] = -2.0 * qx / s2;
  G[1 * 8 + 4] = -2.0 * qy / s2;
  G[2 * 8 + 4] = -2.0 * qz / s2;
  G[0 * 8 + 5] = 2.0 * qw / s2;
  G[1 * 8 + 5] = 2.0 * qz / s2;
  G[2 * 8 + 5] = -2.0 * qy / s2;
  G[0 * 8 + 6] = -2.0 * qz / s2;
  G[1 * 8 + 6] = 2.0 * qw / s2;
  G[2 * 8 + 6] = 2.0 * qx / s2;
  G[0 * 8 + 7] = 2.0 * qy / s2;
  G[1 * 8 + 7] = -2.0 * qx / s2;
  G[2 * 8 + 7] = 2.0 * qw / s2;
}

// Half pure-left-multiply matrix of a quaternion, 4 x 3 row-major
// (0.5 * energy._pure_left_mul, energy.py:192-202): row 0 = -u, rows 1..3 = w I - [u]x.
__device__ __forceinline__ void half_left_mul(double w, double x, double y, double z, double P[12]) {
  P[0] = 0.5 * -x;  P[1] = 0.5 * -y;  P[2] = 0.5 * -z;
  P[3] = 0.5 * w;   P[4] = 0.5 * z;   P[5] = 0.5 * -y;
  P[6] = 0.5 * -z;  P[7] = 0.5 * w;   P[8] = 0.5 * x;
  P[9] = 0.5 * y;   P[10] = 0.5 * -x; P[11] = 0.5 * w;
}

// The increment basis K (8 x 6) of one warp (energy.warp_increment_basis,
// energy.py:205-219) in compact form: Kr = 0.5 L(real), Kd = 0.5 L(dual);
// K[0:4,0:3] = Kr, K[4:8,0:3] = Kd, K[4:8,3:6] = Kr, K[0:4,3:6] = 0.
struct Basis {
  double Kr[12];
  double Kd[12];
};

__device__ __forceinline__ void make_basis(const double* W, Basis& K) {
  half_left_mul(W[0], W[1], W[2], W[3], K.Kr);
  half_left_mul(W[4], W[5], W[6], W[7], K.Kd);
}

// acc_d = sum_e g[e] * K[e][d] accumulated in e order from 0.0 (kernels.py:204-210);
// the structural zeros of K are skipped, which leaves the IEEE result unchanged.
__device__ __forceinline__ void basis_project(const double g[8], const double* Kr, const double* Kd,
                                             double acc[6]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double a = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) a += g[e] * Kr[e * 3 + d];
#pragma unroll
    for (int e = 0; e < 4; ++e) a += g[4 + e] * Kd[e * 3 + d];
    acc[d] = a;
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double a = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) a += g[4 + e] * Kr[e * 3 + d];
    acc[3 + d] = a;
  }
}

// Same projection against a dense (8,6) basis row-major (operator-level path, where the
// basis arrives as an input exactly like kernels.icp_reduce's `basis` argument).
__device__ __forceinline__ void basis_project_dense(const double g[8], const double* K, double acc[6]) {
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    double a = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) a += g[e] * K[e * 6 + d];
    acc[d] = a;
  }
}

// Rank-1 fold of one scalar row into 27 accumulators (kernels.py:47-53).
__device__ __forceinline__ void fold_row(double* acc, const double J[6], double wv) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = i; j < 6; ++j) acc[triu_col(i, j)] += J[i] * J[j];
    acc[21 + i] += J[i] * wv;
  }
}

// Tukey square-root weight |1 - u^2| inside |u| < 1 (kernels.py:184-192).
// tukey_sqrt with a precomputed 1/scale and sqrt(w^2) = w (ulp-level; solver-internal)
__device__ __forceinline__ double tukey_fast(double r, double inv_scale) {
  const double u = r * inv_scale;
  return fabs(u) < 1.0 ? 1.0 - u * u : 0.0;
}

__device__ __forceinline__ double tukey_sqrt(double r, double scale) {
  const double u = r / scale;
  if (fabs(u) < 1.0) {
    const double w = 1.0 - u * u;
    return sqrt(w * w);
  }
  return 0.0;
}

// Rigid transform of a (not necessarily unit) dual quaternion
// (geometry.dq_to_transform_batch, geometry.py:238-264): R row-major 3x3, t.
__device__ __forceinline__ void dq_to_transform(const double* W, double R[9], double t[3]) {
  const double w = W[0], x = W[1], y = W[2], z = W[3];
  const double dw = W[4], dx = W[5], dy = W[6], dz = W[7];
  const double s2 = w * w + x * x + y * y + z * z;
  R[0] = (w * w + x * x - y * y - z * z) / s2;
  R[1] = (2.0 * (x * y - w * z)) / s2;
  R[2] = (2.0 * (x * z + w * y)) / s2;
  R[3] = (2.0 * (x * y + w * z)) / s2;
  R[4] = (w * w - x * x + y * y - z * z) / s2;
  R[5] = (2.0 * (y * z - w * x)) / s2;
  R[6] = (2.0 * (x * z - w * y)) / s2;
  R[7] = (2.0 * (y * z + w * x)) / s2;
  R[8] = (w * w - x * x - y * y + z * z) / s2;
  // t = 2 (qw du - dw qu - du x qu) / s2 (cross3 order: geometry.py:51-63)
  const double c0 = dy * z - dz * y;
  const double c1 = dz * x - dx * z;
  const double c2 = dx * y - dy * x;
  t[0] = 2.0 * (w * dx - dw * x - c0) / s2;
  t[1] = 2.0 * (w * dy - dw * y - c1) / s2;
  t[2] = 2.0 * (w * dz - dw * z - c2) / s2;
}

// dq_to_transform with one reciprocal instead of 12 divisions (ulp-level difference;
// used inside the LM solver, whose parity is tolerance-based)
__device__ __forceinline__ void dq_to_transform_fast(const double* W, double R[9], double t[3]) {
  const double w = W[0], x = W[1], y = W[2], z = W[3];
  const double dw = W[4], dx = W[5], dy = W[6], dz = W[7];
  const double s2 = w * w + x * x + y * y + z * z;
  const double is = 1.0 / s2;
  R[0] = (w * w + x * x - y * y - z * z) * is;
  R[1] = (2.0 * (x * y - w * z)) * is;
  R[2] = (2.0 * (x * z + w * y)) * is;
  R[3] = (2.0 * (x * y + w * z)) * is;
  R[4] = (w * w - x * x + y * y - z * z) * is;
  R[5] = (2.0 * (y * z - w * x)) * is;
  R[6] = (2.0 * (x * z - w * y)) * is;
  R[7] = (2.0 * (y * z + w * x)) * is;
  R[8] = (w * w - x * x - y * y + z * z) * is;
  // t = 2 (qw du - dw qu - du x qu) / s2 (cross3 order: geometry.py:51-63)
  const double c0 = dy * z - dz * y;
  const double c1 = dz * x - dx * z;
  const double c2 = dx * y - dy * x;
  t[0] = 2.0 * (w * dx - dw * x - c0) * is;
  t[1] = 2.0 * (w * dy - dw * y - c1) * is;
  t[2] = 2.0 * (w * dz - dw * z - c2) * is;
}

__device__ __forceinline__ void xform(const double R[9], const double t[3], double px, double py,
                                      double pz, double o[3]) {
  o[0] = R[0] * px + R[1] * py + R[2] * pz + t[0];
  o[1] = R[3] * px + R[4] * py + R[5] * pz + t[1];
  o[2] = R[6] * px + R[7] * py + R[8] * pz + t[2];
}

// ---------------------------------------------------------------------------------
// ARAP rows of one connection, evaluated for ONE endpoint bin (kernels.py:341-467).
// The reference walks each edge once and folds rows into both endpoint bins; the
// device walks each control's incident edges and evaluates only the rows binned to
// that control, so the per-control sums need no atomics. `side` = 0 when the bin is
// edges[e,0], 1 when it is edges[e,1].
// ---------------------------------------------------------------------------------

// One bending-angle row (kernels.py:287-338). Returns the row's weighted value wv;
// when jac, J receives the row of bin `role` (0 = the rotating side a, 1 = side b).
__device__ __forceinline__ double angle_row(double ax, double ay, double az, double bx, double by,
                                            double bz, double patx, double paty, double patz,
                                            double pbtx, double pbty, double pbtz, double sw,
                                            int role, bool jac, double J[6]) {
  const double na = sqrt(ax * ax + ay * ay + az * az);
  const double nb = sqrt(bx * bx + by * by + bz * bz);
  const bool ok = na > ANGLE_MIN_NORM && nb > ANGLE_MIN_NORM;
  const double na_s = ok ? na : 1.0;
  const double nb_s = ok ? nb : 1.0;
  const double ahx = ax / na_s, ahy = ay / na_s, ahz = az / na_s;
  const double bhx = bx / nb_s, bhy = by / nb_s, bhz = bz / nb_s;
  double cth = ahx * bhx + ahy * bhy + ahz * bhz;
  if (cth > 1.0) cth = 1.0;
  else if (cth < -1.0) cth = -1.0;
  const bool near_zero = (1.0 - cth) < ANGLE_COLLINEAR_EPS;
  const bool near_pi = (1.0 + cth) < ANGLE_COLLINEAR_EPS;
  const double val = (ok && !near_zero) ? acos(cth) : 0.0;
  const double wv = sw * val;
  if (!jac) return wv;
  const bool grad_ok = ok && !near_zero && !near_pi;
  const double inv_sin = grad_ok ? -1.0 / sqrt(fmax(1.0 - cth * cth, 1e-300)) : 0.0;
  const double gbx = inv_sin * (ahx - cth * bhx) / nb_s;
  const double gby = inv_sin * (ahy - cth * bhy) / nb_s;
  const double gbz = inv_sin * (ahz - cth * bhz) / nb_s;
  if (role == 0) {
    const double gax = inv_sin * (bhx - cth * ahx) / na_s;
    const double gay = inv_sin * (bhy - cth * ahy) / na_s;
    const double gaz = inv_sin * (bhz - cth * ahz) / na_s;
    J[0] = sw * ((ay * gaz - az * gay) - (paty * gbz - patz * gby));
    J[1] = sw * ((az * gax - ax * gaz) - (patz * gbx - patx * gbz));
    J[2] = sw * ((ax * gay - ay * gax) - (patx * gby - paty * gbx));
    J[3] = sw * (-gbx);
    J[4] = sw * (-gby);
    J[5] = sw * (-gbz);
  } else {
    J[0] = sw * (pbty * gbz - pbtz * gby);
    J[1] = sw * (pbtz * gbx - pbtx * gbz);
    J[2] = sw * (pbtx * gby - pbty * gbx);
    J[3] = sw * gbx;
    J[4] = sw * gby;
    J[5] = sw * gbz;
  }
  return wv;
}

// Unit-weight bending-angle row of one direction with BOTH bins' Jacobians
// (kernels.py:287-338 with sw = 1): Ja for the rotating side a, Jb for side b; returns
// the angle value. angle_row(...) with weight sw equals sw * (these rows, this value).
// 1/sqrt(x) for normal positive x: MUFU estimate + two Newton steps (~1 ulp), without the
// special-case branches of the full-precision rsqrt (solver-internal rows only)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx, y * y, 1.5);
  y = y * fma(-hx, y * y, 1.5);
  return y;
}

__device__ __forceinline__ double angle_unit(double ax, double ay, double az, double bx, double by,
                                             double bz, double patx, double paty, double patz,
                                             double pbtx, double pbty, double pbtz, double Ja[6],
                                             double Jb[6]) {
  // reciprocal norms instead of 12 divisions (ulp-level; the LM solver's parity is
  // tolerance-based; the operator-level arap_reduce keeps the reference's divisions)
  const double sa = ax * ax + ay * ay + az * az;
  const double sb = bx * bx + by * by + bz * bz;
  const bool ok = sa > ANGLE_MIN_NORM * ANGLE_MIN_NORM && sb > ANGLE_MIN_NORM * ANGLE_MIN_NORM;
  const double ia = ok ? rsqrt_nr(sa) : 1.0;
  const double ib = ok ? rsqrt_nr(sb) : 1.0;
  const double ahx = ax * ia, ahy = ay * ia, ahz = az * ia;
  const double bhx = bx * ib, bhy = by * ib, bhz = bz * ib;
  double cth = ahx * bhx + ahy * bhy + ahz * bhz;
  if (cth > 1.0) cth = 1.0;
  else if (cth < -1.0) cth = -1.0;
  const bool near_zero = (1.0 - cth) < ANGLE_COLLINEAR_EPS;
  const bool near_pi = (1.0 + cth) < ANGLE_COLLINEAR_EPS;
  const double val = (ok && !near_zero) ? acos(cth) : 0.0;
  const bool grad_ok = ok && !near_zero && !near_pi;
  const double inv_sin = grad_ok ? -rsqrt_nr(fmax(1.0 - cth * cth, 1e-300)) : 0.0;
  const double fa = inv_sin * ia, fb = inv_sin * ib;
  const double gax = fa * (bhx - cth * ahx);
  const double gay = fa * (bhy - cth * ahy);
  const double gaz = fa * (bhz - cth * ahz);
  const double gbx = fb * (ahx - cth * bhx);
  const double gby = fb * (ahy - cth * bhy);
  const double gbz = fb * (ahz - cth * bhz);
  Ja[0] = (ay * gaz - az * gay) - (paty * gbz - patz * gby);
  Ja[1] = (az * gax - ax * gaz) - (patz * gbx - patx * gbz);
  Ja[2] = (ax * gay - ay * gax) - (patx * gby - paty * gbx);
  Ja[3] = -gbx;
  Ja[4] = -gby;
  Ja[5] = -gbz;
  Jb[0] = pbty * gbz - pbtz * gby;
  Jb[1] = pbtz * gbx - pbtx * gbz;
  Jb[2] = pbtx * gby - pbty * gbx;
  Jb[3] = gbx;
  Jb[4] = gby;
  Jb[5] = gbz;
  return val;
}

// Four quaternion-component rotation rows sharing one bin, rotation columns only
// (kernels.py:470-480).
__device__ __forceinline__ void fold_quad(double* acc, const double J4[12], double d0, double d1,
                                          double d2, double d3, double sw) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = i; j < 3; ++j) {
      const double a = J4[0 * 3 + i] * J4[0 * 3 + j] + J4[1 * 3 + i] * J4[1 * 3 + j] +
                       J4[2 * 3 + i] * J4[2 * 3 + j] + J4[3 * 3 + i] * J4[3 * 3 + j];
      acc[triu_col(i, j)] += sw * sw * a;
    }
    acc[21 + i] += sw * sw * (J4[0 * 3 + i] * d0 + J4[1 * 3 + i] * d1 + J4[2 * 3 + i] * d2 +
                              J4[3 * 3 + i] * d3);
  }
}

// All rigidity rows of edge (i0, i1) that land in the bin of endpoint `side`.
// R0/t0/W0 belong to edges[e,0], R1/t1/W1 to edges[e,1]. Adds the bin's cost to
// *cost and, when jac, the rows' normal-equation contributions to acc[27].
__device__ __forceinline__ void arap_edge_bin(const double p0[3], const double p1[3],
                                              const double R0[9], const double t0[3],
                                              const double R1[9], const double t1[3],
                                              const double* W0, const double* W1, double ew,
                                              double wa0, double wa1, double angle_weight,
                                              double rotation_weight, int side, bool jac,
                                              double* acc, double* cost) {
  const double base = ew * 0.5 * (wa0 + wa1);
  double p0t[3], p1t[3];
  xform(R0, t0, p0[0], p0[1], p0[2], p0t);
  xform(R1, t1, p1[0], p1[1], p1[2], p1t);
  double J[6];

  // length preservation (kernels.py:366-398)
  const double rx = p1[0] - p0[0], ry = p1[1] - p0[1], rz = p1[2] - p0[2];
  const double rest = sqrt(rx * rx + ry * ry + rz * rz);
  const double bx = p1t[0] - p0t[0], by = p1t[1] - p0t[1], bz = p1t[2] - p0t[2];
  const double ln = sqrt(bx * bx + by * by + bz * bz);
  const double val = ln - rest;
  const double sw = sqrt(0.5 * base);
  const double wv = sw * val;
  *cost += wv * wv;
  if (jac) {
    double bhx, bhy, bhz;
    if (ln > 1e-9) {
      bhx = bx / ln; bhy = by / ln; bhz = bz / ln;
    } else {
      bhx = bhy = bhz = 0.0;
    }
    if (side == 0) {
      J[0] = sw * (p0t[1] * (-bhz) - p0t[2] * (-bhy));
      J[1] = sw * (p0t[2] * (-bhx) - p0t[0] * (-bhz));
      J[2] = sw * (p0t[0] * (-bhy) - p0t[1] * (-bhx));
      J[3] = sw * (-bhx);
      J[4] = sw * (-bhy);
      J[5] = sw * (-bhz);
    } else {
      J[0] = sw * (p1t[1] * bhz - p1t[2] * bhy);
      J[1] = sw * (p1t[2] * bhx - p1t[0] * bhz);
      J[2] = sw * (p1t[0] * bhy - p1t[1] * bhx);
      J[3] = sw * bhx;
      J[4] = sw * bhy;
      J[5] = sw * bhz;
    }
    fold_row(acc, J, wv);
  }

  // bending angle, both directions (kernels.py:400-417)
  const double sw_a = sqrt(0.5 * base * angle_weight);
  double c01[3], c10[3];
  xform(R0, t0, p1[0], p1[1], p1[2], c01);
  xform(R1, t1, p0[0], p0[1], p0[2], c10);
  // direction 0 -> 1: a-side bin is i0, b-side bin is i1
  const double wv01 = angle_row(c01[0] - p0t[0], c01[1] - p0t[1], c01[2] - p0t[2],
                                p1t[0] - p0t[0], p1t[1] - p0t[1], p1t[2] - p0t[2],
                                p0t[0], p0t[1], p0t[2], p1t[0], p1t[1], p1t[2], sw_a,
                                side == 0 ? 0 : 1, jac, J);
  *cost += wv01 * wv01;
  if (jac) fold_row(acc, J, wv01);
  // direction 1 -> 0: a-side bin is i1, b-side bin is i0
  const double wv10 = angle_row(c10[0] - p1t[0], c10[1] - p1t[1], c10[2] - p1t[2],
                                p0t[0] - p1t[0], p0t[1] - p1t[1], p0t[2] - p1t[2],
                                p1t[0], p1t[1], p1t[2], p0t[0], p0t[1], p0t[2], sw_a,
                                side == 0 ? 1 : 0, jac, J);
  *cost += wv10 * wv10;
  if (jac) fold_row(acc, J, wv10);

  // rotation consistency of the real parts (kernels.py:419-461)
  const double sw_r = sqrt(0.5 * base * rotation_weight);
  const double q0w = W0[0], q0x = W0[1], q0y = W0[2], q0z = W0[3];
  const double q1w = W1[0], q1x = W1[1], q1y = W1[2], q1z = W1[3];
  const double dq = q0w * q1w + q0x * q1x + q0y * q1y + q0z * q1z;
  const double sg = dq < 0.0 ? -1.0 : 1.0;
  const double d0 = q0w - sg * q1w;
  const double d1 = q0x - sg * q1x;
  const double d2 = q0y - sg * q1y;
  const double d3 = q0z - sg * q1z;
  *cost += sw_r * sw_r * (d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3);
  if (jac) {
    double J4[12];
    if (side == 0) {
      J4[0] = -0.5 * q0x; J4[1] = -0.5 * q0y; J4[2] = -0.5 * q0z;
      J4[3] = 0.5 * q0w;  J4[4] = 0.5 * q0z;  J4[5] = -0.5 * q0y;
      J4[6] = -0.5 * q0z; J4[7] = 0.5 * q0w;  J4[8] = 0.5 * q0x;
      J4[9] = 0.5 * q0y;  J4[10] = -0.5 * q0x; J4[11] = 0.5 * q0w;
    } else {
      const double h = -sg * 0.5;
      J4[0] = h * q1x * -1.0; J4[1] = h * q1y * -1.0; J4[2] = h * q1z * -1.0;
      J4[3] = h * q1w;        J4[4] = h * q1z;        J4[5] = h * -q1y;
      J4[6] = h * -q1z;       J4[7] = h * q1w;        J4[8] = h * q1x;
      J4[9] = h * q1y;        J4[10] = h * -q1x;      J4[11] = h * q1w;
    }
    fold_quad(acc, J4, d0, d1, d2, d3, sw_r);
  }
}

// ---------------------------------------------------------------------------------
// Damped 6x6 solve (solver._assemble + _solve_damped, solver.py:206-258).
// ---------------------------------------------------------------------------------

// From 27 reduced columns: M = A + lam diag(max(diag A, 1e-12)), Cholesky, then the
// reference's forward/backward substitution order. Returns false on a non-positive
// pivot (LAPACK potrf failure), with delta zeroed.
__device__ __forceinline__ bool damped_solve6(const double* part, double lam, double delta[6]) {
  double M[36];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i; j < 6; ++j) {
      const double v = part[triu_col(i, j)];
      M[i * 6 + j] = v;
      M[j * 6 + i] = v;
    }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double d = fmax(M[i * 6 + i], 1e-12);
    M[i * 6 + i] = M[i * 6 + i] + lam * d;
  }
  double L[36];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double s = M[j * 6 + j];
#pragma unroll
    for (int q = 0; q < j; ++q) s -= L[j * 6 + q] * L[j * 6 + q];
    if (!(s > 0.0)) ok = false;
    const double ljj = sqrt(s);
    L[j * 6 + j] = ljj;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double v = M[i * 6 + j];
#pragma unroll
      for (int q = 0; q < j; ++q) v -= L[i * 6 + q] * L[j * 6 + q];
      L[i * 6 + j] = v / ljj;
    }
  }
  if (!ok) {
#pragma unroll
    for (int i = 0; i < 6; ++i) delta[i] = 0.0;
    return false;
  }
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double acc = -part[21 + i];
#pragma unroll
    for (int j = 0; j < i; ++j) acc -= L[i * 6 + j] * y[j];
    y[i] = acc / L[i * 6 + i];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double acc = y[i];
#pragma unroll
    for (int j = i + 1; j < 6; ++j) acc -= L[j * 6 + i] * delta[j];
    delta[i] = acc / L[i * 6 + i];
  }
  return true;
}

// Hamilton product (geometry.quat_mul, geometry.py:29-43).
__device__ __forceinline__ void quat_mul(const double* a, const double* b, double* o) {
  o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  o[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  o[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

// Left-compose exp(delta) and renormalize (solver.apply_step solver.py:261-264 with
// geometry.dq_exp 300-304, quat_from_axis_angle 78-85 (np.sinc form), dq_mul 155-161,
// dq_normalize 164-178).
__device__ __forceinline__ void apply_step_one(const double* W, const double* delta, double* out) {
  const double o0 = delta[0], o1 = delta[1], o2 = delta[2];
  const double angle = sqrt(o0 * o0 + o1 * o1 + o2 * o2);
  // 0.5 * np.sinc(angle / (2 pi)); numpy 2.x: y = pi x, y := eps where y == 0, sin(y)/y
  const double xs = angle / (2.0 * M_PI);
  double y = M_PI * xs;
  if (y == 0.0) y = 2.220446049250313e-16;
  const double half_sinc = 0.5 * (sin(y) / y);
  const double er[4] = {cos(0.5 * angle), o0 * half_sinc, o1 * half_sinc, o2 * half_sinc};
  const double pv[4] = {0.0, delta[3], delta[4], delta[5]};
  double ed[4];
  quat_mul(pv, er, ed);
#pragma unroll
  for (int i = 0; i < 4; ++i) ed[i] = 0.5 * ed[i];
  double real[4], d1[4], d2[4];
  quat_mul(er, W, real);
  quat_mul(er, W + 4, d1);
  quat_mul(ed, W, d2);
  double dual[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) dual[i] = d1[i] + d2[i];
  const double norm = sqrt(real[0] * real[0] + real[1] * real[1] + real[2] * real[2] + real[3] * real[3]);
  double r[4], d[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r[i] = real[i] / norm;
    d[i] = dual[i] / norm;
  }
  const double dot = r[0] * d[0] + r[1] * d[1] + r[2] * d[2] + r[3] * d[3];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[i] = r[i];
    out[4 + i] = d[i] - dot * r[i];
  }
}

// apply_step_one with one sincos and one reciprocal (ulp-level; LM solver only)
__device__ __forceinline__ void apply_step_one_fast(const double* W, const double* delta, double* out) {
  const double o0 = delta[0], o1 = delta[1], o2 = delta[2];
  const double angle = sqrt(o0 * o0 + o1 * o1 + o2 * o2);
  // 0.5 * np.sinc(angle / (2 pi)); numpy 2.x: y = pi x, y := eps where y == 0, sin(y)/y
  const double xs = angle / (2.0 * M_PI);
  double y = M_PI * xs;
  if (y == 0.0) y = 2.220446049250313e-16;
  double sy, cy;
  sincos(y, &sy, &cy);  // y = angle / 2 up to an ulp
  const double half_sinc = 0.5 * (sy / y);
  const double er[4] = {cy, o0 * half_sinc, o1 * half_sinc, o2 * half_sinc};
  const double pv[4] = {0.0, delta[3], delta[4], delta[5]};
  double ed[4];
  quat_mul(pv, er, ed);
#pragma unroll
  for (int i = 0; i < 4; ++i) ed[i] = 0.5 * ed[i];
  double real[4], d1[4], d2[4];
  quat_mul(er, W, real);
  quat_mul(er, W + 4, d1);
  quat_mul(ed, W, d2);
  double dual[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) dual[i] = d1[i] + d2[i];
  const double inorm =
      rsqrt_nr(real[0] * real[0] + real[1] * real[1] + real[2] * real[2] + real[3] * real[3]);
  double r[4], d[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r[i] = real[i] * inorm;
    d[i] = dual[i] * inorm;
  }
  const double dot = r[0] * d[0] + r[1] * d[1] + r[2] * d[2] + r[3] * d[3];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[i] = r[i];
    out[4 + i] = d[i] - dot * r[i];
  }
}

}  // namespace dt
