// dt_solver.cu -- one frame of the deformation solve (solver.solve_frame,
// solver.py:267-378) as ONE kernel launch per frame: a thread-block cluster owns a
// sequence, keeps the control warps in shared memory and runs the whole
// Levenberg-Marquardt loop (relink -> linearize -> per-control 6x6 damped solves ->
// tentative value pass -> accept / reject -> damping ladder) on the device, with
// cluster barriers (barrier.cluster, ~0.2 us) between phases instead of kernel
// boundaries or host round trips.
//
// Work split inside a cluster of C CTAs x 256 threads:
//   per-point phases (warp + rasterize + linearize) stride over the template points,
//   per-control phases give each control to one warp, which gathers that control's
//   rows through static CSR lists (template binding, incident edges) and a per-frame
//   CSR (feature matches) and folds them in a fixed order, so every reduction is
//   deterministic and independent of C; totals over controls are summed in a fixed
//   order by every CTA redundantly, so all CTAs take identical control decisions.
// Several sequences (BASELINE config 5) run as several clusters of the same launch.

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "dt_common.cuh"
#include "dt_math.cuh"
#include "dt_ops.cuh"
#include "dt_solver.cuh"

namespace cg = cooperative_groups;

namespace dt {

constexpr int NWARPS = SOLVER_THREADS / 32;
constexpr int SCR_COLS = 30;  // 27 partial + support + icp cost + feature cost

size_t solver_smem_bytes(int m) {
  return sizeof(double) * ((size_t)8 * m + (size_t)NWARPS * 32 * SCR_COLS);
}

// L2-coherent loads for data produced by other CTAs of the cluster.
__device__ __forceinline__ double ld(const double* p) { return __ldcg(p); }
__device__ __forceinline__ uint8_t ldu8(const uint8_t* p) {
  return (uint8_t)__ldcg(reinterpret_cast<const unsigned char*>(p));
}
__device__ __forceinline__ int ldi(const int* p) { return __ldcg(p); }

struct Ctx {
  int C, r, tid, warp, lane, gw, GW, gt, GT;
};

__device__ __forceinline__ void load_warps(const SolverArgs& A, const double* src, double* s_w) {
  const int n = 8 * A.m;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_w[i] = ld(src + i);
}

// Blend of template point p at the warps in shared memory.
__device__ __forceinline__ void blend_point(const SolverArgs& A, const double* s_w, int64_t p,
                                            double B[8], double sgn[KMAX]) {
  int idx[KMAX];
  double w[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s)
    if (s < A.k) {
      idx[s] = A.bidx[p * A.k + s];
      w[s] = A.bw[p * A.k + s];
    }
  blend_at(s_w, idx, w, A.k, B, sgn);
}

__device__ __forceinline__ void blend_match(const SolverArgs& A, const double* s_w, int64_t j,
                                            double B[8], double sgn[KMAX]) {
  int idx[KMAX];
  double w[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s)
    if (s < A.k) {
      idx[s] = A.fbidx[j * A.k + s];
      w[s] = A.fbw[j * A.k + s];
    }
  blend_at(s_w, idx, w, A.k, B, sgn);
}

__device__ __forceinline__ unsigned sign_bits(const double sgn[KMAX], int k) {
  unsigned bits = 0;
#pragma unroll
  for (int s = 0; s < KMAX; ++s)
    if (s < k && sgn[s] < 0.0) bits |= 1u << s;
  return bits;
}

// Phase A, one template point: warp, project, gate (kernels.py:483-569), then the
// point-to-plane residual, its Tukey weight and (jac) its blend gradient
// (kernels.py:173-197). Returns whether the point has a valid correspondence.
__device__ __forceinline__ bool point_relink(const SolverArgs& A, const double* s_w, int64_t p, bool jac) {
  double B[8], sgn[KMAX];
  blend_point(A, s_w, p, B, sgn);
  const double px = A.tp[3 * p], py = A.tp[3 * p + 1], pz = A.tp[3 * p + 2];
  double x0, x1, x2, s2;
  apply_blend(B, px, py, pz, x0, x1, x2, s2);
  double r0, r1, r2;
  rotate_normal(B, A.tn[3 * p], A.tn[3 * p + 1], A.tn[3 * p + 2], r0, r1, r2);
  double o[3], g[3];
  int ui, vi;
  // projection and gates (identical to rasterize_one in dt_ops.cu)
  bool ok = false;
  if (x2 > 0.0) {
    const double uf = rint(A.fx * x0 / x2 + A.cx);
    const double vf = rint(A.fy * x1 / x2 + A.cy);
    if (uf >= 0.0 && uf < (double)A.width && vf >= 0.0 && vf < (double)A.height) {
      ui = (int)uf;
      vi = (int)vf;
      const int64_t pix = (int64_t)vi * A.width + ui;
      if (A.dvalid[pix]) {
        const double d = A.depth[pix];
        o[0] = ((double)ui - A.cx) / A.fx * d;
        o[1] = ((double)vi - A.cy) / A.fy * d;
        o[2] = d;
        g[0] = A.onrm[3 * pix];
        g[1] = A.onrm[3 * pix + 1];
        g[2] = A.onrm[3 * pix + 2];
        if (g[0] * g[0] + g[1] * g[1] + g[2] * g[2] > 0.25) {
          const double dx = o[0] - x0, dy = o[1] - x1, dz = d - x2;
          if (sqrt(dx * dx + dy * dy + dz * dz) < A.gate &&
              g[0] * r0 + g[1] * r1 + g[2] * r2 > A.cos_gate)
            ok = true;
        }
      }
    }
  }
  A.cvalid[p] = ok ? 1 : 0;
  if (!ok) return false;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    A.cobs[3 * p + i] = o[i];
    A.cnrm[3 * p + i] = g[i];
  }
  const double r = g[0] * (x0 - o[0]) + g[1] * (x1 - o[1]) + g[2] * (x2 - o[2]);
  A.pr_r[p] = r;
  A.pr_rs[p] = tukey_sqrt(r, A.tukey);
  A.pr_sgn[p] = (uint8_t)sign_bits(sgn, A.k);
  if (jac) {
    double G[24];
    blend_gradient(B, px, py, pz, x0, x1, x2, s2, G);
#pragma unroll
    for (int e = 0; e < 8; ++e) A.pr_gn[8 * p + e] = g[0] * G[e] + g[1] * G[8 + e] + g[2] * G[16 + e];
  }
  return true;
}

// Phase A, one active feature match (kernels.py:239-250).
__device__ __forceinline__ void match_lin(const SolverArgs& A, const double* s_w, int64_t j, bool jac) {
  double B[8], sgn[KMAX];
  blend_match(A, s_w, j, B, sgn);
  const double px = A.fp[3 * j], py = A.fp[3 * j + 1], pz = A.fp[3 * j + 2];
  double x0, x1, x2, s2;
  apply_blend(B, px, py, pz, x0, x1, x2, s2);
  A.fr_res[3 * j] = x0 - A.fo[3 * j];
  A.fr_res[3 * j + 1] = x1 - A.fo[3 * j + 1];
  A.fr_res[3 * j + 2] = x2 - A.fo[3 * j + 2];
  A.fr_sgn[j] = (uint8_t)sign_bits(sgn, A.k);
  if (jac) blend_gradient(B, px, py, pz, x0, x1, x2, s2, A.fr_G + 24 * j);
}

// Per-control gather of the data rows (icp + feature) in jac or value mode. In
// tentative mode (`tent`) the residuals are re-evaluated at the warps in shared memory
// with the frozen robust weights and the linearization's correspondences
// (solver.py:333-335); otherwise the stored per-point records are used.
__device__ __forceinline__ void control_data(const SolverArgs& A, const double* s_w, int c, int64_t n_act,
                             bool jac, bool tent, double* acc /*30*/) {
  const int lane = threadIdx.x & 31;
  Basis K;
  if (jac) make_basis(s_w + 8 * c, K);
  double* sup = &acc[27];
  double* cicp = &acc[28];
  double* cfeat = &acc[29];
  const int k = A.k;
  const int q1 = ldi(A.cptr + c + 1);
  for (int q = ldi(A.cptr + c) + lane; q < q1; q += 32) {
    const int e = ldi(A.cent + q);
    const int64_t p = e >> 3;
    const int s = e & 7;
    if (!ldu8(A.cvalid + p)) continue;
    const double a = A.bw[p * k + s];
    const double rs = ld(A.pr_rs + p);
    double r;
    unsigned sbits;
    if (tent) {
      double B[8], sgn[KMAX];
      blend_point(A, s_w, p, B, sgn);
      double x0, x1, x2, s2;
      apply_blend(B, A.tp[3 * p], A.tp[3 * p + 1], A.tp[3 * p + 2], x0, x1, x2, s2);
      r = ld(A.cnrm + 3 * p) * (x0 - ld(A.cobs + 3 * p)) +
          ld(A.cnrm + 3 * p + 1) * (x1 - ld(A.cobs + 3 * p + 1)) +
          ld(A.cnrm + 3 * p + 2) * (x2 - ld(A.cobs + 3 * p + 2));
      sbits = 0;
    } else {
      r = ld(A.pr_r + p);
      sbits = ldu8(A.pr_sgn + p);
    }
    *sup += rs * rs * a;
    const double sw = rs * sqrt(a);
    const double wv = sw * r;
    *cicp += wv * wv;
    if (jac) {
      double gn[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) gn[i] = ld(A.pr_gn + 8 * p + i);
      const double sg = ((sbits >> s) & 1u) ? -1.0 : 1.0;
      const double coef = sw * a * sg;
      double pr[6], J[6];
      basis_project(gn, K.Kr, K.Kd, pr);
#pragma unroll
      for (int d = 0; d < 6; ++d) J[d] = coef * pr[d];
      fold_row(acc, J, wv);
    }
  }
  if (A.mptr != nullptr && n_act > 0) {
    const int m1 = ldi(A.mptr + c + 1);
    for (int q = ldi(A.mptr + c) + lane; q < m1; q += 32) {
      const int e = ldi(A.ment + q);
      const int64_t j = e / k;
      const int s = e - (int)j * k;
      const double a = A.fbw[e];
      double res[3];
      unsigned sbits;
      if (tent) {
        double B[8], sgn[KMAX];
        blend_match(A, s_w, j, B, sgn);
        double x0, x1, x2, s2;
        apply_blend(B, A.fp[3 * j], A.fp[3 * j + 1], A.fp[3 * j + 2], x0, x1, x2, s2);
        res[0] = x0 - A.fo[3 * j];
        res[1] = x1 - A.fo[3 * j + 1];
        res[2] = x2 - A.fo[3 * j + 2];
        sbits = 0;
      } else {
        res[0] = ld(A.fr_res + 3 * j);
        res[1] = ld(A.fr_res + 3 * j + 1);
        res[2] = ld(A.fr_res + 3 * j + 2);
        sbits = ldu8(A.fr_sgn + j);
      }
      const double w_pair = A.fw * A.fwt[j] * a;
      *sup += w_pair;
      const double sw = sqrt(w_pair);
      const double wv0 = sw * res[0], wv1 = sw * res[1], wv2 = sw * res[2];
      *cfeat += wv0 * wv0 + wv1 * wv1 + wv2 * wv2;
      if (jac) {
        const double sg = ((sbits >> s) & 1u) ? -1.0 : 1.0;
        const double coef = sw * a * sg;
        double GK[18];
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) {
          double g[8], pr[6];
#pragma unroll
          for (int i = 0; i < 8; ++i) g[i] = ld(A.fr_G + 24 * j + 8 * comp + i);
          basis_project(g, K.Kr, K.Kd, pr);
#pragma unroll
          for (int d = 0; d < 6; ++d) GK[comp * 6 + d] = coef * pr[d];
        }
#pragma unroll
        for (int i = 0; i < 6; ++i) {
#pragma unroll
          for (int jj = i; jj < 6; ++jj)
            acc[triu_col(i, jj)] += GK[i] * GK[jj] + GK[6 + i] * GK[6 + jj] + GK[12 + i] * GK[12 + jj];
          acc[21 + i] += GK[i] * wv0 + GK[6 + i] * wv1 + GK[12 + i] * wv2;
        }
      }
    }
  }
}

// Per-control gather of the rigidity rows over the control's incident edges.
__device__ __forceinline__ void control_arap(const SolverArgs& A, const double* s_w, int c, const double* wa,
                             bool jac, double* acc /*27*/, double* cost) {
  const int lane = threadIdx.x & 31;
  const int q1 = ldi(A.iptr + c + 1);
  for (int q = ldi(A.iptr + c) + lane; q < q1; q += 32) {
    const int e2 = ldi(A.ient + q);
    const int e = e2 >> 1, side = e2 & 1;
    const int i0 = A.edges[2 * e], i1 = A.edges[2 * e + 1];
    double R0[9], t0[3], R1[9], t1[3];
    dq_to_transform(s_w + 8 * i0, R0, t0);
    dq_to_transform(s_w + 8 * i1, R1, t1);
    arap_edge_bin(A.cpts + 3 * i0, A.cpts + 3 * i1, R0, t0, R1, t1, s_w + 8 * i0, s_w + 8 * i1,
                  A.ew[e], ld(wa + i0), ld(wa + i1), A.angle_w, A.rot_w, side, jac, acc, cost);
  }
}

// Sum three per-control cost columns over all controls in a fixed order (warp 0,
// lane-strided then xor tree); every CTA evaluates it identically. Result broadcast
// through s_out[0..2]. Must be called by the whole CTA.
__device__ void total3(const double* c3, int m, double* s_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (warp == 0) {
    double a = 0.0, b = 0.0, d = 0.0;
    for (int i = lane; i < m; i += 32) {
      a += ld(c3 + 3 * i);
      b += ld(c3 + 3 * i + 1);
      d += ld(c3 + 3 * i + 2);
    }
    a = warp_sum(a);
    b = warp_sum(b);
    d = warp_sum(d);
    if (lane == 0) {
      s_out[0] = a;
      s_out[1] = b;
      s_out[2] = d;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(SOLVER_THREADS, 1) k_solve_frame(const SolverArgs* __restrict__ all) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  __shared__ SolverArgs A;
  __shared__ double s_tot[8];
  __shared__ double s_misc[8];
  __shared__ int s_cnt[NWARPS];
  extern __shared__ double smem[];
  if (threadIdx.x == 0) A = all[blockIdx.x / C];
  __syncthreads();
  double* s_w = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* s_scr = smem + 8 * A.m + warp * 32 * SCR_COLS;
  const int gw = rank * NWARPS + warp, GW = C * NWARPS;
  const int64_t gt = (int64_t)rank * blockDim.x + threadIdx.x, GT = (int64_t)C * blockDim.x;
  const int m = A.m;
  const int64_t n = A.n;
  const int64_t n_act = A.n_active ? *A.n_active : 0;

  for (int c = gw; c < m; c += GW)
    if (lane == 0) A.lam[c] = A.lam_init;

  double* cur = A.warp_a;
  double* tent = A.warp_b;
  int accepted_steps = 0, rejected_steps = 0, n_hist = 0;
  bool converged = false, stalled = false;
  double final_step_norm = 0.0;
  int outer_done = 0;
  int lam_pending = -1;
  int parity = 0;

  for (int outer = 0; outer < A.max_outer; ++outer) {
    outer_done = outer + 1;
    // ---- Phase A: relink + linearize every point and match at `cur` ----
    load_warps(A, cur, s_w);
    __syncthreads();
    for (int64_t p = gt; p < n; p += GT) point_relink(A, s_w, p, true);
    for (int64_t j = gt; j < n_act; j += GT) match_lin(A, s_w, j, true);
    cluster.sync();
    if (lam_pending >= 0 && rank == 0) {
      // lambda_history of the previous outer iteration (solver.py:345); lam is not
      // touched again before the next cluster barrier
      if (warp == 0) {
        double lo = INFINITY, hi = -INFINITY;
        for (int i = lane; i < m; i += 32) {
          const double v = ld(A.lam + i);
          lo = fmin(lo, v);
          hi = fmax(hi, v);
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        if (lane == 0) {
          A.lam_hist[2 * lam_pending] = lo;
          A.lam_hist[2 * lam_pending + 1] = hi;
        }
      }
      lam_pending = -1;
    }
    lam_pending = -1;
    // ---- Phase B: per-control data rows -> partial, support, wa ----
    for (int c = gw; c < m; c += GW) {
      double acc[SCR_COLS];
#pragma unroll
      for (int i = 0; i < SCR_COLS; ++i) acc[i] = 0.0;
      control_data(A, s_w, c, n_act, true, false, acc);
      double out[SCR_COLS];
      warp_column_sum<SCR_COLS>(acc, s_scr, out);
      if (lane < 27) A.partial[27 * c + lane] = out[lane];
      if (lane == 27) A.wa[c] = A.arap_w * fmax(out[27], A.data_floor);
      if (lane == 28) A.cost3[3 * c] = out[28];
      if (lane == 29) A.cost3[3 * c + 1] = out[29];
    }
    cluster.sync();
    // ---- Phase C: per-control rigidity rows, then the first damped solve ----
    for (int c = gw; c < m; c += GW) {
      double acc[28];
#pragma unroll
      for (int i = 0; i < 28; ++i) acc[i] = 0.0;
      control_arap(A, s_w, c, A.wa, true, acc, &acc[27]);
      double out[28];
      warp_column_sum<28>(acc, s_scr, out);
      if (lane < 27) A.partial[27 * c + lane] = A.partial[27 * c + lane] + out[lane];
      if (lane == 27) A.cost3[3 * c + 2] = out[27];
    }
    bool accepted = false;
    double cost_before = 0.0, cost_after = 0.0;
    bool have_before = false;
    for (int attempt = 0; attempt <= A.max_retries; ++attempt) {
      // damped solve per owned control (solver.py:217-258)
      double* okn = A.oknorm + (size_t)parity * 2 * m;
      for (int c = gw; c < m; c += GW) {
        __syncwarp();
        if (lane == 0) {
          double part[27], d[6];
          for (int i = 0; i < 27; ++i) part[i] = ld(A.partial + 27 * c + i);
          const bool good = damped_solve6(part, ld(A.lam + c), d);
          double nn = 0.0;
          for (int i = 0; i < 6; ++i) {
            A.delta[6 * c + i] = d[i];
            nn += d[i] * d[i];
          }
          okn[2 * c] = good ? 1.0 : 0.0;
          okn[2 * c + 1] = sqrt(nn);
        }
      }
      cluster.sync();
      if (!have_before) {
        total3(A.cost3, m, s_tot);
        cost_before = s_tot[0] + s_tot[1] + s_tot[2];
        have_before = true;
      }
      // all ok? max step norm (identical in every CTA)
      __syncthreads();
      if (warp == 0) {
        double allok = 1.0, mx = 0.0;
        for (int i = lane; i < m; i += 32) {
          allok = fmin(allok, ld(okn + 2 * i));
          mx = fmax(mx, ld(okn + 2 * i + 1));
        }
        allok = warp_min(allok);
        mx = warp_max(mx);
        if (lane == 0) {
          s_misc[0] = allok;
          s_misc[1] = mx;
        }
      }
      __syncthreads();
      const bool all_ok = s_misc[0] > 0.5;
      const double step_norm = s_misc[1];
      parity ^= 1;
      if (!all_ok) {
        // raise the damping of the failed controls only, retry (solver.py:321-326)
        for (int c = gw; c < m; c += GW)
          if (lane == 0 && ld(okn + 2 * c) < 0.5) A.lam[c] = fmin(A.lam[c] * A.lam_inc, A.lam_max);
        ++rejected_steps;
        continue;
      }
      final_step_norm = step_norm;
      if (step_norm < A.step_tol) {
        converged = true;
        break;
      }
      // tentative warps (solver.py:332)
      for (int c = gw; c < m; c += GW)
        if (lane < 8) {
          double out8[8];
          apply_step_one(cur + 8 * c, A.delta + 6 * c, out8);
          // every lane evaluates the same step; lane l stores component l
          tent[8 * c + lane] = out8[lane];
        }
      cluster.sync();
      // value pass at the tentative warps with frozen robust and rigidity weights
      load_warps(A, tent, s_w);
      __syncthreads();
      for (int c = gw; c < m; c += GW) {
        double acc[SCR_COLS];
#pragma unroll
        for (int i = 0; i < SCR_COLS; ++i) acc[i] = 0.0;
        control_data(A, s_w, c, n_act, false, true, acc);
        double ca = 0.0;
        control_arap(A, s_w, c, A.wa, false, acc, &ca);
        acc[27] = ca;  // reuse the support slot for the rigidity cost
        double out[SCR_COLS];
        warp_column_sum<SCR_COLS>(acc, s_scr, out);
        if (lane == 28) A.cost3_t[3 * c] = out[28];
        if (lane == 29) A.cost3_t[3 * c + 1] = out[29];
        if (lane == 27) A.cost3_t[3 * c + 2] = out[27];
      }
      cluster.sync();
      total3(A.cost3_t, m, s_tot);
      cost_after = s_tot[0] + s_tot[1] + s_tot[2];
      if (cost_after < cost_before) {
        double* tmp = cur;
        cur = tent;
        tent = tmp;
        for (int c = gw; c < m; c += GW)
          if (lane == 0) A.lam[c] = fmax(A.lam[c] * A.lam_dec, A.lam_min);
        ++accepted_steps;
        if (rank == 0 && threadIdx.x == 0) {
          A.cost_hist[2 * n_hist] = cost_before;
          A.cost_hist[2 * n_hist + 1] = cost_after;
        }
        ++n_hist;
        accepted = true;
        break;
      }
      for (int c = gw; c < m; c += GW)
        if (lane == 0) A.lam[c] = fmin(A.lam[c] * A.lam_inc, A.lam_max);
      ++rejected_steps;
    }
    lam_pending = outer;
    if (converged) break;
    if (!accepted) {
      stalled = true;
      if (rank == 0 && threadIdx.x == 0) A.stalled_hist[outer] = 1;
      continue;
    }
    if (cost_before - cost_after <= A.cost_tol * fmax(cost_before, 1e-30)) {
      converged = true;
      break;
    }
  }

  // ---- final report: relink at the solution, recompute robust and rigidity weights
  // (solver.py:360-376) ----
  load_warps(A, cur, s_w);
  __syncthreads();
  int my_valid = 0;
  for (int64_t p = gt; p < n; p += GT) my_valid += point_relink(A, s_w, p, false) ? 1 : 0;
  for (int64_t j = gt; j < n_act; j += GT) match_lin(A, s_w, j, false);
  // per-CTA count of correspondences
  for (int o = 16; o > 0; o >>= 1) my_valid += __shfl_xor_sync(0xffffffffu, my_valid, o);
  if (lane == 0) s_cnt[warp] = my_valid;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < NWARPS; ++w) t += s_cnt[w];
    A.cta_counts[rank] = t;
  }
  // final warps out
  for (int c = gw; c < m; c += GW)
    if (lane < 8) A.warps_out[8 * c + lane] = ld(cur + 8 * c + lane);
  cluster.sync();
  if (lam_pending >= 0 && rank == 0 && warp == 0) {
    double lo = INFINITY, hi = -INFINITY;
    for (int i = lane; i < m; i += 32) {
      const double v = ld(A.lam + i);
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (lane == 0) {
      A.lam_hist[2 * lam_pending] = lo;
      A.lam_hist[2 * lam_pending + 1] = hi;
    }
  }
  for (int c = gw; c < m; c += GW) {
    double acc[SCR_COLS];
#pragma unroll
    for (int i = 0; i < SCR_COLS; ++i) acc[i] = 0.0;
    control_data(A, s_w, c, n_act, false, false, acc);
    double out[SCR_COLS];
    warp_column_sum<SCR_COLS>(acc, s_scr, out);
    if (lane == 27) {
      const double wv = A.arap_w * fmax(out[27], A.data_floor);
      A.wa[c] = wv;
      A.wa_out[c] = wv;
    }
    if (lane == 28) A.cost3[3 * c] = out[28];
    if (lane == 29) A.cost3[3 * c + 1] = out[29];
  }
  cluster.sync();
  for (int c = gw; c < m; c += GW) {
    double acc[28];
#pragma unroll
    for (int i = 0; i < 28; ++i) acc[i] = 0.0;
    control_arap(A, s_w, c, A.wa, false, acc, &acc[27]);
    double out[28];
    warp_column_sum<28>(acc, s_scr, out);
    if (lane == 27) A.cost3[3 * c + 2] = out[27];
  }
  cluster.sync();
  total3(A.cost3, m, s_tot);
  if (rank == 0 && threadIdx.x == 0) {
    dt_report* R = A.report;
    R->icp_cost = s_tot[0];
    R->feature_cost = s_tot[1];
    R->arap_cost = s_tot[2];
    R->total_cost = s_tot[0] + s_tot[1] + s_tot[2];
    int nc = 0;
    for (int i = 0; i < C; ++i) nc += __ldcg(A.cta_counts + i);
    R->n_correspondences = nc;
    R->outer_iterations = outer_done;
    R->accepted_steps = accepted_steps;
    R->rejected_steps = rejected_steps;
    R->stalled = stalled ? 1 : 0;
    R->converged = converged ? 1 : 0;
    R->final_step_norm = final_step_norm;
    R->n_cost_history = n_hist;
  }
}

static int g_max_cluster[16] = {0};

int solver_max_cluster(int device) {
  if (device < 0 || device >= 16) return 8;
  if (g_max_cluster[device] > 0) return g_max_cluster[device];
  int best = 1;
  cudaFuncSetAttribute(k_solve_frame, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const size_t smem = solver_smem_bytes(1024);
  cudaFuncSetAttribute(k_solve_frame, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int c = 16; c >= 1; c >>= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c, 1, 1);
    cfg.blockDim = dim3(SOLVER_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k_solve_frame, &cfg) == cudaSuccess && nclusters > 0) {
      best = c;
      break;
    }
    cudaGetLastError();
  }
  g_max_cluster[device] = best;
  return best;
}

int solver_pick_cluster(int device, int requested, int m_max) {
  (void)m_max;
  const int mx = solver_max_cluster(device);
  if (requested <= 0) return mx;
  int c = 1;
  while (c * 2 <= requested && c * 2 <= mx) c *= 2;
  return c;
}

int solver_launch(const SolverArgs* d_args, int n_seq, int cluster, int m_max, cudaStream_t s) {
  const size_t smem = solver_smem_bytes(m_max);
  DT_REQUIRE(smem <= 227 * 1024, DT_ERR_UNSUPPORTED,
             "control graph too large for the shared-memory warp table (m=%d)", m_max);
  DT_CHECK_CUDA(cudaFuncSetAttribute(k_solve_frame, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DT_CHECK_CUDA(cudaFuncSetAttribute(k_solve_frame, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_seq * cluster), 1, 1);
  cfg.blockDim = dim3(SOLVER_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DT_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_solve_frame, d_args));
  return DT_OK;
}

}  // namespace dt
