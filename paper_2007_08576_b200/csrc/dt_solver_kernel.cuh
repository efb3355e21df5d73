// dt_solver_kernel.cuh -- body of the persistent LM kernel (included by dt_solver.cu).
//
// Work units inside the sync domain (C CTAs x 16 warps):
//   * points / matches / edges: one item per lane, fixed 32-item chunks whose partial
//     sums land in csum (deterministic, independent of C);
//   * controls: a team of TEAM warps of one CTA per control; each warp folds every
//     TEAM-th block of 32 rows into its own FP64 tensor-core Gram, the team combines the
//     Grams in warp order (deterministic, independent of C).
// Barriers per outer iteration: P1 | P2 | P3 (+ first solve) | value pass -- the
// tentative step is applied redundantly by every CTA into its own shared memory, so it
// costs no barrier.

constexpr int TEAM = 4;
constexpr int TEAMS_PER_CTA = NWARPS / TEAM;

// Sum of the three chunk-sum segments in a fixed order (thread-strided, warp xor tree,
// warps in order), identical in every CTA. Must be called by the whole CTA.
__device__ __forceinline__ void block_totals(const double* cs_p, int np, const double* cs_m, int nm,
                                             const double* cs_e, int ne, double* s_part,
                                             double out[3]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a = 0.0, b = 0.0, e = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) a += ld(cs_p + i);
  for (int i = threadIdx.x; i < nm; i += blockDim.x) b += ld(cs_m + i);
  for (int i = threadIdx.x; i < ne; i += blockDim.x) e += ld(cs_e + i);
  a = warp_sum(a);
  b = warp_sum(b);
  e = warp_sum(e);
  __syncthreads();
  if (lane == 0) {
    s_part[3 * warp] = a;
    s_part[3 * warp + 1] = b;
    s_part[3 * warp + 2] = e;
  }
  __syncthreads();
  double ta = 0.0, tb = 0.0, te = 0.0;
  for (int w = 0; w < NWARPS; ++w) {
    ta += s_part[3 * w];
    tb += s_part[3 * w + 1];
    te += s_part[3 * w + 2];
  }
  out[0] = ta;
  out[1] = tb;
  out[2] = te;
}

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

template <bool GRID>
__global__ void __launch_bounds__(SOLVER_THREADS, 1) k_solve_frame(const SolverArgs* __restrict__ all) {
  Dom<GRID> dom;
  const int C = dom.size();
  const int rank = dom.rank();
  __shared__ SolverArgs A;
  __shared__ double s_part[3 * NWARPS];
  __shared__ double s_sup[NWARPS];
  __shared__ double s_col[TEAMS_PER_CTA][32];
  __shared__ int s_cnt[NWARPS];
  extern __shared__ double smem[];
  if (threadIdx.x == 0) A = all[dom.seq()];
  __syncthreads();
  const int m = A.m;
  const int64_t n = A.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / TEAM, tw = warp % TEAM;
  double* s_w = smem;
  double* s_T = smem + 8 * m;
  double* stage = smem + 20 * m + warp * (STAGE + GOUT);
  double* gout = stage + STAGE;
  // work items are dealt round-robin over the CTAs first (item i -> CTA i % C), so
  // every SM of the domain gets a share of each phase
  const int gw = warp * C + rank, GW = C * NWARPS;
  const int gw_rev = (NWARPS - 1 - warp) * C + rank;
  const int gt = rank * (int)blockDim.x + (int)threadIdx.x, GT = C * (int)blockDim.x;
  const int gteam = team * C + rank, GTEAM = C * TEAMS_PER_CTA;
  const int team_rounds = (m + GTEAM - 1) / GTEAM;
  const int64_t n_act = A.n_active ? *A.n_active : 0;
  const int nch_p = (int)((n + CHUNK - 1) / CHUNK);
  const int nch_m = (int)((n_act + CHUNK - 1) / CHUNK);
  const int nch_e = (A.n_edges + CHUNK - 1) / CHUNK;
  double* cs_p = A.csum;
  double* cs_m = A.csum + A.nch_p;
  double* cs_e = cs_m + A.nch_m;
  unsigned long long* lam_hist = reinterpret_cast<unsigned long long*>(A.lam_hist);
  long long* tr = A.trace;
  int tn = 0;
  TRACE(0);

  for (int c = gt; c < m; c += GT) A.lam[c] = A.lam_init;
  for (int i = gt; i < A.max_outer; i += GT) {
    lam_hist[2 * i] = dbits(INFINITY);  // min over positive doubles = min of their bits
    lam_hist[2 * i + 1] = 0ull;
  }

  double* cur = A.warp_a;
  double* tent = A.warp_b;
  int accepted_steps = 0, rejected_steps = 0, n_hist = 0, outer_done = 0;
  bool converged = false, stalled = false;
  double final_step_norm = 0.0;
  int parity = 0;

  for (int outer = 0; outer < A.max_outer; ++outer) {
    outer_done = outer + 1;
    // ---- P1: relink + linearize at `cur`; icp / feature cost of the iterate ----
    load_state(A, cur, s_w, s_T);
    TRACE(12);
    for (int ch = gw; ch < nch_p + nch_m; ch += GW) {
      double acc = 0.0;
      if (ch < nch_p) {
        const int64_t p = (int64_t)ch * CHUNK + lane;
        int vdummy;
        if (p < n) acc = point_relink(A, s_w, p, true, &vdummy);
        acc = warp_sum(acc);
        if (lane == 0) cs_p[ch] = acc;
      } else {
        const int64_t j = (int64_t)(ch - nch_p) * CHUNK + lane;
        if (j < n_act) acc = match_eval(A, s_w, j, true, true);
        acc = warp_sum(acc);
        if (lane == 0) cs_m[ch - nch_p] = acc;
      }
    }
    DSYNC(1);

    // ---- P2: unit rigidity rows of every connection (no wa needed), on the warps at
    // the end of the domain; data rows -> normal equations (Gram on the FP64 tensor
    // cores) on the teams ----
    for (int ch = gw_rev; ch < nch_e; ch += GW) {
      const int e = ch * CHUNK + lane;
      if (e < A.n_edges) edge_unit_rows(A, s_T, e, A.erows + (size_t)ER * e);
    }
    TRACE(22);
    for (int r = 0; r < team_rounds; ++r) {
      const int c = r * GTEAM + gteam;
      Gram G;
      double sup = 0.0;
      if (c < m) {
        Basis K;
        make_basis(s_w + 8 * c, K);
        const int q0 = ldi(A.cptr + c), q1 = ldi(A.cptr + c + 1);
        for (int base = q0 + 32 * tw; base < q1; base += 32 * TEAM) {
          const int q = base + lane;
          double row[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (q < q1) {
            const int e = ldi(A.cent + q);
            const int64_t p = e >> 3;
            const int s = e & 7;
            if (ldu8(A.cvalid + p)) {
              const double a = A.bw[p * A.k + s];
              const double rs = ld(A.pr_rs + p);
              sup += rs * rs * a;
              const double sw = rs * sqrt(a);
              const double sg = ((ldu8(A.pr_sgn + p) >> s) & 1u) ? -1.0 : 1.0;
              const double coef = sw * a * sg;
              double gn[8], pr[6];
#pragma unroll
              for (int i = 0; i < 8; ++i) gn[i] = ld(A.pr_gn + 8 * p + i);
              basis_project(gn, K.Kr, K.Kd, pr);
#pragma unroll
              for (int d = 0; d < 6; ++d) row[d] = coef * pr[d];
              row[6] = sw * ld(A.pr_r + p);
            }
          }
          gram_push(G, stage, row);
        }
        if (n_act > 0) {
          const int m0 = ldi(A.mptr + c), m1 = ldi(A.mptr + c + 1);
          for (int base = m0 + 32 * tw; base < m1; base += 32 * TEAM) {
            const int q = base + lane;
            const bool live = q < m1;
            int64_t j = 0;
            double coef = 0.0, sw = 0.0;
            if (live) {
              const int e = ldi(A.ment + q);
              j = e / A.k;
              const int s = e - (int)j * A.k;
              const double a = A.fbw[e];
              const double w_pair = A.fw * A.fwt[j] * a;
              sup += w_pair;
              sw = sqrt(w_pair);
              const double sg = ((ldu8(A.fr_sgn + j) >> s) & 1u) ? -1.0 : 1.0;
              coef = sw * a * sg;
            }
#pragma unroll 1
            for (int comp = 0; comp < 3; ++comp) {
              double row[8] = {0, 0, 0, 0, 0, 0, 0, 0};
              if (live) {
                double g[8], pr[6];
#pragma unroll
                for (int i = 0; i < 8; ++i) g[i] = ld(A.fr_G + 24 * j + 8 * comp + i);
                basis_project(g, K.Kr, K.Kd, pr);
#pragma unroll
                for (int d = 0; d < 6; ++d) row[d] = coef * pr[d];
                row[6] = sw * ld(A.fr_res + 3 * j + comp);
              }
              gram_push(G, stage, row);
            }
          }
        }
      }
      gram_store(G, gout);
      sup = warp_sum(sup);
      if (lane == 0) s_sup[warp] = sup;
      __syncthreads();
      if (tw == 0 && c < m) {
        // combine the team's Grams in warp order
        if (lane < 27) {
          double v = 0.0;
          for (int w = 0; w < TEAM; ++w) v += gram_col(gout + w * (STAGE + GOUT), lane);
          A.partial[27 * c + lane] = v;
        }
        if (lane == 27) {
          double su = 0.0;
          for (int w = 0; w < TEAM; ++w) su += s_sup[warp + w];
          A.wa[c] = A.arap_w * fmax(su, A.data_floor);
        }
      }
      __syncthreads();
    }
    DSYNC(2);

    // ---- P3: rigidity rows -> normal equations + first damped solve; rigidity cost ----
    double* okn = A.oknorm + (size_t)parity * 2 * m;
    for (int r = 0; r < team_rounds; ++r) {
      const int c = r * GTEAM + gteam;
      Gram G;
      if (c < m) {
        const int q0 = ldi(A.iptr + c), q1 = ldi(A.iptr + c + 1);
        for (int base = q0 + 32 * tw; base < q1; base += 32 * TEAM) {
          const int q = base + lane;
          const bool live = q < q1;
          int i0 = 0, i1 = 0, side = 0;
          double sw = 0.0, swa = 0.0, swr = 0.0;
          const double* er = A.erows;
          if (live) {
            const int e2 = ldi(A.ient + q);
            const int e = e2 >> 1;
            side = e2 & 1;
            i0 = A.edges[2 * e];
            i1 = A.edges[2 * e + 1];
            const double base_w = A.ew[e] * 0.5 * (ld(A.wa + i0) + ld(A.wa + i1));
            sw = sqrt(0.5 * base_w);
            swa = sqrt(0.5 * base_w * A.angle_w);
            swr = sqrt(0.5 * base_w * A.rot_w);
            er = A.erows + (size_t)ER * e;
          }
          double row[8];
          // length row of this bin
#pragma unroll
          for (int i = 0; i < 6; ++i) row[i] = live ? sw * ld(er + 6 * side + i) : 0.0;
          row[6] = live ? sw * ld(er + 12) : 0.0;
          row[7] = 0.0;
          gram_push(G, stage, row);
          // angle 0->1: bin 0 is side a ([13,19)), bin 1 side b ([19,25))
#pragma unroll
          for (int i = 0; i < 6; ++i) row[i] = live ? swa * ld(er + 13 + 6 * side + i) : 0.0;
          row[6] = live ? swa * ld(er + 25) : 0.0;
          gram_push(G, stage, row);
          // angle 1->0: bin 1 is side a ([26,32)), bin 0 side b ([32,38))
#pragma unroll
          for (int i = 0; i < 6; ++i) row[i] = live ? swa * ld(er + 32 - 6 * side + i) : 0.0;
          row[6] = live ? swa * ld(er + 38) : 0.0;
          gram_push(G, stage, row);
#pragma unroll 1
          for (int rr = 0; rr < 4; ++rr) {
            if (live) {
              rotation_row(s_w, i0, i1, side, swr, rr, row);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) row[i] = 0.0;
            }
            gram_push(G, stage, row);
          }
        }
      }
      gram_store(G, gout);
      TRACE(32);
      __syncthreads();
      if (tw == 0 && c < m) {
        if (lane < 27) {
          double v = 0.0;
          for (int w = 0; w < TEAM; ++w) v += gram_col(gout + w * (STAGE + GOUT), lane);
          v = ld(A.partial + 27 * c + lane) + v;
          A.partial[27 * c + lane] = v;
          s_col[team][lane] = v;
        }
        __syncwarp();
        if (lane == 0) {
          double d[6];
          const bool good = solve6(s_col[team], ld(A.lam + c), d);
          double nn = 0.0;
          for (int i = 0; i < 6; ++i) {
            A.delta[6 * c + i] = d[i];
            nn += d[i] * d[i];
          }
          okn[2 * c] = good ? 1.0 : 0.0;
          okn[2 * c + 1] = sqrt(nn);
        }
      }
      __syncthreads();
      TRACE(34);
    }
    for (int ch = gw_rev; ch < nch_e; ch += GW) {
      double acc = 0.0;
      const int e = ch * CHUNK + lane;
      if (e < A.n_edges) acc = edge_cost_rows(A, s_w, A.wa, A.erows + (size_t)ER * e, e);
      acc = warp_sum(acc);
      if (lane == 0) cs_e[ch] = acc;
    }
    bool accepted = false;
    double cost_before = 0.0, cost_after = 0.0;
    for (int attempt = 0; attempt <= A.max_retries; ++attempt) {
      if (attempt > 0) {
        okn = A.oknorm + (size_t)parity * 2 * m;
        for (int c = gt; c < m; c += GT) {
          double part[27], d[6];
          for (int i = 0; i < 27; ++i) part[i] = ld(A.partial + 27 * c + i);
          const bool good = solve6(part, A.lam[c], d);
          double nn = 0.0;
          for (int i = 0; i < 6; ++i) {
            A.delta[6 * c + i] = d[i];
            nn += d[i] * d[i];
          }
          okn[2 * c] = good ? 1.0 : 0.0;
          okn[2 * c + 1] = sqrt(nn);
        }
      }
      DSYNC(attempt == 0 ? 3 : 4);
      // prefetch this thread's step inputs (one control per thread when m <= 512)
      double pW[8], pD[6];
      const int pc = threadIdx.x;
      if (pc < m) {
#pragma unroll
        for (int i = 0; i < 8; ++i) pW[i] = ld(cur + 8 * pc + i);
#pragma unroll
        for (int i = 0; i < 6; ++i) pD[i] = ld(A.delta + 6 * pc + i);
      }
      if (attempt == 0) {
        double t3[3];
        block_totals(cs_p, nch_p, cs_m, nch_m, cs_e, nch_e, s_part, t3);
        cost_before = t3[0] + t3[1] + t3[2];
      }
      TRACE(53);
      // all solves ok? largest step norm (identical in every CTA)
      {
        double allok = 1.0, mx = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
          allok = fmin(allok, ld(okn + 2 * i));
          mx = fmax(mx, ld(okn + 2 * i + 1));
        }
        allok = warp_min(allok);
        mx = warp_max(mx);
        __syncthreads();
        if (lane == 0) {
          s_part[2 * warp] = allok;
          s_part[2 * warp + 1] = mx;
        }
        __syncthreads();
        allok = 1.0;
        mx = 0.0;
        for (int w = 0; w < NWARPS; ++w) {
          allok = fmin(allok, s_part[2 * w]);
          mx = fmax(mx, s_part[2 * w + 1]);
        }
        __syncthreads();
        parity ^= 1;
        if (!(allok > 0.5)) {
          // raise the damping of the failed controls only, retry (solver.py:321-326)
          for (int c = gt; c < m; c += GT)
            if (ld(okn + 2 * c) < 0.5) A.lam[c] = fmin(A.lam[c] * A.lam_inc, A.lam_max);
          ++rejected_steps;
          continue;
        }
        final_step_norm = mx;
        if (mx < A.step_tol) {  // checked before the step (solver.py:327-331)
          converged = true;
          break;
        }
      }
      TRACE(54);
      // ---- tentative warps, applied redundantly by every CTA (no barrier) ----
      __syncthreads();
      if (pc < m) apply_step_one(pW, pD, s_w + 8 * pc);
      for (int c = threadIdx.x + blockDim.x; c < m; c += blockDim.x) {
        double W[8], d[6];
        for (int i = 0; i < 8; ++i) W[i] = ld(cur + 8 * c + i);
        for (int i = 0; i < 6; ++i) d[i] = ld(A.delta + 6 * c + i);
        apply_step_one(W, d, s_w + 8 * c);
      }
      __syncthreads();
      TRACE(55);
      for (int c = threadIdx.x; c < m; c += blockDim.x)
        dq_to_transform(s_w + 8 * c, s_T + 12 * c, s_T + 12 * c + 9);
      for (int c = gt; c < m; c += GT)
        for (int i = 0; i < 8; ++i) tent[8 * c + i] = s_w[8 * c + i];
      __syncthreads();
      TRACE(52);
      // ---- P6: cost at the tentative warps, frozen weights and correspondences ----
      for (int ch = gw; ch < nch_p + nch_m + nch_e; ch += GW) {
        double acc = 0.0;
        if (ch < nch_p) {
          const int64_t p = (int64_t)ch * CHUNK + lane;
          if (p < n) acc = point_value(A, s_w, p);
          acc = warp_sum(acc);
          if (lane == 0) cs_p[ch] = acc;
        } else if (ch < nch_p + nch_m) {
          const int64_t j = (int64_t)(ch - nch_p) * CHUNK + lane;
          if (j < n_act) acc = match_eval(A, s_w, j, false, false);
          acc = warp_sum(acc);
          if (lane == 0) cs_m[ch - nch_p] = acc;
        } else {
          const int e = (ch - nch_p - nch_m) * CHUNK + lane;
          if (e < A.n_edges) acc = edge_value(A, s_w, s_T, A.wa, e);
          acc = warp_sum(acc);
          if (lane == 0) cs_e[ch - nch_p - nch_m] = acc;
        }
      }
      DSYNC(6);
      {
        double t3[3];
        block_totals(cs_p, nch_p, cs_m, nch_m, cs_e, nch_e, s_part, t3);
        cost_after = t3[0] + t3[1] + t3[2];
      }
      if (cost_after < cost_before) {
        double* tmp = cur;
        cur = tent;
        tent = tmp;
        for (int c = gt; c < m; c += GT) A.lam[c] = fmax(A.lam[c] * A.lam_dec, A.lam_min);
        ++accepted_steps;
        if (rank == 0 && threadIdx.x == 0) {
          A.cost_hist[2 * n_hist] = cost_before;
          A.cost_hist[2 * n_hist + 1] = cost_after;
        }
        ++n_hist;
        accepted = true;
        break;
      }
      for (int c = gt; c < m; c += GT) A.lam[c] = fmin(A.lam[c] * A.lam_inc, A.lam_max);
      ++rejected_steps;
    }
    // lambda_history (solver.py:345): min / max of the final per-control damping of this
    // outer iteration, folded by the owners with order-independent integer atomics
    for (int c0 = gt - lane; c0 < m; c0 += GT) {
      const int c = c0 + lane;
      unsigned long long lo = ~0ull, hi = 0ull;
      if (c < m) lo = hi = dbits(A.lam[c]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      if (lane == 0) {
        atomicMin(lam_hist + 2 * outer, lo);
        atomicMax(lam_hist + 2 * outer + 1, hi);
      }
    }
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
  load_state(A, cur, s_w, s_T);
  int my_valid = 0;
  for (int ch = gw; ch < nch_p + nch_m; ch += GW) {
    double acc = 0.0;
    if (ch < nch_p) {
      const int64_t p = (int64_t)ch * CHUNK + lane;
      int v = 0;
      if (p < n) acc = point_relink(A, s_w, p, false, &v);
      my_valid += v;
      acc = warp_sum(acc);
      if (lane == 0) cs_p[ch] = acc;
    } else {
      const int64_t j = (int64_t)(ch - nch_p) * CHUNK + lane;
      if (j < n_act) acc = match_eval(A, s_w, j, true, false);
      acc = warp_sum(acc);
      if (lane == 0) cs_m[ch - nch_p] = acc;
    }
  }
  for (int o = 16; o > 0; o >>= 1) my_valid += __shfl_xor_sync(0xffffffffu, my_valid, o);
  if (lane == 0) s_cnt[warp] = my_valid;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < NWARPS; ++w) t += s_cnt[w];
    A.counts[rank] = t;
  }
  for (int c = gt; c < m; c += GT)
    for (int i = 0; i < 8; ++i) A.warps_out[8 * c + i] = s_w[8 * c + i];
  DSYNC(7);
  // support per control with the recomputed robust weights -> wa
  for (int c = gw; c < m; c += GW) {
    double sup = 0.0;
    const int q0 = ldi(A.cptr + c), q1 = ldi(A.cptr + c + 1);
    for (int q = q0 + lane; q < q1; q += 32) {
      const int e = ldi(A.cent + q);
      const int64_t p = e >> 3;
      if (!ldu8(A.cvalid + p)) continue;
      const double rs = ld(A.pr_rs + p);
      sup += rs * rs * A.bw[p * A.k + (e & 7)];
    }
    if (n_act > 0) {
      const int m0 = ldi(A.mptr + c), m1 = ldi(A.mptr + c + 1);
      for (int q = m0 + lane; q < m1; q += 32) {
        const int e = ldi(A.ment + q);
        sup += A.fw * A.fwt[e / A.k] * A.fbw[e];
      }
    }
    sup = warp_sum(sup);
    if (lane == 0) {
      const double w = A.arap_w * fmax(sup, A.data_floor);
      A.wa[c] = w;
      A.wa_out[c] = w;
    }
  }
  DSYNC(8);
  for (int ch = gw; ch < nch_e; ch += GW) {
    double acc = 0.0;
    const int e = ch * CHUNK + lane;
    if (e < A.n_edges) acc = edge_value(A, s_w, s_T, A.wa, e);
    acc = warp_sum(acc);
    if (lane == 0) cs_e[ch] = acc;
  }
  DSYNC(9);
  double parts[3];
  block_totals(cs_p, nch_p, cs_m, nch_m, cs_e, nch_e, s_part, parts);
  if (rank == 0 && threadIdx.x == 0) {
    dt_report* R = A.report;
    R->icp_cost = parts[0];
    R->feature_cost = parts[1];
    R->arap_cost = parts[2];
    R->total_cost = parts[0] + parts[1] + parts[2];
    int nc = 0;
    for (int i = 0; i < C; ++i) nc += __ldcg(A.counts + i);
    R->n_correspondences = nc;
    R->outer_iterations = outer_done;
    R->accepted_steps = accepted_steps;
    R->rejected_steps = rejected_steps;
    R->stalled = stalled ? 1 : 0;
    R->converged = converged ? 1 : 0;
    R->final_step_norm = final_step_norm;
    R->n_cost_history = n_hist;
  }
  TRACE(99);
  if (tr && rank == 0 && threadIdx.x == 0) tr[0] = tn;
}
