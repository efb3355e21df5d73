// dt_solver_kernel.cuh -- body of the persistent LM kernel (included by dt_solver.cu).
//
// Work units inside the sync domain (C CTAs x 8 warps), dealt round-robin over the CTAs:
//   * points / matches / edges: one item per lane, fixed 32-item chunks whose partial
//     sums are folded by the last-arriving warp (red_commit; deterministic, independent
//     of C);
//   * controls: a team of TEAM warps of one CTA per control; each lane folds its rows
//     into 32 FP64 accumulators, a warp reduce-scatter leaves lane l with accumulator l,
//     the team combines its warps in warp order (deterministic, independent of C).
// Barriers per accepted outer iteration: P2 | P3 | value pass. The solvers publish the
// tentative warps, every CTA loads them into its own shared memory, and the value pass
// also relinearizes at the tentative warps into the second buffer ("speculative
// relinearization"), so an accepted step starts the next iteration directly at P2; a
// stalled iteration keeps its linearization -- the reference recomputes it at the same
// warps, bit for bit the same -- and only re-solves.


// one of the two linearization buffers
struct PBuf {
  double* rec;  // n x 8 correspondence records [o0 o1 o2 rs g0 g1 g2 valid]
  double* row;  // (n*k) x 8 rows at control-CSR positions
};

__device__ __forceinline__ PBuf pbuf(const SolverArgs& A, int b) {
  const int64_t n = A.n;
  return {A.crec + (size_t)b * n * 8, A.prow + (size_t)b * n * A.k * 8};
}

// 256-bit global accesses (LDG/STG.E.ENL2.256): a 64-byte row or record is two of them.
// Volatile so they are never merged with or hoisted above a domain barrier.
__device__ __forceinline__ void st256(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
// data written by other CTAs in an earlier phase (L1-cacheable: barriers invalidate L1)
__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.ca.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
// read-only for the whole launch (template statics, the frame's pixel records)
__device__ __forceinline__ void ld256_nc(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
__device__ __forceinline__ void ld256_nc_i(const int* p, int v[8]) {
  asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "l"(p));
}

__device__ __forceinline__ double* mrows(const SolverArgs& A, int b) {
  return A.mrow + (size_t)b * A.ma_cap * A.k * 3 * 8;
}

__device__ __forceinline__ double* erows_buf(const SolverArgs& A, int b) {
  return A.erow + (size_t)b * 2 * A.n_edges * EROW;
}

__device__ __forceinline__ double* evals_buf(const SolverArgs& A, int b) {
  return A.evals + (size_t)b * 3 * A.n_edges;
}

__device__ __forceinline__ void store_row(double* dst, const double r[8]) {
  st256(dst, r[0], r[1], r[2], r[3]);
  st256(dst + 4, r[4], r[5], r[6], r[7]);
}

__device__ __forceinline__ void load_row(const double* src, double r[8]) {
  ld256(src, r[0], r[1], r[2], r[3]);
  ld256(src + 4, r[4], r[5], r[6], r[7]);
}

// Relink point p at the warps in smem (kernels.py:483-569) and linearize it into `nb`
// (kernels.py:173-197): the correspondence + robust weight, and for every slot the
// normal-equation row of its control [J0..J5, sqrt(w) r, sqrt(w)] (J = sw alpha sign
// (gn . K_c), sw = rs sqrt(alpha)) at the slot's control-CSR position. Returns the
// point's icp cost under the Tukey weight of the new residual. With `ob`, *cost_old
// receives the point's cost at these warps under the frozen correspondence and robust
// weight of record `ob` (the value pass, solver.py:333-335).
// Everything point p's step reads that does not depend on the warps: the template point
// and normal, its binding (+ sqrt alpha, CSR positions) and -- for the value pass -- the
// frozen correspondence of record `ob`. Issued before the value pass's decide prologue so
// this L2 round trip overlaps it.
template <int KM>
struct PointIn {
  int idx[KM], pos[KM];
  double a[KM], sqa[KM];
  double px, py, pz, tn0, tn1, tn2;
  double oo0, oo1, oo2, on0, on1, on2, ors;
  uint8_t ovalid;
};

template <int KM>
__device__ __forceinline__ void point_load(const SolverArgs& A, int64_t p, const PBuf* ob,
                                           PointIn<KM>& in) {
  in.ovalid = 0;
  in.oo0 = in.oo1 = in.oo2 = in.on0 = in.on1 = in.on2 = in.ors = 0.0;
  if (ob) {  // the frozen correspondence record: two 256-bit loads
    double v;
    ld256(ob->rec + 8 * p, in.oo0, in.oo1, in.oo2, in.ors);
    ld256(ob->rec + 8 * p + 4, in.on0, in.on1, in.on2, v);
    in.ovalid = v != 0.0 ? 1 : 0;
  }
  if constexpr (KM == 4) {
    // the packed statics: five 256-bit loads instead of 22 scalar ones
    const double* q = A.pst + 16 * p;
    ld256_nc(q, in.a[0], in.a[1], in.a[2], in.a[3]);
    ld256_nc(q + 4, in.sqa[0], in.sqa[1], in.sqa[2], in.sqa[3]);
    double pad;
    ld256_nc(q + 8, in.px, in.py, in.pz, pad);
    ld256_nc(q + 12, in.tn0, in.tn1, in.tn2, pad);
    int ip[8];
    ld256_nc_i(A.pi8 + 8 * p, ip);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      in.idx[s] = ip[s];
      in.pos[s] = ip[4 + s];
      DT_DCHECK(ip[s] >= 0 && ip[s] < A.m && ip[4 + s] >= 0 && ip[4 + s] < A.n * 4);
    }
  } else {
    const int kk = A.k;
#pragma unroll
    for (int s = 0; s < KM; ++s)
      if (s < kk) {
        in.idx[s] = A.bidx[p * kk + s];
        in.a[s] = A.bw[p * kk + s];
        in.pos[s] = __ldg(A.cpos + p * kk + s);
        in.sqa[s] = __ldg(A.bws + p * kk + s);  // sqrt(alpha), correctly rounded: the reference's
      }
    in.px = A.tp[3 * p];
    in.py = A.tp[3 * p + 1];
    in.pz = A.tp[3 * p + 2];
    in.tn0 = A.tn[3 * p];
    in.tn1 = A.tn[3 * p + 1];
    in.tn2 = A.tn[3 * p + 2];
  }
}

// The gates of the projective association and the point's cost terms are written with
// explicit rounding intrinsics, which the compiler never contracts into FMAs: they decide
// discrete outcomes, and the value pass's cost at an unchanged iterate must equal the
// linearization's cost bit for bit (or a zero step would be "accepted") -- whatever the
// translation unit's -fmad setting (_build.py SOURCE_FLAGS).
__device__ __forceinline__ double dot3_rn(double a0, double a1, double a2, double b0, double b1,
                                          double b2) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
}

// n . (x - o) and the cost (sw r)^2 of one slot, identical in both passes
__device__ __forceinline__ double plane_res(double n0, double n1, double n2, double x0, double x1,
                                            double x2, double o0, double o1, double o2) {
  return dot3_rn(n0, n1, n2, __dsub_rn(x0, o0), __dsub_rn(x1, o1), __dsub_rn(x2, o2));
}

template <int KM>
__device__ __forceinline__ double point_step(const SolverArgs& A, const double* s_w, int64_t p,
                                             const PointIn<KM>& in, bool value_pass,
                                             const PBuf& nb, double* cost_old, int* valid_out,
                                             long long* dbg = nullptr) {
#ifdef DT_WARP_TRACE
#define PSTAMP(i)                        \
  do {                                   \
    if (dbg) dbg[i] = clock64();         \
  } while (0)
#else
#define PSTAMP(i) \
  do {            \
  } while (0)
#endif
  PSTAMP(0);
  const int kk = KM == 4 ? 4 : A.k;
  const int* pos = in.pos;
  const double* sqa = in.sqa;
  const double* a = in.a;
  const double px = in.px, py = in.py, pz = in.pz;
  double B[8], sgn[KM];
  blend_at_k<KM>(s_w, in.idx, in.a, kk, B, sgn);
  PSTAMP(1);
  double x0, x1, x2, s2;
  apply_blend(B, px, py, pz, x0, x1, x2, s2);
  PSTAMP(2);
  if (value_pass) {
    double co = 0.0;
    if (in.ovalid) {
      const double r = plane_res(in.on0, in.on1, in.on2, x0, x1, x2, in.oo0, in.oo1, in.oo2);
#pragma unroll
      for (int s = 0; s < KM; ++s)
        if (s < kk) {
          const double wv = __dmul_rn(__dmul_rn(in.ors, sqa[s]), r);
          co = __dadd_rn(co, __dmul_rn(wv, wv));
        }
    }
    *cost_old = co;
  }
  double r0, r1, r2;
  rotate_normal(B, in.tn0, in.tn1, in.tn2, r0, r1, r2);
  bool ok = false;
  double o0 = 0, o1 = 0, o2 = 0, g0 = 0, g1 = 0, g2 = 0;
  // projection and gates, in the reference's IEEE order (kernels.py:537-568)
  if (x2 > 0.0) {
    const double uf = rint(__dadd_rn(__ddiv_rn(__dmul_rn(A.fx, x0), x2), A.cx));
    const double vf = rint(__dadd_rn(__ddiv_rn(__dmul_rn(A.fy, x1), x2), A.cy));
    if (uf >= 0.0 && uf < (double)A.width && vf >= 0.0 && vf < (double)A.height) {
      const int ui = (int)uf, vi = (int)vf;
      const int64_t pix = (int64_t)vi * A.width + ui;
      DT_DCHECK(pix >= 0 && pix < (int64_t)A.width * A.height);
      // the pixel's depth (NaN = invalid) and normal: one 256-bit load
      double d, h0, h1, h2;
      ld256_nc(A.pixrec + 4 * pix, d, h0, h1, h2);
      PSTAMP(3);
      if (d == d) {
        o0 = __dmul_rn(__ddiv_rn(__dsub_rn((double)ui, A.cx), A.fx), d);
        o1 = __dmul_rn(__ddiv_rn(__dsub_rn((double)vi, A.cy), A.fy), d);
        o2 = d;
        g0 = h0;
        g1 = h1;
        g2 = h2;
        if (dot3_rn(g0, g1, g2, g0, g1, g2) > 0.25) {
          const double dx = __dsub_rn(o0, x0), dy = __dsub_rn(o1, x1), dz = __dsub_rn(d, x2);
          ok = __dsqrt_rn(dot3_rn(dx, dy, dz, dx, dy, dz)) < A.gate &&
               dot3_rn(g0, g1, g2, r0, r1, r2) > A.cos_gate;
        }
      }
    }
  }
  *valid_out = ok ? 1 : 0;
  if (!ok) {
    const double z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    st256(nb.rec + 8 * p + 4, 0.0, 0.0, 0.0, 0.0);  // valid = 0 (the rest is never read)
#pragma unroll
    for (int s = 0; s < KM; ++s)
      if (s < kk) store_row(nb.row + 8 * (size_t)pos[s], z);
    return 0.0;
  }
  const double r = plane_res(g0, g1, g2, x0, x1, x2, o0, o1, o2);
  const double rs = tukey_fast(r, A.inv_tukey);
  PSTAMP(4);
  st256(nb.rec + 8 * p, o0, o1, o2, rs);
  st256(nb.rec + 8 * p + 4, g0, g1, g2, 1.0);
  double G[24];
  blend_gradient_fast(B, px, py, pz, x0, x1, x2, s2, G);
  double gn[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) gn[e] = g0 * G[e] + g1 * G[8 + e] + g2 * G[16 + e];
  PSTAMP(5);
  double cost = 0.0;
#pragma unroll
  for (int s = 0; s < KM; ++s)
    if (s < kk) {
      const int c = in.idx[s];
      const double sw = __dmul_rn(rs, sqa[s]);
      const double wv = __dmul_rn(sw, r);
      cost = __dadd_rn(cost, __dmul_rn(wv, wv));
      const double coef = sw * a[s] * sgn[s];
      Basis K;
      make_basis(s_w + 8 * c, K);
      double pr[6], row[8];
      basis_project(gn, K.Kr, K.Kd, pr);
#pragma unroll
      for (int d = 0; d < 6; ++d) row[d] = coef * pr[d];
      row[6] = wv;
      row[7] = sw;
      store_row(nb.row + 8 * (size_t)pos[s], row);
    }
  PSTAMP(6);
  return cost;
}

// One active match at the warps in smem (kernels.py:239-250): for every slot the three
// rows [J0..J5, sqrt(w) res_c, (c == 0 ? sqrt(w) : 0)] at the slot's match-CSR position;
// returns its feature cost (no robust weight, so the same value serves the value pass
// and the relinearization).
template <int KM>
__device__ __forceinline__ double match_step(const SolverArgs& A, const double* s_w, int64_t j,
                                             double* rows) {
  const int kk = KM == 4 ? 4 : A.k;
  double B[8], sgn[KM], a[KM];
  blend_rows<KM>(s_w, A.fbidx, A.fbw, j, kk, B, sgn, a);
  const double px = A.fp[3 * j], py = A.fp[3 * j + 1], pz = A.fp[3 * j + 2];
  double x0, x1, x2, s2;
  apply_blend(B, px, py, pz, x0, x1, x2, s2);
  const double res[3] = {x0 - A.fo[3 * j], x1 - A.fo[3 * j + 1], x2 - A.fo[3 * j + 2]};
  double G[24];
  blend_gradient_fast(B, px, py, pz, x0, x1, x2, s2, G);
  const double w = A.fwt[j];
  double cost = 0.0;
#pragma unroll
  for (int s = 0; s < KM; ++s)
    if (s < kk) {
      const int c = A.fbidx[j * kk + s];
      DT_DCHECK(c >= 0 && c < A.m && __ldg(A.mpos + j * kk + s) >= 0 &&
                __ldg(A.mpos + j * kk + s) < A.ma_cap * kk);
      const double sw = sqrt(A.fw * w * a[s]);
      const double v0 = sw * res[0], v1 = sw * res[1], v2 = sw * res[2];
      cost = __dadd_rn(cost, dot3_rn(v0, v1, v2, v0, v1, v2));
      const double coef = sw * a[s] * sgn[s];
      Basis K;
      make_basis(s_w + 8 * c, K);
      double* dst = rows + 24 * (size_t)__ldg(A.mpos + j * kk + s);
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) {
        double pr[6], row[8];
        basis_project(G + 8 * comp, K.Kr, K.Kd, pr);
#pragma unroll
        for (int d = 0; d < 6; ++d) row[d] = coef * pr[d];
        row[6] = sw * res[comp];
        row[7] = comp == 0 ? sw : 0.0;
        store_row(dst + 8 * comp, row);
      }
    }
  return cost;
}

// ---------------------------------------------------------------------------------
// Last-arriver reductions. Every item (a chunk of 32 points / matches / edges, or one
// control) commits its value(s); the last warp to commit an item of a 32-item group folds
// the group in a fixed order, the last group folds the groups in a fixed order and
// publishes the total. The folds never depend on which warp or CTA produced an item nor
// on the arrival order, so totals are deterministic and independent of the launch shape,
// and after the domain barrier every CTA reads one line instead of every item value
// (all-CTA reads of the item arrays hot-spot L2: ~8 us per phase measured).
// ---------------------------------------------------------------------------------

struct RedSlot {
  double* gsum;    // [2][G] group values
  double* total;   // [2]
  unsigned* gcnt;  // [G] per-group commit counters (reset by the group's last arriver)
  unsigned* tcnt;  // group counter (reset by the last group)
  int G;
};

// slots: 0 points (value-pass cost, relinearization cost), 1 matches, 2 rigidity cost of
// the iterate (P3) and of the solution, 3 controls (all solves ok = min, max step norm),
// 4 rigidity cost in the value pass
__device__ __forceinline__ RedSlot red_slot(const SolverArgs& A, int s) {
  const int G = A.red_g;
  double* base = A.red + (size_t)s * (2 * G + 2);
  unsigned* cb = A.redc + (size_t)s * (G + 1);
  return {base, base + 2 * G, cb, cb + G, G};
}

// OP 0: sum; OP 1: (min, max)
template <int OP>
__device__ __forceinline__ double red_op(int k, double a, double b) {
  if (OP == 0) return a + b;
  return k == 0 ? fmin(a, b) : fmax(a, b);
}

template <int OP>
__device__ __forceinline__ double red_id(int k) {
  return OP == 0 ? 0.0 : (k == 0 ? INFINITY : -INFINITY);
}

template <int OP>
__device__ __forceinline__ double warp_red(int k, double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_op<OP>(k, v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// item value arrays of a slot (chunk-sum scratch in A.csum): slot 0 points (2 arrays),
// slot 1 matches, slots 2 / 4 edges
__device__ __forceinline__ double* red_vals(const SolverArgs& A, int slot, int k) {
  const int nch_tot = A.nch_p + A.nch_m + A.nch_e;
  if (slot == 0) return A.csum + (k == 0 ? 0 : nch_tot);
  if (slot == 1) return A.csum + A.nch_p;
  return A.csum + A.nch_p + A.nch_m;
}

__device__ __forceinline__ const double* red_total(const SolverArgs& A, int slot) {
  return A.red + (size_t)slot * (2 * A.red_g + 2) + 2 * A.red_g;
}

// Commit item ch (of nch) with the warp-uniform values v[NV]. Whole warp. The slot's
// pointers are derived from A (shared memory) on use, not kept in registers.
template <int NV, int OP>
__device__ __noinline__ void red_commit(const SolverArgs& A, int slot, int ch, int nch,
                                        const double (&v)[NV]) {
  const RedSlot R = red_slot(A, slot);
  double* vals[2] = {red_vals(A, slot, 0), red_vals(A, slot, 1)};
  const int lane = threadIdx.x & 31;
  const int g = ch >> 5;
  DT_DCHECK(ch >= 0 && ch < nch && g < R.G);
  unsigned old = 0;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) vals[k][ch] = v[k];
    __threadfence();
    old = atomicAdd(R.gcnt + g, 1u);
  }
  old = __shfl_sync(0xffffffffu, old, 0);
  const int gs = min(32, nch - 32 * g);
  if ((int)old != gs - 1) return;
  __threadfence();
  double x[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    x[k] = lane < gs ? ldl2(vals[k] + 32 * g + lane) : red_id<OP>(k);
    x[k] = warp_red<OP>(k, x[k]);
  }
  unsigned old2 = 0;
  if (lane == 0) {
    R.gcnt[g] = 0;
#pragma unroll
    for (int k = 0; k < NV; ++k) R.gsum[k * R.G + g] = x[k];
    __threadfence();
    old2 = atomicAdd(R.tcnt, 1u);
  }
  old2 = __shfl_sync(0xffffffffu, old2, 0);
  const int ng = (nch + 31) >> 5;
  if ((int)old2 != ng - 1) return;
  __threadfence();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double acc = red_id<OP>(k);
    for (int q = lane; q < ng; q += 32) acc = red_op<OP>(k, acc, ldl2(R.gsum + k * R.G + q));
    x[k] = warp_red<OP>(k, acc);
  }
  if (lane == 0) {
    *R.tcnt = 0;
#pragma unroll
    for (int k = 0; k < NV; ++k) R.total[k] = x[k];
  }
}

// the tentative warp of control c, exp(delta) * W (solver.py:261-264), and its rigid
// transform, published for every CTA's value pass
__device__ __forceinline__ void publish_tentative(const SolverArgs& A, int c, const double W[8],
                                                  const double d[6], double* tent) {
  double tw[8], T[12];
  apply_step_one_fast(W, d, tw);
  dq_to_transform_fast(tw, T, T + 9);
  double2* t2 = reinterpret_cast<double2*>(tent + 8 * c);
#pragma unroll
  for (int i = 0; i < 4; ++i) t2[i] = make_double2(tw[2 * i], tw[2 * i + 1]);
  double2* T2 = reinterpret_cast<double2*>(A.tentT + 12 * c);
#pragma unroll
  for (int i = 0; i < 6; ++i) T2[i] = make_double2(T[2 * i], T[2 * i + 1]);
}

// damped solve of control c from the stored normal equations -> delta, ok / |delta|,
// and the tentative warp from the current one
__device__ __forceinline__ void resolve_control(const SolverArgs& A, int c, double lam, double* ok,
                                                double* nrm, const double* cur, double* tent) {
  double part[27], d[6], W[8];
#pragma unroll
  for (int i = 0; i < 27; ++i) part[i] = ld(A.partial + 27 * c + i);
#pragma unroll
  for (int i = 0; i < 8; ++i) W[i] = ld(cur + 8 * c + i);
  const bool good = solve6(part, lam, d);
  double nn = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    A.delta[6 * c + i] = d[i];
    nn += d[i] * d[i];
  }
  ok[c] = good ? 1.0 : 0.0;
  nrm[c] = sqrt(nn);
  publish_tentative(A, c, W, d, tent);
}

// Work units of the relinearizing passes (P1, P6): 32-item chunks of points, matches and
// edges, dealt round-robin over the domain's warps (unit u -> warp u mod GW). When the
// chunks outnumber the warps by `extra`, the warps that take a second unit would finish
// last; the order below makes those units edge chunks handed to warps whose first unit
// was an edge chunk too -- two edge chunks outlast one point chunk less than a point and
// an edge chunk do. Order: edge chunks [0, extra), point chunks, match chunks, edge chunks
// [extra, nch_e).
struct Unit {
  int kind;  // 0 point chunk, 1 match chunk, 2 edge chunk
  int ch;    // chunk index within its kind
};

__device__ __forceinline__ Unit unit_of(int u, int nch_p, int nch_m, int nch_e, int extra) {
  if (u < extra) return {2, u};
  u -= extra;
  if (u < nch_p) return {0, u};
  u -= nch_p;
  if (u < nch_m) return {1, u};
  return {2, extra + (u - nch_m)};
}

// BIG: control graphs whose state does not fit in shared memory (m > M_MAX_SMEM): the
// warps and tentative transforms are read in place from global memory (L1-cached after
// each barrier), the current transforms and the damping live in this CTA's slice of
// A.gstate; everything else is the same kernel.
// TM: warps per control team in P2 / P3 -- 2 when every control gets its own team in
// one round (the pair halves each control's fold), 1 when the controls outnumber the
// teams (one warp per control halves the number of rounds; the host picks).
template <bool GRID, int KM, bool BIG, int TM>
__global__ void __launch_bounds__(SOLVER_THREADS, 1) k_solve_frame(const SolverArgs* __restrict__ all) {
  constexpr int TEAM = TM;
  constexpr int TEAMS_PER_CTA = NWARPS / TM;
  Dom<GRID> dom;
  const int C = dom.size();
  const int rank = dom.rank();
  __shared__ SolverArgs A;
  __shared__ double s_part[8 * NWARPS];
  __shared__ double s_tot[8];
  __shared__ double s_sup[NWARPS];
  __shared__ double s_col[TEAMS_PER_CTA][32];
  __shared__ int s_cnt[NWARPS];
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t s_bar;  // completion of the bulk tentative-state loads
  if (threadIdx.x == 0) {
    A = all[dom.seq()];
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t bar_phase = 0;
  const int m = A.m;
  const int64_t n = A.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / TEAM, tw = warp % TEAM;
  double* s_w = BIG ? A.warp_a : smem;
  double* const s_Tcur = BIG ? A.gstate + (size_t)rank * 13 * m : smem + 8 * m;
  double* s_T = s_Tcur;
  double* s_lam = BIG ? s_Tcur + 12 * m : smem + 20 * m;  // per-control damping, per CTA
  double* gout = (BIG ? smem : smem + 21 * m) + warp * GOUT;
  // work items are dealt round-robin over the CTAs first (item i -> CTA i % C), so
  // every SM of the domain gets a share of each phase
  const int gw = warp * C + rank, GW = C * NWARPS;
  const int gw_rev = (NWARPS - 1 - warp) * C + rank;
  const int gt = rank * (int)blockDim.x + (int)threadIdx.x, GT = C * (int)blockDim.x;
  // per-control work (re-solves, tentative store) is interleaved over the CTAs --
  // control c belongs to CTA c % C -- so no CTA becomes the straggler
  const int gc = (int)threadIdx.x * C + rank;
  const int gteam = team * C + rank, GTEAM = C * TEAMS_PER_CTA;
  const int team_rounds = (m + GTEAM - 1) / GTEAM;
  const int64_t n_act = A.n_active ? *A.n_active : 0;
  const int nch_p = (int)((n + CHUNK - 1) / CHUNK);
  const int nch_m = (int)((n_act + CHUNK - 1) / CHUNK);
  const int nch_e = (A.n_edges + CHUNK - 1) / CHUNK;
  const int nch_tot = A.nch_p + A.nch_m + A.nch_e;
  // second-round units of the relinearizing passes (see unit_of)
  const int extra = min(nch_e / 2, max(0, nch_p + nch_m + nch_e - GW));
  // chunk-sum set 0: value pass (points, matches, edges) and the rigidity cost of the
  // iterate; set 1: icp / feature cost of each (speculative) relinearization

  long long* tr = A.trace;
  int tn = 0, nbar = 0;
  TRACE(0);

  for (int c = threadIdx.x; c < m; c += blockDim.x) s_lam[c] = A.lam_init;

  double* cur = A.warp_a;
  double* tent = A.warp_b;
  int pb = 0;               // record buffer holding the linearization at `cur`
  bool smem_is_cur = true;  // s_w / s_T hold `cur`
  bool need_lin = true;     // P2 / P3 must be evaluated at `cur`
  int accepted_steps = 0, rejected_steps = 0, n_hist = 0, outer_done = 0;
  bool converged = false, stalled = false;
  double final_step_norm = 0.0;
  int parity = 0;
  double cb_icp = 0.0, cb_feat = 0.0, cb_arap = 0.0;
  double pd0 = 0.0, pd1 = 0.0;  // P2 -> P3: this team-lane's data column, team rounds 0 / 1

  // ---- P1: relink + linearize at the warm start (buffer 0): points, matches, unit
  // rigidity rows of the connections ----
  if (rank == 0)  // this launch's stall flags (written by CTA 0 thread 0 after barriers)
    for (int i = threadIdx.x; i < A.max_outer; i += blockDim.x) A.stalled_hist[i] = 0;
  if (BIG) {
    s_w = cur;  // the host copied the warm start into warp_a
    s_T = s_Tcur;
    load_transforms(A, s_w, s_T);
  } else {
    // the warm start straight from the last solution; this CTA's slice of it into `cur`
    // (first read from global memory after the P1 barrier)
    load_state(A, A.warps_out, s_w, s_T, &s_bar, bar_phase);
    for (int c = gc; c < m; c += GT)
#pragma unroll
      for (int i = 0; i < 8; ++i) cur[8 * c + i] = s_w[8 * c + i];
  }
  TRACE(12);
  {
    const PBuf nb = pbuf(A, 0);
    double* nm = mrows(A, 0);
    double* ne = erows_buf(A, 0);
    double* nv = evals_buf(A, 0);
    for (int u = gw; u < nch_p + nch_m + nch_e; u += GW) {
      const Unit un = unit_of(u, nch_p, nch_m, nch_e, extra);
      const int ch = un.ch;
      double acc = 0.0;
      if (un.kind == 0) {
        const int64_t p = (int64_t)ch * CHUNK + lane;
        int vd;
        if (p < n) {
          PointIn<KM> pin;
          point_load<KM>(A, p, nullptr, pin);
          acc = point_step<KM>(A, s_w, p, pin, false, nb, nullptr, &vd);
        }
        acc = warp_sum(acc);
        red_commit<2, 0>(A, 0, ch, nch_p, {0.0, acc});
      } else if (un.kind == 1) {
        const int64_t j = (int64_t)ch * CHUNK + lane;
        if (j < n_act) acc = match_step<KM>(A, s_w, j, nm);
        acc = warp_sum(acc);
        red_commit<1, 0>(A, 1, ch, nch_m, {acc});
      } else {
        const int e = ch * CHUNK + lane;
        double v[3];
        if (e < A.n_edges) edge_unit_rows(A, s_T, e, ne, nv, v);
      }
    }
  }
  DSYNC(1);
  if (threadIdx.x == 0) s_tot[0] = ld(red_total(A, 0) + 1);
  if (threadIdx.x == 1) s_tot[1] = nch_m > 0 ? ld(red_total(A, 1)) : 0.0;
  __syncthreads();
  cb_icp = s_tot[0];
  cb_feat = s_tot[1];

  for (int outer = 0; outer < A.max_outer; ++outer) {
    outer_done = outer + 1;
    // [0, m) ok, [m, 2m) |delta|, [2m, 3m) rigidity cost of the control's bins
    double* okn = A.oknorm + (size_t)parity * 3 * m;
    if (need_lin) {
      const double* prow = pbuf(A, pb).row;
      const double* mrow = mrows(A, pb);
      const double* erow = erows_buf(A, pb);
      // ---- P2: each control's data rows (contiguous at its CSR positions) -> normal
      // equations + support (per-lane FMA accumulation, warp reduce-scatter) ----
      TRACE(22);
      for (int r = 0; r < team_rounds; ++r) {
        const int c = r * GTEAM + gteam;
        double acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.0;
        if (c < m) {
          const int q0 = __ldg(A.cptr + c), q1 = __ldg(A.cptr + c + 1);
          int m0 = 0, m1 = 0;
          if (n_act > 0) {
            m0 = ldi(A.mptr + c);
            m1 = ldi(A.mptr + c + 1);
          }
          DT_DCHECK(0 <= q0 && q0 <= q1 && q1 <= A.n * A.k && 0 <= m0 && m0 <= m1 &&
                    m1 <= A.ma_cap * A.k);
          const int np_rows = q1 - q0, total = np_rows + 3 * (m1 - m0);
          const double* pbase = prow + 8 * (size_t)q0;
          const double* mbase = mrow + 24 * (size_t)m0;
          // two row blocks in flight per warp: blocks b and b + TEAM, pushed in order
          for (int base = 32 * tw; base < total; base += 64 * TEAM) {
            double ra[8] = {0, 0, 0, 0, 0, 0, 0, 0}, rb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const int ia = base + lane, ib = base + 32 * TEAM + lane;
            if (ia < np_rows) load_row(pbase + 8 * (size_t)ia, ra);
            else if (ia < total) load_row(mbase + 8 * (size_t)(ia - np_rows), ra);
            if (ib < np_rows) load_row(pbase + 8 * (size_t)ib, rb);
            else if (ib < total) load_row(mbase + 8 * (size_t)(ib - np_rows), rb);
            acc_row(acc, ra);
            if (base + 32 * TEAM < total) acc_row(acc, rb);
          }
        }
        TRACE(23);
        gout[lane] = warp_reduce_scatter(acc);
        __syncthreads();
        if (tw == 0 && c < m) {
          // combine the team's warps in warp order; accumulator 28 = support. The same
          // team folds this control's rigidity rows in P3, so the data columns stay in a
          // register (P3 publishes data + rigidity for the re-solves)
          if (lane < 27) {
            double v = 0.0;
            for (int w = 0; w < TEAM; ++w) v += gout[w * GOUT + lane];
            if (r == 0) pd0 = v;
            else if (r == 1) pd1 = v;
            else A.partial[27 * c + lane] = v;
          }
          if (lane == 28) {
            double su = 0.0;
            for (int w = 0; w < TEAM; ++w) su += gout[w * GOUT + 28];
            A.wa[c] = A.arap_w * fmax(su, A.data_floor);
          }
        }
        __syncthreads();
        TRACE(24);
      }
      DSYNC(2);

      // ---- P3: rigidity rows -> normal equations + first damped solve; rigidity cost
      // of the iterate from the stored rows ----
      for (int r = 0; r < team_rounds; ++r) {
        const int c = r * GTEAM + gteam;
        double acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.0;
        if (c < m) {
          const int q0 = __ldg(A.iptr + c), q1 = __ldg(A.iptr + c + 1);
          const double wac = ld(A.wa + c);
          for (int base = q0 + 32 * tw; base < q1; base += 32 * TEAM) {
            const int q = base + lane;
            const bool live = q < q1;
            int i0 = c, i1 = c, side = 0;
            double sw = 0.0, swa = 0.0, swr = 0.0;
            double u0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, u1[8] = {0, 0, 0, 0, 0, 0, 0, 0},
                   u2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (live) {
              const int info = __ldg(A.iinfo + q);
              const int o = info >> 1;
              DT_DCHECK(q < 2 * A.n_edges && o >= 0 && o < m);
              side = info & 1;
              const double* er = erow + (size_t)EROW * q;
              load_row(er, u0);
              load_row(er + 8, u1);
              load_row(er + 16, u2);
              const double wao = ld(A.wa + o);
              i0 = side == 0 ? c : o;
              i1 = side == 0 ? o : c;
              const double base_w =
                  __ldg(A.iew + q) * 0.5 * (side == 0 ? wac + wao : wao + wac);
              sw = sqrt(0.5 * base_w);
              swa = sw * A.sq_angle_w;  // = sqrt(0.5 base angle_w) to an ulp
              swr = sw * A.sq_rot_w;
            }
            if (live) {
              double row[8];
              // length, angle 0->1, angle 1->0 rows of this bin (unit rows x weight)
#pragma unroll
              for (int i = 0; i < 8; ++i) row[i] = sw * u0[i];
              acc_row(acc, row);
#pragma unroll
              for (int i = 0; i < 8; ++i) row[i] = swa * u1[i];
              acc_row(acc, row);
#pragma unroll
              for (int i = 0; i < 8; ++i) row[i] = swa * u2[i];
              acc_row(acc, row);
#pragma unroll
              for (int rr = 0; rr < 4; ++rr) {
                rotation_row(s_w, i0, i1, side, swr, rr, row);
                acc_rot(acc, row);
              }
            }
          }
        }
        TRACE(33);
        gout[lane] = warp_reduce_scatter(acc);
        TRACE(32);
        __syncthreads();
        if (tw == 0 && c < m) {
          if (lane < 27) {
            double v = 0.0;
            for (int w = 0; w < TEAM; ++w) v += gout[w * GOUT + lane];
            v = (r == 0 ? pd0 : (r == 1 ? pd1 : ld(A.partial + 27 * c + lane))) + v;
            A.partial[27 * c + lane] = v;
            s_col[team][lane] = v;
          }
          if (lane == 27) {
            // accumulator 27 of the rigidity rows = the rigidity cost of this control's
            // bins (each connection's rows go to both bins: the bins sum to its cost)
            double v = 0.0;
            for (int w = 0; w < TEAM; ++w) v += gout[w * GOUT + 27];
            okn[2 * m + c] = v;
          }
          __syncwarp();
          double okv = 0.0, nrm = 0.0;
          if (lane == 0) {
            double d[6];
            const bool good = solve6(s_col[team], s_lam[c], d);
            double nn = 0.0;
            for (int i = 0; i < 6; ++i) {
              A.delta[6 * c + i] = d[i];
              nn += d[i] * d[i];
            }
            okv = good ? 1.0 : 0.0;
            nrm = sqrt(nn);
            publish_tentative(A, c, s_w + 8 * c, d, tent);
          }
          if (lane == 0) {
            okn[c] = okv;
            okn[m + c] = nrm;
          }
        }
        __syncthreads();
        TRACE(34);
      }
    } else {
      // after a stall the iterate and its linearization are unchanged: re-solve the
      // stored normal equations with the raised damping (solver.py:348-355)
      for (int c = gc; c < m; c += GT) resolve_control(A, c, s_lam[c], okn, okn + m, cur, tent);
    }
    bool accepted = false;
    double cost_before = 0.0, cost_after = 0.0;
    for (int attempt = 0; attempt <= A.max_retries; ++attempt) {
      if (attempt > 0) {
        okn = A.oknorm + (size_t)parity * 3 * m;
        for (int c = gc; c < m; c += GT) resolve_control(A, c, s_lam[c], okn, okn + m, cur, tent);
      }
      DSYNC(attempt == 0 ? 3 : 4);
      // this warp's first value-pass point: its warp-independent inputs are loaded now,
      // overlapping the decide prologue's round trip
      PointIn<KM> pin0;
      const Unit u0 = unit_of(gw, nch_p, nch_m, nch_e, extra);
      const int64_t p0 = (int64_t)u0.ch * CHUNK + lane;
      const bool pre = u0.kind == 0 && gw < nch_p + nch_m + nch_e && p0 < n;
      if (pre) {
        const PBuf ob0 = pbuf(A, pb);
        point_load<KM>(A, p0, &ob0, pin0);
      }
      // The solvers published every control's tentative warp and transform; load them
      // into shared memory together with the per-control solve results (one round
      // trip), then decide (all solves ok? largest step norm; after a fresh
      // linearization also the rigidity cost of the iterate) -- identical in every CTA.
      const bool want_e = attempt == 0 && need_lin;
      const int pc = threadIdx.x;
      if (BIG) {
        s_w = tent;  // read in place
        s_T = A.tentT;
      } else if (threadIdx.x == 0) {
        // tentative warps (8m) and transforms (12m) -> s_w / s_T by two bulk copies; the
        // proxy fence orders this CTA's earlier generic shared-memory accesses (and the
        // barrier-acquired global writes) before the async-proxy copies
        asm volatile("fence.proxy.async;" ::: "memory");
        mbar_expect_tx(&s_bar, (uint32_t)(160 * m));
        bulk_g2s(s_w, tent, (uint32_t)(64 * m), &s_bar);
        bulk_g2s(s_T, A.tentT, (uint32_t)(96 * m), &s_bar);
      }
      double o_ok = 1.0, o_nm = 0.0, o_ar = 0.0;
      if (pc < m) {
        o_ok = ld(okn + pc);
        o_nm = ld(okn + m + pc);
        if (want_e) o_ar = ld(okn + 2 * m + pc);
      }
      smem_is_cur = false;
      TRACE(57);
      {
        double allok = o_ok, mx = o_nm, es = o_ar;
        for (int i = pc + blockDim.x; i < m; i += blockDim.x) {
          allok = fmin(allok, ld(okn + i));
          mx = fmax(mx, ld(okn + m + i));
          if (want_e) es += ld(okn + 2 * m + i);
        }
        allok = warp_min(allok);
        mx = warp_max(mx);
        es = warp_sum(es);
        __syncthreads();
        if (lane == 0) {
          s_part[3 * warp] = allok;
          s_part[3 * warp + 1] = mx;
          s_part[3 * warp + 2] = es;
        }
        if (!BIG) {
          mbar_wait(&s_bar, bar_phase);  // the tentative warps / transforms are in smem
          bar_phase ^= 1;
        }
        __syncthreads();
        allok = 1.0;
        mx = 0.0;
        es = 0.0;
        for (int w = 0; w < NWARPS; ++w) {
          allok = fmin(allok, s_part[3 * w]);
          mx = fmax(mx, s_part[3 * w + 1]);
          es += s_part[3 * w + 2];
        }
        if (want_e) cb_arap = es;
        if (attempt == 0) cost_before = (cb_icp + cb_feat) + cb_arap;
        TRACE(53);
        parity ^= 1;
        if (!(allok > 0.5)) {
          // raise the damping of the failed controls only, retry (solver.py:321-326)
          for (int c = threadIdx.x; c < m; c += blockDim.x)
            if (ld(okn + c) < 0.5) s_lam[c] = fmin(s_lam[c] * A.lam_inc, A.lam_max);
          __syncthreads();
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
      TRACE(52);
      // ---- P6: cost at the tentative warps with frozen weights and correspondences
      // (set 0) + speculative relinearization there (buffer 1 - pb, costs in set 1) ----
      {
        const PBuf ob = pbuf(A, pb);
        const PBuf nb = pbuf(A, 1 - pb);
        double* nm = mrows(A, 1 - pb);
        double* ne = erows_buf(A, 1 - pb);
        double* nv = evals_buf(A, 1 - pb);
        for (int u = gw; u < nch_p + nch_m + nch_e; u += GW) {
          const Unit un = unit_of(u, nch_p, nch_m, nch_e, extra);
          const int ch = un.ch;
          if (un.kind == 0) {
            const int64_t p = (int64_t)ch * CHUNK + lane;
            double co = 0.0, cn = 0.0;
            int vd;
            long long* dbg = nullptr;
#ifdef DT_WARP_TRACE
            if (A.arrivals && outer == 1 && attempt == 0 && lane == 0 && rank < 8)
              dbg = A.arrivals + 2 + (size_t)1024 * A.arr_cap + 20000 + (rank * NWARPS + warp) * 8;
#endif
            if (p < n) {
              if (u == gw && pre) {
                cn = point_step<KM>(A, s_w, p, pin0, true, nb, &co, &vd, dbg);
              } else {
                PointIn<KM> pin;
                point_load<KM>(A, p, &ob, pin);
                cn = point_step<KM>(A, s_w, p, pin, true, nb, &co, &vd, dbg);
              }
            }
            co = warp_sum(co);
            cn = warp_sum(cn);
            red_commit<2, 0>(A, 0, ch, nch_p, {co, cn});
          } else if (un.kind == 1) {
            const int64_t j = (int64_t)ch * CHUNK + lane;
            double cf = 0.0;
            if (j < n_act) cf = match_step<KM>(A, s_w, j, nm);
            cf = warp_sum(cf);
            red_commit<1, 0>(A, 1, ch, nch_m, {cf});
          } else {
            const int e = ch * CHUNK + lane;
            double acc = 0.0;
            if (e < A.n_edges) {
              double v[3];
              edge_unit_rows(A, s_T, e, ne, nv, v);
              acc = edge_cost_vals(A, s_w, A.wa, e, v[0], v[1], v[2]);
            }
            acc = warp_sum(acc);
            red_commit<1, 0>(A, 4, ch, nch_e, {acc});
          }
        }
      }
#ifdef DT_WARP_TRACE
      // debug: per-warp end of the value pass on every CTA, first attempt of outer 1
      if (A.arrivals && outer == 1 && attempt == 0 && lane == 0)
        A.arrivals[2 + (size_t)1024 * A.arr_cap + (size_t)rank * NWARPS + warp] = gtimer();
#endif
      DSYNC(6);
      // value pass (points, matches, edges) + cost of the speculative relinearization
      if (threadIdx.x == 0) s_tot[0] = ld(red_total(A, 0));
      if (threadIdx.x == 1) s_tot[1] = ld(red_total(A, 0) + 1);
      if (threadIdx.x == 2) s_tot[2] = nch_m > 0 ? ld(red_total(A, 1)) : 0.0;
      if (threadIdx.x == 3) s_tot[3] = nch_e > 0 ? ld(red_total(A, 4)) : 0.0;
      __syncthreads();
      cost_after = (s_tot[0] + s_tot[2]) + s_tot[3];
      TRACE(63);
      if (cost_after < cost_before) {
        double* tmp = cur;
        cur = tent;
        tent = tmp;
        pb = 1 - pb;
        smem_is_cur = true;
        cb_icp = s_tot[1];
        cb_feat = s_tot[2];
        for (int c = threadIdx.x; c < m; c += blockDim.x)
          s_lam[c] = fmax(s_lam[c] * A.lam_dec, A.lam_min);
        TRACE(64);
        ++accepted_steps;
        if (rank == 0 && threadIdx.x == 0) {
          A.cost_hist[2 * n_hist] = cost_before;
          A.cost_hist[2 * n_hist + 1] = cost_after;
        }
        ++n_hist;
        accepted = true;
        break;
      }
      for (int c = threadIdx.x; c < m; c += blockDim.x)
        s_lam[c] = fmin(s_lam[c] * A.lam_inc, A.lam_max);
      __syncthreads();
      ++rejected_steps;
    }
    // lambda_history (solver.py:345): min / max of the final per-control damping of this
    // outer iteration -- every CTA holds the same s_lam; one warp of CTA (outer % C)
    // records it
    __syncthreads();
    if (rank == outer % C && warp == NWARPS - 1) {
      double lo = INFINITY, hi = -INFINITY;
      for (int c = lane; c < m; c += 32) {
        lo = fmin(lo, s_lam[c]);
        hi = fmax(hi, s_lam[c]);
      }
      lo = warp_min(lo);
      hi = warp_max(hi);
      if (lane == 0) {
        A.lam_hist[2 * outer] = lo;
        A.lam_hist[2 * outer + 1] = hi;
      }
    }
    TRACE(65);
    if (converged) break;
    if (!accepted) {
      stalled = true;
      need_lin = false;
      if (rank == 0 && threadIdx.x == 0) A.stalled_hist[outer] = 1;
      continue;
    }
    need_lin = true;
    if (cost_before - cost_after <= A.cost_tol * fmax(cost_before, 1e-30)) {
      converged = true;
      break;
    }
  }

  // ---- final report (solver.py:360-376). Record buffer pb is the relinearization at
  // the solution (robust weights recomputed there), so only the support -> rigidity
  // weights and the rigidity cost with them remain ----
  if (BIG) {
    if (!smem_is_cur) {
      s_w = cur;
      s_T = s_Tcur;
      load_transforms(A, s_w, s_T);
    }
  } else if (!smem_is_cur) {
    load_state(A, cur, s_w, s_T, &s_bar, bar_phase);
  }
  TRACE(72);
  {
    const PBuf cb = pbuf(A, pb);
    int my_valid = 0;
    for (int64_t p = gt; p < n; p += GT) my_valid += ld(cb.rec + 8 * p + 7) != 0.0 ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) my_valid += __shfl_xor_sync(0xffffffffu, my_valid, o);
    if (lane == 0) s_cnt[warp] = my_valid;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < NWARPS; ++w) t += s_cnt[w];
      A.counts[rank] = t;
    }
    for (int c = gc; c < m; c += GT)
      for (int i = 0; i < 8; ++i) A.warps_out[8 * c + i] = s_w[8 * c + i];

    // support per control from its rows' last column: sum of sw^2 = rs^2 alpha (points)
    // + w_pair (matches, component-0 rows)
    const double* prow = cb.row;
    const double* mrow = mrows(A, pb);
    for (int c = gw; c < m; c += GW) {
      double sup = 0.0;
      const int q0 = __ldg(A.cptr + c), q1 = __ldg(A.cptr + c + 1);
      for (int q = q0 + lane; q < q1; q += 32) {
        const double v = ld(prow + 8 * (size_t)q + 7);
        sup += v * v;
      }
      if (n_act > 0) {
        const int m0 = ldi(A.mptr + c), m1 = ldi(A.mptr + c + 1);
        for (int q = m0 + lane; q < m1; q += 32) {
          const double v = ld(mrow + 24 * (size_t)q + 7);
          sup += v * v;
        }
      }
      sup = warp_sum(sup);
      if (lane == 0) {
        const double w = A.arap_w * fmax(sup, A.data_floor);
        A.wa[c] = w;
        A.wa_out[c] = w;
      }
    }
  }
  DSYNC(8);
  for (int ch = gw; ch < nch_e; ch += GW) {
    double acc = 0.0;
    const int e = ch * CHUNK + lane;
    if (e < A.n_edges) {
      const double* ev = evals_buf(A, pb) + 3 * e;
      acc = edge_cost_vals(A, s_w, A.wa, e, ld(ev), ld(ev + 1), ld(ev + 2));
    }
    acc = warp_sum(acc);
    red_commit<1, 0>(A, 2, ch, nch_e, {acc});
  }
  DSYNC(9);
  const double t_arap = nch_e > 0 ? ld(red_total(A, 2)) : 0.0;
  if (rank == 0 && threadIdx.x == 0) {
    dt_report* R = A.report;
    R->icp_cost = cb_icp;
    R->feature_cost = cb_feat;
    R->arap_cost = t_arap;
    R->total_cost = (cb_icp + cb_feat) + t_arap;
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
  // the frame's output (tracking.py:87, warpfield.warp_all): every template point and
  // normal through the solution's blended warps, which are already in shared memory --
  // the same device functions as dt_warp_all, so the same bits, without a launch; after
  // the last barrier, so no CTA waits for it
  if (A.out_p) {
    for (int64_t p = gt; p < n; p += GT) {
      double B[8], sgn[KMAX];
      blend_at(s_w, A.bidx + p * A.k, A.bw + p * A.k, A.k, B, sgn);
      double x0, x1, x2, s2;
      apply_blend(B, A.tp[3 * p], A.tp[3 * p + 1], A.tp[3 * p + 2], x0, x1, x2, s2);
      double r0, r1, r2;
      rotate_normal(B, A.tn[3 * p], A.tn[3 * p + 1], A.tn[3 * p + 2], r0, r1, r2);
      A.out_p[3 * p] = x0;
      A.out_p[3 * p + 1] = x1;
      A.out_p[3 * p + 2] = x2;
      A.out_n[3 * p] = r0;
      A.out_n[3 * p + 1] = r1;
      A.out_n[3 * p + 2] = r2;
    }
  }
  TRACE(99);
  if (tr && rank == 0 && threadIdx.x == 0) tr[0] = tn;
  if (A.arrivals && rank == 0 && threadIdx.x == 0) {
    A.arrivals[0] = C;
    A.arrivals[1] = nbar;
  }
}
