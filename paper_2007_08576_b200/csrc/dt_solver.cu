// dt_solver.cu -- one frame of the deformation solve (solver.solve_frame,
// solver.py:267-378) as ONE persistent kernel launch: the whole Levenberg-Marquardt loop
// (relink -> linearize -> per-control normal equations -> damped 6x6 solves -> tentative
// value pass -> accept / reject -> damping ladder) runs on the device with barriers
// between phases instead of kernel boundaries or host round trips.
//
// Two sync domains from one kernel body:
//   * cluster mode: a thread-block cluster (<= 16 CTAs, barrier.cluster) owns one
//     sequence; many sequences run concurrently on their own streams (BASELINE config 5);
//   * grid mode: a cooperative grid of one 256-thread CTA per SM owns one sequence
//     (lowest latency, the default for a single sequence).
//
// Phases (each ends at a domain barrier; details in dt_solver_kernel.cuh):
//   P1  (once) points & matches at the warm start: warp + project + gate + residual +
//       Tukey + blend gradient (kernels.py:483-569, 173-197, 239-250), normal-equation
//       rows at control-CSR positions; unit rigidity rows of every connection
//   P2  controls: fold the data rows -> 27 normal-equation columns + support -> rigidity
//       weight wa (energy.py:394-402)
//   P3  controls: fold the rigidity rows (kernels.py:341-467) with the fresh wa, damped
//       6x6 Cholesky (solver.py:217-258), publish delta + the tentative warp
//       exp(delta) * W (solver.py:261-264) and its rigid transform
//   P6  decide (solver.py:321-331), then points / matches / edges: cost at the tentative
//       warps with frozen robust and rigidity weights (solver.py:333-335) + speculative
//       relinearization there; accept iff strictly lower (solver.py:336)
//   final: support -> wa at the solution, its rigidity cost, the report and (grid mode)
//       the output warp of the template (tracking.py:87)
// Every reduction is deterministic and independent of the launch shape: normal equations
// are folded per control in CSR order, costs per fixed 32-item chunk then folded in chunk
// order, and every CTA evaluates the totals identically, so all CTAs take the same
// control-flow decisions.

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>

#include <cmath>
#include <cstdint>

#include "dt_common.cuh"
#include "dt_math.cuh"
#include "dt_ops.cuh"
#include "dt_solver.cuh"

namespace cg = cooperative_groups;

namespace dt {

constexpr int NWARPS = SOLVER_THREADS / 32;
constexpr int GOUT = 32;  // per-warp reduce-scatter readout (one accumulator per lane)

size_t solver_smem_bytes(int m) {
  if (m > M_MAX_SMEM) return sizeof(double) * (size_t)NWARPS * GOUT;  // global-state variant
  return sizeof(double) * ((size_t)21 * m + (size_t)NWARPS * GOUT);
}

// Loads of data produced by other CTAs in an earlier phase: L1-cacheable (every domain
// barrier has acquire semantics and invalidates L1 -- measured, tools/l1_probe.cu), so
// the several loads of one line within a phase (e.g. the four 16-byte pieces of a
// normal-equation row) are served by one L2 fill instead of one L2 trip each.
__device__ __forceinline__ double ld(const double* p) { return __ldca(p); }
__device__ __forceinline__ uint8_t ldu8(const uint8_t* p) {
  return (uint8_t)__ldca(reinterpret_cast<const unsigned char*>(p));
}
__device__ __forceinline__ int ldi(const int* p) { return __ldca(p); }
// data published by other CTAs WITHIN the phase (last-arriver reductions): L2 only
__device__ __forceinline__ double ldl2(const double* p) { return __ldcg(p); }

// Bulk (non-tensor TMA) global -> shared copies completing on an mbarrier: one thread
// streams a whole per-control table into shared memory while the others go on.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------------
// Per-lane normal-equation accumulation (FP64 FMA) + warp reduce-scatter. Each lane
// folds its rows [J0..J5, wv, sw] into 32 accumulators:
//   [0, 21) triu(J^T J) in kernels.py:41-44 order, [21, 27) J^T wv,
//   27: wv^2 (the rows' cost), 28: sw^2 (support), 29-31 unused;
// the reduce-scatter (31 shuffles) leaves lane l with the warp's sum of accumulator l.
// On B200 the FP64 tensor core (DMMA.8x8x4, mma.sync.m8n8k4.f64) runs at the DFMA rate
// (tools/fp64_probe.cu: 36 vs 34 TFLOP/s), so the 29 useful products per row beat the 64
// of an 8x8 Gram (the first version of these folds; ~3x slower end to end).
// ---------------------------------------------------------------------------------

__device__ __forceinline__ void acc_row(double (&a)[32], const double r[8]) {
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i; j < 6; ++j) a[triu_col(i, j)] = fma(r[i], r[j], a[triu_col(i, j)]);
#pragma unroll
  for (int i = 0; i < 6; ++i) a[21 + i] = fma(r[i], r[6], a[21 + i]);
  a[27] = fma(r[6], r[6], a[27]);
  a[28] = fma(r[7], r[7], a[28]);
}

// a rotation row: J3..J5 and sw are zero
__device__ __forceinline__ void acc_rot(double (&a)[32], const double r[8]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) a[triu_col(i, j)] = fma(r[i], r[j], a[triu_col(i, j)]);
#pragma unroll
  for (int i = 0; i < 3; ++i) a[21 + i] = fma(r[i], r[6], a[21 + i]);
  a[27] = fma(r[6], r[6], a[27]);
}

__device__ __forceinline__ double warp_reduce_scatter(double (&a)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = up ? a[i] : a[i + s];
      const double keep = up ? a[i + s] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return a[0];
}

// ---------------------------------------------------------------------------------
// sync domains
// ---------------------------------------------------------------------------------

template <bool GRID>
struct Dom;

template <>
struct Dom<false> {
  cg::cluster_group g;
  __device__ Dom() : g(cg::this_cluster()) {}
  __device__ int rank() const { return (int)g.block_rank(); }
  __device__ int size() const { return (int)g.num_blocks(); }
  __device__ int seq() const { return (int)(blockIdx.x / g.num_blocks()); }
  __device__ void sync() { g.sync(); }
};

template <>
struct Dom<true> {
  cg::grid_group g;
  __device__ Dom() : g(cg::this_grid()) {}
  __device__ int rank() const { return (int)blockIdx.x; }
  __device__ int size() const { return (int)gridDim.x; }
  __device__ int seq() const { return 0; }
  __device__ void sync() { g.sync(); }
};

// ---------------------------------------------------------------------------------
// state in shared memory: warps and their rigid transforms
// ---------------------------------------------------------------------------------

__device__ __forceinline__ void load_state(const SolverArgs& A, const double* src, double* s_w,
                                           double* s_T, uint64_t* bar, uint32_t& phase) {
  __syncthreads();
  if (threadIdx.x == 0) {  // the warps (8m doubles) by one bulk copy
    asm volatile("fence.proxy.async;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)(64 * A.m));
    bulk_g2s(s_w, src, (uint32_t)(64 * A.m), bar);
  }
  mbar_wait(bar, phase);
  phase ^= 1;
  for (int c = threadIdx.x; c < A.m; c += blockDim.x)
    dq_to_transform_fast(s_w + 8 * c, s_T + 12 * c, s_T + 12 * c + 9);
  __syncthreads();
}

// global-state variant: the warps stay where they are; this CTA's transforms of them
__device__ __forceinline__ void load_transforms(const SolverArgs& A, const double* w, double* T) {
  __syncthreads();
  for (int c = threadIdx.x; c < A.m; c += blockDim.x)
    dq_to_transform_fast(w + 8 * c, T + 12 * c, T + 12 * c + 9);
  __syncthreads();
}

template <int KM, typename IdxT>
__device__ __forceinline__ void blend_rows(const double* s_w, const IdxT* bidx, const double* bw,
                                           int64_t i, int k, double B[8], double sgn[KM],
                                           double a[KM]) {
  int idx[KM];
#pragma unroll
  for (int s = 0; s < KM; ++s)
    if (s < k) {
      idx[s] = bidx[i * k + s];
      a[s] = bw[i * k + s];
    }
  blend_at_k<KM>(s_w, idx, a, k, B, sgn);
}

// d(action)/dB with one reciprocal of |q|^2 (the Jacobian does not need the
// reference's per-entry division; values agree to the last ulp or two)
__device__ __forceinline__ void blend_gradient_fast(const double B[8], double px, double py,
                                                    double pz, double x0, double x1, double x2,
                                                    double s2, double* G) {
  const double is = 1.0 / s2;
  const double qw = B[0], qx = B[1], qy = B[2], qz = B[3];
  const double dw = B[4], dx = B[5], dy = B[6], dz = B[7];
  const double qup = qx * px + qy * py + qz * pz;
  G[0] = (2.0 * qw * px + 2.0 * (qy * pz - qz * py) + 2.0 * dx - 2.0 * x0 * qw) * is;
  G[8] = (2.0 * qw * py + 2.0 * (qz * px - qx * pz) + 2.0 * dy - 2.0 * x1 * qw) * is;
  G[16] = (2.0 * qw * pz + 2.0 * (qx * py - qy * px) + 2.0 * dz - 2.0 * x2 * qw) * is;
  G[1] = (2.0 * qup - 2.0 * dw - 2.0 * x0 * qx) * is;
  G[9] = (-2.0 * py * qx + 2.0 * qy * px - 2.0 * qw * pz - 2.0 * dz - 2.0 * x1 * qx) * is;
  G[17] = (-2.0 * pz * qx + 2.0 * qz * px + 2.0 * qw * py + 2.0 * dy - 2.0 * x2 * qx) * is;
  G[2] = (-2.0 * px * qy + 2.0 * qx * py + 2.0 * qw * pz + 2.0 * dz - 2.0 * x0 * qy) * is;
  G[10] = (2.0 * qup - 2.0 * dw - 2.0 * x1 * qy) * is;
  G[18] = (-2.0 * pz * qy + 2.0 * qz * py - 2.0 * qw * px - 2.0 * dx - 2.0 * x2 * qy) * is;
  G[3] = (-2.0 * px * qz + 2.0 * qx * pz - 2.0 * qw * py - 2.0 * dy - 2.0 * x0 * qz) * is;
  G[11] = (-2.0 * py * qz + 2.0 * qy * pz + 2.0 * qw * px + 2.0 * dx - 2.0 * x1 * qz) * is;
  G[19] = (2.0 * qup - 2.0 * dw - 2.0 * x2 * qz) * is;
  G[4] = -2.0 * qx * is;
  G[12] = -2.0 * qy * is;
  G[20] = -2.0 * qz * is;
  G[5] = 2.0 * qw * is;
  G[13] = 2.0 * qz * is;
  G[21] = -2.0 * qy * is;
  G[6] = -2.0 * qz * is;
  G[14] = 2.0 * qw * is;
  G[22] = 2.0 * qx * is;
  G[7] = 2.0 * qy * is;
  G[15] = -2.0 * qx * is;
  G[23] = 2.0 * qw * is;
}

// ---------------------------------------------------------------------------------
// rigidity rows, evaluated once per connection (kernels.py:341-467)
// ---------------------------------------------------------------------------------
// The rigidity weight of a connection only scales its rows (sqrt(0.5 base w_term)), so
// the unit-weight rows of BOTH endpoint bins are evaluated once per edge in P2 -- in
// parallel with the data gather, before the weights wa exist -- and stored at the bins'
// control-CSR positions (ipos), 3 rows x 8 per position:
//   [length J of the bin, length value, 0]
//   [angle 0->1 J of the bin, angle 0->1 value, 0]   (bin 0 = side a, bin 1 = side b)
//   [angle 1->0 J of the bin, angle 1->0 value, 0]   (bin 1 = side a, bin 0 = side b)
// so P3 streams each control's rows contiguously. The rotation rows need only the two
// quaternions and are rebuilt from shared memory.

constexpr int EROW = 24;

__device__ __forceinline__ void store_row8(double* dst, const double* J6, double v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(J6[0]), "d"(J6[1]),
               "d"(J6[2]), "d"(J6[3])
               : "memory");
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4), "d"(J6[4]), "d"(J6[5]),
               "d"(v), "d"(0.0)
               : "memory");
}

// Writes the unit rows of edge e into `erow` (at the bins' CSR positions) and its three
// values into `evals`; returns the values in v[3].
__device__ __forceinline__ void edge_unit_rows(const SolverArgs& A, const double* s_T, int e,
                                               double* erow, double* evals, double v[3]) {
  const int i0 = A.edges[2 * e], i1 = A.edges[2 * e + 1];
  DT_DCHECK(e >= 0 && e < A.n_edges && i0 >= 0 && i0 < A.m && i1 >= 0 && i1 < A.m);
  DT_DCHECK(__ldg(A.ipos + 2 * e) < 2 * A.n_edges && __ldg(A.ipos + 2 * e + 1) < 2 * A.n_edges);
  const double* p0 = A.cpts + 3 * i0;
  const double* p1 = A.cpts + 3 * i1;
  const double* T0 = s_T + 12 * i0;
  const double* T1 = s_T + 12 * i1;
  double p0t[3], p1t[3], c01[3], c10[3];
  xform(T0, T0 + 9, p0[0], p0[1], p0[2], p0t);
  xform(T1, T1 + 9, p1[0], p1[1], p1[2], p1t);
  xform(T0, T0 + 9, p1[0], p1[1], p1[2], c01);
  xform(T1, T1 + 9, p0[0], p0[1], p0[2], c10);
  // length (kernels.py:366-398)
  const double rx = p1[0] - p0[0], ry = p1[1] - p0[1], rz = p1[2] - p0[2];
  const double rest = sqrt(rx * rx + ry * ry + rz * rz);
  const double bx = p1t[0] - p0t[0], by = p1t[1] - p0t[1], bz = p1t[2] - p0t[2];
  const double ln2 = bx * bx + by * by + bz * bz;
  const double iln = rsqrt_nr(fmax(ln2, 1e-300));
  // |b| correctly rounded like `rest`, so an undeformed connection has a length residual
  // of exactly 0 as in the reference (an ulp-level |b| would leave ~1e-26 of rigidity
  // cost at rest and let the LM accept noise steps where the reference stalls)
  const double ln = sqrt(ln2);
  double bhx = 0.0, bhy = 0.0, bhz = 0.0;
  if (ln > 1e-9) {
    bhx = bx * iln;
    bhy = by * iln;
    bhz = bz * iln;
  }
  const double L0[6] = {p0t[1] * (-bhz) - p0t[2] * (-bhy), p0t[2] * (-bhx) - p0t[0] * (-bhz),
                        p0t[0] * (-bhy) - p0t[1] * (-bhx), -bhx, -bhy, -bhz};
  const double L1[6] = {p1t[1] * bhz - p1t[2] * bhy, p1t[2] * bhx - p1t[0] * bhz,
                        p1t[0] * bhy - p1t[1] * bhx, bhx, bhy, bhz};
  const double lv = ln - rest;
  // bending angle, both directions (kernels.py:400-417)
  double A01a[6], A01b[6], A10a[6], A10b[6];
  const double v01 = angle_unit(c01[0] - p0t[0], c01[1] - p0t[1], c01[2] - p0t[2],
                                p1t[0] - p0t[0], p1t[1] - p0t[1], p1t[2] - p0t[2], p0t[0], p0t[1],
                                p0t[2], p1t[0], p1t[1], p1t[2], A01a, A01b);
  const double v10 = angle_unit(c10[0] - p1t[0], c10[1] - p1t[1], c10[2] - p1t[2],
                                p0t[0] - p1t[0], p0t[1] - p1t[1], p0t[2] - p1t[2], p1t[0], p1t[1],
                                p1t[2], p0t[0], p0t[1], p0t[2], A10a, A10b);
  double* r0 = erow + (size_t)EROW * __ldg(A.ipos + 2 * e);
  double* r1 = erow + (size_t)EROW * __ldg(A.ipos + 2 * e + 1);
  store_row8(r0, L0, lv);
  store_row8(r0 + 8, A01a, v01);
  store_row8(r0 + 16, A10b, v10);
  store_row8(r1, L1, lv);
  store_row8(r1 + 8, A01b, v01);
  store_row8(r1 + 16, A10a, v10);
  evals[3 * e] = lv;
  evals[3 * e + 1] = v01;
  evals[3 * e + 2] = v10;
  v[0] = lv;
  v[1] = v01;
  v[2] = v10;
}

// rotation row r (0..3) of the bin `side` of edge (i0, i1) with weight sw: the 0.5 left
// product of the bin's quaternion, rotation columns only (kernels.py:419-461)
__device__ __forceinline__ void rotation_row(const double* s_w, int i0, int i1, int side, double sw,
                                             int r, double row[8]) {
  const double* q0 = s_w + 8 * i0;
  const double* q1 = s_w + 8 * i1;
  const double dq = q0[0] * q1[0] + q0[1] * q1[1] + q0[2] * q1[2] + q0[3] * q1[3];
  const double sg = dq < 0.0 ? -1.0 : 1.0;
  const double d = q0[r] - sg * q1[r];
  double P[12];
  if (side == 0) {
    half_left_mul(q0[0], q0[1], q0[2], q0[3], P);
  } else {
    const double h = -sg * 0.5;
    P[0] = h * q1[1] * -1.0; P[1] = h * q1[2] * -1.0; P[2] = h * q1[3] * -1.0;
    P[3] = h * q1[0];        P[4] = h * q1[3];        P[5] = h * -q1[2];
    P[6] = h * -q1[3];       P[7] = h * q1[0];        P[8] = h * q1[1];
    P[9] = h * q1[2];        P[10] = h * -q1[1];      P[11] = h * q1[0];
  }
  row[0] = sw * P[3 * r];
  row[1] = sw * P[3 * r + 1];
  row[2] = sw * P[3 * r + 2];
  row[3] = row[4] = row[5] = 0.0;
  row[6] = sw * d;
  row[7] = 0.0;
}

// rigidity cost of one connection from its three values (length, angle 0->1, angle
// 1->0) and the rotation term from the quaternions in smem: 2 x the bin cost, in
// arap_edge_bin's accumulation order (kernels.py:341-467)
__device__ __forceinline__ double edge_cost_vals(const SolverArgs& A, const double* s_w,
                                                 const double* wa, int e, double lv, double v01,
                                                 double v10) {
  const int i0 = A.edges[2 * e], i1 = A.edges[2 * e + 1];
  const double base = A.ew[e] * 0.5 * (ld(wa + i0) + ld(wa + i1));
  // (sqrt(0.5 base w) v)^2 without the square roots: the same value to an ulp
  const double hb = 0.5 * base;
  const double hba = hb * A.angle_w;
  const double* q0 = s_w + 8 * i0;
  const double* q1 = s_w + 8 * i1;
  const double dq = q0[0] * q1[0] + q0[1] * q1[1] + q0[2] * q1[2] + q0[3] * q1[3];
  const double sg = dq < 0.0 ? -1.0 : 1.0;
  const double d0 = q0[0] - sg * q1[0], d1 = q0[1] - sg * q1[1], d2 = q0[2] - sg * q1[2],
               d3 = q0[3] - sg * q1[3];
  double c = hb * (lv * lv);
  c += hba * (v01 * v01);
  c += hba * (v10 * v10);
  c += hb * A.rot_w * (d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3);
  return 2.0 * c;
}

// ---------------------------------------------------------------------------------
// Cholesky of the damped 6x6 system on a packed lower triangle (solver.py:217-258):
// M = A + lam diag(max(diag A, 1e-12)); forward / backward substitution in the
// reference's order. false (delta = 0) on a non-positive pivot.
template <int J>
__device__ __forceinline__ void chol_col(double (&L)[21], double (&inv)[6], bool& ok) {
  double s = L[J * (J + 1) / 2 + J];
#pragma unroll
  for (int q = 0; q < J; ++q) s -= L[J * (J + 1) / 2 + q] * L[J * (J + 1) / 2 + q];
  ok = ok && (s > 0.0);
  // 1/l_jj = rsqrt(s) in one MUFU + Newton chain, l_jj = s / sqrt(s) (ulp-level vs
  // sqrt + division; the pivot test s > 0 is the reference's)
  const double il = rsqrt_nr(fmax(s, 1e-300));
  inv[J] = il;
  L[J * (J + 1) / 2 + J] = s * il;
#pragma unroll
  for (int i = J + 1; i < 6; ++i) {
    double v = L[i * (i + 1) / 2 + J];
#pragma unroll
    for (int q = 0; q < J; ++q) v -= L[i * (i + 1) / 2 + q] * L[J * (J + 1) / 2 + q];
    L[i * (i + 1) / 2 + J] = v * inv[J];
  }
}

__device__ __forceinline__ bool solve6(const double* part, double lam, double delta[6]) {
  double L[21];  // row-major packed lower triangle: L[i(i+1)/2 + j]
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) L[i * (i + 1) / 2 + j] = part[triu_col(j, i)];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double a = L[i * (i + 1) / 2 + i];
    L[i * (i + 1) / 2 + i] = a + lam * fmax(a, 1e-12);
  }
  bool ok = true;
  double inv[6];  // one reciprocal per pivot instead of a division per entry
  // one column per instantiation: the sqrt slow-path call inside a loop would keep the
  // compiler from unrolling it and push L[] to local memory
  chol_col<0>(L, inv, ok);
  chol_col<1>(L, inv, ok);
  chol_col<2>(L, inv, ok);
  chol_col<3>(L, inv, ok);
  chol_col<4>(L, inv, ok);
  chol_col<5>(L, inv, ok);
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
    for (int j = 0; j < i; ++j) acc -= L[i * (i + 1) / 2 + j] * y[j];
    y[i] = acc * inv[i];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double acc = y[i];
#pragma unroll
    for (int j = i + 1; j < 6; ++j) acc -= L[j * (j + 1) / 2 + i] * delta[j];
    delta[i] = acc * inv[i];
  }
  return true;
}

#define TRACE(code)                                                \
  do {                                                             \
    if (tr && rank == 0 && threadIdx.x == 0 && tn < A.trace_cap) { \
      tr[1 + 2 * tn] = (code);                                     \
      tr[2 + 2 * tn] = gtimer();                                   \
      ++tn;                                                        \
    }                                                              \
  } while (0)
#define DSYNC(phase)                                                       \
  do {                                                                     \
    TRACE(10 * (phase));                                                   \
    if (A.arrivals && threadIdx.x == 0 && nbar < A.arr_cap)                \
      A.arrivals[2 + (size_t)rank * A.arr_cap + nbar] = gtimer();          \
    ++nbar;                                                                \
    dom.sync();                                                            \
    TRACE(10 * (phase) + 1);                                               \
  } while (0)

#include "dt_solver_kernel.cuh"

// KM = 4: the reference's bind_k (SolverConfig / RunConfig default, warpfield.py:157);
// KM = 8: any k <= 8 with runtime slot guards
template __global__ void k_solve_frame<false, 4, false, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 4, false, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<false, 8, false, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 8, false, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<false, 4, true, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 4, true, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<false, 8, true, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 8, true, 2>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<false, 4, false, 1>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 4, false, 1>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<false, 8, false, 1>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 8, false, 1>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<false, 4, true, 1>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 4, true, 1>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<false, 8, true, 1>(const SolverArgs* __restrict__);
template __global__ void k_solve_frame<true, 8, true, 1>(const SolverArgs* __restrict__);

template <bool GRID>
static void* solver_fn(int k, bool big, int team) {
  if (team == 1) {
    if (big) return k == 4 ? (void*)k_solve_frame<GRID, 4, true, 1> : (void*)k_solve_frame<GRID, 8, true, 1>;
    return k == 4 ? (void*)k_solve_frame<GRID, 4, false, 1> : (void*)k_solve_frame<GRID, 8, false, 1>;
  }
  if (big) return k == 4 ? (void*)k_solve_frame<GRID, 4, true, 2> : (void*)k_solve_frame<GRID, 8, true, 2>;
  return k == 4 ? (void*)k_solve_frame<GRID, 4, false, 2> : (void*)k_solve_frame<GRID, 8, false, 2>;
}

// per-device cache of the occupancy probe (a hardware property; atomic so concurrent
// tracker creation on several host threads is race-free)
static std::atomic<int> g_max_cluster[16];

int solver_max_cluster(int device) {
  if (device < 0 || device >= 16) return 8;
  const int cached = g_max_cluster[device].load(std::memory_order_relaxed);
  if (cached > 0) return cached;
  int best = 1;
  auto* fn = k_solve_frame<false, 8, false, 2>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const size_t smem = solver_smem_bytes(1024);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters > 0) {
      best = c;
      break;
    }
    cudaGetLastError();
  }
  g_max_cluster[device].store(best, std::memory_order_relaxed);
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

int solver_grid_blocks(int device, int m_max) {
  auto* fn = m_max > M_MAX_SMEM ? k_solve_frame<true, 8, true, 2> : k_solve_frame<true, 8, false, 2>;
  const size_t smem = solver_smem_bytes(m_max);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, SOLVER_THREADS, smem) != cudaSuccess)
    per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return per_sm >= 1 ? sms : 0;  // one CTA per SM
}

// Warps per control team in P2 / P3: pairs while one round of the full grid's teams
// (148 CTAs x 4) covers every control, single warps for larger graphs (config 4, 1,026
// controls: 0.83 -> 0.76 ms). A function of m alone -- not of the launch shape -- because
// the team width fixes the fold order, and results must not depend on the cluster size.
static int solver_team(int m) {
#ifdef DT_TEAM_OVERRIDE
  (void)m;
  return DT_TEAM_OVERRIDE;
#else
  return m > 592 ? 1 : 2;
#endif
}

int solver_launch(const SolverArgs* d_args, int n_seq, int cluster, int m_max, int k, int grid_mode,
                  cudaStream_t s) {
  DT_REQUIRE(k >= 1 && k <= KMAX, DT_ERR_UNSUPPORTED, "bind_k=%d outside the device path (<= %d)", k,
             KMAX);
  const size_t smem = solver_smem_bytes(m_max);
  const bool big = m_max > M_MAX_SMEM;
  if (grid_mode) {
    DT_REQUIRE(n_seq == 1, DT_ERR_UNSUPPORTED, "grid mode runs one sequence per launch");
    int dev = 0;
    DT_CHECK_CUDA(cudaGetDevice(&dev));
    const int blocks = solver_grid_blocks(dev, m_max);
    DT_REQUIRE(blocks > 0, DT_ERR_UNSUPPORTED, "solver kernel cannot be co-resident for a grid launch");
    void* fn = solver_fn<true>(k, big, solver_team(m_max));
    DT_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void* params[] = {(void*)&d_args};
    DT_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(blocks), dim3(SOLVER_THREADS),
                                              params, smem, s));
    return DT_OK;
  }
  void* fn = solver_fn<false>(k, big, solver_team(m_max));
  DT_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DT_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
  void* params[] = {(void*)&d_args};
  DT_CHECK_CUDA(cudaLaunchKernelExC(&cfg, fn, params));
  return DT_OK;
}

}  // namespace dt
