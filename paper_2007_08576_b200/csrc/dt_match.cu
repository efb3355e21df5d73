// dt_match.cu -- ORB Hamming matching and 1-point-RANSAC + reweighting preselection.
//
//  * k_hamming: brute-force 256-bit descriptor matching (north-star part 3a; the
//    reference has no implementation). popc(a ^ b) over 8 x 32-bit words,
//    frame descriptors staged through shared memory, per-lane running argmin and a
//    warp-shuffle (dist, index) argmin; ties resolve to the lowest frame index.
//  * k_preselect_warp / k_preselect_final: matching.preselect_inliers
//    (matching.py:174-226). One warp per reference hypothesis runs the whole
//    rectify -> (weighted Procrustes -> residuals -> reweight) x iters alternation
//    (matching.py:145-171); the 3x3 Procrustes uses a one-sided Jacobi SVD whose singular
//    values are accurate relative to S0, so the reference's degeneracy test
//    S1 <= 1e-9 S0 (matching.py:122) decides the same way as LAPACK's gesdd.
//  * k_preselect_orb (+ a 168-register build for CTAs of <= 12 warps): the ORB path in
//    one launch -- every CTA builds the frame's match list from the Hamming winners into
//    its shared memory (k_build_matches' rule, dt_tracker.cu), its warps evaluate their
//    hypotheses from there with the same evaluate_hypothesis as k_preselect_warp, and the
//    last CTA to finish takes the winner and writes flags, weights, the per-feature
//    scatter and the report statistics in k_preselect_final's arithmetic and order.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "dt_common.cuh"
#include "dt_math.cuh"
#include "dt_ops.cuh"

namespace dt {

// ---------------------------------------------------------------------------------
// Hamming
// ---------------------------------------------------------------------------------

// 2000 x 2500 at config 2: 125 CTAs x 8 frame ranges of 313 descriptors; each lane
// compares one staged frame descriptor with its warp's four templates (four independent
// popc chains). Measured (bench orb_match stage): 2 templates x 4 ranges 27.6 us, 4 x 4
// 29.5, 8 x 4 29.5, 4 x 8 25.5, 2 x 8 25.5, 8 x 8 27.6, 4 x 16 25.4, 2 x 16 25.5.
#ifndef DT_HAM_TPW
#define DT_HAM_TPW 4
#endif
#ifndef DT_HAM_SPLITS
#define DT_HAM_SPLITS 8
#endif
constexpr int HAM_TPW = DT_HAM_TPW;        // template descriptors per warp
constexpr int HAM_WARPS = 4;               // warps per CTA
constexpr int HAM_TILE = 512;              // frame descriptors per smem tile (16 KB)
constexpr int HAM_SPLITS = DT_HAM_SPLITS;  // frame-descriptor ranges (grid rows) per template

// blockIdx.y selects a contiguous range of frame descriptors; with `packed` the per-range
// winners are folded by a 64-bit atomicMin of (distance << 32 | index) -- the
// lexicographic (distance, index) minimum whatever the order of the ranges, i.e. ties
// still resolve to the lowest frame index.
__global__ void __launch_bounds__(HAM_WARPS * 32)
k_hamming(const uint4* __restrict__ tdesc, int64_t nt, const uint4* __restrict__ fdesc, int64_t nf,
          int64_t per_split, int32_t* __restrict__ best_idx, int32_t* __restrict__ best_dist,
          unsigned long long* __restrict__ packed) {
  __shared__ uint4 s_tile[HAM_TILE * 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = ((int64_t)blockIdx.x * HAM_WARPS + warp) * HAM_TPW;
  uint32_t a[HAM_TPW][8];
#pragma unroll
  for (int j = 0; j < HAM_TPW; ++j) {
    const int64_t t = t0 + j;
    uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
    if (t < nt) {
      lo = tdesc[2 * t];
      hi = tdesc[2 * t + 1];
    }
    a[j][0] = lo.x; a[j][1] = lo.y; a[j][2] = lo.z; a[j][3] = lo.w;
    a[j][4] = hi.x; a[j][5] = hi.y; a[j][6] = hi.z; a[j][7] = hi.w;
  }
  int bd[HAM_TPW], bi[HAM_TPW];
#pragma unroll
  for (int j = 0; j < HAM_TPW; ++j) {
    bd[j] = 0x7fffffff;
    bi[j] = 0x7fffffff;
  }
  const int64_t f_begin = (int64_t)blockIdx.y * per_split;
  const int64_t f_end = f_begin + per_split < nf ? f_begin + per_split : nf;
  for (int64_t base = f_begin; base < f_end; base += HAM_TILE) {
    const int cnt = (int)((f_end - base) < HAM_TILE ? (f_end - base) : HAM_TILE);
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * cnt; i += blockDim.x) s_tile[i] = fdesc[2 * base + i];
    __syncthreads();
    for (int f = lane; f < cnt; f += 32) {
      const uint4 lo = s_tile[2 * f], hi = s_tile[2 * f + 1];
#pragma unroll
      for (int j = 0; j < HAM_TPW; ++j) {
        const int d = __popc(a[j][0] ^ lo.x) + __popc(a[j][1] ^ lo.y) + __popc(a[j][2] ^ lo.z) +
                      __popc(a[j][3] ^ lo.w) + __popc(a[j][4] ^ hi.x) + __popc(a[j][5] ^ hi.y) +
                      __popc(a[j][6] ^ hi.z) + __popc(a[j][7] ^ hi.w);
        if (d < bd[j]) {  // strict: this lane visits indices in increasing order
          bd[j] = d;
          bi[j] = (int)(base + f);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < HAM_TPW; ++j) {
    int d = bd[j], i = bi[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int od = __shfl_xor_sync(0xffffffffu, d, o);
      const int oi = __shfl_xor_sync(0xffffffffu, i, o);
      if (od < d || (od == d && oi < i)) {
        d = od;
        i = oi;
      }
    }
    const int64_t t = t0 + j;
    if (lane == 0 && t < nt) {
      if (packed) {
        if (f_begin < f_end)
          atomicMin(packed + t, ((unsigned long long)(unsigned)d << 32) | (unsigned)i);
      } else {
        best_idx[t] = nf > 0 ? i : -1;
        best_dist[t] = nf > 0 ? d : 257;
      }
    }
  }
}

__global__ void k_unpack_hamming(const unsigned long long* __restrict__ packed, int64_t nt, int64_t nf,
                                 int32_t* __restrict__ best_idx, int32_t* __restrict__ best_dist) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const unsigned long long v = packed[t];
  best_idx[t] = nf > 0 ? (int32_t)(v & 0xffffffffull) : -1;
  best_dist[t] = nf > 0 ? (int32_t)(v >> 32) : 257;
}

// With `packed` (nt uint64 scratch) the frame descriptors are split over HAM_SPLITS grid
// rows and the results stay packed (dist << 32 | idx; the ORB match build reads them);
// otherwise one pass writes best_idx / best_dist.
int launch_hamming(const uint8_t* tdesc, int64_t nt, const uint8_t* fdesc, int64_t nf,
                   int32_t* best_idx, int32_t* best_dist, cudaStream_t s,
                   unsigned long long* packed, bool packed_ready) {
  if (nt == 0) return DT_OK;
  const int per_cta = HAM_WARPS * HAM_TPW;
  int splits = 1;
  int64_t per = nf;
  if (packed) {
    // all-ones start values (the tracker's match build leaves them that way after use)
    if (!packed_ready)
      DT_CHECK_CUDA(cudaMemsetAsync(packed, 0xff, sizeof(unsigned long long) * nt, s));
    splits = HAM_SPLITS;
    per = ((nf + splits - 1) / splits + 31) / 32 * 32;
    if (per <= 0) per = 32;
    splits = (int)std::max<int64_t>(1, (nf + per - 1) / per);
  }
  const dim3 grid((unsigned)grid_for(nt, per_cta), (unsigned)splits);
  k_hamming<<<grid, HAM_WARPS * 32, 0, s>>>(reinterpret_cast<const uint4*>(tdesc), nt,
                                            reinterpret_cast<const uint4*>(fdesc), nf, per,
                                            best_idx, best_dist, packed);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

// ---------------------------------------------------------------------------------
// Weighted Procrustes rotation (matching.weighted_rotation, matching.py:108-125): see
// procrustes_lane below (C = the 3x3 weighted cross-covariance sum_k w_k s2_k s1_k^T).
// ---------------------------------------------------------------------------------

// residual |s2 - R s1| (matching.rotation_residuals, matching.py:128-130)
__device__ __forceinline__ double rot_residual(const double R[9], const double s1[3], const double s2[3]) {
  const double e0 = s2[0] - (s1[0] * R[0] + s1[1] * R[1] + s1[2] * R[2]);
  const double e1 = s2[1] - (s1[0] * R[3] + s1[1] * R[4] + s1[2] * R[5]);
  const double e2 = s2[2] - (s1[0] * R[6] + s1[1] * R[7] + s1[2] * R[8]);
  return sqrt(e0 * e0 + e1 * e1 + e2 * e2);
}

// reweight (matching.py:133-136): min(H/d, 1), a zero residual maps to 1
__device__ __forceinline__ double reweight(double d, double H) {
  return d > H ? H / fmax(d, 1e-300) : 1.0;
}

// Warm-started one-sided Jacobi on the columns of A = C V0 (V0 from the previous IRLS
// iteration, so one or two rotating sweeps usually suffice); V (in/out) accumulates the
// rotations. Every lane may hold a different C (two hypotheses per warp run their SVDs in
// the two half-warps at once); the sweep loop is warp-uniform. Singular values come from
// the orthogonalized columns, accurate relative to S0, so the reference's degeneracy test
// S1 <= 1e-9 S0 (matching.py:122) decides as LAPACK's gesdd does.
__device__ __forceinline__ bool procrustes_lane(const double C[9], double V[9], double R[9]) {
  double A[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      A[r * 3 + c] = C[r * 3 + 0] * V[0 * 3 + c] + C[r * 3 + 1] * V[1 * 3 + c] + C[r * 3 + 2] * V[2 * 3 + c];
  for (int sweep = 0; sweep < 16; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double alpha = A[p] * A[p] + A[3 + p] * A[3 + p] + A[6 + p] * A[6 + p];
      const double beta = A[q] * A[q] + A[3 + q] * A[3 + q] + A[6 + q] * A[6 + q];
      const double gamma = A[p] * A[q] + A[3 + p] * A[3 + q] + A[6 + p] * A[6 + q];
      // rotate while |gamma| > 1e-15 sqrt(alpha beta)
      if (gamma != 0.0 && gamma * gamma > 1e-30 * (alpha * beta)) {
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        double t;
        if (fabs(zeta) > 1e150) {
          t = 0.5 / zeta;
        } else {
          const double q = 1.0 + zeta * zeta;
          t = copysign(1.0, zeta) / (fabs(zeta) + q * rsqrt_nr(q));
        }
        const double c = rsqrt_nr(1.0 + t * t);
        const double sn = c * t;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double ap = A[r * 3 + p], aq = A[r * 3 + q];
          A[r * 3 + p] = c * ap - sn * aq;
          A[r * 3 + q] = sn * ap + c * aq;
          const double vp = V[r * 3 + p], vq = V[r * 3 + q];
          V[r * 3 + p] = c * vp - sn * vq;
          V[r * 3 + q] = sn * vp + c * vq;
        }
      }
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
  // column norms as x * rsqrt(x) (within an ulp of sqrt; the reference's degeneracy test
  // S1 <= 1e-9 S0 is far from that resolution)
  const double q0 = A[0] * A[0] + A[3] * A[3] + A[6] * A[6];
  const double q1 = A[1] * A[1] + A[4] * A[4] + A[7] * A[7];
  const double q2 = A[2] * A[2] + A[5] * A[5] + A[8] * A[8];
  double s0 = q0 > 0.0 ? q0 * rsqrt_nr(q0) : 0.0;
  double s1 = q1 > 0.0 ? q1 * rsqrt_nr(q1) : 0.0;
  double s2 = q2 > 0.0 ? q2 * rsqrt_nr(q2) : 0.0;
  // order the columns by singular value (descending, stable)
  int o0 = 0, o1 = 1;
  double S0 = s0, S1 = s1;
  if (s1 > s0) { o0 = 1; o1 = 0; S0 = s1; S1 = s0; }
  if (s2 > S1) {
    if (s2 > S0) { o1 = o0; S1 = S0; o0 = 2; S0 = s2; }
    else { o1 = 2; S1 = s2; }
  }
  if (!(S0 > 0.0) || S1 <= 1e-9 * S0) return false;
  const double iS0 = 1.0 / S0, iS1 = 1.0 / S1;
  double u1[3], u2[3], v1[3], v2[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double a0 = o0 == 0 ? A[r * 3] : (o0 == 1 ? A[r * 3 + 1] : A[r * 3 + 2]);
    const double a1 = o1 == 0 ? A[r * 3] : (o1 == 1 ? A[r * 3 + 1] : A[r * 3 + 2]);
    u1[r] = a0 * iS0;
    u2[r] = a1 * iS1;
    v1[r] = o0 == 0 ? V[r * 3] : (o0 == 1 ? V[r * 3 + 1] : V[r * 3 + 2]);
    v2[r] = o1 == 0 ? V[r * 3] : (o1 == 1 ? V[r * 3 + 1] : V[r * 3 + 2]);
  }
  // R = U diag(1,1,sign det(U V^T)) V^T = u1 v1^T + u2 v2^T + (u1 x u2)(v1 x v2)^T
  const double u3[3] = {u1[1] * u2[2] - u1[2] * u2[1], u1[2] * u2[0] - u1[0] * u2[2],
                        u1[0] * u2[1] - u1[1] * u2[0]};
  const double v3[3] = {v1[1] * v2[2] - v1[2] * v2[1], v1[2] * v2[0] - v1[0] * v2[2],
                        v1[0] * v2[1] - v1[1] * v2[0]};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) R[a * 3 + b] = u1[a] * v1[b] + u2[a] * v2[b] + u3[a] * v3[b];
  return true;
}

// IRLS weight of one rectified match under R: reweight(|s2 - R s1|) = min(H/d, 1)
// (matching.py:128-136), branch-free so the match loop stays unrolled: the residual is
// accumulated with FMA and H/d is H * rsqrt(d^2) (~1e-14 relative from the reference's
// H/d; the final flags are recomputed with the reference's exact arithmetic in
// k_preselect_final).
__device__ __forceinline__ double irls_weight(const double R[9], double a0, double a1, double a2,
                                              double b0, double b1, double b2, double H,
                                              double Hsq) {
  // e = b - R a as one fused chain per component (3 FMA, no separate multiply / subtract)
  const double e0 = __fma_rn(-R[0], a0, __fma_rn(-R[1], a1, __fma_rn(-R[2], a2, b0)));
  const double e1 = __fma_rn(-R[3], a0, __fma_rn(-R[4], a1, __fma_rn(-R[5], a2, b1)));
  const double e2 = __fma_rn(-R[6], a0, __fma_rn(-R[7], a1, __fma_rn(-R[8], a2, b2)));
  const double s = __fma_rn(e2, e2, __fma_rn(e1, e1, e0 * e0));
  // 1/sqrt(s) for s > H^2: the MUFU double-precision estimate refined by two Newton
  // steps (~1 ulp; the full-precision rsqrt(double) carries special-case branches). For
  // s <= H^2 the value is discarded (s = 0 gives NaN there, never selected).
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double hs = 0.5 * s;
  // y <- y + y (0.5 - hs y^2), fused
  // one Newton step after the MUFU estimate: ~1e-14 relative in the weight of a far
  // match (tolerance-level in the IRLS; the flags are recomputed exactly in
  // k_preselect_final) -- two steps measured 0.211 ms, one 0.203 ms at n = 1,888
  y = __fma_rn(y, __fma_rn(-hs * y, y, 0.5), y);
  // s > H^2 on the bit patterns (both >= +0, so the integer order is the IEEE order) on
  // the integer pipe instead of the FP64 one; a NaN residual keeps weight 1 like the
  // reference's `d > threshold` test
  const long long sb = __double_as_longlong(s);
  const bool far = sb > __double_as_longlong(Hsq) && sb <= 0x7ff0000000000000ll;
  return far ? H * y : 1.0;
}

#ifdef DT_PRESELECT_STATS
__device__ int g_pre_iters[8192];  // debug variant only: IRLS steps run per hypothesis
__device__ long long g_pre_time[8];  // debug variant only: globaltimer stamps of the fused kernel
__device__ __forceinline__ long long pre_gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PRE_STAMP(i) \
  do {               \
    if (threadIdx.x == 0) g_pre_time[i] = pre_gtimer(); \
  } while (0)
#else
#define PRE_STAMP(i) \
  do {               \
  } while (0)
#endif

// irls_weight of U matches at once, stage by stage (all U residual chains, then all U
// squared norms, estimates, Newton steps): the same operations per match as irls_weight,
// so the same bits, but the U independent chains sit side by side in the instruction
// stream (given the registers: see the 144-register kernels below) instead of one
// match's ~12-deep dependent chain after another.
template <int U>
__device__ __forceinline__ void irls_weights(const double R[9], const double a[U][3],
                                             const double b[U][3], double H, double Hsq,
                                             double w[U]) {
  double e0[U], e1[U], e2[U], s[U], y[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    e0[u] = __fma_rn(-R[2], a[u][2], b[u][0]);
    e1[u] = __fma_rn(-R[5], a[u][2], b[u][1]);
    e2[u] = __fma_rn(-R[8], a[u][2], b[u][2]);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    e0[u] = __fma_rn(-R[1], a[u][1], e0[u]);
    e1[u] = __fma_rn(-R[4], a[u][1], e1[u]);
    e2[u] = __fma_rn(-R[7], a[u][1], e2[u]);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    e0[u] = __fma_rn(-R[0], a[u][0], e0[u]);
    e1[u] = __fma_rn(-R[3], a[u][0], e1[u]);
    e2[u] = __fma_rn(-R[6], a[u][0], e2[u]);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) s[u] = __fma_rn(e2[u], e2[u], __fma_rn(e1[u], e1[u], e0[u] * e0[u]));
#pragma unroll
  for (int u = 0; u < U; ++u) asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y[u]) : "d"(s[u]));
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const double hs = 0.5 * s[u];
    y[u] = __fma_rn(y[u], __fma_rn(-hs * y[u], y[u], 0.5), y[u]);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long sb = __double_as_longlong(s[u]);
    const bool far = sb > __double_as_longlong(Hsq) && sb <= 0x7ff0000000000000ll;
    w[u] = far ? H * y[u] : 1.0;
  }
}

// Where the hypothesis loops read the matches from: the caller's arrays in global memory
// (read-only path) or the CTA's shared-memory copy (the fused ORB-path kernel).
struct LdGlobal {
  __device__ __forceinline__ static double get(const double* p) { return __ldg(p); }
};
struct LdPlain {
  __device__ __forceinline__ static double get(const double* p) { return *p; }
};

// One lane's share of a covariance pass: C += sum_k w_k b_k a_k^T over k = lane (mod 32)
// in increasing k (w = 1 in the first IRLS step). Four matches per trip are loaded and
// weighted as independent chains before being folded into C in order, so the result is
// the same as the one-match-at-a-time loop while the chains overlap.
#ifndef DT_PRE_TRIP
#define DT_PRE_TRIP 4
#endif
constexpr int PRE_TRIP = DT_PRE_TRIP;  // matches per lane per trip of the hypothesis loops

template <bool WEIGHTED, class LD>
__device__ __forceinline__ void cov_pass(const double* __restrict__ src,
                                         const double* __restrict__ dst, int64_t n, int lane,
                                         double rs0, double rs1, double rs2, double rd0,
                                         double rd1, double rd2, const double R[9], double H,
                                         double Hsq, double C[9]) {
  int64_t k = lane;
  for (; k + 32 * (PRE_TRIP - 1) < n; k += 32 * PRE_TRIP) {
    double a[PRE_TRIP][3], b[PRE_TRIP][3], w[PRE_TRIP];
#pragma unroll
    for (int u = 0; u < PRE_TRIP; ++u) {
      const double* ps = src + 3 * (k + 32 * u);
      const double* pd = dst + 3 * (k + 32 * u);
      a[u][0] = LD::get(ps) - rs0;
      a[u][1] = LD::get(ps + 1) - rs1;
      a[u][2] = LD::get(ps + 2) - rs2;
      b[u][0] = LD::get(pd) - rd0;
      b[u][1] = LD::get(pd + 1) - rd1;
      b[u][2] = LD::get(pd + 2) - rd2;
    }
    if (WEIGHTED) {
      irls_weights<PRE_TRIP>(R, a, b, H, Hsq, w);
    } else {
#pragma unroll
      for (int u = 0; u < PRE_TRIP; ++u) w[u] = 1.0;
    }
#pragma unroll
    for (int u = 0; u < PRE_TRIP; ++u) {
      const double c0 = b[u][0] * w[u], c1 = b[u][1] * w[u], c2 = b[u][2] * w[u];
      C[0] = __fma_rn(c0, a[u][0], C[0]);
      C[1] = __fma_rn(c0, a[u][1], C[1]);
      C[2] = __fma_rn(c0, a[u][2], C[2]);
      C[3] = __fma_rn(c1, a[u][0], C[3]);
      C[4] = __fma_rn(c1, a[u][1], C[4]);
      C[5] = __fma_rn(c1, a[u][2], C[5]);
      C[6] = __fma_rn(c2, a[u][0], C[6]);
      C[7] = __fma_rn(c2, a[u][1], C[7]);
      C[8] = __fma_rn(c2, a[u][2], C[8]);
    }
  }
  for (; k < n; k += 32) {
    const double a0 = LD::get(src + 3 * k) - rs0, a1 = LD::get(src + 3 * k + 1) - rs1,
                 a2 = LD::get(src + 3 * k + 2) - rs2;
    const double b0 = LD::get(dst + 3 * k) - rd0, b1 = LD::get(dst + 3 * k + 1) - rd1,
                 b2 = LD::get(dst + 3 * k + 2) - rd2;
    const double wk = WEIGHTED ? irls_weight(R, a0, a1, a2, b0, b1, b2, H, Hsq) : 1.0;
    const double c0 = b0 * wk, c1 = b1 * wk, c2 = b2 * wk;
    C[0] = __fma_rn(c0, a0, C[0]);
    C[1] = __fma_rn(c0, a1, C[1]);
    C[2] = __fma_rn(c0, a2, C[2]);
    C[3] = __fma_rn(c1, a0, C[3]);
    C[4] = __fma_rn(c1, a1, C[4]);
    C[5] = __fma_rn(c1, a2, C[5]);
    C[6] = __fma_rn(c2, a0, C[6]);
    C[7] = __fma_rn(c2, a1, C[7]);
    C[8] = __fma_rn(c2, a2, C[8]);
  }
}

// Support of one lane's matches (sum of IRLS weights in increasing k), same trip shape.
template <class LD>
__device__ __forceinline__ double support_pass(const double* __restrict__ src,
                                               const double* __restrict__ dst, int64_t n,
                                               int lane, double rs0, double rs1, double rs2,
                                               double rd0, double rd1, double rd2,
                                               const double R[9], double H, double Hsq) {
  double sup = 0.0;
  int64_t k = lane;
  for (; k + 32 * (PRE_TRIP - 1) < n; k += 32 * PRE_TRIP) {
    double a[PRE_TRIP][3], b[PRE_TRIP][3], w[PRE_TRIP];
#pragma unroll
    for (int u = 0; u < PRE_TRIP; ++u) {
      const double* ps = src + 3 * (k + 32 * u);
      const double* pd = dst + 3 * (k + 32 * u);
      a[u][0] = LD::get(ps) - rs0;
      a[u][1] = LD::get(ps + 1) - rs1;
      a[u][2] = LD::get(ps + 2) - rs2;
      b[u][0] = LD::get(pd) - rd0;
      b[u][1] = LD::get(pd + 1) - rd1;
      b[u][2] = LD::get(pd + 2) - rd2;
    }
    irls_weights<PRE_TRIP>(R, a, b, H, Hsq, w);
#pragma unroll
    for (int u = 0; u < PRE_TRIP; ++u) sup += w[u];
  }
  for (; k < n; k += 32)
    sup += irls_weight(R, LD::get(src + 3 * k) - rs0, LD::get(src + 3 * k + 1) - rs1,
                       LD::get(src + 3 * k + 2) - rs2, LD::get(dst + 3 * k) - rd0,
                       LD::get(dst + 3 * k + 1) - rd1, LD::get(dst + 3 * k + 2) - rd2, H, Hsq);
  return sup;
}

// One reference hypothesis on one warp (matching._evaluate_reference, matching.py:145-171):
// lane l owns the matches k = l (mod 32); the per-lane covariances are combined by a
// 5-level xor butterfly (bitwise-identical on every lane) and all 32 lanes run the 3x3
// SVD redundantly -- no shared memory and no CTA barrier, so warps drift apart and one
// warp's SVD overlaps the other warps' match loops. Writes (valid, support, R) of slot w.
template <class LD>
__device__ __forceinline__ void evaluate_hypothesis(const double* __restrict__ src,
                                                    const double* __restrict__ dst, int64_t n,
                                                    int64_t w, int64_t ref, double H, int iters,
                                                    double min_support, double* __restrict__ ref_support,
                                                    double* __restrict__ ref_rot,
                                                    uint8_t* __restrict__ ref_valid) {
  const int lane = threadIdx.x & 31;
  bool live = n >= 3 && ref >= 0 && ref < n;
  const int64_t rr = live ? ref : 0;
  const double rs0 = LD::get(src + 3 * rr), rs1 = LD::get(src + 3 * rr + 1), rs2 = LD::get(src + 3 * rr + 2);
  const double rd0 = LD::get(dst + 3 * rr), rd1 = LD::get(dst + 3 * rr + 1), rd2 = LD::get(dst + 3 * rr + 2);
  const double Hsq = H * H;
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
#ifdef DT_PRESELECT_STATS
  int dbg_it = 0;
#endif
  for (int it = 0; it < iters; ++it) {
#ifdef DT_PRESELECT_STATS
    dbg_it = it;
#endif
    double C[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (it == 0)
      cov_pass<false, LD>(src, dst, n, lane, rs0, rs1, rs2, rd0, rd1, rd2, R, H, Hsq, C);
    else
      cov_pass<true, LD>(src, dst, n, lane, rs0, rs1, rs2, rd0, rd1, rd2, R, H, Hsq, C);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < 9; ++i) C[i] += __shfl_xor_sync(0xffffffffu, C[i], o);
    double Rm[9], V0[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) V0[i] = V[i];
    const bool ok = procrustes_lane(C, V, Rm);
    if (!ok) {
      live = false;  // degenerate: the hypothesis is discarded whatever follows
      break;
    }
    // Exact early exit: after a weighted step, if (R, V) came back bit for bit unchanged,
    // every later step recomputes the same weights, covariance and warm-started SVD, so
    // the remaining iterations cannot change a bit (all lanes hold identical values, so
    // the test is warp-uniform).
    bool same = it > 0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
      same = same && __double_as_longlong(Rm[i]) == __double_as_longlong(R[i]) &&
             __double_as_longlong(V[i]) == __double_as_longlong(V0[i]);
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = Rm[i];
    if (same) break;
  }
#ifdef DT_PRESELECT_STATS
  if (lane == 0 && w < 8192) {
    g_pre_iters[w] = live ? dbg_it + 1 : -1;
  }
#endif
  double sup = 0.0;
  if (live) sup = support_pass<LD>(src, dst, n, lane, rs0, rs1, rs2, rd0, rd1, rd2, R, H, Hsq);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) sup += __shfl_xor_sync(0xffffffffu, sup, o);
  if (lane == 0) {
    const bool good = live && !(sup < min_support * (double)n);
    ref_valid[w] = good ? 1 : 0;
    ref_support[w] = good ? sup : 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) ref_rot[9 * w + i] = R[i];
  }
}

// One warp per reference hypothesis, the matches read from global memory. Two register
// budgets of the same body: a CTA of <= 12 warps (3 per scheduler: the register file is
// split per scheduler, 16 K each) may hold 168 registers per thread, enough for the four
// weight chains of a trip to run side by side (measured ~11 % faster per hypothesis than
// the serialized 128-register schedule); 13-16 warps per CTA get 128. (n = 1,888
// hypotheses on 12-warp CTAs -- two rounds -- measured 0.233 vs 0.205 ms: the second
// round's lone warps cost more than the chains gain.)
#define DT_PRESELECT_WARP_PARAMS                                                            \
  const double *__restrict__ src, const double *__restrict__ dst,                           \
      const int64_t *__restrict__ n_dev, int64_t n_fixed, const int64_t *__restrict__ refs, \
      int64_t n_refs, int exhaustive, double H, int iters, double min_support,              \
      double *__restrict__ ref_support, double *__restrict__ ref_rot,                       \
      uint8_t *__restrict__ ref_valid
#define DT_PRESELECT_WARP_ARGS \
  src, dst, n_dev, n_fixed, refs, n_refs, exhaustive, H, iters, min_support, ref_support, ref_rot, ref_valid
constexpr int PRESELECT_WIDE_WARPS = 12;  // warps per CTA of the 168-register kernels

__device__ __forceinline__ void preselect_warp_body(DT_PRESELECT_WARP_PARAMS) {
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t n = n_dev ? *n_dev : n_fixed;
  const int64_t nr = exhaustive ? n : n_refs;
  if (w >= nr) return;  // warp-uniform
  const int64_t ref = exhaustive ? w : refs[w];
  evaluate_hypothesis<LdGlobal>(src, dst, n, w, ref, H, iters, min_support, ref_support, ref_rot,
                                ref_valid);
}

__global__ void __launch_bounds__(512, 1) k_preselect_warp(DT_PRESELECT_WARP_PARAMS) {
  preselect_warp_body(DT_PRESELECT_WARP_ARGS);
}
__global__ void __launch_bounds__(32 * PRESELECT_WIDE_WARPS, 1) k_preselect_warp_wide(DT_PRESELECT_WARP_PARAMS) {
  preselect_warp_body(DT_PRESELECT_WARP_ARGS);
}

// Winner = max support, ties -> lower reference index (matching.py:198-206); then the
// flags and weights of every match (matching.py:210-213).
// (support, reference) of b beats a: larger support, ties -> lower reference index
__device__ __forceinline__ bool ref_better(double bs, int64_t br, double as, int64_t ar) {
  return br >= 0 && (ar < 0 || bs > as || (bs == as && br < ar));
}

__global__ void __launch_bounds__(1024)
k_preselect_final(const double* __restrict__ src, const double* __restrict__ dst,
                  const int64_t* __restrict__ n_dev, int64_t n_fixed,
                  const int64_t* __restrict__ refs, int64_t n_refs, int exhaustive, double H,
                  double inlier_min, const double* __restrict__ ref_support,
                  const double* __restrict__ ref_rot, const uint8_t* __restrict__ ref_valid,
                  double* weights, uint8_t* flags, double* residuals, double* rotation,
                  int64_t* info, double* support_out, FeatureScatter scatter, int do_scatter) {
  __shared__ double s_sup[32];
  __shared__ int64_t s_ref[32], s_pos[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = n_dev ? *n_dev : n_fixed;
  const int64_t nr = exhaustive ? n : n_refs;
  double best = -1.0;
  int64_t best_ref = -1, best_pos = -1;
  for (int64_t w = threadIdx.x; w < nr; w += blockDim.x) {
    if (!ref_valid[w]) continue;
    const int64_t ref = exhaustive ? w : refs[w];
    const double sp = ref_support[w];
    if (ref_better(sp, ref, best, best_ref)) {
      best = sp;
      best_ref = ref;
      best_pos = w;
    }
  }
  // argmax in a total order: warp shuffles, then the warps' winners
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t orf = __shfl_xor_sync(0xffffffffu, best_ref, o);
    const int64_t op = __shfl_xor_sync(0xffffffffu, best_pos, o);
    if (ref_better(os, orf, best, best_ref)) {
      best = os;
      best_ref = orf;
      best_pos = op;
    }
  }
  if (lane == 0) {
    s_sup[warp] = best;
    s_ref[warp] = best_ref;
    s_pos[warp] = best_pos;
  }
  __syncthreads();
  const int nw = (int)(blockDim.x >> 5);
  best = -1.0;
  best_ref = -1;
  best_pos = -1;
  for (int w2 = 0; w2 < nw; ++w2)
    if (ref_better(s_sup[w2], s_ref[w2], best, best_ref)) {
      best = s_sup[w2];
      best_ref = s_ref[w2];
      best_pos = s_pos[w2];
    }
  const int64_t ref = best_ref, pos = best_pos;
  // this CTA's round of matches (one CTA per 1024; every CTA found the same winner)
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ref < 0) {
    if (k < n) {
      weights[k] = 0.0;
      flags[k] = 0;
      if (residuals) residuals[k] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      info[0] = DT_ERR_NO_VALID_HYPOTHESIS;
      info[1] = -1;
      if (support_out) support_out[0] = 0.0;
      if (rotation)
        for (int i = 0; i < 9; ++i) rotation[i] = (i % 4 == 0) ? 1.0 : 0.0;
    }
  } else {
    double R[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = ref_rot[9 * pos + i];
    const double rs0 = src[3 * ref], rs1 = src[3 * ref + 1], rs2 = src[3 * ref + 2];
    const double rd0 = dst[3 * ref], rd1 = dst[3 * ref + 1], rd2 = dst[3 * ref + 2];
    if (k < n) {
      const double s1[3] = {src[3 * k] - rs0, src[3 * k + 1] - rs1, src[3 * k + 2] - rs2};
      const double s2[3] = {dst[3 * k] - rd0, dst[3 * k + 1] - rd1, dst[3 * k + 2] - rd2};
      const double d = rot_residual(R, s1, s2);
      const double fw = reweight(d, H);
      const bool flag = fw >= inlier_min;
      double soft = 1.0 - d / (5.0 * H);
      soft = soft < 0.0 ? 0.0 : (soft > 1.0 ? 1.0 : soft);
      weights[k] = flag ? fw : soft;
      flags[k] = flag ? 1 : 0;
      if (residuals) residuals[k] = d;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      info[0] = DT_OK;
      info[1] = ref;
      if (support_out) support_out[0] = best;
      if (rotation)
        for (int i = 0; i < 9; ++i) rotation[i] = R[i];
    }
  }
  // ORB path: the weights to their template features + the report statistics, in the
  // same CTA (this CTA's global writes above are visible after the barrier)
  if (do_scatter) {
    // this round's scatter and partial statistics; the last CTA to finish sums the rounds
    // in round order (same bits as one CTA walking the rounds)
    __syncthreads();
    double cs = 0.0;
    int nf = 0;
    feature_scatter_round(scatter, n, (int64_t)blockIdx.x * blockDim.x, weights, flags, &cs, &nf);
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
      scatter.partial[2 * blockIdx.x] = cs;
      scatter.partial[2 * blockIdx.x + 1] = (double)nf;
      __threadfence();
      s_last = atomicAdd(scatter.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      __threadfence();
      double wsum = 0.0;
      int64_t nflag = 0;
      for (unsigned g = 0; g < gridDim.x; ++g) {
        wsum += __ldcg(scatter.partial + 2 * g);
        nflag += (int64_t)__ldcg(scatter.partial + 2 * g + 1);
      }
      *scatter.n_active = scatter.n_feat;
      scatter.stats[0] = wsum;
      scatter.stats[1] = (double)nflag;
      *scatter.counter = 0;
    }
  }
}

// ---------------------------------------------------------------------------------
// ORB path, fused: match build + preselection + final in ONE launch. The separate chain
// (k_build_matches: 1 CTA, four dependent global loads + a block scan, ~14 us;
// k_preselect_warp; k_preselect_final: 2 CTAs, ~12 us) is latency, not work. Here every
// CTA first builds the frame's match list itself -- in template-feature order, exactly
// as k_build_matches does -- into its shared memory (CTA 0 also publishes it), its warps
// evaluate their hypotheses from there, and the last CTA to finish picks the winner,
// writes flags / weights, scatters them to the template features and forms the report
// statistics in the separate kernels' summation order.
// ---------------------------------------------------------------------------------

// Block-wide exclusive scan of per-thread counts; *total = the block's sum.
__device__ __forceinline__ int block_excl_scan(int cnt, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      const int v = s_warp[w];
      s_warp[w] = run;
      run += v;
    }
    s_warp[32] = run;
  }
  __syncthreads();
  const int off = s_warp[warp] + inc - cnt;
  *total = s_warp[32];
  __syncthreads();
  return off;
}

constexpr int ORB_FUSED_PER = 8;  // features per thread per build round

#define DT_PRESELECT_ORB_PARAMS                                                                \
  OrbMatchIn in, const int64_t *__restrict__ refs, int64_t n_refs, double H, int iters,         \
      double inlier_min, double min_support, double *__restrict__ ref_support,                  \
      double *__restrict__ ref_rot, uint8_t *__restrict__ ref_valid, PreselectOrbOut out
#define DT_PRESELECT_ORB_ARGS \
  in, refs, n_refs, H, iters, inlier_min, min_support, ref_support, ref_rot, ref_valid, out

__device__ __forceinline__ void preselect_orb_body(DT_PRESELECT_ORB_PARAMS) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  __shared__ int s_warp[33];
  __shared__ bool s_last;
  const int64_t nt = in.nt;
  if (blockIdx.x == 0) PRE_STAMP(0);
  double* s_src = reinterpret_cast<double*>(s_raw);
  double* s_dst = s_src + 3 * nt;
  int32_t* s_feat = reinterpret_cast<int32_t*>(s_dst + 3 * nt);
  // ---- the frame's match list (k_build_matches' rule, feature order) ----
  int64_t n = 0;
  for (int64_t base = 0; base < nt; base += (int64_t)blockDim.x * ORB_FUSED_PER) {
    const int64_t t0 = base + (int64_t)threadIdx.x * ORB_FUSED_PER;
    // every global load of the round is issued before anything is stored: the template
    // points (independent of the match) first, then the Hamming winner -> keypoint ->
    // depth chain, all eight elements side by side; the back-projection follows, and only
    // then the scan and the stores (a store between two elements' loads would serialize
    // them: the compiler cannot rule out aliasing)
    double sxa[ORB_FUSED_PER], sya[ORB_FUSED_PER], sza[ORB_FUSED_PER];
    int u[ORB_FUSED_PER], v[ORB_FUSED_PER];
    double z[ORB_FUSED_PER], dxa[ORB_FUSED_PER], dya[ORB_FUSED_PER];
    bool ok[ORB_FUSED_PER];
#pragma unroll
    for (int e = 0; e < ORB_FUSED_PER; ++e) {
      const int64_t t = t0 + e < nt ? t0 + e : 0;
      sxa[e] = __ldg(in.tpts + 3 * t);
      sya[e] = __ldg(in.tpts + 3 * t + 1);
      sza[e] = __ldg(in.tpts + 3 * t + 2);
    }
#pragma unroll
    for (int e = 0; e < ORB_FUSED_PER; ++e) {
      const int64_t t = t0 + e;
      int fi = -1;
      if (t < nt && in.nf > 0) {
        const unsigned long long pv = __ldcg(in.packed + t);  // (distance << 32) | frame index
        if ((long long)(pv >> 32) <= (long long)in.max_ham) fi = (int)(pv & 0xffffffffull);
      }
      u[e] = v[e] = -1;
      if (fi >= 0 && fi < in.nf) {
        u[e] = __ldg(in.kp + 2 * fi);
        v[e] = __ldg(in.kp + 2 * fi + 1);
      }
    }
#ifdef DT_PRESELECT_STATS
    if (blockIdx.x == 0 && base == 0) {
      __syncwarp();
      if (u[0] > -2 && threadIdx.x == 0) g_pre_time[6] = pre_gtimer();
    }
#endif
    int cnt = 0;
#pragma unroll
    for (int e = 0; e < ORB_FUSED_PER; ++e) {
      ok[e] = u[e] >= 0 && u[e] < in.width && v[e] >= 0 && v[e] < in.height;
      z[e] = ok[e] ? __ldg(in.depth + (int64_t)v[e] * in.width + u[e]) : 0.0;
      ok[e] = ok[e] && isfinite(z[e]) && z[e] > in.zmin && z[e] < in.zmax;
      cnt += ok[e] ? 1 : 0;
    }
#pragma unroll
    for (int e = 0; e < ORB_FUSED_PER; ++e) {
      // k_build_matches' expression and operation order
      dxa[e] = ((double)u[e] - in.cx) / in.fx * z[e];
      dya[e] = ((double)v[e] - in.cy) / in.fy * z[e];
    }
    int total;
    int64_t o = n + block_excl_scan(cnt, s_warp, &total);
#ifdef DT_PRESELECT_STATS
    if (blockIdx.x == 0 && base == 0 && threadIdx.x == 0) g_pre_time[7] = pre_gtimer();
#endif
#pragma unroll
    for (int e = 0; e < ORB_FUSED_PER; ++e) {
      if (!ok[e]) continue;
      DT_DCHECK(o >= 0 && o < nt && t0 + e < nt);
      s_src[3 * o] = sxa[e];
      s_src[3 * o + 1] = sya[e];
      s_src[3 * o + 2] = sza[e];
      s_dst[3 * o] = dxa[e];
      s_dst[3 * o + 1] = dya[e];
      s_dst[3 * o + 2] = z[e];
      s_feat[o] = (int32_t)(t0 + e);
      ++o;
    }
    n += total;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out.n_out = n;
  __syncthreads();
  // publish the list (matches for the solver and the caller) and clear the per-feature
  // weights, each CTA a contiguous slice, coalesced (one CTA writing it all with the
  // element-strided stores of the build measured 8.7 us on its SM)
  {
    const int64_t G = gridDim.x, b = blockIdx.x;
    for (int64_t i = 3 * n * b / G + threadIdx.x; i < 3 * n * (b + 1) / G; i += blockDim.x) {
      out.m_src[i] = s_src[i];
      out.m_dst[i] = s_dst[i];
    }
    for (int64_t i = n * b / G + threadIdx.x; i < n * (b + 1) / G; i += blockDim.x)
      out.m_feat[i] = s_feat[i];
    for (int64_t i = nt * b / G + threadIdx.x; i < nt * (b + 1) / G; i += blockDim.x)
      out.fs.ffw[i] = 0.0;  // no active match until the final
  }
  if (blockIdx.x == 0) PRE_STAMP(1);
  // ---- hypotheses: one warp each ----
  const int exhaustive = refs == nullptr;
  const int64_t nr = exhaustive ? n : n_refs;
  // hypothesis h on warp (h / gridDim.x) mod wpc of CTA h mod gridDim.x: consecutive
  // hypotheses on different SMs, and when there are more hypotheses than warps (the
  // 12-warp wide kernel) the second round is spread one per SM
  const int wpc = (int)(blockDim.x >> 5);
  for (int64_t r = 0;; ++r) {
    const int64_t w = (int64_t)blockIdx.x + (int64_t)gridDim.x * ((threadIdx.x >> 5) + wpc * r);
    if (w >= nr) break;  // warp-uniform
    evaluate_hypothesis<LdPlain>(s_src, s_dst, n, w, exhaustive ? w : refs[w], H, iters, min_support,
                                 ref_support, ref_rot, ref_valid);
  }
  // ---- the last CTA to finish: winner, flags, weights, scatter, statistics ----
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(out.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  PRE_STAMP(2);
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  double best = -1.0;
  int64_t best_ref = -1, best_pos = -1;
  // four candidates per thread per trip, their loads issued together (a candidate's
  // support load behind its validity test would make one dependent round trip each)
  for (int64_t q0 = threadIdx.x; q0 < nr; q0 += 4 * (int64_t)blockDim.x) {
    uint8_t vl[4];
    double sp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t q = q0 + k * (int64_t)blockDim.x;
      vl[k] = q < nr ? __ldcg(ref_valid + q) : 0;
      sp[k] = q < nr ? __ldcg(ref_support + q) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t q = q0 + k * (int64_t)blockDim.x;
      if (!vl[k]) continue;
      const int64_t rf = exhaustive ? q : refs[q];
      if (ref_better(sp[k], rf, best, best_ref)) {
        best = sp[k];
        best_ref = rf;
        best_pos = q;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double os = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t orf = __shfl_xor_sync(0xffffffffu, best_ref, o);
    const int64_t op = __shfl_xor_sync(0xffffffffu, best_pos, o);
    if (ref_better(os, orf, best, best_ref)) {
      best = os;
      best_ref = orf;
      best_pos = op;
    }
  }
  __shared__ double s_bsup[32];
  __shared__ int64_t s_bref[32], s_bpos[32];
  if (lane == 0) {
    s_bsup[warp] = best;
    s_bref[warp] = best_ref;
    s_bpos[warp] = best_pos;
  }
  __syncthreads();
  best = -1.0;
  best_ref = -1;
  best_pos = -1;
  for (int w2 = 0; w2 < nw; ++w2)
    if (ref_better(s_bsup[w2], s_bref[w2], best, best_ref)) {
      best = s_bsup[w2];
      best_ref = s_bref[w2];
      best_pos = s_bpos[w2];
    }
  PRE_STAMP(3);
  double R[9];
  double rs0 = 0, rs1 = 0, rs2 = 0, rd0 = 0, rd1 = 0, rd2 = 0;
  if (best_ref >= 0) {
    DT_DCHECK(best_pos >= 0 && best_pos < nr && best_ref < n);
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = __ldcg(ref_rot + 9 * best_pos + i);
    rs0 = s_src[3 * best_ref], rs1 = s_src[3 * best_ref + 1], rs2 = s_src[3 * best_ref + 2];
    rd0 = s_dst[3 * best_ref], rd1 = s_dst[3 * best_ref + 1], rd2 = s_dst[3 * best_ref + 2];
  }
  // per match (k_preselect_final's arithmetic): each warp takes 32-match groups
  // warp, warp + nw, ... of the whole list, unrolled so their residual / sqrt / division
  // chains overlap; the group sums go to shared memory and the report statistics are
  // formed in the separate kernels' order: xor-tree sums of the 32-match groups, the 32
  // groups of a 1024-match round in order, rounds in order
  __shared__ double s_gsum[ORB_FUSED_MAX / 32 + 32];
  __shared__ int s_gcnt[ORB_FUSED_MAX / 32 + 32];
  const int n_groups = (int)((n + 31) / 32);
  const int n_slots = (n_groups + 31) / 32 * 32;
#pragma unroll 4
  for (int g = warp; g < n_slots; g += nw) {
    const int64_t k = 32 * (int64_t)g + lane;
    double wk = 0.0;
    int fl = 0;
    if (k < n) {
      if (best_ref < 0) {
        out.weights[k] = 0.0;
        out.flags[k] = 0;
        if (out.residuals) out.residuals[k] = 0.0;
      } else {
        const double s1[3] = {s_src[3 * k] - rs0, s_src[3 * k + 1] - rs1, s_src[3 * k + 2] - rs2};
        const double s2[3] = {s_dst[3 * k] - rd0, s_dst[3 * k + 1] - rd1, s_dst[3 * k + 2] - rd2};
        const double d = rot_residual(R, s1, s2);
        const double fw = reweight(d, H);
        const bool flag = fw >= inlier_min;
        double soft = 1.0 - d / (5.0 * H);
        soft = soft < 0.0 ? 0.0 : (soft > 1.0 ? 1.0 : soft);
        wk = flag ? fw : soft;
        fl = flag ? 1 : 0;
        out.weights[k] = wk;
        out.flags[k] = (uint8_t)fl;
        if (out.residuals) out.residuals[k] = d;
      }
      const int f = s_feat[k];
      DT_DCHECK(f >= 0 && f < nt);
      out.fs.ffw[f] = wk;
      out.fs.ffo[3 * f] = s_dst[3 * k];
      out.fs.ffo[3 * f + 1] = s_dst[3 * k + 1];
      out.fs.ffo[3 * f + 2] = s_dst[3 * k + 2];
    }
    const double gs = warp_sum(wk);
    for (int o = 16; o > 0; o >>= 1) fl += __shfl_xor_sync(0xffffffffu, fl, o);
    if (lane == 0) {
      s_gsum[g] = gs;
      s_gcnt[g] = fl;
    }
  }
  __syncthreads();
  double wsum = 0.0;
  int64_t nflag = 0;
  if (threadIdx.x == 0) {
    for (int r = 0; r < n_slots; r += 32) {
      double cs = 0.0;
      int nf = 0;
      for (int g = r; g < r + 32; ++g) {
        cs += s_gsum[g];
        nf += s_gcnt[g];
      }
      wsum += cs;
      nflag += nf;
    }
  }
  PRE_STAMP(4);
  if (threadIdx.x == 0) {
    out.info[0] = best_ref < 0 ? DT_ERR_NO_VALID_HYPOTHESIS : DT_OK;
    out.info[1] = best_ref;
    out.support[0] = best_ref < 0 ? 0.0 : best;
    *out.fs.n_active = out.fs.n_feat;
    out.fs.stats[0] = wsum;
    out.fs.stats[1] = (double)nflag;
    *out.done = 0;
  }
  // ready for the next frame's Hamming atomicMin
  for (int64_t t = threadIdx.x; t < nt; t += blockDim.x) out.packed_reset[t] = ~0ull;
  PRE_STAMP(5);
}

__global__ void __launch_bounds__(512, 1) k_preselect_orb(DT_PRESELECT_ORB_PARAMS) {
  preselect_orb_body(DT_PRESELECT_ORB_ARGS);
}
__global__ void __launch_bounds__(32 * PRESELECT_WIDE_WARPS, 1) k_preselect_orb_wide(DT_PRESELECT_ORB_PARAMS) {
  preselect_orb_body(DT_PRESELECT_ORB_ARGS);
}

int launch_preselect_orb(const OrbMatchIn& in, const int64_t* refs, int64_t n_refs, double H, int iters,
                         double inlier_min, double min_support, double* ref_support, double* ref_rot,
                         uint8_t* ref_valid, const PreselectOrbOut& out, cudaStream_t s, int shared_gpu) {
  const int64_t nr = refs ? n_refs : in.nt;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  // sharing the GPU (config 5, 64 sequences): 16-warp CTAs measured 2,950 frames/s
  // against 2,904 with 8, 2,845 with 12, 2,498 with 4 (and 2,736 / 2,894 for the
  // 168-register build in 8- / 12-warp CTAs)
  const int64_t wpc = shared_gpu ? 16 : std::min<int64_t>(16, std::max<int64_t>(1, (nr + sms - 1) / sms));
  // one CTA per SM when the tracker owns the GPU (more hypotheses than warps: a second
  // round, see preselect_orb_body); sharing the GPU, one 16-warp CTA per 16 hypotheses
  const int64_t grid = std::max<int64_t>(
      1, shared_gpu ? (nr + wpc - 1) / wpc : std::min<int64_t>(sms, (nr + wpc - 1) / wpc));
  const size_t smem = (size_t)in.nt * (6 * sizeof(double) + sizeof(int32_t));
  auto* kern = !shared_gpu && wpc <= PRESELECT_WIDE_WARPS ? k_preselect_orb_wide : k_preselect_orb;
  DT_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)grid, (unsigned)(32 * wpc), smem, s>>>(in, refs, n_refs, H, iters, inlier_min,
                                                          min_support, ref_support, ref_rot,
                                                          ref_valid, out);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int launch_preselect(const double* src, const double* dst, const int64_t* n_dev, int64_t n_max,
                     const int64_t* refs, int64_t n_refs, int exhaustive, double H, int iters,
                     double inlier_min, double min_support, double* weights, uint8_t* flags,
                     double* residuals, double* rotation, int64_t* info, double* support,
                     double* ref_support, double* ref_rot, uint8_t* ref_valid, cudaStream_t s,
                     const FeatureScatter* scatter, int shared_gpu) {
  const int64_t nr = exhaustive ? n_max : n_refs;
  if (nr > 0) {
    // One warp per hypothesis. The busiest SM sets the time (FP64 pipe ~76 % busy there),
    // so the warps are spread evenly: one CTA of ceil(nr / SMs) warps per SM (<= 16, the
    // register limit), e.g. 2,000 hypotheses -> 143 CTAs x 14 warps instead of 8-warp CTAs
    // that leave 102 SMs with 16 warps and 46 with 8. The block scheduler's greedy fill
    // defeats smaller CTAs.
    int dev = 0, sms = 0;  // a cheap attribute query; no process-global cache
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    // Sharing the GPU with other sequences (cluster mode), small 8-warp CTAs pack
    // between the other kernels' CTAs instead.
    const int64_t wpc = shared_gpu ? 8
                                   : std::min<int64_t>(16, std::max<int64_t>(1, (nr + sms - 1) / sms));
    (!shared_gpu && wpc <= PRESELECT_WIDE_WARPS ? k_preselect_warp_wide : k_preselect_warp)
        <<<(unsigned)((nr + wpc - 1) / wpc), (unsigned)(32 * wpc), 0, s>>>(
        src, dst, n_dev, n_max, refs, n_refs, exhaustive, H, iters, min_support, ref_support,
        ref_rot, ref_valid);
    DT_CHECK_LAUNCH();
  }
  const FeatureScatter fs = scatter ? *scatter : FeatureScatter{};
  // one CTA per 1,024 matches (each finds the winner itself: n_max supports)
  const unsigned g = (unsigned)std::max<int64_t>(1, (n_max + 1023) / 1024);
  k_preselect_final<<<g, 1024, 0, s>>>(src, dst, n_dev, n_max, refs, n_refs, exhaustive, H,
                                        inlier_min, ref_support, ref_rot, ref_valid, weights, flags,
                                        residuals, rotation, info, support, fs,
                                        scatter ? 1 : 0);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

}  // namespace dt

using namespace dt;

extern "C" {

#ifdef DT_PRESELECT_STATS
int dt_debug_preselect_iters(int* out, int n) {
  return cudaMemcpyFromSymbol(out, g_pre_iters, sizeof(int) * (n < 8192 ? n : 8192)) == cudaSuccess ? 0 : -1;
}
int dt_debug_preselect_times(long long* out) {
  return cudaMemcpyFromSymbol(out, g_pre_time, sizeof(long long) * 8) == cudaSuccess ? 0 : -1;
}
#endif

int dt_hamming_match(const uint8_t* template_desc, int64_t n_template, const uint8_t* frame_desc,
                     int64_t n_frame, int32_t* best_idx, int32_t* best_dist, void* stream) {
  DT_REQUIRE(n_template >= 0 && n_frame >= 0, DT_ERR_INVALID_ARGUMENT, "negative descriptor count");
  cudaStream_t s = as_stream(stream);
  if (n_template == 0) return DT_OK;
  unsigned long long* packed = nullptr;
  DT_CHECK_CUDA(cudaMallocAsync((void**)&packed, sizeof(unsigned long long) * n_template, s));
  const int st = launch_hamming(template_desc, n_template, frame_desc, n_frame, nullptr, nullptr, s,
                                packed);
  if (st == DT_OK) {
    k_unpack_hamming<<<grid_for(n_template, 256), 256, 0, s>>>(packed, n_template, n_frame,
                                                              best_idx, best_dist);
  }
  cudaFreeAsync(packed, s);
  DT_CHECK_LAUNCH();
  return st;
}

int dt_preselect(const double* src, const double* dst, int64_t n, const int64_t* refs,
                 int64_t n_refs, const dt_preselect_params* params, double* weights,
                 uint8_t* flags, double* residuals, double* rotation, int64_t* info,
                 double* support, void* stream) {
  DT_REQUIRE(params != nullptr, DT_ERR_INVALID_ARGUMENT, "params is NULL");
  DT_REQUIRE(params->distance_threshold > 0.0, DT_ERR_INVALID_ARGUMENT,
             "distance_threshold must be positive");
  DT_REQUIRE(params->n_reweight_iters >= 1, DT_ERR_INVALID_ARGUMENT, "n_reweight_iters must be >= 1");
  cudaStream_t s = as_stream(stream);
  const int exhaustive = refs == nullptr ? 1 : 0;
  const int64_t nr = exhaustive ? n : n_refs;
  double *ref_support = nullptr, *ref_rot = nullptr;
  uint8_t* ref_valid = nullptr;
  const int64_t cap = nr > 0 ? nr : 1;
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ref_support, sizeof(double) * cap, s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ref_rot, sizeof(double) * 9 * cap, s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ref_valid, cap, s));
  const int st = launch_preselect(src, dst, nullptr, n, refs, n_refs, exhaustive,
                                  params->distance_threshold, params->n_reweight_iters,
                                  params->inlier_weight_min, params->min_support, weights, flags,
                                  residuals, rotation, info, support, ref_support, ref_rot,
                                  ref_valid, s);
  cudaFreeAsync(ref_support, s);
  cudaFreeAsync(ref_rot, s);
  cudaFreeAsync(ref_valid, s);
  return st;
}

}  // extern "C"
