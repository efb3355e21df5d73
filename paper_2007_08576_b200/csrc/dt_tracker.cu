// dt_tracker.cu -- device-resident tracker: one sequence, one stream.
//
// Per frame (tracking.track_frame, tracking.py:67-95):
//   depth -> normals + validity            k_observation_normals   (correspond.py:36-73)
//   [ORB] Hamming match + back-projection  k_hamming, k_build_matches (north-star 3a)
//   preselection (+ ORB feature scatter)   k_preselect_warp/final  (matching.py:174-226)
//   [pairs] binding, active matches, CSR   k_bind_points, k_active, k_csr_*_dev
//                                                                  (solver.py:113-119, 292-296)
//   LM solve                               k_solve_frame           (solver.py:267-378)
//   output warp                            in the solver's final phase (grid mode) or
//                                          k_warp_all_i32 (cluster mode) (warpfield.py:236-250)
// All launches go to the tracker's stream; the steady-state ORB frame replays as one CUDA
// graph; the host only waits at the end of the frame when it asked for host outputs.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "dt_common.cuh"
#include "dt_math.cuh"
#include "dt_ops.cuh"
#include "dt_solver.cuh"

namespace dt {

// ---------------------------------------------------------------------------------
// small device kernels of the frame pipeline
// ---------------------------------------------------------------------------------

__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }

// Block-wide exclusive scan of 0/1 flags for a 1024-thread CTA. Returns this thread's
// offset; *total receives the block count.
__device__ __forceinline__ int block_scan_flag(bool flag, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  const int in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) s_warp[warp] = __popc(bal);
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
  const int off = s_warp[warp] + in_warp;
  *total = s_warp[32];
  __syncthreads();
  return off;
}

// Block-wide exclusive scan of per-thread counts (1024-thread CTA, warp shuffles + one
// pass over the warp totals). Returns this thread's offset; *total = the block's sum.
__device__ __forceinline__ int block_scan_count(int cnt, int* s_warp, int* total) {
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

// ORB path: keep, in template-feature order, every feature whose best frame match passes
// the Hamming gate and lands on a valid depth pixel; the observed point is the keypoint
// back-projected through the frame's depth (geometry.back_project, geometry.py:387-396).
// Each thread owns BM_PER consecutive features per round, so every load of a round is in
// flight before the single block scan.
constexpr int BM_PER = 4;

__global__ void __launch_bounds__(1024)
k_build_matches(int64_t nt, unsigned long long* __restrict__ packed,
                int max_ham, const int32_t* __restrict__ kp, int64_t nf,
                const double* __restrict__ depth, double zmin, double zmax, int width,
                int height, double fx, double fy, double cx, double cy,
                const double* __restrict__ tpts, double* __restrict__ src,
                double* __restrict__ dst, int32_t* __restrict__ feat_id, int64_t* __restrict__ n_out,
                double* __restrict__ ffw) {
  __shared__ int s_warp[33];
  int64_t base_out = 0;
  for (int64_t base = 0; base < nt; base += (int64_t)blockDim.x * BM_PER) {
    const int64_t t0 = base + (int64_t)threadIdx.x * BM_PER;
    int fi[BM_PER], u[BM_PER], v[BM_PER];
    bool ok[BM_PER];
#pragma unroll
    for (int e = 0; e < BM_PER; ++e) {
      const int64_t t = t0 + e;
      fi[e] = -1;
      if (ffw && t < nt) ffw[t] = 0.0;  // features without an active match keep weight 0
      if (t < nt && nf > 0) {
        const unsigned long long v = packed[t];  // (distance << 32) | frame index
        packed[t] = ~0ull;                       // ready for the next frame's atomicMin
        if ((long long)(v >> 32) <= (long long)max_ham) fi[e] = (int)(v & 0xffffffffull);
      }
    }
#pragma unroll
    for (int e = 0; e < BM_PER; ++e) {
      u[e] = v[e] = -1;
      if (fi[e] >= 0 && fi[e] < nf) {
        u[e] = kp[2 * fi[e]];
        v[e] = kp[2 * fi[e] + 1];
      }
    }
    // the depth-validity test of the observation (correspond.valid_depth_mask,
    // correspond.py:23-26) evaluated here from the depth itself: the matching chain has
    // no dependency on the observation-normals kernel
    double z[BM_PER];
#pragma unroll
    for (int e = 0; e < BM_PER; ++e) {
      ok[e] = u[e] >= 0 && u[e] < width && v[e] >= 0 && v[e] < height;
      z[e] = ok[e] ? depth[(int64_t)v[e] * width + u[e]] : 0.0;
    }
    int cnt = 0;
#pragma unroll
    for (int e = 0; e < BM_PER; ++e) {
      ok[e] = ok[e] && isfinite(z[e]) && z[e] > zmin && z[e] < zmax;
      cnt += ok[e] ? 1 : 0;
    }
    int total;
    int64_t o = base_out + block_scan_count(cnt, s_warp, &total);
#pragma unroll
    for (int e = 0; e < BM_PER; ++e) {
      if (!ok[e]) continue;
      const int64_t t = t0 + e;
      const double d = z[e];
      src[3 * o] = tpts[3 * t];
      src[3 * o + 1] = tpts[3 * t + 1];
      src[3 * o + 2] = tpts[3 * t + 2];
      dst[3 * o] = ((double)u[e] - cx) / fx * d;
      dst[3 * o + 1] = ((double)v[e] - cy) / fy * d;
      dst[3 * o + 2] = d;
      feat_id[o] = (int32_t)t;
      ++o;
    }
    base_out += total;
  }
  if (threadIdx.x == 0) *n_out = base_out;
}

// Active matches (weights > 0, solver.py:113) in order, plus the report statistics
// n_preselected and match_weight_sum (solver.py:368-370), summed in a fixed order.
__global__ void __launch_bounds__(1024)
k_active(const int64_t* __restrict__ n_dev, const double* __restrict__ weights,
         const uint8_t* __restrict__ flags, const double* __restrict__ src,
         const double* __restrict__ dst, const int32_t* __restrict__ bidx,
         const double* __restrict__ bw, int k, int use, double* __restrict__ fp,
         double* __restrict__ fo, double* __restrict__ fwt, int32_t* __restrict__ fbidx,
         double* __restrict__ fbw, int64_t* __restrict__ n_active, double* __restrict__ stats) {
  __shared__ int s_warp[33];
  __shared__ double s_sum[32];
  const int64_t n = use ? *n_dev : 0;
  int64_t base_out = 0;
  double wsum = 0.0;
  int64_t nflag = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t j = base + threadIdx.x;
    const bool in = j < n;
    const double w = in ? weights[j] : 0.0;
    const bool act = in && w > 0.0;
    // fixed-order chunk sum of the weights
    double v = warp_sum(w);
    if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = v;
    int flg = (in && flags[j]) ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) flg += __shfl_xor_sync(0xffffffffu, flg, o);
    int total;
    const int off = block_scan_flag(act, s_warp, &total);
    if (threadIdx.x == 0) {
      double cs = 0.0;
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) cs += s_sum[w2];
      wsum += cs;
    }
    if (act) {
      const int64_t o = base_out + off;
      for (int i = 0; i < 3; ++i) {
        fp[3 * o + i] = src[3 * j + i];
        fo[3 * o + i] = dst[3 * j + i];
      }
      fwt[o] = w;
      for (int s = 0; s < k; ++s) {
        fbidx[o * k + s] = bidx[j * k + s];
        fbw[o * k + s] = bw[j * k + s];
      }
    }
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = flg;  // reuse after scan
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) nflag += s_warp[w2];
    __syncthreads();
    base_out += total;
  }
  if (threadIdx.x == 0) {
    *n_active = base_out;
    stats[0] = wsum;
    stats[1] = (double)nflag;
  }
}

// Control -> (match * k + slot) CSR over the active matches, count read on the device.
__global__ void k_csr_count_dev(const int32_t* __restrict__ keys, const int64_t* __restrict__ n_dev,
                                int k, int m, int* __restrict__ cnt) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= m) return;
  const int64_t ne = *n_dev * k;
  int total = 0;
  for (int64_t base = 0; base < ne; base += 32) {
    const int64_t e = base + lane;
    const bool hit = e < ne && keys[e] == warp;
    total += __popc(__ballot_sync(0xffffffffu, hit));
  }
  if (lane == 0) cnt[warp] = total;
}

__global__ void __launch_bounds__(1024) k_scan_counts(const int* __restrict__ cnt, int m, int* __restrict__ ptr) {
  __shared__ int s_part[1024];
  const int t = threadIdx.x;
  const int per = (m + blockDim.x - 1) / blockDim.x;
  const int lo = min(m, t * per), hi = min(m, lo + per);
  int s = 0;
  for (int i = lo; i < hi; ++i) s += cnt[i];
  s_part[t] = s;
  __syncthreads();
  if (t == 0) {
    int run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int v = s_part[i];
      s_part[i] = run;
      run += v;
    }
    ptr[m] = run;
  }
  __syncthreads();
  int run = s_part[t];
  for (int i = lo; i < hi; ++i) {
    ptr[i] = run;
    run += cnt[i];
  }
}

__global__ void k_csr_fill_dev(const int32_t* __restrict__ keys, const int64_t* __restrict__ n_dev,
                               int k, int m, const int* __restrict__ ptr, int* __restrict__ ent,
                               int* __restrict__ pos_of) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= m) return;
  const int64_t ne = *n_dev * k;
  int pos = ptr[warp];
  for (int64_t base = 0; base < ne; base += 32) {
    const int64_t e = base + lane;
    const bool hit = e < ne && keys[e] == warp;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const int q = pos + __popc(bal & ((1u << lane) - 1u));
      ent[q] = (int)e;
      pos_of[e] = q;
    }
    pos += __popc(bal);
  }
}

// Output warp as its own launch (cluster mode: a sequence's solver has only a few CTAs,
// so the full-GPU kernel finishes sooner than the solver's final phase would)
__global__ void k_warp_all_i32(const double* __restrict__ pts, const double* __restrict__ nrm,
                               const int32_t* __restrict__ bidx, const double* __restrict__ alpha,
                               int64_t n, int k, const double* __restrict__ warps, double* out_p,
                               double* out_n) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double B[8], sgn[KMAX];
  blend_at(warps, bidx + c * k, alpha + c * k, k, B, sgn);
  double x0, x1, x2, s2;
  apply_blend(B, pts[3 * c], pts[3 * c + 1], pts[3 * c + 2], x0, x1, x2, s2);
  double r0, r1, r2;
  rotate_normal(B, nrm[3 * c], nrm[3 * c + 1], nrm[3 * c + 2], r0, r1, r2);
  out_p[3 * c] = x0;
  out_p[3 * c + 1] = x1;
  out_p[3 * c + 2] = x2;
  out_n[3 * c] = r0;
  out_n[3 * c + 1] = r1;
  out_n[3 * c + 2] = r2;
}

int launch_warp_all_i32(const double* pts, const double* nrm, const int32_t* bidx,
                        const double* alpha, int64_t n, int k, const double* warps, double* out_p,
                        double* out_n, cudaStream_t s) {
  if (n == 0) return DT_OK;
  k_warp_all_i32<<<grid_for(n, 128), 128, 0, s>>>(pts, nrm, bidx, alpha, n, k, warps, out_p, out_n);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

}  // namespace dt

using namespace dt;

// ---------------------------------------------------------------------------------
// tracker state
// ---------------------------------------------------------------------------------

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool pooled = false;  // from the stream-ordered pool (cudaMallocAsync)
};

struct dt_tracker {
  dt_config cfg;
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n = 0, k = 0, m = 0, ne = 0;
  int cluster = 1;
  int grid_mode = 0;
  int launches = 0;
  bool args_dirty = false;
  bool profiling = false;
  long long* trace = nullptr;
  int trace_cap = 0;
  double* red = nullptr;     // last-arriver reduction slots
  unsigned* redc = nullptr;
  int red_g = 0;
  long long* arrivals = nullptr;  // 2 + 1024 * arr_cap per-CTA barrier arrival stamps
  int arr_cap = 0;
  bool last_used = false;
  cudaEvent_t ev[DT_N_PHASES + 1] = {};
  std::vector<DevBuf> bufs;
  // buffers replaced by a growing dalloc: freed at the next synchronising call (reap)
  std::vector<DevBuf> retired;
  // bumped by every allocation: a captured frame graph is only replayed while the
  // buffers it was captured with are still the live ones
  uint64_t buf_gen = 0;
  // template / graph
  double *tp = nullptr, *tn = nullptr, *bw = nullptr, *bws = nullptr, *cpts = nullptr, *ew = nullptr;
  int32_t *bidx = nullptr, *edges = nullptr;
  int *cptr = nullptr, *cent = nullptr, *iptr = nullptr, *ient = nullptr;
  // frame
  double *depth = nullptr, *onrm = nullptr;  // onrm: caller-supplied normals only
  // features (ORB path)
  int64_t n_feat = 0;
  uint8_t* tdesc = nullptr;
  double* tfeat_pts = nullptr;
  int32_t* tfeat_bidx = nullptr;
  double* tfeat_bw = nullptr;
  uint8_t* fdesc = nullptr;
  int32_t* fkp = nullptr;
  int64_t fdesc_cap = 0;
  int32_t *ham_idx = nullptr, *ham_dist = nullptr;
  unsigned long long* ham_packed = nullptr;  // (distance << 32) | index per template feature
  // ORB path: the solver's match arrays are indexed by template feature -- points,
  // binding and the control -> (feature, slot) CSR are static (set_features); per frame
  // only the observed points and weights change (0 = not an active match)
  int *fptr = nullptr, *fent = nullptr, *fpos = nullptr;
  double *ffo = nullptr, *ffw = nullptr;
  bool orb_static = false;
  // CUDA graph of the ORB frame body (everything after the input staging), captured once
  // per input signature and replayed: one launch instead of ~14 stream operations
  // [0] no pre-solver wait, [1] / [2] the pipelined path waiting on ev_out_copied[0 / 1]
  // captured frame bodies, per (pre-solver wait variant) x (input set: own buffers or
  // one of the two staging slots of the pipelined path)
  static constexpr int NG = 9;
  cudaGraphExec_t gexec[NG] = {};
  int64_t g_nframe[NG] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
  int g_launches[NG] = {};
  bool g_used[NG] = {};
  uint64_t g_gen[NG] = {};
  // input set of the frame being enqueued: 0 = the tracker's own depth / descriptor /
  // keypoint buffers, 1 + s = staging slot s (read in place, no device-to-device copy)
  int in_set = 0;
  bool graphs_off = false;
  // pipelined submission (dt_track_frame_submit / dt_tracker_wait): host inputs are staged
  // into one of two device slots on a copy stream while the previous frame computes;
  // outputs are copied back on the copy stream while the next frame computes
  cudaStream_t copy_stream = nullptr;  // host -> device staging
  // the frame's observation normals run on aux_stream beside the ORB matching chain
  // (only the solver needs them): fork / join events, captured into the frame graph
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t out_stream = nullptr;   // device -> host outputs (not queued behind staging)
  cudaEvent_t ev_in_ready[2] = {nullptr, nullptr}, ev_in_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_out_copied[2] = {nullptr, nullptr};
  cudaEvent_t pre_solver_wait = nullptr;  // compute stream waits on it before the solver
  bool own_stream = false;
  double* fs_partial = nullptr;   // preselection feature scatter: per-round partials
  unsigned* fs_counter = nullptr;  // created by dt_tracker_create (destroyed with the tracker)
  double* in_depth[2] = {nullptr, nullptr};
  // PFM-payload inputs (DT_DEPTH_PFM): the f32 bytes are staged here, then decoded on the
  // device into the f64 depth (own buffers / the pipelined slots)
  float* dstage = nullptr;
  float* in_dstage[2] = {nullptr, nullptr};
  // the pipelined path's staged match pairs / references (pairs path)
  double* in_msrc[2] = {nullptr, nullptr};
  double* in_mdst[2] = {nullptr, nullptr};
  int64_t* in_refs[2] = {nullptr, nullptr};
  int64_t in_pair_cap = 0, in_refs_cap = 0;
  uint8_t* in_desc[2] = {nullptr, nullptr};
  int32_t* in_kp[2] = {nullptr, nullptr};
  int64_t in_desc_cap = 0;
  int64_t* stage_info[2] = {nullptr, nullptr};   // device snapshot: info[4], stats[3], report,
                                                 // cost / lambda / stall histories
  int stage_words = 0;
  int64_t* h_stage[2] = {nullptr, nullptr};      // pinned host copy of the snapshot
  struct Pending {
    bool active = false, used = false;
    int32_t frame_id = 0;
    dt_frame_output out;
  } pend[2];
  int64_t pipe_next = 0;   // frames submitted
  int64_t pipe_waited = 0; // frames waited for
  // matches
  int64_t match_cap = 0;
  double *m_src = nullptr, *m_dst = nullptr, *m_w = nullptr, *m_res = nullptr, *m_bw = nullptr;
  uint8_t* m_flags = nullptr;
  int32_t *m_bidx = nullptr, *m_feat = nullptr;
  int64_t* refs = nullptr;
  int64_t refs_cap = 0;
  double *ref_support = nullptr, *ref_rot = nullptr;
  uint8_t* ref_valid = nullptr;
  int64_t* info = nullptr;      // [0] status [1] ref, [2] n_match, [3] n_active
  double* pstats = nullptr;     // [0] support [1] rotation... (support only)
  double* astats = nullptr;     // [0] weight sum [1] n flags
  double *fp = nullptr, *fo = nullptr, *fwt = nullptr, *fbw = nullptr;
  int32_t* fbidx = nullptr;
  int *mptr = nullptr, *ment = nullptr, *mcnt = nullptr, *mpos = nullptr;
  int *cpos = nullptr, *ipos = nullptr, *iinfo = nullptr;
  double* iew = nullptr;
  // solver state
  double *warp_a = nullptr, *warp_b = nullptr, *warps_out = nullptr, *lam = nullptr, *wa = nullptr;
  double *partial = nullptr, *csum = nullptr, *delta = nullptr, *oknorm = nullptr, *tentT = nullptr;
  double *erow = nullptr, *evals = nullptr;
  double *crec = nullptr, *prow = nullptr, *mrow = nullptr;
  double* pst = nullptr;     // k = 4: packed per-point statics (n x 16)
  int* pi8 = nullptr;        // k = 4: bind index + CSR position (n x 8)
  double* pixrec = nullptr;  // per pixel {depth or NaN, normal xyz}
  int* counts = nullptr;
  dt_report* report = nullptr;
  double *cost_hist = nullptr, *lam_hist = nullptr, *wa_out = nullptr;
  double* gstate = nullptr;  // m > M_MAX_SMEM: per-CTA solver state
  int32_t* stalled_hist = nullptr;
  int* bad_flag = nullptr;
  // outputs
  double *out_p = nullptr, *out_n = nullptr;
  SolverArgs host_args;
  SolverArgs* dev_args = nullptr;
  SolverArgs* dev_args_slot = nullptr;  // [2], pipelined path: depth read from the slots
  // pinned staging for the report / stats
  dt_report* h_report = nullptr;
  int64_t* h_info = nullptr;
  double* h_stats = nullptr;
};

namespace {

// (Re)allocate a zeroed device buffer owned by the tracker. A buffer being replaced
// (capacity growth) is retired -- queued work may still read it -- and freed by reap()
// at the next point where the tracker's streams are idle.
template <typename T>
int dalloc(dt_tracker* t, T** out, size_t count) {
  void* p = nullptr;
  const size_t bytes = sizeof(T) * (count > 0 ? count : 1);
  // Outside a capture: from the stream-ordered pool on the tracker stream (returning 84
  // buffers with cudaFree at the end of a run measured 4 ms to 0.9 s, varying with the
  // driver's state; the pool returns them without a device-wide synchronization), zeroed
  // and complete before any other stream of the tracker can touch it. Inside a capture
  // (a frame that grows a buffer): a plain allocation, as a pool allocation there would
  // become a graph-owned memory node.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  DT_CHECK_CUDA(cudaStreamIsCapturing(t->stream, &cs));
  const bool pooled = cs == cudaStreamCaptureStatusNone;
  if (pooled) {
    DT_CHECK_CUDA(cudaMallocAsync(&p, bytes, t->stream));
    DT_CHECK_CUDA(cudaMemsetAsync(p, 0, bytes, t->stream));
    DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  } else {
    DT_CHECK_CUDA(cudaMalloc(&p, bytes));
    DT_CHECK_CUDA(cudaMemsetAsync(p, 0, bytes, t->stream));
  }
  if (*out != nullptr) {
    for (size_t i = 0; i < t->bufs.size(); ++i)
      if (t->bufs[i].p == static_cast<void*>(*out)) {
        t->retired.push_back(t->bufs[i]);
        t->bufs.erase(t->bufs.begin() + (std::ptrdiff_t)i);
        break;
      }
  }
  t->bufs.push_back({p, bytes, pooled});
  *out = static_cast<T*>(p);
  ++t->buf_gen;
  return DT_OK;
}

cudaError_t free_buf(dt_tracker* t, const DevBuf& b) {
  return b.pooled ? cudaFreeAsync(b.p, t->stream) : cudaFree(b.p);
}

// free retired buffers once every stream of the tracker has drained (never called
// while a stream is being captured)
int reap(dt_tracker* t) {
  if (t->retired.empty()) return DT_OK;
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  if (t->copy_stream) DT_CHECK_CUDA(cudaStreamSynchronize(t->copy_stream));
  if (t->out_stream) DT_CHECK_CUDA(cudaStreamSynchronize(t->out_stream));
  for (const DevBuf& b : t->retired) DT_CHECK_CUDA(free_buf(t, b));
  t->retired.clear();
  return DT_OK;
}

#define DT_TRY(expr)        \
  do {                      \
    int _st = (expr);       \
    if (_st != DT_OK) return _st; \
  } while (0)

template <typename T>
int upload(dt_tracker* t, T* dst, const T* src, size_t count) {
  if (count == 0) return DT_OK;
  DT_CHECK_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyHostToDevice, t->stream));
  return DT_OK;
}

int ensure_match_capacity(dt_tracker* t, int64_t cap) {
  if (cap <= t->match_cap) return DT_OK;
  cap = std::max<int64_t>(cap, 64);
  const int64_t k = t->k;
  DT_TRY(dalloc(t, &t->m_src, 3 * cap));
  DT_TRY(dalloc(t, &t->m_dst, 3 * cap));
  DT_TRY(dalloc(t, &t->m_w, cap));
  DT_TRY(dalloc(t, &t->m_res, cap));
  DT_TRY(dalloc(t, &t->m_flags, cap));
  DT_TRY(dalloc(t, &t->m_bidx, k * cap));
  DT_TRY(dalloc(t, &t->m_bw, k * cap));
  DT_TRY(dalloc(t, &t->m_feat, cap));
  DT_TRY(dalloc(t, &t->ref_support, cap));
  DT_TRY(dalloc(t, &t->ref_rot, 9 * cap));
  DT_TRY(dalloc(t, &t->ref_valid, cap));
  DT_TRY(dalloc(t, &t->fp, 3 * cap));
  DT_TRY(dalloc(t, &t->fo, 3 * cap));
  DT_TRY(dalloc(t, &t->fwt, cap));
  DT_TRY(dalloc(t, &t->fbidx, k * cap));
  DT_TRY(dalloc(t, &t->fbw, k * cap));
  DT_TRY(dalloc(t, &t->ment, k * cap));
  DT_TRY(dalloc(t, &t->mpos, k * cap));
  DT_TRY(dalloc(t, &t->mrow, 2 * k * cap * 3 * 8));
  t->match_cap = cap;
  {
    const int64_t nch = (t->n + CHUNK - 1) / CHUNK + (cap + CHUNK - 1) / CHUNK +
                        (t->ne + CHUNK - 1) / CHUNK;
    DT_TRY(dalloc(t, &t->csum, 2 * nch));
    int64_t items = std::max<int64_t>(std::max<int64_t>((t->n + CHUNK - 1) / CHUNK, (cap + CHUNK - 1) / CHUNK),
                                      std::max<int64_t>((t->ne + CHUNK - 1) / CHUNK, t->m));
    t->red_g = (int)((items + 31) / 32);
    DT_TRY(dalloc(t, &t->red, (size_t)RED_SLOTS * (2 * t->red_g + 2)));
    DT_TRY(dalloc(t, &t->redc, (size_t)RED_SLOTS * (t->red_g + 1)));
  }
  t->args_dirty = true;
  return DT_OK;
}

void fill_args(dt_tracker* t) {
  SolverArgs& a = t->host_args;
  const dt_config& c = t->cfg;
  a.n = (int)t->n;
  a.k = (int)t->k;
  a.m = (int)t->m;
  a.n_edges = (int)t->ne;
  a.height = c.height;
  a.width = c.width;
  a.max_outer = c.max_outer_iters;
  a.max_retries = c.max_retries;
  a.fx = c.fx; a.fy = c.fy; a.cx = c.cx; a.cy = c.cy;
  a.gate = c.gate_distance;
  a.cos_gate = c.cos_gate;
  a.tukey = c.tukey_scale;
  a.fw = c.feature_weight;
  a.arap_w = c.arap_weight;
  a.angle_w = c.angle_weight;
  a.rot_w = c.rotation_weight;
  a.sq_angle_w = std::sqrt(c.angle_weight);
  a.sq_rot_w = std::sqrt(c.rotation_weight);
  a.inv_tukey = 1.0 / c.tukey_scale;
  a.data_floor = c.data_floor;
  a.lam_init = c.lambda_init;
  a.lam_dec = c.lambda_decrease;
  a.lam_inc = c.lambda_increase;
  a.lam_min = c.lambda_min;
  a.lam_max = c.lambda_max;
  a.step_tol = c.step_tol;
  a.cost_tol = c.cost_tol;
  a.tp = t->tp; a.tn = t->tn; a.bidx = t->bidx; a.bw = t->bw; a.bws = t->bws;
  a.cptr = t->cptr; a.cent = t->cent; a.cpos = t->cpos;
  a.cpts = t->cpts; a.edges = t->edges; a.ew = t->ew; a.iptr = t->iptr; a.ient = t->ient;
  a.ipos = t->ipos; a.iinfo = t->iinfo; a.iew = t->iew;
  a.pst = t->pst; a.pi8 = t->pi8; a.pixrec = t->pixrec;
  a.n_active = t->info + 3;
  if (t->orb_static) {
    a.fp = t->tfeat_pts; a.fo = t->ffo; a.fwt = t->ffw; a.fbidx = t->tfeat_bidx; a.fbw = t->tfeat_bw;
    a.mptr = t->fptr; a.ment = t->fent; a.mpos = t->fpos;
  } else {
    a.fp = t->fp; a.fo = t->fo; a.fwt = t->fwt; a.fbidx = t->fbidx; a.fbw = t->fbw;
    a.mptr = t->mptr; a.ment = t->ment; a.mpos = t->mpos;
  }
  a.warp_a = t->warp_a; a.warp_b = t->warp_b; a.warps_out = t->warps_out;
  a.lam = t->lam; a.wa = t->wa; a.partial = t->partial; a.csum = t->csum;
  a.gstate = t->gstate;
  a.erow = t->erow; a.evals = t->evals;
  a.nch_p = (int)((t->n + CHUNK - 1) / CHUNK);
  a.nch_m = (int)((t->match_cap + CHUNK - 1) / CHUNK);
  a.nch_e = (int)((t->ne + CHUNK - 1) / CHUNK);
  a.delta = t->delta; a.oknorm = t->oknorm; a.tentT = t->tentT;
  a.crec = t->crec; a.prow = t->prow; a.mrow = t->mrow;
  a.ma_cap = (int)t->match_cap;
  a.counts = t->counts;
  a.report = t->report;
  a.cost_hist = t->cost_hist;
  a.lam_hist = t->lam_hist;
  a.stalled_hist = t->stalled_hist;
  a.wa_out = t->wa_out;
  // grid mode folds the output warp into the solver's final phase
  a.out_p = t->grid_mode ? t->out_p : nullptr;
  a.out_n = t->grid_mode ? t->out_n : nullptr;
  a.trace = t->profiling ? t->trace : nullptr;
  a.trace_cap = t->trace_cap;
  a.arrivals = t->profiling ? t->arrivals : nullptr;
  a.arr_cap = t->arr_cap;
  a.red = t->red;
  a.redc = t->redc;
  a.red_g = t->red_g;
}

// the solver's arguments (one block per input set: the solver reads the frame through the
// pixel records every input set writes into the same buffer, so the blocks are equal)
int push_args(dt_tracker* t) {
  fill_args(t);
  t->args_dirty = false;
  DT_CHECK_CUDA(cudaMemcpyAsync(t->dev_args, &t->host_args, sizeof(SolverArgs),
                                cudaMemcpyHostToDevice, t->stream));
  if (t->dev_args_slot) {
    const SolverArgs v[2] = {t->host_args, t->host_args};
    DT_CHECK_CUDA(cudaMemcpyAsync(t->dev_args_slot, v, sizeof(v), cudaMemcpyHostToDevice, t->stream));
  }
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  return DT_OK;
}

// cluster_size <= 0: one cooperative grid over every SM (lowest latency for one
// sequence), falling back to the largest cluster; > 0: cluster of that size
void pick_mode(dt_tracker* t) {
  t->grid_mode = 0;
  t->cluster = solver_pick_cluster(t->device, t->cfg.cluster_size > 0 ? t->cfg.cluster_size : 0,
                                   (int)t->m);
  if (t->cfg.cluster_size <= 0 && solver_grid_blocks(t->device, (int)t->m) > 0) t->grid_mode = 1;
}

int validate_config(const dt_config* c) {
  DT_REQUIRE(c != nullptr, DT_ERR_INVALID_ARGUMENT, "config is NULL");
  DT_REQUIRE(c->max_outer_iters >= 1 && c->max_retries >= 0, DT_ERR_INVALID_ARGUMENT,
             "iteration budgets must be positive");
  DT_REQUIRE(c->lambda_min > 0.0 && c->lambda_min <= c->lambda_init && c->lambda_init <= c->lambda_max,
             DT_ERR_INVALID_ARGUMENT, "lambda_init must lie inside [lambda_min, lambda_max]");
  DT_REQUIRE(c->lambda_decrease < 1.0 && c->lambda_increase > 1.0, DT_ERR_INVALID_ARGUMENT,
             "damping factors must shrink on accept and grow on reject");
  DT_REQUIRE(c->tukey_scale > 0.0, DT_ERR_INVALID_ARGUMENT, "tukey_scale must be positive");
  DT_REQUIRE(c->width > 0 && c->height > 0 && c->fx > 0.0 && c->fy > 0.0, DT_ERR_INVALID_ARGUMENT,
             "invalid camera");
  return DT_OK;
}

// stable counting sort of (key, entry) by key on the host (template-time CSR)
void host_csr(const std::vector<int>& keys, const std::vector<int>& ents, int m,
              std::vector<int>& ptr, std::vector<int>& out) {
  ptr.assign(m + 1, 0);
  for (int kk : keys) ptr[kk + 1]++;
  for (int i = 0; i < m; ++i) ptr[i + 1] += ptr[i];
  out.assign(keys.size(), 0);
  std::vector<int> pos(ptr.begin(), ptr.end() - 1);
  for (size_t i = 0; i < keys.size(); ++i) out[pos[keys[i]]++] = ents[i];
}

__global__ void k_i64_to_i32(const int64_t* __restrict__ a, int64_t n, int m, int32_t* __restrict__ b,
                             int* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = a[i];
  if (v < 0 || v >= m) *bad = 1;
  b[i] = (int32_t)(v < 0 ? 0 : (v >= m ? m - 1 : v));
}

// binding (n, k) int64 + f64 from the caller -> the tracker's int32 / f64 buffers
int upload_binding(dt_tracker* t, const int64_t* bidx, const double* bw, int64_t n, bool on_dev,
                   int32_t* dst_idx, double* dst_w) {
  cudaStream_t s = t->stream;
  const int64_t cnt = n * t->k;
  if (cnt == 0) return DT_OK;
  if (on_dev) {
    k_i64_to_i32<<<grid_for(cnt, 256), 256, 0, s>>>(bidx, cnt, (int)t->m, dst_idx, t->bad_flag);
    DT_CHECK_LAUNCH();
  } else {
    std::vector<int32_t> tmp(cnt);
    for (int64_t i = 0; i < cnt; ++i) {
      DT_REQUIRE(bidx[i] >= 0 && bidx[i] < t->m, DT_ERR_INVALID_ARGUMENT, "binding index out of range");
      tmp[i] = (int32_t)bidx[i];
    }
    DT_CHECK_CUDA(cudaMemcpyAsync(dst_idx, tmp.data(), sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, s));
    DT_CHECK_CUDA(cudaStreamSynchronize(s));  // tmp is stack-owned
  }
  DT_CHECK_CUDA(cudaMemcpyAsync(dst_w, bw, sizeof(double) * cnt,
                                on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  return DT_OK;
}

// The C-ABI size contract of dt_frame_input (include/deformtrack_b200.h): the caller's
// arrays are only dereferenced after these checks pass.
int check_frame_input(const dt_tracker* t, const dt_frame_input* in) {
  DT_REQUIRE(in != nullptr, DT_ERR_INVALID_ARGUMENT, "frame input is NULL");
  DT_REQUIRE(in->depth != nullptr, DT_ERR_INVALID_ARGUMENT, "depth is required");
  DT_REQUIRE(in->height == t->cfg.height && in->width == t->cfg.width, DT_ERR_INVALID_ARGUMENT,
             "depth is %dx%d but the tracker's camera is %dx%d", (int)in->width, (int)in->height,
             (int)t->cfg.width, (int)t->cfg.height);
  DT_REQUIRE(in->on_device == 0 || in->on_device == 1, DT_ERR_INVALID_ARGUMENT, "on_device must be 0 or 1");
  DT_REQUIRE(in->depth_kind == DT_DEPTH_F64 || in->depth_kind == DT_DEPTH_PFM, DT_ERR_INVALID_ARGUMENT,
             "unknown depth_kind %d", (int)in->depth_kind);
  DT_REQUIRE(in->depth_kind == DT_DEPTH_F64 || in->normals == nullptr, DT_ERR_INVALID_ARGUMENT,
             "precomputed normals need an f64 depth");
  DT_REQUIRE(in->n_pairs >= 0 && in->n_frame >= 0 && in->n_refs >= 0, DT_ERR_INVALID_ARGUMENT,
             "negative count");
  DT_REQUIRE(in->n_frame <= (int64_t)1 << 24 && in->n_pairs <= (int64_t)1 << 26, DT_ERR_INVALID_ARGUMENT,
             "match / descriptor count out of range");
  if (in->use_matches && in->frame_desc != nullptr) {
    DT_REQUIRE(in->frame_kp != nullptr, DT_ERR_INVALID_ARGUMENT, "frame descriptors without keypoints");
    DT_REQUIRE(t->n_feat > 0, DT_ERR_INVALID_ARGUMENT, "frame descriptors given but no template features set");
  } else if (in->use_matches && in->n_pairs > 0) {
    DT_REQUIRE(in->match_src != nullptr && in->match_dst != nullptr, DT_ERR_INVALID_ARGUMENT,
               "match pairs missing");
    DT_REQUIRE((in->match_bidx == nullptr) == (in->match_bw == nullptr), DT_ERR_INVALID_ARGUMENT,
               "match_bidx and match_bw come together");
  }
  if (in->n_refs > 0) {
    DT_REQUIRE(in->refs != nullptr, DT_ERR_INVALID_ARGUMENT, "n_refs > 0 but refs is NULL");
    if (!in->on_device) {
      const int64_t lim = in->frame_desc != nullptr ? t->n_feat : in->n_pairs;
      for (int64_t i = 0; i < in->n_refs; ++i)
        DT_REQUIRE(in->refs[i] >= 0 && in->refs[i] < lim, DT_ERR_INVALID_ARGUMENT,
                   "reference index %lld outside [0, %lld)", (long long)in->refs[i], (long long)lim);
    }
  }
  return DT_OK;
}

void mark(dt_tracker* t, int i) {
  if (t->profiling) cudaEventRecord(t->ev[i], t->stream);
}

int enqueue_frame(dt_tracker* t, const dt_frame_input* in, bool* used_matches) {
  cudaStream_t s = t->stream;
  const dt_config& c = t->cfg;
  const int64_t npix = (int64_t)c.width * c.height;
  const cudaMemcpyKind kind = in->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  DT_REQUIRE(in->depth != nullptr, DT_ERR_INVALID_ARGUMENT, "depth is required");
  t->launches = 0;
  mark(t, 0);
  // warm start: the previous solution (or set_warps) is in warps_out
  // (the shared-memory solver reads the warm start straight from warps_out)
  if (t->m > M_MAX_SMEM)
    DT_CHECK_CUDA(cudaMemcpyAsync(t->warp_a, t->warps_out, sizeof(double) * 8 * t->m,
                                  cudaMemcpyDeviceToDevice, s));
  // input set: the tracker's buffers (copied into) or a staging slot (read in place)
  const int set = t->in_set;
  double* dep = set ? t->in_depth[set - 1] : t->depth;
  DT_REQUIRE(!set || in->depth == dep, DT_ERR_INVALID_ARGUMENT, "staged depth mismatch");
  if (in->depth_kind == DT_DEPTH_PFM) {
    // the file's f32 payload in, decoded on the device (fileio.read_pfm)
    if (!t->dstage) DT_TRY(dalloc(t, &t->dstage, npix));
    DT_CHECK_CUDA(cudaMemcpyAsync(t->dstage, in->depth, sizeof(float) * npix, kind, s));
    DT_TRY(launch_depth_from_pfm(t->dstage, c.height, c.width, 0, dep, s));
    ++t->launches;
  } else if (in->depth != dep) {
    DT_CHECK_CUDA(cudaMemcpyAsync(dep, in->depth, sizeof(double) * npix, kind, s));
  }
  // the solver reads the frame as 32-byte pixel records {depth or NaN, normal}; they are
  // produced on the aux stream beside the matching chain (serially when profiling, so the
  // per-stage events keep their meaning)
  const bool fork = !t->profiling;
  cudaStream_t ns = s;
  if (fork) {
    DT_CHECK_CUDA(cudaEventRecord(t->ev_fork, s));
    DT_CHECK_CUDA(cudaStreamWaitEvent(t->aux_stream, t->ev_fork, 0));
    ns = t->aux_stream;
  }
  if (in->normals) {
    if (!t->onrm) DT_TRY(dalloc(t, &t->onrm, 3 * npix));
    DT_CHECK_CUDA(cudaMemcpyAsync(t->onrm, in->normals, sizeof(double) * 3 * npix, kind, ns));
    DT_TRY(launch_pack_pixels(dep, t->onrm, npix, c.z_min, c.z_max, t->pixrec, ns));
  } else {
    DT_TRY(launch_observation_normals(dep, c.height, c.width, c.fx, c.fy, c.cx, c.cy, c.z_min,
                                      c.z_max, nullptr, nullptr, ns, t->pixrec));
  }
  if (fork) DT_CHECK_CUDA(cudaEventRecord(t->ev_join, t->aux_stream));
  ++t->launches;
  mark(t, 1);

  // ---- matches ----
  bool use = in->use_matches != 0;
  int64_t n_max = 0;
  bool orb_fused = false;
  const int32_t* orb_kp = nullptr;
  if (use && in->frame_desc != nullptr) {
    DT_REQUIRE(t->n_feat > 0, DT_ERR_INVALID_ARGUMENT, "frame descriptors given but no template features set");
    if (!set && in->n_frame > t->fdesc_cap) {
      const int64_t cap = std::max<int64_t>(in->n_frame, 256);
      DT_TRY(dalloc(t, &t->fdesc, 32 * cap));
      DT_TRY(dalloc(t, &t->fkp, 2 * cap));
      t->fdesc_cap = cap;
    }
    uint8_t* fdesc = set ? t->in_desc[set - 1] : t->fdesc;
    int32_t* fkp = set ? t->in_kp[set - 1] : t->fkp;
    DT_REQUIRE(!set || (in->frame_desc == fdesc && in->frame_kp == fkp), DT_ERR_INVALID_ARGUMENT,
               "staged descriptors mismatch");
    if (in->frame_desc != fdesc)
      DT_CHECK_CUDA(cudaMemcpyAsync(fdesc, in->frame_desc, 32 * in->n_frame, kind, s));
    if (in->frame_kp != fkp)
      DT_CHECK_CUDA(cudaMemcpyAsync(fkp, in->frame_kp, sizeof(int32_t) * 2 * in->n_frame, kind, s));
    DT_TRY(launch_hamming(t->tdesc, t->n_feat, fdesc, in->n_frame, nullptr, nullptr, s,
                          t->ham_packed, true));
    ++t->launches;
    // the match build runs inside the fused preselection when the template's features fit
    // its shared-memory copy (in cluster mode too: 8-warp CTAs, config 5 measured 2,855
    // vs 2,732 frames/s with the separate chain)
    orb_fused = t->n_feat <= ORB_FUSED_MAX;
    orb_kp = fkp;
    if (!orb_fused) {
      k_build_matches<<<1, 1024, 0, s>>>(t->n_feat, t->ham_packed, c.max_hamming, fkp,
                                         in->n_frame, dep, c.z_min, c.z_max, c.width, c.height, c.fx,
                                         c.fy, c.cx, c.cy, t->tfeat_pts, t->m_src, t->m_dst, t->m_feat,
                                         t->info + 2, t->ffw);
      DT_CHECK_LAUNCH();
      ++t->launches;
    }
    n_max = t->n_feat;
  } else if (use && in->n_pairs > 0) {
    DT_TRY(ensure_match_capacity(t, in->n_pairs));
    DT_CHECK_CUDA(cudaMemcpyAsync(t->m_src, in->match_src, sizeof(double) * 3 * in->n_pairs, kind, s));
    DT_CHECK_CUDA(cudaMemcpyAsync(t->m_dst, in->match_dst, sizeof(double) * 3 * in->n_pairs, kind, s));
    k_set_i64<<<1, 1, 0, s>>>(t->info + 2, in->n_pairs);
    DT_CHECK_LAUNCH();
    if (in->match_bidx != nullptr && in->match_bw != nullptr) {
      // caller-supplied binding (e.g. the reference's kd-tree tie order)
      DT_TRY(upload_binding(t, in->match_bidx, in->match_bw, in->n_pairs, in->on_device != 0,
                            t->m_bidx, t->m_bw));
    } else {
      // per-frame binding of the match template points, sigma = graph sampling radius
      // (solver.py:292-296)
      DT_TRY(launch_bind_points_i32(t->m_src, in->n_pairs, t->cpts, (int)t->m, (int)t->k,
                                    c.sampling_radius, t->m_bidx, t->m_bw, s));
    }
    t->launches += 2;
    n_max = in->n_pairs;
  } else {
    use = false;
  }
  *used_matches = use;
  mark(t, 2);
  if (use && in->match_w != nullptr && in->frame_desc == nullptr) {
    // weights given by the caller (already annotated MatchSet): no preselection
    DT_CHECK_CUDA(cudaMemcpyAsync(t->m_w, in->match_w, sizeof(double) * in->n_pairs, kind, s));
    DT_CHECK_CUDA(cudaMemsetAsync(t->m_flags, 0, in->n_pairs, s));
    k_set_i64<<<1, 1, 0, s>>>(t->info, DT_OK);
    DT_CHECK_LAUNCH();
    ++t->launches;
  } else if (use) {
    int exhaustive = 1;
    int64_t n_refs = 0;
    if (in->refs != nullptr && in->n_refs > 0) {
      if (in->n_refs > t->refs_cap) {
        DT_TRY(dalloc(t, &t->refs, in->n_refs));
        t->refs_cap = in->n_refs;
      }
      DT_CHECK_CUDA(cudaMemcpyAsync(t->refs, in->refs, sizeof(int64_t) * in->n_refs, kind, s));
      exhaustive = 0;
      n_refs = in->n_refs;
    }
    if (!exhaustive && n_refs > t->match_cap) DT_TRY(ensure_match_capacity(t, n_refs));
    // ORB path: the final preselection kernel also scatters the weights to the template
    // features (matches indexed by feature: static points / binding / CSR)
    FeatureScatter fs{t->n_feat, t->m_dst, t->m_feat, t->ffo, t->ffw, t->info + 3, t->astats,
                      t->fs_partial, t->fs_counter};
    if (orb_fused) {
      const OrbMatchIn mi{t->n_feat, t->ham_packed, c.max_hamming, orb_kp, in->n_frame, dep,
                          c.z_min, c.z_max, c.width, c.height, c.fx, c.fy, c.cx, c.cy, t->tfeat_pts};
      const PreselectOrbOut mo{t->m_src, t->m_dst, t->m_feat, t->info + 2, t->m_w, t->m_flags,
                               t->m_res, t->info, t->pstats, fs, t->ham_packed, t->fs_counter};
      DT_TRY(launch_preselect_orb(mi, exhaustive ? nullptr : t->refs, n_refs,
                                  c.preselect.distance_threshold, c.preselect.n_reweight_iters,
                                  c.preselect.inlier_weight_min, c.preselect.min_support,
                                  t->ref_support, t->ref_rot, t->ref_valid, mo, s,
                                  t->grid_mode ? 0 : 1));
      ++t->launches;
    } else {
    DT_TRY(launch_preselect(t->m_src, t->m_dst, t->info + 2, n_max, t->refs, n_refs, exhaustive,
                            c.preselect.distance_threshold, c.preselect.n_reweight_iters,
                            c.preselect.inlier_weight_min, c.preselect.min_support, t->m_w,
                            t->m_flags, t->m_res, nullptr, t->info, t->pstats, t->ref_support,
                            t->ref_rot, t->ref_valid, s,
                            in->frame_desc != nullptr ? &fs : nullptr, t->grid_mode ? 0 : 1));
    t->launches += 2;
    }
  } else {
    k_set_i64<<<1, 1, 0, s>>>(t->info + 2, 0);
    DT_CHECK_LAUNCH();
    ++t->launches;
  }
  mark(t, 3);
  const bool orb_static = use && in->frame_desc != nullptr;
  if (orb_static != t->orb_static) {
    t->orb_static = orb_static;
    t->args_dirty = true;
  }
  if (!orb_static) {
    k_active<<<1, 1024, 0, s>>>(t->info + 2, t->m_w, t->m_flags, t->m_src, t->m_dst, t->m_bidx,
                                t->m_bw, (int)t->k, use ? 1 : 0, t->fp, t->fo, t->fwt, t->fbidx,
                                t->fbw, t->info + 3, t->astats);
    DT_CHECK_LAUNCH();
    const int cthreads = 256;
    const int cblocks = grid_for(t->m * 32, cthreads);
    k_csr_count_dev<<<cblocks, cthreads, 0, s>>>(t->fbidx, t->info + 3, (int)t->k, (int)t->m, t->mcnt);
    DT_CHECK_LAUNCH();
    k_scan_counts<<<1, 1024, 0, s>>>(t->mcnt, (int)t->m, t->mptr);
    DT_CHECK_LAUNCH();
    k_csr_fill_dev<<<cblocks, cthreads, 0, s>>>(t->fbidx, t->info + 3, (int)t->k, (int)t->m, t->mptr,
                                                t->ment, t->mpos);
    DT_CHECK_LAUNCH();
    t->launches += 4;
  }
  mark(t, 4);

  // ---- solve ----
  if (fork) DT_CHECK_CUDA(cudaStreamWaitEvent(s, t->ev_join, 0));  // the pixel records
  if (t->args_dirty) DT_TRY(push_args(t));
  if (t->pre_solver_wait) DT_CHECK_CUDA(cudaStreamWaitEvent(s, t->pre_solver_wait, 0));
  DT_TRY(solver_launch(t->in_set ? t->dev_args_slot + (t->in_set - 1) : t->dev_args, 1, t->cluster,
                       (int)t->m, (int)t->k, t->grid_mode, s));
  ++t->launches;
  mark(t, 5);
  // ---- output warp (tracking.py:87): in grid mode done by the solver's final phase ----
  if (!t->grid_mode) {
    DT_TRY(launch_warp_all_i32(t->tp, t->tn, t->bidx, t->bw, t->n, (int)t->k, t->warps_out,
                               t->out_p, t->out_n, s));
    ++t->launches;
  }
  mark(t, 6);
  return DT_OK;
}

int collect_outputs(dt_tracker* t, const dt_frame_input* in, dt_frame_output* out, bool used) {
  cudaStream_t s = t->stream;
  if (out == nullptr) return DT_OK;
  if (out->warps)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->warps, t->warps_out, sizeof(double) * 8 * t->m, cudaMemcpyDeviceToHost, s));
  if (out->points)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->points, t->out_p, sizeof(double) * 3 * t->n, cudaMemcpyDeviceToHost, s));
  if (out->normals)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->normals, t->out_n, sizeof(double) * 3 * t->n, cudaMemcpyDeviceToHost, s));
  if (out->control_data_weights)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->control_data_weights, t->wa_out, sizeof(double) * t->m,
                                  cudaMemcpyDeviceToHost, s));
  const int64_t cap = std::min<int64_t>(out->match_capacity, t->match_cap);
  if (cap > 0) {
    if (out->match_weights)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->match_weights, t->m_w, sizeof(double) * cap, cudaMemcpyDeviceToHost, s));
    if (out->match_flags)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->match_flags, t->m_flags, cap, cudaMemcpyDeviceToHost, s));
    if (out->match_src)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->match_src, t->m_src, sizeof(double) * 3 * cap, cudaMemcpyDeviceToHost, s));
    if (out->match_dst)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->match_dst, t->m_dst, sizeof(double) * 3 * cap, cudaMemcpyDeviceToHost, s));
  }
  {
    const int it = t->cfg.max_outer_iters;
    if (out->cost_history)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->cost_history, t->cost_hist, sizeof(double) * 2 * it, cudaMemcpyDeviceToHost, s));
    if (out->lambda_history)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->lambda_history, t->lam_hist, sizeof(double) * 2 * it, cudaMemcpyDeviceToHost, s));
    if (out->stalled)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->stalled, t->stalled_hist, sizeof(int32_t) * it, cudaMemcpyDeviceToHost, s));
  }
  DT_CHECK_CUDA(cudaMemcpyAsync(t->h_report, t->report, sizeof(dt_report), cudaMemcpyDeviceToHost, s));
  DT_CHECK_CUDA(cudaMemcpyAsync(t->h_info, t->info, sizeof(int64_t) * 4, cudaMemcpyDeviceToHost, s));
  DT_CHECK_CUDA(cudaMemcpyAsync(t->h_stats, t->astats, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
  DT_CHECK_CUDA(cudaMemcpyAsync(t->h_stats + 2, t->pstats, sizeof(double), cudaMemcpyDeviceToHost, s));
  DT_CHECK_CUDA(cudaStreamSynchronize(s));
  dt_report* R = t->h_report;
  R->frame_id = in->frame_id;
  if (used) {
    R->n_matches = (int32_t)t->h_info[2];
    R->n_preselected = (int32_t)t->h_stats[1];
    R->match_weight_sum = t->h_stats[0];
    R->preselect_status = (int32_t)t->h_info[0];
    R->preselect_reference = (int32_t)t->h_info[1];
    R->preselect_support = t->h_stats[2];
  } else {
    R->n_matches = 0;
    R->n_preselected = 0;
    R->match_weight_sum = 0.0;
    R->preselect_status = DT_OK;
    R->preselect_reference = -1;
    R->preselect_support = 0.0;
  }
  if (out->report) *out->report = *R;
  return DT_OK;
}

void drop_graph(dt_tracker* t) {
  for (int i = 0; i < dt_tracker::NG; ++i) {
    if (t->gexec[i]) cudaGraphExecDestroy(t->gexec[i]);
    t->gexec[i] = nullptr;
    t->g_nframe[i] = -1;
  }
}

// A frame through the CUDA graph when it is the steady-state ORB case (depth + frame
// descriptors, no precomputed normals, profiling off, solver arguments already on the
// device): stage the inputs into the tracker's own buffers, then replay the captured
// body. Anything else -- or a failed capture -- runs the stream-ordered path.
int run_frame(dt_tracker* t, const dt_frame_input* in, bool* used) {
  const int set = t->in_set;
  const int64_t cap = set ? t->in_desc_cap : t->fdesc_cap;
  const bool eligible = !t->graphs_off && !t->profiling && !t->args_dirty && in->depth != nullptr &&
                        in->normals == nullptr && in->use_matches && in->frame_desc != nullptr &&
                        in->frame_kp != nullptr && in->n_frame > 0 && in->n_frame <= cap &&
                        t->orb_static;
  if (!eligible) return enqueue_frame(t, in, used);
  cudaStream_t s = t->stream;
  dt_frame_input gin = *in;
  gin.on_device = 1;
  if (set == 0) {
    // own input buffers: copy the caller's arrays in, then replay
    const cudaMemcpyKind kind = in->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const int64_t npix = (int64_t)t->cfg.width * t->cfg.height;
    if (in->depth_kind == DT_DEPTH_PFM) {
      if (!t->dstage) return enqueue_frame(t, in, used);  // first PFM frame: allocate first
      DT_CHECK_CUDA(cudaMemcpyAsync(t->dstage, in->depth, sizeof(float) * npix, kind, s));
      DT_TRY(launch_depth_from_pfm(t->dstage, t->cfg.height, t->cfg.width, 0, t->depth, s));
    } else {
      DT_CHECK_CUDA(cudaMemcpyAsync(t->depth, in->depth, sizeof(double) * npix, kind, s));
    }
    gin.depth_kind = DT_DEPTH_F64;
    DT_CHECK_CUDA(cudaMemcpyAsync(t->fdesc, in->frame_desc, 32 * in->n_frame, kind, s));
    DT_CHECK_CUDA(cudaMemcpyAsync(t->fkp, in->frame_kp, sizeof(int32_t) * 2 * in->n_frame, kind, s));
    gin.depth = t->depth;
    gin.frame_desc = t->fdesc;
    gin.frame_kp = t->fkp;
  }  // else: a staging slot, read in place by its own graph
  const int gw = t->pre_solver_wait == nullptr ? 0
                 : (t->copy_stream && t->pre_solver_wait == t->ev_out_copied[0] ? 1 : 2);
  const int gi = 3 * gw + set;
  // re-capture when the descriptor count changed or any buffer was reallocated since the
  // capture (a replay would read the replaced buffers)
  if (t->gexec[gi] == nullptr || t->g_nframe[gi] != in->n_frame || t->g_gen[gi] != t->buf_gen) {
    if (t->gexec[gi]) cudaGraphExecDestroy(t->gexec[gi]);
    t->gexec[gi] = nullptr;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      t->graphs_off = true;
      return enqueue_frame(t, &gin, used);
    }
    bool u = false;
    const int st = enqueue_frame(t, &gin, &u);
    const cudaError_t ce = cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge = nullptr;
    if (st != DT_OK || ce != cudaSuccess || g == nullptr ||
        cudaGraphInstantiate(&ge, g, 0) != cudaSuccess || t->args_dirty) {
      cudaGetLastError();
      if (g) cudaGraphDestroy(g);
      if (ge) cudaGraphExecDestroy(ge);
      t->graphs_off = true;  // capture unsupported here: stream-ordered from now on
      return enqueue_frame(t, &gin, used);
    }
    cudaGraphDestroy(g);
    t->gexec[gi] = ge;
    t->g_nframe[gi] = in->n_frame;
    t->g_launches[gi] = t->launches;
    t->g_used[gi] = u;
    t->g_gen[gi] = t->buf_gen;  // after the capture: it may have grown a buffer itself
  }
  DT_CHECK_CUDA(cudaGraphLaunch(t->gexec[gi], s));
  t->launches = t->g_launches[gi];
  *used = t->g_used[gi];
  return DT_OK;
}

}  // namespace

extern "C" {

// Everything after the allocation of the handle; on failure dt_tracker_create destroys
// the partly built tracker (buffers, streams, events) instead of leaking it.
static int tracker_init(dt_tracker* t, const dt_config* cfg, const double* t_points, const double* t_normals,
                const int64_t* bind_idx, const double* bind_w, int64_t n, int64_t k,
                const double* ctrl_points, const double* warps, int64_t m,
                const int64_t* edges, const double* edge_weights, int64_t n_edges,
                int device, void* stream) {
  t->cfg = *cfg;
  t->device = device;
  t->n = n;
  t->k = k;
  t->m = m;
  t->ne = n_edges;
  if (stream) {
    t->stream = as_stream(stream);
  } else {
    DT_CHECK_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    t->own_stream = true;
  }
  DT_CHECK_CUDA(cudaStreamCreateWithFlags(&t->aux_stream, cudaStreamNonBlocking));
  DT_CHECK_CUDA(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
  DT_CHECK_CUDA(cudaEventCreateWithFlags(&t->ev_join, cudaEventDisableTiming));
  const int64_t npix = (int64_t)cfg->width * cfg->height;
  // static data
  std::vector<int32_t> bidx32(n * k), edges32(2 * n_edges);
  for (int64_t i = 0; i < n * k; ++i) {
    DT_REQUIRE(bind_idx[i] >= 0 && bind_idx[i] < m, DT_ERR_INVALID_ARGUMENT, "bind index out of range");
    bidx32[i] = (int32_t)bind_idx[i];
  }
  for (int64_t i = 0; i < 2 * n_edges; ++i) {
    DT_REQUIRE(edges[i] >= 0 && edges[i] < m, DT_ERR_INVALID_ARGUMENT, "edge index out of range");
    edges32[i] = (int32_t)edges[i];
  }
  // control -> (point, slot), encoded (p << 3) | slot, in point order
  std::vector<int> keys(n * k), ents(n * k), cptr, cent;
  for (int64_t p = 0; p < n; ++p)
    for (int64_t s = 0; s < k; ++s) {
      keys[p * k + s] = bidx32[p * k + s];
      ents[p * k + s] = (int)((p << 3) | s);
    }
  host_csr(keys, ents, (int)m, cptr, cent);
  std::vector<int> ekeys(2 * n_edges), eents(2 * n_edges), iptr, ient;
  for (int64_t e = 0; e < n_edges; ++e)
    for (int s = 0; s < 2; ++s) {
      ekeys[2 * e + s] = edges32[2 * e + s];
      eents[2 * e + s] = (int)((e << 1) | s);
    }
  host_csr(ekeys, eents, (int)m, iptr, ient);
  // inverse maps: the CSR position of every (point, slot) and (edge, side), and per edge
  // position the other endpoint + side and the edge weight (static per sequence)
  std::vector<int> cpos(n * k), ipos(2 * n_edges), iinfo(2 * n_edges);
  std::vector<double> iew(2 * n_edges);
  for (size_t q = 0; q < cent.size(); ++q) cpos[(cent[q] >> 3) * k + (cent[q] & 7)] = (int)q;
  for (size_t q = 0; q < ient.size(); ++q) {
    const int e = ient[q] >> 1, side = ient[q] & 1;
    ipos[2 * e + side] = (int)q;
    iinfo[q] = (edges32[2 * e + (1 - side)] << 1) | side;
    iew[q] = edge_weights[e];
  }

  DT_TRY(dalloc(t, &t->tp, 3 * n));
  DT_TRY(dalloc(t, &t->tn, 3 * n));
  DT_TRY(dalloc(t, &t->bidx, k * n));
  DT_TRY(dalloc(t, &t->bw, k * n));
  DT_TRY(dalloc(t, &t->bws, k * n));
  DT_TRY(dalloc(t, &t->cptr, m + 1));
  DT_TRY(dalloc(t, &t->cent, k * n));
  DT_TRY(dalloc(t, &t->cpts, 3 * m));
  DT_TRY(dalloc(t, &t->edges, 2 * n_edges));
  DT_TRY(dalloc(t, &t->ew, n_edges));
  DT_TRY(dalloc(t, &t->iptr, m + 1));
  DT_TRY(dalloc(t, &t->ient, 2 * n_edges));
  DT_TRY(dalloc(t, &t->cpos, k * n));
  DT_TRY(dalloc(t, &t->ipos, 2 * n_edges));
  DT_TRY(dalloc(t, &t->iinfo, 2 * n_edges));
  DT_TRY(dalloc(t, &t->iew, 2 * n_edges));
  DT_TRY(upload(t, t->tp, t_points, 3 * n));
  DT_TRY(upload(t, t->tn, t_normals, 3 * n));
  DT_TRY(upload(t, t->bidx, bidx32.data(), k * n));
  DT_TRY(upload(t, t->bw, bind_w, k * n));
  {
    std::vector<double> bws(k * n);
    for (int64_t i = 0; i < k * n; ++i) bws[i] = std::sqrt(bind_w[i]);
    DT_TRY(upload(t, t->bws, bws.data(), bws.size()));
    DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));  // bws is stack-owned
  }
  DT_TRY(upload(t, t->cptr, cptr.data(), m + 1));
  DT_TRY(upload(t, t->cent, cent.data(), cent.size()));
  DT_TRY(upload(t, t->cpts, ctrl_points, 3 * m));
  DT_TRY(upload(t, t->edges, edges32.data(), 2 * n_edges));
  DT_TRY(upload(t, t->ew, edge_weights, n_edges));
  DT_TRY(upload(t, t->iptr, iptr.data(), m + 1));
  DT_TRY(upload(t, t->ient, ient.data(), ient.size()));
  DT_TRY(upload(t, t->cpos, cpos.data(), cpos.size()));
  DT_TRY(upload(t, t->ipos, ipos.data(), ipos.size()));
  DT_TRY(upload(t, t->iinfo, iinfo.data(), iinfo.size()));
  DT_TRY(upload(t, t->iew, iew.data(), iew.size()));
  // frame buffers
  DT_TRY(dalloc(t, &t->depth, npix));
  DT_TRY(dalloc(t, &t->pixrec, 4 * npix));
  if (k == 4) {
    // the relink's per-point statics packed for 256-bit loads (dt_solver.cuh SolverArgs)
    std::vector<double> pst(16 * n);
    std::vector<int> pi8(8 * n);
    for (int64_t p = 0; p < n; ++p) {
      for (int s2 = 0; s2 < 4; ++s2) {
        pst[16 * p + s2] = bind_w[4 * p + s2];
        pst[16 * p + 4 + s2] = std::sqrt(bind_w[4 * p + s2]);
        pi8[8 * p + s2] = bidx32[4 * p + s2];
        pi8[8 * p + 4 + s2] = cpos[4 * p + s2];
      }
      for (int c = 0; c < 3; ++c) {
        pst[16 * p + 8 + c] = t_points[3 * p + c];
        pst[16 * p + 12 + c] = t_normals[3 * p + c];
      }
      pst[16 * p + 11] = pst[16 * p + 15] = 0.0;
    }
    DT_TRY(dalloc(t, &t->pst, 16 * n));
    DT_TRY(dalloc(t, &t->pi8, 8 * n));
    DT_TRY(upload(t, t->pst, pst.data(), pst.size()));
    DT_TRY(upload(t, t->pi8, pi8.data(), pi8.size()));
    DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));  // pst / pi8 are stack-owned
  }
  DT_TRY(dalloc(t, &t->info, 4));
  DT_TRY(dalloc(t, &t->pstats, 2));
  DT_TRY(dalloc(t, &t->astats, 2));
  DT_TRY(dalloc(t, &t->mptr, m + 1));
  DT_TRY(dalloc(t, &t->mcnt, m));
  DT_TRY(ensure_match_capacity(t, 64));
  // solver state
  DT_TRY(dalloc(t, &t->warp_a, 8 * m));
  DT_TRY(dalloc(t, &t->warp_b, 8 * m));
  DT_TRY(dalloc(t, &t->warps_out, 8 * m));
  DT_TRY(dalloc(t, &t->lam, m));
  DT_TRY(dalloc(t, &t->wa, m));
  DT_TRY(dalloc(t, &t->partial, 27 * m));
  DT_TRY(dalloc(t, &t->delta, 6 * m));
  DT_TRY(dalloc(t, &t->oknorm, 6 * m));
  DT_TRY(dalloc(t, &t->tentT, 12 * m));
  DT_TRY(dalloc(t, &t->crec, 2 * 8 * n));
  DT_TRY(dalloc(t, &t->prow, 2 * k * n * 8));
  DT_TRY(dalloc(t, &t->counts, 1024));
  DT_TRY(dalloc(t, &t->erow, 2 * 2 * 24 * (n_edges > 0 ? n_edges : 1)));
  DT_TRY(dalloc(t, &t->evals, 2 * 3 * (n_edges > 0 ? n_edges : 1)));
  DT_TRY(dalloc(t, &t->bad_flag, 1));
  DT_TRY(dalloc(t, &t->report, 1));
  DT_TRY(dalloc(t, &t->cost_hist, 2 * cfg->max_outer_iters));
  DT_TRY(dalloc(t, &t->lam_hist, 2 * cfg->max_outer_iters));
  DT_TRY(dalloc(t, &t->stalled_hist, cfg->max_outer_iters));
  DT_TRY(dalloc(t, &t->wa_out, m));
  DT_TRY(dalloc(t, &t->out_p, 3 * n));
  DT_TRY(dalloc(t, &t->out_n, 3 * n));
  DT_TRY(dalloc(t, &t->dev_args, 1));
  DT_CHECK_CUDA(cudaMallocHost((void**)&t->h_report, sizeof(dt_report)));
  DT_CHECK_CUDA(cudaMallocHost((void**)&t->h_info, sizeof(int64_t) * 4));
  DT_CHECK_CUDA(cudaMallocHost((void**)&t->h_stats, sizeof(double) * 4));
  DT_CHECK_CUDA(cudaMemcpyAsync(t->warps_out, warps, sizeof(double) * 8 * m, cudaMemcpyHostToDevice, t->stream));
  if (m > M_MAX_SMEM) {
    // large control graph: the global-state solver variant keeps per-CTA transforms and
    // damping here (one slice per CTA of the largest domain: the grid or a cluster)
    int sms = 0;
    DT_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DT_TRY(dalloc(t, &t->gstate, (size_t)std::max(sms, 16) * 13 * m));
  }
  pick_mode(t);
  DT_TRY(push_args(t));
  return DT_OK;
}

int dt_tracker_create(const dt_config* cfg, const double* t_points, const double* t_normals,
                      const int64_t* bind_idx, const double* bind_w, int64_t n, int64_t k,
                      const double* ctrl_points, const double* warps, int64_t m,
                      const int64_t* edges, const double* edge_weights, int64_t n_edges,
                      int device, void* stream, dt_tracker** out) {
  DT_TRY(validate_config(cfg));
  DT_REQUIRE(out != nullptr, DT_ERR_INVALID_ARGUMENT, "out is NULL");
  DT_REQUIRE(m >= 1, DT_ERR_EMPTY_TEMPLATE, "control graph is empty");
  DT_REQUIRE(k >= 1 && k <= KMAX, DT_ERR_UNSUPPORTED, "bind_k outside [1, %d]", KMAX);
  DT_REQUIRE(bind_idx != nullptr && bind_w != nullptr, DT_ERR_NOT_BOUND,
             "template must be bound to the control graph first");
  DT_REQUIRE(n < (1ll << 28), DT_ERR_UNSUPPORTED, "template too large");
  DT_CHECK_CUDA(cudaSetDevice(device));
  dt_tracker* t = new (std::nothrow) dt_tracker();
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "out of host memory");
  const int st = tracker_init(t, cfg, t_points, t_normals, bind_idx, bind_w, n, k, ctrl_points,
                              warps, m, edges, edge_weights, n_edges, device, stream);
  if (st != DT_OK) {
    dt_tracker_destroy(t);
    return st;
  }
  *out = t;
  return DT_OK;
}

int dt_tracker_destroy(dt_tracker* t) {
  if (!t) return DT_OK;
  cudaStreamSynchronize(t->stream);
  drop_graph(t);
  if (t->copy_stream) {
    cudaStreamSynchronize(t->copy_stream);
    cudaStreamDestroy(t->copy_stream);
  }
  if (t->out_stream) {
    cudaStreamSynchronize(t->out_stream);
    cudaStreamDestroy(t->out_stream);
  }
  for (int i = 0; i < 2; ++i) {
    for (cudaEvent_t e : {t->ev_in_ready[i], t->ev_in_free[i], t->ev_done[i], t->ev_out_copied[i]})
      if (e) cudaEventDestroy(e);
    if (t->h_stage[i]) cudaFreeHost(t->h_stage[i]);
  }
  for (auto& e : t->ev)
    if (e) cudaEventDestroy(e);
  if (t->aux_stream) {
    cudaStreamSynchronize(t->aux_stream);
    cudaStreamDestroy(t->aux_stream);
  }
  if (t->ev_fork) cudaEventDestroy(t->ev_fork);
  if (t->ev_join) cudaEventDestroy(t->ev_join);
  // the device buffers come from the stream-ordered pool: returning them is a pool
  // operation, not a synchronous cudaFree each (84 of those measured 4 ms to 0.9 s at
  // the end of a run, varying with the driver's state)
  for (const DevBuf& b : t->bufs) free_buf(t, b);
  for (const DevBuf& b : t->retired) free_buf(t, b);
  cudaStreamSynchronize(t->stream);
  if (t->own_stream) cudaStreamDestroy(t->stream);
  if (t->h_report) cudaFreeHost(t->h_report);
  if (t->h_info) cudaFreeHost(t->h_info);
  if (t->h_stats) cudaFreeHost(t->h_stats);
  delete t;
  return DT_OK;
}

int dt_tracker_set_features(dt_tracker* t, const uint8_t* desc, const double* points, int64_t n_features,
                            const int64_t* bind_idx, const double* bind_w) {
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker is NULL");
  DT_REQUIRE(n_features >= 0, DT_ERR_INVALID_ARGUMENT, "negative feature count");
  DT_REQUIRE(n_features == 0 || (desc != nullptr && points != nullptr), DT_ERR_INVALID_ARGUMENT,
             "descriptors and points are required");
  DT_TRY(dt_tracker_sync(t));  // frames in flight still read the current feature buffers
  drop_graph(t);
  t->n_feat = n_features;
  DT_TRY(ensure_match_capacity(t, n_features));
  DT_TRY(dalloc(t, &t->tdesc, 32 * n_features));
  DT_TRY(dalloc(t, &t->tfeat_pts, 3 * n_features));
  DT_TRY(dalloc(t, &t->tfeat_bidx, t->k * n_features));
  DT_TRY(dalloc(t, &t->tfeat_bw, t->k * n_features));
  DT_TRY(dalloc(t, &t->ham_idx, n_features));
  DT_TRY(dalloc(t, &t->ham_dist, n_features));
  DT_TRY(dalloc(t, &t->ham_packed, n_features));
  DT_CHECK_CUDA(cudaMemsetAsync(t->ham_packed, 0xff, sizeof(unsigned long long) * std::max<int64_t>(1, n_features),
                                t->stream));
  DT_TRY(upload(t, t->tdesc, desc, 32 * n_features));
  DT_TRY(upload(t, t->tfeat_pts, points, 3 * n_features));
  // the match binding depends only on the template-side point (SURVEY §8a invariant):
  // bind every feature once, sigma = graph sampling radius (solver.py:292-296)
  if (bind_idx != nullptr && bind_w != nullptr) {
    DT_TRY(upload_binding(t, bind_idx, bind_w, n_features, false, t->tfeat_bidx, t->tfeat_bw));
  } else {
    DT_TRY(launch_bind_points_i32(t->tfeat_pts, n_features, t->cpts, (int)t->m, (int)t->k,
                                  t->cfg.sampling_radius, t->tfeat_bidx, t->tfeat_bw, t->stream));
  }
  // static control -> (feature, slot) CSR of the ORB path, built on the host once
  {
    const int64_t k = t->k;
    std::vector<int32_t> fb(n_features * k);
    if (n_features > 0) {
      DT_CHECK_CUDA(cudaMemcpyAsync(fb.data(), t->tfeat_bidx, sizeof(int32_t) * fb.size(),
                                    cudaMemcpyDeviceToHost, t->stream));
      DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
    }
    for (const int32_t key : fb)
      DT_REQUIRE(key >= 0 && key < t->m, DT_ERR_INVALID_ARGUMENT,
                 "feature bind index %d outside the control graph (m=%lld)", key, (long long)t->m);
    std::vector<int> keys(fb.begin(), fb.end()), ents(n_features * k), fptr, fent;
    for (int64_t i = 0; i < n_features * k; ++i) ents[i] = (int)i;
    host_csr(keys, ents, (int)t->m, fptr, fent);
    std::vector<int> fpos(n_features * k);
    for (size_t q = 0; q < fent.size(); ++q) fpos[fent[q]] = (int)q;
    DT_TRY(dalloc(t, &t->fptr, t->m + 1));
    DT_TRY(dalloc(t, &t->fent, std::max<int64_t>(1, n_features * k)));
    DT_TRY(dalloc(t, &t->fpos, std::max<int64_t>(1, n_features * k)));
    DT_TRY(dalloc(t, &t->ffo, 3 * std::max<int64_t>(1, n_features)));
    DT_TRY(dalloc(t, &t->ffw, std::max<int64_t>(1, n_features)));
    DT_TRY(dalloc(t, &t->fs_partial, 2 * (n_features / 1024 + 2)));
    DT_TRY(dalloc(t, &t->fs_counter, 1));
    DT_TRY(upload(t, t->fptr, fptr.data(), fptr.size()));
    if (!fent.empty()) {
      DT_TRY(upload(t, t->fent, fent.data(), fent.size()));
      DT_TRY(upload(t, t->fpos, fpos.data(), fpos.size()));
    }
    DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  }
  DT_TRY(push_args(t));
  return DT_OK;
}

int dt_tracker_set_warps(dt_tracker* t, const double* warps, int from_device) {
  DT_REQUIRE(t != nullptr && warps != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  // a pipelined frame may still be copying warps_out to its host buffer
  DT_TRY(dt_tracker_sync(t));
  DT_CHECK_CUDA(cudaMemcpyAsync(t->warps_out, warps, sizeof(double) * 8 * t->m,
                                from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                t->stream));
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  return DT_OK;
}

int dt_tracker_get_warps(dt_tracker* t, double* warps_host) {
  DT_REQUIRE(t != nullptr && warps_host != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_CHECK_CUDA(cudaMemcpyAsync(warps_host, t->warps_out, sizeof(double) * 8 * t->m,
                                cudaMemcpyDeviceToHost, t->stream));
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  return DT_OK;
}

int dt_tracker_set_config(dt_tracker* t, const dt_config* cfg) {
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker is NULL");
  DT_TRY(dt_tracker_sync(t));  // frames in flight use the current histories / staging
  drop_graph(t);
  DT_TRY(validate_config(cfg));
  DT_REQUIRE(cfg->width == t->cfg.width && cfg->height == t->cfg.height, DT_ERR_INVALID_ARGUMENT,
             "camera size cannot change on a live tracker");
  if (cfg->max_outer_iters > t->cfg.max_outer_iters) {
    DT_TRY(dalloc(t, &t->cost_hist, 2 * cfg->max_outer_iters));
    DT_TRY(dalloc(t, &t->lam_hist, 2 * cfg->max_outer_iters));
    DT_TRY(dalloc(t, &t->stalled_hist, cfg->max_outer_iters));
  }
  t->cfg = *cfg;
  pick_mode(t);
  DT_TRY(push_args(t));
  return DT_OK;
}

int dt_tracker_wait(dt_tracker* t);

int dt_tracker_sync(dt_tracker* t) {
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker is NULL");
  while (t->pipe_waited < t->pipe_next) DT_TRY(dt_tracker_wait(t));  // drain the pipeline
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  return reap(t);
}

int dt_track_frame(dt_tracker* t, const dt_frame_input* in, dt_frame_output* out) {
  DT_REQUIRE(t != nullptr && in != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_TRY(check_frame_input(t, in));
  bool used = false;
  DT_TRY(run_frame(t, in, &used));
  t->last_used = used;
  DT_TRY(collect_outputs(t, in, out, used));
  return reap(t);
}

int dt_tracker_get_history(dt_tracker* t, double* cost_history, double* lambda_history,
                           int32_t* stalled);
}  // extern "C"

namespace {

constexpr int STAGE_BASE = 4 + 3 + (int)((sizeof(dt_report) + 7) / 8);
// snapshot words for `it` outer iterations: the base + cost (2 it) + lambda (2 it) + stalled (it)
inline int stage_words(int it) { return STAGE_BASE + 5 * it; }

__global__ void k_stage_outputs(const int64_t* __restrict__ info, const double* __restrict__ astats,
                                const double* __restrict__ pstats, const dt_report* __restrict__ rep,
                                const double* __restrict__ cost_hist, const double* __restrict__ lam_hist,
                                const int32_t* __restrict__ stalled, int it, int64_t* __restrict__ stage) {
  const int i = threadIdx.x;
  if (i < 4) stage[i] = info[i];
  if (i < 2) reinterpret_cast<double*>(stage + 4)[i] = astats[i];
  if (i == 0) reinterpret_cast<double*>(stage + 4)[2] = pstats[0];
  const int nw = (int)((sizeof(dt_report) + 7) / 8);
  if (i < nw) stage[7 + i] = reinterpret_cast<const int64_t*>(rep)[i];
  double* h = reinterpret_cast<double*>(stage + STAGE_BASE);
  for (int j = i; j < 2 * it; j += blockDim.x) {
    h[j] = cost_hist[j];
    h[2 * it + j] = lam_hist[j];
  }
  for (int j = i; j < it; j += blockDim.x) stage[STAGE_BASE + 4 * it + j] = stalled[j];
}

int ensure_pipeline(dt_tracker* t, int64_t n_desc) {
  if (!t->copy_stream) {
    DT_CHECK_CUDA(cudaStreamCreateWithFlags(&t->copy_stream, cudaStreamNonBlocking));
    DT_CHECK_CUDA(cudaStreamCreateWithFlags(&t->out_stream, cudaStreamNonBlocking));
    const int64_t npix = (int64_t)t->cfg.width * t->cfg.height;
    for (int i = 0; i < 2; ++i) {
      DT_CHECK_CUDA(cudaEventCreateWithFlags(&t->ev_in_ready[i], cudaEventDisableTiming));
      DT_CHECK_CUDA(cudaEventCreateWithFlags(&t->ev_in_free[i], cudaEventDisableTiming));
      DT_CHECK_CUDA(cudaEventCreateWithFlags(&t->ev_done[i], cudaEventDisableTiming));
      DT_CHECK_CUDA(cudaEventCreateWithFlags(&t->ev_out_copied[i], cudaEventDisableTiming));
      DT_TRY(dalloc(t, &t->in_depth[i], npix));
      DT_TRY(dalloc(t, &t->stage_info[i], stage_words(t->cfg.max_outer_iters)));
      DT_CHECK_CUDA(cudaMallocHost((void**)&t->h_stage[i],
                                   sizeof(int64_t) * stage_words(t->cfg.max_outer_iters)));
    }
    DT_TRY(dalloc(t, &t->dev_args_slot, 2));
    t->stage_words = stage_words(t->cfg.max_outer_iters);
    t->args_dirty = true;  // the per-slot solver arguments still have to be written
  }
  if (t->stage_words < stage_words(t->cfg.max_outer_iters)) {  // more iterations since (set_config)
    t->stage_words = stage_words(t->cfg.max_outer_iters);
    for (int i = 0; i < 2; ++i) {
      DT_TRY(dalloc(t, &t->stage_info[i], t->stage_words));
      DT_CHECK_CUDA(cudaFreeHost(t->h_stage[i]));
      DT_CHECK_CUDA(cudaMallocHost((void**)&t->h_stage[i], sizeof(int64_t) * t->stage_words));
    }
  }
  if (n_desc > t->in_desc_cap) {
    const int64_t cap = std::max<int64_t>(n_desc, 256);
    for (int i = 0; i < 2; ++i) {
      DT_TRY(dalloc(t, &t->in_desc[i], 32 * cap));
      DT_TRY(dalloc(t, &t->in_kp[i], 2 * cap));
    }
    t->in_desc_cap = cap;
    drop_graph(t);  // captured bodies read the old staging buffers
  }
  return DT_OK;
}

// staging slots of the pipelined path for match pairs / references / PFM payloads
int ensure_pipeline_pairs(dt_tracker* t, int64_t n_pairs, int64_t n_refs, bool pfm) {
  if (n_pairs > t->in_pair_cap) {
    const int64_t cap = std::max<int64_t>(n_pairs, 256);
    for (int i = 0; i < 2; ++i) {
      DT_TRY(dalloc(t, &t->in_msrc[i], 3 * cap));
      DT_TRY(dalloc(t, &t->in_mdst[i], 3 * cap));
    }
    t->in_pair_cap = cap;
  }
  if (n_refs > t->in_refs_cap) {
    const int64_t cap = std::max<int64_t>(n_refs, 64);
    for (int i = 0; i < 2; ++i) DT_TRY(dalloc(t, &t->in_refs[i], cap));
    t->in_refs_cap = cap;
  }
  if (pfm && !t->in_dstage[0]) {
    const int64_t npix = (int64_t)t->cfg.width * t->cfg.height;
    for (int i = 0; i < 2; ++i) DT_TRY(dalloc(t, &t->in_dstage[i], npix));
  }
  return DT_OK;
}

// host side of a finished pipelined frame: the report from the staged snapshot
void finish_pending(dt_tracker* t, int slot) {
  dt_tracker::Pending& pd = t->pend[slot];
  const int64_t* st = t->h_stage[slot];
  const double* stats = reinterpret_cast<const double*>(st + 4);
  dt_report R;
  std::memcpy(&R, st + 7, sizeof(dt_report));
  R.frame_id = pd.frame_id;
  if (pd.used) {
    R.n_matches = (int32_t)st[2];
    R.n_preselected = (int32_t)stats[1];
    R.match_weight_sum = stats[0];
    R.preselect_status = (int32_t)st[0];
    R.preselect_reference = (int32_t)st[1];
    R.preselect_support = stats[2];
  } else {
    R.n_matches = R.n_preselected = 0;
    R.match_weight_sum = R.preselect_support = 0.0;
    R.preselect_status = DT_OK;
    R.preselect_reference = -1;
  }
  if (pd.out.report) *pd.out.report = R;
  const int it = t->cfg.max_outer_iters;
  const double* h = reinterpret_cast<const double*>(st + STAGE_BASE);
  if (pd.out.cost_history) std::memcpy(pd.out.cost_history, h, sizeof(double) * 2 * it);
  if (pd.out.lambda_history) std::memcpy(pd.out.lambda_history, h + 2 * it, sizeof(double) * 2 * it);
  if (pd.out.stalled)
    for (int j = 0; j < it; ++j) pd.out.stalled[j] = (int32_t)st[STAGE_BASE + 4 * it + j];
  pd.active = false;
}

}  // namespace

extern "C" {

int dt_tracker_wait(dt_tracker* t) {
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker is NULL");
  if (t->pipe_waited >= t->pipe_next) return DT_OK;  // nothing in flight
  const int slot = (int)(t->pipe_waited % 2);
  DT_CHECK_CUDA(cudaEventSynchronize(t->ev_out_copied[slot]));
  finish_pending(t, slot);
  ++t->pipe_waited;
  return DT_OK;
}

int dt_track_frame_submit(dt_tracker* t, const dt_frame_input* in, dt_frame_output* out) {
  DT_REQUIRE(t != nullptr && in != nullptr && out != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_REQUIRE(!in->on_device, DT_ERR_INVALID_ARGUMENT, "dt_track_frame_submit takes host inputs");
  DT_TRY(check_frame_input(t, in));
  DT_REQUIRE(in->depth != nullptr, DT_ERR_INVALID_ARGUMENT, "depth is required");
  DT_REQUIRE(in->normals == nullptr, DT_ERR_UNSUPPORTED, "the pipelined path computes the normals itself");
  DT_REQUIRE(in->match_w == nullptr && in->match_bidx == nullptr, DT_ERR_UNSUPPORTED,
             "the pipelined path preselects and binds the pairs itself");
  // at most two frames in flight
  if (t->pipe_next - t->pipe_waited >= 2) DT_TRY(dt_tracker_wait(t));
  const int64_t nd = in->frame_desc ? in->n_frame : 0;
  const int64_t np = (in->use_matches && in->frame_desc == nullptr) ? in->n_pairs : 0;
  const int64_t nref = in->refs != nullptr ? in->n_refs : 0;
  DT_TRY(ensure_pipeline(t, nd));
  DT_TRY(ensure_pipeline_pairs(t, np, nref, in->depth_kind == DT_DEPTH_PFM));
  const int slot = (int)(t->pipe_next % 2);
  const int64_t npix = (int64_t)t->cfg.width * t->cfg.height;
  cudaStream_t cs = t->copy_stream, s = t->stream;
  // stage the inputs once the frame that used this slot has consumed them
  DT_CHECK_CUDA(cudaStreamWaitEvent(cs, t->ev_in_free[slot], 0));
  const bool pfm = in->depth_kind == DT_DEPTH_PFM;
  if (pfm)  // the file's f32 payload (half the bytes); decoded on the compute stream
    DT_CHECK_CUDA(cudaMemcpyAsync(t->in_dstage[slot], in->depth, sizeof(float) * npix,
                                  cudaMemcpyHostToDevice, cs));
  else
    DT_CHECK_CUDA(cudaMemcpyAsync(t->in_depth[slot], in->depth, sizeof(double) * npix,
                                  cudaMemcpyHostToDevice, cs));
  if (np > 0) {
    DT_CHECK_CUDA(cudaMemcpyAsync(t->in_msrc[slot], in->match_src, sizeof(double) * 3 * np,
                                  cudaMemcpyHostToDevice, cs));
    DT_CHECK_CUDA(cudaMemcpyAsync(t->in_mdst[slot], in->match_dst, sizeof(double) * 3 * np,
                                  cudaMemcpyHostToDevice, cs));
  }
  if (nref > 0)
    DT_CHECK_CUDA(cudaMemcpyAsync(t->in_refs[slot], in->refs, sizeof(int64_t) * nref,
                                  cudaMemcpyHostToDevice, cs));
  if (nd > 0) {
    DT_CHECK_CUDA(cudaMemcpyAsync(t->in_desc[slot], in->frame_desc, 32 * nd, cudaMemcpyHostToDevice, cs));
    DT_CHECK_CUDA(cudaMemcpyAsync(t->in_kp[slot], in->frame_kp, sizeof(int32_t) * 2 * nd,
                                  cudaMemcpyHostToDevice, cs));
  }
  DT_CHECK_CUDA(cudaEventRecord(t->ev_in_ready[slot], cs));
  // compute: wait for the inputs; the solver (which rewrites warps / report / weights)
  // waits until the previous frame's outputs are copied out
  DT_CHECK_CUDA(cudaStreamWaitEvent(s, t->ev_in_ready[slot], 0));
  // a previous frame whose annotated matches are still being copied out: its preselection
  // arrays must not be rewritten before that copy (the usual pre-solver wait covers the
  // solver's outputs only)
  if (t->pipe_next > 0 && t->pend[1 - slot].active &&
      (t->pend[1 - slot].out.match_weights || t->pend[1 - slot].out.match_flags) &&
      t->pend[1 - slot].out.match_capacity > 0)
    DT_CHECK_CUDA(cudaStreamWaitEvent(s, t->ev_out_copied[1 - slot], 0));
  if (pfm) DT_TRY(launch_depth_from_pfm(t->in_dstage[slot], t->cfg.height, t->cfg.width, 0,
                                        t->in_depth[slot], s));
  dt_frame_input din = *in;
  din.on_device = 1;
  din.depth_kind = DT_DEPTH_F64;
  din.depth = t->in_depth[slot];
  din.frame_desc = nd > 0 ? t->in_desc[slot] : nullptr;
  din.frame_kp = nd > 0 ? t->in_kp[slot] : nullptr;
  if (np > 0) {
    din.match_src = t->in_msrc[slot];
    din.match_dst = t->in_mdst[slot];
  }
  if (nref > 0) din.refs = t->in_refs[slot];
  t->pre_solver_wait = t->pipe_next > 0 ? t->ev_out_copied[1 - slot] : nullptr;
  t->in_set = 1 + slot;  // the frame reads the staging slot in place
  bool used = false;
  const int st = run_frame(t, &din, &used);
  t->pre_solver_wait = nullptr;
  t->in_set = 0;
  DT_TRY(st);
  t->last_used = used;
  DT_CHECK_CUDA(cudaEventRecord(t->ev_in_free[slot], s));
  k_stage_outputs<<<1, 64, 0, s>>>(t->info, t->astats, t->pstats, t->report, t->cost_hist, t->lam_hist,
                                   t->stalled_hist, t->cfg.max_outer_iters, t->stage_info[slot]);
  DT_CHECK_LAUNCH();
  DT_CHECK_CUDA(cudaEventRecord(t->ev_done[slot], s));
  // outputs back on their own stream while the next frame computes (a single copy stream
  // would queue the next frame's input staging behind this frame's output copies)
  cudaStream_t os = t->out_stream;
  DT_CHECK_CUDA(cudaStreamWaitEvent(os, t->ev_done[slot], 0));
  if (out->warps)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->warps, t->warps_out, sizeof(double) * 8 * t->m, cudaMemcpyDeviceToHost, os));
  if (out->points)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->points, t->out_p, sizeof(double) * 3 * t->n, cudaMemcpyDeviceToHost, os));
  if (out->normals)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->normals, t->out_n, sizeof(double) * 3 * t->n, cudaMemcpyDeviceToHost, os));
  if (out->control_data_weights)
    DT_CHECK_CUDA(cudaMemcpyAsync(out->control_data_weights, t->wa_out, sizeof(double) * t->m,
                                  cudaMemcpyDeviceToHost, os));
  const int64_t mcap = std::min<int64_t>(out->match_capacity, t->match_cap);
  if (mcap > 0) {
    // the annotated matches (MatchSet weights / flags): the next frame's preselection
    // waits for these copies (wait_matches below)
    if (out->match_weights)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->match_weights, t->m_w, sizeof(double) * mcap, cudaMemcpyDeviceToHost, os));
    if (out->match_flags)
      DT_CHECK_CUDA(cudaMemcpyAsync(out->match_flags, t->m_flags, mcap, cudaMemcpyDeviceToHost, os));
  }
  DT_CHECK_CUDA(cudaMemcpyAsync(t->h_stage[slot], t->stage_info[slot], sizeof(int64_t) * t->stage_words,
                                cudaMemcpyDeviceToHost, os));
  DT_CHECK_CUDA(cudaEventRecord(t->ev_out_copied[slot], os));
  dt_tracker::Pending& pd = t->pend[slot];
  pd.active = true;
  pd.used = used;
  pd.frame_id = in->frame_id;
  pd.out = *out;
  ++t->pipe_next;
  return DT_OK;
}

int dt_tracker_get_history(dt_tracker* t, double* cost_history, double* lambda_history,
                           int32_t* stalled) {
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker is NULL");
  const int it = t->cfg.max_outer_iters;
  if (cost_history)
    DT_CHECK_CUDA(cudaMemcpyAsync(cost_history, t->cost_hist, sizeof(double) * 2 * it, cudaMemcpyDeviceToHost, t->stream));
  if (lambda_history)
    DT_CHECK_CUDA(cudaMemcpyAsync(lambda_history, t->lam_hist, sizeof(double) * 2 * it, cudaMemcpyDeviceToHost, t->stream));
  if (stalled)
    DT_CHECK_CUDA(cudaMemcpyAsync(stalled, t->stalled_hist, sizeof(int32_t) * it, cudaMemcpyDeviceToHost, t->stream));
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  return DT_OK;
}

int dt_tracker_device_outputs(dt_tracker* t, double** warps, double** points, double** normals) {
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker is NULL");
  if (warps) *warps = t->warps_out;
  if (points) *points = t->out_p;
  if (normals) *normals = t->out_n;
  return DT_OK;
}

int dt_tracker_last_launches(dt_tracker* t) { return t ? t->launches : 0; }

int dt_track_frame_async(dt_tracker* t, const dt_frame_input* in) {
  DT_REQUIRE(t != nullptr && in != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_TRY(check_frame_input(t, in));
  bool used = false;
  DT_TRY(run_frame(t, in, &used));
  t->last_used = used;
  return DT_OK;
}

int dt_tracker_collect(dt_tracker* t, const dt_frame_input* in, dt_frame_output* out) {
  DT_REQUIRE(t != nullptr && in != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  return collect_outputs(t, in, out, t->last_used);
}

int dt_tracker_get_trace(dt_tracker* t, long long* buf, int cap) {
  DT_REQUIRE(t != nullptr && buf != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!t->trace) return 0;
  long long n = 0;
  DT_CHECK_CUDA(cudaMemcpyAsync(&n, t->trace, sizeof(long long), cudaMemcpyDeviceToHost, t->stream));
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  const long long cnt = std::min<long long>(n, cap);
  if (cnt > 0)
    DT_CHECK_CUDA(cudaMemcpyAsync(buf, t->trace + 1, sizeof(long long) * 2 * cnt,
                                  cudaMemcpyDeviceToHost, t->stream));
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  return (int)cnt;
}

int dt_tracker_get_arrivals(dt_tracker* t, long long* buf, int cap) {
  DT_REQUIRE(t != nullptr && buf != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!t->arrivals) return 0;
  long long hdr[2] = {0, 0};
  DT_CHECK_CUDA(cudaMemcpyAsync(hdr, t->arrivals, sizeof(hdr), cudaMemcpyDeviceToHost, t->stream));
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  // the header + every CTA's stamps (+ the debug per-warp area when cap reaches it)
  const long long alloc = 2 + 1024LL * t->arr_cap + 1024LL * 32;
  const long long want = std::min<long long>(cap, cap > 2 + 1024LL * t->arr_cap
                                                      ? alloc
                                                      : 2 + hdr[0] * (long long)t->arr_cap);
  if (want > 0)
    DT_CHECK_CUDA(cudaMemcpyAsync(buf, t->arrivals, sizeof(long long) * want, cudaMemcpyDeviceToHost,
                                  t->stream));
  DT_CHECK_CUDA(cudaStreamSynchronize(t->stream));
  return t->arr_cap;
}

void* dt_tracker_stream(dt_tracker* t) { return t ? (void*)t->stream : nullptr; }

int dt_tracker_set_profiling(dt_tracker* t, int on) {
  DT_REQUIRE(t != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker is NULL");
  drop_graph(t);
  if (on && !t->ev[0])
    for (auto& e : t->ev) DT_CHECK_CUDA(cudaEventCreate(&e));
  if (on && !t->trace) {
    t->trace_cap = 4096;
    DT_TRY(dalloc(t, &t->trace, 1 + 2 * (size_t)t->trace_cap));
    t->arr_cap = 256;
    DT_TRY(dalloc(t, &t->arrivals, 2 + 1024 * (size_t)t->arr_cap + 1024 * 32));
  }
  t->profiling = on != 0;
  DT_TRY(push_args(t));
  return DT_OK;
}

int dt_tracker_get_phase_ms(dt_tracker* t, float* ms) {
  DT_REQUIRE(t != nullptr && ms != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_REQUIRE(t->profiling, DT_ERR_INVALID_ARGUMENT, "profiling is off");
  DT_CHECK_CUDA(cudaEventSynchronize(t->ev[DT_N_PHASES]));
  for (int i = 0; i < DT_N_PHASES; ++i) DT_CHECK_CUDA(cudaEventElapsedTime(&ms[i], t->ev[i], t->ev[i + 1]));
  return DT_OK;
}

int dt_track_frames_batched(dt_tracker** trackers, const dt_frame_input* inputs,
                            dt_frame_output* outputs, int32_t n_trackers, void* stream) {
  (void)stream;
  // independent sequences: each tracker enqueues on its own stream; the streams overlap
  // on the device (one cluster per sequence)
  DT_REQUIRE(n_trackers >= 0 && (n_trackers == 0 || (trackers != nullptr && inputs != nullptr)),
             DT_ERR_INVALID_ARGUMENT, "NULL argument");
  for (int32_t i = 0; i < n_trackers; ++i) {
    DT_REQUIRE(trackers[i] != nullptr, DT_ERR_INVALID_ARGUMENT, "tracker %d is NULL", (int)i);
    DT_TRY(check_frame_input(trackers[i], &inputs[i]));
  }
  std::vector<char> used(n_trackers, 0);
  for (int32_t i = 0; i < n_trackers; ++i) {
    bool u = false;
    DT_TRY(enqueue_frame(trackers[i], &inputs[i], &u));
    used[i] = u ? 1 : 0;
  }
  for (int32_t i = 0; i < n_trackers; ++i)
    DT_TRY(collect_outputs(trackers[i], &inputs[i], outputs ? &outputs[i] : nullptr, used[i] != 0));
  return DT_OK;
}

}  // extern "C"
