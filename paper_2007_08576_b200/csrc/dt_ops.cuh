// dt_ops.cuh -- internal declarations shared between the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dt_common.cuh"

namespace dt {

// Per-correspondence ICP record (stage 1 of kernels.icp_reduce): raw residual, robust
// square-root weight, gradient of r w.r.t. the blended warp (n_obs^T G), blend signs.
struct IcpRow {
  double r;
  double rs;
  double gn[8];
  unsigned sgn;
};

// Per-match feature record (stage 1 of kernels.feature_reduce).
struct FeatRow {
  double res[3];
  double w;
  double G[24];
  unsigned sgn;
};

template <typename KeyT>
int build_csr(const KeyT* keys, int64_t ne, int m, int* ptr, int* ent, int* scratch_cnt,
              cudaStream_t s);

int launch_depth_from_pfm(const float* payload, int64_t h, int64_t w, int big_endian, double* depth,
                          cudaStream_t s);
int launch_observation_normals(const double* depth, int64_t h, int64_t w, double fx, double fy,
                               double cx, double cy, double zmin, double zmax, double* normals,
                               uint8_t* valid, cudaStream_t s, double* pix = nullptr);
// the solver's 32-byte pixel records {depth or NaN, normal xyz} from depth + given normals
int launch_pack_pixels(const double* depth, const double* normals, int64_t npix, double zmin,
                       double zmax, double* pix, cudaStream_t s);
int launch_bind_points_i32(const double* pts, int64_t n, const double* ctrl, int m, int k,
                           double sigma, int32_t* idx, double* w, cudaStream_t s);

// ORB path: scatter the preselected pairs back to their template features (weight 0 for
// every feature without an active match) and the report statistics n_preselected and
// match_weight_sum (solver.py:368-370), summed in a fixed order (warp sums of each
// 1024-thread round, warps in order). Whole CTA of 1024 threads.
struct FeatureScatter {
  int64_t n_feat;
  const double* dst;       // (n, 3) observed points of the compacted matches
  const int32_t* feat_id;  // (n,) template feature of each match
  double* ffo;             // (n_feat, 3) observed point per feature
  double* ffw;             // (n_feat,) weight per feature (zeroed by the match build)
  int64_t* n_active;
  double* stats;           // [match_weight_sum, n_preselected]
  double* partial;         // scratch: 2 per 1024-match round
  unsigned* counter;       // scratch: rounds done (reset by the last)
};

// One 1024-match round [base, base + blockDim) of the ORB-path scatter: the weights and
// observed points to their template features; returns (to thread 0) the round's weight
// sum (warp sums in warp order) and flag count -- the rounds are then summed in round
// order, the order k_active uses (solver.py:368-370).
__device__ __forceinline__ void feature_scatter_round(const FeatureScatter& F, int64_t n,
                                                      int64_t base, const double* weights,
                                                      const uint8_t* flags, double* cs_out,
                                                      int* flg_out) {
  __shared__ double s_fsum[32];
  __shared__ int s_fcnt[32];
  const int64_t j = base + threadIdx.x;
  const bool in = j < n;
  const double w = in ? weights[j] : 0.0;
  if (in) {
    const int f = F.feat_id[j];
    F.ffw[f] = w;
    F.ffo[3 * f] = F.dst[3 * j];
    F.ffo[3 * f + 1] = F.dst[3 * j + 1];
    F.ffo[3 * f + 2] = F.dst[3 * j + 2];
  }
  const double v = warp_sum(w);
  int flg = (in && flags[j]) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) flg += __shfl_xor_sync(0xffffffffu, flg, o);
  if ((threadIdx.x & 31) == 0) {
    s_fsum[threadIdx.x >> 5] = v;
    s_fcnt[threadIdx.x >> 5] = flg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double cs = 0.0;
    int nf = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) {
      cs += s_fsum[w2];
      nf += s_fcnt[w2];
    }
    *cs_out = cs;
    *flg_out = nf;
  }
}

// dt_match.cu
int launch_hamming(const uint8_t* tdesc, int64_t nt, const uint8_t* fdesc, int64_t nf,
                   int32_t* best_idx, int32_t* best_dist, cudaStream_t s,
                   unsigned long long* packed = nullptr, bool packed_ready = false);
struct PreselectWork;
// ORB path: the Hamming winners -> match list (k_build_matches' rule) inputs
struct OrbMatchIn {
  int64_t nt;                          // template features
  const unsigned long long* packed;    // (nt) (distance << 32) | frame index
  int max_ham;
  const int32_t* kp;                   // (nf, 2) frame keypoints
  int64_t nf;
  const double* depth;
  double zmin, zmax;
  int width, height;
  double fx, fy, cx, cy;
  const double* tpts;                  // (nt, 3) template feature points
};
struct PreselectOrbOut {
  double* m_src;       // (n, 3) compacted matches (published by CTA 0)
  double* m_dst;
  int32_t* m_feat;
  int64_t* n_out;
  double* weights;     // (n) preselected weights / flags / residuals
  uint8_t* flags;
  double* residuals;
  int64_t* info;       // [status, winning reference]
  double* support;     // winning support
  FeatureScatter fs;   // the scatter to template features + report statistics
  unsigned long long* packed_reset;  // = packed: reset for the next frame's atomicMin
  unsigned* done;      // CTAs finished (the last resets it)
};
// Match build + preselection + final of the ORB path in one launch (dt_match.cu). The
// feature count must fit the shared-memory copy (ORB_FUSED_MAX).
constexpr int64_t ORB_FUSED_MAX = 4000;
int launch_preselect_orb(const OrbMatchIn& in, const int64_t* refs, int64_t n_refs, double H, int iters,
                         double inlier_min, double min_support, double* ref_support, double* ref_rot,
                         uint8_t* ref_valid, const PreselectOrbOut& out, cudaStream_t s, int shared_gpu);
int launch_preselect(const double* src, const double* dst, const int64_t* n_dev, int64_t n_max,
                     const int64_t* refs, int64_t n_refs, int exhaustive, double H, int iters,
                     double inlier_min, double min_support, double* weights, uint8_t* flags,
                     double* residuals, double* rotation, int64_t* info, double* support,
                     double* ref_support, double* ref_rot, uint8_t* ref_valid, cudaStream_t s,
                     const FeatureScatter* scatter = nullptr, int shared_gpu = 0);

// dt_solver.cu
int solver_max_cluster(int device);

}  // namespace dt
