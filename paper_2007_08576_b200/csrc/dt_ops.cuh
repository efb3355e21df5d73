// dt_ops.cuh -- internal declarations shared between the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

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

int launch_observation_normals(const double* depth, int64_t h, int64_t w, double fx, double fy,
                               double cx, double cy, double zmin, double zmax, double* normals,
                               uint8_t* valid, cudaStream_t s);
int launch_bind_points_i32(const double* pts, int64_t n, const double* ctrl, int m, int k,
                           double sigma, int32_t* idx, double* w, cudaStream_t s);

// dt_match.cu
int launch_hamming(const uint8_t* tdesc, int64_t nt, const uint8_t* fdesc, int64_t nf,
                   int32_t* best_idx, int32_t* best_dist, cudaStream_t s,
                   unsigned long long* packed = nullptr);
struct PreselectWork;
int launch_preselect(const double* src, const double* dst, const int64_t* n_dev, int64_t n_max,
                     const int64_t* refs, int64_t n_refs, int exhaustive, double H, int iters,
                     double inlier_min, double min_support, double* weights, uint8_t* flags,
                     double* residuals, double* rotation, int64_t* info, double* support,
                     double* ref_support, double* ref_rot, uint8_t* ref_valid, cudaStream_t s);

// dt_solver.cu
int solver_max_cluster(int device);

}  // namespace dt
