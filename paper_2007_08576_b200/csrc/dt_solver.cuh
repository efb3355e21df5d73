// dt_solver.cuh -- the fused per-frame Levenberg-Marquardt solver (solver.solve_frame,
// solver.py:267-378) as one thread-block-cluster kernel per sequence.
#pragma once

#include <cstdint>

#include "../../include/deformtrack_b200.h"

namespace dt {

struct SolverArgs {
  // sizes
  int n, k, m, n_edges, height, width, max_outer, max_retries;
  // camera, gates and energy weights
  double fx, fy, cx, cy, gate, cos_gate;
  double tukey, fw, arap_w, angle_w, rot_w, data_floor;
  // damping schedule and tolerances (SolverConfig, solver.py:43-71)
  double lam_init, lam_dec, lam_inc, lam_min, lam_max, step_tol, cost_tol;
  // bound template (static per sequence)
  const double* tp;
  const double* tn;
  const int32_t* bidx;
  const double* bw;
  const int* cptr;   // control -> template (point, slot) entries, encoded (p << 3) | slot
  const int* cent;
  // control graph (static)
  const double* cpts;
  const int32_t* edges;
  const double* ew;
  const int* iptr;   // control -> incident (edge << 1) | side
  const int* ient;
  // frame observation
  const double* depth;
  const uint8_t* dvalid;
  const double* onrm;
  // active feature matches of the frame (compacted on the device)
  const int64_t* n_active;
  const double* fp;
  const double* fo;
  const double* fwt;
  const int32_t* fbidx;
  const double* fbw;
  const int* mptr;   // control -> (match * k + slot) entries
  const int* ment;
  // solver state / scratch
  double* warp_a;    // warm start in, scratch
  double* warp_b;    // scratch
  double* warps_out; // solution
  double* lam;
  double* wa;
  double* partial;   // m x 27
  double* cost3;     // m x 3 (icp, feature, arap) of the linearization pass
  double* cost3_t;   // m x 3 of the tentative (value) pass
  double* delta;     // m x 6
  double* oknorm;    // 2 parities x m x 2 (ok, step norm)
  uint8_t* cvalid;   // per template point: correspondence valid
  double* cobs;      // n x 3 observed point
  double* cnrm;      // n x 3 observed normal
  double* pr_r;      // n raw residual
  double* pr_rs;     // n robust sqrt weight (frozen for the tentative passes)
  double* pr_gn;     // n x 8 gradient of r w.r.t. the blend
  uint8_t* pr_sgn;   // n blend signs (bit per slot)
  double* fr_res;    // Ma x 3
  double* fr_G;      // Ma x 24
  uint8_t* fr_sgn;   // Ma
  int* cta_counts;   // cluster-size scratch
  // outputs
  dt_report* report;
  double* cost_hist;  // max_outer x 2
  double* lam_hist;   // max_outer x 2
  int32_t* stalled_hist;
  double* wa_out;     // m control_data_weights
};

constexpr int SOLVER_THREADS = 256;

size_t solver_smem_bytes(int m);
int solver_launch(const SolverArgs* d_args, int n_seq, int cluster, int m_max, cudaStream_t s);
int solver_pick_cluster(int device, int requested, int m_max);

}  // namespace dt
