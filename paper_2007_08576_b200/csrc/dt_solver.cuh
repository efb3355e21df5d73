// dt_solver.cuh -- the fused per-frame Levenberg-Marquardt solver (solver.solve_frame,
// solver.py:267-378) as one persistent kernel per frame: either one thread-block
// cluster per sequence (batched sequences) or one cooperative grid over every SM
// (lowest single-sequence latency).
#pragma once

#include <cstdint>

#include "../../include/deformtrack_b200.h"

namespace dt {

#ifndef DT_SOLVER_THREADS
#define DT_SOLVER_THREADS 256
#endif
constexpr int SOLVER_THREADS = DT_SOLVER_THREADS;
constexpr int CHUNK = 32;  // items per deterministic partial sum (one per lane)

struct SolverArgs {
  // sizes
  int n, k, m, n_edges, height, width, max_outer, max_retries;
  int nch_p, nch_m, nch_e;  // value-pass chunk counts (points, matches, edges)
  // camera, gates and energy weights
  double fx, fy, cx, cy, gate, cos_gate;
  double tukey, fw, arap_w, angle_w, rot_w, data_floor;
  double sq_angle_w, sq_rot_w;  // sqrt(angle_w), sqrt(rot_w)
  double inv_tukey;             // 1 / tukey scale
  // damping schedule and tolerances (SolverConfig, solver.py:43-71)
  double lam_init, lam_dec, lam_inc, lam_min, lam_max, step_tol, cost_tol;
  // bound template (static per sequence)
  const double* tp;
  const double* tn;
  const int32_t* bidx;
  const double* bw;
  const double* bws;  // (n*k) sqrt of the binding weights (correctly rounded, = the reference's sqrt(alpha))
  const int* cptr;   // control -> template (point, slot) entries, encoded (p << 3) | slot
  const int* cent;
  const int* cpos;   // (n*k) inverse: CSR position of (point, slot)
  // control graph (static)
  const double* cpts;
  const int32_t* edges;
  const double* ew;
  const int* iptr;   // control -> incident (edge << 1) | side
  const int* ient;
  const int* ipos;   // (2E) inverse: CSR position of (edge, side)
  const int* iinfo;  // (2E) per CSR position: (other endpoint << 1) | side
  const double* iew; // (2E) per CSR position: edge weight
  // k = 4 only: the per-point static inputs of a relink packed for 256-bit loads
  const double* pst;  // n x 16: alpha[4], sqrt(alpha)[4], template point xyz + pad, normal xyz + pad
  const int* pi8;     // n x 8: bind index[4], control-CSR position[4]
  // frame observation: per pixel {depth if valid else NaN, observed normal xyz} (32 B)
  const double* pixrec;
  // active feature matches of the frame (compacted on the device)
  const int64_t* n_active;
  const double* fp;
  const double* fo;
  const double* fwt;
  const int32_t* fbidx;
  const double* fbw;
  const int* mptr;   // control -> (match * k + slot) entries
  const int* ment;
  const int* mpos;   // (Ma*k) inverse: CSR position of (match, slot)
  // solver state / scratch
  double* warp_a;    // warm start in, scratch
  double* warp_b;    // scratch
  double* warps_out; // solution
  double* lam;
  double* wa;
  double* gstate;    // m > M_MAX_SMEM only: per CTA 12m transforms + m damping
  double* partial;   // m x 27 normal-equation columns
  double* csum;      // 2 sets x (nch_p + nch_m + nch_e) deterministic chunk sums
  double* erow;      // 2 x (2E) x 24: per CSR position the 3 unit rigidity rows of that
                     // bin (length, angle 0->1, angle 1->0; [J0..J5, value, 0])
  double* evals;     // 2 x (E) x 3: length / angle 0->1 / angle 1->0 values
  double* delta;     // m x 6
  double* tentT;     // m x 12 rigid transforms (R, t) of the tentative warps
  double* oknorm;    // 2 parities x 3m: ok, step norm, rigidity cost of the control's bins
  // linearization, double-buffered: the value pass at a tentative iterate relinearizes
  // there speculatively into the other buffer, which becomes current when the step is
  // accepted. Per point: the correspondence + robust weight (frozen for the tentative
  // value passes); per (point, slot) and (match, slot, component): the normal-equation
  // row [J0..J5, sqrt(w) r, sqrt(w)] of its control, stored at its control-CSR position
  // so that every control's rows are contiguous
  double* crec;      // 2 x n x 8 correspondence records (64 B): observed point xyz, robust
                     // sqrt weight, observed normal xyz, valid (1 / 0)
  double* prow;      // 2 x (n*k) x 8 point rows
  double* mrow;      // 2 x (Ma*k*3) x 8 match rows
  int ma_cap;        // match capacity Ma (stride between the two match row buffers)
  int* counts;       // per-CTA correspondence counts (<= 1024 CTAs)
  // outputs
  dt_report* report;
  double* cost_hist;  // max_outer x 2
  double* lam_hist;   // max_outer x 2
  int32_t* stalled_hist;
  double* wa_out;     // m control_data_weights
  double* out_p;      // optional (n x 3): the template warped by the solution (tracking.py:87)
  double* out_n;      // optional (n x 3): its rotated normals
  // optional in-kernel phase trace (CTA 0, thread 0): trace[0] = count, then
  // (code, globaltimer ns) pairs
  long long* trace;
  int trace_cap;
  // optional per-CTA barrier arrival stamps: arrivals[0] = CTAs, [1] = count,
  // arrivals[2 + rank * arr_cap + b]
  long long* arrivals;
  int arr_cap;
  // last-arriver reduction slots (see red_commit): RED_SLOTS x (2 G + 2) doubles and
  // RED_SLOTS x (G + 1) counters, G = red_g groups of 32 items
  double* red;
  unsigned* redc;
  int red_g;
};

constexpr int RED_SLOTS = 5;

// control graphs up to this size keep their state in shared memory; larger ones run the
// global-state kernel variant (needs SolverArgs::gstate)
constexpr int M_MAX_SMEM = 1300;
size_t solver_smem_bytes(int m);
// mode: 0 = one cluster of `cluster` CTAs per sequence; 1 = one cooperative grid over
// every SM for a single sequence
int solver_launch(const SolverArgs* d_args, int n_seq, int cluster, int m_max, int k, int grid_mode,
                  cudaStream_t s);
int solver_pick_cluster(int device, int requested, int m_max);
int solver_grid_blocks(int device, int m_max);

}  // namespace dt
