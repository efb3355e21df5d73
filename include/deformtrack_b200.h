/*
 * deformtrack_b200.h -- C-ABI of the B200 (sm_100a) deformation-tracking hot path.
 *
 * The reference (arXiv 2007.08576, /root/reference/pkg/src/deformtrack) is a pure
 * Python/numba package with no FFI of its own. The entry points below replace the
 * reference functions named in each comment one for one: the operator-level ones
 * mirror the numba kernels' positional signatures (kernels.py) and the numpy
 * helpers around them, the frame-level ones mirror solver.solve_frame /
 * tracking.track_frame. INTEGRATION.md shows the ctypes binding a maintainer of the
 * reference would add.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch types cross this boundary;
 *   - operator-level calls take DEVICE pointers and a cudaStream_t passed as void*;
 *     they are asynchronous on that stream;
 *   - dtypes follow the reference: float64 for geometry, int64 for indices, uint8 for
 *     boolean masks (numpy bool is one byte);
 *   - every call returns a dt_status; dt_last_error() gives the message of the last
 *     failure on the calling thread;
 *   - the library holds no global numeric state (the reference's process-global
 *     numba.set_num_threads, solver.py:288, has no equivalent here); one dt_tracker
 *     handle per sequence, one stream per handle; different handles may be driven from
 *     different host threads, one handle from one thread at a time;
 *   - array sizes are trusted: the Python layer (paper_2007_08576_b200) checks shapes
 *     before calling; index arrays are range-checked where the kernels would otherwise
 *     read out of bounds (template / feature / match bindings, edges).
 */
#ifndef DEFORMTRACK_B200_H
#define DEFORMTRACK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror deformtrack/exceptions.py:4-49. */
typedef enum {
  DT_OK = 0,
  DT_ERR_INVALID_ARGUMENT = 1,     /* ValueError                                  */
  DT_ERR_CUDA = 2,                 /* CUDA runtime failure (no reference twin)    */
  DT_ERR_NO_VALID_HYPOTHESIS = 3,  /* exceptions.NoValidHypothesis (matching.py:184,208) */
  DT_ERR_EMPTY_TEMPLATE = 4,       /* exceptions.EmptyTemplate (warpfield.py:86,172)     */
  DT_ERR_ALL_ZERO_WEIGHTS = 5,     /* exceptions.AllZeroWeights (geometry.py:173)        */
  DT_ERR_UNSUPPORTED = 6,          /* configuration outside what the device path covers  */
  DT_ERR_NOT_BOUND = 7             /* solver.py:282-283 "template must be bound"         */
} dt_status;

const char* dt_last_error(void);
/* Library version string and the sm arch it was compiled for. */
const char* dt_version(void);
/* Number of SMs and the largest thread-block cluster the solver kernel can use. */
int dt_device_info(int device, int* sm_count, int* max_cluster);

/* ------------------------------------------------------------------------------
 * Operator level (device pointers). Each replaces one reference function.
 * ---------------------------------------------------------------------------- */

/* correspond.compute_observation_normals (correspond.py:36-73) fused with
 * valid_depth_mask (correspond.py:23-26).  depth (h,w) f64 -> normals (h,w,3) f64,
 * valid (h,w) u8. */
int dt_observation_normals(const double* depth, int64_t h, int64_t w,
                           double fx, double fy, double cx, double cy,
                           double z_min, double z_max,
                           double* normals, uint8_t* valid, void* stream);

/* kernels.warp_and_rasterize (kernels.py:483-569). pixels are (u,v) int64, -1 where
 * the point found no valid pair. */
int dt_warp_and_rasterize(const double* points, const double* normals,
                          const int64_t* bind_idx, const double* alpha,
                          int64_t n, int64_t k, const double* warps, int64_t m,
                          const double* depth, const uint8_t* depth_valid,
                          const double* obs_normals, int64_t height, int64_t width,
                          double fx, double fy, double cx, double cy,
                          double gate_distance, double cos_gate,
                          double* out_p, double* out_n, uint8_t* valid,
                          double* obs_p, double* obs_n, int64_t* pixels,
                          void* stream);

/* kernels.icp_reduce (kernels.py:148-220). basis (m,8,6) as warp_increment_basis
 * (energy.py:205-219). partial (m,27), support (m), cost (m), r (n). */
int dt_icp_reduce(const double* points, const double* obs_normals, const double* obs_points,
                  const int64_t* bind_idx, const double* alpha, int64_t n, int64_t k,
                  const double* warps, const double* basis, int64_t m,
                  double tukey_scale, const double* frozen, int use_frozen, int want_jac,
                  double* partial, double* support, double* cost, double* r,
                  void* stream);

/* kernels.feature_reduce (kernels.py:222-284). */
int dt_feature_reduce(const double* points, const double* obs_points, const double* match_w,
                      const int64_t* bind_idx, const double* alpha, int64_t n, int64_t k,
                      const double* warps, const double* basis, int64_t m,
                      double feature_weight, int want_jac,
                      double* partial, double* support, double* cost, void* stream);

/* kernels.arap_reduce (kernels.py:341-467). R (m,3,3), t (m,3) as
 * geometry.dq_to_transform_batch (geometry.py:238-264); edges (e,2) int64. */
int dt_arap_reduce(const double* ctrl_points, const double* R, const double* t,
                   const double* warps, const int64_t* edges, const double* edge_weights,
                   int64_t n_edges, const double* wa, int64_t m,
                   double angle_weight, double rotation_weight, int want_jac,
                   double* partial, double* cost, void* stream);

/* solver._solve_damped (solver.py:217-258). A (m,6,6), b (m,6), lam (m) ->
 * delta (m,6), ok (m) u8. */
int dt_solve_damped(const double* A, const double* b, const double* lam, int64_t m,
                    double* delta, uint8_t* ok, void* stream);

/* solver.apply_step (solver.py:261-264). */
int dt_apply_step(const double* warps, const double* delta, int64_t m, double* out,
                  void* stream);

/* energy.warp_increment_basis (energy.py:205-219): warps (m,8) -> (m,8,6). */
int dt_warp_increment_basis(const double* warps, int64_t m, double* basis, void* stream);

/* geometry.dq_to_transform_batch (geometry.py:238-264): warps (m,8) -> R (m,3,3), t (m,3). */
int dt_dq_to_transform(const double* warps, int64_t m, double* R, double* t, void* stream);

/* warpfield.warp_all (warpfield.py:236-250). */
int dt_warp_all(const double* points, const double* normals, const int64_t* bind_idx,
                const double* alpha, int64_t n, int64_t k, const double* warps,
                double* out_p, double* out_n, void* stream);

/* warpfield.bind_points (warpfield.py:157-194): brute-force k-nearest controls,
 * nearest first (ties -> lower control index), normalized Gaussian weights. */
int dt_bind_points(const double* points, int64_t n, const double* ctrl, int64_t m,
                   int64_t k, double sigma, int64_t* idx, double* w, void* stream);

/* Brute-force Hamming matching of 256-bit ORB descriptors (north-star part 3a; no
 * reference twin). For every template descriptor: the frame
 * descriptor with the smallest popcount(a xor b), ties -> lowest frame index. */
int dt_hamming_match(const uint8_t* template_desc, int64_t n_template,
                     const uint8_t* frame_desc, int64_t n_frame,
                     int32_t* best_idx, int32_t* best_dist, void* stream);

/* matching.preselect_inliers (matching.py:174-226) with the reference indices given
 * explicitly (refs, n_refs): the host draws them with numpy's Generator exactly as
 * matching.py:189-193 does, or passes arange(n) (exhaustive).
 * Outputs (device): weights (n) f64, flags (n) u8, residuals (n) f64, rotation (9) f64,
 * info: int64[2] = {status (DT_OK or DT_ERR_NO_VALID_HYPOTHESIS), reference index},
 * support: f64[1]. */
typedef struct {
  double distance_threshold;   /* PreselectConfig.distance_threshold (matching.py:69) */
  int32_t n_reweight_iters;    /* PreselectConfig.n_reweight_iters                   */
  double inlier_weight_min;    /* PreselectConfig.inlier_weight_min                  */
  double min_support;          /* PreselectConfig.min_support                        */
} dt_preselect_params;

int dt_preselect(const double* src, const double* dst, int64_t n,
                 const int64_t* refs, int64_t n_refs, const dt_preselect_params* params,
                 double* weights, uint8_t* flags, double* residuals, double* rotation,
                 int64_t* info, double* support, void* stream);

/* ------------------------------------------------------------------------------
 * Template time: graph construction on the device. HOST arrays in
 * and out (once per sequence); bit-identical to the reference.
 * ---------------------------------------------------------------------------- */

/* warpfield.sample_control_points' greedy radius thinning (warpfield.py:77-109): the
 * storage-order indices of the accepted control points (capacity n) and their count. */
int dt_sample_control_points(const double* points, int64_t n, double radius,
                             int64_t* control_index, int64_t* m_out, int device);

/* Candidate connections of warpfield.build_connections (warpfield.py:112-137): every pair
 * i < j with squared distance <= d2_max (the reference's order of evaluation), in
 * lexicographic order, with that squared distance. edges (capacity x 2) int64, d2
 * (capacity) f64; *e_out = the candidate count (pass edges = NULL to query it). The
 * caller applies the reference's weight expression and prune. */
int dt_connection_candidates(const double* ctrl, int64_t m, double d2_max, int64_t* edges,
                             double* d2, int64_t capacity, int64_t* e_out, int device);
/* The whole of build_connections (warpfield.py:112-137) on the device: the pairs i < j of
 * the m controls (lexicographic) with weight w = exp(-|c_i - c_j|^2 / 2 sigma^2) >= prune,
 * into edges (e,2) / weights (e). The weights agree with the reference's numpy exp to an
 * ulp (numpy's exp is not correctly rounded; CUDA's is within 1 ulp), so a pair exactly at
 * the prune boundary may differ; dt_connection_candidates + the host's own exp is the
 * bit-identical route. Call with edges = NULL for the count. HOST arrays. */
int dt_build_connections(const double* ctrl, int64_t m, double sigma, double prune,
                         int64_t* edges, double* weights, int64_t capacity, int64_t* e_out,
                         int device);

/* Local-PCA normals of an unordered cloud (correspond.estimate_point_normals,
 * correspond.py:198-220): the k nearest points (itself included; exact, ties at the
 * k-th neighbour -> lower index), smallest-eigenvalue eigenvector of their scatter,
 * oriented toward the camera (n . p < 0), unit length. points / normals are host
 * (n x 3) f64; k <= 16; n < 3 or k < 3 gives (0, 0, -1) everywhere. */
int dt_estimate_point_normals(const double* points, int64_t n, int64_t k, double* normals,
                              int device);

/* ORB front end (not in the reference): FAST-9 corners,
 * 3x3 non-maximum suppression, uniform suppression (best per_cell per cell of `cell`
 * px, then the best n_max), intensity-centroid orientation in 30 sectors and 256-bit
 * rotated BRIEF on 5x5 box sums. pattern_rot (30 x 256 x 4 int8: the test offsets
 * (ax, ay, bx, by) rotated to each sector) and boundaries (31 x 2 f64 sector-boundary
 * unit vectors) are built by the caller (paper_2007_08576_b200.orb). One context per
 * image size; outputs in order of score (descending), ties by pixel index. */
typedef struct dt_orb dt_orb;
int dt_orb_create(int height, int width, int threshold, int cell, int per_cell, int n_max,
                  const int8_t* pattern_rot, const double* boundaries, int device, dt_orb** out);
int dt_orb_destroy(dt_orb* orb);
/* image: h x w uint8 (host, or device with on_device); outputs host arrays with room for
 * n_max: keypoints (n, 2) int32 (u, v), descriptors (n, 32) uint8, scores and sectors
 * int32 (each may be NULL); *n_out = n. */
int dt_orb_detect(dt_orb* orb, const uint8_t* image, int on_device, int32_t* keypoints,
                  uint8_t* descriptors, int32_t* scores, int32_t* sectors, int64_t* n_out);
/* Device pointers to the last detection's keypoints (n, 2) int32 and descriptors
 * (n, 32) uint8 (valid until the next dt_orb_detect on this context): pass them to
 * dt_track_frame with on_device = 1 to keep the whole image -> warps path on the GPU. */
int dt_orb_last(dt_orb* orb, const int32_t** keypoints, const uint8_t** descriptors, int64_t* n);

/* ------------------------------------------------------------------------------
 * Frame level: a device-resident tracker (one per sequence / stream).
 * Replaces solver.solve_frame (solver.py:267-378) and tracking.track_frame
 * (tracking.py:67-95): preselect -> bind matches -> LM loop -> warp_all, with the
 * whole Levenberg-Marquardt loop running on the device in one cluster kernel.
 * ---------------------------------------------------------------------------- */

typedef struct dt_tracker dt_tracker;

typedef struct {
  /* EnergyWeights (energy.py:49-65) */
  double feature_weight, arap_weight, angle_weight, rotation_weight, tukey_scale, data_floor;
  /* SolverConfig (solver.py:43-71) */
  int32_t max_outer_iters;
  double lambda_init, lambda_decrease, lambda_increase, lambda_min, lambda_max;
  int32_t max_retries;
  double step_tol, cost_tol, gate_distance, cos_gate; /* cos_gate = cos(deg2rad(gate_angle_deg)) */
  /* PreselectConfig (matching.py:58-80) */
  dt_preselect_params preselect;
  /* camera (geometry.PinholeCamera, geometry.py:355-370) + DepthSection (config.py:36-43) */
  double fx, fy, cx, cy;
  int32_t width, height;
  double z_min, z_max;
  /* sampling radius of the graph: sigma of the per-frame match binding (solver.py:292-296) */
  double sampling_radius;
  /* device execution: thread-block cluster size of the solver kernel (0 = auto) */
  int32_t cluster_size;
  /* Hamming gate for descriptor matching (256 = keep every best match) */
  int32_t max_hamming;
} dt_config;

/* EnergyReport (energy.py:107-168) scalar fields. The per-iteration histories are
 * read with dt_tracker_get_history. */
typedef struct {
  double icp_cost, feature_cost, arap_cost, total_cost;
  double match_weight_sum, final_step_norm;
  double preselect_support;
  int32_t n_correspondences, n_matches, n_preselected;
  int32_t outer_iterations, accepted_steps, rejected_steps;
  int32_t stalled, converged, n_cost_history;
  int32_t preselect_status;     /* DT_OK or DT_ERR_NO_VALID_HYPOTHESIS (tracking.py:56-64) */
  int32_t preselect_reference;  /* winning reference index, -1 when none */
  int32_t frame_id;
} dt_report;

/* Create a tracker from host arrays: the bound template (Template, warpfield.py:25-47)
 * and the control graph (ControlGraph, warpfield.py:50-74) with its warm-start warps. */
int dt_tracker_create(const dt_config* cfg,
                      const double* t_points, const double* t_normals,
                      const int64_t* bind_idx, const double* bind_w, int64_t n, int64_t k,
                      const double* ctrl_points, const double* warps, int64_t m,
                      const int64_t* edges, const double* edge_weights, int64_t n_edges,
                      int device, void* stream, dt_tracker** out);
int dt_tracker_destroy(dt_tracker* t);
/* Template-side ORB features: 256-bit descriptors (T,32) u8 and their frame-0 3D
 * points (T,3) f64 (host). The features' control binding (solver.py:292-296: k nearest
 * controls, sigma = graph sampling radius) depends only on these fixed points, so it is
 * computed once here: taken from bind_idx (T,k) int64 / bind_w (T,k) f64 when given
 * (e.g. the reference's kd-tree order), else on the device (ties -> lower index). */
int dt_tracker_set_features(dt_tracker* t, const uint8_t* desc, const double* points,
                            int64_t n_features, const int64_t* bind_idx, const double* bind_w);
/* Warm-start warps (m,8) f64: host (from_device=0) or device pointer. */
int dt_tracker_set_warps(dt_tracker* t, const double* warps, int from_device);
int dt_tracker_get_warps(dt_tracker* t, double* warps_host);
int dt_tracker_set_config(dt_tracker* t, const dt_config* cfg);
int dt_tracker_sync(dt_tracker* t);

/* Per-frame inputs. Pointers are HOST pointers unless `on_device` is set, in which case
 * they are device pointers already resident in HBM. Any optional input may be NULL.
 *   depth            (h,w) f64 mm                         required
 *   normals          (h,w,3) f64; NULL -> computed on the device from depth
 *   match_src/dst    (n_pairs,3) f64 MatchSet pairs (matching.py:21-55)
 *   frame_desc/kp    (n_frame,32) u8 + (n_frame,2) int32 (u,v) keypoints: the ORB path,
 *                    matched against the template features set above
 *   match_w          (n_pairs) f64 weights of ALREADY annotated pairs: preselection is
 *                    skipped (the solver.solve_frame contract, solver.py:267); NULL ->
 *                    the pairs are preselected on the device first (track_frame)
 *   match_bidx/bw    (n_pairs,k) int64 / f64 binding of the pairs' template points;
 *                    NULL -> bound on the device per frame (k nearest, ties -> lower index)
 *   refs             (n_refs) int64 preselect references; NULL -> exhaustive arange(n)
 *   use_matches      0 = no feature term this frame
 *   height, width    the depth image's dimensions
 *   depth_kind       DT_DEPTH_F64: (h,w) f64 row-major (the reference's Observation.depth);
 *                    DT_DEPTH_PFM: the raw payload of a grayscale PFM file -- (h,w) f32,
 *                    little-endian, rows bottom-up (fileio.write_pfm, fileio.py:131-139) --
 *                    copied as is (half the bytes) and decoded on the device
 * Size contract (checked on every call, DT_ERR_INVALID_ARGUMENT otherwise): height /
 * width equal the tracker's camera; counts are non-negative; every array a non-zero
 * count refers to is non-NULL; match_bidx / match_bw come together; host-side refs lie
 * in [0, n_pairs) (pairs path) or [0, n_features) (ORB path). Keypoints outside the
 * image are not an error: they produce no match.
 */
#define DT_DEPTH_F64 0
#define DT_DEPTH_PFM 1

typedef struct {
  const double* depth;  /* DT_DEPTH_PFM: points at the f32 payload (cast) */
  const double* normals;
  const double* match_src;
  const double* match_dst;
  const double* match_w;
  const int64_t* match_bidx;
  const double* match_bw;
  int64_t n_pairs;
  const uint8_t* frame_desc;
  const int32_t* frame_kp;
  int64_t n_frame;
  const int64_t* refs;
  int64_t n_refs;
  int32_t use_matches;
  int32_t on_device;
  int32_t frame_id;
  int32_t height, width;  /* dimensions of depth / normals: must equal dt_config's */
  int32_t depth_kind;     /* DT_DEPTH_F64 or DT_DEPTH_PFM (see below) */
} dt_frame_input;

/* Per-frame outputs (HOST pointers; any may be NULL to skip that copy).
 *   warps (m,8), points (n,3), normals (n,3), match_weights / match_flags (n_matches),
 *   match_src / match_dst (n_matches,3) (the ORB path's MatchSet), control_data_weights (m),
 *   report, and the frame's per-iteration histories (energy.EnergyReport cost_history /
 *   lambda_history, solver.py:345-355): the first report.n_cost_history rows of
 *   cost_history and report.outer_iterations rows of lambda_history / stalled are set.
 *   The pipelined path (dt_track_frame_submit) fills them from the frame's own snapshot. */
typedef struct {
  double* warps;
  double* points;
  double* normals;
  double* match_weights;
  uint8_t* match_flags;
  double* match_src;
  double* match_dst;
  int64_t match_capacity;
  double* control_data_weights;
  dt_report* report;
  double* cost_history;    /* (max_outer_iters,2) [before, after] of the accepted steps */
  double* lambda_history;  /* (max_outer_iters,2) [min, max] damping per outer iteration */
  int32_t* stalled;        /* (max_outer_iters) 1 where the iteration stalled */
} dt_frame_output;

/* Run one frame (asynchronous on the tracker stream; results valid after
 * dt_tracker_sync). The warps solved here become the warm start of the next frame. */
int dt_track_frame(dt_tracker* t, const dt_frame_input* in, dt_frame_output* out);
/* Enqueue one frame without any host output or synchronization (inputs may be host or
 * device pointers as flagged); results stay resident (dt_tracker_device_outputs) and
 * dt_tracker_collect copies them out later. */
int dt_track_frame_async(dt_tracker* t, const dt_frame_input* in);
int dt_tracker_collect(dt_tracker* t, const dt_frame_input* in, dt_frame_output* out);
/* Pipelined streaming (host inputs): dt_track_frame_submit stages the frame's depth and
 * ORB features (HOST pointers) into one of two device slots on a copy stream while the
 * previous frame computes, runs the frame, and copies warps / points / normals /
 * control_data_weights back into `out` (pinned host memory recommended) while the next
 * frame computes. At most two frames are in flight (submit waits for the oldest when
 * needed); `out` must stay valid until dt_tracker_wait returns for that frame.
 * dt_tracker_wait waits for the oldest frame in flight and fills its out->report.
 * Frames are still solved strictly in order (each warm-starts from the previous). */
int dt_track_frame_submit(dt_tracker* t, const dt_frame_input* in, dt_frame_output* out);
int dt_tracker_wait(dt_tracker* t);
/* The tracker's CUDA stream (cudaStream_t). */
void* dt_tracker_stream(dt_tracker* t);
/* Per-phase device timing of each frame (CUDA events between the pipeline stages):
 * ms[0] depth normals, [1] ORB Hamming + match build, [2] preselection,
 * [3] active matches + control CSR, [4] LM solver kernel, [5] output warp. */
#define DT_N_PHASES 6
int dt_tracker_set_profiling(dt_tracker* t, int on);
int dt_tracker_get_phase_ms(dt_tracker* t, float* ms);
/* With profiling on, the solver kernel stamps (phase code, globaltimer ns) pairs at every
 * cluster barrier of the last frame; returns the number of pairs copied into buf. */
int dt_tracker_get_trace(dt_tracker* t, long long* buf, int cap);
/* With profiling on, every CTA of the solver also stamps its ARRIVAL time at each barrier:
 * buf[0] = CTAs, buf[1] = barriers stamped, buf[2 + cta * per_cta + b] = ns. Copies at
 * most cap values; returns per_cta (the stride), 0 when profiling is off. */
int dt_tracker_get_arrivals(dt_tracker* t, long long* buf, int cap);
/* Per-outer-iteration histories of the last frame (host): cost_history
 * (max_outer_iters,2), lambda_history (max_outer_iters,2), stalled (max_outer_iters). */
int dt_tracker_get_history(dt_tracker* t, double* cost_history, double* lambda_history,
                           int32_t* stalled);
/* Device pointers of the resident per-frame outputs (for zero-copy consumers). */
int dt_tracker_device_outputs(dt_tracker* t, double** warps, double** points, double** normals);
/* Counters: kernels launched by the last dt_track_frame call. */
int dt_tracker_last_launches(dt_tracker* t);

/* Run one frame on each of several trackers (independent sequences, BASELINE config 5):
 * every frame is enqueued on its own tracker's stream before any is collected, so the
 * sequences overlap on the device (in cluster mode each solver occupies one thread-block
 * cluster); then each tracker's outputs are collected as dt_track_frame would return
 * them (outputs may be NULL). All trackers must live on the current device. `stream` is
 * reserved (pass NULL). */
int dt_track_frames_batched(dt_tracker** trackers, const dt_frame_input* inputs,
                            dt_frame_output* outputs, int32_t n_trackers, void* stream);

/* ---------------------------------------------------------------------------------
 * Stereo depth (PAPER.md:25 -- upstream of the observation, not in the
 * reference, algorithm defined by oracle/stereo.py): a rectified grey pair (uint8 (h,w),
 * left pixel x <-> right pixel x - d) -> depth (h,w) f64 = fx B / disparity, NaN where
 * no match survives. ZNCC over a (2r+1)^2 window (r in [1,5]) for d in [0, max_disp),
 * winner-take-all both ways, left-right check within lr_tol, minimum correlation
 * min_ncc, parabolic sub-pixel. dt_stereo_compute takes HOST or DEVICE images (on_device)
 * and copies depth / disparity (f64) / winner (int32, -1 = none) to HOST buffers (any may
 * be NULL); dt_stereo_last hands out the device depth for dt_track_frame (on_device = 1).
 * ------------------------------------------------------------------------------- */
typedef struct dt_stereo dt_stereo;
int dt_stereo_create(int height, int width, int max_disp, int radius, double fx, double baseline,
                     double min_ncc, int lr_tol, int device, dt_stereo** out);
int dt_stereo_destroy(dt_stereo* s);
int dt_stereo_compute(dt_stereo* s, const uint8_t* left, const uint8_t* right, int on_device,
                      double* depth, double* disparity, int32_t* winner);
int dt_stereo_last(dt_stereo* s, const double** depth);

/* ---------------------------------------------------------------------------------
 * File-format codecs (fileio.py:23-259). HOST memory, no device.
 * dt_format_reals: `rows` lines of `cols` space-separated reals, each printed exactly as
 *   Python's repr() prints it (shortest round-trip digits; fixed notation for decimal
 *   exponents -4 < e <= 16, else d.ddde+XX), '\n' after each row -- the reference's ascii
 *   PLY body byte for byte. Returns the bytes written, or -(bytes needed) when
 *   `capacity` is too small, -1 on bad arguments.
 * dt_parse_reals: whitespace-separated decimal reals -> out (correctly rounded, the
 *   values Python's float() gives); returns the count parsed (stops at capacity), or
 *   -2 - i when token i is malformed, -1 on bad arguments.
 * dt_depth_from_pfm: device decode of a PFM payload already in DEVICE memory: (h,w) f32
 *   rows bottom-up (big_endian = 0 for the reference's negative scale) -> (h,w) f64
 *   rows top-down (fileio.read_pfm, fileio.py:142-160), on `stream`.
 * ------------------------------------------------------------------------------- */
int64_t dt_format_reals(const double* values, int64_t rows, int64_t cols, char* out,
                        int64_t capacity);
int64_t dt_parse_reals(const char* text, int64_t length, double* out, int64_t capacity);
int dt_depth_from_pfm(const float* payload, int64_t h, int64_t w, int big_endian, double* depth,
                      void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DEFORMTRACK_B200_H */
