// dt_ops.cu -- operator-level sm_100a kernels, one per reference function, and their
// C-ABI entry points (include/deformtrack_b200.h). The fused per-frame solver
// (dt_solver.cu) reuses the same row math from dt_math.cuh.
//
// Reductions are per control point and deterministic: a control's rows are gathered
// through a CSR list in row order and summed by one warp in a fixed association, so
// results are bitwise reproducible run to run and independent of grid size (the
// reference's determinism contract, kernels.py:9-13), without float atomics.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "dt_common.cuh"
#include "dt_math.cuh"
#include "dt_ops.cuh"

namespace dt {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

// ---------------------------------------------------------------------------------
// Observation normals (correspond.py:23-26 valid mask, 29-33 back-projection,
// 36-73 central-difference normals oriented toward the camera).
// ---------------------------------------------------------------------------------

__device__ __forceinline__ bool depth_ok(double z, double zmin, double zmax) {
  return isfinite(z) && z > zmin && z < zmax;
}

// 32-byte pixel record of the solver's projective association (one 256-bit load at the
// projected pixel): {depth if valid_depth_mask else NaN, observed normal x, y, z}
__device__ __forceinline__ void store_pixel(double* rec, double z, bool zok, double n0, double n1,
                                            double n2) {
  const double d = zok ? z : __longlong_as_double(0x7ff8000000000000ll);
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(rec), "d"(d), "d"(n0), "d"(n1),
               "d"(n2)
               : "memory");
}

__global__ void k_observation_normals(const double* __restrict__ depth, int h, int w, double fx,
                                      double fy, double cx, double cy, double zmin, double zmax,
                                      double* __restrict__ normals, uint8_t* __restrict__ valid,
                                      double* __restrict__ pix) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)h * w) return;
  const int v = (int)(i / w);
  const int u = (int)(i - (int64_t)v * w);
  const double z = depth[i];
  if (valid) valid[i] = depth_ok(z, zmin, zmax) ? 1 : 0;
  double n0 = 0.0, n1 = 0.0, n2 = 0.0;
  if (h >= 3 && w >= 3 && v >= 1 && v < h - 1 && u >= 1 && u < w - 1) {
    const double zr = depth[i + 1], zl = depth[i - 1], zd = depth[i + w], zu = depth[i - w];
    // back_project: x = (u - cx) / fx * z
    const double xr = ((double)(u + 1) - cx) / fx * zr, yr = ((double)v - cy) / fy * zr;
    const double xl = ((double)(u - 1) - cx) / fx * zl, yl = ((double)v - cy) / fy * zl;
    const double xd = ((double)u - cx) / fx * zd, yd = ((double)(v + 1) - cy) / fy * zd;
    const double xu = ((double)u - cx) / fx * zu, yu = ((double)(v - 1) - cy) / fy * zu;
    const double dx0 = xr - xl, dx1 = yr - yl, dx2 = zr - zl;
    const double dy0 = xd - xu, dy1 = yd - yu, dy2 = zd - zu;
    double c0 = dx1 * dy2 - dx2 * dy1;
    double c1 = dx2 * dy0 - dx0 * dy2;
    double c2 = dx0 * dy1 - dx1 * dy0;
    bool ok = depth_ok(z, zmin, zmax) && depth_ok(zr, zmin, zmax) && depth_ok(zl, zmin, zmax) &&
              depth_ok(zd, zmin, zmax) && depth_ok(zu, zmin, zmax);
    const double norm = sqrt(c0 * c0 + c1 * c1 + c2 * c2);
    ok = ok && norm > 1e-12;
    if (ok) {
      const double den = norm > 1e-12 ? norm : 1.0;
      n0 = c0 / den;
      n1 = c1 / den;
      n2 = c2 / den;
      const double px = ((double)u - cx) / fx * z, py = ((double)v - cy) / fy * z;
      if (n0 * px + n1 * py + n2 * z > 0.0) {
        n0 = -n0;
        n1 = -n1;
        n2 = -n2;
      }
    }
  }
  if (normals) {
    normals[3 * i + 0] = n0;
    normals[3 * i + 1] = n1;
    normals[3 * i + 2] = n2;
  }
  if (pix) store_pixel(pix + 4 * i, z, depth_ok(z, zmin, zmax), n0, n1, n2);
}

// pixel records from a depth map + caller-supplied observation normals
__global__ void k_pack_pixels(const double* __restrict__ depth, const double* __restrict__ normals,
                              int64_t npix, double zmin, double zmax, double* __restrict__ pix) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  const double z = depth[i];
  store_pixel(pix + 4 * i, z, depth_ok(z, zmin, zmax), normals[3 * i], normals[3 * i + 1],
              normals[3 * i + 2]);
}

int launch_pack_pixels(const double* depth, const double* normals, int64_t npix, double zmin,
                       double zmax, double* pix, cudaStream_t s) {
  if (npix == 0) return DT_OK;
  k_pack_pixels<<<grid_for(npix, 256), 256, 0, s>>>(depth, normals, npix, zmin, zmax, pix);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

// PFM payload (f32, rows bottom-up, little- or big-endian) -> f64 depth, rows top-down
// (fileio.read_pfm, fileio.py:142-160: frombuffer(...).reshape(h, w)[::-1].astype(f64))
__global__ void k_depth_from_pfm(const float* __restrict__ payload, int h, int w, int big_endian,
                                 double* __restrict__ depth) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)h * w) return;
  const int v = (int)(i / w), u = (int)(i - (int64_t)v * w);
  const float* src = payload + (int64_t)(h - 1 - v) * w + u;
  float f = __ldg(src);
  if (big_endian) f = __int_as_float((int)__byte_perm(__float_as_uint(f), 0, 0x0123));
  depth[i] = (double)f;
}

int launch_depth_from_pfm(const float* payload, int64_t h, int64_t w, int big_endian, double* depth,
                          cudaStream_t s) {
  if (h * w == 0) return DT_OK;
  k_depth_from_pfm<<<grid_for(h * w, 256), 256, 0, s>>>(payload, (int)h, (int)w, big_endian, depth);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int launch_observation_normals(const double* depth, int64_t h, int64_t w, double fx, double fy,
                               double cx, double cy, double zmin, double zmax, double* normals,
                               uint8_t* valid, cudaStream_t s, double* pix) {
  if (h * w == 0) return DT_OK;
  k_observation_normals<<<grid_for(h * w, 256), 256, 0, s>>>(depth, (int)h, (int)w, fx, fy, cx, cy,
                                                            zmin, zmax, normals, valid, pix);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

// ---------------------------------------------------------------------------------
// Warp + projective association (kernels.py:483-569).
// ---------------------------------------------------------------------------------

// Project a warped point and gate the pair (kernels.py:537-568). Returns true when the
// pair survives; fills obs point / normal and the pixel.
__device__ __forceinline__ bool rasterize_one(double x0, double x1, double x2, double r0, double r1,
                                              double r2, const double* __restrict__ depth,
                                              const uint8_t* __restrict__ dvalid,
                                              const double* __restrict__ onrm, int height,
                                              int width, double fx, double fy, double cx,
                                              double cy, double gate, double cos_gate,
                                              double obs[3], double g[3], int& ui, int& vi) {
#ifdef DT_DEBUG_RASTER
#define DBG(...) printf(__VA_ARGS__)
#else
#define DBG(...)
#endif
  if (!(x2 > 0.0)) { DBG("x2 %g\n", x2); return false; }
  const double uf = rint(fx * x0 / x2 + cx);
  const double vf = rint(fy * x1 / x2 + cy);
  DBG("uf %.17g vf %.17g w %d h %d\n", uf, vf, width, height);
  if (!(uf >= 0.0 && uf < (double)width && vf >= 0.0 && vf < (double)height)) return false;
  ui = (int)uf;
  vi = (int)vf;
  const int64_t pix = (int64_t)vi * width + ui;
  DBG("ui %d vi %d pix %lld valid %d\n", ui, vi, (long long)pix, (int)dvalid[pix]);
  if (!dvalid[pix]) return false;
  const double d = depth[pix];
  const double ox = ((double)ui - cx) / fx * d;
  const double oy = ((double)vi - cy) / fy * d;
  const double gx = onrm[3 * pix + 0], gy = onrm[3 * pix + 1], gz = onrm[3 * pix + 2];
  DBG("d %.17g g %.17g %.17g %.17g\n", d, gx, gy, gz);
  if (gx * gx + gy * gy + gz * gz <= 0.25) return false;
  const double dx = ox - x0, dy = oy - x1, dz = d - x2;
  DBG("dist %.17g gate %g\n", sqrt(dx * dx + dy * dy + dz * dz), gate);
  if (sqrt(dx * dx + dy * dy + dz * dz) >= gate) return false;
  DBG("cos %.17g cg %.17g\n", gx * r0 + gy * r1 + gz * r2, cos_gate);
  if (gx * r0 + gy * r1 + gz * r2 <= cos_gate) return false;
  obs[0] = ox;
  obs[1] = oy;
  obs[2] = d;
  g[0] = gx;
  g[1] = gy;
  g[2] = gz;
  return true;
}

__global__ void k_warp_and_rasterize(const double* __restrict__ pts, const double* __restrict__ nrm,
                                     const int64_t* __restrict__ bidx,
                                     const double* __restrict__ alpha, int64_t n, int k,
                                     const double* __restrict__ warps,
                                     const double* __restrict__ depth,
                                     const uint8_t* __restrict__ dvalid,
                                     const double* __restrict__ onrm, int height, int width,
                                     double fx, double fy, double cx, double cy, double gate,
                                     double cos_gate, double* out_p, double* out_n,
                                     uint8_t* valid, double* obs_p, double* obs_n,
                                     int64_t* pixels) {
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
  double o[3] = {0.0, 0.0, 0.0}, g[3] = {0.0, 0.0, 0.0};
  int ui = -1, vi = -1;
  const bool ok = rasterize_one(x0, x1, x2, r0, r1, r2, depth, dvalid, onrm, height, width, fx, fy,
                                cx, cy, gate, cos_gate, o, g, ui, vi);
  valid[c] = ok ? 1 : 0;
  obs_p[3 * c] = ok ? o[0] : 0.0;
  obs_p[3 * c + 1] = ok ? o[1] : 0.0;
  obs_p[3 * c + 2] = ok ? o[2] : 0.0;
  obs_n[3 * c] = ok ? g[0] : 0.0;
  obs_n[3 * c + 1] = ok ? g[1] : 0.0;
  obs_n[3 * c + 2] = ok ? g[2] : 0.0;
  pixels[2 * c] = ok ? ui : -1;
  pixels[2 * c + 1] = ok ? vi : -1;
}

// ---------------------------------------------------------------------------------
// Deterministic CSR by control: entry e (row * k + slot) with key[e] = control. For each
// control, one warp scans the keys in order and appends matching entries with a
// ballot/popc prefix, so every list is in increasing entry order.
// ---------------------------------------------------------------------------------

template <typename KeyT>
__global__ void k_csr_count(const KeyT* __restrict__ keys, int64_t ne, int m, int* __restrict__ cnt) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= m) return;
  int total = 0;
  for (int64_t base = 0; base < ne; base += 32) {
    const int64_t e = base + lane;
    const bool hit = e < ne && (int)keys[e] == warp;
    total += __popc(__ballot_sync(0xffffffffu, hit));
  }
  if (lane == 0) cnt[warp] = total;
}

__global__ void __launch_bounds__(1024) k_exclusive_scan(const int* __restrict__ cnt, int m, int* __restrict__ ptr) {
  // single block; m is at most a few thousand controls
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

template <typename KeyT>
__global__ void k_csr_fill(const KeyT* __restrict__ keys, int64_t ne, int m,
                           const int* __restrict__ ptr, int* __restrict__ ent) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= m) return;
  int pos = ptr[warp];
  for (int64_t base = 0; base < ne; base += 32) {
    const int64_t e = base + lane;
    const bool hit = e < ne && (int)keys[e] == warp;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (hit) ent[pos + __popc(bal & ((1u << lane) - 1u))] = (int)e;
    pos += __popc(bal);
  }
}

template <typename KeyT>
int build_csr(const KeyT* keys, int64_t ne, int m, int* ptr, int* ent, int* scratch_cnt,
              cudaStream_t s) {
  const int threads = 256;
  const int blocks = grid_for((int64_t)m * 32, threads);
  k_csr_count<KeyT><<<blocks, threads, 0, s>>>(keys, ne, m, scratch_cnt);
  DT_CHECK_LAUNCH();
  k_exclusive_scan<<<1, 1024, 0, s>>>(scratch_cnt, m, ptr);
  DT_CHECK_LAUNCH();
  k_csr_fill<KeyT><<<blocks, threads, 0, s>>>(keys, ne, m, ptr, ent);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

template int build_csr<int64_t>(const int64_t*, int64_t, int, int*, int*, int*, cudaStream_t);
template int build_csr<int32_t>(const int32_t*, int64_t, int, int*, int*, int*, cudaStream_t);

// ---------------------------------------------------------------------------------
// ICP rows (kernels.py:148-220). Stage 1: one thread per correspondence computes the
// residual, the robust factor and the gradient of r w.r.t. the blend (gn, 8 values).
// Stage 2: one warp per control gathers its (row, slot) entries.
// ---------------------------------------------------------------------------------

__global__ void k_icp_rows(const double* __restrict__ pts, const double* __restrict__ onrm,
                           const double* __restrict__ obs, const int64_t* __restrict__ bidx,
                           const double* __restrict__ alpha, int64_t n, int k,
                           const double* __restrict__ warps, double tukey,
                           const double* __restrict__ frozen, int use_frozen, int want_jac,
                           double* __restrict__ r_out, IcpRow* __restrict__ rows) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double B[8], sgn[KMAX];
  blend_at(warps, bidx + c * k, alpha + c * k, k, B, sgn);
  const double px = pts[3 * c], py = pts[3 * c + 1], pz = pts[3 * c + 2];
  double x0, x1, x2, s2;
  apply_blend(B, px, py, pz, x0, x1, x2, s2);
  const double n0 = onrm[3 * c], n1 = onrm[3 * c + 1], n2 = onrm[3 * c + 2];
  const double r = n0 * (x0 - obs[3 * c]) + n1 * (x1 - obs[3 * c + 1]) + n2 * (x2 - obs[3 * c + 2]);
  r_out[c] = r;
  IcpRow row;
  row.r = r;
  row.rs = use_frozen ? frozen[c] : tukey_sqrt(r, tukey);
  unsigned bits = 0;
  for (int s = 0; s < k; ++s)
    if (sgn[s] < 0.0) bits |= 1u << s;
  row.sgn = bits;
  if (want_jac) {
    double G[24];
    blend_gradient(B, px, py, pz, x0, x1, x2, s2, G);
#pragma unroll
    for (int e = 0; e < 8; ++e) row.gn[e] = n0 * G[e] + n1 * G[8 + e] + n2 * G[16 + e];
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) row.gn[e] = 0.0;
  }
  rows[c] = row;
}

// One entry (row c, slot s) of an ICP row binned to control `ci` (kernels.py:198-212).
__device__ __forceinline__ void icp_entry(const IcpRow& row, double a, const double* K, bool dense,
                                          const double* Kr, const double* Kd, int slot,
                                          bool jac, double* acc, double& support, double& cost) {
  const double rs = row.rs;
  support += rs * rs * a;
  const double sw = rs * sqrt(a);
  const double wv = sw * row.r;
  cost += wv * wv;
  if (jac) {
    const double sg = ((row.sgn >> slot) & 1u) ? -1.0 : 1.0;
    const double coef = sw * a * sg;
    double pr[6];
    if (dense) basis_project_dense(row.gn, K, pr);
    else basis_project(row.gn, Kr, Kd, pr);
    double J[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) J[d] = coef * pr[d];
    fold_row(acc, J, wv);
  }
}

__global__ void k_icp_gather(const IcpRow* __restrict__ rows, const double* __restrict__ alpha,
                             int k, const double* __restrict__ basis, const int* __restrict__ ptr,
                             const int* __restrict__ ent, int m, int want_jac,
                             double* __restrict__ partial, double* __restrict__ support,
                             double* __restrict__ cost) {
  extern __shared__ double s_scr[];
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ci = blockIdx.x * (blockDim.x >> 5) + wib;
  double* scr = s_scr + wib * 32 * 29;
  if (ci >= m) return;
  double acc[29];
#pragma unroll
  for (int i = 0; i < 29; ++i) acc[i] = 0.0;
  const double* K = basis + (int64_t)ci * 48;
  for (int q = ptr[ci] + lane; q < ptr[ci + 1]; q += 32) {
    const int e = ent[q];
    const int c = e / k, s = e - c * k;
    icp_entry(rows[c], alpha[e], K, true, nullptr, nullptr, s, want_jac != 0, acc, acc[27], acc[28]);
  }
  double out[29];
  warp_column_sum<29>(acc, scr, out);
  if (lane < 27) partial[(int64_t)ci * 27 + lane] = want_jac ? out[lane] : 0.0;
  if (lane == 27) support[ci] = out[27];
  if (lane == 28) cost[ci] = out[28];
}

// ---------------------------------------------------------------------------------
// Feature rows (kernels.py:222-284).
// ---------------------------------------------------------------------------------

__global__ void k_feature_rows(const double* __restrict__ pts, const double* __restrict__ obs,
                               const double* __restrict__ mw, const int64_t* __restrict__ bidx,
                               const double* __restrict__ alpha, int64_t n, int k,
                               const double* __restrict__ warps, int want_jac,
                               FeatRow* __restrict__ rows) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double B[8], sgn[KMAX];
  blend_at(warps, bidx + c * k, alpha + c * k, k, B, sgn);
  const double px = pts[3 * c], py = pts[3 * c + 1], pz = pts[3 * c + 2];
  double x0, x1, x2, s2;
  apply_blend(B, px, py, pz, x0, x1, x2, s2);
  FeatRow row;
  row.res[0] = x0 - obs[3 * c];
  row.res[1] = x1 - obs[3 * c + 1];
  row.res[2] = x2 - obs[3 * c + 2];
  row.w = mw[c];
  unsigned bits = 0;
  for (int s = 0; s < k; ++s)
    if (sgn[s] < 0.0) bits |= 1u << s;
  row.sgn = bits;
  if (want_jac) blend_gradient(B, px, py, pz, x0, x1, x2, s2, row.G);
  else
    for (int e = 0; e < 24; ++e) row.G[e] = 0.0;
  rows[c] = row;
}

__device__ __forceinline__ void feature_entry(const FeatRow& row, double a, double fw,
                                              const double* K, bool dense, const double* Kr,
                                              const double* Kd, int slot, bool jac, double* acc,
                                              double& support, double& cost) {
  const double w_pair = fw * row.w * a;
  support += w_pair;
  const double sw = sqrt(w_pair);
  const double wv0 = sw * row.res[0], wv1 = sw * row.res[1], wv2 = sw * row.res[2];
  cost += wv0 * wv0 + wv1 * wv1 + wv2 * wv2;
  if (jac) {
    const double sg = ((row.sgn >> slot) & 1u) ? -1.0 : 1.0;
    const double coef = sw * a * sg;
    double GK[18];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      double pr[6];
      if (dense) basis_project_dense(row.G + comp * 8, K, pr);
      else basis_project(row.G + comp * 8, Kr, Kd, pr);
#pragma unroll
      for (int d = 0; d < 6; ++d) GK[comp * 6 + d] = coef * pr[d];
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
      for (int j = i; j < 6; ++j)
        acc[triu_col(i, j)] += GK[i] * GK[j] + GK[6 + i] * GK[6 + j] + GK[12 + i] * GK[12 + j];
      acc[21 + i] += GK[i] * wv0 + GK[6 + i] * wv1 + GK[12 + i] * wv2;
    }
  }
}

__global__ void k_feature_gather(const FeatRow* __restrict__ rows, const double* __restrict__ alpha,
                                 int k, const double* __restrict__ basis, double fw,
                                 const int* __restrict__ ptr, const int* __restrict__ ent, int m,
                                 int want_jac, double* __restrict__ partial,
                                 double* __restrict__ support, double* __restrict__ cost) {
  extern __shared__ double s_scr[];
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ci = blockIdx.x * (blockDim.x >> 5) + wib;
  double* scr = s_scr + wib * 32 * 29;
  if (ci >= m) return;
  double acc[29];
#pragma unroll
  for (int i = 0; i < 29; ++i) acc[i] = 0.0;
  const double* K = basis + (int64_t)ci * 48;
  for (int q = ptr[ci] + lane; q < ptr[ci + 1]; q += 32) {
    const int e = ent[q];
    const int c = e / k, s = e - c * k;
    feature_entry(rows[c], alpha[e], fw, K, true, nullptr, nullptr, s, want_jac != 0, acc, acc[27],
                  acc[28]);
  }
  double out[29];
  warp_column_sum<29>(acc, scr, out);
  if (lane < 27) partial[(int64_t)ci * 27 + lane] = want_jac ? out[lane] : 0.0;
  if (lane == 27) support[ci] = out[27];
  if (lane == 28) cost[ci] = out[28];
}

// ---------------------------------------------------------------------------------
// ARAP rows (kernels.py:341-467): one warp per control over its incident edges.
// ---------------------------------------------------------------------------------

__global__ void k_arap_gather(const double* __restrict__ cpts, const double* __restrict__ R,
                              const double* __restrict__ t, const double* __restrict__ warps,
                              const int64_t* __restrict__ edges, const double* __restrict__ ew,
                              const double* __restrict__ wa, double angle_w, double rot_w,
                              const int* __restrict__ ptr, const int* __restrict__ ent, int m,
                              int want_jac, double* __restrict__ partial, double* __restrict__ cost) {
  extern __shared__ double s_scr[];
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ci = blockIdx.x * (blockDim.x >> 5) + wib;
  double* scr = s_scr + wib * 32 * 28;
  if (ci >= m) return;
  double acc[28];
#pragma unroll
  for (int i = 0; i < 28; ++i) acc[i] = 0.0;
  for (int q = ptr[ci] + lane; q < ptr[ci + 1]; q += 32) {
    const int e2 = ent[q];
    const int e = e2 >> 1, side = e2 & 1;
    const int64_t i0 = edges[2 * (int64_t)e], i1 = edges[2 * (int64_t)e + 1];
    arap_edge_bin(cpts + 3 * i0, cpts + 3 * i1, R + 9 * i0, t + 3 * i0, R + 9 * i1, t + 3 * i1,
                  warps + 8 * i0, warps + 8 * i1, ew[e], wa[i0], wa[i1], angle_w, rot_w, side,
                  want_jac != 0, acc, &acc[27]);
  }
  double out[28];
  warp_column_sum<28>(acc, scr, out);
  if (lane < 27) partial[(int64_t)ci * 27 + lane] = want_jac ? out[lane] : 0.0;
  if (lane == 27) cost[ci] = out[27];
}

// keys of the incidence list: entry 2e + side -> edges[e, side]
__global__ void k_edge_keys(const int64_t* __restrict__ edges, int64_t ne, int32_t* keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * ne) return;
  keys[i] = (int32_t)edges[i];
}

// ---------------------------------------------------------------------------------
// Small per-control kernels.
// ---------------------------------------------------------------------------------

__global__ void k_solve_damped(const double* __restrict__ A, const double* __restrict__ b,
                               const double* __restrict__ lam, int64_t m, double* __restrict__ delta,
                               uint8_t* __restrict__ ok) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double part[27];
  const double* Ac = A + 36 * c;
  // the lower triangle feeds the factorization (numpy.linalg.cholesky reads 'L')
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) part[triu_col(i, j)] = Ac[j * 6 + i];
  for (int i = 0; i < 6; ++i) part[21 + i] = -b[6 * c + i];
  double d[6];
  const bool good = damped_solve6(part, lam[c], d);
  for (int i = 0; i < 6; ++i) delta[6 * c + i] = d[i];
  ok[c] = good ? 1 : 0;
}

__global__ void k_apply_step(const double* __restrict__ warps, const double* __restrict__ delta,
                             int64_t m, double* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  apply_step_one(warps + 8 * c, delta + 6 * c, out + 8 * c);
}

__global__ void k_basis(const double* __restrict__ warps, int64_t m, double* __restrict__ basis) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  Basis K;
  make_basis(warps + 8 * c, K);
  double* o = basis + 48 * c;
  for (int i = 0; i < 48; ++i) o[i] = 0.0;
  for (int e = 0; e < 4; ++e)
    for (int d = 0; d < 3; ++d) {
      o[e * 6 + d] = K.Kr[e * 3 + d];
      o[(4 + e) * 6 + d] = K.Kd[e * 3 + d];
      o[(4 + e) * 6 + 3 + d] = K.Kr[e * 3 + d];
    }
}

__global__ void k_dq_to_transform(const double* __restrict__ warps, int64_t m, double* __restrict__ R,
                                  double* __restrict__ t) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  dq_to_transform(warps + 8 * c, R + 9 * c, t + 3 * c);
}

__global__ void k_warp_all(const double* __restrict__ pts, const double* __restrict__ nrm,
                           const int64_t* __restrict__ bidx, const double* __restrict__ alpha,
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

// k-nearest controls (warpfield.py:157-194), brute force over the control set with the
// ordering key (squared distance, control index).
template <typename IdxT>
__global__ void k_bind_points(const double* __restrict__ pts, int64_t n,
                              const double* __restrict__ ctrl, int m, int k, double sigma,
                              IdxT* __restrict__ out_idx, double* __restrict__ out_w) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double px = pts[3 * p], py = pts[3 * p + 1], pz = pts[3 * p + 2];
  double bd[KMAX];
  int bi[KMAX];
  const int keff = k < m ? k : m;
  for (int s = 0; s < KMAX; ++s) {
    bd[s] = INFINITY;
    bi[s] = 0x7fffffff;
  }
  for (int c = 0; c < m; ++c) {
    const double dx = px - ctrl[3 * c], dy = py - ctrl[3 * c + 1], dz = pz - ctrl[3 * c + 2];
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 < bd[keff - 1]) {
      int s = keff - 1;
      while (s > 0 && d2 < bd[s - 1]) {
        bd[s] = bd[s - 1];
        bi[s] = bi[s - 1];
        --s;
      }
      bd[s] = d2;
      bi[s] = c;
    }
  }
  double w[KMAX];
  const double den = 2.0 * sigma * sigma;
  double row_sum = 0.0;
  for (int s = 0; s < keff; ++s) {
    const double dist = sqrt(bd[s]);
    w[s] = exp(-(dist * dist) / den);
    row_sum += w[s];
  }
  if (row_sum <= 0.0) {
    for (int s = 0; s < keff; ++s) w[s] = s == 0 ? 1.0 : 0.0;
    row_sum = 0.0;
    for (int s = 0; s < keff; ++s) row_sum += w[s];
  }
  for (int s = 0; s < k; ++s) {
    if (s < keff) {
      out_idx[p * k + s] = (IdxT)bi[s];
      out_w[p * k + s] = w[s] / row_sum;
    } else {
      out_idx[p * k + s] = (IdxT)bi[0];
      out_w[p * k + s] = 0.0;
    }
  }
}

template __global__ void k_bind_points<int64_t>(const double*, int64_t, const double*, int, int,
                                                double, int64_t*, double*);
template __global__ void k_bind_points<int32_t>(const double*, int64_t, const double*, int, int,
                                                double, int32_t*, double*);

int launch_bind_points_i32(const double* pts, int64_t n, const double* ctrl, int m, int k,
                           double sigma, int32_t* idx, double* w, cudaStream_t s) {
  if (n == 0) return DT_OK;
  k_bind_points<int32_t><<<grid_for(n, 128), 128, 0, s>>>(pts, n, ctrl, m, k, sigma, idx, w);
  DT_CHECK_LAUNCH();
  return DT_OK;
}


}  // namespace dt

using namespace dt;

// =================================================================================
// C-ABI
// =================================================================================

extern "C" {

const char* dt_last_error(void) { return g_last_error.c_str(); }

const char* dt_version(void) { return "deformtrack_b200 0.1 (sm_100a)"; }

int dt_device_info(int device, int* sm_count, int* max_cluster) {
  int sms = 0;
  DT_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (sm_count) *sm_count = sms;
  if (max_cluster) *max_cluster = solver_max_cluster(device);
  return DT_OK;
}

int dt_observation_normals(const double* depth, int64_t h, int64_t w, double fx, double fy,
                           double cx, double cy, double z_min, double z_max, double* normals,
                           uint8_t* valid, void* stream) {
  DT_REQUIRE(h >= 0 && w >= 0, DT_ERR_INVALID_ARGUMENT, "negative image size");
  return launch_observation_normals(depth, h, w, fx, fy, cx, cy, z_min, z_max, normals, valid,
                                    as_stream(stream));
}

int dt_depth_from_pfm(const float* payload, int64_t h, int64_t w, int big_endian, double* depth,
                      void* stream) {
  DT_REQUIRE(h >= 0 && w >= 0, DT_ERR_INVALID_ARGUMENT, "negative image size");
  DT_REQUIRE(h * w == 0 || (payload != nullptr && depth != nullptr), DT_ERR_INVALID_ARGUMENT, "NULL buffer");
  return launch_depth_from_pfm(payload, h, w, big_endian, depth, as_stream(stream));
}

int dt_warp_and_rasterize(const double* points, const double* normals, const int64_t* bind_idx,
                          const double* alpha, int64_t n, int64_t k, const double* warps,
                          int64_t m, const double* depth, const uint8_t* depth_valid,
                          const double* obs_normals, int64_t height, int64_t width, double fx,
                          double fy, double cx, double cy, double gate_distance, double cos_gate,
                          double* out_p, double* out_n, uint8_t* valid, double* obs_p,
                          double* obs_n, int64_t* pixels, void* stream) {
  DT_REQUIRE(k >= 1 && k <= KMAX, DT_ERR_UNSUPPORTED, "bind_k=%lld outside [1, %d]", (long long)k, KMAX);
  (void)m;
  if (n == 0) return DT_OK;
  k_warp_and_rasterize<<<grid_for(n, 128), 128, 0, as_stream(stream)>>>(
      points, normals, bind_idx, alpha, n, (int)k, warps, depth, depth_valid, obs_normals,
      (int)height, (int)width, fx, fy, cx, cy, gate_distance, cos_gate, out_p, out_n, valid, obs_p,
      obs_n, pixels);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int dt_icp_reduce(const double* points, const double* obs_normals, const double* obs_points,
                  const int64_t* bind_idx, const double* alpha, int64_t n, int64_t k,
                  const double* warps, const double* basis, int64_t m, double tukey_scale,
                  const double* frozen, int use_frozen, int want_jac, double* partial,
                  double* support, double* cost, double* r, void* stream) {
  DT_REQUIRE(k >= 1 && k <= KMAX, DT_ERR_UNSUPPORTED, "bind_k outside [1, %d]", KMAX);
  cudaStream_t s = as_stream(stream);
  if (m == 0) return DT_OK;
  IcpRow* rows = nullptr;
  int *ptr = nullptr, *ent = nullptr, *cnt = nullptr;
  const int64_t ne = n * k;
  DT_CHECK_CUDA(cudaMallocAsync((void**)&rows, sizeof(IcpRow) * (n > 0 ? n : 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ptr, sizeof(int) * (m + 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ent, sizeof(int) * (ne > 0 ? ne : 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&cnt, sizeof(int) * m, s));
  if (n > 0) {
    k_icp_rows<<<grid_for(n, 128), 128, 0, s>>>(points, obs_normals, obs_points, bind_idx, alpha,
                                                 n, (int)k, warps, tukey_scale, frozen, use_frozen,
                                                 want_jac, r, rows);
    DT_CHECK_LAUNCH();
  }
  int st = build_csr<int64_t>(bind_idx, ne, (int)m, ptr, ent, cnt, s);
  if (st != DT_OK) return st;
  const int wpb = 4;
  k_icp_gather<<<grid_for(m, wpb), wpb * 32, wpb * 32 * 29 * sizeof(double), s>>>(
      rows, alpha, (int)k, basis, ptr, ent, (int)m, want_jac, partial, support, cost);
  DT_CHECK_LAUNCH();
  cudaFreeAsync(rows, s);
  cudaFreeAsync(ptr, s);
  cudaFreeAsync(ent, s);
  cudaFreeAsync(cnt, s);
  return DT_OK;
}

int dt_feature_reduce(const double* points, const double* obs_points, const double* match_w,
                      const int64_t* bind_idx, const double* alpha, int64_t n, int64_t k,
                      const double* warps, const double* basis, int64_t m, double feature_weight,
                      int want_jac, double* partial, double* support, double* cost, void* stream) {
  DT_REQUIRE(k >= 1 && k <= KMAX, DT_ERR_UNSUPPORTED, "bind_k outside [1, %d]", KMAX);
  cudaStream_t s = as_stream(stream);
  if (m == 0) return DT_OK;
  FeatRow* rows = nullptr;
  int *ptr = nullptr, *ent = nullptr, *cnt = nullptr;
  const int64_t ne = n * k;
  DT_CHECK_CUDA(cudaMallocAsync((void**)&rows, sizeof(FeatRow) * (n > 0 ? n : 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ptr, sizeof(int) * (m + 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ent, sizeof(int) * (ne > 0 ? ne : 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&cnt, sizeof(int) * m, s));
  if (n > 0) {
    k_feature_rows<<<grid_for(n, 128), 128, 0, s>>>(points, obs_points, match_w, bind_idx, alpha, n,
                                                     (int)k, warps, want_jac, rows);
    DT_CHECK_LAUNCH();
  }
  int st = build_csr<int64_t>(bind_idx, ne, (int)m, ptr, ent, cnt, s);
  if (st != DT_OK) return st;
  const int wpb = 4;
  k_feature_gather<<<grid_for(m, wpb), wpb * 32, wpb * 32 * 29 * sizeof(double), s>>>(
      rows, alpha, (int)k, basis, feature_weight, ptr, ent, (int)m, want_jac, partial, support,
      cost);
  DT_CHECK_LAUNCH();
  cudaFreeAsync(rows, s);
  cudaFreeAsync(ptr, s);
  cudaFreeAsync(ent, s);
  cudaFreeAsync(cnt, s);
  return DT_OK;
}

int dt_arap_reduce(const double* ctrl_points, const double* R, const double* t,
                   const double* warps, const int64_t* edges, const double* edge_weights,
                   int64_t n_edges, const double* wa, int64_t m, double angle_weight,
                   double rotation_weight, int want_jac, double* partial, double* cost,
                   void* stream) {
  cudaStream_t s = as_stream(stream);
  if (m == 0) return DT_OK;
  int32_t* keys = nullptr;
  int *ptr = nullptr, *ent = nullptr, *cnt = nullptr;
  const int64_t ne = 2 * n_edges;
  DT_CHECK_CUDA(cudaMallocAsync((void**)&keys, sizeof(int32_t) * (ne > 0 ? ne : 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ptr, sizeof(int) * (m + 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&ent, sizeof(int) * (ne > 0 ? ne : 1), s));
  DT_CHECK_CUDA(cudaMallocAsync((void**)&cnt, sizeof(int) * m, s));
  if (ne > 0) {
    k_edge_keys<<<grid_for(ne, 256), 256, 0, s>>>(edges, n_edges, keys);
    DT_CHECK_LAUNCH();
  }
  int st = build_csr<int32_t>(keys, ne, (int)m, ptr, ent, cnt, s);
  if (st != DT_OK) return st;
  const int wpb = 4;
  k_arap_gather<<<grid_for(m, wpb), wpb * 32, wpb * 32 * 28 * sizeof(double), s>>>(
      ctrl_points, R, t, warps, edges, edge_weights, wa, angle_weight, rotation_weight, ptr, ent,
      (int)m, want_jac, partial, cost);
  DT_CHECK_LAUNCH();
  cudaFreeAsync(keys, s);
  cudaFreeAsync(ptr, s);
  cudaFreeAsync(ent, s);
  cudaFreeAsync(cnt, s);
  return DT_OK;
}

int dt_solve_damped(const double* A, const double* b, const double* lam, int64_t m, double* delta,
                    uint8_t* ok, void* stream) {
  if (m == 0) return DT_OK;
  k_solve_damped<<<grid_for(m, 128), 128, 0, as_stream(stream)>>>(A, b, lam, m, delta, ok);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int dt_apply_step(const double* warps, const double* delta, int64_t m, double* out, void* stream) {
  if (m == 0) return DT_OK;
  k_apply_step<<<grid_for(m, 128), 128, 0, as_stream(stream)>>>(warps, delta, m, out);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int dt_warp_increment_basis(const double* warps, int64_t m, double* basis, void* stream) {
  if (m == 0) return DT_OK;
  k_basis<<<grid_for(m, 128), 128, 0, as_stream(stream)>>>(warps, m, basis);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int dt_dq_to_transform(const double* warps, int64_t m, double* R, double* t, void* stream) {
  if (m == 0) return DT_OK;
  k_dq_to_transform<<<grid_for(m, 128), 128, 0, as_stream(stream)>>>(warps, m, R, t);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int dt_warp_all(const double* points, const double* normals, const int64_t* bind_idx,
                const double* alpha, int64_t n, int64_t k, const double* warps, double* out_p,
                double* out_n, void* stream) {
  DT_REQUIRE(k >= 1 && k <= KMAX, DT_ERR_UNSUPPORTED, "bind_k outside [1, %d]", KMAX);
  if (n == 0) return DT_OK;
  k_warp_all<<<grid_for(n, 128), 128, 0, as_stream(stream)>>>(points, normals, bind_idx, alpha, n,
                                                               (int)k, warps, out_p, out_n);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

int dt_bind_points(const double* points, int64_t n, const double* ctrl, int64_t m, int64_t k,
                   double sigma, int64_t* idx, double* w, void* stream) {
  DT_REQUIRE(m > 0, DT_ERR_EMPTY_TEMPLATE, "cannot bind to an empty control set");
  DT_REQUIRE(sigma > 0.0, DT_ERR_INVALID_ARGUMENT, "binding sigma must be positive");
  DT_REQUIRE(k >= 1 && k <= KMAX, DT_ERR_UNSUPPORTED, "bind_k outside [1, %d]", KMAX);
  if (n == 0) return DT_OK;
  k_bind_points<int64_t><<<grid_for(n, 128), 128, 0, as_stream(stream)>>>(points, n, ctrl, (int)m,
                                                                         (int)k, sigma, idx, w);
  DT_CHECK_LAUNCH();
  return DT_OK;
}

}  // extern "C"
