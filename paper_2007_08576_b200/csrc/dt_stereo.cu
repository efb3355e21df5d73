// Stereo depth on the device (the paper's GPU stereo
// matcher upstream of the observation, Fig. 1): a rectified grey pair -> the (h, w) f64
// depth map dt_track_frame consumes. The reference ships no stereo (depth
// arrives as a map), so the algorithm is defined by the restatement in oracle/stereo.py
// and matched exactly:
//
//   k_box_stats   exact integer window sums S, SS of both images ((2r+1)^2 windows)
//   k_wta_left    per left pixel, every disparity: the cross sum from shared-memory
//                 tiles (left window in registers), ZNCC in IEEE double from the exact
//                 integers, winner-take-all (ties -> smaller disparity)
//   k_wta_right   the same per right pixel (right window in registers)
//   k_finish      left-right consistency, minimum correlation, sub-pixel parabola,
//                 depth = fx B / disparity (NaN where no match survives)
//
// Integer sums are exact and the double expressions follow the oracle's operation order
// (the library builds with -fmad=false; sqrt and division are IEEE round-to-nearest), so
// winners, disparities and depths equal the oracle's bit for bit.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "dt_common.cuh"

#ifndef DT_TRY
#define DT_TRY(expr)        \
  do {                      \
    int _st = (expr);       \
    if (_st != DT_OK)       \
      return _st;           \
  } while (0)
#endif

struct dt_stereo {
  int h = 0, w = 0, max_disp = 0, radius = 0, lr_tol = 1, device = 0;
  double fxb = 0.0, min_ncc = 0.5;
  cudaStream_t stream = nullptr;
  uint8_t *left = nullptr, *right = nullptr;
  int32_t *sl = nullptr, *sll = nullptr, *sr = nullptr, *srr = nullptr;
  int32_t *dl = nullptr, *dr = nullptr, *win = nullptr;
  double *cl = nullptr, *depth = nullptr, *disp = nullptr;
};

namespace dt {
namespace {

constexpr int ST_BX = 32, ST_BY = 8;
constexpr int ST_RMAX = 5;  // window radius limit (11 x 11)

// ZNCC from exact window sums, in the oracle's operation order (oracle/stereo.py)
__device__ __forceinline__ double zncc(long long n, long long SL, long long SLL, long long SR,
                                       long long SRR, long long SLR, bool& ok) {
  const long long num = n * SLR - SL * SR;
  const long long vl = n * SLL - SL * SL;
  const long long vr = n * SRR - SR * SR;
  ok = vl > 0 && vr > 0;
  return (double)num / sqrt((double)vl * (double)vr);
}

__global__ void k_box_stats(const uint8_t* __restrict__ img, int h, int w, int r,
                            int32_t* __restrict__ s, int32_t* __restrict__ ss) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  int a = 0, b = 0;
  if (y >= r && y < h - r && x >= r && x < w - r)
    for (int i = -r; i <= r; ++i)
      for (int j = -r; j <= r; ++j) {
        const int v = __ldg(img + (int64_t)(y + i) * w + (x + j));
        a += v;
        b += v * v;
      }
  s[(int64_t)y * w + x] = a;
  ss[(int64_t)y * w + x] = b;
}

// LEFT = true: thread per left pixel x, partner right pixel x - d; LEFT = false: thread
// per right pixel x, partner left pixel x + d. The thread's own window sits in registers
// (RAD is a template parameter so the window unrolls); the partner image's rows of the
// tile in shared memory.
template <bool LEFT, int RAD>
__global__ void __launch_bounds__(ST_BX* ST_BY)
k_wta(const uint8_t* __restrict__ L, const uint8_t* __restrict__ R, int h, int w, int D,
      const int32_t* __restrict__ sl, const int32_t* __restrict__ sll, const int32_t* __restrict__ sr,
      const int32_t* __restrict__ srr, int32_t* __restrict__ best_d, double* __restrict__ best_c) {
  extern __shared__ uint8_t s_tile[];
  constexpr int r = RAD, k = 2 * RAD + 1;
  const int x0 = blockIdx.x * ST_BX, y0 = blockIdx.y * ST_BY;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x = x0 + tx, y = y0 + ty;
  // partner tile: rows y0 - r .. y0 + BY + r, columns (left pass) x0 - r - (D-1) ..
  // x0 + BX + r, (right pass) x0 - r .. x0 + BX + r + D - 1
  const int tw = ST_BX + 2 * r + D - 1, th = ST_BY + 2 * r;
  const int cx0 = LEFT ? x0 - r - (D - 1) : x0 - r;
  const uint8_t* P = LEFT ? R : L;
  for (int i = ty * ST_BX + tx; i < tw * th; i += ST_BX * ST_BY) {
    const int yy = y0 - r + i / tw, xx = cx0 + i % tw;
    s_tile[i] = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? __ldg(P + (int64_t)yy * w + xx) : 0;
  }
  __syncthreads();
  if (x >= w || y >= h) return;
  const bool rows_ok = y >= r && y < h - r && x >= r && x < w - r;
  int own[k * k];
  const uint8_t* O = LEFT ? L : R;
#pragma unroll
  for (int i = 0; i < k; ++i)
#pragma unroll
    for (int j = 0; j < k; ++j)
      own[i * k + j] = rows_ok ? __ldg(O + (int64_t)(y - r + i) * w + (x - r + j)) : 0;
  const long long n = (long long)k * k;
  const long long S1 = rows_ok ? (LEFT ? sl : sr)[(int64_t)y * w + x] : 0;
  const long long SS1 = rows_ok ? (LEFT ? sll : srr)[(int64_t)y * w + x] : 0;
  int bd = -1;
  double bc = -INFINITY;
  if (rows_ok) {
    for (int d = 0; d < D; ++d) {
      const int px = LEFT ? x - d : x + d;  // partner pixel
      if (px - r < 0 || px + r >= w) continue;
      // partner window: tile column of (px - r) is px - r - cx0
      const int c0 = px - r - cx0;
      int cross = 0;
#pragma unroll
      for (int i = 0; i < k; ++i) {
        const uint8_t* row = s_tile + (ty + i) * tw + c0;
#pragma unroll
        for (int j = 0; j < k; ++j) cross += own[i * k + j] * (int)row[j];
      }
      const long long S2 = (LEFT ? sr : sl)[(int64_t)y * w + px];
      const long long SS2 = (LEFT ? srr : sll)[(int64_t)y * w + px];
      bool ok;
      const double c = LEFT ? zncc(n, S1, SS1, S2, SS2, cross, ok) : zncc(n, S2, SS2, S1, SS1, cross, ok);
      if (ok && c > bc) {  // strict: ascending d keeps the smaller disparity on ties
        bc = c;
        bd = d;
      }
    }
  }
  best_d[(int64_t)y * w + x] = bd;
  if (best_c) best_c[(int64_t)y * w + x] = bc;
}

// Two-phase variant: one CTA per (32-pixel segment, row).
//  Phase 1 -- one lane per disparity (warp c: disparities 32c .. 32c + 31): each lane walks
//  the segment left to right keeping its window cross sum up to date with one entering and
//  one leaving column (2 (2r+1) multiply-adds per step instead of (2r+1)^2) and scores
//  every pixel in float from the exact integer sums, float(num) * rsqrt(float(vl) *
//  float(vr)) (relative error < 1e-6, |c| <= 1); a warp max and a ballot per pixel record
//  the disparities within 1e-5 of the warp's best, and the per-warp maxima go to shared
//  memory.
//  Phase 2 -- one lane per pixel: over the disparities recorded within 1e-5 of the
//  pixel's overall float maximum, in ascending order, the oracle's double ZNCC from the
//  window cross sum (recomputed for those few): the exact maximum is among them, so the
//  winner (ties -> smaller disparity) and its correlation are k_wta's bit for bit, at a
//  few double divisions and square roots per pixel instead of one per disparity.
constexpr int SL_SEG = 32;

template <bool LEFT, int RAD>
__global__ void k_wta_slide(const uint8_t* __restrict__ L, const uint8_t* __restrict__ R, int h,
                            int w, int D, const int32_t* __restrict__ sl,
                            const int32_t* __restrict__ sll, const int32_t* __restrict__ sr,
                            const int32_t* __restrict__ srr, int32_t* __restrict__ best_d,
                            double* __restrict__ best_c) {
  extern __shared__ __align__(16) uint8_t s_raw[];
  constexpr int r = RAD, k = 2 * RAD + 1;
  const int x0 = blockIdx.x * SL_SEG, y = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  // own rows: columns x0 - r .. x0 + SEG - 1 + r; partner rows: (left pass) columns
  // x0 - r - (D - 1) .. x0 + SEG - 1 + r, (right pass) x0 - r .. x0 + SEG - 1 + r + D - 1
  const int ow = SL_SEG + 2 * r, pw = SL_SEG + 2 * r + D - 1;
  uint8_t* s_own = s_raw;
  uint8_t* s_par = s_raw + k * ow;
  float* s_fmax = reinterpret_cast<float*>(s_raw + ((k * (ow + pw) + 15) / 16) * 16);
  unsigned* s_mask = reinterpret_cast<unsigned*>(s_fmax + nw * SL_SEG);
  const uint8_t* O = LEFT ? L : R;
  const uint8_t* P = LEFT ? R : L;
  const int ox0 = x0 - r, px0 = LEFT ? x0 - r - (D - 1) : x0 - r;
  for (int i = threadIdx.x; i < k * ow; i += blockDim.x) {
    const int yy = y - r + i / ow, xx = ox0 + i % ow;
    s_own[i] = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? __ldg(O + (int64_t)yy * w + xx) : 0;
  }
  for (int i = threadIdx.x; i < k * pw; i += blockDim.x) {
    const int yy = y - r + i / pw, xx = px0 + i % pw;
    s_par[i] = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? __ldg(P + (int64_t)yy * w + xx) : 0;
  }
  __syncthreads();
  const bool rows_ok = y >= r && y < h - r;
  const long long n = (long long)k * k;
  const int32_t* So = LEFT ? sl : sr;
  const int32_t* SSo = LEFT ? sll : srr;
  const int32_t* Sp = LEFT ? sr : sl;
  const int32_t* SSp = LEFT ? srr : sll;
  // ---- phase 1 ----
  {
    const int d = warp * 32 + lane;
    // column product sum at own tile column c: own(c) x partner(c -/+ d)
    auto col = [&](int c) {
      const int pc = c + (LEFT ? (D - 1) - d : d);
      int a = 0;
#pragma unroll
      for (int i = 0; i < k; ++i) a += (int)s_own[i * ow + c] * (int)s_par[i * pw + pc];
      return a;
    };
    int cross = 0;
    if (d < D) {
#pragma unroll
      for (int j = 0; j < k; ++j) cross += col(j);  // the window of x0
    }
    for (int t = 0; t < SL_SEG; ++t) {
      const int x = x0 + t;
      if (d < D && t > 0) cross += col(t + 2 * r) - col(t - 1);
      float cf = -INFINITY;
      const int px = LEFT ? x - d : x + d;
      if (d < D && rows_ok && x >= r && x < w - r && px - r >= 0 && px + r < w) {
        const int64_t po = (int64_t)y * w + x, pp = (int64_t)y * w + px;
        const long long S1 = So[po], SS1 = SSo[po], S2 = Sp[pp], SS2 = SSp[pp];
        const long long num = n * (long long)cross - S1 * S2;
        const long long vo = n * SS1 - S1 * S1, vp = n * SS2 - S2 * S2;
        if (vo > 0 && vp > 0) cf = (float)num * rsqrtf((float)vo * (float)vp);
      }
      float m = cf;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      const unsigned bits = __ballot_sync(0xffffffffu, cf != -INFINITY && cf >= m - 1e-5f);
      if (lane == 0) {
        s_fmax[warp * SL_SEG + t] = m;
        s_mask[warp * SL_SEG + t] = bits;
      }
    }
  }
  __syncthreads();
  // ---- phase 2: one lane per pixel ----
  if ((int)threadIdx.x < SL_SEG) {
    const int t = threadIdx.x, x = x0 + t;
    if (x < w) {
      float m = -INFINITY;
      for (int c2 = 0; c2 < nw; ++c2) m = fmaxf(m, s_fmax[c2 * SL_SEG + t]);
      const float cut = m - 1e-5f;
      double bc = -INFINITY;
      int bd = -1;
      if (m != -INFINITY) {
        const int64_t po = (int64_t)y * w + x;
        const long long S1 = So[po], SS1 = SSo[po];
        for (int c2 = 0; c2 < nw; ++c2) {
          if (!(s_fmax[c2 * SL_SEG + t] >= cut)) continue;  // no disparity of this warp near the top
          unsigned bits = s_mask[c2 * SL_SEG + t];
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int d = c2 * 32 + b;
            const int px = LEFT ? x - d : x + d;
            // the window cross sum from the tiles (own columns t .. t + 2r)
            int cross = 0;
            for (int i = 0; i < k; ++i)
              for (int j = 0; j < k; ++j)
                cross += (int)s_own[i * ow + t + j] *
                         (int)s_par[i * pw + t + j + (LEFT ? (D - 1) - d : d)];
            const int64_t pp = (int64_t)y * w + px;
            const long long S2 = Sp[pp], SS2 = SSp[pp];
            const long long num = n * (long long)cross - S1 * S2;
            const long long vo = n * SS1 - S1 * S1, vp = n * SS2 - S2 * S2;
            if ((float)num * rsqrtf((float)vo * (float)vp) < cut) continue;
            bool ok;
            const double v = LEFT ? zncc(n, S1, SS1, S2, SS2, cross, ok)
                                  : zncc(n, S2, SS2, S1, SS1, cross, ok);
            if (ok && v > bc) {  // ascending disparities: strict > keeps the smaller
              bc = v;
              bd = d;
            }
          }
        }
      }
      best_d[(int64_t)y * w + x] = bd;
      if (best_c) best_c[(int64_t)y * w + x] = bc;
    }
  }
}

// ZNCC of left pixel (y, x) at disparity d straight from the images (sub-pixel
// neighbours); ok = false where the oracle has no cost
__device__ double ncc_at(const uint8_t* __restrict__ L, const uint8_t* __restrict__ R, int h, int w,
                         int r, int y, int x, int d, const int32_t* __restrict__ sl,
                         const int32_t* __restrict__ sll, const int32_t* __restrict__ sr,
                         const int32_t* __restrict__ srr, bool& ok) {
  ok = false;
  if (y < r || y >= h - r || x - d - r < 0 || x + r >= w) return 0.0;
  int cross = 0;
  for (int i = -r; i <= r; ++i)
    for (int j = -r; j <= r; ++j)
      cross += (int)__ldg(L + (int64_t)(y + i) * w + x + j) * (int)__ldg(R + (int64_t)(y + i) * w + x + j - d);
  const long long n = (long long)(2 * r + 1) * (2 * r + 1);
  const int64_t pl = (int64_t)y * w + x, pr = (int64_t)y * w + x - d;
  return zncc(n, sl[pl], sll[pl], sr[pr], srr[pr], cross, ok);
}

__global__ void k_finish(const uint8_t* __restrict__ L, const uint8_t* __restrict__ R, int h, int w,
                         int D, int r, int lr_tol, double min_ncc, double fxb,
                         const int32_t* __restrict__ sl, const int32_t* __restrict__ sll,
                         const int32_t* __restrict__ sr, const int32_t* __restrict__ srr,
                         const int32_t* __restrict__ dL, const double* __restrict__ cL,
                         const int32_t* __restrict__ dR, int32_t* __restrict__ win,
                         double* __restrict__ disp, double* __restrict__ depth) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const int64_t p = (int64_t)y * w + x;
  const int d = dL[p];
  bool keep = d >= 0 && cL[p] >= min_ncc && x - d >= 0;
  if (keep) {
    const int drx = dR[(int64_t)y * w + (x - d)];
    keep = drx >= 0 && abs(drx - d) <= lr_tol;
  }
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  if (!keep) {
    win[p] = -1;
    disp[p] = nan;
    depth[p] = nan;
    return;
  }
  double delta = 0.0;
  if (d > 0 && d < D - 1) {
    bool okm, okp;
    const double cm = ncc_at(L, R, h, w, r, y, x, d - 1, sl, sll, sr, srr, okm);
    const double cp = ncc_at(L, R, h, w, r, y, x, d + 1, sl, sll, sr, srr, okp);
    if (okm && okp) {
      const double c0 = cL[p];
      const double den = (cm - 2.0 * c0) + cp;
      if (den < 0.0) delta = (cm - cp) / (2.0 * den);
    }
  }
  const double ds = (double)d + delta;
  win[p] = d;
  disp[p] = ds;
  depth[p] = ds > 0.0 ? fxb / ds : nan;
}

template <int RAD>
void launch_wta_r(dim3 grd, dim3 blk, size_t tile, cudaStream_t st, dt_stereo* s) {
#ifdef DT_STEREO_TILE_WTA
  k_wta<true, RAD><<<grd, blk, tile, st>>>(s->left, s->right, s->h, s->w, s->max_disp, s->sl,
                                           s->sll, s->sr, s->srr, s->dl, s->cl);
  k_wta<false, RAD><<<grd, blk, tile, st>>>(s->left, s->right, s->h, s->w, s->max_disp, s->sl,
                                            s->sll, s->sr, s->srr, s->dr, nullptr);
#else
  (void)grd;
  (void)blk;
  (void)tile;
  const int D = s->max_disp, r = RAD, k = 2 * RAD + 1, nw = (D + 31) / 32;
  const int ow = SL_SEG + 2 * r, pw = SL_SEG + 2 * r + D - 1;
  const size_t smem = (size_t)(k * (ow + pw) + 15) / 16 * 16 + (size_t)nw * SL_SEG * (sizeof(float) + sizeof(unsigned));
  const dim3 g2((s->w + SL_SEG - 1) / SL_SEG, s->h), b2(32 * nw);
  k_wta_slide<true, RAD><<<g2, b2, smem, st>>>(s->left, s->right, s->h, s->w, D, s->sl, s->sll,
                                               s->sr, s->srr, s->dl, s->cl);
  k_wta_slide<false, RAD><<<g2, b2, smem, st>>>(s->left, s->right, s->h, s->w, D, s->sl, s->sll,
                                                s->sr, s->srr, s->dr, nullptr);
#endif
}

int launch_wta(int r, dim3 grd, dim3 blk, size_t tile, cudaStream_t st, dt_stereo* s) {
  switch (r) {
    case 1: launch_wta_r<1>(grd, blk, tile, st, s); break;
    case 2: launch_wta_r<2>(grd, blk, tile, st, s); break;
    case 3: launch_wta_r<3>(grd, blk, tile, st, s); break;
    case 4: launch_wta_r<4>(grd, blk, tile, st, s); break;
    case 5: launch_wta_r<5>(grd, blk, tile, st, s); break;
    default: DT_REQUIRE(false, DT_ERR_UNSUPPORTED, "window radius %d", r);
  }
  return DT_OK;
}

}  // namespace
}  // namespace dt

using namespace dt;

extern "C" {

int dt_stereo_create(int height, int width, int max_disp, int radius, double fx, double baseline,
                     double min_ncc, int lr_tol, int device, dt_stereo** out) {
  DT_REQUIRE(out != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL handle");
  *out = nullptr;
  DT_REQUIRE(height > 0 && width > 0 && max_disp >= 1 && max_disp <= 1024, DT_ERR_INVALID_ARGUMENT,
             "bad image size or disparity range");
  DT_REQUIRE(radius >= 1 && radius <= ST_RMAX, DT_ERR_UNSUPPORTED, "window radius must lie in [1, %d]",
             ST_RMAX);
  DT_REQUIRE(fx > 0.0 && baseline > 0.0 && lr_tol >= 0, DT_ERR_INVALID_ARGUMENT,
             "need fx > 0, baseline > 0, lr_tol >= 0");
  DT_CHECK_CUDA(cudaSetDevice(device));
  dt_stereo* s = new dt_stereo();
  s->h = height;
  s->w = width;
  s->max_disp = max_disp;
  s->radius = radius;
  s->lr_tol = lr_tol;
  s->device = device;
  s->fxb = fx * baseline;
  s->min_ncc = min_ncc;
  const size_t np = (size_t)height * width;
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->left, 2 * np);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->sl, sizeof(int32_t) * 7 * np);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->cl, sizeof(double) * 3 * np);
  if (e != cudaSuccess) {
    dt_stereo_destroy(s);
    DT_CHECK_CUDA(e);
  }
  s->right = s->left + np;
  s->sll = s->sl + np;
  s->sr = s->sl + 2 * np;
  s->srr = s->sl + 3 * np;
  s->dl = s->sl + 4 * np;
  s->dr = s->sl + 5 * np;
  s->win = s->sl + 6 * np;
  s->depth = s->cl + np;
  s->disp = s->cl + 2 * np;
  *out = s;
  return DT_OK;
}

int dt_stereo_destroy(dt_stereo* s) {
  if (!s) return DT_OK;
  if (s->stream) {
    cudaStreamSynchronize(s->stream);
    cudaStreamDestroy(s->stream);
  }
  cudaFree(s->left);
  cudaFree(s->sl);
  cudaFree(s->cl);
  delete s;
  return DT_OK;
}

int dt_stereo_compute(dt_stereo* s, const uint8_t* left, const uint8_t* right, int on_device,
                      double* depth, double* disparity, int32_t* winner) {
  DT_REQUIRE(s != nullptr && left != nullptr && right != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_CHECK_CUDA(cudaSetDevice(s->device));
  const int h = s->h, w = s->w, r = s->radius, D = s->max_disp;
  const size_t np = (size_t)h * w;
  cudaStream_t st = s->stream;
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  DT_CHECK_CUDA(cudaMemcpyAsync(s->left, left, np, kind, st));
  DT_CHECK_CUDA(cudaMemcpyAsync(s->right, right, np, kind, st));
  const dim3 blk(ST_BX, ST_BY), grd((w + ST_BX - 1) / ST_BX, (h + ST_BY - 1) / ST_BY);
  k_box_stats<<<grd, blk, 0, st>>>(s->left, h, w, r, s->sl, s->sll);
  k_box_stats<<<grd, blk, 0, st>>>(s->right, h, w, r, s->sr, s->srr);
  DT_CHECK_LAUNCH();
  const size_t tile = (size_t)(ST_BX + 2 * r + D - 1) * (ST_BY + 2 * r);
  DT_TRY(launch_wta(r, grd, blk, tile, st, s));
  DT_CHECK_LAUNCH();
  k_finish<<<grd, blk, 0, st>>>(s->left, s->right, h, w, D, r, s->lr_tol, s->min_ncc, s->fxb, s->sl,
                                s->sll, s->sr, s->srr, s->dl, s->cl, s->dr, s->win, s->disp, s->depth);
  DT_CHECK_LAUNCH();
  if (depth) DT_CHECK_CUDA(cudaMemcpyAsync(depth, s->depth, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
  if (disparity)
    DT_CHECK_CUDA(cudaMemcpyAsync(disparity, s->disp, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
  if (winner) DT_CHECK_CUDA(cudaMemcpyAsync(winner, s->win, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, st));
  DT_CHECK_CUDA(cudaStreamSynchronize(st));
  return DT_OK;
}

int dt_stereo_last(dt_stereo* s, const double** depth) {
  DT_REQUIRE(s != nullptr && depth != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  *depth = s->depth;
  return DT_OK;
}

}  // extern "C"
