// dt_template.cu -- template-time graph construction on the device:
//
//  * dt_sample_control_points: warpfield.sample_control_points' greedy radius thinning
//    (warpfield.py:77-109) -- visit points in storage order, accept a point when its
//    squared distance to every accepted control is >= radius^2. The accepted set is the
//    lexicographically-first maximal independent set of the "closer than radius" conflict
//    graph in storage order; it is computed exactly by monotone rounds: a point is
//    accepted once every EARLIER conflicting point is rejected, rejected as soon as one
//    of them is accepted. Conflicts come from a uniform grid of cell size slightly above
//    the radius (so every conflict lies in the 27 neighbouring cells), and the squared
//    distances are evaluated in the reference's IEEE order (-fmad=false), so the result
//    is bit-identical to the sequential loop.
//  * dt_connection_candidates: the pairs (i < j) of build_connections
//    (warpfield.py:112-137) whose Gaussian weight can reach the prune threshold, in
//    lexicographic order, with their squared distances in the reference's order; the host
//    layer evaluates the weights with the reference's own numpy expression and applies the
//    exact prune, so edges and weights are bit-identical.
//
// Template-time only (once per sequence): host arrays in / out, internal device buffers.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "dt_common.cuh"

#ifndef DT_TRY
#define DT_TRY(expr)        \
  do {                      \
    int _st = (expr);       \
    if (_st != DT_OK)       \
      return _st;           \
  } while (0)
#endif

namespace dt {

namespace {

struct Grid {
  double ox, oy, oz, h;
  int64_t gx, gy, gz;
};

__device__ __forceinline__ int64_t cell_of(const Grid& g, double x, double y, double z, int64_t* c) {
  c[0] = (int64_t)floor((x - g.ox) / g.h);
  c[1] = (int64_t)floor((y - g.oy) / g.h);
  c[2] = (int64_t)floor((z - g.oz) / g.h);
  c[0] = c[0] < 0 ? 0 : (c[0] >= g.gx ? g.gx - 1 : c[0]);
  c[1] = c[1] < 0 ? 0 : (c[1] >= g.gy ? g.gy - 1 : c[1]);
  c[2] = c[2] < 0 ? 0 : (c[2] >= g.gz ? g.gz - 1 : c[2]);
  return c[0] + g.gx * (c[1] + g.gy * c[2]);
}

__global__ void k_cell_keys(const double* __restrict__ p, int64_t n, Grid g, int64_t* __restrict__ key) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c[3];
  key[i] = cell_of(g, p[3 * i], p[3 * i + 1], p[3 * i + 2], c);
}

// first index of `key` in the sorted array (lower bound)
__device__ __forceinline__ int64_t lower_bound(const int64_t* __restrict__ a, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// squared distance in the reference's order: sum((chosen - p)^2, axis=1)
__device__ __forceinline__ double d2_ref(const double* __restrict__ p, int64_t j, int64_t i) {
  const double dx = p[3 * j] - p[3 * i];
  const double dy = p[3 * j + 1] - p[3 * i + 1];
  const double dz = p[3 * j + 2] - p[3 * i + 2];
  return (dx * dx + dy * dy) + dz * dz;
}

// earlier conflicting points of every point (j < i, d2 < r^2): count (fill == nullptr)
// or write at off[i]
__global__ void k_conflicts(const double* __restrict__ p, int64_t n, Grid g, double r2,
                            const int64_t* __restrict__ skey, const int32_t* __restrict__ sidx,
                            const int64_t* __restrict__ off, int32_t* __restrict__ cnt,
                            int32_t* __restrict__ fill) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c[3];
  cell_of(g, p[3 * i], p[3 * i + 1], p[3 * i + 2], c);
  int32_t k = 0;
  int64_t o = fill ? off[i] : 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
        if (x < 0 || y < 0 || z < 0 || x >= g.gx || y >= g.gy || z >= g.gz) continue;
        const int64_t key = x + g.gx * (y + g.gy * z);
        for (int64_t q = lower_bound(skey, n, key); q < n && skey[q] == key; ++q) {
          const int32_t j = sidx[q];
          if (j >= i) continue;
          if (d2_ref(p, j, i) < r2) {
            if (fill) fill[o++] = j;
            ++k;
          }
        }
      }
  if (!fill) cnt[i] = k;
}

// one monotone round of the storage-order greedy: 0 undecided, 1 accepted, 2 rejected
__global__ void k_mis_round(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ nb,
                            int8_t* __restrict__ state, int* __restrict__ undecided) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || state[i] != 0) return;
  bool pending = false;
  for (int64_t q = off[i]; q < off[i + 1]; ++q) {
    const int8_t s = ((volatile int8_t*)state)[nb[q]];
    if (s == 1) {
      state[i] = 2;
      return;
    }
    if (s == 0) pending = true;
  }
  if (!pending) state[i] = 1;
  else atomicAdd(undecided, 1);
}

// connections of row i: j > i with d2 <= thr (candidates: d2out = d2); with two_s2 > 0
// the weight w = exp(-d2 / two_s2) is formed here too (the reference's operation order)
// and only w >= prune is kept (d2out = w; build_connections, warpfield.py:112-137, up to
// the last ulp of exp)
__global__ void k_conn(const double* __restrict__ c, int64_t m, double thr,
                       const int64_t* __restrict__ off, int32_t* __restrict__ cnt,
                       int64_t* __restrict__ edges, double* __restrict__ d2out,
                       double two_s2 = 0.0, double prune = 0.0) {
  const int64_t i = blockIdx.x;
  if (i >= m) return;
  __shared__ int s_warp[32];
  int64_t base = edges ? off[i] : 0;
  int total = 0;
  for (int64_t j0 = i + 1; j0 < m; j0 += blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    bool keep = false;
    double d2 = 0.0;
    if (j < m) {
      // reference order: sum((pts[ii] - pts[jj])**2, axis=1)
      const double dx = c[3 * i] - c[3 * j], dy = c[3 * i + 1] - c[3 * j + 1],
                   dz = c[3 * i + 2] - c[3 * j + 2];
      d2 = (dx * dx + dy * dy) + dz * dz;
      keep = d2 <= thr;
      if (keep && two_s2 > 0.0) {
        d2 = exp(-d2 / two_s2);  // the weight
        keep = d2 >= prune;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    int before = 0, blk = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) before += s_warp[w];
      blk += s_warp[w];
    }
    if (keep && edges) {
      const int64_t o = base + total + before + __popc(bal & ((1u << lane) - 1u));
      edges[2 * o] = i;
      edges[2 * o + 1] = j;
      d2out[o] = d2;
    }
    total += blk;
    __syncthreads();
  }
  if (!edges && threadIdx.x == 0) cnt[i] = total;
}

template <typename T>
int dmalloc(T** p, size_t count) {
  DT_CHECK_CUDA(cudaMalloc((void**)p, sizeof(T) * (count > 0 ? count : 1)));
  return DT_OK;
}

// ---------------------------------------------------------------------------------
// correspond.estimate_point_normals (correspond.py:198-220): the k nearest points of
// every point (itself included; exact brute force with the key (squared distance,
// index), i.e. ties at the k-th neighbour go to the lower index), their mean and 3x3
// scatter in nearest-first order, the eigenvector of the smallest eigenvalue (cyclic
// Jacobi), oriented toward the camera at the origin (n . p < 0) and normalized.
// One thread per point; candidates stream through shared memory in tiles.
// ---------------------------------------------------------------------------------
constexpr int NRM_KMAX = 16;
constexpr int NRM_TILE = 256;

__device__ __forceinline__ bool key_less(double d, int j, double e, int i) {
  return d < e || (d == e && j < i);
}

__device__ void sym3_min_eigvec(double a00, double a01, double a02, double a11, double a12,
                                double a22, double v[3]) {
  double a[3][3] = {{a00, a01, a02}, {a01, a11, a12}, {a02, a12, a22}};
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double dia = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (off == 0.0 || off <= 1e-36 * dia) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      if (a[p][q] == 0.0) continue;
      const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
      const double t = th == 0.0 ? 1.0 : copysign(1.0, th) / (fabs(th) + sqrt(th * th + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const double ap = a[r][p], aq = a[r][q];
        a[r][p] = c * ap - sn * aq;
        a[r][q] = sn * ap + c * aq;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const double ap = a[p][r], aq = a[q][r];
        a[p][r] = c * ap - sn * aq;
        a[q][r] = sn * ap + c * aq;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const double vp = V[r][p], vq = V[r][q];
        V[r][p] = c * vp - sn * vq;
        V[r][q] = sn * vp + c * vq;
      }
    }
  }
  int im = 0;
  if (a[1][1] < a[im][im]) im = 1;
  if (a[2][2] < a[im][im]) im = 2;
  v[0] = V[0][im];
  v[1] = V[1][im];
  v[2] = V[2][im];
}

__global__ void __launch_bounds__(NRM_TILE)
k_point_normals(const double* __restrict__ pts, int64_t n, int k, double* __restrict__ out) {
  __shared__ double sx[NRM_TILE], sy[NRM_TILE], sz[NRM_TILE];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < n;
  double px = 0.0, py = 0.0, pz = 0.0;
  if (live) {
    px = pts[3 * i];
    py = pts[3 * i + 1];
    pz = pts[3 * i + 2];
  }
  double bd[NRM_KMAX];
  int bi[NRM_KMAX];
#pragma unroll
  for (int s = 0; s < NRM_KMAX; ++s) {
    bd[s] = INFINITY;
    bi[s] = 0x7fffffff;
  }
  double thr = INFINITY;  // key of the current k-th neighbour
  int thi = 0x7fffffff;
  for (int64_t base = 0; base < n; base += NRM_TILE) {
    const int64_t j = base + threadIdx.x;
    __syncthreads();
    if (j < n) {
      sx[threadIdx.x] = pts[3 * j];
      sy[threadIdx.x] = pts[3 * j + 1];
      sz[threadIdx.x] = pts[3 * j + 2];
    }
    __syncthreads();
    const int cnt = (int)(n - base < NRM_TILE ? n - base : NRM_TILE);
    if (!live) continue;
    for (int u = 0; u < cnt; ++u) {
      const double dx = sx[u] - px, dy = sy[u] - py, dz = sz[u] - pz;
      const double d = dx * dx + dy * dy + dz * dz;
      const int jj = (int)(base + u);
      if (!key_less(d, jj, thr, thi)) continue;
      // sorted insertion of (d, jj)
#pragma unroll
      for (int s = NRM_KMAX - 1; s > 0; --s) {
        if (key_less(d, jj, bd[s - 1], bi[s - 1])) {
          bd[s] = bd[s - 1];
          bi[s] = bi[s - 1];
        } else if (key_less(d, jj, bd[s], bi[s])) {
          bd[s] = d;
          bi[s] = jj;
        }
      }
      if (key_less(d, jj, bd[0], bi[0])) {
        bd[0] = d;
        bi[0] = jj;
      }
#pragma unroll
      for (int s = 0; s < NRM_KMAX; ++s)
        if (s == k - 1) {
          thr = bd[s];
          thi = bi[s];
        }
    }
  }
  if (!live) return;
  // neighbourhood mean and scatter in nearest-first order
  double mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
  for (int s = 0; s < NRM_KMAX; ++s)
    if (s < k) {
      mx += pts[3 * (int64_t)bi[s]];
      my += pts[3 * (int64_t)bi[s] + 1];
      mz += pts[3 * (int64_t)bi[s] + 2];
    }
  mx /= (double)k;
  my /= (double)k;
  mz /= (double)k;
  double c00 = 0, c01 = 0, c02 = 0, c11 = 0, c12 = 0, c22 = 0;
#pragma unroll
  for (int s = 0; s < NRM_KMAX; ++s)
    if (s < k) {
      const double x = pts[3 * (int64_t)bi[s]] - mx, y = pts[3 * (int64_t)bi[s] + 1] - my,
                   z = pts[3 * (int64_t)bi[s] + 2] - mz;
      c00 += x * x;
      c01 += x * y;
      c02 += x * z;
      c11 += y * y;
      c12 += y * z;
      c22 += z * z;
    }
  double v[3];
  sym3_min_eigvec(c00, c01, c02, c11, c12, c22, v);
  if (v[0] * px + v[1] * py + v[2] * pz > 0.0) {
    v[0] = -v[0];
    v[1] = -v[1];
    v[2] = -v[2];
  }
  const double nn = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  const double den = nn > 0.0 ? nn : 1.0;
  out[3 * i] = v[0] / den;
  out[3 * i + 1] = v[1] / den;
  out[3 * i + 2] = v[2] / den;
}

struct Freer {
  std::vector<void*> ptrs;
  ~Freer() {
    for (void* p : ptrs) cudaFree(p);
  }
};

}  // namespace

}  // namespace dt

using namespace dt;

extern "C" {

int dt_sample_control_points(const double* points, int64_t n, double radius, int64_t* control_index,
                             int64_t* m_out, int device) {
  DT_REQUIRE(points != nullptr && control_index != nullptr && m_out != nullptr,
             DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_REQUIRE(n > 0, DT_ERR_EMPTY_TEMPLATE, "cannot sample control points from an empty template");
  DT_REQUIRE(radius > 0.0, DT_ERR_INVALID_ARGUMENT, "sampling radius must be positive");
  DT_REQUIRE(n < (1ll << 31), DT_ERR_UNSUPPORTED, "template too large");
  DT_CHECK_CUDA(cudaSetDevice(device));
  cudaStream_t s = nullptr;
  // grid: cell size just above the radius, so every conflict is in a neighbouring cell
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      DT_REQUIRE(std::isfinite(points[3 * i + d]), DT_ERR_INVALID_ARGUMENT, "non-finite template point");
      lo[d] = std::min(lo[d], points[3 * i + d]);
      hi[d] = std::max(hi[d], points[3 * i + d]);
    }
  Grid g;
  g.h = radius * (1.0 + 1e-6);
  g.ox = lo[0];
  g.oy = lo[1];
  g.oz = lo[2];
  g.gx = (int64_t)std::floor((hi[0] - lo[0]) / g.h) + 1;
  g.gy = (int64_t)std::floor((hi[1] - lo[1]) / g.h) + 1;
  g.gz = (int64_t)std::floor((hi[2] - lo[2]) / g.h) + 1;
  DT_REQUIRE((double)g.gx * g.gy * g.gz < 4e18, DT_ERR_UNSUPPORTED, "grid too large");
  Freer fr;
  double* d_p;
  int64_t *d_key, *d_off;
  int32_t *d_cnt, *d_sidx;
  int8_t* d_state;
  int* d_und;
  DT_TRY(dmalloc(&d_p, 3 * n));
  fr.ptrs.push_back(d_p);
  DT_TRY(dmalloc(&d_key, n));
  fr.ptrs.push_back(d_key);
  DT_TRY(dmalloc(&d_off, n + 1));
  fr.ptrs.push_back(d_off);
  DT_TRY(dmalloc(&d_cnt, n));
  fr.ptrs.push_back(d_cnt);
  DT_TRY(dmalloc(&d_sidx, n));
  fr.ptrs.push_back(d_sidx);
  DT_TRY(dmalloc(&d_state, n));
  fr.ptrs.push_back(d_state);
  DT_TRY(dmalloc(&d_und, 1));
  fr.ptrs.push_back(d_und);
  DT_CHECK_CUDA(cudaMemcpy(d_p, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  const int T = 256;
  const unsigned B = (unsigned)((n + T - 1) / T);
  k_cell_keys<<<B, T, 0, s>>>(d_p, n, g, d_key);
  DT_CHECK_LAUNCH();
  // sort (key, index) by key on the host (template time)
  std::vector<int64_t> key(n);
  DT_CHECK_CUDA(cudaMemcpy(key.data(), d_key, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  std::vector<int32_t> order(n);
  for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
  std::vector<int64_t> skey(n);
  for (int64_t i = 0; i < n; ++i) skey[i] = key[order[i]];
  DT_CHECK_CUDA(cudaMemcpy(d_key, skey.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
  DT_CHECK_CUDA(cudaMemcpy(d_sidx, order.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  const double r2 = radius * radius;
  k_conflicts<<<B, T, 0, s>>>(d_p, n, g, r2, d_key, d_sidx, nullptr, d_cnt, nullptr);
  DT_CHECK_LAUNCH();
  std::vector<int32_t> cnt(n);
  DT_CHECK_CUDA(cudaMemcpy(cnt.data(), d_cnt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  std::vector<int64_t> off(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) off[i + 1] = off[i] + cnt[i];
  DT_CHECK_CUDA(cudaMemcpy(d_off, off.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  int32_t* d_nb;
  DT_TRY(dmalloc(&d_nb, off[n]));
  fr.ptrs.push_back(d_nb);
  k_conflicts<<<B, T, 0, s>>>(d_p, n, g, r2, d_key, d_sidx, d_off, nullptr, d_nb);
  DT_CHECK_LAUNCH();
  DT_CHECK_CUDA(cudaMemset(d_state, 0, n));
  // monotone rounds until every point is decided (several rounds per host check)
  for (int64_t round = 0;; round += 8) {
    DT_CHECK_CUDA(cudaMemset(d_und, 0, sizeof(int)));
    for (int r = 0; r < 8; ++r) {
      if (r == 7) DT_CHECK_CUDA(cudaMemset(d_und, 0, sizeof(int)));
      k_mis_round<<<B, T, 0, s>>>(n, d_off, d_nb, d_state, d_und);
      DT_CHECK_LAUNCH();
    }
    int und = 0;
    DT_CHECK_CUDA(cudaMemcpy(&und, d_und, sizeof(int), cudaMemcpyDeviceToHost));
    if (und == 0) break;
    DT_REQUIRE(round < 4 * n, DT_ERR_CUDA, "control sampling did not converge");
  }
  std::vector<int8_t> state(n);
  DT_CHECK_CUDA(cudaMemcpy(state.data(), d_state, n, cudaMemcpyDeviceToHost));
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (state[i] == 1) control_index[m++] = i;
  *m_out = m;
  return DT_OK;
}

int dt_connection_candidates(const double* ctrl, int64_t m, double d2_max, int64_t* edges,
                             double* d2, int64_t capacity, int64_t* e_out, int device) {
  DT_REQUIRE(ctrl != nullptr && e_out != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_REQUIRE(m >= 0 && m < (1ll << 31), DT_ERR_INVALID_ARGUMENT, "bad control count");
  *e_out = 0;
  if (m < 2) return DT_OK;
  DT_CHECK_CUDA(cudaSetDevice(device));
  Freer fr;
  double *d_c, *d_d2;
  int64_t *d_off, *d_e;
  int32_t* d_cnt;
  DT_TRY(dmalloc(&d_c, 3 * m));
  fr.ptrs.push_back(d_c);
  DT_TRY(dmalloc(&d_off, m + 1));
  fr.ptrs.push_back(d_off);
  DT_TRY(dmalloc(&d_cnt, m));
  fr.ptrs.push_back(d_cnt);
  DT_CHECK_CUDA(cudaMemcpy(d_c, ctrl, sizeof(double) * 3 * m, cudaMemcpyHostToDevice));
  k_conn<<<(unsigned)m, 256>>>(d_c, m, d2_max, nullptr, d_cnt, nullptr, nullptr);
  DT_CHECK_LAUNCH();
  std::vector<int32_t> cnt(m);
  DT_CHECK_CUDA(cudaMemcpy(cnt.data(), d_cnt, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
  std::vector<int64_t> off(m + 1, 0);
  for (int64_t i = 0; i < m; ++i) off[i + 1] = off[i] + cnt[i];
  const int64_t e = off[m];
  *e_out = e;
  if (edges == nullptr || d2 == nullptr) return DT_OK;  // count query
  DT_REQUIRE(capacity >= e, DT_ERR_INVALID_ARGUMENT, "edge capacity %lld < %lld",
             (long long)capacity, (long long)e);
  DT_TRY(dmalloc(&d_e, 2 * e));
  fr.ptrs.push_back(d_e);
  DT_TRY(dmalloc(&d_d2, e));
  fr.ptrs.push_back(d_d2);
  DT_CHECK_CUDA(cudaMemcpy(d_off, off.data(), sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice));
  k_conn<<<(unsigned)m, 256>>>(d_c, m, d2_max, d_off, nullptr, d_e, d_d2);
  DT_CHECK_LAUNCH();
  DT_CHECK_CUDA(cudaMemcpy(edges, d_e, sizeof(int64_t) * 2 * e, cudaMemcpyDeviceToHost));
  DT_CHECK_CUDA(cudaMemcpy(d2, d_d2, sizeof(double) * e, cudaMemcpyDeviceToHost));
  return DT_OK;
}

int dt_build_connections(const double* ctrl, int64_t m, double sigma, double prune,
                         int64_t* edges, double* weights, int64_t capacity, int64_t* e_out,
                         int device) {
  DT_REQUIRE(ctrl != nullptr && e_out != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_REQUIRE(m >= 0 && m < (1ll << 31), DT_ERR_INVALID_ARGUMENT, "bad control count");
  DT_REQUIRE(sigma > 0.0 && prune > 0.0 && prune <= 1.0, DT_ERR_INVALID_ARGUMENT,
             "need sigma > 0 and 0 < prune <= 1");
  *e_out = 0;
  if (m < 2) return DT_OK;
  DT_CHECK_CUDA(cudaSetDevice(device));
  // w >= prune <=> d2 <= -2 sigma^2 ln(prune): a hair above it bounds the candidates, the
  // weight itself decides
  const double two_s2 = 2.0 * sigma * sigma;
  const double thr = -std::log(prune) * two_s2 * (1.0 + 1e-9);
  Freer fr;
  double *d_c, *d_w;
  int64_t *d_off, *d_e;
  int32_t* d_cnt;
  DT_TRY(dmalloc(&d_c, 3 * m));
  fr.ptrs.push_back(d_c);
  DT_TRY(dmalloc(&d_off, m + 1));
  fr.ptrs.push_back(d_off);
  DT_TRY(dmalloc(&d_cnt, m));
  fr.ptrs.push_back(d_cnt);
  DT_CHECK_CUDA(cudaMemcpy(d_c, ctrl, sizeof(double) * 3 * m, cudaMemcpyHostToDevice));
  k_conn<<<(unsigned)m, 256>>>(d_c, m, thr, nullptr, d_cnt, nullptr, nullptr, two_s2, prune);
  DT_CHECK_LAUNCH();
  std::vector<int32_t> cnt(m);
  DT_CHECK_CUDA(cudaMemcpy(cnt.data(), d_cnt, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
  std::vector<int64_t> off(m + 1, 0);
  for (int64_t i = 0; i < m; ++i) off[i + 1] = off[i] + cnt[i];
  const int64_t e = off[m];
  *e_out = e;
  if (edges == nullptr || weights == nullptr) return DT_OK;  // count query
  DT_REQUIRE(capacity >= e, DT_ERR_INVALID_ARGUMENT, "edge capacity %lld < %lld",
             (long long)capacity, (long long)e);
  DT_TRY(dmalloc(&d_e, 2 * e));
  fr.ptrs.push_back(d_e);
  DT_TRY(dmalloc(&d_w, e));
  fr.ptrs.push_back(d_w);
  DT_CHECK_CUDA(cudaMemcpy(d_off, off.data(), sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice));
  k_conn<<<(unsigned)m, 256>>>(d_c, m, thr, d_off, nullptr, d_e, d_w, two_s2, prune);
  DT_CHECK_LAUNCH();
  DT_CHECK_CUDA(cudaMemcpy(edges, d_e, sizeof(int64_t) * 2 * e, cudaMemcpyDeviceToHost));
  DT_CHECK_CUDA(cudaMemcpy(weights, d_w, sizeof(double) * e, cudaMemcpyDeviceToHost));
  return DT_OK;
}

int dt_estimate_point_normals(const double* points, int64_t n, int64_t k, double* normals,
                              int device) {
  DT_REQUIRE(points != nullptr && normals != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_REQUIRE(n >= 0 && n < (1ll << 31), DT_ERR_UNSUPPORTED, "point count out of range");
  DT_REQUIRE(k >= 1, DT_ERR_INVALID_ARGUMENT, "k must be positive");
  const int64_t ke = std::min<int64_t>(k, n);
  if (n < 3 || ke < 3) {  // too few points: the camera-facing default (correspond.py:205-207)
    for (int64_t i = 0; i < n; ++i) {
      normals[3 * i] = 0.0;
      normals[3 * i + 1] = 0.0;
      normals[3 * i + 2] = -1.0;
    }
    return DT_OK;
  }
  DT_REQUIRE(ke <= NRM_KMAX, DT_ERR_UNSUPPORTED, "k=%lld above the device limit %d", (long long)ke,
             NRM_KMAX);
  DT_CHECK_CUDA(cudaSetDevice(device));
  Freer fr;
  double *d_p, *d_n;
  DT_TRY(dmalloc(&d_p, 3 * n));
  fr.ptrs.push_back(d_p);
  DT_TRY(dmalloc(&d_n, 3 * n));
  fr.ptrs.push_back(d_n);
  DT_CHECK_CUDA(cudaMemcpy(d_p, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  k_point_normals<<<(unsigned)((n + NRM_TILE - 1) / NRM_TILE), NRM_TILE>>>(d_p, n, (int)ke, d_n);
  DT_CHECK_LAUNCH();
  DT_CHECK_CUDA(cudaMemcpy(normals, d_n, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
  return DT_OK;
}

}  // extern "C"
