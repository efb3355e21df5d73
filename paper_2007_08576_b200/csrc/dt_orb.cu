// ORB front end on the device ("FAST + uniform
// suppression + rBRIEF"): the stage upstream of the Hamming matcher (a4) that turns a
// grey image into the frame keypoints / 256-bit descriptors dt_track_frame consumes.
// The reference has no ORB code; the algorithm is defined by the restatement
// in oracle/orb.py and matched exactly:
//
//   k_fast_score    FAST-9 score per pixel (16-pixel circle of radius 3)
//   k_box5          5x5 box sums (the BRIEF test values)
//   k_nms_collect   3x3 non-maximum suppression, candidates keyed (cell, -score, index)
//   cub radix sort  -> k_cell_rank: the best `per_cell` of every cell, keyed (-score, index)
//   cub radix sort  -> the best n_max overall
//   k_describe      one warp per keypoint: intensity-centroid moments over the r = 15 disc,
//                   sector by exact sign tests, 256 rotated tests -> 32 bytes
//
// All integer arithmetic (scores, moments, box sums) is exact; the sector test uses the
// host's boundary table with IEEE products (-fmad=false), so the device output equals the
// oracle's bit for bit. One dt_orb context per image size holds the tables and scratch.

#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
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

constexpr int ORB_BORDER = 21;
constexpr int ORB_BINS = 30;
constexpr int ORB_TESTS = 256;

__constant__ int8_t c_circle[32];  // 16 (dx, dy)

__global__ void k_fast_score(const uint8_t* __restrict__ img, int h, int w, int32_t* __restrict__ score) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  int best = 0;
  if (x >= 3 && x < w - 3 && y >= 3 && y < h - 3) {
    const int c = __ldg(img + (int64_t)y * w + x);
    int ring[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      ring[k] = __ldg(img + (int64_t)(y + c_circle[2 * k + 1]) * w + (x + c_circle[2 * k]));
#pragma unroll
    for (int sg = 0; sg < 2; ++sg) {
      int d[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) d[k] = sg == 0 ? ring[k] - c : c - ring[k];
#pragma unroll
      for (int s0 = 0; s0 < 16; ++s0) {
        int mn = d[s0];
#pragma unroll
        for (int k = 1; k < 9; ++k) mn = min(mn, d[(s0 + k) & 15]);
        best = max(best, mn);
      }
    }
  }
  score[(int64_t)y * w + x] = best;
}

__global__ void k_box5(const uint8_t* __restrict__ img, int h, int w, int32_t* __restrict__ box) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  int s = 0;
#pragma unroll
  for (int dy = -2; dy <= 2; ++dy)
#pragma unroll
    for (int dx = -2; dx <= 2; ++dx) {
      const int yy = y + dy, xx = x + dx;
      if (yy >= 0 && yy < h && xx >= 0 && xx < w) s += __ldg(img + (int64_t)yy * w + xx);
    }
  box[(int64_t)y * w + x] = s;
}

// Sort keys, packed as tight as the image allows so the radix sorts run few passes:
// key = cell << (ib + 8) | (255 - score) << ib | pixel index, ib = bits of an index.
// candidates: corners (score > threshold) inside the descriptor border that no 3x3
// neighbour beats in the order (score, -index)
__global__ void k_nms_collect(const int32_t* __restrict__ score, int h, int w, int threshold,
                              int cell, int ncx, int ib, unsigned long long* __restrict__ keys,
                              unsigned* __restrict__ count, int cap) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x < ORB_BORDER || y < ORB_BORDER || x >= w - ORB_BORDER || y >= h - ORB_BORDER) return;
  const int64_t i = (int64_t)y * w + x;
  const int s = score[i];
  if (s <= threshold) return;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dx == 0 && dy == 0) continue;
      const int64_t j = i + (int64_t)dy * w + dx;
      const int t = score[j];
      if (t > s || (t == s && j < i)) return;
    }
  const unsigned slot = atomicAdd(count, 1u);
  if ((int)slot >= cap) return;
  const unsigned long long cid = (unsigned long long)((y / cell) * ncx + x / cell);
  keys[slot] = (cid << (ib + 8)) | ((unsigned long long)(255 - s) << ib) | (unsigned long long)i;
}

// rank of every sorted candidate inside its cell (sorted by cell, then -score, index):
// the first `per_cell` pass on, re-keyed (255 - score) << ib | index
__global__ void k_cell_rank(const unsigned long long* __restrict__ sorted, int n, int per_cell,
                            int ib, unsigned long long* __restrict__ out,
                            unsigned* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = sorted[i];
  if (k == ~0ull) return;  // padding (the sorts run over the full capacity, no host sync)
  const unsigned long long cell = k >> (ib + 8);
  int lo = 0, hi = i;  // first position with this cell
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((sorted[mid] >> (ib + 8)) < cell) lo = mid + 1;
    else hi = mid;
  }
  if (i - lo >= per_cell) return;
  out[atomicAdd(count, 1u)] = k & ((1ull << (ib + 8)) - 1);
}

// one warp per keypoint
__global__ void k_describe(const uint8_t* __restrict__ img, const int32_t* __restrict__ box, int w,
                           const unsigned long long* __restrict__ sel,
                           const unsigned* __restrict__ n_sel, int n_max, int ib,
                           const int16_t* __restrict__ disc, int n_disc,
                           const double* __restrict__ bnd, const int8_t* __restrict__ rot,
                           int32_t* __restrict__ kp, uint8_t* __restrict__ desc,
                           int32_t* __restrict__ score, int32_t* __restrict__ bins) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int n = min((int)*n_sel, n_max);
  if (k >= n) return;
  const unsigned long long key = sel[k];
  const int64_t lin = (int64_t)(key & ((1ull << ib) - 1));
  const int y = (int)(lin / w), x = (int)(lin - (int64_t)y * w);
  long long m10 = 0, m01 = 0;
  for (int q = lane; q < n_disc; q += 32) {
    const int ox = disc[2 * q], oy = disc[2 * q + 1];
    const long long v = __ldg(img + (int64_t)(y + oy) * w + (x + ox));
    m10 += ox * v;
    m01 += oy * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m10 += __shfl_xor_sync(0xffffffffu, m10, o);
    m01 += __shfl_xor_sync(0xffffffffu, m01, o);
  }
  // sector j: cross(b_j, v) >= 0 and cross(b_{j+1}, v) < 0 (oracle/orb.py sector_of)
  int bin = 0;
  if (m10 == 0 && m01 == 0) {
    bin = ORB_BINS / 2;
  } else {
    const double vx = (double)m10, vy = (double)m01;
    int found = -1;
    if (lane < ORB_BINS) {
      const double c0 = bnd[2 * lane] * vy - bnd[2 * lane + 1] * vx;
      const double c1 = bnd[2 * lane + 2] * vy - bnd[2 * lane + 3] * vx;
      if (c0 >= 0.0 && c1 < 0.0) found = lane;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, found >= 0);
    bin = hit ? __ffs(hit) - 1 : 0;
  }
  // tests 8 lane .. 8 lane + 7 -> byte `lane`
  const int8_t* t = rot + ((size_t)bin * ORB_TESTS + 8 * lane) * 4;
  unsigned byte = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ax = t[4 * j], ay = t[4 * j + 1], bx = t[4 * j + 2], by = t[4 * j + 3];
    const int va = __ldg(box + (int64_t)(y + ay) * w + (x + ax));
    const int vb = __ldg(box + (int64_t)(y + by) * w + (x + bx));
    byte |= (va < vb ? 1u : 0u) << j;
  }
  desc[(size_t)k * 32 + lane] = (uint8_t)byte;
  if (lane == 0) {
    kp[2 * k] = x;
    kp[2 * k + 1] = y;
    score[k] = 255 - (int)((key >> ib) & 0xff);
    bins[k] = bin;
  }
}

}  // namespace
}  // namespace dt

using namespace dt;

struct dt_orb {
  int device = 0;
  int h = 0, w = 0, threshold = 20, cell = 32, per_cell = 8, n_max = 2500;
  cudaStream_t stream = nullptr;
  uint8_t* img = nullptr;
  int32_t *score = nullptr, *box = nullptr;
  unsigned long long *keys = nullptr, *keys2 = nullptr, *sel = nullptr, *sel2 = nullptr;
  unsigned* counts = nullptr;  // [2]
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int cap = 0;
  int16_t* disc = nullptr;
  int n_disc = 0;
  double* bnd = nullptr;
  int8_t* rot = nullptr;
  int32_t *o_kp = nullptr, *o_score = nullptr, *o_bin = nullptr;
  int64_t n_last = 0;
  uint8_t* o_desc = nullptr;
};

namespace {

void orb_free(dt_orb* o) {
  if (!o) return;
  for (void* p : {(void*)o->img, (void*)o->score, (void*)o->box, (void*)o->keys, (void*)o->keys2,
                  (void*)o->sel, (void*)o->sel2, (void*)o->counts, o->tmp, (void*)o->disc,
                  (void*)o->bnd, (void*)o->rot, (void*)o->o_kp, (void*)o->o_score,
                  (void*)o->o_bin, (void*)o->o_desc})
    if (p) cudaFree(p);
  if (o->stream) cudaStreamDestroy(o->stream);
  delete o;
}

template <typename T>
int orb_alloc(T** p, size_t n) {
  DT_CHECK_CUDA(cudaMalloc((void**)p, sizeof(T) * std::max<size_t>(n, 1)));
  return DT_OK;
}

int orb_init(dt_orb* o, const int8_t* pattern_rot, const double* boundaries) {
  const size_t npix = (size_t)o->h * o->w;
  DT_CHECK_CUDA(cudaStreamCreateWithFlags(&o->stream, cudaStreamNonBlocking));
  o->cap = (int)std::min<size_t>(npix / 4 + 1024, (size_t)1 << 24);
  DT_TRY(orb_alloc(&o->img, npix));
  DT_TRY(orb_alloc(&o->score, npix));
  DT_TRY(orb_alloc(&o->box, npix));
  DT_TRY(orb_alloc(&o->keys, o->cap));
  DT_TRY(orb_alloc(&o->keys2, o->cap));
  DT_TRY(orb_alloc(&o->sel, o->cap));
  DT_TRY(orb_alloc(&o->sel2, o->cap));
  DT_TRY(orb_alloc(&o->counts, 2));
  size_t b1 = 0, b2 = 0;
  DT_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, o->keys, o->keys2, o->cap, 0, 64));
  DT_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b2, o->sel, o->sel2, o->cap, 0, 40));
  o->tmp_bytes = std::max(b1, b2);
  DT_TRY(orb_alloc((char**)&o->tmp, o->tmp_bytes));
  // disc offsets of the orientation moments (r = 15), row-major
  std::vector<int16_t> disc;
  for (int oy = -15; oy <= 15; ++oy)
    for (int ox = -15; ox <= 15; ++ox)
      if (ox * ox + oy * oy <= 225) {
        disc.push_back((int16_t)ox);
        disc.push_back((int16_t)oy);
      }
  o->n_disc = (int)(disc.size() / 2);
  DT_TRY(orb_alloc(&o->disc, disc.size()));
  DT_CHECK_CUDA(cudaMemcpy(o->disc, disc.data(), sizeof(int16_t) * disc.size(), cudaMemcpyHostToDevice));
  DT_TRY(orb_alloc(&o->bnd, 2 * (ORB_BINS + 1)));
  DT_CHECK_CUDA(cudaMemcpy(o->bnd, boundaries, sizeof(double) * 2 * (ORB_BINS + 1), cudaMemcpyHostToDevice));
  DT_TRY(orb_alloc(&o->rot, (size_t)ORB_BINS * ORB_TESTS * 4));
  DT_CHECK_CUDA(cudaMemcpy(o->rot, pattern_rot, (size_t)ORB_BINS * ORB_TESTS * 4, cudaMemcpyHostToDevice));
  DT_TRY(orb_alloc(&o->o_kp, 2 * (size_t)o->n_max));
  DT_TRY(orb_alloc(&o->o_score, o->n_max));
  DT_TRY(orb_alloc(&o->o_bin, o->n_max));
  DT_TRY(orb_alloc(&o->o_desc, 32 * (size_t)o->n_max));
  static const int8_t circle[32] = {0, -3, 1, -3, 2, -2, 3, -1, 3, 0, 3, 1, 2, 2, 1, 3,
                                    0, 3, -1, 3, -2, 2, -3, 1, -3, 0, -3, -1, -2, -2, -1, -3};
  DT_CHECK_CUDA(cudaMemcpyToSymbol(c_circle, circle, sizeof(circle)));
  return DT_OK;
}

}  // namespace

extern "C" {

int dt_orb_create(int height, int width, int threshold, int cell, int per_cell, int n_max,
                  const int8_t* pattern_rot, const double* boundaries, int device, dt_orb** out) {
  DT_REQUIRE(out != nullptr && pattern_rot != nullptr && boundaries != nullptr,
             DT_ERR_INVALID_ARGUMENT, "NULL argument");
  DT_REQUIRE(height > 2 * ORB_BORDER && width > 2 * ORB_BORDER, DT_ERR_INVALID_ARGUMENT,
             "image smaller than the descriptor border (%d px)", ORB_BORDER);
  DT_REQUIRE(threshold >= 0 && threshold < 255 && cell >= 1 && per_cell >= 1 && n_max >= 1,
             DT_ERR_INVALID_ARGUMENT, "invalid ORB parameters");
  DT_REQUIRE((int64_t)height * width < (1ll << 31), DT_ERR_UNSUPPORTED, "image too large");
  DT_CHECK_CUDA(cudaSetDevice(device));
  dt_orb* o = new (std::nothrow) dt_orb();
  DT_REQUIRE(o != nullptr, DT_ERR_INVALID_ARGUMENT, "out of host memory");
  o->device = device;
  o->h = height;
  o->w = width;
  o->threshold = threshold;
  o->cell = cell;
  o->per_cell = per_cell;
  o->n_max = n_max;
  const int st = orb_init(o, pattern_rot, boundaries);
  if (st != DT_OK) {
    orb_free(o);
    return st;
  }
  *out = o;
  return DT_OK;
}

int dt_orb_destroy(dt_orb* o) {
  if (o) cudaStreamSynchronize(o->stream);
  orb_free(o);
  return DT_OK;
}

// image (h x w uint8, host or device per on_device); outputs host arrays of capacity
// n_max: keypoints (n, 2) int32 (u, v), descriptors (n, 32) uint8, scores, sectors; *n_out.
int dt_orb_detect(dt_orb* o, const uint8_t* image, int on_device, int32_t* keypoints,
                  uint8_t* descriptors, int32_t* scores, int32_t* sectors, int64_t* n_out) {
  DT_REQUIRE(o != nullptr && image != nullptr && n_out != nullptr, DT_ERR_INVALID_ARGUMENT,
             "NULL argument");
  DT_CHECK_CUDA(cudaSetDevice(o->device));
  cudaStream_t s = o->stream;
  const int h = o->h, w = o->w;
  const size_t npix = (size_t)h * w;
  const uint8_t* img = image;
  if (!on_device) {
    DT_CHECK_CUDA(cudaMemcpyAsync(o->img, image, npix, cudaMemcpyHostToDevice, s));
    img = o->img;
  }
  const dim3 blk(32, 8), grd((unsigned)((w + 31) / 32), (unsigned)((h + 7) / 8));
  DT_CHECK_CUDA(cudaMemsetAsync(o->counts, 0, 2 * sizeof(unsigned), s));
  // every stage runs over the fixed capacity with all-ones padding keys (sorted last), so
  // the whole detection is stream-ordered: one host sync, at the end, for the count
  DT_CHECK_CUDA(cudaMemsetAsync(o->keys, 0xff, sizeof(unsigned long long) * o->cap, s));
  DT_CHECK_CUDA(cudaMemsetAsync(o->sel, 0xff, sizeof(unsigned long long) * o->cap, s));
  k_fast_score<<<grd, blk, 0, s>>>(img, h, w, o->score);
  DT_CHECK_LAUNCH();
  k_box5<<<grd, blk, 0, s>>>(img, h, w, o->box);
  DT_CHECK_LAUNCH();
  const int ncx = (w + o->cell - 1) / o->cell;
  const int ncells = ncx * ((h + o->cell - 1) / o->cell);
  int ib = 1, cb = 1;
  while ((1ll << ib) < (long long)npix) ++ib;
  while ((1 << cb) < ncells) ++cb;
  k_nms_collect<<<grd, blk, 0, s>>>(o->score, h, w, o->threshold, o->cell, ncx, ib, o->keys,
                                    o->counts, o->cap);
  DT_CHECK_LAUNCH();
  size_t tb = o->tmp_bytes;
  DT_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(o->tmp, tb, o->keys, o->keys2, o->cap, 0,
                                               ib + 8 + cb, s));
  k_cell_rank<<<(o->cap + 255) / 256, 256, 0, s>>>(o->keys2, o->cap, o->per_cell, ib, o->sel,
                                                   o->counts + 1);
  DT_CHECK_LAUNCH();
  tb = o->tmp_bytes;
  DT_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(o->tmp, tb, o->sel, o->sel2, o->cap, 0, ib + 8, s));
  k_describe<<<(o->n_max + 7) / 8, 256, 0, s>>>(img, o->box, w, o->sel2, o->counts + 1, o->n_max, ib,
                                                o->disc, o->n_disc, o->bnd, o->rot, o->o_kp,
                                                o->o_desc, o->o_score, o->o_bin);
  DT_CHECK_LAUNCH();
  unsigned cnt[2] = {0, 0};
  DT_CHECK_CUDA(cudaMemcpyAsync(cnt, o->counts, sizeof(cnt), cudaMemcpyDeviceToHost, s));
  DT_CHECK_CUDA(cudaStreamSynchronize(s));
  const int n = (int)std::min<unsigned>(cnt[1], (unsigned)o->n_max);
  if (n > 0) {
    if (keypoints)
      DT_CHECK_CUDA(cudaMemcpyAsync(keypoints, o->o_kp, sizeof(int32_t) * 2 * n, cudaMemcpyDeviceToHost, s));
    if (descriptors)
      DT_CHECK_CUDA(cudaMemcpyAsync(descriptors, o->o_desc, 32 * (size_t)n, cudaMemcpyDeviceToHost, s));
    if (scores)
      DT_CHECK_CUDA(cudaMemcpyAsync(scores, o->o_score, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    if (sectors)
      DT_CHECK_CUDA(cudaMemcpyAsync(sectors, o->o_bin, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  }
  DT_CHECK_CUDA(cudaStreamSynchronize(s));
  o->n_last = n;
  *n_out = n;
  return DT_OK;
}

// device-resident results of the last dt_orb_detect (valid until the next call): feed
// them to dt_track_frame with on_device = 1, no host round trip
int dt_orb_last(dt_orb* o, const int32_t** keypoints, const uint8_t** descriptors, int64_t* n) {
  DT_REQUIRE(o != nullptr, DT_ERR_INVALID_ARGUMENT, "NULL argument");
  if (keypoints) *keypoints = o->o_kp;
  if (descriptors) *descriptors = o->o_desc;
  if (n) *n = o->n_last;
  return DT_OK;
}

}  // extern "C"
