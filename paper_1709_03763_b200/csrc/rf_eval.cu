// rf_eval.cu -- the evaluation metrics' exact nearest-neighbour grid index on
// the device (reference /root/reference/pkg/src/refusion/
// evaluation.py:100-229, GridIndex).
//
// Build (:117-138): cells = floor(p / cell_size) as int64, packed like
// _pack_cells (21 bits per axis, bias 2^20, int64 wrap-around), points
// stably sorted by key (cub radix sort of (key, index) pairs), one group
// per distinct key.  Query (:140-214): per query point the rings of cells
// at Chebyshev distance k = k_near, k_near + 1, ... are scanned (binary
// search of each ring cell among the group keys) until the best squared
// distance is <= (k * cell_size)^2 or the rings have left the occupied box;
// queries far outside the box (k_near > 8) or not settled within 3 rings
// take the exact linear scan.  Squared distances group as (dx*dx + dy*dy) +
// dz*dz, IEEE f64 without contraction, as both the reference's ring scan
// and its nn_min_d2 do, so every result is the exact minimum over all
// indexed points -- bit-identical to the reference -- and the returned
// distance is its IEEE square root.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cmath>
#include <climits>
#include <cstdint>

#include "refusion_b200.h"

namespace {

constexpr long long kPackBias = 1LL << 20;
constexpr int kFarRingCutoff = 8;     // evaluation.py:36
constexpr int kExpandRingCutoff = 3;  // evaluation.py:41

__device__ __forceinline__ long long pack_cell(long long x, long long y, long long z) {
  // ((x + B) << 42) | ((y + B) << 21) | (z + B) in int64 arithmetic (wraps)
  const unsigned long long ux = static_cast<unsigned long long>(x + kPackBias) << 42;
  const unsigned long long uy = static_cast<unsigned long long>(y + kPackBias) << 21;
  const unsigned long long uz = static_cast<unsigned long long>(z + kPackBias);
  return static_cast<long long>(ux | uy | uz);
}

__device__ __forceinline__ long long cell_of(double p, double cell) {
  return static_cast<long long>(floor(p / cell));  // np.floor(points / cell).astype(int64)
}

__global__ void k_grid_keys(const double* __restrict__ pts, long long n, double cell,
                            long long* __restrict__ keys, long long* __restrict__ idx,
                            long long* __restrict__ lohi) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long cx = cell_of(pts[3 * i], cell), cy = cell_of(pts[3 * i + 1], cell),
                  cz = cell_of(pts[3 * i + 2], cell);
  keys[i] = pack_cell(cx, cy, cz);
  idx[i] = i;
  atomicMin(&lohi[0], cx);
  atomicMin(&lohi[1], cy);
  atomicMin(&lohi[2], cz);
  atomicMax(&lohi[3], cx);
  atomicMax(&lohi[4], cy);
  atomicMax(&lohi[5], cz);
}

__global__ void k_grid_gather(const double* __restrict__ pts, const long long* __restrict__ idx,
                              const long long* __restrict__ skeys, long long n,
                              double* __restrict__ sorted, int* __restrict__ head) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long j = idx[i];
  sorted[3 * i] = pts[3 * j];
  sorted[3 * i + 1] = pts[3 * j + 1];
  sorted[3 * i + 2] = pts[3 * j + 2];
  head[i] = (i == 0 || skeys[i] != skeys[i - 1]) ? 1 : 0;
}

__global__ void k_grid_groups(const long long* __restrict__ skeys, const int* __restrict__ head,
                              const int* __restrict__ gpos, long long n,
                              long long* __restrict__ gkeys, long long* __restrict__ gstart) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (head[i]) {
    gkeys[gpos[i]] = skeys[i];
    gstart[gpos[i]] = i;
  }
  if (i == n - 1) gstart[gpos[i] + head[i]] = n;  // one past the last group
}

struct GridView {
  const double* pts;       // sorted by cell key
  const long long* gkeys;  // distinct keys, ascending
  const long long* gstart; // group g = points [gstart[g], gstart[g+1])
  long long n, groups;
  long long lo[3], hi[3];
  double cell;
};

__device__ __forceinline__ long long find_group(const GridView& g, long long key) {
  long long a = 0, b = g.groups;
  while (a < b) {
    const long long m = (a + b) >> 1;
    if (g.gkeys[m] < key) a = m + 1;
    else b = m;
  }
  return (a < g.groups && g.gkeys[a] == key) ? a : -1;
}

__device__ __forceinline__ double fold(const double* p, long long a, long long b, double qx,
                                       double qy, double qz, double best) {
  for (long long j = a; j < b; ++j) {
    const double dx = p[3 * j] - qx, dy = p[3 * j + 1] - qy, dz = p[3 * j + 2] - qz;
    double d2 = dx * dx + dy * dy;
    d2 = d2 + dz * dz;
    best = d2 < best ? d2 : best;
  }
  return best;
}

__global__ void k_grid_query(GridView g, const double* __restrict__ q, long long m,
                             double* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double qx = q[3 * i], qy = q[3 * i + 1], qz = q[3 * i + 2];
  const long long c[3] = {cell_of(qx, g.cell), cell_of(qy, g.cell), cell_of(qz, g.cell)};
  long long k_near = 0, k_far = 0;
  for (int a = 0; a < 3; ++a) {
    k_near = max(k_near, max(max(g.lo[a] - c[a], c[a] - g.hi[a]), 0LL));
    k_far = max(k_far, max(max(g.hi[a] - c[a], c[a] - g.lo[a]), 0LL));
  }
  double best = CUDART_INF;
  bool brute = k_near > kFarRingCutoff;
  for (long long k = k_near; !brute; ++k) {
    if (k - k_near > kExpandRingCutoff) {
      brute = true;
      break;
    }
    // the cells at Chebyshev distance exactly k from the query's cell
    for (long long dz = -k; dz <= k; ++dz)
      for (long long dy = -k; dy <= k; ++dy) {
        const bool face = (dz == -k || dz == k || dy == -k || dy == k);
        for (long long dx = -k; dx <= k; dx += (face || k == 0) ? 1 : 2 * k) {
          const long long gi = find_group(g, pack_cell(c[0] + dx, c[1] + dy, c[2] + dz));
          if (gi >= 0) best = fold(g.pts, g.gstart[gi], g.gstart[gi + 1], qx, qy, qz, best);
          if (k == 0) break;
        }
      }
    const double t = static_cast<double>(k) * g.cell;
    if (best <= t * t || k >= k_far) break;
  }
  if (brute) best = fold(g.pts, 0, g.n, qx, qy, qz, best);
  out[i] = sqrt(best);
}

}  // namespace

struct rf_grid_index {
  int device = 0;
  double cell = 0.0;
  long long n = 0, groups = 0;
  long long lohi[6] = {0, 0, 0, 0, 0, 0};
  double* pts = nullptr;
  long long* gkeys = nullptr;
  long long* gstart = nullptr;
};

extern "C" {

rf_status rf_grid_index_create(const double* points, int64_t n, double cell_size,
                               rf_grid_index** out, void* stream) {
  if (!out || !points || n <= 0 || !(cell_size > 0.0)) return RF_INVALID_ARG;
  *out = nullptr;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* g = new rf_grid_index;
  cudaGetDevice(&g->device);
  g->cell = cell_size;
  g->n = n;
  long long *keys = nullptr, *idx = nullptr, *skeys = nullptr, *sidx = nullptr, *lohi = nullptr;
  int *head = nullptr, *gpos = nullptr;
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys, skeys, idx, sidx,
                                  static_cast<int>(n), 0, 64, s);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, head, gpos, static_cast<int>(n), s);
  void* tmp = nullptr;
  bool ok = n < (1LL << 31) &&
            cudaMallocAsync(&keys, 8 * n, s) == cudaSuccess &&
            cudaMallocAsync(&idx, 8 * n, s) == cudaSuccess &&
            cudaMallocAsync(&skeys, 8 * n, s) == cudaSuccess &&
            cudaMallocAsync(&sidx, 8 * n, s) == cudaSuccess &&
            cudaMallocAsync(&lohi, 8 * 6, s) == cudaSuccess &&
            cudaMallocAsync(&head, 4 * n, s) == cudaSuccess &&
            cudaMallocAsync(&gpos, 4 * n, s) == cudaSuccess &&
            cudaMallocAsync(&tmp, std::max(sort_bytes, scan_bytes), s) == cudaSuccess &&
            cudaMalloc(&g->pts, 24 * n) == cudaSuccess;
  if (ok) {
    const long long init[6] = {LLONG_MAX, LLONG_MAX, LLONG_MAX, LLONG_MIN, LLONG_MIN, LLONG_MIN};
    cudaMemcpyAsync(lohi, init, sizeof(init), cudaMemcpyHostToDevice, s);
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    k_grid_keys<<<blocks, 256, 0, s>>>(points, n, cell_size, keys, idx, lohi);
    // stable sort by the signed key (np.argsort(keys, kind="stable"))
    cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, keys, skeys, idx, sidx,
                                    static_cast<int>(n), 0, 64, s);
    k_grid_gather<<<blocks, 256, 0, s>>>(points, sidx, skeys, n, g->pts, head);
    cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, head, gpos, static_cast<int>(n), s);
    int last_pos = 0, last_head = 0;
    cudaMemcpyAsync(&last_pos, gpos + n - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&last_head, head + n - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(g->lohi, lohi, sizeof(g->lohi), cudaMemcpyDeviceToHost, s);
    ok = cudaStreamSynchronize(s) == cudaSuccess;
    g->groups = static_cast<long long>(last_pos) + last_head;
    ok = ok && cudaMalloc(&g->gkeys, 8 * g->groups) == cudaSuccess &&
         cudaMalloc(&g->gstart, 8 * (g->groups + 1)) == cudaSuccess;
    if (ok) {
      k_grid_groups<<<blocks, 256, 0, s>>>(skeys, head, gpos, n, g->gkeys, g->gstart);
      ok = cudaStreamSynchronize(s) == cudaSuccess;
    }
  }
  void* bufs[] = {keys, idx, skeys, sidx, lohi, head, gpos, tmp};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, s);
  if (!ok || cudaGetLastError() != cudaSuccess) {
    cudaStreamSynchronize(s);
    if (g->pts) cudaFree(g->pts);
    if (g->gkeys) cudaFree(g->gkeys);
    if (g->gstart) cudaFree(g->gstart);
    delete g;
    return RF_CUDA;
  }
  *out = g;
  return RF_OK;
}

rf_status rf_grid_index_query(rf_grid_index* g, const double* queries, int64_t m, double* out,
                              void* stream) {
  if (!g || m < 0 || (m > 0 && (!queries || !out))) return RF_INVALID_ARG;
  if (m == 0) return RF_OK;
  GridView v;
  v.pts = g->pts;
  v.gkeys = g->gkeys;
  v.gstart = g->gstart;
  v.n = g->n;
  v.groups = g->groups;
  for (int a = 0; a < 3; ++a) {
    v.lo[a] = g->lohi[a];
    v.hi[a] = g->lohi[3 + a];
  }
  v.cell = g->cell;
  k_grid_query<<<static_cast<unsigned>((m + 127) / 128), 128, 0,
                 static_cast<cudaStream_t>(stream)>>>(v, queries, m, out);
  return cudaGetLastError() == cudaSuccess ? RF_OK : RF_CUDA;
}

rf_status rf_grid_index_destroy(rf_grid_index* g) {
  if (!g) return RF_OK;
  cudaDeviceSynchronize();
  cudaFree(g->pts);
  cudaFree(g->gkeys);
  cudaFree(g->gstart);
  delete g;
  return RF_OK;
}

}  // extern "C"
