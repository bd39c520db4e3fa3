// Exact k-nearest-neighbour mean distance on the device — replaces splatlab
// scene_io.mean_knn_distance (scene_io.py:304-311, scipy cKDTree query of
// k + 1 neighbours with the self match dropped), the scale initialisation
// of init_from_sfm / init_random (scene_io.py:314-366).
//
// Uniform grid over the bounding box (about two points per occupied cell):
//   1. bounding box (one block-reduce kernel);
//   2. cell id per point, CUB radix sort of (cell, point) pairs;
//   3. cell ranges from neighbouring cell ids (dense [start, end) per cell);
//   4. one thread per query point searches Chebyshev shells of cells around
//      its own cell, keeping the k best squared distances (float64, like the
//      reference), and stops once the k-th best distance is <= r h after
//      shell r (every point in shell r + 1 is at least r h away).  Exact.
#include <cub/device/device_radix_sort.cuh>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kMaxK = 16;

struct Grid {
  double lo[3];
  double h, inv_h;
  int dim[3];
};

__global__ void bbox_kernel(const double* __restrict__ pts, int64_t n, double* __restrict__ box) {
  // box[0..2] = min, box[3..5] = max; one block, strided
  __shared__ double s[6][256];
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = pts[3 * i + c];
      mn[c] = fmin(mn[c], v);
      mx[c] = fmax(mx[c], v);
    }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    s[c][threadIdx.x] = mn[c];
    s[3 + c][threadIdx.x] = mx[c];
  }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        s[c][threadIdx.x] = fmin(s[c][threadIdx.x], s[c][threadIdx.x + w]);
        s[3 + c][threadIdx.x] = fmax(s[3 + c][threadIdx.x], s[3 + c][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) box[threadIdx.x] = s[threadIdx.x][0];
}

__device__ __forceinline__ int cell_coord(double v, double lo, double inv_h, int dim) {
  const int c = int(floor((v - lo) * inv_h));
  return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__global__ void cell_ids_kernel(const double* __restrict__ pts, int64_t n, Grid g, uint32_t* __restrict__ cell,
                                uint32_t* __restrict__ idx) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cx = cell_coord(pts[3 * i + 0], g.lo[0], g.inv_h, g.dim[0]);
  const int cy = cell_coord(pts[3 * i + 1], g.lo[1], g.inv_h, g.dim[1]);
  const int cz = cell_coord(pts[3 * i + 2], g.lo[2], g.inv_h, g.dim[2]);
  cell[i] = uint32_t((cz * g.dim[1] + cy) * g.dim[0] + cx);
  idx[i] = uint32_t(i);
}

__global__ void cell_ranges_kernel(const uint32_t* __restrict__ cell, int64_t n, int2* __restrict__ ranges) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cell[i];
  if (i == 0 || cell[i - 1] != c) ranges[c].x = int(i);
  if (i == n - 1 || cell[i + 1] != c) ranges[c].y = int(i + 1);
}

template <int K>
__global__ void knn_kernel(const double* __restrict__ pts, const double* __restrict__ sorted_pts,
                           const uint32_t* __restrict__ sorted_idx, const int2* __restrict__ ranges, int64_t n, Grid g,
                           float* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double px = pts[3 * i + 0], py = pts[3 * i + 1], pz = pts[3 * i + 2];
  const int cx = cell_coord(px, g.lo[0], g.inv_h, g.dim[0]);
  const int cy = cell_coord(py, g.lo[1], g.inv_h, g.dim[1]);
  const int cz = cell_coord(pz, g.lo[2], g.inv_h, g.dim[2]);
  double best[K];
#pragma unroll
  for (int k = 0; k < K; ++k) best[k] = 1e300;   // ascending squared distances
  const int rmax = max(g.dim[0], max(g.dim[1], g.dim[2]));
  for (int r = 0; r <= rmax; ++r) {
    for (int dz = -r; dz <= r; ++dz) {
      const int z = cz + dz;
      if (z < 0 || z >= g.dim[2]) continue;
      for (int dy = -r; dy <= r; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= g.dim[1]) continue;
        const bool face = (dz == -r || dz == r || dy == -r || dy == r);
        // interior rows of the shell only need their two end cells
        for (int dx = -r; dx <= r; dx += (face || r == 0) ? 1 : 2 * r) {
          const int x = cx + dx;
          if (x < 0 || x >= g.dim[0]) continue;
          const int2 rg = ranges[(z * g.dim[1] + y) * g.dim[0] + x];
          for (int j = rg.x; j < rg.y; ++j) {
            if (sorted_idx[j] == uint32_t(i)) continue;   // the self match (scene_io.py:310)
            const double ex = sorted_pts[3 * j + 0] - px, ey = sorted_pts[3 * j + 1] - py,
                         ez = sorted_pts[3 * j + 2] - pz;
            double d2 = ex * ex + ey * ey + ez * ez;
            if (d2 < best[K - 1]) {   // insertion into the ascending list
#pragma unroll
              for (int k = K - 1; k >= 0; --k) {
                const double prev = k > 0 ? best[k - 1] : -1.0;
                if (k > 0 && prev > d2) {
                  best[k] = prev;
                } else {
                  best[k] = d2;
                  break;
                }
              }
            }
          }
        }
      }
    }
    // every point of shell r + 1 is at least r h away from this point
    const double reach = double(r) * g.h;
    if (best[K - 1] <= reach * reach) break;
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += sqrt(best[k]);
  out[i] = float(s / double(K));
}

__global__ void gather_points_kernel(const double* __restrict__ pts, const uint32_t* __restrict__ idx, int64_t n,
                                     double* __restrict__ sorted_pts) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t i = idx[j];
#pragma unroll
  for (int c = 0; c < 3; ++c) sorted_pts[3 * j + c] = pts[3 * size_t(i) + c];
}

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace gs

// Workspace: points as float64 (the caller converts), cell ids / indices
// (double-buffered), the sorted points, the dense cell ranges and CUB's
// scratch.  max_cells bounds the grid (the caller passes ~2 n).
extern "C" int gs_knn_workspace_size(int64_t n, int64_t max_cells, size_t* bytes) {
  if (!bytes || n < 0 || max_cells < 1 || max_cells > int64_t(INT32_MAX)) return GS_ERR_INVALID_ARG;
  size_t temp = 0;
  const int nn = int(n > 0 ? n : 1);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, nn, 0, 32);
  if (e != cudaSuccess) return gs::record_cuda_error(e);
  const size_t un = size_t(nn);
  *bytes = gs::align_up(64) + 4 * gs::align_up(4 * un) + gs::align_up(24 * un) +
           gs::align_up(8 * size_t(max_cells)) + gs::align_up(temp);
  return GS_OK;
}

extern "C" int gs_knn_mean_distance(const double* points, int64_t n, int32_t k, int64_t max_cells, void* workspace,
                                    size_t workspace_bytes, float* out, void* stream) {
  using namespace gs;
  if (!points || !out || n < 0 || k < 1 || k > kMaxK || max_cells < 1) return GS_ERR_INVALID_ARG;
  if (n == 0) return GS_OK;
  if (n <= k || n > int64_t(INT32_MAX)) return GS_ERR_INVALID_ARG;   // needs k neighbours besides self
  size_t need = 0;
  int st = gs_knn_workspace_size(n, max_cells, &need);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < need) return GS_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  size_t off = 0;
  auto take = [&](size_t b) {
    char* p = ws + off;
    off += align_up(b);
    return p;
  };
  const size_t un = size_t(n);
  double* box = reinterpret_cast<double*>(take(64));
  uint32_t* cell_in = reinterpret_cast<uint32_t*>(take(4 * un));
  uint32_t* cell_out = reinterpret_cast<uint32_t*>(take(4 * un));
  uint32_t* idx_in = reinterpret_cast<uint32_t*>(take(4 * un));
  uint32_t* idx_out = reinterpret_cast<uint32_t*>(take(4 * un));
  double* sorted_pts = reinterpret_cast<double*>(take(24 * un));
  int2* ranges = reinterpret_cast<int2*>(take(8 * size_t(max_cells)));
  void* temp = take(0);
  size_t temp_bytes = workspace_bytes - off;

  // the grid needs the bounding box on the host (one small read)
  bbox_kernel<<<1, 256, 0, s>>>(points, n, box);
  if ((st = check_launch()) != GS_OK) return st;
  double hb[6];
  cudaError_t e = cudaMemcpyAsync(hb, box, sizeof(hb), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return record_cuda_error(e);
  Grid g;
  double ext[3], vol = 1.0;
  for (int c = 0; c < 3; ++c) {
    g.lo[c] = hb[c];
    ext[c] = fmax(hb[3 + c] - hb[c], 1e-12);
    vol *= ext[c];
  }
  // cell edge for ~max_cells / 2 cells over the box, at least one cell per axis
  double h = cbrt(vol / (0.5 * double(max_cells)));
  for (;;) {
    int64_t cells = 1;
    for (int c = 0; c < 3; ++c) {
      g.dim[c] = int(fmin(fmax(ceil(ext[c] / h), 1.0), 1e6));
      cells *= g.dim[c];
    }
    if (cells <= max_cells) break;
    h *= 1.1;
  }
  g.h = h;
  g.inv_h = 1.0 / h;
  const int64_t ncells = int64_t(g.dim[0]) * g.dim[1] * g.dim[2];
  const int block = 256;
  const unsigned grid = unsigned((n + block - 1) / block);
  cell_ids_kernel<<<grid, block, 0, s>>>(points, n, g, cell_in, idx_in);
  if ((st = check_launch()) != GS_OK) return st;
  e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, cell_in, cell_out, idx_in, idx_out, int(n), 0, 32, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  if ((e = cudaMemsetAsync(ranges, 0, 8 * size_t(ncells), s)) != cudaSuccess) return record_cuda_error(e);
  cell_ranges_kernel<<<grid, block, 0, s>>>(cell_out, n, ranges);
  if ((st = check_launch()) != GS_OK) return st;
  gather_points_kernel<<<grid, block, 0, s>>>(points, idx_out, n, sorted_pts);
  if ((st = check_launch()) != GS_OK) return st;
  switch (k) {
#define GS_KNN_CASE(KK)                                                                                    \
  case KK:                                                                                                 \
    knn_kernel<KK><<<unsigned((n + 127) / 128), 128, 0, s>>>(points, sorted_pts, idx_out, ranges, n, g, out); \
    break;
    GS_KNN_CASE(1) GS_KNN_CASE(2) GS_KNN_CASE(3) GS_KNN_CASE(4) GS_KNN_CASE(5) GS_KNN_CASE(6) GS_KNN_CASE(7)
    GS_KNN_CASE(8) GS_KNN_CASE(9) GS_KNN_CASE(10) GS_KNN_CASE(11) GS_KNN_CASE(12) GS_KNN_CASE(13)
    GS_KNN_CASE(14) GS_KNN_CASE(15) GS_KNN_CASE(16)
#undef GS_KNN_CASE
    default:
      return GS_ERR_INVALID_ARG;
  }
  return check_launch();
}
