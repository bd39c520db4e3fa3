// K2-K5 binning — replaces splatlab rasterizer.bin_and_sort (rasterizer.py:69-124).
//
// The reference duplicates every splat into every tile of its radius box,
// packs (tile << 32 | float32-depth bits) keys and runs ONE stable argsort
// over K instances (45 significant bits at 1080p = 6 radix passes over K).
// Here the same lexicographic order (tile, float32 depth, splat index) is
// produced depth-first, which moves most of the sorting from K to N:
//   1. depth sort: stable radix sort of (depth bits, gaussian id) over N
//      (ties keep index order, exactly like the reference's stable sort);
//   2. per-Gaussian instance counts gathered in depth order, exclusive scan
//      -> instance offsets and K (one D2H read);
//   3. emission: each Gaussian writes (tile id, gaussian id) for every tile
//      of its rectangle, in depth-sorted Gaussian order;
//   4. stable radix sort of the instances on the tile id only
//      (ceil(log2 T) bits = 2 passes at 1080p and 4K);
//   5. tile ranges from neighbouring tile ids (rasterizer.py:118-123).
// HBM traffic per instance: 8 B written by emission + 2 x 16 B per tile pass,
// against 6 x 24 B for a 64-bit key sort.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr uint32_t kCulledKey = 0xFFFFFFFFu;

__global__ void depth_keys_kernel(const float* __restrict__ depth, const int32_t* __restrict__ tiles,
                                  uint32_t* __restrict__ keys, uint32_t* __restrict__ ids, int64_t n) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n) return;
  // positive float32 bit patterns order like the floats (rasterizer.py:55-62)
  keys[g] = tiles[g] > 0 ? __float_as_uint(depth[g]) : kCulledKey;
  ids[g] = uint32_t(g);
}

__global__ void gather_counts_kernel(const uint32_t* __restrict__ order, const int32_t* __restrict__ tiles,
                                     uint64_t* __restrict__ counts, int64_t n) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  counts[r] = uint64_t(tiles[order[r]]);
}

__global__ void total_kernel(const uint64_t* __restrict__ offsets, const uint64_t* __restrict__ counts, int64_t n,
                             const int32_t* __restrict__ status, uint64_t* __restrict__ out) {
  out[0] = offsets[n - 1] + counts[n - 1];
  out[1] = uint64_t(status[0]);
}

// One thread per depth-ranked Gaussian; instances of one Gaussian are emitted
// in row-major tile order (rasterizer.py:105-111).
__global__ void emit_instances_kernel(const uint32_t* __restrict__ order, const uint64_t* __restrict__ offsets,
                                      const uint64_t* __restrict__ counts, const int4* __restrict__ rect,
                                      int tiles_x, uint32_t* __restrict__ tile_keys, uint32_t* __restrict__ ids,
                                      int64_t n) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint64_t cnt = counts[r];
  if (cnt == 0) return;
  const uint32_t g = order[r];
  const int4 rc = rect[g];
  uint64_t o = offsets[r];
  for (int ty = rc.y; ty <= rc.w; ++ty) {
    const uint32_t row = uint32_t(ty) * uint32_t(tiles_x);
    for (int tx = rc.x; tx <= rc.z; ++tx) {
      tile_keys[o] = row + uint32_t(tx);
      ids[o] = g;
      ++o;
    }
  }
}

__global__ void tile_ranges_kernel(const uint32_t* __restrict__ tile_keys, int64_t k, int2* __restrict__ ranges) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const uint32_t t = tile_keys[i];
  if (i == 0 || tile_keys[i - 1] != t) ranges[t].x = int(i);
  if (i == k - 1 || tile_keys[i + 1] != t) ranges[t].y = int(i + 1);
}

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t depth_keys_in, depth_keys_out, ids_in, ids_out, counts, offsets, total, tile_keys_in, tile_keys_out,
      inst_ids_in, cub_temp, bytes;
};

int bits_for(int64_t tiles) {
  int b = 1;
  while ((int64_t(1) << b) < tiles) ++b;
  return b;
}

int make_layout(int64_t n, int64_t tiles, int64_t kcap, Layout* L) {
  size_t temp_depth = 0, temp_scan = 0, temp_tiles = 0;
  const int nn = int(n > 0 ? n : 1);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, temp_depth, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, nn, 0, 32);
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cub::DeviceScan::ExclusiveSum(nullptr, temp_scan, (const uint64_t*)nullptr, (uint64_t*)nullptr, nn);
  if (e != cudaSuccess) return record_cuda_error(e);
  const int kk = int(kcap > 0 ? kcap : 1);
  e = cub::DeviceRadixSort::SortPairs(nullptr, temp_tiles, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                      (const uint32_t*)nullptr, (uint32_t*)nullptr, kk, 0, bits_for(tiles));
  if (e != cudaSuccess) return record_cuda_error(e);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes);
    return o;
  };
  const size_t un = size_t(nn), uk = size_t(kk);
  L->depth_keys_in = take(4 * un);
  L->depth_keys_out = take(4 * un);
  L->ids_in = take(4 * un);
  L->ids_out = take(4 * un);
  L->counts = take(8 * un);
  L->offsets = take(8 * un);
  L->total = take(16);
  L->tile_keys_in = take(4 * uk);
  L->tile_keys_out = take(4 * uk);
  L->inst_ids_in = take(4 * uk);
  size_t temp = temp_depth;
  if (temp_scan > temp) temp = temp_scan;
  if (temp_tiles > temp) temp = temp_tiles;
  L->cub_temp = take(temp);
  L->bytes = off;
  return GS_OK;
}

}  // namespace
}  // namespace gs

extern "C" int gs_bin_workspace_size(int64_t n, int32_t width, int32_t height, int64_t k_capacity, size_t* bytes) {
  if (!bytes || n < 0 || width <= 0 || height <= 0 || k_capacity < 0) return GS_ERR_INVALID_ARG;
  const int64_t tiles = int64_t((width + gs::kTile - 1) / gs::kTile) * int64_t((height + gs::kTile - 1) / gs::kTile);
  if (tiles > gs::kMaxTiles) return GS_ERR_RESOURCE_LIMIT;
  gs::Layout L;
  int st = gs::make_layout(n, tiles, k_capacity, &L);
  if (st != GS_OK) return st;
  *bytes = L.bytes;
  return GS_OK;
}

extern "C" int gs_bin_and_sort(const gs_splats_t* splats, int32_t width, int32_t height, void* workspace,
                               size_t workspace_bytes, int64_t k_capacity, uint32_t* sorted_ids, int32_t* ranges,
                               int64_t* k_out, void* stream) {
  using namespace gs;
  if (!splats || !k_out || width <= 0 || height <= 0 || k_capacity < 0) return GS_ERR_INVALID_ARG;
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * int64_t(tiles_y);
  if (tiles > kMaxTiles) return GS_ERR_RESOURCE_LIMIT;  // rasterizer.py:76-79
  if (tiles > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  const int64_t n = splats->n;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  *k_out = 0;
  cudaError_t e;
  if (ranges) {
    e = cudaMemsetAsync(ranges, 0, size_t(tiles) * 2 * sizeof(int32_t), s);
    if (e != cudaSuccess) return record_cuda_error(e);
  }
  if (n == 0) return GS_OK;
  if (n > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  Layout L;
  int st = make_layout(n, tiles, k_capacity, &L);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(workspace);
  auto* dk_in = reinterpret_cast<uint32_t*>(ws + L.depth_keys_in);
  auto* dk_out = reinterpret_cast<uint32_t*>(ws + L.depth_keys_out);
  auto* id_in = reinterpret_cast<uint32_t*>(ws + L.ids_in);
  auto* id_out = reinterpret_cast<uint32_t*>(ws + L.ids_out);
  auto* counts = reinterpret_cast<uint64_t*>(ws + L.counts);
  auto* offsets = reinterpret_cast<uint64_t*>(ws + L.offsets);
  auto* total = reinterpret_cast<uint64_t*>(ws + L.total);
  auto* tk_in = reinterpret_cast<uint32_t*>(ws + L.tile_keys_in);
  auto* tk_out = reinterpret_cast<uint32_t*>(ws + L.tile_keys_out);
  auto* iid_in = reinterpret_cast<uint32_t*>(ws + L.inst_ids_in);
  void* temp = ws + L.cub_temp;
  size_t temp_bytes = workspace_bytes - L.cub_temp;

  const int block = 256;
  const unsigned gn = unsigned((n + block - 1) / block);
  depth_keys_kernel<<<gn, block, 0, s>>>(splats->depth, splats->tiles_touched, dk_in, id_in, n);
  if ((st = check_launch()) != GS_OK) return st;
  e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, dk_in, dk_out, id_in, id_out, int(n), 0, 32, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  gather_counts_kernel<<<gn, block, 0, s>>>(id_out, splats->tiles_touched, counts, n);
  if ((st = check_launch()) != GS_OK) return st;
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offsets, int(n), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  total_kernel<<<1, 1, 0, s>>>(offsets, counts, n, splats->status, total);
  if ((st = check_launch()) != GS_OK) return st;
  uint64_t host_total[2] = {0, 0};
  e = cudaMemcpyAsync(host_total, total, sizeof(host_total), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return record_cuda_error(e);
  if (host_total[1] & 1u) return GS_ERR_ZERO_QUATERNION;
  const uint64_t K = host_total[0];
  *k_out = int64_t(K);
  if (K > uint64_t(kMaxInstances)) return GS_ERR_RESOURCE_LIMIT;  // rasterizer.py:99-101
  if (K > uint64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  if (int64_t(K) > k_capacity) return GS_ERR_CAPACITY;
  if (K == 0) return GS_OK;
  if (!sorted_ids || !ranges) return GS_ERR_INVALID_ARG;

  emit_instances_kernel<<<gn, block, 0, s>>>(id_out, offsets, counts, reinterpret_cast<const int4*>(splats->rect),
                                             tiles_x, tk_in, iid_in, n);
  if ((st = check_launch()) != GS_OK) return st;
  e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, tk_in, tk_out, iid_in, sorted_ids, int(K), 0,
                                      bits_for(tiles), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  const unsigned gk = unsigned((K + block - 1) / block);
  tile_ranges_kernel<<<gk, block, 0, s>>>(tk_out, int64_t(K), reinterpret_cast<int2*>(ranges));
  return check_launch();
}
