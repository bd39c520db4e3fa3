// K2-K5 binning — replaces splatlab rasterizer.bin_and_sort (rasterizer.py:69-124).
//
// The reference duplicates every splat into every tile of its radius box,
// packs (tile << 32 | float32-depth bits) keys and runs ONE stable argsort
// over K instances (45 significant bits at 1080p = 6 radix passes over K).
// Here the same lexicographic order (tile, float32 depth, splat index) is
// produced depth-first, which moves most of the sorting from K to N:
//   1. depth order: stable radix sort of (depth bits, gaussian id) over N
//      (ties keep index order, exactly like the reference's stable sort);
//   2. per-Gaussian instance counts read in depth order by the exclusive scan
//      -> instance offsets and K, kept on the device (no host round trip);
//   3. emission: warps write (tile id, gaussian id) for 32 depth-ranked
//      Gaussians at a time into their contiguous output range, coalesced;
//      slots [K, capacity) are padded with the largest tile key;
//   4. stable radix sort of the capacity-sized instance list on the tile id
//      only (16-bit keys and ceil(log2 T) bits = 2 passes at 1080p and 4K);
//   5. tile ranges from neighbouring tile ids over the first K sorted keys
//      (rasterizer.py:118-123).
// Steps 2-5 can run per band of tile rows (gs_bin_rows_async) on the shared
// depth order (gs_depth_order): each band is an independent instance list,
// so the latency-bound sort of one band overlaps the compute-bound blend of
// another on a second stream.  The per-tile lists are identical to the
// full-frame binning's.
// HBM traffic per instance: 6 B written by emission + 2 x 12 B per tile
// pass + 2 B for ranges, against 6 x 24 B for a 64-bit key sort.  Every
// kernel after the scan reads K from device memory, so the whole binning is
// enqueued without synchronising (CUDA-graph capturable); the grids and the
// sort length are the caller's instance capacity and K > capacity is
// reported through a device flag (gs_bin_and_sort_async) or, in the
// synchronous entry point, as GS_ERR_CAPACITY after one stream sync.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr uint32_t kCulledKey = 0xFFFFFFFFu;

// kinfo[] (device, int64): [0] K, [1] flags, [2] K clamped to the capacity
constexpr int64_t kFlagZeroQuat = 1, kFlagCapacity = 2, kFlagLimit = 4;


__global__ void depth_keys_kernel(const float* __restrict__ depth, const int32_t* __restrict__ tiles,
                                  uint32_t* __restrict__ keys, uint32_t* __restrict__ ids, int64_t n) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n) return;
  // positive float32 bit patterns order like the floats (rasterizer.py:55-62)
  keys[g] = tiles[g] > 0 ? __float_as_uint(depth[g]) : kCulledKey;
  ids[g] = uint32_t(g);
}

// Tile rows [y0, y1) of a band; full = the whole frame (counts are then the
// preprocess' tiles_touched, and no rectangle is read).
struct RowBand {
  int y0, y1;
  bool full;
};

// instances of Gaussian g inside the band: its tile rectangle clipped to the rows
__device__ __forceinline__ uint32_t band_count(uint32_t g, const int32_t* __restrict__ tiles,
                                               const int4* __restrict__ rect, RowBand b) {
  const int32_t t = tiles[g];
  if (t <= 0) return 0u;   // culled or off-screen (its rect may be stale)
  if (b.full) return uint32_t(t);
  const int4 rc = rect[g];
  const int r0 = max(rc.y, b.y0), r1 = min(rc.w, b.y1 - 1);
  return r1 >= r0 ? uint32_t(rc.z - rc.x + 1) * uint32_t(r1 - r0 + 1) : 0u;
}

// per-Gaussian instance count in depth order, read on the fly by the scan
struct DepthCount {
  const uint32_t* order;
  const int32_t* tiles;
  const int4* rect;
  RowBand band;
  __host__ __device__ __forceinline__ uint64_t operator()(int64_t r) const {
#ifdef __CUDA_ARCH__
    return uint64_t(band_count(order[r], tiles, rect, band));
#else
    return 0;
#endif
  }
};

__global__ void total_kernel(const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ order,
                             const int32_t* __restrict__ tiles, const int4* __restrict__ rect, RowBand band,
                             int64_t n, int64_t capacity, const int32_t* __restrict__ status,
                             int64_t* __restrict__ kinfo) {
  const uint64_t K = offsets[n - 1] + uint64_t(band_count(order[n - 1], tiles, rect, band));
  int64_t flags = (status[0] & 1) ? kFlagZeroQuat : 0;
  if (K > uint64_t(kMaxInstances) || K > uint64_t(INT32_MAX)) flags |= kFlagLimit;  // rasterizer.py:99-101
  if (K > uint64_t(capacity)) flags |= kFlagCapacity;
  kinfo[0] = int64_t(K);
  kinfo[1] = flags;
  kinfo[2] = int64_t(K < uint64_t(capacity) ? K : uint64_t(capacity));
}

// Warp-cooperative emission.  A warp owns 32 consecutive depth-ranked
// Gaussians whose instances occupy one contiguous output range (32-bit
// positions: the capacity is < 2^31, and positions past it are dropped).
// The warp sweeps that range 32 positions at a time: each lane finds the
// Gaussian owning its position (the number of lanes whose range ends at or
// before it: a monotone predicate, so Gaussians without instances in the
// band are skipped correctly) and derives the tile from the local index,
// row-major over the (band-clipped) rectangle (rasterizer.py:105-111).
template <typename KeyT>
__global__ void __launch_bounds__(256)
emit_instances_kernel(const uint32_t* __restrict__ order, const uint64_t* __restrict__ offsets,
                      const int32_t* __restrict__ tiles_touched, const int4* __restrict__ rect, RowBand band,
                      int tiles_x, KeyT* __restrict__ tile_keys, uint32_t* __restrict__ ids, int64_t n,
                      int64_t capacity) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  uint32_t off = 0u, end = 0u, g = 0u;
  int4 rc = make_int4(0, 0, 0, 0);
  bool in = r < n;
  if (in) {
    g = order[r];
    const uint32_t cnt = band_count(g, tiles_touched, rect, band);
    off = uint32_t(offsets[r]);
    end = off + cnt;
    if (cnt) {
      rc = rect[g];
      rc.y = max(rc.y, band.y0);   // first row of the rectangle inside the band
    }
  }
  const uint32_t base = __shfl_sync(0xffffffffu, off, 0);
  const uint32_t warp_end = __reduce_max_sync(0xffffffffu, end);
  if (!in) end = warp_end;   // keep the lane ends non-decreasing
  const int w = rc.z - rc.x + 1;
  for (uint32_t ob = base; ob < warp_end; ob += 32) {
    const uint32_t o = ob + lane;
    int owner = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      const uint32_t e = __shfl_sync(0xffffffffu, end, owner + step - 1);
      if (e <= o) owner += step;
    }
    owner = min(owner, 31);
    const uint32_t k = o - __shfl_sync(0xffffffffu, off, owner);
    const int ow = __shfl_sync(0xffffffffu, w, owner);
    const int ox = __shfl_sync(0xffffffffu, rc.x, owner);
    const int oy = __shfl_sync(0xffffffffu, rc.y, owner);
    const uint32_t og = __shfl_sync(0xffffffffu, g, owner);
    if (o < warp_end && int64_t(o) < capacity) {
      const uint32_t row = k / uint32_t(ow);
      const uint32_t col = k - row * uint32_t(ow);
      tile_keys[o] = KeyT((uint32_t(oy) + row) * uint32_t(tiles_x) + uint32_t(ox) + col);
      ids[o] = og;
    }
  }
}

// Instance slots [K, capacity) get the largest key (all tile bits set) so the
// capacity-sized sort leaves them behind every real instance (a stable sort
// keeps them after the real instances of the last tile too).
template <typename KeyT>
__global__ void pad_instances_kernel(const int64_t* __restrict__ kinfo, int64_t capacity, KeyT* __restrict__ keys,
                                     uint32_t* __restrict__ ids) {
  for (int64_t i = kinfo[2] + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < capacity;
       i += int64_t(gridDim.x) * blockDim.x) {
    keys[i] = KeyT(~KeyT(0));
    ids[i] = 0u;
  }
}

// Tile ranges: each thread inspects 16 bytes of sorted keys plus its two
// neighbours and records [start, end) where the tile id changes.
template <typename KeyT>
__global__ void tile_ranges_kernel(const KeyT* __restrict__ keys, const int64_t* __restrict__ kinfo,
                                   int2* __restrict__ ranges) {
  constexpr int kPer = 16 / sizeof(KeyT);
  const int64_t k = kinfo[2];
  const int64_t i0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kPer;
  if (i0 >= k || kinfo[1] != 0) return;
  KeyT v[kPer];
  if (i0 + kPer <= k) {
    const uint4 raw = *reinterpret_cast<const uint4*>(keys + i0);
    const KeyT* rv = reinterpret_cast<const KeyT*>(&raw);
#pragma unroll
    for (int j = 0; j < kPer; ++j) v[j] = rv[j];
  } else {
#pragma unroll
    for (int j = 0; j < kPer; ++j) v[j] = (i0 + j < k) ? keys[i0 + j] : KeyT(0);
  }
  KeyT prev = i0 > 0 ? keys[i0 - 1] : KeyT(0);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int64_t i = i0 + j;
    if (i >= k) break;
    if (i == 0 || v[j] != prev) ranges[v[j]].x = int(i);
    const bool last = (i == k - 1) || (j + 1 < kPer ? v[j + 1] != v[j] : keys[i + 1] != v[j]);
    if (last) ranges[v[j]].y = int(i + 1);
    prev = v[j];
  }
}

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

int bits_for(int64_t tiles) {
  int b = 1;
  while ((int64_t(1) << b) < tiles) ++b;
  return b;
}

bool small_keys(int64_t tiles) { return tiles <= 65536; }

// Depth-order workspace: keys / ids double buffers + CUB scratch.
struct DepthLayout {
  size_t keys_in, keys_out, ids_in, cub_temp, bytes;
};
// Band workspace: offsets, kinfo (sync entry point), instance keys / ids + scratch.
struct RowsLayout {
  size_t offsets, kinfo, tile_keys_in, tile_keys_out, inst_ids_in, cub_temp, bytes;
};

template <typename KeyT>
cudaError_t sort_tiles(void* temp, size_t& temp_bytes, const KeyT* kin, KeyT* kout, const uint32_t* vin,
                       uint32_t* vout, int64_t count, int bits, cudaStream_t s) {
  return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kin, kout, vin, vout, int(count), 0, bits, s);
}

template <typename F>
size_t carve(F&& plan) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes);
    return o;
  };
  plan(take);
  return off;
}

int depth_layout(int64_t n, DepthLayout* L) {
  size_t temp = 0;
  const int nn = int(n > 0 ? n : 1);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, nn, 0, 32);
  if (e != cudaSuccess) return record_cuda_error(e);
  const size_t un = size_t(nn);
  L->bytes = carve([&](auto take) {
    L->keys_in = take(4 * un);
    L->keys_out = take(4 * un);
    L->ids_in = take(4 * un);
    L->cub_temp = take(temp);
  });
  return GS_OK;
}

int rows_layout(int64_t n, int64_t tiles, int64_t kcap, RowsLayout* L) {
  size_t temp_scan = 0, temp_tiles = 0;
  const int nn = int(n > 0 ? n : 1);
  cub::TransformInputIterator<uint64_t, DepthCount, cub::CountingInputIterator<int64_t>> in(
      cub::CountingInputIterator<int64_t>(0), DepthCount{nullptr, nullptr, nullptr, RowBand{0, 0, true}});
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, temp_scan, in, (uint64_t*)nullptr, nn);
  if (e != cudaSuccess) return record_cuda_error(e);
  if (kcap > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  const int64_t kk = kcap > 0 ? kcap : 1;
  const size_t key_bytes = small_keys(tiles) ? 2 : 4;
  if (small_keys(tiles))
    e = sort_tiles<uint16_t>(nullptr, temp_tiles, nullptr, nullptr, nullptr, nullptr, kk, bits_for(tiles), nullptr);
  else
    e = sort_tiles<uint32_t>(nullptr, temp_tiles, nullptr, nullptr, nullptr, nullptr, kk, bits_for(tiles), nullptr);
  if (e != cudaSuccess) return record_cuda_error(e);
  const size_t un = size_t(nn), uk = size_t(kk);
  L->bytes = carve([&](auto take) {
    L->offsets = take(8 * un);
    L->kinfo = take(4 * sizeof(int64_t));
    L->tile_keys_in = take(key_bytes * uk + 16);
    L->tile_keys_out = take(key_bytes * uk + 16);
    L->inst_ids_in = take(4 * uk);
    L->cub_temp = take(temp_scan > temp_tiles ? temp_scan : temp_tiles);
  });
  return GS_OK;
}

// The full-frame binning workspace: the depth order (order array + its
// workspace) followed by one band workspace.
struct FullLayout {
  DepthLayout D;
  RowsLayout R;
  size_t order, depth_ws, rows_ws, bytes;
};

int full_layout(int64_t n, int64_t tiles, int64_t kcap, FullLayout* L) {
  int st = depth_layout(n, &L->D);
  if (st != GS_OK) return st;
  if ((st = rows_layout(n, tiles, kcap, &L->R)) != GS_OK) return st;
  const size_t un = size_t(n > 0 ? n : 1);
  L->bytes = carve([&](auto take) {
    L->order = take(4 * un);
    L->depth_ws = take(L->D.bytes);
    L->rows_ws = take(L->R.bytes);
  });
  return GS_OK;
}

// Emission in depth order, padding to the capacity, a stable sort of the
// capacity-sized instance list on the tile bits only (ceil(log2 T): 2 radix
// passes at 1080p and 4K) and the tile ranges — all sized by the host-known
// capacity, with K itself read on the device.
template <typename KeyT>
int tile_sort(const uint32_t* order, const uint64_t* offsets, const int32_t* counts, const int4* rect, RowBand band,
              int tiles_x, int64_t tiles, int64_t n, int64_t cap, const int64_t* kinfo, char* ws,
              const RowsLayout& L, size_t temp_bytes, uint32_t* sorted_ids, int2* ranges, cudaStream_t s) {
  auto* tk_in = reinterpret_cast<KeyT*>(ws + L.tile_keys_in);
  auto* tk_out = reinterpret_cast<KeyT*>(ws + L.tile_keys_out);
  auto* iid_in = reinterpret_cast<uint32_t*>(ws + L.inst_ids_in);
  const int block = 256;
  emit_instances_kernel<KeyT><<<unsigned((n + block - 1) / block), block, 0, s>>>(
      order, offsets, counts, rect, band, tiles_x, tk_in, iid_in, n, cap);
  int st = check_launch();
  if (st != GS_OK) return st;
  pad_instances_kernel<KeyT><<<4 * 148, block, 0, s>>>(kinfo, cap, tk_in, iid_in);
  if ((st = check_launch()) != GS_OK) return st;
  cudaError_t e = sort_tiles<KeyT>(ws + L.cub_temp, temp_bytes, tk_in, tk_out, iid_in, sorted_ids, cap,
                                   bits_for(tiles), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  constexpr int kPer = 16 / sizeof(KeyT);
  const int64_t threads = (cap + kPer - 1) / kPer;
  tile_ranges_kernel<KeyT><<<unsigned((threads + block - 1) / block), block, 0, s>>>(tk_out, kinfo, ranges);
  return check_launch();
}

// Step 1: order[r] = id of the r-th Gaussian by (float32 depth, index);
// culled Gaussians last.
int depth_enqueue(const gs_splats_t* splats, void* workspace, size_t workspace_bytes, uint32_t* order,
                  cudaStream_t s) {
  const int64_t n = splats->n;
  if (n == 0) return GS_OK;
  if (n > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  DepthLayout L;
  int st = depth_layout(n, &L);
  if (st != GS_OK) return st;
  if (!workspace || !order || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(workspace);
  auto* dk_in = reinterpret_cast<uint32_t*>(ws + L.keys_in);
  auto* dk_out = reinterpret_cast<uint32_t*>(ws + L.keys_out);
  auto* id_in = reinterpret_cast<uint32_t*>(ws + L.ids_in);
  size_t temp_bytes = workspace_bytes - L.cub_temp;
  const int block = 256;
  depth_keys_kernel<<<unsigned((n + block - 1) / block), block, 0, s>>>(splats->depth, splats->tiles_touched, dk_in,
                                                                        id_in, n);
  if ((st = check_launch()) != GS_OK) return st;
  cudaError_t e =
      cub::DeviceRadixSort::SortPairs(ws + L.cub_temp, temp_bytes, dk_in, dk_out, id_in, order, int(n), 0, 32, s);
  return e == cudaSuccess ? GS_OK : record_cuda_error(e);
}

// Steps 2-5 for one band of tile rows; K and the flags land in kinfo.
// ranges entries are written only for tiles holding instances (the caller
// zeroes the frame's ranges once).
int rows_enqueue(const gs_splats_t* splats, const uint32_t* order, int32_t width, int32_t height, RowBand band,
                 void* workspace, size_t workspace_bytes, int64_t k_capacity, uint32_t* sorted_ids, int32_t* ranges,
                 int64_t* kinfo, cudaStream_t s) {
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * int64_t(tiles_y);
  const int64_t n = splats->n;
  cudaError_t e;
  if (n == 0) {
    e = cudaMemsetAsync(kinfo, 0, 3 * sizeof(int64_t), s);
    return e == cudaSuccess ? GS_OK : record_cuda_error(e);
  }
  if (n > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  if (!order || (k_capacity > 0 && (!sorted_ids || !ranges))) return GS_ERR_INVALID_ARG;
  if (band.y0 < 0 || band.y1 > tiles_y || band.y0 >= band.y1) return GS_ERR_INVALID_ARG;
  band.full = band.y0 == 0 && band.y1 == tiles_y;
  RowsLayout L;
  int st = rows_layout(n, tiles, k_capacity, &L);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(workspace);
  auto* offsets = reinterpret_cast<uint64_t*>(ws + L.offsets);
  void* temp = ws + L.cub_temp;
  size_t temp_bytes = workspace_bytes - L.cub_temp;
  const int4* rect = reinterpret_cast<const int4*>(splats->rect);
  {
    cub::TransformInputIterator<uint64_t, DepthCount, cub::CountingInputIterator<int64_t>> in(
        cub::CountingInputIterator<int64_t>(0), DepthCount{order, splats->tiles_touched, rect, band});
    e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, offsets, int(n), s);
  }
  if (e != cudaSuccess) return record_cuda_error(e);
  total_kernel<<<1, 1, 0, s>>>(offsets, order, splats->tiles_touched, rect, band, n, k_capacity, splats->status,
                               kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  if (k_capacity == 0) return GS_OK;
  if (small_keys(tiles))
    return tile_sort<uint16_t>(order, offsets, splats->tiles_touched, rect, band, tiles_x, tiles, n, k_capacity,
                               kinfo, ws, L, temp_bytes, sorted_ids, reinterpret_cast<int2*>(ranges), s);
  return tile_sort<uint32_t>(order, offsets, splats->tiles_touched, rect, band, tiles_x, tiles, n, k_capacity, kinfo,
                             ws, L, temp_bytes, sorted_ids, reinterpret_cast<int2*>(ranges), s);
}

// Full frame: zero the ranges, depth order, one band over all tile rows.
int bin_enqueue(const gs_splats_t* splats, int32_t width, int32_t height, void* workspace, size_t workspace_bytes,
                int64_t k_capacity, uint32_t* sorted_ids, int32_t* ranges, int64_t* kinfo, cudaStream_t s) {
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * int64_t(tiles_y);
  const int64_t n = splats->n;
  if (ranges) {
    cudaError_t e = cudaMemsetAsync(ranges, 0, size_t(tiles) * 2 * sizeof(int32_t), s);
    if (e != cudaSuccess) return record_cuda_error(e);
  }
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(kinfo, 0, 3 * sizeof(int64_t), s);
    return e == cudaSuccess ? GS_OK : record_cuda_error(e);
  }
  if (n > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  FullLayout L;
  int st = full_layout(n, tiles, k_capacity, &L);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(workspace);
  auto* order = reinterpret_cast<uint32_t*>(ws + L.order);
  st = depth_enqueue(splats, ws + L.depth_ws, L.D.bytes, order, s);
  if (st != GS_OK) return st;
  return rows_enqueue(splats, order, width, height, RowBand{0, tiles_y, true}, ws + L.rows_ws,
                      workspace_bytes - L.rows_ws, k_capacity, sorted_ids, ranges, kinfo, s);
}

int check_dims(int32_t width, int32_t height) {
  if (width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  const int64_t tiles = int64_t((width + kTile - 1) / kTile) * int64_t((height + kTile - 1) / kTile);
  if (tiles > kMaxTiles) return GS_ERR_RESOURCE_LIMIT;  // rasterizer.py:76-79
  if (tiles > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  return GS_OK;
}

}  // namespace
}  // namespace gs

extern "C" int gs_bin_workspace_size(int64_t n, int32_t width, int32_t height, int64_t k_capacity, size_t* bytes) {
  if (!bytes || n < 0 || k_capacity < 0) return GS_ERR_INVALID_ARG;
  int st = gs::check_dims(width, height);
  if (st != GS_OK) return st;
  const int64_t tiles = int64_t((width + gs::kTile - 1) / gs::kTile) * int64_t((height + gs::kTile - 1) / gs::kTile);
  gs::FullLayout L;
  st = gs::full_layout(n, tiles, k_capacity, &L);
  if (st != GS_OK) return st;
  *bytes = L.bytes;
  return GS_OK;
}

extern "C" int gs_bin_and_sort_async(const gs_splats_t* splats, int32_t width, int32_t height, void* workspace,
                                     size_t workspace_bytes, int64_t k_capacity, uint32_t* sorted_ids,
                                     int32_t* ranges, int64_t* k_info, void* stream) {
  using namespace gs;
  if (!splats || !k_info || k_capacity < 0) return GS_ERR_INVALID_ARG;
  int st = check_dims(width, height);
  if (st != GS_OK) return st;
  return bin_enqueue(splats, width, height, workspace, workspace_bytes, k_capacity, sorted_ids, ranges, k_info,
                     static_cast<cudaStream_t>(stream));
}

extern "C" int gs_depth_order_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return GS_ERR_INVALID_ARG;
  gs::DepthLayout L;
  int st = gs::depth_layout(n, &L);
  if (st != GS_OK) return st;
  *bytes = L.bytes;
  return GS_OK;
}

extern "C" int gs_depth_order(const gs_splats_t* splats, void* workspace, size_t workspace_bytes, uint32_t* order,
                              void* stream) {
  if (!splats) return GS_ERR_INVALID_ARG;
  return gs::depth_enqueue(splats, workspace, workspace_bytes, order, static_cast<cudaStream_t>(stream));
}

extern "C" int gs_bin_rows_workspace_size(int64_t n, int32_t width, int32_t height, int64_t k_capacity,
                                          size_t* bytes) {
  if (!bytes || n < 0 || k_capacity < 0) return GS_ERR_INVALID_ARG;
  int st = gs::check_dims(width, height);
  if (st != GS_OK) return st;
  const int64_t tiles = int64_t((width + gs::kTile - 1) / gs::kTile) * int64_t((height + gs::kTile - 1) / gs::kTile);
  gs::RowsLayout L;
  st = gs::rows_layout(n, tiles, k_capacity, &L);
  if (st != GS_OK) return st;
  *bytes = L.bytes;
  return GS_OK;
}

extern "C" int gs_bin_rows_async(const gs_splats_t* splats, const uint32_t* order, int32_t width, int32_t height,
                                 int32_t tile_row_begin, int32_t tile_row_end, void* workspace,
                                 size_t workspace_bytes, int64_t k_capacity, uint32_t* sorted_ids, int32_t* ranges,
                                 int64_t* k_info, void* stream) {
  using namespace gs;
  if (!splats || !k_info || k_capacity < 0) return GS_ERR_INVALID_ARG;
  int st = check_dims(width, height);
  if (st != GS_OK) return st;
  return rows_enqueue(splats, order, width, height, RowBand{tile_row_begin, tile_row_end, false}, workspace,
                      workspace_bytes, k_capacity, sorted_ids, ranges, k_info, static_cast<cudaStream_t>(stream));
}

extern "C" int gs_bin_and_sort(const gs_splats_t* splats, int32_t width, int32_t height, void* workspace,
                               size_t workspace_bytes, int64_t k_capacity, uint32_t* sorted_ids, int32_t* ranges,
                               int64_t* k_out, void* stream) {
  using namespace gs;
  if (!splats || !k_out || k_capacity < 0) return GS_ERR_INVALID_ARG;
  int st = check_dims(width, height);
  if (st != GS_OK) return st;
  *k_out = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t tiles = int64_t((width + kTile - 1) / kTile) * int64_t((height + kTile - 1) / kTile);
  if (splats->n == 0) {
    if (ranges) {
      cudaError_t e = cudaMemsetAsync(ranges, 0, size_t(tiles) * 2 * sizeof(int32_t), s);
      if (e != cudaSuccess) return record_cuda_error(e);
    }
    return GS_OK;
  }
  if (!workspace) return GS_ERR_INVALID_ARG;
  FullLayout L;
  st = full_layout(splats->n, tiles, k_capacity, &L);
  if (st != GS_OK) return st;
  if (workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  int64_t* kinfo = reinterpret_cast<int64_t*>(static_cast<char*>(workspace) + L.rows_ws + L.R.kinfo);
  // with no instance buffers only K is computed (capacity 0)
  const int64_t cap = (sorted_ids && ranges) ? k_capacity : 0;
  st = bin_enqueue(splats, width, height, workspace, workspace_bytes, cap, sorted_ids, ranges, kinfo, s);
  if (st != GS_OK) return st;
  int64_t host[3] = {0, 0, 0};
  cudaError_t e = cudaMemcpyAsync(host, kinfo, sizeof(host), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return record_cuda_error(e);
  *k_out = host[0];
  if (host[1] & kFlagZeroQuat) return GS_ERR_ZERO_QUATERNION;
  if (host[1] & kFlagLimit) return GS_ERR_RESOURCE_LIMIT;  // rasterizer.py:99-101
  if (host[1] & kFlagCapacity) return GS_ERR_CAPACITY;
  if (host[0] > 0 && (!sorted_ids || !ranges)) return GS_ERR_INVALID_ARG;
  return GS_OK;
}
