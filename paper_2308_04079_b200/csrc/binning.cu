// K2-K5 binning — replaces splatlab rasterizer.bin_and_sort (rasterizer.py:69-124)
// and make_keys (rasterizer.py:55-62).  Hand-written for sm_100a; no library
// sort or scan.
//
// The reference duplicates every splat into every tile of its radius box,
// packs (tile << 32 | float32-depth bits) keys and runs ONE stable argsort
// over the K instances.  The same lexicographic order (tile, float32 depth,
// Gaussian index) is produced here without ever sorting the K instances:
//
//   1. depth order over the N Gaussians: a stable LSD radix sort of the
//      float32 depth bits (4 x 8-bit digits; culled Gaussians carry the
//      largest key), one "onesweep" kernel per digit: warp-level match_any
//      ranks + per-warp digit counts, decoupled look-back across blocks for
//      the global digit offsets (digit totals come from one histogram kernel
//      over all four digits).  The last pass also gathers each Gaussian's
//      tile rectangle into depth order.
//   2. super-tile buckets: the tiles are grouped into super-tiles of 8 x 4
//      tiles (32 = one warp, one lane per tile; 16 x 8 / 32 x 16 with 2 x 2 /
//      4 x 4 tiles per lane for very large frames).  Every Gaussian is
//      appended, in depth order, to the bucket of every super-tile its
//      rectangle meets, with its rectangle clipped to that super-tile (a
//      stable counting sort: per-chunk bucket counts, one exclusive scan,
//      then an ordered scatter with match_any ranks inside each warp).
//   3. windows: each bucket is cut into windows of 512 entries.  One warp
//      per window counts, per lane (= tile), the entries covering its tile;
//      a prefix over the bucket's windows gives every (window, tile) its
//      offset inside the tile's list, and the tiles' totals.
//   4. one exclusive scan of the tile totals in tile order gives the tile
//      ranges [start, end) (rasterizer.py:118-123) and K.
//   5. one warp per window walks its entries again, every lane appending the
//      Gaussian id to its own tile's list when the entry covers the tile —
//      in bucket order, i.e. depth order, so ties keep the index order of the
//      reference's stable sort.  The optional 64-bit keys (tile << 32 |
//      depth bits) are written alongside.
//
// HBM traffic (c3: N = 3M, K = 30.8M, ~5.8M bucket entries): the sort moves
// 16 B / Gaussian / pass, the buckets 8 B / entry written + read twice, the
// instance list is written once (4 B / instance); nothing of size K is read
// back.  K never leaves the device: every kernel after the histogram reads
// the flags in k_info and returns early when the frame overflowed the
// caller's capacity (the ranges are then all empty), so the whole binning
// is enqueued without a host synchronisation and is CUDA-graph capturable.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr uint32_t kCulledKey = 0xFFFFFFFFu;
// kinfo[] (device, int64): [0] K, [1] flags, [2] K clamped to the capacity
constexpr int64_t kFlagZeroQuat = 1, kFlagCapacity = 2, kFlagLimit = 4;

// depth sort
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef GS_SCAN_ITEMS
#define GS_SCAN_ITEMS 16
#endif
constexpr int kItems = GS_SCAN_ITEMS;          // scan items per thread
constexpr int kScanTile = kThreads * kItems;   // 4096 values per scan block
#ifndef GS_SORT_ITEMS
#define GS_SORT_ITEMS 12   // 3072 keys per block: 8 / 12 / 16 -> 0.454 / 0.446 / 0.457 ms at c3 (1.299 / 1.274 / 1.289 at 6M/4K)
#endif
constexpr int kSortItems = GS_SORT_ITEMS;      // depth keys per thread and sort pass
constexpr int kSortTile = kThreads * kSortItems;
constexpr int kRadix = 256;
constexpr int kPasses = 4;
constexpr uint64_t kStAgg = uint64_t(1) << 32, kStPre = uint64_t(2) << 32;

// super-tile buckets and walk windows
constexpr int kMaxSuper = 4096;                 // bucket scatter keeps kWarps x S cursors in smem
// Gaussians per bucketing block, chosen per frame: small chunks give the
// count / scatter more blocks, but M and Mw grow with S x chunks, so 1024 for
// up to 512 super-tiles (1080p: 0.466 -> 0.456 ms) and 2048 above (4K, S =
// 1020: 1.335 -> 1.304 ms with 2048 vs 4096; 1.446 with 1024)
constexpr int kChunkSmall = 1024, kChunkLarge = 2048, kChunkSmallMaxS = 512;
inline int chunk_for(int S) { return S <= kChunkSmallMaxS ? kChunkSmall : kChunkLarge; }
#ifndef GS_BIN_WINDOW
#define GS_BIN_WINDOW 1024
#endif
constexpr int kWindow = GS_BIN_WINDOW;          // bucket entries per walk window
constexpr uint32_t kEmptyRect = 0x0000FFFFu;    // packed local rect that covers nothing (x0 = y0 = 255 > x1 = y1 = 0)

struct Grid {
  int tiles_x, tiles_y;
  int lq;        // log2 tiles per lane per dimension (0, 1, 2)
  int sx, sy;    // super-tile grid
  int S;
};

__host__ __device__ __forceinline__ int super_w(const Grid& g) { return 8 << g.lq; }
__host__ __device__ __forceinline__ int super_h(const Grid& g) { return 4 << g.lq; }

// Look-back status words (flag << 32 | count) are self-contained, so relaxed
// gpu-scope accesses suffice (a volatile access would be system-scope).
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back for one counter of block b: the exclusive prefix over
// blocks [0, b), walking back over the predecessors' status words
// (base + p * stride) GS_LOOKBACK at a time (one memory round trip each)
// until an inclusive prefix is met.
#ifndef GS_LOOKBACK
#define GS_LOOKBACK 4   // predecessors per round trip: 2 / 3 / 4 / 6 / 8 -> 0.457 / 0.453 / 0.454 / 0.457 / 0.462 ms at c3
#endif
__device__ __forceinline__ uint32_t look_back(const uint64_t* base, int64_t stride, int64_t b) {
  constexpr int kW = GS_LOOKBACK;   // predecessors read per memory round trip
  uint32_t excl = 0;
  for (int64_t p = b - 1; p >= 0; p -= kW) {
    uint64_t v[kW];
#pragma unroll
    for (int i = 0; i < kW; ++i) v[i] = p - i >= 0 ? ld_status(base + (p - i) * stride) : kStPre;
    bool done = false;
#pragma unroll
    for (int i = 0; i < kW; ++i) {
      if (!done) {
        while (v[i] == 0) v[i] = ld_status(base + (p - i) * stride);   // not yet published
        excl += uint32_t(v[i]);
        done = (v[i] & kStPre) != 0;
      }
    }
    if (done) break;
  }
  return excl;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// The lanes holding the same BITS-bit value as this lane (among the lanes
// with valid set; invalid lanes get 0): one ballot per bit.  MATCH.ANY does
// the same in one instruction but issues at a small fraction of the ballot
// rate on sm_100.
#ifndef GS_BIN_MATCH
#define GS_BIN_MATCH 0
#endif
template <int BITS>
__device__ __forceinline__ uint32_t peer_mask(uint32_t v, bool valid) {
  if (GS_BIN_MATCH) {
    // invalid lanes get a value no valid lane can hold
    const uint32_t m = __match_any_sync(0xffffffffu, valid ? v : 0xFFFFFFFFu);
    return valid ? m : 0u;
  }
  uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int i = 0; i < BITS; ++i) {
    const bool bit = (v >> i) & 1u;
    const uint32_t b = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? b : ~b;
  }
  return valid ? peers : 0u;
}

__device__ __forceinline__ uint32_t warp_inclusive_sum(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Exclusive prefix of v over the block (blockDim.x multiple of 32, <= 1024);
// *total receives the block sum.  s_warp: >= 32 words of smem.
__device__ __forceinline__ uint32_t block_exclusive_sum(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t incl = warp_inclusive_sum(v);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < nw ? s_warp[lane] : 0u;
    const uint32_t wi = warp_inclusive_sum(w);
    if (lane < nw) s_warp[lane] = wi - w;
    if (lane == nw - 1) s_warp[32] = wi;
  }
  __syncthreads();
  const uint32_t r = s_warp[warp] + incl - v;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// 1. depth order

__device__ __forceinline__ uint32_t depth_key(const float* depth, const int32_t* tiles, int64_t g) {
  // positive float32 bit patterns order like the floats (rasterizer.py:55-62);
  // Gaussians without instances (culled / off-screen) go last
  return tiles[g] > 0 ? __float_as_uint(depth[g]) : kCulledKey;
}

// Digit histograms of all four passes + K = sum of tiles_touched (u64).
// kHistItems consecutive Gaussians per thread, loaded as vectors up front
// (one memory round trip per thread instead of a dependent grid-stride loop).
#ifndef GS_HIST_ITEMS
#define GS_HIST_ITEMS 16   // Gaussians per thread: 4 / 8 / 16 -> 0.446 / 0.434 / 0.430 ms binning at c3
#endif
constexpr int kHistItems = GS_HIST_ITEMS;
__global__ void __launch_bounds__(kThreads) depth_hist_kernel(const float* __restrict__ depth,
                                                             const int32_t* __restrict__ tiles, int64_t n,
                                                             uint32_t* __restrict__ hist, int64_t* __restrict__ kinfo) {
  pdl_wait();
  __shared__ uint32_t s_h[kPasses * kRadix];
  for (int i = threadIdx.x; i < kPasses * kRadix; i += kThreads) s_h[i] = 0;
  __syncthreads();
  const int64_t i0 = (int64_t(blockIdx.x) * kThreads + threadIdx.x) * kHistItems;
  uint32_t dk[kHistItems];
  int32_t tt[kHistItems];
  const bool vec = i0 + kHistItems <= n && ((reinterpret_cast<uintptr_t>(depth) | reinterpret_cast<uintptr_t>(tiles)) & 15u) == 0;
  if (vec) {
#pragma unroll
    for (int q = 0; q < kHistItems / 4; ++q) {
      const uint4 d4 = reinterpret_cast<const uint4*>(depth + i0)[q];
      const int4 t4 = reinterpret_cast<const int4*>(tiles + i0)[q];
      dk[4 * q] = d4.x; dk[4 * q + 1] = d4.y; dk[4 * q + 2] = d4.z; dk[4 * q + 3] = d4.w;
      tt[4 * q] = t4.x; tt[4 * q + 1] = t4.y; tt[4 * q + 2] = t4.z; tt[4 * q + 3] = t4.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kHistItems; ++j) {
      const bool ok = i0 + j < n;
      dk[j] = ok ? __float_as_uint(depth[i0 + j]) : 0u;
      tt[j] = ok ? tiles[i0 + j] : -1;   // -1: past the end, not counted
    }
  }
  uint64_t ksum = 0;
#pragma unroll
  for (int j = 0; j < kHistItems; ++j) {
    const bool ok = tt[j] >= 0;
    const uint32_t key = tt[j] > 0 ? dk[j] : kCulledKey;
    ksum += tt[j] > 0 ? uint64_t(tt[j]) : 0u;
    // the top digit takes a handful of values per frame: one atomic per
    // distinct value of the warp; the lower digits are spread over the bins
    uint32_t todo = __ballot_sync(0xffffffffu, ok);
    const uint32_t top = key >> 24;
    while (todo) {
      const uint32_t v = __shfl_sync(0xffffffffu, top, __ffs(todo) - 1);
      const uint32_t m = __ballot_sync(0xffffffffu, ok && top == v) & todo;
      if ((threadIdx.x & 31) == __ffs(todo) - 1) atomicAdd(&s_h[3 * kRadix + v], uint32_t(__popc(m)));
      todo &= ~m;
    }
    if (ok) {
#pragma unroll
      for (int p = 0; p < kPasses - 1; ++p) atomicAdd(&s_h[p * kRadix + ((key >> (8 * p)) & 0xFFu)], 1u);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
  if ((threadIdx.x & 31) == 0 && ksum)
    atomicAdd(reinterpret_cast<unsigned long long*>(kinfo), static_cast<unsigned long long>(ksum));
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kRadix; i += kThreads)
    if (s_h[i]) atomicAdd(&hist[i], s_h[i]);
}

// One block of 1024 threads: exclusive digit offsets of every pass, and the
// frame's flags (rasterizer.py:99-101 instance limit, caller capacity,
// zero quaternion from the projection).
__global__ void __launch_bounds__(1024) sort_setup_kernel(const uint32_t* __restrict__ hist,
                                                          uint32_t* __restrict__ digit_base,
                                                          const int32_t* __restrict__ status, int64_t capacity,
                                                          int64_t* __restrict__ kinfo) {
  pdl_wait();
  __shared__ uint32_t s_w[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;   // pass = t / 256 = warp / 8
  const uint32_t v = hist[t];
  const uint32_t incl = warp_inclusive_sum(v);
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t before = 0;
  for (int w = warp & ~7; w < warp; ++w) before += s_w[w];
  digit_base[t] = before + incl - v;
  if (t == 0) {
    const uint64_t K = uint64_t(kinfo[0]);
    int64_t flags = (status[0] & 1) ? kFlagZeroQuat : 0;
    if (K > uint64_t(kMaxInstances) || K > uint64_t(INT32_MAX)) flags |= kFlagLimit;
    if (K > uint64_t(capacity)) flags |= kFlagCapacity;
    kinfo[1] = flags;
    kinfo[2] = int64_t(K < uint64_t(capacity) ? K : uint64_t(capacity));
  }
}

// One stable LSD pass over 8 digit bits.  Block = 4096 keys (8 warps x 16
// items, item j of lane l at warp offset 32 j + l, so the in-warp order is
// (j, lane)); the block index comes from a ticket so a block only waits on
// blocks that are already running.  The block's keys are first placed in
// shared memory in (digit, stable rank) order and then written out, thread i
// writing staged slot i: consecutive threads of one digit write consecutive
// global positions, so the scatter is coalesced in runs (~16 keys per digit
// per block) instead of one 4-byte sector write per key.  kFirst: keys from
// depth / tiles_touched and values = Gaussian index.  kLast: writes only
// the depth order (the values); bucket_count gathers the rectangles.
#ifndef GS_SORT_RANK_OR
#define GS_SORT_RANK_OR 1
#endif
#ifndef GS_SORT_MIN_BLOCKS
#define GS_SORT_MIN_BLOCKS 4
#endif
template <bool kFirst, bool kLast>
__global__ void __launch_bounds__(kThreads, GS_SORT_MIN_BLOCKS) onesweep_kernel(
    const float* __restrict__ depth, const int32_t* __restrict__ tiles, const int4* __restrict__ rect,
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ ids_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ ids_out, int4* __restrict__ drect_out, const uint32_t* __restrict__ digit_base,
    uint64_t* status, uint32_t* ticket, int shift, int64_t n, const int64_t* __restrict__ kinfo) {
  pdl_wait();
  __shared__ uint32_t s_cnt[kWarps][kRadix];
  __shared__ uint32_t s_local[kRadix];
  __shared__ uint32_t s_delta[kRadix];
  __shared__ uint32_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];
  __shared__ uint32_t s_w[33];
  __shared__ uint32_t s_block;
  if (kinfo[1] != 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_block = atomicAdd(ticket, 1u);
  // peer masks by shared-memory OR: the ranking phase borrows s_keys as
  // [kWarps][kRadix] bitmask bins (lane bits), cleared again by each digit's leader
  uint32_t* bins = s_keys + warp * kRadix;
  for (int i = tid; i < kWarps * kRadix; i += kThreads) {
    (&s_cnt[0][0])[i] = 0u;
    if (GS_SORT_RANK_OR) s_keys[i] = 0u;
  }
  __syncthreads();
  const uint32_t b = s_block;
  const int64_t base = int64_t(b) * kSortTile + warp * (32 * kSortItems);
  uint32_t key[kSortItems], val[kSortItems], rank[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + j * 32 + lane;
    if (kFirst) {
      key[j] = i < n ? depth_key(depth, tiles, i) : kCulledKey;
      val[j] = uint32_t(i);
    } else {
      key[j] = i < n ? keys_in[i] : kCulledKey;
      val[j] = i < n ? ids_in[i] : 0u;
    }
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const bool ok = base + j * 32 + lane < n;
    const uint32_t d = (key[j] >> shift) & 0xFFu;
    uint32_t peers;
    if (GS_SORT_RANK_OR) {
      // the lanes holding digit d set their bits in bins[d]; OR is order-free
      if (ok) atomicOr(&bins[d], 1u << lane);
      __syncwarp();
      peers = ok ? bins[d] : 0u;
    } else {
      peers = peer_mask<8>(d, ok);
    }
    const uint32_t c = ok ? s_cnt[warp][d] : 0u;
    rank[j] = c + __popc(peers & lt);
    __syncwarp();
    if (ok && lane == 31 - __clz(peers)) {
      s_cnt[warp][d] = c + __popc(peers);
      if (GS_SORT_RANK_OR) bins[d] = 0u;
    }
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = tid;   // kThreads == kRadix
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_cnt[w][d];
      s_cnt[w][d] = total;
      total += c;
    }
    uint32_t block_total;
    const uint32_t local = block_exclusive_sum(total, s_w, &block_total);
    s_local[d] = local;
    uint64_t* st = status + int64_t(b) * kRadix + d;
    uint32_t excl = 0;
    if (b == 0) {
      st_status(st, kStPre | total);
    } else {
      st_status(st, kStAgg | total);
      excl = look_back(status + d, kRadix, b);
      st_status(st, kStPre | (excl + total));
    }
    s_delta[d] = digit_base[d] + excl - local;   // global position = staged slot + delta
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    if (base + j * 32 + lane >= n) continue;
    const uint32_t d = (key[j] >> shift) & 0xFFu;
    const uint32_t lp = s_local[d] + s_cnt[warp][d] + rank[j];
    s_keys[lp] = key[j];
    s_vals[lp] = val[j];
  }
  __syncthreads();
  const int64_t left = n - int64_t(b) * kSortTile;
  const int cnt = left < kSortTile ? int(left) : kSortTile;
  if (kLast) {
    for (int i = tid; i < cnt; i += kThreads) {
      const uint32_t k = s_keys[i];
      ids_out[uint32_t(i) + s_delta[(k >> shift) & 0xFFu]] = s_vals[i];
    }
  } else {
    for (int i = tid; i < cnt; i += kThreads) {
      const uint32_t k = s_keys[i], v = s_vals[i];
      const uint32_t pos = uint32_t(i) + s_delta[(k >> shift) & 0xFFu];
      ids_out[pos] = v;
      keys_out[pos] = k;
    }
  }
}

// ---------------------------------------------------------------------------
// 2. super-tile buckets

struct SuperRect {
  int x0, y0, x1, y1;   // inclusive super-tile rectangle; empty when x1 < x0
};

__device__ __forceinline__ SuperRect super_rect(int4 rc, const Grid& g) {
  if (rc.x > rc.z) return SuperRect{0, 0, -1, -1};
  const int sw = 3 + g.lq, sh = 2 + g.lq;
  return SuperRect{rc.x >> sw, rc.y >> sh, rc.z >> sw, rc.w >> sh};
}

// per chunk of kChunk depth-ranked Gaussians: the number of Gaussians meeting
// each super-tile -> M[s * chunks + chunk]
// The rectangles are gathered into depth order here (drect[r] =
// rect[order[r]]; the Gaussians without instances, which the sort put last,
// get the empty rectangle), with the gathers of a thread issued together.
// Counts are kept per warp range of the chunk (kChunk / kWarps Gaussians, the
// ranges bucket_scatter's warps own): M[s * chunks + chunk] = their sum and
// Mw[(chunk * kWarps + w) * S + s] (u16) the warp range's own count, from
// which the scatter's warps take their cursor bases without recounting.
template <int kChunk>
__global__ void __launch_bounds__(kThreads) bucket_count_kernel(const int4* __restrict__ rect,
                                                               const uint32_t* __restrict__ order,
                                                               const uint32_t* __restrict__ hist, int4* __restrict__ drect,
                                                               int64_t n, Grid g, uint32_t* __restrict__ M,
                                                               uint16_t* __restrict__ Mw, int64_t chunks,
                                                               const int64_t* __restrict__ kinfo) {
  pdl_wait();
  extern __shared__ uint32_t s_h[];   // [kWarps][S]
  if (kinfo[1] != 0) return;
  for (int s = threadIdx.x; s < kWarps * g.S; s += kThreads) s_h[s] = 0u;
  // Gaussians with instances: every key except the culled 0xFFFFFFFF (depth > 0, so no other key has top byte 0xFF)
  const int64_t visible = n - int64_t(hist[3 * kRadix + 255]);
  __syncthreads();
  const int64_t r0 = int64_t(blockIdx.x) * kChunk;
  constexpr int kPer = kChunk / kThreads;
  int4 rc[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int64_t r = r0 + threadIdx.x + u * kThreads;
    rc[u] = r < visible ? rect[order[r]] : make_int4(0, 0, -1, -1);
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int64_t r = r0 + threadIdx.x + u * kThreads;
    if (r >= n) break;
    drect[r] = rc[u];
    const SuperRect q = super_rect(rc[u], g);
    uint32_t* h = s_h + ((threadIdx.x + u * kThreads) / (kChunk / kWarps)) * g.S;
    for (int y = q.y0; y <= q.y1; ++y)
      for (int x = q.x0; x <= q.x1; ++x) atomicAdd(&h[y * g.sx + x], 1u);
  }
  __syncthreads();
  for (int s = threadIdx.x; s < g.S; s += kThreads) {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_h[w * g.S + s];
      Mw[(int64_t(blockIdx.x) * kWarps + w) * g.S + s] = uint16_t(c);
      sum += c;
    }
    M[int64_t(s) * chunks + blockIdx.x] = sum;
  }
}

// In-place exclusive scan of a u32 array (single pass, decoupled look-back
// of one value per block).  *total_out = the sum.
__global__ void __launch_bounds__(kThreads) scan_kernel(uint32_t* data, int64_t len, uint64_t* status, uint32_t* ticket,
                                                        uint32_t* total_out, const int64_t* __restrict__ kinfo) {
  pdl_wait();
  __shared__ uint32_t s_w[33];
  __shared__ uint32_t s_block, s_excl;
  if (kinfo[1] != 0) return;
  if (threadIdx.x == 0) s_block = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t b = s_block;
  const int64_t i0 = int64_t(b) * kScanTile + int64_t(threadIdx.x) * kItems;
  uint32_t v[kItems];
  uint32_t sum = 0;
  if (i0 + kItems <= len) {
    const uint4* p = reinterpret_cast<const uint4*>(data + i0);
#pragma unroll
    for (int q = 0; q < kItems / 4; ++q) {
      const uint4 u = p[q];
      v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kItems; ++j) v[j] = i0 + j < len ? data[i0 + j] : 0u;
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) sum += v[j];
  uint32_t total;
  const uint32_t excl_t = block_exclusive_sum(sum, s_w, &total);
  if (threadIdx.x == 0) {
    uint32_t excl = 0;
    uint64_t* st = status + b;
    if (b == 0) {
      st_status(st, kStPre | total);
    } else {
      st_status(st, kStAgg | total);
      excl = look_back(status, 1, b);
      st_status(st, kStPre | (excl + total));
    }
    s_excl = excl;
    if (int64_t(b + 1) * kScanTile >= len) *total_out = excl + total;   // the last block
  }
  __syncthreads();
  uint32_t run = s_excl + excl_t;
  if (i0 + kItems <= len) {
    uint4* p = reinterpret_cast<uint4*>(data + i0);
#pragma unroll
    for (int q = 0; q < kItems / 4; ++q) {
      uint4 u;
      u.x = run; run += v[4 * q];
      u.y = run; run += v[4 * q + 1];
      u.z = run; run += v[4 * q + 2];
      u.w = run; run += v[4 * q + 3];
      p[q] = u;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kItems; ++j)
      if (i0 + j < len) {
        data[i0 + j] = run;
        run += v[j];
      }
  }
}

// One block of 1024 threads: bucket starts (from the scanned M), the window
// starts of every bucket and the window -> bucket map.
// bstart[S] = entries, wstart[S] = windows.
__global__ void __launch_bounds__(1024) window_setup_kernel(const uint32_t* __restrict__ M, int64_t chunks,
                                                            const uint32_t* __restrict__ m_total, Grid g,
                                                            uint32_t* __restrict__ bstart, uint32_t* __restrict__ wstart,
                                                            uint32_t* __restrict__ wmap,
                                                            const int64_t* __restrict__ kinfo) {
  pdl_wait();
  __shared__ uint32_t s_w[33];
  if (kinfo[1] != 0) return;
  constexpr int kPer = kMaxSuper / 1024;
  const int s0 = threadIdx.x * kPer;
  uint32_t st[kPer], nw[kPer];
  uint32_t sum = 0;
  const uint32_t total = *m_total;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int s = s0 + k;
    st[k] = s < g.S ? M[int64_t(s) * chunks] : total;
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int s = s0 + k;
    const uint32_t end = s + 1 < g.S ? (k + 1 < kPer ? st[k + 1] : M[int64_t(s + 1) * chunks]) : total;
    nw[k] = s < g.S ? (end - st[k] + kWindow - 1) / kWindow : 0u;
    sum += nw[k];
  }
  uint32_t wtot;
  uint32_t run = block_exclusive_sum(sum, s_w, &wtot);
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int s = s0 + k;
    if (s < g.S) {
      bstart[s] = st[k];
      wstart[s] = run;
      for (uint32_t w = 0; w < nw[k]; ++w) wmap[run + w] = uint32_t(s);
    }
    run += nw[k];
  }
  if (threadIdx.x == 0) {
    bstart[g.S] = total;
    wstart[g.S] = wtot;
  }
}

// Ordered scatter of the bucket entries.  Each warp owns 512 consecutive
// depth-ranked Gaussians; its per-bucket cursors (smem, kWarps x S) start at
// the chunk's scanned count plus the counts of the warp's predecessors in
// the block.  The warp flattens its Gaussians' (Gaussian, super-tile) pairs
// 32 at a time in (depth rank, super-tile) order; lanes hitting the same
// bucket (found by ballots over the bucket bits) are ranked by lane, so every
// bucket receives its Gaussians in depth order.  Entry = (Gaussian id,
// rectangle clipped to the super-tile, local tile coordinates packed
// x0 | y0 << 8 | x1 << 16 | y1 << 24).  (Staging the block's entries in
// shared memory for coalesced writes measured slower: 116-133 vs 96 us at c3.)
template <bool kOrBins, int kChunk>
__global__ void __launch_bounds__(kThreads) bucket_scatter_kernel(const int4* __restrict__ drect,
                                                                 const uint32_t* __restrict__ order, int64_t n, Grid g,
                                                                 const uint32_t* __restrict__ M,
                                                                 const uint16_t* __restrict__ Mw, int64_t chunks,
                                                                 uint2* __restrict__ entries, int64_t capacity,
                                                                 const int64_t* __restrict__ kinfo) {
  pdl_wait();
  extern __shared__ uint32_t s_cur[];   // [kWarps][S] cursors, then [kWarps][S] bytes of bucket stamps
  if (kinfo[1] != 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = g.S;
  for (int i = tid; i < kWarps * S; i += kThreads) s_cur[i] = 0u;
  __syncthreads();
  const int64_t rw = int64_t(blockIdx.x) * kChunk + warp * (kChunk / kWarps);
  uint32_t* cur = s_cur + warp * S;
  uint8_t* stamp = reinterpret_cast<uint8_t*>(s_cur + kWarps * S) + warp * S;
  uint32_t* bins = s_cur + kWarps * S + warp * S;   // kOrBins: [kWarps][S] lane bitmasks
  if (kOrBins)
    for (int i = tid; i < kWarps * S; i += kThreads) s_cur[kWarps * S + i] = 0u;
  // each warp range's cursors start at the chunk's scanned count plus the
  // counts of the ranges before it (bucket_count's Mw)
  for (int s = tid; s < S; s += kThreads) {
    uint32_t run = M[int64_t(s) * chunks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      s_cur[w * S + s] = run;
      run += Mw[(int64_t(blockIdx.x) * kWarps + w) * S + s];
    }
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  const int sw = super_w(g), sh = super_h(g);
  for (int i = 0; i < kChunk / kWarps; i += 32) {
    const int64_t r = rw + i + lane;
    int4 rc = make_int4(0, 0, -1, -1);
    uint32_t gid = 0;
    if (r < n) {
      rc = drect[r];
      gid = order[r];
    }
    const SuperRect q = super_rect(rc, g);
    const int nsx = q.x1 - q.x0 + 1;
    const uint32_t cnt = q.x1 >= q.x0 ? uint32_t(nsx * (q.y1 - q.y0 + 1)) : 0u;
    // jj / nsx = umulhi(jj, ceil(2^32 / nsx)), exact for jj * nsx < 2^32
    const uint32_t magic = nsx > 1 ? 0xFFFFFFFFu / uint32_t(nsx) + 1u : 0u;
    const uint32_t end = warp_inclusive_sum(cnt);   // non-decreasing over the lanes
    const uint32_t off = end - cnt;
    const uint32_t tot = __shfl_sync(0xffffffffu, end, 31);
    for (uint32_t ob = 0; ob < tot; ob += 32) {
      const uint32_t o = ob + lane;
      int owner = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t e = __shfl_sync(0xffffffffu, end, owner + step - 1);
        if (e <= o) owner += step;
      }
      owner = min(owner, 31);
      const uint32_t jj = o - __shfl_sync(0xffffffffu, off, owner);
      const int onsx = __shfl_sync(0xffffffffu, nsx, owner);
      const uint32_t omagic = __shfl_sync(0xffffffffu, magic, owner);
      const int ox0 = __shfl_sync(0xffffffffu, q.x0, owner);
      const int oy0 = __shfl_sync(0xffffffffu, q.y0, owner);
      const int rx0 = __shfl_sync(0xffffffffu, rc.x, owner);
      const int ry0 = __shfl_sync(0xffffffffu, rc.y, owner);
      const int rx1 = __shfl_sync(0xffffffffu, rc.z, owner);
      const int ry1 = __shfl_sync(0xffffffffu, rc.w, owner);
      const uint32_t og = __shfl_sync(0xffffffffu, gid, owner);
      const bool valid = o < tot;
      int s = 0, bx = 0, by = 0;
      if (valid) {
        const int jy = onsx == 1 ? int(jj) : int(__umulhi(jj, omagic));
        bx = ox0 + int(jj) - jy * onsx;
        by = oy0 + jy;
        s = by * g.sx + bx;
      }
      uint32_t pos = 0;
      if (kOrBins) {
        // peer masks by shared-memory OR into per-warp bucket bins (order-free)
        if (valid) atomicOr(&bins[s], 1u << lane);
        __syncwarp();
        const uint32_t peers = valid ? bins[s] : 0u;
        const uint32_t c = valid ? cur[s] : 0u;
        pos = c + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == 31 - __clz(peers)) {
          cur[s] = c + __popc(peers);
          bins[s] = 0u;
        }
        __syncwarp();
        if (valid) {
          const int tx0 = bx * sw, ty0 = by * sh;
          const uint32_t lx0 = uint32_t(max(rx0, tx0) - tx0), ly0 = uint32_t(max(ry0, ty0) - ty0);
          const uint32_t lx1 = uint32_t(min(rx1, tx0 + sw - 1) - tx0), ly1 = uint32_t(min(ry1, ty0 + sh - 1) - ty0);
          if (int64_t(pos) < capacity) entries[pos] = make_uint2(og, lx0 | (ly0 << 8) | (lx1 << 16) | (ly1 << 24));
        }
        continue;
      }
      // the warp's 32 pairs usually lie in 32 distinct buckets: detect a
      // shared bucket with a byte stamp per bucket (a lane whose stamp was
      // overwritten shares its bucket), and rank by lane only then
      if (valid) stamp[s] = uint8_t(lane);
      __syncwarp();
      const bool shared = valid && stamp[s] != uint8_t(lane);
      if (!__any_sync(0xffffffffu, shared)) {
        if (valid) {
          pos = cur[s];
          cur[s] = pos + 1u;
        }
      } else {
        const uint32_t peers = peer_mask<12>(uint32_t(s), valid);
        const uint32_t c = valid ? cur[s] : 0u;
        __syncwarp();
        if (valid && lane == 31 - __clz(peers)) cur[s] = c + __popc(peers);
        pos = c + __popc(peers & lt);
      }
      __syncwarp();
      if (valid) {
        const int tx0 = bx * sw, ty0 = by * sh;
        const uint32_t lx0 = uint32_t(max(rx0, tx0) - tx0), ly0 = uint32_t(max(ry0, ty0) - ty0);
        const uint32_t lx1 = uint32_t(min(rx1, tx0 + sw - 1) - tx0), ly1 = uint32_t(min(ry1, ty0 + sh - 1) - ty0);
        if (int64_t(pos) < capacity) entries[pos] = make_uint2(og, lx0 | (ly0 << 8) | (lx1 << 16) | (ly1 << 24));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 3-5. windows, tile ranges, instance lists

// Lane l of a super-tile warp owns the Q x Q tiles at local (((l & 7) Q + a),
// ((l >> 3) Q + b)), sub-tile index a + Q b.
template <int Q>
__device__ __forceinline__ bool covers(uint32_t packed, int lane, int a, int b) {
  const int x = (lane & 7) * Q + a, y = (lane >> 3) * Q + b;
  return x >= int(packed & 0xFFu) && x <= int((packed >> 16) & 0xFFu) && y >= int((packed >> 8) & 0xFFu) &&
         y <= int(packed >> 24);
}

// Q = 1: the 32-lane coverage mask of an entry (bit 8 row + col).
__device__ __forceinline__ uint32_t cover_mask(uint32_t packed) {
  const uint32_t x0 = packed & 0xFFu, y0 = (packed >> 8) & 0xFFu, x1 = (packed >> 16) & 0xFFu, y1 = packed >> 24;
  if (x1 < x0 || y1 < y0) return 0u;
  const uint32_t cols = (0xFFu >> (7u - x1)) & (0xFFu << x0) & 0xFFu;
  const uint32_t rows = (0x01010101u >> (8u * (3u - y1))) & (0x01010101u << (8u * y0));
  return cols * rows;
}

// 32 x 32 bit-matrix transpose across the warp: lane r holds row r (bit c =
// column c); lane c receives column c (bit r = row r).  Five butterfly steps.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int j = 16, i = 0; j >= 1; j >>= 1, ++i) {
    const uint32_t m = i == 0 ? 0x0000FFFFu : i == 1 ? 0x00FF00FFu : i == 2 ? 0x0F0F0F0Fu : i == 3 ? 0x33333333u
                                                                                                  : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

struct WindowRange {
  uint32_t s, e0, e1;
};

__device__ __forceinline__ WindowRange window_range(uint32_t w, const uint32_t* __restrict__ wmap,
                                                    const uint32_t* __restrict__ bstart,
                                                    const uint32_t* __restrict__ wstart) {
  WindowRange r;
  r.s = wmap[w];
  r.e0 = bstart[r.s] + (w - wstart[r.s]) * uint32_t(kWindow);
  r.e1 = min(r.e0 + uint32_t(kWindow), bstart[r.s + 1]);
  return r;
}

__device__ __forceinline__ int64_t lane_tile(const Grid& g, uint32_t s, int lane, int a, int b, int Q) {
  const int tx = int(s % uint32_t(g.sx)) * (8 * Q) + (lane & 7) * Q + a;
  const int ty = int(s / uint32_t(g.sx)) * (4 * Q) + (lane >> 3) * Q + b;
  return (tx < g.tiles_x && ty < g.tiles_y) ? int64_t(ty) * g.tiles_x + tx : int64_t(-1);
}

// cnt[w][lane][sub] = entries of window w covering the lane's tile
template <int Q>
__global__ void __launch_bounds__(kThreads) window_count_kernel(const uint2* __restrict__ entries,
                                                               const uint32_t* __restrict__ wmap,
                                                               const uint32_t* __restrict__ bstart,
                                                               const uint32_t* __restrict__ wstart, Grid g,
                                                               uint32_t* __restrict__ cnt,
                                                               const int64_t* __restrict__ kinfo) {
  pdl_wait();
  if (kinfo[1] != 0) return;
  const int lane = threadIdx.x & 31;
  const uint32_t nwin = wstart[g.S];
  const uint32_t stride = gridDim.x * kWarps;
  for (uint32_t w = blockIdx.x * kWarps + (threadIdx.x >> 5); w < nwin; w += stride) {
    const WindowRange wr = window_range(w, wmap, bstart, wstart);
    uint32_t c[Q * Q];
#pragma unroll
    for (int k = 0; k < Q * Q; ++k) c[k] = 0u;
    for (uint32_t eb = wr.e0; eb < wr.e1; eb += 32) {
      const uint32_t e = eb + lane;
      const uint32_t packed = e < wr.e1 ? entries[e].y : kEmptyRect;
      if (Q == 1) {
        // lane k holds entry k's tile mask; after the transpose lane t holds
        // the entries covering tile t
        c[0] += __popc(transpose32(cover_mask(packed), lane));
      } else {
        const int m = int(min(32u, wr.e1 - eb));
        for (int k = 0; k < m; ++k) {
          const uint32_t p = __shfl_sync(0xffffffffu, packed, k);
#pragma unroll
          for (int b = 0; b < Q; ++b)
#pragma unroll
            for (int a = 0; a < Q; ++a) c[a + Q * b] += covers<Q>(p, lane, a, b) ? 1u : 0u;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < Q * Q; ++k) cnt[(int64_t(w) * 32 + lane) * (Q * Q) + k] = c[k];
  }
}

// One warp per super-tile: exclusive prefix of the counts over the bucket's
// windows (in place) and the tile totals.
template <int Q>
__global__ void __launch_bounds__(kThreads) window_prefix_kernel(const uint32_t* __restrict__ wstart, Grid g,
                                                                uint32_t* __restrict__ cnt,
                                                                uint32_t* __restrict__ tile_total,
                                                                const int64_t* __restrict__ kinfo) {
  pdl_wait();
  if (kinfo[1] != 0) return;
  const uint32_t s = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (s >= uint32_t(g.S)) return;
  const int lane = threadIdx.x & 31;
  const uint32_t w0 = wstart[s], w1 = wstart[s + 1];
  uint32_t run[Q * Q];
#pragma unroll
  for (int k = 0; k < Q * Q; ++k) run[k] = 0u;
  constexpr int kBatch = Q == 1 ? 8 : 2;
  for (uint32_t w = w0; w < w1; w += kBatch) {
    uint32_t v[kBatch][Q * Q];
#pragma unroll
    for (int i = 0; i < kBatch; ++i)
#pragma unroll
      for (int k = 0; k < Q * Q; ++k) v[i][k] = w + i < w1 ? cnt[(int64_t(w + i) * 32 + lane) * (Q * Q) + k] : 0u;
#pragma unroll
    for (int i = 0; i < kBatch; ++i)
#pragma unroll
      for (int k = 0; k < Q * Q; ++k)
        if (w + i < w1) {
          cnt[(int64_t(w + i) * 32 + lane) * (Q * Q) + k] = run[k];
          run[k] += v[i][k];
        }
  }
#pragma unroll
  for (int b = 0; b < Q; ++b)
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      const int64_t t = lane_tile(g, s, lane, a, b, Q);
      if (t >= 0) tile_total[t] = run[a + Q * b];
    }
}

// One block of 1024 threads: exclusive scan of the tile totals in tile order
// -> ranges [start, end), empty tiles [0, 0] (rasterizer.py:118-123), in
// rounds of 4096 consecutive tiles (4 per thread: coalesced loads and
// stores) carrying the running total.  A flagged frame gets all-empty ranges.
__global__ void __launch_bounds__(1024) tile_ranges_kernel(const uint32_t* __restrict__ tile_total, int64_t tiles,
                                                           int2* __restrict__ ranges,
                                                           const int64_t* __restrict__ kinfo) {
  pdl_wait();
  __shared__ uint32_t s_w[33];
  const bool flagged = kinfo[1] != 0;
  uint32_t carry = 0;
  for (int64_t base = 0; base < tiles; base += 4 * 1024) {
    const int64_t t0 = base + 4 * int64_t(threadIdx.x);
    uint32_t c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = (!flagged && t0 + u < tiles) ? tile_total[t0 + u] : 0u;
    uint32_t total;
    uint32_t run = carry + block_exclusive_sum(c[0] + c[1] + c[2] + c[3], s_w, &total);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (t0 + u < tiles) ranges[t0 + u] = c[u] ? make_int2(int(run), int(run + c[u])) : make_int2(0, 0);
      run += c[u];
    }
    carry += total;
  }
}

// One warp per window: every lane appends, in entry (= depth) order, the
// Gaussian of each entry covering its tile to that tile's list (and the
// 64-bit key when requested).
template <int Q>
__global__ void __launch_bounds__(kThreads) instance_write_kernel(
    const uint2* __restrict__ entries, const uint32_t* __restrict__ wmap, const uint32_t* __restrict__ bstart,
    const uint32_t* __restrict__ wstart, Grid g, const uint32_t* __restrict__ cnt, const int2* __restrict__ ranges,
    const float* __restrict__ depth, uint32_t* __restrict__ ids, unsigned long long* __restrict__ keys,
    const int64_t* __restrict__ kinfo) {
  pdl_wait();
  if (kinfo[1] != 0) return;
  const int lane = threadIdx.x & 31;
  const uint32_t nwin = wstart[g.S];
  const uint32_t stride = gridDim.x * kWarps;
  for (uint32_t w = blockIdx.x * kWarps + (threadIdx.x >> 5); w < nwin; w += stride) {
    const WindowRange wr = window_range(w, wmap, bstart, wstart);
    uint32_t cur[Q * Q];
    int64_t tile[Q * Q];
#pragma unroll
    for (int b = 0; b < Q; ++b)
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        const int k = a + Q * b;
        tile[k] = lane_tile(g, wr.s, lane, a, b, Q);
        cur[k] = tile[k] >= 0 ? uint32_t(ranges[tile[k]].x) + cnt[(int64_t(w) * 32 + lane) * (Q * Q) + k] : 0u;
      }
    for (uint32_t eb = wr.e0; eb < wr.e1; eb += 32) {
      const uint32_t e = eb + lane;
      const uint2 ent = e < wr.e1 ? entries[e] : make_uint2(0u, kEmptyRect);
      if (Q == 1) {
        const uint32_t mask = cover_mask(ent.y);
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const uint32_t m = __shfl_sync(0xffffffffu, mask, k);
          const uint32_t id = __shfl_sync(0xffffffffu, ent.x, k);
          if ((m >> lane) & 1u) {
            ids[cur[0]] = id;
            if (keys) keys[cur[0]] = (static_cast<unsigned long long>(tile[0]) << 32) | __float_as_uint(depth[id]);
            ++cur[0];
          }
        }
      } else {
        const int m = int(min(32u, wr.e1 - eb));
        for (int k = 0; k < m; ++k) {
          const uint32_t p = __shfl_sync(0xffffffffu, ent.y, k);
          const uint32_t id = __shfl_sync(0xffffffffu, ent.x, k);
#pragma unroll
          for (int b = 0; b < Q; ++b)
#pragma unroll
            for (int a = 0; a < Q; ++a) {
              const int kk = a + Q * b;
              if (covers<Q>(p, lane, a, b)) {
                ids[cur[kk]] = id;
                if (keys)
                  keys[cur[kk]] = (static_cast<unsigned long long>(tile[kk]) << 32) | __float_as_uint(depth[id]);
                ++cur[kk];
              }
            }
        }
      }
    }
  }
}

// Q = 1 with staged writes: each lane collects its tile's ids in a 64-slot
// shared-memory ring; whenever a lane holds 32 unwritten ids the warp writes
// them together (one coalesced 128-byte store), and the remainder at the end
// of the window.  One scattered 4-byte store per instance would cost one L2
// sector write each (measured: the L2 write-request rate, not HBM, then
// bounds the pass: 265 vs 172 us at c3).  The walk is bit-transposed: lane t
// receives the mask of the 32 loaded entries covering its tile.
constexpr int kRing = 64, kRingStride = kRing + 1;
constexpr int kWriteWarps = kWarps;
constexpr size_t kStagedSmem = sizeof(uint32_t) * kWarps * 32 * kRingStride;


template <bool kKeys>
__global__ void __launch_bounds__(kThreads) instance_write_staged_kernel(
    const uint2* __restrict__ entries, const uint32_t* __restrict__ wmap, const uint32_t* __restrict__ bstart,
    const uint32_t* __restrict__ wstart, Grid g, const uint32_t* __restrict__ cnt, const int2* __restrict__ ranges,
    const float* __restrict__ depth, uint32_t* __restrict__ ids, unsigned long long* __restrict__ keys,
    const int64_t* __restrict__ kinfo) {
  pdl_wait();
  extern __shared__ uint32_t s_ring[];
  __shared__ uint32_t s_eid[kWarps][32];
  if (kinfo[1] != 0) return;
  const int lane = threadIdx.x & 31;
  uint32_t* ring = s_ring + (threadIdx.x >> 5) * 32 * kRingStride;
  uint32_t* mine = ring + lane * kRingStride;
  uint32_t* eid = s_eid[threadIdx.x >> 5];
  const uint32_t mine_s = smem_u32(mine), eid_s = smem_u32(eid), ring_s = smem_u32(ring);
  // flush of lane f's ring: 32 (or count) ids from slot `from` to ids[dst...]
  auto flush = [&](int f, uint32_t from, uint32_t dst, uint32_t count, int64_t tile_f) {
    if (uint32_t(lane) < count) {
      uint32_t id;
      asm volatile("ld.shared.u32 %0, [%1];"
                   : "=r"(id)
                   : "r"(ring_s + 4u * (uint32_t(f) * kRingStride + ((from + uint32_t(lane)) & (kRing - 1))))
                   : "memory");
      ids[dst + lane] = id;
      if (kKeys) keys[dst + lane] = (static_cast<unsigned long long>(tile_f) << 32) | __float_as_uint(depth[id]);
    }
  };
  const uint32_t nwin = wstart[g.S];
  const uint32_t stride = gridDim.x * kWarps;
  for (uint32_t w = blockIdx.x * kWarps + (threadIdx.x >> 5); w < nwin; w += stride) {
    const WindowRange wr = window_range(w, wmap, bstart, wstart);
    const int64_t tile = lane_tile(g, wr.s, lane, 0, 0, 1);
    uint32_t cur = tile >= 0 ? uint32_t(ranges[tile].x) + cnt[int64_t(w) * 32 + lane] : 0u;   // next unwritten slot
    uint32_t wp = 0, fp = 0;   // ids staged / written
    for (uint32_t eb = wr.e0; eb < wr.e1; eb += 32) {
      const uint32_t e = eb + lane;
      const uint2 ent = e < wr.e1 ? entries[e] : make_uint2(0u, kEmptyRect);
      eid[lane] = ent.x;
      // lane t: the entries (bit k = entry eb + k) covering tile t, in depth order
      uint32_t col = transpose32(cover_mask(ent.y), lane);
      __syncwarp();
      const uint32_t cnt = uint32_t(__popc(col));
      const int rounds = __reduce_max_sync(0xffffffffu, cnt);
      // branch-free rounds on raw shared addresses.  The column is bit-reversed
      // once, so the leading one (one CLZ) is the next entry in depth order;
      // round r writes ring slot wp + r: a lane whose column is exhausted
      // writes past its staged ids (slots < fp + 64, since wp - fp < 32 before
      // and rounds <= 32), which are overwritten before they are flushed
      uint32_t colr = __brev(col);
      uint32_t wb = 4u * (wp & (kRing - 1));
      for (int r = 0; r < rounds; ++r) {
        const uint32_t k = uint32_t(__clz(colr)) & 31u;   // 32 (exhausted) -> 0
        uint32_t id;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(id) : "r"(eid_s + 4u * k) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(mine_s + wb), "r"(id) : "memory");
        wb = (wb + 4u) & (4u * kRing - 1u);
        colr &= 0x7FFFFFFFu >> k;   // clears the leading one (no-op on an exhausted column)
      }
      wp += cnt;
      __syncwarp();
      // at most 32 ids were staged since the last flush, so a lane holds < 64
      uint32_t full = __ballot_sync(0xffffffffu, wp - fp >= 32u);
      while (full) {   // any order (distinct destinations): highest lane first, one FLO per pick
        const int f = 31 - __clz(full);
        full ^= 1u << f;
        flush(f, __shfl_sync(0xffffffffu, fp, f), __shfl_sync(0xffffffffu, cur, f), 32u,
              kKeys ? __shfl_sync(0xffffffffu, tile, f) : int64_t(0));
        if (lane == f) {
          fp += 32u;
          cur += 32u;
        }
      }
      __syncwarp();
    }
    uint32_t rest = __ballot_sync(0xffffffffu, wp != fp);
    while (rest) {
      const int f = 31 - __clz(rest);
      rest ^= 1u << f;
      flush(f, __shfl_sync(0xffffffffu, fp, f), __shfl_sync(0xffffffffu, cur, f),
            __shfl_sync(0xffffffffu, wp - fp, f), kKeys ? __shfl_sync(0xffffffffu, tile, f) : int64_t(0));
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// host side

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

int make_grid(int width, int height, Grid* g) {
  g->tiles_x = (width + kTile - 1) / kTile;
  g->tiles_y = (height + kTile - 1) / kTile;
  for (int lq = 0; lq <= 2; ++lq) {
    const int64_t sx = (g->tiles_x + (8 << lq) - 1) / (8 << lq), sy = (g->tiles_y + (4 << lq) - 1) / (4 << lq);
    if (sx * sy <= kMaxSuper) {
      g->lq = lq;
      g->sx = int(sx);
      g->sy = int(sy);
      g->S = int(sx * sy);
      return GS_OK;
    }
  }
  return GS_ERR_RESOURCE_LIMIT;   // > 2M tiles (> 537 Mpx frames)
}

struct Layout {
  Grid g;
  int64_t n, cap, tiles, blocks, chunk, chunks, mlen, wmax;
  size_t zero, zero_bytes;                              // memset region
  size_t hist, tickets, mtotal, sort_status, scan_status;  // inside it
  size_t digit_base, keys_a, keys_b, ids_a, ids_b, order, drect, m, mw, bstart, wstart, wmap, entries, cnt, tile_total,
      kinfo, bytes;
};

int layout(int64_t n, int width, int height, int64_t cap, Layout* L) {
  int st = make_grid(width, height, &L->g);
  if (st != GS_OK) return st;
  if (cap > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  const int q2 = 1 << (2 * L->g.lq);
  L->n = n;
  L->cap = cap;
  L->tiles = int64_t(L->g.tiles_x) * L->g.tiles_y;
  L->blocks = (n + kSortTile - 1) / kSortTile;
  L->chunk = chunk_for(L->g.S);
  L->chunks = (n + L->chunk - 1) / L->chunk;
  L->mlen = int64_t(L->g.S) * L->chunks;
  L->wmax = (cap + kWindow - 1) / kWindow + L->g.S;
  const size_t un = size_t(n > 0 ? n : 1), ub = size_t(L->blocks > 0 ? L->blocks : 1);
  const size_t scan_blocks = size_t((L->mlen + kScanTile - 1) / kScanTile) + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes);
    return o;
  };
  L->zero = off;
  L->hist = take(sizeof(uint32_t) * kPasses * kRadix);
  L->tickets = take(sizeof(uint32_t) * 8);
  L->mtotal = take(sizeof(uint32_t) * 8);
  L->sort_status = take(sizeof(uint64_t) * kPasses * kRadix * ub);
  L->scan_status = take(sizeof(uint64_t) * scan_blocks);
  L->zero_bytes = off - L->zero;
  L->digit_base = take(sizeof(uint32_t) * kPasses * kRadix);
  L->keys_a = take(4 * un);
  L->keys_b = take(4 * un);
  L->ids_a = take(4 * un);
  L->ids_b = take(4 * un);
  L->order = take(4 * un);
  L->drect = take(16 * un);
  L->m = take(4 * size_t(L->mlen > 0 ? L->mlen : 1) + 16);
  L->mw = take(2 * size_t(L->mlen > 0 ? L->mlen : 1) * kWarps + 16);   // per warp range, u16
  L->bstart = take(4 * size_t(L->g.S + 1));
  L->wstart = take(4 * size_t(L->g.S + 1));
  L->wmap = take(4 * size_t(L->wmax));
  L->entries = take(8 * size_t(cap > 0 ? cap : 1));
  L->cnt = take(4 * size_t(L->wmax) * 32 * q2);
  L->tile_total = take(4 * size_t(L->tiles));
  L->kinfo = take(4 * sizeof(int64_t));
  L->bytes = off;
  return GS_OK;
}

template <typename T>
T* at(char* ws, size_t off) {
  return reinterpret_cast<T*>(ws + off);
}

cudaError_t smem_opt_in(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

template <int Q>
int walk(const Layout& L, char* ws, const float* depth, uint32_t* ids, int2* ranges, unsigned long long* keys,
         const int64_t* kinfo, cudaStream_t s) {
  const Grid g = L.g;
#ifndef GS_WALK_CTAS_PER_SM
#define GS_WALK_CTAS_PER_SM 8
#endif
  const int persistent = 148 * GS_WALK_CTAS_PER_SM;   // resident 8-warp blocks per SM x 148 SMs
  launch_pdl(window_count_kernel<Q>, persistent, kThreads, 0, s, at<uint2>(ws, L.entries), at<uint32_t>(ws, L.wmap),
                                                        at<uint32_t>(ws, L.bstart), at<uint32_t>(ws, L.wstart), g,
                                                        at<uint32_t>(ws, L.cnt), kinfo);
  int st = check_launch();
  if (st != GS_OK) return st;
  launch_pdl(window_prefix_kernel<Q>, unsigned((g.S + kWarps - 1) / kWarps), kThreads, 0, s, 
      at<uint32_t>(ws, L.wstart), g, at<uint32_t>(ws, L.cnt), at<uint32_t>(ws, L.tile_total), kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  launch_pdl(tile_ranges_kernel, 1, 1024, 0, s, at<uint32_t>(ws, L.tile_total), L.tiles, ranges, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  if (Q == 1) {
    const void* fn = keys ? reinterpret_cast<const void*>(instance_write_staged_kernel<true>)
                          : reinterpret_cast<const void*>(instance_write_staged_kernel<false>);
    cudaError_t e = smem_opt_in(fn, kStagedSmem);
    if (e != cudaSuccess) return record_cuda_error(e);
    if (keys)
      launch_pdl(instance_write_staged_kernel<true>, 148 * 3, kThreads, kStagedSmem, s, 
          at<uint2>(ws, L.entries), at<uint32_t>(ws, L.wmap), at<uint32_t>(ws, L.bstart), at<uint32_t>(ws, L.wstart),
          g, at<uint32_t>(ws, L.cnt), ranges, depth, ids, keys, kinfo);
    else
      launch_pdl(instance_write_staged_kernel<false>, 148 * 3, kThreads, kStagedSmem, s, 
        at<uint2>(ws, L.entries), at<uint32_t>(ws, L.wmap), at<uint32_t>(ws, L.bstart), at<uint32_t>(ws, L.wstart),
        g, at<uint32_t>(ws, L.cnt), ranges, depth, ids, keys, kinfo);
  } else {
    launch_pdl(instance_write_kernel<Q>, persistent, kThreads, 0, s, at<uint2>(ws, L.entries), at<uint32_t>(ws, L.wmap),
                                                            at<uint32_t>(ws, L.bstart), at<uint32_t>(ws, L.wstart), g,
                                                            at<uint32_t>(ws, L.cnt), ranges, depth, ids, keys, kinfo);
  }
  return check_launch();
}

// Step 2 of the binning (bucket counts, their scan, the window setup and the
// ordered bucket scatter) for a chunk size.
template <int kChunk>
int bucket(const Layout& L, char* ws, const gs_splats_t* splats, const uint32_t* order, int4* drect,
           const uint32_t* hist, uint32_t* tickets, int64_t cap, int64_t* kinfo, cudaStream_t s) {
  const Grid g = L.g;
  const int64_t n = L.n;
  const int4* rect = reinterpret_cast<const int4*>(splats->rect);
  uint32_t* M = at<uint32_t>(ws, L.m);
  const size_t smem_count = sizeof(uint32_t) * kWarps * size_t(g.S);
  uint16_t* Mw = at<uint16_t>(ws, L.mw);
  cudaError_t e = smem_opt_in(reinterpret_cast<const void*>(bucket_count_kernel<kChunk>), smem_count);
  if (e != cudaSuccess) return record_cuda_error(e);
  launch_pdl(bucket_count_kernel<kChunk>, unsigned(L.chunks), kThreads, smem_count, s, rect, order, hist, drect, n, g,
             M, Mw, L.chunks, kinfo);
  int st = check_launch();
  if (st != GS_OK) return st;
  uint32_t* mtotal = at<uint32_t>(ws, L.mtotal);
  launch_pdl(scan_kernel, unsigned((L.mlen + kScanTile - 1) / kScanTile), kThreads, 0, s, M, L.mlen,
             at<uint64_t>(ws, L.scan_status), tickets + 4, mtotal, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  launch_pdl(window_setup_kernel, 1, 1024, 0, s, M, L.chunks, mtotal, g, at<uint32_t>(ws, L.bstart),
             at<uint32_t>(ws, L.wstart), at<uint32_t>(ws, L.wmap), kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  // cursors + OR bins (<= 2048 super-tiles) or cursors + byte stamps
  const bool or_bins = g.S <= 2048;
  const size_t smem_scatter = (sizeof(uint32_t) + (or_bins ? sizeof(uint32_t) : 1)) * kWarps * size_t(g.S);
  const void* scatter_fn = or_bins ? reinterpret_cast<const void*>(bucket_scatter_kernel<true, kChunk>)
                                   : reinterpret_cast<const void*>(bucket_scatter_kernel<false, kChunk>);
  if ((e = smem_opt_in(scatter_fn, smem_scatter)) != cudaSuccess) return record_cuda_error(e);
  if (or_bins)
    launch_pdl(bucket_scatter_kernel<true, kChunk>, unsigned(L.chunks), kThreads, smem_scatter, s, drect, order, n, g,
               M, Mw, L.chunks, at<uint2>(ws, L.entries), cap, kinfo);
  else
    launch_pdl(bucket_scatter_kernel<false, kChunk>, unsigned(L.chunks), kThreads, smem_scatter, s, drect, order, n,
               g, M, Mw, L.chunks, at<uint2>(ws, L.entries), cap, kinfo);
  return check_launch();
}

// The whole binning, enqueued on `s` without synchronising.  ranges /
// sorted_ids may be NULL only with capacity 0 (K and the flags only).
int bin_enqueue(const gs_splats_t* splats, int32_t width, int32_t height, void* workspace, size_t workspace_bytes,
                int64_t cap, uint32_t* sorted_ids, int32_t* ranges_raw, uint64_t* keys, int64_t* kinfo,
                cudaStream_t s) {
  const int64_t n = splats->n;
  if (n > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  Layout L;
  int st = layout(n, width, height, cap, &L);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  if (cap > 0 && (!sorted_ids || !ranges_raw)) return GS_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(workspace);
  int2* ranges = reinterpret_cast<int2*>(ranges_raw);
  cudaError_t e = zero_async(kinfo, 3 * sizeof(int64_t), ws + L.zero, L.zero_bytes, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  if (n == 0) {
    if (ranges) e = cudaMemsetAsync(ranges, 0, size_t(L.tiles) * sizeof(int2), s);
    return e == cudaSuccess ? GS_OK : record_cuda_error(e);
  }
  const Grid g = L.g;
  uint32_t* hist = at<uint32_t>(ws, L.hist);
  uint32_t* tickets = at<uint32_t>(ws, L.tickets);
  uint32_t* digit_base = at<uint32_t>(ws, L.digit_base);
  uint64_t* sort_status = at<uint64_t>(ws, L.sort_status);
  const unsigned blocks = unsigned(L.blocks);
  launch_pdl(depth_hist_kernel, unsigned((n + int64_t(kThreads) * kHistItems - 1) / (int64_t(kThreads) * kHistItems)), kThreads, 0, s, splats->depth, splats->tiles_touched, n, hist, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  launch_pdl(sort_setup_kernel, 1, 1024, 0, s, hist, digit_base, splats->status, cap, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  if (cap == 0) {   // K and the flags only
    if (ranges) e = cudaMemsetAsync(ranges, 0, size_t(L.tiles) * sizeof(int2), s);
    return e == cudaSuccess ? GS_OK : record_cuda_error(e);
  }
  // 1. depth order: passes 0..3 over the 8-bit digits (A -> B -> A -> order / drect)
  const int4* rect = reinterpret_cast<const int4*>(splats->rect);
  uint32_t *ka = at<uint32_t>(ws, L.keys_a), *kb = at<uint32_t>(ws, L.keys_b);
  uint32_t *ia = at<uint32_t>(ws, L.ids_a), *ib = at<uint32_t>(ws, L.ids_b);
  uint32_t* order = at<uint32_t>(ws, L.order);
  int4* drect = at<int4>(ws, L.drect);
  const size_t pass_status = size_t(kRadix) * L.blocks;
  launch_pdl(onesweep_kernel<true, false>, blocks, kThreads, 0, s, splats->depth, splats->tiles_touched, rect, nullptr,
                                                           nullptr, ka, ia, nullptr, digit_base, sort_status,
                                                           tickets + 0, 0, n, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  launch_pdl(onesweep_kernel<false, false>, blocks, kThreads, 0, s, nullptr, nullptr, nullptr, ka, ia, kb, ib, nullptr,
                                                            digit_base + kRadix, sort_status + pass_status,
                                                            tickets + 1, 8, n, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  launch_pdl(onesweep_kernel<false, false>, blocks, kThreads, 0, s, nullptr, nullptr, nullptr, kb, ib, ka, ia, nullptr,
                                                            digit_base + 2 * kRadix, sort_status + 2 * pass_status,
                                                            tickets + 2, 16, n, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  launch_pdl(onesweep_kernel<false, true>, blocks, kThreads, 0, s, nullptr, splats->tiles_touched, rect, ka, ia, nullptr,
                                                           order, drect, digit_base + 3 * kRadix,
                                                           sort_status + 3 * pass_status, tickets + 3, 24, n, kinfo);
  if ((st = check_launch()) != GS_OK) return st;
  // 2. super-tile buckets
  st = L.chunk == kChunkSmall ? bucket<kChunkSmall>(L, ws, splats, order, drect, hist, tickets, cap, kinfo, s)
                              : bucket<kChunkLarge>(L, ws, splats, order, drect, hist, tickets, cap, kinfo, s);
  if (st != GS_OK) return st;
  // 3-5. windows, ranges, instance lists
  unsigned long long* k64 = reinterpret_cast<unsigned long long*>(keys);
  switch (g.lq) {
    case 0: return walk<1>(L, ws, splats->depth, sorted_ids, ranges, k64, kinfo, s);
    case 1: return walk<2>(L, ws, splats->depth, sorted_ids, ranges, k64, kinfo, s);
    default: return walk<4>(L, ws, splats->depth, sorted_ids, ranges, k64, kinfo, s);
  }
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
  gs::Layout L;
  st = gs::layout(n, width, height, k_capacity, &L);
  if (st != GS_OK) return st;
  *bytes = L.bytes;
  return GS_OK;
}

extern "C" int gs_bin_and_sort_async(const gs_splats_t* splats, int32_t width, int32_t height, void* workspace,
                                     size_t workspace_bytes, int64_t k_capacity, uint32_t* sorted_ids,
                                     int32_t* ranges, uint64_t* keys, int64_t* k_info, void* stream) {
  using namespace gs;
  if (!splats || !k_info || k_capacity < 0) return GS_ERR_INVALID_ARG;
  int st = check_dims(width, height);
  if (st != GS_OK) return st;
  return bin_enqueue(splats, width, height, workspace, workspace_bytes, k_capacity, sorted_ids, ranges, keys, k_info,
                     static_cast<cudaStream_t>(stream));
}

extern "C" int gs_bin_and_sort(const gs_splats_t* splats, int32_t width, int32_t height, void* workspace,
                               size_t workspace_bytes, int64_t k_capacity, uint32_t* sorted_ids, int32_t* ranges,
                               uint64_t* keys, int64_t* k_out, void* stream) {
  using namespace gs;
  if (!splats || !k_out || k_capacity < 0) return GS_ERR_INVALID_ARG;
  int st = check_dims(width, height);
  if (st != GS_OK) return st;
  *k_out = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Layout L;
  st = layout(splats->n, width, height, k_capacity, &L);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  int64_t* kinfo = reinterpret_cast<int64_t*>(static_cast<char*>(workspace) + L.kinfo);
  // with no instance buffers only K is computed (capacity 0)
  const int64_t cap = (sorted_ids && ranges) ? k_capacity : 0;
  st = bin_enqueue(splats, width, height, workspace, workspace_bytes, cap, sorted_ids, ranges, keys, kinfo, s);
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
