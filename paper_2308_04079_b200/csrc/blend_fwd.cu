// K6 blend_fwd — replaces splatlab rasterizer.render_forward / _blend_tile
// (rasterizer.py:152-240).
//
// One CTA per 16x16 tile: 8 consumer warps (one pixel per thread, each warp
// an 8x4 pixel block) + 1 producer warp, warp-specialised over a ring of
// kStages shared-memory batch buffers guarded by mbarriers:
//   producer: for each kBatch-entry batch of the tile's sorted instance list,
//     loads the Gaussian ids, gathers the 48-byte splat records (words 0-2)
//     with cp.async, folds the tile origin into them and computes each
//     splat's 8-bit warp coverage mask
//     (warp_cover_mask) and arrives on full[stage];
//   consumers: wait on full[stage], visit (front to back, by ballot over the
//     mask bits) only the splats that can reach alpha >= 1/255 in their
//     block, then arrive on empty[stage].
// Warps therefore drift apart by up to kStages-1 batches instead of meeting
// at a CTA barrier after every batch (the v1 kernel's dominant stall).
// A pixel stops before its accumulated opacity would exceed 0.9999
// (rasterizer.py:179-180); in training mode a pixel whose float32 T_new is
// too close to the threshold to decide (kSatGuard) is re-blended in float64
// by the tile's consumer warps after the blend (exact_pixel: the
// reference's stop, T_final and last contributor).  Once every consumer
// warp is done the CTA stops
// (rasterizer.py:194-195): the last warp to finish raises s_stop, which the
// producer and any waiting consumer poll.  gs_blend_forward_ordered launches
// the tiles in a given order (heaviest first) and can record each tile's work.
#include "gs_common.cuh"

namespace gs {
namespace {

#ifndef GS_FWD_EXACT
#define GS_FWD_EXACT 0   // exact ellipse-vs-block masks (see warp_cover_mask)
#endif
#ifndef GS_FWD_BATCH
#define GS_FWD_BATCH 32
#endif
#ifndef GS_FWD_STAGES
#define GS_FWD_STAGES 12
#endif
constexpr int kBatch = GS_FWD_BATCH;
constexpr int kStages = GS_FWD_STAGES;
#ifndef GS_FWD_PARTS
#define GS_FWD_PARTS 1   // CTAs per tile: 2 = one CTA per 16x8 half tile (4 consumer warps)
#endif
constexpr int kParts = GS_FWD_PARTS;
constexpr int kConsumerWarps = 8 / kParts;
#ifndef GS_FWD_PRODUCERS
#define GS_FWD_PRODUCERS 1   // producer warps; producer p fills batches p, p + P, ... (kStages % P == 0)
#endif
constexpr int kProducers = GS_FWD_PRODUCERS;
constexpr int kThreads = (kConsumerWarps + kProducers) * 32;

#ifndef GS_FWD_TMA
#define GS_FWD_TMA 0     // 1: the producer gathers the records with TMA tile::gather4 (see produce_batch_tma)
#endif

#if GS_FWD_TMA
// TMA variant: record words 0-3 of each splat land as one 64-byte row
// (rec4[4 e + w] = word w of splat e), four splats per gather4 (256 B)
struct alignas(128) FwdStage {
  float4 rec4[4 * kBatch];
  float4 m[kBatch];      // (-k1 . mean_rel, -k2 . mean_rel, alpha, 0)
  uint32_t id[kBatch];
  uint8_t mask[kBatch];
};
__device__ __forceinline__ float4 stage_k(const FwdStage& st, int j) { return st.rec4[4 * j + 1]; }
__device__ __forceinline__ float4 stage_col(const FwdStage& st, int j) { return st.rec4[4 * j + 2]; }
struct RawRec {};
constexpr size_t kSmemBytes = sizeof(FwdStage) * kStages + 128;   // + alignment slack
#else
struct FwdStage {
  float4 k[kBatch];      // eigenbasis rows (record word 1), see make_tile_splat
  float4 m[kBatch];      // (-k1 . mean_rel, -k2 . mean_rel, alpha, 0)
  float4 col[kBatch];
  uint32_t id[kBatch];
  uint8_t mask[kBatch];
};
__device__ __forceinline__ float4 stage_k(const FwdStage& st, int j) { return st.k[j]; }
__device__ __forceinline__ float4 stage_col(const FwdStage& st, int j) { return st.col[j]; }
struct RawRec {          // the producer's landing buffer for the cp.async gathers
  float4 r0[kBatch];
};
constexpr size_t kSmemBytes = sizeof(FwdStage) * kStages + sizeof(RawRec) * kProducers;
#endif

#if GS_FWD_TMA
// TMA producer: lane l < ceil(cnt / 4) issues one tile::gather4 of splats
// 4l..4l+3 (record rows of the 2-D tensor map over rec: 20 floats x N, box
// 16 x 1), completing on the stage's tma mbarrier; the rows past cnt repeat
// the last id (never read).  Then the tile-relative record and coverage mask.
__device__ __forceinline__ void produce_batch_tma(FwdStage& st, uint64_t* tma_bar, uint32_t parity,
                                                  const CUtensorMap* tmap, const float4* __restrict__ rec,
                                                  const uint32_t* __restrict__ ids, int base, int cnt, int lane,
                                                  float tile_x0, float tile_y0, int mask_shift) {
  static_assert(kBatch == 32, "one id per lane");
  const uint32_t gid = __ldg(ids + base + min(lane, cnt - 1));
  if (lane < cnt) st.id[lane] = gid;
  const int ng = (cnt + 3) >> 2;
  const int r0 = __shfl_sync(0xffffffffu, int(gid), (4 * lane + 0) & 31);
  const int r1 = __shfl_sync(0xffffffffu, int(gid), (4 * lane + 1) & 31);
  const int r2 = __shfl_sync(0xffffffffu, int(gid), (4 * lane + 2) & 31);
  const int r3 = __shfl_sync(0xffffffffu, int(gid), (4 * lane + 3) & 31);
  if (lane == 0) mbar_arrive_expect_tx(tma_bar, uint32_t(ng) * 256u);
  __syncwarp();
  if (lane < ng) tma_gather4(&st.rec4[16 * lane], tmap, tma_bar, 0, r0, r1, r2, r3);
  while (!mbar_try_wait(tma_bar, parity)) {
  }
  if (lane < cnt) {
    const float4 w0 = st.rec4[4 * lane], k = st.rec4[4 * lane + 1];
    const float alpha = st.rec4[4 * lane + 2].w;
    float2 ctr;
    make_tile_splat(w0, k, alpha, tile_x0, tile_y0, st.m[lane], ctr);
    st.mask[lane] = uint8_t(warp_cover_mask<GS_FWD_EXACT != 0>(w0, k, alpha, tile_x0, tile_y0) >> mask_shift);
  }
}
#endif

#if !GS_FWD_TMA
__device__ __forceinline__ void produce_batch(FwdStage& st, RawRec& raw, const float4* __restrict__ rec,
                                              const uint32_t* __restrict__ ids, int base, int cnt, int lane,
                                              float tile_x0, float tile_y0, int mask_shift) {
  uint32_t gid[kBatch / 32];
#pragma unroll
  for (int u = 0; u < kBatch / 32; ++u) {
    const int e = lane + 32 * u;
    gid[u] = e < cnt ? __ldg(ids + base + e) : 0u;
  }
#pragma unroll
  for (int u = 0; u < kBatch / 32; ++u) {
    const int e = lane + 32 * u;
    if (e < cnt) {
      const float4* src = rec + kRecWords * size_t(gid[u]);
      st.id[e] = gid[u];
      cp_async16(&raw.r0[e], src + 0);
      cp_async16(&st.k[e], src + 1);
      cp_async16(&st.col[e], src + 2);
    }
  }
  cp_async_wait_all();
#pragma unroll
  for (int u = 0; u < kBatch / 32; ++u) {
    const int e = lane + 32 * u;
    if (e < cnt) {
      const float4 r0 = raw.r0[e], k = st.k[e];
      const float alpha = st.col[e].w;
      float2 ctr;
      make_tile_splat(r0, k, alpha, tile_x0, tile_y0, st.m[e], ctr);
      // kParts = 2: only the half tile's blocks (mask_shift = part * 4 rows of 4 px)
      st.mask[e] = kParts == 1
                       ? uint8_t(warp_cover_mask<GS_FWD_EXACT != 0>(r0, k, alpha, tile_x0, tile_y0))
                       : uint8_t(warp_cover_mask<GS_FWD_EXACT != 0, 4, kConsumerWarps / 2>(
                             r0, k, alpha, tile_x0, tile_y0 + float(mask_shift / kConsumerWarps * (kTile / kParts))));
    }
  }
}
#endif

// ---------------------------------------------------------------------------
// Exact float64 re-blend of a flagged pixel (training).  The forward appends
// every pixel whose stop float32 cannot decide (kSatGuard) to a list and
// stores its float32 last contributor L as last = -3 - L; blend_exact_kernel
// then re-blends each listed pixel with a whole CTA.  Every candidate up to
// L was accepted with float32 T_new >= thr (1 + kSatGuard), hence with exact
// T_new >= thr: those are included exactly when their float64 alpha is > 0
// (rasterizer.py:171-180; the 1/255 and 0.99 decisions are already the
// reference's).  Their product and colour are block prefix products over the
// list prefix; then the candidates after L are visited in order until the
// exact stop (1 - T_new > 0.9999), as the reference's sequential rule.
#ifndef GS_FIX_CTAS_PER_SM
#define GS_FIX_CTAS_PER_SM 6
#endif
constexpr int kFixThreads = 256, kFixItems = 2, kFixPass = kFixThreads * kFixItems;

struct FixShared {
  double wscan[kFixThreads / 32];
  double total;
  double col[3][kFixThreads / 32];
  double tail_a[kFixThreads];
  float4 tail_c[kFixThreads];   // the candidates' colours (the serial walk reads them)
  int stop;
  int item;
};

__device__ __forceinline__ void consumer_sync() { __syncthreads(); }

// float64 alpha of one list entry at pixel centre (fx, fy), reference
// arithmetic (rasterizer.py:171-177); a cheap float32 exclusion skips the
// exp for entries whose exponent is far below log2(1/255)
__device__ __forceinline__ double exact_alpha(const float4* __restrict__ rec, uint32_t id, double fx, double fy,
                                              float4& col) {
  const float4* r = rec + kRecWords * size_t(id);
  const float4 r0 = r[0], k = r[1];
  const float mx = float(fx - double(r0.x)) - r0.z, my = float(fy - double(r0.y)) - r0.w;
  const float v1 = fmaf(k.x, mx, k.y * my), v2 = fmaf(k.z, mx, k.w * my);
  if (-(v1 * v1 + v2 * v2) < -8.004f) return 0.0;   // log2(e) power < log2(1/255) - 0.01
  const float4 r3 = r[3], r4 = r[4];
  col = r[2];
  const double dx = fx - (double(r0.x) + double(r0.z));
  const double dy = fy - (double(r0.y) + double(r0.w));
  const double ca = double(r3.x) + double(r4.x), cb = double(r3.y) + double(r4.y);
  const double cc = double(r3.z) + double(r4.z), al = double(col.w) + double(r4.w);
  const double power = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy;
  const double g = power > 0.0 ? 0.0 : exp(power);
  const double a = fmin(0.99, al * g);   // ALPHA_CLAMP
  return a < 1.0 / 255.0 ? 0.0 : a;      // ALPHA_EPS
}

// exclusive product of v over the consumer threads; *total = the product
__device__ __forceinline__ double consumer_exclusive_product(double v, FixShared& sh, double* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl *= t;
  }
  if (lane == 31) sh.wscan[warp] = incl;
  consumer_sync();
  if (threadIdx.x == 0) {
    double run = 1.0;
    for (int w = 0; w < kFixThreads / 32; ++w) {
      const double x = sh.wscan[w];
      sh.wscan[w] = run;
      run *= x;
    }
    sh.total = run;
  }
  consumer_sync();
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  excl = (lane == 0 ? 1.0 : excl) * sh.wscan[warp];
  *total = sh.total;
  consumer_sync();
  return excl;
}

__device__ void exact_pixel(const float4* __restrict__ rec, const uint32_t* __restrict__ ids, int2 range, int px,
                            int py, int last_f32, int width, float3 bg, float* __restrict__ image,
                            float* __restrict__ t_final, int32_t* __restrict__ last, FixShared& sh) {
  const double fx = double(px) + 0.5, fy = double(py) + 0.5;   // rasterizer.py:142
  double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
  // 1. the accepted prefix [range.x, last_f32]
  for (int base = range.x; base <= last_f32; base += kFixPass) {
    double a[kFixItems];
    float4 col[kFixItems];
    const int i0 = base + int(threadIdx.x) * kFixItems;
    double local = 1.0;
#pragma unroll
    for (int u = 0; u < kFixItems; ++u) {
      col[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      a[u] = i0 + u <= last_f32 ? exact_alpha(rec, ids[i0 + u], fx, fy, col[u]) : 0.0;
      local *= 1.0 - a[u];
    }
    double pass;
    double tb = T * consumer_exclusive_product(local, sh, &pass);
#pragma unroll
    for (int u = 0; u < kFixItems; ++u) {
      const double w = tb * a[u];
      cr += w * col[u].x;
      cg += w * col[u].y;
      cb += w * col[u].z;
      tb *= 1.0 - a[u];
    }
    T *= pass;
  }
  // colour sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cr += __shfl_xor_sync(0xffffffffu, cr, o);
    cg += __shfl_xor_sync(0xffffffffu, cg, o);
    cb += __shfl_xor_sync(0xffffffffu, cb, o);
  }
  if (lane == 0) {
    sh.col[0][warp] = cr;
    sh.col[1][warp] = cg;
    sh.col[2][warp] = cb;
  }
  if (threadIdx.x == 0) sh.stop = 0;
  consumer_sync();
  // 2. the candidates after it, in order, until the exact stop (thread 0
  //    walks each batch's alphas; the float32 stop candidate is the first)
  double c[3] = {0.0, 0.0, 0.0};
  if (threadIdx.x == 0)
    for (int w = 0; w < kFixThreads / 32; ++w)
      for (int k = 0; k < 3; ++k) c[k] += sh.col[k][w];
  int lst = last_f32;
  for (int base = last_f32 + 1; base < range.y; base += kFixThreads) {
    const int i = base + int(threadIdx.x);
    float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
    sh.tail_a[threadIdx.x] = i < range.y ? exact_alpha(rec, ids[i], fx, fy, col) : 0.0;
    sh.tail_c[threadIdx.x] = col;
    consumer_sync();
    if (threadIdx.x == 0) {
      for (int u = 0; u < kFixThreads && base + u < range.y; ++u) {
        const double a = sh.tail_a[u];
        if (a <= 0.0) continue;
        const double t_new = T * (1.0 - a);
        if ((1.0 - t_new) > 0.9999) {   // SATURATION
          sh.stop = 1;
          break;
        }
        const float4 cc = sh.tail_c[u];
        c[0] += T * a * cc.x;
        c[1] += T * a * cc.y;
        c[2] += T * a * cc.z;
        T = t_new;
        lst = base + u;
      }
    }
    consumer_sync();
    if (sh.stop) break;
  }
  if (threadIdx.x == 0) {
    const size_t p = size_t(py) * width + px;
    image[3 * p + 0] = float(c[0] + T * double(bg.x));   // rasterizer.py:197
    image[3 * p + 1] = float(c[1] + T * double(bg.y));
    image[3 * p + 2] = float(c[2] + T * double(bg.z));
    t_final[p] = float(T);
    last[p] = lst;
  }
  consumer_sync();
}

// Persistent CTAs take the listed pixels one at a time (fix[0] = count,
// fix[1] = work counter, fix[2 + i] = pixel index).
__global__ void __launch_bounds__(kFixThreads, GS_FIX_CTAS_PER_SM) blend_exact_kernel(const float4* __restrict__ rec,
                                                                 const uint32_t* __restrict__ ids,
                                                                 const int2* __restrict__ ranges, int width,
                                                                 int tiles_x, float3 bg, float* __restrict__ image,
                                                                 float* __restrict__ t_final,
                                                                 int32_t* __restrict__ last, int32_t* fix) {
  pdl_begin();
  __shared__ FixShared sh;
  const int count = *reinterpret_cast<volatile int32_t*>(fix);
  for (;;) {
    if (threadIdx.x == 0) sh.item = atomicAdd(fix + 1, 1);
    __syncthreads();
    const int item = sh.item;
    __syncthreads();
    if (item >= count) return;
    const int64_t q = fix[2 + item];
    const int px = int(q % width), py = int(q / width);
    exact_pixel(rec, ids, ranges[(py / kTile) * tiles_x + px / kTile], px, py, -3 - last[q], width, bg, image,
                t_final, last, sh);
  }
}

#ifdef GS_FWD_MIN_BLOCKS
#define GS_FWD_LB __launch_bounds__(kThreads, GS_FWD_MIN_BLOCKS)
#else
#define GS_FWD_LB __launch_bounds__(kThreads)
#endif
template <bool kTraining>
__global__ void GS_FWD_LB
blend_fwd_kernel(const float4* __restrict__ rec, const uint32_t* __restrict__ ids, const int2* __restrict__ ranges,
                 int width, int height, int tiles_x, int tile0, float3 bg, float* __restrict__ image,
                 float* __restrict__ t_final, int32_t* __restrict__ last, const int32_t* __restrict__ tile_order,
                 int32_t* __restrict__ tile_work, int32_t* __restrict__ fix, const __grid_constant__ CUtensorMap tmap) {
  pdl_begin();
  extern __shared__ __align__(128) unsigned char smem_raw[];
#if GS_FWD_TMA
  FwdStage* stages = reinterpret_cast<FwdStage*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  RawRec* raw = nullptr;
  __shared__ uint64_t tma_bar[kStages];
#else
  FwdStage* stages = reinterpret_cast<FwdStage*>(smem_raw);
  RawRec* raw = reinterpret_cast<RawRec*>(smem_raw + sizeof(FwdStage) * kStages);
#endif
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ int s_done, s_stop, s_work;
  static_assert(kStages % kProducers == 0, "every stage must have a single producer");

  const int tile = tile_order ? tile_order[int(blockIdx.x) / kParts] : tile0 + int(blockIdx.x) / kParts;
  const int part = int(blockIdx.x) % kParts;   // this CTA's rows: [part * 16 / kParts, (part + 1) * 16 / kParts)
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const float tile_x0 = float(tx * kTile), tile_y0 = float(ty * kTile);
  const int2 range = ranges[tile];
  const int nb = (range.y - range.x + kBatch - 1) / kBatch;

  if (t == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 32);
      mbar_init(&empty_bar[s], kConsumerWarps);
#if GS_FWD_TMA
      mbar_init(&tma_bar[s], 1);
#endif
    }
    s_done = 0;
    s_stop = 0;
    s_work = 0;
#if GS_FWD_TMA
    fence_mbarrier_init();
#endif
  }
  __syncthreads();

  if (warp >= kConsumerWarps) {  // ---------------- producer warp(s)
    const int prod = warp - kConsumerWarps;
    int b = prod;
    for (; b < nb; b += kProducers) {
      const int s = b % kStages;
      bool stop = false;
      if (b >= kStages) {
        while (!mbar_try_wait(&empty_bar[s], uint32_t((b / kStages) - 1) & 1u))
          if (ld_volatile(&s_stop)) {
            stop = true;
            break;
          }
      }
      if (stop || ld_volatile(&s_stop)) break;
      const int base = range.x + b * kBatch;
#if GS_FWD_TMA
      (void)raw;
      produce_batch_tma(stages[s], &tma_bar[s], uint32_t(b / kStages) & 1u, &tmap, rec, ids, base,
                        min(kBatch, range.y - base), lane, tile_x0, tile_y0, part * kConsumerWarps);
#else
      produce_batch(stages[s], raw[prod], rec, ids, base, min(kBatch, range.y - base), lane, tile_x0, tile_y0,
                    part * kConsumerWarps);
#endif
      mbar_arrive(&full_bar[s]);
    }
    // the tile's work (splats handed to the consumers) for the next frame's schedule
    if (kProducers == 1) {
      if (tile_work && lane == 0) tile_work[tile] = b * kBatch;
    } else if (tile_work) {
      if (lane == 0) atomicMax(&s_work, b - kProducers + 1);   // batches handed, up to the producers' stagger
      asm volatile("bar.sync 1, %0;" ::"r"(kProducers * 32) : "memory");
      if (prod == 0 && lane == 0) tile_work[tile] = min(s_work, nb) * kBatch;
    }
    return;
  }

  // ---------------- consumer warps
  const int px = tx * kTile + tile_px(t);
  const int py = ty * kTile + tile_py(t) + part * (kTile / kParts);
  const bool inside = (px < width) && (py < height);
  const float fx = float(px) + 0.5f, fy = float(py) + 0.5f;  // rasterizer.py:142
  const float lx = float(tile_px(t)) + 0.5f, ly = float(tile_py(t) + part * (kTile / kParts)) + 0.5f;
  float T = 1.0f;
  float cr = 0.0f, cg = 0.0f, cb = 0.0f;
  int32_t last_idx = -1;
  float t_stop = 0.0f;    // T_new of the splat the pixel stopped before (training: kSatGuard check)
  bool done = !inside;
  bool warp_done = __all_sync(0xffffffffu, done);
  if (warp_done && lane == 0 && atomicAdd(&s_done, 1) == kConsumerWarps - 1) s_stop = 1;

  for (int b = 0; b < nb; ++b) {
    const int s = b % kStages;
    bool stop = false;
    while (!mbar_try_wait(&full_bar[s], uint32_t(b / kStages) & 1u)) {
      if (ld_volatile(&s_stop)) {
        stop = true;
        break;
      }
    }
    if (__any_sync(0xffffffffu, stop)) break;
    if (!warp_done) {
      const FwdStage& st = stages[s];
      const int base = range.x + b * kBatch;
      const int cnt = min(kBatch, range.y - base);
      for (int c0 = 0; c0 < cnt; c0 += 32) {
        const int jl = c0 + lane;
        unsigned live = __ballot_sync(0xffffffffu, jl < cnt && ((st.mask[jl] >> warp) & 1u));
        while (live) {
          const int j = c0 + __ffs(live) - 1;
          live &= live - 1;
          // branch-light body: finished lanes evaluate too (free under SIMT)
          // and are masked by `take`
          const AlphaEval e = eval_alpha_tile(lx, ly, fx, fy, stage_k(st, j), st.m[j], rec, st.id, j);
          const float t_new = T * (1.0f - e.a);   // used only when blended
          const bool blend = !done && e.ok;
          const bool sat = t_new < (kTraining ? kTransSatHi : kTransSat);  // 1 - T_new > 0.9999
          const bool stopping = blend && sat;
          done = done || stopping;
          if (kTraining) t_stop = stopping ? t_new : t_stop;
          if (blend && !sat) {
            const float4 c = stage_col(st, j);
            const float w = T * e.a;
            cr = fmaf(w, c.x, cr);
            cg = fmaf(w, c.y, cg);
            cb = fmaf(w, c.z, cb);
            T = t_new;
            if (kTraining) last_idx = base + j;
          }
        }
        if (__all_sync(0xffffffffu, done)) break;
      }
      if (__all_sync(0xffffffffu, done)) {
        warp_done = true;
        if (lane == 0 && atomicAdd(&s_done, 1) == kConsumerWarps - 1) s_stop = 1;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }

  if (!inside) return;
  const size_t p = size_t(py) * width + px;
  image[3 * p + 0] = fmaf(T, bg.x, cr);  // rasterizer.py:197
  image[3 * p + 1] = fmaf(T, bg.y, cg);
  image[3 * p + 2] = fmaf(T, bg.z, cb);
  if (kTraining) {
    t_final[p] = T;
    if (t_stop >= kTransSatLo) {   // the stop is undecidable in float32: list it for blend_exact_kernel
      last[p] = -3 - last_idx;
      fix[2 + atomicAdd(fix, 1)] = int32_t(p);
    } else {
      last[p] = last_idx;
    }
  }
}

template <bool kTraining>
int launch(const int32_t* order, int32_t* work, const float4* rec, int64_t n, const uint32_t* ids, const int2* rg,
           int width, int height, int tiles_x, int tile0,
           int64_t ntiles, float3 bg, float* image, float* t_final, int32_t* last, int32_t* fix, cudaStream_t s) {
  CUtensorMap tmap{};
#if GS_FWD_TMA
  {   // 2-D map over the records: 20 floats x n rows (80-byte stride), box 16 x 1 (words 0-3)
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return GS_ERR_CUDA;
      encode = reinterpret_cast<EncodeFn>(fn);
    }
    const cuuint64_t dims[2] = {cuuint64_t(kRecWords * 4), cuuint64_t(n > 0 ? n : 1)};
    const cuuint64_t strides[1] = {cuuint64_t(kRecWords * 16)};
    const cuuint32_t box[2] = {16, 1}, estr[2] = {1, 1};
    if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float4*>(rec), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return GS_ERR_CUDA;
  }
#else
  (void)n;
#endif
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(blend_fwd_kernel<kTraining>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kSmemBytes));
    if (e != cudaSuccess) return record_cuda_error(e);
    configured = true;
  }
  if (ntiles <= 0) return GS_OK;
  if (kTraining) {
    cudaError_t e = zero_async(fix, 2 * sizeof(int32_t), nullptr, 0, s);
    if (e != cudaSuccess) return record_cuda_error(e);
  }
  launch_pdl(blend_fwd_kernel<kTraining>, unsigned(ntiles * kParts), kThreads, kSmemBytes, s, rec, ids, rg, width, height, tiles_x,
                                                                             tile0, bg, image, t_final, last,
                                                                             order, work, fix, tmap);
  int st = check_launch();
  if (st != GS_OK || !kTraining) return st;
  launch_pdl(blend_exact_kernel, 148 * GS_FIX_CTAS_PER_SM, kFixThreads, 0, s, rec, ids, rg, width, tiles_x, bg, image, t_final, last, fix);
  return check_launch();
}

int blend_forward_rows(const gs_splats_t* splats, const uint32_t* sorted_ids, const int32_t* ranges, int32_t width,
                       int32_t height, int32_t row_begin, int32_t row_end, const float background[3],
                       int32_t training, float* image, float* t_final, int32_t* last, int32_t* scratch, void* stream,
                       const int32_t* tile_order = nullptr, int32_t* tile_work = nullptr) {
  if (!splats || !ranges || !image || !background || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  if (training && (!t_final || !last || !scratch)) return GS_ERR_INVALID_ARG;
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * tiles_y;
  if (tiles > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  if (row_begin < 0 || row_end > tiles_y || row_begin > row_end) return GS_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float3 bg = make_float3(background[0], background[1], background[2]);
  const float4* rec = reinterpret_cast<const float4*>(splats->rec);
  const int2* rg = reinterpret_cast<const int2*>(ranges);
  const int tile0 = row_begin * tiles_x;
  const int64_t ntiles = int64_t(row_end - row_begin) * tiles_x;
  if (training)
    return launch<true>(tile_order, tile_work, rec, splats->n, sorted_ids, rg, width, height, tiles_x, tile0, ntiles, bg, image,
                        t_final, last, scratch, s);
  return launch<false>(tile_order, tile_work, rec, splats->n, sorted_ids, rg, width, height, tiles_x, tile0, ntiles, bg, image,
                       nullptr, nullptr, nullptr, s);
}

}  // namespace
}  // namespace gs

extern "C" int gs_blend_forward(const gs_splats_t* splats, const uint32_t* sorted_ids, const int32_t* ranges,
                                int32_t width, int32_t height, const float background[3], int32_t training,
                                float* image, float* t_final, int32_t* last, int32_t* scratch, void* stream) {
  if (width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  return gs::blend_forward_rows(splats, sorted_ids, ranges, width, height, 0, (height + gs::kTile - 1) / gs::kTile,
                                background, training, image, t_final, last, scratch, stream);
}

// The full frame with the tiles visited in `tile_order` (a permutation of
// [0, tiles), device int32).
extern "C" int gs_blend_forward_ordered(const gs_splats_t* splats, const uint32_t* sorted_ids, const int32_t* ranges,
                                        int32_t width, int32_t height, const float background[3], int32_t training,
                                        const int32_t* tile_order, int32_t* tile_work, float* image, float* t_final,
                                        int32_t* last, int32_t* scratch, void* stream) {
  if (height <= 0) return GS_ERR_INVALID_ARG;
  return gs::blend_forward_rows(splats, sorted_ids, ranges, width, height, 0, (height + gs::kTile - 1) / gs::kTile,
                                background, training, image, t_final, last, scratch, stream, tile_order, tile_work);
}
