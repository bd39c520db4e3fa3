// K7 blend_bwd — replaces splatlab rasterizer.render_backward
// (rasterizer.py:253-316) and gradients.backward_blend (gradients.py:30-94).
//
// One CTA per 16x8 half tile (GS_BWD_PARTS = 2): 4 consumer warps (8x4
// pixel blocks) + 1 producer warp over a kStages-deep ring of shared-memory
// batches with mbarriers, like the forward; the two halves of a tile run as
// independent CTAs (less warp drift per ring, overlapping start-ups), and
// gs_blend_backward_scheduled launches the tiles heaviest first.
// Each CTA walks its list back to front from the largest last contributor
// of its pixels (gradients.py:48-52), re-evaluating alpha with the forward's
// exact code so the contributor sets coincide.  Each pixel rebuilds T_before
// by dividing out (1 - a) (gradients.py:67-70) and carries the composited
// tail (gradients.py:75-78) as a running sum.
//
// Reduction: a warp processes the splats of its coverage mask in pairs; the
// 2 x 9 per-lane partial gradients are summed across the warp by a
// transposed (reduce-scatter) butterfly — 22 shuffles per pair instead of
// 2 x 45 — leaving each of 8 lane pairs one summed component, which goes
// straight to global memory as a fire-and-forget float reduction (RED) into
// the splat's screen-gradient row: L2 absorbs them (measured 1.39 ms vs
// 1.45 ms for shared-memory CAS accumulators flushed per (splat, tile)).
// The terms' constant factors are applied once per reduced value.
//
// Conic gradient in the conic's eigenbasis: instead of d_conic (a, b, c) =
// -1/2 sum dL/dpower (dx^2, 2 dx dy, dy^2) (gradients.py:90-93) the kernel
// accumulates the moments M = sum dL/dpower (v1^2, v1 v2, v2^2) of the
// eigenbasis offsets v = K d the exponent is built from (log2(e) power =
// -|v|^2).  For an elongated conic the x/y sums are dominated by the long
// axis and carry the short axis' component only to float32 rounding of the
// large one, which d Sigma' = -A G A then multiplies by cond(A); the moments
// keep each axis at its own relative precision.  The projection backward
// forms d Sigma' = 2 / log2(e)^2 K^T M K in float64 (preprocess_bwd.cu);
// SplatGrads2D.d_conic converts M back to the reference's d_conic.
// coverage masks: box + eigen-metric ball + the directional separating-axis
// test (GS_COVER_BALL 2, gs_common.cuh): 0.980 vs 0.991 ms here; the
// forward keeps 1 (its single producer warp: 0.664 vs 0.569 ms with 2)
#ifndef GS_COVER_BALL
#define GS_COVER_BALL 2
#endif
#include "gs_common.cuh"

namespace gs {
namespace {

#ifndef GS_WAIT_NS
#define GS_WAIT_NS 2000
#endif
#ifndef GS_BWD_MIN_BLOCKS
#define GS_BWD_MIN_BLOCKS 7  // half-tile CTAs: <= 56 registers (no spills), 7 CTAs (35 warps) per SM: 0.926 -> 0.907 ms (8: spills, 0.944)
#endif
#ifndef GS_BWD_EXACT_MASK
#define GS_BWD_EXACT_MASK 0   // 1: exact ellipse-vs-block masks (slower since the ball test: 1.031 vs 0.994 ms)
#endif
#ifndef GS_BWD_BATCH
#define GS_BWD_BATCH 64
#endif
constexpr int kBatch = GS_BWD_BATCH;
#ifndef GS_BWD_STAGES
#define GS_BWD_STAGES 4
#endif
constexpr int kStages = GS_BWD_STAGES;
#ifndef GS_BWD_PARTS
#define GS_BWD_PARTS 2   // CTAs per tile: 2 = one CTA per 16x8 half tile (4 consumer warps)
#endif
constexpr int kParts = GS_BWD_PARTS;
constexpr int kConsumerWarps = 8 / kParts;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kG = 2;    // splats per reduction group (group_reduce2)
constexpr int kC = 9;    // gradient components per splat

#ifndef GS_BWD_STATS
#define GS_BWD_STATS 0
#endif
#if GS_BWD_STATS
__device__ unsigned long long g_bwd_hist[33];   // visited (warp, splat) pairs by active-lane count
#endif

struct BwdStage {
  float4 k[kBatch];      // eigenbasis rows (record word 1), see make_tile_splat
  float4 m[kBatch];      // (-k1 . mean_rel, -k2 . mean_rel, alpha, 0)
  float4 col[kBatch];
  uint32_t id[kBatch];
  uint8_t mask[kBatch];
};
struct RawRec {          // the producer's landing buffer for the cp.async gathers
  float4 r0[kBatch];
};
constexpr size_t kSmemBytes = sizeof(BwdStage) * kStages + sizeof(RawRec);
// deterministic mode: per stage, each consumer warp's reduced partials
// [warp][slot][component], combined by the producer in warp order
struct DetPart {
  float v[kConsumerWarps][kBatch][kC];
};
constexpr size_t kSmemBytesDet = kSmemBytes + sizeof(DetPart) * kStages;

// deterministic mode: the producer sums the released stage's warp partials
// in warp order into the per-instance rows part_out[pos][tile part][kC]
// (one row per (sorted instance, half tile)), and clears them.
__device__ __forceinline__ void det_flush(DetPart& dp, int lo, int cnt, int part, float* __restrict__ part_out,
                                          int lane) {
  for (int e = lane; e < cnt; e += 32) {
    float* row = part_out + (size_t(lo + e) * kParts + part) * kC;
#pragma unroll
    for (int c = 0; c < kC; ++c) {
      float acc = 0.0f;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        acc += dp.v[w][e][c];
        dp.v[w][e][c] = 0.0f;
      }
      row[c] = acc;
    }
  }
}

// Two-splat variant: sum v[0..17] over the warp.  On return lane l holds, in
// `out`, component ((l >> 1) & 7) of splat (l >> 4) (lanes l and l^1 hold the
// same value) and `out8` holds component 8 of splat (l >> 4).
// 37 instructions per splat with 18 live floats.
__device__ __forceinline__ void group_reduce2(float (&v)[2 * kC], int lane, float& out, float& out8) {
  const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
  float x[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const float send = b16 ? v[i] : v[i + 9];
    const float keep = b16 ? v[i + 9] : v[i];
    x[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float c8 = x[8];
  c8 += __shfl_xor_sync(0xffffffffu, c8, 8);
  c8 += __shfl_xor_sync(0xffffffffu, c8, 4);
  c8 += __shfl_xor_sync(0xffffffffu, c8, 2);
  c8 += __shfl_xor_sync(0xffffffffu, c8, 1);
  out8 = c8;
  float y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b8 ? x[i] : x[i + 4];
    const float keep = b8 ? x[i + 4] : x[i];
    y[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float z[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b4 ? y[i] : y[i + 2];
    const float keep = b4 ? y[i + 2] : y[i];
    z[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  const float send = b2 ? z[0] : z[1];
  float w = (b2 ? z[1] : z[0]) + __shfl_xor_sync(0xffffffffu, send, 2);
  out = w + __shfl_xor_sync(0xffffffffu, w, 1);
}

// batch b covers sorted positions [lo, top) counted back from the tile's end
__device__ __forceinline__ void batch_bounds(int b, int tile_top, int range_lo, int& lo, int& cnt) {
  const int top = tile_top - b * kBatch;
  lo = max(range_lo, top - kBatch);
  cnt = top - lo;
}

// kDet: no float atomics; every (instance, half tile) gets its own partial
// row, summed in a fixed order per splat afterwards (det_reduce_kernel), so
// runs are bit-identical (the reference's deterministic=True,
// rasterizer.py:32-41).  top_out[tile * kParts + part] = the CTA's last
// processed sorted position + 1 (rows at or above it are never written).
template <bool kDet>
__global__ void __launch_bounds__(kThreads, kDet ? 3 : GS_BWD_MIN_BLOCKS)
blend_bwd_kernel(const float* __restrict__ d_image, const float4* __restrict__ rec, const uint32_t* __restrict__ ids,
                 const int2* __restrict__ ranges, const float* __restrict__ t_final, const int32_t* __restrict__ last,
                 int width, int height, int tiles_x, int tile0, float3 bg, float4* __restrict__ grads2d,
                 const int32_t* __restrict__ tile_order, float* __restrict__ part_out, int32_t* __restrict__ top_out) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BwdStage* stages = reinterpret_cast<BwdStage*>(smem_raw);
  RawRec* raw = reinterpret_cast<RawRec*>(smem_raw + sizeof(BwdStage) * kStages);
  DetPart* dparts = reinterpret_cast<DetPart*>(smem_raw + kSmemBytes);
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ int s_warp_max[kConsumerWarps + 1];

  // tile_order (optional): the launch visits tiles in this order (e.g. the
  // longest lists first, so the light tiles fill the last wave)
  const int tile = tile_order ? tile_order[int(blockIdx.x) / kParts] : tile0 + int(blockIdx.x) / kParts;
  const int part = int(blockIdx.x) % kParts;   // this CTA's rows: [part * 16 / kParts, (part + 1) * 16 / kParts)
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const bool consumer = warp < kConsumerWarps;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + tile_px(t);
  const int py = ty * kTile + tile_py(t) + part * (kTile / kParts);
  const bool inside = consumer && (px < width) && (py < height);
  const float fx = float(px) + 0.5f, fy = float(py) + 0.5f;
  const float lx = float(tile_px(t)) + 0.5f, ly = float(tile_py(t) + part * (kTile / kParts)) + 0.5f;
  const float tile_x0 = float(tx * kTile), tile_y0 = float(ty * kTile);
  const int2 range = ranges[tile];

  float T = 1.0f, dlx = 0.0f, dly = 0.0f, dlz = 0.0f;
  int32_t last_idx = -1;
  if (inside) {
    const size_t p = size_t(py) * width + px;
    T = t_final[p];
    last_idx = last[p];
    dlx = d_image[3 * p + 0];
    dly = d_image[3 * p + 1];
    dlz = d_image[3 * p + 2];
  }
  // a tile with an all-zero gradient contributes nothing (rasterizer.py:286-287)
  const bool nonzero = (dlx != 0.0f) || (dly != 0.0f) || (dlz != 0.0f);
  if (kDet && t == 0) top_out[tile * kParts + part] = range.x;   // nothing written (yet)
  if (!__syncthreads_or(nonzero)) return;
  // needed = max(last_local) + 1 (gradients.py:48-52)
  const int warp_last = __reduce_max_sync(0xffffffffu, last_idx);
  if (lane == 0) s_warp_max[warp] = warp_last;
  if (t == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 32);
      // deterministic mode: every consumer lane arrives (each releases its own
      // partial-row writes to the producer that combines them)
      mbar_init(&empty_bar[s], kDet ? kConsumerWarps * 32 : kConsumerWarps);
    }
  }
  __syncthreads();
  int tile_last = s_warp_max[0];
#pragma unroll
  for (int w = 1; w < kConsumerWarps; ++w) tile_last = max(tile_last, s_warp_max[w]);
  if (tile_last < range.x) return;
  const int tile_top = tile_last + 1;
  const int nb = (tile_top - range.x + kBatch - 1) / kBatch;
  if (kDet && t == 0) top_out[tile * kParts + part] = tile_top;

  if (!consumer) {  // ---------------- producer warp
    if (kDet)
      for (int i = lane; i < int(sizeof(DetPart) * kStages / sizeof(float)); i += 32)
        reinterpret_cast<float*>(dparts)[i] = 0.0f;
    for (int b = 0; b < nb; ++b) {
      const int s = b % kStages;
      if (b >= kStages) {
        while (!mbar_try_wait_sleep(&empty_bar[s], uint32_t((b / kStages) - 1) & 1u, GS_WAIT_NS)) {
        }
        if (kDet) {   // batch b - kStages is complete: its rows, in warp order
          int plo, pcnt;
          batch_bounds(b - kStages, tile_top, range.x, plo, pcnt);
          det_flush(dparts[s], plo, pcnt, part, part_out, lane);
          __syncwarp();
        }
      }
      {
        int lo, cnt;
        batch_bounds(b, tile_top, range.x, lo, cnt);
        BwdStage& st = stages[s];
        uint32_t gid[kBatch / 32];
#pragma unroll
        for (int u = 0; u < kBatch / 32; ++u) {
          const int e = lane + 32 * u;
          gid[u] = e < cnt ? __ldg(ids + lo + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kBatch / 32; ++u) {
          const int e = lane + 32 * u;
          if (e < cnt) {
            const float4* src = rec + kRecWords * size_t(gid[u]);
            st.id[e] = gid[u];
            cp_async16(&raw->r0[e], src + 0);
            cp_async16(&st.k[e], src + 1);
            cp_async16(&st.col[e], src + 2);
          }
        }
        cp_async_wait_all();
#pragma unroll
        for (int u = 0; u < kBatch / 32; ++u) {
          const int e = lane + 32 * u;
          if (e < cnt) {
            const float4 r0 = raw->r0[e], k = st.k[e];
            const float alpha = st.col[e].w;
            float2 ctr;
            make_tile_splat(r0, k, alpha, tile_x0, tile_y0, st.m[e], ctr);
            st.mask[e] = uint8_t(warp_cover_mask<GS_BWD_EXACT_MASK != 0, 4, kConsumerWarps / 2>(
                r0, k, alpha, tile_x0, tile_y0 + float(part * (kTile / kParts))));
          }
        }
        mbar_arrive(&full_bar[s]);
      }
    }
    if (kDet)   // the last kStages batches
      for (int b = max(nb - kStages, 0); b < nb; ++b) {
        const int s = b % kStages;
        while (!mbar_try_wait_sleep(&empty_bar[s], uint32_t(b / kStages) & 1u, GS_WAIT_NS)) {
        }
        int plo, pcnt;
        batch_bounds(b, tile_top, range.x, plo, pcnt);
        det_flush(dparts[s], plo, pcnt, part, part_out, lane);
      }
    return;
  }

  // ---------------- consumer warps
  // composited tail behind the current splat, starts at the background term
  float S = T * (dlx * bg.x + dly * bg.y + dlz * bg.z);
  for (int b = 0; b < nb; ++b) {
    const int s = b % kStages;
    while (!mbar_try_wait_sleep(&full_bar[s], uint32_t(b / kStages) & 1u, GS_WAIT_NS)) {
    }
    int lo, cnt;
    batch_bounds(b, tile_top, range.x, lo, cnt);
    BwdStage& st = stages[s];
    if (lo <= warp_last) {
      const int jmax = min(cnt - 1, warp_last - lo);
      // this lane takes batch slots j < lim (its last contributor and before);
      // padding slots of a short group carry j = -1, i.e. 0xffffffff unsigned
      const uint32_t lim = uint32_t(max(last_idx - lo + 1, 0));
      for (int c = jmax; c >= 0; c -= 32) {
        // lane l looks at splat c - 31 + l: the highest set bit is the
        // backmost remaining splat (one FLO per pick)
        const int jl = c - 31 + lane;
        unsigned live = __ballot_sync(0xffffffffu, jl >= 0 && ((st.mask[jl] >> warp) & 1u));
        while (live) {
          int js[kG];
#pragma unroll
          for (int u = 0; u < kG; ++u) {
            const int hb = 31 - __clz(live);   // -1 when empty
            js[u] = live ? c - 31 + hb : -1;
            live &= ~(1u << (hb & 31));
          }
          float v[kG * kC];
          bool any = false;
#pragma unroll
          for (int u = 0; u < kG; ++u) {
            const int j = max(js[u], 0);
            const float4 kk = st.k[j];
            const AlphaEval e = eval_alpha_tile(lx, ly, fx, fy, kk, st.m[j], rec, st.id, j);
            // branch-free body: lanes past their last contributor (or the
            // padding slots of a short group) evaluate with a = 0, which
            // leaves T and S unchanged and zeroes every gradient term
            const bool use = (uint32_t(js[u]) < lim) && e.ok;
            any |= use;
#if GS_BWD_STATS
            {
              const uint32_t bu = __ballot_sync(0xffffffffu, use);
              if (lane == 0 && js[u] >= 0) atomicAdd(&g_bwd_hist[__popc(bu)], 1ull);
            }
#endif
            const float a = use ? e.a : 0.0f;
            // 1 - a >= 0.01: MUFU reciprocal (~1 ulp), no IEEE/denormal sequence
            const float inv = rcp_approx(1.0f - a);
            T = use ? T * inv : T;  // transmittance just before this splat
            const float w = T * a;
            const float4 col = st.col[j];
            const float dc = col.x * dlx + col.y * dly + col.z * dlz;
            // clamped alphas pass no gradient (gradients.py:83-84)
            const float d_a = (use && e.live) ? T * dc - S * inv : 0.0f;  // gradients.py:81
            S = fmaf(w, dc, S);
            v[u * kC + 6] = w * dlx;
            v[u * kC + 7] = w * dly;
            v[u * kC + 8] = w * dlz;
            // dp = dL/d(log2(e) power) up to sign; the row holds its
            // eigenbasis moments sum dp (v1, v2, 1, v1^2, v1 v2, v2^2), from
            // which the projection backward forms d_mean2d = 2/log2(e) K^T
            // (sum dp v), d_alpha = sum dp / alpha and d_conic (see above)
            const float dp = d_a * e.a_raw;
            const float dpv1 = dp * e.v1, dpv2 = dp * e.v2;
            v[u * kC + 0] = dpv1;                                // S1
            v[u * kC + 1] = dpv2;                                // S2
            v[u * kC + 2] = dp;                                  // S0
            v[u * kC + 3] = dpv1 * e.v1;                         // conic moment M11
            v[u * kC + 4] = dpv1 * e.v2;                         // M12
            v[u * kC + 5] = dpv2 * e.v2;                         // M22
          }
          if (!__any_sync(0xffffffffu, any)) continue;
          float out, out8;
          group_reduce2(v, lane, out, out8);
          const int j = (lane & 16) ? js[1] : js[0];
          const int comp = (lane >> 1) & 7;
          if (j >= 0 && (lane & 1) == 0) {
            if (kDet) {   // this warp's partial, combined in warp order by the producer
              dparts[s].v[warp][j][comp] = out;
              if (comp == 0) dparts[s].v[warp][j][8] = out8;
            } else {
              // fire-and-forget reductions into the (N,12) screen-gradient rows
              float* row = reinterpret_cast<float*>(grads2d) + 12 * size_t(st.id[j]);
              atomicAdd(row + comp + comp / 3, out);
              if (comp == 0) atomicAdd(row + 10, out8);
            }
          }
        }
      }
    }
    __syncwarp();
    if (kDet || lane == 0) mbar_arrive(&empty_bar[s]);
  }
}

int blend_backward_rows(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                        const int32_t* ranges, const float* t_final, const int32_t* last, int32_t width,
                        int32_t height, int32_t row_begin, int32_t row_end, const float background[3],
                        float* grads2d, void* stream, const int32_t* tile_order = nullptr,
                        float* part_out = nullptr, int32_t* top_out = nullptr) {
  if (!d_image || !splats || !ranges || !t_final || !last || !grads2d || !background || width <= 0 ||
      height <= 0)
    return GS_ERR_INVALID_ARG;
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * tiles_y;
  if (tiles > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  if (row_begin < 0 || row_end > tiles_y || row_begin > row_end) return GS_ERR_INVALID_ARG;
  if (splats->n == 0 || row_begin == row_end) return GS_OK;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(blend_bwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kSmemBytes));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(blend_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kSmemBytesDet));
    if (e != cudaSuccess) return record_cuda_error(e);
    configured = true;
  }
  const float3 bg = make_float3(background[0], background[1], background[2]);
  const int64_t ntiles = int64_t(row_end - row_begin) * tiles_x;
  if (part_out)
    launch_pdl(blend_bwd_kernel<true>, unsigned(ntiles * kParts), kThreads, kSmemBytesDet, static_cast<cudaStream_t>(stream), 
        d_image, reinterpret_cast<const float4*>(splats->rec), sorted_ids, reinterpret_cast<const int2*>(ranges),
        t_final, last, width, height, tiles_x, row_begin * tiles_x, bg, reinterpret_cast<float4*>(grads2d),
        tile_order, part_out, top_out);
  else
    launch_pdl(blend_bwd_kernel<false>, unsigned(ntiles * kParts), kThreads, kSmemBytes, static_cast<cudaStream_t>(stream), 
        d_image, reinterpret_cast<const float4*>(splats->rec), sorted_ids, reinterpret_cast<const int2*>(ranges),
        t_final, last, width, height, tiles_x, row_begin * tiles_x, bg, reinterpret_cast<float4*>(grads2d),
        tile_order, nullptr, nullptr);
  return check_launch();
}

}  // namespace
}  // namespace gs

extern "C" int gs_blend_backward(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                                 const int32_t* ranges, const float* t_final, const int32_t* last, int32_t width,
                                 int32_t height, const float background[3], float* grads2d, void* stream) {
  using namespace gs;
  if (!splats || !grads2d || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  cudaError_t e = cudaMemsetAsync(grads2d, 0, size_t(splats->n) * GS_GRAD2D_FLOATS * sizeof(float),
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return record_cuda_error(e);
  return blend_backward_rows(d_image, splats, sorted_ids, ranges, t_final, last, width, height, 0,
                             (height + kTile - 1) / kTile, background, grads2d, stream);
}

// The full frame with the tiles visited in `tile_order` (a permutation of
// [0, tiles), device int32), e.g. by descending list length.
extern "C" int gs_blend_backward_ordered(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                                         const int32_t* ranges, const float* t_final, const int32_t* last,
                                         int32_t width, int32_t height, const float background[3],
                                         const int32_t* tile_order, float* grads2d, void* stream) {
  using namespace gs;
  if (!splats || !grads2d || !tile_order || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  cudaError_t e = cudaMemsetAsync(grads2d, 0, size_t(splats->n) * GS_GRAD2D_FLOATS * sizeof(float),
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return record_cuda_error(e);
  return blend_backward_rows(d_image, splats, sorted_ids, ranges, t_final, last, width, height, 0,
                             (height + kTile - 1) / kTile, background, grads2d, stream, tile_order);
}

// ---------------------------------------------------------------------------
// Longest-first tile schedule for the backward: a tile's work is its number
// of back-to-front splats, need = max(last contributor) - start + 1
// (gradients.py:48-52), known from the forward's training record.  Tiles are
// bucketed by need on a 1/64-octave scale and visited from the heaviest
// bucket down, so the light tiles fill the last wave instead of a few heavy
// ones trailing it.  Scratch: 2 T + 2048 ints.
namespace gs {
namespace {
constexpr int kSchedBuckets = 1024;   // 1/64-octave buckets: close to an exact descending sort

__device__ __forceinline__ int need_bucket(int need) {
  return need <= 0 ? 0 : min(kSchedBuckets - 1, 1 + int(__log2f(float(need)) * 64.0f));
}

// one warp per tile: max of `last` over the tile's pixels -> the tile's work
__global__ void tile_need_kernel(const int32_t* __restrict__ last, const int2* __restrict__ ranges, int width,
                                 int height, int tiles_x, int tiles, int32_t* __restrict__ bucket_of,
                                 int32_t* __restrict__ hist) {
  pdl_begin();
  const int tile = int((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (tile >= tiles) return;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  int m = -1;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int p = lane + 32 * k;             // 16 x 16 pixels, row-major within the tile
    const int px = tx * kTile + (p & 15), py = ty * kTile + (p >> 4);
    if (px < width && py < height) m = max(m, last[size_t(py) * width + px]);
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane == 0) {
    const int2 r = ranges[tile];
    const int b = need_bucket(m >= r.x ? m - r.x + 1 : 0);
    bucket_of[tile] = b;
    atomicAdd(&hist[b], 1);
  }
}

// bucket of a given per-tile work (gs_tile_schedule)
__global__ void tile_bucket_kernel(const int32_t* __restrict__ work, int tiles, int32_t* __restrict__ bucket_of,
                                   int32_t* __restrict__ hist) {
  pdl_begin();
  const int t = int(int64_t(blockIdx.x) * blockDim.x + threadIdx.x);
  if (t >= tiles) return;
  const int b = need_bucket(work[t]);
  bucket_of[t] = b;
  atomicAdd(&hist[b], 1);
}

// exclusive scan over the buckets from the heaviest down (one block of
// kSchedBuckets threads; thread i owns bucket kSchedBuckets - 1 - i)
__global__ void __launch_bounds__(kSchedBuckets) tile_sched_scan_kernel(const int32_t* __restrict__ hist,
                                                                        int32_t* __restrict__ cursor) {
  pdl_begin();
  __shared__ int warp_tot[kSchedBuckets / 32];
  const int i = threadIdx.x, lane = i & 31, w = i >> 5;
  const int b = kSchedBuckets - 1 - i;
  const int c = hist[b];
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = lane < kSchedBuckets / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += v;
    }
    if (lane < kSchedBuckets / 32) warp_tot[lane] = t;   // inclusive over warps
  }
  __syncthreads();
  cursor[b] = incl - c + (w > 0 ? warp_tot[w - 1] : 0);
}

__global__ void tile_sched_scatter_kernel(const int32_t* __restrict__ bucket_of, int32_t* __restrict__ cursor,
                                          int tiles, int32_t* __restrict__ order) {
  pdl_begin();
  const int t = int(int64_t(blockIdx.x) * blockDim.x + threadIdx.x);
  if (t < tiles) order[atomicAdd(&cursor[bucket_of[t]], 1)] = t;
}
}  // namespace
}  // namespace gs

// The longest-first order alone (scratch[0, tiles) receives it).
extern "C" int gs_blend_backward_schedule(const int32_t* ranges, const int32_t* last, int32_t width, int32_t height,
                                          int32_t* scratch, void* stream) {
  using namespace gs;
  if (!scratch || !ranges || !last || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles64 = int64_t(tiles_x) * tiles_y;
  if (tiles64 > int64_t(INT32_MAX) / 4) return GS_ERR_RESOURCE_LIMIT;
  const int tiles = int(tiles64);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* order = scratch;
  int32_t* bucket_of = scratch + tiles;
  int32_t* hist = scratch + 2 * tiles;
  int32_t* cursor = hist + kSchedBuckets;
  cudaError_t e = cudaMemsetAsync(hist, 0, kSchedBuckets * sizeof(int32_t), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  launch_pdl(tile_need_kernel, unsigned((int64_t(tiles) * 32 + 255) / 256), 256, 0, s, 
      last, reinterpret_cast<const int2*>(ranges), width, height, tiles_x, tiles, bucket_of, hist);
  launch_pdl(tile_sched_scan_kernel, 1, kSchedBuckets, 0, s, hist, cursor);
  launch_pdl(tile_sched_scatter_kernel, unsigned((tiles + 255) / 256), 256, 0, s, bucket_of, cursor, tiles, order);
  return check_launch();
}

// The blend kernel alone: accumulates into the caller's grads2d (no
// clearing), tiles in `tile_order` (nullable: row-major).
extern "C" int gs_blend_backward_accumulate(const float* d_image, const gs_splats_t* splats,
                                            const uint32_t* sorted_ids, const int32_t* ranges, const float* t_final,
                                            const int32_t* last, int32_t width, int32_t height,
                                            const float background[3], const int32_t* tile_order, float* grads2d,
                                            void* stream) {
  using namespace gs;
  if (!splats || !grads2d || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  return blend_backward_rows(d_image, splats, sorted_ids, ranges, t_final, last, width, height, 0,
                             (height + kTile - 1) / kTile, background, grads2d, stream, tile_order);
}

extern "C" int gs_blend_backward_scheduled(const float* d_image, const gs_splats_t* splats,
                                           const uint32_t* sorted_ids, const int32_t* ranges, const float* t_final,
                                           const int32_t* last, int32_t width, int32_t height,
                                           const float background[3], int32_t* scratch, float* grads2d,
                                           void* stream) {
  if (!splats || !grads2d) return GS_ERR_INVALID_ARG;
  const int st = gs_blend_backward_schedule(ranges, last, width, height, scratch, stream);
  if (st != GS_OK) return st;
  return gs_blend_backward_ordered(d_image, splats, sorted_ids, ranges, t_final, last, width, height, background,
                                   scratch, grads2d, stream);
}

// Longest-first order of `tiles` tiles from any per-tile work estimate
// (e.g. the forward's gs_blend_forward_ordered tile_work of the previous frame).
// scratch: device int32[tiles + 2048]; order: device int32[tiles].
extern "C" int gs_tile_schedule(const int32_t* work, int32_t tiles, int32_t* scratch, int32_t* order, void* stream) {
  using namespace gs;
  if (!work || !scratch || !order || tiles < 0) return GS_ERR_INVALID_ARG;
  if (tiles == 0) return GS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* bucket_of = scratch;
  int32_t* hist = scratch + tiles;
  int32_t* cursor = hist + kSchedBuckets;
  cudaError_t e = cudaMemsetAsync(hist, 0, kSchedBuckets * sizeof(int32_t), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  launch_pdl(tile_bucket_kernel, unsigned((tiles + 255) / 256), 256, 0, s, work, tiles, bucket_of, hist);
  launch_pdl(tile_sched_scan_kernel, 1, kSchedBuckets, 0, s, hist, cursor);
  launch_pdl(tile_sched_scatter_kernel, unsigned((tiles + 255) / 256), 256, 0, s, bucket_of, cursor, tiles, order);
  return check_launch();
}

// ---------------------------------------------------------------------------
// Deterministic backward (the reference's deterministic=True / workers=1
// contract, rasterizer.py:32-41, test_cli.py:24-35: bit-identical runs).
// The blend writes one partial row per (sorted instance, half tile) — no
// float atomics — and each splat's rows are then summed in a fixed order:
// its tiles in row-major order over its rectangle (the reference's own
// expansion order, rasterizer.py:105-111), the two halves of a tile in order.
// The instance position of (splat, k-th tile of its rectangle) comes from an
// inverse index built from the sorted list.
namespace gs {
namespace {

constexpr int kScanBlock = 1024;

// off[g] = exclusive prefix of max(tiles_touched, 0): block sums, then a
// single-block scan of the sums, then the per-block add
__global__ void __launch_bounds__(kScanBlock) det_count_kernel(const int32_t* __restrict__ tiles, int64_t n,
                                                               uint32_t* __restrict__ off, uint32_t* __restrict__ sums) {
  pdl_begin();
  __shared__ uint32_t s_w[32];
  const int64_t g = int64_t(blockIdx.x) * kScanBlock + threadIdx.x;
  const uint32_t v = g < n ? uint32_t(max(tiles[g], 0)) : 0u;
  uint32_t incl = v;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    s_w[lane] = x;   // inclusive over warps
  }
  __syncthreads();
  const uint32_t excl = incl - v + (w > 0 ? s_w[w - 1] : 0u);
  if (g < n) off[g] = excl;
  if (threadIdx.x == kScanBlock - 1) sums[blockIdx.x] = excl + v;
}

__global__ void __launch_bounds__(kScanBlock) det_sums_kernel(uint32_t* __restrict__ sums, int64_t blocks) {
  pdl_begin();
  __shared__ uint32_t s_run;
  if (threadIdx.x == 0) s_run = 0u;
  __syncthreads();
  for (int64_t b0 = 0; b0 < blocks; b0 += kScanBlock) {
    const int64_t b = b0 + threadIdx.x;
    const uint32_t v = b < blocks ? sums[b] : 0u;
    // serial-per-chunk scan by a warp-free simple approach: one thread per element
    uint32_t incl = v;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    __shared__ uint32_t s_w[32];
    if (lane == 31) s_w[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t x = s_w[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (int(threadIdx.x) >= o) x += t;
      }
      s_w[threadIdx.x] = x;
    }
    __syncthreads();
    const int w = threadIdx.x >> 5;
    const uint32_t excl = s_run + incl - v + (w > 0 ? s_w[w - 1] : 0u);
    if (b < blocks) sums[b] = excl;
    __syncthreads();
    if (threadIdx.x == kScanBlock - 1) s_run = excl + v;
    __syncthreads();
  }
}

__global__ void det_add_kernel(uint32_t* __restrict__ off, const uint32_t* __restrict__ sums, int64_t n) {
  pdl_begin();
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < n) off[g] += sums[g / kScanBlock];
}

// inv[off[g] + k] = sorted position of (g, k-th tile of its rectangle); one warp per tile
__global__ void det_inverse_kernel(const uint32_t* __restrict__ ids, const int2* __restrict__ ranges,
                                   const int4* __restrict__ rect, const uint32_t* __restrict__ off, int tiles_x,
                                   int64_t tiles, uint32_t* __restrict__ inv) {
  pdl_begin();
  const int64_t tile = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (tile >= tiles) return;
  const int tx = int(tile % tiles_x), ty = int(tile / tiles_x);
  const int2 r = ranges[tile];
  for (int pos = r.x + (threadIdx.x & 31); pos < r.y; pos += 32) {
    const uint32_t g = ids[pos];
    const int4 rc = rect[g];
    inv[off[g] + uint32_t((ty - rc.y) * (rc.z - rc.x + 1) + (tx - rc.x))] = uint32_t(pos);
  }
}

// one thread per splat: its partial rows in the fixed order -> the (N,12) row
__global__ void det_reduce_kernel(const int32_t* __restrict__ tiles, const int4* __restrict__ rect,
                                  const uint32_t* __restrict__ off, const uint32_t* __restrict__ inv,
                                  const float* __restrict__ part_rows, const int32_t* __restrict__ top,
                                  int tiles_x, int64_t n, float* __restrict__ grads2d) {
  pdl_begin();
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n) return;
  float acc[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) acc[c] = 0.0f;
  if (tiles[g] > 0) {
    const int4 rc = rect[g];
    uint32_t k = off[g];
    for (int ty = rc.y; ty <= rc.w; ++ty)
      for (int tx = rc.x; tx <= rc.z; ++tx, ++k) {
        const int64_t t = int64_t(ty) * tiles_x + tx;
        const uint32_t pos = inv[k];
#pragma unroll
        for (int part = 0; part < kParts; ++part)
          if (int64_t(pos) < int64_t(top[t * kParts + part])) {
            const float* row = part_rows + (size_t(pos) * kParts + part) * kC;
#pragma unroll
            for (int c = 0; c < kC; ++c) acc[c] += row[c];
          }
      }
  }
  float4* out = reinterpret_cast<float4*>(grads2d) + 3 * g;
  out[0] = make_float4(acc[0], acc[1], acc[2], 0.0f);
  out[1] = make_float4(acc[3], acc[4], acc[5], 0.0f);
  out[2] = make_float4(acc[6], acc[7], acc[8], 0.0f);
}

struct DetLayout {
  size_t part_rows, inv, off, sums, top, bytes;
};

inline size_t det_align(size_t x) { return (x + 255) & ~size_t(255); }

int det_layout(int64_t n, int32_t width, int32_t height, int64_t cap, DetLayout* L) {
  if (n < 0 || cap < 0 || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  if (cap > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  const int64_t tiles = int64_t((width + kTile - 1) / kTile) * ((height + kTile - 1) / kTile);
  const size_t un = size_t(n > 0 ? n : 1), uc = size_t(cap > 0 ? cap : 1);
  size_t o = 0;
  L->part_rows = o; o += det_align(sizeof(float) * uc * kParts * kC);
  L->inv = o; o += det_align(sizeof(uint32_t) * uc);
  L->off = o; o += det_align(sizeof(uint32_t) * un);
  L->sums = o; o += det_align(sizeof(uint32_t) * (un / kScanBlock + 1));
  L->top = o; o += det_align(sizeof(int32_t) * size_t(tiles) * kParts);
  L->bytes = o;
  return GS_OK;
}

}  // namespace
}  // namespace gs

extern "C" int gs_blend_backward_det_workspace_size(int64_t n, int32_t width, int32_t height, int64_t k_capacity,
                                                    size_t* bytes) {
  if (!bytes) return GS_ERR_INVALID_ARG;
  gs::DetLayout L;
  const int st = gs::det_layout(n, width, height, k_capacity, &L);
  if (st == GS_OK) *bytes = L.bytes;
  return st;
}

extern "C" int gs_blend_backward_deterministic(const float* d_image, const gs_splats_t* splats,
                                               const uint32_t* sorted_ids, const int32_t* ranges,
                                               const float* t_final, const int32_t* last, int32_t width,
                                               int32_t height, const float background[3],
                                               const int32_t* tile_order, void* workspace, size_t workspace_bytes,
                                               int64_t k_capacity, float* grads2d, void* stream) {
  using namespace gs;
  if (!splats || !grads2d || !ranges || !sorted_ids || !workspace) return GS_ERR_INVALID_ARG;
  DetLayout L;
  int st = det_layout(splats->n, width, height, k_capacity, &L);
  if (st != GS_OK) return st;
  if (workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  const int64_t n = splats->n;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return GS_OK;
  char* ws = static_cast<char*>(workspace);
  float* part_rows = reinterpret_cast<float*>(ws + L.part_rows);
  uint32_t* inv = reinterpret_cast<uint32_t*>(ws + L.inv);
  uint32_t* off = reinterpret_cast<uint32_t*>(ws + L.off);
  uint32_t* sums = reinterpret_cast<uint32_t*>(ws + L.sums);
  int32_t* top = reinterpret_cast<int32_t*>(ws + L.top);
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * tiles_y;
  st = blend_backward_rows(d_image, splats, sorted_ids, ranges, t_final, last, width, height, 0, tiles_y, background,
                           grads2d, stream, tile_order, part_rows, top);
  if (st != GS_OK) return st;
  const int64_t blocks = (n + kScanBlock - 1) / kScanBlock;
  launch_pdl(det_count_kernel, unsigned(blocks), kScanBlock, 0, s, splats->tiles_touched, n, off, sums);
  launch_pdl(det_sums_kernel, 1, kScanBlock, 0, s, sums, blocks);
  launch_pdl(det_add_kernel, unsigned((n + 255) / 256), 256, 0, s, off, sums, n);
  const int4* rect = reinterpret_cast<const int4*>(splats->rect);
  launch_pdl(det_inverse_kernel, unsigned((tiles * 32 + 255) / 256), 256, 0, s, 
      sorted_ids, reinterpret_cast<const int2*>(ranges), rect, off, tiles_x, tiles, inv);
  launch_pdl(det_reduce_kernel, unsigned((n + 255) / 256), 256, 0, s, splats->tiles_touched, rect, off, inv, part_rows, top,
                                                              tiles_x, n, grads2d);
  return check_launch();
}

#if GS_BWD_STATS
extern "C" int gs_debug_bwd_hist(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, gs::g_bwd_hist, sizeof(unsigned long long) * 33);
  if (e == cudaSuccess && reset) {
    unsigned long long z[33] = {};
    e = cudaMemcpyToSymbol(gs::g_bwd_hist, z, sizeof(z));
  }
  return e == cudaSuccess ? 0 : 1;
}
#endif
