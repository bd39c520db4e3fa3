// K6 blend_fwd — replaces splatlab rasterizer.render_forward / _blend_tile
// (rasterizer.py:152-240).
//
// One 256-thread CTA per 16x16 tile, one pixel per thread, each warp an 8x4
// pixel block.  The tile's sorted instance list is walked front to back in
// batches of 256: every thread gathers one splat record (48 of its 64 B)
// into shared memory and computes the splat's 8-bit warp coverage mask
// (warp_cover_mask).  Each warp then visits, in order, only the splats whose
// mask bit is set (a ballot over 32 mask bits at a time), so splats that
// cannot reach alpha >= 1/255 anywhere in its block cost no pixel work.
// A pixel stops before its accumulated opacity would exceed 0.9999
// (rasterizer.py:179-180); the CTA leaves the list as soon as
// __syncthreads_count says every pixel is done (rasterizer.py:194-195).
#include "gs_common.cuh"

namespace gs {
namespace {

template <bool kTraining>
__global__ void __launch_bounds__(kTilePixels)
blend_fwd_kernel(const float4* __restrict__ rec, const uint32_t* __restrict__ ids, const int2* __restrict__ ranges,
                 int width, int height, int tiles_x, float3 bg, float* __restrict__ image,
                 float* __restrict__ t_final, int32_t* __restrict__ last) {
  __shared__ float4 s_r0[kTilePixels];
  __shared__ float4 s_r1[kTilePixels];
  __shared__ float4 s_col[kTilePixels];
  __shared__ uint32_t s_id[kTilePixels];
  __shared__ uint8_t s_mask[kTilePixels];

  const int tile = blockIdx.x;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + tile_px(t);
  const int py = ty * kTile + tile_py(t);
  const bool inside = (px < width) && (py < height);
  const float fx = float(px) + 0.5f, fy = float(py) + 0.5f;  // rasterizer.py:142
  const float tile_x0 = float(tx * kTile), tile_y0 = float(ty * kTile);

  const int2 range = ranges[tile];
  float T = 1.0f;
  float cr = 0.0f, cg = 0.0f, cb = 0.0f;
  int32_t last_idx = -1;
  bool done = !inside;

  for (int base = range.x; base < range.y; base += kTilePixels) {
    if (__syncthreads_count(done) == kTilePixels) break;
    const int i = base + t;
    if (i < range.y) {
      const uint32_t g = ids[i];
      const float4 r0 = rec[4 * size_t(g) + 0];
      const float4 r1 = rec[4 * size_t(g) + 1];
      s_id[t] = g;
      s_r0[t] = r0;
      s_r1[t] = r1;
      s_col[t] = rec[4 * size_t(g) + 2];
      s_mask[t] = uint8_t(warp_cover_mask(r0, r1, tile_x0, tile_y0));
    }
    __syncthreads();
    if (__all_sync(0xffffffffu, done)) continue;
    const int cnt = min(kTilePixels, range.y - base);
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int jl = c0 + lane;
      unsigned live = __ballot_sync(0xffffffffu, jl < cnt && ((s_mask[jl] >> warp) & 1u));
      while (live) {
        const int j = c0 + __ffs(live) - 1;
        live &= live - 1;
        if (done) continue;
        const AlphaEval e = eval_alpha(fx, fy, s_r0[j], s_r1[j], rec, s_id[j]);
        if (e.a == 0.0f) continue;
        const float t_new = T * (1.0f - e.a);
        if (t_new < kTransSat) {  // 1 - T_new > 0.9999
          done = true;
          continue;
        }
        const float4 c = s_col[j];
        const float w = T * e.a;
        cr = fmaf(w, c.x, cr);
        cg = fmaf(w, c.y, cg);
        cb = fmaf(w, c.z, cb);
        T = t_new;
        if (kTraining) last_idx = base + j;
      }
      if (__all_sync(0xffffffffu, done)) break;
    }
  }
  if (!inside) return;
  const size_t p = size_t(py) * width + px;
  image[3 * p + 0] = fmaf(T, bg.x, cr);  // rasterizer.py:197
  image[3 * p + 1] = fmaf(T, bg.y, cg);
  image[3 * p + 2] = fmaf(T, bg.z, cb);
  if (kTraining) {
    t_final[p] = T;
    last[p] = last_idx;
  }
}

}  // namespace
}  // namespace gs

extern "C" int gs_blend_forward(const gs_splats_t* splats, const uint32_t* sorted_ids, const int32_t* ranges,
                                int32_t width, int32_t height, const float background[3], int32_t training,
                                float* image, float* t_final, int32_t* last, void* stream) {
  using namespace gs;
  if (!splats || !ranges || !image || !background || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  if (training && (!t_final || !last)) return GS_ERR_INVALID_ARG;
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * tiles_y;
  if (tiles > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float3 bg = make_float3(background[0], background[1], background[2]);
  const float4* rec = reinterpret_cast<const float4*>(splats->rec);
  const int2* rg = reinterpret_cast<const int2*>(ranges);
  if (training)
    blend_fwd_kernel<true><<<unsigned(tiles), kTilePixels, 0, s>>>(rec, sorted_ids, rg, width, height, tiles_x, bg,
                                                                  image, t_final, last);
  else
    blend_fwd_kernel<false><<<unsigned(tiles), kTilePixels, 0, s>>>(rec, sorted_ids, rg, width, height, tiles_x, bg,
                                                                   image, nullptr, nullptr);
  return check_launch();
}
