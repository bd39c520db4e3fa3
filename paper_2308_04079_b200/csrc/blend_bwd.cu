// K7 blend_bwd — replaces splatlab rasterizer.render_backward
// (rasterizer.py:253-316) and gradients.backward_blend (gradients.py:30-94).
//
// Same CTA-per-tile layout as the forward.  Each tile walks its list back to
// front from the largest last contributor of its pixels (gradients.py:48-52),
// re-evaluating alpha with the forward's exact code so the contributor sets
// coincide.  Each pixel rebuilds T_before by dividing out (1 - a)
// (gradients.py:67-70) and carries the composited tail (gradients.py:75-78)
// as a running sum.  The nine per-splat partial gradients of a warp are
// summed with xor shuffles and committed with three float4 atomics per warp,
// only when at least one lane contributed.
#include "gs_common.cuh"

namespace gs {
namespace {

__global__ void __launch_bounds__(kTilePixels)
blend_bwd_kernel(const float* __restrict__ d_image, const float4* __restrict__ rec, const uint32_t* __restrict__ ids,
                 const int2* __restrict__ ranges, const float* __restrict__ t_final, const int32_t* __restrict__ last,
                 int width, int height, int tiles_x, float3 bg, float4* __restrict__ grads2d) {
  __shared__ float4 s_r0[kTilePixels];
  __shared__ float4 s_r1[kTilePixels];
  __shared__ float4 s_col[kTilePixels];
  __shared__ uint32_t s_id[kTilePixels];
  __shared__ int s_warp_max[kTilePixels / 32];

  const int tile = blockIdx.x;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int px = tx * kTile + (t & (kTile - 1));
  const int py = ty * kTile + (t >> 4);
  const bool inside = (px < width) && (py < height);
  const float fx = float(px) + 0.5f, fy = float(py) + 0.5f;
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
  if (!__syncthreads_or(nonzero)) return;
  // needed = max(last_local) + 1 (gradients.py:48-52)
  int wmax = __reduce_max_sync(0xffffffffu, last_idx);
  if (lane == 0) s_warp_max[warp] = wmax;
  __syncthreads();
  int tile_last = s_warp_max[0];
#pragma unroll
  for (int w = 1; w < kTilePixels / 32; ++w) tile_last = max(tile_last, s_warp_max[w]);
  if (tile_last < range.x) return;

  // composited tail behind the current splat, starts at the background term
  float S = T * (dlx * bg.x + dly * bg.y + dlz * bg.z);

  for (int top = tile_last + 1; top > range.x; top -= kTilePixels) {
    const int lo = max(range.x, top - kTilePixels);
    __syncthreads();
    const int i = lo + t;
    if (i < top) {
      const uint32_t g = ids[i];
      s_id[t] = g;
      s_r0[t] = rec[4 * size_t(g) + 0];
      s_r1[t] = rec[4 * size_t(g) + 1];
      s_col[t] = rec[4 * size_t(g) + 2];
    }
    __syncthreads();
    for (int j = top - lo - 1; j >= 0; --j) {
      const int gi = lo + j;
      float g_mx = 0.f, g_my = 0.f, g_al = 0.f, g_ca = 0.f, g_cb = 0.f, g_cc = 0.f, g_r = 0.f, g_g = 0.f, g_b = 0.f;
      bool contrib = false;
      if (gi <= last_idx) {
        const float4 r1 = s_r1[j];
        const AlphaEval e = eval_alpha(fx, fy, s_r0[j], r1, rec, s_id[j]);
        if (e.a > 0.0f) {
          contrib = true;
          const float inv = __frcp_rn(1.0f - e.a);
          T = T * inv;  // transmittance just before this splat
          const float w = T * e.a;
          const float4 c = s_col[j];
          const float dc = c.x * dlx + c.y * dly + c.z * dlz;
          const float d_a = T * dc - S * inv;  // gradients.py:81
          S = fmaf(w, dc, S);
          g_r = w * dlx;
          g_g = w * dly;
          g_b = w * dlz;
          if (e.live) {  // clamped alphas pass no gradient (gradients.py:83-84)
            g_al = d_a * e.g;
            const float dp = d_a * e.a_raw;
            g_mx = dp * (r1.x * e.dx + r1.y * e.dy);
            g_my = dp * (r1.y * e.dx + r1.z * e.dy);
            g_ca = -0.5f * dp * e.dx * e.dx;
            g_cb = -dp * e.dx * e.dy;
            g_cc = -0.5f * dp * e.dy * e.dy;
          }
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
        g_mx = warp_sum(g_mx);
        g_my = warp_sum(g_my);
        g_al = warp_sum(g_al);
        g_ca = warp_sum(g_ca);
        g_cb = warp_sum(g_cb);
        g_cc = warp_sum(g_cc);
        g_r = warp_sum(g_r);
        g_g = warp_sum(g_g);
        g_b = warp_sum(g_b);
        if (lane < 3) {
          float4* row = grads2d + 3 * size_t(s_id[j]);
          float4 v;
          if (lane == 0) v = make_float4(g_mx, g_my, g_al, 0.0f);
          else if (lane == 1) v = make_float4(g_ca, g_cb, g_cc, 0.0f);
          else v = make_float4(g_r, g_g, g_b, 0.0f);
          atomicAdd(row + lane, v);
        }
      }
    }
  }
}

}  // namespace
}  // namespace gs

extern "C" int gs_blend_backward(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                                 const int32_t* ranges, const float* t_final, const int32_t* last, int32_t width,
                                 int32_t height, const float background[3], float* grads2d, void* stream) {
  using namespace gs;
  if (!d_image || !splats || !ranges || !t_final || !last || !grads2d || !background || width <= 0 ||
      height <= 0)
    return GS_ERR_INVALID_ARG;
  const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
  const int64_t tiles = int64_t(tiles_x) * tiles_y;
  if (tiles > int64_t(INT32_MAX)) return GS_ERR_RESOURCE_LIMIT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(grads2d, 0, size_t(splats->n) * GS_GRAD2D_FLOATS * sizeof(float), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  if (splats->n == 0) return GS_OK;
  const float3 bg = make_float3(background[0], background[1], background[2]);
  blend_bwd_kernel<<<unsigned(tiles), kTilePixels, 0, s>>>(
      d_image, reinterpret_cast<const float4*>(splats->rec), sorted_ids, reinterpret_cast<const int2*>(ranges),
      t_final, last, width, height, tiles_x, bg, reinterpret_cast<float4*>(grads2d));
  return check_launch();
}
