// K1 preprocess_fwd — replaces splatlab core.project (core.py:266-345) and the
// per-splat tile rectangle of rasterizer.bin_and_sort (rasterizer.py:86-97).
//
// One thread per Gaussian.  The geometry chain that decides integers
// (culling, radius, tile rectangle, float32 depth key) runs in float64 with
// non-contracted IEEE operations, mirroring the float64 reference, so radii
// and binning agree bit-for-bit.  Appearance (SH colour) runs in float32.
// Besides the hi/lo split of mean, conic and alpha, each record carries the
// conic's scaled eigenbasis (conic_basis, float64) from which the blends
// evaluate the exponent as a sum of two squares.
#include "project.cuh"

namespace gs {
namespace {

#ifndef GS_PREFWD_MINB
#define GS_PREFWD_MINB 6   // 80 registers, no spills: 0.196 vs 0.208 ms at the default 94
#endif
__global__ void __launch_bounds__(128, GS_PREFWD_MINB)
preprocess_fwd_kernel(gs_params_t p, DevCamera cam, int degree, gs_splats_t out) {
  pdl_begin();
  const int64_t g0 = int64_t(blockIdx.x) * blockDim.x;
  const int64_t g = g0 + threadIdx.x;
  // The block's SH rows (one contiguous 192 B x 128 span) are bulk-prefetched
  // into L2 by the TMA unit while the float64 geometry runs; the colour step
  // then reads each thread's row from L2.  No shared-memory staging, no block
  // barrier, and culled Gaussians never touch their SH bytes.
  if (threadIdx.x == 0) {
    const int64_t nbk = min(int64_t(blockDim.x), p.n - g0);
    const int rows = (degree + 1) * (degree + 1);
    // SH (N,16,3): the active rows of every Gaussian lie inside its 192-B record
    prefetch_l2_span(p.sh + 48 * g0, size_t(48 * (nbk - 1) + 3 * rows) * sizeof(float));
  }
  float pm0 = 0.f, pm1 = 0.f, pm2 = 0.f, pl0 = 0.f, pl1 = 0.f, pl2 = 0.f, pop = 0.f;
  float4 qf = make_float4(1.f, 0.f, 0.f, 0.f);
  if (g < p.n) {
    pm0 = __ldg(p.means + 3 * g + 0); pm1 = __ldg(p.means + 3 * g + 1); pm2 = __ldg(p.means + 3 * g + 2);
    qf = __ldg(reinterpret_cast<const float4*>(p.rotations) + g);
    pl0 = __ldg(p.log_scales + 3 * g + 0); pl1 = __ldg(p.log_scales + 3 * g + 1);
    pl2 = __ldg(p.log_scales + 3 * g + 2);
    pop = __ldg(p.opacity_logits + g);
  }
  if (g >= p.n) return;

  const float4* shrow = reinterpret_cast<const float4*>(p.sh) + 12 * g;
  project_gaussian(pm0, pm1, pm2, qf, pl0, pl1, pl2, pop, [&](int k) { return __ldg(shrow + k); }, cam, degree, out,
                   g);
}

}  // namespace
}  // namespace gs

extern "C" int gs_preprocess_forward(const gs_params_t* params, const gs_camera_t* camera,
                                     int32_t active_sh_degree, gs_splats_t* splats, void* stream) {
  if (!params || !camera || !splats) return GS_ERR_INVALID_ARG;
  if (active_sh_degree < 0 || active_sh_degree > 3) return GS_ERR_INVALID_ARG;
  if (camera->width <= 0 || camera->height <= 0 || !(camera->fx > 0) || !(camera->fy > 0) ||
      !(camera->near_plane > 0))
    return GS_ERR_INVALID_ARG;
  if (params->n < 0 || splats->n != params->n) return GS_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = gs::zero_async(splats->status, sizeof(int32_t), nullptr, 0, s);
  if (e != cudaSuccess) return gs::record_cuda_error(e);
  if (params->n == 0) return GS_OK;
  const gs::DevCamera cam = gs::make_dev_camera(*camera);
  const int block = 128;
  const unsigned grid = unsigned((params->n + block - 1) / block);
  gs::launch_pdl(gs::preprocess_fwd_kernel, grid, block, 0, s, *params, cam, active_sh_degree, *splats);
  return gs::check_launch();
}
