// Model / PLY record (de)interleaving on the device — the data formats either
// side of the hot path: splatlab scene_io
// _records_from_cloud / _cloud_from_records (scene_io.py:377-391) and the
// export_ply vertex layout (scene_io.py:417-439).
//
// A trained scene goes from file bytes to the rasterizer's SoA parameter
// tensors with ONE host->device copy of the packed records and one kernel
// (and back for save/export), instead of a host-side transpose of N x 59
// floats.  Record layouts (little-endian float32):
//   GS_LAYOUT_MODEL (59): mean(3) log_scale(3) rotation(4) opacity(1)
//                         sh(48) channel-major (16 R, 16 G, 16 B)
//   GS_LAYOUT_PLY   (62): x y z nx ny nz (normals 0) f_dc(3) f_rest(45)
//                         channel-major over coefficients 1..15, opacity,
//                         scale(3), rot(4)
// One warp moves 32 records; each thread stages its record through shared
// memory so the global reads and writes of both sides are coalesced.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kRecThreads = 128;
constexpr int kMaxRecFloats = GS_PLY_FLOATS;

__device__ __forceinline__ int record_floats(int layout) {
  return layout == GS_LAYOUT_PLY ? GS_PLY_FLOATS : GS_MODEL_FLOATS;
}

// position of SoA value `v` (0..58: means 0-2, log_scales 3-5, rotations
// 6-9, opacity 10, sh 11 + 3 * coeff + channel) in the record; -1 = none
__device__ __forceinline__ int record_slot(int layout, int v) {
  if (layout == GS_LAYOUT_MODEL) {
    if (v < 11) return v;                       // mean, log_scale, rotation, opacity
    const int k = v - 11, coeff = k / 3, ch = k - 3 * coeff;
    return 11 + ch * 16 + coeff;                // channel-major SH
  }
  if (v < 3) return v;                          // x y z
  if (v < 6) return 55 + (v - 3);               // scale_0..2
  if (v < 10) return 58 + (v - 6);              // rot_0..3
  if (v == 10) return 54;                       // opacity
  const int k = v - 11, coeff = k / 3, ch = k - 3 * coeff;
  if (coeff == 0) return 6 + ch;                // f_dc_ch
  return 9 + ch * 15 + (coeff - 1);             // f_rest, channel-major
}

__device__ __forceinline__ float* soa_ptr(const gs_params_t& p, int v, int64_t g) {
  float* means = const_cast<float*>(p.means);
  float* ls = const_cast<float*>(p.log_scales);
  float* rot = const_cast<float*>(p.rotations);
  float* op = const_cast<float*>(p.opacity_logits);
  float* sh = const_cast<float*>(p.sh);
  if (v < 3) return means + 3 * g + v;
  if (v < 6) return ls + 3 * g + (v - 3);
  if (v < 10) return rot + 4 * g + (v - 6);
  if (v == 10) return op + g;
  return sh + 48 * g + (v - 11);
}

__global__ void __launch_bounds__(kRecThreads)
pack_records_kernel(gs_params_t p, int layout, float* __restrict__ out) {
  __shared__ float s[kRecThreads * kMaxRecFloats];
  const int nf = record_floats(layout);
  const int64_t g0 = int64_t(blockIdx.x) * kRecThreads;
  const int nb = int(min(int64_t(kRecThreads), p.n - g0));
  // SoA -> shared (records, zero-filled unused slots), group by group so the
  // global reads of each group are contiguous
  for (int i = threadIdx.x; i < nb * nf; i += kRecThreads) s[i] = 0.0f;
  __syncthreads();
  for (int i = threadIdx.x; i < nb * 59; i += kRecThreads) {
    // i enumerates (value v, gaussian) with the gaussian fastest inside each group
    const int grp_sizes[5] = {3, 3, 4, 1, 48};
    int v0 = 0, rem = i, grp = 0;
    for (; grp < 5; ++grp) {
      const int span = grp_sizes[grp] * nb;
      if (rem < span) break;
      rem -= span;
      v0 += grp_sizes[grp];
    }
    const int j = rem / grp_sizes[grp], c = rem - j * grp_sizes[grp];   // gaussian j, component c
    const int v = v0 + c;
    s[j * nf + record_slot(layout, v)] = *soa_ptr(p, v, g0 + j);
  }
  __syncthreads();
  float* dst = out + g0 * nf;
  for (int i = threadIdx.x; i < nb * nf; i += kRecThreads) dst[i] = s[i];
}

__global__ void __launch_bounds__(kRecThreads)
unpack_records_kernel(const float* __restrict__ rec, gs_params_t p) {
  __shared__ float s[kRecThreads * GS_MODEL_FLOATS];
  const int nf = GS_MODEL_FLOATS;
  const int64_t g0 = int64_t(blockIdx.x) * kRecThreads;
  const int nb = int(min(int64_t(kRecThreads), p.n - g0));
  const float* src = rec + g0 * nf;
  for (int i = threadIdx.x; i < nb * nf; i += kRecThreads) s[i] = src[i];
  __syncthreads();
  for (int i = threadIdx.x; i < nb * 59; i += kRecThreads) {
    const int grp_sizes[5] = {3, 3, 4, 1, 48};
    int v0 = 0, rem = i, grp = 0;
    for (; grp < 5; ++grp) {
      const int span = grp_sizes[grp] * nb;
      if (rem < span) break;
      rem -= span;
      v0 += grp_sizes[grp];
    }
    const int j = rem / grp_sizes[grp], c = rem - j * grp_sizes[grp];
    const int v = v0 + c;
    *soa_ptr(p, v, g0 + j) = s[j * nf + record_slot(GS_LAYOUT_MODEL, v)];
  }
}

}  // namespace
}  // namespace gs

extern "C" int gs_pack_records(const gs_params_t* params, int32_t layout, float* out, void* stream) {
  using namespace gs;
  if (!params || !out || params->n < 0) return GS_ERR_INVALID_ARG;
  if (layout != GS_LAYOUT_MODEL && layout != GS_LAYOUT_PLY) return GS_ERR_INVALID_ARG;
  if (params->n == 0) return GS_OK;
  if (!params->means || !params->rotations || !params->log_scales || !params->opacity_logits || !params->sh)
    return GS_ERR_INVALID_ARG;
  const int64_t blocks = (params->n + kRecThreads - 1) / kRecThreads;
  pack_records_kernel<<<unsigned(blocks), kRecThreads, 0, static_cast<cudaStream_t>(stream)>>>(*params, layout,
                                                                                               out);
  return check_launch();
}

extern "C" int gs_unpack_records(const float* records, gs_params_t* params_out, void* stream) {
  using namespace gs;
  if (!records || !params_out || params_out->n < 0) return GS_ERR_INVALID_ARG;
  if (params_out->n == 0) return GS_OK;
  if (!params_out->means || !params_out->rotations || !params_out->log_scales || !params_out->opacity_logits ||
      !params_out->sh)
    return GS_ERR_INVALID_ARG;
  const int64_t blocks = (params_out->n + kRecThreads - 1) / kRecThreads;
  unpack_records_kernel<<<unsigned(blocks), kRecThreads, 0, static_cast<cudaStream_t>(stream)>>>(records,
                                                                                                 *params_out);
  return check_launch();
}
