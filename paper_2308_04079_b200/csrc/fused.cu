// Fused single-call entry points: the reference's render_view
// (optimizer.py:212-219: project -> bin_and_sort -> render_forward) and its
// backward pair render_backward + backward_project (rasterizer.py:253-316,
// gradients.py:192-259), each one C call enqueueing every kernel of the
// stage on the caller's stream with no host synchronisation.  They compose
// the stage entry points; the drop-in torch.autograd.Function binds these.
#include "gs_common.cuh"

extern "C" int gs_forward(const gs_params_t* params, const gs_camera_t* camera, int32_t active_sh_degree,
                          gs_splats_t* splats, void* bin_workspace, size_t bin_workspace_bytes, int64_t k_capacity,
                          uint32_t* sorted_ids, int32_t* ranges, int64_t* k_info, const float background[3],
                          int32_t training, const int32_t* tile_order, float* image, float* t_final, int32_t* last,
                          int32_t* scratch, void* stream) {
  if (!params || !camera || !splats || !k_info) return GS_ERR_INVALID_ARG;
  int st = gs_preprocess_forward(params, camera, active_sh_degree, splats, stream);
  if (st != GS_OK) return st;
  st = gs_bin_and_sort_async(splats, camera->width, camera->height, bin_workspace, bin_workspace_bytes, k_capacity,
                             sorted_ids, ranges, nullptr, k_info, stream);
  if (st != GS_OK) return st;
  return gs_blend_forward_ordered(splats, sorted_ids, ranges, camera->width, camera->height, background, training,
                                  tile_order, nullptr, image, t_final, last, scratch, stream);
}

extern "C" int gs_backward(const float* d_image, const gs_params_t* params, const gs_camera_t* camera,
                           int32_t active_sh_degree, const gs_splats_t* splats, const uint32_t* sorted_ids,
                           const int32_t* ranges, const float* t_final, const int32_t* last,
                           const float background[3], int32_t* sched_scratch, float* grads2d,
                           const gs_grads_t* grads, const gs_stats_t* stats, void* stream) {
  if (!camera || !splats || !grads) return GS_ERR_INVALID_ARG;
  int st = sched_scratch
               ? gs_blend_backward_scheduled(d_image, splats, sorted_ids, ranges, t_final, last, camera->width,
                                             camera->height, background, sched_scratch, grads2d, stream)
               : gs_blend_backward(d_image, splats, sorted_ids, ranges, t_final, last, camera->width, camera->height,
                                   background, grads2d, stream);
  if (st != GS_OK) return st;
  return gs_preprocess_backward(params, camera, active_sh_degree, splats, grads2d, grads, 0, stats, stream);
}

extern "C" int gs_backward_prepared(const float* d_image, const gs_params_t* params, const gs_camera_t* camera,
                                    int32_t active_sh_degree, const gs_splats_t* splats, const uint32_t* sorted_ids,
                                    const int32_t* ranges, const float* t_final, const int32_t* last,
                                    const float background[3], const int32_t* sched_scratch, float* grads2d,
                                    const gs_grads_t* grads, const gs_stats_t* stats, void* stream) {
  if (!camera || !splats || !grads || !sched_scratch) return GS_ERR_INVALID_ARG;
  int st = gs_blend_backward_accumulate(d_image, splats, sorted_ids, ranges, t_final, last, camera->width,
                                        camera->height, background, sched_scratch, grads2d, stream);
  if (st != GS_OK) return st;
  return gs_preprocess_backward(params, camera, active_sh_degree, splats, grads2d, grads, 0, stats, stream);
}
