/*
 * gs_rasterizer.h — C ABI of the B200-native differentiable Gaussian-splatting
 * rasterizer (libgs_b200.so).
 *
 * This is the drop-in boundary for the hot path of arXiv 2308.04079 as the
 * reference package `splatlab` (/root/reference/pkg/src/splatlab) structures
 * it.  The reference has no native FFI: its hot path is the Python function
 * trio render_view / render_backward / backward_project plus the Adam step.
 * Every entry point below replaces one of those functions (or one stage
 * inside them) and is bound from Python through ctypes.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers owned by the caller (torch's
 *     caching allocator in the Python host layer).  The library never
 *     allocates or frees device memory and keeps no global mutable state.
 *   - Work is enqueued on the caller's stream (`stream` is a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  Only gs_bin_and_sort
 *     synchronises that stream once (to read the instance count K);
 *     gs_bin_and_sort_async keeps K on the device.
 *   - Parameter layouts are the reference's (core.py:36-50): means (N,3),
 *     rotations (N,4) raw (r,i,j,k) quaternions, log_scales (N,3),
 *     opacity_logits (N,), sh (N,16,3) coefficient-major / channel-minor.
 *     Device arithmetic: float32 storage; the projection geometry (view
 *     transform, EWA covariance, radius, tile rectangle, depth) runs in
 *     float64 so radii, keys and tile ranges match the float64 reference.
 *   - Return value: GS_OK or a GS_ERR_* code.  The Python host layer maps the
 *     codes to the reference's exception types.
 */
#ifndef GS_RASTERIZER_H
#define GS_RASTERIZER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 2
#define GS_TILE_SIZE 16        /* rasterizer.py:13 TILE_SIZE */
#define GS_SH_COEFFS 16        /* sh.py:25 NUM_COEFFS */
#define GS_REC_FLOATS 20       /* floats per projected-splat record, see gs_splats_t */
#define GS_GRAD2D_FLOATS 12    /* floats per screen-space gradient row, see gs_blend_backward */
#define GS_MODEL_FLOATS 59     /* scene_io.py:374-376 model record (236 B) */
#define GS_PLY_FLOATS 62       /* scene_io.py:417-439 PLY vertex */
#define GS_LAYOUT_MODEL 0
#define GS_LAYOUT_PLY 1

enum gs_status {
  GS_OK = 0,
  GS_ERR_INVALID_ARG = 1,      /* ValueError: bad camera / SH degree (core.py:135-141, sh.py:37-38),
                                  backward without training record (rasterizer.py:265-266)          */
  GS_ERR_ZERO_QUATERNION = 2,  /* InvalidPrimitiveError (core.py:164-165)                          */
  GS_ERR_RESOURCE_LIMIT = 3,   /* ResourceLimitError: > 2^32-1 tiles or > 2^31 instances
                                  (rasterizer.py:76-79, 99-101)                                    */
  GS_ERR_CAPACITY = 4,         /* caller's instance buffers hold fewer than K entries;
                                  *k_out carries the K required                                    */
  GS_ERR_CUDA = 5              /* a CUDA runtime error; see gs_last_cuda_error()                    */
};

/* Pinhole camera (core.py:113-146).  View space x-right, y-down, z-forward;
 * pixel centres at (col+0.5, row+0.5). */
typedef struct gs_camera {
  double rotation[9];          /* world-to-view rotation, row-major */
  double translation[3];       /* world-to-view translation */
  double fx, fy, cx, cy;
  int32_t width, height;
  double near_plane;           /* Camera.near, default 0.2 */
} gs_camera_t;

/* Raw Gaussian parameters (GaussianCloud, core.py:36-50), float32, device. */
typedef struct gs_params {
  const float* means;          /* (N,3) */
  const float* rotations;      /* (N,4) raw quaternion, normalised on use */
  const float* log_scales;     /* (N,3) */
  const float* opacity_logits; /* (N,)  */
  const float* sh;             /* (N,16,3) */
  int64_t n;
} gs_params_t;

/* Per-view projected splats, N rows indexed by Gaussian (the device
 * counterpart of ProjectedSplats, core.py:236-263, kept in N-space instead of
 * compacted; a row is a survivor of project() iff radii[row] > 0).
 *
 *   rec (N,20) float32, five 16-byte words per row:
 *     [0..3]   mean2d.x (hi), mean2d.y (hi), mean2d.x (lo), mean2d.y (lo)
 *     [4..7]   conic eigenbasis k = (k1.x, k1.y, k2.x, k2.y), k_i = sqrt(log2(e) lambda_i / 2) e_i,
 *              so log2(e) * power = -(k1.d)^2 - (k2.d)^2 for d = pixel - mean2d
 *     [8..11]  color r, g, b, alpha (hi)
 *     [12..15] conic a, b, c (hi), clamp mask (bits 0..2 as float: channel active)
 *     [16..19] conic a, b, c (lo), alpha (lo)
 *   hi + lo reproduces the float64 value to ~2^-48; the blend kernels gather
 *   words 0..2 per (splat, tile) and read words 3..4 only for the rare pairs
 *   whose alpha sits at a threshold.
 *   depth (N,)  float32 view-space z (the sort key's source, rasterizer.py:61)
 *   radii (N,)  int32 ceil(3 sqrt(lambda_max)), 0 = culled
 *   rect  (N,4) int32 clipped inclusive tile rectangle x0,y0,x1,y1
 *   tiles_touched (N,) int32 (x1-x0+1)(y1-y0+1) or 0 (rasterizer.py:86-97)
 *   status (1,) int32 device word; bit 0 set when a survivor had a zero quaternion.
 * Rows with radii == 0 leave rec/depth/rect undefined. */
typedef struct gs_splats {
  float* rec;
  float* depth;
  int32_t* radii;
  int32_t* rect;
  int32_t* tiles_touched;
  int32_t* status;
  int64_t n;
} gs_splats_t;

/* Parameter gradients (GaussianGrads, gradients.py:13-27), device float32,
 * same shapes as gs_params_t.  view_pos_grad_norm (N,) may be NULL. */
typedef struct gs_grads {
  float* d_means;
  float* d_rotations;
  float* d_log_scales;
  float* d_opacity_logits;
  float* d_sh;
  float* view_pos_grad_norm;
} gs_grads_t;

/* Densification statistics (TrainState, optimizer.py:106-108, updated at
 * optimizer.py:252-255).  Any pointer may be NULL to skip that statistic. */
typedef struct gs_stats {
  float* accum_pos_grad;       /* (N,) += view_pos_grad_norm for survivors */
  int32_t* accum_count;        /* (N,) += 1 for survivors */
  float* max_radius_frac;      /* (N,) = max(., radius / image height) */
} gs_stats_t;

/* One Adam parameter group (optimizer.py:263-293).  Elements whose index e
 * satisfies (e % period) < head use lr_head instead of lr (period a multiple
 * of 4, head <= 4; the SH DC row:
 * period 48, head 3, optimizer.py:268-269).  period <= 0 disables it. */
typedef struct gs_adam_group {
  float* param;
  const float* grad;
  float* exp_avg;
  float* exp_avg_sq;
  int64_t numel;
  float lr;
  float lr_head;
  int32_t period;
  int32_t head;
} gs_adam_group_t;

/* Parameters + Adam moments of a cloud, PARAM_GROUPS order (optimizer.py:85):
 * means (N,3), log_scales (N,3), rotations (N,4), opacity_logits (N,),
 * sh (N,16,3); float32, device. */
typedef struct gs_cloud_state {
  float* param[5];
  float* exp_avg[5];
  float* exp_avg_sq[5];
  int64_t n;
} gs_cloud_state_t;

/* densify_and_prune settings (TrainConfig, optimizer.py:20-70), resolved
 * for one call. */
typedef struct gs_densify_config {
  double grad_threshold;         /* densify_grad_threshold                       */
  double split_scale_threshold;  /* resolve_split_threshold(scene_extent)        */
  double split_log_factor;       /* log(split_factor)                            */
  double prune_alpha;            /* prune_alpha_threshold                        */
  double prune_world_scale;      /* prune_world_percent * scene_extent           */
  double prune_screen_fraction;  /* prune_screen_fraction                        */
  int32_t prune_big;             /* iteration > opacity_reset_interval           */
  int32_t reset_opacity;         /* iteration > 0 && iteration % interval == 0   */
  float reset_logit;             /* logit(opacity_reset_alpha)                   */
} gs_densify_config_t;

/* ---- library info ------------------------------------------------------ */
int gs_abi_version(void);
const char* gs_status_string(int status);
/* Copies the last CUDA error string seen by the library into buf. */
int gs_last_cuda_error(char* buf, size_t len);
/* Diagnostics: FP32 FMA throughput probe used by bench.py as the roofline
 * denominator of the blend kernels (blocks x 256 threads x iters x 8 FMAs;
 * scratch: >= blocks floats, device). */
int gs_fp32_fma_probe(float* scratch, int32_t blocks, int32_t iters, void* stream);

/* ---- K1 preprocess: replaces core.project (core.py:266-345) ------------- */
/* Culls (near plane, guard band, det <= 0), builds the EWA conic, radius,
 * tile rectangle, SH colour and sigmoid opacity for every Gaussian. */
int gs_preprocess_forward(const gs_params_t* params, const gs_camera_t* camera,
                          int32_t active_sh_degree, gs_splats_t* splats, void* stream);

/* ---- K2-K5 binning: replaces rasterizer.bin_and_sort (rasterizer.py:69-124)
 * and make_keys (rasterizer.py:55-62).
 * Orders every (tile, splat) instance by (tile, float32 depth, Gaussian
 * index) — the reference's stable sort on (tile<<32 | depth bits) — and
 * writes the Gaussian id of every sorted instance plus per-tile [start,end)
 * ranges (T,2) int32 (empty tiles [0,0]).  keys (nullable, device uint64
 * (capacity,)) additionally receives the reference's sort key of every
 * sorted instance, (tile << 32) | float32 bits of depth (TileBinning.keys,
 * rasterizer.py:48).  Hand-written kernels only (see binning.cu): a depth
 * radix sort over the Gaussians, super-tile buckets, per-tile lists.
 * gs_bin_and_sort synchronises `stream` once to read K, written to *k_out
 * (host).  Returns GS_ERR_CAPACITY (and K) when k_capacity < K; the
 * instance buffers then hold unspecified values. */
int gs_bin_workspace_size(int64_t n, int32_t width, int32_t height, int64_t k_capacity,
                          size_t* bytes);
int gs_bin_and_sort(const gs_splats_t* splats, int32_t width, int32_t height,
                    void* workspace, size_t workspace_bytes, int64_t k_capacity,
                    uint32_t* sorted_ids, int32_t* ranges, uint64_t* keys, int64_t* k_out, void* stream);
/* Same binning, enqueued without any host synchronisation (CUDA-graph
 * capturable): K never leaves the device.  k_info is a caller-owned DEVICE
 * int64[3]: [0] = K, [1] = flags (1: zero quaternion among the survivors,
 * 2: K > k_capacity, 4: K > 2^31 instances), [2] = min(K, k_capacity).
 * When flags != 0 the ranges stay empty and the caller must check k_info
 * (e.g. one step later) and re-run with a larger capacity / raise. */
int gs_bin_and_sort_async(const gs_splats_t* splats, int32_t width, int32_t height,
                          void* workspace, size_t workspace_bytes, int64_t k_capacity,
                          uint32_t* sorted_ids, int32_t* ranges, uint64_t* keys, int64_t* k_info,
                          void* stream);

/* ---- K6 forward blend: replaces rasterizer.render_forward (rasterizer.py:201-240)
 * image (H,W,3) float32.  When training != 0, t_final (H,W) float32 and
 * last (H,W) int32 (global sorted index of the last blended instance, -1 =
 * none; rasterizer.py:131, 225-231) are written too, and every saturation
 * stop is the reference's float64 decision: pixels whose float32
 * transmittance is within 1e-4 (relative) of the stop are re-blended in
 * float64; scratch (training only, else NULL): device int32[2 + W*H]. */
int gs_blend_forward(const gs_splats_t* splats, const uint32_t* sorted_ids, const int32_t* ranges,
                     int32_t width, int32_t height, const float background[3], int32_t training,
                     float* image, float* t_final, int32_t* last, int32_t* scratch, void* stream);

/* gs_blend_forward with the tiles launched in `tile_order` (nullable; a
 * permutation of [0, tiles), device int32, e.g. the previous backward's
 * longest-first schedule of the same view, or gs_tile_schedule of the
 * previous frame's tile_work).  tile_work (nullable, device int32[tiles])
 * receives each tile's work (splats handed to the blend before it stopped).
 * The outputs do not depend on the order. */
int gs_blend_forward_ordered(const gs_splats_t* splats, const uint32_t* sorted_ids, const int32_t* ranges,
                             int32_t width, int32_t height, const float background[3], int32_t training,
                             const int32_t* tile_order, int32_t* tile_work, float* image, float* t_final,
                             int32_t* last, int32_t* scratch, void* stream);

/* Longest-first tile order from a per-tile work estimate (1/64-octave
 * buckets, heaviest first).  scratch: device int32[tiles + 2048]. */
int gs_tile_schedule(const int32_t* work, int32_t tiles, int32_t* scratch, int32_t* order, void* stream);

/* ---- K7 backward blend: replaces rasterizer.render_backward (rasterizer.py:253-316)
 * with gradients.backward_blend (gradients.py:30-94).
 * grads2d (N,12) float32 is zeroed and then accumulated with the eigenbasis
 * moments of dp = dL/da * a_raw over the offsets v = K (pixel - mean2d)
 * (K = record words 4..7; log2(e) power = -|v|^2):
 *   [0..3]  S1 = sum dp v1, S2 = sum dp v2, S0 = sum dp, 0
 *   [4..7]  M11 = sum dp v1^2, M12 = sum dp v1 v2, M22 = sum dp v2^2, 0
 *   [8..11] d_color r, g, b, 0
 * The reference's SplatGrads2D (rasterizer.py:243-250) follows as
 * d_mean2d = 2 / log2(e) K^T (S1, S2), d_alpha = S0 / alpha and
 * d_conic = (-Q_xx / 2, -Q_xy, -Q_yy / 2) with Q = K^-1 M K^-T
 * (the host mirror's SplatGrads2D properties). */
int gs_blend_backward(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                      const int32_t* ranges, const float* t_final, const int32_t* last,
                      int32_t width, int32_t height, const float background[3],
                      float* grads2d, void* stream);

/* gs_blend_backward with the tiles visited in `tile_order` (a permutation of
 * [0, tiles), device int32). */
int gs_blend_backward_ordered(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                              const int32_t* ranges, const float* t_final, const int32_t* last, int32_t width,
                              int32_t height, const float background[3], const int32_t* tile_order,
                              float* grads2d, void* stream);

/* gs_blend_backward on a longest-first tile schedule built on the device from
 * the training record: a tile's work is max(last contributor) - start + 1
 * (gradients.py:48-52); heavy tiles start first so light ones fill the last
 * wave.  scratch: caller-owned device int32[2 * tiles + 2048]. */
int gs_blend_backward_scheduled(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                                const int32_t* ranges, const float* t_final, const int32_t* last, int32_t width,
                                int32_t height, const float background[3], int32_t* scratch, float* grads2d,
                                void* stream);

/* The two halves of gs_blend_backward_scheduled: the longest-first order into
 * scratch[0, tiles) (scratch: device int32[2 * tiles + 2048]), and the blend
 * kernel alone, accumulating into a caller-cleared grads2d (tile_order
 * nullable: row-major). */
int gs_blend_backward_schedule(const int32_t* ranges, const int32_t* last, int32_t width, int32_t height,
                               int32_t* scratch, void* stream);
int gs_blend_backward_accumulate(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                                 const int32_t* ranges, const float* t_final, const int32_t* last, int32_t width,
                                 int32_t height, const float background[3], const int32_t* tile_order,
                                 float* grads2d, void* stream);

/* Deterministic backward blend (the reference's deterministic=True /
 * workers=1 contract, rasterizer.py:32-41: bit-identical runs): no float
 * atomics — one partial row per (sorted instance, half tile), summed per
 * splat in a fixed order (its tiles row-major, rasterizer.py:105-111).
 * grads2d is fully written (no clearing needed).  tile_order nullable.
 * workspace: gs_blend_backward_det_workspace_size(n, W, H, k_capacity)
 * bytes, k_capacity >= K (the instance buffers' length). */
int gs_blend_backward_det_workspace_size(int64_t n, int32_t width, int32_t height, int64_t k_capacity,
                                         size_t* bytes);
int gs_blend_backward_deterministic(const float* d_image, const gs_splats_t* splats, const uint32_t* sorted_ids,
                                    const int32_t* ranges, const float* t_final, const int32_t* last,
                                    int32_t width, int32_t height, const float background[3],
                                    const int32_t* tile_order, void* workspace, size_t workspace_bytes,
                                    int64_t k_capacity, float* grads2d, void* stream);

/* ---- K8 backward preprocess: replaces gradients.backward_project
 * (gradients.py:192-259) and the densification statistics update of
 * train_step (optimizer.py:252-255).  accumulate = 0 overwrites `grads`
 * (culled rows exactly 0), 1 adds to them (multi-view batches).
 * stats may be NULL. */
int gs_preprocess_backward(const gs_params_t* params, const gs_camera_t* camera,
                           int32_t active_sh_degree, const gs_splats_t* splats,
                           const float* grads2d, const gs_grads_t* grads, int32_t accumulate,
                           const gs_stats_t* stats, void* stream);

/* gs_preprocess_backward leaving the densify statistics untouched when
 * *skip != 0 (device int32 from gs_step_guard, e.g. max-reduced over the
 * ranks): a multi-view step enqueues its backward before the host has read
 * the loss (optimizer.py:245-246 raises before any update). */
int gs_preprocess_backward_guarded(const gs_params_t* params, const gs_camera_t* camera,
                                   int32_t active_sh_degree, const gs_splats_t* splats,
                                   const float* grads2d, const gs_grads_t* grads, int32_t accumulate,
                                   const gs_stats_t* stats, const int32_t* skip, void* stream);

/* ---- K8+K9 fused: backward_project + densify statistics + dense Adam in one
 * pass (gradients.py:192-259, optimizer.py:252-257 and 263-293 back to back,
 * as train_step runs them).  The parameters in *params are UPDATED IN PLACE.
 * groups[5] in PARAM_GROUPS order (means, log_scales, rotations,
 * opacity_logits, sh; optimizer.py:85): exp_avg / exp_avg_sq / lr are used
 * (groups[4].lr_head = SH DC learning rate); param / grad fields are ignored.
 * grads_out (nullable, any member nullable) additionally receives the
 * gradients.  Bit-identical to gs_preprocess_backward + gs_adam_step. */
int gs_preprocess_backward_adam(const gs_params_t* params, const gs_camera_t* camera,
                                int32_t active_sh_degree, const gs_splats_t* splats, const float* grads2d,
                                const gs_adam_group_t* groups, double beta1, double beta2, double eps,
                                double bias1, double bias2, const gs_stats_t* stats,
                                const gs_grads_t* grads_out, void* stream);

/* The same with a device-side step guard: when *skip != 0 (device int32,
 * written by gs_step_guard on the same stream) the launch applies nothing.
 * Lets a training step enqueue its backward and Adam before the host has
 * read the loss: the reference's divergence check (optimizer.py:245-246,
 * raise before any update) and the binning-capacity retry stay exact. */
int gs_preprocess_backward_adam_guarded(const gs_params_t* params, const gs_camera_t* camera,
                                        int32_t active_sh_degree, const gs_splats_t* splats,
                                        const float* grads2d, const gs_adam_group_t* groups, double beta1,
                                        double beta2, double eps, double bias1, double bias2,
                                        const gs_stats_t* stats, const gs_grads_t* grads_out,
                                        const int32_t* skip, void* stream);

/* gs_preprocess_backward_adam_guarded that ALSO projects the updated
 * parameters for the next iteration's view (gs_preprocess_forward with
 * next_camera / next_active_sh_degree into next_splats, bit-identical to
 * calling it after this launch), from the values the update leaves in
 * registers and shared memory: the next forward skips K1 and its 236-B
 * parameter read per Gaussian (optimizer.py:222-260 steps i and i+1 run
 * back to back).  When *skip != 0 nothing is updated and the next view is
 * projected from the unchanged parameters.  next_splats must not alias
 * splats (this step's records are still read). */
int gs_preprocess_backward_adam_project(const gs_params_t* params, const gs_camera_t* camera,
                                        int32_t active_sh_degree, const gs_splats_t* splats,
                                        const float* grads2d, const gs_adam_group_t* groups, double beta1,
                                        double beta2, double eps, double bias1, double bias2,
                                        const gs_stats_t* stats, const gs_grads_t* grads_out,
                                        const int32_t* skip, const gs_camera_t* next_camera,
                                        int32_t next_active_sh_degree, gs_splats_t* next_splats, void* stream);

/* *skip =(k_info[1] != 0 (binning overflow / limit flags) || loss[0] not finite).
 * report (nullable; 8 doubles, device memory or mapped pinned host memory):
 * [loss[0..3], k_info[0..2], skip] -- the step's one host read, without a
 * separate copy. */
int gs_step_guard(const float* loss, const int64_t* k_info, int32_t* skip, double* report, void* stream);

/* ---- K9 fused Adam: replaces optimizer._adam_step (optimizer.py:263-293)
 * over all groups in one launch; bias1 = 1-beta1^t, bias2 = 1-beta2^t. */
int gs_adam_step(const gs_adam_group_t* groups, int32_t num_groups, double beta1, double beta2,
                 double eps, double bias1, double bias2, void* stream);
/* gs_adam_step applying nothing when *skip != 0 (device int32). */
int gs_adam_step_guarded(const gs_adam_group_t* groups, int32_t num_groups, double beta1, double beta2,
                         double eps, double bias1, double bias2, const int32_t* skip, void* stream);

/* ---- fused single-call stages --------------------------
 * gs_forward = gs_preprocess_forward + gs_bin_and_sort_async +
 * gs_blend_forward_ordered (render_view, optimizer.py:212-219): no host
 * synchronisation; K and the flags land in k_info (see
 * gs_bin_and_sort_async), tile_order nullable, scratch as gs_blend_forward.
 * gs_backward = the backward blend (longest-first when sched_scratch, device
 * int32[2 T + 2048], is given) + gs_preprocess_backward (render_backward +
 * backward_project, rasterizer.py:253-316, gradients.py:192-259); grads
 * overwritten, stats nullable. */
int gs_forward(const gs_params_t* params, const gs_camera_t* camera, int32_t active_sh_degree,
               gs_splats_t* splats, void* bin_workspace, size_t bin_workspace_bytes, int64_t k_capacity,
               uint32_t* sorted_ids, int32_t* ranges, int64_t* k_info, const float background[3],
               int32_t training, const int32_t* tile_order, float* image, float* t_final, int32_t* last,
               int32_t* scratch, void* stream);
int gs_backward(const float* d_image, const gs_params_t* params, const gs_camera_t* camera,
                int32_t active_sh_degree, const gs_splats_t* splats, const uint32_t* sorted_ids,
                const int32_t* ranges, const float* t_final, const int32_t* last, const float background[3],
                int32_t* sched_scratch, float* grads2d, const gs_grads_t* grads, const gs_stats_t* stats,
                void* stream);
/* gs_backward after its setup was enqueued ahead (gs_blend_backward_schedule
 * into sched_scratch and grads2d cleared, e.g. on a side stream while the
 * loss runs): gs_blend_backward_accumulate + gs_preprocess_backward. */
int gs_backward_prepared(const float* d_image, const gs_params_t* params, const gs_camera_t* camera,
                         int32_t active_sh_degree, const gs_splats_t* splats, const uint32_t* sorted_ids,
                         const int32_t* ranges, const float* t_final, const int32_t* last,
                         const float background[3], const int32_t* sched_scratch, float* grads2d,
                         const gs_grads_t* grads, const gs_stats_t* stats, void* stream);

/* ---- adaptive density control: replaces
 * optimizer.densify_and_prune (optimizer.py:304-374).
 * gs_densify_classify counts clones and splits (synchronises `stream`);
 * the caller then draws z = rng.standard_normal((2*n_split, 3)) from the
 * training RNG (optimizer.py:335), uploads it (float32, device) and calls
 * gs_densify_apply, which writes the densified, pruned, (opacity-reset)
 * cloud and its moments into `out` (capacity >= N - n_split + n_clone +
 * 2 n_split rows) in the reference's row order and reports the surviving
 * row count (synchronises).  Densify statistics are left to the caller to
 * reset (optimizer.py:372). */
int gs_densify_workspace_size(int64_t n, size_t* bytes);
int gs_densify_classify(const gs_cloud_state_t* cloud, const gs_stats_t* stats, const gs_densify_config_t* cfg,
                        void* workspace, size_t workspace_bytes, int64_t* n_clone, int64_t* n_split, void* stream);
int gs_densify_apply(const gs_cloud_state_t* cloud, const gs_stats_t* stats, const gs_densify_config_t* cfg,
                     int64_t n_clone, int64_t n_split, const float* z, void* workspace, size_t workspace_bytes,
                     gs_cloud_state_t* out, int64_t* n_out, void* stream);

/* ---- training loss: replaces optimizer.loss
 * (optimizer.py:141-163) with ssim_map/ssim_backward (ssim.py:50-84).
 * image, target (H,W,3) float32; loss_out (4,) float32 device:
 * [total loss, mean |image-target|, mean SSIM, mean squared error (the
 * step's PSNR, optimizer.py:257-259)]; d_image (H,W,3) float32 =
 * d loss / d image.  workspace: gs_loss_workspace_size bytes, device. */
int gs_loss_workspace_size(int32_t width, int32_t height, size_t* bytes);
int gs_l1_dssim_loss(const float* image, const float* target, int32_t width, int32_t height, double lambda_dssim,
                     void* workspace, size_t workspace_bytes, float* loss_out, float* d_image, void* stream);

/* ---- model / PLY records: replaces scene_io
 * _records_from_cloud / _cloud_from_records (scene_io.py:377-391) and the
 * export_ply vertex packing (scene_io.py:417-439).  `out` / `records` are
 * DEVICE arrays of n x GS_MODEL_FLOATS (layout GS_LAYOUT_MODEL: mean,
 * log_scale, rotation, opacity, SH channel-major) or n x GS_PLY_FLOATS
 * (GS_LAYOUT_PLY: x y z, zero normals, f_dc, f_rest channel-major, opacity,
 * scale, rot) little-endian float32, i.e. the file body byte for byte. */
int gs_pack_records(const gs_params_t* params, int32_t layout, float* out, void* stream);
int gs_unpack_records(const float* records, gs_params_t* params_out, void* stream);

/* ---- initialisation: replaces scene_io.mean_knn_distance
 * (scene_io.py:304-311; scipy cKDTree, k + 1 neighbours with the self
 * match dropped), the per-point scale of init_from_sfm / init_random
 * (scene_io.py:314-366).  points: DEVICE (n,3) float64; out: DEVICE (n,)
 * float32 mean distance to the k nearest other points (exact, float64
 * distances, uniform-grid shell search).  Requires n > k; 1 <= k <= 16;
 * max_cells bounds the grid (e.g. 2 n).  Synchronises `stream` once to read
 * the bounding box. */
int gs_knn_workspace_size(int64_t n, int64_t max_cells, size_t* bytes);
int gs_knn_mean_distance(const double* points, int64_t n, int32_t k, int64_t max_cells, void* workspace,
                         size_t workspace_bytes, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GS_RASTERIZER_H */
