// Adaptive density control — replaces splatlab optimizer.densify_and_prune
// (optimizer.py:304-374): clone small / split large high-gradient Gaussians,
// prune transparent or oversized ones, optionally reset opacity, keeping the
// Adam moments index-aligned (new rows start with zero moments).
//
// Device pipeline (stream compaction over N x 177 floats of parameters and
// moments):
//   classify   per Gaussian: hot / clone / split flags (optimizer.py:315-323),
//              counts to the host (one sync: the host then draws the split
//              samples from the reference's own RNG stream, optimizer.py:335)
//   rank scan  one 64-bit exclusive scan gives keep and clone ranks at once
//   scatter    inverse maps kept_at / clone_at / split_at
//   virtual    for each row of the densified cloud [kept | clones | children
//              copy 0 | children copy 1] (optimizer.py:326-345) the prune test
//              (optimizer.py:357-360) -> survivor flags
//   compact    exclusive scan of the survivors, then every surviving row is
//              written once (parameters, moments or zeros, opacity reset
//              optimizer.py:368-370).
#include <cub/device/device_scan.cuh>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kWidth[5] = {3, 3, 4, 1, 48};  // means, log_scales, rotations, opacity_logits, sh

struct State {
  float* p[5];
  float* m[5];
  float* v[5];
};

__device__ __forceinline__ int width_of(int gidx) {
  return gidx == 0 ? 3 : gidx == 1 ? 3 : gidx == 2 ? 4 : gidx == 3 ? 1 : 48;
}

__device__ __forceinline__ double max_scale_of(const float* ls) {
  return fmax(fmax(exp(double(ls[0])), exp(double(ls[1]))), exp(double(ls[2])));
}

__global__ void classify_kernel(State s, int64_t n, gs_stats_t stats, gs_densify_config_t cfg, uint8_t* flags,
                                uint64_t* packed, unsigned long long* counters) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int clone = 0, split = 0;
  if (i < n) {
    const int32_t cnt = stats.accum_count[i];
    const double mean_grad = double(stats.accum_pos_grad[i]) / double(cnt > 1 ? cnt : 1);
    const bool hot = (mean_grad > double(cfg.grad_threshold)) && (cnt > 0);
    const bool big = max_scale_of(s.p[1] + 3 * i) > double(cfg.split_scale_threshold);
    split = hot && big;
    clone = hot && !big;
    flags[i] = uint8_t(split ? 2 : clone ? 1 : 0);
    packed[i] = uint64_t(split ? 0 : 1) | (uint64_t(clone) << 32);
  }
  const int nc = __reduce_add_sync(0xffffffffu, clone), ns = __reduce_add_sync(0xffffffffu, split);
  if ((threadIdx.x & 31) == 0) {
    if (nc) atomicAdd(&counters[0], (unsigned long long)nc);
    if (ns) atomicAdd(&counters[1], (unsigned long long)ns);
  }
}

__global__ void scatter_kernel(const uint8_t* flags, const uint64_t* ranks, int64_t n, uint32_t* kept_at,
                               uint32_t* clone_at, uint32_t* split_at) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t r = ranks[i];
  const uint32_t keep_rank = uint32_t(r & 0xffffffffu), clone_rank = uint32_t(r >> 32);
  const uint8_t f = flags[i];
  if (f != 2) kept_at[keep_rank] = uint32_t(i);
  if (f == 1) clone_at[clone_rank] = uint32_t(i);
  if (f == 2) split_at[uint32_t(i) - keep_rank] = uint32_t(i);
}

// Row v of the densified cloud: its source row and kind (0 kept, 1 clone, 2 child).
struct Virtual {
  int64_t n_keep, n_clone, n_split;
  const uint32_t *kept_at, *clone_at, *split_at;
};

__device__ __forceinline__ void source_of(const Virtual& V, int64_t v, uint32_t& src, int& kind, int64_t& child) {
  if (v < V.n_keep) {
    src = V.kept_at[v];
    kind = 0;
  } else if (v < V.n_keep + V.n_clone) {
    src = V.clone_at[v - V.n_keep];
    kind = 1;
  } else {
    child = v - V.n_keep - V.n_clone;  // doubled = concat(parents, parents) (optimizer.py:332)
    src = V.split_at[child % V.n_split];
    kind = 2;
  }
}

// child parameters (optimizer.py:333-343): means + R(q/|q|) (s * z), log_scales - log(split_factor)
__device__ __forceinline__ void child_params(const State& s, uint32_t src, const float* z, double log_factor,
                                             float mean[3], float ls[3]) {
  const float4 qf = reinterpret_cast<const float4*>(s.p[2])[src];
  const double qn = sqrt(double(qf.x) * qf.x + double(qf.y) * qf.y + double(qf.z) * qf.z + double(qf.w) * qf.w);
  double R[9];
  quat_to_rot(qf.x / qn, qf.y / qn, qf.z / qn, qf.w / qn, R);
  const float* pls = s.p[1] + 3 * size_t(src);
  const double sz[3] = {exp(double(pls[0])) * double(z[0]), exp(double(pls[1])) * double(z[1]),
                        exp(double(pls[2])) * double(z[2])};
  const float* pm = s.p[0] + 3 * size_t(src);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    mean[r] = float(double(pm[r]) + (R[3 * r + 0] * sz[0] + R[3 * r + 1] * sz[1] + R[3 * r + 2] * sz[2]));
    ls[r] = float(double(pls[r]) - log_factor);
  }
}

__global__ void prune_kernel(State s, Virtual V, const float* z, const float* max_radius_frac, gs_densify_config_t cfg,
                             int64_t total, uint32_t* survive) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= total) return;
  uint32_t src;
  int kind;
  int64_t child = 0;
  source_of(V, v, src, kind, child);
  // sigmoid(opacity) < threshold (optimizer.py:357)
  const double alpha = 1.0 / (1.0 + exp(-double(s.p[3][src])));
  bool prune = alpha < double(cfg.prune_alpha);
  if (cfg.prune_big) {  // optimizer.py:358-360
    double max_scale;
    if (kind == 2) {  // the child's float64 log scales, as the reference tests them
      const float* pls = s.p[1] + 3 * size_t(src);
      max_scale = fmax(fmax(exp(double(pls[0]) - cfg.split_log_factor), exp(double(pls[1]) - cfg.split_log_factor)),
                       exp(double(pls[2]) - cfg.split_log_factor));
    } else {
      max_scale = max_scale_of(s.p[1] + 3 * size_t(src));
    }
    const double radius = (kind == 0 && max_radius_frac) ? double(max_radius_frac[src]) : 0.0;
    prune = prune || (max_scale > double(cfg.prune_world_scale)) || (radius > double(cfg.prune_screen_fraction));
  }
  survive[v] = prune ? 0u : 1u;
}

__global__ void write_kernel(State s, Virtual V, const float* z, gs_densify_config_t cfg, int64_t total,
                             const uint32_t* survive, const uint32_t* final_index, State out) {
  const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= total || !survive[v]) return;
  uint32_t src;
  int kind;
  int64_t child = 0;
  source_of(V, v, src, kind, child);
  const int64_t d = final_index[v];
  float cm[3], cls[3];
  if (kind == 2) child_params(s, src, z + 3 * child, cfg.split_log_factor, cm, cls);
#pragma unroll
  for (int gi = 0; gi < 5; ++gi) {
    const int w = width_of(gi);
    const float* sp = s.p[gi] + w * size_t(src);
    float* dp = out.p[gi] + w * size_t(d);
    float* dm = out.m[gi] + w * size_t(d);
    float* dv = out.v[gi] + w * size_t(d);
    const float* sm = s.m[gi] + w * size_t(src);
    const float* sv = s.v[gi] + w * size_t(src);
    for (int k = 0; k < w; ++k) {
      float val = sp[k];
      if (kind == 2 && gi == 0) val = cm[k];
      if (kind == 2 && gi == 1) val = cls[k];
      if (gi == 3 && cfg.reset_opacity) val = cfg.reset_logit;  // optimizer.py:368-370
      dp[k] = val;
      dm[k] = kind == 0 ? sm[k] : 0.0f;  // new Gaussians start with zero moments
      dv[k] = kind == 0 ? sv[k] : 0.0f;
    }
  }
}

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t flags, packed, ranks, kept_at, clone_at, split_at, survive, final_index, counters, temp, bytes;
};

int make_layout(int64_t n, Layout* L) {
  const int64_t m = 2 * (n > 0 ? n : 1);
  size_t t1 = 0, t2 = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, t1, (const uint64_t*)nullptr, (uint64_t*)nullptr, int(n > 0 ? n : 1));
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cub::DeviceScan::ExclusiveSum(nullptr, t2, (const uint32_t*)nullptr, (uint32_t*)nullptr, int(m));
  if (e != cudaSuccess) return record_cuda_error(e);
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += align_up(b); return o; };
  const size_t un = size_t(n > 0 ? n : 1);
  L->flags = take(un);
  L->packed = take(8 * un);
  L->ranks = take(8 * un);
  L->kept_at = take(4 * un);
  L->clone_at = take(4 * un);
  L->split_at = take(4 * un);
  L->survive = take(4 * size_t(m));
  L->final_index = take(4 * size_t(m));
  L->counters = take(32);
  L->temp = take(t1 > t2 ? t1 : t2);
  L->bytes = off;
  return GS_OK;
}

State to_state(const gs_cloud_state_t& c) {
  State s;
  for (int g = 0; g < 5; ++g) {
    s.p[g] = c.param[g];
    s.m[g] = c.exp_avg[g];
    s.v[g] = c.exp_avg_sq[g];
  }
  return s;
}

}  // namespace
}  // namespace gs

extern "C" int gs_densify_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0 || n > int64_t(INT32_MAX) / 2) return GS_ERR_INVALID_ARG;
  gs::Layout L;
  int st = gs::make_layout(n, &L);
  if (st != GS_OK) return st;
  *bytes = L.bytes;
  return GS_OK;
}

extern "C" int gs_densify_classify(const gs_cloud_state_t* cloud, const gs_stats_t* stats,
                                   const gs_densify_config_t* cfg, void* workspace, size_t workspace_bytes,
                                   int64_t* n_clone, int64_t* n_split, void* stream) {
  using namespace gs;
  if (!cloud || !stats || !cfg || !n_clone || !n_split || !stats->accum_pos_grad || !stats->accum_count)
    return GS_ERR_INVALID_ARG;
  const int64_t n = cloud->n;
  Layout L;
  int st = make_layout(n, &L);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(workspace);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  cudaError_t e = cudaMemsetAsync(counters, 0, 32, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  *n_clone = *n_split = 0;
  if (n == 0) return GS_OK;
  classify_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(to_state(*cloud), n, *stats, *cfg,
                                                            reinterpret_cast<uint8_t*>(ws + L.flags),
                                                            reinterpret_cast<uint64_t*>(ws + L.packed), counters);
  if ((st = check_launch()) != GS_OK) return st;
  unsigned long long host[2] = {0, 0};
  e = cudaMemcpyAsync(host, counters, sizeof(host), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return record_cuda_error(e);
  *n_clone = int64_t(host[0]);
  *n_split = int64_t(host[1]);
  return GS_OK;
}

extern "C" int gs_densify_apply(const gs_cloud_state_t* cloud, const gs_stats_t* stats, const gs_densify_config_t* cfg,
                                int64_t n_clone, int64_t n_split, const float* z, void* workspace,
                                size_t workspace_bytes, gs_cloud_state_t* out, int64_t* n_out, void* stream) {
  using namespace gs;
  if (!cloud || !cfg || !out || !n_out || (n_split > 0 && !z)) return GS_ERR_INVALID_ARG;
  const int64_t n = cloud->n;
  const int64_t n_keep = n - n_split;
  const int64_t total = n_keep + n_clone + 2 * n_split;
  if (n_clone < 0 || n_split < 0 || n_keep < 0 || out->n < total) return GS_ERR_INVALID_ARG;
  Layout L;
  int st = make_layout(n, &L);
  if (st != GS_OK) return st;
  if (!workspace || workspace_bytes < L.bytes) return GS_ERR_INVALID_ARG;
  char* ws = static_cast<char*>(workspace);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  *n_out = 0;
  if (total == 0) return GS_OK;
  auto* flags = reinterpret_cast<uint8_t*>(ws + L.flags);
  auto* packed = reinterpret_cast<uint64_t*>(ws + L.packed);
  auto* ranks = reinterpret_cast<uint64_t*>(ws + L.ranks);
  auto* kept_at = reinterpret_cast<uint32_t*>(ws + L.kept_at);
  auto* clone_at = reinterpret_cast<uint32_t*>(ws + L.clone_at);
  auto* split_at = reinterpret_cast<uint32_t*>(ws + L.split_at);
  auto* survive = reinterpret_cast<uint32_t*>(ws + L.survive);
  auto* final_index = reinterpret_cast<uint32_t*>(ws + L.final_index);
  void* temp = ws + L.temp;
  size_t temp_bytes = workspace_bytes - L.temp;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, packed, ranks, int(n), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  scatter_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(flags, ranks, n, kept_at, clone_at, split_at);
  if ((st = check_launch()) != GS_OK) return st;
  const Virtual V{n_keep, n_clone, n_split, kept_at, clone_at, split_at};
  const State S = to_state(*cloud);
  const unsigned gt = unsigned((total + 255) / 256);
  prune_kernel<<<gt, 256, 0, s>>>(S, V, z, stats ? stats->max_radius_frac : nullptr, *cfg, total, survive);
  if ((st = check_launch()) != GS_OK) return st;
  temp_bytes = workspace_bytes - L.temp;
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, survive, final_index, int(total), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  write_kernel<<<gt, 256, 0, s>>>(S, V, z, *cfg, total, survive, final_index, to_state(*out));
  if ((st = check_launch()) != GS_OK) return st;
  uint32_t last_idx = 0, last_surv = 0;
  e = cudaMemcpyAsync(&last_idx, final_index + total - 1, 4, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cudaMemcpyAsync(&last_surv, survive + total - 1, 4, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return record_cuda_error(e);
  *n_out = int64_t(last_idx) + int64_t(last_surv);
  return GS_OK;
}
