// K9 adam_fused — replaces splatlab optimizer._adam_step (optimizer.py:263-293).
//
// One launch updates every parameter group.  Dense over all N rows, exactly
// like the reference (culled rows with zero gradient still decay their
// moments and move).  Each thread handles 4 consecutive elements of one
// group with 16-byte vector loads where the group is 16-byte aligned.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kMaxGroups = 8;

struct AdamArgs {
  gs_adam_group_t g[kMaxGroups];
  int64_t quad_start[kMaxGroups + 1];  // prefix over ceil(numel/4)
  int num_groups;
  float beta1, beta2, one_m_beta1, one_m_beta2, eps;
  float inv_bias1, inv_bias2;
};

__device__ __forceinline__ void adam_elem(float& p, float gr, float& m, float& v, float lr, const AdamArgs& a) {
  adam_update(p, gr, m, v, lr, AdamCoef{a.beta1, a.beta2, a.one_m_beta1, a.one_m_beta2, a.eps, a.inv_bias1,
                                        a.inv_bias2});
}

__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a, const int32_t* __restrict__ skip) {
  pdl_begin();
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= a.quad_start[a.num_groups]) return;
  if (skip != nullptr && *skip != 0) return;   // the step guard (gs_step_guard) vetoed this step
  int gi = 0;
  while (gi + 1 < a.num_groups && q >= a.quad_start[gi + 1]) ++gi;
  const gs_adam_group_t& G = a.g[gi];
  const int64_t e0 = (q - a.quad_start[gi]) * 4;
  // period % 4 == 0 (checked on the host): the quad is a row head iff its quad
  // index is a multiple of period / 4; components c < head then use lr_head
  const bool head_quad = G.period > 0 && uint32_t((q - a.quad_start[gi]) % uint32_t(G.period / 4)) == 0u;
  const bool vec = ((reinterpret_cast<uintptr_t>(G.param) | reinterpret_cast<uintptr_t>(G.grad) |
                     reinterpret_cast<uintptr_t>(G.exp_avg) | reinterpret_cast<uintptr_t>(G.exp_avg_sq)) & 15) == 0;
  if (vec && e0 + 4 <= G.numel) {
    float4 p = *reinterpret_cast<const float4*>(G.param + e0);
    const float4 gr = *reinterpret_cast<const float4*>(G.grad + e0);
    float4 m = *reinterpret_cast<const float4*>(G.exp_avg + e0);
    float4 v = *reinterpret_cast<const float4*>(G.exp_avg_sq + e0);
    float* pp = &p.x; const float* pg = &gr.x; float* pm = &m.x; float* pv = &v.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = e0 + k;
      const float lr = (head_quad && k < G.head) ? G.lr_head : G.lr;
      adam_elem(pp[k], pg[k], pm[k], pv[k], lr, a);
    }
    *reinterpret_cast<float4*>(G.param + e0) = p;
    *reinterpret_cast<float4*>(G.exp_avg + e0) = m;
    *reinterpret_cast<float4*>(G.exp_avg_sq + e0) = v;
  } else {
    for (int k = 0; k < 4; ++k) {
      const int64_t e = e0 + k;
      if (e >= G.numel) break;
      const float lr = (head_quad && k < G.head) ? G.lr_head : G.lr;
      float p = G.param[e], m = G.exp_avg[e], v = G.exp_avg_sq[e];
      adam_elem(p, G.grad[e], m, v, lr, a);
      G.param[e] = p;
      G.exp_avg[e] = m;
      G.exp_avg_sq[e] = v;
    }
  }
}

}  // namespace
}  // namespace gs

namespace gs {
namespace {
int adam_step(const gs_adam_group_t* groups, int32_t num_groups, double beta1, double beta2, double eps, double bias1,
              double bias2, const int32_t* skip, void* stream) {
  if (!groups || num_groups <= 0 || num_groups > kMaxGroups) return GS_ERR_INVALID_ARG;
  if (!(bias1 > 0) || !(bias2 > 0)) return GS_ERR_INVALID_ARG;
  AdamArgs a;
  a.num_groups = num_groups;
  a.quad_start[0] = 0;
  for (int i = 0; i < num_groups; ++i) {
    a.g[i] = groups[i];
    if (groups[i].numel < 0 || (groups[i].period > 0 && (groups[i].period % 4 != 0 || groups[i].head > 4)))
      return GS_ERR_INVALID_ARG;
    if (groups[i].numel > 0 &&
        (!groups[i].param || !groups[i].grad || !groups[i].exp_avg || !groups[i].exp_avg_sq))
      return GS_ERR_INVALID_ARG;
    a.quad_start[i + 1] = a.quad_start[i] + (groups[i].numel + 3) / 4;
  }
  a.beta1 = float(beta1);
  a.beta2 = float(beta2);
  a.one_m_beta1 = float(1.0 - beta1);
  a.one_m_beta2 = float(1.0 - beta2);
  a.eps = float(eps);
  a.inv_bias1 = float(1.0 / bias1);
  a.inv_bias2 = float(1.0 / bias2);
  const int64_t quads = a.quad_start[num_groups];
  if (quads == 0) return GS_OK;
  const int block = 256;
  launch_pdl(adam_kernel, unsigned((quads + block - 1) / block), block, 0, static_cast<cudaStream_t>(stream), a, skip);
  return check_launch();
}
}  // namespace
}  // namespace gs

extern "C" int gs_adam_step(const gs_adam_group_t* groups, int32_t num_groups, double beta1, double beta2, double eps,
                            double bias1, double bias2, void* stream) {
  return gs::adam_step(groups, num_groups, beta1, beta2, eps, bias1, bias2, nullptr, stream);
}

// gs_adam_step applying nothing when *skip != 0 (device int32, gs_step_guard)
extern "C" int gs_adam_step_guarded(const gs_adam_group_t* groups, int32_t num_groups, double beta1, double beta2,
                                    double eps, double bias1, double bias2, const int32_t* skip, void* stream) {
  return gs::adam_step(groups, num_groups, beta1, beta2, eps, bias1, bias2, skip, stream);
}
