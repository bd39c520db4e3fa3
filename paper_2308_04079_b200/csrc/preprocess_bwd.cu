// K8 preprocess_bwd — replaces splatlab gradients.backward_project
// (gradients.py:192-259, with backward_invert_cov2d 97-113,
// backward_conic_to_cov3d 116-123, backward_cov3d_to_scale_rotation 126-189,
// sh_basis_jacobian sh.py:66-109) and the densification statistics update of
// optimizer.train_step (optimizer.py:252-255).
//
// One thread per Gaussian.  Nothing from the forward's geometry is cached:
// the view position, J, U = JW, Sigma and the conic are recomputed from the
// parameters (cheaper in HBM bytes than storing the reference's 40-float
// backward cache per splat); precision per stage: see GS_BWD_REAL.  The SH path reuses the
// forward's float32 basis and the stored clamp mask.
#include "project.cuh"

namespace gs {
namespace {

// Gradients of one surviving Gaussian g.  Writes the non-SH outputs and the
// statistics; returns the SH basis b and the masked colour gradient dcol,
// whose outer product is the (16,3) d_sh row (written by the caller through
// shared memory).  shrow: the Gaussian's staged SH coefficients.
// Per-Gaussian inputs, loaded before the block's SH staging so their
// latency overlaps it.
struct GradInputs {
  float4 ga, gb, gc;   // grads2d row: moments (S1, S2, S0), conic moments (M11, M12, M22), (d_r, d_g, d_b)
  float4 k;            // the conic's eigenbasis rows (record word 1) the blends built the exponent from
  float4 q;            // raw quaternion
  float m0, m1, m2, l0, l1, l2, op, mask;
};

__device__ __forceinline__ void load_inputs(const gs_params_t& p, const float4* __restrict__ rec,
                                            const float4* __restrict__ g2d, int64_t g, GradInputs& in) {
  in.ga = __ldg(g2d + 3 * g + 0);
  in.gb = __ldg(g2d + 3 * g + 1);
  in.gc = __ldg(g2d + 3 * g + 2);
  in.mask = __ldg(rec + kRecWords * g + 3).w;
  in.k = __ldg(rec + kRecWords * g + 1);
  in.q = __ldg(reinterpret_cast<const float4*>(p.rotations) + g);
  in.m0 = __ldg(p.means + 3 * g + 0); in.m1 = __ldg(p.means + 3 * g + 1); in.m2 = __ldg(p.means + 3 * g + 2);
  in.l0 = __ldg(p.log_scales + 3 * g + 0); in.l1 = __ldg(p.log_scales + 3 * g + 1);
  in.l2 = __ldg(p.log_scales + 3 * g + 2);
  in.op = __ldg(p.opacity_logits + g);
}

// Non-SH gradients of one Gaussian (the SH row is b (x) dcol).
struct GradOut {
  float dmean[3];
  float dlogs[3];
  float4 drot;
  float dlogit;
  float norm;   // view_pos_grad_norm = |d_mean2d| (gradients.py:258)
};

__device__ __forceinline__ void zero_grads(GradOut& o) {
  o.dmean[0] = o.dmean[1] = o.dmean[2] = 0.0f;
  o.dlogs[0] = o.dlogs[1] = o.dlogs[2] = 0.0f;
  o.drot = make_float4(0.f, 0.f, 0.f, 0.f);
  o.dlogit = 0.0f;
  o.norm = 0.0f;
}

template <typename Real>
__device__ __forceinline__ void grad_one_t(const GradInputs& in, const DevCamera& cam, int degree,
                                         const float4* shrow, GradOut& o, float (&b)[16], float (&dcol)[3]) {
  Real cR[9], ct[3], ccen[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) cR[k] = Real(cam.R[k]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ct[k] = Real(cam.t[k]);
    ccen[k] = Real(cam.center[k]);
  }
  const Real cfx = Real(cam.fx), cfy = Real(cam.fy);
  const float4 ga = in.ga, gb = in.gb, gc = in.gc;
  const int mask = int(in.mask);

  // --- opacity through the sigmoid (gradients.py:217): d_alpha = S0 / alpha
  //     (S0 = sum dL/da a_raw with a_raw = alpha g), so d_logit = S0 (1 - alpha)
  const Real alpha = Real(1.0) / (Real(1.0) + exp(-Real(in.op)));
  const float d_logit = float(Real(ga.z) * (Real(1.0) - alpha));

  // --- view position, Jacobian, U = J W (core.py:279, 298-303)
  const Real mx = in.m0, my = in.m1, mz = in.m2;
  Real view[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    view[i] = mx * cR[3 * i + 0] + my * cR[3 * i + 1] + mz * cR[3 * i + 2] + ct[i];
  const Real x = view[0], y = view[1], z = view[2];
  // gradients only from here on (no integer is decided): reciprocals are
  // formed once and multiplied, ~1e-16 relative from the divided form
  const Real inv_z = Real(1.0) / z, inv_z2 = inv_z * inv_z, inv_z3 = inv_z2 * inv_z;
  const Real j00 = cfx * inv_z, j02 = -cfx * x * inv_z2, j11 = cfy * inv_z, j12 = -cfy * y * inv_z2;
  Real U[6];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    U[c] = j00 * cR[c] + j02 * cR[6 + c];
    U[3 + c] = j11 * cR[3 + c] + j12 * cR[6 + c];
  }

  // --- covariance from the raw quaternion and log scales (core.py:187-201),
  //     always float64: the rotation gradient below relies on R R^T = I and
  //     a symmetric dSigma to cancel (to ~1e-16 of |d log_scale| for isotropic Gaussians)
  using Cov = double;
  const float4 qf = in.q;
  const Cov qn = sqrt(Cov(qf.x) * qf.x + Cov(qf.y) * qf.y + Cov(qf.z) * qf.z + Cov(qf.w) * qf.w);
  const Cov q[4] = {qf.x / qn, qf.y / qn, qf.z / qn, qf.w / qn};
  Cov R[9];
  quat_to_rot(q[0], q[1], q[2], q[3], R);
  const Cov s[3] = {exp(Cov(in.l0)), exp(Cov(in.l1)), exp(Cov(in.l2))};
  Cov M[9];
  Real S[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) M[3 * i + j] = R[3 * i + j] * s[j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      S[3 * i + k] = Real(M[3 * i + 0] * M[3 * k + 0] + M[3 * i + 1] * M[3 * k + 1] + M[3 * i + 2] * M[3 * k + 2]);
  Real US[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) US[3 * r + k] = U[3 * r + 0] * S[k] + U[3 * r + 1] * S[3 + k] + U[3 * r + 2] * S[6 + k];
  // --- conic moments -> floored screen covariance.  The reference forms
  //     d_conic = -1/2 sum dp d d^T and dS' = -A G A (gradients.py:97-113);
  //     with d = K^-1 v and A = 2 / log2(e) K^T K (the blends' exponent,
  //     gs_common.cuh: conic_basis) that is dS' = 2 / log2(e)^2 K^T M K,
  //     which never mixes the axes' magnitudes (see blend_bwd.cu).
  const Real k1x = in.k.x, k1y = in.k.y, k2x = in.k.z, k2y = in.k.w;
  const Real M11 = gb.x, M12 = gb.y, M22 = gb.z;
  const Real P1x = M11 * k1x + M12 * k2x, P1y = M11 * k1y + M12 * k2y;
  const Real P2x = M12 * k1x + M22 * k2x, P2y = M12 * k1y + M22 * k2y;
  const Real cm = Real(2.0 / (1.4426950408889634 * 1.4426950408889634));
  const Real dC00 = cm * (k1x * P1x + k2x * P2x);
  const Real dC01 = cm * (k1x * P1y + k2x * P2y);
  const Real dC10 = dC01;
  const Real dC11 = cm * (k1y * P1y + k2y * P2y);
  // d_mean2d = 2 / log2(e) K^T (S1, S2) from the row's moments (float32, like
  // the per-pixel products the blends summed before)
  const float fmx = (2.0f / 1.4426950408889634f) * fmaf(in.k.x, ga.x, in.k.z * ga.y);
  const float fmy = (2.0f / 1.4426950408889634f) * fmaf(in.k.y, ga.x, in.k.w * ga.y);

  // --- screen covariance -> world covariance: dSigma = U^T dS' U (gradients.py:116-123)
  Real dCU[6];  // dS' U  (2x3)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dCU[c] = dC00 * U[c] + dC01 * U[3 + c];
    dCU[3 + c] = dC10 * U[c] + dC11 * U[3 + c];
  }
  Real dS[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dS[3 * i + j] = U[i] * dCU[j] + U[3 + i] * dCU[3 + j];

  // --- Sigma = M M^T -> log scales and raw quaternion (gradients.py:126-189), float64
  Cov dSs[9];  // symmetrised dSigma
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dSs[3 * i + j] = Cov(0.5) * (Cov(dS[3 * i + j]) + Cov(dS[3 * j + i]));
  Cov dM[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dM[3 * i + k] = Cov(2.0) * (dSs[3 * i + 0] * M[0 + k] + dSs[3 * i + 1] * M[3 + k] + dSs[3 * i + 2] * M[6 + k]);
  Cov d_logs[3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    d_logs[k] = (dM[k] * R[k] + dM[3 + k] * R[3 + k] + dM[6 + k] * R[6 + k]) * s[k];
  // dR = dM * diag(s); contract with dR/dq of quat_to_rot
  Cov dR[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dR[3 * i + j] = dM[3 * i + j] * s[j];
  const Cov qr = q[0], qi = q[1], qj = q[2], qk = q[3];
  const Cov dqr = Cov(2.0) * (-qk * dR[1] + qj * dR[2] + qk * dR[3] - qi * dR[5] - qj * dR[6] + qi * dR[7]);
  const Cov dqi = Cov(2.0) * (qj * dR[1] + qk * dR[2] + qj * dR[3] - Cov(2.0) * qi * dR[4] - qr * dR[5] + qk * dR[6] +
                            qr * dR[7] - Cov(2.0) * qi * dR[8]);
  const Cov dqj = Cov(2.0) * (-Cov(2.0) * qj * dR[0] + qi * dR[1] + qr * dR[2] + qi * dR[3] + qk * dR[5] - qr * dR[6] +
                            qk * dR[7] - Cov(2.0) * qj * dR[8]);
  const Cov dqk = Cov(2.0) * (-Cov(2.0) * qk * dR[0] - qr * dR[1] + qi * dR[2] + qr * dR[3] - Cov(2.0) * qk * dR[4] +
                            qj * dR[5] + qi * dR[6] + qj * dR[7]);
  const Cov qdot = qr * dqr + qi * dqi + qj * dqj + qk * dqk;
  const Cov inv_qn = Cov(1.0) / qn;
  const float4 d_rot = make_float4(float((dqr - qr * qdot) * inv_qn), float((dqi - qi * qdot) * inv_qn),
                                   float((dqj - qj * qdot) * inv_qn), float((dqk - qk * qdot) * inv_qn));

  // --- view position: J^T d_mean2d plus the dependence of J on the mean
  //     (gradients.py:236-255)
  const Real dmx = fmx, dmy = fmy;
  Real dt[3] = {j00 * dmx, j11 * dmy, j02 * dmx + j12 * dmy};
  Real dU[6];  // 2 dS' U Sigma
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int l = 0; l < 3; ++l)
      dU[3 * r + l] = Real(2.0) * (dCU[3 * r + 0] * S[l] + dCU[3 * r + 1] * S[3 + l] + dCU[3 * r + 2] * S[6 + l]);
  Real dJ[6];  // dU W^T
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dJ[3 * r + k] = dU[3 * r + 0] * cR[3 * k + 0] + dU[3 * r + 1] * cR[3 * k + 1] +
                      dU[3 * r + 2] * cR[3 * k + 2];
  dt[0] += dJ[2] * (-cfx * inv_z2);
  dt[1] += dJ[5] * (-cfy * inv_z2);
  dt[2] += dJ[0] * (-cfx * inv_z2) + dJ[2] * (Real(2.0) * cfx * x * inv_z3) + dJ[4] * (-cfy * inv_z2) +
           dJ[5] * (Real(2.0) * cfy * y * inv_z3);

  // --- colour: clamp mask, SH coefficients, direction path (gradients.py:219-226)
  const Real ddx = mx - ccen[0], ddy = my - ccen[1], ddz = mz - ccen[2];
  const Real dist = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
  const Real inv_dist_r = Real(1.0) / dist;
  const float vx = float(ddx * inv_dist_r), vy = float(ddy * inv_dist_r), vz = float(ddz * inv_dist_r);
  sh_basis(vx, vy, vz, degree, b);
  dcol[0] = (mask & 1) ? gc.x : 0.0f;
  dcol[1] = (mask & 2) ? gc.y : 0.0f;
  dcol[2] = (mask & 4) ? gc.z : 0.0f;
  float shv[48];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const float4 q4 = shrow[k];
    shv[4 * k + 0] = q4.x; shv[4 * k + 1] = q4.y; shv[4 * k + 2] = q4.z; shv[4 * k + 3] = q4.w;
  }
  float db[16];
  const int nrows = (degree + 1) * (degree + 1);
#pragma unroll
  for (int k = 0; k < 16; ++k)
    db[k] = k < nrows ? dcol[0] * shv[3 * k + 0] + dcol[1] * shv[3 * k + 1] + dcol[2] * shv[3 * k + 2] : 0.0f;
  float gdx, gdy, gdz;
  sh_basis_vjp(vx, vy, vz, degree, db, gdx, gdy, gdz);
  const float vdot = vx * gdx + vy * gdy + vz * gdz;
  const float inv_dist = float(inv_dist_r);
  const float dms[3] = {(gdx - vx * vdot) * inv_dist, (gdy - vy * vdot) * inv_dist, (gdz - vz * vdot) * inv_dist};

  // --- d_means = d_t W + d_mean_sh (gradients.py:257)
  float dmean[3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
    dmean[j] = float(dt[0] * cR[j] + dt[1] * cR[3 + j] + dt[2] * cR[6 + j]) + dms[j];
  o.norm = sqrtf(fmx * fmx + fmy * fmy);  // gradients.py:258
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o.dmean[k] = dmean[k];
    o.dlogs[k] = float(d_logs[k]);
  }
  o.drot = d_rot;
  o.dlogit = d_logit;
}

// Precision of the backward projection chain (gradients only: no integer is
// decided here, the forward keeps float64 for radii / keys).  GS_BWD_REAL =
// float runs view position, J, U, the conic and dSigma' in float32; the
// covariance R, M and the dM -> (d log_scale, d quaternion) chain stay
// float64 (see grad_one_t).  The float32 variant was 10% faster but drifted
// 0.1-0.7% from the reference in d_rotations on adversarial fuzz scenes
// (test_fuzz_scenes_vs_oracle), so the default is float64 throughout; the
// cost of float64 is mostly its divisions, formed once as reciprocals
// (fused backward + Adam 1.027 -> 0.933 ms at c3).
#ifndef GS_BWD_REAL
#define GS_BWD_REAL double
#endif
__device__ __forceinline__ void grad_one(const GradInputs& in, const DevCamera& cam, int degree,
                                         const float4* shrow, GradOut& o, float (&b)[16], float (&dcol)[3]) {
  grad_one_t<GS_BWD_REAL>(in, cam, degree, shrow, o, b, dcol);
}

__device__ __forceinline__ void store_grads(const gs_grads_t& out, int64_t g, const GradOut& o, bool accumulate) {
  if (accumulate) {
    for (int k = 0; k < 3; ++k) out.d_means[3 * g + k] += o.dmean[k];
    for (int k = 0; k < 3; ++k) out.d_log_scales[3 * g + k] += o.dlogs[k];
    float4 r = reinterpret_cast<float4*>(out.d_rotations)[g];
    r.x += o.drot.x; r.y += o.drot.y; r.z += o.drot.z; r.w += o.drot.w;
    reinterpret_cast<float4*>(out.d_rotations)[g] = r;
    out.d_opacity_logits[g] += o.dlogit;
  } else {
    for (int k = 0; k < 3; ++k) out.d_means[3 * g + k] = o.dmean[k];
    for (int k = 0; k < 3; ++k) out.d_log_scales[3 * g + k] = o.dlogs[k];
    reinterpret_cast<float4*>(out.d_rotations)[g] = o.drot;
    out.d_opacity_logits[g] = o.dlogit;
  }
  if (out.view_pos_grad_norm) out.view_pos_grad_norm[g] = o.norm;
}

// densification statistics over every survivor (optimizer.py:252-255)
__device__ __forceinline__ void update_stats(const gs_stats_t& stats, int64_t g, float norm, int32_t radius,
                                             int height) {
  if (stats.accum_pos_grad) stats.accum_pos_grad[g] += norm;
  if (stats.accum_count) stats.accum_count[g] += 1;
  if (stats.max_radius_frac) {
    const float frac = float(double(radius) / double(height));
    stats.max_radius_frac[g] = fmaxf(stats.max_radius_frac[g], frac);
  }
}

// d_sh row (gradients.py:221) as float4 k of the (16,3) row: basis (x) dcol
__device__ __forceinline__ float4 dsh_quad(const float (&b)[16], const float (&dcol)[3], int k) {
  const int e0 = 4 * k;
  return make_float4(b[(e0 + 0) / 3] * dcol[(e0 + 0) % 3], b[(e0 + 1) / 3] * dcol[(e0 + 1) % 3],
                     b[(e0 + 2) / 3] * dcol[(e0 + 2) % 3], b[(e0 + 3) / 3] * dcol[(e0 + 3) % 3]);
}

__global__ void __launch_bounds__(128, 4)
preprocess_bwd_kernel(gs_params_t p, DevCamera cam, int degree, const float4* __restrict__ rec,
                      const int32_t* __restrict__ radii, const float4* __restrict__ g2d, gs_grads_t out,
                      int accumulate, gs_stats_t stats, const int32_t* __restrict__ stats_skip) {
  pdl_begin();
  __shared__ float4 s_sh[128 * kShStride];
  if (stats_skip != nullptr && *stats_skip != 0) stats = gs_stats_t{nullptr, nullptr, nullptr};
  const int64_t g0 = int64_t(blockIdx.x) * blockDim.x;
  const int64_t g = g0 + threadIdx.x;
  const bool valid = g < p.n;
  const int32_t radius = valid ? radii[g] : 0;
  GradInputs in;
  if (valid) load_inputs(p, rec, g2d, g, in);
  stage_sh_rows(p.sh, p.n, g0, s_sh);
  __syncthreads();
  float b[16], dcol[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < 16; ++k) b[k] = 0.0f;
  GradOut o;
  if (radius > 0) {
    grad_one(in, cam, degree, s_sh + threadIdx.x * kShStride, o, b, dcol);
    store_grads(out, g, o, accumulate);
    update_stats(stats, g, o.norm, radius, cam.height);
  } else if (valid && !accumulate) {  // culled: exactly zero gradient (gradients.py:13-27)
    zero_grads(o);
    store_grads(out, g, o, false);
  }
  // d_sh = basis (x) masked d_color (gradients.py:221), written through shared
  // memory so the (N,16,3) stores are coalesced
  __syncthreads();
  if (accumulate) {
    stage_sh_rows(out.d_sh, p.n, g0, s_sh);
    __syncthreads();
  }
  if (valid) {
    float4* row = s_sh + threadIdx.x * kShStride;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      float4 v = dsh_quad(b, dcol, k);
      if (accumulate) {
        const float4 o = row[k];
        v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
      }
      row[k] = v;
    }
  }
  __syncthreads();
  store_sh_rows(s_sh, p.n, g0, out.d_sh);
}

// ---------------------------------------------------------------------------
// Fused backward preprocess + densify statistics + dense Adam: the same
// per-Gaussian gradient as preprocess_bwd_kernel, consumed in registers /
// shared memory by the Adam update (optimizer.py:263-293) instead of being
// written to HBM and re-read by a second kernel (saves 472 B per Gaussian).
// Bit-identical to preprocess_bwd_kernel followed by adam_kernel.
struct FusedAdam {
  float* m[5];   // exp_avg:    means, log_scales, rotations, opacity_logits, sh
  float* v[5];   // exp_avg_sq: same order (optimizer.py:85 PARAM_GROUPS)
  float lr[5];
  float lr_sh_dc;
  AdamCoef c;
};

#ifndef GS_BWDADAM_MINB
#define GS_BWDADAM_MINB 5
#endif
#ifndef GS_BWDADAM_SWEEP_U
#define GS_BWDADAM_SWEEP_U 4
#endif
// The next view's projection (kProject): after the update every thread
// stages its Gaussian's new parameters in shared memory (in place of the
// gradients it consumed) and runs K1's per-Gaussian projection on them for
// `ncam`, writing the next forward's splats `nout`, so that forward does not
// re-read the 236 B of parameters per Gaussian the update just wrote.
struct NextView {
  DevCamera cam;
  int degree;
  gs_splats_t out;
};

template <bool kProject>
__global__ void __launch_bounds__(128, GS_BWDADAM_MINB)
preprocess_bwd_adam_kernel(gs_params_t p, DevCamera cam, int degree, const float4* __restrict__ rec,
                           const int32_t* __restrict__ radii, const float4* __restrict__ g2d, gs_grads_t out,
                           gs_stats_t stats, FusedAdam A, const int32_t* __restrict__ skip, NextView next) {
  pdl_begin();
  // device-side step guard (gs_step_guard): a step whose loss is not finite
  // or whose binning overflowed applies nothing — parameters, moments and
  // statistics stay untouched, as the reference raises before updating (the
  // next view is then projected from the unchanged parameters)
  const bool apply = skip == nullptr || *skip == 0;
  if (!kProject && !apply) return;
  extern __shared__ __align__(16) float4 smem4[];
  float4* s_sh = smem4;                      // staged SH coefficients (the SH parameters)
  float4* s_dsh = smem4;  // d_sh rows: each thread overwrites its own SH row after grad_one read it
  float4* s_grot = smem4 + 128 * kShStride;  // (128) rotation grads
  float* s_gmean = reinterpret_cast<float*>(s_grot + 128);  // (128*3)
  float* s_glogs = s_gmean + 128 * 3;                       // (128*3)
  float* s_gop = s_glogs + 128 * 3;                         // (128)
  const int64_t g0 = int64_t(blockIdx.x) * blockDim.x;
  const int64_t g = g0 + threadIdx.x;
  const bool valid = g < p.n;
  const int32_t radius = valid ? radii[g] : 0;
  GradInputs in;
  if (valid) load_inputs(p, rec, g2d, g, in);
  stage_sh_rows(p.sh, p.n, g0, s_sh);
  __syncthreads();
  float b[16], dcol[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < 16; ++k) b[k] = 0.0f;
  GradOut o;
  zero_grads(o);
  if (radius > 0 && apply) {
    grad_one(in, cam, degree, s_sh + threadIdx.x * kShStride, o, b, dcol);
    update_stats(stats, g, o.norm, radius, cam.height);
  }
  // gradients -> shared memory, group-major, so every Adam group below is a
  // coalesced sweep over the block's contiguous span
  const int tid = threadIdx.x;
  if (valid) {
    if (out.d_means && apply) store_grads(out, g, o, false);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      s_gmean[3 * tid + k] = o.dmean[k];
      s_glogs[3 * tid + k] = o.dlogs[k];
    }
    s_grot[tid] = o.drot;
    s_gop[tid] = o.dlogit;
    float4* row = s_dsh + tid * kShStride;
#pragma unroll
    for (int k = 0; k < 12; ++k) row[k] = dsh_quad(b, dcol, k);
  }
  __syncthreads();
  if (out.d_sh && apply) store_sh_rows(s_dsh, p.n, g0, out.d_sh);
  const int64_t left = p.n - g0;
  const int nb = left < int64_t(blockDim.x) ? int(left) : int(blockDim.x);
  {  // dense Adam: means, log_scales (N,3); rotations (N,4); opacity (N,)
    float* __restrict__ pm = const_cast<float*>(p.means) + 3 * g0;
    float* __restrict__ pl = const_cast<float*>(p.log_scales) + 3 * g0;
    float* __restrict__ mm = A.m[0] + 3 * g0;
    float* __restrict__ vm = A.v[0] + 3 * g0;
    float* __restrict__ ml = A.m[1] + 3 * g0;
    float* __restrict__ vl = A.v[1] + 3 * g0;
    // 3 * nb <= 3 * blockDim.x: at most 3 iterations, all loads issued first
    float x[3], m[3], v[3], y[3], m2[3], v2[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int f = tid + u * int(blockDim.x);
      if (f < 3 * nb) {
        x[u] = pm[f]; m[u] = mm[f]; v[u] = vm[f];
        y[u] = pl[f]; m2[u] = ml[f]; v2[u] = vl[f];
      }
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int f = tid + u * int(blockDim.x);
      if (f < 3 * nb && apply) {
        adam_update(x[u], s_gmean[f], m[u], v[u], A.lr[0], A.c);
        adam_update(y[u], s_glogs[f], m2[u], v2[u], A.lr[1], A.c);
        pm[f] = x[u]; mm[f] = m[u]; vm[f] = v[u];
        pl[f] = y[u]; ml[f] = m2[u]; vl[f] = v2[u];
      }
      if (kProject && f < 3 * nb) {   // element f is this thread's alone: the new value replaces its gradient
        s_gmean[f] = x[u];
        s_glogs[f] = y[u];
      }
    }
    if (tid < nb) {
      float4* pr = reinterpret_cast<float4*>(const_cast<float*>(p.rotations)) + g0 + tid;
      float4* mr = reinterpret_cast<float4*>(A.m[2]) + g0 + tid;
      float4* vr = reinterpret_cast<float4*>(A.v[2]) + g0 + tid;
      float4 q = *pr;
      float* po = const_cast<float*>(p.opacity_logits) + g0 + tid;
      float op = *po;
      if (apply) {
        float4 m = *mr, v = *vr;
        const float4 gq = s_grot[tid];
        adam_update(q.x, gq.x, m.x, v.x, A.lr[2], A.c);
        adam_update(q.y, gq.y, m.y, v.y, A.lr[2], A.c);
        adam_update(q.z, gq.z, m.z, v.z, A.lr[2], A.c);
        adam_update(q.w, gq.w, m.w, v.w, A.lr[2], A.c);
        *pr = q; *mr = m; *vr = v;
        float mo = A.m[3][g0 + tid], vo = A.v[3][g0 + tid];
        adam_update(op, s_gop[tid], mo, vo, A.lr[3], A.c);
        *po = op; A.m[3][g0 + tid] = mo; A.v[3][g0 + tid] = vo;
      }
      if (kProject) {   // this thread's own Gaussian
        s_grot[tid] = q;
        s_gop[tid] = op;
      }
    }
  }
  // dense Adam on the SH rows: coalesced float4 sweep over the block's span;
  // element 0..2 of each 48-float row (the DC band) uses lr_sh_dc
  float4* __restrict__ shp = reinterpret_cast<float4*>(const_cast<float*>(p.sh)) + g0 * 12;
  float4* __restrict__ m4 = reinterpret_cast<float4*>(A.m[4]) + g0 * 12;
  float4* __restrict__ v4 = reinterpret_cast<float4*>(A.v[4]) + g0 * 12;
  const int total = nb * 12, step = blockDim.x;
  constexpr int kU = GS_BWDADAM_SWEEP_U;  // kU x 3 float4 loads in flight per thread
  for (int f0 = threadIdx.x; f0 < total; f0 += kU * step) {
    float4 pq[kU], mq[kU], vq[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int f = f0 + u * step;
      if (f < total) {
        pq[u] = shp[f];
        mq[u] = m4[f];
        vq[u] = v4[f];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int f = f0 + u * step;
      if (f >= total) break;
      const int j = f / 12, k = f - j * 12;
      if (apply) {
        const float4 gq = s_dsh[j * kShStride + k];
        const float lr0 = (k == 0) ? A.lr_sh_dc : A.lr[4];
        adam_update(pq[u].x, gq.x, mq[u].x, vq[u].x, lr0, A.c);
        adam_update(pq[u].y, gq.y, mq[u].y, vq[u].y, lr0, A.c);
        adam_update(pq[u].z, gq.z, mq[u].z, vq[u].z, lr0, A.c);
        adam_update(pq[u].w, gq.w, mq[u].w, vq[u].w, A.lr[4], A.c);
        shp[f] = pq[u];
        m4[f] = mq[u];
        v4[f] = vq[u];
      }
      if (kProject) s_dsh[j * kShStride + k] = pq[u];   // the element's new value replaces its gradient
    }
  }
  if (kProject) {
    __syncthreads();
    if (tid < nb) {
      const float4 q = s_grot[tid];
      const float4* row = s_dsh + tid * kShStride;
      project_gaussian(s_gmean[3 * tid + 0], s_gmean[3 * tid + 1], s_gmean[3 * tid + 2], q, s_glogs[3 * tid + 0],
                       s_glogs[3 * tid + 1], s_glogs[3 * tid + 2], s_gop[tid], [&](int k) { return row[k]; },
                       next.cam, next.degree, next.out, g);
    }
  }
}

}  // namespace
}  // namespace gs

namespace {
// shared by the guarded entry and the one that also projects the next view
int launch_backward_adam(const gs_params_t* params, const gs_camera_t* camera, int32_t active_sh_degree,
                         const gs_splats_t* splats, const float* grads2d, const gs_adam_group_t* groups, double beta1,
                         double beta2, double eps, double bias1, double bias2, const gs_stats_t* stats,
                         const gs_grads_t* grads_out, const int32_t* skip, const gs_camera_t* next_camera,
                         int32_t next_degree, gs_splats_t* next_splats, cudaStream_t s) {
  if (!params || !camera || !splats || !grads2d || !groups) return GS_ERR_INVALID_ARG;
  if (active_sh_degree < 0 || active_sh_degree > 3) return GS_ERR_INVALID_ARG;
  if (splats->n != params->n || !(bias1 > 0) || !(bias2 > 0)) return GS_ERR_INVALID_ARG;
  const bool project = next_splats != nullptr;
  if (project) {
    if (!next_camera || next_degree < 0 || next_degree > 3 || next_splats->n != params->n) return GS_ERR_INVALID_ARG;
    if (next_camera->width <= 0 || next_camera->height <= 0 || !(next_camera->fx > 0) || !(next_camera->fy > 0) ||
        !(next_camera->near_plane > 0))
      return GS_ERR_INVALID_ARG;
    if (next_splats->rec == splats->rec) return GS_ERR_INVALID_ARG;   // the kernel still reads this step's records
    cudaError_t e = gs::zero_async(next_splats->status, sizeof(int32_t), nullptr, 0, s);
    if (e != cudaSuccess) return gs::record_cuda_error(e);
  }
  if (params->n == 0) return GS_OK;
  for (int i = 0; i < 5; ++i)
    if (!groups[i].exp_avg || !groups[i].exp_avg_sq) return GS_ERR_INVALID_ARG;
  gs::FusedAdam A;
  for (int i = 0; i < 5; ++i) {
    A.m[i] = groups[i].exp_avg;
    A.v[i] = groups[i].exp_avg_sq;
    A.lr[i] = groups[i].lr;
  }
  A.lr_sh_dc = groups[4].lr_head;
  A.c = gs::AdamCoef{float(beta1), float(beta2), float(1.0 - beta1), float(1.0 - beta2), float(eps),
                     float(1.0 / bias1), float(1.0 / bias2)};
  gs_stats_t st = {nullptr, nullptr, nullptr};
  if (stats) st = *stats;
  gs_grads_t go = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  if (grads_out) go = *grads_out;
  const size_t smem = (128 * gs::kShStride + 128) * sizeof(float4) + 128 * 7 * sizeof(float);
  static bool configured = false;
  if (!configured) {
    for (const void* fn : {reinterpret_cast<const void*>(gs::preprocess_bwd_adam_kernel<false>),
                           reinterpret_cast<const void*>(gs::preprocess_bwd_adam_kernel<true>)}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return gs::record_cuda_error(e);
    }
    configured = true;
  }
  const gs::DevCamera cam = gs::make_dev_camera(*camera);
  gs::NextView next{};
  if (project) {
    next.cam = gs::make_dev_camera(*next_camera);
    next.degree = next_degree;
    next.out = *next_splats;
  }
  const unsigned grid = unsigned((params->n + 127) / 128);
  const float4* rec = reinterpret_cast<const float4*>(splats->rec);
  const float4* g2 = reinterpret_cast<const float4*>(grads2d);
  if (project)
    gs::launch_pdl(gs::preprocess_bwd_adam_kernel<true>, grid, 128, smem, s, *params, cam, active_sh_degree, rec, splats->radii,
                                                                 g2, go, st, A, skip, next);
  else
    gs::launch_pdl(gs::preprocess_bwd_adam_kernel<false>, grid, 128, smem, s, *params, cam, active_sh_degree, rec, splats->radii,
                                                                  g2, go, st, A, skip, next);
  return gs::check_launch();
}
}  // namespace

extern "C" int gs_preprocess_backward_adam_guarded(const gs_params_t* params, const gs_camera_t* camera,
                                                   int32_t active_sh_degree, const gs_splats_t* splats,
                                                   const float* grads2d, const gs_adam_group_t* groups, double beta1,
                                                   double beta2, double eps, double bias1, double bias2,
                                                   const gs_stats_t* stats, const gs_grads_t* grads_out,
                                                   const int32_t* skip, void* stream) {
  return launch_backward_adam(params, camera, active_sh_degree, splats, grads2d, groups, beta1, beta2, eps, bias1,
                              bias2, stats, grads_out, skip, nullptr, 0, nullptr, static_cast<cudaStream_t>(stream));
}

extern "C" int gs_preprocess_backward_adam_project(const gs_params_t* params, const gs_camera_t* camera,
                                                   int32_t active_sh_degree, const gs_splats_t* splats,
                                                   const float* grads2d, const gs_adam_group_t* groups, double beta1,
                                                   double beta2, double eps, double bias1, double bias2,
                                                   const gs_stats_t* stats, const gs_grads_t* grads_out,
                                                   const int32_t* skip, const gs_camera_t* next_camera,
                                                   int32_t next_active_sh_degree, gs_splats_t* next_splats,
                                                   void* stream) {
  if (!next_splats) return GS_ERR_INVALID_ARG;
  return launch_backward_adam(params, camera, active_sh_degree, splats, grads2d, groups, beta1, beta2, eps, bias1,
                              bias2, stats, grads_out, skip, next_camera, next_active_sh_degree, next_splats,
                              static_cast<cudaStream_t>(stream));
}

extern "C" int gs_preprocess_backward_adam(const gs_params_t* params, const gs_camera_t* camera,
                                           int32_t active_sh_degree, const gs_splats_t* splats,
                                           const float* grads2d, const gs_adam_group_t* groups, double beta1,
                                           double beta2, double eps, double bias1, double bias2,
                                           const gs_stats_t* stats, const gs_grads_t* grads_out, void* stream) {
  return gs_preprocess_backward_adam_guarded(params, camera, active_sh_degree, splats, grads2d, groups, beta1, beta2,
                                             eps, bias1, bias2, stats, grads_out, nullptr, stream);
}

namespace gs {
namespace {
__global__ void step_guard_kernel(const float* loss, const int64_t* k_info, int32_t* skip, double* report) {
  pdl_begin();
  const float v = loss[0];
  const int32_t sk = (k_info[1] != 0 || !isfinite(v)) ? 1 : 0;
  skip[0] = sk;
  if (report) {   // the step's host-visible summary, written straight into (mapped) pinned memory
    for (int i = 0; i < 4; ++i) report[i] = double(loss[i]);
    for (int i = 0; i < 3; ++i) report[4 + i] = double(k_info[i]);
    report[7] = double(sk);
    __threadfence_system();
  }
}
}  // namespace
}  // namespace gs

extern "C" int gs_step_guard(const float* loss, const int64_t* k_info, int32_t* skip, double* report,
                             void* stream) {
  if (!loss || !k_info || !skip) return GS_ERR_INVALID_ARG;
  gs::launch_pdl(gs::step_guard_kernel, 1, 1, 0, static_cast<cudaStream_t>(stream), loss, k_info, skip, report);
  return gs::check_launch();
}

namespace gs {
namespace {
int preprocess_backward(const gs_params_t* params, const gs_camera_t* camera, int32_t active_sh_degree,
                        const gs_splats_t* splats, const float* grads2d, const gs_grads_t* grads, int32_t accumulate,
                        const gs_stats_t* stats, const int32_t* skip, void* stream) {
  if (!params || !camera || !splats || !grads2d || !grads) return GS_ERR_INVALID_ARG;
  if (active_sh_degree < 0 || active_sh_degree > 3) return GS_ERR_INVALID_ARG;
  if (splats->n != params->n) return GS_ERR_INVALID_ARG;
  if (params->n == 0) return GS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  gs_stats_t st = {nullptr, nullptr, nullptr};
  if (stats) st = *stats;
  const DevCamera cam = make_dev_camera(*camera);
  const int block = 128;
  const unsigned grid = unsigned((params->n + block - 1) / block);
  launch_pdl(preprocess_bwd_kernel, grid, block, 0, s, *params, cam, active_sh_degree,
                                               reinterpret_cast<const float4*>(splats->rec), splats->radii,
                                               reinterpret_cast<const float4*>(grads2d), *grads, accumulate, st,
                                               skip);
  return check_launch();
}
}  // namespace
}  // namespace gs

extern "C" int gs_preprocess_backward(const gs_params_t* params, const gs_camera_t* camera, int32_t active_sh_degree,
                                      const gs_splats_t* splats, const float* grads2d, const gs_grads_t* grads,
                                      int32_t accumulate, const gs_stats_t* stats, void* stream) {
  return gs::preprocess_backward(params, camera, active_sh_degree, splats, grads2d, grads, accumulate, stats, nullptr,
                                 stream);
}

// The same, with the densify statistics left untouched when *skip != 0
// (device int32 from gs_step_guard, e.g. reduced over the ranks): the
// multi-view step enqueues its backward before the host has read the loss.
extern "C" int gs_preprocess_backward_guarded(const gs_params_t* params, const gs_camera_t* camera,
                                              int32_t active_sh_degree, const gs_splats_t* splats,
                                              const float* grads2d, const gs_grads_t* grads, int32_t accumulate,
                                              const gs_stats_t* stats, const int32_t* skip, void* stream) {
  return gs::preprocess_backward(params, camera, active_sh_degree, splats, grads2d, grads, accumulate, stats, skip,
                                 stream);
}
