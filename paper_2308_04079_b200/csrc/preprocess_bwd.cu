// K8 preprocess_bwd — replaces splatlab gradients.backward_project
// (gradients.py:192-259, with backward_invert_cov2d 97-113,
// backward_conic_to_cov3d 116-123, backward_cov3d_to_scale_rotation 126-189,
// sh_basis_jacobian sh.py:66-109) and the densification statistics update of
// optimizer.train_step (optimizer.py:252-255).
//
// One thread per Gaussian.  Nothing from the forward's geometry is cached:
// the view position, J, U = JW, Sigma and the conic are recomputed in
// float64 from the parameters (cheaper in HBM bytes than storing the
// reference's 40-float backward cache per splat).  The SH path reuses the
// forward's float32 basis and the stored clamp mask.
#include "gs_common.cuh"

namespace gs {
namespace {

// Gradients of one surviving Gaussian g.  Writes the non-SH outputs and the
// statistics; returns the SH basis b and the masked colour gradient dcol,
// whose outer product is the (16,3) d_sh row (written by the caller through
// shared memory).  shrow: the Gaussian's staged SH coefficients.
// Per-Gaussian inputs, loaded before the block's SH staging so their
// latency overlaps it.
struct GradInputs {
  float4 ga, gb, gc;   // grads2d row: (d_mx, d_my, d_alpha), (d_ca, d_cb, d_cc), (d_r, d_g, d_b)
  float4 q;            // raw quaternion
  float m0, m1, m2, l0, l1, l2, op, mask;
};

__device__ __forceinline__ void load_inputs(const gs_params_t& p, const float4* __restrict__ rec,
                                            const float4* __restrict__ g2d, int64_t g, GradInputs& in) {
  in.ga = __ldg(g2d + 3 * g + 0);
  in.gb = __ldg(g2d + 3 * g + 1);
  in.gc = __ldg(g2d + 3 * g + 2);
  in.mask = __ldg(rec + 4 * g + 2).w;
  in.q = __ldg(reinterpret_cast<const float4*>(p.rotations) + g);
  in.m0 = __ldg(p.means + 3 * g + 0); in.m1 = __ldg(p.means + 3 * g + 1); in.m2 = __ldg(p.means + 3 * g + 2);
  in.l0 = __ldg(p.log_scales + 3 * g + 0); in.l1 = __ldg(p.log_scales + 3 * g + 1);
  in.l2 = __ldg(p.log_scales + 3 * g + 2);
  in.op = __ldg(p.opacity_logits + g);
}

__device__ __forceinline__ void grad_one(const GradInputs& in, const DevCamera& cam, int degree,
                                         const gs_grads_t& out, int accumulate, const gs_stats_t& stats,
                                         int64_t g, int32_t radius, const float4* shrow, float (&b)[16],
                                         float (&dcol)[3]) {
  const float4 ga = in.ga, gb = in.gb, gc = in.gc;
  const int mask = int(in.mask);

  // --- opacity through the sigmoid (gradients.py:217)
  const double alpha = 1.0 / (1.0 + exp(-double(in.op)));
  const float d_logit = float(double(ga.z) * alpha * (1.0 - alpha));

  // --- view position, Jacobian, U = J W (core.py:279, 298-303)
  const double mx = in.m0, my = in.m1, mz = in.m2;
  double view[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    view[i] = mx * cam.R[3 * i + 0] + my * cam.R[3 * i + 1] + mz * cam.R[3 * i + 2] + cam.t[i];
  const double x = view[0], y = view[1], z = view[2];
  const double z2 = z * z, z3 = z2 * z;
  const double j00 = cam.fx / z, j02 = -cam.fx * x / z2, j11 = cam.fy / z, j12 = -cam.fy * y / z2;
  double U[6];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    U[c] = j00 * cam.R[c] + j02 * cam.R[6 + c];
    U[3 + c] = j11 * cam.R[3 + c] + j12 * cam.R[6 + c];
  }

  // --- covariance from the raw quaternion and log scales (core.py:187-201)
  const float4 qf = in.q;
  const double qn = sqrt(double(qf.x) * qf.x + double(qf.y) * qf.y + double(qf.z) * qf.z + double(qf.w) * qf.w);
  const double q[4] = {qf.x / qn, qf.y / qn, qf.z / qn, qf.w / qn};
  double R[9];
  quat_to_rot(q[0], q[1], q[2], q[3], R);
  const double s[3] = {exp(double(in.l0)), exp(double(in.l1)), exp(double(in.l2))};
  double M[9], S[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) M[3 * i + j] = R[3 * i + j] * s[j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      S[3 * i + k] = M[3 * i + 0] * M[3 * k + 0] + M[3 * i + 1] * M[3 * k + 1] + M[3 * i + 2] * M[3 * k + 2];
  double US[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) US[3 * r + k] = U[3 * r + 0] * S[k] + U[3 * r + 1] * S[3 + k] + U[3 * r + 2] * S[6 + k];
  const double ca = US[0] * U[0] + US[1] * U[1] + US[2] * U[2] + kLowpass;
  const double cb = US[0] * U[3] + US[1] * U[4] + US[2] * U[5];
  const double cc = US[3] * U[3] + US[4] * U[4] + US[5] * U[5] + kLowpass;
  const double det = ca * cc - cb * cb;
  const double A0 = cc / det, A1 = -cb / det, A2 = ca / det;  // conic (core.py:316)

  // --- conic -> floored screen covariance: dS' = -A G A (gradients.py:97-113)
  const double G0 = gb.x, G1 = 0.5 * double(gb.y), G2 = gb.z;
  const double AG00 = A0 * G0 + A1 * G1, AG01 = A0 * G1 + A1 * G2;
  const double AG10 = A1 * G0 + A2 * G1, AG11 = A1 * G1 + A2 * G2;
  const double dC00 = -(AG00 * A0 + AG01 * A1);
  const double dC01 = -(AG00 * A1 + AG01 * A2);
  const double dC10 = -(AG10 * A0 + AG11 * A1);
  const double dC11 = -(AG10 * A1 + AG11 * A2);

  // --- screen covariance -> world covariance: dSigma = U^T dS' U (gradients.py:116-123)
  double dCU[6];  // dS' U  (2x3)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dCU[c] = dC00 * U[c] + dC01 * U[3 + c];
    dCU[3 + c] = dC10 * U[c] + dC11 * U[3 + c];
  }
  double dS[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dS[3 * i + j] = U[i] * dCU[j] + U[3 + i] * dCU[3 + j];

  // --- Sigma = M M^T -> log scales and raw quaternion (gradients.py:126-189)
  double dM[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dM[3 * i + k] = 2.0 * (dS[3 * i + 0] * M[0 + k] + dS[3 * i + 1] * M[3 + k] + dS[3 * i + 2] * M[6 + k]);
  double d_logs[3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    d_logs[k] = (dM[k] * R[k] + dM[3 + k] * R[3 + k] + dM[6 + k] * R[6 + k]) * s[k];
  // dR = dM * diag(s); contract with dR/dq of quat_to_rot
  double dR[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dR[3 * i + j] = dM[3 * i + j] * s[j];
  const double qr = q[0], qi = q[1], qj = q[2], qk = q[3];
  const double dqr = 2.0 * (-qk * dR[1] + qj * dR[2] + qk * dR[3] - qi * dR[5] - qj * dR[6] + qi * dR[7]);
  const double dqi = 2.0 * (qj * dR[1] + qk * dR[2] + qj * dR[3] - 2.0 * qi * dR[4] - qr * dR[5] + qk * dR[6] +
                            qr * dR[7] - 2.0 * qi * dR[8]);
  const double dqj = 2.0 * (-2.0 * qj * dR[0] + qi * dR[1] + qr * dR[2] + qi * dR[3] + qk * dR[5] - qr * dR[6] +
                            qk * dR[7] - 2.0 * qj * dR[8]);
  const double dqk = 2.0 * (-2.0 * qk * dR[0] - qr * dR[1] + qi * dR[2] + qr * dR[3] - 2.0 * qk * dR[4] +
                            qj * dR[5] + qi * dR[6] + qj * dR[7]);
  const double qdot = qr * dqr + qi * dqi + qj * dqj + qk * dqk;
  const float4 d_rot = make_float4(float((dqr - qr * qdot) / qn), float((dqi - qi * qdot) / qn),
                                   float((dqj - qj * qdot) / qn), float((dqk - qk * qdot) / qn));

  // --- view position: J^T d_mean2d plus the dependence of J on the mean
  //     (gradients.py:236-255)
  const double dmx = ga.x, dmy = ga.y;
  double dt[3] = {j00 * dmx, j11 * dmy, j02 * dmx + j12 * dmy};
  double dU[6];  // 2 dS' U Sigma
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int l = 0; l < 3; ++l)
      dU[3 * r + l] = 2.0 * (dCU[3 * r + 0] * S[l] + dCU[3 * r + 1] * S[3 + l] + dCU[3 * r + 2] * S[6 + l]);
  double dJ[6];  // dU W^T
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dJ[3 * r + k] = dU[3 * r + 0] * cam.R[3 * k + 0] + dU[3 * r + 1] * cam.R[3 * k + 1] +
                      dU[3 * r + 2] * cam.R[3 * k + 2];
  dt[0] += dJ[2] * (-cam.fx / z2);
  dt[1] += dJ[5] * (-cam.fy / z2);
  dt[2] += dJ[0] * (-cam.fx / z2) + dJ[2] * (2.0 * cam.fx * x / z3) + dJ[4] * (-cam.fy / z2) +
           dJ[5] * (2.0 * cam.fy * y / z3);

  // --- colour: clamp mask, SH coefficients, direction path (gradients.py:219-226)
  const double ddx = mx - cam.center[0], ddy = my - cam.center[1], ddz = mz - cam.center[2];
  const double dist = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
  const float vx = float(ddx / dist), vy = float(ddy / dist), vz = float(ddz / dist);
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
  const float inv_dist = float(1.0 / dist);
  const float dms[3] = {(gdx - vx * vdot) * inv_dist, (gdy - vy * vdot) * inv_dist, (gdz - vz * vdot) * inv_dist};

  // --- d_means = d_t W + d_mean_sh (gradients.py:257)
  float dmean[3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
    dmean[j] = float(dt[0] * cam.R[j] + dt[1] * cam.R[3 + j] + dt[2] * cam.R[6 + j]) + dms[j];
  const float norm = sqrtf(ga.x * ga.x + ga.y * ga.y);  // gradients.py:258

  if (accumulate) {
    for (int k = 0; k < 3; ++k) out.d_means[3 * g + k] += dmean[k];
    for (int k = 0; k < 3; ++k) out.d_log_scales[3 * g + k] += float(d_logs[k]);
    float4 r = reinterpret_cast<float4*>(out.d_rotations)[g];
    r.x += d_rot.x; r.y += d_rot.y; r.z += d_rot.z; r.w += d_rot.w;
    reinterpret_cast<float4*>(out.d_rotations)[g] = r;
    out.d_opacity_logits[g] += d_logit;
  } else {
    for (int k = 0; k < 3; ++k) out.d_means[3 * g + k] = dmean[k];
    for (int k = 0; k < 3; ++k) out.d_log_scales[3 * g + k] = float(d_logs[k]);
    reinterpret_cast<float4*>(out.d_rotations)[g] = d_rot;
    out.d_opacity_logits[g] = d_logit;
  }
  if (out.view_pos_grad_norm) out.view_pos_grad_norm[g] = norm;
  // densification statistics over every survivor (optimizer.py:252-255)
  if (stats.accum_pos_grad) stats.accum_pos_grad[g] += norm;
  if (stats.accum_count) stats.accum_count[g] += 1;
  if (stats.max_radius_frac) {
    const float frac = float(double(radius) / double(cam.height));
    stats.max_radius_frac[g] = fmaxf(stats.max_radius_frac[g], frac);
  }
}

__global__ void __launch_bounds__(128, 4)
preprocess_bwd_kernel(gs_params_t p, DevCamera cam, int degree, const float4* __restrict__ rec,
                      const int32_t* __restrict__ radii, const float4* __restrict__ g2d, gs_grads_t out,
                      int accumulate, gs_stats_t stats) {
  __shared__ float4 s_sh[128 * kShStride];
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
  if (radius > 0) {
    grad_one(in, cam, degree, out, accumulate, stats, g, radius, s_sh + threadIdx.x * kShStride, b, dcol);
  } else if (valid && !accumulate) {  // culled: exactly zero gradient (gradients.py:13-27)
    for (int k = 0; k < 3; ++k) out.d_means[3 * g + k] = 0.0f;
    for (int k = 0; k < 3; ++k) out.d_log_scales[3 * g + k] = 0.0f;
    reinterpret_cast<float4*>(out.d_rotations)[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    out.d_opacity_logits[g] = 0.0f;
    if (out.view_pos_grad_norm) out.view_pos_grad_norm[g] = 0.0f;
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
      const int e0 = 4 * k;
      float4 v = make_float4(b[(e0 + 0) / 3] * dcol[(e0 + 0) % 3], b[(e0 + 1) / 3] * dcol[(e0 + 1) % 3],
                             b[(e0 + 2) / 3] * dcol[(e0 + 2) % 3], b[(e0 + 3) / 3] * dcol[(e0 + 3) % 3]);
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

}  // namespace
}  // namespace gs

extern "C" int gs_preprocess_backward(const gs_params_t* params, const gs_camera_t* camera, int32_t active_sh_degree,
                                      const gs_splats_t* splats, const float* grads2d, const gs_grads_t* grads,
                                      int32_t accumulate, const gs_stats_t* stats, void* stream) {
  if (!params || !camera || !splats || !grads2d || !grads) return GS_ERR_INVALID_ARG;
  if (active_sh_degree < 0 || active_sh_degree > 3) return GS_ERR_INVALID_ARG;
  if (splats->n != params->n) return GS_ERR_INVALID_ARG;
  if (params->n == 0) return GS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  gs_stats_t st = {nullptr, nullptr, nullptr};
  if (stats) st = *stats;
  const gs::DevCamera cam = gs::make_dev_camera(*camera);
  const int block = 128;
  const unsigned grid = unsigned((params->n + block - 1) / block);
  gs::preprocess_bwd_kernel<<<grid, block, 0, s>>>(*params, cam, active_sh_degree,
                                                   reinterpret_cast<const float4*>(splats->rec), splats->radii,
                                                   reinterpret_cast<const float4*>(grads2d), *grads, accumulate, st);
  return gs::check_launch();
}
