// Per-Gaussian projection (splatlab core.project, core.py:266-345, and the
// tile rectangle of rasterizer.bin_and_sort, rasterizer.py:86-97), shared by
// preprocess_fwd_kernel (K1) and the fused backward + Adam kernel that
// projects the updated parameters for the next view
// (gs_preprocess_backward_adam_project).  The geometry chain that decides
// integers (culling, radius, tile rectangle, float32 depth key) runs in
// float64 with non-contracted IEEE operations, mirroring the float64
// reference, so radii and binning agree bit-for-bit; appearance (SH colour)
// runs in float32.  sh_row(k) returns float4 k of the Gaussian's (16,3) SH
// row (a global or a shared-memory load).
#pragma once
#include "gs_common.cuh"

namespace gs {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

template <typename ShRow>
__device__ __forceinline__ void project_gaussian(float pm0, float pm1, float pm2, float4 qf, float pl0, float pl1,
                                                 float pl2, float pop, ShRow sh_row, const DevCamera& cam,
                                                 int degree, const gs_splats_t& out, int64_t g) {
  // view = means @ W^T + t (core.py:279)
  const double mx = pm0, my = pm1, mz = pm2;
  double view[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    view[i] = dadd(dadd(dadd(dmul(mx, cam.R[3 * i + 0]), dmul(my, cam.R[3 * i + 1])), dmul(mz, cam.R[3 * i + 2])),
                   cam.t[i]);
  const double x = view[0], y = view[1], z = view[2];

  int32_t radius_out = 0;
  int32_t tiles = 0;
  // near-plane cull (core.py:281); NaN compares false and is culled like numpy
  if (!(z >= cam.near_plane)) {
    out.radii[g] = 0;
    out.tiles_touched[g] = 0;
    return;
  }
  // screen position and guard band (core.py:286-293)
  const double u = dadd(__ddiv_rn(dmul(cam.fx, x), z), cam.cx);
  const double v = dadd(__ddiv_rn(dmul(cam.fy, y), z), cam.cy);
  // |ndc| <= 1.3 decided on a product with the host's reciprocal of the
  // half extent (within 2 ulp of the quotient); only a product within 1e-12
  // of the band edge (or NaN) takes the correctly rounded division
  const double ax = dsub(u, cam.cx), ay = dsub(v, cam.cy);
  double ndc_x = dmul(ax, cam.inv_half_w), ndc_y = dmul(ay, cam.inv_half_h);
  if (!(fabs(fabs(ndc_x) - kGuardBand) > 1e-12)) ndc_x = __ddiv_rn(ax, dmul(0.5, double(cam.width)));
  if (!(fabs(fabs(ndc_y) - kGuardBand) > 1e-12)) ndc_y = __ddiv_rn(ay, dmul(0.5, double(cam.height)));
  if (!(fabs(ndc_x) <= kGuardBand && fabs(ndc_y) <= kGuardBand)) {
    out.radii[g] = 0;
    out.tiles_touched[g] = 0;
    return;
  }

  // world covariance Sigma = M M^T, M = R(q/|q|) diag(exp(s)) (core.py:187-201)

  double qr = qf.x, qi = qf.y, qj = qf.z, qk = qf.w;
  const double qn = sqrt(dadd(dadd(dadd(dmul(qr, qr), dmul(qi, qi)), dmul(qj, qj)), dmul(qk, qk)));
  if (qn == 0.0) {  // InvalidPrimitiveError (core.py:164-165)
    atomicOr(out.status, 1);
    out.radii[g] = 0;
    out.tiles_touched[g] = 0;
    return;
  }
  qr = __ddiv_rn(qr, qn); qi = __ddiv_rn(qi, qn); qj = __ddiv_rn(qj, qn); qk = __ddiv_rn(qk, qn);
  double R[9];
  quat_to_rot(qr, qi, qj, qk, R);
  const double s0 = exp(double(pl0));
  const double s1 = exp(double(pl1));
  const double s2 = exp(double(pl2));
  double M[9];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    M[3 * i + 0] = dmul(R[3 * i + 0], s0);
    M[3 * i + 1] = dmul(R[3 * i + 1], s1);
    M[3 * i + 2] = dmul(R[3 * i + 2], s2);
  }
  // M M^T is symmetric bit for bit (the same products, summed in the same
  // order): the upper triangle is computed and mirrored
  double S[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = i; k < 3; ++k) {
      S[3 * i + k] = dadd(dadd(dmul(M[3 * i + 0], M[3 * k + 0]), dmul(M[3 * i + 1], M[3 * k + 1])),
                          dmul(M[3 * i + 2], M[3 * k + 2]));
      S[3 * k + i] = S[3 * i + k];
    }

  // EWA: J (core.py:298-302), U = J W, Sigma' = U Sigma U^T (303-304)
  const double zz = dmul(z, z);
  const double j00 = __ddiv_rn(cam.fx, z);
  const double j02 = __ddiv_rn(dmul(-cam.fx, x), zz);
  const double j11 = __ddiv_rn(cam.fy, z);
  const double j12 = __ddiv_rn(dmul(-cam.fy, y), zz);
  double U[6];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    U[c] = dadd(dmul(j00, cam.R[c]), dmul(j02, cam.R[6 + c]));
    U[3 + c] = dadd(dmul(j11, cam.R[3 + c]), dmul(j12, cam.R[6 + c]));
  }
  double US[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      US[3 * r + k] = dadd(dadd(dmul(U[3 * r + 0], S[0 * 3 + k]), dmul(U[3 * r + 1], S[1 * 3 + k])),
                           dmul(U[3 * r + 2], S[2 * 3 + k]));
  const double c00 = dadd(dadd(dmul(US[0], U[0]), dmul(US[1], U[1])), dmul(US[2], U[2]));
  const double c01 = dadd(dadd(dmul(US[0], U[3]), dmul(US[1], U[4])), dmul(US[2], U[5]));
  const double c11 = dadd(dadd(dmul(US[3], U[3]), dmul(US[4], U[4])), dmul(US[5], U[5]));
  const double ca = dadd(c00, kLowpass);  // core.py:305-307
  const double cb = c01;
  const double cc = dadd(c11, kLowpass);
  const double det = dsub(dmul(ca, cc), dmul(cb, cb));  // core.py:309
  if (!(det > 0.0)) {
    out.radii[g] = 0;
    out.tiles_touched[g] = 0;
    return;
  }
  // conic, lambda_max, radius (core.py:316-319)
  const double mid = dmul(0.5, dadd(ca, cc));
  const double lam = dadd(mid, sqrt(fmax(dsub(dmul(mid, mid), det), 0.0)));
  const double rad_d = ceil(dmul(kRadiusSigmas, sqrt(lam)));
  radius_out = rad_d >= 2147483647.0 ? 2147483647 : int32_t(rad_d);

  // tile rectangle, inclusive, clipped (rasterizer.py:86-97)
  // x / 16 == x * 2^-4 exactly (power-of-two scaling), without a division
  constexpr double kInvTile = 1.0 / double(kTile);
  static_assert((kTile & (kTile - 1)) == 0, "tile size must be a power of two");
  const double x0d = floor(dmul(dsub(u, rad_d), kInvTile));
  const double x1d = floor(dmul(dadd(u, rad_d), kInvTile));
  const double y0d = floor(dmul(dsub(v, rad_d), kInvTile));
  const double y1d = floor(dmul(dadd(v, rad_d), kInvTile));
  const double txm = double(cam.tiles_x - 1), tym = double(cam.tiles_y - 1);
  const bool valid = (x1d >= 0.0) && (x0d < double(cam.tiles_x)) && (y1d >= 0.0) && (y0d < double(cam.tiles_y));
  const int32_t x0 = int32_t(fmin(fmax(x0d, 0.0), txm));
  const int32_t x1 = int32_t(fmin(fmax(x1d, 0.0), txm));
  const int32_t y0 = int32_t(fmin(fmax(y0d, 0.0), tym));
  const int32_t y1 = int32_t(fmin(fmax(y1d, 0.0), tym));
  if (valid) {
    const int64_t cnt = int64_t(x1 - x0 + 1) * int64_t(y1 - y0 + 1);
    tiles = cnt > 2147483647 ? 2147483647 : int32_t(cnt);
  }

  // SH colour along the unit camera->mean direction (core.py:321-326)
  const double dx = dsub(mx, cam.center[0]), dy = dsub(my, cam.center[1]), dz = dsub(mz, cam.center[2]);
  const double dist = sqrt(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
  // float32 colour path: one reciprocal instead of three divisions
  const double inv_dist = __drcp_rn(dist);
  const float vx = float(dmul(dx, inv_dist)), vy = float(dmul(dy, inv_dist)), vz = float(dmul(dz, inv_dist));
  float b[16];
  sh_basis(vx, vy, vz, degree, b);
  const int nrows = (degree + 1) * (degree + 1);
  float shv[48];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const float4 q4 = (4 * k < 3 * nrows) ? sh_row(k) : make_float4(0.f, 0.f, 0.f, 0.f);
    shv[4 * k + 0] = q4.x; shv[4 * k + 1] = q4.y; shv[4 * k + 2] = q4.z; shv[4 * k + 3] = q4.w;
  }
  float col[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (k < nrows) {
      col[0] = fmaf(b[k], shv[3 * k + 0], col[0]);
      col[1] = fmaf(b[k], shv[3 * k + 1], col[1]);
      col[2] = fmaf(b[k], shv[3 * k + 2], col[2]);
    }
  }
  int mask = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    col[c] += 0.5f;
    if (col[c] > 0.0f) mask |= (1 << c);
    col[c] = fmaxf(col[c], 0.0f);
  }
  // sigmoid opacity (core.py:327)
  const double alpha = __drcp_rn(1.0 + exp(-double(pop)));   // == 1.0 / (...) (both correctly rounded)

  const float ux_hi = float(u), uy_hi = float(v);
  const float ux_lo = float(dsub(u, double(ux_hi))), uy_lo = float(dsub(v, double(uy_hi)));
  // split float64 -> (hi, lo) float32 pairs for the blend's threshold guard
  // the conic from one reciprocal of det (within 2 ulp of the quotients: far
  // below the 48 bits its hi/lo pair keeps; it decides no integer)
  const double rdet = __drcp_rn(det);   // det(conic) = 1 / det(cov2d)
  const double c0 = dmul(cc, rdet), c1 = dmul(-cb, rdet), c2 = dmul(ca, rdet);
  const float c0h = float(c0), c1h = float(c1), c2h = float(c2), ah = float(alpha);
  float4* rec = reinterpret_cast<float4*>(out.rec) + kRecWords * g;
  rec[0] = make_float4(ux_hi, uy_hi, ux_lo, uy_lo);
  rec[1] = conic_basis(c0, c1, c2, rdet);
  rec[2] = make_float4(col[0], col[1], col[2], ah);
  rec[3] = make_float4(c0h, c1h, c2h, float(mask));
  rec[4] = make_float4(float(dsub(c0, double(c0h))), float(dsub(c1, double(c1h))), float(dsub(c2, double(c2h))),
                       float(dsub(alpha, double(ah))));
  out.depth[g] = float(z);
  reinterpret_cast<int4*>(out.rect)[g] = make_int4(x0, y0, x1, y1);
  out.radii[g] = radius_out;
  out.tiles_touched[g] = tiles;
}

}  // namespace gs
