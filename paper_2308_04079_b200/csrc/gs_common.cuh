// gs_common.cuh — device-side constants and math shared by every kernel.
//
// The constants restate the reference's module-level constants
// (core.py:13-18, rasterizer.py:13-25, sh.py:6-23).  The alpha evaluation
// used by the forward and the backward blend is ONE inline function built
// from non-contractible intrinsics, so both passes see bit-identical alphas
// and therefore identical contributor sets (gradients.py:54-65).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cstdlib>
#include <utility>   // CUtensorMap (the TMA descriptor type; the encoder is fetched at run time)
#include <cuda_runtime.h>

#include "../../include/gs_rasterizer.h"

namespace gs {

constexpr int kTile = GS_TILE_SIZE;             // rasterizer.py:13
constexpr int kTilePixels = kTile * kTile;      // 256 pixels = 256 threads per tile CTA
constexpr double kLowpass = 0.3;                // core.py:13 LOWPASS_FLOOR
constexpr double kGuardBand = 1.3;              // core.py:16 GUARD_BAND
constexpr double kRadiusSigmas = 3.0;           // core.py:18 RADIUS_SIGMAS
constexpr float kAlphaEps = 1.0f / 255.0f;      // rasterizer.py:17 ALPHA_EPS
constexpr float kAlphaClamp = 0.99f;            // rasterizer.py:18 ALPHA_CLAMP
// rasterizer.py:19 SATURATION = 0.9999; "1 - T_new > 0.9999" is evaluated as
// T_new < 1 - 0.9999 so float32 keeps full relative precision near T = 1e-4
// (1.0f - T would quantise T to ulp(1) = 6e-8, i.e. 6e-4 relative).
constexpr float kTransSat = float(1.0 - 0.9999);
// Saturation guard (training forward): the float32 transmittance differs
// from the float64 reference's by ~sum_i eps_a a_i / (1 - a_i) relative
// (float32 alphas are ~1e-7..2e-6 relative off, the 1/255 and 0.99
// decisions are exact), ~1e-5 at the stop for realistic alpha mixes.  A
// pixel whose T_new lands within kSatGuard (relative) of the threshold is
// flagged (last = kLastPending) and re-blended exactly in float64 by the
// fix-up kernel, so every stop decision is the reference's.
constexpr float kSatGuard = 1e-4f;
constexpr float kTransSatLo = kTransSat * (1.0f - kSatGuard);
constexpr float kTransSatHi = kTransSat * (1.0f + kSatGuard);
constexpr int32_t kLastPending = -2;
constexpr int64_t kMaxInstances = int64_t(1) << 31;    // rasterizer.py:25
constexpr int64_t kMaxTiles = (int64_t(1) << 32) - 1;  // rasterizer.py:24

// Real SH constants (sh.py:6-23).
constexpr float kC0 = 0.28209479177387814f;
constexpr float kC1 = 0.4886025119029199f;
constexpr float kC2_0 = 1.0925484305920792f;
constexpr float kC2_1 = -1.0925484305920792f;
constexpr float kC2_2 = 0.31539156525252005f;
constexpr float kC2_3 = -1.0925484305920792f;
constexpr float kC2_4 = 0.5462742152960396f;
constexpr float kC3_0 = -0.5900435899266435f;
constexpr float kC3_1 = 2.890611442640554f;
constexpr float kC3_2 = -0.4570457994644658f;
constexpr float kC3_3 = 0.3731763325901154f;
constexpr float kC3_4 = -0.4570457994644658f;
constexpr float kC3_5 = 1.445305721320277f;
constexpr float kC3_6 = -0.5900435899266435f;

// Camera as the kernels see it (passed by value in the kernel parameters).
struct DevCamera {
  double R[9];
  double t[3];
  double center[3];   // -R^T t (core.py:143-146)
  double fx, fy, cx, cy;
  double near_plane;
  double inv_half_w, inv_half_h;   // 1 / (0.5 width), 1 / (0.5 height): the guard-band test's fast path
  int width, height;
  int tiles_x, tiles_y;
};

__host__ inline DevCamera make_dev_camera(const gs_camera_t& c) {
  DevCamera d;
  for (int i = 0; i < 9; ++i) d.R[i] = c.rotation[i];
  for (int i = 0; i < 3; ++i) d.t[i] = c.translation[i];
  for (int i = 0; i < 3; ++i)
    d.center[i] = -(c.rotation[0 * 3 + i] * c.translation[0] + c.rotation[1 * 3 + i] * c.translation[1] +
                    c.rotation[2 * 3 + i] * c.translation[2]);
  d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy;
  d.near_plane = c.near_plane;
  d.inv_half_w = 1.0 / (0.5 * double(c.width));
  d.inv_half_h = 1.0 / (0.5 * double(c.height));
  d.width = c.width; d.height = c.height;
  d.tiles_x = (c.width + kTile - 1) / kTile;
  d.tiles_y = (c.height + kTile - 1) / kTile;
  return d;
}

// ---------------------------------------------------------------------------
// Alpha of one splat at one pixel (rasterizer.py:171-177, gradients.py:54-61).
//   power = -0.5 (a dx^2 + c dy^2) - b dx dy ; G = 0 if power > 0 else e^power
//   a_raw = alpha G ; a = min(0.99, a_raw) ; a < 1/255 -> skipped
// Fast path in float32: dx uses the split (hi, lo) screen mean so the
// subtraction keeps ~f64 accuracy at 4K coordinates, and explicit _rn
// intrinsics are never fused or re-associated, so the forward and the
// backward see bit-identical alphas (identical contributor sets).
// Threshold guard: when a_raw lies within kGuard (relative) of 1/255 or of
// 0.99 the pair is re-evaluated in float64 from the split records
// (mean, conic and opacity hi + lo), so the skip / clamp decisions agree with
// the float64 reference.  The float32 fast path is accurate to < 5e-6
// relative for every conic conditioning (eigenbasis form, see
// make_tile_splat), kGuard = 1e-5 covers it; about 4e-5 of pairs take the
// slow path.
struct AlphaEval {
  float v1, v2, g, a_raw, a;   // v: eigenbasis offsets; a: clamped and eps-skipped alpha (0 = skip)
  bool live;                   // a_raw < 0.99: the pair passes gradient to alpha/power
  bool ok;                     // the pair is blended (a >= 1/255); for ok = false a is not
                               // zeroed on the float32 path (callers select on ok)
};

#ifndef GS_ALPHA_GUARD
#define GS_ALPHA_GUARD 1e-5f
#endif
constexpr float kGuard = GS_ALPHA_GUARD;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// one MUFU.RCP (the value __fdividef(1, x) computes for normal x, without
// its denormal-range rescaling sequence)
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Record layout (gs_splats_t.rec, kRecWords x float4 per Gaussian):
//   r0 = (mx_hi, my_hi, mx_lo, my_lo)      r1 = k = (k1.x, k1.y, k2.x, k2.y)  (conic_basis)
//   r2 = (r, g, b, alpha_hi)               r3 = (ca_hi, cb_hi, cc_hi, mask)
//   r4 = (ca_lo, cb_lo, cc_lo, alpha_lo)
// The blend producers gather r0..r2 (48 B); r3, r4 are read by the float64
// slow path and the projection backward only.
constexpr int kRecWords = 5;

// Returns (G, a_raw, a, live) by value (registers, no local memory).
static __device__ __noinline__ float4 alpha_f64(float px, float py, const float4* __restrict__ r) {
  const float4 r0 = r[0], r2 = r[2], r3 = r[3], r4 = r[4];
  const double dx = double(px) - (double(r0.x) + double(r0.z));
  const double dy = double(py) - (double(r0.y) + double(r0.w));
  const double ca = double(r3.x) + double(r4.x), cb = double(r3.y) + double(r4.y), cc = double(r3.z) + double(r4.z);
  const double al = double(r2.w) + double(r4.w);
  const double power = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy;
  const double g = power > 0.0 ? 0.0 : exp(power);
  const double ar = al * g;
  const double a = ar < 0.99 ? ar : 0.99;
  return make_float4(float(g), float(ar), (a < 1.0 / 255.0) ? 0.0f : float(a), ar < 0.99 ? 1.0f : 0.0f);
}

__device__ __forceinline__ void eval_alpha_f64(float px, float py, const float4* __restrict__ r, AlphaEval& e) {
  const float4 v = alpha_f64(px, py, r);
  e.g = v.x;
  e.a_raw = v.y;
  e.a = v.z;
  e.live = v.w != 0.0f;
}

// ---------------------------------------------------------------------------
// SH coefficient staging for the per-Gaussian kernels.  A block of B threads
// owns B consecutive Gaussians whose (B,16,3) coefficients are one
// contiguous 192*B-byte span: it is read with consecutive float4 loads
// (coalesced) into shared memory rows padded to 13 float4, so each thread's
// 12 float4 row reads are bank-conflict free (row stride 52 words).
constexpr int kShStride = 13;

__device__ __forceinline__ void stage_sh_rows(const float* __restrict__ src_rows, int64_t n, int64_t g0,
                                              float4* __restrict__ s) {
  const int64_t left = n - g0;
  const int nb = left < int64_t(blockDim.x) ? int(left) : int(blockDim.x);
  const float4* src = reinterpret_cast<const float4*>(src_rows) + g0 * 12;
  const int total = nb * 12, step = blockDim.x;
  int f = threadIdx.x;
  // four loads in flight per thread before the shared-memory stores
  for (; f + 3 * step < total; f += 4 * step) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(src + f + u * step);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int ff = f + u * step, j = ff / 12;
      s[j * kShStride + (ff - j * 12)] = v[u];
    }
  }
  for (; f < total; f += step) {
    const int j = f / 12;
    s[j * kShStride + (f - j * 12)] = __ldg(src + f);
  }
}

__device__ __forceinline__ void store_sh_rows(const float4* __restrict__ s, int64_t n, int64_t g0,
                                              float* __restrict__ dst_rows) {
  const int64_t left = n - g0;
  const int nb = left < int64_t(blockDim.x) ? int(left) : int(blockDim.x);
  float4* dst = reinterpret_cast<float4*>(dst_rows) + g0 * 12;
  for (int f = threadIdx.x; f < nb * 12; f += blockDim.x) {
    const int j = f / 12;
    dst[f] = s[j * kShStride + (f - j * 12)];
  }
}

// ---------------------------------------------------------------------------
// Tile CTA pixel layout: warp w covers the 8x4 pixel block at
// ((w & 1) * 8, (w >> 1) * 4) of the 16x16 tile; lane l covers pixel
// (l & 7, l >> 3) of that block.
__device__ __forceinline__ int tile_px(int t) { return ((t >> 5) & 1) * 8 + (t & 7); }
__device__ __forceinline__ int tile_py(int t) { return (t >> 6) * 4 + ((t & 31) >> 3); }

// Warp coverage mask of one splat: bit w is set when the splat can reach
// alpha >= 1/255 at some pixel centre of warp w's block.  The set
// {alpha * exp(-Q/2) >= 1/255} is the ellipse Q(d) = d^T conic d <= 2 tau,
// tau = ln(255 alpha); its axis-aligned box has half-extents
// sqrt(2 tau Sigma'_xx), sqrt(2 tau Sigma'_yy).  tau and the box are
// inflated so the test is conservative against float32 rounding: a pair is
// skipped only if the reference would skip it (a < 1/255), so culling never
// changes a result bit.
// Warp w's 8x4 block starts at ((w & 1) * 8, (w >> 1) * 4) of the tile.
// kExact adds the exact ellipse-vs-block test (cheaper consumers, busier
// producer: it pays in the backward, not in the forward, whose producer
// then becomes the bottleneck — measured bwd 1.359 -> 1.336 ms, fwd 0.673 -> 1.01 ms).
#ifndef GS_COVER_BALL
#define GS_COVER_BALL 1
#endif
#ifndef GS_COVER_BALL_EXACT
#define GS_COVER_BALL_EXACT 0
#endif
#ifndef GS_COVER_FAST
#define GS_COVER_FAST 1   // separable box + incremental centre images (branch-free); 0: per-block loop
#endif
// |(a, b)| by the MUFU reciprocal square root (0 for a zero vector)
__device__ __forceinline__ float fast_norm(float a, float b) {
  const float q = fmaf(a, a, b * b);
  return q > 0.0f ? q * rsqrtf(q) : 0.0f;
}

// kRows: block rows tested from tile_y0 (a half-tile CTA passes 2 and its
// half's origin, so only its own four blocks are tested)
template <bool kExact = false, int kBlockH = 4, int kRows = kTile / kBlockH>
__device__ __forceinline__ uint32_t warp_cover_mask(float4 r0, float4 k, float alpha, float tile_x0, float tile_y0) {
  constexpr int kWarps = 2 * kRows;
  constexpr uint32_t kAll = (1u << kWarps) - 1u;
  if (alpha < kAlphaEps * (1.0f - 1e-5f)) return 0u;
  // alpha 2^-(|k d|^2) >= 1/255  <=>  |k d|^2 <= tau = log2(255 alpha)
  const float tau = fmaxf(__log2f(255.0f * alpha), 0.0f) * 1.0001f + 1e-4f;
  // det k = f1 f2 (ex^2 + ey^2): a sum of same-signed terms, no cancellation
  const float detk = k.x * k.w - k.y * k.z;
  if (!(detk > 0.0f)) return kAll;  // degenerate basis: never cull
  // the contour's half extents: sqrt(tau) |row of k^-1|.  The square roots
  // and the division are the MUFU approximations (a few ulp): every bound
  // below carries a 1e-3 relative inflation, so the masks stay conservative
  const float sqrt_tau = tau * rsqrtf(tau);   // tau >= 1e-4 > 0
  const float kex = fast_norm(k.x, k.z), key = fast_norm(k.y, k.w);   // |K e_x|, |K e_y|
  const float st = __fdividef(sqrt_tau, detk);
  const float hx = st * key * 1.001f + 0.05f;
  const float hy = st * kex * 1.001f + 0.05f;
  const float mx = r0.x + r0.z, my = r0.y + r0.w;
#if GS_COVER_BALL
  // !kExact: a cheap conservative metric test after the box test: in the
  // eigenbasis the contour is the disk |v| <= sqrt(tau), v = K (p - mean);
  // the block's pixel centres lie within hw |K e_x| + hh |K e_y| of its
  // centre's image (triangle inequality), so the block is missed when
  // |K (c - mean)| exceeds sqrt(tau) plus that radius
  const float ball_r = sqrt_tau + 3.5f * kex + (0.5f * float(kBlockH - 1)) * key;
  const float ball_r2 = ball_r * ball_r * 1.0002f + 1e-3f;
  const float sat_r2 = tau * 1.0002f + 1e-3f;   // (GS_COVER_BALL >= 2) the contour radius^2, inflated
#endif
#if GS_COVER_BALL && GS_COVER_FAST
  if (!kExact) {
    // branch-free form: the box test is separable (2 block columns x kRows
    // rows), and the block centres' images c' = K (c - mean) step by the
    // constant 8 K e_x per column and kBlockH K e_y per row
    const float cx0 = tile_x0 + 4.0f - mx, cy0 = tile_y0 + 0.5f * float(kBlockH) - my;
    const float u00 = fmaf(k.x, cx0, k.y * cy0), v00 = fmaf(k.z, cx0, k.w * cy0);
    const float dux = 8.0f * k.x, dvx = 8.0f * k.z, duy = float(kBlockH) * k.y, dvy = float(kBlockH) * k.w;
    bool okx[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float x0 = tile_x0 + float(c * 8) + 0.5f;
      okx[c] = (mx + hx >= x0) && (mx - hx <= x0 + 7.0f);
    }
    uint32_t m = 0u;
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const float y0 = tile_y0 + float(r * kBlockH) + 0.5f;
      const bool oky = (my + hy >= y0) && (my - hy <= y0 + float(kBlockH - 1));
      const float ur = fmaf(float(r), duy, u00), vr = fmaf(float(r), dvy, v00);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float u = c ? ur + dux : ur, v = c ? vr + dvx : vr;
        const float d2 = fmaf(u, u, v * v);
        bool pass = okx[c] && oky && d2 <= ball_r2;
#if GS_COVER_BALL >= 2
        const float hh = 0.5f * float(kBlockH - 1);
        const float A = (3.5f * fabsf(fmaf(u, k.x, v * k.z)) + hh * fabsf(fmaf(u, k.y, v * k.w))) * 1.001f + 1e-3f;
        const float e = d2 - A;
        pass = pass && !(e > 0.0f && e * e > sat_r2 * d2);
#endif
        m |= pass ? (1u << (2 * r + c)) : 0u;
      }
    }
    return m;
  }
#endif
  // exact test for the blocks whose box overlaps the contour's box: the
  // minimum of the convex |k d|^2 over the block's pixel-centre rectangle (0
  // when the mean is inside, else on one of the four edges; the edge
  // minimiser comes from the expanded form, the value is evaluated as a sum
  // of squares), against the inflated tau.  The rectangle is padded by 0.01 px.
  const float qa = k.x * k.x + k.z * k.z, qb = k.x * k.y + k.z * k.w, qc = k.y * k.y + k.w * k.w;
  const float rb_c = -qb / qc, rb_a = -qb / qa;
  const float lim = tau * 1.0001f + 1e-4f;
  uint32_t m = 0u;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const float x0 = tile_x0 + float((w & 1) * 8) + 0.5f, y0 = tile_y0 + float((w >> 1) * kBlockH) + 0.5f;
    if (!(mx + hx >= x0 && mx - hx <= x0 + 7.0f && my + hy >= y0 && my - hy <= y0 + float(kBlockH - 1))) continue;
#if GS_COVER_BALL
    if (!kExact || GS_COVER_BALL_EXACT) {   // with kExact: a cheap pre-filter of the exact test
      const float cx = x0 + 3.5f - mx, cy = y0 + 0.5f * float(kBlockH - 1) - my;
      const float u = fmaf(k.x, cx, k.y * cy), v = fmaf(k.z, cx, k.w * cy);
      const float d2 = fmaf(u, u, v * v);
      if (d2 > ball_r2) continue;
#if GS_COVER_BALL >= 2
      // separating axis through the centre's image c' = (u, v): the block's
      // image (a parallelogram, half-edges 3.5 K e_x and hh K e_y) reaches at
      // most A / |c'| towards the origin along c', A = 3.5 |c'.K e_x| + hh
      // |c'.K e_y|; missed when |c'| - A / |c'| > sqrt(tau), i.e. (squared,
      // for d2 > A) (d2 - A)^2 > tau' d2
      const float hh = 0.5f * float(kBlockH - 1);
      const float A = (3.5f * fabsf(fmaf(u, k.x, v * k.z)) + hh * fabsf(fmaf(u, k.y, v * k.w))) * 1.001f + 1e-3f;
      const float e = d2 - A;
      if (e > 0.0f && e * e > sat_r2 * d2) continue;
#endif
    }
#endif
    if (kExact) {
      const float xa = x0 - 0.01f - mx, xb = x0 + 7.01f - mx;
      const float ya = y0 - 0.01f - my, yb = y0 + float(kBlockH - 1) + 0.01f - my;
      float q = 0.0f;
      if (!(xa <= 0.0f && xb >= 0.0f && ya <= 0.0f && yb >= 0.0f)) {
        q = 3.0e38f;
        auto sq = [&](float x, float y) {
          const float u = fmaf(k.x, x, k.y * y), v = fmaf(k.z, x, k.w * y);
          return fmaf(u, u, v * v);
        };
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float x = e ? xb : xa;
          q = fminf(q, sq(x, fminf(fmaxf(rb_c * x, ya), yb)));
          const float yy = e ? yb : ya;
          q = fminf(q, sq(fminf(fmaxf(rb_a * yy, xa), xb), yy));
        }
      }
      if (!(q <= lim)) continue;
    }
    m |= 1u << w;
  }
  return m;
}

// ---------------------------------------------------------------------------
// Adam update of one element (optimizer.py:288-293), shared by the standalone
// Adam kernel and the fused backward+Adam kernel; explicit _rn intrinsics so
// both produce bit-identical parameters and moments.
//   m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2 ; p -= lr (m/bias1) / (sqrt(v/bias2) + eps)
struct AdamCoef {
  float beta1, beta2, one_m_beta1, one_m_beta2, eps, inv_bias1, inv_bias2;
};

__device__ __forceinline__ void adam_update(float& p, float g, float& m, float& v, float lr, const AdamCoef& c) {
  m = __fadd_rn(__fmul_rn(c.beta1, m), __fmul_rn(c.one_m_beta1, g));
  v = __fadd_rn(__fmul_rn(c.beta2, v), __fmul_rn(__fmul_rn(c.one_m_beta2, g), g));
  const float denom = __fadd_rn(__fsqrt_rn(__fmul_rn(v, c.inv_bias2)), c.eps);
  // denom >= eps = 1e-15 is a normal float: __fdividef is accurate to 2 ulp
  p = __fsub_rn(p, __fdividef(__fmul_rn(lr, __fmul_rn(m, c.inv_bias1)), denom));
}

// ---------------------------------------------------------------------------
// mbarrier / cp.async helpers (sm_90+ PTX) for the pipelined blend kernels.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// arrive (release.cta): this thread's prior shared-memory writes become
// visible to threads that observe the phase completion
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait.parity (acquire.cta): true once the phase with this parity completed
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the waiting warp sleeps (up to
// `hint_ns`, or until the phase completes) instead of spinning, so a waiting
// producer or consumer does not steal issue slots from the warps that work.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
      : "memory");
  return ok != 0;
}
// TMA: arrive on an mbarrier announcing `bytes` of asynchronous transactions
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// make freshly initialised mbarriers visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbarrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// TMA tile::gather4: rows r0..r3 of a 2-D tensor map, columns [c0, c0 + box
// width), into 4 consecutive smem rows; completes `box bytes x 4` on `bar`
__device__ __forceinline__ void tma_gather4(void* smem_dst, const CUtensorMap* tmap, uint64_t* bar, int c0, int r0,
                                            int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Bulk L2 prefetch of a global span (TMA unit, no registers or shared
// memory involved).  The span is trimmed to whole 16-byte units inside
// [ptr, ptr + bytes) so it never touches memory outside the buffer.
__device__ __forceinline__ void prefetch_l2_span(const void* ptr, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
  const uintptr_t lo = (a + 15) & ~uintptr_t(15), hi = (a + bytes) & ~uintptr_t(15);
  if (hi <= lo) return;
  size_t n = hi - lo;
  const char* q = reinterpret_cast<const char*>(lo);
  while (n) {   // one bulk op moves < 2^32 bytes; keep each <= 1 MiB
    const uint32_t chunk = uint32_t(n < (size_t(1) << 20) ? n : (size_t(1) << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(chunk) : "memory");
    q += chunk;
    n -= chunk;
  }
}

__device__ __forceinline__ int ld_volatile(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

// ---------------------------------------------------------------------------
// The exponent is evaluated as a sum of two squares in the conic's eigenbasis,
//   p2 = log2(e) * power = -(v1^2 + v2^2),   v_i = k_i . (p - mean),
//   k_i = sqrt(log2(e) * lambda_i / 2) * e_i   (lambda_i, e_i: conic eigenpairs)
// so no cancellation occurs for elongated (near-singular) conics: the
// expanded form a dx^2 + 2b dx dy + c dy^2 loses ~cond(conic) * 6e-8 of
// relative accuracy in float32, which for needle-like splats (cond ~1e4)
// exceeds the parity tolerance.  conic_basis runs once per Gaussian in the
// projection (float64, from the float64 conic and its determinant).
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float4 conic_basis(double a, double b, double c, double det) {
  const double h = 0.5 * (a - c);
  const double r = sqrt(h * h + b * b);
  const double l1 = 0.5 * (a + c) + r;             // larger eigenvalue, no cancellation
  const double l2 = l1 > 0.0 ? fmax(det, 0.0) / l1 : 0.0;  // smaller one from the determinant
  double ex = h >= 0.0 ? h + r : b, ey = h >= 0.0 ? b : r - h;  // whichever form does not cancel
  const double nn = sqrt(ex * ex + ey * ey);
  if (nn > 0.0) {
    const double inv = 1.0 / nn;
    ex *= inv;
    ey *= inv;
  } else {
    ex = 1.0;
    ey = 0.0;
  }
  const double f1 = sqrt(0.5 * double(kLog2e) * l1), f2 = sqrt(0.5 * double(kLog2e) * l2);
  return make_float4(float(f1 * ex), float(f1 * ey), float(-f2 * ey), float(f2 * ex));
}

// Per-(splat, tile) blend record, built once by the producer warp from r0, r1:
//   k   = r1
//   m   = (-k1 . mean_rel, -k2 . mean_rel, alpha, 0)
//   ctr = mean_rel = mean - tile origin (the backward's d_conic offsets)
// so a pixel costs four FFMA + FMUL + FFMA, and p2 <= 0 by construction.
// Both blend kernels evaluate from the same records with the same
// intrinsics, so their alphas (and contributor sets) are bit-identical; near
// the 1/255 and 0.99 thresholds the float64 slow path (eval_alpha_f64)
// decides from the global hi/lo record.
__device__ __forceinline__ void make_tile_splat(float4 r0, float4 k, float alpha, float tile_x0, float tile_y0,
                                                float4& m, float2& ctr) {
  // tile-relative mean in float32 (two roundings, < 1 ulp of |mean_rel|)
  const float mx = __fadd_rn(__fsub_rn(r0.x, tile_x0), r0.z);
  const float my = __fadd_rn(__fsub_rn(r0.y, tile_y0), r0.w);
  m = make_float4(-__fmaf_rn(k.x, mx, __fmul_rn(k.y, my)), -__fmaf_rn(k.z, mx, __fmul_rn(k.w, my)), alpha, 0.0f);
  ctr = make_float2(mx, my);
}

// Alpha of one (pixel, splat) pair (rasterizer.py:171-177).  lx, ly:
// tile-local pixel centre (col + 0.5); px, py: absolute pixel centre.
// e.ok says whether the pair is blended (min(0.99, a_raw) >= 1/255 iff
// a_raw >= 1/255) and e.a is min(0.99, a_raw) without the skip zeroing,
// which the callers fold into their own selects.  Within kGuard of either
// threshold the pair is re-evaluated in float64 from the hi/lo record, so
// the skip and clamp decisions are the reference's.
__device__ __forceinline__ AlphaEval eval_alpha_tile(float lx, float ly, float px, float py, float4 k, float4 m,
                                                         const float4* __restrict__ rec, const uint32_t* s_id, int j) {
  AlphaEval e;
  e.v1 = __fmaf_rn(k.x, lx, __fmaf_rn(k.y, ly, m.x));
  e.v2 = __fmaf_rn(k.z, lx, __fmaf_rn(k.w, ly, m.y));
  const float p2 = __fmaf_rn(-e.v1, e.v1, -__fmul_rn(e.v2, e.v2));
  e.g = ex2_approx(p2);
  e.a_raw = __fmul_rn(m.z, e.g);
  if (fabsf(e.a_raw - kAlphaEps) <= kGuard * kAlphaEps || fabsf(e.a_raw - kAlphaClamp) <= kGuard) {
    eval_alpha_f64(px, py, rec + kRecWords * size_t(s_id[j]), e);
    e.ok = e.a > 0.0f;
    return e;
  }
  e.live = e.a_raw < kAlphaClamp;
  e.ok = e.a_raw >= kAlphaEps;
  e.a = fminf(kAlphaClamp, e.a_raw);
  return e;
}

// ---------------------------------------------------------------------------
// Geometry (float64).  Quaternion -> rotation (core.py:170-184).
template <typename Real>
__device__ __forceinline__ void quat_to_rot(Real r, Real i, Real j, Real k, Real R[9]) {
  R[0] = 1.0 - 2.0 * (j * j + k * k);
  R[1] = 2.0 * (i * j - r * k);
  R[2] = 2.0 * (i * k + r * j);
  R[3] = 2.0 * (i * j + r * k);
  R[4] = 1.0 - 2.0 * (i * i + k * k);
  R[5] = 2.0 * (j * k - r * i);
  R[6] = 2.0 * (i * k - r * j);
  R[7] = 2.0 * (j * k + r * i);
  R[8] = 1.0 - 2.0 * (i * i + j * j);
}

// SH basis (sh.py:32-63), float32, zero above the active degree.
__device__ __forceinline__ void sh_basis(float x, float y, float z, int degree, float b[16]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) b[k] = 0.0f;
  b[0] = kC0;
  if (degree >= 1) {
    b[1] = -kC1 * y;
    b[2] = kC1 * z;
    b[3] = -kC1 * x;
  }
  if (degree >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = kC2_0 * x * y;
    b[5] = kC2_1 * y * z;
    b[6] = kC2_2 * (2.0f * zz - xx - yy);
    b[7] = kC2_3 * x * z;
    b[8] = kC2_4 * (xx - yy);
    if (degree >= 3) {
      b[9] = kC3_0 * y * (3.0f * xx - yy);
      b[10] = kC3_1 * x * y * z;
      b[11] = kC3_2 * y * (4.0f * zz - xx - yy);
      b[12] = kC3_3 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
      b[13] = kC3_4 * x * (4.0f * zz - xx - yy);
      b[14] = kC3_5 * z * (xx - yy);
      b[15] = kC3_6 * x * (xx - 3.0f * yy);
    }
  }
}

// d(basis)/d(direction) contracted with d_basis (sh.py:66-109):
// returns sum_k d_basis[k] * d basis_k / d dir.
__device__ __forceinline__ void sh_basis_vjp(float x, float y, float z, int degree, const float db[16],
                                             float& gx, float& gy, float& gz) {
  gx = gy = gz = 0.0f;
  if (degree >= 1) {
    gy += -kC1 * db[1];
    gz += kC1 * db[2];
    gx += -kC1 * db[3];
  }
  if (degree >= 2) {
    gx += kC2_0 * y * db[4];
    gy += kC2_0 * x * db[4];
    gy += kC2_1 * z * db[5];
    gz += kC2_1 * y * db[5];
    gx += kC2_2 * (-2.0f * x) * db[6];
    gy += kC2_2 * (-2.0f * y) * db[6];
    gz += kC2_2 * (4.0f * z) * db[6];
    gx += kC2_3 * z * db[7];
    gz += kC2_3 * x * db[7];
    gx += kC2_4 * (2.0f * x) * db[8];
    gy += kC2_4 * (-2.0f * y) * db[8];
  }
  if (degree >= 3) {
    const float xx = x * x, yy = y * y, zz = z * z;
    gx += kC3_0 * 6.0f * x * y * db[9];
    gy += kC3_0 * (3.0f * xx - 3.0f * yy) * db[9];
    gx += kC3_1 * y * z * db[10];
    gy += kC3_1 * x * z * db[10];
    gz += kC3_1 * x * y * db[10];
    gx += kC3_2 * (-2.0f * x * y) * db[11];
    gy += kC3_2 * (4.0f * zz - xx - 3.0f * yy) * db[11];
    gz += kC3_2 * 8.0f * y * z * db[11];
    gx += kC3_3 * (-6.0f * x * z) * db[12];
    gy += kC3_3 * (-6.0f * y * z) * db[12];
    gz += kC3_3 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * db[12];
    gx += kC3_4 * (4.0f * zz - 3.0f * xx - yy) * db[13];
    gy += kC3_4 * (-2.0f * x * y) * db[13];
    gz += kC3_4 * 8.0f * x * z * db[13];
    gx += kC3_5 * 2.0f * x * z * db[14];
    gy += kC3_5 * (-2.0f * y * z) * db[14];
    gz += kC3_5 * (xx - yy) * db[14];
    gx += kC3_6 * (3.0f * xx - 3.0f * yy) * db[15];
    gy += kC3_6 * (-6.0f * x * y) * db[15];
  }
}

// Status plumbing shared by the C-ABI entry points.
int record_cuda_error(cudaError_t err);
int check_launch();

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  A kernel launched with launch_pdl may be
// scheduled while its stream predecessor's last blocks still run (its blocks
// take the SM slots the predecessor's tail frees); every such kernel begins
// with pdl_begin(): griddepcontrol.wait blocks until the predecessor grid has
// completed and its memory is visible (so no read or write of this kernel can
// race it), then launch_dependents lets the successor do the same.  After a
// kernel that never triggers (a library kernel, a memset) the wait returns
// at once and the launch is an ordinary stream-ordered one.
#ifndef GS_PDL
#define GS_PDL 1
#endif

#ifndef GS_PDL_TRIGGER
#define GS_PDL_TRIGGER 1
#endif
__device__ __forceinline__ void pdl_begin() {
#if GS_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if GS_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
#endif
}

// wait only: the successor launches when this grid's blocks exit (implicit
// trigger).  The binning's kernels use it: an early trigger puts the next
// kernel's waiting blocks beside the tail of the look-back passes (bin_and_sort
// 0.485 ms with it, 0.471 without); the loss kernels gain from it (0.211 ->
// 0.203 ms); the blends and the per-Gaussian kernels are indifferent.
__device__ __forceinline__ void pdl_wait() {
#if GS_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// GS_PDL_LAUNCH=0 in the environment launches every kernel without the
// programmatic attribute (A/B measurements; read once)
inline int pdl_launch_enabled() {
  static const int on = [] {
    const char* v = std::getenv("GS_PDL_LAUNCH");
    return (v && v[0] == '0') ? 0 : 1;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (GS_PDL && pdl_launch_enabled()) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);   // errors surface through check_launch()
}

// Zero up to two word ranges as a programmatically launched kernel (a
// cudaMemsetAsync node between two kernels would break the launch chain).
static __global__ void zero_words_kernel(uint32_t* a, int64_t na, uint32_t* b, int64_t nb) {
  pdl_begin();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < na + nb; i += stride) {
    if (i < na) a[i] = 0u;
    else b[i - na] = 0u;
  }
}

// bytes must be multiples of 4 (else a memset); returns the launch status
inline cudaError_t zero_async(void* a, size_t a_bytes, void* b, size_t b_bytes, cudaStream_t s) {
  if ((a_bytes | b_bytes) & 3u) {
    cudaError_t e = a_bytes ? cudaMemsetAsync(a, 0, a_bytes, s) : cudaSuccess;
    if (e == cudaSuccess && b_bytes) e = cudaMemsetAsync(b, 0, b_bytes, s);
    return e;
  }
  const int64_t words = int64_t((a_bytes + b_bytes) / 4);
  if (words == 0) return cudaSuccess;
  const int64_t blocks = (words + 1023) / 1024;
  launch_pdl(zero_words_kernel, unsigned(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, s,
             static_cast<uint32_t*>(a), int64_t(a_bytes / 4), static_cast<uint32_t*>(b), int64_t(b_bytes / 4));
  return cudaGetLastError();
}

}  // namespace gs
