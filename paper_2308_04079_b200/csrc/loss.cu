// L1 + D-SSIM training loss and its image gradient — replaces splatlab
// optimizer.loss (optimizer.py:141-163) with ssim_map / ssim_backward
// (ssim.py:50-84): 11x11 Gaussian window (sigma 1.5), separable, zero
// padding, per channel.
//
// Two tiled passes over 32x16 output tiles with a 5-pixel halo staged in
// shared memory:
//   pass 1: the five filtered moments (mu_x, mu_y, E[x^2], E[y^2], E[xy]) in
//           shifted float32, the SSIM value (float64), the three adjoint source maps
//           (d_mu_x, d_E[x^2], d_E[xy]) and block partial sums of SSIM and |x-y|;
//   pass 2: the adjoint filter of the source maps (the symmetric, zero-padded
//           filter is self-adjoint, ssim.py:24-31) plus the L1 sign term.
// A 1-thread finalize kernel turns the sums into the scalar loss.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kR = 5;         // window radius (11 taps)
#ifndef GS_SSIM_REAL
#define GS_SSIM_REAL double   // per-pixel SSIM and adjoint precision
#endif
using SsimReal = GS_SSIM_REAL;
constexpr double kC1 = 0.01 * 0.01;
constexpr double kC2 = 0.03 * 0.03;

struct Window {
  float w[11];
  double wd[11];
  float rowsum;   // sum of the 11 float32 taps
  double total;   // (sum of the float32 taps)^2: the 2-D filter's mass
};

__host__ Window make_window() {
  Window W;
  double s = 0.0, v[11];
  for (int i = 0; i < 11; ++i) {
    const double x = double(i) - 5.0;
    v[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
    s += v[i];
  }
  double fs = 0.0;
  float rs = 0.0f;
  for (int i = 0; i < 11; ++i) {
    W.wd[i] = v[i] / s;
    W.w[i] = float(W.wd[i]);
    fs += double(W.w[i]);
    rs += W.w[i];
  }
  W.rowsum = rs;
  W.total = fs * fs;
  return W;
}

// pass 1 -------------------------------------------------------------------
// The five filtered moments are accumulated in float32 on values shifted by
// kShift (sigma^2 and the covariance are shift-invariant; mu is shifted back
// exactly): |x - 0.5| <= 0.5 for images in [0, 1] keeps the E[x^2] - mu^2
// cancellation error near 1e-7 absolute, four orders below the SSIM
// constant C2 = 9e-4 that every variance is added to.  Zero padding is
// staged as the shifted value of 0.  The per-pixel SSIM value and its
// adjoint are formed in float64.
//
// Tiles of kTW x kTH outputs (42 x 26 inputs with the halo), 384 threads,
// register blocking: a horizontal item filters kRunX consecutive outputs of
// one row and channel from one register window; a vertical item filters
// kRunY consecutive rows of one column and channel.  One horizontal round
// (3 x 26 x 4 = 312 items) and one vertical round (3 x 32 x 4 = 384 items).
constexpr float kShift = 0.5f;
constexpr int kTW = 32, kTH = 16;
constexpr int kInW = kTW + 2 * kR, kInH = kTH + 2 * kR;   // 42 x 26
constexpr int kLossThreads = 384;
constexpr int kRunX = 8, kRunY = 4;
constexpr int kWinX = kRunX + 10, kWinY = kRunY + 10;
// input rows padded to 44 floats (176 B): a run's 18-tap window is read as
// five 16-byte loads (the 20 floats from c0, c0 a multiple of 8), and the
// 8 lanes of a quarter warp (4 runs x 2 rows) hit disjoint banks
constexpr int kPitchIn = 44, kPitchH = kTW + 1;
static_assert(kPitchIn >= kInW + 2 && kPitchIn % 4 == 0, "input pitch");

struct FwdSmem {
  alignas(16) float x[3][kInH][kPitchIn];
  alignas(16) float y[3][kInH][kPitchIn];
  float h[3][5][kInH][kPitchH];   // horizontal pass: channel, moment, row, col
  double red[kLossThreads / 32];
};
struct BwdSmem {
  alignas(16) float src[9][kInH][kPitchIn];
  float h[9][kInH][kPitchH];
};

__device__ __forceinline__ double block_sum384(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kLossThreads / 32; ++i) s += red[i];
  return s;
}

__global__ void __launch_bounds__(kLossThreads)
ssim_forward_kernel(const float* __restrict__ img, const float* __restrict__ gt, int W, int H, Window win,
                    double d_map, float* __restrict__ src, double* __restrict__ sums) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  const int t = threadIdx.x;
  const int ox = blockIdx.x * kTW, oy = blockIdx.y * kTH;
  for (int i = t; i < kInH * kInW; i += kLossThreads) {
    const int r = i / kInW, c = i - r * kInW;
    const int gx = ox + c - kR, gy = oy + r - kR;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    const size_t p = in ? (size_t(gy) * W + gx) * 3 : 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      sm.x[ch][r][c] = (in ? img[p + ch] : 0.0f) - kShift;
      sm.y[ch][r][c] = (in ? gt[p + ch] : 0.0f) - kShift;
    }
  }
  __syncthreads();
  // horizontal: each input of the run's window is read once (16-byte loads),
  // its three products formed once, and scattered into the (up to 8) outputs
  // whose taps cover it: 5 FFMA per tap and output
  constexpr int kRunsX = kTW / kRunX;
  for (int i = t; i < 3 * kInH * kRunsX; i += kLossThreads) {
    const int ch = i / (kInH * kRunsX), rem = i - ch * (kInH * kRunsX);
    const int r = rem / kRunsX, c0 = (rem - r * kRunsX) * kRunX;
    const float4* xr = reinterpret_cast<const float4*>(&sm.x[ch][r][c0]);
    const float4* yr = reinterpret_cast<const float4*>(&sm.y[ch][r][c0]);
    float acc[kRunX][5];
#pragma unroll
    for (int o = 0; o < kRunX; ++o)
#pragma unroll
      for (int j = 0; j < 5; ++j) acc[o][j] = 0.f;
#pragma unroll
    for (int q = 0; q < (kWinX + 3) / 4; ++q) {
      const float4 xq = xr[q], yq = yr[q];
      const float xs[4] = {xq.x, xq.y, xq.z, xq.w}, ys[4] = {yq.x, yq.y, yq.z, yq.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = 4 * q + e;   // window position
        if (k < kWinX) {
          const float xv = xs[e], yv = ys[e];
          const float pxx = xv * xv, pyy = yv * yv, pxy = xv * yv;
#pragma unroll
          for (int o = 0; o < kRunX; ++o) {
            if (k - o >= 0 && k - o < 11) {
              const float w = win.w[k - o];
              acc[o][0] = fmaf(w, xv, acc[o][0]);
              acc[o][1] = fmaf(w, yv, acc[o][1]);
              acc[o][2] = fmaf(w, pxx, acc[o][2]);
              acc[o][3] = fmaf(w, pyy, acc[o][3]);
              acc[o][4] = fmaf(w, pxy, acc[o][4]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < kRunX; ++o)
#pragma unroll
      for (int j = 0; j < 5; ++j) sm.h[ch][j][r][c0 + o] = acc[o][j];
  }
  __syncthreads();
  // vertical: item = (channel, column, run of kRunY output rows); 384 items
  double ssim_sum = 0.0, l1_sum = 0.0, sq_sum = 0.0;
  {
    constexpr int kRunsY = kTH / kRunY;
    const int ch = t / (kTW * kRunsY), rem = t - ch * (kTW * kRunsY);
    const int c = rem % kTW, r0 = (rem / kTW) * kRunY;
    float m[kRunY][5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      float v[kWinY];
#pragma unroll
      for (int k = 0; k < kWinY; ++k) v[k] = sm.h[ch][j][r0 + k][c];
#pragma unroll
      for (int o = 0; o < kRunY; ++o) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 11; ++k) acc = fmaf(win.w[k], v[o + k], acc);
        m[o][j] = acc;
      }
    }
    const int gx = ox + c;
#pragma unroll
    for (int o = 0; o < kRunY; ++o) {
      const int gy = oy + r0 + o;
      if (gx < W && gy < H) {
        const size_t p = size_t(gy) * W + gx;
        // moments of the shifted values: sigma^2 / covariance directly, means shifted back
        const SsimReal msx = m[o][0], msy = m[o][1];
        const SsimReal sx = SsimReal(m[o][2]) - msx * msx, sy = SsimReal(m[o][3]) - msy * msy;
        const SsimReal sxy = SsimReal(m[o][4]) - msx * msy;
        const SsimReal mu_x = msx + SsimReal(kShift) * SsimReal(win.total), mu_y = msy + SsimReal(kShift) * SsimReal(win.total);
        const SsimReal a1 = SsimReal(2.0) * mu_x * mu_y + SsimReal(kC1), a2 = SsimReal(2.0) * sxy + SsimReal(kC2);
        const SsimReal b1 = mu_x * mu_x + mu_y * mu_y + SsimReal(kC1), b2 = sx + sy + SsimReal(kC2);
        // one float64 division per pixel and channel: 1/b1 = b2/(b1 b2), 1/b2 = b1/(b1 b2)
        const SsimReal inv = SsimReal(1.0) / (b1 * b2);
        ssim_sum += (a1 * a2) * inv;
        // ssim_backward (ssim.py:67-84) with a constant d_map
        const SsimReal d_a1 = SsimReal(d_map) * a2 * inv, d_a2 = SsimReal(d_map) * a1 * inv;
        const SsimReal d_b1 = -d_a1 * (a1 * b2 * inv), d_b2 = -d_a2 * (a2 * b1 * inv);
        const SsimReal d_mu = SsimReal(2.0) * mu_y * d_a1 + SsimReal(2.0) * mu_x * d_b1 - SsimReal(2.0) * mu_y * d_a2 - SsimReal(2.0) * mu_x * d_b2;
        // planar source maps [3 x 3][H x W]: coalesced rows for both passes
        // pixel-major source maps (9 floats per pixel): planar maps were
        // measured slower in the backward's halo load (91 vs 78 us)
        src[9 * p + 3 * 0 + ch] = float(d_mu);
        src[9 * p + 3 * 1 + ch] = float(d_b2);
        src[9 * p + 3 * 2 + ch] = float(SsimReal(2.0) * d_a2);
        const SsimReal diff = SsimReal(img[3 * p + ch]) - SsimReal(gt[3 * p + ch]);
        l1_sum += fabs(diff);
        sq_sum += diff * diff;   // for the step's PSNR (optimizer.py:257-259)
      }
    }
  }
  const double s1 = block_sum384(ssim_sum, sm.red);
  const double s2 = block_sum384(l1_sum, sm.red);
  const double s3 = block_sum384(sq_sum, sm.red);
  if (t == 0) {   // per-block partials, summed in a fixed order by the finalize kernel (deterministic)
    const size_t b = size_t(blockIdx.y) * gridDim.x + blockIdx.x;
    sums[3 * b + 0] = s1;
    sums[3 * b + 1] = s2;
    sums[3 * b + 2] = s3;
  }
}

// pass 2 -------------------------------------------------------------------
// Same tiling: horizontal runs over the nine source maps, then vertical runs
// of kRunY rows per (channel, column) that combine the three filtered maps
// of the channel with the L1 sign term.
__global__ void __launch_bounds__(kLossThreads)
ssim_backward_kernel(const float* __restrict__ img, const float* __restrict__ gt, const float* __restrict__ src,
                     int W, int H, Window win, float l1_scale, float* __restrict__ d_image) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
  const int t = threadIdx.x;
  const int ox = blockIdx.x * kTW, oy = blockIdx.y * kTH;
  for (int i = t; i < kInH * kInW; i += kLossThreads) {
    const int r = i / kInW, c = i - r * kInW;
    const int gx = ox + c - kR, gy = oy + r - kR;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    const size_t p = in ? (size_t(gy) * W + gx) * 9 : 0;
#pragma unroll
    for (int j = 0; j < 9; ++j) sm.src[j][r][c] = in ? src[p + j] : 0.0f;
  }
  __syncthreads();
  // horizontal runs of 8 outputs, windows read with 16-byte loads (runs of 4
  // balance the 384 threads better, 4.9 vs 2.4 -> 3 rounds, but measured
  // slower: 93 vs 79 us, the doubled item count's index arithmetic)
  constexpr int kRunB = kRunX, kRunsB = kTW / kRunB, kWinB = kRunB + 10;
  for (int i = t; i < 9 * kInH * kRunsB; i += kLossThreads) {
    const int j = i / (kInH * kRunsB), rem = i - j * (kInH * kRunsB);
    const int r = rem / kRunsB, c0 = (rem - r * kRunsB) * kRunB;
    const float4* vr = reinterpret_cast<const float4*>(&sm.src[j][r][c0]);
    float v[4 * ((kWinB + 3) / 4)];
#pragma unroll
    for (int q = 0; q < (kWinB + 3) / 4; ++q) {
      const float4 f = vr[q];
      v[4 * q + 0] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
    }
#pragma unroll
    for (int o = 0; o < kRunB; ++o) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < 11; ++k) acc = fmaf(win.w[k], v[o + k], acc);
      sm.h[j][r][c0 + o] = acc;
    }
  }
  __syncthreads();
  constexpr int kRunsY = kTH / kRunY;
  const int ch = t / (kTW * kRunsY), rem = t - ch * (kTW * kRunsY);
  const int c = rem % kTW, r0 = (rem / kTW) * kRunY;
  float f[3][kRunY];
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    float v[kWinY];
#pragma unroll
    for (int k = 0; k < kWinY; ++k) v[k] = sm.h[3 * m + ch][r0 + k][c];
#pragma unroll
    for (int o = 0; o < kRunY; ++o) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < 11; ++k) acc = fmaf(win.w[k], v[o + k], acc);
      f[m][o] = acc;
    }
  }
  const int gx = ox + c;
#pragma unroll
  for (int o = 0; o < kRunY; ++o) {
    const int gy = oy + r0 + o;
    if (gx < W && gy < H) {
      const size_t p = size_t(gy) * W + gx;
      const float x = img[3 * p + ch], y = gt[3 * p + ch];
      const float diff = x - y;
      const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);  // np.sign
      d_image[3 * p + ch] = sgn * l1_scale + f[0][o] + 2.0f * x * f[1][o] + y * f[2][o];
    }
  }
}

// one block of 256 threads: the block partials in a fixed order (strided
// per thread, then a fixed shared-memory tree), so the loss is bit-identical
// run to run
constexpr int kFinThreads = 1024;
__global__ void __launch_bounds__(kFinThreads) loss_finalize_kernel(const double* __restrict__ part, int64_t blocks,
                                                                    double count, double lambda,
                                                                    float* __restrict__ loss) {
  pdl_begin();
  __shared__ double red[3][kFinThreads];
  // strided per thread with four loads in flight, then a fixed tree: the
  // summation order depends only on the block count (deterministic)
  double a[4][3] = {};
  int64_t b = threadIdx.x;
  for (; b + 3 * kFinThreads < blocks; b += 4 * kFinThreads)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < 3; ++k) a[u][k] += __ldg(part + 3 * (b + u * kFinThreads) + k);
  for (; b < blocks; b += kFinThreads)
#pragma unroll
    for (int k = 0; k < 3; ++k) a[0][k] += __ldg(part + 3 * b + k);
  for (int k = 0; k < 3; ++k) red[k][threadIdx.x] = (a[0][k] + a[1][k]) + (a[2][k] + a[3][k]);
  __syncthreads();
  for (int w = kFinThreads / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w)
      for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double sums[3] = {red[0][0], red[1][0], red[2][0]};
    const double l1 = sums[1] / count;
    const double dssim = (1.0 - sums[0] / count) / 2.0;
    loss[0] = float((1.0 - lambda) * l1 + lambda * dssim);
    loss[1] = float(l1);
    loss[2] = float(sums[0] / count);
    loss[3] = float(sums[2] / count);   // mean squared error
  }
}

}  // namespace
}  // namespace gs

namespace {
size_t loss_blocks(int32_t width, int32_t height) {
  return size_t((width + gs::kTW - 1) / gs::kTW) * size_t((height + gs::kTH - 1) / gs::kTH);
}
size_t loss_src_offset(int32_t width, int32_t height) {
  return (3 * sizeof(double) * loss_blocks(width, height) + 255) & ~size_t(255);
}
}  // namespace

extern "C" int gs_loss_workspace_size(int32_t width, int32_t height, size_t* bytes) {
  if (!bytes || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  *bytes = loss_src_offset(width, height) + size_t(width) * height * 9 * sizeof(float);
  return GS_OK;
}

extern "C" int gs_l1_dssim_loss(const float* image, const float* target, int32_t width, int32_t height, double lambda,
                                void* workspace, size_t workspace_bytes, float* loss_out, float* d_image,
                                void* stream) {
  using namespace gs;
  if (!image || !target || !loss_out || !d_image || !workspace || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  if (!(lambda >= 0.0 && lambda <= 1.0)) return GS_ERR_INVALID_ARG;
  size_t need = 0;
  gs_loss_workspace_size(width, height, &need);
  if (workspace_bytes < need) return GS_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* sums = static_cast<double*>(workspace);
  float* src = reinterpret_cast<float*>(static_cast<char*>(workspace) + loss_src_offset(width, height));
  cudaError_t e = cudaSuccess;
  const double count = double(width) * height * 3.0;
  const Window win = make_window();
  static bool configured = false;
  if (!configured) {
    e = cudaFuncSetAttribute(ssim_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FwdSmem)));
    if (e != cudaSuccess) return record_cuda_error(e);
    e = cudaFuncSetAttribute(ssim_backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(BwdSmem)));
    if (e != cudaSuccess) return record_cuda_error(e);
    configured = true;
  }
  const dim3 grid((width + kTW - 1) / kTW, (height + kTH - 1) / kTH);
  // d_map = -lambda / (2 count) everywhere (optimizer.py:159)
  launch_pdl(ssim_forward_kernel, grid, kLossThreads, sizeof(FwdSmem), s, image, target, width, height, win,
                                                                   -lambda / (2.0 * count), src, sums);
  int st = check_launch();
  if (st != GS_OK) return st;
  launch_pdl(ssim_backward_kernel, grid, kLossThreads, sizeof(BwdSmem), s, image, target, src, width, height, win,
                                                                    float((1.0 - lambda) / count), d_image);
  if ((st = check_launch()) != GS_OK) return st;
  launch_pdl(loss_finalize_kernel, 1, kFinThreads, 0, s, sums, int64_t(loss_blocks(width, height)), count, lambda, loss_out);
  return check_launch();
}
