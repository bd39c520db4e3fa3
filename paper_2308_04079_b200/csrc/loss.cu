// L1 + D-SSIM training loss and its image gradient — replaces splatlab
// optimizer.loss (optimizer.py:141-163) with ssim_map / ssim_backward
// (ssim.py:50-84): 11x11 Gaussian window (sigma 1.5), separable, zero
// padding, per channel.
//
// Two tiled passes over 16x16 output tiles with a 5-pixel halo staged in
// shared memory:
//   pass 1: the five filtered moments (mu_x, mu_y, E[x^2], E[y^2], E[xy]) in
//           float64, the SSIM value, the three adjoint source maps
//           (d_mu_x, d_E[x^2], d_E[xy]) and block partial sums of SSIM and |x-y|;
//   pass 2: the adjoint filter of the source maps (the symmetric, zero-padded
//           filter is self-adjoint, ssim.py:24-31) plus the L1 sign term.
// A 1-thread finalize kernel turns the sums into the scalar loss.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kT = 16;        // output tile edge
constexpr int kR = 5;         // window radius (11 taps)
constexpr int kIn = kT + 2 * kR;  // 26
constexpr double kC1 = 0.01 * 0.01;
constexpr double kC2 = 0.03 * 0.03;

struct Window {
  float w[11];
  double wd[11];
};

__host__ Window make_window() {
  Window W;
  double s = 0.0, v[11];
  for (int i = 0; i < 11; ++i) {
    const double x = double(i) - 5.0;
    v[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
    s += v[i];
  }
  for (int i = 0; i < 11; ++i) {
    W.wd[i] = v[i] / s;
    W.w[i] = float(W.wd[i]);
  }
  return W;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// pass 1 -------------------------------------------------------------------
__global__ void __launch_bounds__(256)
ssim_forward_kernel(const float* __restrict__ img, const float* __restrict__ gt, int W, int H, Window win,
                    double d_map, float* __restrict__ src, double* __restrict__ sums) {
  __shared__ float s_x[kIn][kIn][3];
  __shared__ float s_y[kIn][kIn][3];
  __shared__ double s_h[kIn][kT][5];   // horizontal pass of one channel: 5 moments
  __shared__ double s_red[8];
  const int t = threadIdx.x;
  const int ox = blockIdx.x * kT, oy = blockIdx.y * kT;
  for (int i = t; i < kIn * kIn; i += 256) {
    const int r = i / kIn, c = i % kIn;
    const int gx = ox + c - kR, gy = oy + r - kR;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    const size_t p = in ? (size_t(gy) * W + gx) * 3 : 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      s_x[r][c][ch] = in ? img[p + ch] : 0.0f;
      s_y[r][c][ch] = in ? gt[p + ch] : 0.0f;
    }
  }
  const int lx = t % kT, ly = t / kT;
  const int gx = ox + lx, gy = oy + ly;
  const bool inside = gx < W && gy < H;
  const size_t p = inside ? size_t(gy) * W + gx : 0;
  double ssim_sum = 0.0, l1_sum = 0.0, sq_sum = 0.0;
  for (int ch = 0; ch < 3; ++ch) {
    __syncthreads();
    for (int i = t; i < kIn * kT; i += 256) {
      const int r = i / kT, c = i % kT;
      double a = 0, b = 0, xx = 0, yy = 0, xy = 0;
#pragma unroll
      for (int k = 0; k < 11; ++k) {
        const double x = s_x[r][c + k][ch], y = s_y[r][c + k][ch], w = win.wd[k];
        a += w * x;
        b += w * y;
        xx += w * x * x;
        yy += w * y * y;
        xy += w * x * y;
      }
      s_h[r][c][0] = a;
      s_h[r][c][1] = b;
      s_h[r][c][2] = xx;
      s_h[r][c][3] = yy;
      s_h[r][c][4] = xy;
    }
    __syncthreads();
    if (inside) {
      double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < 11; ++k)
#pragma unroll
        for (int j = 0; j < 5; ++j) m[j] += win.wd[k] * s_h[ly + k][lx][j];
      const double mu_x = m[0], mu_y = m[1];
      const double sx = m[2] - mu_x * mu_x, sy = m[3] - mu_y * mu_y, sxy = m[4] - mu_x * mu_y;
      const double a1 = 2.0 * mu_x * mu_y + kC1, a2 = 2.0 * sxy + kC2;
      const double b1 = mu_x * mu_x + mu_y * mu_y + kC1, b2 = sx + sy + kC2;
      ssim_sum += (a1 * a2) / (b1 * b2);
      // ssim_backward (ssim.py:67-84) with a constant d_map
      const double denom = b1 * b2;
      const double d_a1 = d_map * a2 / denom, d_a2 = d_map * a1 / denom;
      const double d_b1 = -d_a1 * (a1 / b1), d_b2 = -d_a2 * (a2 / b2);
      const double d_mu = 2.0 * mu_y * d_a1 + 2.0 * mu_x * d_b1 - 2.0 * mu_y * d_a2 - 2.0 * mu_x * d_b2;
      src[9 * p + 3 * 0 + ch] = float(d_mu);
      src[9 * p + 3 * 1 + ch] = float(d_b2);
      src[9 * p + 3 * 2 + ch] = float(2.0 * d_a2);
      const double diff = double(s_x[ly + kR][lx + kR][ch]) - double(s_y[ly + kR][lx + kR][ch]);
      l1_sum += fabs(diff);
      sq_sum += diff * diff;   // for the step's PSNR (optimizer.py:257-259)
    }
  }
  const double s1 = block_sum(ssim_sum, s_red);
  const double s2 = block_sum(l1_sum, s_red);
  const double s3 = block_sum(sq_sum, s_red);
  if (t == 0) {
    atomicAdd(&sums[0], s1);
    atomicAdd(&sums[1], s2);
    atomicAdd(&sums[2], s3);
  }
}

// pass 2 -------------------------------------------------------------------
__global__ void __launch_bounds__(256)
ssim_backward_kernel(const float* __restrict__ img, const float* __restrict__ gt, const float* __restrict__ src,
                     int W, int H, Window win, float l1_scale, float* __restrict__ d_image) {
  __shared__ float s_s[kIn][kIn][9];
  __shared__ float s_h[kIn][kT][9];
  const int t = threadIdx.x;
  const int ox = blockIdx.x * kT, oy = blockIdx.y * kT;
  for (int i = t; i < kIn * kIn; i += 256) {
    const int r = i / kIn, c = i % kIn;
    const int gx = ox + c - kR, gy = oy + r - kR;
    const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
    const size_t p = in ? (size_t(gy) * W + gx) * 9 : 0;
#pragma unroll
    for (int j = 0; j < 9; ++j) s_s[r][c][j] = in ? src[p + j] : 0.0f;
  }
  __syncthreads();
  for (int i = t; i < kIn * kT; i += 256) {
    const int r = i / kT, c = i % kT;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      float a = 0.0f;
#pragma unroll
      for (int k = 0; k < 11; ++k) a = fmaf(win.w[k], s_s[r][c + k][j], a);
      s_h[r][c][j] = a;
    }
  }
  __syncthreads();
  const int lx = t % kT, ly = t / kT;
  const int gx = ox + lx, gy = oy + ly;
  if (gx >= W || gy >= H) return;
  const size_t p = size_t(gy) * W + gx;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float f[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 11; ++k)
#pragma unroll
      for (int m = 0; m < 3; ++m) f[m] = fmaf(win.w[k], s_h[ly + k][lx][3 * m + ch], f[m]);
    const float x = img[3 * p + ch], y = gt[3 * p + ch];
    const float diff = x - y;
    const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);  // np.sign
    d_image[3 * p + ch] = sgn * l1_scale + f[0] + 2.0f * x * f[1] + y * f[2];
  }
}

__global__ void loss_finalize_kernel(const double* __restrict__ sums, double count, double lambda,
                                     float* __restrict__ loss) {
  const double l1 = sums[1] / count;
  const double dssim = (1.0 - sums[0] / count) / 2.0;
  loss[0] = float((1.0 - lambda) * l1 + lambda * dssim);
  loss[1] = float(l1);
  loss[2] = float(sums[0] / count);
  loss[3] = float(sums[2] / count);   // mean squared error
}

}  // namespace
}  // namespace gs

extern "C" int gs_loss_workspace_size(int32_t width, int32_t height, size_t* bytes) {
  if (!bytes || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
  *bytes = 256 + size_t(width) * height * 9 * sizeof(float);
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
  float* src = reinterpret_cast<float*>(static_cast<char*>(workspace) + 256);
  cudaError_t e = cudaMemsetAsync(sums, 0, 3 * sizeof(double), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  const double count = double(width) * height * 3.0;
  const Window win = make_window();
  const dim3 grid((width + kT - 1) / kT, (height + kT - 1) / kT);
  // d_map = -lambda / (2 count) everywhere (optimizer.py:159)
  ssim_forward_kernel<<<grid, 256, 0, s>>>(image, target, width, height, win, -lambda / (2.0 * count), src,
                                           sums);
  int st = check_launch();
  if (st != GS_OK) return st;
  ssim_backward_kernel<<<grid, 256, 0, s>>>(image, target, src, width, height, win, float((1.0 - lambda) / count),
                                            d_image);
  if ((st = check_launch()) != GS_OK) return st;
  loss_finalize_kernel<<<1, 1, 0, s>>>(sums, count, lambda, loss_out);
  return check_launch();
}
