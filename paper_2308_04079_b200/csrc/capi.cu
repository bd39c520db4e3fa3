// Library-level C-ABI helpers: version, status strings, CUDA error capture.
#include <cstdio>
#include <cstring>

#include "gs_common.cuh"

namespace gs {

// Per-thread copy of the last CUDA error (the library holds no other state).
static thread_local char g_last_error[256] = "";

int record_cuda_error(cudaError_t err) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(err), cudaGetErrorString(err));
  return GS_ERR_CUDA;
}

int check_launch() {
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? GS_OK : record_cuda_error(err);
}

}  // namespace gs

namespace gs {
namespace {
// FP32 FMA throughput probe: 8 independent FMA chains per thread, enough
// resident warps to saturate every SM's FMA pipes.
__global__ void __launch_bounds__(256) fma_probe_kernel(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = float(threadIdx.x + k) * 1e-3f;
  const float b = 0.999f, c = 1e-4f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  }
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1.0f) out[blockIdx.x] = s;  // never true; keeps the chains alive
}
}  // namespace
}  // namespace gs

extern "C" int gs_fp32_fma_probe(float* scratch, int32_t blocks, int32_t iters, void* stream) {
  if (!scratch || blocks <= 0 || iters <= 0) return GS_ERR_INVALID_ARG;
  gs::fma_probe_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(scratch, iters);
  return gs::check_launch();
}

extern "C" int gs_abi_version(void) { return GS_ABI_VERSION; }

extern "C" const char* gs_status_string(int status) {
  switch (status) {
    case GS_OK: return "ok";
    case GS_ERR_INVALID_ARG: return "invalid argument";
    case GS_ERR_ZERO_QUATERNION: return "zero-norm quaternion cannot be normalized";
    case GS_ERR_RESOURCE_LIMIT: return "resource limit exceeded (tiles or instances)";
    case GS_ERR_CAPACITY: return "instance buffer capacity too small";
    case GS_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

extern "C" int gs_last_cuda_error(char* buf, size_t len) {
  if (!buf || len == 0) return GS_ERR_INVALID_ARG;
  std::strncpy(buf, gs::g_last_error, len - 1);
  buf[len - 1] = '\0';
  return GS_OK;
}
