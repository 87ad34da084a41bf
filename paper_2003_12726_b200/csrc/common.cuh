// Shared device helpers for the PXST B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdio.h>

#include "pxst_b200.h"

namespace pxst {

// ---------------------------------------------------------------------------
// error reporting (thread-local message, int status codes)
// ---------------------------------------------------------------------------
int set_error(int code, const char* fmt, ...);
void count_launch(int n = 1);

#define PXST_CHECK_CUDA(expr)                                                    \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess)                                                       \
      return ::pxst::set_error(PXST_ECUDA, "%s failed: %s (%s:%d)", #expr,       \
                               cudaGetErrorString(_e), __FILE__, __LINE__);      \
  } while (0)

#define PXST_CHECK_LAUNCH()                                                      \
  do {                                                                           \
    ::pxst::count_launch();                                                      \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess)                                                       \
      return ::pxst::set_error(PXST_ECUDA, "kernel launch failed: %s (%s:%d)",   \
                               cudaGetErrorString(_e), __FILE__, __LINE__);      \
  } while (0)

#define PXST_REQUIRE(cond, ...)                                                  \
  do {                                                                           \
    if (!(cond)) return ::pxst::set_error(PXST_EINVAL, __VA_ARGS__);             \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Device-side bounds / invariant checks, compiled in with -DPXST_CHECKED
// (tools/checked_run.sh: the checked library runs the GPU tests; this pool
// has compute-sanitizer closed).  A failure prints the condition and traps.
#ifdef PXST_CHECKED
#define PXST_DCHECK(cond)                                                           \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("PXST_DCHECK failed: %s at %s:%d (block %d,%d,%d thread %d)\n", #cond, \
             __FILE__, __LINE__, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);   \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define PXST_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

// Keep memory freed with cudaFreeAsync in the device's default pool across
// synchronisations (the default release threshold of 0 hands it back to the
// OS at every sync, making the next cudaMallocAsync re-map pages: ms per call).
void retain_pool_memory();

// Stream-ordered scratch buffer, released on the stream at scope exit.
struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  int alloc(size_t bytes, cudaStream_t stream) {
    s = stream;
    retain_pool_memory();
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, stream);
    if (e != cudaSuccess) {
      p = nullptr;
      return set_error(PXST_ENOMEM, "cudaMallocAsync(%zu) failed: %s", bytes,
                       cudaGetErrorString(e));
    }
    return PXST_OK;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

constexpr int kMaxGridY = 65535;

// Blocks for a grid-stride loop over n items.
inline int grid_1d(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return static_cast<int>(b);
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Split coordinate: x = i + f with integer i = floor(x) and f in [0,1)
// (interp.py:39-42).  Computed in float64 exactly as the reference does.
struct Split {
  int i;
  double f;
};
__device__ __forceinline__ Split split(double x) {
  double fl = floor(x);
  return Split{static_cast<int>(fl), x - fl};
}

// Inclusive in-grid test 0 <= i+f <= n-1 for integer row i and frac f
// (interp.py:67).
__device__ __forceinline__ bool inside_1d(int i, double f, int64_t n) {
  return i >= 0 && (i < n - 1 || (i == n - 1 && f == 0.0));
}

// Masked bilinear read with renormalisation (interp.py:53-85) at integer
// base (i, j) and fractions (fx, fy).  Reads the global masked image fm and
// validity.  Returns whether the sample is valid; v receives num/den.
__device__ __forceinline__ bool masked_read(const float* __restrict__ fm,
                                            const uint8_t* __restrict__ valid, int64_t os,
                                            int64_t of, int i, int j, double fx, double fy,
                                            float& v) {
  if (!inside_1d(i, fx, os) || !inside_1d(j, fy, of)) return false;
  const int r0 = i, c0 = j;
  const int r1 = min(r0 + 1, static_cast<int>(os - 1));
  const int c1 = min(c0 + 1, static_cast<int>(of - 1));
  const float gx = static_cast<float>(fx), gy = static_cast<float>(fy);
  const float w00 = (1.f - gx) * (1.f - gy), w01 = (1.f - gx) * gy;
  const float w10 = gx * (1.f - gy), w11 = gx * gy;
  const int64_t a00 = (int64_t)r0 * of + c0, a01 = (int64_t)r0 * of + c1;
  const int64_t a10 = (int64_t)r1 * of + c0, a11 = (int64_t)r1 * of + c1;
  const bool m00 = __ldg(valid + a00), m01 = __ldg(valid + a01);
  const bool m10 = __ldg(valid + a10), m11 = __ldg(valid + a11);
  // den > 0 decided exactly from the float64 fractions (w00 > 0 always).
  const bool any = m00 || (fy > 0.0 && m01) || (fx > 0.0 && m10) || (fx > 0.0 && fy > 0.0 && m11);
  if (!any) return false;
  float den = 0.f, num = 0.f;
  if (m00) { den += w00; num = fmaf(w00, __ldg(fm + a00), num); }
  if (m01) { den += w01; num = fmaf(w01, __ldg(fm + a01), num); }
  if (m10) { den += w10; num = fmaf(w10, __ldg(fm + a10), num); }
  if (m11) { den += w11; num = fmaf(w11, __ldg(fm + a11), num); }
  v = num / den;
  return true;
}

}  // namespace pxst
