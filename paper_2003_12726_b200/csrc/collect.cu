// Elementwise reductions for the single-process multi-GPU path
// (multigpu.py): a device adds a peer's copy of an accumulator into its own.
// Integer sums are exact (the fixed-point splat images), so any order of the
// peers gives the same bits; the float64 per-frame sums are added by every
// device in the same fixed peer order.
#include <algorithm>
#include <string.h>

#include "common.cuh"

namespace pxst {
namespace {

__global__ void k_add_i64(long long* __restrict__ dst, const long long* __restrict__ src,
                          int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

__global__ void k_add_f64(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

__global__ void k_or_u8(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] |= src[i];
}

// Mean and variance (ddof 0, as numpy's var) of the cells flagged valid: one
// block, every thread sums its strided share in a fixed order, a fixed tree
// adds the threads -- deterministic; two passes (mean, then squared
// deviations) like numpy.  out = (count, mean, var).
__global__ void __launch_bounds__(1024) k_masked_moments(const double* __restrict__ v,
                                                        const uint8_t* __restrict__ valid,
                                                        int64_t n, double* __restrict__ out) {
  __shared__ double sh[1024];
  __shared__ double s_mean, s_cnt;
  auto block_sum = [&](double x) {
    sh[threadIdx.x] = x;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
  };
  double c = 0.0, a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024)
    if (valid[i]) { c += 1.0; a += v[i]; }
  const double cnt = block_sum(c), sum = block_sum(a);
  if (threadIdx.x == 0) { s_cnt = cnt; s_mean = cnt > 0.0 ? sum / cnt : 0.0; }
  __syncthreads();
  const double mean = s_mean;
  double q = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024)
    if (valid[i]) { const double d = v[i] - mean; q += d * d; }
  const double ss = block_sum(q);
  if (threadIdx.x == 0) {
    out[0] = s_cnt;
    out[1] = mean;
    out[2] = s_cnt > 0.0 ? ss / s_cnt : 0.0;
  }
}

// Frame stack of another element type -> the float32 stack the kernels read
// (the reference takes any dtype and casts per use: recon.py:91
// scan.frames[...].astype(np.float64)).  The stack is uploaded in its own
// type -- half the bytes for 16-bit detector counts, no host-side conversion
// pass -- and converted here, 4 elements per thread.
template <class T>
__global__ void k_to_f32(const T* __restrict__ src, int64_t n, float* __restrict__ dst) {
  // 16 bytes of source per thread and step (one vector load), float4 stores;
  // both arrays are 16-byte aligned (checked by the caller), the tail goes
  // element by element.  (One element per thread ran at a fifth of the
  // memory rate for 16-bit counts.)
  constexpr int V = 16 / sizeof(T);
  const int64_t nv = n / V;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src);
  for (int64_t i = t0; i < nv; i += stride) {
    const uint4 raw = __ldg(s4 + i);
    T e[V];
    memcpy(e, &raw, 16);
    float f[V];
#pragma unroll
    for (int k = 0; k < V; ++k) f[k] = static_cast<float>(e[k]);   // RN, as numpy's astype
    if (V >= 4) {
#pragma unroll
      for (int k = 0; k < V; k += 4)
        reinterpret_cast<float4*>(dst + i * V)[k / 4] = make_float4(f[k], f[k + 1], f[k + 2], f[k + 3]);
    } else {
      reinterpret_cast<float2*>(dst + i * V)[0] = make_float2(f[0], f[V - 1]);
    }
  }
  for (int64_t i = nv * V + t0; i < n; i += stride) dst[i] = static_cast<float>(src[i]);
}
template <class T>
int launch_to_f32(const void* src, int64_t n, float* dst, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const int blocks = static_cast<int>(std::min<int64_t>((n / V + 255) / 256 + 1, 148 * 16));
  k_to_f32<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(src), n, dst);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

}  // namespace
}  // namespace pxst

using namespace pxst;

extern "C" int pxst_stack_to_f32(const void* src, int type_code, int64_t n, float* dst,
                                 void* stream) {
  PXST_REQUIRE(src && dst && n >= 0, "bad arguments");
  PXST_REQUIRE(((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0,
               "stack buffers must be 16-byte aligned");
  if (n == 0) return PXST_OK;
  cudaStream_t s = as_stream(stream);
  switch (type_code) {
    case PXST_U8: return launch_to_f32<uint8_t>(src, n, dst, s);
    case PXST_I8: return launch_to_f32<int8_t>(src, n, dst, s);
    case PXST_U16: return launch_to_f32<uint16_t>(src, n, dst, s);
    case PXST_I16: return launch_to_f32<int16_t>(src, n, dst, s);
    case PXST_U32: return launch_to_f32<uint32_t>(src, n, dst, s);
    case PXST_I32: return launch_to_f32<int32_t>(src, n, dst, s);
    case PXST_U64: return launch_to_f32<unsigned long long>(src, n, dst, s);
    case PXST_I64: return launch_to_f32<long long>(src, n, dst, s);
    case PXST_F64: return launch_to_f32<double>(src, n, dst, s);
    default: PXST_REQUIRE(false, "unknown element type code %d", type_code);
  }
  return PXST_OK;
}

extern "C" int pxst_masked_moments(const double* v, const uint8_t* valid, int64_t n, double* out,
                                   void* stream) {
  PXST_REQUIRE(v && valid && out && n >= 0, "bad arguments");
  k_masked_moments<<<1, 1024, 0, as_stream(stream)>>>(v, valid, n, out);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_add_i64(int64_t* dst, const int64_t* src, int64_t n, void* stream) {
  PXST_REQUIRE(dst && src && n >= 0, "bad arguments");
  if (n == 0) return PXST_OK;
  k_add_i64<<<grid_1d(n, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<long long*>(dst), reinterpret_cast<const long long*>(src), n);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_add_f64(double* dst, const double* src, int64_t n, void* stream) {
  PXST_REQUIRE(dst && src && n >= 0, "bad arguments");
  if (n == 0) return PXST_OK;
  k_add_f64<<<grid_1d(n, 256), 256, 0, as_stream(stream)>>>(dst, src, n);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_or_u8(uint8_t* dst, const uint8_t* src, int64_t n, void* stream) {
  PXST_REQUIRE(dst && src && n >= 0, "bad arguments");
  if (n == 0) return PXST_OK;
  k_or_u8<<<grid_1d(n, 256), 256, 0, as_stream(stream)>>>(dst, src, n);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}
