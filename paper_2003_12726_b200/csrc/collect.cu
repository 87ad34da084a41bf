// Elementwise reductions for the single-process multi-GPU path
// (multigpu.py): a device adds a peer's copy of an accumulator into its own.
// Integer sums are exact (the fixed-point splat images), so any order of the
// peers gives the same bits; the float64 per-frame sums are added by every
// device in the same fixed peer order.
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

}  // namespace
}  // namespace pxst

using namespace pxst;

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
