// split_half_recon's counter-based sample split (analysis.py:294-303,
// :326-335): every (frame, ss, fs) sample of the stack is
// assigned to half A or B by one bit of a SplitMix64 finaliser of its flat
// index.  The weights feed K2's frame-weight path (recon.py:94-95, 150-161).
#include "common.cuh"

namespace pxst {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ unsigned split_bit(unsigned long long seed, unsigned long long idx) {
  unsigned long long x = idx + seed * 0x9E3779B97F4A7C15ull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return static_cast<unsigned>(x & 1ull);
}

__global__ void k_split_weights(unsigned long long seed, int64_t n, int half,
                                float4* __restrict__ fw4, float* __restrict__ fw) {
  // four samples per thread (16-byte stores), scalar tail
  const int64_t n4 = n / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4;
       q += (int64_t)gridDim.x * blockDim.x) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned b = split_bit(seed, static_cast<unsigned long long>(4 * q + k));
      v[k] = static_cast<float>(half ? 1u - b : b);
    }
    fw4[q] = make_float4(v[0], v[1], v[2], v[3]);
  }
  for (int64_t q = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned b = split_bit(seed, static_cast<unsigned long long>(q));
    fw[q] = static_cast<float>(half ? 1u - b : b);
  }
}

__global__ void k_split_counts(unsigned long long seed, const int32_t* __restrict__ good,
                               int64_t n_good, int64_t plane, int32_t* __restrict__ counts) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < plane;
       p += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = 0;
    for (int64_t k = 0; k < n_good; ++k)
      c += split_bit(seed, static_cast<unsigned long long>(good[k]) * plane + p);
    counts[p] = c;
  }
}

}  // namespace
}  // namespace pxst

using namespace pxst;

extern "C" int pxst_split_weights(uint64_t seed, int64_t n_frames, int64_t ss, int64_t fs,
                                  int half, float* fw, void* stream) {
  PXST_REQUIRE(fw, "NULL pointer");
  PXST_REQUIRE(n_frames >= 0 && ss >= 0 && fs >= 0, "bad stack shape");
  PXST_REQUIRE(half == 0 || half == 1, "half must be 0 (A) or 1 (B)");
  const int64_t n = n_frames * ss * fs;
  if (n == 0) return PXST_OK;
  PXST_REQUIRE((reinterpret_cast<uintptr_t>(fw) & 15) == 0, "fw must be 16-byte aligned");
  k_split_weights<<<grid_1d(n / 4 + 1, kThreads), kThreads, 0, as_stream(stream)>>>(
      seed, n, half, reinterpret_cast<float4*>(fw), fw);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_split_counts(uint64_t seed, const int32_t* good, int64_t n_good, int64_t ss,
                                 int64_t fs, int32_t* counts_a, void* stream) {
  PXST_REQUIRE(counts_a && (good || n_good == 0), "NULL pointer");
  PXST_REQUIRE(n_good >= 0 && ss > 0 && fs > 0, "bad shape");
  k_split_counts<<<grid_1d(ss * fs, kThreads), kThreads, 0, as_stream(stream)>>>(
      seed, good, n_good, ss * fs, counts_a);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}
