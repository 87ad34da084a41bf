// Host/device utilities shared by the search kernels: patch-valid maps,
// window offsets, TMA descriptor encoding.
#include <stdlib.h>

#include "search_common.cuh"
#include "tma.cuh"

namespace pxst {
namespace {

// Patch-valid map (pv_tile_block), one 32 x 16 output tile per block.
__global__ void __launch_bounds__(256) k_pv_tile(const uint8_t* __restrict__ valid,
                                                 const float* __restrict__ fm, int os, int of,
                                                 int lr, int hr, int lc, int hc,
                                                 uint8_t* __restrict__ pv, float* __restrict__ fmn) {
  __shared__ PvShared sm;
  pv_tile_block(sm, blockIdx.x, blockIdx.y, threadIdx.x, threadIdx.y, valid, fm, os, of, lr, hr,
                lc, hc, pv, fmn);
}

__global__ void k_span_max(const TileGeo* __restrict__ geo, int64_t n, int* out) {
  __shared__ int sr[32], sc[32];
  int mr = -1, mc = -1;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    mr = max(mr, geo[k].span_r);
    mc = max(mc, geo[k].span_c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sr[w] = mr; sc[w] = mc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) { mr = max(mr, sr[i]); mc = max(mc, sc[i]); }
    mr = max(mr, sr[0]);
    mc = max(mc, sc[0]);
    out[0] = mr;
    out[1] = mc;
  }
}

}  // namespace

int tile_span_max_dev(const TileGeo* geo, int64_t n, int* out_dev, cudaStream_t s) {
  k_span_max<<<1, 1024, 0, s>>>(geo, n, out_dev);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

int tile_span_max(const TileGeo* geo, int64_t n, int* out, cudaStream_t s) {
  Scratch d;
  if (int e = d.alloc(2 * sizeof(int), s)) return e;
  k_span_max<<<1, 1024, 0, s>>>(geo, n, d.as<int>());
  PXST_CHECK_LAUNCH();
  PXST_CHECK_CUDA(cudaMemcpyAsync(out, d.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  PXST_CHECK_CUDA(cudaStreamSynchronize(s));
  return PXST_OK;
}

int make_pv(const pxst_ref* ref, int lr, int hr, int lc, int hc, uint8_t* pv, float* fmn,
            cudaStream_t s) {
  PXST_REQUIRE(lr <= hr && lc <= hc && hr - lr <= kPvMaxHalo && hc - lc <= kPvMaxHalo,
               "patch extent too large");
  dim3 g((unsigned)((ref->of + kPvC - 1) / kPvC), (unsigned)((ref->os + kPvR - 1) / kPvR));
  PXST_REQUIRE(g.y <= kMaxGridY, "reference image too tall");
  k_pv_tile<<<g, dim3(32, 8), 0, s>>>(ref->valid, ref->fm, static_cast<int>(ref->os),
                              static_cast<int>(ref->of), lr, hr, lc, hc, pv, fmn);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

__global__ void k_fill_offsets(double* __restrict__ out, int na, int nb, double step) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < na + nb) {
    const int n = i < na ? na : nb, k0 = i < na ? i : i - na;
    const double k = static_cast<double>(k0 - (n - 1) / 2);
    out[i] = step > 0.0 ? step * k : k;          // window_offsets, on the device
  }
}

int fill_offsets(double* out, int na, int nb, double step, cudaStream_t s) {
  // A device fill instead of a pageable host->device copy, which would
  // synchronise the stream before it starts.
  k_fill_offsets<<<(na + nb + 127) / 128, 128, 0, s>>>(out, na, nb, step);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

std::vector<double> window_offsets(int64_t half, double step) {
  std::vector<double> o;
  if (step <= 0.0) {
    for (int64_t k = -half; k <= half; ++k) o.push_back(static_cast<double>(k));
  } else {
    // Python round() (recon.py:55): ties to even, as nearbyint in the default
    // rounding mode (llround would round 0.5 away from zero)
    const int64_t kh = static_cast<int64_t>(nearbyint(static_cast<double>(half) / step));
    for (int64_t k = -kh; k <= kh; ++k) o.push_back(step * static_cast<double>(k));
  }
  return o;
}

int steps_per_pixel(double step) {
  if (step <= 0.0) return 1;
  const double q = 1.0 / step;
  const double qr = nearbyint(q);
  if (qr >= 1.0 && qr <= 16.0 && fabs(q - qr) < 1e-9 && fabs(step * qr - 1.0) < 1e-12)
    return static_cast<int>(qr);
  return 0;
}

int check_ref(const pxst_ref* r) {
  PXST_REQUIRE(r && r->fm && r->valid && r->os > 0 && r->of > 0, "bad reference image");
  PXST_REQUIRE(r->os * r->of < (int64_t(1) << 31), "reference image too large");
  return PXST_OK;
}

bool force_generic() {
  const char* v = getenv("PXST_FORCE_GENERIC");
  return v && v[0] == '1';
}

int encode_tmap_2d_f32(CUtensorMap* map, const float* base, int64_t rows, int64_t cols,
                       int64_t pitch_elems, int box_rows, int box_cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
      return set_error(PXST_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch_elems * 4)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                      strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(PXST_ECUDA, "cuTensorMapEncodeTiled failed (%d): rows %lld cols %lld box %dx%d",
                     static_cast<int>(r), (long long)rows, (long long)cols, box_rows, box_cols);
  return PXST_OK;
}

}  // namespace pxst
