// K1 object formation (recon.py:99-141) and the interp primitives
// (interp.py:53-135).
//
// The reference accumulates the bilinear splat in float64 with np.bincount
// (interp.py:114-122).  The splat is bound by the L2 atomic units, so here a
// sample's four corners go out as two 16-byte float32 REDs (splat_grouped:
// 2 RED lane-ops per sample instead of 8 float64 ones) into at most 32
// float32 images, each covering a contiguous range of >= 24 frames (and
// <= N/32 frames for long stacks); a fixed-order float64 fold sums the
// images.  An image sums positive terms of a few dozen frames, so its
// relative error stays ~1e-7-1e-6 (the 1e-5 bar of SURVEY 8(c)); the
// summation order inside an image varies run to run.
#include "common.cuh"

namespace pxst {
namespace {

constexpr int kTR = 4, kTC = 32, kThreads = kTR * kTC;  // 4 rows x 32 fs pixels
constexpr int kFB = 8;                 // frames per load batch (loads before REDs)
constexpr int kTab = 256;              // frames per shared-memory frame table chunk
constexpr int64_t kMaxImages = 32;     // float32 chunk images per splat
constexpr int64_t kMinImageFrames = 24;  // frames summed per image, at least
constexpr int64_t kImageBytes = int64_t(1) << 30;
#ifndef PXST_K1_OCC
#define PXST_K1_OCC 8
#endif

// One thread per work pixel over the frame slice blockIdx.z.  Lanes of a
// warp are consecutive fs pixels, so the corner REDs of a warp land on a few
// consecutive cells (the cheap, row-coalesced atomic pattern).  Each sample
// issues two 16-byte float32 REDs (splat_grouped) into the chunk image of
// its frame batch; a batch's frame loads are all issued before its REDs.
__global__ void __launch_bounds__(kThreads, PXST_K1_OCC)
k_object_splat(pxst_scan sc, const double* __restrict__ u, const double* __restrict__ di,
               const double* __restrict__ dj, int64_t n0, int64_t m0, int64_t os, int64_t of,
               int64_t frame_lo, int64_t frame_hi, int64_t frames_per_z, float4* __restrict__ img,
               int bpi, unsigned long long* __restrict__ n_drop) {
  __shared__ double t_di[kTab], t_dj[kTab];
  __shared__ int64_t t_off[kTab];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = sc.roi[0] + (int64_t)blockIdx.y * kTR + warp;
  const int64_t c = sc.roi[2] + (int64_t)blockIdx.x * kTC + lane;
  const bool inroi = r < sc.roi[1] && c < sc.roi[3];
  const int64_t p = inroi ? r * sc.fs + c : 0;
  const bool live = inroi && sc.work[p] != 0;
  const int64_t plane = sc.ss * sc.fs;
  const double u0 = live ? u[p] : 0.0, u1 = live ? u[plane + p] : 0.0;
  const double w = live ? sc.w64[p] : 1.0;
  const double w2 = w * w;                       // recon.py:136
  const double inv_w = 1.0 / w;                  // value = I / W (interp.py:112), <= 1 ulp
  const double os1 = static_cast<double>(os - 1), of1 = static_cast<double>(of - 1);
  const int64_t n_o = os * of;
  const int64_t k_begin = frame_lo + (int64_t)blockIdx.z * frames_per_z;
  const int64_t k_end = min(frame_hi, k_begin + frames_per_z);
  unsigned long long dropped = 0;
  for (int64_t kc = k_begin; kc < k_end; kc += kTab) {
    const int nt = static_cast<int>(k_end - kc < kTab ? k_end - kc : kTab);
    __syncthreads();
    for (int t = threadIdx.x; t < nt; t += kThreads) {
      const int64_t f = sc.good[kc + t];
      t_di[t] = di[f];
      t_dj[t] = dj[f];
      t_off[t] = f * plane;
    }
    __syncthreads();
    // every lane runs the loop (the splat is warp-cooperative); lanes
    // without a work pixel splat nothing
    for (int b0 = 0; b0 < nt; b0 += kFB) {
      float4* out = img + ((kc - frame_lo + b0) / kFB / bpi) * n_o;
      float Iv[kFB];
#pragma unroll
      for (int b = 0; b < kFB; ++b)
        Iv[b] = (live && b0 + b < nt) ? __ldg(sc.frames + t_off[b0 + b] + p) : 0.f;
#pragma unroll
      for (int b = 0; b < kFB; ++b) {
        if (b0 + b >= nt) break;
        const double x = u0 - t_di[b0 + b] - static_cast<double>(n0);   // recon.py:138
        const double y = u1 - t_dj[b0 + b] - static_cast<double>(m0);
        const bool in = x >= 0.0 && x <= os1 && y >= 0.0 && y <= of1;   // interp.py:103-107
        dropped += (live && !in) ? 1 : 0;
        const bool act = live && in;
        const Split sx = split(act ? x : 0.0), sy = split(act ? y : 0.0);
        const double vw = (static_cast<double>(Iv[b]) * inv_w) * w2;   // value*weight (interp.py:112)
        splat_grouped_warp(out, (int64_t)sx.i * of + sy.i, sx.f, sy.f, vw, w2, act);
      }
    }
  }
  if (n_drop && dropped) atomicAdd(n_drop, dropped);
}

// Fold grouped float32 chunk images into float64 (num, den), fixed order:
// cell (r, c) = sum_z g_z(r, c).lo + g_z(r-1, c).hi.
__global__ void k_group_fold(const float4* __restrict__ img, int n_img, int64_t os, int64_t of,
                             double* __restrict__ num, double* __restrict__ den) {
  const int64_t n = os * of;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0, b = 0.0;
    const bool up = q >= of;
    for (int z = 0; z < n_img; ++z) {
      const float4 g = __ldg(img + (int64_t)z * n + q);
      a += g.x;
      b += g.y;
      if (up) {
        const float4 h = __ldg(img + (int64_t)z * n + q - of);
        a += h.z;
        b += h.w;
      }
    }
    num[q] += a;
    den[q] += b;
  }
}

// Normalise (interp.py:126-135): i_ref = num/den where den > 0 else 0.
__global__ void k_object_finish(const double* __restrict__ num, const double* __restrict__ den,
                                int64_t n, double* i_ref, double* wsum, float* fm,
                                uint8_t* valid) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double vv = num[q];
    const double ww = den[q];
    const bool ok = ww > 0.0;
    const double out = ok ? vv / ww : 0.0;
    if (i_ref) i_ref[q] = out;
    if (wsum) wsum[q] = ww;
    if (fm) fm[q] = static_cast<float>(out);
    if (valid) valid[q] = ok ? 1 : 0;
  }
}

__global__ void k_gather(pxst_ref ref, const double* __restrict__ x, const double* __restrict__ y,
                         int64_t n, double* vals, uint8_t* ok) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double xx = x[q], yy = y[q];
    float v = 0.f;
    bool good = false;
    if (isfinite(xx) && isfinite(yy) && fabs(xx) < 2e9 && fabs(yy) < 2e9) {
      const Split sx = split(xx), sy = split(yy);
      good = masked_read(ref.fm, ref.valid, ref.os, ref.of, sx.i, sy.i, sx.f, sy.f, v);
    }
    vals[q] = good ? static_cast<double>(v) : 0.0;
    ok[q] = good ? 1 : 0;
  }
}

__global__ void k_splat_f64(double* acc_v, double* acc_w, int64_t os, int64_t of,
                            const double* __restrict__ x, const double* __restrict__ y,
                            const double* __restrict__ value, const double* __restrict__ weight,
                            int64_t n, unsigned long long* n_drop) {
  unsigned long long dropped = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double xx = x[q], yy = y[q];
    if (!(xx >= 0.0 && xx <= static_cast<double>(os - 1) && yy >= 0.0 &&
          yy <= static_cast<double>(of - 1))) {
      ++dropped;
      continue;
    }
    const Split sx = split(xx), sy = split(yy);
    const double wt = weight ? weight[q] : 1.0;
    const double vw = value[q] * wt;
    const int r0 = sx.i, c0 = sy.i;
    const int r1 = min(r0 + 1, static_cast<int>(os - 1));
    const int c1 = min(c0 + 1, static_cast<int>(of - 1));
    const double gx = 1.0 - sx.f, gy = 1.0 - sy.f;
    const double cw[4] = {gx * gy, gx * sy.f, sx.f * gy, sx.f * sy.f};
    const int64_t cell[4] = {(int64_t)r0 * of + c0, (int64_t)r0 * of + c1,
                             (int64_t)r1 * of + c0, (int64_t)r1 * of + c1};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      atomicAdd(acc_v + cell[k], vw * cw[k]);
      atomicAdd(acc_w + cell[k], wt * cw[k]);
    }
  }
  if (dropped) atomicAdd(n_drop, dropped);
}

}  // namespace

int check_scan(const pxst_scan* sc);

int64_t chunk_images(int64_t blocks, int64_t frames_per_block, int64_t n_cells, int* n_img) {
  // An image sums >= kMinImageFrames frames (fewer images: less zeroing and
  // folding traffic) and, for long stacks, <= blocks / kMaxImages blocks;
  // the scratch stays <= kImageBytes.
  int64_t cap = kImageBytes / (static_cast<int64_t>(sizeof(float4)) * (n_cells > 0 ? n_cells : 1));
  if (cap > kMaxImages) cap = kMaxImages;
  if (cap < 1) cap = 1;
  int64_t bpi = (blocks + cap - 1) / cap;
  const int64_t min_bpi = (kMinImageFrames + frames_per_block - 1) / frames_per_block;
  if (bpi < min_bpi) bpi = min_bpi;
  *n_img = static_cast<int>((blocks + bpi - 1) / bpi);
  return bpi;
}

int fold_groups(const float4* img, int n_img, int64_t os, int64_t of, double* num, double* den,
                cudaStream_t s) {
  k_group_fold<<<grid_1d(os * of, 256), 256, 0, s>>>(img, n_img, os, of, num, den);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

int launch_object_splat(const pxst_scan* sc, const double* u, const double* di,
                        const double* dj, int64_t n0, int64_t m0, int64_t os, int64_t of,
                        int64_t frame_lo, int64_t frame_hi, double* num, double* den,
                        unsigned long long* n_drop, cudaStream_t s) {
  const int64_t nk = frame_hi - frame_lo;
  if (nk <= 0) return PXST_OK;
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  dim3 g((unsigned)((cw + kTC - 1) / kTC), (unsigned)((rw + kTR - 1) / kTR));
  PXST_REQUIRE(g.y <= kMaxGridY, "ROI too tall");
  // Frame slices (grid.z) so the launch holds ~3 waves of resident CTAs.
  int dev = 0, sms = 148, per_sm = 1;
  PXST_CHECK_CUDA(cudaGetDevice(&dev));
  PXST_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PXST_CHECK_CUDA(
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_object_splat, kThreads, 0));
  const int64_t resident = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t n_batches = (nk + kFB - 1) / kFB;
  int64_t n_z = (3 * resident + (int64_t)g.x * g.y - 1) / ((int64_t)g.x * g.y);
  n_z = n_z < 1 ? 1 : (n_z > n_batches ? n_batches : n_z);
  const int64_t fpz = ((n_batches + n_z - 1) / n_z) * kFB;
  g.z = static_cast<unsigned>((nk + fpz - 1) / fpz);
  const int64_t n = os * of;
  int n_img;
  const int64_t bpi = chunk_images(n_batches, kFB, n, &n_img);
  Scratch acc;
  if (int e = acc.alloc(sizeof(float4) * n * n_img, s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(float4) * n * n_img, s));
  k_object_splat<<<g, kThreads, 0, s>>>(*sc, u, di, dj, n0, m0, os, of, frame_lo, frame_hi, fpz,
                                        acc.as<float4>(), (int)bpi, n_drop);
  PXST_CHECK_LAUNCH();
  return fold_groups(acc.as<float4>(), n_img, os, of, num, den, s);
}

int launch_object_finish(const double* num, const double* den, int64_t n, double* i_ref,
                         double* wsum, float* fm, uint8_t* valid, cudaStream_t s) {
  k_object_finish<<<grid_1d(n, 256), 256, 0, s>>>(num, den, n, i_ref, wsum, fm, valid);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

}  // namespace pxst

using namespace pxst;

extern "C" int pxst_object_splat(const pxst_scan* sc, const double* u, const double* di,
                                 const double* dj, int64_t n0, int64_t m0, int64_t os,
                                 int64_t of, int64_t frame_lo, int64_t frame_hi, double* num,
                                 double* den, unsigned long long* n_dropped, void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(u && di && dj && num && den, "NULL pointer");
  PXST_REQUIRE(os > 0 && of > 0 && os * of < (int64_t(1) << 40), "bad grid shape");
  PXST_REQUIRE(0 <= frame_lo && frame_lo <= frame_hi && frame_hi <= sc->n_good,
               "bad frame range");
  return launch_object_splat(sc, u, di, dj, n0, m0, os, of, frame_lo, frame_hi, num, den,
                             n_dropped, as_stream(stream));
}

extern "C" int pxst_object_finish(const double* num, const double* den, int64_t n,
                                  double* i_ref, double* wsum, float* fm, uint8_t* valid,
                                  void* stream) {
  PXST_REQUIRE(num && den && n > 0, "bad accumulators");
  return launch_object_finish(num, den, n, i_ref, wsum, fm, valid, as_stream(stream));
}

extern "C" int pxst_object_map(const pxst_scan* sc, const double* u,
                               const double* di, const double* dj, int64_t n0, int64_t m0,
                               int64_t os, int64_t of, double* i_ref, double* wsum, float* fm,
                               uint8_t* valid, void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(os > 0 && of > 0 && os * of < (int64_t(1) << 40), "bad grid shape");
  cudaStream_t s = as_stream(stream);
  const int64_t n = os * of;
  Scratch acc;
  if (int e = acc.alloc(sizeof(double) * 2 * n, s)) return e;
  double* num = acc.as<double>();
  PXST_CHECK_CUDA(cudaMemsetAsync(num, 0, sizeof(double) * 2 * n, s));
  if (int e = launch_object_splat(sc, u, di, dj, n0, m0, os, of, 0, sc->n_good, num, num + n,
                                  nullptr, s))
    return e;
  return launch_object_finish(num, num + n, n, i_ref, wsum, fm, valid, s);
}

extern "C" int pxst_gather(const pxst_ref* ref, const double* x, const double* y, int64_t n,
                           double* vals, uint8_t* ok, void* stream) {
  PXST_REQUIRE(ref && ref->fm && ref->valid && ref->os > 0 && ref->of > 0, "bad reference");
  PXST_REQUIRE(x && y && vals && ok, "NULL pointer");
  if (n <= 0) return PXST_OK;
  k_gather<<<grid_1d(n, 256), 256, 0, as_stream(stream)>>>(*ref, x, y, n, vals, ok);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_splat(double* acc_v, double* acc_w, int64_t os, int64_t of, const double* x,
                          const double* y, const double* value, const double* weight, int64_t n,
                          int64_t* n_dropped, void* stream) {
  PXST_REQUIRE(acc_v && acc_w && os > 0 && of > 0, "bad accumulators");
  PXST_REQUIRE(x && y && value, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  Scratch cnt;
  if (int e = cnt.alloc(sizeof(unsigned long long), s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), s));
  if (n > 0) {
    k_splat_f64<<<grid_1d(n, 256), 256, 0, s>>>(acc_v, acc_w, os, of, x, y, value, weight, n,
                                                 cnt.as<unsigned long long>());
    PXST_CHECK_LAUNCH();
  }
  unsigned long long h = 0;
  PXST_CHECK_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  PXST_CHECK_CUDA(cudaStreamSynchronize(s));
  if (n_dropped) *n_dropped = static_cast<int64_t>(h);
  return PXST_OK;
}
