// K4 error maps (recon.py:388-438), one pass over the stack.
//
// eps = (valid ? (I - W v)^2 : (I - W)^2) / sigma2 per (frame, work pixel);
// per_pixel = sum over frames (float64, in-thread), per_frame = sum over
// pixels (deterministic: per-CTA partials, fixed-order final sum), total =
// sum of per_frame, reference_plane = normalise(splat(eps, weight 1)) where
// every sample is splatted, invalid ones included, out-of-grid
// points dropped (interp.py:103-107).  The splat goes through float32
// grouped chunk images and a float64 fold like K1 (splat.cu header).
#include "common.cuh"

namespace pxst {

int check_scan(const pxst_scan* sc);
int launch_object_finish(const double* num, const double* den, int64_t n, double* i_ref,
                         double* wsum, float* fm, uint8_t* valid, cudaStream_t s);

namespace {

constexpr int kTR = 8, kTC = 32, kThreads = kTR * kTC;
constexpr int kFB = 8;  // frames per reduction batch
constexpr int kLB = 2;  // frames per load batch (loads issued before the batch's REDs)

struct ErrArgs {
  pxst_scan sc;
  const double* u;
  const double* di;
  const double* dj;
  const float* fm;
  const uint8_t* valid;
  int64_t os, of, n0, m0;
  const double* fm64;  // nullable float64 image
  const double* sigma2;
  float4* img;   // grouped reference-plane images [n_img][os*of]
  int bpi;       // reduction batches (kFB frames) per image
};

// Per-pixel sums, per-(frame, CTA) partials, reference-plane splat.
__global__ void __launch_bounds__(kThreads, 2) k_err_pass(ErrArgs a, double* per_pixel,
                                                       double* part, int64_t n_ctas) {
  __shared__ double red[kThreads / 32][kFB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = a.sc.roi[0] + (int64_t)blockIdx.y * kTR + warp;
  const int64_t col = a.sc.roi[2] + (int64_t)blockIdx.x * kTC + lane;
  const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const bool inroi = row < a.sc.roi[1] && col < a.sc.roi[3];
  const int64_t p = inroi ? row * a.sc.fs + col : 0;
  const bool live = inroi && a.sc.work[p] != 0;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const double u0 = live ? a.u[p] : 0.0, u1 = live ? a.u[plane + p] : 0.0;
  const double W64 = live ? a.sc.w64[p] : 0.0;
  const double s2 = live ? a.sigma2[p] : 1.0;
  const double os1 = static_cast<double>(a.os - 1), of1 = static_cast<double>(a.of - 1);
  __shared__ double t_di[kFB], t_dj[kFB];
  __shared__ int64_t t_off[kFB];
  double pix = 0.0;
  for (int64_t k0 = 0; k0 < a.sc.n_good; k0 += kFB) {
    if (threadIdx.x < kFB && k0 + threadIdx.x < a.sc.n_good) {
      const int64_t f = a.sc.good[k0 + threadIdx.x];
      t_di[threadIdx.x] = a.di[f];
      t_dj[threadIdx.x] = a.dj[f];
      t_off[threadIdx.x] = f * plane;
    }
    __syncthreads();   // also orders the previous batch's red[] reads before reuse
    float4* img = a.img + (int64_t)((k0 / kFB) / a.bpi) * a.os * a.of;
    double e[kFB];
#pragma unroll
    for (int h = 0; h < kFB; h += kLB) {
    // Phase A: every load of the sub-batch is issued before any RED of it
    // (REDs pin the program order of later loads).
    float Iv[kLB];
    bool inb[kLB];
    double fxb[kLB], fyb[kLB];
    int64_t a00[kLB];
    int dc[kLB], dr[kLB];               // corner offsets (clipped at the grid edge)
    double v4[kLB][4];
    uint8_t m4[kLB][4];
#pragma unroll
    for (int b = 0; b < kLB; ++b) {
      const int64_t k = k0 + h + b;
      const bool act = live && k < a.sc.n_good;
      const double x = u0 - t_di[h + b] - static_cast<double>(a.n0);   // recon.py:418
      const double y = u1 - t_dj[h + b] - static_cast<double>(a.m0);
      inb[b] = act && x >= 0.0 && x <= os1 && y >= 0.0 && y <= of1;
      Iv[b] = act ? __ldg(a.sc.frames + t_off[h + b] + p) : 0.f;
      const Split sx = split(inb[b] ? x : 0.0), sy = split(inb[b] ? y : 0.0);
      fxb[b] = sx.f;
      fyb[b] = sy.f;
      dr[b] = sx.i + 1 < a.os ? static_cast<int>(a.of) : 0;
      dc[b] = sy.i + 1 < a.of ? 1 : 0;
      a00[b] = (int64_t)sx.i * a.of + sy.i;
      const int64_t ad[4] = {a00[b], a00[b] + dc[b], a00[b] + dr[b], a00[b] + dr[b] + dc[b]};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        m4[b][q] = inb[b] ? __ldg(a.valid + ad[q]) : 0;
        // fm / fm64 are 0 on invalid cells (where(m, f, 0), interp.py:64)
        v4[b][q] = !inb[b] ? 0.0 : (a.fm64 ? __ldg(a.fm64 + ad[q])
                                           : static_cast<double>(__ldg(a.fm + ad[q])));
      }
    }
    // Phase B: residuals, sums, reference-plane splat.
#pragma unroll
    for (int b = 0; b < kLB; ++b) {
      e[h + b] = 0.0;
      const int64_t k = k0 + h + b;
      if (!(live && k < a.sc.n_good)) continue;
      const double fx = fxb[b], fy = fyb[b], gx = 1.0 - fx, gy = 1.0 - fy;
      const double cw[4] = {gx * gy, gx * fy, fx * gy, fx * fy};
      bool ok = false;
      double v = 0.0;
      if (inb[b]) {                                   // interp.py:70-84
        const double den = cw[0] * m4[b][0] + cw[1] * m4[b][1] + cw[2] * m4[b][2] +
                           cw[3] * m4[b][3];
        const double nm = cw[0] * v4[b][0] + cw[1] * v4[b][1] + cw[2] * v4[b][2] +
                          cw[3] * v4[b][3];
        ok = den > 0.0;
        v = ok ? nm / den : 0.0;
      }
      const double I = static_cast<double>(Iv[b]);
      const double r = ok ? I - W64 * v : I - W64;  // recon.py:421
      const double eps = (r * r) / s2;                // recon.py:422
      e[h + b] = eps;
      pix += eps;
      if (inb[b])                                     // recon.py:425
        splat_grouped(img, a00[b], fx, fy, eps, 1.0);
    }
    }
#pragma unroll
    for (int b = 0; b < kFB; ++b) {
      const double v = warp_sum(e[b]);
      if (lane == 0) red[warp][b] = v;
    }
    __syncthreads();
    if (threadIdx.x < kFB && k0 + threadIdx.x < a.sc.n_good) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) s += red[w][threadIdx.x];
      part[(k0 + threadIdx.x) * n_ctas + cta] = s;
    }
  }
  if (live) per_pixel[p] = pix;
}

// per_frame[good[k]] = sum over CTAs in a fixed order (one block per frame).
__global__ void k_err_frames(pxst_scan sc, const double* __restrict__ part, int64_t n_ctas,
                             double* per_frame, double* frame_tmp) {
  __shared__ double sh[32];
  const int64_t k = blockIdx.x;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < n_ctas; c += blockDim.x) s += part[k * n_ctas + c];
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    per_frame[sc.good[k]] = t;
    frame_tmp[k] = t;
  }
}

// total = sum of per_frame over good frames (recon.py:433), fixed order.
__global__ void k_err_total(const double* __restrict__ frame_tmp, int64_t n, double* total) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) s += frame_tmp[k];
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    *total = t;
  }
}

}  // namespace
}  // namespace pxst

using namespace pxst;

namespace pxst {
namespace {

// One pass: per_frame (zeroed, then good frames filled), per_pixel (zeroed,
// then this scan's ROI filled), reference-plane accumulators added into
// num/den (caller-initialised), optional total.
int error_pass(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref, const double* u,
               const double* di, const double* dj, double* per_frame, double* per_pixel,
               double* num, double* den, double* total, cudaStream_t s) {
  const int64_t plane = sc->ss * sc->fs;
  PXST_CHECK_CUDA(cudaMemsetAsync(per_frame, 0, sizeof(double) * sc->n_frames, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(per_pixel, 0, sizeof(double) * plane, s));
  if (total) PXST_CHECK_CUDA(cudaMemsetAsync(total, 0, sizeof(double), s));
  if (sc->n_good == 0) return PXST_OK;
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  dim3 g((unsigned)((cw + kTC - 1) / kTC), (unsigned)((rw + kTR - 1) / kTR));
  PXST_REQUIRE(g.y <= kMaxGridY, "ROI too tall");
  const int64_t n_ctas = (int64_t)g.x * g.y;
  Scratch part;
  if (int e = part.alloc(sizeof(double) * (n_ctas + 1) * sc->n_good, s)) return e;
  const int64_t n_o = ref->os * ref->of;
  int n_img;
  const int64_t bpi = chunk_images((sc->n_good + kFB - 1) / kFB, n_o, &n_img);
  Scratch img;
  if (int e = img.alloc(sizeof(float4) * n_o * n_img, s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(img.p, 0, sizeof(float4) * n_o * n_img, s));
  double* ftmp = part.as<double>() + n_ctas * sc->n_good;
  ErrArgs a{*sc,        u,          di,          dj,      ref->fm,
            ref->valid, ref->os,    ref->of,     ref->n0, ref->m0,
            ref->fm64,  st->sigma2, img.as<float4>(), (int)bpi};
  k_err_pass<<<g, kThreads, 0, s>>>(a, per_pixel, part.as<double>(), n_ctas);
  PXST_CHECK_LAUNCH();
  k_err_frames<<<(unsigned)sc->n_good, 256, 0, s>>>(*sc, part.as<double>(), n_ctas, per_frame,
                                                    ftmp);
  PXST_CHECK_LAUNCH();
  if (total) {
    k_err_total<<<1, 1024, 0, s>>>(ftmp, sc->n_good, total);
    PXST_CHECK_LAUNCH();
  }
  return fold_groups(img.as<float4>(), n_img, ref->os, ref->of, num, den, s);
}

int check_err_args(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(ref && ref->fm && ref->valid && ref->os > 0 && ref->of > 0, "bad reference");
  PXST_REQUIRE(st && st->sigma2, "stats descriptor is NULL");
  return PXST_OK;
}

}  // namespace
}  // namespace pxst

extern "C" int pxst_error_maps(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref,
                               const double* u, const double* di, const double* dj,
                               double* per_frame, double* per_pixel, double* ref_plane,
                               double* total, void* stream) {
  if (int e = check_err_args(sc, st, ref)) return e;
  PXST_REQUIRE(u && di && dj && per_frame && per_pixel && ref_plane && total, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t n_o = ref->os * ref->of;
  Scratch acc;
  if (int e = acc.alloc(sizeof(double) * 2 * n_o, s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double) * 2 * n_o, s));
  if (int e = error_pass(sc, st, ref, u, di, dj, per_frame, per_pixel, acc.as<double>(),
                         acc.as<double>() + n_o, total, s))
    return e;
  return launch_object_finish(acc.as<double>(), acc.as<double>() + n_o, n_o, ref_plane, nullptr,
                              nullptr, nullptr, s);
}

extern "C" int pxst_error_partials(const pxst_scan* sc, const pxst_stats* st,
                                   const pxst_ref* ref, const double* u, const double* di,
                                   const double* dj, double* per_frame, double* per_pixel,
                                   double* plane_num, double* plane_den, void* stream) {
  if (int e = check_err_args(sc, st, ref)) return e;
  PXST_REQUIRE(u && di && dj && per_frame && per_pixel && plane_num && plane_den,
               "NULL pointer");
  return error_pass(sc, st, ref, u, di, dj, per_frame, per_pixel, plane_num, plane_den, nullptr,
                    as_stream(stream));
}
