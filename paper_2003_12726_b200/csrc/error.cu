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

constexpr int kTR = 4, kTC = 32, kThreads = kTR * kTC, kWarps = kThreads / 32;
constexpr int kFB = 8;    // frames per reduction batch
constexpr int kLB = 2;    // frames per load batch (loads issued before the batch's REDs)
constexpr int kTab = 256; // frames per shared-memory frame table chunk
#ifndef PXST_K4_OCC
#define PXST_K4_OCC 6   // resident CTAs per SM (80 registers; 4 measured slower)
#endif

struct ErrArgs {
  pxst_scan sc;
  const double* u;
  const double* di;
  const double* dj;
  const double2* grp;  // grouped reference (k_group_ref), NaN = invalid cell
  int64_t os, of, n0, m0;
  const double* sigma2;
  float4* img;         // grouped reference-plane images [n_img][os*of]
  int bpi;             // reduction batches (kFB frames) per image
  int64_t frames_per_z;
  // fused next-object splat (pxst_error_maps_splat): K1 of the next
  // iteration reads the same samples at the same positions u - delta,
  // relative to its own grid, read from device memory (n0, m0, os, of)
  float4* img_b;       // grouped object images [n_img_b][cap_b], NULL = not fused
  int bpi_b;
  const int64_t* grid_b;
  int64_t cap_b;       // cells per image; a grid with os*of > cap_b is not splatted
};

// g[r][c] = (v(r, c), v(r+1, c)) with v = the float64 masked reference where
// valid and NaN elsewhere (and past the last row): one 16-byte load fetches a
// bilinear column pair, and the NaN doubles as the validity bit.
__global__ void k_group_ref(const double* __restrict__ fm64, const float* __restrict__ fm,
                            const uint8_t* __restrict__ valid, int64_t os, int64_t of,
                            double2* __restrict__ g) {
  const int64_t n = os * of;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    auto v = [&](int64_t i) {
      return valid[i] ? (fm64 ? fm64[i] : static_cast<double>(fm[i])) : nan;
    };
    g[q] = make_double2(v(q), q + of < n ? v(q + of) : nan);
  }
}

// Fixed-order butterfly all-reduce of 8 values over a warp: afterwards lane l
// holds the warp sum of value index ((l>>4)&1)*4 + ((l>>3)&1)*2 + ((l>>2)&1)
// (9 float64 shuffles instead of 40).
__device__ __forceinline__ double warp_sum8(double (&v)[8], int lane) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool hi = lane & 16;
    const double send = hi ? v[j] : v[j + 4], keep = hi ? v[j + 4] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool hi = lane & 8;
    const double send = hi ? v[j] : v[j + 2], keep = hi ? v[j + 2] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool hi = lane & 4;
    const double send = hi ? v[0] : v[1], keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

// One thread per work pixel over the frame slice blockIdx.z: per-pixel slice
// sums, per-(frame, warp) partials, reference-plane splat.  No barrier inside
// the frame loop (the frame table is refreshed every kTab frames).
template <bool FUSE>
__global__ void __launch_bounds__(kThreads, PXST_K4_OCC) k_err_pass(ErrArgs a, double* pix_part,
                                                       double* part, int64_t n_warps) {
  __shared__ double t_di[kTab], t_dj[kTab];
  __shared__ int64_t t_off[kTab];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = a.sc.roi[0] + (int64_t)blockIdx.y * kTR + warp;
  const int64_t col = a.sc.roi[2] + (int64_t)blockIdx.x * kTC + lane;
  const int64_t gwarp = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kWarps + warp;
  const bool inroi = row < a.sc.roi[1] && col < a.sc.roi[3];
  const int64_t p = inroi ? row * a.sc.fs + col : 0;
  const bool live = inroi && a.sc.work[p] != 0;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const double u0 = live ? a.u[p] : 0.0, u1 = live ? a.u[plane + p] : 0.0;
  const double W64 = live ? a.sc.w64[p] : 0.0;
  const double s2 = live ? a.sigma2[p] : 1.0;
  const double W2 = W64 * W64;                               // recon.py:136
  const double inv_s2 = live ? 1.0 / s2 : 0.0;               // one division per pixel
  const double inv_W = live ? 1.0 / W64 : 0.0;
  int64_t n0b = 0, m0b = 0, osb = 1, ofb = 1;
  if (FUSE) {
    n0b = a.grid_b[0];
    m0b = a.grid_b[1];
    osb = a.grid_b[2];
    ofb = a.grid_b[3];
  }
  const bool splat_b = FUSE && osb > 0 && ofb > 0 && osb * ofb <= a.cap_b;
  const double osb1 = static_cast<double>(osb - 1), ofb1 = static_cast<double>(ofb - 1);
  const double os1 = static_cast<double>(a.os - 1), of1 = static_cast<double>(a.of - 1);
  const int64_t n_o = a.os * a.of;
  const int64_t k_begin = (int64_t)blockIdx.z * a.frames_per_z;
  const int64_t k_end = min(a.sc.n_good, k_begin + a.frames_per_z);
  double pix = 0.0;
  for (int64_t kc = k_begin; kc < k_end; kc += kTab) {
    const int nt = static_cast<int>(k_end - kc < kTab ? k_end - kc : kTab);
    __syncthreads();
    for (int t = threadIdx.x; t < nt; t += kThreads) {
      const int64_t f = a.sc.good[kc + t];
      t_di[t] = a.di[f];
      t_dj[t] = a.dj[f];
      t_off[t] = f * plane;
    }
    __syncthreads();
    for (int b0 = 0; b0 < nt; b0 += kFB) {
      float4* img = a.img + ((kc + b0) / kFB / a.bpi) * n_o;
      float4* img_b = FUSE ? a.img_b + ((kc + b0) / kFB / a.bpi_b) * a.cap_b : nullptr;
      double e[kFB];
#pragma unroll
      for (int h = 0; h < kFB; h += kLB) {
        // Phase A: every load of the sub-batch is issued before any RED of it.
        float Iv[kLB];
        bool inb[kLB];
        double fxb[kLB], fyb[kLB];
        int64_t a00[kLB];
        double2 g0[kLB], g1[kLB];
#pragma unroll
        for (int b = 0; b < kLB; ++b) {
          const int t = b0 + h + b;
          const bool act = live && t < nt;
          const double x = u0 - t_di[t] - static_cast<double>(a.n0);   // recon.py:418
          const double y = u1 - t_dj[t] - static_cast<double>(a.m0);
          inb[b] = act && x >= 0.0 && x <= os1 && y >= 0.0 && y <= of1;
          Iv[b] = act ? __ldg(a.sc.frames + t_off[t] + p) : 0.f;
          const Split sx = split(inb[b] ? x : 0.0), sy = split(inb[b] ? y : 0.0);
          fxb[b] = sx.f;
          fyb[b] = sy.f;
          a00[b] = (int64_t)sx.i * a.of + sy.i;
          const double2 z2 = make_double2(0.0, 0.0);
          g0[b] = inb[b] ? __ldg(a.grp + a00[b]) : z2;
          // fy == 0 <=> the reference's clipped column (interp.py:44-45), weight 0
          g1[b] = inb[b] && sy.f > 0.0 ? __ldg(a.grp + a00[b] + 1) : z2;
        }
        // Phase B: residuals, sums, reference-plane splat.
#pragma unroll
        for (int b = 0; b < kLB; ++b) {
          const double fx = fxb[b], fy = fyb[b], gx = 1.0 - fx, gy = 1.0 - fy;
          const double cw[4] = {gx * gy, gx * fy, fx * gy, fx * fy};
          // corners 00, 01, 10, 11 (interp.py:70-84 order)
          const double cv[4] = {g0[b].x, g1[b].x, g0[b].y, g1[b].y};
          double den = 0.0, nm = 0.0;
          bool all = true;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool m = cv[q] == cv[q];           // NaN = invalid cell
            all = all && m;
            den = fma(cw[q], m ? 1.0 : 0.0, den);    // cw * {0, 1} is exact: = den + cw m
            nm = fma(cw[q], m ? cv[q] : 0.0, nm);
          }
          const bool ok = inb[b] && den > 0.0;
          // all four corners valid: den = 1 to a few ulp, and 1/den = 2 - den to
          // ~1e-31 -- no division on the common path
          const double v = !ok ? 0.0 : (all ? nm * (2.0 - den) : nm / den);
          const double I = static_cast<double>(Iv[b]);
          const double r = ok ? I - W64 * v : I - W64;  // recon.py:421
          const double eps = (live && b0 + h + b < nt) ? (r * r) * inv_s2 : 0.0;   // recon.py:422
          e[h + b] = eps;
          pix += eps;
          if (inb[b])                                   // recon.py:425
            splat_grouped(img, a00[b], fx, fy, eps, 1.0);
          if (FUSE) {                                   // next K1 (recon.py:135-138)
            const int t = b0 + h + b < nt ? b0 + h + b : 0;
            const double xb = u0 - t_di[t] - static_cast<double>(n0b);
            const double yb = u1 - t_dj[t] - static_cast<double>(m0b);
            const bool in_b = splat_b && live && b0 + h + b < nt && xb >= 0.0 && xb <= osb1 &&
                              yb >= 0.0 && yb <= ofb1;   // interp.py:103-107
            const Split sx = split(in_b ? xb : 0.0), sy = split(in_b ? yb : 0.0);
            if (in_b)
              splat_grouped(img_b, (int64_t)sx.i * ofb + sy.i, sx.f, sy.f, (I * inv_W) * W2, W2);
          }
        }
      }
      const double sum = warp_sum8(e, lane);
      const int idx = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      if ((lane & 3) == 0 && b0 + idx < nt) part[(kc + b0 + idx) * n_warps + gwarp] = sum;
    }
  }
  if (live) pix_part[(int64_t)blockIdx.z * plane + p] = pix;
}

// per_pixel[p] = sum over frame slices (fixed order) on work pixels.
__global__ void k_err_pixels(pxst_scan sc, const double* __restrict__ pix_part, int n_z,
                             double* per_pixel) {
  const int64_t cw = sc.roi[3] - sc.roi[2], n = (sc.roi[1] - sc.roi[0]) * cw;
  const int64_t plane = sc.ss * sc.fs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = (sc.roi[0] + q / cw) * sc.fs + sc.roi[2] + q % cw;
    if (!sc.work[p]) continue;
    double t = 0.0;
    for (int z = 0; z < n_z; ++z) t += pix_part[z * plane + p];
    per_pixel[p] = t;
  }
}

// per_frame[good[k]] = sum over warps in a fixed order (one block per frame).
__global__ void k_err_frames(pxst_scan sc, const double* __restrict__ part, int64_t n_warps,
                             double* per_frame, double* frame_tmp) {
  __shared__ double sh[32];
  const int64_t k = blockIdx.x;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < n_warps; c += blockDim.x) s += part[k * n_warps + c];
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
// The next iteration's object grid for the fused splat (its num/den are
// added into, like pxst_object_splat).
struct NextObject {
  const int64_t* grid;   // device (n0, m0, os, of)
  int64_t capacity;      // cells of num / den and of each image
  double* num;
  double* den;
};

// Grid rule of recon.py:126-132 on device: grid = (n0, m0, os, of) from the
// bbox values of pxst_bbox.
__global__ void k_grid_rule(const double* __restrict__ b, int64_t* __restrict__ grid) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t n0 = static_cast<int64_t>(floor(b[0] - b[5]));
    const int64_t m0 = static_cast<int64_t>(floor(b[2] - b[7]));
    grid[0] = n0;
    grid[1] = m0;
    grid[2] = static_cast<int64_t>(floor(b[1] - b[4])) - n0 + 2;
    grid[3] = static_cast<int64_t>(floor(b[3] - b[6])) - m0 + 2;
  }
}

// Fold of grouped images whose grid lives in device memory (image stride cap).
__global__ void k_group_fold_dev(const float4* __restrict__ img, int n_img, int64_t cap,
                                 const int64_t* __restrict__ grid, double* __restrict__ num,
                                 double* __restrict__ den) {
  const int64_t os = grid[2], of = grid[3], n = os * of;
  if (!(os > 0 && of > 0 && n <= cap)) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    double x = 0.0, y = 0.0;
    const bool up = q >= of;
    for (int z = 0; z < n_img; ++z) {
      const float4 g = __ldg(img + (int64_t)z * cap + q);
      x += g.x;
      y += g.y;
      if (up) {
        const float4 h = __ldg(img + (int64_t)z * cap + q - of);
        x += h.z;
        y += h.w;
      }
    }
    num[q] += x;
    den[q] += y;
  }
}

int error_pass(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref, const double* u,
               const double* di, const double* dj, double* per_frame, double* per_pixel,
               double* num, double* den, double* total, const NextObject* nx, cudaStream_t s) {
  const int64_t plane = sc->ss * sc->fs;
  PXST_CHECK_CUDA(cudaMemsetAsync(per_frame, 0, sizeof(double) * sc->n_frames, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(per_pixel, 0, sizeof(double) * plane, s));
  if (total) PXST_CHECK_CUDA(cudaMemsetAsync(total, 0, sizeof(double), s));
  if (sc->n_good == 0) return PXST_OK;
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  dim3 g((unsigned)((cw + kTC - 1) / kTC), (unsigned)((rw + kTR - 1) / kTR));
  PXST_REQUIRE(g.y <= kMaxGridY, "ROI too tall");
  const int64_t n_warps = (int64_t)g.x * g.y * kWarps;
  // Frame slices (grid.z): enough threads for ~3 waves of resident CTAs when
  // the ROI alone cannot fill the GPU (config 1: 131k pixels).
  int dev = 0, sms = 148, per_sm = 1;
  PXST_CHECK_CUDA(cudaGetDevice(&dev));
  PXST_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PXST_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, nx ? k_err_pass<true> : k_err_pass<false>, kThreads, 0));
  const int64_t resident = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t n_batches = (sc->n_good + kFB - 1) / kFB;
  int64_t n_z = (3 * resident + (int64_t)g.x * g.y - 1) / ((int64_t)g.x * g.y);
  n_z = n_z < 1 ? 1 : (n_z > n_batches ? n_batches : n_z);
  const int64_t fpz = ((n_batches + n_z - 1) / n_z) * kFB;
  n_z = (sc->n_good + fpz - 1) / fpz;
  g.z = static_cast<unsigned>(n_z);
  Scratch part;
  if (int e = part.alloc(sizeof(double) * ((n_warps + 1) * sc->n_good + n_z * plane), s)) return e;
  double* ftmp = part.as<double>() + n_warps * sc->n_good;
  double* pix_part = ftmp + sc->n_good;
  const int64_t n_o = ref->os * ref->of;
  int n_img;
  const int64_t bpi = chunk_images(n_batches, kFB, n_o, &n_img);
  Scratch img, grp;
  if (int e = img.alloc(sizeof(float4) * n_o * n_img, s)) return e;
  if (int e = grp.alloc(sizeof(double2) * n_o, s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(img.p, 0, sizeof(float4) * n_o * n_img, s));
  k_group_ref<<<grid_1d(n_o, 256), 256, 0, s>>>(ref->fm64, ref->fm, ref->valid, ref->os, ref->of,
                                                grp.as<double2>());
  PXST_CHECK_LAUNCH();
  ErrArgs a{};
  a.sc = *sc;
  a.u = u;
  a.di = di;
  a.dj = dj;
  a.grp = grp.as<double2>();
  a.os = ref->os;
  a.of = ref->of;
  a.n0 = ref->n0;
  a.m0 = ref->m0;
  a.sigma2 = st->sigma2;
  a.img = img.as<float4>();
  a.bpi = static_cast<int>(bpi);
  a.frames_per_z = fpz;
  Scratch img_b;
  int n_img_b = 0;
  if (nx) {
    const int64_t n_b = nx->capacity;
    a.bpi_b = static_cast<int>(chunk_images(n_batches, kFB, n_b, &n_img_b));
    if (int e = img_b.alloc(sizeof(float4) * n_b * n_img_b, s)) return e;
    PXST_CHECK_CUDA(cudaMemsetAsync(img_b.p, 0, sizeof(float4) * n_b * n_img_b, s));
    a.img_b = img_b.as<float4>();
    a.grid_b = nx->grid;
    a.cap_b = n_b;
    k_err_pass<true><<<g, kThreads, 0, s>>>(a, pix_part, part.as<double>(), n_warps);
  } else {
    k_err_pass<false><<<g, kThreads, 0, s>>>(a, pix_part, part.as<double>(), n_warps);
  }
  PXST_CHECK_LAUNCH();
  if (nx) {
    k_group_fold_dev<<<grid_1d(nx->capacity, 256), 256, 0, s>>>(
        img_b.as<float4>(), n_img_b, nx->capacity, nx->grid, nx->num, nx->den);
    PXST_CHECK_LAUNCH();
  }
  k_err_pixels<<<grid_1d(rw * cw, 256), 256, 0, s>>>(*sc, pix_part, (int)n_z, per_pixel);
  PXST_CHECK_LAUNCH();
  k_err_frames<<<(unsigned)sc->n_good, 256, 0, s>>>(*sc, part.as<double>(), n_warps, per_frame,
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
                         acc.as<double>() + n_o, total, nullptr, s))
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
                    nullptr, as_stream(stream));
}

extern "C" int pxst_grid_rule(const double* bbox, int64_t* grid, void* stream) {
  PXST_REQUIRE(bbox && grid, "NULL pointer");
  k_grid_rule<<<1, 32, 0, as_stream(stream)>>>(bbox, grid);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_error_maps_splat(const pxst_scan* sc, const pxst_stats* st,
                                     const pxst_ref* ref, const double* u, const double* di,
                                     const double* dj, double* per_frame, double* per_pixel,
                                     double* ref_plane, double* total, const int64_t* grid,
                                     int64_t capacity, double* num, double* den, void* stream) {
  if (int e = check_err_args(sc, st, ref)) return e;
  PXST_REQUIRE(u && di && dj && per_frame && per_pixel && ref_plane && total && grid && num &&
                   den,
               "NULL pointer");
  PXST_REQUIRE(capacity > 0 && capacity < (int64_t(1) << 40), "bad capacity");
  cudaStream_t s = as_stream(stream);
  const int64_t n_o = ref->os * ref->of;
  Scratch acc;
  if (int e = acc.alloc(sizeof(double) * 2 * n_o, s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double) * 2 * n_o, s));
  const NextObject nx{grid, capacity, num, den};
  if (int e = error_pass(sc, st, ref, u, di, dj, per_frame, per_pixel, acc.as<double>(),
                         acc.as<double>() + n_o, total, &nx, s))
    return e;
  return launch_object_finish(acc.as<double>(), acc.as<double>() + n_o, n_o, ref_plane, nullptr,
                              nullptr, nullptr, s);
}
