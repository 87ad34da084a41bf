// K4 error maps (recon.py:388-438), one pass over the stack.
//
// eps = (valid ? (I - W v)^2 : (I - W)^2) / sigma2 per (frame, work pixel);
// per_pixel = sum over frames (float64, in-thread over a frame slice, slices
// added in a fixed order), per_frame = sum over pixels (per-CTA partials,
// fixed-order final sum), total = sum of per_frame, reference_plane =
// normalise(splat(eps, weight 1)) where every sample is splatted, invalid ones
// included, out-of-grid points dropped (interp.py:103-107).  The
// pass is mode 1 / 2 of fixsplat.cu: the plane is accumulated in exact int64
// fixed point (bit-reproducible, independent of the work split), and mode 2
// also forms the next iteration's object from the same samples.
#include "fixsplat.cuh"

namespace pxst {

int check_scan(const pxst_scan* sc);
struct FixArgs;
int launch_abs_max(const pxst_scan* sc, double* out, cudaStream_t s);
int launch_quanta(const pxst_scan* sc, const double* absmax, const double* sigma2,
                  const pxst_ref* ref, int kind, double* quanta, cudaStream_t s);
int launch_fix_finish(const FixAcc& acc, const int64_t* grid, int64_t n, double* out, double* wsum,
                      float* fm, uint8_t* valid, cudaStream_t s);
int launch_error_fix(const pxst_scan* sc, const pxst_ref* ref, const double* u, const double* di,
                     const double* dj, const double* sigma2, const double2* grp, const FixAcc& plane,
                     const FixAcc* next, const int64_t* grid_b, int64_t cap_b, double* pix_part,
                     double* part, int* n_z, int64_t* n_cta, cudaStream_t s);
int fix_pass_slices(const pxst_scan* sc, int64_t nk, int mode, int64_t* n_cta);

namespace {

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

// per_frame[good[k]] = sum over CTAs in a fixed order (one block per frame).
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

// One pass: per_frame (zeroed, then good frames filled), per_pixel (zeroed,
// then this scan's ROI filled), reference-plane int64 terms added into
// `plane` (caller-initialised), optional total; with `next`, the next
// iteration's object terms added into it (grid read from the device).
int error_pass(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref, const double* u,
               const double* di, const double* dj, double* per_frame, double* per_pixel,
               const FixAcc& plane, double* total, const FixAcc* next, const int64_t* grid_b,
               int64_t cap_b, cudaStream_t s) {
  const int64_t plane_px = sc->ss * sc->fs;
  PXST_CHECK_CUDA(cudaMemsetAsync(per_frame, 0, sizeof(double) * sc->n_frames, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(per_pixel, 0, sizeof(double) * plane_px, s));
  if (total) PXST_CHECK_CUDA(cudaMemsetAsync(total, 0, sizeof(double), s));
  if (sc->n_good == 0) return PXST_OK;
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  int64_t n_cta = 0;
  const int n_z = fix_pass_slices(sc, sc->n_good, next ? 2 : 1, &n_cta);
  const int64_t n_o = ref->os * ref->of;
  Scratch part, grp;
  if (int e = part.alloc(sizeof(double) * ((n_cta + 1) * sc->n_good + (int64_t)n_z * plane_px), s))
    return e;
  double* ftmp = part.as<double>() + n_cta * sc->n_good;
  double* pix_part = ftmp + sc->n_good;
  if (int e = grp.alloc(sizeof(double2) * n_o, s)) return e;
  k_group_ref<<<grid_1d(n_o, 256), 256, 0, s>>>(ref->fm64, ref->fm, ref->valid, ref->os, ref->of,
                                                grp.as<double2>());
  PXST_CHECK_LAUNCH();
  int nz2 = 0;
  int64_t nc2 = 0;
  if (int e = launch_error_fix(sc, ref, u, di, dj, st->sigma2, grp.as<double2>(), plane, next,
                               grid_b, cap_b, pix_part, part.as<double>(), &nz2, &nc2, s))
    return e;
  PXST_REQUIRE(nz2 == n_z && nc2 == n_cta, "error pass layout mismatch");
  k_err_pixels<<<grid_1d(rw * cw, 256), 256, 0, s>>>(*sc, pix_part, n_z, per_pixel);
  PXST_CHECK_LAUNCH();
  k_err_frames<<<(unsigned)sc->n_good, 256, 0, s>>>(*sc, part.as<double>(), n_cta, per_frame,
                                                    ftmp);
  PXST_CHECK_LAUNCH();
  if (total) {
    k_err_total<<<1, 1024, 0, s>>>(ftmp, sc->n_good, total);
    PXST_CHECK_LAUNCH();
  }
  return PXST_OK;
}

int check_err_args(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(ref && ref->fm && ref->valid && ref->os > 0 && ref->of > 0, "bad reference");
  PXST_REQUIRE(ref->os * ref->of < (int64_t(1) << 31), "reference image too large");
  PXST_REQUIRE(st && st->sigma2, "stats descriptor is NULL");
  return PXST_OK;
}

FixAcc fix_acc(const pxst_accum* acc) {
  return FixAcc{reinterpret_cast<long long*>(acc->num), reinterpret_cast<long long*>(acc->den),
                reinterpret_cast<long long*>(acc->num_fine),
                reinterpret_cast<long long*>(acc->den_fine), acc->touched, acc->quanta};
}

// Plane accumulators + quanta in one scratch block, the error pass, the
// normalisation into ref_plane.
int error_maps_full(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref,
                    const double* u, const double* di, const double* dj, const double* absmax,
                    double* per_frame, double* per_pixel, double* ref_plane, double* total,
                    const FixAcc* next, const int64_t* grid_b, int64_t cap_b, cudaStream_t s) {
  const int64_t n_o = ref->os * ref->of;
  Scratch acc;
  if (int e = acc.alloc(sizeof(int64_t) * 4 * n_o + 4 * sizeof(double), s)) return e;
  int64_t* num = acc.as<int64_t>();
  double* q = reinterpret_cast<double*>(num + 4 * n_o);
  double* amax = q + 2;
  PXST_CHECK_CUDA(cudaMemsetAsync(num, 0, sizeof(int64_t) * 4 * n_o, s));
  if (!absmax) {
    if (int e = launch_abs_max(sc, amax, s)) return e;
    absmax = amax;
  }
  if (int e = launch_quanta(sc, absmax, st->sigma2, ref, 1, q, s)) return e;
  const FixAcc plane{reinterpret_cast<long long*>(num), reinterpret_cast<long long*>(num + n_o),
                     reinterpret_cast<long long*>(num + 2 * n_o),
                     reinterpret_cast<long long*>(num + 3 * n_o), nullptr, q};
  if (int e = error_pass(sc, st, ref, u, di, dj, per_frame, per_pixel, plane, total, next, grid_b,
                         cap_b, s))
    return e;
  return launch_fix_finish(plane, nullptr, n_o, ref_plane, nullptr, nullptr, nullptr, s);
}

}  // namespace
}  // namespace pxst

extern "C" int pxst_plane_quanta(const pxst_scan* sc, const double* absmax, const pxst_stats* st,
                                 const pxst_ref* ref, double* quanta, void* stream) {
  if (int e = check_err_args(sc, st, ref)) return e;
  PXST_REQUIRE(absmax && quanta, "NULL pointer");
  return launch_quanta(sc, absmax, st->sigma2, ref, 1, quanta, as_stream(stream));
}

extern "C" int pxst_error_maps(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref,
                               const double* u, const double* di, const double* dj,
                               const double* absmax, double* per_frame, double* per_pixel,
                               double* ref_plane, double* total, void* stream) {
  if (int e = check_err_args(sc, st, ref)) return e;
  PXST_REQUIRE(u && di && dj && per_frame && per_pixel && ref_plane && total, "NULL pointer");
  return error_maps_full(sc, st, ref, u, di, dj, absmax, per_frame, per_pixel, ref_plane, total,
                         nullptr, nullptr, 0, as_stream(stream));
}

extern "C" int pxst_error_partials(const pxst_scan* sc, const pxst_stats* st,
                                   const pxst_ref* ref, const double* u, const double* di,
                                   const double* dj, double* per_frame, double* per_pixel,
                                   const pxst_accum* plane, void* stream) {
  if (int e = check_err_args(sc, st, ref)) return e;
  PXST_REQUIRE(u && di && dj && per_frame && per_pixel && plane && plane->num && plane->den &&
                   plane->num_fine && plane->den_fine && plane->quanta,
               "NULL pointer");
  return error_pass(sc, st, ref, u, di, dj, per_frame, per_pixel, fix_acc(plane), nullptr,
                    nullptr, nullptr, 0, as_stream(stream));
}

extern "C" int pxst_grid_rule(const double* bbox, int64_t* grid, void* stream) {
  PXST_REQUIRE(bbox && grid, "NULL pointer");
  k_grid_rule<<<1, 32, 0, as_stream(stream)>>>(bbox, grid);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_error_maps_splat(const pxst_scan* sc, const pxst_stats* st,
                                     const pxst_ref* ref, const double* u, const double* di,
                                     const double* dj, const double* absmax, double* per_frame,
                                     double* per_pixel, double* ref_plane, double* total,
                                     const int64_t* grid, int64_t capacity,
                                     const pxst_accum* next, void* stream) {
  if (int e = check_err_args(sc, st, ref)) return e;
  PXST_REQUIRE(u && di && dj && per_frame && per_pixel && ref_plane && total && grid && next &&
                   next->num && next->den && next->num_fine && next->den_fine && next->quanta,
               "NULL pointer");
  PXST_REQUIRE(capacity > 0 && capacity < (int64_t(1) << 40), "bad capacity");
  const FixAcc nx = fix_acc(next);
  return error_maps_full(sc, st, ref, u, di, dj, absmax, per_frame, per_pixel, ref_plane, total,
                         &nx, grid, capacity, as_stream(stream));
}
