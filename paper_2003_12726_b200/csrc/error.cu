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
int launch_error_fix(const pxst_scan* sc, const pxst_ref* ref, const double* u, const double* di,
                     const double* dj, const double* sigma2, const double2* grp, const FixAcc& plane,
                     const FixAcc* next, const int64_t* grid_b, int64_t cap_b, double* pix_part,
                     double* part, int* n_z, int64_t* n_cta, cudaStream_t s);
int fix_pass_slices(const pxst_scan* sc, int64_t nk, int mode, int64_t* n_cta);

namespace {

// The pass's reductions in one launch (block roles; 256 threads):
//   [0, n_good)            per_frame[good[k]] = sum over the pass's CTAs in a
//                          fixed order; the last frame block to finish
//                          (ticket) adds total = sum of per_frame over good
//                          frames (recon.py:433), fixed order;
//   [n_good, +nb_plane)    the reference plane's normalisation (optional);
//   [.., +nb_pixel)        per_pixel[p] = sum over frame slices (fixed order)
//                          on work pixels, 0 elsewhere (the whole detector).
struct ErrEpi {
  pxst_scan sc;
  const double* pix_part;   // [n_z][ss * fs]
  int n_z;
  const double* part;       // [n_good][n_cta]
  int64_t n_cta;
  double* per_pixel;
  double* per_frame;
  double* ftmp;             // [n_good]
  double* total;            // nullable
  unsigned* ticket;         // zero at start
  FixAcc plane;
  double* ref_plane;        // nullable: no normalisation
  int64_t n_o, nb_plane;
};

__global__ void __launch_bounds__(256) k_err_epilogue(ErrEpi e) {
  __shared__ double sh[32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t b = blockIdx.x;
  if (b < e.sc.n_good) {
    double s = 0.0;
    for (int64_t c = threadIdx.x; c < e.n_cta; c += blockDim.x) s += e.part[b * e.n_cta + c];
    s = warp_sum(s);
    if (lane == 0) sh[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += sh[w];
      e.per_frame[e.sc.good[b]] = t;
      e.ftmp[b] = t;
      if (e.total) {
        __threadfence();
        s_last = atomicAdd(e.ticket, 1u) == static_cast<unsigned>(e.sc.n_good - 1);
      }
    }
    if (!e.total) return;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double s2 = 0.0;
    for (int64_t k = threadIdx.x; k < e.sc.n_good; k += blockDim.x) s2 += __ldcg(e.ftmp + k);
    s2 = warp_sum(s2);
    __syncthreads();
    if (lane == 0) sh[warp] = s2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += sh[w];
      *e.total = t;
    }
    return;
  }
  if (b < e.sc.n_good + e.nb_plane) {
    const int64_t i = (b - e.sc.n_good) * blockDim.x + threadIdx.x;
    if (i < e.n_o) fix_finish_cell(e.plane, i, e.ref_plane, nullptr, nullptr, nullptr);
    return;
  }
  const int64_t plane = e.sc.ss * e.sc.fs;
  const int64_t p = (b - e.sc.n_good - e.nb_plane) * blockDim.x + threadIdx.x;
  if (p >= plane) return;
  const int64_t r = p / e.sc.fs, c = p % e.sc.fs;
  double t = 0.0;
  if (r >= e.sc.roi[0] && r < e.sc.roi[1] && c >= e.sc.roi[2] && c < e.sc.roi[3] && e.sc.work[p])
    for (int z = 0; z < e.n_z; ++z) t += e.pix_part[z * plane + p];
  e.per_pixel[p] = t;
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

// One pass: per_frame (zeroed, then good frames filled), per_pixel (the
// ROI's work pixels filled, 0 elsewhere), reference-plane int64 terms added
// into `plane` (caller-initialised; with `absmax` its quanta are computed
// here first), optional total and normalised plane (ref_plane); with
// `next`, the next iteration's object terms added into it (grid read from
// the device).  ticket: two zeroed words.  Launches: prologue (quanta,
// grouped reference, per_frame zero), the fused pass, the epilogue.
int error_pass(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref, const double* u,
               const double* di, const double* dj, double* per_frame, double* per_pixel,
               const FixAcc& plane, const double* absmax, double* ref_plane, double* total,
               const FixAcc* next, const int64_t* grid_b, int64_t cap_b, unsigned* ticket,
               cudaStream_t s) {
  const int64_t plane_px = sc->ss * sc->fs;
  const int64_t n_o = ref->os * ref->of;
  if (sc->n_good == 0) {
    PXST_CHECK_CUDA(cudaMemsetAsync(per_frame, 0, sizeof(double) * sc->n_frames, s));
    PXST_CHECK_CUDA(cudaMemsetAsync(per_pixel, 0, sizeof(double) * plane_px, s));
    if (total) PXST_CHECK_CUDA(cudaMemsetAsync(total, 0, sizeof(double), s));
    if (ref_plane) PXST_CHECK_CUDA(cudaMemsetAsync(ref_plane, 0, sizeof(double) * n_o, s));
    return PXST_OK;
  }
  int64_t n_cta = 0;
  const int n_z = fix_pass_slices(sc, sc->n_good, next ? 2 : 1, &n_cta);
  Scratch part, grp;
  if (int e = part.alloc(sizeof(double) * ((n_cta + 1) * sc->n_good + (int64_t)n_z * plane_px), s))
    return e;
  double* ftmp = part.as<double>() + n_cta * sc->n_good;
  double* pix_part = ftmp + sc->n_good;
  if (int e = grp.alloc(sizeof(double2) * n_o, s)) return e;
  QuantaJob j{};
  j.sc = *sc;
  j.sigma2 = st->sigma2;
  j.fm64 = ref->fm64;
  j.fm = ref->fm;
  j.valid = ref->valid;
  j.os = ref->os;
  j.of = ref->of;
  j.absmax = absmax;
  j.kind = 1;
  j.quanta = absmax ? const_cast<double*>(plane.q) : nullptr;
  j.ticket = ticket;
  j.grp = grp.as<double2>();
  j.zero = per_frame;
  j.n_zero = sc->n_frames;
  if (int e = launch_quanta_job(j, s)) return e;
  int nz2 = 0;
  int64_t nc2 = 0;
  if (int e = launch_error_fix(sc, ref, u, di, dj, st->sigma2, grp.as<double2>(), plane, next,
                               grid_b, cap_b, pix_part, part.as<double>(), &nz2, &nc2, s))
    return e;
  PXST_REQUIRE(nz2 == n_z && nc2 == n_cta, "error pass layout mismatch");
  ErrEpi ep{};
  ep.sc = *sc;
  ep.pix_part = pix_part;
  ep.n_z = n_z;
  ep.part = part.as<double>();
  ep.n_cta = n_cta;
  ep.per_pixel = per_pixel;
  ep.per_frame = per_frame;
  ep.ftmp = ftmp;
  ep.total = total;
  ep.ticket = ticket + 1;
  ep.plane = plane;
  ep.ref_plane = ref_plane;
  ep.n_o = n_o;
  ep.nb_plane = ref_plane ? (n_o + 255) / 256 : 0;
  const int64_t blocks = sc->n_good + ep.nb_plane + (plane_px + 255) / 256;
  PXST_REQUIRE(blocks < (int64_t(1) << 31), "error maps too large");
  k_err_epilogue<<<(unsigned)blocks, 256, 0, s>>>(ep);
  PXST_CHECK_LAUNCH();
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

// Plane accumulators, quanta and the two tickets in one zeroed scratch
// block, the error pass with the normalisation into ref_plane.
int error_maps_full(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref,
                    const double* u, const double* di, const double* dj, const double* absmax,
                    double* per_frame, double* per_pixel, double* ref_plane, double* total,
                    const FixAcc* next, const int64_t* grid_b, int64_t cap_b, cudaStream_t s) {
  const int64_t n_o = ref->os * ref->of;
  Scratch acc;
  const size_t bytes = sizeof(int64_t) * 4 * n_o + 4 * sizeof(double) + 2 * sizeof(unsigned);
  if (int e = acc.alloc(bytes, s)) return e;
  int64_t* num = acc.as<int64_t>();
  double* q = reinterpret_cast<double*>(num + 4 * n_o);
  double* amax = q + 2;
  unsigned* ticket = reinterpret_cast<unsigned*>(q + 4);
  PXST_CHECK_CUDA(cudaMemsetAsync(num, 0, bytes, s));
  if (!absmax) {
    if (int e = launch_abs_max(sc, amax, s)) return e;
    absmax = amax;
  }
  const FixAcc plane{reinterpret_cast<long long*>(num), reinterpret_cast<long long*>(num + n_o),
                     reinterpret_cast<long long*>(num + 2 * n_o),
                     reinterpret_cast<long long*>(num + 3 * n_o), nullptr, q};
  return error_pass(sc, st, ref, u, di, dj, per_frame, per_pixel, plane, absmax, ref_plane, total,
                    next, grid_b, cap_b, ticket, s);
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
  cudaStream_t s = as_stream(stream);
  Scratch ticket;
  if (int e = ticket.alloc(2 * sizeof(unsigned), s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(ticket.p, 0, 2 * sizeof(unsigned), s));
  return error_pass(sc, st, ref, u, di, dj, per_frame, per_pixel, fix_acc(plane), nullptr,
                    nullptr, nullptr, nullptr, nullptr, 0, ticket.as<unsigned>(), s);
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
