// K0 stack statistics and bbox reductions.
//
// var_pm      recon.py:257-260   sum_n (I-W)^2 (times fw when given)
// sigma2      recon.py:410-412   population variance over good frames,
//                                floored at 1e-8 * max(W_work)^2
// frame_norm  recon.py:367       sum_p (I_n - W)^2
// bbox        recon.py:126-132   min/max of u over work px, of di/dj over good frames
#include "common.cuh"

namespace pxst {
namespace {

constexpr int kThreads = 256;

// Deterministic block reduction helpers (fixed tree).
template <class T, class Op>
__device__ T block_reduce(T v, Op op, T* sh) {
  const T ident = Op::identity();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < nw ? sh[lane] : ident;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;  // valid in thread 0
}

// Max of N values at once (one pair of barriers for all N; min(x) is taken
// as -max(-x)).  Result valid in warp 0.
template <int N>
__device__ void block_max_n(double (&v)[N], double (*sh)[32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = fmax(v[i], __shfl_xor_sync(0xffffffffu, v[i], o));
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) sh[i][w] = v[i];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = lane < nw ? sh[i][lane] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = fmax(v[i], __shfl_xor_sync(0xffffffffu, v[i], o));
  }
}

struct Sum {
  __device__ static double identity() { return 0.0; }
  __device__ double operator()(double a, double b) const { return a + b; }
};
struct Min {
  __device__ static double identity() { return INFINITY; }
  __device__ double operator()(double a, double b) const { return fmin(a, b); }
};
struct Max {
  __device__ static double identity() { return -INFINITY; }
  __device__ double operator()(double a, double b) const { return fmax(a, b); }
};

// Block partials of max W and work-pixel count over the ROI rectangle.
__global__ void k_wmax_partial(pxst_scan sc, double* part_max, double* part_cnt) {
  __shared__ double sh[32];
  const int64_t rw = sc.roi[1] - sc.roi[0], cw = sc.roi[3] - sc.roi[2];
  const int64_t n = rw * cw;
  double mx = -INFINITY, cnt = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = sc.roi[0] + k / cw, c = sc.roi[2] + k % cw;
    const int64_t p = r * sc.fs + c;
    if (sc.work[p]) { mx = fmax(mx, sc.w64[p]); cnt += 1; }
  }
  mx = block_reduce(mx, Max(), sh);
  cnt = block_reduce(cnt, Sum(), sh);
  if (threadIdx.x == 0) { part_max[blockIdx.x] = mx; part_cnt[blockIdx.x] = cnt; }
}

__global__ void k_wmax_final(const double* part_max, const double* part_cnt, int nb,
                             double* scalars) {
  __shared__ double sh[32];
  double mx = -INFINITY, cnt = 0;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) { mx = fmax(mx, part_max[k]); cnt += part_cnt[k]; }
  mx = block_reduce(mx, Max(), sh);
  cnt = block_reduce(cnt, Sum(), sh);
  if (threadIdx.x == 0) {
    scalars[0] = cnt > 0 ? mx : 1.0;   // recon.py:411 uses 1.0 for an empty set
    scalars[2] = cnt;
  }
}

// Per-pixel statistics: one thread per ROI pixel, sequential over good
// frames (the same order as numpy's axis-0 reduction).
__global__ void k_pixel_stats(pxst_scan sc, const float* __restrict__ fw,
                              const double* __restrict__ scalars, double* var_pm,
                              double* sigma2) {
  const int64_t c = sc.roi[2] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = sc.roi[0] + blockIdx.y;
  if (c >= sc.roi[3]) return;
  const int64_t p = r * sc.fs + c;
  if (!sc.work[p]) return;
  const double w = sc.w64[p];
  const int64_t plane = sc.ss * sc.fs;
  const float* fp = sc.frames + p;
  const float* wp = fw ? fw + p : nullptr;
  // Loads kU frames ahead of the adds (memory-level parallelism: one thread
  // per pixel has too few loads in flight otherwise); the adds stay in frame
  // order, so the sums are bit-identical to the sequential loop.
  constexpr int kU = 8;
  double vs = 0.0, sum = 0.0;
  for (int64_t k0 = 0; k0 < sc.n_good; k0 += kU) {
    float I32[kU], F32[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int64_t k = k0 + j < sc.n_good ? k0 + j : sc.n_good - 1;
      const int64_t off = static_cast<int64_t>(__ldg(sc.good + k)) * plane;
      I32[j] = __ldg(fp + off);
      F32[j] = wp ? __ldg(wp + off) : 1.0f;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j)
      if (k0 + j < sc.n_good) {
        const double I = static_cast<double>(I32[j]);
        const double d = I - w;
        double t = d * d;
        if (wp) t = static_cast<double>(F32[j]) * t;
        vs += t;
        sum += I;
      }
  }
  const double mean = sum / static_cast<double>(sc.n_good);
  double ss = 0.0;
  for (int64_t k0 = 0; k0 < sc.n_good; k0 += kU) {
    float I32[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int64_t k = k0 + j < sc.n_good ? k0 + j : sc.n_good - 1;
      I32[j] = __ldg(fp + static_cast<int64_t>(__ldg(sc.good + k)) * plane);
    }
#pragma unroll
    for (int j = 0; j < kU; ++j)
      if (k0 + j < sc.n_good) {
        const double d = static_cast<double>(I32[j]) - mean;
        ss += d * d;
      }
  }
  const double wmax = scalars[0];
  const double floor_ = 1e-8 * wmax * wmax;
  var_pm[p] = vs;
  sigma2[p] = fmax(ss / static_cast<double>(sc.n_good), floor_);
}

// Per-frame normaliser and |I|W mass: one block per good frame.
// Per-frame sums over the ROI's work pixels, split over gridDim.y slices of
// rows (enough blocks to fill the GPU; one block per frame left most SMs
// idle), partial[k * slices + slice]; k_frame_final adds the slices in order.
__global__ void k_frame_stats(pxst_scan sc, double* part_norm, double* part_iw,
                              double* part_i) {
  __shared__ double sh[32];
  const int64_t k = blockIdx.x;
  const int slices = gridDim.y, sl = blockIdx.y;
  const int64_t f = sc.good[k];
  const int64_t rw = sc.roi[1] - sc.roi[0], cw = sc.roi[3] - sc.roi[2];
  const int64_t r_lo = sc.roi[0] + rw * sl / slices, r_hi = sc.roi[0] + rw * (sl + 1) / slices;
  const float* fr = sc.frames + f * sc.ss * sc.fs;
  double acc = 0.0, iw = 0.0, ia = 0.0;
  constexpr int kR = 4;                          // rows in flight per thread
  for (int64_t r0 = r_lo; r0 < r_hi; r0 += kR)
    for (int64_t c = threadIdx.x; c < cw; c += blockDim.x) {
      float I32[kR];
      double w[kR];
      bool m[kR];
#pragma unroll
      for (int j = 0; j < kR; ++j) {             // all loads first
        const bool in = r0 + j < r_hi;
        const int64_t p = (in ? r0 + j : r0) * sc.fs + sc.roi[2] + c;
        I32[j] = __ldg(fr + p);
        w[j] = sc.w64[p];
        m[j] = in && sc.work[p];
      }
#pragma unroll
      for (int j = 0; j < kR; ++j)
        if (m[j]) {
          const double I = static_cast<double>(I32[j]);
          const double d = I - w[j];
          acc += d * d;
          iw += fabs(I) * w[j];
          ia += fabs(I);
        }
    }
  acc = block_reduce(acc, Sum(), sh);
  iw = block_reduce(iw, Sum(), sh);
  ia = block_reduce(ia, Sum(), sh);
  if (threadIdx.x == 0) {
    part_norm[k * slices + sl] = acc;
    part_iw[k * slices + sl] = iw;
    part_i[k * slices + sl] = ia;
  }
}

__global__ void k_frame_final(const double* __restrict__ part_norm,
                              const double* __restrict__ part_iw, const double* __restrict__ part_i,
                              int64_t n_good, int slices, double* frame_norm, double* frame_iw,
                              double* frame_i) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_good;
       k += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int j = 0; j < slices; ++j) {
      a += part_norm[k * slices + j];
      b += part_iw[k * slices + j];
      c += part_i[k * slices + j];
    }
    frame_norm[k] = a;
    frame_iw[k] = b;
    frame_i[k] = c;
  }
}

__global__ void k_sum_final(const double* a, const double* b, int64_t n, double* out_a,
                            double* out_b) {
  __shared__ double sh[32];
  double sa = 0, sb = 0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) { sa += a[k]; sb += b[k]; }
  sa = block_reduce(sa, Sum(), sh);
  sb = block_reduce(sb, Sum(), sh);
  if (threadIdx.x == 0) { *out_a = sa; *out_b = sb; }
}

// bbox of the work pixels' u (min/max of u0, u1) and of the good frames'
// translations, one launch: every block reduces its share of the ROI to
// part[4 * block]; the last block to finish (ticket, zero at start) folds the
// partials, reduces di / dj and writes out[8] and, when given, the grid rule
// of recon.py:126-132: grid = (n0, m0, os, of).
__global__ void k_bbox(pxst_scan sc, const double* __restrict__ u, const double* __restrict__ di,
                       const double* __restrict__ dj, double* part, unsigned* ticket, double* out,
                       int64_t* grid) {
  __shared__ double sh[8][32];
  __shared__ bool s_last;
  const int64_t rw = sc.roi[1] - sc.roi[0], cw = sc.roi[3] - sc.roi[2];
  const int64_t n = rw * cw, plane = sc.ss * sc.fs;
  // (-min u0, max u0, -min u1, max u1)
  double v[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = (sc.roi[0] + k / cw) * sc.fs + sc.roi[2] + k % cw;
    if (!sc.work[p]) continue;
    const double x = u[p], y = u[plane + p];
    v[0] = fmax(v[0], -x); v[1] = fmax(v[1], x); v[2] = fmax(v[2], -y); v[3] = fmax(v[3], y);
  }
  block_max_n<4>(v, sh);
  if (threadIdx.x == 0) {
    double* o = part + 4 * blockIdx.x;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // (-min u0, max u0, -min u1, max u1, -min di, max di, -min dj, max dj)
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = -INFINITY;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x)
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = fmax(r[i], __ldcg(part + 4 * k + i));
  for (int64_t k = threadIdx.x; k < sc.n_good; k += blockDim.x) {
    const int64_t f = sc.good[k];
    const double a = di[f], b = dj[f];
    r[4] = fmax(r[4], -a); r[5] = fmax(r[5], a); r[6] = fmax(r[6], -b); r[7] = fmax(r[7], b);
  }
  block_max_n<8>(r, sh);
  if (threadIdx.x == 0) {
    const double a0 = -r[0], b0 = r[1], a1 = -r[2], b1 = r[3];
    const double c0 = -r[4], d0 = r[5], c1 = -r[6], d1 = r[7];
    out[0] = a0; out[1] = b0; out[2] = a1; out[3] = b1;
    out[4] = c0; out[5] = d0; out[6] = c1; out[7] = d1;
    if (grid) {
      const int64_t n0 = static_cast<int64_t>(floor(a0 - d0));
      const int64_t m0 = static_cast<int64_t>(floor(a1 - d1));
      grid[0] = n0;
      grid[1] = m0;
      grid[2] = static_cast<int64_t>(floor(b0 - c0)) - n0 + 2;
      grid[3] = static_cast<int64_t>(floor(b1 - c1)) - m0 + 2;
    }
  }
}

int partial_blocks(const pxst_scan* sc) {
  const int64_t n = (sc->roi[1] - sc->roi[0]) * (sc->roi[3] - sc->roi[2]);
  int64_t nb = (n + kThreads * 2 - 1) / (kThreads * 2);   // latency-bound: many short blocks
  if (nb < 1) nb = 1;
  if (nb > 1184) nb = 1184;  // 8 x 148 SMs
  return static_cast<int>(nb);
}

}  // namespace

int check_scan(const pxst_scan* sc) {
  PXST_REQUIRE(sc != nullptr, "scan descriptor is NULL");
  PXST_REQUIRE(sc->frames && sc->good && sc->w64 && sc->w32 && sc->work,
               "scan descriptor has a NULL device pointer");
  PXST_REQUIRE(sc->n_frames > 0 && sc->ss > 0 && sc->fs > 0, "empty frame stack");
  PXST_REQUIRE(sc->n_good >= 0 && sc->n_good <= sc->n_frames, "bad n_good");
  PXST_REQUIRE(0 <= sc->roi[0] && sc->roi[0] < sc->roi[1] && sc->roi[1] <= sc->ss &&
                   0 <= sc->roi[2] && sc->roi[2] < sc->roi[3] && sc->roi[3] <= sc->fs,
               "empty or out-of-range ROI");
  PXST_REQUIRE(sc->ss * sc->fs < (int64_t(1) << 31), "detector too large");
  return PXST_OK;
}

}  // namespace pxst

using namespace pxst;

namespace {

// K0 per-pixel part: max W (scalars[0], scalars[2]), var_pm, sigma2.
int pixel_part(const pxst_scan* sc, const float* fw, const pxst_stats* st, cudaStream_t s) {
  const int64_t plane = sc->ss * sc->fs;
  PXST_CHECK_CUDA(cudaMemsetAsync(st->var_pm, 0, sizeof(double) * plane, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(st->sigma2, 0, sizeof(double) * plane, s));
  const int nb = partial_blocks(sc);
  Scratch part;
  if (int e = part.alloc(sizeof(double) * 2 * nb, s)) return e;
  double* pm = part.as<double>();
  double* pc = pm + nb;
  k_wmax_partial<<<nb, kThreads, 0, s>>>(*sc, pm, pc);
  PXST_CHECK_LAUNCH();
  k_wmax_final<<<1, 1024, 0, s>>>(pm, pc, nb, st->scalars);
  PXST_CHECK_LAUNCH();
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  dim3 g((unsigned)((cw + 127) / 128), (unsigned)rw);
  PXST_REQUIRE(rw <= kMaxGridY, "ROI too tall");
  k_pixel_stats<<<g, 128, 0, s>>>(*sc, fw, st->scalars, st->var_pm, st->sigma2);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

// K0 per-frame part: frame_norm, scalars[1], scalars[3].
int frame_part(const pxst_scan* sc, const pxst_stats* st, cudaStream_t s) {
  const int64_t rows = sc->roi[1] - sc->roi[0];
  int64_t slices = (4 * 148 + sc->n_good - 1) / sc->n_good;
  slices = slices < 1 ? 1 : (slices > rows ? rows : slices);
  if (slices > 64) slices = 64;
  Scratch fpart;
  if (int e = fpart.alloc(sizeof(double) * (3 * slices + 2) * sc->n_good, s)) return e;
  double* pn = fpart.as<double>();
  double* fiw = pn + 3 * slices * sc->n_good;
  double* fi = fiw + sc->n_good;
  k_frame_stats<<<dim3((unsigned)sc->n_good, (unsigned)slices), 256, 0, s>>>(
      *sc, pn, pn + slices * sc->n_good, pn + 2 * slices * sc->n_good);
  PXST_CHECK_LAUNCH();
  k_frame_final<<<grid_1d(sc->n_good, 128), 128, 0, s>>>(
      pn, pn + slices * sc->n_good, pn + 2 * slices * sc->n_good, sc->n_good, (int)slices,
      st->frame_norm, fiw, fi);
  PXST_CHECK_LAUNCH();
  k_sum_final<<<1, 1024, 0, s>>>(fiw, fi, sc->n_good, st->scalars + 1, st->scalars + 3);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

}  // namespace

extern "C" int pxst_stack_stats_parts(const pxst_scan* sc, const float* fw,
                                      const pxst_stats* st, int parts, void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(st && st->var_pm && st->sigma2 && st->frame_norm && st->scalars,
               "stats descriptor has a NULL pointer");
  PXST_REQUIRE(sc->n_good > 0, "no good frames");
  PXST_REQUIRE(parts >= 1 && parts <= 3, "parts must be PXST_STATS_PIXEL and/or _FRAME");
  cudaStream_t s = as_stream(stream);
  if (parts & PXST_STATS_PIXEL)
    if (int e = pixel_part(sc, fw, st, s)) return e;
  if (parts & PXST_STATS_FRAME)
    if (int e = frame_part(sc, st, s)) return e;
  return PXST_OK;
}

extern "C" int pxst_stack_stats(const pxst_scan* sc, const float* fw, const pxst_stats* st,
                                void* stream) {
  return pxst_stack_stats_parts(sc, fw, st, PXST_STATS_PIXEL | PXST_STATS_FRAME, stream);
}

extern "C" int pxst_bbox_grid(const pxst_scan* sc, const double* u, const double* di,
                              const double* dj, double* out, int64_t* grid, void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(u && di && dj && out, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  const int nb = partial_blocks(sc);
  Scratch part;
  if (int e = part.alloc(sizeof(double) * 4 * nb + sizeof(unsigned), s)) return e;
  unsigned* ticket = reinterpret_cast<unsigned*>(part.as<double>() + 4 * nb);
  PXST_CHECK_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  k_bbox<<<nb, kThreads, 0, s>>>(*sc, u, di, dj, part.as<double>(), ticket, out, grid);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_bbox(const pxst_scan* sc, const double* u, const double* di,
                         const double* dj, double* out, void* stream) {
  return pxst_bbox_grid(sc, u, di, dj, out, nullptr, stream);
}
