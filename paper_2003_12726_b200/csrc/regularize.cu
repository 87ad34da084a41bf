// Pixel-map regularisation, SURVEY 8(f) rows 1-2 (recon.py:298-311):
//   * mask-aware Gaussian smoothing of the displacement (recon.py:210-218),
//   * irrotational projection by least-squares integration
//     (integration.py:61-134).
//
// Both act on [ss, fs] float64 planes (~1M cells at config 3), so they are
// memory/latency-bound and run replicated on every rank after the u
// all-gather.  Arithmetic follows the reference's operation order with
// explicitly rounded float64 ops (no FMA contraction):
//   * the separable filter is scipy's symmetric correlate1d
//     (out = x[0] w0 + sum_{k=r..1} (x[-k] + x[k]) w_k, mode "nearest"),
//     axis 0 then axis 1;
//   * the normal operator, right-hand side and CG updates are the numpy
//     expressions of integration.py:35-50, 84-113.  Dot products are
//     deterministic two-level reductions (their order differs from BLAS
//     ddot, so CG iterates agree with the reference to rounding, and the
//     converged potentials to ~tol).
// The CG loop is device resident: per iteration three kernels read and
// write a small device state (rs, alpha, beta, best residual, done flag);
// batches of iterations are replayed as a CUDA graph and the host reads the
// done flag once per batch.
#include <math.h>

#include <vector>

#include "common.cuh"

namespace pxst {
namespace {

constexpr int kThreads = 256;
constexpr int kRedBlocks = 592;     // 148 SMs x 4: partial-sum count of a dot product
constexpr int kBatch = 32;          // CG iterations per graph replay (even: p ping-pong)

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// ---------------------------------------------------------------------------
// Gaussian smoothing
// ---------------------------------------------------------------------------
// Field f of the filter input: 0, 1 = (u_f - identity_f) * M, 2 = M.
__device__ __forceinline__ double smooth_src(const double* __restrict__ u,
                                             const uint8_t* __restrict__ m, int64_t ss,
                                             int64_t fs, int f, int64_t i, int64_t j) {
  const int64_t q = i * fs + j;
  const double w = m[q] ? 1.0 : 0.0;
  if (f == 2) return w;
  const double id = f == 0 ? static_cast<double>(i) : static_cast<double>(j);
  return dmul(dsub(u[f * ss * fs + q], id), w);
}

// Pass along axis 0 (scipy correlate1d, mode nearest) of the three fields.
__global__ void k_smooth_axis0(const double* __restrict__ u, const uint8_t* __restrict__ m,
                               int64_t ss, int64_t fs, const double* __restrict__ wt, int r,
                               double* __restrict__ out) {
  const int64_t n = ss * fs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 3 * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int f = static_cast<int>(t / n);
    const int64_t q = t % n, i = q / fs, j = q % fs;
    double o = dmul(smooth_src(u, m, ss, fs, f, i, j), wt[0]);
    for (int k = r; k >= 1; --k) {
      const int64_t lo = i - k < 0 ? 0 : i - k, hi = i + k >= ss ? ss - 1 : i + k;
      o = dadd(o, dmul(dadd(smooth_src(u, m, ss, fs, f, lo, j), smooth_src(u, m, ss, fs, f, hi, j)),
                       wt[k]));
    }
    out[t] = o;
  }
}

// Pass along axis 1 of the three planes of `in`.
__global__ void k_smooth_axis1(const double* __restrict__ in, int64_t ss, int64_t fs,
                               const double* __restrict__ wt, int r, double* __restrict__ out) {
  const int64_t n = ss * fs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 3 * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row0 = (t / fs) * fs, j = t % fs;
    double o = dmul(in[t], wt[0]);
    for (int k = r; k >= 1; --k) {
      const int64_t lo = j - k < 0 ? 0 : j - k, hi = j + k >= fs ? fs - 1 : j + k;
      o = dadd(o, dmul(dadd(in[row0 + lo], in[row0 + hi]), wt[k]));
    }
    out[t] = o;
  }
}

// u = identity + (M && den > 0 ? num / den : u - identity) (recon.py:216-218, :303-304).
__global__ void k_smooth_apply(double* __restrict__ u, const uint8_t* __restrict__ m, int64_t ss,
                               int64_t fs, const double* __restrict__ g) {
  const int64_t n = ss * fs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double den = g[2 * n + q];
    const bool ok = m[q] && den > 0.0;
    const int64_t i = q / fs, j = q % fs;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const double id = f == 0 ? static_cast<double>(i) : static_cast<double>(j);
      const double d = dsub(u[f * n + q], id);
      u[f * n + q] = dadd(id, ok ? __ddiv_rn(g[f * n + q], den) : d);
    }
  }
}

// ---------------------------------------------------------------------------
// CG on the masked Poisson normal operator
// ---------------------------------------------------------------------------
struct CgState {
  double rs, bnorm, best_res, tol, beta;
  long long it, maxiter;
  long long anchor;
  int done, improved;
  double rz;           // preconditioned variant: r . M r
};

__device__ __forceinline__ double link_w(const uint8_t* m, int64_t a, int64_t b) {
  return (m[a] && m[b]) ? 1.0 : 0.0;
}

// Gather form of out[:-1] -= d; out[1:] += d along both axes
// (integration.py:40-49), terms in the reference's order.
template <class F>
__device__ __forceinline__ double normal_op(const uint8_t* __restrict__ m, int64_t ss, int64_t fs,
                                            int64_t i, int64_t j, F val) {
  const int64_t q = i * fs + j;
  double o = 0.0;
  const double c = val(q);
  if (i + 1 < ss) o = dsub(o, dmul(link_w(m, q, q + fs), dsub(val(q + fs), c)));
  if (i > 0) o = dadd(o, dmul(link_w(m, q - fs, q), dsub(c, val(q - fs))));
  if (j + 1 < fs) o = dsub(o, dmul(link_w(m, q, q + 1), dsub(val(q + 1), c)));
  if (j > 0) o = dadd(o, dmul(link_w(m, q - 1, q), dsub(c, val(q - 1))));
  return o;
}

// Deterministic block sum of v; thread 0 returns the total.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[kThreads / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < kThreads / 32; ++k) t += sh[k];
  __syncthreads();
  return t;
}

// Fixed-order sum of the kRedBlocks partials (every caller gets the same value).
__device__ __forceinline__ double sum_partials(const double* __restrict__ part) {
  __shared__ double tot;
  double v = 0.0;
  for (int k = threadIdx.x; k < kRedBlocks; k += kThreads) v += part[k];
  v = block_sum(v);
  if (threadIdx.x == 0) tot = v;
  __syncthreads();
  return tot;
}

__global__ void k_anchor(const uint8_t* __restrict__ m, int64_t n, unsigned long long* anchor) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    if (m[q]) atomicMin(anchor, static_cast<unsigned long long>(q));
}

// b (integration.py:84-91); r = b; p = 0; phi = best = 0; partial b.b.
__global__ void k_cg_init(const double* __restrict__ gx, const double* __restrict__ gy,
                          const uint8_t* __restrict__ m, int64_t ss, int64_t fs,
                          double* __restrict__ r, double* __restrict__ p0,
                          double* __restrict__ p1, double* __restrict__ phi,
                          double* __restrict__ best, double* __restrict__ part) {
  const int64_t n = ss * fs;
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / fs, j = q % fs;
    double o = 0.0;
    if (i + 1 < ss) o = dsub(o, dmul(link_w(m, q, q + fs), gx[q]));
    if (i > 0) o = dadd(o, dmul(link_w(m, q - fs, q), gx[q - fs]));
    if (j + 1 < fs) o = dsub(o, dmul(link_w(m, q, q + 1), gy[q]));
    if (j > 0) o = dadd(o, dmul(link_w(m, q - 1, q), gy[q - 1]));
    r[q] = o;                   // r = b - A 0 = b
    p0[q] = 0.0;
    p1[q] = 0.0;
    phi[q] = 0.0;
    best[q] = 0.0;
    acc += o * o;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_cg_start(const double* __restrict__ part, CgState* st) {
  const double rs = sum_partials(part);
  if (threadIdx.x == 0) {
    const double bn = sqrt(rs);
    st->rs = rs;
    st->bnorm = bn != 0.0 ? bn : 1.0;                 // `or 1.0` (integration.py:96)
    st->best_res = sqrt(rs) / st->bnorm;
    st->beta = 0.0;
    st->it = 0;
    st->improved = 0;
    st->done = !(st->best_res > st->tol && st->it < st->maxiter);
  }
}

// p_new = r + beta p_old (p = r at the first iteration: beta = 0, p_old = 0);
// ap = A p_new; partial p_new . ap.
__global__ void k_cg_apply(const uint8_t* __restrict__ m, int64_t ss, int64_t fs,
                           const double* __restrict__ r, const double* __restrict__ p_old,
                           double* __restrict__ p_new, double* __restrict__ ap,
                           double* __restrict__ part, const CgState* __restrict__ st) {
  if (st->done) return;
  const double beta = st->beta;
  const int64_t anchor = st->anchor;
  const int64_t n = ss * fs;
  auto pn = [&](int64_t q) { return dadd(r[q], dmul(beta, p_old[q])); };
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / fs, j = q % fs;
    const double pq = pn(q);
    double o = normal_op(m, ss, fs, i, j, pn);
    if (q == anchor) o = dadd(o, pq);
    p_new[q] = pq;
    ap[q] = o;
    acc += pq * o;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// alpha = rs / p.ap; (best = phi if the previous iterate improved);
// phi += alpha p; r -= alpha ap; partial r.r.
__global__ void k_cg_update(const double* __restrict__ p, const double* __restrict__ ap,
                            double* __restrict__ phi, double* __restrict__ r,
                            double* __restrict__ best, int64_t n,
                            const double* __restrict__ part_pap, double* __restrict__ part_rr,
                            const CgState* __restrict__ st) {
  if (st->done) return;
  const double alpha = st->rs / sum_partials(part_pap);
  const bool save = st->improved;
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double ph = phi[q];
    if (save) best[q] = ph;
    phi[q] = dadd(ph, dmul(alpha, p[q]));
    const double rq = dsub(r[q], dmul(alpha, ap[q]));
    r[q] = rq;
    acc += rq * rq;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part_rr[blockIdx.x] = t;
}

__global__ void k_cg_step(const double* __restrict__ part_rr, CgState* st) {
  if (st->done) return;
  const double rs_new = sum_partials(part_rr);
  if (threadIdx.x == 0) {
    const double res = sqrt(rs_new) / st->bnorm;
    st->improved = res < st->best_res;
    if (st->improved) st->best_res = res;
    st->beta = rs_new / st->rs;
    st->rs = rs_new;
    st->it += 1;
    st->done = !(res > st->tol && st->it < st->maxiter);
  }
}

// phi_out = best - best[anchor] (best = phi when the last iterate improved).
__global__ void k_cg_finish(const double* __restrict__ phi, const double* __restrict__ best,
                            int64_t n, const CgState* __restrict__ st, double* __restrict__ out) {
  const double* src = st->improved ? phi : best;
  const double a = src[st->anchor];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = dsub(src[q], a);
}

// ---------------------------------------------------------------------------
// Multigrid-preconditioned CG (solver 1).  Same normal operator, right-hand
// side, stopping rule on |r|/|b|, best-iterate tracking and gauge as the plain
// CG; the search directions come from M r, M = one symmetric V(1,1)-cycle of
// aggregation multigrid: level l+1 merges 2x2 cells of level l, its link
// weights are the summed fine links between merged cells (the Galerkin
// product P^T A P for piecewise-constant P keeps the 5-point form), the
// anchor term follows its cell, damped Jacobi (w = 0.8) smooths, the
// piecewise-constant coarse correction is over-corrected by 1.8 (the usual
// remedy for plain aggregation; a constant scale keeps M symmetric), and the
// coarsest level (<= 16x16) takes 64 Jacobi sweeps in one CTA.  Two kernels
// per level and V-cycle: the pre-smoothed z = w D^-1 r is recomputed where
// needed instead of stored.  Converges to the same potential (to the
// tolerance) in ~30-40 iterations instead of thousands (256x512: 31 vs 2673,
// 1024x1024: 37 vs 7152); `iterations` reports the PCG count.
// ---------------------------------------------------------------------------
constexpr double kOmega = 0.8;
#ifndef PXST_MG_OVERCORRECT
#define PXST_MG_OVERCORRECT 1.8
#endif
constexpr double kOverCorrect = PXST_MG_OVERCORRECT;
constexpr int kCoarsest = 16;
constexpr int kCoarseSweeps = 64;
constexpr int kMaxLevels = 16;

struct MgLevel {
  int64_t s, f, anchor;
  double *wx, *wy, *diag, *r, *t;   // t = the level's V-cycle output
};

__device__ __forceinline__ double mg_apply(const double* __restrict__ wx,
                                           const double* __restrict__ wy,
                                           const double* __restrict__ diag, int64_t s, int64_t f,
                                           const double* __restrict__ x, int64_t i, int64_t j) {
  const int64_t q = i * f + j;
  double o = diag[q] * x[q];
  if (i + 1 < s) o -= wx[q] * x[q + f];
  if (i > 0) o -= wx[q - f] * x[q - f];
  if (j + 1 < f) o -= wy[q] * x[q + 1];
  if (j > 0) o -= wy[q - 1] * x[q - 1];
  return o;
}

__global__ void k_mg_fine_weights(const uint8_t* __restrict__ m, int64_t s, int64_t f,
                                  double* __restrict__ wx, double* __restrict__ wy) {
  const int64_t n = s * f;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / f, j = q % f;
    wx[q] = i + 1 < s ? link_w(m, q, q + f) : 0.0;
    wy[q] = j + 1 < f ? link_w(m, q, q + 1) : 0.0;
  }
}

__global__ void k_mg_coarsen(const double* __restrict__ wx, const double* __restrict__ wy,
                             int64_t s, int64_t f, double* __restrict__ cwx,
                             double* __restrict__ cwy, int64_t cs, int64_t cf) {
  const int64_t n = cs * cf;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t I = q / cf, J = q % cf;
    const int64_t i1 = 2 * I + 1, j1 = 2 * J + 1;
    double x = 0.0, y = 0.0;
    if (i1 < s && I + 1 < cs) {                 // links from row 2I+1 down to 2I+2
      x += wx[i1 * f + 2 * J];
      if (j1 < f) x += wx[i1 * f + j1];
    }
    if (j1 < f && J + 1 < cf) {                 // links from col 2J+1 right to 2J+2
      y += wy[(2 * I) * f + j1];
      if (i1 < s) y += wy[i1 * f + j1];
    }
    cwx[q] = x;
    cwy[q] = y;
  }
}

__global__ void k_mg_diag(const double* __restrict__ wx, const double* __restrict__ wy,
                          int64_t s, int64_t f, int64_t anchor, double* __restrict__ diag) {
  const int64_t n = s * f;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / f, j = q % f;
    double d = wx[q] + wy[q];
    if (i > 0) d += wx[q - f];
    if (j > 0) d += wy[q - 1];
    diag[q] = d + (q == anchor ? 1.0 : 0.0);
  }
}

// Pre-smoothing from zero is one damped Jacobi step, z = w D^-1 r; the
// kernels below recompute it where they need it instead of storing it.
__device__ __forceinline__ double mg_pre(const MgLevel& L, int64_t q) {
  const double d = L.diag[q];
  return d > 0.0 ? kOmega * L.r[q] / d : 0.0;
}

// coarse r(I, J) = sum over the 2x2 children of the pre-smoothed residual
// r - A z, z = w D^-1 r
__global__ void k_mg_restrict(MgLevel L, MgLevel C, const CgState* __restrict__ st) {
  if (st->done) return;
  const int64_t n = C.s * C.f;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t I = q / C.f, J = q % C.f;
    double acc = 0.0;
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
      for (int dj = 0; dj < 2; ++dj) {
        const int64_t i = 2 * I + di, j = 2 * J + dj;
        if (i < L.s && j < L.f) {
          const int64_t c = i * L.f + j;
          double az = L.diag[c] * mg_pre(L, c);
          if (i + 1 < L.s) az -= L.wx[c] * mg_pre(L, c + L.f);
          if (i > 0) az -= L.wx[c - L.f] * mg_pre(L, c - L.f);
          if (j + 1 < L.f) az -= L.wy[c] * mg_pre(L, c + 1);
          if (j > 0) az -= L.wy[c - 1] * mg_pre(L, c - 1);
          acc += L.r[c] - az;
        }
      }
    C.r[q] = acc;
  }
}

// coarse-grid correction (piecewise constant, scaled by kOverCorrect) on the
// pre-smoothed z, then one damped Jacobi step: t = z + w D^-1 (r - A z)
__global__ void k_mg_post(MgLevel L, const double* __restrict__ zc, int64_t cf,
                          const CgState* __restrict__ st) {
  if (st->done) return;
  const int64_t n = L.s * L.f;
  auto zz = [&](int64_t c, int64_t i, int64_t j) {
    return L.diag[c] > 0.0 ? mg_pre(L, c) + kOverCorrect * zc[(i / 2) * cf + j / 2] : 0.0;
  };
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / L.f, j = q % L.f;
    const double d = L.diag[q];
    if (!(d > 0.0)) {
      L.t[q] = 0.0;
      continue;
    }
    const double z0 = zz(q, i, j);
    double az = d * z0;
    if (i + 1 < L.s) az -= L.wx[q] * zz(q + L.f, i + 1, j);
    if (i > 0) az -= L.wx[q - L.f] * zz(q - L.f, i - 1, j);
    if (j + 1 < L.f) az -= L.wy[q] * zz(q + 1, i, j + 1);
    if (j > 0) az -= L.wy[q - 1] * zz(q - 1, i, j - 1);
    L.t[q] = z0 + kOmega * (L.r[q] - az) / d;
  }
}

// coarsest level: kCoarseSweeps damped Jacobi sweeps from zero in one CTA
__global__ void k_mg_coarsest(MgLevel L, const CgState* __restrict__ st) {
  if (st->done) return;
  __shared__ double za[kCoarsest * kCoarsest], zb[kCoarsest * kCoarsest];
  const int64_t n = L.s * L.f;
  for (int64_t q = threadIdx.x; q < n; q += blockDim.x) za[q] = 0.0;
  __syncthreads();
  double* cur = za;
  double* nxt = zb;
  for (int it = 0; it < kCoarseSweeps; ++it) {
    for (int64_t q = threadIdx.x; q < n; q += blockDim.x) {
      const int64_t i = q / L.f, j = q % L.f;
      const double d = L.diag[q];
      nxt[q] = d > 0.0 ? cur[q] + kOmega * (L.r[q] - mg_apply(L.wx, L.wy, L.diag, L.s, L.f, cur, i, j)) / d
                       : 0.0;
    }
    __syncthreads();
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  for (int64_t q = threadIdx.x; q < n; q += blockDim.x) L.t[q] = cur[q];
}

// PCG: p_new = z + beta p_old (fused into the operator apply), Ap, p.Ap
__global__ void k_pcg_apply(const uint8_t* __restrict__ m, int64_t ss, int64_t fs,
                            const double* __restrict__ z, const double* __restrict__ p_old,
                            double* __restrict__ p_new, double* __restrict__ ap,
                            double* __restrict__ part, const CgState* __restrict__ st) {
  if (st->done) return;
  const double beta = st->beta;
  const int64_t anchor = st->anchor;
  const int64_t n = ss * fs;
  auto pn = [&](int64_t q) { return dadd(z[q], dmul(beta, p_old[q])); };
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / fs, j = q % fs;
    const double pq = pn(q);
    double o = normal_op(m, ss, fs, i, j, pn);
    if (q == anchor) o = dadd(o, pq);
    p_new[q] = pq;
    ap[q] = o;
    acc += pq * o;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// alpha = rz / p.Ap, then the same phi / r / best update as the plain CG
__global__ void k_pcg_update(const double* __restrict__ p, const double* __restrict__ ap,
                             double* __restrict__ phi, double* __restrict__ r,
                             double* __restrict__ best, int64_t n,
                             const double* __restrict__ part_pap, double* __restrict__ part_rr,
                             const CgState* __restrict__ st) {
  if (st->done) return;
  const double alpha = st->rz / sum_partials(part_pap);
  const bool save = st->improved;
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double ph = phi[q];
    if (save) best[q] = ph;
    phi[q] = dadd(ph, dmul(alpha, p[q]));
    const double rq = dsub(r[q], dmul(alpha, ap[q]));
    r[q] = rq;
    acc += rq * rq;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part_rr[blockIdx.x] = t;
}

// residual norm, best tracking, done flag (beta comes later, from r.z)
__global__ void k_pcg_step(const double* __restrict__ part_rr, CgState* st) {
  if (st->done) return;
  const double rs_new = sum_partials(part_rr);
  if (threadIdx.x == 0) {
    const double res = sqrt(rs_new) / st->bnorm;
    st->improved = res < st->best_res;
    if (st->improved) st->best_res = res;
    st->rs = rs_new;
    st->it += 1;
    st->done = !(res > st->tol && st->it < st->maxiter);
  }
}

__global__ void k_pcg_dot(const double* __restrict__ r, const double* __restrict__ z, int64_t n,
                          double* __restrict__ part, const CgState* __restrict__ st) {
  if (st->done) return;
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    acc += r[q] * z[q];
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// beta = (r.z)_new / (r.z); first = true at the start (beta = 0)
__global__ void k_pcg_beta(const double* __restrict__ part, CgState* st, int first) {
  if (st->done) return;
  const double rz_new = sum_partials(part);
  if (threadIdx.x == 0) {
    st->beta = first ? 0.0 : rz_new / st->rz;
    st->rz = rz_new;
  }
}

// displacement planes for the projection: d_f = u_f - identity_f.
__global__ void k_disp(const double* __restrict__ u, int64_t ss, int64_t fs,
                       double* __restrict__ gx, double* __restrict__ gy) {
  const int64_t n = ss * fs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    gx[q] = dsub(u[q], static_cast<double>(q / fs));
    gy[q] = dsub(u[n + q], static_cast<double>(q % fs));
  }
}

// u = identity + grad(phi) on the support (integration.py:19-31; recon.py:309-310).
__global__ void k_apply_grad(double* __restrict__ u, const uint8_t* __restrict__ m, int64_t ss,
                             int64_t fs, const double* __restrict__ phi) {
  const int64_t n = ss * fs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    if (!m[q]) continue;
    const int64_t i = q / fs, j = q % fs;
    const double gx = i + 1 < ss ? dsub(phi[q + fs], phi[q]) : dsub(phi[q], phi[q - fs]);
    const double gy = j + 1 < fs ? dsub(phi[q + 1], phi[q]) : dsub(phi[q], phi[q - 1]);
    u[q] = dadd(static_cast<double>(i), gx);
    u[n + q] = dadd(static_cast<double>(j), gy);
  }
}

// numpy's pairwise summation (used by ndarray.sum for float64).
double numpy_sum(const double* a, size_t n) {
  if (n < 8) {
    double res = 0.0;
    for (size_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    size_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  size_t n2 = n / 2;
  n2 -= n2 % 8;
  return numpy_sum(a, n2) + numpy_sum(a + n2, n - n2);
}

// scipy.ndimage._gaussian_kernel1d(sigma, 0, radius) with radius = int(4 sigma + 0.5).
std::vector<double> gaussian_weights(double sigma) {
  const int r = static_cast<int>(4.0 * sigma + 0.5);
  std::vector<double> phi(2 * r + 1);
  const double sigma2 = sigma * sigma;
  for (int k = -r; k <= r; ++k)
    phi[k + r] = exp(-0.5 / sigma2 * static_cast<double>(static_cast<int64_t>(k) * k));
  const double s = numpy_sum(phi.data(), phi.size());
  std::vector<double> half(r + 1);
  for (int k = 0; k <= r; ++k) half[k] = phi[k + r] / s;
  return half;
}

int cg_solve(const double* gx, const double* gy, const uint8_t* m, int64_t ss, int64_t fs,
             double tol, int64_t maxiter, double* phi_out, pxst_cg_info* info, cudaStream_t s) {
  const int64_t n = ss * fs;
  const int grid = grid_1d(n, kThreads) < kRedBlocks ? grid_1d(n, kThreads) : kRedBlocks;
  Scratch buf, stb;
  if (int e = buf.alloc(sizeof(double) * (6 * n + 2 * kRedBlocks), s)) return e;
  if (int e = stb.alloc(sizeof(CgState) + sizeof(unsigned long long), s)) return e;
  double* r = buf.as<double>();
  double* p0 = r + n;
  double* p1 = p0 + n;
  double* ap = p1 + n;
  double* phi = ap + n;
  double* best = phi + n;
  double* part_a = best + n;
  double* part_b = part_a + kRedBlocks;
  CgState* st = stb.as<CgState>();
  unsigned long long* anchor = reinterpret_cast<unsigned long long*>(st + 1);
  PXST_CHECK_CUDA(cudaMemsetAsync(part_a, 0, sizeof(double) * 2 * kRedBlocks, s));

  // anchor = first mask pixel (np.argwhere order); an empty mask is the
  // reference's ValueError (integration.py:80-81).
  PXST_CHECK_CUDA(cudaMemsetAsync(anchor, 0xff, sizeof(unsigned long long), s));
  k_anchor<<<grid_1d(n, kThreads), kThreads, 0, s>>>(m, n, anchor);
  PXST_CHECK_LAUNCH();
  unsigned long long h_anchor = 0;
  PXST_CHECK_CUDA(cudaMemcpyAsync(&h_anchor, anchor, sizeof(h_anchor), cudaMemcpyDeviceToHost, s));
  PXST_CHECK_CUDA(cudaStreamSynchronize(s));
  PXST_REQUIRE(h_anchor != ~0ull, "integrate_gradient: mask has no good pixels");

  CgState h{};
  h.tol = tol;
  h.maxiter = maxiter > 0 ? maxiter : 20 * n;             // integration.py:93-94
  h.anchor = static_cast<long long>(h_anchor);
  PXST_CHECK_CUDA(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  k_cg_init<<<grid, kThreads, 0, s>>>(gx, gy, m, ss, fs, r, p0, p1, phi, best, part_a);
  PXST_CHECK_LAUNCH();
  k_cg_start<<<1, kThreads, 0, s>>>(part_a, st);
  PXST_CHECK_LAUNCH();

  // Batches of kBatch iterations, captured once on a private stream and
  // replayed until the device sets `done` (kernels of finished batches
  // return at once).
  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int rc = PXST_OK;
  auto fail = [&](cudaError_t e, const char* what) {
    rc = set_error(PXST_ECUDA, "%s failed: %s", what, cudaGetErrorString(e));
  };
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) { fail(e, "cudaStreamCreate"); return rc; }
  e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev, 0);
  if (e == cudaSuccess) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    for (int k = 0; k < kBatch; ++k) {
      double* po = (k & 1) ? p1 : p0;
      double* pn = (k & 1) ? p0 : p1;
      k_cg_apply<<<grid, kThreads, 0, cs>>>(m, ss, fs, r, po, pn, ap, part_a, st);
      k_cg_update<<<grid, kThreads, 0, cs>>>(pn, ap, phi, r, best, n, part_a, part_b, st);
      k_cg_step<<<1, kThreads, 0, cs>>>(part_b, st);
    }
    e = cudaStreamEndCapture(cs, &graph);
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  int done = 0;
  long long launched = 0;
  while (e == cudaSuccess && !done) {
    e = cudaGraphLaunch(exec, cs);
    launched += 3 * kBatch;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  }
  if (e != cudaSuccess) fail(e, "CG graph");
  count_launch(static_cast<int>(launched));
  if (e == cudaSuccess) {
    k_cg_finish<<<grid_1d(n, kThreads), kThreads, 0, cs>>>(phi, best, n, st, phi_out);
    e = cudaGetLastError();
    count_launch();
    if (e == cudaSuccess) e = cudaEventRecord(ev, cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev, 0);
    if (e != cudaSuccess) fail(e, "CG finish");
  }
  if (rc == PXST_OK && info) {
    e = cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      fail(e, "CG info");
    } else {
      info->iterations = h.it;
      info->residual = h.best_res;
      info->converged = h.best_res <= tol;
    }
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  if (ev) cudaEventDestroy(ev);
  cudaStreamDestroy(cs);
  return rc;
}

int mgcg_solve(const double* gx, const double* gy, const uint8_t* m, int64_t ss, int64_t fs,
               double tol, int64_t maxiter, double* phi_out, pxst_cg_info* info, cudaStream_t s) {
  const int64_t n = ss * fs;
  const int grid = grid_1d(n, kThreads) < kRedBlocks ? grid_1d(n, kThreads) : kRedBlocks;
  // level sizes
  int64_t ls[kMaxLevels], lf[kMaxLevels];
  int nl = 1;
  ls[0] = ss;
  lf[0] = fs;
  while (nl < kMaxLevels && (ls[nl - 1] > kCoarsest || lf[nl - 1] > kCoarsest)) {
    ls[nl] = (ls[nl - 1] + 1) / 2;
    lf[nl] = (lf[nl - 1] + 1) / 2;
    ++nl;
  }
  int64_t lvl_cells = 0;
  for (int l = 0; l < nl; ++l) lvl_cells += ls[l] * lf[l];
  Scratch buf, stb, mg;
  if (int e = buf.alloc(sizeof(double) * (6 * n + 3 * kRedBlocks), s)) return e;
  if (int e = stb.alloc(sizeof(CgState) + sizeof(unsigned long long), s)) return e;
  // per level: wx, wy, diag, t (+ r for l >= 1)
  if (int e = mg.alloc(sizeof(double) * 5 * lvl_cells, s)) return e;
  double* r = buf.as<double>();
  double* p0 = r + n;
  double* p1 = p0 + n;
  double* ap = p1 + n;
  double* phi = ap + n;
  double* best = phi + n;
  double* part_a = best + n;
  double* part_b = part_a + kRedBlocks;
  double* part_c = part_b + kRedBlocks;
  CgState* st = stb.as<CgState>();
  unsigned long long* anchor = reinterpret_cast<unsigned long long*>(st + 1);
  PXST_CHECK_CUDA(cudaMemsetAsync(part_a, 0, sizeof(double) * 3 * kRedBlocks, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(anchor, 0xff, sizeof(unsigned long long), s));
  k_anchor<<<grid_1d(n, kThreads), kThreads, 0, s>>>(m, n, anchor);
  PXST_CHECK_LAUNCH();
  unsigned long long h_anchor = 0;
  PXST_CHECK_CUDA(cudaMemcpyAsync(&h_anchor, anchor, sizeof(h_anchor), cudaMemcpyDeviceToHost, s));
  PXST_CHECK_CUDA(cudaStreamSynchronize(s));
  PXST_REQUIRE(h_anchor != ~0ull, "integrate_gradient: mask has no good pixels");

  MgLevel lv[kMaxLevels];
  double* cur = mg.as<double>();
  const int64_t ai = static_cast<int64_t>(h_anchor) / fs, aj = static_cast<int64_t>(h_anchor) % fs;
  for (int l = 0; l < nl; ++l) {
    const int64_t c = ls[l] * lf[l];
    lv[l].s = ls[l];
    lv[l].f = lf[l];
    lv[l].anchor = (ai >> l) * lf[l] + (aj >> l);
    lv[l].wx = cur; cur += c;
    lv[l].wy = cur; cur += c;
    lv[l].diag = cur; cur += c;
    lv[l].t = cur; cur += c;
    lv[l].r = l == 0 ? r : cur;
    cur += c;
  }
  k_mg_fine_weights<<<grid_1d(n, kThreads), kThreads, 0, s>>>(m, ss, fs, lv[0].wx, lv[0].wy);
  PXST_CHECK_LAUNCH();
  for (int l = 0; l + 1 < nl; ++l) {
    k_mg_coarsen<<<grid_1d(ls[l + 1] * lf[l + 1], kThreads), kThreads, 0, s>>>(
        lv[l].wx, lv[l].wy, ls[l], lf[l], lv[l + 1].wx, lv[l + 1].wy, ls[l + 1], lf[l + 1]);
    PXST_CHECK_LAUNCH();
  }
  for (int l = 0; l < nl; ++l) {
    k_mg_diag<<<grid_1d(ls[l] * lf[l], kThreads), kThreads, 0, s>>>(lv[l].wx, lv[l].wy, ls[l],
                                                                     lf[l], lv[l].anchor,
                                                                     lv[l].diag);
    PXST_CHECK_LAUNCH();
  }

  CgState h{};
  h.tol = tol;
  h.maxiter = maxiter > 0 ? maxiter : 20 * n;             // integration.py:93-94
  h.anchor = static_cast<long long>(h_anchor);
  PXST_CHECK_CUDA(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  k_cg_init<<<grid, kThreads, 0, s>>>(gx, gy, m, ss, fs, r, p0, p1, phi, best, part_a);
  PXST_CHECK_LAUNCH();
  k_cg_start<<<1, kThreads, 0, s>>>(part_a, st);
  PXST_CHECK_LAUNCH();

  auto vcycle = [&](cudaStream_t q) {
    for (int l = 0; l + 1 < nl; ++l)
      k_mg_restrict<<<grid_1d(ls[l + 1] * lf[l + 1], kThreads), kThreads, 0, q>>>(lv[l],
                                                                                  lv[l + 1], st);
    k_mg_coarsest<<<1, 256, 0, q>>>(lv[nl - 1], st);
    for (int l = nl - 2; l >= 0; --l)
      k_mg_post<<<grid_1d(ls[l] * lf[l], kThreads), kThreads, 0, q>>>(lv[l], lv[l + 1].t,
                                                                       lf[l + 1], st);
  };
  const int per_iter_launches = 5 + 2 * (nl - 1) + 1;
  // z0 = M r, rz = r.z, p0 stays 0 so the first p is z
  vcycle(s);
  k_pcg_dot<<<grid, kThreads, 0, s>>>(r, lv[0].t, n, part_c, st);
  k_pcg_beta<<<1, kThreads, 0, s>>>(part_c, st, 1);
  PXST_CHECK_LAUNCH();
  count_launch(per_iter_launches - 3);

  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int rc = PXST_OK;
  auto fail = [&](cudaError_t e, const char* what) {
    rc = set_error(PXST_ECUDA, "%s failed: %s", what, cudaGetErrorString(e));
  };
  constexpr int kMgBatch = 8;    // PCG iterations per graph replay (even: p ping-pong)
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) { fail(e, "cudaStreamCreate"); return rc; }
  e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev, 0);
  if (e == cudaSuccess) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    for (int k = 0; k < kMgBatch; ++k) {
      double* po = (k & 1) ? p1 : p0;
      double* pn = (k & 1) ? p0 : p1;
      k_pcg_apply<<<grid, kThreads, 0, cs>>>(m, ss, fs, lv[0].t, po, pn, ap, part_a, st);
      k_pcg_update<<<grid, kThreads, 0, cs>>>(pn, ap, phi, r, best, n, part_a, part_b, st);
      k_pcg_step<<<1, kThreads, 0, cs>>>(part_b, st);
      vcycle(cs);
      k_pcg_dot<<<grid, kThreads, 0, cs>>>(r, lv[0].t, n, part_c, st);
      k_pcg_beta<<<1, kThreads, 0, cs>>>(part_c, st, 0);
    }
    e = cudaStreamEndCapture(cs, &graph);
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  int done = 0;
  long long launched = 0;
  while (e == cudaSuccess && !done) {
    e = cudaGraphLaunch(exec, cs);
    launched += (long long)per_iter_launches * kMgBatch;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  }
  if (e != cudaSuccess) fail(e, "MG-PCG graph");
  count_launch(static_cast<int>(launched));
  if (e == cudaSuccess) {
    k_cg_finish<<<grid_1d(n, kThreads), kThreads, 0, cs>>>(phi, best, n, st, phi_out);
    e = cudaGetLastError();
    count_launch();
    if (e == cudaSuccess) e = cudaEventRecord(ev, cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev, 0);
    if (e != cudaSuccess) fail(e, "MG-PCG finish");
  }
  if (rc == PXST_OK && info) {
    e = cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      fail(e, "MG-PCG info");
    } else {
      info->iterations = h.it;
      info->residual = h.best_res;
      info->converged = h.best_res <= tol;
    }
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  if (ev) cudaEventDestroy(ev);
  cudaStreamDestroy(cs);
  return rc;
}

int solve(int solver, const double* gx, const double* gy, const uint8_t* m, int64_t ss,
          int64_t fs, double tol, int64_t maxiter, double* phi, pxst_cg_info* info,
          cudaStream_t s) {
  return solver == 1 ? mgcg_solve(gx, gy, m, ss, fs, tol, maxiter, phi, info, s)
                     : cg_solve(gx, gy, m, ss, fs, tol, maxiter, phi, info, s);
}

}  // namespace
}  // namespace pxst

using namespace pxst;

extern "C" int pxst_smooth_displacement(double* u, const uint8_t* support, int64_t ss, int64_t fs,
                                        double sigma, void* stream) {
  PXST_REQUIRE(u && support, "NULL pointer");
  PXST_REQUIRE(ss > 0 && fs > 0, "bad plane shape");
  PXST_REQUIRE(sigma >= 0.0 && sigma < 1e4, "sigma must be in [0, 1e4)");
  if (sigma == 0.0) return PXST_OK;
  cudaStream_t s = as_stream(stream);
  const std::vector<double> w = gaussian_weights(sigma);
  const int r = static_cast<int>(w.size()) - 1;
  const int64_t n = ss * fs;
  Scratch buf;
  if (int e = buf.alloc(sizeof(double) * (6 * n + w.size()), s)) return e;
  double* g1 = buf.as<double>();
  double* g2 = g1 + 3 * n;
  double* wt = g2 + 3 * n;
  PXST_CHECK_CUDA(cudaMemcpyAsync(wt, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice, s));
  k_smooth_axis0<<<grid_1d(3 * n, kThreads), kThreads, 0, s>>>(u, support, ss, fs, wt, r, g1);
  PXST_CHECK_LAUNCH();
  k_smooth_axis1<<<grid_1d(3 * n, kThreads), kThreads, 0, s>>>(g1, ss, fs, wt, r, g2);
  PXST_CHECK_LAUNCH();
  k_smooth_apply<<<grid_1d(n, kThreads), kThreads, 0, s>>>(u, support, ss, fs, g2);
  PXST_CHECK_LAUNCH();
  // the host weight vector must outlive the async copy
  PXST_CHECK_CUDA(cudaStreamSynchronize(s));
  return PXST_OK;
}

extern "C" int pxst_integrate_gradient(const double* gx, const double* gy, const uint8_t* mask,
                                       int64_t ss, int64_t fs, double tol, int64_t maxiter,
                                       int solver, double* phi, pxst_cg_info* info,
                                       void* stream) {
  PXST_REQUIRE(gx && gy && mask && phi, "NULL pointer");
  PXST_REQUIRE(ss >= 2 && fs >= 2, "integrate_gradient needs at least a 2x2 grid");
  PXST_REQUIRE(tol >= 0.0, "tol must be >= 0");
  PXST_REQUIRE(solver == 0 || solver == 1, "solver must be 0 (CG) or 1 (MG-PCG)");
  return solve(solver, gx, gy, mask, ss, fs, tol, maxiter, phi, info, as_stream(stream));
}

extern "C" int pxst_project_irrotational(double* u, const uint8_t* support, int64_t ss,
                                         int64_t fs, double tol, int64_t maxiter, int solver,
                                         pxst_cg_info* info, void* stream) {
  PXST_REQUIRE(u && support, "NULL pointer");
  PXST_REQUIRE(ss >= 2 && fs >= 2, "integrate_gradient needs at least a 2x2 grid");
  PXST_REQUIRE(tol >= 0.0, "tol must be >= 0");
  cudaStream_t s = as_stream(stream);
  const int64_t n = ss * fs;
  Scratch buf;
  if (int e = buf.alloc(sizeof(double) * 3 * n, s)) return e;
  double* gx = buf.as<double>();
  double* gy = gx + n;
  double* phi = gy + n;
  k_disp<<<grid_1d(n, kThreads), kThreads, 0, s>>>(u, ss, fs, gx, gy);
  PXST_CHECK_LAUNCH();
  PXST_REQUIRE(solver == 0 || solver == 1, "solver must be 0 (CG) or 1 (MG-PCG)");
  if (int e = solve(solver, gx, gy, support, ss, fs, tol, maxiter, phi, info, s)) return e;
  k_apply_grad<<<grid_1d(n, kThreads), kThreads, 0, s>>>(u, support, ss, fs, phi);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}
