// K3: per-frame translation grid search (recon.py:336-385).
//
// One CTA per (searched frame, band of 16 detector rows): the band's object
// window for that frame is staged in shared memory (cp.async), threads stride
// over the band's pixels accumulating the phase group's Ka x Kb trial window
// in registers (same engine as K2), then a deterministic CTA reduction writes
// float32 partials[frame][band][trial].  A per-frame epilogue sums the bands
// in float64 (fixed order), normalises by sum_p (I_n - W)^2, takes the
// first-occurrence argmin and applies the reference's always-on paraboloid
// (offset in grid-index units added in pixels).
//
// Sub-pixel grids with integral 1/step (config 4: 0.25 px) decompose into
// q^2 phase groups, each an integer window of the engine: trial k = q m + rho
// sits at floor(x - step*rho) - m with the same fractions for every m.
#include "search_common.cuh"

namespace pxst {

int check_scan(const pxst_scan* sc);

namespace {

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = ok ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Stage the [wr0, wr0+WR) x [wc0, wc0+WC) window of fm into smem (row pitch
// WC), zero outside the grid.  Warps walk rows, lanes walk columns.
__device__ __forceinline__ void stage_window(float* dst, const float* __restrict__ fm, int64_t os,
                                             int64_t of, int wr0, int wc0, int WR, int WC) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < WR; r += nw) {
    const int gr = wr0 + r;
    const bool rok = gr >= 0 && gr < os;
    const float* srow = fm + (rok ? (int64_t)gr * of : 0);
    for (int c = lane; c < WC; c += 32) {
      const int gc = wc0 + c;
      const bool ok = rok && gc >= 0 && gc < of;
      cp_async4(dst + r * WC + c, ok ? srow + gc : fm, ok);
    }
  }
}

constexpr int kTrThreads = 256;
constexpr int kTrBand = 16;   // detector rows per band

struct TransArgs {
  pxst_scan sc;
  const double* u;
  const double* di;
  const double* dj;
  const float* fm;
  const uint8_t* valid;
  const uint8_t* pv;
  int64_t os, of, n0, m0;
  const double* band_mm;   // [n_bands][4] min/max u0, min/max u1 over work px
  int64_t n_bands;
  int64_t frame_lo;        // first searched frame (index into good)
  // phase group
  double ph_a, ph_b;       // sub-pixel phase shifts s*rho (0 for integer grids)
  int mhi_a, mhi_b;        // largest integer step of the phase group
  int q_a, q_b;            // steps per pixel (1/step)
  int rho_a, rho_b;
  int kh_a, kh_b;          // full-grid half counts (offset index = k + kh)
  int na_full, nb_full;
  float* partial;          // [n_frames_chunk][n_bands][na_full*nb_full]
  int win_cap;
};

template <int KA, int KB>
__global__ void __launch_bounds__(kTrThreads, (KA * KB <= 81) ? 2 : 1) k_trans_partial(TransArgs a) {
  extern __shared__ float win[];
  __shared__ float red[kTrThreads / 32][KA * KB];
  const int band = blockIdx.x;
  const int64_t kk = blockIdx.y;                       // frame within the chunk
  const int64_t f = a.sc.good[a.frame_lo + kk];
  const int64_t r_lo = a.sc.roi[0] + (int64_t)band * kTrBand;
  const int64_t r_hi = min(a.sc.roi[1], r_lo + kTrBand);
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2];
  const int64_t nq = (r_hi - r_lo) * cw;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const double mn0 = a.band_mm[4 * band], mx0 = a.band_mm[4 * band + 1];
  const double mn1 = a.band_mm[4 * band + 2], mx1 = a.band_mm[4 * band + 3];

  float acc[KA][KB];
#pragma unroll
  for (int t = 0; t < KA; ++t)
#pragma unroll
    for (int s = 0; s < KB; ++s) acc[t][s] = 0.f;

  if (mn0 <= mx0) {
    // x_rho = (u0 - di - n0) - s*rho; trial m -> base row floor(x_rho) - m,
    // engine row t <-> m = mhi - t (recon.py:373-374 sign convention).
    const double xs = a.di[f] + static_cast<double>(a.n0) + a.ph_a;
    const double ys = a.dj[f] + static_cast<double>(a.m0) + a.ph_b;
    const int WR = clamp_span(floor(mx0 - mn0)) + KA + 2;
    const int WC = clamp_span(floor(mx1 - mn1)) + KB + 2;
    const bool use_win = WR * WC <= a.win_cap && fabs(mn0) < 1e9 && fabs(mn1) < 1e9;
    const int wr0 = use_win ? static_cast<int>(floor(mn0 - xs)) - a.mhi_a : 0;
    const int wc0 = use_win ? static_cast<int>(floor(mn1 - ys)) - a.mhi_b : 0;
    if (use_win) stage_window(win, a.fm, a.os, a.of, wr0, wc0, WR, WC);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const float* frame = a.sc.frames + f * plane;
    for (int64_t q = threadIdx.x; q < nq; q += kTrThreads) {
      const int64_t p = (r_lo + q / cw) * a.sc.fs + a.sc.roi[2] + q % cw;
      if (!a.sc.work[p]) continue;
      const double x = (a.u[p] - a.di[f] - static_cast<double>(a.n0)) - a.ph_a;
      const double y = (a.u[plane + p] - a.dj[f] - static_cast<double>(a.m0)) - a.ph_b;
      const double xf = floor(x), yf = floor(y);
      const double fxd = x - xf, fyd = y - yf;
      const bool finite = fabs(x) < 1e9 && fabs(y) < 1e9;
      const int i = finite ? static_cast<int>(xf) : -(1 << 30);
      const int j = finite ? static_cast<int>(yf) : -(1 << 30);
      const float I = __ldg(frame + p);
      const float W = a.sc.w32[p];
      const int pr = i - a.mhi_a, pc = j - a.mhi_b;
      bool fast = use_win && i >= 0 && i < a.os && j >= 0 && j < a.of &&
                  a.pv[(int64_t)i * a.of + j] != 0;
      const int lr = pr - wr0, lc = pc - wc0;
      fast = fast && lr >= 0 && lr + KA + 1 <= WR && lc >= 0 && lc + KB + 1 <= WC;
      if (fast) {
        const float fx = static_cast<float>(fxd), fy = static_cast<float>(fyd);
        engine_fast<KA, KB>(win + lr * WC + lc, WC, fx, fy, W * (1.f - fx), W * fx, I, acc);
      } else {
        engine_slow<KA, KB>(a.fm, a.valid, a.os, a.of, pr, pc, fxd, fyd, W, I, 1.f, acc);
      }
    }
  }
  // Deterministic CTA reduction: warp shuffles, then fixed-order sum of warps.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < KA; ++t)
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      const float v = warp_sumf(acc[t][s]);
      if (lane == 0) red[warp][t * KB + s] = v;
    }
  __syncthreads();
  const int nk = a.na_full * a.nb_full;
  float* out = a.partial + (kk * a.n_bands + band) * (int64_t)nk;
  for (int e = threadIdx.x; e < KA * KB; e += kTrThreads) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kTrThreads / 32; ++w) v += red[w][e];
    const int t = e / KB, s = e % KB;
    const int ia = a.q_a * (a.mhi_a - t) + a.rho_a + a.kh_a;
    const int ib = a.q_b * (a.mhi_b - s) + a.rho_b + a.kh_b;
    out[ia * a.nb_full + ib] = v;
  }
}

// Generic K3: one CTA per (searched frame, full-grid trial), float64.
__global__ void k_trans_generic(TransArgs a, const double* __restrict__ offs_a,
                                const double* __restrict__ offs_b, double* __restrict__ errs) {
  __shared__ double sh[32];
  const int64_t kk = blockIdx.y;
  const int t = blockIdx.x;
  const int64_t f = a.sc.good[a.frame_lo + kk];
  const int nb = a.nb_full;
  const double oa = offs_a[t / nb], ob = offs_b[t % nb];
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2], rw = a.sc.roi[1] - a.sc.roi[0];
  const int64_t plane = a.sc.ss * a.sc.fs;
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < cw * rw; q += blockDim.x) {
    const int64_t p = (a.sc.roi[0] + q / cw) * a.sc.fs + a.sc.roi[2] + q % cw;
    if (!a.sc.work[p]) continue;
    const double x = a.u[p] - (a.di[f] + oa) - a.n0;           // recon.py:373
    const double y = a.u[plane + p] - (a.dj[f] + ob) - a.m0;   // recon.py:374
    const double I = static_cast<double>(__ldg(a.sc.frames + f * plane + p));
    const double W = a.sc.w64[p];
    float v = 0.f;
    bool ok = false;
    if (fabs(x) < 1e9 && fabs(y) < 1e9) {
      const Split sx = split(x), sy = split(y);
      ok = masked_read(a.fm, a.valid, a.os, a.of, sx.i, sy.i, sx.f, sy.f, v);
    }
    const double r = ok ? I - W * static_cast<double>(v) : I - W;
    acc += r * r;
  }
  acc = warp_sum(acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    errs[kk * (int64_t)(a.na_full * a.nb_full) + t] = s;
  }
}

// Per-frame epilogue: sum partials over bands (fixed order, float64),
// normalise, first-occurrence argmin, paraboloid when interior (always, in
// grid-index units added as pixels: recon.py:380-384), write translations.
template <class T>
__global__ void k_trans_epilogue(pxst_scan sc, const double* __restrict__ frame_norm,
                                 const T* __restrict__ part, int64_t n_bands, int64_t frame_lo,
                                 int na, int nb, const double* __restrict__ offs_a,
                                 const double* __restrict__ offs_b, const double* di,
                                 const double* dj, double* di_out, double* dj_out,
                                 double* err_out) {
  extern __shared__ double e[];
  __shared__ double bv[32];
  __shared__ int bi[32];
  const int64_t kk = blockIdx.x;
  const int64_t k = frame_lo + kk;
  const int64_t f = sc.good[k];
  const double norm = frame_norm[k];
  const int nk = na * nb;
  const T* pp = part + kk * n_bands * nk;
  for (int t = threadIdx.x; t < nk; t += blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < n_bands; ++b) s += static_cast<double>(pp[b * nk + t]);
    e[t] = norm > 0.0 ? s / norm : s;
  }
  __syncthreads();
  if (err_out)
    for (int t = threadIdx.x; t < nk; t += blockDim.x) err_out[kk * nk + t] = e[t];
  if (!(norm > 0.0)) return;                                  // recon.py:367-369
  double v = INFINITY;
  int idx = 0x7fffffff;
  for (int t = threadIdx.x; t < nk; t += blockDim.x)
    if (e[t] < v) { v = e[t]; idx = t; }
  // (value, index) lexicographic min == numpy first-occurrence argmin
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov < v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { bv[warp] = v; bi[warp] = idx; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  v = bv[0];
  idx = bi[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
    if (bv[w] < v || (bv[w] == v && bi[w] < idx)) { v = bv[w]; idx = bi[w]; }
  if (idx == 0x7fffffff) idx = 0;   // all NaN/inf: numpy would pick the first
  const int ia = idx / nb, ib = idx % nb;
  double da = 0.0, db = 0.0;
  if (ia > 0 && ia < na - 1 && ib > 0 && ib < nb - 1) {
    double q[9];
    for (int d = 0; d < 9; ++d) q[d] = e[(ia + d / 3 - 1) * nb + (ib + d % 3 - 1)];
    paraboloid(q, da, db);
  }
  di_out[f] = di[f] + offs_a[ia] + da;                        // recon.py:383-384
  dj_out[f] = dj[f] + offs_b[ib] + db;
}

// band bbox of u over work pixels
__global__ void k_band_mm(pxst_scan sc, const double* __restrict__ u, int band_rows,
                          double* out) {
  const int band = blockIdx.x;
  const int64_t r_lo = sc.roi[0] + (int64_t)band * band_rows;
  const int64_t r_hi = min(sc.roi[1], r_lo + band_rows);
  const int64_t cw = sc.roi[3] - sc.roi[2];
  const int64_t plane = sc.ss * sc.fs;
  double a0 = INFINITY, b0 = -INFINITY, a1 = INFINITY, b1 = -INFINITY;
  for (int64_t q = threadIdx.x; q < (r_hi - r_lo) * cw; q += blockDim.x) {
    const int64_t p = (r_lo + q / cw) * sc.fs + sc.roi[2] + q % cw;
    if (!sc.work[p]) continue;
    a0 = fmin(a0, u[p]); b0 = fmax(b0, u[p]);
    a1 = fmin(a1, u[plane + p]); b1 = fmax(b1, u[plane + p]);
  }
  __shared__ double sh[4][32];
  a0 = warp_min(a0); b0 = warp_max(b0); a1 = warp_min(a1); b1 = warp_max(b1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sh[0][warp] = a0; sh[1][warp] = b0; sh[2][warp] = a1; sh[3][warp] = b1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      a0 = fmin(a0, sh[0][w]); b0 = fmax(b0, sh[1][w]);
      a1 = fmin(a1, sh[2][w]); b1 = fmax(b1, sh[3][w]);
    }
    out[4 * band] = sh[0][0] < a0 ? sh[0][0] : a0;
    out[4 * band + 1] = sh[1][0] > b0 ? sh[1][0] : b0;
    out[4 * band + 2] = sh[2][0] < a1 ? sh[2][0] : a1;
    out[4 * band + 3] = sh[3][0] > b1 ? sh[3][0] : b1;
  }
}

// ----------------------------------------------------------------------------
using TrKernel = void (*)(TransArgs);
struct TrEntry { int ka, kb; TrKernel fn; };
#define TR(a, b) TrEntry{a, b, k_trans_partial<a, b>}
const TrEntry kTrTable[] = {
    TR(1, 1), TR(3, 3), TR(5, 5), TR(7, 7), TR(9, 9), TR(11, 11), TR(13, 13),
    TR(8, 8), TR(8, 9), TR(9, 8), TR(9, 9),
};
#undef TR

TrKernel find_tr(int ka, int kb) {
  for (const auto& e : kTrTable)
    if (e.ka == ka && e.kb == kb) return e.fn;
  return nullptr;
}

}  // namespace
}  // namespace pxst

using namespace pxst;

extern "C" int pxst_translation_search(const pxst_scan* sc, const pxst_stats* st,
                                       const pxst_ref* ref, const double* u, const double* di,
                                       const double* dj, int64_t half_ss, int64_t half_fs,
                                       double subpixel_step, int64_t frame_lo, int64_t frame_hi,
                                       double* di_out, double* dj_out, double* err_out,
                                       void* stream) {
  if (int e = check_scan(sc)) return e;
  if (int e = check_ref(ref)) return e;
  PXST_REQUIRE(st && st->frame_norm, "stats descriptor is NULL");
  PXST_REQUIRE(u && di && dj && di_out && dj_out, "NULL pointer");
  PXST_REQUIRE(half_ss >= 0 && half_fs >= 0, "search window halves must be >= 0");
  PXST_REQUIRE(subpixel_step == 0.0 || (subpixel_step > 0.0 && subpixel_step <= 1.0),
               "subpixel_grid step must be in (0, 1]");
  PXST_REQUIRE(0 <= frame_lo && frame_lo <= frame_hi && frame_hi <= sc->n_good,
               "bad frame range");
  cudaStream_t s = as_stream(stream);
  if (frame_hi == frame_lo) return PXST_OK;

  const std::vector<double> oa = window_offsets(half_ss, subpixel_step);
  const std::vector<double> ob = window_offsets(half_fs, subpixel_step);
  const int na = static_cast<int>(oa.size()), nb = static_cast<int>(ob.size());
  const int nk = na * nb;
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];

  Scratch offs;
  if (int e = offs.alloc(sizeof(double) * (na + nb), s)) return e;
  PXST_CHECK_CUDA(cudaMemcpyAsync(offs.p, oa.data(), sizeof(double) * na,
                                  cudaMemcpyHostToDevice, s));
  PXST_CHECK_CUDA(cudaMemcpyAsync(offs.as<double>() + na, ob.data(), sizeof(double) * nb,
                                  cudaMemcpyHostToDevice, s));
  const double* d_oa = offs.as<double>();
  const double* d_ob = d_oa + na;

  TransArgs a{};
  a.sc = *sc;
  a.u = u; a.di = di; a.dj = dj;
  a.fm = ref->fm; a.valid = ref->valid;
  a.os = ref->os; a.of = ref->of; a.n0 = ref->n0; a.m0 = ref->m0;
  a.na_full = na; a.nb_full = nb;

  // Phase decomposition of the (sub-pixel) grid into integer sub-grids.
  const int qa = steps_per_pixel(subpixel_step), qb = qa;
  bool fast = qa > 0 && !force_generic();
  const int kha = (na - 1) / 2, khb = (nb - 1) / 2;
  struct Phase { int rho_a, rho_b, mlo_a, mhi_a, mlo_b, mhi_b; TrKernel fn; };
  std::vector<Phase> phases;
  if (fast) {
    for (int ra_ = 0; ra_ < qa && fast; ++ra_)
      for (int rb_ = 0; rb_ < qb && fast; ++rb_) {
        // k = q*m + rho in [-kh, kh]
        auto mrange = [](int q, int rho, int kh, int& lo, int& hi) {
          lo = static_cast<int>(ceil((-kh - rho) / static_cast<double>(q)));
          hi = static_cast<int>(floor((kh - rho) / static_cast<double>(q)));
        };
        Phase ph{ra_, rb_, 0, 0, 0, 0, nullptr};
        mrange(qa, ra_, kha, ph.mlo_a, ph.mhi_a);
        mrange(qb, rb_, khb, ph.mlo_b, ph.mhi_b);
        if (ph.mhi_a < ph.mlo_a || ph.mhi_b < ph.mlo_b) continue;
        ph.fn = find_tr(ph.mhi_a - ph.mlo_a + 1, ph.mhi_b - ph.mlo_b + 1);
        if (!ph.fn) fast = false;
        phases.push_back(ph);
      }
  }

  const int64_t n_search = frame_hi - frame_lo;
  if (fast) {
    const int64_t n_bands = (rw + kTrBand - 1) / kTrBand;
    Scratch mm, pvbuf, pvtmp;
    if (int e = mm.alloc(sizeof(double) * 4 * n_bands, s)) return e;
    k_band_mm<<<(unsigned)n_bands, 256, 0, s>>>(*sc, u, kTrBand, mm.as<double>());
    PXST_CHECK_LAUNCH();
    // union patch box over phases, relative to floor(x_rho): rows
    // [-max mhi, -min mlo + 1]
    int mhi_a = -1 << 20, mlo_a = 1 << 20, mhi_b = -1 << 20, mlo_b = 1 << 20;
    for (const auto& ph : phases) {
      mhi_a = max(mhi_a, ph.mhi_a); mlo_a = min(mlo_a, ph.mlo_a);
      mhi_b = max(mhi_b, ph.mhi_b); mlo_b = min(mlo_b, ph.mlo_b);
    }
    if (int e = pvbuf.alloc(ref->os * ref->of, s)) return e;
    if (int e = make_pv(ref, -mhi_a, -mlo_a + 1, -mhi_b, -mlo_b + 1, pvbuf.as<uint8_t>(), pvtmp,
                        s))
      return e;
    a.pv = pvbuf.as<uint8_t>();
    a.band_mm = mm.as<double>();
    a.n_bands = n_bands;
    a.q_a = qa; a.q_b = qb; a.kh_a = kha; a.kh_b = khb;
    // window: band footprint (~0.8 x 16 rows) x full width, capped at 96 KB
    a.win_cap = 96 * 1024 / 4;
    const size_t smem = sizeof(float) * a.win_cap;
    // frame chunks so the partial buffer stays <= 256 MB
    int64_t chunk = (256ll << 20) / (4 * n_bands * nk);
    if (chunk < 1) chunk = 1;
    if (chunk > kMaxGridY) chunk = kMaxGridY;
    Scratch part;
    if (int e = part.alloc(sizeof(float) * min(chunk, n_search) * n_bands * nk, s)) return e;
    a.partial = part.as<float>();
    for (const auto& ph : phases)
      PXST_CHECK_CUDA(cudaFuncSetAttribute(ph.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    for (int64_t c0 = frame_lo; c0 < frame_hi; c0 += chunk) {
      const int64_t c1 = min(frame_hi, c0 + chunk);
      a.frame_lo = c0;
      for (const auto& ph : phases) {
        a.rho_a = ph.rho_a; a.rho_b = ph.rho_b;
        a.mhi_a = ph.mhi_a; a.mhi_b = ph.mhi_b;
        a.ph_a = subpixel_step > 0.0 ? subpixel_step * ph.rho_a : 0.0;
        a.ph_b = subpixel_step > 0.0 ? subpixel_step * ph.rho_b : 0.0;
        dim3 g((unsigned)n_bands, (unsigned)(c1 - c0));
        ph.fn<<<g, kTrThreads, smem, s>>>(a);
        PXST_CHECK_LAUNCH();
      }
      k_trans_epilogue<float><<<(unsigned)(c1 - c0), 256, sizeof(double) * nk, s>>>(
          *sc, st->frame_norm, part.as<float>(), n_bands, c0, na, nb, d_oa, d_ob, di, dj,
          di_out, dj_out, err_out ? err_out + (c0 - frame_lo) * nk : nullptr);
      PXST_CHECK_LAUNCH();
    }
    return PXST_OK;
  }
  // generic path
  int64_t chunk = (256ll << 20) / (8 * (int64_t)nk);
  if (chunk < 1) chunk = 1;
  if (chunk > kMaxGridY) chunk = kMaxGridY;
  Scratch errs;
  if (int e = errs.alloc(sizeof(double) * min(chunk, n_search) * nk, s)) return e;
  for (int64_t c0 = frame_lo; c0 < frame_hi; c0 += chunk) {
    const int64_t c1 = min(frame_hi, c0 + chunk);
    a.frame_lo = c0;
    dim3 g((unsigned)nk, (unsigned)(c1 - c0));
    k_trans_generic<<<g, 256, 0, s>>>(a, d_oa, d_ob, errs.as<double>());
    PXST_CHECK_LAUNCH();
    k_trans_epilogue<double><<<(unsigned)(c1 - c0), 256, sizeof(double) * nk, s>>>(
        *sc, st->frame_norm, errs.as<double>(), 1, c0, na, nb, d_oa, d_ob, di, dj, di_out,
        dj_out, err_out ? err_out + (c0 - frame_lo) * nk : nullptr);
    PXST_CHECK_LAUNCH();
  }
  return PXST_OK;
}
