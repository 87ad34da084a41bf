// K2 pixel-map grid search and K3 translation grid search.
//
// Reference: recon.py:144-170 (_candidate_errors), :183-207 (_refine_batch),
// :221-296 (update_pixel_map), :336-385 (update_translations),
// interp.py:53-85 (masked bilinear read).
//
// Design:
//  * For integer offsets the fractional part of u - delta - origin is the
//    same for every trial, so each (frame, pixel) sample splits
//    once into an exact integer base (float64 floor) and float32 fractions,
//    and the whole (Ka x Kb) window is evaluated from one (Ka+1) x (Kb+1)
//    patch of the object.
//  * The patch is walked row by row: each row is interpolated along fs once
//    (h = (1-fy) o_b + fy o_{b+1}), and every trial is then
//        r = I - A h_prev - B h_cur,  acc += r*r     (A = W(1-fx), B = W fx)
//    i.e. 3 FFMA per trial plus 2(Ka+1)Kb/(KaKb) for the rows.
//    The Ka x Kb accumulators live in registers (169 at R=6).
//  * Per frame, the CTA stages the object window covering its pixel tile's
//    footprint (shifted by delta_n) in shared memory with cp.async, double
//    buffered; the per-sample "fast" path reads only shared memory.
//  * A sample whose patch leaves the grid or touches an invalid cell
//    (wsum == 0) takes the exact slow path: masked renormalised read with the
//    reference's inclusive inside test and (I - W)^2 fallback, per trial,
//    from global memory.  This is rare (< 1 % of samples) and keeps results
//    identical in semantics to the reference.
//  * Epilogue in registers: first-occurrence argmin (strict <, row-major
//    flat index a*Kb + b as numpy), 3x3 paraboloid in float64 on the
//    normalised errors, static-pixel rule.
#include "common.cuh"

#include <vector>

namespace pxst {

int check_scan(const pxst_scan* sc);

namespace {

// ----------------------------------------------------------------------------
// cp.async helpers
// ----------------------------------------------------------------------------
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

// Stage the [wr0, wr0+WR) x [wc0, wc0+WC) window of fm into smem (row stride
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

// ----------------------------------------------------------------------------
// trial engines
// ----------------------------------------------------------------------------
// Fast path: whole (KA+1) x (KB+1) patch valid and inside; `win` points at the
// patch origin in shared memory.  acc[t][s] += (I - W * bilinear)^2 for the
// trial whose base cell is (patch row t, patch col s).
template <int KA, int KB>
__device__ __forceinline__ void engine_fast(const float* __restrict__ win, int ld, float fx,
                                            float fy, float A, float B, float I,
                                            float (&acc)[KA][KB]) {
  const float gy = 1.f - fy;
  float hp[KB];
  {
    float o[KB + 1];
#pragma unroll
    for (int s = 0; s <= KB; ++s) o[s] = win[s];
#pragma unroll
    for (int s = 0; s < KB; ++s) hp[s] = fmaf(fy, o[s + 1], gy * o[s]);
  }
#pragma unroll
  for (int t = 0; t < KA; ++t) {
    const float* rp = win + (t + 1) * ld;
    float o[KB + 1], hc[KB];
#pragma unroll
    for (int s = 0; s <= KB; ++s) o[s] = rp[s];
#pragma unroll
    for (int s = 0; s < KB; ++s) hc[s] = fmaf(fy, o[s + 1], gy * o[s]);
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      float r = fmaf(-A, hp[s], I);
      r = fmaf(-B, hc[s], r);
      acc[t][s] = fmaf(r, r, acc[t][s]);
    }
#pragma unroll
    for (int s = 0; s < KB; ++s) hp[s] = hc[s];
  }
}

// Exact slow path for one sample: per trial, masked renormalised bilinear
// read (interp.py:53-85) from global memory, inclusive inside test, and the
// (I - W)^2 fallback for invalid trials (recon.py:150, 161).  `fwv` is the
// sample's frame weight (1 without weights).
template <int KA, int KB>
__device__ __forceinline__ void engine_slow(const float* __restrict__ fm,
                                            const uint8_t* __restrict__ valid, int64_t os,
                                            int64_t of, int pr, int pc, double fx, double fy,
                                            float W, float I, float fwv, float (&acc)[KA][KB]) {
  const float d0 = I - W;
  const float fb = fwv * (d0 * d0);
#pragma unroll
  for (int t = 0; t < KA; ++t) {
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      float v;
      float add = fb;
      if (masked_read(fm, valid, os, of, pr + t, pc + s, fx, fy, v)) {
        const float r = fmaf(-W, v, I);
        add = fwv * (r * r);
      }
      acc[t][s] += add;
    }
  }
}

// float64 3x3 least-squares paraboloid (recon.py:183-207); e is row-major
// [ss offset -1,0,1][fs offset -1,0,1].
__device__ __forceinline__ void paraboloid(const double (&e)[9], double& dss, double& dfs) {
  double s0 = 0, sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const double X = static_cast<double>(q / 3 - 1), Y = static_cast<double>(q % 3 - 1);
    s0 += e[q];
    sx += e[q] * X;
    sy += e[q] * Y;
    sxx += e[q] * (X * X);
    syy += e[q] * (Y * Y);
    sxy += e[q] * (X * Y);
  }
  const double b = sx / 6.0, c = sy / 6.0, f = sxy / 4.0;
  const double d = (-2.0 * s0 + 3.0 * sxx) / 6.0;
  const double g = (-2.0 * s0 + 3.0 * syy) / 6.0;
  const double det = 4.0 * d * g - f * f;
  if (d > 0.0 && det > 0.0) {
    dss = fmin(fmax((-2.0 * g * b + f * c) / det, -1.0), 1.0);
    dfs = fmin(fmax((-2.0 * d * c + f * b) / det, -1.0), 1.0);
  } else {
    dss = 0.0;
    dfs = 0.0;
  }
}

// ----------------------------------------------------------------------------
// patch-valid map: pv[i][j] = every cell of rows [i+lr, i+hr] x cols
// [j+lc, j+hc] exists and is valid.  Two separable passes.
// ----------------------------------------------------------------------------
__global__ void k_pv_rows(const uint8_t* __restrict__ valid, int64_t os, int64_t of, int lc,
                          int hc, uint8_t* __restrict__ tmp) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < os * of;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / of, j = q % of;
    uint8_t ok = (j + lc >= 0 && j + hc < of) ? 1 : 0;
    for (int c = lc; ok && c <= hc; ++c) ok = valid[i * of + j + c];
    tmp[q] = ok;
  }
}
__global__ void k_pv_cols(const uint8_t* __restrict__ tmp, int64_t os, int64_t of, int lr,
                          int hr, uint8_t* __restrict__ pv) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < os * of;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / of, j = q % of;
    uint8_t ok = (i + lr >= 0 && i + hr < os) ? 1 : 0;
    for (int r = lr; ok && r <= hr; ++r) ok = tmp[(i + r) * of + j];
    pv[q] = ok;
  }
}

int make_pv(const pxst_ref* ref, int lr, int hr, int lc, int hc, uint8_t* pv, Scratch& tmp,
            cudaStream_t s) {
  const int64_t n = ref->os * ref->of;
  if (int e = tmp.alloc(n, s)) return e;
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  k_pv_rows<<<(unsigned)b, 256, 0, s>>>(ref->valid, ref->os, ref->of, lc, hc, tmp.as<uint8_t>());
  PXST_CHECK_LAUNCH();
  k_pv_cols<<<(unsigned)b, 256, 0, s>>>(tmp.as<uint8_t>(), ref->os, ref->of, lr, hr, pv);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

// ----------------------------------------------------------------------------
// K2: pixel-map search (integer window), fast engine.
// ----------------------------------------------------------------------------
constexpr int kPixTR = 4, kPixTC = 32, kPixThreads = kPixTR * kPixTC;

struct PixArgs {
  pxst_scan sc;
  const double* u;
  const double* di;
  const double* dj;
  const float* fm;
  const uint8_t* valid;
  const uint8_t* pv;
  int64_t os, of, n0, m0;
  const float* fw;      // nullable
  const double* var;    // normaliser [ss*fs]
  double* u_out;
  double* err_out;
  int refine;
  int win_cap;          // floats per window buffer
};

__device__ __forceinline__ int clamp_span(double v) {
  return v < 0.0 ? 0 : (v > 4096.0 ? 4096 : static_cast<int>(v));
}

template <int KA, int KB>
__global__ void __launch_bounds__(kPixThreads, 2) k_pixel_search(PixArgs a) {
  constexpr int RA = (KA - 1) / 2, RB = (KB - 1) / 2;
  extern __shared__ float smem[];
  __shared__ double red[4][4];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = a.sc.roi[0] + (int64_t)blockIdx.y * kPixTR + warp;
  const int64_t col = a.sc.roi[2] + (int64_t)blockIdx.x * kPixTC + lane;
  const bool inroi = row < a.sc.roi[1] && col < a.sc.roi[3];
  const int64_t p = inroi ? row * a.sc.fs + col : 0;
  const bool live = inroi && a.sc.work[p] != 0;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const double u0 = live ? a.u[p] : 0.0, u1 = live ? a.u[plane + p] : 0.0;

  // Block bounding box of u over live pixels (fixes the window geometry).
  double mn0 = warp_min(live ? u0 : INFINITY), mx0 = warp_max(live ? u0 : -INFINITY);
  double mn1 = warp_min(live ? u1 : INFINITY), mx1 = warp_max(live ? u1 : -INFINITY);
  if (lane == 0) { red[warp][0] = mn0; red[warp][1] = mx0; red[warp][2] = mn1; red[warp][3] = mx1; }
  __syncthreads();
  mn0 = red[0][0]; mx0 = red[0][1]; mn1 = red[0][2]; mx1 = red[0][3];
#pragma unroll
  for (int w = 1; w < kPixTR; ++w) {
    mn0 = fmin(mn0, red[w][0]); mx0 = fmax(mx0, red[w][1]);
    mn1 = fmin(mn1, red[w][2]); mx1 = fmax(mx1, red[w][3]);
  }
  if (!(mn0 <= mx0)) return;  // no live pixel in this tile (uniform)
  const int WR = clamp_span(floor(mx0 - mn0)) + KA + 2;
  const int WC = clamp_span(floor(mx1 - mn1)) + KB + 2;
  const bool use_win = WR * WC <= a.win_cap && isfinite(mn0) && isfinite(mn1) &&
                       fabs(mn0) < 1e9 && fabs(mn1) < 1e9;
  float* buf0 = smem;
  float* buf1 = smem + a.win_cap;
  const double n0d = static_cast<double>(a.n0), m0d = static_cast<double>(a.m0);

  const float W = live ? a.sc.w32[p] : 0.f;
  float acc[KA][KB];
#pragma unroll
  for (int t = 0; t < KA; ++t)
#pragma unroll
    for (int s = 0; s < KB; ++s) acc[t][s] = 0.f;

  const int64_t K = a.sc.n_good;
  if (use_win) {
    const int64_t f = a.sc.good[0];
    stage_window(buf0, a.fm, a.os, a.of,
                 static_cast<int>(floor(mn0 - a.di[f] - n0d)) - RA,
                 static_cast<int>(floor(mn1 - a.dj[f] - m0d)) - RB, WR, WC);
  }
  cp_async_commit();
  float I_next = live ? __ldg(a.sc.frames + (int64_t)a.sc.good[0] * plane + p) : 0.f;

  for (int64_t k = 0; k < K; ++k) {
    const int64_t f = a.sc.good[k];
    float* cur = (k & 1) ? buf1 : buf0;
    const float I = I_next;
    if (k + 1 < K) {
      const int64_t fn = a.sc.good[k + 1];
      if (use_win)
        stage_window((k & 1) ? buf0 : buf1, a.fm, a.os, a.of,
                     static_cast<int>(floor(mn0 - a.di[fn] - n0d)) - RA,
                     static_cast<int>(floor(mn1 - a.dj[fn] - m0d)) - RB, WR, WC);
      if (live) I_next = __ldg(a.sc.frames + fn * plane + p);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (live) {
      const double dI = a.di[f], dJ = a.dj[f];
      const double x = u0 - dI - n0d;                 // recon.py:148
      const double y = u1 - dJ - m0d;
      const double xf = floor(x), yf = floor(y);
      const double fxd = x - xf, fyd = y - yf;
      const bool finite = fabs(x) < 1e9 && fabs(y) < 1e9;
      const int i = finite ? static_cast<int>(xf) : -(1 << 30);
      const int j = finite ? static_cast<int>(yf) : -(1 << 30);
      float fwv = 1.f;
      if (a.fw) fwv = __ldg(a.fw + f * plane + p);
      bool fast = use_win && fwv >= 0.f && i >= 0 && i < a.os && j >= 0 && j < a.of &&
                  a.pv[(int64_t)i * a.of + j] != 0;
      const int wr0 = static_cast<int>(floor(mn0 - dI - n0d)) - RA;
      const int wc0 = static_cast<int>(floor(mn1 - dJ - m0d)) - RB;
      const int lr = i - RA - wr0, lc = j - RB - wc0;
      fast = fast && lr >= 0 && lr + KA + 1 <= WR && lc >= 0 && lc + KB + 1 <= WC;
      if (fast) {
        const float fx = static_cast<float>(fxd), fy = static_cast<float>(fyd);
        float sI = I, sW = W;
        if (a.fw) {
          const float sq = sqrtf(fwv);
          sI *= sq;
          sW *= sq;
        }
        engine_fast<KA, KB>(cur + lr * WC + lc, WC, fx, fy, sW * (1.f - fx), sW * fx, sI, acc);
      } else {
        engine_slow<KA, KB>(a.fm, a.valid, a.os, a.of, i - RA, j - RB, fxd, fyd, W, I, fwv,
                            acc);
      }
    }
    __syncthreads();
  }
  if (!live) return;

  // ---- epilogue: normalise, argmin (first occurrence), refine, write ----
  const double var = a.var[p];
  const bool active = var > 0.0;
  float best = acc[0][0];
  int bt = 0, bs = 0;
#pragma unroll
  for (int t = 0; t < KA; ++t)
#pragma unroll
    for (int s = 0; s < KB; ++s)
      if (acc[t][s] < best) { best = acc[t][s]; bt = t; bs = s; }
  double sh_ss = static_cast<double>(bt - RA), sh_fs = static_cast<double>(bs - RB);
  if (KA >= 3 && KB >= 3 && a.refine && active && bt > 0 && bt < KA - 1 && bs > 0 &&
      bs < KB - 1) {
    float r0[KB], r1[KB], r2[KB];
#pragma unroll
    for (int s = 0; s < KB; ++s) { r0[s] = 0.f; r1[s] = 0.f; r2[s] = 0.f; }
#pragma unroll
    for (int t = 0; t < KA; ++t) {
#pragma unroll
      for (int s = 0; s < KB; ++s) {
        // The opaque copy stops the optimiser from turning this select chain
        // into a dynamically indexed load, which would demote acc[][] to
        // local memory for the whole kernel.
        float v = acc[t][s];
        asm("" : "+f"(v));
        r0[s] = (t == bt - 1) ? v : r0[s];
        r1[s] = (t == bt) ? v : r1[s];
        r2[s] = (t == bt + 1) ? v : r2[s];
      }
    }
    double e[9];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
      for (int s = 0; s < KB; ++s) {
        const bool m = (s == bs - 1 + d);
        float v0 = r0[s], v1 = r1[s], v2 = r2[s];
        asm("" : "+f"(v0), "+f"(v1), "+f"(v2));
        c0 = m ? v0 : c0;
        c1 = m ? v1 : c1;
        c2 = m ? v2 : c2;
      }
      e[d] = c0;
      e[3 + d] = c1;
      e[6 + d] = c2;
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) e[q] /= var;
    double dss, dfs;
    paraboloid(e, dss, dfs);
    sh_ss += dss;
    sh_fs += dfs;
  }
  if (!active) { sh_ss = 0.0; sh_fs = 0.0; }     // recon.py:289-292
  a.u_out[p] = u0 + sh_ss;                       // recon.py:294-296
  a.u_out[plane + p] = u1 + sh_fs;
  a.err_out[p] = active ? static_cast<double>(best) / var : 0.0;
}

// ----------------------------------------------------------------------------
// Generic K2 (any window, sub-pixel grids): one thread per (pixel, trial),
// float64, straight restatement of recon.py:144-170.  Writes the raw error
// stack errs[t][q] for the ROI rectangle q; the epilogue kernel finishes.
// ----------------------------------------------------------------------------
__global__ void k_pixel_generic(PixArgs a, const double* __restrict__ offs_a,
                                const double* __restrict__ offs_b, int na, int nb,
                                double* __restrict__ errs) {
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2], rw = a.sc.roi[1] - a.sc.roi[0];
  const int64_t nq = cw * rw;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (q >= nq) return;
  const int64_t p = (a.sc.roi[0] + q / cw) * a.sc.fs + a.sc.roi[2] + q % cw;
  if (!a.sc.work[p]) return;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const double u0 = a.u[p], u1 = a.u[plane + p];
  const double W = a.sc.w64[p];
  const double oa = offs_a[t / nb], ob = offs_b[t % nb];
  double acc = 0.0;
  for (int64_t k = 0; k < a.sc.n_good; ++k) {
    const int64_t f = a.sc.good[k];
    const double I = static_cast<double>(__ldg(a.sc.frames + f * plane + p));
    const double fwv = a.fw ? static_cast<double>(__ldg(a.fw + f * plane + p)) : 1.0;
    const double x = (u0 - a.di[f] - a.n0) + oa;
    const double y = (u1 - a.dj[f] - a.m0) + ob;
    float v = 0.f;
    bool ok = false;
    if (fabs(x) < 1e9 && fabs(y) < 1e9) {
      const Split sx = split(x), sy = split(y);
      ok = masked_read(a.fm, a.valid, a.os, a.of, sx.i, sy.i, sx.f, sy.f, v);
    }
    const double r = ok ? I - W * static_cast<double>(v) : I - W;
    acc += fwv * (r * r);
  }
  errs[(int64_t)t * nq + q] = acc;
}

__global__ void k_pixel_generic_epilogue(PixArgs a, const double* __restrict__ offs_a,
                                         const double* __restrict__ offs_b, int na, int nb,
                                         int refine_ok, const double* __restrict__ errs) {
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2], rw = a.sc.roi[1] - a.sc.roi[0];
  const int64_t nq = cw * rw;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int64_t p = (a.sc.roi[0] + q / cw) * a.sc.fs + a.sc.roi[2] + q % cw;
  if (!a.sc.work[p]) return;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const double var = a.var[p];
  const bool active = var > 0.0;
  const double nv = active ? var : 1.0;
  int best = 0;
  double bv = errs[q] / nv;
  for (int t = 1; t < na * nb; ++t) {
    const double v = errs[(int64_t)t * nq + q] / nv;
    if (v < bv) { bv = v; best = t; }
  }
  const int ia = best / nb, ib = best % nb;
  double sh_ss = offs_a[ia], sh_fs = offs_b[ib];
  if (refine_ok && active && ia > 0 && ia < na - 1 && ib > 0 && ib < nb - 1) {
    double e[9];
    for (int d = 0; d < 9; ++d)
      e[d] = errs[(int64_t)((ia + d / 3 - 1) * nb + (ib + d % 3 - 1)) * nq + q] / nv;
    double dss, dfs;
    paraboloid(e, dss, dfs);
    sh_ss += dss;
    sh_fs += dfs;
  }
  if (!active) { sh_ss = 0.0; sh_fs = 0.0; }
  a.u_out[p] = a.u[p] + sh_ss;
  a.u_out[plane + p] = a.u[plane + p] + sh_fs;
  a.err_out[p] = active ? bv : 0.0;
}

// ----------------------------------------------------------------------------
// K3: translation search.  One CTA per (searched frame, band of detector
// rows); threads stride over the band's pixels accumulating the phase
// group's Ka x Kb window in registers, then a deterministic CTA reduction
// writes float32 partials[frame][band][full grid index].
// ----------------------------------------------------------------------------
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
// dispatch tables
// ----------------------------------------------------------------------------
using PixKernel = void (*)(PixArgs);
using TrKernel = void (*)(TransArgs);

struct PixEntry { int ka, kb; PixKernel fn; };
struct TrEntry { int ka, kb; TrKernel fn; };

#define PIX(a, b) PixEntry{a, b, k_pixel_search<a, b>}
const PixEntry kPixTable[] = {
    PIX(1, 1),  PIX(3, 3),  PIX(5, 5),  PIX(7, 7),  PIX(9, 9),  PIX(11, 11), PIX(13, 13),
    PIX(1, 3),  PIX(1, 5),  PIX(1, 7),  PIX(1, 9),  PIX(1, 11), PIX(1, 13),  PIX(1, 15),
    PIX(1, 17), PIX(3, 1),  PIX(5, 1),  PIX(7, 1),  PIX(9, 1),  PIX(11, 1),  PIX(13, 1),
    PIX(15, 1), PIX(17, 1),
};
#undef PIX
#define TR(a, b) TrEntry{a, b, k_trans_partial<a, b>}
const TrEntry kTrTable[] = {
    TR(1, 1), TR(3, 3), TR(5, 5), TR(7, 7), TR(9, 9), TR(11, 11), TR(13, 13),
    TR(8, 8), TR(8, 9), TR(9, 8), TR(9, 9),
};
#undef TR

PixKernel find_pix(int ka, int kb) {
  for (const auto& e : kPixTable)
    if (e.ka == ka && e.kb == kb) return e.fn;
  return nullptr;
}
TrKernel find_tr(int ka, int kb) {
  for (const auto& e : kTrTable)
    if (e.ka == ka && e.kb == kb) return e.fn;
  return nullptr;
}

bool force_generic() {
  const char* v = getenv("PXST_FORCE_GENERIC");
  return v && v[0] == '1';
}

// Offsets of SearchWindow.offsets (recon.py:51-57).
std::vector<double> window_offsets(int64_t half, double step) {
  std::vector<double> o;
  if (step <= 0.0) {
    for (int64_t k = -half; k <= half; ++k) o.push_back(static_cast<double>(k));
  } else {
    const int64_t kh = static_cast<int64_t>(llround(static_cast<double>(half) / step));
    for (int64_t k = -kh; k <= kh; ++k) o.push_back(step * static_cast<double>(k));
  }
  return o;
}

int check_ref(const pxst_ref* r) {
  PXST_REQUIRE(r && r->fm && r->valid && r->os > 0 && r->of > 0, "bad reference image");
  PXST_REQUIRE(r->os * r->of < (int64_t(1) << 31), "reference image too large");
  return PXST_OK;
}

// Integer steps per pixel for a sub-pixel grid, or 0 when 1/step is not an
// integer (then only the generic kernels apply).
int steps_per_pixel(double step) {
  if (step <= 0.0) return 1;
  const double q = 1.0 / step;
  const double qr = nearbyint(q);
  if (qr >= 1.0 && qr <= 16.0 && fabs(q - qr) < 1e-9 && fabs(step * qr - 1.0) < 1e-12)
    return static_cast<int>(qr);
  return 0;
}

}  // namespace
}  // namespace pxst

using namespace pxst;

extern "C" int pxst_pixel_map_search(const pxst_scan* sc, const pxst_stats* st,
                                     const pxst_ref* ref, const double* u_in, const double* di,
                                     const double* dj, int64_t half_ss, int64_t half_fs,
                                     double subpixel_step, int refine, const float* fw,
                                     const double* var_fw, double* u_out, double* err_out,
                                     void* stream) {
  if (int e = check_scan(sc)) return e;
  if (int e = check_ref(ref)) return e;
  PXST_REQUIRE(st && st->var_pm, "stats descriptor is NULL");
  PXST_REQUIRE(u_in && di && dj && u_out && err_out, "NULL pointer");
  PXST_REQUIRE(half_ss >= 0 && half_fs >= 0, "search window halves must be >= 0");
  PXST_REQUIRE(subpixel_step == 0.0 || (subpixel_step > 0.0 && subpixel_step <= 1.0),
               "subpixel_grid step must be in (0, 1]");
  PXST_REQUIRE(!fw || var_fw, "frame weights need their normaliser var_fw");
  cudaStream_t s = as_stream(stream);
  const int64_t plane = sc->ss * sc->fs;
  PXST_CHECK_CUDA(cudaMemcpyAsync(u_out, u_in, sizeof(double) * 2 * plane,
                                  cudaMemcpyDeviceToDevice, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(err_out, 0, sizeof(double) * plane, s));
  if (sc->n_good == 0) return PXST_OK;

  PixArgs a{};
  a.sc = *sc;
  a.u = u_in; a.di = di; a.dj = dj;
  a.fm = ref->fm; a.valid = ref->valid;
  a.os = ref->os; a.of = ref->of; a.n0 = ref->n0; a.m0 = ref->m0;
  a.fw = fw;
  a.var = fw ? var_fw : st->var_pm;
  a.u_out = u_out; a.err_out = err_out;
  a.refine = refine;

  const std::vector<double> oa = window_offsets(half_ss, subpixel_step);
  const std::vector<double> ob = window_offsets(half_fs, subpixel_step);
  const int na = static_cast<int>(oa.size()), nb = static_cast<int>(ob.size());
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];

  PixKernel fn = (subpixel_step == 0.0 && !force_generic()) ? find_pix(na, nb) : nullptr;
  if (fn) {
    const int ra = (na - 1) / 2, rb = (nb - 1) / 2;
    Scratch pvbuf, pvtmp;
    if (int e = pvbuf.alloc(ref->os * ref->of, s)) return e;
    if (int e = make_pv(ref, -ra, ra + 1, -rb, rb + 1, pvbuf.as<uint8_t>(), pvtmp, s)) return e;
    a.pv = pvbuf.as<uint8_t>();
    // window buffer: room for a tile footprint up to ~2x magnification
    a.win_cap = (2 * kPixTR + na + 6) * (2 * kPixTC + nb + 6);
    const size_t smem = sizeof(float) * 2 * a.win_cap;
    PXST_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    dim3 g((unsigned)((cw + kPixTC - 1) / kPixTC), (unsigned)((rw + kPixTR - 1) / kPixTR));
    PXST_REQUIRE(g.y <= kMaxGridY, "ROI too tall");
    fn<<<g, kPixThreads, smem, s>>>(a);
    PXST_CHECK_LAUNCH();
    return PXST_OK;
  }
  // generic path
  const int64_t nq = cw * rw;
  Scratch offs, errs;
  if (int e = offs.alloc(sizeof(double) * (na + nb), s)) return e;
  PXST_CHECK_CUDA(cudaMemcpyAsync(offs.p, oa.data(), sizeof(double) * na,
                                  cudaMemcpyHostToDevice, s));
  PXST_CHECK_CUDA(cudaMemcpyAsync(offs.as<double>() + na, ob.data(), sizeof(double) * nb,
                                  cudaMemcpyHostToDevice, s));
  if (int e = errs.alloc(sizeof(double) * nq * na * nb, s)) return e;
  PXST_REQUIRE(na * nb <= kMaxGridY, "search window too large");
  dim3 g((unsigned)((nq + 127) / 128), (unsigned)(na * nb));
  k_pixel_generic<<<g, 128, 0, s>>>(a, offs.as<double>(), offs.as<double>() + na, na, nb,
                                    errs.as<double>());
  PXST_CHECK_LAUNCH();
  const int refine_ok = refine && subpixel_step == 0.0 && na >= 3 && nb >= 3;  // recon.py:273
  k_pixel_generic_epilogue<<<(unsigned)((nq + 127) / 128), 128, 0, s>>>(
      a, offs.as<double>(), offs.as<double>() + na, na, nb, refine_ok, errs.as<double>());
  PXST_CHECK_LAUNCH();
  // CUDA stream-ordered frees of offs/errs happen after the kernels.
  cudaError_t e = cudaGetLastError();
  (void)e;
  return PXST_OK;
}

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
