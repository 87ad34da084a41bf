// Shared pieces of the grid-search kernels (K2 pixel map, K3 translations).
//
// Reference: recon.py:144-170 (_candidate_errors), :183-207 (_refine_batch),
// interp.py:53-85 (masked bilinear read).
//
// Trial engine: for integer offsets the fractional part of
// u - delta - origin is the same for every trial, so one (frame, pixel)
// sample splits once into an exact integer base (float64 floor) and float32
// fractions, and the whole Ka x Kb window is evaluated from a single
// (Ka+1) x (Kb+1) patch of the object.  The patch is walked row by row: each
// row is interpolated along fs once (h = (1-fy) o_b + fy o_{b+1}) and every
// trial is
//     r = I - A h_prev - B h_cur,  acc += r*r        (A = W(1-fx), B = W fx)
// i.e. 3 FFMA per trial + 2 (Ka+1) Kb / (Ka Kb) per trial for the rows.
#pragma once

#include <vector>

#include "common.cuh"

namespace pxst {

// ---------------------------------------------------------------------------
// Packed (FFMA2) engine.  sm_100 executes fma.rn.f32x2 at the full FP32 rate
// with half the issue slots (measured 73.8 TFLOP/s, profiles/microbench_r01.json).
//
// Two changes to the plain engine above cut its FP32 work per trial from
// ~5.2 to ~4.1 lane operations and its issue slots by a third:
//  * Row interpolation in one FMA.  h = gy o_b + fy o_{b+1} (gy = 1 - fy) is
//    carried as h' = o_b + rho o_{b+1} with rho = fy / gy (MUFU reciprocal,
//    ~1 ulp: it scales the o_{b+1} term only) and the factor gy
//    folded into the trial weights (A' = A gy, B' = B gy), so every trial is
//    still r = I - A' h'_prev - B' h'_cur = I - A h_prev - B h_cur.  fy is
//    kept <= 1 - 2^-24, so gy > 0; the relative rounding of A' h' matches
//    that of A h (h' is one fused rounding, the gy scale one more).
//  * Trial columns paired at a distance H = ceil(KB / 2): the register pair k
//    holds trials (t, k) and (t, k + H).  The patch row then packs as
//    Q_k = (o_k, o_{k+H}) with every value in exactly one register, and the
//    row's h' pairs are one FFMA2 each, h'_(k, k+H) = Q_k + rho Q_{k+1}
//    (the plain (2k, 2k+1) pairing needs the misaligned pair (o_{2k+1},
//    o_{2k+2})).
// ---------------------------------------------------------------------------
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(f32x2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// MUFU reciprocal, flush-to-zero (~1 ulp).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// MUFU square root (frame weights of the split-half path).
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int KA, int KB>
struct PackedAcc {
  static constexpr int H = (KB + 1) / 2;      // pair distance
  static constexpr int NP = KB / 2;           // register pairs per trial row
  static constexpr bool ODD = (KB % 2) != 0;  // single column NP (= H - 1)
  f32x2 p[KA][NP > 0 ? NP : 1];
  float s[KA];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int t = 0; t < KA; ++t) {
#pragma unroll
      for (int k = 0; k < NP; ++k) p[t][k] = 0ull;
      s[t] = 0.f;
    }
  }
  __device__ __forceinline__ float get(int t, int c) const {  // t, c compile-time in loops
    if (ODD && c == NP) return s[t];
    float lo, hi;
    unpack2(p[t][c < NP ? c : c - H], lo, hi);
    return c < NP ? lo : hi;
  }
};

// One patch row: o_0 .. o_KB packed as Q_k = (o_k, o_{k+H}) (+ o_KB alone when
// KB is even), and its h' values in the accumulator layout.
template <int KB>
struct PatchRow {
  static constexpr int H = (KB + 1) / 2, NP = KB / 2;
  static constexpr bool ODD = (KB % 2) != 0;
  f32x2 h[NP > 0 ? NP : 1];
  float hs;

  __device__ __forceinline__ void load(const float* __restrict__ rp, float rho) {
    float o[KB + 1];
#pragma unroll
    for (int c = 0; c <= KB; ++c) o[c] = rp[c];
    f32x2 q[H + 1];
#pragma unroll
    for (int k = 0; k < H; ++k) q[k] = pack2(o[k], o[k + H]);
    if (!ODD) q[H] = pack2(o[H], o[KB]);            // (o_H, o_2H) for the last pair
    const f32x2 rho2 = pack2(rho, rho);
#pragma unroll
    for (int k = 0; k < NP; ++k) h[k] = ffma2(rho2, q[k + 1], q[k]);
    hs = ODD ? fmaf(rho, o[H], o[H - 1]) : 0.f;
  }
};

template <int KA, int KB>
__device__ __forceinline__ void engine_fast2(const float* __restrict__ win, int ld, float fx,
                                             float fy, float A, float B, float I,
                                             PackedAcc<KA, KB>& acc) {
  constexpr int NP = PackedAcc<KA, KB>::NP;
  constexpr bool ODD = PackedAcc<KA, KB>::ODD;
  fy = fminf(fy, 0x1.fffffep-1f);
  const float gy = 1.f - fy;
  const float rho = fy * rcp_approx(gy);   // gy in [2^-24, 1]: no denormal path needed
  const float Ap = A * gy, Bp = B * gy;
  const f32x2 nA2 = pack2(-Ap, -Ap), nB2 = pack2(-Bp, -Bp), I2 = pack2(I, I);
  PatchRow<KB> prev, cur;
  prev.load(win, rho);
#pragma unroll
  for (int t = 0; t < KA; ++t) {
    cur.load(win + (t + 1) * ld, rho);
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      f32x2 r = ffma2(nA2, prev.h[k], I2);
      r = ffma2(nB2, cur.h[k], r);
      acc.p[t][k] = ffma2(r, r, acc.p[t][k]);
    }
    if (ODD) {
      float r = fmaf(-Ap, prev.hs, I);
      r = fmaf(-Bp, cur.hs, r);
      acc.s[t] = fmaf(r, r, acc.s[t]);
    }
    prev = cur;
  }
}

// One-row engine for KA == 1 windows when the sample's ss fraction is 0:
// the r0 + 1 corners carry zero weight (B = 0), so the second patch row and
// its half of each trial drop out (config 2: u_ss = x and no ss scan, every
// fx = 0).  Same values as engine_fast2 with B = 0.
template <int KB>
__device__ __forceinline__ void engine_row1(const float* __restrict__ win, float fy, float A,
                                            float I, PackedAcc<1, KB>& acc) {
  constexpr int NP = PackedAcc<1, KB>::NP;
  constexpr bool ODD = PackedAcc<1, KB>::ODD;
  fy = fminf(fy, 0x1.fffffep-1f);
  const float gy = 1.f - fy;
  const float rho = fy * rcp_approx(gy);
  const float Ap = A * gy;
  const f32x2 nA2 = pack2(-Ap, -Ap), I2 = pack2(I, I);
  PatchRow<KB> row;
  row.load(win, rho);
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const f32x2 r = ffma2(nA2, row.h[k], I2);
    acc.p[0][k] = ffma2(r, r, acc.p[0][k]);
  }
  if (ODD) {
    const float r = fmaf(-Ap, row.hs, I);
    acc.s[0] = fmaf(r, r, acc.s[0]);
  }
}

// ---------------------------------------------------------------------------
// Exact trials (the slow fix-up kernels), read from a float32 copy of the
// reference with NaN on invalid cells (make_pv's fmn), so one load gives value
// and validity.  Everything that is constant over a sample's trials (integer
// shifts keep its fractions) is hoisted into ExactSample; a trial then costs
// four loads and the masked renormalisation of masked_read, in the same
// float32 operation order.
// ---------------------------------------------------------------------------
struct ExactSample {
  float w00, w01, w10, w11;   // bilinear weights (masked_read's float32 formulas)
  bool fxp, fyp;              // fx > 0, fy > 0 decided on the float64 fractions
  float I, W, fwv, fb;        // fb = fwv (I - W)^2, the invalid-trial fallback
};

__device__ __forceinline__ ExactSample exact_sample(double fx, double fy, float W, float I,
                                                    float fwv) {
  ExactSample e;
  const float gx = static_cast<float>(fx), gy = static_cast<float>(fy);
  e.w00 = (1.f - gx) * (1.f - gy);
  e.w01 = (1.f - gx) * gy;
  e.w10 = gx * (1.f - gy);
  e.w11 = gx * gy;
  e.fxp = fx > 0.0;
  e.fyp = fy > 0.0;
  e.I = I;
  e.W = W;
  e.fwv = fwv;
  const float d0 = I - W;
  e.fb = fwv * (d0 * d0);
  return e;
}

// Same trial read straight from a NaN-encoded copy of the reference in
// global memory (make_pv's fmn): four independent L1/L2 loads, no staging.
// Branch-free, 32-bit cell indices (callers guarantee os * of < 2^31): the
// four loads always go to clamped in-grid cells and the reference's rules
// are applied by selects.  Corners past the last row/column carry zero
// weight and are excluded by the fx/fy flags; a base outside the grid (or a
// weighted corner past its edge) gives the (I - W)^2 fallback.
__device__ __forceinline__ float trial_global(const float* __restrict__ fmn, int os, int of,
                                              int row, int col, const ExactSample& e) {
  const bool rin = (row >= 0 && row < os - 1) || (row == os - 1 && !e.fxp);
  const bool cin = (col >= 0 && col < of - 1) || (col == of - 1 && !e.fyp);
  const int r0 = min(max(row, 0), os - 1), c0 = min(max(col, 0), of - 1);
  const int dr = r0 + 1 < os ? of : 0, dc = c0 + 1 < of ? 1 : 0;
  const float* p0 = fmn + (r0 * of + c0);
  const float v00 = __ldg(p0), v01 = __ldg(p0 + dc);
  const float v10 = __ldg(p0 + dr), v11 = __ldg(p0 + dr + dc);
  const bool m00 = v00 == v00;
  const bool m01 = e.fyp && v01 == v01;
  const bool m10 = e.fxp && v10 == v10;
  const bool m11 = e.fxp && e.fyp && v11 == v11;
  float den = m00 ? e.w00 : 0.f;
  float num = m00 ? e.w00 * v00 : 0.f;
  den += m01 ? e.w01 : 0.f;
  num = fmaf(m01 ? e.w01 : 0.f, m01 ? v01 : 0.f, num);
  den += m10 ? e.w10 : 0.f;
  num = fmaf(m10 ? e.w10 : 0.f, m10 ? v10 : 0.f, num);
  den += m11 ? e.w11 : 0.f;
  num = fmaf(m11 ? e.w11 : 0.f, m11 ? v11 : 0.f, num);
  const float r = fmaf(-e.W, __fdividef(num, den), e.I);
  const bool ok = rin && cin && (m00 || m01 || m10 || m11);
  return ok ? e.fwv * (r * r) : e.fb;
}

// trial_global for a cell whose 2x2 corners are all on the grid (the caller
// checked the whole patch): no bounds tests or clamps, identical arithmetic.
__device__ __forceinline__ float trial_interior(const float* __restrict__ p0, int of,
                                                const ExactSample& e) {
  const float v00 = __ldg(p0), v01 = __ldg(p0 + 1);
  const float v10 = __ldg(p0 + of), v11 = __ldg(p0 + of + 1);
  const bool m00 = v00 == v00;
  const bool m01 = e.fyp && v01 == v01;
  const bool m10 = e.fxp && v10 == v10;
  const bool m11 = e.fxp && e.fyp && v11 == v11;
  float den = m00 ? e.w00 : 0.f;
  float num = m00 ? e.w00 * v00 : 0.f;
  den += m01 ? e.w01 : 0.f;
  num = fmaf(m01 ? e.w01 : 0.f, m01 ? v01 : 0.f, num);
  den += m10 ? e.w10 : 0.f;
  num = fmaf(m10 ? e.w10 : 0.f, m10 ? v10 : 0.f, num);
  den += m11 ? e.w11 : 0.f;
  num = fmaf(m11 ? e.w11 : 0.f, m11 ? v11 : 0.f, num);
  const float r = fmaf(-e.W, __fdividef(num, den), e.I);
  return (m00 || m01 || m10 || m11) ? e.fwv * (r * r) : e.fb;
}

// Same trial from four corner values in registers (off-grid cells carry
// kOffGrid, a NaN with its own payload, so one value gives position, validity
// and value).  Equal to trial_global: the reference's bounds rule (row in
// [0, os-1), or os-1 with zero row weight; likewise for columns) is "base
// corner on the grid and every corner with nonzero weight on the grid".
constexpr unsigned kOffGrid = 0xffc0beefu;
__device__ __forceinline__ bool on_grid(float v) { return __float_as_uint(v) != kOffGrid; }

__device__ __forceinline__ float trial_patch(float v00, float v01, float v10, float v11,
                                             const ExactSample& e) {
  const bool in = on_grid(v00) && (!e.fxp || on_grid(v10)) && (!e.fyp || on_grid(v01));
  const bool m00 = v00 == v00;
  const bool m01 = e.fyp && v01 == v01;
  const bool m10 = e.fxp && v10 == v10;
  const bool m11 = e.fxp && e.fyp && v11 == v11;
  float den = m00 ? e.w00 : 0.f;
  float num = m00 ? e.w00 * v00 : 0.f;
  den += m01 ? e.w01 : 0.f;
  num = fmaf(m01 ? e.w01 : 0.f, m01 ? v01 : 0.f, num);
  den += m10 ? e.w10 : 0.f;
  num = fmaf(m10 ? e.w10 : 0.f, m10 ? v10 : 0.f, num);
  den += m11 ? e.w11 : 0.f;
  num = fmaf(m11 ? e.w11 : 0.f, m11 ? v11 : 0.f, num);
  const float r = fmaf(-e.W, __fdividef(num, den), e.I);
  return (in && (m00 || m01 || m10 || m11)) ? e.fwv * (r * r) : e.fb;
}




// Exact trial from the padded (value, mask) copy of the reference (fm2,
// pv_tile_block): cell = (v, m) with m = 1 valid (v = the masked float32
// value), m = 0 invalid (v = 0), m = -inf off the grid (the padding border,
// v = 0).  num = sum w v and den = sum w m are plain FMA chains in
// masked_read's corner order -- an invalid cell adds w * 0 to both, exactly
// what the select forms above add -- and den > 0 holds iff every corner with
// nonzero weight is on the grid and one of them is valid (a weighted off-grid
// corner makes den -inf, or NaN with a zero weight: both fail the test), the
// reference's rule (interp.py:67-85).  Callers alias zero-weight corners onto
// weighted ones (dr = 0 when fx == 0, dc = 0 when fy == 0).  i0 / i1 = the
// cell index of the trial's base in rows r0 / r0 + dr.
template <bool DC1>
__device__ __forceinline__ float trial_pad(const float2* __restrict__ fm2, unsigned i0,
                                           unsigned i1, int dc, const ExactSample& e) {
  // (unsigned 32-bit cell indices: one IMAD.WIDE per row pointer)
  const float2* p0 = fm2 + i0;
  const float2* p1 = fm2 + i1;
  const float2 c00 = __ldg(p0), c01 = __ldg(p0 + (DC1 ? 1 : dc));
  const float2 c10 = __ldg(p1), c11 = __ldg(p1 + (DC1 ? 1 : dc));
  float den = e.w00 * c00.y;
  float num = e.w00 * c00.x;
  den = fmaf(e.w01, c01.y, den);
  num = fmaf(e.w01, c01.x, num);
  den = fmaf(e.w10, c10.y, den);
  num = fmaf(e.w10, c10.x, num);
  den = fmaf(e.w11, c11.y, den);
  num = fmaf(e.w11, c11.x, num);
  const float r = fmaf(-e.W, num * rcp_approx(den), e.I);
  return den > 0.f ? e.fwv * (r * r) : e.fb;
}

// float64 3x3 least-squares paraboloid (recon.py:183-207); e is row-major
// [ss offset -1,0,1][fs offset -1,0,1].  Offsets clipped to [-1, 1]; (0,0)
// when the Hessian is not positive definite.
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

// Per-tile geometry of the TMA object windows (bounding box of u over the
// tile's work pixels).
struct TileGeo {
  double umin0, umin1;  // NaN when the tile has no work pixel
  int span_r, span_c;   // floor(max u - min u) per axis over the tile's work pixels
                        // (clamped to 4096; -1 when not finite)
};

// The tile's object window fits a TMA box of box_r x box_c when its span plus
// the patch extent (need_r/need_c: window rows/cols beyond the span, incl.
// floor() slack and the 4-column alignment of the box origin) fit.
__host__ __device__ inline bool tile_fits(const TileGeo& g, int need_r, int need_c, int box_r,
                                          int box_c) {
  return g.span_r >= 0 && g.span_c >= 0 && g.span_r + need_r <= box_r &&
         g.span_c + need_c <= box_c;
}

// Per-tile geometry -> TileGeo (device helper used by the tile kernels).
__device__ __forceinline__ TileGeo make_tile_geo(double mn0, double mx0, double mn1, double mx1) {
  TileGeo g;
  if (!(mn0 <= mx0)) {
    g.umin0 = g.umin1 = NAN;
    g.span_r = g.span_c = -1;
    return g;
  }
  g.umin0 = mn0;
  g.umin1 = mn1;
  const bool finite = fabs(mn0) < 1e9 && fabs(mx0) < 1e9 && fabs(mn1) < 1e9 && fabs(mx1) < 1e9;
  const double sr = floor(mx0 - mn0), sc = floor(mx1 - mn1);
  g.span_r = finite ? (sr > 4096.0 ? 4096 : static_cast<int>(sr)) : -1;
  g.span_c = finite ? (sc > 4096.0 ? 4096 : static_cast<int>(sc)) : -1;
  return g;
}

// Host: largest spans over tiles with work pixels -> out[2] (synchronises).
int tile_span_max(const TileGeo* geo, int64_t n, int* out, cudaStream_t s);
// Same reduction left on the device: out_dev[2] (no synchronisation).
int tile_span_max_dev(const TileGeo* geo, int64_t n, int* out_dev, cudaStream_t s);
// out = window_offsets of the na-point window then of the nb-point window
// (n = 2 kh + 1 points each), written on the device (no host copy).
int fill_offsets(double* out, int na, int nb, double step, cudaStream_t s);

__host__ __device__ inline int slot_floats(int br, int bc) { return (br * bc + 31) / 32 * 32; }
// TMA on this stack faults ("illegal instruction") unless the box starts on a
// 16-byte boundary in the innermost dimension (measured: fp32 column
// coordinates must be multiples of 4; tools/tma_probe4.cu), so window origins
// are aligned down and the patch offset absorbs the difference.
__host__ __device__ inline int align4_down(int c) { return c - (((c % 4) + 4) % 4); }

__device__ __forceinline__ int clamp_span(double v) {
  return v < 0.0 ? 0 : (v > 4096.0 ? 4096 : static_cast<int>(v));
}

// Patch-valid map tile (see make_pv): pv[i][j] = every cell of rows
// [i+lr, i+hr] x cols [j+lc, j+hc] exists and is valid, as a separable AND
// over a kPvR x kPvC output tile with its halo staged in shared memory;
// optionally also the NaN-encoded float32 reference of the tile's cells
// (fmn).  32 x 8 threads (tx, ty).
constexpr int kPvC = 32, kPvR = 16, kPvMaxHalo = 64;
struct PvShared {
  uint8_t v[kPvR + kPvMaxHalo][kPvC + kPvMaxHalo];
  uint8_t rowok[kPvR + kPvMaxHalo][kPvC];
};
__device__ __forceinline__ void pv_tile_block(PvShared& sm, int bx, int by, int tx, int ty,
                                              const uint8_t* __restrict__ valid,
                                              const float* __restrict__ fm, int os, int of, int lr,
                                              int hr, int lc, int hc, uint8_t* __restrict__ pv,
                                              float* __restrict__ fmn,
                                              float2* __restrict__ fm2 = nullptr, int pad = 0) {
  const int i0 = by * kPvR, j0 = bx * kPvC;
  const int th = kPvR + hr - lr, tw = kPvC + hc - lc;
  for (int rr = ty; rr < th; rr += 8)
    for (int cc = tx; cc < tw; cc += 32) {
      const int r = i0 + lr + rr, c = j0 + lc + cc;
      sm.v[rr][cc] = (r >= 0 && r < os && c >= 0 && c < of) ? valid[r * of + c] : 0;
    }
  __syncthreads();
  for (int rr = ty; rr < th; rr += 8) {
    uint8_t ok = 1;
    for (int d = 0; d <= hc - lc; ++d) ok &= sm.v[rr][tx + d];
    sm.rowok[rr][tx] = ok;
  }
  __syncthreads();
  const int j = j0 + tx;
  for (int rr = ty; rr < kPvR; rr += 8) {
    const int i = i0 + rr;
    if (i >= os || j >= of) continue;
    uint8_t ok = 1;
    for (int d = 0; d <= hr - lr; ++d) ok &= sm.rowok[rr + d][tx];
    pv[i * of + j] = ok;
    if (fmn) fmn[i * of + j] = valid[i * of + j] ? fm[i * of + j] : __int_as_float(0x7fc00000);
  }
  if (fm2) {
    // padded (value, mask) copy (trial_pad): the tile's cells, and for tiles on
    // the image's edge the pad-wide border next to them (mask -inf)
    const int ofp = of + 2 * pad;
    const int rlo = by == 0 ? -pad : 0, clo = bx == 0 ? -pad : 0;
    const int rhi = i0 + kPvR >= os ? os - i0 + pad : kPvR;
    const int chi = j0 + kPvC >= of ? of - j0 + pad : kPvC;
    for (int rr = rlo + ty; rr < rhi; rr += 8)
      for (int cc = clo + tx; cc < chi; cc += 32) {
        const int i = i0 + rr, jj = j0 + cc;
        float2 v = make_float2(0.f, __int_as_float(0xff800000));
        if (i >= 0 && i < os && jj >= 0 && jj < of)
          v = valid[i * of + jj] ? make_float2(fm[i * of + jj], 1.f) : make_float2(0.f, 0.f);
        fm2[(int64_t)(i + pad) * ofp + (jj + pad)] = v;
      }
  }
}

// Host helpers ---------------------------------------------------------------
// Patch-valid map: pv[i][j] = every cell of rows [i+lr, i+hr] x cols
// [j+lc, j+hc] exists and is valid; with fmn != NULL also the NaN-encoded
// reference (NaN on invalid cells, read by the exact fix-ups) in the same launch.
int make_pv(const pxst_ref* ref, int lr, int hr, int lc, int hc, uint8_t* pv, float* fmn,
            cudaStream_t s);
// Offsets of SearchWindow.offsets (recon.py:51-57).
std::vector<double> window_offsets(int64_t half, double step);
// Integer steps per pixel of a sub-pixel grid (0 when 1/step is not integral).
int steps_per_pixel(double step);
int check_ref(const pxst_ref* r);
bool force_generic();

}  // namespace pxst
