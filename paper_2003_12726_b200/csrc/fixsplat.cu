// Deterministic splat pass shared by K1 (object formation, recon.py:99-141)
// and K4 (error maps, recon.py:388-438): see fixsplat.cuh for the number
// format.
//
// One CTA per 8 x 64 detector tile and frame slice (grid.z).  The CTA walks
// its frames in batches of 8 and groups consecutive batches into "sessions"
// whose joint object footprint (the tile's u bounding box shifted by each
// frame's translation) fits a shared-memory region of RC cells and whose
// term count per cell stays <= 2047 (bounded by the tile's largest number of
// pixels reaching one cell in one frame, from a shared-memory histogram of
// the tile's u).  A session zeroes the region, adds every sample's corner
// terms with 32-bit shared atomics on (lo, hi) limbs, then adds the region's
// nonzero cells to the global int64 accumulators (one RED.64 per cell and
// value instead of two 16-byte REDs per sample and image).  A batch whose
// footprint alone exceeds the region (a pathological map) adds its terms to
// the global accumulators directly -- the same integers, so the same result.
//
// Modes: 0 = object splat (value I/W, weight W^2: recon.py:135-138);
// 1 = error maps (masked bilinear read of the reference, eps = r^2/sigma^2,
// per-pixel / per-frame sums, reference-plane splat of eps with weight 1,
// recon.py:414-431); 2 = mode 1 fused with the next iteration's object
// splat (same samples, positions relative to the next grid read from the
// device, recon.py:504-516).
#include <stdlib.h>

#include <type_traits>

#include "fixsplat.cuh"

namespace pxst {
namespace {

// Tile 8 rows x 64 columns: warp w takes row w, lane l its columns 2l and
// 2l + 1 (one per pass e), so the 32 samples of one instruction are two
// detector columns apart and land on distinct cells (adjacent columns often
// share a cell at magnification < 1: same-address shared atomics serialise).
constexpr int kXR = 8, kXC = 64, kXT = 256, kXW = kXT / 32;  // tile, threads, warps
constexpr int kXB = 8;        // (frame-table chunks are multiples of this)
#ifndef PXST_FIX_TAB
#define PXST_FIX_TAB 128
#endif
constexpr int kXTab = PXST_FIX_TAB;   // frames per shared frame-table chunk (multiple of kXB)

// Region values: mode 0 object num, den; modes 1, 2 plane num, den, plane
// num fine band (see plane_band); mode 2 adds the next object's num, den.
#ifndef PXST_FIX_RC1
#define PXST_FIX_RC1 2048
#endif
#ifndef PXST_FIX_RC2
#define PXST_FIX_RC2 1280
#endif
#ifndef PXST_FIX_OCC12
#define PXST_FIX_OCC12 3
#endif
template <int MODE> struct FixCfg { static constexpr int NV = 2, RC = 3072; };
template <> struct FixCfg<1> { static constexpr int NV = 3, RC = PXST_FIX_RC1; };
template <> struct FixCfg<2> { static constexpr int NV = 5, RC = PXST_FIX_RC2; };

template <int MODE>
constexpr size_t fix_smem_bytes() {
  return sizeof(unsigned) * 2 * FixCfg<MODE>::NV * FixCfg<MODE>::RC;
}

}  // namespace

struct FixArgs {
  pxst_scan sc;
  const double* u;
  const double* di;
  const double* dj;
  int64_t n0, m0, os, of;      // primary grid: the object (mode 0) or the reference (1, 2)
  int64_t k_lo, k_hi;          // good-frame range of the launch
  int64_t frames_per_z;        // frames per grid.z slice (fix_slices)
  FixAcc A;                    // mode 0: object; modes 1, 2: reference plane
  FixAcc B;                    // mode 2: next object
  const int64_t* grid_b;       // mode 2: device (n0, m0, os, of) of the next object
  int64_t cap_b;               //   cells of B; a next grid larger than this is not splatted
  const double2* grp;          // modes 1, 2: grouped float64 reference, NaN = invalid
  const double* sigma2;
  double* pix_part;            // [n_z][ss*fs] per-pixel eps sums of each slice
  double* part;                // [n_good][n_cta] per-frame eps sums of each CTA
  int64_t n_cta;
  unsigned long long* n_drop;  // mode 0, nullable: out-of-grid samples
  int no_region;               // debug (PXST_FIX_NO_REGION=1): every term straight to global memory
};

namespace {

__device__ __forceinline__ void red64(long long* p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// One term t = scaled * w of an image: coarse corners into the shared region
// (limbs) or, without a region, into the global int64 image; tiny-weight
// corners into the fine image (see kFineW).
struct TermSink {
  unsigned* lo;       // region limbs of this value (lo, hi = lo + NV*RC) or nullptr
  int* hi;
  long long* g;       // global coarse image
  long long* gf;      // global fine image
};

// A term into the region's limbs (coarse, corner weight >= kFineW): lo at
// slo[idx], hi at slo[idx + HI] (HI = NV * RC words, an immediate offset).
// Every nonzero corner weight >= kFineW: the smallest nonzero one is
// min(fx, 1-fx) min(fy, 1-fy) over the axes with a nonzero fraction
// (float32 classification; exact fractions 0 stay 0).
__device__ __forceinline__ bool small_corner_ok(double fx, double fy) {
  const float x = static_cast<float>(fx), y = static_cast<float>(fy);
  const float mx = x > 0.f ? fminf(x, 1.f - x) : 1.f;
  const float my = y > 0.f ? fminf(y, 1.f - y) : 1.f;
  return mx * my >= static_cast<float>(kFineW) * 1.0001f;
}

template <int HI>
__device__ __forceinline__ void region_term(unsigned* slo, int idx, double scaled, double w) {
  PXST_DCHECK(idx >= 0 && idx < HI);
  unsigned lo;
  int hi;
  fix_limbs(scaled, w, lo, hi);
  atomicAdd(slo + idx, lo);
  atomicAdd(reinterpret_cast<int*>(slo) + idx + HI, hi);
}

// The same term through a 32-bit shared-memory address (the hot path):
// lo at [addr], hi at [addr + HIB]; value planes and the c0 + 1 corner are
// immediate offsets (OFF) from one address register.
template <int HIB, int OFF>
__device__ __forceinline__ void region_red(unsigned addr, double scaled, double w) {
  unsigned lo;
  int hi;
  fix_limbs(scaled, w, lo, hi);
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(addr), "r"(lo), "n"(OFF));
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(addr), "r"(hi), "n"(OFF + HIB));
}

// A term straight into the global images (no region; and tiny-weight
// corners, |t| < 2^51 fine quanta).
__device__ __forceinline__ void global_term(long long* g, long long* gf, int64_t cell,
                                            double scaled, double w) {
  PXST_DCHECK(cell >= 0);
  if (w >= kFineW) red64(g + cell, fix_value(scaled, w));
  else if (w > 0.0) red64(gf + cell, fix_value(scaled * 0x1p20, w));
}

// The plane numerator eps * w_c: eps is bounded loosely (pxst_plane_quanta:
// (max|I| + max W max|ref|)^2 / min sigma^2, often 10^4 x the typical eps),
// so a coarse-weight term below 2^21 coarse quanta goes to a second band in
// units of q * 2^-20 (the fine image) and keeps >= 20 significant bits.
// The rule compares exponents: with scaled = m1 2^e1 and w = m2 2^e2
// (m in [1, 2)), band <=> e1 + e2 < 20, so a band term is below 2^21 coarse
// quanta (< 2^41 fine quanta) and a coarse term at least 2^20.  band_key is
// the per-sample part: plane_band(key, w) = hi word of w below key.
__device__ __forceinline__ int band_key(double scaled) {
  const int e1 = (__double2hiint(scaled) >> 20) & 0x7ff;          // biased exponent, 0 for 0
  return min(2 * 1023 + 20 - e1, 2047) << 20;   // (a zero / denormal eps: every term in the band)
}
__device__ __forceinline__ bool plane_band(int key, double w) {   // w >= 0
  return __double2hiint(w) < key;
}

#ifndef PXST_FIX_OCC0
#define PXST_FIX_OCC0 3
#endif
template <int MODE>
__global__ void __launch_bounds__(kXT, MODE == 0 ? PXST_FIX_OCC0 : PXST_FIX_OCC12) k_fix_pass(FixArgs a) {
  constexpr int NV = FixCfg<MODE>::NV, RC = FixCfg<MODE>::RC;
  constexpr bool ERR = MODE != 0;
  extern __shared__ __align__(16) unsigned char fx_raw[];
  unsigned* slo = reinterpret_cast<unsigned*>(fx_raw);              // [NV][RC]
  int* shi = reinterpret_cast<int*>(slo + NV * RC);                 // [NV][RC]
  __shared__ double t_di[kXTab], t_dj[kXTab];
  __shared__ int64_t t_off[kXTab];
  __shared__ int4 t_ft[kXTab];                                      // frame footprints
  __shared__ double s_red[kXW][4];
  __shared__ double s_frw[ERR ? kXW : 1][ERR ? kXTab : 1];   // per-frame sums of each warp
  __shared__ int s_cmax;
  __shared__ int4 s_sess[2];   // session footprint (R0, R1, C0, C1), (end frame, region)
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(slo));

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int64_t plane = a.sc.ss * a.sc.fs;
  // Sample positions: t = u - d (recon.py:138, one rounding), split as
  // floor(t) and t - floor(t), the grid origin subtracted from the integer.
  // The reference rounds t - origin once more before its split
  // (interp.py:39-42): at most one ulp of the position, far inside the parity
  // bars, and the bilinear value is continuous across a floor that flips.  In
  // exchange the split does not depend on the grid, so the fused pass
  // (mode 2) shares every weight between the reference grid and the next
  // object's grid, whose cells differ by the origins' integer offset.
  // (|t| < 1e9 on the region path -- the footprints are finite -- and
  // checked on the direct path.)
  const int n0i = static_cast<int>(a.n0), m0i = static_cast<int>(a.m0);
  const int os_1 = static_cast<int>(a.os - 1), of_1 = static_cast<int>(a.of - 1);
  const int of = static_cast<int>(a.of);

  int64_t p[2];
  bool live[2];
  double u0[2], u1[2], Wv[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int64_t row = a.sc.roi[0] + (int64_t)blockIdx.y * kXR + warp;
    const int64_t col = a.sc.roi[2] + (int64_t)blockIdx.x * kXC + 2 * lane + e;
    const bool in = row < a.sc.roi[1] && col < a.sc.roi[3];
    p[e] = in ? row * a.sc.fs + col : 0;
    live[e] = in && a.sc.work[p[e]] != 0;
    u0[e] = live[e] ? a.u[p[e]] : 0.0;
    u1[e] = live[e] ? a.u[plane + p[e]] : 0.0;
    Wv[e] = live[e] ? a.sc.w64[p[e]] : 1.0;
  }
  // tile bounding box of u over its work pixels
  double b0 = fmin(live[0] ? u0[0] : INFINITY, live[1] ? u0[1] : INFINITY);
  double b1 = fmax(live[0] ? u0[0] : -INFINITY, live[1] ? u0[1] : -INFINITY);
  double b2 = fmin(live[0] ? u1[0] : INFINITY, live[1] ? u1[1] : INFINITY);
  double b3 = fmax(live[0] ? u1[0] : -INFINITY, live[1] ? u1[1] : -INFINITY);
  b0 = warp_min(b0); b1 = warp_max(b1); b2 = warp_min(b2); b3 = warp_max(b3);
  if (lane == 0) { s_red[warp][0] = b0; s_red[warp][1] = b1; s_red[warp][2] = b2; s_red[warp][3] = b3; }
  if (threadIdx.x == 0) s_cmax = 0;
  __syncthreads();
  double umin0 = s_red[0][0], umax0 = s_red[0][1], umin1 = s_red[0][2], umax1 = s_red[0][3];
#pragma unroll
  for (int w = 1; w < kXW; ++w) {
    umin0 = fmin(umin0, s_red[w][0]); umax0 = fmax(umax0, s_red[w][1]);
    umin1 = fmin(umin1, s_red[w][2]); umax1 = fmax(umax1, s_red[w][3]);
  }
  const int64_t k_begin = a.k_lo + (int64_t)blockIdx.z * a.frames_per_z;
  const int64_t k_end = min(a.k_hi, k_begin + a.frames_per_z);
  if (!(umin0 <= umax0)) {   // no work pixel: only the per-frame partials need writing
    if (ERR)
      for (int64_t k = k_begin + threadIdx.x; k < k_end; k += kXT) a.part[k * a.n_cta + cta] = 0.0;
    return;
  }

  // Largest number of this tile's pixels whose corners reach one cell in one
  // frame: a pixel in u-bin b reaches cells b - D + {-1, 0, 1} per axis
  // (D = the frame's integer shift), so the max over 3 x 3 blocks of the
  // tile's u-bin histogram bounds it.
  const bool fin = fabs(umin0) < 1e9 && fabs(umax0) < 1e9 && fabs(umin1) < 1e9 && fabs(umax1) < 1e9;
  const int hb0 = fin ? __double2int_rd(umin0) : 0, hb1 = fin ? __double2int_rd(umin1) : 0;
  const int hh = fin ? __double2int_rd(umax0) - hb0 + 1 : 1 << 20;
  const int hw = fin ? __double2int_rd(umax1) - hb1 + 1 : 1 << 20;
  int cmax;
  if (hh <= 2 * RC && hw <= 2 * RC && hh * hw <= NV * RC) {
    for (int i = threadIdx.x; i < hh * hw; i += kXT) slo[i] = 0u;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (live[e])
        atomicAdd(&slo[(__double2int_rd(u0[e]) - hb0) * hw + (__double2int_rd(u1[e]) - hb1)], 1u);
    __syncthreads();
    int m = 0;
    for (int i = threadIdx.x; i < hh * hw; i += kXT) {
      const int r = i / hw, c = i % hw;
      int sum = 0;
      for (int dr = -1; dr <= 1; ++dr)
        for (int dc = -1; dc <= 1; ++dc) {
          const int rr = r + dr, cc = c + dc;
          if (rr >= 0 && rr < hh && cc >= 0 && cc < hw) sum += static_cast<int>(slo[rr * hw + cc]);
        }
      m = max(m, sum);
    }
    atomicMax(&s_cmax, m);
    __syncthreads();
    cmax = s_cmax;
  } else {
    cmax = 2 * kXT;   // every pixel of the tile
  }
  // frames per session: <= 2047 terms per cell (a map whose bounding box is
  // not finite takes the direct path throughout)
  const int max_frames = cmax > 0 ? kFixMaxTerms / cmax : 1 << 30;

  // accumulator scales
  const double qa_n = 1.0 / a.A.q[0], qa_d = 1.0 / a.A.q[1];
  double qb_n = 0.0, qb_d = 0.0;
  int64_t dn = 0, dm = 0, osb = 1, ofb = 1;
  bool splat_b = false;
  if (MODE == 2) {
    qb_n = 1.0 / a.B.q[0];
    qb_d = 1.0 / a.B.q[1];
    dn = a.n0 - a.grid_b[0];
    dm = a.m0 - a.grid_b[1];
    osb = a.grid_b[2];
    ofb = a.grid_b[3];
    splat_b = osb > 0 && ofb > 0 && osb * ofb <= a.cap_b;
  }
  const int dni = static_cast<int>(dn), dmi = static_cast<int>(dm);
  const int osb_1 = static_cast<int>(osb - 1), ofb_1 = static_cast<int>(ofb - 1);
  double W2[2], vsc[2], isig[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    W2[e] = Wv[e] * Wv[e];                                    // recon.py:136
    vsc[e] = live[e] ? W2[e] / Wv[e] : 0.0;                   // (value = I / W) * W^2 per unit I
    isig[e] = (ERR && live[e]) ? 1.0 / a.sigma2[p[e]] : 0.0;  // recon.py:422
  }
  const TermSink kAn{slo, shi, a.A.num, a.A.num_f};
  const TermSink kAd{slo + RC, shi + RC, a.A.den, a.A.den_f};
  const TermSink kBn{slo + 2 * RC, shi + 2 * RC, a.B.num, a.B.num_f};
  const TermSink kBd{slo + 3 * RC, shi + 3 * RC, a.B.den, a.B.den_f};
  constexpr int kBandV = MODE == 2 ? 4 : 2;        // the plane numerator's fine band
  const TermSink kAnB{slo + kBandV * RC, shi + kBandV * RC, a.A.num_f, nullptr};
  double pix[2] = {0.0, 0.0};
  unsigned dropped = 0;
  const bool count_drop = !ERR && a.n_drop != nullptr;

  for (int64_t kc = k_begin; kc < k_end; kc += kXTab) {
    const int nt = static_cast<int>(min((int64_t)kXTab, k_end - kc));
    __syncthreads();
    for (int t = threadIdx.x; t < nt; t += kXT) {
      const int64_t f = a.sc.good[kc + t];
      const double dI = a.di[f], dJ = a.dj[f];
      t_di[t] = dI;
      t_dj[t] = dJ;
      t_off[t] = f * plane;
      // the tile's cells for this frame (primary grid; + 1 row / column for
      // the r0 + 1 / c0 + 1 corners)
      t_ft[t] = fin ? make_int4(__double2int_rd(umin0 - dI) - n0i, __double2int_rd(umax0 - dI) - n0i + 1,
                                __double2int_rd(umin1 - dJ) - m0i, __double2int_rd(umax1 - dJ) - m0i + 1)
                    : make_int4(0, 1 << 20, 0, 1 << 20);
    }
    __syncthreads();
    for (int s0 = 0; s0 < nt;) {
      // session: consecutive frames whose joint footprint fits the region
      // (formed by thread 0, broadcast through shared memory)
      if (threadIdx.x == 0) {
        int4 fb = t_ft[s0];
        int s1 = s0 + 1;
        const bool reg = fin && max_frames > 0 && !a.no_region &&
                         (int64_t)(fb.y - fb.x + 1) * (fb.w - fb.z + 1) <= RC;
        if (reg) {
          while (s1 < nt && s1 - s0 < max_frames) {
            const int4 g = t_ft[s1];
            const int4 u = make_int4(min(fb.x, g.x), max(fb.y, g.y), min(fb.z, g.z),
                                     max(fb.w, g.w));
            if ((int64_t)(u.y - u.x + 1) * (u.w - u.z + 1) > RC) break;
            fb = u;
            ++s1;
          }
        }
        s_sess[0] = fb;
        s_sess[1] = make_int4(s1, reg ? 1 : 0, 0, 0);
      }
      __syncthreads();
      const int4 fb = s_sess[0];
      const int s1 = s_sess[1].x;
      const bool region = s_sess[1].y != 0;
      const int R0 = fb.x, C0 = fb.z;
      const int nc = region ? fb.w - fb.z + 1 : 0;
      const int ncell = region ? (fb.y - fb.x + 1) * nc : 0;
      if (region) {
        for (int i = threadIdx.x; i < ncell; i += kXT) {
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            slo[v * RC + i] = 0u;
            shi[v * RC + i] = 0;
          }
        }
        __syncthreads();
      }
      // ---- the session's samples, one frame at a time (the next frame's
      // stack values in flight); region / direct are two compiled bodies
      auto session = [&](auto region_c) {
        constexpr bool REG = decltype(region_c)::value;
        constexpr int HIB = NV * RC * 4;           // lo -> hi limb, bytes
        constexpr int VB = RC * 4;                 // value plane stride, bytes
        float In[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) In[e] = live[e] ? __ldg(a.sc.frames + t_off[s0] + p[e]) : 0.f;
        for (int t = s0; t < s1; ++t) {
          const float Ic[2] = {In[0], In[1]};
          {
            const int64_t off = t_off[t + 1 < s1 ? t + 1 : t];
#pragma unroll
            for (int e = 0; e < 2; ++e) In[e] = live[e] ? __ldg(a.sc.frames + off + p[e]) : 0.f;
          }
          const double dI = t_di[t], dJ = t_dj[t];
          double ef = 0.0;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool act = live[e];
            const double tx = u0[e] - dI, ty = u1[e] - dJ;    // recon.py:138, 418
            const int ri = __double2int_rd(tx), ci = __double2int_rd(ty);
            const double fx = tx - static_cast<double>(ri), fy = ty - static_cast<double>(ci);
            const int r0 = ri - n0i, c0 = ci - m0i;
            // inside: 0 <= x <= os - 1 per axis (interp.py:67, 103-107)
            const bool fin_s = REG || (fabs(tx) < 1e9 && fabs(ty) < 1e9);
            const bool inA = act && fin_s && r0 >= 0 && c0 >= 0 &&
                             (r0 < os_1 || (r0 == os_1 && fx == 0.0)) &&
                             (c0 < of_1 || (c0 == of_1 && fy == 0.0));
            const double gx = 1.0 - fx, gy = 1.0 - fy;
            const double cw[4] = {gx * gy, gx * fy, fx * gy, fx * fy};   // corners 00 01 10 11
            const double I = static_cast<double>(Ic[e]);
            double sAn, sAd;
            int bkey = 0;
            if (ERR) {
              // masked bilinear read (interp.py:53-85) of the grouped reference:
              // g[r][c] = (v(r, c), v(r + 1, c)), NaN = invalid cell.  (A lane
              // without a work pixel has I = 0, W = 1, 1/sigma2 = 0: eps = 0.)
              const double2 z2 = make_double2(0.0, 0.0);
              const int a00 = r0 * of + c0;                   // os * of < 2^31 (check_ref)
              const double2 g0 = inA ? __ldg(a.grp + a00) : z2;
              const double2 g1 = (inA && fy > 0.0) ? __ldg(a.grp + a00 + 1) : z2;
              const double cv[4] = {g0.x, g1.x, g0.y, g1.y};
              const bool anynan = (g0.x != g0.x) || (g1.x != g1.x) || (g0.y != g0.y) || (g1.y != g1.y);
              double den, nm;
              bool all = true;
              if (!__any_sync(0xffffffffu, anynan)) {
                // every corner of every lane valid: the same sums without selects
                den = ((cw[0] + cw[1]) + cw[2]) + cw[3];
                nm = fma(cw[3], cv[3], fma(cw[2], cv[2], fma(cw[1], cv[1], cw[0] * cv[0])));
              } else {
                den = 0.0;
                nm = 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const bool m = cv[q] == cv[q];
                  all = all && m;
                  den = fma(cw[q], m ? 1.0 : 0.0, den);
                  nm = fma(cw[q], m ? cv[q] : 0.0, nm);
                }
              }
              const bool ok = inA && den > 0.0;
              const double v = !ok ? 0.0 : (all ? nm * (2.0 - den) : nm / den);
              const double r = I - Wv[e] * v;                           // recon.py:421
              const double rr = ok ? r : I - Wv[e];
              const double eps = (rr * rr) * isig[e];                   // recon.py:422
              pix[e] += eps;
              ef += eps;
              sAn = eps * qa_n;       // plane: value eps, weight 1 (recon.py:425)
              sAd = qa_d;
              bkey = band_key(sAn);
            } else {
              dropped += (count_drop && act && !inA) ? 1u : 0u;
              sAn = I * vsc[e] * qa_n;   // value * weight = (I / W) W^2 (interp.py:112-122)
              sAd = W2[e] * qa_d;
            }
            // hot path: every corner weight 0 (nothing to add) or >= kFineW;
            // the others, and the direct sessions, take the per-corner path
            // (smallest nonzero corner weight = min(fx, 1-fx) min(fy, 1-fy)
            // over the axes with a nonzero fraction; classified in float32:
            // only the routing depends on it)
            const bool hot = REG && small_corner_ok(fx, fy);
            // warp-uniform: skip the r0+1 / c0+1 corners when no lane weights
            // them (config 2: u_ss = x, every fx = 0)
            const bool need_r1 = __any_sync(0xffffffffu, inA && hot && fx > 0.0);
            const bool need_c1 = __any_sync(0xffffffffu, inA && hot && fy > 0.0);
            if (inA && hot) {
              const int l = (r0 - R0) * nc + (c0 - C0);
              PXST_DCHECK(r0 >= R0 && c0 >= C0 && l >= 0 && l + nc + 1 < ncell);
              const unsigned a0 = sbase + 4u * static_cast<unsigned>(l);
              const unsigned a1 = a0 + 4u * static_cast<unsigned>(nc);
              // one corner: numerator (plane: coarse or fine band by its size),
              // denominator; a zero-weight corner adds 0 (no branch)
              auto corner = [&](unsigned ad, auto off_c, double w) {
                constexpr int OFF = decltype(off_c)::value;
                if (ERR) {
                  const bool band = plane_band(bkey, w);
                  const unsigned an = ad + (band ? kBandV * VB : 0);
                  const double sn = __hiloint2double(__double2hiint(sAn) + (band ? (20 << 20) : 0),
                                                     __double2loint(sAn));
                  region_red<HIB, OFF>(an, sn, w);
                } else {
                  region_red<HIB, OFF>(ad, sAn, w);
                }
                region_red<HIB, OFF + VB>(ad, sAd, w);
              };
              corner(a0, std::integral_constant<int, 0>{}, cw[0]);
              if (need_c1) corner(a0, std::integral_constant<int, 4>{}, cw[1]);
              if (need_r1) {
                corner(a1, std::integral_constant<int, 0>{}, cw[2]);
                if (need_c1) corner(a1, std::integral_constant<int, 4>{}, cw[3]);
              }
            } else if (inA) {
              const int64_t cell = (int64_t)r0 * a.of + c0;
              const int64_t dcell[4] = {0, 1, a.of, a.of + 1};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (ERR && cw[q] >= kFineW && plane_band(bkey, cw[q]))
                  red64(a.A.num_f + cell + dcell[q], fix_value(sAn * 0x1p20, cw[q]));
                else
                  global_term(a.A.num, a.A.num_f, cell + dcell[q], sAn, cw[q]);
                global_term(a.A.den, a.A.den_f, cell + dcell[q], sAd, cw[q]);
                if (!ERR && a.A.touched && cw[q] > 0.0 && cw[q] < kFineW)
                  a.A.touched[cell + dcell[q]] = 1;
              }
            }
            if (MODE == 2) {
              // the next object's own position, as make_reference computes it
              // (recon.py:138: u - d - origin), so the terms equal a separate
              // object formation bit for bit
              // (same split, same weights: only the cell differs, by the
              // origins' offset; a separate object formation computes exactly
              // these terms, so the fused object equals it bit for bit)
              const int r0b = r0 + dni, c0b = c0 + dmi;
              const bool inB = splat_b && act && fin_s && r0b >= 0 && c0b >= 0 &&
                               (r0b < osb_1 || (r0b == osb_1 && fx == 0.0)) &&
                               (c0b < ofb_1 || (c0b == ofb_1 && fy == 0.0));
              const double* cwb = cw;
              const double sBn = I * vsc[e] * qb_n, sBd = W2[e] * qb_d;
              const bool hotb = hot;
              const bool need_r1b = __any_sync(0xffffffffu, inB && hotb && fx > 0.0);
              const bool need_c1b = __any_sync(0xffffffffu, inB && hotb && fy > 0.0);
              if (inB && hotb) {
                // next-grid cell (r0b, c0b) in the region's (reference-grid) frame
                const int l = (r0 - R0) * nc + (c0 - C0);
                PXST_DCHECK(l >= 0 && l + nc + 1 < ncell);
                const unsigned b0 = sbase + 4u * static_cast<unsigned>(l) + 2 * VB;
                const unsigned b1 = b0 + 4u * static_cast<unsigned>(nc);
                auto cornerb = [&](unsigned ad, auto off_c, double w) {
                  constexpr int OFF = decltype(off_c)::value;
                  region_red<HIB, OFF>(ad, sBn, w);
                  region_red<HIB, OFF + VB>(ad, sBd, w);
                };
                cornerb(b0, std::integral_constant<int, 0>{}, cwb[0]);
                if (need_c1b) cornerb(b0, std::integral_constant<int, 4>{}, cwb[1]);
                if (need_r1b) {
                  cornerb(b1, std::integral_constant<int, 0>{}, cwb[2]);
                  if (need_c1b) cornerb(b1, std::integral_constant<int, 4>{}, cwb[3]);
                }
              } else if (inB) {
                const int64_t cellb = (int64_t)r0b * ofb + c0b;
                const int64_t dcb[4] = {0, 1, ofb, ofb + 1};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  global_term(a.B.num, a.B.num_f, cellb + dcb[q], sBn, cwb[q]);
                  global_term(a.B.den, a.B.den_f, cellb + dcb[q], sBd, cwb[q]);
                  if (a.B.touched && cwb[q] > 0.0 && cwb[q] < kFineW) a.B.touched[cellb + dcb[q]] = 1;
                }
              }
            }
          }
          if (ERR) {       // this warp's share of the frame's sum (CTA sum at chunk end)
            const double sum = warp_sum(ef);
            if (lane == 0) s_frw[warp][t] = sum;
          }
        }
      };
      if (region)
        session(std::integral_constant<bool, true>{});
      else
        session(std::integral_constant<bool, false>{});
      // ---- flush the region into the int64 images
      if (region) {
        __syncthreads();
        for (int i = threadIdx.x; i < ncell; i += kXT) {
          const int r = R0 + i / nc, c = C0 + i % nc;
          const long long vn = fix_join(slo[i], shi[i]);
          const long long vd = fix_join(slo[RC + i], shi[RC + i]);
          if (vn != 0 || vd != 0) {
            PXST_DCHECK(r >= 0 && r < a.os && c >= 0 && c < a.of);
            const int64_t cell = (int64_t)r * of + c;
            if (vn) red64(a.A.num + cell, vn);
            if (vd) red64(a.A.den + cell, vd);
          }
          if (ERR) {
            const long long vb = fix_join(slo[kBandV * RC + i], shi[kBandV * RC + i]);
            if (vb) red64(a.A.num_f + (int64_t)r * of + c, vb);
          }
          if (MODE == 2) {
            const long long wn = fix_join(slo[2 * RC + i], shi[2 * RC + i]);
            const long long wd = fix_join(slo[3 * RC + i], shi[3 * RC + i]);
            if (wn != 0 || wd != 0) {
              PXST_DCHECK(r + dn >= 0 && r + dn < osb && c + dm >= 0 && c + dm < ofb);
              const int64_t cell = (int64_t)(r + dn) * ofb + (c + dm);
              if (wn) red64(a.B.num + cell, wn);
              if (wd) red64(a.B.den + cell, wd);
            }
          }
        }
        __syncthreads();
      }
      s0 = s1;
    }
    if (ERR) {   // per-frame sums of the chunk: the CTA's warps in a fixed order
      __syncthreads();
      for (int t = threadIdx.x; t < nt; t += kXT) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kXW; ++w) sum += s_frw[w][t];
        a.part[(kc + t) * a.n_cta + cta] = sum;
      }
    }
  }
  if (ERR) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (live[e]) a.pix_part[(int64_t)blockIdx.z * plane + p[e]] = pix[e];
  }
  if (!ERR && a.n_drop) {
    dropped += __shfl_xor_sync(0xffffffffu, dropped, 16);
    dropped += __shfl_xor_sync(0xffffffffu, dropped, 8);
    dropped += __shfl_xor_sync(0xffffffffu, dropped, 4);
    dropped += __shfl_xor_sync(0xffffffffu, dropped, 2);
    dropped += __shfl_xor_sync(0xffffffffu, dropped, 1);
    if (lane == 0 && dropped) atomicAdd(a.n_drop, static_cast<unsigned long long>(dropped));
  }
}

// ---------------------------------------------------------------------------
// scales
// ---------------------------------------------------------------------------
// Order-independent max of non-negative doubles (their bit patterns order
// like the values).
__device__ __forceinline__ void atomic_max_nonneg(double* p, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(p),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}
__device__ __forceinline__ void atomic_min_nonneg(double* p, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(p),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

// max |I| over the whole stack (a bound for every sample of every frame set)
__global__ void k_abs_max(const float* __restrict__ frames, int64_t n, double* out) {
  float m = 0.f;
  const int64_t n4 = n / 4;
  const float4* f4 = reinterpret_cast<const float4*>(frames);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(f4 + i);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(__ldg(frames + i)));
  // NaN / inf samples: an infinite bound (quantum 2^-41 of 1, see fix_quantum)
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) m = fmaxf(m, red[k]);
    atomic_max_nonneg(out, static_cast<double>(m));
  }
}

// Scale statistics and quanta in one launch.  Every block reduces its share
// of the ROI's work pixels (max W, min sigma2: kind 1 only) and of the
// reference's valid cells (max |ref|) to part[3 * block]; the last block to
// finish (ticket) folds the partials and writes the quanta:
//   kind 0 (object): q_num from max |I| max W, q_den from max W^2;
//   kind 1 (reference plane): q_num from the eps bound
//   (max|I| + max W max(1, max|ref|))^2 / min sigma2, q_den from 1.
// The same loops also write K4's grouped reference (g[r][c] = (v(r, c),
// v(r + 1, c)), v = the float64 masked reference where valid, NaN elsewhere
// and past the last row: one 16-byte load fetches a bilinear column pair and
// the NaN doubles as the validity bit) and zero-fill an array.
__global__ void __launch_bounds__(256) k_quanta_pass(QuantaJob j, double* __restrict__ part) {
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = t0; q < j.n_zero; q += stride) j.zero[q] = 0.0;
  const int64_t n_ref = j.valid ? j.os * j.of : 0;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  double rmax = 0.0;
  for (int64_t q = t0; q < n_ref; q += stride) {
    const bool ok = j.valid[q] != 0;
    const double v = ok ? (j.fm64 ? j.fm64[q] : static_cast<double>(j.fm[q])) : nan;
    if (ok) rmax = fmax(rmax, fabs(v));
    if (j.grp) {
      const int64_t q1 = q + j.of;
      const double v1 = q1 < n_ref && j.valid[q1] ? (j.fm64 ? j.fm64[q1] : static_cast<double>(j.fm[q1]))
                                                  : nan;
      j.grp[q] = make_double2(v, v1);
    }
  }
  if (!j.quanta) return;
  const int64_t cw = j.sc.roi[3] - j.sc.roi[2], n = (j.sc.roi[1] - j.sc.roi[0]) * cw;
  double wmax = 0.0, smin = INFINITY;
  for (int64_t q = t0; q < n; q += stride) {
    const int64_t p = (j.sc.roi[0] + q / cw) * j.sc.fs + j.sc.roi[2] + q % cw;
    if (!j.sc.work[p]) continue;
    wmax = fmax(wmax, fabs(j.sc.w64[p]));
    if (j.sigma2) smin = fmin(smin, j.sigma2[p]);
  }
  __shared__ double red[3][32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  wmax = warp_max(wmax);
  smin = warp_min(smin);
  rmax = warp_max(rmax);
  if (lane == 0) { red[0][w] = wmax; red[1][w] = smin; red[2][w] = rmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < nw; ++k) {
      wmax = fmax(wmax, red[0][k]);
      smin = fmin(smin, red[1][k]);
      rmax = fmax(rmax, red[2][k]);
    }
    part[3 * blockIdx.x] = wmax;
    part[3 * blockIdx.x + 1] = smin;
    part[3 * blockIdx.x + 2] = rmax;
    __threadfence();
    s_last = atomicAdd(j.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  wmax = 0.0; smin = INFINITY; rmax = 0.0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
    wmax = fmax(wmax, __ldcg(part + 3 * k));
    smin = fmin(smin, __ldcg(part + 3 * k + 1));
    rmax = fmax(rmax, __ldcg(part + 3 * k + 2));
  }
  wmax = warp_max(wmax);
  smin = warp_min(smin);
  rmax = warp_max(rmax);
  __syncthreads();
  if (lane == 0) { red[0][w] = wmax; red[1][w] = smin; red[2][w] = rmax; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int k = 1; k < nw; ++k) {
    wmax = fmax(wmax, red[0][k]);
    smin = fmin(smin, red[1][k]);
    rmax = fmax(rmax, red[2][k]);
  }
  const double amax = *j.absmax;
  const int hk = fix_headroom(j.sc.n_good);
  if (j.kind == 0) {
    j.quanta[0] = fix_quantum(amax * wmax, hk);
    j.quanta[1] = fix_quantum(wmax * wmax, hk);
  } else {
    const double r = amax + wmax * fmax(1.0, rmax);
    const double sg = smin > 0.0 && isfinite(smin) ? smin : 1.0;
    j.quanta[0] = fix_quantum(r * r / sg, hk);
    j.quanta[1] = fix_quantum(1.0, hk);
  }
}

// ---------------------------------------------------------------------------
// finish
// ---------------------------------------------------------------------------
// Normalise (fix_finish_cell) the first n cells, or the grid's when given.
__global__ void k_fix_finish(FixAcc acc, const int64_t* __restrict__ grid, int64_t n, double* out,
                             double* wsum, float* fm, uint8_t* valid) {
  if (grid) {
    const int64_t gn = grid[2] * grid[3];
    if (!(grid[2] > 0 && grid[3] > 0)) return;
    n = gn < n ? gn : n;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    fix_finish_cell(acc, i, out, wsum, fm, valid);
}

// The frame shards' all-reduce fused with the normalisation (single-process
// multi-GPU path, pxst_object_finish_peers): the W peers' accumulators are
// read where they lie (P2P loads over NVLink on a multi-GPU box), their int64
// terms added -- exact, so every device computes the same bits whatever the
// order -- the cells [lo, hi) of this device's slice normalised
// (fix_finish_cell) and the results stored into every peer's output images
// (P2P stores): reduce-scatter, normalise and all-gather in one kernel, 34
// bytes read and 21 written per cell and peer instead of five all-reduced
// images followed by W finishes of the whole grid.
struct PeerFinish {
  FixAcc acc[kMaxPeers];
  double* out[kMaxPeers];
  double* wsum[kMaxPeers];
  float* fm[kMaxPeers];
  uint8_t* valid[kMaxPeers];
  int w;
  int64_t lo, hi;
};
__global__ void k_fix_finish_peers(PeerFinish a) {
  const double qn = a.acc[0].q[0], qd = a.acc[0].q[1];   // full-scan quanta: equal on every peer
  for (int64_t i = a.lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long num = 0, den = 0, num_f = 0, den_f = 0;
    unsigned touched = 0;
    for (int j = 0; j < a.w; ++j) {
      num += a.acc[j].num[i];
      den += a.acc[j].den[i];
      num_f += a.acc[j].num_f[i];
      den_f += a.acc[j].den_f[i];
      if (a.acc[j].touched) touched |= a.acc[j].touched[i];
    }
    // fix_finish_cell on the summed integers
    const double d = static_cast<double>(den) * qd + static_cast<double>(den_f) * (qd * 0x1p-20);
    const double nm = static_cast<double>(num) * qn + static_cast<double>(num_f) * (qn * 0x1p-20);
    const bool pos = d > 0.0;
    const bool ok = pos || (a.acc[0].touched && touched != 0);
    const double v = pos ? nm / d : 0.0;
    const double ws = pos ? d : (ok ? qd * 0x1p-62 : 0.0);
    for (int j = 0; j < a.w; ++j) {
      if (a.out[j]) a.out[j][i] = v;
      if (a.wsum[j]) a.wsum[j][i] = ws;
      if (a.fm[j]) a.fm[j][i] = ok ? static_cast<float>(v) : 0.f;
      if (a.valid[j]) a.valid[j][i] = ok ? 1 : 0;
    }
  }
}

}  // namespace

int launch_fix_finish_peers(const FixAcc* accs, int w, int64_t lo, int64_t hi, double* const* out,
                            double* const* wsum, float* const* fm, uint8_t* const* valid,
                            cudaStream_t s) {
  PXST_REQUIRE(w >= 1 && w <= kMaxPeers, "peer count out of range");
  if (hi <= lo) return PXST_OK;
  PeerFinish a{};
  for (int j = 0; j < w; ++j) {
    a.acc[j] = accs[j];
    a.out[j] = out ? out[j] : nullptr;
    a.wsum[j] = wsum ? wsum[j] : nullptr;
    a.fm[j] = fm ? fm[j] : nullptr;
    a.valid[j] = valid ? valid[j] : nullptr;
  }
  a.w = w;
  a.lo = lo;
  a.hi = hi;
  k_fix_finish_peers<<<grid_1d(hi - lo, 256), 256, 0, s>>>(a);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int check_scan(const pxst_scan* sc);

int launch_abs_max(const pxst_scan* sc, double* out, cudaStream_t s) {
  PXST_CHECK_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
  const int64_t n = sc->n_frames * sc->ss * sc->fs;
  if (n <= 0) return PXST_OK;
  k_abs_max<<<148 * 8, 256, 0, s>>>(sc->frames, n, out);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

int launch_quanta_job(const QuantaJob& j, cudaStream_t s) {
  const int64_t n_roi = (j.sc.roi[1] - j.sc.roi[0]) * (j.sc.roi[3] - j.sc.roi[2]);
  const int64_t n_ref = j.valid ? j.os * j.of : 0;
  const int g = std::min(grid_1d(std::max(std::max(n_roi, n_ref), j.n_zero), 256), 8 * 148);
  Scratch part;
  if (j.quanta)
    if (int e = part.alloc(3 * sizeof(double) * g, s)) return e;
  k_quanta_pass<<<g, 256, 0, s>>>(j, part.as<double>());
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

int launch_quanta(const pxst_scan* sc, const double* absmax, const double* sigma2,
                  const pxst_ref* ref, int kind, double* quanta, cudaStream_t s) {
  Scratch t;
  if (int e = t.alloc(sizeof(unsigned), s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(t.p, 0, sizeof(unsigned), s));
  QuantaJob j{};
  j.sc = *sc;
  j.sigma2 = kind == 1 ? sigma2 : nullptr;
  if (ref) {
    j.fm64 = ref->fm64;
    j.fm = ref->fm;
    j.valid = ref->valid;
    j.os = ref->os;
    j.of = ref->of;
  }
  j.absmax = absmax;
  j.kind = kind;
  j.quanta = quanta;
  j.ticket = t.as<unsigned>();
  return launch_quanta_job(j, s);
}

// Frame slices (grid.z) of a pass over nk frames with n_cta tiles when
// `resident` CTAs fit the GPU: balanced slices (sizes differ by at most one
// frame), their number chosen by a wave model -- ceil(CTAs / resident) waves,
// each costing a slice's frames plus the per-CTA setup (bounding box,
// histogram, frame table: about kSetupFrames frames' worth of instructions).
// (Round 2 used ~3 waves of slices rounded up to 8 frames: 121 frames gave
// five slices of 24 and one of a single frame, 13 % of the instructions.)
constexpr int kSetupFrames = 4;
static void fix_slices(int64_t nk, int64_t n_cta, int64_t resident, int64_t* n_z, int64_t* fpz) {
  int64_t best_z = 1;
  double best = 0.0;
  const int64_t zmax = nk < 64 ? (nk < 1 ? 1 : nk) : 64;
  for (int64_t z = 1; z <= zmax; ++z) {
    const int64_t f = (nk + z - 1) / z;
    const int64_t zz = (nk + f - 1) / f;                   // slices actually used
    const int64_t waves = (n_cta * zz + resident - 1) / resident;
    const double cost = static_cast<double>(waves) * static_cast<double>(f + kSetupFrames);
    if (z == 1 || cost < best) { best = cost; best_z = zz; }
  }
  *fpz = (nk + best_z - 1) / best_z;
  if (*fpz < 1) *fpz = 1;
  *n_z = (nk + *fpz - 1) / *fpz;
  if (*n_z < 1) *n_z = 1;
}

template <int MODE>
int launch_fix_pass(FixArgs& a, int* n_z_out, cudaStream_t s) {
  if (const char* v = getenv("PXST_FIX_NO_REGION")) a.no_region = v[0] == '1';
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2], rw = a.sc.roi[1] - a.sc.roi[0];
  dim3 g((unsigned)((cw + kXC - 1) / kXC), (unsigned)((rw + kXR - 1) / kXR));
  PXST_REQUIRE(g.y <= kMaxGridY, "ROI too tall");
  a.n_cta = (int64_t)g.x * g.y;
  const int64_t nk = a.k_hi - a.k_lo;
  constexpr size_t smem = fix_smem_bytes<MODE>();
  PXST_CHECK_CUDA(cudaFuncSetAttribute(k_fix_pass<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  // frame slices (grid.z): ~3 waves of resident CTAs when the ROI alone
  // cannot fill the GPU
  int dev = 0, sms = 148, per_sm = 1;
  PXST_CHECK_CUDA(cudaGetDevice(&dev));
  PXST_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PXST_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fix_pass<MODE>, kXT,
                                                                smem));
  const int64_t resident = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  int64_t n_z;
  fix_slices(nk, a.n_cta, resident, &n_z, &a.frames_per_z);
  g.z = static_cast<unsigned>(n_z);
  if (n_z_out) *n_z_out = static_cast<int>(n_z);
  if (nk <= 0) return PXST_OK;
  k_fix_pass<MODE><<<g, kXT, smem, s>>>(a);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

// slices the launch would use (the caller sizes pix_part with it)
int fix_pass_slices(const pxst_scan* sc, int64_t nk, int mode, int64_t* n_cta) {
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  const int64_t ctas = ((cw + kXC - 1) / kXC) * ((rw + kXR - 1) / kXR);
  if (n_cta) *n_cta = ctas;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = mode == 2 ? fix_smem_bytes<2>() : mode == 1 ? fix_smem_bytes<1>() : fix_smem_bytes<0>();
  if (mode == 2) {
    cudaFuncSetAttribute(k_fix_pass<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fix_pass<2>, kXT, smem);
  } else if (mode == 1) {
    cudaFuncSetAttribute(k_fix_pass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fix_pass<1>, kXT, smem);
  } else {
    cudaFuncSetAttribute(k_fix_pass<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fix_pass<0>, kXT, smem);
  }
  const int64_t resident = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  int64_t n_z, fpz;
  fix_slices(nk, ctas, resident, &n_z, &fpz);
  return static_cast<int>(n_z);
}

template int launch_fix_pass<0>(FixArgs&, int*, cudaStream_t);
template int launch_fix_pass<1>(FixArgs&, int*, cudaStream_t);
template int launch_fix_pass<2>(FixArgs&, int*, cudaStream_t);

int launch_fix_finish(const FixAcc& acc, const int64_t* grid, int64_t n, double* out, double* wsum,
                      float* fm, uint8_t* valid, cudaStream_t s) {
  if (n <= 0) return PXST_OK;
  k_fix_finish<<<grid_1d(n, 256), 256, 0, s>>>(acc, grid, n, out, wsum, fm, valid);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

}  // namespace pxst

namespace pxst {

int launch_object_fix(const pxst_scan* sc, const double* u, const double* di, const double* dj,
                      int64_t n0, int64_t m0, int64_t os, int64_t of, int64_t frame_lo,
                      int64_t frame_hi, const FixAcc& acc, unsigned long long* n_drop,
                      cudaStream_t s) {
  FixArgs a{};
  a.sc = *sc;
  a.u = u;
  a.di = di;
  a.dj = dj;
  a.n0 = n0;
  a.m0 = m0;
  a.os = os;
  a.of = of;
  a.k_lo = frame_lo;
  a.k_hi = frame_hi;
  a.A = acc;
  a.n_drop = n_drop;
  return launch_fix_pass<0>(a, nullptr, s);
}

}  // namespace pxst

namespace pxst {

int launch_error_fix(const pxst_scan* sc, const pxst_ref* ref, const double* u, const double* di,
                     const double* dj, const double* sigma2, const double2* grp, const FixAcc& plane,
                     const FixAcc* next, const int64_t* grid_b, int64_t cap_b, double* pix_part,
                     double* part, int* n_z, int64_t* n_cta, cudaStream_t s) {
  FixArgs a{};
  a.sc = *sc;
  a.u = u;
  a.di = di;
  a.dj = dj;
  a.n0 = ref->n0;
  a.m0 = ref->m0;
  a.os = ref->os;
  a.of = ref->of;
  a.k_lo = 0;
  a.k_hi = sc->n_good;
  a.A = plane;
  a.grp = grp;
  a.sigma2 = sigma2;
  a.pix_part = pix_part;
  a.part = part;
  int e;
  if (next) {
    a.B = *next;
    a.grid_b = grid_b;
    a.cap_b = cap_b;
    e = launch_fix_pass<2>(a, n_z, s);
  } else {
    e = launch_fix_pass<1>(a, n_z, s);
  }
  if (n_cta) *n_cta = a.n_cta;
  return e;
}

}  // namespace pxst
