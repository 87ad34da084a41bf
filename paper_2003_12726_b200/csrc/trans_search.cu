// K3: per-frame translation grid search (recon.py:336-385).
//
// err(n, a, b) = sum over work pixels of the masked-bilinear residual^2 at
// u - (delta_n + off) - origin (note the minus sign, recon.py:373-374).
//
// Pipeline (integer grids and sub-pixel grids with integral 1/step):
//   1. k_tile_geo3   per 16x64 pixel tile: u bounding box and span; the host
//                    sizes the TMA box from the largest span.
//   2. k_trans_fast  one CTA per searched frame walks every tile of the ROI:
//                    each tile's object window for the frame is fetched by TMA
//                    into a 4-slot ring (mbarrier full/empty), every thread
//                    (4 pixels per tile) runs the FFMA2 trial engine into
//                    registers across all tiles, one deterministic CTA
//                    reduction (float64) writes partial[frame][trial].  Samples
//                    whose patch leaves the grid or touches an invalid cell are
//                    skipped; their tiles are flagged in a per-frame bitmap and
//                    the frame is listed.
//   3. k_trans_slow  one block per listed frame: its 8 warps take the frame's
//                    flagged tiles in turn, re-derive eligibility over each
//                    tile's pixels lane-parallel and, for every skipped sample,
//                    evaluate the trials with lanes over trials (exact masked
//                    read of the NaN-encoded reference, (I-W)^2 fallback) into
//                    registers; the warps' sums are added in warp order, one
//                    add per trial into the frame's partial (deterministic).
//   4. k_trans_epilogue per frame: normalise by sum_p (I_n-W)^2 in place,
//                    first-occurrence argmin, always-on paraboloid when interior
//                    (grid-index units added in pixels).
// Sub-pixel grids with q = 1/step integral decompose into q^2 phase groups:
// trial k = q m + rho sits at floor(x - step*rho) - m with fractions common
// to every m, i.e. an integer window of the same engine (one launch per
// phase).  Other grids use k_trans_generic (float64, CTA per (frame, trial)).
#include <stdio.h>
#include <stdlib.h>

#include "search_common.cuh"
#include "tma.cuh"

namespace pxst {

int check_scan(const pxst_scan* sc);

namespace {

constexpr int kTR = 16, kTC = 64;           // pixel tile
constexpr int kThreads = 256;              // 8 warps: warp w -> tile rows 2w, 2w+1
constexpr int kNB = 4;                      // TMA ring depth
constexpr int kSlowPerLane = 6;             // ceil(max phase window 13x13 / 32)

struct TransArgs {
  pxst_scan sc;
  const double* u;
  const double* di;
  const double* dj;
  const float* fm;
  const uint8_t* valid;
  const uint8_t* pv;         // patch-valid map for the union box over phases
  const float* fmn;          // NaN-encoded reference (slow fix-up)
  int64_t os, of, n0, m0;
  const TileGeo* geo;        // [n_bands][n_ct]
  const int4* rec16;         // per-pixel records in the fast kernel's (tile, e, thread) order:
  const float2* rec8;        //   (floor u0, floor u1, frac u0, frac u1), (W or 0, pixel offset)
  int n_ct;                  // column tiles per band
  int64_t n_bands;
  int64_t n_tiles;           // n_bands * n_ct
  int64_t frame_lo;          // first searched frame of this launch (index into good)
  // phase group
  double ph_a, ph_b;         // sub-pixel phase shifts step*rho (0 for integer grids)
  int mhi_a, mhi_b;          // largest integer step m of the phase group
  int ka, kb;                // phase window (= template args in the fast kernel)
  int q_a, q_b;              // steps per pixel (1/step)
  int rho_a, rho_b;
  int kh_a, kh_b;            // full-grid half counts (offset index = k + kh)
  int na_full, nb_full;
  int box_r, box_c;          // TMA box
  double* partial;           // [chunk frames][na_full*nb_full]
  unsigned long long* tilebits;    // [chunk frames][words] flagged tiles
  int tile_words;
  unsigned* slow_list;       // frames (within the chunk) with flagged tiles
  unsigned* slow_n;
  unsigned long long* dbg;   // nullable debug counters (PXST_DEBUG)
  const int* sat;            // summed-area table of pv == 0, [(os + 1)][(of + 1)] (nullable)
};

// Summed-area table of the patch-invalid cells (two passes: rows, then
// columns), so a (tile, frame) can ask "is every sample base of this tile on a
// patch-valid cell?" with four loads that do not depend on the samples'
// geometry -- the per-sample patch-valid lookup was the one load of the fast
// kernel that waits for the sample's own floor (28 % of the 7 x 7 kernel's
// stall samples sat on the long scoreboard).
__global__ void k_sat_rows(const uint8_t* __restrict__ pv, int os, int of, int* __restrict__ sat) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > os) return;
  int* row = sat + (int64_t)r * (of + 1);
  row[0] = 0;
  if (r == 0) {
    for (int c = 0; c < of; ++c) row[c + 1] = 0;
    return;
  }
  int acc = 0;
  const uint8_t* p = pv + (int64_t)(r - 1) * of;
  for (int c = 0; c < of; ++c) {
    acc += p[c] == 0 ? 1 : 0;
    row[c + 1] = acc;
  }
}
__global__ void k_sat_cols(int os, int of, int* __restrict__ sat) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > of) return;
  int acc = 0;
  for (int r = 0; r <= os; ++r) {
    int* q = sat + (int64_t)r * (of + 1) + c;
    acc += *q;
    *q = acc;
  }
}
// invalid cells among rows [r0, r1] x columns [c0, c1] (inclusive, inside the grid)
__device__ __forceinline__ int sat_count(const int* __restrict__ sat, int of, int r0, int r1, int c0,
                                         int c1) {
  const int w = of + 1;
  return __ldg(sat + (r1 + 1) * w + (c1 + 1)) - __ldg(sat + r0 * w + (c1 + 1)) -
         __ldg(sat + (r1 + 1) * w + c0) + __ldg(sat + r0 * w + c0);
}

// Boxes cover a 16x64 tile's footprint; the host grows them from the measured spans.
__host__ __device__ inline int box_rows3(int ka) { return ka + 24; }
__host__ __device__ inline int box_cols3(int kb) { return ((kb + 76 + 3) / 4) * 4; }
// Window rows / cols beyond the tile's u span: the patch, one of floor()
// slack, one for the sub-pixel phase shift, and 3 columns of box alignment.
__host__ __device__ inline int need_rows3(int ka) { return ka + 3; }
__host__ __device__ inline int need_cols3(int kb) { return kb + 6; }

// ---------------------------------------------------------------------------
// 1. tile geometry (16 x 64 tiles)
// ---------------------------------------------------------------------------
__global__ void k_tile_geo3(pxst_scan sc, const double* __restrict__ u, TileGeo* geo) {
  __shared__ double red[kThreads / 32][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t plane = sc.ss * sc.fs;
  double mn0 = INFINITY, mx0 = -INFINITY, mn1 = INFINITY, mx1 = -INFINITY;
  for (int e = threadIdx.x; e < kTR * kTC; e += kThreads) {
    const int64_t row = sc.roi[0] + (int64_t)blockIdx.y * kTR + e / kTC;
    const int64_t col = sc.roi[2] + (int64_t)blockIdx.x * kTC + e % kTC;
    if (row >= sc.roi[1] || col >= sc.roi[3]) continue;
    const int64_t p = row * sc.fs + col;
    if (!sc.work[p]) continue;
    mn0 = fmin(mn0, u[p]); mx0 = fmax(mx0, u[p]);
    mn1 = fmin(mn1, u[plane + p]); mx1 = fmax(mx1, u[plane + p]);
  }
  mn0 = warp_min(mn0); mx0 = warp_max(mx0); mn1 = warp_min(mn1); mx1 = warp_max(mx1);
  if (lane == 0) { red[warp][0] = mn0; red[warp][1] = mx0; red[warp][2] = mn1; red[warp][3] = mx1; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < kThreads / 32; ++w) {
    mn0 = fmin(red[0][0], red[w][0]); red[0][0] = mn0;
    mx0 = fmax(red[0][1], red[w][1]); red[0][1] = mx0;
    mn1 = fmin(red[0][2], red[w][2]); red[0][2] = mn1;
    mx1 = fmax(red[0][3], red[w][3]); red[0][3] = mx1;
  }
  mn0 = red[0][0]; mx0 = red[0][1]; mn1 = red[0][2]; mx1 = red[0][3];
  geo[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = make_tile_geo(mn0, mx0, mn1, mx1);
}

struct Sample3 {
  int i, j;
  double fx, fy;
  int lr, lc;
  bool fast;
};

// Geometry of one (frame, pixel) sample for the current phase, shared by the
// fast and slow kernels.  x_rho = (u0 - d - n0) - step*rho; trial m sits at
// floor(x_rho) - m; the engine patch starts at floor(x_rho) - mhi.
__device__ __forceinline__ Sample3 make_sample3(const TransArgs& a, const TileGeo& g, double u0,
                                                double u1, double dI, double dJ) {
  const double n0d = static_cast<double>(a.n0), m0d = static_cast<double>(a.m0);
  Sample3 s;
  const double x = (u0 - dI - n0d) - a.ph_a;
  const double y = (u1 - dJ - m0d) - a.ph_b;
  const double xf = floor(x), yf = floor(y);
  s.fx = x - xf;
  s.fy = y - yf;
  const bool finite = fabs(x) < 1e9 && fabs(y) < 1e9;
  s.i = finite ? static_cast<int>(xf) : -(1 << 30);
  s.j = finite ? static_cast<int>(yf) : -(1 << 30);
  s.fast = false;
  s.lr = s.lc = 0;
  if (tile_fits(g, need_rows3(a.ka), need_cols3(a.kb), a.box_r, a.box_c)) {
    const int wr0 = static_cast<int>(floor((g.umin0 - dI - n0d) - a.ph_a)) - a.mhi_a;
    const int wc0 = align4_down(static_cast<int>(floor((g.umin1 - dJ - m0d) - a.ph_b)) - a.mhi_b);
    s.lr = s.i - a.mhi_a - wr0;
    s.lc = s.j - a.mhi_b - wc0;
    s.fast = s.i >= 0 && s.i < a.os && s.j >= 0 && s.j < a.of &&
             a.pv[(int64_t)s.i * a.of + s.j] != 0 && s.lr >= 0 && s.lr + a.ka + 1 <= a.box_r &&
             s.lc >= 0 && s.lc + a.kb + 1 <= a.box_c;
  }
  return s;
}

// Per-pixel records (k_k3_records, once per call): what the fast kernel needs
// of a pixel, in the order its threads read it -- record (it, e, tid) for tile
// it, pixel slot e of thread tid (tile_pixel).
// rec16 = (floor u0, floor u1, bits of frac u0, bits of frac u1) with u split
// in float64 once (floor exact, fraction rounded to float32); rec8 = (W for a
// work pixel else 0, bits of the pixel's 32-bit offset in a frame).  A frame's
// CTA then needs one 16-byte and one 8-byte load per pixel plus the stack
// value, and no 64-bit row / column arithmetic (ncu: half of the 7 x 7
// kernel's instructions were per-sample loads, address arithmetic and float64
// geometry).  i0 = kNoPixel marks pixels off the ROI / work set / not finite.
constexpr int kNoPixel = 1 << 30;
__device__ __forceinline__ int64_t rec_index(int64_t it, int e, int tid) {
  return (it * 4 + e) * kThreads + tid;
}
// Pixel slot e of thread tid -> (row, column) inside the 16 x 64 tile, and back.
// 0 (default): a warp = 32 pixels of one row (rows 2w + (e >> 1), columns
// lane + 32 (e & 1)).  PXST_K3_BLOCKS = 1: a warp's lanes form a 4 x 8 pixel
// block per slot (rows 4e .. 4e+3, columns 8w .. 8w+7, row pitch = 8 mod 32)
// as in K2.  ncu puts 33 % of the row mapping's shared-memory wavefronts on
// bank conflicts, yet the block mapping measured slower (config 3: 34.1 vs
// 31.9 ms, config 4: 289 vs 285 ms): its stack reads are four 32-byte pieces
// per warp instead of one 128-byte line.
#ifndef PXST_K3_BLOCKS
#define PXST_K3_BLOCKS 0
#endif
__device__ __forceinline__ void tile_pixel(int e, int tid, int& tr, int& tc) {
  const int lane = tid & 31, warp = tid >> 5;
  if (PXST_K3_BLOCKS) {
    tr = 4 * e + (lane >> 3);
    tc = 8 * warp + (lane & 7);
  } else {
    tr = 2 * warp + (e >> 1);
    tc = lane + 32 * (e & 1);
  }
}
__device__ __forceinline__ int64_t rec_index_of(int64_t it, int tr, int tc) {
  if (PXST_K3_BLOCKS) return rec_index(it, tr >> 2, (tc >> 3) * 32 + ((tr & 3) << 3) + (tc & 7));
  return rec_index(it, (tr & 1) * 2 + (tc >> 5), (tr >> 1) * 32 + (tc & 31));
}
__global__ void __launch_bounds__(kThreads) k_k3_records(pxst_scan sc, const double* __restrict__ u,
                                                        int n_ct, int4* __restrict__ rec16,
                                                        float2* __restrict__ rec8) {
  const int64_t it = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int64_t plane = sc.ss * sc.fs;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int tr, tc;
    tile_pixel(e, threadIdx.x, tr, tc);
    const int64_t row = sc.roi[0] + (int64_t)blockIdx.y * kTR + tr;
    const int64_t col = sc.roi[2] + (int64_t)blockIdx.x * kTC + tc;
    const bool in = row < sc.roi[1] && col < sc.roi[3];
    const int64_t p = in ? row * sc.fs + col : 0;
    bool live = in && sc.work[p] != 0 && plane < (int64_t(1) << 31);
    int4 r = make_int4(kNoPixel, 0, 0, 0);
    if (live) {
      const double u0 = u[p], u1 = u[plane + p];
      live = fabs(u0) < 1e9 && fabs(u1) < 1e9;
      if (live) {
        const double a = floor(u0), b = floor(u1);
        r = make_int4(static_cast<int>(a), static_cast<int>(b),
                      __float_as_int(static_cast<float>(u0 - a)),
                      __float_as_int(static_cast<float>(u1 - b)));
      }
    }
    const int64_t k = rec_index(it, e, threadIdx.x);
    rec16[k] = r;
    rec8[k] = make_float2(live ? sc.w32[p] : 0.f, __int_as_float(static_cast<int>(p)));
  }
}

// Frame constants of the split geometry: d + origin + phase = id + fd per axis.
struct FrameSplit {
  int id0, id1;
  float fd0, fd1;
  bool ok;
};
__device__ __forceinline__ FrameSplit frame_split(const TransArgs& a, double dI, double dJ) {
  const double x = (dI + static_cast<double>(a.n0)) + a.ph_a;
  const double y = (dJ + static_cast<double>(a.m0)) + a.ph_b;
  FrameSplit f;
  f.ok = fabs(x) < 1e9 && fabs(y) < 1e9;
  const double xa = f.ok ? floor(x) : 0.0, ya = f.ok ? floor(y) : 0.0;
  f.id0 = static_cast<int>(xa);
  f.id1 = static_cast<int>(ya);
  f.fd0 = f.ok ? static_cast<float>(x - xa) : 0.f;
  f.fd1 = f.ok ? static_cast<float>(y - ya) : 0.f;
  return f;
}

// Sample geometry from a pixel record and the frame split: x = (iu - id) +
// (fu - fd), one float32 subtract and a carry per axis.  The base may differ
// from make_sample3's float64 floor by one where x is within ~1e-7 of an
// integer; the trial positions, and so the bilinear values (continuous there:
// a fast sample's patch is valid and on the grid), are the same to float32
// rounding.  Both the fast kernel and the fix-up's classification use this
// function; the fix-up's exact trials keep make_sample3's float64 split.
struct Sample3f {
  int i, j;
  float fx, fy;
  int lr, lc;
  bool pre;
  uint8_t pvb;
  __device__ __forceinline__ bool fast() const { return pre && pvb != 0; }
};
__device__ __forceinline__ Sample3f make_sample3_split(const TransArgs& a, int4 r,
                                                       const FrameSplit& f, bool fits, int wr0,
                                                       int wc0, bool allv = false) {
  Sample3f s;
  float dx = __int_as_float(r.z) - f.fd0, dy = __int_as_float(r.w) - f.fd1;
  int i = r.x - f.id0, j = r.y - f.id1;
  if (dx < 0.f) { dx += 1.f; --i; }
  if (dy < 0.f) { dy += 1.f; --j; }
  if (dx >= 1.f) { dx = 0.f; ++i; }
  if (dy >= 1.f) { dy = 0.f; ++j; }
  s.fx = dx;
  s.fy = dy;
  const bool on = r.x != kNoPixel && f.ok;
  s.i = on ? i : -(1 << 30);
  s.j = on ? j : -(1 << 30);
  s.lr = s.i - a.mhi_a - wr0;
  s.lc = s.j - a.mhi_b - wc0;
  const int os = static_cast<int>(a.os), of = static_cast<int>(a.of);
  const bool in = static_cast<unsigned>(s.i) < static_cast<unsigned>(os) &&
                  static_cast<unsigned>(s.j) < static_cast<unsigned>(of);
  // allv (warp-uniform): every sample base of this tile and frame is on a
  // patch-valid cell (sat_count == 0 over the tile's base rectangle): no lookup
  s.pvb = allv ? 1 : (fits ? __ldg(a.pv + (in ? s.i * of + s.j : 0)) : 0);
  s.pre = fits && in && static_cast<unsigned>(s.lr) <= static_cast<unsigned>(a.box_r - a.ka - 1) &&
          static_cast<unsigned>(s.lc) <= static_cast<unsigned>(a.box_c - a.kb - 1);
  return s;
}

// full-grid trial index of phase-local engine trial (t, s)
__device__ __forceinline__ int full_index(const TransArgs& a, int t, int s) {
  const int ia = a.q_a * (a.mhi_a - t) + a.rho_a + a.kh_a;
  const int ib = a.q_b * (a.mhi_b - s) + a.rho_b + a.kh_b;
  return ia * a.nb_full + ib;
}

// ---------------------------------------------------------------------------
// 2. fast kernel: one CTA per searched frame
// ---------------------------------------------------------------------------
template <int KA, int KB>
#ifndef PXST_K3_OCC2_BELOW
#define PXST_K3_OCC2_BELOW 82   // up to 9 x 9 at 2 CTAs/SM: the 128-register cap spills a few
                                  // values but the doubled warps win (config 4: -11 %)
#endif
#ifndef PXST_K3_OCC3_BELOW
#define PXST_K3_OCC3_BELOW 0
#endif
__global__ void __launch_bounds__(kThreads, (KA * KB < PXST_K3_OCC3_BELOW)   ? 3
                                            : (KA * KB < PXST_K3_OCC2_BELOW) ? 2
                                                                             : 1)
    k_trans_fast(const __grid_constant__ CUtensorMap tmap, TransArgs a) {
  extern __shared__ __align__(128) unsigned char ring_raw[];
  __shared__ __align__(8) uint64_t full[kNB], empty[kNB];
  __shared__ double red[kThreads / 32][KA * KB];
  __shared__ int any_flag;
  unsigned char* base = ring_raw + ((128u - (smem_addr(ring_raw) & 127u)) & 127u);
  float* ring = reinterpret_cast<float*>(base);
  const int box = slot_floats(a.box_r, a.box_c);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t kk = blockIdx.x;                     // frame within this launch's chunk
  const int64_t f = a.sc.good[a.frame_lo + kk];
  const double dI = a.di[f], dJ = a.dj[f];
  const int64_t plane = a.sc.ss * a.sc.fs;
  const float* frame = a.sc.frames + f * plane;
  const double n0d = static_cast<double>(a.n0), m0d = static_cast<double>(a.m0);
  const unsigned bytes = static_cast<unsigned>(a.box_r * a.box_c * sizeof(float));
  unsigned long long* bits = a.tilebits + kk * a.tile_words;

  PackedAcc<KA, KB> acc;
  acc.zero();

  auto issue = [&](int64_t it) {
    const TileGeo g = a.geo[it];
    const int b = static_cast<int>(it % kNB);
    if (tile_fits(g, need_rows3(KA), need_cols3(KB), a.box_r, a.box_c)) {
      const int wr0 = static_cast<int>(floor((g.umin0 - dI - n0d) - a.ph_a)) - a.mhi_a;
      const int wc0 =
          align4_down(static_cast<int>(floor((g.umin1 - dJ - m0d) - a.ph_b)) - a.mhi_b);
      mbar_arrive_expect_tx(&full[b], bytes);
      tma_load_2d(ring + b * box, &tmap, wc0, wr0, &full[b]);
    } else {
      mbar_arrive(&full[b]);           // nothing to fetch: complete the phase directly
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmap);
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kThreads);
    }
    mbar_fence_init();
    any_flag = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int64_t it = 0; it < (a.n_tiles < kNB ? a.n_tiles : kNB); ++it) issue(it);

  // Per-pixel inputs from the records (k_k3_records) and the stack; windows of
  // 9 x 9 and more (1 CTA per SM, registers to spare) fetch tile it + 1's while
  // tile it runs.
  struct Raw3 {
    int4 r16[4];
    float W[4], I[4];
  };
  auto load_raw = [&](int64_t it, Raw3& R) {
    const int4* r16 = a.rec16 + rec_index(it, 0, threadIdx.x);
    const float2* r8 = a.rec8 + rec_index(it, 0, threadIdx.x);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      R.r16[e] = __ldg(r16 + e * kThreads);
      const float2 w = __ldg(r8 + e * kThreads);
      R.W[e] = w.x;
      R.I[e] = __ldg(frame + static_cast<unsigned>(__float_as_int(w.y)));
    }
  };
  constexpr bool kPipe = !(KA * KB < PXST_K3_OCC2_BELOW);
  Raw3 nxt;
  if (kPipe) load_raw(0, nxt);
  const FrameSplit fs_ = frame_split(a, dI, dJ);

  for (int64_t it = 0; it < a.n_tiles; ++it) {
    const int b = static_cast<int>(it % kNB);
    const unsigned ph = static_cast<unsigned>((it / kNB) & 1);
    const TileGeo g = a.geo[it];
    Raw3 cur;
    if (kPipe) {
      cur = nxt;
      if (it + 1 < a.n_tiles) load_raw(it + 1, nxt);
    } else {
      load_raw(it, cur);
    }
    // the tile's window origin for this frame (as issue() computed it)
    const bool fits = tile_fits(g, need_rows3(KA), need_cols3(KB), a.box_r, a.box_c);
    const int wr0 = static_cast<int>(floor((g.umin0 - dI - n0d) - a.ph_a)) - a.mhi_a;
    const int jb = static_cast<int>(floor((g.umin1 - dJ - m0d) - a.ph_b));
    const int wc0 = align4_down(jb - a.mhi_b);
    // the tile's sample bases lie in rows [wr0 + mhi_a, + span_r + 1], columns
    // [jb, + span_c + 1] (one more each side: the float32 split may move a
    // base by one where x is within 1e-7 of an integer)
    bool allv = false;
    if (a.sat && fits) {
      const int i0 = wr0 + a.mhi_a - 1, i1 = wr0 + a.mhi_a + g.span_r + 2;
      const int j0 = jb - 1, j1 = jb + g.span_c + 2;
      if (i0 >= 0 && j0 >= 0 && i1 < static_cast<int>(a.os) && j1 < static_cast<int>(a.of))
        allv = sat_count(a.sat, static_cast<int>(a.of), i0, i1, j0, j1) == 0;
    }
    float I[4], W[4], fx[4], fy[4];
    int off[4];                        // patch origin offset in the slot, -1 = not fast
    bool tile_slow = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool live = cur.r16[e].x != kNoPixel;
      I[e] = cur.I[e];
      W[e] = cur.W[e];                 // 0 off the work set
      const Sample3f sm = make_sample3_split(a, cur.r16[e], fs_, fits, wr0, wc0, allv);
      fx[e] = sm.fx;
      fy[e] = sm.fy;
      off[e] = (live && sm.fast()) ? sm.lr * a.box_c + sm.lc : -1;
      tile_slow |= live && !sm.fast();
      if (a.dbg && live) {   // [samples, !fits, !in-grid, !pv, !box]
        atomicAdd(a.dbg, 1ull);
        if (!sm.fast()) {
          const bool ing = sm.i >= 0 && sm.i < a.os && sm.j >= 0 && sm.j < a.of;
          if (!fits)
            atomicAdd(a.dbg + 1, 1ull);
          else if (!ing) atomicAdd(a.dbg + 2, 1ull);
          else if (!a.pv[(int64_t)sm.i * a.of + sm.j]) atomicAdd(a.dbg + 3, 1ull);
          else atomicAdd(a.dbg + 4, 1ull);
        }
      }
    }
    if (__any_sync(0xffffffffu, tile_slow) && lane == 0) {
      atomicOr(&bits[it >> 6], 1ull << (it & 63));
      any_flag = 1;
    }
    mbar_wait(&full[b], ph);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      PXST_DCHECK(off[e] < 0 || off[e] + KA * a.box_c + KB + a.box_c + 1 < box);
      if (off[e] >= 0)
        engine_fast2<KA, KB>(ring + b * box + off[e], a.box_c, fx[e], fy[e],
                             W[e] * (1.f - fx[e]), W[e] * fx[e], I[e], acc);
    }
    mbar_arrive(&empty[b]);
    if (threadIdx.x == 0 && it + kNB < a.n_tiles) {
      mbar_wait(&empty[b], ph);
      issue(it + kNB);
    }
  }
  // deterministic CTA reduction: float32 warp shuffles, then a fixed-order
  // float64 sum of the warps
#pragma unroll
  for (int t = 0; t < KA; ++t)
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      const float v = warp_sumf(acc.get(t, s));
      if (lane == 0) red[warp][t * KB + s] = static_cast<double>(v);
    }
  __syncthreads();
  double* out = a.partial + kk * (int64_t)(a.na_full * a.nb_full);
  for (int e = threadIdx.x; e < KA * KB; e += kThreads) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) v += red[w][e];
    out[full_index(a, e / KB, e % KB)] = v;
  }
  if (any_flag && threadIdx.x == 0) {   // hand the flagged tiles to k_trans_slow
    const unsigned slot = atomicAdd(a.slow_n, 1u);
    a.slow_list[slot] = static_cast<unsigned>(kk);
  }
}

// ---------------------------------------------------------------------------
// 3. slow fix-up: warp per listed frame
// ---------------------------------------------------------------------------
// One block per listed frame: its 8 warps take the frame's flagged tiles in
// turn (a warp per frame left the launch waiting on the frame with the most
// flagged tiles), then the warps' partial sums are added in warp order.
constexpr int kSlowWarps = 8;
__global__ void __launch_bounds__(32 * kSlowWarps) k_trans_slow(TransArgs a) {
  __shared__ float red[kSlowWarps][kSlowPerLane * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned n = *a.slow_n;
  const int nk_ph = a.ka * a.kb, nk = a.na_full * a.nb_full;
  const int os = static_cast<int>(a.os), of = static_cast<int>(a.of);
  int ta[kSlowPerLane], tb[kSlowPerLane];   // patch coordinates of the lane's trials
  int to[kSlowPerLane];                     // and their cell offsets from the patch corner
#pragma unroll
  for (int j = 0; j < kSlowPerLane; ++j) {
    const int t = lane + 32 * j;
    ta[j] = t / a.kb;
    tb[j] = t % a.kb;
    to[j] = ta[j] * of + tb[j];
  }
  const int64_t plane = a.sc.ss * a.sc.fs;
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2];
  for (int64_t e = blockIdx.x; e < n; e += gridDim.x) {
    const int64_t kk = a.slow_list[e];
    const int64_t f = a.sc.good[a.frame_lo + kk];
    const double dI = a.di[f], dJ = a.dj[f];
    const float* frame = a.sc.frames + f * plane;
    const unsigned long long* bits = a.tilebits + kk * a.tile_words;
    const FrameSplit fs_ = frame_split(a, dI, dJ);
    const double n0d = static_cast<double>(a.n0), m0d = static_cast<double>(a.m0);
    float part[kSlowPerLane];
#pragma unroll
    for (int j = 0; j < kSlowPerLane; ++j) part[j] = 0.f;
    int flagged = 0;
    for (int64_t it = 0; it < a.n_tiles; ++it) {
      if (!((bits[it >> 6] >> (it & 63)) & 1ull)) continue;     // only flagged tiles
      if ((flagged++ % kSlowWarps) != warp) continue;           // this warp's share
      const int64_t band = it / a.n_ct;
      const int ct = static_cast<int>(it % a.n_ct);
      const TileGeo g = a.geo[it];
      const bool fits = tile_fits(g, need_rows3(a.ka), need_cols3(a.kb), a.box_r, a.box_c);
      const int wr0 = static_cast<int>(floor((g.umin0 - dI - n0d) - a.ph_a)) - a.mhi_a;
      const int wc0 = align4_down(static_cast<int>(floor((g.umin1 - dJ - m0d) - a.ph_b)) - a.mhi_b);
      const int64_t r_lo = a.sc.roi[0] + band * kTR;
      const int64_t r_hi = min(a.sc.roi[1], r_lo + kTR);
      const int64_t c_lo = (int64_t)ct * kTC;
      const int64_t c_hi = min(cw, c_lo + kTC);
      const int64_t npx = (r_hi - r_lo) * (c_hi - c_lo);
      for (int64_t q0 = 0; q0 < npx; q0 += 32) {
        // lane-parallel classification of 32 pixels; each lane keeps its
        // sample and inputs for the broadcast below
        const int64_t ql = q0 + lane;
        bool slow = false;
        Sample3 sl{};
        float Il = 0.f, Wl = 0.f;
        if (ql < npx) {
          const int64_t rr = ql / (c_hi - c_lo), cc = c_lo + ql % (c_hi - c_lo);
          const int64_t p = (r_lo + rr) * a.sc.fs + a.sc.roi[2] + cc;
          if (a.sc.work[p]) {
            // skipped <=> the fast kernel's own test (the split geometry on the
            // pixel's record); the exact trials use the float64 split
            const int tr = static_cast<int>(rr), tc = static_cast<int>(cc - c_lo);
            const int4 r16 = a.rec16[rec_index_of(it, tr, tc)];
            slow = !make_sample3_split(a, r16, fs_, fits, wr0, wc0).fast();
            if (slow) {
              sl = make_sample3(a, g, a.u[p], a.u[plane + p], dI, dJ);
              Il = __ldg(frame + p);
              Wl = a.sc.w32[p];
            }
          }
        }
        unsigned mask = __ballot_sync(0xffffffffu, slow);
        while (mask) {
          const int bsel = __ffs(mask) - 1;
          mask &= mask - 1;
          const int pr0 = __shfl_sync(0xffffffffu, sl.i, bsel) - a.mhi_a;
          const int pc0 = __shfl_sync(0xffffffffu, sl.j, bsel) - a.mhi_b;
          const ExactSample es = exact_sample(__shfl_sync(0xffffffffu, sl.fx, bsel),
                                              __shfl_sync(0xffffffffu, sl.fy, bsel),
                                              __shfl_sync(0xffffffffu, Wl, bsel),
                                              __shfl_sync(0xffffffffu, Il, bsel), 1.f);
          if (pr0 >= 0 && pc0 >= 0 && pr0 + a.ka < os && pc0 + a.kb < of) {   // warp-uniform
            const float* w0 = a.fmn + (pr0 * of + pc0);
#pragma unroll
            for (int j = 0; j < kSlowPerLane; ++j)
              if (lane + 32 * j < nk_ph) part[j] += trial_interior(w0 + to[j], of, es);
          } else {
#pragma unroll
            for (int j = 0; j < kSlowPerLane; ++j)
              if (lane + 32 * j < nk_ph)
                part[j] += trial_global(a.fmn, os, of, pr0 + ta[j], pc0 + tb[j], es);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kSlowPerLane; ++j) red[warp][lane + 32 * j] = part[j];
    __syncthreads();
    if (warp == 0) {
      double* out = a.partial + kk * (int64_t)nk;
#pragma unroll
      for (int j = 0; j < kSlowPerLane; ++j) {
        const int t = lane + 32 * j;
        float v = red[0][t];
        for (int w = 1; w < kSlowWarps; ++w) v += red[w][t];
        if (t < nk_ph) out[full_index(a, t / a.kb, t % a.kb)] += static_cast<double>(v);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// generic (any grid): one CTA per (searched frame, full-grid trial), float64
// ---------------------------------------------------------------------------
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

// ---------------------------------------------------------------------------
// 4. per-frame epilogue
// ---------------------------------------------------------------------------
__global__ void k_trans_epilogue(pxst_scan sc, const double* __restrict__ frame_norm,
                                 double* part, int64_t frame_lo, int na,
                                 int nb, const double* __restrict__ offs_a,
                                 const double* __restrict__ offs_b, const double* di,
                                 const double* dj, double* di_out, double* dj_out,
                                 double* err_out) {
  __shared__ double bv[32];
  __shared__ int bi[32];
  const int64_t kk = blockIdx.x;
  const int64_t k = frame_lo + kk;
  const int64_t f = sc.good[k];
  const double norm = frame_norm[k];
  const int nk = na * nb;
  // normalised in place in the frame's partial row (any window size: no
  // shared-memory copy of the nk errors)
  double* e = part + kk * nk;
  if (norm > 0.0)
    for (int t = threadIdx.x; t < nk; t += blockDim.x) e[t] = e[t] / norm;
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
  if (ia > 0 && ia < na - 1 && ib > 0 && ib < nb - 1) {       // recon.py:381-382
    double q[9];
    for (int d = 0; d < 9; ++d) q[d] = e[(ia + d / 3 - 1) * nb + (ib + d % 3 - 1)];
    paraboloid(q, da, db);
  }
  di_out[f] = di[f] + offs_a[ia] + da;                        // recon.py:383-384
  dj_out[f] = dj[f] + offs_b[ib] + db;
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
using FastKernel = void (*)(const __grid_constant__ CUtensorMap, TransArgs);
struct FastEntry { int ka, kb; FastKernel fn; };
#define TR(a, b) FastEntry{a, b, k_trans_fast<a, b>}
const FastEntry kTable[] = {
    TR(1, 1), TR(3, 3), TR(5, 5), TR(7, 7), TR(9, 9), TR(11, 11), TR(13, 13),
    TR(8, 8), TR(8, 9), TR(9, 8),
};
#undef TR

FastKernel find_fast(int ka, int kb) {
  for (const auto& e : kTable)
    if (e.ka == ka && e.kb == kb) return e.fn;
  return nullptr;
}

}  // namespace
}  // namespace pxst

using namespace pxst;

namespace {
int translation_search(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref,
                       const double* u, const double* di, const double* dj, int64_t half_ss,
                       int64_t half_fs, double subpixel_step, int64_t frame_lo, int64_t frame_hi,
                       double* di_out, double* dj_out, double* err_out, const int32_t* span_hint,
                       void* stream);
}

extern "C" int pxst_translation_search(const pxst_scan* sc, const pxst_stats* st,
                                       const pxst_ref* ref, const double* u, const double* di,
                                       const double* dj, int64_t half_ss, int64_t half_fs,
                                       double subpixel_step, int64_t frame_lo, int64_t frame_hi,
                                       double* di_out, double* dj_out, double* err_out,
                                       void* stream) {
  return translation_search(sc, st, ref, u, di, dj, half_ss, half_fs, subpixel_step, frame_lo,
                            frame_hi, di_out, dj_out, err_out, nullptr, stream);
}

extern "C" int pxst_translation_search_ex(const pxst_scan* sc, const pxst_stats* st,
                                          const pxst_ref* ref, const double* u, const double* di,
                                          const double* dj, int64_t half_ss, int64_t half_fs,
                                          double subpixel_step, int64_t frame_lo,
                                          int64_t frame_hi, double* di_out, double* dj_out,
                                          double* err_out, const int32_t* span_hint,
                                          void* stream) {
  return translation_search(sc, st, ref, u, di, dj, half_ss, half_fs, subpixel_step, frame_lo,
                            frame_hi, di_out, dj_out, err_out, span_hint, stream);
}

extern "C" int pxst_tile_spans3(const pxst_scan* sc, const double* u, int32_t* spans,
                                void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(u && spans, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  const int n_ct = static_cast<int>((cw + kTC - 1) / kTC);
  const int64_t n_bands = (rw + kTR - 1) / kTR;
  PXST_REQUIRE(n_bands <= kMaxGridY, "ROI too tall");
  Scratch geo;
  if (int e = geo.alloc(sizeof(TileGeo) * n_ct * n_bands, s)) return e;
  k_tile_geo3<<<dim3((unsigned)n_ct, (unsigned)n_bands), kThreads, 0, s>>>(*sc, u,
                                                                            geo.as<TileGeo>());
  PXST_CHECK_LAUNCH();
  return tile_span_max_dev(geo.as<TileGeo>(), (int64_t)n_ct * n_bands, spans, s);
}

namespace {
int translation_search(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref,
                       const double* u, const double* di, const double* dj, int64_t half_ss,
                       int64_t half_fs, double subpixel_step, int64_t frame_lo, int64_t frame_hi,
                       double* di_out, double* dj_out, double* err_out, const int32_t* span_hint,
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
  if (int e = fill_offsets(offs.as<double>(), na, nb, subpixel_step, s)) return e;
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
  struct Phase { int rho_a, rho_b, mlo_a, mhi_a, mlo_b, mhi_b; FastKernel fn; };
  std::vector<Phase> phases;
  if (fast) {
    auto mrange = [](int q, int rho, int kh, int& lo, int& hi) {   // k = q*m + rho in [-kh, kh]
      lo = static_cast<int>(ceil((-kh - rho) / static_cast<double>(q)));
      hi = static_cast<int>(floor((kh - rho) / static_cast<double>(q)));
    };
    for (int ra_ = 0; ra_ < qa && fast; ++ra_)
      for (int rb_ = 0; rb_ < qb && fast; ++rb_) {
        Phase ph{ra_, rb_, 0, 0, 0, 0, nullptr};
        mrange(qa, ra_, kha, ph.mlo_a, ph.mhi_a);
        mrange(qb, rb_, khb, ph.mlo_b, ph.mhi_b);
        if (ph.mhi_a < ph.mlo_a || ph.mhi_b < ph.mlo_b) continue;
        ph.fn = find_fast(ph.mhi_a - ph.mlo_a + 1, ph.mhi_b - ph.mlo_b + 1);
        if (!ph.fn) fast = false;
        phases.push_back(ph);
      }
  }

  const int64_t n_search = frame_hi - frame_lo;
  // frame chunks so the partial buffer stays <= 256 MB
  int64_t chunk = (256ll << 20) / (8 * (int64_t)nk);
  chunk = chunk < kMaxGridY ? chunk : kMaxGridY;
  chunk = chunk > 1 ? chunk : 1;
  const int64_t cmax = min(chunk, n_search);
  Scratch part;
  if (int e = part.alloc(sizeof(double) * cmax * nk, s)) return e;
  a.partial = part.as<double>();

  if (fast) {
    int max_ka = 0, max_kb = 0, mhi_a = -1 << 20, mlo_a = 1 << 20, mhi_b = -1 << 20,
        mlo_b = 1 << 20;
    for (const auto& ph : phases) {
      max_ka = max(max_ka, ph.mhi_a - ph.mlo_a + 1);
      max_kb = max(max_kb, ph.mhi_b - ph.mlo_b + 1);
      mhi_a = max(mhi_a, ph.mhi_a); mlo_a = min(mlo_a, ph.mlo_a);
      mhi_b = max(mhi_b, ph.mhi_b); mlo_b = min(mlo_b, ph.mlo_b);
    }
    a.box_r = box_rows3(max_ka);
    a.box_c = box_cols3(max_kb);
    a.n_ct = static_cast<int>((cw + kTC - 1) / kTC);
    a.n_bands = (rw + kTR - 1) / kTR;
    a.n_tiles = a.n_bands * a.n_ct;
    PXST_REQUIRE(a.n_bands <= kMaxGridY, "ROI too tall");
    a.q_a = qa; a.q_b = qb; a.kh_a = kha; a.kh_b = khb;
    a.tile_words = static_cast<int>((a.n_tiles + 63) / 64);

    Scratch geo, pvbuf, fmnbuf, fmpad, lst, tb, satbuf;
    if (int e = geo.alloc(sizeof(TileGeo) * a.n_tiles, s)) return e;
    a.geo = geo.as<TileGeo>();
    k_tile_geo3<<<dim3((unsigned)a.n_ct, (unsigned)a.n_bands), kThreads, 0, s>>>(
        *sc, u, geo.as<TileGeo>());
    PXST_CHECK_LAUNCH();
    Scratch rec16, rec8;             // per-pixel records of the fast kernel (k_k3_records)
    if (int e = rec16.alloc(sizeof(int4) * a.n_tiles * 4 * kThreads, s)) return e;
    if (int e = rec8.alloc(sizeof(float2) * a.n_tiles * 4 * kThreads, s)) return e;
    k_k3_records<<<dim3((unsigned)a.n_ct, (unsigned)a.n_bands), kThreads, 0, s>>>(
        *sc, u, a.n_ct, rec16.as<int4>(), rec8.as<float2>());
    PXST_CHECK_LAUNCH();
    a.rec16 = rec16.as<int4>();
    a.rec8 = rec8.as<float2>();
    // Box from the largest tile footprint, <= 256 columns and <= 40 KB per
    // slot; tiles beyond the cap take the exact path.
    int span[2];
    if (span_hint) {             // from pxst_tile_spans3; a stale hint only costs speed
      span[0] = span_hint[0];
      span[1] = span_hint[1];
    } else if (int e = tile_span_max(geo.as<TileGeo>(), a.n_tiles, span, s)) {
      return e;
    }
    a.box_r = max(a.box_r, span[0] + need_rows3(max_ka));
    a.box_c = max(a.box_c, span[1] + need_cols3(max_kb));
    a.box_c = (a.box_c + 3) / 4 * 4;
    if (PXST_K3_BLOCKS) {        // row pitch = 8 (mod 32): a warp's 4 block rows tile the banks
      const int c8 = (a.box_c + 23) / 32 * 32 + 8;
      if (c8 <= 256) a.box_c = c8;     // (a TMA box dimension is at most 256)
    }
    if (a.box_c > 256) a.box_c = 256;
    while (a.box_r > 16 && a.box_r * a.box_c * 4 > 40 * 1024) --a.box_r;
    // union patch box over phases, relative to floor(x_rho): rows
    // [-max mhi, -min mlo + 1]
    if (int e = pvbuf.alloc(ref->os * ref->of, s)) return e;
    if (int e = fmnbuf.alloc(sizeof(float) * ref->os * ref->of, s)) return e;
    if (int e = make_pv(ref, -mhi_a, -mlo_a + 1, -mhi_b, -mlo_b + 1, pvbuf.as<uint8_t>(),
                        fmnbuf.as<float>(), s))
      return e;
    a.pv = pvbuf.as<uint8_t>();
    a.fmn = fmnbuf.as<float>();
    // Off by default (PXST_K3_SAT=1 turns it on): measured neutral to slightly
    // slower -- config 3 K3 31.15 ms without, 31.71 ms with; config 4 282.9 /
    // 283.4 ms -- the four table loads cost what the skipped lookups save.
    if (getenv("PXST_K3_SAT") && (ref->os + 1) * (ref->of + 1) < (int64_t(1) << 31)) {
      if (int e = satbuf.alloc(sizeof(int) * (ref->os + 1) * (ref->of + 1), s)) return e;
      const int os_i = static_cast<int>(ref->os), of_i = static_cast<int>(ref->of);
      k_sat_rows<<<(os_i + 1 + 127) / 128, 128, 0, s>>>(pvbuf.as<uint8_t>(), os_i, of_i,
                                                       satbuf.as<int>());
      PXST_CHECK_LAUNCH();
      k_sat_cols<<<(of_i + 1 + 127) / 128, 128, 0, s>>>(os_i, of_i, satbuf.as<int>());
      PXST_CHECK_LAUNCH();
      a.sat = satbuf.as<int>();
    }
    // TMA descriptor (16-byte row pitch)
    const float* tbase = ref->fm;
    int64_t pitch = ref->of;
    if (ref->of % 4 != 0 || (reinterpret_cast<uintptr_t>(ref->fm) & 15)) {
      pitch = (ref->of + 3) / 4 * 4;
      if (int e = fmpad.alloc(sizeof(float) * pitch * ref->os, s)) return e;
      PXST_CHECK_CUDA(cudaMemcpy2DAsync(fmpad.p, pitch * sizeof(float), ref->fm,
                                        ref->of * sizeof(float), ref->of * sizeof(float), ref->os,
                                        cudaMemcpyDeviceToDevice, s));
      tbase = fmpad.as<float>();
    }
    CUtensorMap tmap;
    if (int e = encode_tmap_2d_f32(&tmap, tbase, ref->os, ref->of, pitch, a.box_r, a.box_c))
      return e;
    const size_t smem = sizeof(float) * kNB * slot_floats(a.box_r, a.box_c) + 128;
    for (const auto& ph : phases)
      PXST_CHECK_CUDA(cudaFuncSetAttribute(ph.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    if (int e = lst.alloc(sizeof(unsigned) * (cmax + 2), s)) return e;
    a.slow_n = lst.as<unsigned>();
    a.slow_list = lst.as<unsigned>() + 1;
    const size_t tb_bytes = sizeof(unsigned long long) * cmax * a.tile_words;
    if (int e = tb.alloc(tb_bytes, s)) return e;
    a.tilebits = tb.as<unsigned long long>();
    Scratch dbg;
    if (getenv("PXST_DEBUG")) {
      if (int e = dbg.alloc(sizeof(unsigned long long) * 8, s)) return e;
      PXST_CHECK_CUDA(cudaMemsetAsync(dbg.p, 0, sizeof(unsigned long long) * 8, s));
      a.dbg = dbg.as<unsigned long long>();
    }
    for (int64_t c0 = frame_lo; c0 < frame_hi; c0 += chunk) {
      const int64_t c1 = min(frame_hi, c0 + chunk);
      a.frame_lo = c0;
      for (const auto& ph : phases) {
        a.rho_a = ph.rho_a; a.rho_b = ph.rho_b;
        a.mhi_a = ph.mhi_a; a.mhi_b = ph.mhi_b;
        a.ka = ph.mhi_a - ph.mlo_a + 1;
        a.kb = ph.mhi_b - ph.mlo_b + 1;
        a.ph_a = subpixel_step > 0.0 ? subpixel_step * ph.rho_a : 0.0;
        a.ph_b = subpixel_step > 0.0 ? subpixel_step * ph.rho_b : 0.0;
        PXST_CHECK_CUDA(cudaMemsetAsync(a.slow_n, 0, sizeof(unsigned), s));
        PXST_CHECK_CUDA(cudaMemsetAsync(a.tilebits, 0, tb_bytes, s));
        ph.fn<<<(unsigned)(c1 - c0), kThreads, smem, s>>>(tmap, a);
        PXST_CHECK_LAUNCH();
        k_trans_slow<<<148 * 4, 32 * kSlowWarps, 0, s>>>(a);
        PXST_CHECK_LAUNCH();
        if (a.dbg) {
          unsigned h = 0;
          unsigned long long d[5];
          PXST_CHECK_CUDA(cudaMemcpyAsync(&h, a.slow_n, sizeof(h), cudaMemcpyDeviceToHost, s));
          PXST_CHECK_CUDA(cudaMemcpyAsync(d, a.dbg, sizeof(d), cudaMemcpyDeviceToHost, s));
          PXST_CHECK_CUDA(cudaStreamSynchronize(s));
          fprintf(stderr, "[pxst] K3 phase (%d,%d) %dx%d: %lld frames, %lld tiles, box %dx%d, "
                  "%u frames with slow tiles; samples %llu, slow: no-fit %llu, outside %llu, "
                  "patch-invalid %llu, box %llu\n", ph.rho_a, ph.rho_b, a.ka, a.kb,
                  (long long)(c1 - c0), (long long)a.n_tiles, a.box_r, a.box_c, h, d[0], d[1],
                  d[2], d[3], d[4]);
          PXST_CHECK_CUDA(cudaMemsetAsync(a.dbg, 0, sizeof(d), s));
        }
      }
      k_trans_epilogue<<<(unsigned)(c1 - c0), 256, 0, s>>>(
          *sc, st->frame_norm, part.as<double>(), c0, na, nb, d_oa, d_ob, di, dj, di_out,
          dj_out, err_out ? err_out + (c0 - frame_lo) * nk : nullptr);
      PXST_CHECK_LAUNCH();
    }
    return PXST_OK;
  }
  // generic path
  for (int64_t c0 = frame_lo; c0 < frame_hi; c0 += chunk) {
    const int64_t c1 = min(frame_hi, c0 + chunk);
    a.frame_lo = c0;
    dim3 g((unsigned)nk, (unsigned)(c1 - c0));
    k_trans_generic<<<g, 256, 0, s>>>(a, d_oa, d_ob, part.as<double>());
    PXST_CHECK_LAUNCH();
    k_trans_epilogue<<<(unsigned)(c1 - c0), 256, 0, s>>>(
        *sc, st->frame_norm, part.as<double>(), c0, na, nb, d_oa, d_ob, di, dj, di_out, dj_out,
        err_out ? err_out + (c0 - frame_lo) * nk : nullptr);
    PXST_CHECK_LAUNCH();
  }
  return PXST_OK;
}
}  // namespace
