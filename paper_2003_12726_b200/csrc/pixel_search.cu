// K2: pixel-map grid search + argmin + paraboloid refinement
// (recon.py:144-170, 183-207, 221-296; sigma = 0, integrate = False).
//
// Pipeline for integer windows (Ka x Kb instantiated):
//   1. k_tile_geo      per 8x16 pixel tile: bounding box of u over its work
//                      pixels -> object-window origin and "window fits" flag
//                      (and u_out = u, err = 0 on the ROI when it is the
//                      whole detector).
//   2. k_pix_fast      1-D grid of work units: whole tiles over all frames
//                      (<= 512 good frames: the first full waves) and
//                      (tile, frame chunk) units for the rest.  Per frame the
//                      tile's object window (box BR x BC, shifted by delta_n)
//                      is fetched by TMA into a 4-deep shared-memory ring
//                      (mbarrier full / empty pairs), each thread runs the
//                      register trial engine for its pixel; samples whose
//                      patch leaves the grid or touches an invalid cell are
//                      skipped and listed.  Whole-tile units finish their
//                      pixels in the kernel (argmin, paraboloid); chunk units
//                      write float32 partial[chunk][trial][pixel].
//   3. k_pix_slow(_rows) one warp per listed (pixel, chunk): lanes classify 32
//                      frames at a time with the same eligibility test, then
//                      add every skipped sample's exact per-trial contribution
//                      (masked renormalised read from a NaN-encoded reference,
//                      (I-W)^2 fallback), in frame order; whole-tile pixels
//                      are finished there.
//   4. k_pix_epilogue  pixels of the chunked tiles, eight lanes per pixel:
//                      float64 sum over chunks, first-occurrence argmin (numpy
//                      order a*Kb + b), paraboloid on the normalised 3x3
//                      patch, static-pixel rule, u_out and the error map.
// Sub-pixel grids and non-instantiated windows use k_pix_generic (float64,
// one thread per (pixel, trial)) followed by the same epilogue.
#include <algorithm>
#include <stdio.h>
#include <stdlib.h>

#include "search_common.cuh"
#include "tma.cuh"

namespace pxst {

int check_scan(const pxst_scan* sc);

namespace {

// Pixel tile 8 x 16 = 2 x 2 warps, each warp a 4 x 8 pixel block.  A warp's
// lanes then read window rows spread over ~5 rows and ~8 columns; with the
// window pitch = 8 (mod 32) this cuts shared-memory bank conflicts on noisy
// maps from 2.16x (warp = one 32-pixel row) to ~1.6x and to 1.0x on smooth
// maps (model of the access pattern, confirmed by ncu).
#ifndef PXST_K2_TILE_ROWS
#define PXST_K2_TILE_ROWS 8
#endif
constexpr int kTR = PXST_K2_TILE_ROWS, kTC = 16, kThreads = kTR * kTC;
constexpr int kCtaPerSm = kThreads <= 128 ? 2 : 1;   // fast-kernel CTAs resident per SM
__device__ __forceinline__ int tile_dr(int tid) { return ((tid >> 5) >> 1) * 4 + ((tid & 31) >> 3); }
__device__ __forceinline__ int tile_dc(int tid) { return ((tid >> 5) & 1) * 8 + (tid & 7); }
#ifndef PXST_K2_RING
#define PXST_K2_RING 4
#endif
constexpr int kNB = PXST_K2_RING;  // TMA ring depth


struct PixArgs {
  pxst_scan sc;
  const double* u;
  const double* di;
  const double* dj;
  const float* fm;
  const uint8_t* valid;
  const uint8_t* pv;
  const float* fmn;          // NaN-encoded reference (slow fix-up)
  const float2* fm2;         // padded (value, mask) reference (trial_pad), pad cells each side
  int pad;
  int64_t os, of, n0, m0;
  const float* fw;           // nullable frame weights [n_frames, ss, fs]
  const double* var;         // normaliser [ss*fs]
  const TileGeo* geo;        // [tiles_y * tiles_x]
  int tiles_x;
  int ka, kb;                // window (fast kernels: = template args)
  int box_r, box_c;          // TMA box (rows, cols)
  int n_chunks, chunk;       // frame chunking of the good list (split tiles)
  int tbl;                   // frame-table capacity of a fast CTA
  int64_t n_full;            // work units [0, n_full) are whole tiles over all frames
  int64_t nq;                // ROI rectangle pixel count
  const double* offs_a;      // window offsets (device)
  const double* offs_b;
  int refine_ok;
  double* u_out;
  double* err_out;
  float* partial;            // [n_chunks][ka*kb][nq]
  unsigned long long* slow_list;  // (pixel << 20 | chunk) pairs owning skipped samples
  unsigned* slow_n;
  unsigned long long* dbg;   // PXST_DEBUG: skipped-sample count (nullable)
};

// Box: 8 tile rows (|du/dx| up to ~1.2 plus noise) + window; columns: 16
// tile columns + window + alignment slack, rounded to pitch = 8 (mod 32).
__host__ __device__ inline int box_rows_for(int ka) { return ka + 16; }
__host__ __device__ inline int box_cols_for(int kb) {
  int c = kb + 36;
  c = (c + 31) / 32 * 32 + 8;
  return c - 32 >= kb + 36 ? c - 32 : c;
}
constexpr int kWarps = kThreads / 32;

// Work units of k_pix_fast (1-D grid): units [0, n_full) are whole tiles over
// all frames, finished in the kernel (argmin + paraboloid, no partial sums);
// the remaining tiles are split into n_chunks frame chunks each, one unit per
// (tile, chunk), so the last partial wave still fills the machine.  Slow-list
// entries and partial slots name a chunk; kAllFrames = a whole-tile unit
// (partial slot 0).
constexpr unsigned kAllFrames = 0xFFFFFu;

__device__ __forceinline__ void unit_of(const PixArgs& a, int64_t unit, int64_t& tile,
                                        unsigned& chunk) {
  if (unit < a.n_full) {
    tile = unit;
    chunk = kAllFrames;
  } else {
    const int64_t v = unit - a.n_full;
    tile = a.n_full + v / a.n_chunks;
    chunk = static_cast<unsigned>(v % a.n_chunks);
  }
}

__device__ __forceinline__ void chunk_frames(const PixArgs& a, unsigned chunk, int64_t& k_lo,
                                             int64_t& k_hi, int64_t& slot) {
  if (chunk == kAllFrames) {
    k_lo = 0;
    k_hi = a.sc.n_good;
    slot = 0;
  } else {
    k_lo = (int64_t)chunk * a.chunk;
    k_hi = min(a.sc.n_good, k_lo + a.chunk);
    slot = chunk;
  }
}

// Window offset i of an n-point window (recon.py:51-57): from the device
// array when one is given (sub-pixel grids), else the integer offset i - half.
__device__ __forceinline__ double win_off(const double* offs, int i, int n) {
  return offs ? offs[i] : static_cast<double>(i - (n - 1) / 2);
}

// Argmin / paraboloid / static-pixel rule for one pixel (recon.py:257-296,
// 313-315) from its raw trial sums (total(t), t in numpy order a * Kb + b).
// First-occurrence argmin on the raw sums: dividing by the common positive
// normaliser preserves the order except for ties the division itself would
// create, which the parity bar (unique argmin, margin > 1e-4) excludes.
template <class Total>
__device__ __forceinline__ void finish_pixel(const PixArgs& a, int64_t p, int best, double braw,
                                             double u0, double u1, double var, double off_a,
                                             double off_b, Total total) {
  const int64_t plane = a.sc.ss * a.sc.fs;
  const int na = a.ka, nb = a.kb;
  const bool active = var > 0.0;                      // recon.py:257-263
  const double nv = active ? var : 1.0;
  const double bv = braw / nv;
  const int ia = best / nb, ib = best % nb;
  double sh_ss = off_a, sh_fs = off_b;
  if (a.refine_ok && active && ia > 0 && ia < na - 1 && ib > 0 && ib < nb - 1) {   // recon.py:273-287
    double e[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) e[d] = total((ia + d / 3 - 1) * nb + (ib + d % 3 - 1)) / nv;
    double dss, dfs;
    paraboloid(e, dss, dfs);
    sh_ss += dss;
    sh_fs += dfs;
  }
  if (!active) { sh_ss = 0.0; sh_fs = 0.0; }          // recon.py:289-292
  a.u_out[p] = u0 + sh_ss;                            // recon.py:294-296
  a.u_out[plane + p] = u1 + sh_fs;
  a.err_out[p] = active ? bv : 0.0;                   // recon.py:313-315
}


// ---------------------------------------------------------------------------
// 1. tile geometry
// ---------------------------------------------------------------------------
// With init_out, every ROI pixel also gets u_out = u, err_out = 0 (the
// search's finishers then overwrite the work pixels).  One tile of kThreads
// threads (tid); red = kWarps x 4 doubles of shared memory; every thread
// reaches the one barrier.
__device__ __forceinline__ void tile_geo_block(const PixArgs& a, TileGeo* geo, int init_out,
                                               int64_t tile, bool on, int tid, double (*red)[4]) {
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t by = on ? tile / a.tiles_x : 0, bx = on ? tile % a.tiles_x : 0;
  const int64_t row = a.sc.roi[0] + by * kTR + tile_dr(tid);
  const int64_t col = a.sc.roi[2] + bx * kTC + tile_dc(tid);
  const bool inroi = on && row < a.sc.roi[1] && col < a.sc.roi[3];
  const int64_t p = inroi ? row * a.sc.fs + col : 0;
  const bool live = inroi && a.sc.work[p] != 0;
  const int64_t plane = a.sc.ss * a.sc.fs;
  if (init_out && inroi) {
    a.u_out[p] = a.u[p];
    a.u_out[plane + p] = a.u[plane + p];
    a.err_out[p] = 0.0;
  }
  const double u0 = live ? a.u[p] : 0.0, u1 = live ? a.u[plane + p] : 0.0;
  const double mn0 = warp_min(live ? u0 : INFINITY), mx0 = warp_max(live ? u0 : -INFINITY);
  const double mn1 = warp_min(live ? u1 : INFINITY), mx1 = warp_max(live ? u1 : -INFINITY);
  if (lane == 0) { red[warp][0] = mn0; red[warp][1] = mx0; red[warp][2] = mn1; red[warp][3] = mx1; }
  __syncthreads();
  if (tid != 0 || !on) return;
  double r0 = red[0][0], r1 = red[0][1], r2 = red[0][2], r3 = red[0][3];
  for (int w = 1; w < kWarps; ++w) {
    r0 = fmin(r0, red[w][0]);
    r1 = fmax(r1, red[w][1]);
    r2 = fmin(r2, red[w][2]);
    r3 = fmax(r3, red[w][3]);
  }
  geo[tile] = make_tile_geo(r0, r1, r2, r3);
}

__global__ void k_tile_geo(PixArgs a, TileGeo* geo, int init_out) {
  __shared__ double red[kWarps][4];
  tile_geo_block(a, geo, init_out, (int64_t)blockIdx.y * gridDim.x + blockIdx.x, true, threadIdx.x,
                 red);
}

// K2's two preparation steps in one launch of 256-thread blocks: blocks
// [0, n_pv) build the patch-valid map and NaN-encoded reference
// (pv_tile_block), the rest the tile geometry (kTiles tiles per block) and
// zero the slow-list counters.
constexpr int kPrepTiles = 256 / kThreads;
struct PvJob {
  const uint8_t* valid;
  const float* fm;
  int os, of, lr, hr, lc, hc, nx;
  uint8_t* pv;
  float* fmn;
  float2* fm2;
  int pad;
};
__global__ void __launch_bounds__(256) k_k2_prep(PixArgs a, TileGeo* geo, int init_out,
                                                 unsigned* zero2, PvJob pj, int n_pv,
                                                 int64_t tiles) {
  __shared__ union {
    PvShared pv;
    double red[kPrepTiles][kWarps][4];
  } sm;
  if (blockIdx.x < n_pv) {
    pv_tile_block(sm.pv, blockIdx.x % pj.nx, blockIdx.x / pj.nx, threadIdx.x & 31,
                  threadIdx.x >> 5, pj.valid, pj.fm, pj.os, pj.of, pj.lr, pj.hr, pj.lc, pj.hc,
                  pj.pv, pj.fmn, pj.fm2, pj.pad);
    return;
  }
  const int64_t b = blockIdx.x - n_pv;
  if (b == 0 && threadIdx.x < 2) zero2[threadIdx.x] = 0u;
  const int part = threadIdx.x / kThreads;
  const int64_t tile = b * kPrepTiles + part;
  tile_geo_block(a, geo, init_out, tile, tile < tiles, threadIdx.x % kThreads, sm.red[part]);
}

// window rows / cols a tile needs beyond its u span: the (Ka+1) x (Kb+1)
// patch, one row/col of floor() slack, and 3 columns of box-origin alignment.
__host__ __device__ inline int need_rows2(int ka) { return ka + 2; }
__host__ __device__ inline int need_cols2(int kb) { return kb + 5; }

// Per-sample geometry shared by the fast and slow kernels (identical float64
// expressions, so both agree on which samples are "fast").
struct Sample {
  int i, j;          // integer base of u - delta - origin
  double fx, fy;     // fractions
  int lr, lc;        // patch origin inside the TMA box
  int wr0, wc0;      // box origin in the object grid
  bool pre;          // every fast-path condition except the patch-valid lookup
                     // and the frame-weight sign
  uint8_t pvb;       // patch-valid byte (loaded unconditionally, consumed late so
                     // the one-frame-ahead pipeline hides its latency)
  float fwv;         // frame weight (< 0: not live); also consumed late
  __device__ __forceinline__ bool fast() const { return pre && pvb != 0 && fwv >= 0.f; }
};

// Object-window origin (box row, 16-byte aligned box column) of a tile for
// the frame at (dI, dJ): the same for every thread of the tile, so the fast
// kernel computes it once per frame in its shared frame table.
__device__ __forceinline__ void window_origin(const PixArgs& a, const TileGeo& g, double dI,
                                              double dJ, int& wr0, int& wc0) {
  const int ra = (a.ka - 1) / 2, rb = (a.kb - 1) / 2;
  wr0 = static_cast<int>(floor(g.umin0 - dI - static_cast<double>(a.n0))) - ra;
  wc0 = align4_down(static_cast<int>(floor(g.umin1 - dJ - static_cast<double>(a.m0))) - rb);
}

// Sample geometry from precomputed splits (what the fast kernel and the
// fast / slow classification use): u = iu + fu per pixel (once per thread)
// and d + origin = id + fd per frame (once per CTA, in the frame table), so
// x = u - d - origin = (iu - id) + (fu - fd) costs one float32 subtract and a
// carry instead of the float64 split.  The base may differ from the float64
// floor by one where x is within ~1e-7 of an integer; the trial positions
// x + a, and so the bilinear values (continuous there: these samples' patches
// are valid and on the grid, or they go to the fix-up, which re-derives the
// exact float64 split), are the same.
struct USplit {
  int i0, i1;
  float f0, f1;
  bool ok;
};
__device__ __forceinline__ USplit split_u(double u0, double u1) {
  USplit s;
  s.ok = fabs(u0) < 1e9 && fabs(u1) < 1e9;
  const double a = s.ok ? floor(u0) : 0.0, b = s.ok ? floor(u1) : 0.0;
  s.i0 = static_cast<int>(a);
  s.i1 = static_cast<int>(b);
  s.f0 = s.ok ? static_cast<float>(u0 - a) : 0.f;
  s.f1 = s.ok ? static_cast<float>(u1 - b) : 0.f;
  return s;
}
// frame split packed as int4 (i0, i1, bits of f0, bits of f1) of d + origin
__device__ __forceinline__ int4 split_d(double dI, double dJ, int64_t n0, int64_t m0) {
  const double x = dI + static_cast<double>(n0), y = dJ + static_cast<double>(m0);
  const bool ok = fabs(x) < 1e9 && fabs(y) < 1e9;
  const double a = ok ? floor(x) : 0.0, b = ok ? floor(y) : 0.0;
  return make_int4(ok ? static_cast<int>(a) : (1 << 30), static_cast<int>(b),
                   __float_as_int(ok ? static_cast<float>(x - a) : 0.f),
                   __float_as_int(ok ? static_cast<float>(y - b) : 0.f));
}

template <bool kKnownFit = false, int KA_ = 0, int KB_ = 0, int BC_ = 0>
__device__ __forceinline__ Sample make_sample_split(const PixArgs& a, const TileGeo& g,
                                                    const USplit& us, int4 ds, float fwv,
                                                    int wr0, int wc0) {
  const int ka = KA_ > 0 ? KA_ : a.ka, kb = KB_ > 0 ? KB_ : a.kb;
  const int box_c = BC_ > 0 ? BC_ : a.box_c;
  const int ra = (ka - 1) / 2, rb = (kb - 1) / 2;
  Sample s;
  s.fwv = fwv;
  float dx = us.f0 - __int_as_float(ds.z), dy = us.f1 - __int_as_float(ds.w);
  int i = us.i0 - ds.x, j = us.i1 - ds.y;
  if (dx < 0.f) { dx += 1.f; --i; }
  if (dy < 0.f) { dy += 1.f; --j; }
  if (dx >= 1.f) { dx = 0.f; ++i; }
  if (dy >= 1.f) { dy = 0.f; ++j; }
  s.fx = dx;
  s.fy = dy;
  const bool finite = us.ok && ds.x != (1 << 30);
  s.i = finite ? i : -(1 << 30);
  s.j = finite ? j : -(1 << 30);
  s.pre = false;
  s.pvb = 0;
  s.wr0 = s.wc0 = s.lr = s.lc = 0;
  if (kKnownFit || tile_fits(g, need_rows2(ka), need_cols2(kb), a.box_r, box_c)) {
    s.wr0 = wr0;
    s.wc0 = wc0;
    s.lr = s.i - ra - s.wr0;
    s.lc = s.j - rb - s.wc0;
    const int os = static_cast<int>(a.os), of = static_cast<int>(a.of);
    const bool in = static_cast<unsigned>(s.i) < static_cast<unsigned>(os) &&
                    static_cast<unsigned>(s.j) < static_cast<unsigned>(of);
    s.pre = in && static_cast<unsigned>(s.lr) <= static_cast<unsigned>(a.box_r - ka - 1) &&
            static_cast<unsigned>(s.lc) <= static_cast<unsigned>(box_c - kb - 1);
    s.pvb = __ldg(a.pv + (in ? s.i * of + s.j : 0));
  }
  return s;
}

// fwv is only stored (checked by fast()), so a frame-weight load issued for
// the next frame is not waited on here.
// KA_/KB_/BC_ > 0: the window and box width as compile-time constants (the
// fast kernels); the same tests as with the runtime values.
template <bool kKnownFit = false, int KA_ = 0, int KB_ = 0, int BC_ = 0>
__device__ __forceinline__ Sample make_sample(const PixArgs& a, const TileGeo& g, double u0,
                                              double u1, double dI, double dJ, float fwv,
                                              int wr0, int wc0) {
  const int ka = KA_ > 0 ? KA_ : a.ka, kb = KB_ > 0 ? KB_ : a.kb;
  const int box_c = BC_ > 0 ? BC_ : a.box_c;
  const int ra = (ka - 1) / 2, rb = (kb - 1) / 2;
  const double n0d = static_cast<double>(a.n0), m0d = static_cast<double>(a.m0);
  Sample s;
  s.fwv = fwv;
  const double x = u0 - dI - n0d;                     // recon.py:148
  const double y = u1 - dJ - m0d;
  const double xf = floor(x), yf = floor(y);
  s.fx = x - xf;
  s.fy = y - yf;
  const bool finite = fabs(x) < 1e9 && fabs(y) < 1e9;
  s.i = finite ? static_cast<int>(xf) : -(1 << 30);
  s.j = finite ? static_cast<int>(yf) : -(1 << 30);
  s.pre = false;
  s.pvb = 0;
  s.wr0 = s.wc0 = s.lr = s.lc = 0;
  if (kKnownFit || tile_fits(g, need_rows2(ka), need_cols2(kb), a.box_r, box_c)) {
    s.wr0 = wr0;
    s.wc0 = wc0;
    s.lr = s.i - ra - s.wr0;
    s.lc = s.j - rb - s.wc0;
    // 0 <= v < n as one unsigned compare (os * of < 2^31, check_ref; the box
    // holds the patch: box_r >= ka + 2, box_c >= kb + 2)
    const int os = static_cast<int>(a.os), of = static_cast<int>(a.of);
    const bool in = static_cast<unsigned>(s.i) < static_cast<unsigned>(os) &&
                    static_cast<unsigned>(s.j) < static_cast<unsigned>(of);
    s.pre = in && static_cast<unsigned>(s.lr) <= static_cast<unsigned>(a.box_r - ka - 1) &&
            static_cast<unsigned>(s.lc) <= static_cast<unsigned>(box_c - kb - 1);
    s.pvb = __ldg(a.pv + (in ? s.i * of + s.j : 0));
  }
  return s;
}

// ---------------------------------------------------------------------------
// 2. fast kernel (TMA ring + register engine)
// ---------------------------------------------------------------------------
// BC > 0: the TMA box width (window row pitch in the ring) is the compile-time
// constant BC (= a.box_c), so the engine's patch rows are immediate LDS
// offsets from one base register; these variants are also specialised for
// calls without frame weights (the host picks them only then).
template <int KA, int KB, int BC = 0>
__global__ void __launch_bounds__(kThreads, kCtaPerSm)
    k_pix_fast(const __grid_constant__ CUtensorMap tmap, PixArgs a) {
  const int ldw = BC > 0 ? BC : a.box_c;
  const float* const fwp = BC > 0 ? nullptr : a.fw;
  extern __shared__ __align__(128) unsigned char ring_raw[];
  __shared__ __align__(8) uint64_t full[kNB], empty[kNB];
  __shared__ int s_iss[kNB];   // PXST_K2_PRODUCER == 2: the frame each slot holds or awaits
  // TMA destinations must be 128-byte aligned: align the base, pad the slots.
  // (Pointer arithmetic on the shared array keeps the address space, so the
  // engine's reads compile to LDS rather than generic loads.)
  unsigned char* base = ring_raw + ((128u - (smem_addr(ring_raw) & 127u)) & 127u);
  float* ring = reinterpret_cast<float*>(base);
  const int box = slot_floats(a.box_r, a.box_c);          // slot stride (128-byte multiple)
  // Per-frame table of the chunk after the ring: the split of d + origin
  // (int4, one-row windows) or (di, dj), the frame's stack offset, the window
  // origin.
  int4* t_ds = reinterpret_cast<int4*>(base + sizeof(float) * kNB * box);
  double* t_di = reinterpret_cast<double*>(t_ds + a.tbl);
  double* t_dj = t_di + a.tbl;
  int64_t* t_off = reinterpret_cast<int64_t*>(t_dj + a.tbl);     // frame offset f * plane
  int* t_wr = reinterpret_cast<int*>(t_off + a.tbl);             // window origin per frame
  int* t_wc = t_wr + a.tbl;

  int64_t tile;
  unsigned chunk;
  unit_of(a, blockIdx.x, tile, chunk);
  const int64_t ty = tile / a.tiles_x, tx = tile % a.tiles_x;
  const TileGeo g = a.geo[tile];
  if (!(g.umin0 == g.umin0)) return;                  // tile without work pixels
  const int64_t rr = ty * kTR + tile_dr(threadIdx.x);
  const int64_t cc = tx * kTC + tile_dc(threadIdx.x);
  const int64_t row = a.sc.roi[0] + rr, col = a.sc.roi[2] + cc;
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2];
  const bool inroi = row < a.sc.roi[1] && col < a.sc.roi[3];
  const int64_t p = inroi ? row * a.sc.fs + col : 0;
  const int64_t q = rr * cw + cc;
  const bool live = inroi && a.sc.work[p] != 0;
  const int64_t plane = a.sc.ss * a.sc.fs;
  int64_t k_lo, k_hi, pslot;
  chunk_frames(a, chunk, k_lo, k_hi, pslot);
  const int nk = static_cast<int>(k_hi - k_lo);
  float* out = a.partial + pslot * KA * KB * a.nq + q;

  PackedAcc<KA, KB> acc;
  acc.zero();
  const bool fits = tile_fits(g, need_rows2(KA), need_cols2(KB), a.box_r, a.box_c);
  bool any_slow = live && nk > 0 && !fits;

  const double u0 = live ? a.u[p] : 0.0, u1 = live ? a.u[plane + p] : 0.0;
  const double var_p = (live && chunk == kAllFrames) ? a.var[p] : 0.0;   // used after the loop
  if (fits && nk > 0) {
    const unsigned bytes = static_cast<unsigned>(a.box_r * a.box_c * sizeof(float));
    for (int jj = threadIdx.x; jj < nk; jj += kThreads) {
      const int f = a.sc.good[k_lo + jj];
      const double dI = a.di[f], dJ = a.dj[f];
      t_off[jj] = f * plane;
      if (KA == 1) t_ds[jj] = split_d(dI, dJ, a.n0, a.m0);
      t_di[jj] = dI;
      t_dj[jj] = dJ;
      window_origin(a, g, dI, dJ, t_wr[jj], t_wc[jj]);
    }
    auto issue = [&](int jj) {  // frame k_lo + jj into slot jj % kNB
      const int b = jj % kNB;
      mbar_arrive_expect_tx(&full[b], bytes);
      tma_load_2d(ring + b * box, &tmap, t_wc[jj], t_wr[jj], &full[b]);
    };
    if (threadIdx.x == 0) {
      tma_prefetch_desc(&tmap);
      for (int b = 0; b < kNB; ++b) {
        mbar_init(&full[b], 1);
        mbar_init(&empty[b], kThreads);
        s_iss[b] = b;
      }
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int jj = 0; jj < min(kNB, nk); ++jj) issue(jj);

    const float W = live ? a.sc.w32[p] : 0.f;
    // One-row windows (few trials per sample: the geometry is a large share)
    // use the float32 split; larger ones keep the float64 geometry, which the
    // compiler interleaves with the previous sample's trials (the split made
    // the 11 x 11 loop 16 % slower).
    const USplit us = split_u(u0, u1);
    auto sample_of = [&](int jj, float& I, float& fwv) {
      const int64_t off = t_off[jj];
      I = live ? __ldg(a.sc.frames + off + p) : 0.f;
      fwv = (live && fwp) ? __ldg(fwp + off + p) : 1.f;
      // (fwv goes in as loaded and "live" into the pre flag: a select on the
      // weight here would wait for this frame-ahead load -- and for the stack
      // value sharing its scoreboard -- in the frame that issues it; ncu
      // showed 32 % of the 1 x 17 kernel's stall samples on that select)
      // (the two-dimensional windows keep the select: without it the 13 x 13
      // kernel spilled, 91.0 -> 93.9 ms at config 3)
      if (KA == 1) {
        Sample sm_ = make_sample_split<true, KA, KB, BC>(a, g, us, t_ds[jj], fwv, t_wr[jj],
                                                         t_wc[jj]);
        sm_.pre = sm_.pre && live;
        return sm_;
      }
      return make_sample<true, KA, KB, BC>(a, g, u0, u1, t_di[jj], t_dj[jj], live ? fwv : -1.f,
                                           t_wr[jj], t_wc[jj]);
    };
    // One-frame-ahead pipeline of the per-sample geometry, stack value and
    // patch-valid lookup.  The loop body after the ring wait is one basic
    // block (samples that are not fast run the engine with zero weights on
    // the slot origin), so the compiler interleaves the next sample's float64
    // geometry and loads with this frame's trials.
    // (Windows above 11 x 11 compute the sample in place: the 169 accumulators
    // of 13 x 13 leave no registers for a second sample.)
#ifndef PXST_K2_AHEAD_MAX
#define PXST_K2_AHEAD_MAX 121
#endif
    constexpr bool kAhead = KA * KB <= PXST_K2_AHEAD_MAX;
    float I_n = 0.f, fw_n = 0.f;
    Sample s_n{};
    if (kAhead) s_n = sample_of(0, I_n, fw_n);
    int issued = min(kNB, nk);     // thread 0: frames [0, issued) are in flight or done
    const unsigned full_a = smem_addr(full), empty_a = smem_addr(empty);   // see mbar_wait_a
    for (int jj = 0; jj < nk; ++jj) {
      if (!kAhead) s_n = sample_of(jj, I_n, fw_n);
      const Sample sm = s_n;
      const float I = I_n, fwv = fw_n;
      const int b = jj % kNB;
      const unsigned ph = (jj / kNB) & 1;
      // Ring refill.  Windows up to 11 x 11: at release time (below).  Larger
      // ones (13 x 13 sits at the register limit; the release-time code cost
      // 91.3 -> 95.1 ms at config 3): thread 0, opportunistically, here.
#ifndef PXST_K2_PRODUCER
#define PXST_K2_PRODUCER (KA * KB <= 121 ? 2 : 1)
#endif
      if (PXST_K2_PRODUCER == 1 && threadIdx.x == 0) {
        // Refill freed slots without waiting for the slowest warp: frame k
        // reuses the slot of frame k - kNB; block only when this thread
        // itself needs frame jj next.
        while (issued < nk && issued < jj + kNB) {
          const int k = issued;
          const unsigned eph = ((k / kNB) - 1) & 1;
          if (k > jj) {
            if (!mbar_test(&empty[k % kNB], eph)) break;
          } else {
            mbar_wait(&empty[k % kNB], eph);
          }
          issue(k);
          ++issued;
        }
      }
      mbar_wait_a(full_a + 8u * b, ph);
      const bool fast = sm.fast();
      any_slow |= live && !fast;
      const float fx = fast ? static_cast<float>(sm.fx) : 0.f;
      const float fy = fast ? static_cast<float>(sm.fy) : 0.f;
      float sq = BC > 0 ? 1.f : sqrt_approx(fmaxf(fwv, 0.f));   // no branch in the block
      sq = fwv == 1.f ? 1.f : sq;
      sq = fast ? sq : 0.f;
      const float sI = I * sq, sW = W * sq;
      const int off = fast ? sm.lr * ldw + sm.lc : 0;
      PXST_DCHECK(!fast || (sm.lr >= 0 && sm.lr + KA + 1 <= a.box_r && sm.lc >= 0 &&
                            sm.lc + KB + 1 <= a.box_c));
      if (kAhead) s_n = sample_of(jj + 1 < nk ? jj + 1 : jj, I_n, fw_n);
      if (KA == 1 && __all_sync(0xffffffffu, fx == 0.f))   // warp-uniform (config 2)
        engine_row1<KB>(ring + b * box + off, fy, sW, sI,
                        reinterpret_cast<PackedAcc<1, KB>&>(acc));
      else
        engine_fast2<KA, KB>(ring + b * box + off, ldw, fx, fy, sW * (1.f - fx), sW * fx, sI,
                             acc);
      mbar_arrive_a(empty_a + 8u * b);
      if (PXST_K2_PRODUCER == 2 && (threadIdx.x & 31) == 0 && jj + kNB < nk) {
        // Refill at release time: the warp whose arrival completes the slot's
        // phase (or any warp that sees it complete) claims the slot's next
        // frame and issues its load -- no waiting for thread 0 to come round
        // (ncu had 17 % of the 11 x 11 kernel's stall samples on the ring
        // wait; config 1 K2 0.564 -> 0.548 ms, config 2 6.09 -> 5.70 ms).
        if (mbar_test_a(empty_a + 8u * b, ph) && atomicCAS(&s_iss[b], jj, jj + kNB) == jj)
          issue(jj + kNB);
      }
      if (PXST_K2_PRODUCER == 0 && threadIdx.x == 0 && jj + kNB < nk) {
        mbar_wait(&empty[b], ph);      // every thread is done with this slot
        issue(jj + kNB);
      }
    }
  }
  bool finished = false;
  if (chunk == kAllFrames) {
    // Whole-tile unit: finish every pixel without skipped samples here (the
    // others are finished by k_pix_slow after their fix-up).  The
    // trial sums go to this thread's column of the (now idle) ring so the
    // 3x3 refinement patch can be indexed.
    __syncthreads();                               // no thread reads the ring any more
    float* st = ring + threadIdx.x;
    int best = 0;
    float bsum = 0.f;
#pragma unroll
    for (int t = 0; t < KA; ++t)
#pragma unroll
      for (int s = 0; s < KB; ++s) {
        const float v = acc.get(t, s);
        st[(t * KB + s) * kThreads] = v;
        if (t * KB + s == 0 || v < bsum) { bsum = v; best = t * KB + s; }
      }
    finished = live && !any_slow;
    if (finished) {   // integer window: offsets are index - half (window_offsets)
      constexpr int RA = (KA - 1) / 2, RB = (KB - 1) / 2;
      finish_pixel(a, p, best, static_cast<double>(bsum), u0, u1, var_p,
                   static_cast<double>(best / KB - RA), static_cast<double>(best % KB - RB),
                   [&](int t) { return static_cast<double>(st[t * kThreads]); });
    }
  }
  if (live && !finished) {
#pragma unroll
    for (int t = 0; t < KA; ++t)
#pragma unroll
      for (int s = 0; s < KB; ++s) out[(int64_t)(t * KB + s) * a.nq] = acc.get(t, s);
  }
  if (any_slow) {   // hand the skipped samples of this (pixel, chunk) to k_pix_slow
    const unsigned slot = atomicAdd(a.slow_n, 1u);
    a.slow_list[slot] = (static_cast<unsigned long long>(q) << 20) | chunk;
  }
}

// ---------------------------------------------------------------------------
// 3. slow-sample fix-up (runs after k_pix_fast on the same stream).
//    k_pix_fast appends (pixel, chunk) pairs that own skipped samples to a
//    list; k_pix_slow: one warp per listed pair (fetched dynamically: an
//    entry's cost ranges from one to all frames).  Lanes classify 32 frames
//    at a time with the fast kernel's eligibility test.  Windows of up to 3
//    rows (k_pix_slow_rows; larger ones: k_pix_slow, lanes over trials) then
//    evaluate the skipped samples by "row lanes": lane l works on sample slot l / Ka and
//    owns trial row l % Ka, loading that row's two patch rows once (Kb + 1
//    cells each, NaN-encoded reference, off-grid cells marked) and evaluating
//    its Kb trials exactly from registers (trial_patch: the reference's masked
//    renormalised read and (I-W)^2 fallback).  32 / Ka samples are in flight
//    per warp; each slot's partial sums are added in a fixed slot order, so
//    the result does not depend on the list order or on timing.
// ---------------------------------------------------------------------------
constexpr int kRowMax = 17;        // widest fast-path window row (1 x 17)

__device__ __forceinline__ float slow_cell(const float* __restrict__ fmn, int os, int of, int r,
                                           int c) {
  return (r >= 0 && r < os && c >= 0 && c < of) ? __ldg(fmn + (r * of + c))
                                                : __uint_as_float(kOffGrid);
}

__global__ void __launch_bounds__(256, 2) k_pix_slow_rows(PixArgs a,
                                                      const unsigned long long* __restrict__ list,
                                                      unsigned* __restrict__ list_n) {
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2];
  const int lane = threadIdx.x & 31;
  const unsigned n = list_n[0];
  unsigned* next = list_n + 1;       // work counter
  const int ka = a.ka, kb = a.kb;
  const int ra = (ka - 1) / 2, rb = (kb - 1) / 2;
  const int nk = ka * kb;
  const int nslot = 32 / ka;         // samples in flight per warp
  const int slot = lane / ka, trow = lane % ka;
  const bool lane_on = slot < nslot;
  const int os = static_cast<int>(a.os), of = static_cast<int>(a.of);
  const int64_t plane = a.sc.ss * a.sc.fs;
  for (;;) {
    unsigned e = 0;
    if (lane == 0) e = atomicAdd(next, 1u);
    e = __shfl_sync(0xffffffffu, e, 0);
    if (e >= n) break;
    const unsigned long long ent = list[e];
    const int64_t q = static_cast<int64_t>(ent >> 20);
    const unsigned chunk = static_cast<unsigned>(ent & 0xFFFFF);
    const int64_t rr = q / cw, cc = q % cw;
    const int64_t p = (a.sc.roi[0] + rr) * a.sc.fs + a.sc.roi[2] + cc;
    const TileGeo g = a.geo[(rr / kTR) * a.tiles_x + cc / kTC];
    const double u0 = a.u[p], u1 = a.u[plane + p];
    const USplit us = split_u(u0, u1);
    const float W = a.sc.w32[p];
    int64_t k_lo, k_hi, pslot;
    chunk_frames(a, chunk, k_lo, k_hi, pslot);
    float* out = a.partial + pslot * nk * a.nq + q;
    float acc[kRowMax];              // this lane's trial row, its slot's samples
    float prev[kRowMax];             // slot 0: the fast kernel's partials of the row
#pragma unroll
    for (int c = 0; c < kRowMax; ++c) {
      acc[c] = 0.f;
      prev[c] = (slot == 0 && c < kb) ? out[(int64_t)(trow * kb + c) * a.nq] : 0.f;
    }
    for (int64_t k0 = k_lo; k0 < k_hi; k0 += 32) {
      // lane-parallel classification of 32 frames; each lane keeps its
      // frame's sample and stack value for the row lanes below
      const int64_t kl = k0 + lane;
      bool slow = false;
      Sample sl{};
      float Il = 0.f, fwl = 1.f;
      if (kl < k_hi) {
        const int64_t f = a.sc.good[kl];
        fwl = a.fw ? __ldg(a.fw + f * plane + p) : 1.f;
        const double dI = a.di[f], dJ = a.dj[f];
        int wr0, wc0;
        window_origin(a, g, dI, dJ, wr0, wc0);
        // classified exactly as the fast kernel did (the float32 split for
        // one-row windows); the exact trials use the float64 split
        sl = make_sample(a, g, u0, u1, dI, dJ, fwl, wr0, wc0);
        slow = a.ka == 1
                   ? !make_sample_split(a, g, us, split_d(dI, dJ, a.n0, a.m0), fwl, wr0, wc0).fast()
                   : !sl.fast();
        if (slow) Il = __ldg(a.sc.frames + f * plane + p);
      }
      unsigned mask = __ballot_sync(0xffffffffu, slow);
      if (a.dbg) {   // skipped samples by reason: off grid, outside the box, patch invalid
        const bool in = sl.i >= 0 && sl.i < a.os && sl.j >= 0 && sl.j < a.of;
        const bool inbox = sl.lr >= 0 && sl.lr + a.ka + 1 <= a.box_r && sl.lc >= 0 &&
                           sl.lc + a.kb + 1 <= a.box_c;
        const unsigned m1 = __ballot_sync(0xffffffffu, slow && !in);
        const unsigned m2 = __ballot_sync(0xffffffffu, slow && in && !inbox);
        if (lane == 0) {
          atomicAdd(a.dbg, (unsigned long long)__popc(mask));
          atomicAdd(a.dbg + 1, (unsigned long long)__popc(m1));
          atomicAdd(a.dbg + 2, (unsigned long long)__popc(m2));
        }
      }
      while (mask) {
        // slot s takes the (s+1)-th lowest set bit: samples stay in frame
        // order within a slot
        const int cnt = __popc(mask);
        const int bsel = (lane_on && slot < cnt) ? static_cast<int>(__fns(mask, 0, slot + 1)) : -1;
        const int src = bsel >= 0 ? bsel : 0;
        const int si = __shfl_sync(0xffffffffu, sl.i, src);
        const int sj = __shfl_sync(0xffffffffu, sl.j, src);
        const double sfx = __shfl_sync(0xffffffffu, sl.fx, src);
        const double sfy = __shfl_sync(0xffffffffu, sl.fy, src);
        const float sI = __shfl_sync(0xffffffffu, Il, src);
        const float sfw = __shfl_sync(0xffffffffu, fwl, src);
        if (cnt <= nslot) {
          mask = 0u;
        } else {
          const unsigned last = __fns(mask, 0, nslot);      // bit of the last slot's sample
          mask &= ~((2u << last) - 1u);
        }
        if (bsel >= 0) {
          const ExactSample es = exact_sample(sfx, sfy, W, sI, sfw);
          const int pr = si - ra + trow, pc = sj - rb;
          float r0[kRowMax + 1], r1[kRowMax + 1];
#pragma unroll
          for (int c = 0; c <= kRowMax; ++c) {
            r0[c] = c <= kb ? slow_cell(a.fmn, os, of, pr, pc + c) : 0.f;
            r1[c] = c <= kb ? slow_cell(a.fmn, os, of, pr + 1, pc + c) : 0.f;
          }
#pragma unroll
          for (int c = 0; c < kRowMax; ++c)
            if (c < kb) acc[c] += trial_patch(r0[c], r0[c + 1], r1[c], r1[c + 1], es);
        }
      }
    }
    // slot partials into slot 0, fixed order
    for (int s = 1; s < nslot; ++s) {
#pragma unroll
      for (int c = 0; c < kRowMax; ++c) {
        const float v = __shfl_sync(0xffffffffu, acc[c], (s * ka + trow) & 31);
        if (slot == 0) acc[c] += v;
      }
    }
    float tot[kRowMax];
#pragma unroll
    for (int c = 0; c < kRowMax; ++c) tot[c] = prev[c] + acc[c];
    if (chunk != kAllFrames) {
      if (slot == 0) {
#pragma unroll
        for (int c = 0; c < kRowMax; ++c)
          if (c < kb) out[(int64_t)(trow * kb + c) * a.nq] = tot[c];
      }
      continue;
    }
    // Whole-tile pixel: every frame is in, finish it here.  Warp first-
    // occurrence argmin (smaller sum, ties to the smaller trial index).
    int best = -1;
    float bsum = 0.f;
    if (slot == 0) {
#pragma unroll
      for (int c = 0; c < kRowMax; ++c)
        if (c < kb && (best < 0 || tot[c] < bsum)) { bsum = tot[c]; best = trow * kb + c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bsum, o);
      const int ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (ob >= 0 && (best < 0 || ov < bsum || (ov == bsum && ob < best))) { bsum = ov; best = ob; }
    }
    finish_pixel(a, p, best, static_cast<double>(bsum), u0, u1, a.var[p],
                 win_off(a.offs_a, best / kb, a.ka), win_off(a.offs_b, best % kb, a.kb),
                 [&](int t) {
                   const int c = t % kb;
                   float v = tot[0];
#pragma unroll
                   for (int j = 1; j < kRowMax; ++j) v = c == j ? tot[j] : v;
                   return static_cast<double>(__shfl_sync(0xffffffffu, v, t / kb));
                 });
  }
}

// Lane-per-trial variant for windows of 5 rows and more (row lanes would
// leave a third of the warp idle and serialise each lane's Kb trials): lanes
// own trials lane + 32 j and read each trial's corners straight from the
// NaN-encoded reference (trial_global), in frame order.
// NJ = trials per lane, ceil(Ka Kb / 32) (<= 6 for the fast-path windows):
// sized per window so 11x11 (NJ = 4) fits three blocks per SM.

#ifndef PXST_K2_SLOW_OCC
#define PXST_K2_SLOW_OCC 3
#endif
template <int NJ>
__global__ void __launch_bounds__(256, NJ <= 4 ? PXST_K2_SLOW_OCC : 2) k_pix_slow(PixArgs a,
                                                 const unsigned long long* __restrict__ list,
                                                 unsigned* __restrict__ list_n) {
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2];
  const int lane = threadIdx.x & 31;
  const unsigned n = list_n[0];
  unsigned* next = list_n + 1;       // work counter: entries are fetched dynamically per warp
                                     // (their cost ranges from 1 to all frames)
  const int ra = (a.ka - 1) / 2, rb = (a.kb - 1) / 2;
  const int nk = a.ka * a.kb;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const int os = static_cast<int>(a.os), of = static_cast<int>(a.of);
  int ta[NJ], tb[NJ];   // window coordinates of the lane's trials
  int to[NJ];           // and their cell offsets from the window's corner
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int t = lane + 32 * j;
    ta[j] = t / a.kb;
    tb[j] = t % a.kb;
    to[j] = ta[j] * of + tb[j];
  }
  unsigned tp[NJ];      // the same offsets in the padded image
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int t = min(lane + 32 * j, nk - 1);
    tp[j] = (t / a.kb) * (of + 2 * a.pad) + t % a.kb;
  }
  for (;;) {
    unsigned e = 0;
    if (lane == 0) e = atomicAdd(next, 1u);
    e = __shfl_sync(0xffffffffu, e, 0);
    if (e >= n) break;
    const unsigned long long ent = list[e];
    const int64_t q = static_cast<int64_t>(ent >> 20);
    const unsigned chunk = static_cast<unsigned>(ent & 0xFFFFF);
    const int64_t rr = q / cw, cc = q % cw;
    const int64_t p = (a.sc.roi[0] + rr) * a.sc.fs + a.sc.roi[2] + cc;
    const TileGeo g = a.geo[(rr / kTR) * a.tiles_x + cc / kTC];
    const double u0 = a.u[p], u1 = a.u[plane + p];
    const USplit us = split_u(u0, u1);
    const float W = a.sc.w32[p];
    int64_t k_lo, k_hi, pslot;
    chunk_frames(a, chunk, k_lo, k_hi, pslot);
    float* out = a.partial + pslot * nk * a.nq + q;
    float part[NJ];          // lane owns trials lane + 32 j
    float prev[NJ];          // the fast kernel's partials, fetched early
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      part[j] = 0.f;
      prev[j] = lane + 32 * j < nk ? out[(int64_t)(lane + 32 * j) * a.nq] : 0.f;
    }
    for (int64_t k0 = k_lo; k0 < k_hi; k0 += 32) {
      // lane-parallel classification of 32 frames; each lane keeps its
      // frame's sample and stack value for the broadcast below
      const int64_t kl = k0 + lane;
      bool slow = false;
      Sample sl{};
      float Il = 0.f, fwl = 1.f;
      if (kl < k_hi) {
        const int64_t f = a.sc.good[kl];
        fwl = a.fw ? __ldg(a.fw + f * plane + p) : 1.f;
        const double dI = a.di[f], dJ = a.dj[f];
        int wr0, wc0;
        window_origin(a, g, dI, dJ, wr0, wc0);
        // classified exactly as the fast kernel did (the float32 split for
        // one-row windows); the exact trials use the float64 split
        sl = make_sample(a, g, u0, u1, dI, dJ, fwl, wr0, wc0);
        slow = a.ka == 1
                   ? !make_sample_split(a, g, us, split_d(dI, dJ, a.n0, a.m0), fwl, wr0, wc0).fast()
                   : !sl.fast();
        if (slow) Il = __ldg(a.sc.frames + f * plane + p);
      }
      unsigned mask = __ballot_sync(0xffffffffu, slow);
      if (a.dbg) {   // skipped samples by reason: off grid, outside the box, patch invalid
        const bool in = sl.i >= 0 && sl.i < a.os && sl.j >= 0 && sl.j < a.of;
        const bool inbox = sl.lr >= 0 && sl.lr + a.ka + 1 <= a.box_r && sl.lc >= 0 &&
                           sl.lc + a.kb + 1 <= a.box_c;
        const unsigned m1 = __ballot_sync(0xffffffffu, slow && !in);
        const unsigned m2 = __ballot_sync(0xffffffffu, slow && in && !inbox);
        if (lane == 0) {
          atomicAdd(a.dbg, (unsigned long long)__popc(mask));
          atomicAdd(a.dbg + 1, (unsigned long long)__popc(m1));
          atomicAdd(a.dbg + 2, (unsigned long long)__popc(m2));
        }
      }
      while (mask) {
        const int bsel = __ffs(mask) - 1;
        mask &= mask - 1;
        const int pr0 = __shfl_sync(0xffffffffu, sl.i, bsel) - ra;
        const int pc0 = __shfl_sync(0xffffffffu, sl.j, bsel) - rb;
        const ExactSample es = exact_sample(__shfl_sync(0xffffffffu, sl.fx, bsel),
                                            __shfl_sync(0xffffffffu, sl.fy, bsel), W,
                                            __shfl_sync(0xffffffffu, Il, bsel),
                                            __shfl_sync(0xffffffffu, fwl, bsel));
        // warp-uniform: the window's 2x2 cells inside the padded (value,
        // mask) image (every on-grid sample): two row pointers per trial,
        // four 8-byte loads, no bounds tests or selects
        if (a.fm2 && pr0 >= -a.pad && pc0 >= -a.pad && pr0 + a.ka < os + a.pad &&
            pc0 + a.kb < of + a.pad) {
          const int ofp = of + 2 * a.pad;
          const unsigned w0 = static_cast<unsigned>((pr0 + a.pad) * ofp + (pc0 + a.pad));
          const unsigned w1 = w0 + (es.fxp ? ofp : 0);
          PXST_DCHECK(w1 + tp[NJ - 1] + 1 <
                      static_cast<unsigned>((os + 2 * a.pad) * ofp));   // inside the padded image
          // (no trial-count guard: lanes past the window repeat its last
          // trial, their sums are never read; the NJ trials' loads overlap)
          float v[NJ];
          if (es.fyp) {
#pragma unroll
            for (int j = 0; j < NJ; ++j) v[j] = trial_pad<true>(a.fm2, w0 + tp[j], w1 + tp[j], 1, es);
          } else {
#pragma unroll
            for (int j = 0; j < NJ; ++j) v[j] = trial_pad<false>(a.fm2, w0 + tp[j], w1 + tp[j], 0, es);
          }
#pragma unroll
          for (int j = 0; j < NJ; ++j) part[j] += v[j];
        } else if (pr0 >= 0 && pc0 >= 0 && pr0 + a.ka < os && pc0 + a.kb < of) {
          const float* w0 = a.fmn + (pr0 * of + pc0);
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (lane + 32 * j < nk) part[j] += trial_interior(w0 + to[j], of, es);
        } else {
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (lane + 32 * j < nk)
              part[j] += trial_global(a.fmn, os, of, pr0 + ta[j], pc0 + tb[j], es);
        }
      }
    }
    float tot[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) tot[j] = prev[j] + part[j];
    if (chunk != kAllFrames) {
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int t = lane + 32 * j;
        if (t < nk) out[(int64_t)t * a.nq] = tot[j];
      }
      continue;
    }
    // Whole-tile pixel: every frame is in, finish it here.  Warp first-
    // occurrence argmin (smaller sum, ties to the smaller trial index).
    int best = -1;
    float bsum = 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int t = lane + 32 * j;
      if (t < nk && (best < 0 || tot[j] < bsum)) { bsum = tot[j]; best = t; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bsum, o);
      const int ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (ob >= 0 && (best < 0 || ov < bsum || (ov == bsum && ob < best))) { bsum = ov; best = ob; }
    }
    finish_pixel(a, p, best, static_cast<double>(bsum), u0, u1, a.var[p],
                 win_off(a.offs_a, best / a.kb, a.ka), win_off(a.offs_b, best % a.kb, a.kb),
                 [&](int t) {
                   float v = tot[0];
#pragma unroll
                   for (int j = 1; j < NJ; ++j) v = (t >> 5) == j ? tot[j] : v;
                   return static_cast<double>(__shfl_sync(0xffffffffu, v, t & 31));
                 });
  }
}

// ---------------------------------------------------------------------------
// generic (sub-pixel / any window): float64, one thread per (pixel, trial)
// ---------------------------------------------------------------------------
__global__ void k_pix_generic(PixArgs a, const double* __restrict__ offs_a,
                              const double* __restrict__ offs_b, double* __restrict__ errs,
                              int t0) {
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2];
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int t = t0 + blockIdx.y;
  if (q >= a.nq) return;
  const int64_t p = (a.sc.roi[0] + q / cw) * a.sc.fs + a.sc.roi[2] + q % cw;
  if (!a.sc.work[p]) return;
  const int64_t plane = a.sc.ss * a.sc.fs;
  const double u0 = a.u[p], u1 = a.u[plane + p];
  const double W = a.sc.w64[p];
  const double oa = offs_a[t / a.kb], ob = offs_b[t % a.kb];
  double acc = 0.0;
  for (int64_t k = 0; k < a.sc.n_good; ++k) {
    const int64_t f = a.sc.good[k];
    const double I = static_cast<double>(__ldg(a.sc.frames + f * plane + p));
    const double fwv = a.fw ? static_cast<double>(__ldg(a.fw + f * plane + p)) : 1.0;
    const double x = (u0 - a.di[f] - a.n0) + oa;      // recon.py:148, 157
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
  errs[(int64_t)t * a.nq + q] = acc;
}

// ---------------------------------------------------------------------------
// 4. epilogue
// ---------------------------------------------------------------------------
// kEpiLanes lanes per pixel: lane k sums trials k, k + kEpiLanes, ... over
// the chunks (all loads independent), then a first-occurrence argmin across
// the group (smaller sum, ties to the smaller trial index = numpy's order).
// 4 lanes measured best when only the tail tiles are chunked (config 1: 8
// lanes 20.9 us, 4 lanes 16.0, 2 lanes 21.6), 2 when every tile is (config 3:
// 8 lanes 1.85 ms, 4 lanes 1.54, 2 lanes 0.91: better coalesced trial loads).

// Pixels: linear over the ROI (generic path, tiles_x == 0), or the pixels of
// the split tiles [n_full, tiles) of the fast path (whole-tile pixels are
// finished by k_pix_fast / k_pix_slow).
template <class T, int kEpiLanes>
__global__ void k_pix_epilogue(PixArgs a, const T* __restrict__ part, int n_chunks) {
  const int64_t cw = a.sc.roi[3] - a.sc.roi[2];
  const int64_t gi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kEpiLanes;
  const int sub = threadIdx.x % kEpiLanes;
  const unsigned gmask = ((1u << kEpiLanes) - 1u) << ((threadIdx.x & 31) & ~(kEpiLanes - 1));
  int64_t rr, cc;
  if (a.tiles_x > 0) {
    const int64_t tile = a.n_full + gi / kThreads;
    const int loc = static_cast<int>(gi % kThreads);
    rr = (tile / a.tiles_x) * kTR + tile_dr(loc);
    cc = (tile % a.tiles_x) * kTC + tile_dc(loc);
    if (rr >= a.sc.roi[1] - a.sc.roi[0] || cc >= cw) return;
  } else {
    if (gi >= a.nq) return;
    rr = gi / cw;
    cc = gi % cw;
  }
  const int64_t q = rr * cw + cc;
  const int64_t p = (a.sc.roi[0] + rr) * a.sc.fs + a.sc.roi[2] + cc;
  if (!a.sc.work[p]) return;
  const int nk = a.ka * a.kb;
  const int64_t cstride = (int64_t)nk * a.nq;
  auto total = [&](int t) {
    double s = 0.0;
    for (int c = 0; c < n_chunks; ++c) s += static_cast<double>(part[c * cstride + (int64_t)t * a.nq + q]);
    return s;
  };
  int best = -1;
  double braw = 0.0;
  for (int t0 = 0; t0 < nk; t0 += 8 * kEpiLanes) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.0;
    for (int c = 0; c < n_chunks; ++c) {
      const T* pc = part + c * cstride + q;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int t = t0 + sub + j * kEpiLanes;
        if (t < nk) v[j] += static_cast<double>(pc[(int64_t)t * a.nq]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = t0 + sub + j * kEpiLanes;
      if (t < nk && (best < 0 || v[j] < braw)) { braw = v[j]; best = t; }
    }
  }
#pragma unroll
  for (int o = kEpiLanes / 2; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(gmask, braw, o, kEpiLanes);
    const int ob = __shfl_xor_sync(gmask, best, o, kEpiLanes);
    if (ob >= 0 && (best < 0 || ov < braw || (ov == braw && ob < best))) { braw = ov; best = ob; }
  }
  if (sub != 0) return;
  const int64_t plane = a.sc.ss * a.sc.fs;
  finish_pixel(a, p, best, braw, a.u[p], a.u[plane + p], a.var[p],
               win_off(a.offs_a, best / a.kb, a.ka), win_off(a.offs_b, best % a.kb, a.kb), total);
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
using FastKernel = void (*)(const __grid_constant__ CUtensorMap, PixArgs);
// fn72: box_c == 72, no frame weights (11 x 11 only: the specialised 13 x 13
// spilled at 255 registers, config 3 K2 93 -> 99 ms)
struct FastEntry { int ka, kb; FastKernel fn; FastKernel fn72; FastKernel fn40; };
#define PIX(a, b) FastEntry{a, b, k_pix_fast<a, b>, nullptr, nullptr}
#define PIX72(a, b) FastEntry{a, b, k_pix_fast<a, b>, k_pix_fast<a, b, 72>, k_pix_fast<a, b, 40>}
const FastEntry kFastTable[] = {
    PIX(1, 1),  PIX(3, 3),  PIX(5, 5),  PIX(7, 7),  PIX(9, 9),  PIX72(11, 11), PIX(13, 13),
    PIX(1, 3),  PIX(1, 5),  PIX(1, 7),  PIX(1, 9),  PIX(1, 11), PIX(1, 13),  PIX(1, 15),
    PIX72(1, 17), PIX(3, 1),  PIX(5, 1),  PIX(7, 1),  PIX(9, 1),  PIX(11, 1),  PIX(13, 1),
    PIX(15, 1), PIX(17, 1),
};
#undef PIX
#undef PIX72

FastKernel find_fast(int ka, int kb, int box_c = 0) {
  for (const auto& e : kFastTable)
    if (e.ka == ka && e.kb == kb)
      return (box_c == 72 && e.fn72) ? e.fn72 : (box_c == 40 && e.fn40) ? e.fn40 : e.fn;
  return nullptr;
}

}  // namespace
}  // namespace pxst

using namespace pxst;

namespace {
int pixel_map_search(const pxst_scan* sc, const pxst_stats* st, const pxst_ref* ref,
                     const double* u_in, const double* di, const double* dj, int64_t half_ss,
                     int64_t half_fs, double subpixel_step, int refine, const float* fw,
                     const double* var_fw, double* u_out, double* err_out,
                     const int32_t* span_hint, void* stream) {
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
  // u_out = u_in, err_out = 0 outside the work set: done by k_tile_geo for the
  // ROI on the fast path when the ROI is the whole detector, else here
  const bool full_roi = sc->roi[0] == 0 && sc->roi[1] == sc->ss && sc->roi[2] == 0 &&
                        sc->roi[3] == sc->fs;
  const bool fast_init = full_roi && sc->n_good > 0 && subpixel_step == 0.0 &&
                         !force_generic() &&
                         find_fast(static_cast<int>(2 * half_ss + 1),
                                   static_cast<int>(2 * half_fs + 1)) != nullptr;
  if (!fast_init) {
    PXST_CHECK_CUDA(cudaMemcpyAsync(u_out, u_in, sizeof(double) * 2 * plane,
                                    cudaMemcpyDeviceToDevice, s));
    PXST_CHECK_CUDA(cudaMemsetAsync(err_out, 0, sizeof(double) * plane, s));
  }
  if (sc->n_good == 0) return PXST_OK;

  const std::vector<double> oa = window_offsets(half_ss, subpixel_step);
  const std::vector<double> ob = window_offsets(half_fs, subpixel_step);
  const int na = static_cast<int>(oa.size()), nb = static_cast<int>(ob.size());
  const int nk = na * nb;
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];

  PixArgs a{};
  a.sc = *sc;
  a.u = u_in; a.di = di; a.dj = dj;
  a.fm = ref->fm; a.valid = ref->valid;
  a.os = ref->os; a.of = ref->of; a.n0 = ref->n0; a.m0 = ref->m0;
  a.fw = fw;
  a.var = fw ? var_fw : st->var_pm;
  a.ka = na; a.kb = nb;
  a.nq = cw * rw;

  FastKernel fn = (subpixel_step == 0.0 && !force_generic()) ? find_fast(na, nb) : nullptr;
  // window offsets: integer windows (the fast path) compute them inline
  Scratch offs;
  const double* d_oa = nullptr;
  const double* d_ob = nullptr;
  if (!fn) {
    if (int e = offs.alloc(sizeof(double) * (na + nb), s)) return e;
    if (int e = fill_offsets(offs.as<double>(), na, nb, subpixel_step, s)) return e;
    d_oa = offs.as<double>();
    d_ob = d_oa + na;
  }
  a.offs_a = d_oa;
  a.offs_b = d_ob;
  a.refine_ok = refine && subpixel_step == 0.0 && na >= 3 && nb >= 3;   // recon.py:273
  a.u_out = u_out;
  a.err_out = err_out;
  const unsigned qblocks = (unsigned)((a.nq + 127) / 128);

  if (fn) {
    const int ra = (na - 1) / 2, rb = (nb - 1) / 2;
    a.box_r = box_rows_for(na);
    a.box_c = box_cols_for(nb);
    a.tiles_x = static_cast<int>((cw + kTC - 1) / kTC);
    const int tiles_y = static_cast<int>((rw + kTR - 1) / kTR);
    PXST_REQUIRE(tiles_y <= kMaxGridY, "ROI too tall");
    const int64_t tiles = (int64_t)a.tiles_x * tiles_y;

    Scratch pvbuf, geo, part, fmpad, fmn, fm2;
    if (int e = pvbuf.alloc(ref->os * ref->of, s)) return e;
    if (int e = fmn.alloc(sizeof(float) * ref->os * ref->of, s)) return e;
    a.fmn = fmn.as<float>();
    // padded (value, mask) copy for the lanes-over-trials fix-up (windows of
    // more than 3 rows); the pad holds every trial corner of an on-grid sample
    a.pad = max(ra, rb) + 2;
    if (na > 3 && (ref->os + 2 * a.pad) * (ref->of + 2 * a.pad) < (int64_t(1) << 31) &&
        !getenv("PXST_K2_NO_PAD")) {
      if (int e = fm2.alloc(sizeof(float2) * (ref->os + 2 * a.pad) * (ref->of + 2 * a.pad), s))
        return e;
      a.fm2 = fm2.as<float2>();
    }
    a.pv = pvbuf.as<uint8_t>();
    if (int e = geo.alloc(sizeof(TileGeo) * tiles, s)) return e;
    a.geo = geo.as<TileGeo>();

    // TMA needs a 16-byte row pitch: pad the object image when of % 4 != 0.
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
    Scratch cnt;                 // slow-list count and work counter, zeroed by k_tile_geo
    if (int e = cnt.alloc(2 * sizeof(unsigned), s)) return e;
    {
      // patch-valid map + NaN-encoded reference (make_pv) and the tile
      // geometry in one launch
      PXST_REQUIRE(2 * ra + 1 <= kPvMaxHalo && 2 * rb + 1 <= kPvMaxHalo, "patch extent too large");
      PvJob pj{ref->valid, ref->fm, static_cast<int>(ref->os), static_cast<int>(ref->of),
               -ra, ra + 1, -rb, rb + 1, static_cast<int>((ref->of + kPvC - 1) / kPvC),
               pvbuf.as<uint8_t>(), fmn.as<float>(), fm2.as<float2>(), a.pad};
      const int64_t n_pv = (int64_t)pj.nx * ((ref->os + kPvR - 1) / kPvR);
      const int64_t blocks = n_pv + (tiles + kPrepTiles - 1) / kPrepTiles;
      PXST_REQUIRE(blocks < (int64_t(1) << 31), "reference image too large");
      k_k2_prep<<<(unsigned)blocks, 256, 0, s>>>(a, geo.as<TileGeo>(), fast_init ? 1 : 0,
                                                 cnt.as<unsigned>(), pj, static_cast<int>(n_pv),
                                                 tiles);
      PXST_CHECK_LAUNCH();
    }
    // Size the TMA box from the largest tile footprint (|du/dx| reaches ~1.8
    // at the edges of the config-3 map), capped at 24 KB per ring slot; tiles
    // beyond the cap take the exact path.
    int span[2];
    if (span_hint) {             // from pxst_tile_spans; a stale hint only costs speed
      span[0] = span_hint[0];
      span[1] = span_hint[1];
    } else if (int e = tile_span_max(geo.as<TileGeo>(), tiles, span, s)) {
      return e;
    }
    // (exactly the largest tile's need: round 2 kept the defaults as a floor
    // and fetched 17 x 72 cells per frame where config 2's tiles need 10 x 30
    // -- its one-row kernel was bound by the L2 -> shared-memory traffic)
#ifndef PXST_K2_TIGHT_BOX
#define PXST_K2_TIGHT_BOX 1
#endif
    if (PXST_K2_TIGHT_BOX && span[0] >= 0 && span[1] >= 0) {
      a.box_r = span[0] + need_rows2(na);
      a.box_c = span[1] + need_cols2(nb);
    } else {
      a.box_r = max(a.box_r, span[0] + need_rows2(na));
      a.box_c = max(a.box_c, span[1] + need_cols2(nb));
    }
    a.box_c = (a.box_c + 23) / 32 * 32 + 8;            // pitch = 8 (mod 32)
    if (a.box_c > 256) a.box_c = 232;
    while (a.box_r > 16 && a.box_r * a.box_c * 4 > 24 * 1024) --a.box_r;
    fn = find_fast(na, nb, fw ? 0 : a.box_c);            // compile-time row pitch if 72
    CUtensorMap tmap;
    if (int e = encode_tmap_2d_f32(&tmap, tbase, ref->os, ref->of, pitch, a.box_r, a.box_c))
      return e;
    // Work units.  Resident CTAs S = 2 per SM.  With <= 512 good frames (one
    // float32 partial holds them) the first floor(tiles / S) full waves are
    // whole tiles finished in the kernel; the remaining R tiles are split into
    // ~S / R frame chunks so the last wave is full.  More frames: every tile
    // is split (<= 512 frames per float32 partial, ~6 waves).
    int sms = 148;
    {
      int dev = 0;
      PXST_CHECK_CUDA(cudaGetDevice(&dev));
      PXST_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int64_t slots = kCtaPerSm * static_cast<int64_t>(sms);
    const int max_chunks = static_cast<int>(sc->n_good / 16 > 1 ? sc->n_good / 16 : 1);
    int n_chunks;
    a.n_full = 0;
    if (sc->n_good <= 512 && tiles >= slots && !getenv("PXST_K2_NO_FUSE")) {
      a.n_full = tiles / slots * slots;
      const int64_t rest = tiles - a.n_full;
      int64_t c = rest > 0 ? slots / rest : 1;
      c = c < 1 ? 1 : c;
      c = c > max_chunks ? max_chunks : c;
      n_chunks = static_cast<int>(c);
    } else {
      n_chunks = static_cast<int>((6 * slots + tiles - 1) / tiles);
      n_chunks = max(n_chunks, static_cast<int>((sc->n_good + 511) / 512));
      n_chunks = n_chunks < max_chunks ? n_chunks : max_chunks;
      n_chunks = n_chunks > 1 ? n_chunks : 1;
    }
    a.chunk = static_cast<int>((sc->n_good + n_chunks - 1) / n_chunks);
    a.n_chunks = static_cast<int>((sc->n_good + a.chunk - 1) / a.chunk);
    a.tbl = a.n_full > 0 ? static_cast<int>(sc->n_good) : a.chunk;
    const int64_t units = a.n_full + (tiles - a.n_full) * a.n_chunks;
    size_t smem = sizeof(float) * kNB * slot_floats(a.box_r, a.box_c) + 128 +
                  (sizeof(int4) + 3 * sizeof(double) + 2 * sizeof(int)) * a.tbl;
    if (a.n_full > 0)      // whole-tile units stage their trial sums in the ring
      smem = std::max(smem, sizeof(float) * nk * kThreads + 128 +
                                (sizeof(int4) + 3 * sizeof(double) + 2 * sizeof(int)) * a.tbl);
    PXST_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    if (int e = part.alloc(sizeof(float) * a.n_chunks * nk * a.nq, s)) return e;
    a.partial = part.as<float>();
    Scratch lst;
    if (int e = lst.alloc(sizeof(unsigned long long) * (a.nq * a.n_chunks + 1), s)) return e;
    unsigned* list_n = cnt.as<unsigned>();
    unsigned long long* list = lst.as<unsigned long long>();
    a.slow_list = list;
    a.slow_n = list_n;
    Scratch dbg;
    if (getenv("PXST_DEBUG")) {
      if (int e = dbg.alloc(3 * sizeof(unsigned long long), s)) return e;
      PXST_CHECK_CUDA(cudaMemsetAsync(dbg.p, 0, 3 * sizeof(unsigned long long), s));
      a.dbg = dbg.as<unsigned long long>();
    }
    PXST_REQUIRE(units < (int64_t(1) << 31), "ROI too large");
    fn<<<(unsigned)units, kThreads, smem, s>>>(tmap, a);
    PXST_CHECK_LAUNCH();
    if (na <= 3)          // 1 x N / 3 x N windows: >= 10 samples in flight per warp
      k_pix_slow_rows<<<2 * sms, 256, 0, s>>>(a, list, list_n);
    else
    {
      const int nj = (nk + 31) / 32;
      switch (nj) {
        case 1: k_pix_slow<1><<<PXST_K2_SLOW_OCC * sms, 256, 0, s>>>(a, list, list_n); break;
        case 2: k_pix_slow<2><<<PXST_K2_SLOW_OCC * sms, 256, 0, s>>>(a, list, list_n); break;
        case 3: k_pix_slow<3><<<PXST_K2_SLOW_OCC * sms, 256, 0, s>>>(a, list, list_n); break;
        case 4: k_pix_slow<4><<<PXST_K2_SLOW_OCC * sms, 256, 0, s>>>(a, list, list_n); break;
        case 5: k_pix_slow<5><<<2 * sms, 256, 0, s>>>(a, list, list_n); break;
        default: k_pix_slow<6><<<2 * sms, 256, 0, s>>>(a, list, list_n); break;
      }
    }
    PXST_CHECK_LAUNCH();
    if (getenv("PXST_DEBUG")) {
      unsigned h = 0;
      unsigned long long hs[3] = {0, 0, 0};
      PXST_CHECK_CUDA(cudaMemcpyAsync(&h, list_n, sizeof(h), cudaMemcpyDeviceToHost, s));
      PXST_CHECK_CUDA(cudaMemcpyAsync(hs, a.dbg, sizeof(hs), cudaMemcpyDeviceToHost, s));
      PXST_CHECK_CUDA(cudaStreamSynchronize(s));
      fprintf(stderr, "[pxst] K2 %dx%d: %lld pixels x %d chunks, %u (pixel, chunk) pairs own "
              "%llu slow samples (%llu off grid, %llu outside the %dx%d box, rest patch "
              "invalid)\n", na, nb, (long long)a.nq, a.n_chunks, h, hs[0], hs[1], hs[2],
              a.box_r, a.box_c);
    }
    const int64_t split_px = (tiles - a.n_full) * kThreads;
    if (split_px > 0) {
      if (a.n_full > 0)
        k_pix_epilogue<float, 4><<<(unsigned)((split_px * 4 + 127) / 128), 128, 0, s>>>(
            a, part.as<float>(), a.n_chunks);
      else
        k_pix_epilogue<float, 2><<<(unsigned)((split_px * 2 + 127) / 128), 128, 0, s>>>(
            a, part.as<float>(), a.n_chunks);
      PXST_CHECK_LAUNCH();
    }
    PXST_CHECK_LAUNCH();
    return PXST_OK;
  }
  // generic path
  Scratch errs;
  if (int e = errs.alloc(sizeof(double) * a.nq * nk, s)) return e;
  for (int t0 = 0; t0 < nk; t0 += kMaxGridY) {       // grid.y <= 65535 trials per launch
    dim3 g(qblocks, (unsigned)std::min(nk - t0, kMaxGridY));
    k_pix_generic<<<g, 128, 0, s>>>(a, d_oa, d_ob, errs.as<double>(), t0);
    PXST_CHECK_LAUNCH();
  }
  k_pix_epilogue<double, 2><<<qblocks * 2, 128, 0, s>>>(a, errs.as<double>(), 1);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}
}  // namespace

extern "C" int pxst_pixel_map_search(const pxst_scan* sc, const pxst_stats* st,
                                     const pxst_ref* ref, const double* u_in, const double* di,
                                     const double* dj, int64_t half_ss, int64_t half_fs,
                                     double subpixel_step, int refine, const float* fw,
                                     const double* var_fw, double* u_out, double* err_out,
                                     void* stream) {
  return pixel_map_search(sc, st, ref, u_in, di, dj, half_ss, half_fs, subpixel_step, refine, fw,
                          var_fw, u_out, err_out, nullptr, stream);
}

extern "C" int pxst_pixel_map_search_ex(const pxst_scan* sc, const pxst_stats* st,
                                        const pxst_ref* ref, const double* u_in,
                                        const double* di, const double* dj, int64_t half_ss,
                                        int64_t half_fs, double subpixel_step, int refine,
                                        const float* fw, const double* var_fw, double* u_out,
                                        double* err_out, const int32_t* span_hint,
                                        void* stream) {
  return pixel_map_search(sc, st, ref, u_in, di, dj, half_ss, half_fs, subpixel_step, refine, fw,
                          var_fw, u_out, err_out, span_hint, stream);
}

extern "C" int pxst_tile_spans(const pxst_scan* sc, const double* u, int32_t* spans,
                               void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(u && spans, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t cw = sc->roi[3] - sc->roi[2], rw = sc->roi[1] - sc->roi[0];
  PixArgs a{};
  a.sc = *sc;
  a.u = u;
  a.tiles_x = static_cast<int>((cw + kTC - 1) / kTC);
  const int tiles_y = static_cast<int>((rw + kTR - 1) / kTR);
  PXST_REQUIRE(tiles_y <= kMaxGridY, "ROI too tall");
  const int64_t tiles = (int64_t)a.tiles_x * tiles_y;
  Scratch geo;
  if (int e = geo.alloc(sizeof(TileGeo) * tiles, s)) return e;
  k_tile_geo<<<dim3((unsigned)a.tiles_x, (unsigned)tiles_y), kThreads, 0, s>>>(a, geo.as<TileGeo>(),
                                                                             0);
  PXST_CHECK_LAUNCH();
  return tile_span_max_dev(geo.as<TileGeo>(), tiles, spans, s);
}
