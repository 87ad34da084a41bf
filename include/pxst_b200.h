/*
 * pxst_b200.h -- C ABI of the B200-native PXST hot path (arXiv 2003.12726).
 *
 * One shared library, libpxst_b200.so, hand-written CUDA for sm_100a.  Every
 * entry point takes DEVICE pointers owned by the caller plus a cudaStream_t
 * passed as `void*` (NULL = legacy default stream), enqueues its kernels on
 * that stream and returns a status code; nothing is synchronised unless the
 * function says so.  No torch types cross this boundary.  The library keeps
 * no global state except a thread-local error string; scratch memory is
 * taken from the stream-ordered allocator (cudaMallocAsync) and released on
 * the same stream before the call returns.
 *
 * The reference (pure NumPy, /root/reference/pkg/src/pxst) has no FFI; the
 * entry points below are what its Python hot path binds to through ctypes
 * (see INTEGRATION.md).  Each cites the reference function it replaces.
 *
 * Conventions shared with the reference (data_model.py:3-12):
 *   - axis order [slow-scan (ss), fast-scan (fs)], row-major, fs fastest;
 *   - u: [2, ss, fs] float64 pixel map in reference-grid pixels;
 *   - di, dj: [n_frames] float64 translations (reference-grid pixels);
 *   - reference grid origin (n0, m0) is subtracted from u - delta.
 */
#ifndef PXST_B200_H
#define PXST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PXST_ABI_VERSION 2

/* status codes */
#define PXST_OK 0
#define PXST_EINVAL 1   /* bad argument: maps to ValueError in the Python shim   */
#define PXST_ECUDA 2    /* CUDA runtime / launch error: maps to RuntimeError     */
#define PXST_ENOMEM 3   /* device allocation failed                              */

/* A scan resident on one device.  Mirrors recon._work_set (recon.py:81-96):
 * the kernels read the stack in place; work pixels are work[ss,fs] != 0
 * (mask & W > 0 & inside the half-open ROI), good frames are good[0..n_good). */
typedef struct pxst_scan {
  const float* frames;    /* [n_frames, ss, fs] float32                          */
  int64_t n_frames, ss, fs;
  const int32_t* good;    /* [n_good] frame indices, ascending                   */
  int64_t n_good;
  const double* w64;      /* [ss, fs] whitefield, float64                        */
  const float* w32;       /* [ss, fs] whitefield, float32 copy                   */
  const uint8_t* work;    /* [ss, fs] work-pixel flags                           */
  int64_t roi[4];         /* ss_min, ss_max, fs_min, fs_max (half-open)          */
} pxst_scan;

/* Per-scan statistics, iteration invariant.  Device buffers
 * allocated by the caller; filled by pxst_stack_stats. */
typedef struct pxst_stats {
  double* var_pm;      /* [ss*fs] sum_n (I-W)^2, pixel-map normaliser (recon.py:257-263) */
  double* sigma2;      /* [ss*fs] population variance over good frames, floored
                          at 1e-8 max(W)^2 (recon.py:410-412); 0 off the work set  */
  double* frame_norm;  /* [n_good] sum_p (I_n-W)^2 (recon.py:367)                   */
  double* scalars;     /* [4]: max W over work px, sum |I| W, n_work, sum |I|        */
} pxst_stats;

/* Reference image on device: fm = i_ref where valid else 0 (float32),
 * valid = wsum > 0 (data_model.py:186-188).  fm64 (nullable) is the same
 * image in float64; the error maps use it when present. */
typedef struct pxst_ref {
  const float* fm;        /* [os, of] */
  const uint8_t* valid;   /* [os, of] */
  int64_t os, of;
  int64_t n0, m0;
  const double* fm64;     /* [os, of] or NULL */
} pxst_ref;

int pxst_abi_version(void);
const char* pxst_last_error(void);
/* Number of kernels this thread has launched through the library (for the
 * bench's gpu_launches count). */
int64_t pxst_launch_count(void);
/* Return the scratch memory the library keeps in the current device's
 * default memory pool to the driver (synchronises the device).  The
 * library raises the pool's release threshold so stream-ordered scratch is
 * not re-mapped at every synchronisation; this undoes the retention (the
 * Python shim's clear_cache() calls it). */
int pxst_release_pool(void);

/* K0: per-scan statistics.  Replaces the fallback/variance/normaliser
 * computations at recon.py:257-260, :367 and :410-412.  `fw` (nullable,
 * [n_frames, ss, fs] float32) gives frame weights; then var_pm is
 * sum_n fw (I-W)^2 as at recon.py:258-260. */
int pxst_stack_stats(const pxst_scan* scan, const float* fw, const pxst_stats* st,
                     void* stream);

/* The same statistics in two independent parts: PXST_STATS_PIXEL = max W,
 * var_pm, sigma2 (what K2 and K4 read); PXST_STATS_FRAME = frame_norm and
 * the |I| sums (what K3 reads).  pxst_stack_stats = both. */
#define PXST_STATS_PIXEL 1
#define PXST_STATS_FRAME 2
int pxst_stack_stats_parts(const pxst_scan* scan, const float* fw, const pxst_stats* st,
                           int parts, void* stream);

/* Bounding box of u over work pixels and of (di, dj) over good frames:
 * out[8] (device, float64) = min u0, max u0, min u1, max u1, min di, max di,
 * min dj, max dj.  Feeds the grid rule of recon.py:126-132. */
int pxst_bbox(const pxst_scan* scan, const double* u, const double* di, const double* dj,
              double* out, void* stream);

/* pxst_bbox and, in the same launch, the grid rule of recon.py:126-132:
 * grid[4] (device, int64, nullable) = (n0, m0, os, of) -- what
 * pxst_grid_rule computes from out. */
int pxst_bbox_grid(const pxst_scan* scan, const double* u, const double* di, const double* dj,
                   double* out, int64_t* grid, void* stream);

/* Deterministic splat accumulators (K1 object numerator / denominator, K4
 * reference-plane numerator / denominator).  Every float64 term t of the
 * reference's bincount (interp.py:113-122) is rounded once to an integer
 * multiple of a power-of-two quantum q (round to nearest even) and the
 * integers are summed exactly in int64, so the images do not depend on the
 * order of the additions, on the kernels' work split or on the number of
 * GPUs: frame shards all-reduce num/den as int64 (exact) and touched with
 * max.  quanta (device, float64[2]) = (q_num, q_den), chosen so that
 * |t| < 2^41 q (pxst_object_quanta / pxst_plane_quanta; ~41 significant
 * bits relative to the largest possible term).  A cell is valid (the
 * reference's wsum > 0, data_model.py:186) when den + den_fine > 0 or a
 * tiny-weight term marked it in touched. */
typedef struct pxst_accum {
  int64_t* num;           /* [cells], units of quanta[0]                        */
  int64_t* den;           /* [cells], units of quanta[1]                        */
  int64_t* num_fine;      /* [cells], units of quanta[0] * 2^-20: terms whose   */
  int64_t* den_fine;      /*   bilinear corner weight is < 2^-10 (cells reached */
                          /*   only by tiny-weight corners keep their precision)*/
  uint8_t* touched;       /* [cells] or NULL: a tiny-weight term landed         */
  const double* quanta;   /* device [2]                                         */
} pxst_accum;

/* Zero `cells` cells of every array of an accumulator (cudaMemsetAsync). */
int pxst_accum_zero(const pxst_accum* acc, int64_t cells, void* stream);

/* max |I| over the whole frame stack (device float64 scalar): the bound the
 * quanta are derived from.  One pass over the stack; cache it per stack. */
int pxst_stack_absmax(const pxst_scan* scan, double* out, void* stream);

/* Quanta of the object accumulators: q_num from max|I| max W, q_den from
 * max W^2 (max W over the ROI's work pixels), with headroom for n_good
 * frames.  Frame shards must use the same quanta (same scan, same absmax). */
int pxst_object_quanta(const pxst_scan* scan, const double* absmax, double* quanta,
                       void* stream);

/* K1 object formation, splat half (recon.py:99-138; interp.py:88-123).
 * Adds, for every good frame in [frame_lo, frame_hi) of scan->good and work
 * pixel, the fixed-point terms of I*W*w_c to acc->num and W^2*w_c to
 * acc->den ([os*of]) at the four bilinear corners of (u0 - di - n0,
 * u1 - dj - m0), and marks acc->touched.  Points outside [0,os-1]x[0,of-1]
 * are dropped whole; their count is added to *n_dropped (device, nullable).
 * Frame ranges let frame shards accumulate partial images that are summed
 * (int64 all-reduce) before pxst_object_finish. */
int pxst_object_splat(const pxst_scan* scan, const double* u, const double* di,
                      const double* dj, int64_t n0, int64_t m0, int64_t os, int64_t of,
                      int64_t frame_lo, int64_t frame_hi, const pxst_accum* acc,
                      unsigned long long* n_dropped, void* stream);

/* K1 normalise (interp.py:126-135): i_ref = num/den where den > 0 else 0,
 * wsum = den (in float64 units), valid = touched (or den > 0 without
 * touched); also writes the float32 masked image fm the search kernels read.
 * Any of the four outputs may be NULL.  (A touched cell whose whole weight
 * rounds below one quantum keeps valid = 1 with i_ref = 0 and a tiny wsum.) */
int pxst_object_finish(const pxst_accum* acc, int64_t n, double* i_ref, double* wsum, float* fm,
                       uint8_t* valid, void* stream);

/* Single-process multi-GPU: the frame shards' all-reduce fused with
 * pxst_object_finish (replaces the NCCL all-reduce of recon.py:133-141's
 * numerator / denominator in the one-process driver).  accs[0..n_peers) are
 * the accumulators of ALL peers (device pointers on n_peers <= 16 devices with
 * peer access enabled; the same full-scan quanta on every peer).  The call
 * runs on the stream's device and handles its slice of cells
 * [cell_lo, cell_hi): it reads every peer's int64 terms where they lie (P2P
 * loads), adds them (exact: the same bits on every device, in any order),
 * normalises, and stores the slice's results into EVERY peer's output images
 * i_ref[j] / wsum[j] / fm[j] / valid[j] (host arrays of n_peers device
 * pointers, any array or entry nullable; P2P stores).  Once every device has
 * run its slice and the devices have been synchronised, each holds the whole
 * object.  Also finishes reference planes (K4 row shards). */
int pxst_object_finish_peers(const pxst_accum* accs, int n_peers, int64_t cell_lo,
                             int64_t cell_hi, double* const* i_ref, double* const* wsum,
                             float* const* fm, uint8_t* const* valid, void* stream);

/* Convenience: absmax + quanta + splat + finish over all good frames for a
 * known grid (recon.make_reference after the bbox of pxst_bbox). */
int pxst_object_map(const pxst_scan* scan, const double* u, const double* di, const double* dj,
                    int64_t n0, int64_t m0, int64_t os, int64_t of, double* i_ref, double* wsum,
                    float* fm, uint8_t* valid, void* stream);

/* K2 pixel-map grid search + argmin + paraboloid refinement
 * (recon.py:144-170, 183-207, 221-296 with sigma = 0, integrate = False).
 * subpixel_step = 0 selects the integer grid -half..half; otherwise
 * step*(-k..k), k = round(half/step) (recon.py:51-57).  fw / var_fw
 * (nullable) carry frame weights and their normaliser.  u_out [2,ss,fs] is
 * a copy of u_in with work pixels updated; err_out [ss,fs] is the selected
 * normalised error (0 off the work set and for static pixels). */
int pxst_pixel_map_search(const pxst_scan* scan, const pxst_stats* st, const pxst_ref* ref,
                          const double* u_in, const double* di, const double* dj,
                          int64_t half_ss, int64_t half_fs, double subpixel_step, int refine,
                          const float* fw, const double* var_fw, double* u_out,
                          double* err_out, void* stream);

/* Same, with the TMA window sizing hint span_hint (host int32[2]) taken from
 * pxst_tile_spans on the same u instead of a device->host read inside the
 * call: with the hint the call never synchronises the stream.  A hint that
 * does not match u costs speed only (tiles whose window does not fit the
 * box take the exact path).  span_hint = NULL behaves as
 * pxst_pixel_map_search. */
int pxst_pixel_map_search_ex(const pxst_scan* scan, const pxst_stats* st, const pxst_ref* ref,
                             const double* u_in, const double* di, const double* dj,
                             int64_t half_ss, int64_t half_fs, double subpixel_step, int refine,
                             const float* fw, const double* var_fw, double* u_out,
                             double* err_out, const int32_t* span_hint, void* stream);

/* Largest per-tile extent of u over the K2 pixel tiles (rows, cols; device
 * int32[2]), the window sizing input of pxst_pixel_map_search_ex.  Depends
 * on u only, so it can be computed (and copied to the host) ahead of time,
 * e.g. on a side stream while the error maps run. */
int pxst_tile_spans(const pxst_scan* scan, const double* u, int32_t* spans, void* stream);

/* K3 per-frame translation grid search (recon.py:336-385), including the
 * reference's quirks: offsets enter as u - (d + off) and the paraboloid
 * offset (grid-index units) is added in pixels whenever the argmin is
 * interior.  Frames in [frame_lo, frame_hi) of scan->good are searched;
 * di_out / dj_out [n_frames] must already hold the input translations (only
 * searched frames with a positive normaliser are overwritten).  err_out
 * (nullable) receives the normalised [n_searched, Ka, Kb] error grids. */
int pxst_translation_search(const pxst_scan* scan, const pxst_stats* st, const pxst_ref* ref,
                            const double* u, const double* di, const double* dj,
                            int64_t half_ss, int64_t half_fs, double subpixel_step,
                            int64_t frame_lo, int64_t frame_hi, double* di_out,
                            double* dj_out, double* err_out, void* stream);

/* Same, with K3's TMA box sized from span_hint (host int32[2], from
 * pxst_tile_spans3 of this u or a bound of it) instead of a device->host
 * read inside the call; a hint that does not match u costs speed only. */
int pxst_translation_search_ex(const pxst_scan* scan, const pxst_stats* st, const pxst_ref* ref,
                               const double* u, const double* di, const double* dj,
                               int64_t half_ss, int64_t half_fs, double subpixel_step,
                               int64_t frame_lo, int64_t frame_hi, double* di_out,
                               double* dj_out, double* err_out, const int32_t* span_hint,
                               void* stream);

/* Largest row / column extent of u over K3's 16x64-pixel tiles (device
 * int32[2], no host wait): the span hint of pxst_translation_search_ex. */
int pxst_tile_spans3(const pxst_scan* scan, const double* u, int32_t* spans, void* stream);

/* Quanta of the reference-plane accumulators (see pxst_accum): q_num from
 * the bound (max|I| + max W max(1, max|ref|))^2 / min sigma2 on eps, q_den
 * from 1 (weight 1).  Row shards must share the full scan's quanta. */
int pxst_plane_quanta(const pxst_scan* scan, const double* absmax, const pxst_stats* st,
                      const pxst_ref* ref, double* quanta, void* stream);

/* K4 error maps (recon.py:388-438), one pass over the stack: per_frame
 * [n_frames] (0 for frames not good), per_pixel [ss,fs], ref_plane [os,of]
 * (normalised reference-plane projection of the residuals, every work sample
 * splatted with weight 1, in exact fixed point: bit-reproducible), total
 * (device scalar).  absmax (nullable) = pxst_stack_absmax of the stack;
 * computed here when NULL. */
int pxst_error_maps(const pxst_scan* scan, const pxst_stats* st, const pxst_ref* ref,
                    const double* u, const double* di, const double* dj, const double* absmax,
                    double* per_frame, double* per_pixel, double* ref_plane, double* total,
                    void* stream);

/* K4 fused with the NEXT iteration's K1 splat: calc_error(ref, u, t) and
 * make_reference(u, t) read the same samples at the same positions
 * u - delta (recon.py:511-516 calls them back to back), so one pass over the
 * stack produces the error maps of `ref` and adds the next object's
 * fixed-point terms into `next` as pxst_object_splat would (next->quanta
 * from pxst_object_quanta).  The next grid (n0, m0, os, of) is read from
 * DEVICE memory `grid` (e.g. written by pxst_bbox + pxst_grid_rule on a side
 * stream), so the call never waits for the host; next holds `capacity` cells
 * (the grid is laid out densely in the first os*of) and a grid with
 * os*of > capacity is not splatted -- the caller, who learns the grid later,
 * then forms the object separately.  Finish it with pxst_object_finish. */
int pxst_error_maps_splat(const pxst_scan* scan, const pxst_stats* st, const pxst_ref* ref,
                          const double* u, const double* di, const double* dj,
                          const double* absmax, double* per_frame, double* per_pixel,
                          double* ref_plane, double* total, const int64_t* grid,
                          int64_t capacity, const pxst_accum* next, void* stream);

/* Grid rule of recon.py:126-132 on the device: grid[4] = (n0, m0, os, of)
 * from the 8 bbox values of pxst_bbox (both device pointers). */
int pxst_grid_rule(const double* bbox, int64_t* grid, void* stream);

/* K4 without the final normalisation, for detector-row shards: per_frame
 * [n_frames] = this ROI's per-frame sums, per_pixel [ss,fs] (this ROI only),
 * and the reference-plane fixed-point terms ADDED into plane ([os,of],
 * caller-zeroed, quanta from pxst_plane_quanta of the FULL scan).  After an
 * all-reduce (sum) of per_frame and of plane->num / plane->den (int64,
 * exact) across shards, pxst_object_finish(plane, ...) yields
 * reference_plane. */
int pxst_error_partials(const pxst_scan* scan, const pxst_stats* st, const pxst_ref* ref,
                        const double* u, const double* di, const double* dj, double* per_frame,
                        double* per_pixel, const pxst_accum* plane, void* stream);

/* Elementwise reductions of the single-process multi-GPU path (device
 * pointers on the stream's device; `src` is a peer's accumulator copied
 * over NVLink): dst += src (int64: the exact fixed-point images; float64: the
 * per-frame error sums, added by every device in the same peer order) and
 * dst |= src (touched flags). */
int pxst_add_i64(int64_t* dst, const int64_t* src, int64_t n, void* stream);
int pxst_add_f64(double* dst, const double* src, int64_t n, void* stream);
int pxst_or_u8(uint8_t* dst, const uint8_t* src, int64_t n, void* stream);

/* Frame stack of another element type -> float32 on the device.  The
 * reference takes frames of any dtype and casts them where it reads them
 * (recon.py:91 scan.frames[good][:, idx_ss, idx_fs].astype(np.float64)); the
 * kernels read a float32 stack, so a stack of detector counts is uploaded in
 * its own type (half the bytes for 16-bit counts, no host conversion pass)
 * and converted here (round to nearest even, as numpy's astype(float32)). */
enum { PXST_U8 = 1, PXST_I8, PXST_U16, PXST_I16, PXST_U32, PXST_I32, PXST_U64, PXST_I64,
       PXST_F64 };
int pxst_stack_to_f32(const void* src, int type_code, int64_t n, float* dst, void* stream);

/* Mean and variance (ddof 0) of v[i] over the cells with valid[i] != 0, in a
 * fixed summation order: out[3] (device) = (count, mean, variance).  The
 * contrast var / mean^2 of the merged reference that
 * geometry.fit_defocus_registration maximises (geometry.py:214-222:
 * ref.i_ref[ref.valid] -> np.var / np.mean ** 2). */
int pxst_masked_moments(const double* v, const uint8_t* valid, int64_t n, double* out,
                        void* stream);

/* Interpolation primitives (interp.py:53-85 and :88-123), for the drop-in
 * interp module and the parity tests.  gather: vals/ok at n points of the
 * masked image.  splat: float64 accumulation into acc_v/acc_w [os,of]
 * (adds to their current contents); returns the dropped count in *n_dropped
 * (host, synchronises the stream). */
int pxst_gather(const pxst_ref* ref, const double* x, const double* y, int64_t n,
                double* vals, uint8_t* ok, void* stream);
int pxst_splat(double* acc_v, double* acc_w, int64_t os, int64_t of, const double* x,
               const double* y, const double* value, const double* weight, int64_t n,
               int64_t* n_dropped, void* stream);

/* ---- pixel-map regularisation (recon.py:298-311) ---- */

/* Mask-aware Gaussian regularisation of the displacement, in place on
 * u [2, ss, fs] (recon.py:210-218 applied at :300-304): per component
 * d = u - identity, num = G(d*M), den = G(M) with G = scipy
 * gaussian_filter(sigma, mode="nearest", truncate 4) (axis 0 then axis 1),
 * u = identity + (M && den > 0 ? num/den : d).  support [ss, fs] is M.
 * The filter taps are computed on the host exactly as scipy does and copied
 * to the device; the call synchronises the stream before returning. */
int pxst_smooth_displacement(double* u, const uint8_t* support, int64_t ss, int64_t fs,
                             double sigma, void* stream);

typedef struct pxst_cg_info {
  int64_t iterations;   /* CG iterations run                                   */
  double residual;      /* best relative residual |r| / |b|                     */
  int converged;        /* residual <= tol                                     */
} pxst_cg_info;

/* Least-squares potential of a gradient field on a mask
 * (integration.py:61-118): conjugate gradients on the masked Poisson normal
 * operator with the anchor term at the first mask pixel (row-major), stopped
 * at |r|/|b| <= tol or maxiter (maxiter <= 0: 20*ss*fs); the best iterate is
 * returned shifted to phi[anchor] = 0.  solver 0 = plain CG (the
 * reference's iteration); solver 1 = the same CG preconditioned by an
 * aggregation-multigrid V-cycle (same operator, stopping rule and gauge;
 * converges to the same potential in far fewer iterations).  gx, gy, phi
 * [ss, fs] float64 (device); info (host, nullable) is written after a stream
 * sync.  Returns PXST_EINVAL if the mask is empty (the reference's
 * ValueError). */
int pxst_integrate_gradient(const double* gx, const double* gy, const uint8_t* mask,
                            int64_t ss, int64_t fs, double tol, int64_t maxiter, int solver,
                            double* phi, pxst_cg_info* info, void* stream);

/* Irrotational projection of the displacement, in place on u [2, ss, fs]
 * (integration.py:121-134 applied at recon.py:305-311): fits phi to
 * (u0 - i, u1 - j) on the support and sets u = identity + grad(phi) there
 * (forward differences, last row/column backward). */
int pxst_project_irrotational(double* u, const uint8_t* support, int64_t ss, int64_t fs,
                              double tol, int64_t maxiter, int solver, pxst_cg_info* info,
                              void* stream);

/* ---- split-half uncertainty (analysis.py:306-361) ---- */

/* The counter-based sample split of split_half_recon (analysis.py:294-303,
 * :326-328): for every flat stack index k in [0, n_frames*ss*fs),
 * bit(k) = SplitMix64-finaliser(k + seed * 0x9E3779B97F4A7C15) & 1 and
 * fw[k] = bit (half 0, "A") or 1 - bit (half 1, "B"), float32, device;
 * fw must be 16-byte aligned.  fw is the frame-weight input of
 * pxst_stack_stats / pxst_pixel_map_search. */
int pxst_split_weights(uint64_t seed, int64_t n_frames, int64_t ss, int64_t fs, int half,
                       float* fw, void* stream);

/* counts_a[p] = sum over good frames of bit(good[k]*ss*fs + p): the half-A
 * sample count per pixel (analysis.py:333-334); half B has n_good - counts_a. */
int pxst_split_counts(uint64_t seed, const int32_t* good, int64_t n_good, int64_t ss, int64_t fs,
                      int32_t* counts_a, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PXST_B200_H */
