// Deterministic bilinear splat (K1 object formation, K4 reference plane).
//
// The reference accumulates the splat terms t = value * weight * w_c in
// float64 with np.bincount (interp.py:113-122), one fixed order.  Here every
// term is rounded once to an integer multiple of a power-of-two quantum q
// (round to nearest even) and the integers are summed exactly: the result is
// independent of the order of the additions, of the kernel's work
// decomposition and of the number of GPUs (frame shards add their int64
// accumulators).  q = 2^e is chosen per accumulator from a bound on |t|
// (|t| < 2^41 q), so a term keeps ~41 significant bits relative to the
// largest possible term (pxst_object_quanta / pxst_plane_quanta).
//
// A term is carried as two 32-bit limbs, lo = v mod 2^21 (unsigned) and
// hi = floor(v / 2^21) (signed, |hi| < 2^20), so a CTA can accumulate up to
// 2047 terms per cell with native 32-bit shared-memory atomics (ATOMS.ADD;
// 64-bit shared atomics are CAS loops, ~6x slower on sm_100a) before its
// region is added to the global int64 accumulators.
#pragma once

#include "common.cuh"

namespace pxst {

constexpr int kFixTermBits = 41;         // |term| < 2^41 quanta
constexpr int kFixLoBits = 21;           // lo limb width
constexpr int kFixMaxTerms = 2047;       // terms per cell per shared-memory session
constexpr double kFixMagic = 6755399441055744.0;            // 1.5 * 2^52
constexpr unsigned long long kFixMagicBits = 0x4338000000000000ull;
// assumed bound on the pixels whose bilinear corners reach one cell in one
// frame (local magnification >= 1/16): sets the headroom of the global int64
// sums, N_good * kFixCellDensity * 2^41 < 2^63 (else q grows by 2^k)
constexpr int kFixCellDensity = 256;

// Limbs of round(scaled * w) (|scaled * w| < 2^41): one DFMA against the
// magic constant puts the rounded integer in the low mantissa bits (the
// magic's low 21 bits are zero, so the limbs need no 64-bit subtract).
__device__ __forceinline__ void fix_limbs(double scaled, double w, unsigned& lo, int& hi) {
  const double x = fma(scaled, w, kFixMagic);
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const unsigned blo = static_cast<unsigned>(b), bhi = static_cast<unsigned>(b >> 32);
  lo = blo & ((1u << kFixLoBits) - 1u);
  hi = static_cast<int>(__funnelshift_r(blo, bhi, kFixLoBits) -
                        static_cast<unsigned>(kFixMagicBits >> kFixLoBits));
}

// The full integer of the same term (for the direct global path).
__device__ __forceinline__ long long fix_value(double scaled, double w) {
  const double x = fma(scaled, w, kFixMagic);
  return __double_as_longlong(x) - static_cast<long long>(kFixMagicBits);
}

__device__ __forceinline__ long long fix_join(unsigned lo, int hi) {
  return static_cast<long long>(hi) * (1ll << kFixLoBits) + static_cast<long long>(lo);
}

// 2^(ceil(log2 m) - 41 + k): the quantum for terms bounded by m.
__device__ __forceinline__ double fix_quantum(double m, int k) {
  if (!(m > 0.0) || !isfinite(m)) m = 1.0;
  int e;
  frexp(m, &e);                        // m = f 2^e, f in [0.5, 1): m <= 2^e
  return ldexp(1.0, e - kFixTermBits + k);
}

// Headroom exponent k of the global sums for n_good frames: at most
// n_good * kFixCellDensity terms of < 2^(41-k) quanta per cell stay < 2^63.
__host__ __device__ inline int fix_headroom(int64_t n_good) {
  const long long c = static_cast<long long>(n_good > 0 ? n_good : 1) * kFixCellDensity;
  int k = 0;
  while ((1ll << (22 + k)) < c) ++k;
  return k;
}

// Terms whose bilinear corner weight is below kFineW = 2^-20 are summed
// apart, in units of q * 2^-kFineShift (a single int64 per term,
// |t| < 2^(41-20+20) = 2^41 fine quanta): a cell reached only by tiny-weight
// corners (e.g. the grid's last row, weighted by the fractions of the
// outermost samples) keeps 20 more bits; a coarse term of weight >= 2^-20
// keeps >= 21.  Such corners are rare (~1e-5 of the samples), so they go
// straight to global memory.
constexpr double kFineW = 0x1p-20;
constexpr int kFineShift = 20;

// Device accumulators of one image, int64: num / den in units of the quanta
// q[0] / q[1], num_f / den_f in units of q * 2^-kFineShift; touched
// (nullable) = a tiny-weight term landed (so that a cell whose whole weight
// rounds to zero stays valid: the reference's wsum > 0, data_model.py:186).
struct FixAcc {
  long long* num;
  long long* den;
  long long* num_f;
  long long* den_f;
  uint8_t* touched;
  const double* q;
};

// Normalise one cell (interp.py:126-135): out = num/den where den > 0 else
// 0, with num = num q + num_f q 2^-20 (likewise den).  The object's validity
// is "a positive-weight term landed": den > 0, or a tiny-weight term marked
// the cell (touched) -- such a cell whose weight rounds to zero keeps
// valid = 1 with value 0 and wsum = q 2^-62.  Every output is nullable.
__device__ __forceinline__ void fix_finish_cell(const FixAcc& acc, int64_t i, double* out,
                                                double* wsum, float* fm, uint8_t* valid) {
  const double qn = acc.q[0], qd = acc.q[1];
  const double d = static_cast<double>(acc.den[i]) * qd +
                   static_cast<double>(acc.den_f[i]) * (qd * 0x1p-20);
  const double nm = static_cast<double>(acc.num[i]) * qn +
                    static_cast<double>(acc.num_f[i]) * (qn * 0x1p-20);
  const bool pos = d > 0.0;
  const bool ok = pos || (acc.touched && acc.touched[i] != 0);
  const double v = pos ? nm / d : 0.0;
  if (out) out[i] = v;
  if (wsum) wsum[i] = pos ? d : (ok ? qd * 0x1p-62 : 0.0);
  if (fm) fm[i] = ok ? static_cast<float>(v) : 0.f;
  if (valid) valid[i] = ok ? 1 : 0;
}

constexpr int kMaxPeers = 16;   // GPUs of one process (pxst_object_finish_peers)

// One launch for the scale statistics and the quanta (and, in the same
// grid-stride loops, K4's grouped reference and a zero fill): see
// k_quanta_pass.  ticket must be zero when the kernel starts.
struct QuantaJob {
  pxst_scan sc;
  const double* sigma2;         // nullable (object quanta: kind 0)
  const double* fm64;           // reference (nullable valid: none)
  const float* fm;
  const uint8_t* valid;
  int64_t os, of;
  const double* absmax;
  int kind;                     // 0 object, 1 reference plane
  double* quanta;               // nullable: side jobs only
  unsigned* ticket;
  double2* grp;                 // nullable: g[r][c] = (v(r, c), v(r + 1, c)), NaN = invalid
  double* zero;                 // nullable: zero[0, n_zero) = 0
  int64_t n_zero;
};
int launch_quanta_job(const QuantaJob& j, cudaStream_t s);

}  // namespace pxst
