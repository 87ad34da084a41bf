// K1 object formation (recon.py:99-141) and the interp primitives
// (interp.py:53-135).
//
// The reference accumulates the bilinear splat in float64 with np.bincount
// (interp.py:114-122).  Here the splat runs through the deterministic
// fixed-point pass of fixsplat.cu (mode 0): every term I/W * W^2 * w_c and
// W^2 * w_c is rounded once to a power-of-two quantum and summed exactly in
// int64, so the object map is bit-identical from run to run, for any frame
// split and any number of GPUs (the int64 images of frame shards add
// exactly).
#include "fixsplat.cuh"

namespace pxst {

struct FixArgs;
template <int MODE> int launch_fix_pass(FixArgs& a, int* n_z_out, cudaStream_t s);
int launch_abs_max(const pxst_scan* sc, double* out, cudaStream_t s);
int launch_quanta(const pxst_scan* sc, const double* absmax, const double* sigma2,
                  const pxst_ref* ref, int kind, double* quanta, cudaStream_t s);
int launch_fix_finish_peers(const FixAcc* accs, int w, int64_t lo, int64_t hi, double* const* out,
                            double* const* wsum, float* const* fm, uint8_t* const* valid,
                            cudaStream_t s);
int launch_fix_finish(const FixAcc& acc, const int64_t* grid, int64_t n, double* out, double* wsum,
                      float* fm, uint8_t* valid, cudaStream_t s);
int launch_object_fix(const pxst_scan* sc, const double* u, const double* di, const double* dj,
                      int64_t n0, int64_t m0, int64_t os, int64_t of, int64_t frame_lo,
                      int64_t frame_hi, const FixAcc& acc, unsigned long long* n_drop,
                      cudaStream_t s);

namespace {

__global__ void k_gather(pxst_ref ref, const double* __restrict__ x, const double* __restrict__ y,
                         int64_t n, double* vals, uint8_t* ok) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double xx = x[q], yy = y[q];
    float v = 0.f;
    bool good = false;
    if (isfinite(xx) && isfinite(yy) && fabs(xx) < 2e9 && fabs(yy) < 2e9) {
      const Split sx = split(xx), sy = split(yy);
      good = masked_read(ref.fm, ref.valid, ref.os, ref.of, sx.i, sy.i, sx.f, sy.f, v);
    }
    vals[q] = good ? static_cast<double>(v) : 0.0;
    ok[q] = good ? 1 : 0;
  }
}

__global__ void k_splat_f64(double* acc_v, double* acc_w, int64_t os, int64_t of,
                            const double* __restrict__ x, const double* __restrict__ y,
                            const double* __restrict__ value, const double* __restrict__ weight,
                            int64_t n, unsigned long long* n_drop) {
  unsigned long long dropped = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double xx = x[q], yy = y[q];
    if (!(xx >= 0.0 && xx <= static_cast<double>(os - 1) && yy >= 0.0 &&
          yy <= static_cast<double>(of - 1))) {
      ++dropped;
      continue;
    }
    const Split sx = split(xx), sy = split(yy);
    const double wt = weight ? weight[q] : 1.0;
    const double vw = value[q] * wt;
    const int r0 = sx.i, c0 = sy.i;
    const int r1 = min(r0 + 1, static_cast<int>(os - 1));
    const int c1 = min(c0 + 1, static_cast<int>(of - 1));
    const double gx = 1.0 - sx.f, gy = 1.0 - sy.f;
    const double cw[4] = {gx * gy, gx * sy.f, sx.f * gy, sx.f * sy.f};
    const int64_t cell[4] = {(int64_t)r0 * of + c0, (int64_t)r0 * of + c1,
                             (int64_t)r1 * of + c0, (int64_t)r1 * of + c1};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      atomicAdd(acc_v + cell[k], vw * cw[k]);
      atomicAdd(acc_w + cell[k], wt * cw[k]);
    }
  }
  if (dropped) atomicAdd(n_drop, dropped);
}

}  // namespace

int check_scan(const pxst_scan* sc);

}  // namespace pxst

using namespace pxst;

static int check_accum(const pxst_accum* acc) {
  PXST_REQUIRE(acc && acc->num && acc->den && acc->num_fine && acc->den_fine && acc->quanta,
               "bad accumulator");
  return PXST_OK;
}

static FixAcc fix_acc(const pxst_accum* acc) {
  return FixAcc{reinterpret_cast<long long*>(acc->num), reinterpret_cast<long long*>(acc->den),
                reinterpret_cast<long long*>(acc->num_fine),
                reinterpret_cast<long long*>(acc->den_fine), acc->touched, acc->quanta};
}

extern "C" int pxst_stack_absmax(const pxst_scan* sc, double* out, void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(out, "NULL pointer");
  return launch_abs_max(sc, out, as_stream(stream));
}

extern "C" int pxst_object_quanta(const pxst_scan* sc, const double* absmax, double* quanta,
                                  void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(absmax && quanta, "NULL pointer");
  return launch_quanta(sc, absmax, nullptr, nullptr, 0, quanta, as_stream(stream));
}

extern "C" int pxst_object_splat(const pxst_scan* sc, const double* u, const double* di,
                                 const double* dj, int64_t n0, int64_t m0, int64_t os,
                                 int64_t of, int64_t frame_lo, int64_t frame_hi,
                                 const pxst_accum* acc, unsigned long long* n_dropped,
                                 void* stream) {
  if (int e = check_scan(sc)) return e;
  if (int e = check_accum(acc)) return e;
  PXST_REQUIRE(u && di && dj, "NULL pointer");
  PXST_REQUIRE(os > 0 && of > 0 && os * of < (int64_t(1) << 40), "bad grid shape");
  PXST_REQUIRE(0 <= frame_lo && frame_lo <= frame_hi && frame_hi <= sc->n_good,
               "bad frame range");
  return launch_object_fix(sc, u, di, dj, n0, m0, os, of, frame_lo, frame_hi, fix_acc(acc),
                           n_dropped, as_stream(stream));
}

extern "C" int pxst_accum_zero(const pxst_accum* acc, int64_t cells, void* stream) {
  if (int e = check_accum(acc)) return e;
  PXST_REQUIRE(cells >= 0, "bad accumulator size");
  cudaStream_t s = as_stream(stream);
  const size_t b = sizeof(int64_t) * cells;
  PXST_CHECK_CUDA(cudaMemsetAsync(acc->num, 0, b, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(acc->den, 0, b, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(acc->num_fine, 0, b, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(acc->den_fine, 0, b, s));
  if (acc->touched) PXST_CHECK_CUDA(cudaMemsetAsync(acc->touched, 0, cells, s));
  return PXST_OK;
}

extern "C" int pxst_object_finish(const pxst_accum* acc, int64_t n, double* i_ref, double* wsum,
                                  float* fm, uint8_t* valid, void* stream) {
  if (int e = check_accum(acc)) return e;
  PXST_REQUIRE(n > 0, "bad accumulator size");
  return launch_fix_finish(fix_acc(acc), nullptr, n, i_ref, wsum, fm, valid, as_stream(stream));
}

extern "C" int pxst_object_finish_peers(const pxst_accum* accs, int n_peers, int64_t cell_lo,
                                        int64_t cell_hi, double* const* i_ref,
                                        double* const* wsum, float* const* fm,
                                        uint8_t* const* valid, void* stream) {
  PXST_REQUIRE(accs && n_peers >= 1 && n_peers <= kMaxPeers, "peer count out of range");
  PXST_REQUIRE(cell_lo >= 0 && cell_hi >= cell_lo, "bad cell range");
  FixAcc fa[kMaxPeers];
  for (int j = 0; j < n_peers; ++j) {
    if (int e = check_accum(accs + j)) return e;
    fa[j] = fix_acc(accs + j);
  }
  return launch_fix_finish_peers(fa, n_peers, cell_lo, cell_hi, i_ref, wsum, fm, valid,
                                 as_stream(stream));
}

extern "C" int pxst_object_map(const pxst_scan* sc, const double* u,
                               const double* di, const double* dj, int64_t n0, int64_t m0,
                               int64_t os, int64_t of, double* i_ref, double* wsum, float* fm,
                               uint8_t* valid, void* stream) {
  if (int e = check_scan(sc)) return e;
  PXST_REQUIRE(u && di && dj, "NULL pointer");
  PXST_REQUIRE(os > 0 && of > 0 && os * of < (int64_t(1) << 40), "bad grid shape");
  cudaStream_t s = as_stream(stream);
  const int64_t n = os * of;
  Scratch buf;
  if (int e = buf.alloc(sizeof(int64_t) * 4 * n + n + 4 * sizeof(double) + 16, s)) return e;
  int64_t* num = buf.as<int64_t>();
  double* q = reinterpret_cast<double*>(num + 4 * n);
  double* amax = q + 2;
  uint8_t* touched = reinterpret_cast<uint8_t*>(q + 4);
  PXST_CHECK_CUDA(cudaMemsetAsync(num, 0, sizeof(int64_t) * 4 * n, s));
  PXST_CHECK_CUDA(cudaMemsetAsync(touched, 0, n, s));
  if (int e = launch_abs_max(sc, amax, s)) return e;
  if (int e = launch_quanta(sc, amax, nullptr, nullptr, 0, q, s)) return e;
  const FixAcc acc{reinterpret_cast<long long*>(num), reinterpret_cast<long long*>(num + n),
                   reinterpret_cast<long long*>(num + 2 * n),
                   reinterpret_cast<long long*>(num + 3 * n), touched, q};
  if (int e = launch_object_fix(sc, u, di, dj, n0, m0, os, of, 0, sc->n_good, acc, nullptr, s))
    return e;
  return launch_fix_finish(acc, nullptr, n, i_ref, wsum, fm, valid, s);
}

extern "C" int pxst_gather(const pxst_ref* ref, const double* x, const double* y, int64_t n,
                           double* vals, uint8_t* ok, void* stream) {
  PXST_REQUIRE(ref && ref->fm && ref->valid && ref->os > 0 && ref->of > 0, "bad reference");
  PXST_REQUIRE(x && y && vals && ok, "NULL pointer");
  if (n <= 0) return PXST_OK;
  k_gather<<<grid_1d(n, 256), 256, 0, as_stream(stream)>>>(*ref, x, y, n, vals, ok);
  PXST_CHECK_LAUNCH();
  return PXST_OK;
}

extern "C" int pxst_splat(double* acc_v, double* acc_w, int64_t os, int64_t of, const double* x,
                          const double* y, const double* value, const double* weight, int64_t n,
                          int64_t* n_dropped, void* stream) {
  PXST_REQUIRE(acc_v && acc_w && os > 0 && of > 0, "bad accumulators");
  PXST_REQUIRE(x && y && value, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  Scratch cnt;
  if (int e = cnt.alloc(sizeof(unsigned long long), s)) return e;
  PXST_CHECK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), s));
  if (n > 0) {
    k_splat_f64<<<grid_1d(n, 256), 256, 0, s>>>(acc_v, acc_w, os, of, x, y, value, weight, n,
                                                 cnt.as<unsigned long long>());
    PXST_CHECK_LAUNCH();
  }
  unsigned long long h = 0;
  PXST_CHECK_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  PXST_CHECK_CUDA(cudaStreamSynchronize(s));
  if (n_dropped) *n_dropped = static_cast<int64_t>(h);
  return PXST_OK;
}
