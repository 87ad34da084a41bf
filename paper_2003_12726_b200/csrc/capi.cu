// C ABI glue: thread-local error string, status codes, launch counter.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace pxst {
namespace {
thread_local char g_err[1024] = "";
thread_local int64_t g_launches = 0;
}  // namespace

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

void count_launch(int n) { g_launches += n; }

void retain_pool_memory() {
  static thread_local int done_mask = 0;   // devices 0..31 configured by this thread
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) return;
  if (done_mask & (1 << dev)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done_mask |= 1 << dev;
}

}  // namespace pxst

extern "C" int pxst_abi_version(void) { return PXST_ABI_VERSION; }
extern "C" const char* pxst_last_error(void) { return pxst::g_err; }
extern "C" int64_t pxst_launch_count(void) { return pxst::g_launches; }

// Hand the scratch memory the library kept in the current device's default
// pool back to the driver (the pool otherwise retains it for the process,
// see retain_pool_memory): waits for the device, then trims to zero bytes.
extern "C" int pxst_release_pool(void) {
  int dev = 0;
  PXST_CHECK_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  PXST_CHECK_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  PXST_CHECK_CUDA(cudaDeviceSynchronize());
  PXST_CHECK_CUDA(cudaMemPoolTrimTo(pool, 0));
  return PXST_OK;
}
