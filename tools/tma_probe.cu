// Bisect TMA/mbarrier issues: runs small kernels, reports which fail.
#include <cstdio>
#include "../paper_2003_12726_b200/csrc/tma.cuh"
using namespace pxst;


__global__ void k_mbar_only(int* out) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, blockDim.x); mbar_fence_init(); }
  __syncthreads();
  mbar_arrive(&bar);
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

template <bool PREF>
__global__ void k_tma(const __grid_constant__ CUtensorMap tmap, float* out, int r0, int c0, int n) {
  extern __shared__ __align__(128) unsigned char raw[];
  __shared__ __align__(8) uint64_t bar;
  float* buf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  if (threadIdx.x == 0) {
    if (PREF) tma_prefetch_desc(&tmap);
    mbar_init(&bar, 1); mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_arrive_expect_tx(&bar, n * 4); tma_load_2d(buf, &tmap, c0, r0, &bar); }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main() {
  int* d; cudaMalloc(&d, 1024);
  k_mbar_only<<<4, 128>>>(d);
  printf("mbar_only: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  const int R = 85, C = 136, BR = 13, BC = 56;
  float* img; cudaMalloc(&img, R * C * 4);
  float* h = new float[R * C]; for (int i = 0; i < R * C; ++i) h[i] = i;
  cudaMemcpy(img, h, R * C * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  int e = encode_tmap_2d_f32(&m, img, R, C, C, BR, BC);
  printf("encode: %d\n", e);
  float* out; cudaMalloc(&out, BR * BC * 4);
  size_t smem = BR * BC * 4 + 128;
  cudaFuncSetAttribute(k_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tma<false><<<1, 128, smem>>>(m, out, 3, 5, BR * BC);
  cudaError_t r = cudaDeviceSynchronize();
  printf("tma: %s\n", cudaGetErrorString(r));
  if (r == cudaSuccess) {
    float* ho = new float[BR * BC]; cudaMemcpy(ho, out, BR * BC * 4, cudaMemcpyDeviceToHost);
    printf("tma value check: %g (expect %g), %g (expect %g)\n", ho[0], h[3 * C + 5], ho[BC + 2], h[4 * C + 7]);
    k_tma<false><<<1, 128, smem>>>(m, out, -2, -3, BR * BC);
    printf("tma oob: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(ho, out, BR * BC * 4, cudaMemcpyDeviceToHost);
    printf("oob value check: %g (expect 0), %g (expect %g)\n", ho[0], ho[2 * BC + 3], h[0]);
    k_tma<true><<<1, 128, smem>>>(m, out, 3, 5, BR * BC);
    printf("tma+prefetch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
