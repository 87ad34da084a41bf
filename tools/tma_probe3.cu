// Which async bulk-copy mechanisms work on this B200 pool?
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra.uni W_%=;\n}\n" :: "r"(sa(b)), "r"(ph) : "memory");
}
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tmap, const CUtensorMap* gmap, const float* src, float* out, int n, int cx, int cy) {
  __shared__ alignas(128) float buf[2048];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(n * 4) : "memory");
    if (MODE == 0) {  // 1-D bulk copy
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(sa(buf)), "l"(src), "r"(n * 4), "r"(sa(&bar)) : "memory");
    } else if (MODE == 1) {  // tensor, param-space map
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(sa(buf)), "l"((uint64_t)&tmap), "r"(0), "r"(0), "r"(sa(&bar)) : "memory");
    } else if (MODE == 2) {  // tensor, global-memory map
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" :: "l"(gmap) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(sa(buf)), "l"(gmap), "r"(0), "r"(0), "r"(sa(&bar)) : "memory");
    } else {  // shared::cta destination form (PTX 8.6+)
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(sa(buf)), "l"((uint64_t)&tmap), "r"(0), "r"(0), "r"(sa(&bar)) : "memory");
    }
  }
  wait(&bar, 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}
int g_cx = 0, g_cy = 0;
template <int M> void run(const char* name, CUtensorMap& m, CUtensorMap* gm, float* src, float* out, int n) {
  k<M><<<1, 128>>>(m, gm, src, out, n, g_cx, g_cy);
  cudaError_t e = cudaDeviceSynchronize();
  float h[4] = {0};
  if (e == cudaSuccess) cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("%-28s %s  out[1]=%g\n", name, cudaGetErrorString(e), h[1]);
}
int main(int argc, char** argv) {
  const int R = argc > 7 ? atoi(argv[7]) : 64, C = argc > 8 ? atoi(argv[8]) : 128;
  float* img; cudaMalloc(&img, R * C * 4);
  float* h = new float[R * C]; for (int i = 0; i < R * C; ++i) h[i] = i;
  cudaMemcpy(img, h, R * C * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 2048 * 4);
  CUtensorMap m;
  cuuint64_t dims[2] = {C, R}; cuuint64_t strides[1] = {C * 4};
  cuuint32_t box[2] = {(cuuint32_t)(argc > 2 ? atoi(argv[2]) : 32), (cuuint32_t)(argc > 3 ? atoi(argv[3]) : 8)}; cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, img, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (argc > 4 && atoi(argv[4])) ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  g_cx = argc > 5 ? atoi(argv[5]) : 0; g_cy = argc > 6 ? atoi(argv[6]) : 0;
  if (mode == 0) run<0>("bulk 1-D", m, gm, img, out, 256);
  if (mode == 1) run<1>("tensor param map", m, gm, img, out, (int)(box[0] * box[1]));
  if (mode == 2) run<2>("tensor global map", m, gm, img, out, 256);
  if (mode == 3) run<3>("tensor shared::cta dst", m, gm, img, out, 256);
  return 0;
}
