// Pipe-rate microbenchmarks for the PXST kernel design on B200 (sm_100a).
// Measures: FFMA (3-register form), FFMA2 (packed f32x2), LDS.32 and LDS.128
// shared-memory bandwidth, REDG.ADD (u64 and f64) spread-address throughput,
// and DFMA. Prints one JSON object. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CH = 16;

__global__ void k_ffma(float* out, float b, float c, int iters) {
  float a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = fmaf(a[i], b, c + 0.0f * a[(i + 1) % CH]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// acc_i = fma(r_i, r_i, acc_i) with r_i = fma(-A, h_i, I): the trial kernel's mix.
__global__ void k_ffma_mix(float* out, float A, float I, int iters) {
  float acc[CH], h[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) { acc[i] = 0.f; h[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      float r = fmaf(-A, h[i], I);
      acc[i] = fmaf(r, r, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) h[i] = h[i] * 0.999f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }

__global__ void k_ffma2(float* out, float b, float c, int iters) {
  unsigned long long a[CH / 2];
  float2 bb = make_float2(b, b), cc = make_float2(c, c);
  unsigned long long br = f2u(bb), cr = f2u(cc);
#pragma unroll
  for (int i = 0; i < CH / 2; ++i) a[i] = f2u(make_float2(threadIdx.x * 1e-3f + i, i + 0.5f));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH / 2; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(br), "l"(cr));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH / 2; ++i) { float2 v = u2f(a[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double b, double c, int iters) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Each lane reads its own conflict-free word: bank = lane.
__global__ void k_lds32(float* out, int iters, int stride) {
  __shared__ float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 0.5f;
  __syncthreads();
  float s = 0;
  int base = (threadIdx.x & 31) + (threadIdx.x >> 5) * 32;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) s += sm[(base + (it * 16 + k) * stride) & 8191];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lds128(float* out, int iters) {
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float s = 0;
  int base = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) { float4 v = sm[(base + (it * 16 + k) * 64) & 2047]; s += v.x + v.w; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_red64(unsigned long long* acc, int n_cells, int iters) {
  unsigned int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    unsigned int h = (tid * 2654435761u + it * 40503u) % n_cells;
    atomicAdd(&acc[h], 1ull);
  }
}

__global__ void k_redf64(double* acc, int n_cells, int iters) {
  unsigned int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    unsigned int h = (tid * 2654435761u + it * 40503u) % n_cells;
    atomicAdd(&acc[h], 1.0);
  }
}

// Coalesced row-contiguous atomics (neighbouring lanes hit neighbouring cells),
// the pattern of a bilinear splat along a detector row.
__global__ void k_redf64_rows(double* acc, int n_cells, int iters) {
  unsigned int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    unsigned int h = ((tid >> 5) * 977u + it * 131u) * 32u % (n_cells - 64) + (threadIdx.x & 31);
    atomicAdd(&acc[h], 1.0);
  }
}


__global__ void k_lds_cyc(float* out, long long* cyc, int iters, int mode) {
  __shared__ float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 0.5f;
  __syncthreads();
  long long t0 = clock64();
  float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* p = sm + w * 64 + lane;
  if (mode == 0) {
    for (int it = 0; it < iters; ++it) {
      const float* q = p + ((it * 256) & 4095);
#pragma unroll
      for (int k = 0; k < 16; k += 4) { s0 += q[k * 64]; s1 += q[k * 64 + 64]; s2 += q[k * 64 + 128]; s3 += q[k * 64 + 192]; }
    }
  } else if (mode == 1) {
    const float2* p2 = reinterpret_cast<const float2*>(sm) + w * 32 + lane;
    for (int it = 0; it < iters; ++it) {
      const float2* q = p2 + ((it * 128) & 2047);
#pragma unroll
      for (int k = 0; k < 8; k += 2) { float2 a = q[k * 64]; float2 b = q[k * 64 + 64]; s0 += a.x; s1 += a.y; s2 += b.x; s3 += b.y; }
    }
  } else {
    const float4* p4 = reinterpret_cast<const float4*>(sm) + w * 32 + lane;
    for (int it = 0; it < iters; ++it) {
      const float4* q = p4 + ((it * 64) & 1023);
#pragma unroll
      for (int k = 0; k < 4; k += 1) { float4 a = reinterpret_cast<const float4*>(sm)[((q - p4) + k * 128 + w * 32 + lane) & 2047]; s0 += a.x; s1 += a.y; s2 += a.z; s3 += a.w; }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Shared-memory u32 atomics: each lane adds into its own word (spread = a
// lane-dependent hash inside a 4096-word window, row = consecutive words).
__global__ void k_atoms(float* out, int iters, int row) {
  __shared__ unsigned sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const unsigned h = row ? ((w * 32 + lane + (it * 8 + k) * 256) & 4095)
                             : (((w * 32 + lane) * 2654435761u + (it * 8 + k) * 40503u) >> 20) & 4095;
      atomicAdd(&sm[h], lane + (unsigned)k + 3u);
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[threadIdx.x & 4095];
}

// Shared-memory f32 atomics (compiled as ATOMS.CAS loops or native adds).
__global__ void k_atoms_f32(float* out, int iters) {
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) atomicAdd(&sm[(w * 32 + lane + (it * 8 + k) * 256) & 4095], 1.f);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[threadIdx.x & 4095];
}

// Shared-memory read-modify-write of float4 cells (LDS.128 + 4 FADD + STS.128).
__global__ void k_rmw128(float* out, int iters) {
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(0, 0, 0, 0);
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* mine = sm + (w * 32 & 2047);   // warps own disjoint 32-cell rows
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float4* c = mine + ((lane + it * 8 + k) & 31);
      float4 v = *c;
      v.x += 1.f; v.y += 2.f; v.z += 3.f; v.w += 4.f;
      *c = v;
      __syncwarp();
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[threadIdx.x & 2047].x;
}

// Shared-memory u64 atomics (ATOMS.CAST.SPIN.64 loops): lanes on consecutive
// words (dup = 1) or pairs of lanes on the same word (dup = 2).
__global__ void k_atoms_u64(float* out, int iters, int dup) {
  __shared__ unsigned long long sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      atomicAdd(&sm[(w * 32 + lane / dup + (it * 8 + k) * 256) & 2047],
                (unsigned long long)(lane + k + 3));
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)sm[threadIdx.x & 2047];
}

// Fixed-point term: DFMA against a magic constant, 64-bit subtract (the
// conversion cost of one accumulation term).
__global__ void k_fix_terms(float* out, int iters, double s) {
  const double magic = 6755399441055744.0;
  long long acc = 0;
  double x = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double y = fma(x + k, s, magic);
      acc += __double_as_longlong(y) - 0x4338000000000000ll;
    }
    x += 1e-7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

__global__ void k_match(float* out, int iters) {
  unsigned acc = 0;
  const unsigned lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += __match_any_sync(0xffffffffu, (lane + it + k) >> 1);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Global REDs into an L2-resident 4 MB image, lanes on consecutive cells of a
// row (the splat pattern): v4.f32 (16 B per lane) vs u64 (8 B per lane).
__global__ void k_red_v4_rows(float4* acc, int n_cells, int iters) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const unsigned h = ((tid >> 5) * 977u + it * 131u) * 32u % (n_cells - 64) + (threadIdx.x & 31);
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(acc + h), "f"(1.f),
                 "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
  }
}
__global__ void k_red_u64_rows(unsigned long long* acc, int n_cells, int iters) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const unsigned h = ((tid >> 5) * 977u + it * 131u) * 32u % (n_cells - 64) + (threadIdx.x & 31);
    atomicAdd(acc + h, 1ull);
  }
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float* fout; double* dout;
  CK(cudaMalloc(&fout, sizeof(float) * sms * 64 * 1024));
  CK(cudaMalloc(&dout, sizeof(double) * sms * 64 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", prop.name, sms, clk_khz);

  auto timeit = [&](auto launch) -> float {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float t; cudaEventElapsedTime(&t, e0, e1); return t / 3;
  };
  const int threads = 256, blocks = sms * 8, iters = 4096;
  double lanes = double(blocks) * threads;
  ms = timeit([&] { k_ffma<<<blocks, threads>>>(fout, 0.999f, 1e-4f, iters); });
  printf(", \"ffma_tflops\": %.2f", lanes * iters * CH * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_ffma_mix<<<blocks, threads>>>(fout, 0.5f, 3.0f, iters / 2); });
  printf(", \"ffma_mix_tflops\": %.2f", lanes * (iters / 2) * (CH * 2 + CH) * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_ffma2<<<blocks, threads>>>(fout, 0.999f, 1e-4f, iters); });
  printf(", \"ffma2_tflops\": %.2f", lanes * iters * CH * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_dfma<<<blocks, threads>>>(dout, 0.999, 1e-4, iters / 8); });
  printf(", \"dfma_tflops\": %.2f", lanes * (iters / 8) * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_lds32<<<blocks, threads>>>(fout, iters / 4, 32); });
  double lds_bytes = lanes * (iters / 4) * 16 * 4;
  printf(", \"lds32_TBps\": %.2f, \"lds32_B_per_clk_sm\": %.1f", lds_bytes / (ms * 1e-3) / 1e12,
         lds_bytes / (ms * 1e-3) / (clk_khz * 1e3) / sms);
  ms = timeit([&] { k_lds32<<<blocks, threads>>>(fout, iters / 4, 33); });
  printf(", \"lds32_stride33_TBps\": %.2f", lds_bytes / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_lds128<<<blocks, threads>>>(fout, iters / 4); });
  printf(", \"lds128_TBps\": %.2f", lanes * (iters / 4) * 16 * 16 / (ms * 1e-3) / 1e12);
  int n_cells = 1 << 22;
  unsigned long long* acc;
  CK(cudaMalloc(&acc, sizeof(double) * n_cells));
  CK(cudaMemset(acc, 0, sizeof(double) * n_cells));
  int aiters = 64;
  ms = timeit([&] { k_red64<<<blocks, threads>>>(acc, n_cells, aiters); });
  printf(", \"redg_u64_Gops\": %.1f", lanes * aiters / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_redf64<<<blocks, threads>>>((double*)acc, n_cells, aiters); });
  printf(", \"redg_f64_Gops\": %.1f", lanes * aiters / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_redf64_rows<<<blocks, threads>>>((double*)acc, n_cells, aiters); });
  printf(", \"redg_f64_rows_Gops\": %.1f", lanes * aiters / (ms * 1e-3) / 1e9);

  {
    long long* cyc; CK(cudaMalloc(&cyc, sizeof(long long) * sms));
    long long hc[1024];
    for (int mode = 0; mode < 3; ++mode) {
      int it = 2048;
      k_lds_cyc<<<sms, 1024>>>(fout, cyc, it, mode);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hc, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
      double mean = 0; for (int i = 0; i < sms; ++i) mean += hc[i]; mean /= sms;
      double bytes = 1024.0 * it * 64;  // 16 floats per iter per thread
      printf(", \"lds_mode%d_B_per_clk_sm\": %.1f", mode, bytes / mean);
    }
  }
  {
    const int ai = 256;
    const double ops = lanes * ai * 8;
    ms = timeit([&] { k_atoms<<<blocks, threads>>>(fout, ai, 0); });
    printf(", \"atoms_u32_spread_lane_ops_per_clk_sm\": %.2f", ops / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    ms = timeit([&] { k_atoms<<<blocks, threads>>>(fout, ai, 1); });
    printf(", \"atoms_u32_row_lane_ops_per_clk_sm\": %.2f", ops / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    ms = timeit([&] { k_atoms_f32<<<blocks, threads>>>(fout, ai); });
    printf(", \"atoms_f32_row_lane_ops_per_clk_sm\": %.2f", ops / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    ms = timeit([&] { k_atoms_u64<<<blocks, threads>>>(fout, ai, 1); });
    printf(", \"atoms_u64_cas_row_lane_ops_per_clk_sm\": %.2f", ops / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    ms = timeit([&] { k_atoms_u64<<<blocks, threads>>>(fout, ai, 2); });
    printf(", \"atoms_u64_cas_dup2_lane_ops_per_clk_sm\": %.2f", ops / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    ms = timeit([&] { k_fix_terms<<<blocks, threads>>>(fout, ai, 1.2345e3); });
    printf(", \"fix_terms_per_clk_sm\": %.2f", ops / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    ms = timeit([&] { k_rmw128<<<blocks, threads>>>(fout, ai); });
    printf(", \"smem_rmw128_lane_ops_per_clk_sm\": %.2f", ops / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    ms = timeit([&] { k_match<<<blocks, threads>>>(fout, ai); });
    printf(", \"match_any_warp_ops_per_clk_sm\": %.3f", ops / 32 / (ms * 1e-3) / (clk_khz * 1e3) / sms);
    const int cells = 1 << 18;   // 4 MB of float4: L2 resident
    ms = timeit([&] { k_red_v4_rows<<<blocks, threads>>>((float4*)acc, cells, aiters); });
    printf(", \"redg_v4f32_rows_Gops\": %.1f", lanes * aiters / (ms * 1e-3) / 1e9);
    ms = timeit([&] { k_red_u64_rows<<<blocks, threads>>>(acc, cells, aiters); });
    printf(", \"redg_u64_rows_Gops\": %.1f", lanes * aiters / (ms * 1e-3) / 1e9);
  }
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
