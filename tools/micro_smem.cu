// Shared-memory throughput on B200 for 64-bit vs 128-bit LDS/STS (volatile asm, no DCE).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_smem tools/micro_smem.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int W>  // W = 8 or 16 bytes per lane
__global__ void __launch_bounds__(512) k_ld(float* out, int iters) {
  __shared__ __align__(16) float sm[8192];
  const int t = threadIdx.x;
  for (int i = t; i < 8192; i += 512) sm[i] = i;
  __syncthreads();
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const unsigned a = base + ((t * W + e * 512 * W + it * 16) & (32768 - 1));
      if (W == 8) {
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
        acc += x + y;
      } else {
        float x, y, z, w;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
        acc += x + y + z + w;
      }
    }
  }
  out[blockIdx.x * 512 + t] = acc;
}
template <int W>
__global__ void __launch_bounds__(512) k_st(float* out, int iters) {
  __shared__ __align__(16) float sm[8192];
  const int t = threadIdx.x;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  float v = t;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const unsigned a = base + ((t * W + e * 512 * W + it * 16) & (32768 - 1));
      if (W == 8)
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v), "f"(v + 1.f));
      else
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v), "f"(v + 1.f), "f"(v + 2.f), "f"(v + 3.f));
      v += 1.f;
    }
  }
  __syncthreads();
  out[blockIdx.x * 512 + t] = sm[(t * 7) & 8191];
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, (size_t)sms * 4 * 512 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4000, blocks = sms * 2;
  auto run = [&](const char* name, void (*k)(float*, int), int w) {
    float ms = 0;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      k<<<blocks, 512>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) printf("%s: %s\n", name, cudaGetErrorString(e));
    }
    double ins = (double)blocks * 512 / 32 * iters * 8;
    printf("%-8s %.3f ms  %.2f warp-inst/clk/SM  %.1f B/clk/SM\n", name, ms, ins / (ms * 1e-3) / sms / 1.965e9,
           ins * 32 * w / (ms * 1e-3) / sms / 1.965e9);
  };
  run("LDS.64", k_ld<8>, 8);
  run("LDS.128", k_ld<16>, 16);
  run("STS.64", k_st<8>, 8);
  run("STS.128", k_st<16>, 16);
  return 0;
}
