// Exchange-primitive throughput on B200: shared-memory STS.64/LDS.64 vs warp SHFL.32.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_xchg tools/micro_xchg.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512) k_lds(float2* out, int iters) {
  __shared__ float2 sm[512 * 8 + 8];
  const int t = threadIdx.x;
  for (int i = t; i < 4096; i += 512) sm[i] = make_float2(i, 1);
  __syncthreads();
  float2 acc = make_float2(0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      float2 v = sm[(t + 512 * e + (it & 1)) & 4095];
      acc.x += v.x; acc.y += v.y;
    }
  }
  out[blockIdx.x * 512 + t] = acc;
}
__global__ void __launch_bounds__(512) k_sts(float2* out, int iters) {
  __shared__ float2 sm[512 * 8 + 8];
  const int t = threadIdx.x;
  float2 v = make_float2(t, 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      sm[(t + 512 * e) & 4095] = v;
      v.x += 1.f;
    }
  }
  __syncthreads();
  out[blockIdx.x * 512 + t] = sm[(t * 7) & 4095];
}
__global__ void __launch_bounds__(512) k_shfl(float2* out, int iters) {
  const int t = threadIdx.x;
  float a[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) a[e] = t + e;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 16; ++e) a[e] = __shfl_xor_sync(0xffffffffu, a[e], (e + 1) & 31) + 1.f;
  }
  float r = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) r += a[e];
  out[blockIdx.x * 512 + t] = make_float2(r, 0);
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float2* out;
  cudaMalloc(&out, (size_t)sms * 4 * 512 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000, blocks = sms * 2;
  auto run = [&](const char* name, void (*k)(float2*, int), double bytes_per_op) {
    float ms = 0;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      k<<<blocks, 512>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    double ops = (double)blocks * 512 / 32 * iters * 16;  // warp instructions
    printf("%-6s %.3f ms  %.2f warp-inst/clk/SM  %.1f B/clk/SM\n", name, ms, ops / (ms * 1e-3) / sms / 1.965e9,
           ops * 32 * bytes_per_op / (ms * 1e-3) / sms / 1.965e9);
  };
  run("LDS.64", k_lds, 8);
  run("STS.64", k_sts, 8);
  run("SHFL", k_shfl, 4);
  return 0;
}
