// FP32 issue/throughput microbenchmark: scalar FFMA/FADD vs packed FFMA2/FADD2 (sm_100a).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_fp tools/micro_fp.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
template <int K>
__global__ void k_ffma(float* out, int iters, float s) {
  float a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = fmaf(a[k], s, 0.5f);
  }
  float r = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) r += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int K>
__global__ void k_fadd(float* out, int iters, float s) {
  float a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = a[k] + s;
  }
  float r = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) r += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int K>
__global__ void k_ffma2(float* out, int iters, float s) {
  u64 a[K];
  u64 sv, h;
  asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
  asm("mov.b64 %0, {%1, %1};" : "=l"(h) : "f"(0.5f));
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float x = threadIdx.x + k;
    asm("mov.b64 %0, {%1, %1};" : "=l"(a[k]) : "f"(x));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = fma2(a[k], sv, h);
  }
  float r = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[k]));
    r += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int K>
__global__ void k_fadd2(float* out, int iters, float s) {
  u64 a[K];
  u64 sv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float x = threadIdx.x + k;
    asm("mov.b64 %0, {%1, %1};" : "=l"(a[k]) : "f"(x));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = add2(a[k], sv);
  }
  float r = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[k]));
    r += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 1 << 26);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  auto run = [&](const char* name, void (*kern)(float*, int, float), double flops_per_op, int ops_per_iter) {
    float ms = 0;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      kern<<<blocks, threads>>>(out, iters, 1.0001f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    double inst = (double)blocks * threads / 32 * iters * ops_per_iter;  // warp instructions
    double fl = (double)blocks * threads * iters * ops_per_iter * flops_per_op;
    printf("%-8s %.3f ms  %.1f Gwarp-inst/s  %.2f TFLOP/s  (%.2f warp-inst/clk/SM @1.965GHz)\n", name, ms,
           inst / ms / 1e6, fl / ms / 1e9, inst / (ms * 1e-3) / sms / 1.965e9);
  };
  run("FFMA", k_ffma<16>, 2, 16);
  run("FFMA2", k_ffma2<16>, 4, 16);
  run("FADD", k_fadd<16>, 1, 16);
  run("FADD2", k_fadd2<16>, 2, 16);
  return 0;
}
