// TMEM (tensor memory) load throughput on B200: tcgen05.ld 32x32b.xK per thread-lane.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_tmem tools/micro_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k_tmem(float* out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s;
  // warp w: lanes 32*(w%4).., columns (w/4)*cols_per
  constexpr int cols_per = 512 / ((WARPS + 3) / 4);
  const uint32_t ta = base + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)((warp / 4) * cols_per);
  // write something
  {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint((float)(threadIdx.x + i));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(ta + (uint32_t)((it & 1) * 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, (size_t)sms * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  auto run = [&](const char* name, void (*k)(float*, int), int warps) {
    float ms = 0;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      k<<<sms, warps * 32>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    }
    double bytes = (double)sms * warps * 32 * iters * 16 * 4;
    printf("%-10s %.3f ms  %.1f B/clk/SM  (%.2f us per 16-col load per warp)\n", name, ms,
           bytes / (ms * 1e-3) / sms / 1.965e9, ms * 1e3 / iters);
  };
  run("tmem 4w", k_tmem<4>, 4);
  run("tmem 8w", k_tmem<8>, 8);
  run("tmem 16w", k_tmem<16>, 16);
  return 0;
}
