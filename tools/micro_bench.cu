// Microbenchmarks that decide the transposed-store design:
//  (1) DSMEM read bandwidth inside a thread-block cluster (ld.shared::cluster),
//  (2) global store throughput when a warp writes S-byte segments scattered with a large
//      stride (the "transposed store" pattern) for S = 8..128,
//  (3) plain coalesced copy for reference.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_bench tools/micro_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

// (1) each CTA fills 64 KB of smem, then repeatedly reads the smem of peer (rank+d)%C
template <int C>
__global__ void __launch_bounds__(512) dsmem_read(float2* sink, int iters, int remote) {
  extern __shared__ float4 sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int n4 = 65536 / 16;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
  cl.sync();
  const unsigned rank = cl.block_rank();
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    const unsigned peer = remote ? (rank + 1 + (it % (C - 1))) % C : rank;
    const float4* p = cl.map_shared_rank(sm, peer);
#pragma unroll 4
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
      float4 v = p[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  cl.sync();
  if (acc.x == -1.f) sink[0] = make_float2(acc.y, acc.z);
}

// (2) scattered segment stores: warp writes 32*8 bytes as (32*8/S) segments of S bytes,
// consecutive segments `stride` bytes apart; total bytes written = total.
__global__ void scatter_store(float2* out, long long n_elems, int seg_elems, long long stride_elems) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  // element index k -> (segment s = k / seg, offset o = k % seg); segments laid out with stride
  const long long nseg_rows = stride_elems / seg_elems;  // segments per "row block"
  for (long long k = t; k < n_elems; k += nthreads) {
    const long long s = k / seg_elems, o = k % seg_elems;
    const long long row = s % (n_elems / stride_elems);      // which row (strided)
    const long long col = s / (n_elems / stride_elems);      // which segment within the row
    out[row * stride_elems + col * seg_elems + o] = make_float2((float)k, 1.f);
    (void)nseg_rows;
  }
}

// (2b) the exact transposed-store pattern of the line passes: CTA g owns G consecutive
// lines of an N x N image and writes out[e][g*G + ll] for all e (in-order CTAs).
template <int G>
__global__ void __launch_bounds__(512) transposed_store(float2* out, int n) {
  const long long g = blockIdx.x;
  const long long line0 = g * G;
  const long long img = line0 / n;
  const int l0 = (int)(line0 % n);
  float2* dst = out + img * (long long)n * n + l0;
  const int per = G * n / 512;
  for (int kk = 0; kk < per; ++kk) {
    const int f = threadIdx.x + kk * 512;
    const int ll = f % G, e = f / G;
    dst[(long long)e * n + ll] = make_float2((float)f, 1.f);
  }
}

__global__ void copy_kernel(const float4* in, float4* out, long long n4) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  for (long long k = t; k < n4; k += nthreads) out[k] = in[k];
}

template <int C>
int run_dsmem(float2* sink, int sms, int remote) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = 65536;
  CK(cudaFuncSetAttribute(dsmem_read<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  int ncl = 0;
  cfg.gridDim = dim3(C * 64);
  CK(cudaOccupancyMaxActiveClusters(&ncl, dsmem_read<C>, &cfg));
  cfg.gridDim = dim3(C * ncl);
  const int iters = 200;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  CK(cudaLaunchKernelEx(&cfg, dsmem_read<C>, sink, 4, remote));
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  CK(cudaLaunchKernelEx(&cfg, dsmem_read<C>, sink, iters, remote));
  cudaEventRecord(b);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double bytes = (double)C * ncl * iters * 65536.0;
  printf("dsmem C=%d remote=%d active_clusters=%d ctas=%d: %.1f GB/s total, %.2f GB/s per CTA\n", C, remote,
         ncl, C * ncl, bytes / ms / 1e6, bytes / ms / 1e6 / (C * ncl));
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  float2* sink;
  CK(cudaMalloc(&sink, 64));
  run_dsmem<2>(sink, sms, 0);
  run_dsmem<2>(sink, sms, 1);
  run_dsmem<4>(sink, sms, 1);
  run_dsmem<8>(sink, sms, 1);

  const long long n = 1ll << 29;  // 4 GiB of float2
  float2* buf;
  float4* buf2;
  CK(cudaMalloc(&buf, n * sizeof(float2)));
  CK(cudaMalloc(&buf2, n * sizeof(float2)));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    copy_kernel<<<sms * 8, 256>>>((const float4*)buf, buf2, n / 2);
    cudaEventRecord(b);
    CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("copy 4 GiB: %.3f ms, %.1f GB/s (read+write)\n", ms, 2.0 * n * 8 / ms / 1e6);
  const long long stride = 4096;  // elements between consecutive rows (32 KB)
  for (int seg : {1, 2, 4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      scatter_store<<<sms * 8, 256>>>(buf, n, seg, stride);
      cudaEventRecord(b);
      CK(cudaDeviceSynchronize());
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("scatter store seg=%3d B stride=%lld B: %.3f ms, %.1f GB/s (write only)\n", seg * 8, stride * 8, ms,
           (double)n * 8 / ms / 1e6);
  }
  {
    const int nn = 4096;
    const long long lines = n / nn;
    auto run = [&](auto kern, int G) {
      float ms2 = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        kern<<<(unsigned)(lines / G), 512>>>(buf, nn);
        cudaEventRecord(b);
        cudaDeviceSynchronize();
        cudaEventElapsedTime(&ms2, a, b);
      }
      printf("transposed store G=%2d (seg %3d B), N=%d: %.3f ms, %.1f GB/s\n", G, G * 8, nn, ms2,
             (double)n * 8 / ms2 / 1e6);
    };
    run(transposed_store<1>, 1);
    run(transposed_store<2>, 2);
    run(transposed_store<4>, 4);
    run(transposed_store<8>, 8);
    run(transposed_store<16>, 16);
  }
  return 0;
}
