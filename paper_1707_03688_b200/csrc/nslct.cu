// C ABI of the B200 NsDLCT: plan / exec / exec_host / plan_info / pass_ms / destroy.
// See include/nslct.h for the contract and kernels.cuh for the pass schedule.
#include <cuda.h>
#include <cudaTypedefs.h>   // PFN_cuTensorMapEncodeTiled (driver entry point, no -lcuda)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>           // types only: NCCL is dlopen'ed at run time (nccl_api below)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/nslct.h"
#include "bluestein.h"
#include "kernels.cuh"
#include "planner.h"

namespace {

thread_local std::string g_err;

nslct_status fail(nslct_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(e_ == cudaErrorMemoryAllocation ? NSLCT_E_OOM : NSLCT_E_CUDA,             \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                      \
  } while (0)

using nslct::PassArgs;
using nslct::Phase;

typedef cudaError_t (*launch_fn)(const PassArgs&, cudaStream_t);
typedef cudaError_t (*attr_fn)();

template <typename T, int LOG2N, int MODE>
cudaError_t launch_pass(const PassArgs& a, cudaStream_t s) {
  using Cfg = nslct::LineCfg<LOG2N>;
  const size_t smem = (size_t)Cfg::G * Cfg::LS * sizeof(nslct::cpx<T>);
  const long long grid = a.n_lines / Cfg::G;
  nslct::line_pass_kernel<T, LOG2N, MODE><<<(unsigned)grid, Cfg::THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int LOG2N, int MODE>
cudaError_t set_attr() {
  using Cfg = nslct::LineCfg<LOG2N>;
  const size_t smem = (size_t)Cfg::G * Cfg::LS * sizeof(nslct::cpx<T>);
  return cudaFuncSetAttribute(nslct::line_pass_kernel<T, LOG2N, MODE>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

nslct_status make_store_map(CUtensorMap* m, void* out, int log2n, long long images);
nslct_status make_slab_store_map(CUtensorMap* m, void* out, int log2n, long long L, long long Lc);
// N = 16384: 512 threads x 2 virtual threads (kernels.cuh line_pass_pair2_kernel); the
// batched transposing passes write through TMA tensor stores (map of the pair-interleaved
// output, G = 2)
template <int MODE, bool SLAB>
cudaError_t launch_pair2(const PassArgs& a, cudaStream_t s) {
  using Cfg = nslct::LineCfg<14>;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (!nslct::ModeIO<MODE>::kStraightOut) {
    if (!SLAB && make_store_map(&map, a.out, 14, a.n_lines >> 14) != NSLCT_OK) return cudaErrorInvalidValue;
    if (SLAB && !a.peer_on && make_slab_store_map(&map, a.out, 14, a.lines_per_img, a.out_chunk) != NSLCT_OK)
      return cudaErrorInvalidValue;
  }
  cudaLaunchConfig_t cfg = {};
  long long grid = a.persist_ctas > 0 ? a.persist_ctas : a.n_lines;
  if (grid > a.n_lines) grid = a.n_lines;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(nslct::kPair2Threads);
  // exchange buffer, TMEM address slot (+ output staging for the transposing passes)
  cfg.dynamicSmemBytes = nslct::ModeIO<MODE>::kStraightOut ? nslct::kPair2SmemSmall : nslct::kPair2Smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if constexpr (SLAB && !nslct::ModeIO<MODE>::kStraightOut) {
    if (a.peer_on) return cudaLaunchKernelEx(&cfg, nslct::line_pass_pair2_kernel<MODE, true, true>, a, map);
  }
  return cudaLaunchKernelEx(&cfg, nslct::line_pass_pair2_kernel<MODE, SLAB, false>, a, map);
}
template <int MODE, bool SLAB>
cudaError_t set_attr_pair2() {
  using Cfg = nslct::LineCfg<14>;
  const int smem = (int)(nslct::ModeIO<MODE>::kStraightOut ? nslct::kPair2SmemSmall : nslct::kPair2Smem);
  if constexpr (SLAB && !nslct::ModeIO<MODE>::kStraightOut) {
    cudaError_t e = cudaFuncSetAttribute(nslct::line_pass_pair2_kernel<MODE, true, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  return cudaFuncSetAttribute(nslct::line_pass_pair2_kernel<MODE, SLAB, false>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}
template <bool SLAB>
struct Pair2Row {
  static void fill(launch_fn* l, attr_fn* at) {
    l[0] = launch_pair2<0, SLAB>; l[1] = launch_pair2<1, SLAB>; l[2] = launch_pair2<2, SLAB>;
    l[3] = launch_pair2<3, SLAB>; l[4] = launch_pair2<4, SLAB>; l[5] = launch_pair2<5, SLAB>;
    at[0] = set_attr_pair2<0, SLAB>; at[1] = set_attr_pair2<1, SLAB>; at[2] = set_attr_pair2<2, SLAB>;
    at[3] = set_attr_pair2<3, SLAB>; at[4] = set_attr_pair2<4, SLAB>; at[5] = set_attr_pair2<5, SLAB>;
  }
};

// large-N TMA-pipelined kernels (N = 8192, complex64): 2-CTA clusters, persistent
template <int LOG2N, int MODE, bool SLAB>
cudaError_t launch_big(const PassArgs& a, cudaStream_t s, const CUtensorMap& map) {
  using Cfg = nslct::BigCfg<LOG2N>;
  cudaLaunchConfig_t cfg = {};
  long long grid = a.persist_ctas > 0 ? a.persist_ctas : a.n_lines;
  if (grid > a.n_lines) grid = a.n_lines;
  grid &= ~1ll;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, nslct::line_pass_big_kernel<LOG2N, MODE, SLAB>, a, map);
}
template <int LOG2N, int MODE, bool SLAB>
cudaError_t set_attr_big() {
  return cudaFuncSetAttribute(nslct::line_pass_big_kernel<LOG2N, MODE, SLAB>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nslct::BigCfg<LOG2N>::SMEM);
}
typedef cudaError_t (*big_fn)(const PassArgs&, cudaStream_t, const CUtensorMap&);
template <int LOG2N, bool SLAB>
struct BigRow {
  static void fill(big_fn* l, attr_fn* at) {
    l[0] = launch_big<LOG2N, 0, SLAB>; l[1] = launch_big<LOG2N, 1, SLAB>; l[2] = launch_big<LOG2N, 2, SLAB>;
    l[3] = launch_big<LOG2N, 3, SLAB>; l[4] = launch_big<LOG2N, 4, SLAB>; l[5] = launch_big<LOG2N, 5, SLAB>;
    at[0] = set_attr_big<LOG2N, 0, SLAB>; at[1] = set_attr_big<LOG2N, 1, SLAB>;
    at[2] = set_attr_big<LOG2N, 2, SLAB>; at[3] = set_attr_big<LOG2N, 3, SLAB>;
    at[4] = set_attr_big<LOG2N, 4, SLAB>; at[5] = set_attr_big<LOG2N, 5, SLAB>;
  }
};

// persistent TMA-pipelined variant: grid = #SMs (one CTA per SM)
constexpr size_t kPipeExtra = 64;   // 3 mbarriers + 3 claimed-group slots + TMEM base
template <typename T, int LOG2N, int MODE>
cudaError_t launch_pipe(const PassArgs& a, cudaStream_t s, int grid, unsigned long long* counter,
                        const CUtensorMap& omap) {
  using Cfg = nslct::PipeCfg<LOG2N>;
  const size_t smem = (size_t)Cfg::NBUF * Cfg::BUF_ELEMS * sizeof(nslct::cpx<T>) + kPipeExtra;
  const long long n_groups = a.n_lines / Cfg::G;
  const long long g = n_groups < grid ? n_groups : grid;
  nslct::line_pass_pipe_kernel<T, LOG2N, MODE><<<(unsigned)g, Cfg::THREADS, smem, s>>>(a, n_groups, counter, omap);
  return cudaGetLastError();
}
template <typename T, int LOG2N, int MODE>
cudaError_t set_attr_pipe() {
  using Cfg = nslct::PipeCfg<LOG2N>;
  const size_t smem = (size_t)Cfg::NBUF * Cfg::BUF_ELEMS * sizeof(nslct::cpx<T>) + kPipeExtra;
  return cudaFuncSetAttribute(nslct::line_pass_pipe_kernel<T, LOG2N, MODE>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}
typedef cudaError_t (*pipe_fn)(const PassArgs&, cudaStream_t, int, unsigned long long*, const CUtensorMap&);

// warp-specialised variant (kernels.cuh line_pass_ws_kernel): passes of modes 1-3
template <int LOG2N, int MODE>
cudaError_t launch_ws(const PassArgs& a, cudaStream_t s, int grid, unsigned long long* counter,
                      const CUtensorMap& omap) {
  using Cfg = nslct::PipeCfg<LOG2N>;
  const size_t smem = (size_t)Cfg::NBUF * Cfg::BUF_ELEMS * sizeof(nslct::cpx<float>) + nslct::kWsExtra;
  const long long n_groups = a.n_lines / Cfg::G;
  const long long g = n_groups < grid ? n_groups : grid;
  nslct::line_pass_ws_kernel<LOG2N, MODE><<<(unsigned)g, 544, smem, s>>>(a, n_groups, counter, omap);
  return cudaGetLastError();
}
template <int LOG2N, int MODE>
cudaError_t set_attr_ws() {
  using Cfg = nslct::PipeCfg<LOG2N>;
  const size_t smem = (size_t)Cfg::NBUF * Cfg::BUF_ELEMS * sizeof(nslct::cpx<float>) + nslct::kWsExtra;
  return cudaFuncSetAttribute(nslct::line_pass_ws_kernel<LOG2N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem);
}
// the warp-specialised kernels for N = 2^lg (1024 ... 4096), pass modes 1 ... 3
struct WsRow {
  pipe_fn launch[3];
  attr_fn attr[3];
};
template <int L>
constexpr WsRow ws_row() {
  return WsRow{{launch_ws<L, 1>, launch_ws<L, 2>, launch_ws<L, 3>},
               {set_attr_ws<L, 1>, set_attr_ws<L, 2>, set_attr_ws<L, 3>}};
}
const WsRow* ws_row_of(int lg) {
  static const WsRow rows[3] = {ws_row<10>(), ws_row<11>(), ws_row<12>()};
  return (lg >= 10 && lg <= 12) ? &rows[lg - 10] : nullptr;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (resolved once)
PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// Tensor map of a pipe pass's transposed (pair-interleaved) output `out` of `images`
// N x N complex64 images, as the kernel's TMA store sees it (kernels.cuh, PipeCfg):
// dim0 = the G*IL-element segment (as 4G floats), dim1 = N/IL rows, dim2 = N/G groups,
// dim3 = images.
nslct_status make_store_map(CUtensorMap* m, void* out, int log2n, long long images) {
  auto fn = encode_tiled();
  if (!fn) return fail(NSLCT_E_CUDA, "cuTensorMapEncodeTiled entry point not available");
  const cuuint64_t n = 1ull << log2n;
  const cuuint64_t G = n <= 4096 ? 8192 / n : 2, IL = 2;   // pipe groups; the pair kernels' 2 lines
  const cuuint64_t dims[4] = {2 * IL * G, n / IL, n / G, (cuuint64_t)images};
  const cuuint64_t strides[3] = {IL * n * 8, IL * G * 8, n * n * 8};
  const cuuint32_t box[4] = {(cuuint32_t)(2 * IL * G), (cuuint32_t)(n / IL < 256 ? n / IL : 256), 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NSLCT_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return NSLCT_OK;
}

// Tensor map of a row-slab transposing pass's output as the N = 16384 pair kernel's TMA
// stores see it (kernels.cuh line_pass_pair2_kernel; layout in PassArgs): 5D view
// {32-byte segment (8 floats), consumer line pair lam/2 (row, 2 Lc elements), producer
// line pair within the sub-block (32 B), sub-block (L Lc elements), block s (L^2)};
// box = one segment x min(L/2, 256) rows.
nslct_status make_slab_store_map(CUtensorMap* m, void* out, int log2n, long long L, long long Lc) {
  auto fn = encode_tiled();
  if (!fn) return fail(NSLCT_E_CUDA, "cuTensorMapEncodeTiled entry point not available");
  const cuuint64_t n = 1ull << log2n;
  const cuuint64_t dims[5] = {8, (cuuint64_t)L / 2, (cuuint64_t)Lc / 2, (cuuint64_t)(L / Lc), n / (cuuint64_t)L};
  const cuuint64_t strides[4] = {(cuuint64_t)Lc * 16, 32, (cuuint64_t)(L * Lc) * 8, (cuuint64_t)(L * L) * 8};
  const cuuint32_t box[5] = {8, (cuuint32_t)(L / 2 < 256 ? L / 2 : 256), 1, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NSLCT_E_CUDA, "cuTensorMapEncodeTiled (slab store) failed (" + std::to_string((int)r) + ")");
  return NSLCT_OK;
}

// Tensor map of a large-N pass's Q16 input (kernels.cuh line_pass_big_kernel): 5D view
// {16 B piece (4 floats), line parity (16 B), mu pair (32 B), line pair (2C elements),
// chunk / image (L C elements)} of `images` blocks of L lines x N elements in chunks of C;
// box = one 16-byte piece x up to 256 mu pairs.
nslct_status make_q16_map(CUtensorMap* m, const void* in, int log2n, long long L, long long C, long long images) {
  auto fn = encode_tiled();
  if (!fn) return fail(NSLCT_E_CUDA, "cuTensorMapEncodeTiled entry point not available");
  const cuuint64_t n = 1ull << log2n;
  const cuuint64_t dims[5] = {4, 2, (cuuint64_t)C / 2, (cuuint64_t)L / 2, (n / (cuuint64_t)C) * (cuuint64_t)images};
  const cuuint64_t strides[4] = {16, 32, (cuuint64_t)C * 16, (cuuint64_t)(L * C) * 8};
  const cuuint32_t box[5] = {4, 1, (cuuint32_t)(C / 2 < 256 ? C / 2 : 256), 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void*>(in), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NSLCT_E_CUDA, "cuTensorMapEncodeTiled (Q16) failed (" + std::to_string((int)r) + ")");
  return NSLCT_OK;
}

constexpr int kModes = 6;   // pass modes 0..5 (kernels.cuh pass_body)

// the non-warp-specialised pipe kernel runs the passes that read the user's input (modes
// 0, 4: measured faster there than the warp-specialised kernel) and the
// three-FFT LC pass of form II (mode 5); modes 1-3 run line_pass_ws_kernel
template <typename T, int LOG2N>
struct PipeRow {
  static void fill(pipe_fn* l, attr_fn* at) {
    l[0] = launch_pipe<T, LOG2N, 0>;
    l[4] = launch_pipe<T, LOG2N, 4>;
    l[5] = launch_pipe<T, LOG2N, 5>;
    at[0] = set_attr_pipe<T, LOG2N, 0>;
    at[4] = set_attr_pipe<T, LOG2N, 4>;
    at[5] = set_attr_pipe<T, LOG2N, 5>;
  }
};

// needs an even number of lines per group; at N = 256 (C2) the persistent kernels measured
// 0.66x the one-CTA-per-group line passes (389k vs 585k transforms/s)
constexpr int kPipeMinLog = 10, kPipeMaxLog = 12;

template <typename T, int LOG2N>
struct Row {
  static void fill(launch_fn* l, attr_fn* at) {
    l[0] = launch_pass<T, LOG2N, 0>;
    l[1] = launch_pass<T, LOG2N, 1>;
    l[2] = launch_pass<T, LOG2N, 2>;
    l[3] = launch_pass<T, LOG2N, 3>;
    l[4] = launch_pass<T, LOG2N, 4>;
    l[5] = launch_pass<T, LOG2N, 5>;
    at[0] = set_attr<T, LOG2N, 0>;
    at[1] = set_attr<T, LOG2N, 1>;
    at[2] = set_attr<T, LOG2N, 2>;
    at[3] = set_attr<T, LOG2N, 3>;
    at[4] = set_attr<T, LOG2N, 4>;
    at[5] = set_attr<T, LOG2N, 5>;
  }
};

constexpr int kMinLog = 5, kMaxLog = 14;
constexpr int kMaxLog128 = 13;  // c128 line buffer of 16384 would exceed shared memory

// fully on-chip small-N variant (F2): one CTA (C = 1) or a C-CTA cluster per image
typedef cudaError_t (*img_fn)(const nslct::ImgArgs&, cudaStream_t, long long);
template <typename T, int LOG2N, int C>
cudaError_t launch_img(const nslct::ImgArgs& a, cudaStream_t s, long long batch) {
  using Cfg = nslct::ImgCfg<T, LOG2N, C>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * C));
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = (C > 1) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, nslct::image_kernel<T, LOG2N, C>, a);
}
template <typename T, int LOG2N, int C>
cudaError_t set_attr_img() {
  using Cfg = nslct::ImgCfg<T, LOG2N, C>;
  return cudaFuncSetAttribute(nslct::image_kernel<T, LOG2N, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)Cfg::SMEM);
}

struct Table {
  img_fn li[2][kMaxLog + 1] = {};   // on-chip kernels: c64 N <= 256, c128 N <= 128
  attr_fn ati[2][kMaxLog + 1] = {};
  launch_fn l[2][kMaxLog + 1][kModes] = {};
  attr_fn at[2][kMaxLog + 1][kModes] = {};
  launch_fn lpair[2][kMaxLog + 1][kModes] = {};   // c64 N = 16384 (cluster pairs): [slab]
  attr_fn atpair[2][kMaxLog + 1][kModes] = {};
  big_fn lbig[2][kMaxLog + 1][kModes] = {};     // c64 N = 8192 (TMA-pipelined): [slab]
  attr_fn atbig[2][kMaxLog + 1][kModes] = {};
  pipe_fn lp[kMaxLog + 1][kModes] = {};   // c64 only
  attr_fn atp[kMaxLog + 1][kModes] = {};
  Table() {
    li[0][5] = launch_img<float, 5, 1>, ati[0][5] = set_attr_img<float, 5, 1>;
    li[0][6] = launch_img<float, 6, 1>, ati[0][6] = set_attr_img<float, 6, 1>;
    li[0][7] = launch_img<float, 7, 1>, ati[0][7] = set_attr_img<float, 7, 1>;
    li[0][8] = launch_img<float, 8, 4>, ati[0][8] = set_attr_img<float, 8, 4>;
    li[1][5] = launch_img<double, 5, 1>, ati[1][5] = set_attr_img<double, 5, 1>;
    li[1][6] = launch_img<double, 6, 1>, ati[1][6] = set_attr_img<double, 6, 1>;
    li[1][7] = launch_img<double, 7, 4>, ati[1][7] = set_attr_img<double, 7, 4>;
    Pair2Row<false>::fill(lpair[0][14], atpair[0][14]);
    Pair2Row<true>::fill(lpair[1][14], atpair[1][14]);
    BigRow<13, false>::fill(lbig[0][13], atbig[0][13]);
    BigRow<13, true>::fill(lbig[1][13], atbig[1][13]);
    PipeRow<float, 10>::fill(lp[10], atp[10]);
    PipeRow<float, 11>::fill(lp[11], atp[11]);
    PipeRow<float, 12>::fill(lp[12], atp[12]);
    Row<float, 5>::fill(l[0][5], at[0][5]);
    Row<float, 6>::fill(l[0][6], at[0][6]);
    Row<float, 7>::fill(l[0][7], at[0][7]);
    Row<float, 8>::fill(l[0][8], at[0][8]);
    Row<float, 9>::fill(l[0][9], at[0][9]);
    Row<float, 10>::fill(l[0][10], at[0][10]);
    Row<float, 11>::fill(l[0][11], at[0][11]);
    Row<float, 12>::fill(l[0][12], at[0][12]);
    Row<float, 13>::fill(l[0][13], at[0][13]);
    Row<float, 14>::fill(l[0][14], at[0][14]);
    Row<double, 5>::fill(l[1][5], at[1][5]);
    Row<double, 6>::fill(l[1][6], at[1][6]);
    Row<double, 7>::fill(l[1][7], at[1][7]);
    Row<double, 8>::fill(l[1][8], at[1][8]);
    Row<double, 9>::fill(l[1][9], at[1][9]);
    Row<double, 10>::fill(l[1][10], at[1][10]);
    Row<double, 11>::fill(l[1][11], at[1][11]);
    Row<double, 12>::fill(l[1][12], at[1][12]);
    Row<double, 13>::fill(l[1][13], at[1][13]);
  }
};
const Table& table() {
  static Table t;
  return t;
}

// ---- fixed-point phase coefficients ------------------------------------------------
// turns -> 64-bit fixed-point fraction of a turn (mod 1).  x - nearbyint(x) is exact in
// fp64 and keeps the full relative precision of a small |x| (reducing a small negative
// x to 1 - |x| first would round it to 2^-53 turns, ~1e-10 turns after scaling by i^2).
uint64_t fx(double turns) {
  const double f = turns - std::nearbyint(turns);   // [-1/2, 1/2], exact
  double v = std::ldexp(f, 64);                      // [-2^63, 2^63], exact
  if (v >= 9223372036854775808.0) v -= 18446744073709551616.0;
  return (uint64_t)(int64_t)v;
}

// Chirp exp(j/2 d^2 (q11 p^2 + 2 q12 p q + q22 q^2)) with centered p = i - h, q = j - h,
// plus `checker` half-turns per index (the centring checkerboard (-1)^(i+j)), as a
// polynomial in array indices (i, j):  t = A i^2 + B ij + C j^2 + Li i + Lj j + K.
struct Poly {
  uint64_t A, B, C, Li, Lj, K;
};
Poly chirp_poly(const nslct::Sym& q, double d, int n, bool checker) {
  const double c0 = d * d / (4.0 * M_PI);
  const uint64_t A = fx(c0 * q.q11), B = fx(2.0 * c0 * q.q12), C = fx(c0 * q.q22);
  const uint64_t h = (uint64_t)(n / 2);
  Poly P;
  P.A = A;
  P.B = B;
  P.C = C;
  // a(i-h)^2 + b(i-h)(j-h) + c(j-h)^2 expanded, all mod 2^64
  P.Li = (uint64_t)0 - (2ull * h * A + h * B);
  P.Lj = (uint64_t)0 - (2ull * h * C + h * B);
  P.K = h * h * (A + B + C);
  if (checker) {
    P.Li += (1ull << 63);
    P.Lj += (1ull << 63);
  }
  return P;
}
// Z_m = exp(2 pi j m(m-1)/2 dd), dd = 2 cC TL^2 (mod 2^64), for the rotation evaluation
// of complex64 chirps (kernels.cuh struct Phase).
void set_rec(Phase* ph, int tl) {
  const uint64_t dd = 2ull * ph->cC * (uint64_t)tl * (uint64_t)tl;
  // structure the kernel exploits (struct Phase::kind): constant along the line, or no
  // element-quadratic step
  ph->kind = (ph->cB == 0 && ph->cC == 0 && ph->cE * (uint64_t)tl == 0) ? 2 : (dd == 0) ? 1 : 0;
  for (int m = 0; m < 8; ++m) {
    const uint64_t t = (uint64_t)(m * (m - 1) / 2) * dd;
    const double ang = 2.0 * M_PI * ((double)(int64_t)t * 5.42101086242752217e-20);   // 2^-64 turns
    ph->zr[m] = (float)std::cos(ang);
    ph->zi[m] = (float)std::sin(ang);
  }
  ph->rec = 1;
}
// complex64 plans: chirp coefficients whose largest phase over the N x N grid is below
// kSnapRad are dropped (set to 0) -- far below the fp32 phase evaluation's own error (the
// complex64 transform's relL2 against the oracle is ~2e-6), and it lets the kernels use the
// cheaper chirp forms of struct Phase::kind.  The HA search often ends on such a point
// (e.g. C4's Q4 has q12, q22 ~ 1e-11 next to q11 = -1.53: a chirp constant along each
// line).  DESIGN.md §6.3.
constexpr double kSnapRad = 1e-6;
nslct::Sym snap_c64(nslct::Sym q, double d, int n) {
  const double m2 = 0.25 * (double)n * (double)n * d * d;   // (n/2 d)^2: largest |z_a z_b|
  auto cut = [&](double v, double w) { return std::fabs(v) * w * m2 < kSnapRad ? 0.0 : v; };
  q.q11 = cut(q.q11, 0.5);
  q.q22 = cut(q.q22, 0.5);
  q.q12 = cut(q.q12, 1.0);
  return q;
}
// roles: line index = i (x) or j (y)
Phase to_phase(const Poly& P, bool line_is_x) {
  Phase ph{};
  if (line_is_x) {
    ph.cA = P.A; ph.cB = P.B; ph.cC = P.C; ph.cL = P.Li; ph.cE = P.Lj; ph.cK = P.K;
  } else {
    ph.cA = P.C; ph.cB = P.B; ph.cC = P.A; ph.cL = P.Lj; ph.cE = P.Li; ph.cK = P.K;
  }
  return ph;
}

}  // namespace

// ---- NCCL, loaded at run time ----------------------------------------------------------
// The library links no NCCL: dlopen("libnccl.so.2") returns the copy already mapped into
// the process (glibc matches the soname -- PyTorch's NCCL when torch is loaded), else the
// one the loader finds.  Only the entry points the slab exchange needs are resolved.
namespace {
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.err = std::string("dlopen(libnccl.so.2): ") + (e ? e : "not found");
      return a;
    }
    bool ok = true;
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) {
        ok = false;
        a.err += std::string(a.err.empty() ? "" : "; ") + "missing " + name;
      }
      return f;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = ok;
    return a;
  }();
  return api;
}
}  // namespace

#define NCCL_TRY(expr)                                                                      \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      return fail(NSLCT_E_NCCL, std::string(#expr) + ": " + nccl_api().GetErrorString(r_)); \
  } while (0)

struct nslct_comm_s {
  ncclComm_t c = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

struct nslct_plan_s {
  int64_t n = 0, batch = 0;
  int log2n = 0;       // power-of-two plans: log2 N; Bluestein plans: log2 M (FFT length)
  int64_t nl = 0;      // line length of the passes: N, or 2N for Ding plans
  bool bluestein = false;   // arbitrary N (row F3): every line DFT by Bluestein, length M
  int64_t n_in = 0;         // input side (fused zero-padding when < n)
  size_t in_img_bytes = 0;  // bytes of one input image (n_in^2 elements)
  void* bq = nullptr;       // Bluestein tables (kernels.cuh TwBluestein)
  void* bhat = nullptr;
  nslct_dtype dtype = NSLCT_C64;
  int device = 0;
  int profile = 0;
  double dx = 0;
  nslct::Plan p;
  size_t elem = 8, bytes = 0;
  void* tw = nullptr;
  void* scratch = nullptr;
  void* h_in = nullptr;   // device staging for exec_host
  void* h_out = nullptr;
  cudaStream_t cs_in = nullptr, cs_out = nullptr;   // exec_host copy streams (H2D, D2H)
  std::vector<cudaEvent_t> cev;                     // exec_host: 2 events per chunk + 1
  PassArgs args[5];
  int n_passes = 5;
  int mode[5] = {0, 1, 2, 1, 3};   // HA schedule; LC (y-axis H) uses 3 passes
  bool slab = false;   // row-slab plan (nslct_plan_slab, or nslct_plan_ex with opts.comm)
  int nranks = 1, rank = 0;
  int64_t L = 0;       // rows of this rank's slab
  int nc = 1;          // slab: exchange chunks per transposing pass; sub-block width lc = L / nc
  int64_t lc = 0;
  nslct_comm_s* comm = nullptr;          // slab plans run by nslct_exec (opts.comm)
  void* xsend = nullptr;                 // comm plans: pass output / all-to-all send buffer
  void* xrecv[2] = {nullptr, nullptr};   // all-to-all receive buffers (alternating passes)
  cudaStream_t cs_comm = nullptr;        // NCCL stream
  std::vector<cudaEvent_t> xev;          // nc chunk events + 1 exchange-done event
  int exchange = NSLCT_EXCHANGE_NCCL;    // comm plans: NCCL send/recv, or stores to peers
  void* peer_recv[2][8] = {};            // PEER: every rank's receive buffer b (own = xrecv[b])
  bool peer_opened[2][8] = {};           //       ... opened through cudaIpcOpenMemHandle
  int* xbar = nullptr;                   // PEER: 4-byte all-reduce "barrier" buffer
  bool pipe = false;   // persistent TMA-pipelined kernels
  bool image = false;  // fully on-chip kernel (one launch per exec)
  bool ws = false;     // warp-specialised pipe kernels for modes 1-3
  bool pair = false;   // large-N cluster-pair line passes (N = 16384, complex64)
  bool big = false;    // large-N TMA-pipelined cluster-pair passes (N = 8192, complex64)
  unsigned long long* counters = nullptr;   // per-pass group counters (pipe mode)
  int num_sms = 148;
  int host_chunk_kb = 0;    // opts.host_chunk_kb (exec_host pipeline chunk; 0 = auto)
  nslct::B0Args b0{};
  nslct::DingArgs ding{};
  struct EvSet {
    cudaEvent_t e[6];
  };
  std::vector<EvSet> ev;  // one set per exec since the last nslct_pass_ms (profile mode)
  size_t ev_used = 0;
};

namespace {
struct DeviceGuard {
  int prev = -1;
  cudaError_t status = cudaSuccess;   // of the cudaSetDevice (plan_internal validates the ordinal)
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) status = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define GUARD_DEVICE(pl)                                                                  \
  DeviceGuard guard((pl)->device);                                                        \
  if (guard.status != cudaSuccess)                                                        \
  return fail(NSLCT_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(guard.status))

void free_plan(nslct_plan_s* pl) {
  if (!pl) return;
  DeviceGuard g(pl->device);
  if (pl->tw) cudaFree(pl->tw);
  if (pl->bq) cudaFree(pl->bq);
  if (pl->bhat) cudaFree(pl->bhat);
  if (pl->scratch) cudaFree(pl->scratch);
  if (pl->xsend) cudaFree(pl->xsend);
  for (void* r : pl->xrecv)
    if (r) cudaFree(r);
  if (pl->cs_comm) cudaStreamDestroy(pl->cs_comm);
  for (int b = 0; b < 2; ++b)
    for (int s = 0; s < 8; ++s)
      if (pl->peer_opened[b][s]) cudaIpcCloseMemHandle(pl->peer_recv[b][s]);
  if (pl->xbar) cudaFree(pl->xbar);
  for (auto e : pl->xev)
    if (e) cudaEventDestroy(e);
  if (pl->counters) cudaFree(pl->counters);
  if (pl->h_in) cudaFree(pl->h_in);
  if (pl->h_out) cudaFree(pl->h_out);
  if (pl->cs_in) cudaStreamDestroy(pl->cs_in);
  if (pl->cs_out) cudaStreamDestroy(pl->cs_out);
  for (auto e : pl->cev)
    if (e) cudaEventDestroy(e);
  for (auto& set : pl->ev)
    for (auto& e : set.e)
      if (e) cudaEventDestroy(e);
  delete pl;
}
}  // namespace

namespace {
constexpr int64_t kBlMaxN = 4096;   // Bluestein FFT length M <= 2^kBlMaxLog

// (cos, sin) of 2 pi num/den, the argument reduced exactly to [-1/8, 1/8] turn around
// the nearest quarter turn before the fp64 cos/sin.
void cis_turns(int64_t num, int64_t den, double* c, double* s) {
  num %= den;
  if (num < 0) num += den;
  const int64_t q4 = (4 * num + den / 2) / den;
  const double r = 2.0 * M_PI * ((double)(4 * num - q4 * den) / (4.0 * (double)den));
  const double cr = std::cos(r), sr = std::sin(r);
  switch (q4 & 3) {
    case 0: *c = cr; *s = sr; break;
    case 1: *c = -sr; *s = cr; break;
    case 2: *c = -cr; *s = -sr; break;
    default: *c = sr; *s = -cr; break;
  }
}

// In-place fp64 radix-2 FFT (forward, e^{-2 pi i jk/M}) of the host table builder.
void host_fft(std::vector<double>& re, std::vector<double>& im) {
  const int64_t m = (int64_t)re.size();
  for (int64_t i = 1, j = 0; i < m; ++i) {
    int64_t bit = m >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      std::swap(re[i], re[j]);
      std::swap(im[i], im[j]);
    }
  }
  for (int64_t len = 2; len <= m; len <<= 1) {
    for (int64_t k = 0; k < len / 2; ++k) {
      double c, sn;
      cis_turns(-k, len, &c, &sn);
      for (int64_t i = k; i < m; i += len) {
        const int64_t u = i, v = i + len / 2;
        const double tr = re[v] * c - im[v] * sn, ti = re[v] * sn + im[v] * c;
        re[v] = re[u] - tr;
        im[v] = im[u] - ti;
        re[u] += tr;
        im[u] += ti;
      }
    }
  }
}

// Bluestein tables of kernels.cuh TwBluestein for a plan of side n and FFT length
// M = 2^log2n:  bq[i] = exp(-j pi (i-h)^2/N), bhat = FFT_M(c)/M with
// c[k mod M] = exp(+j pi k^2/N) for |k| < N.  Phases reduced exactly: k^2 mod 2N.
nslct_status bluestein_tables(nslct_plan_s* pl) {
  const int64_t n = pl->nl, m = int64_t(1) << pl->log2n, h = n / 2;
  std::vector<double> bre(n), bim(n), cre(m, 0.0), cim(m, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t d = i - h;
    cis_turns(-((d * d) % (2 * n)), 2 * n, &bre[i], &bim[i]);
  }
  for (int64_t k = -(n - 1); k <= n - 1; ++k) {
    const int64_t pos = (k + m) % m;
    cis_turns((k * k) % (2 * n), 2 * n, &cre[pos], &cim[pos]);
  }
  host_fft(cre, cim);
  const size_t e = pl->elem;
  std::vector<unsigned char> hb(n * e), hh(m * e);
  auto put = [&](unsigned char* dst, int64_t i, double re, double im) {
    if (e == 8) {
      float* f = reinterpret_cast<float*>(dst);
      f[2 * i] = (float)re;
      f[2 * i + 1] = (float)im;
    } else {
      double* f = reinterpret_cast<double*>(dst);
      f[2 * i] = re;
      f[2 * i + 1] = im;
    }
  };
  for (int64_t i = 0; i < n; ++i) put(hb.data(), i, bre[i], bim[i]);
  for (int64_t k = 0; k < m; ++k) put(hh.data(), k, cre[k] / (double)m, cim[k] / (double)m);
  CUDA_TRY(cudaMalloc(&pl->bq, n * e));
  CUDA_TRY(cudaMalloc(&pl->bhat, m * e));
  CUDA_TRY(cudaMemcpy(pl->bq, hb.data(), n * e, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(pl->bhat, hh.data(), m * e, cudaMemcpyHostToDevice));
  return NSLCT_OK;
}
}  // namespace

extern "C" {

void nslct_opts_default(nslct_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->dx = 0.0;
  o->variant = NSLCT_VARIANT_HA;
  o->dispatch = NSLCT_DISPATCH_REVERSIBLE;
  o->device = -1;
  o->profile = 0;
}

int nslct_abi_version(void) { return NSLCT_ABI_VERSION; }

const char* nslct_last_error(void) { return g_err.c_str(); }

nslct_status nslct_plan(nslct_plan_t* plan, int64_t n, const double abcd[16], int64_t batch,
                        nslct_dtype dtype) {
  nslct_opts o;
  nslct_opts_default(&o);
  return nslct_plan_ex(plan, n, abcd, batch, dtype, &o);
}

// The chain's H is rank one along y, H = (0,0;0,h) (Eq. LC12 with the F_y form; LC plans
// with that axis, or a FIXED_H plan given such an H): the 3-pass schedule applies.
static bool lc_y(const nslct::Plan& p) {
  return p.kind != 0 && p.H.q11 == 0.0 && p.H.q12 == 0.0 && p.H.q22 != 0.0;
}

// PEER exchange (NSLCT_EXCHANGE_PEER): map every rank's two receive buffers into this
// process.  Collective over the plan's communicator: each rank publishes the CUDA IPC
// handles of its xrecv[0..1] by an NCCL all-gather, then opens the other ranks' (its own
// buffers are used directly).
static nslct_status peer_setup(nslct_plan_s* pl) {
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(NSLCT_E_NCCL, api.err);
  const int P = pl->nranks;
  constexpr size_t H = sizeof(cudaIpcMemHandle_t);   // 64 bytes
  std::vector<unsigned char> mine(2 * H), all((size_t)P * 2 * H);
  for (int b = 0; b < 2; ++b)
    CUDA_TRY(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(mine.data() + b * H), pl->xrecv[b]));
  unsigned char* dev = nullptr;
  CUDA_TRY(cudaMalloc(&dev, (size_t)(P + 1) * 2 * H));
  cudaError_t e = cudaMemcpy(dev + (size_t)P * 2 * H, mine.data(), 2 * H, cudaMemcpyHostToDevice);
  ncclResult_t r = ncclSuccess;
  if (e == cudaSuccess) r = api.AllGather(dev + (size_t)P * 2 * H, dev, 2 * H, ncclInt8, pl->comm->c, pl->cs_comm);
  if (e == cudaSuccess && r == ncclSuccess) e = cudaStreamSynchronize(pl->cs_comm);
  if (e == cudaSuccess && r == ncclSuccess) e = cudaMemcpy(all.data(), dev, all.size(), cudaMemcpyDeviceToHost);
  cudaFree(dev);
  if (r != ncclSuccess) return fail(NSLCT_E_NCCL, std::string("ncclAllGather(IPC handles): ") + api.GetErrorString(r));
  if (e != cudaSuccess) return fail(NSLCT_E_CUDA, std::string("IPC handle exchange: ") + cudaGetErrorString(e));
  for (int s = 0; s < P; ++s)
    for (int b = 0; b < 2; ++b) {
      if (s == pl->rank) {
        pl->peer_recv[b][s] = pl->xrecv[b];
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, all.data() + ((size_t)s * 2 + b) * H, H);
      CUDA_TRY(cudaIpcOpenMemHandle(&pl->peer_recv[b][s], h, cudaIpcMemLazyEnablePeerAccess));
      pl->peer_opened[b][s] = true;
    }
  CUDA_TRY(cudaMalloc(&pl->xbar, sizeof(int)));
  CUDA_TRY(cudaMemset(pl->xbar, 0, sizeof(int)));
  return NSLCT_OK;
}

static nslct_status plan_internal(nslct_plan_t* plan, int64_t n, const double abcd[16], int64_t batch,
                                  nslct_dtype dtype, const nslct_opts* opts, int nranks, int rank);

nslct_status nslct_plan_ex(nslct_plan_t* plan, int64_t n, const double abcd[16], int64_t batch,
                           nslct_dtype dtype, const nslct_opts* opts) {
  if (opts && opts->comm) {   // one transform, row slabs over the communicator's ranks
    const nslct_comm_s* c = static_cast<const nslct_comm_s*>(opts->comm);
    if (batch != 1) return fail(NSLCT_E_ARG, "a comm (row-slab) plan transforms one image: batch must be 1");
    return plan_internal(plan, n, abcd, 1, dtype, opts, c->nranks, c->rank);
  }
  return plan_internal(plan, n, abcd, batch, dtype, opts, 0, 0);
}

nslct_status nslct_plan_slab(nslct_plan_t* plan, int64_t n, const double abcd[16], int nranks, int rank,
                             nslct_dtype dtype, const nslct_opts* opts) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NSLCT_E_ARG, "bad nranks/rank");
  return plan_internal(plan, n, abcd, 1, dtype, opts, nranks, rank);
}

static nslct_status plan_internal(nslct_plan_t* plan, int64_t n, const double abcd[16], int64_t batch,
                                  nslct_dtype dtype, const nslct_opts* opts, int nranks, int rank) {
  g_err.clear();
  if (!plan || !abcd) return fail(NSLCT_E_ARG, "null plan or abcd pointer");
  *plan = nullptr;
  nslct_opts o;
  if (opts)
    o = *opts;
  else
    nslct_opts_default(&o);
  if (dtype != NSLCT_C64 && dtype != NSLCT_C128) return fail(NSLCT_E_ARG, "bad dtype");
  if (batch < 1) return fail(NSLCT_E_ARG, "batch must be >= 1");
  if (o.variant < 0 || o.variant > 3 || o.dispatch < 0 || o.dispatch > 1 || o.schedule < 0 || o.schedule > 2)
    return fail(NSLCT_E_ARG, "bad variant/dispatch option");
  if (o.kernels < 0 || o.kernels > NSLCT_KERNELS_GENERIC) return fail(NSLCT_E_ARG, "bad kernels option");
  int lg = 0;
  while ((int64_t(1) << lg) < n && lg < 62) ++lg;
  const bool pow2 = n >= 1 && (int64_t(1) << lg) == n && lg >= kMinLog && lg <= kMaxLog &&
                    !(dtype == NSLCT_C128 && lg > kMaxLog128);
  if (!pow2) {   // arbitrary N: Bluestein line DFTs of length M = 2^lg >= 2N - 1 (row F3)
    if (n < 2 || n > kBlMaxN)
      return fail(NSLCT_E_UNSUPPORTED_N,
                  "N must be a power of two in [32, 16384] (c128: <= 8192) or any N in [2, 4096]");
    lg = nslct::kBlMinLog;
    while ((int64_t(1) << lg) < 2 * n - 1) ++lg;
  }
  const int64_t n_in = (o.n_in > 0) ? o.n_in : n;
  if (n_in > n) return fail(NSLCT_E_ARG, "n_in must be <= n");
  if (!(std::isfinite(o.dx)) || (o.dx > 0 && !(o.dx < 1e30)))
    return fail(NSLCT_E_ARG, "bad dx");

  const bool slab = nranks > 0;
  int64_t L = n, Lc = n;
  int nc = 1;
  if (slab) {
    if (n % nranks) return fail(NSLCT_E_ARG, "nranks must divide n");
    L = n / nranks;
    const int64_t TL = n / 16;
    const int64_t TB = (n <= 2048) ? 256 : (n <= 8192 ? 512 : 1024);
    const int64_t G = (TB / TL < n) ? TB / TL : n;
    if (L % G) return fail(NSLCT_E_ARG, "slab height n/nranks must be a multiple of the lines per CTA");
    // exchange chunks: sub-blocks of lc = L/nc producer lines (PassArgs::out_chunk); each
    // chunk a whole number of CTA line groups (and of line pairs)
    const int want = (o.exchange_chunks > 0) ? o.exchange_chunks : 2;
    if (want != 1 && want != 2 && want != 4 && want != 8)
      return fail(NSLCT_E_ARG, "exchange_chunks must be 0, 1, 2, 4 or 8");
    nc = want;
    while (nc > 1 && ((L / nc) % G || (L / nc) % 2)) nc /= 2;
    Lc = L / nc;
  }
  if (o.comm && !slab) return fail(NSLCT_E_ARG, "opts.comm: use nslct_plan_ex (not nslct_plan_slab)");
  if (o.exchange != NSLCT_EXCHANGE_NCCL && o.exchange != NSLCT_EXCHANGE_PEER) return fail(NSLCT_E_ARG, "bad exchange");
  if (o.comm && o.exchange == NSLCT_EXCHANGE_PEER && nranks > 8)
    return fail(NSLCT_E_ARG, "the peer-store exchange supports at most 8 ranks");
  std::string err;
  nslct::Plan p;
  int st = nslct::make_plan(abcd, o.variant, o.dispatch, o.h_fixed, &p, &err);
  if (st) return fail((nslct_status)st, err);
  if (slab && p.kind == 0) return fail(NSLCT_E_ARG, "B = 0 has no row-slab form");
  if (slab && (!pow2 || n_in != n)) return fail(NSLCT_E_ARG, "row-slab plans need a power-of-two N and no padding");
  if (p.kind == 3 && (slab || n_in != n)) return fail(NSLCT_E_ARG, "Ding plans have no row-slab or padded form");
  // line length of the passes: n, or 2n for Ding's two-times upsampled DFT
  const int64_t nl = (p.kind == 3) ? 2 * n : n;
  bool pow2l = pow2;
  if (p.kind == 3) {
    lg = 0;
    while ((int64_t(1) << lg) < nl && lg < 62) ++lg;
    pow2l = (int64_t(1) << lg) == nl && lg >= kMinLog && lg <= kMaxLog && !(dtype == NSLCT_C128 && lg > kMaxLog128);
    if (!pow2l) {
      if (nl > kBlMaxN)
        return fail(NSLCT_E_UNSUPPORTED_N, "Ding plans: 2N must be a power of two <= 16384 (c128: 8192) or <= 4096");
      lg = nslct::kBlMinLog;
      while ((int64_t(1) << lg) < 2 * nl - 1) ++lg;
    }
  }

  nslct_plan_s* pl = new (std::nothrow) nslct_plan_s();
  if (!pl) return fail(NSLCT_E_OOM, "host allocation failed");
  pl->n = n;
  pl->batch = batch;
  pl->log2n = lg;
  pl->nl = nl;
  pl->bluestein = !pow2l;
  pl->n_in = n_in;
  pl->dtype = dtype;
  pl->p = p;
  pl->profile = o.profile;
  pl->dx = (o.dx > 0) ? o.dx : std::sqrt(2.0 * M_PI / (double)n);
  pl->elem = (dtype == NSLCT_C64) ? 8 : 16;
  pl->bytes = (size_t)batch * (size_t)n * (size_t)n * pl->elem;
  pl->in_img_bytes = (size_t)n_in * (size_t)n_in * pl->elem;
  pl->slab = slab;
  pl->nranks = slab ? nranks : 1;
  pl->rank = slab ? rank : 0;
  pl->L = L;
  pl->nc = nc;
  pl->lc = Lc;
  pl->comm = static_cast<nslct_comm_s*>(o.comm);
  pl->exchange = o.exchange;
  if (o.device >= 0) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || o.device >= count) {
      delete pl;
      return fail(NSLCT_E_ARG, "opts.device " + std::to_string(o.device) + " is not a CUDA device ordinal (" +
                                   std::to_string(count) + " devices)");
    }
    pl->device = o.device;
  } else {
    cudaError_t e = cudaGetDevice(&pl->device);
    if (e != cudaSuccess) {
      delete pl;
      return fail(NSLCT_E_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    }
  }
  pl->host_chunk_kb = o.host_chunk_kb;
  nslct_status result = NSLCT_OK;
  do {
    DeviceGuard guard(pl->device);
    if (guard.status != cudaSuccess) {
      result = fail(NSLCT_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(guard.status));
      break;
    }
    const int ti = (dtype == NSLCT_C64) ? 0 : 1;
    const double dx = pl->dx;
    const double dw = 2.0 * M_PI / ((double)n * dx);  // frequency grid
    if (p.kind == 0) {
      // B = 0: chirp exp(j/2 z'^T C D^T z') and sqrt(det D) (Eq. Intro20)
      nslct::M2 C = p.Cb, D = p.Db;
      nslct::M2 CDt = {C.a * D.a + C.b * D.b, C.a * D.c + C.b * D.d, C.c * D.a + C.d * D.b,
                       C.c * D.c + C.d * D.d};
      nslct::Sym S = {CDt.a, CDt.d, 0.5 * (CDt.b + CDt.c)};
      Poly P = chirp_poly(S, dx, (int)n, false);
      double detD = D.a * D.d - D.b * D.c;
      nslct::B0Args& b = pl->b0;
      b.n = (int)n;
      b.total = batch * n * n;
      b.d11 = D.a; b.d12 = D.b; b.d21 = D.c; b.d22 = D.d;
      b.amp_re = detD >= 0 ? std::sqrt(detD) : 0.0;
      b.amp_im = detD >= 0 ? 0.0 : std::sqrt(-detD);
      b.ph = to_phase(P, true);
      b.n_in = (int)n_in;
      b.in_off = (int)(n / 2 - n_in / 2);
      break;
    }
    // twiddles exp(-2 pi i k/N) in fp64, stored at the run precision (N = M for Bluestein)
    if (pl->bluestein) {
      nslct_status st = bluestein_tables(pl);
      if (st != NSLCT_OK) { result = st; break; }
    }
    {
      const int64_t nt = int64_t(1) << lg;
      const size_t tw_bytes = (size_t)nt * pl->elem;
      unsigned char* host = new (std::nothrow) unsigned char[tw_bytes];
      if (!host) { result = fail(NSLCT_E_OOM, "host twiddles"); break; }
      for (int64_t k = 0; k < nt; ++k) {
        // reduce k/N to [-1/8, 1/8] turns around the nearest quarter for accuracy
        double s, c;
        const int64_t q4 = (4 * k + nt / 2) / nt;         // nearest quarter turn
        const double r = 2.0 * M_PI * ((double)(4 * k - q4 * nt) / (4.0 * (double)nt));
        const double cr = std::cos(r), sr = std::sin(r);
        switch (q4 & 3) {
          case 0: c = cr; s = sr; break;
          case 1: c = -sr; s = cr; break;
          case 2: c = -cr; s = -sr; break;
          default: c = sr; s = -cr; break;
        }
        if (dtype == NSLCT_C64) {
          float* f = reinterpret_cast<float*>(host);
          f[2 * k] = (float)c;
          f[2 * k + 1] = (float)(-s);
        } else {
          double* f = reinterpret_cast<double*>(host);
          f[2 * k] = c;
          f[2 * k + 1] = -s;
        }
      }
      cudaError_t e = cudaMalloc(&pl->tw, tw_bytes);
      if (e == cudaSuccess) e = cudaMemcpy(pl->tw, host, tw_bytes, cudaMemcpyHostToDevice);
      delete[] host;
      if (e != cudaSuccess) {
        result = fail(e == cudaErrorMemoryAllocation ? NSLCT_E_OOM : NSLCT_E_CUDA,
                      std::string("twiddles: ") + cudaGetErrorString(e));
        break;
      }
    }
    if (pl->comm) {   // row slabs over a communicator: send + 2 receive buffers, NCCL stream
      if (pl->comm->device != pl->device) {
        result = fail(NSLCT_E_ARG, "opts.comm was initialised on another device than the plan's");
        break;
      }
      const size_t sb = (size_t)L * (size_t)n * pl->elem;
      cudaError_t e = (o.exchange == NSLCT_EXCHANGE_NCCL) ? cudaMalloc(&pl->xsend, sb) : cudaSuccess;
      if (e == cudaSuccess) e = cudaMalloc(&pl->xrecv[0], sb);
      if (e == cudaSuccess) e = cudaMalloc(&pl->xrecv[1], sb);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pl->cs_comm, cudaStreamNonBlocking);
      for (int i = 0; i <= nc && e == cudaSuccess; ++i) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) pl->xev.push_back(ev);
      }
      if (e != cudaSuccess) {
        result = fail(e == cudaErrorMemoryAllocation ? NSLCT_E_OOM : NSLCT_E_CUDA,
                      std::string("slab exchange buffers: ") + cudaGetErrorString(e));
        break;
      }
      if (o.exchange == NSLCT_EXCHANGE_PEER) {
        nslct_status st = peer_setup(pl);
        if (st != NSLCT_OK) {
          result = st;
          break;
        }
      }
    }
    if (!slab) {
      const size_t sb = (p.kind == 3) ? 2 * (size_t)batch * (size_t)nl * (size_t)nl * pl->elem : pl->bytes;
      cudaError_t e = cudaMalloc(&pl->scratch, sb);
      if (e != cudaSuccess) {
        result = fail(e == cudaErrorMemoryAllocation ? NSLCT_E_OOM : NSLCT_E_CUDA,
                      std::string("scratch: ") + cudaGetErrorString(e));
        break;
      }
    }
    const nslct::Sym zero = {0, 0, 0};
    const double invn = 1.0 / (double)n;
    // K1: CM_r(Q0) + checkerboard;  K2: CM_w(Q1)/N;  K3: CM_r(Q2)/N;  K4: CM_w(Q3)/N;
    // K5: CM_r(Q4)/N + checkerboard.
    // power-of-two plans: the centred DFT is S W S (kernels.cuh header); the outer
    // checkerboards S ride on the first and last chirps.  Bluestein DFTs are centred
    // by construction: no checkerboard.
    const bool ck = !pl->bluestein;
    auto qs = [&](const nslct::Sym& q, double d) { return ti == 0 ? snap_c64(q, d, (int)n) : q; };
    Poly P0 = chirp_poly(p.q_active[0] ? qs(p.Q[0], dx) : zero, dx, (int)n, ck);
    Poly P1 = chirp_poly(qs(p.Q[1], dw), dw, (int)n, false);
    Poly P2 = chirp_poly(qs(p.Q[2], dx), dx, (int)n, false);
    Poly P3 = chirp_poly(qs(p.Q[3], dw), dw, (int)n, false);
    Poly P4 = chirp_poly(p.q_active[4] ? qs(p.Q[4], dx) : zero, dx, (int)n, ck);
    const Phase ph[5] = {to_phase(P0, true), to_phase(P1, false), to_phase(P2, true),
                         to_phase(P3, false), to_phase(P4, true)};
    // inverse FFTs are unnormalised; the last pass applies 1/N^4 (two 2D inverses)
    const double sc[5] = {1.0, 1.0, 1.0, 1.0, invn * invn * invn * invn};
    const int sign_only[5] = {(p.q_active[0] || !ck) ? 0 : 1, 0, 0, 0, (p.q_active[4] || !ck) ? 0 : 1};
    for (int k = 0; k < 5; ++k) {
      pl->args[k] = PassArgs{};
      pl->args[k].tw = pl->tw;
      pl->args[k].n_lines = batch * n;
      pl->args[k].ph = ph[k];
      pl->args[k].scale = sc[k];
      pl->args[k].sign_only = sign_only[k];
    }
    if (lc_y(p) && !pl->bluestein) {
      // LC-NsDLCT with H = (0,0;0,h) (Eq. LC12 with F_y): the 1D CC along y merges with
      // the neighbouring y-axis FFTs, 3 passes.  S_x / S_y are the
      // one-axis centring checkerboards left over when a 1D and a 2D DFT meet.
      const uint64_t HALF = 1ull << 63;
      Poly Pq1 = chirp_poly(p.Q[1], dw, (int)n, false);   // rank-1 y chirp: 1D freq grid
      Poly Pq3 = chirp_poly(p.Q[3], dw, (int)n, false);   // rank-1 y chirp (form II)
      Poly Psx2 = chirp_poly(p.Q[2], dx, (int)n, false);
      Psx2.Li += HALF;                                      // S_x * CM(Q2)
      const double inv3 = invn * invn * invn;               // W_y^-1 and one 2D W^-1
      pl->n_passes = 3;
      if (p.kind == 1) {
        pl->mode[0] = 4; pl->mode[1] = 1; pl->mode[2] = 3;
        PassArgs& a0 = pl->args[0];          // S_y, FFT_y, CM_wy(Q1), IFFT_y, S_x CM(Q2), FFT_y
        a0.ph = Phase{};
        a0.sign_only = 2;
        a0.ph_b = to_phase(Pq1, true);
        a0.ph_c = to_phase(Psx2, true);
        a0.sign_c = 0;
        pl->args[1].ph = to_phase(P3, false); // FFT_x, CM_w(Q3), IFFT_x
        pl->args[2] = pl->args[4];            // IFFT_y, CM(Q4) S / N^3
        pl->args[2].scale = inv3;
      } else {
        pl->mode[0] = 0; pl->mode[1] = 1; pl->mode[2] = 5;
        // pass 0: S CM(Q0), FFT_y (as the HA K1); pass 1: FFT_x, CM_w(Q1), IFFT_x
        PassArgs& a2 = pl->args[2];          // IFFT_y, S_x CM(Q2), FFT_y, CM_wy(Q3), IFFT_y, S_y / N^3
        a2.ph = to_phase(Psx2, true);
        a2.sign_only = 0;
        a2.ph_b = to_phase(Pq3, true);
        a2.ph_c = Phase{};
        a2.sign_c = 2;
        a2.scale = inv3;
      }
    }
    for (int k = 0; k < 5; ++k) {
      pl->args[k].lines_per_img = (int)L;
      pl->args[k].line_offset = slab ? (int)(rank * L) : 0;
      pl->args[k].in_chunk = (slab && k > 0) ? (int)Lc : (int)n;
      pl->args[k].in_chunk_stride = (slab && k > 0) ? L * Lc : n * n;
      {   // PassArgs::in_eoff (N = 16384 pair kernel, chunks of >= 1024 elements)
        const long long C = pl->args[k].in_chunk, CS = (slab && k > 0) ? L * Lc : 0;
        for (int e = 0; e < 16; ++e) {
          const long long i0 = 1024ll * e;
          pl->args[k].in_eoff[e] = (C >= 1024) ? (i0 / C) * CS + 2 * (i0 % C) : 0;
        }
      }
      pl->args[k].out_chunk = (int)Lc;
      pl->args[k].line_base = 0;
      pl->args[k].n_lines = slab ? L : batch * n;
      pl->args[k].n_in = (k == 0 && n_in != n) ? (int)n_in : 0;
      pl->args[k].in_off = (k == 0 && n_in != n) ? (int)(n / 2 - n_in / 2) : 0;
    }
    if (p.kind == 3) {
      // Ding (Eq. Ding12): pass 0 = CM(B^-1 A) on the input zero-padded to 2N x 2N (+ the
      // input-side centring checkerboard on power-of-two grids), W_y; pass 1 = W_x; then
      // the gather (kernels.cuh ding_gather_kernel) from the 2N grid to the N x N output.
      Poly Pa = chirp_poly(p.Q[0], dx, (int)nl, ck);
      for (int k = 0; k < 2; ++k) {
        PassArgs& a = pl->args[k];
        a = PassArgs{};
        a.tw = pl->tw;
        a.ph = (k == 0) ? to_phase(Pa, true) : Phase{};
        a.scale = 1.0;
        a.sign_only = 0;
        a.lines_per_img = (int)nl;
        a.in_chunk = (int)nl;
        a.in_chunk_stride = nl * nl;
        a.out_chunk = (int)nl;
        a.n_lines = batch * nl;
        a.n_in = (k == 0) ? (int)n : 0;
        a.in_off = (k == 0) ? (int)(nl / 2 - n / 2) : 0;
      }
      pl->n_passes = 3;   // two line passes + the gather
      pl->mode[0] = pl->mode[1] = 0;
      nslct::DingArgs& d = pl->ding;
      d.n = (int)n;
      d.n2 = (int)nl;
      d.d11 = p.Db.a; d.d12 = p.Db.b; d.d21 = p.Db.c; d.d22 = p.Db.d;
      const double dwl = 2.0 * M_PI / ((double)nl * dx);   // DFT grid of the upsampled F
      d.ratio = dx / dwl;
      const double detD = p.Db.a * p.Db.d - p.Db.b * p.Db.c;
      const double sr = detD >= 0 ? std::sqrt(detD) : 0.0, si = detD >= 0 ? 0.0 : std::sqrt(-detD);
      const double c = dx * dx / (2.0 * M_PI);                // dx dy / (j 2 pi) = -j c
      d.amp_re = si * c;
      d.amp_im = -sr * c;
      d.ph = to_phase(chirp_poly(p.Q[4], dx, (int)n, false), true);
      d.checker = ck ? 1 : 0;
    }
    {
      int sms = 0;
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl->device) == cudaSuccess && sms > 0)
        pl->num_sms = sms;
      const bool plain = pow2 && n_in == n && p.kind != 3;   // neither Bluestein, padded nor Ding
      // opts.kernels = NSLCT_KERNELS_GENERIC: the one-CTA-per-line-group kernels everywhere
      // (same operator; the reference for A/B checks of the specialised kernels)
      const bool special = o.kernels == NSLCT_KERNELS_AUTO;
      pl->pipe = (plain && special && !slab && ti == 0 && lg >= kPipeMinLog && lg <= kPipeMaxLog);
      // L2 prefetch one claim ahead in the persistent kernels: one grid of groups ahead
      // (the group this CTA most likely claims next).  Measured on the C4 bench (DESIGN.md
      // §6.6): K1 1.51 -> 1.32 ms, K2-K5 +0.5-1% -- so on the first pass only.
      if (pl->pipe) pl->args[0].l2_ahead = pl->num_sms;
      // ... and on the last pass (one FFT + a chirp; K5 1.47 -> 1.37 ms at C4 since the chirps
      // became cheaper, profiles/r02f_l2ahead_ab.txt)
      if (pl->pipe) pl->args[pl->n_passes - 1].l2_ahead = pl->num_sms;
      // complex64 chirps by anchored rotation recurrences (kernels.cuh struct Phase) on
      // every pass: measured K5 1.71 -> 1.66 ms, K2-K4 -1.4..-2% on the C4 bench (DESIGN.md
      // §6.3)
      if (ti == 0) {
        const int tl = (1 << lg) / 16;
        for (int k = 0; k < 5; ++k) {
          set_rec(&pl->args[k].ph, tl);
          set_rec(&pl->args[k].ph_b, tl);
          set_rec(&pl->args[k].ph_c, tl);
        }
      }
      const bool large = plain && ti == 0 && (lg == 13 || lg == 14) && (L % 2 == 0) && (Lc % 16 == 0);
      // N = 8192: the TMA-pipelined kernel (Q16 intermediates); N = 16384: the cluster-pair
      // kernel (pair-interleaved intermediates) -- measured faster at each size (kernels.cuh)
      pl->big = large && special && lg == 13;
      pl->pair = large && special && lg == 14;
      for (int k = 0; k < 5 && (pl->pair || pl->big); ++k) pl->args[k].persist_ctas = (pl->num_sms / 2) * 2;
      for (int m = 0; m < kModes && (pl->pair || pl->big); ++m) {
        cudaError_t e = pl->big ? table().atbig[slab ? 1 : 0][lg][m]() : table().atpair[slab ? 1 : 0][lg][m]();
        if (e != cudaSuccess) {
          result = fail(NSLCT_E_CUDA, std::string("cudaFuncSetAttribute(large N): ") + cudaGetErrorString(e));
          break;
        }
      }
      if (result != NSLCT_OK) break;
      // warp-specialised kernels for the passes after the first (measured K2-K5 -0.6..-1.6%,
      // K1 +2.4% -- so not for mode 0)
      pl->ws = pl->pipe;
      if (pl->ws) {
        const WsRow* row = ws_row_of(lg);
        cudaError_t e = row ? cudaSuccess : cudaErrorInvalidValue;
        for (int m = 1; m <= 3 && e == cudaSuccess; ++m) e = row->attr[m - 1]();
        if (e != cudaSuccess) {
          result = fail(NSLCT_E_CUDA, std::string("cudaFuncSetAttribute(ws): ") + cudaGetErrorString(e));
          break;
        }
      }
      const bool have = plain && !slab && table().li[ti][lg] != nullptr;
      if (o.schedule == NSLCT_SCHEDULE_ON_CHIP && !have && pl->p.kind != 0) {
        result = fail(NSLCT_E_UNSUPPORTED_N, "no on-chip kernel for this N / dtype (c64 N <= 256, c128 N <= 128)");
        break;
      }
      // AUTO: on chip for N <= 64, where it beat the line passes at every batch size
      pl->image = have && (o.schedule == NSLCT_SCHEDULE_ON_CHIP || (o.schedule == NSLCT_SCHEDULE_AUTO && lg <= 6));
    }
    if (pl->image) {
      cudaError_t e = table().ati[ti][lg]();
      if (e != cudaSuccess) {
        result = fail(NSLCT_E_CUDA, std::string("cudaFuncSetAttribute(on-chip): ") + cudaGetErrorString(e));
        break;
      }
    }
    if (pl->pipe) {
      cudaError_t e = cudaMalloc(&pl->counters, 8 * sizeof(unsigned long long));
      if (e != cudaSuccess) {
        result = fail(NSLCT_E_OOM, std::string("counters: ") + cudaGetErrorString(e));
        break;
      }
    }
    for (int m = 0; m < kModes && pl->pipe; ++m) {
      if (!table().atp[lg][m]) continue;   // modes 1-3 run the warp-specialised kernel
      cudaError_t e = table().atp[lg][m]();
      if (e != cudaSuccess) {
        result = fail(NSLCT_E_CUDA, std::string("cudaFuncSetAttribute(pipe): ") + cudaGetErrorString(e));
        break;
      }
    }
    if (result != NSLCT_OK) break;
    for (int m = 0; m < 4 && pl->bluestein; ++m) {
      cudaError_t e = nslct::bl_attr(ti, lg, m)();
      if (e != cudaSuccess) {
        result = fail(NSLCT_E_CUDA, std::string("cudaFuncSetAttribute(bluestein): ") + cudaGetErrorString(e));
        break;
      }
    }
    for (int m = 0; m < kModes && !pl->bluestein; ++m) {
      cudaError_t e = table().at[ti][lg][m]();
      if (e != cudaSuccess) {
        result = fail(NSLCT_E_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        break;
      }
    }
    if (result != NSLCT_OK) break;
  } while (0);
  if (result != NSLCT_OK) {
    free_plan(pl);
    return result;
  }
  *plan = pl;
  return NSLCT_OK;
}

static nslct_status launch_large(nslct_plan_t pl, int k, const PassArgs& a, cudaStream_t s);

// one pipe pass: the transposed passes get the tensor map of their output
static nslct_status launch_pipe_pass(nslct_plan_t pl, int k, const PassArgs& a, cudaStream_t s) {
  const int m = pl->mode[k];
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (!(m == 3 || m == 5)) {   // not a straight-output mode (kernels.cuh ModeIO)
    nslct_status st = make_store_map(&map, a.out, pl->log2n, a.n_lines >> pl->log2n);
    if (st != NSLCT_OK) return st;
  }
  if (m >= 1 && m <= 3)
    CUDA_TRY(ws_row_of(pl->log2n)->launch[m - 1](a, s, pl->num_sms, pl->counters + k, map));
  else
    CUDA_TRY(table().lp[pl->log2n][m](a, s, pl->num_sms, pl->counters + k, map));
  return NSLCT_OK;
}

// The passes of `nimg` consecutive images starting at image img0 of the plan's batch
// (in/out already offset to image img0; the scratch is offset here).
static nslct_status run_images(nslct_plan_t pl, const void* in, void* out, int64_t img0, int64_t nimg,
                               cudaStream_t s, bool profile) {
  const int ti = (pl->dtype == NSLCT_C64) ? 0 : 1;
  unsigned char* sbase = static_cast<unsigned char*>(pl->scratch);
  void* scratch = sbase ? sbase + (size_t)img0 * (size_t)pl->nl * (size_t)pl->nl * pl->elem : nullptr;
  cudaEvent_t* ev = nullptr;
  if (profile) {
    if (pl->ev_used == pl->ev.size()) {
      nslct_plan_s::EvSet set{};
      for (auto& e : set.e) CUDA_TRY(cudaEventCreate(&e));
      pl->ev.push_back(set);
    }
    ev = pl->ev[pl->ev_used].e;
  }
  if (pl->p.kind == 0) {
    nslct::B0Args b = pl->b0;
    b.in = in;
    b.out = out;
    b.total = nimg * pl->n * pl->n;
    const long long blocks = nimg * pl->n;   // one CTA per output row
    if (in == out) return fail(NSLCT_E_ARG, "the B = 0 gather cannot run in place");
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
    if (ti == 0)
      nslct::b0_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(b);
    else
      nslct::b0_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(b);
    CUDA_TRY(cudaGetLastError());
    if (ev) {
      CUDA_TRY(cudaEventRecord(ev[1], s));
      ++pl->ev_used;
    }
    return NSLCT_OK;
  }
  if (pl->image) {   // F2: every pass in one kernel, the image in shared memory
    nslct::ImgArgs ia;
    ia.in = in;
    ia.out = out;
    ia.tw = pl->tw;
    for (int k = 0; k < 5; ++k) {
      ia.pass[k] = pl->args[k];
      ia.pass[k].n_lines = nimg * pl->n;
      ia.mode[k] = pl->mode[k];
    }
    ia.n_passes = pl->n_passes;
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
    CUDA_TRY(table().li[ti][pl->log2n](ia, s, nimg));
    if (ev) {
      CUDA_TRY(cudaEventRecord(ev[1], s));
      ++pl->ev_used;
    }
    return NSLCT_OK;
  }
  if (pl->p.kind == 3) {   // Ding: two line passes of length 2N, then the affine gather
    const size_t img2 = (size_t)pl->nl * (size_t)pl->nl * pl->elem;
    void* s1 = scratch;
    void* s2 = sbase + (size_t)pl->batch * img2 + (size_t)img0 * img2;
    nslct::BlArgs bl{pl->bq, pl->bhat, (int)pl->nl};
    const void* src = in;
    for (int k = 0; k < 2; ++k) {
      void* dst = (k == 0) ? s1 : s2;
      if (ev) CUDA_TRY(cudaEventRecord(ev[k], s));
      PassArgs a = pl->args[k];
      a.in = src;
      a.out = dst;
      a.n_lines = nimg * pl->nl;
      if (pl->bluestein)
        CUDA_TRY(nslct::bl_launcher(ti, pl->log2n, 0)(a, bl, nimg, s));
      else
        CUDA_TRY(table().l[ti][pl->log2n][0](a, s));
      src = dst;
    }
    nslct::DingArgs d = pl->ding;
    d.in = s2;
    d.out = out;
    d.total = nimg * pl->n * pl->n;
    const long long blocks = (d.total + 255) / 256;
    if (ev) CUDA_TRY(cudaEventRecord(ev[2], s));
    if (ti == 0)
      nslct::ding_gather_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(d);
    else
      nslct::ding_gather_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(d);
    CUDA_TRY(cudaGetLastError());
    if (ev) {
      CUDA_TRY(cudaEventRecord(ev[3], s));
      ++pl->ev_used;
    }
    return NSLCT_OK;
  }
  if (pl->bluestein) {   // arbitrary N: Bluestein line passes (kernels.cuh bl_pass_kernel)
    nslct::BlArgs bl{pl->bq, pl->bhat, (int)pl->n};
    const int np = pl->n_passes;
    const void* src = in;
    for (int k = 0; k < np; ++k) {
      void* dst = (k == np - 1) ? out : ((k % 2 == 0) ? scratch : out);
      if (ev) CUDA_TRY(cudaEventRecord(ev[k], s));
      PassArgs a = pl->args[k];
      a.in = src;
      a.out = dst;
      a.n_lines = nimg * pl->n;
      CUDA_TRY(nslct::bl_launcher(ti, pl->log2n, pl->mode[k])(a, bl, nimg, s));
      src = dst;
    }
    if (ev) {
      CUDA_TRY(cudaEventRecord(ev[np], s));
      ++pl->ev_used;
    }
    return NSLCT_OK;
  }
  if (pl->pipe) CUDA_TRY(cudaMemsetAsync(pl->counters, 0, 5 * sizeof(unsigned long long), s));
  // pass k writes the scratch (k even) or out (k odd); the last pass writes out in place.
  // HA: K1 in->S, K2 S->out, K3 out->S, K4 S->out, K5 out->out; LC-y: in->S, S->out, out->out
  const int np = pl->n_passes;
  const void* src = in;
  for (int k = 0; k < np; ++k) {
    void* dst = (k == np - 1) ? out : ((k % 2 == 0) ? scratch : out);
    if (ev) CUDA_TRY(cudaEventRecord(ev[k], s));
    PassArgs a = pl->args[k];
    a.in = src;
    a.out = dst;
    a.n_lines = nimg * pl->n;
    if (pl->pipe) {
      nslct_status st = launch_pipe_pass(pl, k, a, s);
      if (st != NSLCT_OK) return st;
    } else if (pl->pair || pl->big) {
      nslct_status st = launch_large(pl, k, a, s);
      if (st != NSLCT_OK) return st;
    } else {
      CUDA_TRY(table().l[ti][pl->log2n][pl->mode[k]](a, s));
    }
    src = dst;
  }
  if (ev) {
    CUDA_TRY(cudaEventRecord(ev[np], s));
    ++pl->ev_used;
  }
  return NSLCT_OK;
}

// One launch of pass k with the large-N kernels (batched or slab): the TMA-pipelined
// kernel gets the tensor map of its Q16 input (not for the passes reading user rows).
static nslct_status launch_large(nslct_plan_t pl, int k, const PassArgs& a, cudaStream_t s) {
  const int sl = pl->slab ? 1 : 0, m = pl->mode[k];
  if (!pl->big) {
    CUDA_TRY(table().lpair[sl][pl->log2n][m](a, s));
    return NSLCT_OK;
  }
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (!(m == 0 || m == 4)) {
    const long long L = pl->slab ? pl->L : pl->n;
    const long long C = pl->slab ? a.in_chunk : pl->n;
    const long long images = pl->slab ? 1 : a.n_lines / pl->n;
    nslct_status st = make_q16_map(&map, a.in, pl->log2n, L, C, images);
    if (st != NSLCT_OK) return st;
  }
  CUDA_TRY(table().lbig[sl][pl->log2n][m](a, s, map));
  return NSLCT_OK;
}

// One launch of pass k of a slab plan (the cluster-pair kernels at N = 8192 / 16384 c64,
// else the generic line pass), over local lines a.line_base + [0, a.n_lines).
static nslct_status launch_slab_pass(nslct_plan_t pl, int k, const PassArgs& a, cudaStream_t s) {
  const int ti = (pl->dtype == NSLCT_C64) ? 0 : 1;
  if (pl->pair || pl->big) return launch_large(pl, k, a, s);
  CUDA_TRY(table().l[ti][pl->log2n][pl->mode[k]](a, s));
  return NSLCT_OK;
}

// The whole row-slab transform of a comm plan on stream s (include/nslct.h nslct_exec):
// pass k in nc chunks of lc lines into the send buffer; after chunk c, the NCCL stream
// moves sub-block (q, c) to every rank q (grouped send/recv, NCCL 2.28 over NVLink /
// NVSwitch) while chunk c+1 computes; pass k+1 waits for the whole exchange and reads the
// receive buffer, which alternates between passes (the exchange of pass k+1 writes the
// other one while pass k+1 still reads this one).
static nslct_status run_slab_comm(nslct_plan_t pl, const void* in, void* out, cudaStream_t s, bool profile) {
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(NSLCT_E_NCCL, api.err);
  cudaEvent_t* ev = nullptr;
  if (profile) {
    if (pl->ev_used == pl->ev.size()) {
      nslct_plan_s::EvSet set{};
      for (auto& e : set.e) CUDA_TRY(cudaEventCreate(&e));
      pl->ev.push_back(set);
    }
    ev = pl->ev[pl->ev_used].e;
  }
  const size_t blk = (size_t)pl->L * (size_t)pl->L * pl->elem;   // bytes of one L x L block
  const size_t sub = (size_t)pl->L * (size_t)pl->lc * pl->elem;  // bytes of one sub-block
  unsigned char* send = static_cast<unsigned char*>(pl->xsend);
  const int np = pl->n_passes;
  const void* src = in;
  for (int k = 0; k < np; ++k) {
    if (ev) CUDA_TRY(cudaEventRecord(ev[k], s));
    PassArgs a = pl->args[k];
    a.in = src;
    if (k == np - 1) {   // straight output, rows of this rank's slab
      a.out = out;
      nslct_status st = launch_slab_pass(pl, k, a, s);
      if (st != NSLCT_OK) return st;
      break;
    }
    unsigned char* recv = static_cast<unsigned char*>(pl->xrecv[k & 1]);
    if (pl->exchange == NSLCT_EXCHANGE_PEER) {
      // the store IS the exchange: row-block q of this pass's output lands in rank q's
      // receive buffer k&1 at block offset rank L^2 (kernels.cuh peer_on); then a
      // stream-ordered barrier over all ranks (a 4-byte NCCL all-reduce): every rank's pass
      // k stores are complete before any rank's pass k+1 reads them, and every rank has
      // finished reading buffer (k+1)&1 (its pass k input) before pass k+1 overwrites it.
      a.out = pl->peer_recv[k & 1][pl->rank];
      a.peer_on = 1;
      a.peer_rank = pl->rank;
      for (int q = 0; q < pl->nranks; ++q) a.peer_out[q] = pl->peer_recv[k & 1][q];
      nslct_status st = launch_slab_pass(pl, k, a, s);
      if (st != NSLCT_OK) return st;
      const ncclResult_t r = api.AllReduce(pl->xbar, pl->xbar, 1, ncclInt32, ncclSum, pl->comm->c, s);
      if (r != ncclSuccess) return fail(NSLCT_E_NCCL, std::string("barrier (ncclAllReduce): ") + api.GetErrorString(r));
      src = recv;
      continue;
    }
    a.out = send;
    for (int c = 0; c < pl->nc; ++c) {
      PassArgs ac = a;
      ac.line_base = (int)(c * pl->lc);
      ac.n_lines = pl->lc;
      nslct_status st = launch_slab_pass(pl, k, ac, s);
      if (st != NSLCT_OK) return st;
      CUDA_TRY(cudaEventRecord(pl->xev[c], s));
      CUDA_TRY(cudaStreamWaitEvent(pl->cs_comm, pl->xev[c], 0));
      ncclResult_t r = api.GroupStart();
      for (int q = 0; q < pl->nranks && r == ncclSuccess; ++q) {
        const size_t off = (size_t)q * blk + (size_t)c * sub;
        r = api.Send(send + off, sub, ncclInt8, q, pl->comm->c, pl->cs_comm);
        if (r == ncclSuccess) r = api.Recv(recv + off, sub, ncclInt8, q, pl->comm->c, pl->cs_comm);
      }
      const ncclResult_t r2 = api.GroupEnd();   // always close the group
      if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(NSLCT_E_NCCL, std::string("slab all-to-all (grouped ncclSend/ncclRecv): ") +
                                      api.GetErrorString(r != ncclSuccess ? r : r2));
    }
    CUDA_TRY(cudaEventRecord(pl->xev[pl->nc], pl->cs_comm));
    CUDA_TRY(cudaStreamWaitEvent(s, pl->xev[pl->nc], 0));
    src = recv;
  }
  if (ev) {
    CUDA_TRY(cudaEventRecord(ev[np], s));
    ++pl->ev_used;
  }
  return NSLCT_OK;
}

nslct_status nslct_exec(nslct_plan_t pl, const void* in, void* out, void* stream) {
  if (!pl) return fail(NSLCT_E_ARG, "null plan");
  if (!in || !out) return fail(NSLCT_E_ARG, "null in/out pointer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(NSLCT_E_ARG, "in/out must be 16-byte aligned");
  if (pl->slab && !pl->comm)
    return fail(NSLCT_E_ARG, "nslct_plan_slab plans run pass by pass (nslct_exec_pass); comm plans run here");
  if (pl->n_in != pl->n && in == out) return fail(NSLCT_E_ARG, "a padded plan cannot run in place");
  GUARD_DEVICE(pl);
  if (pl->comm) return run_slab_comm(pl, in, out, reinterpret_cast<cudaStream_t>(stream), pl->profile != 0);
  return run_images(pl, in, out, 0, pl->batch, reinterpret_cast<cudaStream_t>(stream),
                    pl->profile != 0);
}

nslct_status nslct_exec_pass(nslct_plan_t pl, int pass, const void* in, void* out, void* stream) {
  if (!pl) return fail(NSLCT_E_ARG, "null plan");
  if (!in || !out) return fail(NSLCT_E_ARG, "null in/out pointer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(NSLCT_E_ARG, "in/out must be 16-byte aligned");
  if (pl->p.kind == 0) return fail(NSLCT_E_ARG, "the B = 0 plan has a single pass: use nslct_exec");
  if (pl->p.kind == 3) return fail(NSLCT_E_ARG, "Ding plans run through nslct_exec");
  if (pass < 0 || pass >= pl->n_passes) return fail(NSLCT_E_ARG, "pass out of range");
  if (pass < pl->n_passes - 1 && in == out) return fail(NSLCT_E_ARG, "transposing passes cannot run in place");
  GUARD_DEVICE(pl);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int ti = (pl->dtype == NSLCT_C64) ? 0 : 1;
  PassArgs a = pl->args[pass];
  a.in = in;
  a.out = out;
  if (pl->bluestein) {
    nslct::BlArgs bl{pl->bq, pl->bhat, (int)pl->n};
    CUDA_TRY(nslct::bl_launcher(ti, pl->log2n, pl->mode[pass])(a, bl, pl->batch, s));
  } else if (pl->pipe) {
    CUDA_TRY(cudaMemsetAsync(pl->counters + pass, 0, sizeof(unsigned long long), s));
    nslct_status st = launch_pipe_pass(pl, pass, a, s);
    if (st != NSLCT_OK) return st;
  } else if (pl->pair || pl->big) {
    return launch_large(pl, pass, a, s);
  } else {
    CUDA_TRY(table().l[ti][pl->log2n][pl->mode[pass]](a, s));
  }
  return NSLCT_OK;
}

// ---- communicator -------------------------------------------------------------------
nslct_status nslct_comm_unique_id(uint8_t unique_id[128]) {
  if (!unique_id) return fail(NSLCT_E_ARG, "null pointer");
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(NSLCT_E_NCCL, api.err);
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId id;
  NCCL_TRY(api.GetUniqueId(&id));
  std::memcpy(unique_id, &id, 128);
  return NSLCT_OK;
}

nslct_status nslct_comm_init(nslct_comm_t* comm, const uint8_t unique_id[128], int rank, int nranks) {
  if (!comm || !unique_id) return fail(NSLCT_E_ARG, "null pointer");
  *comm = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NSLCT_E_ARG, "bad rank / nranks");
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(NSLCT_E_NCCL, api.err);
  nslct_comm_s* c = new (std::nothrow) nslct_comm_s();
  if (!c) return fail(NSLCT_E_OOM, "host allocation failed");
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) {
    delete c;
    return fail(NSLCT_E_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, 128);
  const ncclResult_t r = api.CommInitRank(&c->c, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(NSLCT_E_NCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
  }
  c->rank = rank;
  c->nranks = nranks;
  *comm = c;
  return NSLCT_OK;
}

nslct_status nslct_comm_info(nslct_comm_t comm, int* rank, int* nranks) {
  if (!comm) return fail(NSLCT_E_ARG, "null communicator");
  if (rank) *rank = comm->rank;
  if (nranks) *nranks = comm->nranks;
  return NSLCT_OK;
}

nslct_status nslct_comm_destroy(nslct_comm_t comm) {
  if (!comm) return NSLCT_OK;
  const NcclApi& api = nccl_api();
  ncclResult_t r = ncclSuccess;
  if (api.ok && comm->c) r = api.CommDestroy(comm->c);
  delete comm;
  if (r != ncclSuccess) return fail(NSLCT_E_NCCL, std::string("ncclCommDestroy: ") + api.GetErrorString(r));
  return NSLCT_OK;
}

// Images per exec_host chunk: about 64 MiB per copy (opts.host_chunk_kb overrides), so
// the H2D of chunk i+1, the passes of chunk i and the D2H of chunk i-1 overlap.
static int64_t host_chunk_images(const nslct_plan_s* pl) {
  const double img = (double)pl->n * (double)pl->n * (double)pl->elem;
  // at most 64 MiB per chunk, and at least ~8 chunks when the batch allows it, so small
  // batches still overlap their copies with the passes
  double mb = std::min(64.0, img * (double)pl->batch / 8.0 / 1048576.0);
  if (pl->host_chunk_kb > 0) mb = (double)pl->host_chunk_kb / 1024.0;
  int64_t c = (int64_t)(mb * 1048576.0 / img);
  if (c < 1) c = 1;
  if (c > pl->batch) c = pl->batch;
  return c;
}

nslct_status nslct_exec_pass_peer(nslct_plan_t pl, int pass, const void* in, void* const* peer_out, int n_peers,
                                  void* stream) {
  if (!pl) return fail(NSLCT_E_ARG, "null plan");
  if (!pl->slab) return fail(NSLCT_E_ARG, "peer-store passes exist for row-slab plans only");
  if (!in || !peer_out) return fail(NSLCT_E_ARG, "null pointer");
  if (n_peers != pl->nranks || n_peers > 8) return fail(NSLCT_E_ARG, "n_peers must equal nranks (<= 8)");
  if (pass < 0 || pass >= pl->n_passes - 1)
    return fail(NSLCT_E_ARG, "only the transposing passes (0 .. n_passes-2) exchange");
  for (int s = 0; s < n_peers; ++s)
    if (!peer_out[s] || (reinterpret_cast<uintptr_t>(peer_out[s]) & 15))
      return fail(NSLCT_E_ARG, "peer buffers must be non-null and 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(in) & 15) return fail(NSLCT_E_ARG, "in must be 16-byte aligned");
  GUARD_DEVICE(pl);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int ti = (pl->dtype == NSLCT_C64) ? 0 : 1;
  PassArgs a = pl->args[pass];
  a.in = in;
  a.out = peer_out[pl->rank];
  a.peer_on = 1;
  a.peer_rank = pl->rank;
  for (int r = 0; r < n_peers; ++r) a.peer_out[r] = peer_out[r];
  if (pl->pair || pl->big) return launch_large(pl, pass, a, s);
  CUDA_TRY(table().l[ti][pl->log2n][pl->mode[pass]](a, s));
  return NSLCT_OK;
}

nslct_status nslct_exec_host(nslct_plan_t pl, const void* host_in, void* host_out, void* stream) {
  if (!pl) return fail(NSLCT_E_ARG, "null plan");
  if (pl->slab) return fail(NSLCT_E_ARG, "slab plans run pass by pass: nslct_exec_pass");
  if (!host_in || !host_out) return fail(NSLCT_E_ARG, "null host pointer");
  if (pl->n_in != pl->n) {
    // output chunks are larger than input chunks: chunk i's device->host copy could
    // overwrite input bytes of a later chunk not yet uploaded
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(host_in), o0 = reinterpret_cast<uintptr_t>(host_out);
    const uintptr_t i1 = i0 + pl->in_img_bytes * (size_t)pl->batch, o1 = o0 + pl->bytes;
    if (i0 < o1 && o0 < i1) return fail(NSLCT_E_ARG, "a zero-padding plan needs disjoint host_in / host_out");
  }
  GUARD_DEVICE(pl);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!pl->h_in) CUDA_TRY(cudaMalloc(&pl->h_in, pl->in_img_bytes * (size_t)pl->batch));
  if (!pl->h_out) CUDA_TRY(cudaMalloc(&pl->h_out, pl->bytes));
  if (!pl->cs_in) CUDA_TRY(cudaStreamCreateWithFlags(&pl->cs_in, cudaStreamNonBlocking));
  if (!pl->cs_out) CUDA_TRY(cudaStreamCreateWithFlags(&pl->cs_out, cudaStreamNonBlocking));
  const int64_t c = host_chunk_images(pl);
  const int64_t nch = (pl->batch + c - 1) / c;
  while ((int64_t)pl->cev.size() < 2 * nch + 1) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pl->cev.push_back(e);
  }
  const size_t img_bytes = (size_t)pl->n * (size_t)pl->n * pl->elem;
  // copies start after whatever the caller queued on `stream` before this call
  CUDA_TRY(cudaEventRecord(pl->cev[2 * nch], s));
  CUDA_TRY(cudaStreamWaitEvent(pl->cs_in, pl->cev[2 * nch], 0));
  for (int64_t i = 0; i < nch; ++i) {
    const int64_t i0 = i * c, ni = (i0 + c <= pl->batch) ? c : pl->batch - i0;
    const size_t off = (size_t)i0 * img_bytes, len = (size_t)ni * img_bytes;
    const size_t off_in = (size_t)i0 * pl->in_img_bytes, len_in = (size_t)ni * pl->in_img_bytes;
    unsigned char* din = static_cast<unsigned char*>(pl->h_in) + off_in;
    unsigned char* dout = static_cast<unsigned char*>(pl->h_out) + off;
    CUDA_TRY(cudaMemcpyAsync(din, static_cast<const unsigned char*>(host_in) + off_in, len_in,
                             cudaMemcpyHostToDevice, pl->cs_in));
    CUDA_TRY(cudaEventRecord(pl->cev[2 * i], pl->cs_in));
    CUDA_TRY(cudaStreamWaitEvent(s, pl->cev[2 * i], 0));
    nslct_status st = run_images(pl, din, dout, i0, ni, s, false);
    if (st != NSLCT_OK) return st;
    CUDA_TRY(cudaEventRecord(pl->cev[2 * i + 1], s));
    CUDA_TRY(cudaStreamWaitEvent(pl->cs_out, pl->cev[2 * i + 1], 0));
    CUDA_TRY(cudaMemcpyAsync(static_cast<unsigned char*>(host_out) + off, dout, len, cudaMemcpyDeviceToHost,
                             pl->cs_out));
  }
  CUDA_TRY(cudaStreamSynchronize(pl->cs_out));
  CUDA_TRY(cudaStreamSynchronize(s));
  return NSLCT_OK;
}

static void describe(const nslct::Plan& p, double dx, nslct_plan_desc* d) {
  std::memset(d, 0, sizeof(*d));
  d->kind = p.kind;
  d->variant = p.variant;
  d->lc_axis = p.lc_axis;
  d->n_passes = (p.kind == 0) ? 1 : (p.kind == 3 || lc_y(p)) ? 3 : 5;
  auto put = [](double* o, const nslct::Sym& s) {
    o[0] = s.q11;
    o[1] = s.q22;
    o[2] = s.q12;
  };
  put(d->H, p.H);
  put(d->Bp, p.Bp);
  put(d->P2, p.P2);
  put(d->P4, p.P4);
  for (int i = 0; i < 5; ++i) {
    if (p.kind != 0 && (i % 2 == 1 || p.q_active[i])) put(d->Q[i], p.Q[i]);
  }
  d->dx = dx;
  d->objective = p.objective;
  d->sym_residual = p.sym_residual;
  d->recomposition_residual = p.recomposition_residual;
  d->dispatch_key = p.key;
}

nslct_status nslct_plan_info(nslct_plan_t pl, nslct_plan_desc* d) {
  if (!pl || !d) return fail(NSLCT_E_ARG, "null pointer");
  describe(pl->p, pl->dx, d);
  if (pl->p.kind != 0) d->n_passes = pl->n_passes;
  d->on_chip = (pl->p.kind != 0 && pl->image) ? 1 : 0;
  d->n_launches = (pl->p.kind == 0 || pl->image) ? 1 : pl->n_passes;
  d->fft_len = (pl->p.kind == 0) ? 0 : (1 << pl->log2n);
  d->n_in = (int)pl->n_in;
  return NSLCT_OK;
}

nslct_status nslct_plan_describe(int64_t n, const double abcd[16], const nslct_opts* opts,
                                 nslct_plan_desc* d) {
  g_err.clear();
  if (!abcd || !d) return fail(NSLCT_E_ARG, "null pointer");
  nslct_opts o;
  if (opts)
    o = *opts;
  else
    nslct_opts_default(&o);
  if (n < 2) return fail(NSLCT_E_ARG, "n must be >= 2");
  if (o.variant < 0 || o.variant > 3 || o.dispatch < 0 || o.dispatch > 1 || o.schedule < 0 || o.schedule > 2)
    return fail(NSLCT_E_ARG, "bad variant/dispatch option");
  std::string err;
  nslct::Plan p;
  int st = nslct::make_plan(abcd, o.variant, o.dispatch, o.h_fixed, &p, &err);
  if (st) return fail((nslct_status)st, err);
  describe(p, (o.dx > 0) ? o.dx : std::sqrt(2.0 * M_PI / (double)n), d);
  return NSLCT_OK;
}

nslct_status nslct_pass_ms(nslct_plan_t pl, float* ms, int capacity, int* n_written) {
  if (!pl || !ms) return fail(NSLCT_E_ARG, "null pointer");
  if (!pl->profile || pl->ev_used == 0) return fail(NSLCT_E_ARG, "plan not profiled / no exec yet");
  GUARD_DEVICE(pl);
  const int np = (pl->p.kind == 0 || pl->image) ? 1 : pl->n_passes;
  if (capacity < np) return fail(NSLCT_E_ARG, "capacity too small");
  for (int k = 0; k < np; ++k) ms[k] = 0.0f;
  for (size_t i = 0; i < pl->ev_used; ++i) {
    cudaEvent_t* e = pl->ev[i].e;
    CUDA_TRY(cudaEventSynchronize(e[np]));
    for (int k = 0; k < np; ++k) {
      float t = 0.0f;
      CUDA_TRY(cudaEventElapsedTime(&t, e[k], e[k + 1]));
      ms[k] += t;
    }
  }
  for (int k = 0; k < np; ++k) ms[k] /= (float)pl->ev_used;
  pl->ev_used = 0;
  if (n_written) *n_written = np;
  return NSLCT_OK;
}

nslct_status nslct_inverse_matrix(const double abcd[16], double out[16]) {
  if (!abcd || !out) return fail(NSLCT_E_ARG, "null pointer");
  // Eq. CCCMCCCM20: (A, B; C, D)^-1 = (D^T, -B^T; -C^T, A^T); row-major
  // 4x4, block (r, c) of M at rows 2r.., columns 2c..
  double m[16];
  std::memcpy(m, abcd, sizeof(m));
  auto at = [&](int br, int bc, int i, int k) { return m[(2 * br + i) * 4 + 2 * bc + k]; };
  for (int i = 0; i < 2; ++i)
    for (int k = 0; k < 2; ++k) {
      out[i * 4 + k] = at(1, 1, k, i);                  // D^T
      out[i * 4 + 2 + k] = -at(0, 1, k, i);             // -B^T
      out[(2 + i) * 4 + k] = -at(1, 0, k, i);           // -C^T
      out[(2 + i) * 4 + 2 + k] = at(0, 0, k, i);        // A^T
    }
  return NSLCT_OK;
}

// ---- FP32 roofline calibration --------------------------------------------------------
// 16 independent FFMA chains per thread, 2048 threads per SM: the FMA pipe's issue-bound
// rate (SURVEY.md §8(d) asks for the measured FP32 ceiling next to the HBM one).
}  // extern "C"
namespace {
__global__ void __launch_bounds__(1024) fp32_peak_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (float)(threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 1.2345f) out[blockIdx.x] = s;   // never true for the launch below; keeps the work
}
}  // namespace
extern "C" {

nslct_status nslct_fp32_peak(int device, double* tflops) {
  if (!tflops) return fail(NSLCT_E_ARG, "null pointer");
  DeviceGuard guard(device);
  if (guard.status != cudaSuccess) return fail(NSLCT_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(guard.status));
  int sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  float* out = nullptr;
  CUDA_TRY(cudaMalloc(&out, (size_t)sms * 2 * sizeof(float)));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  const int iters = 1 << 16;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, 0);
    fp32_peak_kernel<<<sms * 2, 1024>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1, 0);
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * 16.0 * iters * (double)sms * 2.0 * 1024.0;
    if (rep > 0 && ms > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  CUDA_TRY(cudaGetLastError());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *tflops = best;
  return NSLCT_OK;
}

nslct_status nslct_destroy(nslct_plan_t pl) {
  free_plan(pl);
  return NSLCT_OK;
}

}  // extern "C"
