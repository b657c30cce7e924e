// Arbitrary-N line passes: kernels.cuh bl_pass_kernel instantiated
// for M = 2^5 .. 2^13, the four modes of the 5-pass schedule, complex64 and complex128.
#include "bluestein.h"

namespace nslct {
namespace {

template <typename T, int LOG2M, int MODE>
cudaError_t launch_bl(const PassArgs& a, const BlArgs& b, long long batch, cudaStream_t s) {
  using Cfg = LineCfg<LOG2M>;
  const size_t smem = (size_t)Cfg::G * Cfg::LS * sizeof(cpx<T>);
  const long long grid = batch * ((b.n + Cfg::G - 1) / Cfg::G);
  bl_pass_kernel<T, LOG2M, MODE><<<(unsigned)grid, Cfg::THREADS, smem, s>>>(a, b);
  return cudaGetLastError();
}
template <typename T, int LOG2M, int MODE>
cudaError_t attr_bl() {
  using Cfg = LineCfg<LOG2M>;
  const size_t smem = (size_t)Cfg::G * Cfg::LS * sizeof(cpx<T>);
  return cudaFuncSetAttribute(bl_pass_kernel<T, LOG2M, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem);
}

struct BlTable {
  bl_launch_fn l[2][kBlMaxLog + 1][4] = {};
  bl_attr_fn at[2][kBlMaxLog + 1][4] = {};
  template <typename T, int LOG2M>
  void row(int ti) {
    l[ti][LOG2M][0] = launch_bl<T, LOG2M, 0>;
    l[ti][LOG2M][1] = launch_bl<T, LOG2M, 1>;
    l[ti][LOG2M][2] = launch_bl<T, LOG2M, 2>;
    l[ti][LOG2M][3] = launch_bl<T, LOG2M, 3>;
    at[ti][LOG2M][0] = attr_bl<T, LOG2M, 0>;
    at[ti][LOG2M][1] = attr_bl<T, LOG2M, 1>;
    at[ti][LOG2M][2] = attr_bl<T, LOG2M, 2>;
    at[ti][LOG2M][3] = attr_bl<T, LOG2M, 3>;
  }
  template <int LOG2M>
  void both() {
    row<float, LOG2M>(0);
    row<double, LOG2M>(1);
    if constexpr (LOG2M < kBlMaxLog) both<LOG2M + 1>();
  }
  BlTable() { both<kBlMinLog>(); }
};
const BlTable& bl_table() {
  static BlTable t;
  return t;
}

}  // namespace

bl_launch_fn bl_launcher(int ti, int log2m, int mode) {
  if (ti < 0 || ti > 1 || log2m < kBlMinLog || log2m > kBlMaxLog || mode < 0 || mode > 3) return nullptr;
  return bl_table().l[ti][log2m][mode];
}
bl_attr_fn bl_attr(int ti, int log2m, int mode) {
  if (ti < 0 || ti > 1 || log2m < kBlMinLog || log2m > kBlMaxLog || mode < 0 || mode > 3) return nullptr;
  return bl_table().at[ti][log2m][mode];
}

}  // namespace nslct
