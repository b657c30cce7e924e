// Launchers of the arbitrary-N (Bluestein) line passes, compiled in their own
// translation unit (bluestein.cu) so the two kernel families build in parallel.
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace nslct {
constexpr int kBlMinLog = 5, kBlMaxLog = 13;   // FFT length M = 2^LOG2M per line: N <= 4096
typedef cudaError_t (*bl_launch_fn)(const PassArgs&, const BlArgs&, long long batch, cudaStream_t);
typedef cudaError_t (*bl_attr_fn)();
// ti: 0 = complex64, 1 = complex128; mode: pass_body modes 0..3 (the 5-pass schedule)
bl_launch_fn bl_launcher(int ti, int log2m, int mode);
bl_attr_fn bl_attr(int ti, int log2m, int mode);
}  // namespace nslct
