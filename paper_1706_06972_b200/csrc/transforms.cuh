// Internal (C++) interface of transforms.cu shared by the other translation units.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

namespace ocsc {
int get_plan(int kind, int dtype, int H, int W, int batch, cufftHandle* out);
int exec_r2c(int dtype, int H, int W, int nplanes, const void* x, void* xh, cudaStream_t s);
int exec_c2r(int dtype, int H, int W, int nplanes, void* xh, void* x, cudaStream_t s);
int grid_for(int64_t n, int threads);
}  // namespace ocsc
