// Transforms: cuFFT plan cache, half/full spectrum plumbing, residue guard.
// Replaces transforms.py:82-211 (numpy pocketfft) of the reference.
#include <cufft.h>
#include <math_constants.h>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "transforms.cuh"

namespace ocsc {

// ------------------------------------------------------------ plan cache --
namespace {
using PlanKey = std::tuple<int, int, int, int, int, int, int64_t>;  // dev, kind, dtype, H, W, batch, stride
std::map<PlanKey, cufftHandle>& plans() {
  static std::map<PlanKey, cufftHandle> m;
  return m;
}
std::mutex& plan_mu() {
  static std::mutex m;
  return m;
}

int cufft_fail(cufftResult r, const char* where) {
  return fail(OCSC_ECUDA, std::string("cuFFT error ") + std::to_string((int)r) + " in " + where);
}
}  // namespace

// kind: 0 = R2C, 1 = C2R, 2 = C2C planes contiguous, 3 = C2C on (P, batch) columns
int get_plan(int kind, int dtype, int H, int W, int batch, cufftHandle* out) {
  int dev = 0;
  OCSC_CUDA(cudaGetDevice(&dev));
  PlanKey key{dev, kind, dtype, H, W, batch, 0};
  std::lock_guard<std::mutex> lk(plan_mu());
  auto it = plans().find(key);
  if (it != plans().end()) {
    *out = it->second;
    return OCSC_OK;
  }
  cufftHandle h;
  cufftResult r = cufftCreate(&h);
  if (r != CUFFT_SUCCESS) return cufft_fail(r, "cufftCreate");
  const bool dbl = dtype == OCSC_F64;
  cufftType type;
  if (kind == 0) type = dbl ? CUFFT_D2Z : CUFFT_R2C;
  else if (kind == 1) type = dbl ? CUFFT_Z2D : CUFFT_C2R;
  else type = dbl ? CUFFT_Z2Z : CUFFT_C2C;
  int rank = H == 1 ? 1 : 2;
  int n2[2] = {H, W};
  int* n = H == 1 ? n2 + 1 : n2;
  size_t ws = 0;
  if (kind == 3) {
    // reference columns: element (pixel q, column k) at q*batch + k
    int emb2[2] = {H, W};
    int* emb = H == 1 ? emb2 + 1 : emb2;
    r = cufftMakePlanMany(h, rank, n, emb, batch, 1, emb, batch, 1, type, batch, &ws);
  } else {
    r = cufftMakePlanMany(h, rank, n, nullptr, 1, 0, nullptr, 1, 0, type, batch, &ws);
  }
  if (r != CUFFT_SUCCESS) {
    cufftDestroy(h);
    return cufft_fail(r, "cufftMakePlanMany");
  }
  plans()[key] = h;
  *out = h;
  return OCSC_OK;
}

int exec_r2c(int dtype, int H, int W, int nplanes, const void* x, void* xh, cudaStream_t s) {
  if (nplanes == 0) return OCSC_OK;
  cufftHandle h;
  int rc = get_plan(0, dtype, H, W, nplanes, &h);
  if (rc) return rc;
  cufftSetStream(h, s);
  cufftResult r = dtype == OCSC_F64
                      ? cufftExecD2Z(h, (cufftDoubleReal*)x, (cufftDoubleComplex*)xh)
                      : cufftExecR2C(h, (cufftReal*)x, (cufftComplex*)xh);
  return r == CUFFT_SUCCESS ? OCSC_OK : cufft_fail(r, "exec R2C");
}

int exec_c2r(int dtype, int H, int W, int nplanes, void* xh, void* x, cudaStream_t s) {
  if (nplanes == 0) return OCSC_OK;
  cufftHandle h;
  int rc = get_plan(1, dtype, H, W, nplanes, &h);
  if (rc) return rc;
  cufftSetStream(h, s);
  cufftResult r = dtype == OCSC_F64
                      ? cufftExecZ2D(h, (cufftDoubleComplex*)xh, (cufftDoubleReal*)x)
                      : cufftExecC2R(h, (cufftComplex*)xh, (cufftReal*)x);
  return r == CUFFT_SUCCESS ? OCSC_OK : cufft_fail(r, "exec C2R");
}

// ---------------------------------------------------------------- kernels --
template <typename T>
__global__ void k_scale(int64_t n, T* x, T s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= s;
}

template <typename T>
__global__ void k_widen(int64_t n, const T* in, cx<T>* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mkc<cx<T>>(in[i], (T)0);
}

template <typename T>
__global__ void k_residue(int64_t n, const cx<T>* sp, const cx<T>* spec, double* stats) {
  double a = 0.0, b = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    a = fmax(a, fabs((double)sp[i].y));
    cx<T> v = spec[i];
    b = fmax(b, sqrt((double)v.x * v.x + (double)v.y * v.y));
    if (isnan((double)sp[i].y)) a = CUDART_INF;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(stats, a);
    atomic_max_nonneg(stats + 1, b);
  }
}

template <typename T>
__global__ void k_real_part(int64_t n, const cx<T>* in, T scale, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i].x * scale;
}

// half (nplanes, H, Wh) -> full columns (P, nplanes)
template <typename T>
__global__ void k_half_to_cols(int H, int W, int nplanes, const cx<T>* half, cx<T>* cols) {
  const int Wh = W / 2 + 1;
  const int64_t total = (int64_t)H * W * nplanes;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int k = (int)(i % nplanes);
    int64_t q = i / nplanes;
    int v = (int)(q % W), u = (int)(q / W);
    cx<T> val;
    if (v < Wh) {
      val = half[((int64_t)k * H + u) * Wh + v];
    } else {
      int uu = (H - u) % H, vv = W - v;
      val = cconj(half[((int64_t)k * H + uu) * Wh + vv]);
    }
    cols[i] = val;
  }
}

template <typename T>
__global__ void k_cols_to_half(int H, int W, int ncols, const cx<T>* cols, cx<T>* half) {
  const int Wh = W / 2 + 1;
  const int64_t total = (int64_t)ncols * H * Wh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int v = (int)(i % Wh);
    int64_t r = i / Wh;
    int u = (int)(r % H);
    int k = (int)(r / H);
    half[i] = cols[((int64_t)u * W + v) * ncols + k];
  }
}

template <typename T>
__global__ void k_herm_defect(int H, int W, int ncols, const cx<T>* cols, double* stats) {
  const int64_t total = (int64_t)H * W * ncols;
  double a = 0.0, b = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int k = (int)(i % ncols);
    int64_t q = i / ncols;
    int v = (int)(q % W), u = (int)(q / W);
    int uu = (H - u) % H, vv = (W - v) % W;
    cx<T> x = cols[i], y = cols[((int64_t)uu * W + vv) * ncols + k];
    double dx = (double)x.x - y.x, dy = (double)x.y + y.y;
    a = fmax(a, sqrt(dx * dx + dy * dy));
    b = fmax(b, sqrt((double)x.x * x.x + (double)x.y * x.y));
    if (isnan(dx) || isnan(dy)) a = CUDART_INF;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(stats, a);
    atomic_max_nonneg(stats + 1, b);
  }
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  return g < 1 ? 1 : (int)g;
}

}  // namespace ocsc

using namespace ocsc;

#define DISPATCH(dtype, CALL_F, CALL_D)                      \
  do {                                                       \
    if ((dtype) == OCSC_F32) { CALL_F; }                     \
    else if ((dtype) == OCSC_F64) { CALL_D; }                \
    else return fail(OCSC_EARG, "dtype must be 4 or 8");     \
  } while (0)

extern "C" int ocsc_fft_prepare(int dtype, int H, int W, int nplanes) {
  if (H <= 0 || W <= 0 || nplanes <= 0) return fail(OCSC_ESHAPE, "fft_prepare: bad extents");
  if (dtype != OCSC_F32 && dtype != OCSC_F64) return fail(OCSC_EARG, "dtype must be 4 or 8");
  cufftHandle h;
  int rc = get_plan(0, dtype, H, W, nplanes, &h);
  return rc ? rc : get_plan(1, dtype, H, W, nplanes, &h);
}

extern "C" int ocsc_rfft2(int dtype, int H, int W, int nplanes, const void* x, void* xh, void* stream) {
  if (H <= 0 || W <= 0 || nplanes < 0) return fail(OCSC_ESHAPE, "rfft2: bad extents");
  if (dtype != OCSC_F32 && dtype != OCSC_F64) return fail(OCSC_EARG, "dtype must be 4 or 8");
  return exec_r2c(dtype, H, W, nplanes, x, xh, as_stream(stream));
}

extern "C" int ocsc_irfft2(int dtype, int H, int W, int nplanes, void* xh, void* x, void* stream) {
  if (H <= 0 || W <= 0 || nplanes < 0) return fail(OCSC_ESHAPE, "irfft2: bad extents");
  if (dtype != OCSC_F32 && dtype != OCSC_F64) return fail(OCSC_EARG, "dtype must be 4 or 8");
  cudaStream_t s = as_stream(stream);
  int rc = exec_c2r(dtype, H, W, nplanes, xh, x, s);
  if (rc) return rc;
  int64_t n = (int64_t)nplanes * H * W;
  if (n == 0) return OCSC_OK;
  DISPATCH(dtype, (k_scale<float><<<grid_for(n, 256), 256, 0, s>>>(n, (float*)x, 1.0f / (float)(H * W))),
           (k_scale<double><<<grid_for(n, 256), 256, 0, s>>>(n, (double*)x, 1.0 / (double)(H * W))));
  OCSC_LAUNCHED("k_scale");
  return OCSC_OK;
}

extern "C" int ocsc_dft_cols(int dtype, int H, int W, int ncols, const void* in, int in_complex,
                             void* out, int inverse, void* stream) {
  if (H <= 0 || W <= 0 || ncols < 0) return fail(OCSC_ESHAPE, "dft_cols: bad extents");
  if (ncols == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  int64_t n = (int64_t)H * W * ncols;
  const void* src = in;
  if (!in_complex) {
    DISPATCH(dtype, (k_widen<float><<<grid_for(n, 256), 256, 0, s>>>(n, (const float*)in, (float2*)out)),
             (k_widen<double><<<grid_for(n, 256), 256, 0, s>>>(n, (const double*)in, (double2*)out)));
    OCSC_LAUNCHED("k_widen");
    src = out;
  }
  cufftHandle h;
  int rc = get_plan(3, dtype, H, W, ncols, &h);
  if (rc) return rc;
  cufftSetStream(h, s);
  int dir = inverse ? CUFFT_INVERSE : CUFFT_FORWARD;
  cufftResult r = dtype == OCSC_F64
                      ? cufftExecZ2Z(h, (cufftDoubleComplex*)src, (cufftDoubleComplex*)out, dir)
                      : cufftExecC2C(h, (cufftComplex*)src, (cufftComplex*)out, dir);
  return r == CUFFT_SUCCESS ? OCSC_OK : cufft_fail(r, "exec C2C cols");
}

extern "C" int ocsc_residue_stats(int dtype, int64_t n, const void* spatial, const void* spec,
                                  double* stats, void* stream) {
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  DISPATCH(dtype,
           (k_residue<float><<<grid_for(n, 256), 256, 0, s>>>(n, (const float2*)spatial, (const float2*)spec, stats)),
           (k_residue<double><<<grid_for(n, 256), 256, 0, s>>>(n, (const double2*)spatial, (const double2*)spec, stats)));
  OCSC_LAUNCHED("k_residue");
  return OCSC_OK;
}

extern "C" int ocsc_real_part(int dtype, int64_t n, const void* in, double scale, void* out, void* stream) {
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  DISPATCH(dtype,
           (k_real_part<float><<<grid_for(n, 256), 256, 0, s>>>(n, (const float2*)in, (float)scale, (float*)out)),
           (k_real_part<double><<<grid_for(n, 256), 256, 0, s>>>(n, (const double2*)in, scale, (double*)out)));
  OCSC_LAUNCHED("k_real_part");
  return OCSC_OK;
}

extern "C" int ocsc_half_to_cols(int dtype, int H, int W, int nplanes, const void* half, void* cols, void* stream) {
  int64_t n = (int64_t)H * W * nplanes;
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  DISPATCH(dtype,
           (k_half_to_cols<float><<<grid_for(n, 256), 256, 0, s>>>(H, W, nplanes, (const float2*)half, (float2*)cols)),
           (k_half_to_cols<double><<<grid_for(n, 256), 256, 0, s>>>(H, W, nplanes, (const double2*)half, (double2*)cols)));
  OCSC_LAUNCHED("k_half_to_cols");
  return OCSC_OK;
}

extern "C" int ocsc_cols_to_half(int dtype, int H, int W, int ncols, const void* cols, void* half, void* stream) {
  int64_t n = (int64_t)H * (W / 2 + 1) * ncols;
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  DISPATCH(dtype,
           (k_cols_to_half<float><<<grid_for(n, 256), 256, 0, s>>>(H, W, ncols, (const float2*)cols, (float2*)half)),
           (k_cols_to_half<double><<<grid_for(n, 256), 256, 0, s>>>(H, W, ncols, (const double2*)cols, (double2*)half)));
  OCSC_LAUNCHED("k_cols_to_half");
  return OCSC_OK;
}

extern "C" int ocsc_hermitian_defect(int dtype, int H, int W, int ncols, const void* cols, double* stats,
                                     void* stream) {
  int64_t n = (int64_t)H * W * ncols;
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  DISPATCH(dtype,
           (k_herm_defect<float><<<grid_for(n, 256), 256, 0, s>>>(H, W, ncols, (const float2*)cols, stats)),
           (k_herm_defect<double><<<grid_for(n, 256), 256, 0, s>>>(H, W, ncols, (const double2*)cols, stats)));
  OCSC_LAUNCHED("k_herm_defect");
  return OCSC_OK;
}
