// Shared device helpers for libocsc_b200 (sm_100a).
//
// Complex values are float2 / double2 (interleaved re, im) -- the layout
// cuFFT and torch.complex64/complex128 use, so spectra cross the C-ABI as
// plain pointers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/ocsc_b200.h"

namespace ocsc {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
void count_launches(int n);  // kernels of this library enqueued (ocsc_kernel_launches)

#define OCSC_CUDA(call)                                   \
  do {                                                    \
    cudaError_t e__ = (call);                             \
    if (e__ != cudaSuccess) return ::ocsc::cuda_fail(e__, #call); \
  } while (0)

#define OCSC_LAUNCHED(name)                                              \
  do {                                                                   \
    ::ocsc::count_launches(1);                                           \
    cudaError_t e__ = cudaGetLastError();                                \
    if (e__ != cudaSuccess) return ::ocsc::cuda_fail(e__, name);         \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// --------------------------------------------------------------- complex --
template <typename T> struct Cx;
template <> struct Cx<float> { using type = float2; };
template <> struct Cx<double> { using type = double2; };
template <typename T> using cx = typename Cx<T>::type;

template <typename C> __host__ __device__ __forceinline__ C mkc(decltype(C::x) r, decltype(C::x) i) {
  C c; c.x = r; c.y = i; return c;
}
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return mkc<C>(a.x + b.x, a.y + b.y); }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return mkc<C>(a.x - b.x, a.y - b.y); }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
  return mkc<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
  return mkc<C>(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
template <typename C> __device__ __forceinline__ C cconj(C a) { return mkc<C>(a.x, -a.y); }
template <typename C, typename S> __device__ __forceinline__ C cscale(C a, S s) { return mkc<C>(a.x * s, a.y * s); }
template <typename C> __device__ __forceinline__ decltype(C::x) cabs2(C a) { return a.x * a.x + a.y * a.y; }
// acc += a * b
template <typename C> __device__ __forceinline__ void cfma(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
// acc += conj(a) * b
template <typename C> __device__ __forceinline__ void cfmac(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
}

// acc += conj(a) * b with the product rounded on its own before the (uncontracted) add, so
// a sum over repeated identical terms is exactly that multiple of one term (duplicating every
// sample of a corpus leaves the averaged history bit-identical, as in the reference's numpy
// sums; reference tests/test_training.py:180-195)
__device__ __forceinline__ void cmacc_sep(double2& acc, double2 a, double2 b) {
  const double px = fma(a.x, b.x, a.y * b.y), py = fma(a.x, b.y, -(a.y * b.x));
  acc.x = __dadd_rn(acc.x, px);
  acc.y = __dadd_rn(acc.y, py);
}
__device__ __forceinline__ void cmacc_sep(float2& acc, float2 a, float2 b) {
  const float px = fmaf(a.x, b.x, a.y * b.y), py = fmaf(a.x, b.y, -(a.y * b.x));
  acc.x = __fadd_rn(acc.x, px);
  acc.y = __fadd_rn(acc.y, py);
}

// ---- 2-wide arithmetic: Blackwell FP32x2 (FADD2/FMUL2/FFMA2) for float2, plain for double2 ----
__device__ __forceinline__ float2 vadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 vsub(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }
__device__ __forceinline__ double2 vadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 vmul(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ double2 vfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
__device__ __forceinline__ double2 vsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
template <typename C> __device__ __forceinline__ C vsplat(decltype(C::x) s) { return mkc<C>(s, s); }

// ---- complex products and +-i combinations in 2-wide form ----------------------------------
// float2: FMUL2 / FFMA2 with a broadcast scalar and a swizzled (LO_HI) operand -- two
// instructions per complex product, one per a -+ i b (the +-1 multiplies are exact, so the
// latter round exactly like the scalar form).  double2: the scalar forms.
__device__ __forceinline__ float2 cmul2(float2 a, float2 b) {  // a * b
  return __ffma2_rn(make_float2(b.y, b.x), make_float2(-a.y, a.y), __fmul2_rn(make_float2(a.x, a.x), b));
}
__device__ __forceinline__ float2 cmulc2(float2 a, float2 b) {  // conj(a) * b
  return __ffma2_rn(make_float2(b.y, b.x), make_float2(a.y, -a.y), __fmul2_rn(make_float2(a.x, a.x), b));
}
__device__ __forceinline__ float2 sub_i(float2 a, float2 b) {  // a - i b
  return __ffma2_rn(make_float2(b.y, b.x), make_float2(1.f, -1.f), a);
}
__device__ __forceinline__ float2 add_i(float2 a, float2 b) {  // a + i b
  return __ffma2_rn(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a);
}
__device__ __forceinline__ float2 vswap(float2 a) { return make_float2(a.y, a.x); }
__device__ __forceinline__ float2 vfma_c(float2 a, float2 b, float2 acc) {  // acc + a * b
  return __ffma2_rn(make_float2(b.y, b.x), make_float2(-a.y, a.y), __ffma2_rn(make_float2(a.x, a.x), b, acc));
}
__device__ __forceinline__ double2 vfma_c(double2 a, double2 b, double2 acc) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc2(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 sub_i(double2 a, double2 b) { return make_double2(a.x + b.y, a.y - b.x); }
__device__ __forceinline__ double2 add_i(double2 a, double2 b) { return make_double2(a.x - b.y, a.y + b.x); }
__device__ __forceinline__ double2 vswap(double2 a) { return make_double2(a.y, a.x); }

template <typename To, typename From> __device__ __forceinline__ cx<To> ccast(From a) {
  return mkc<cx<To>>((To)a.x, (To)a.y);
}

// ------------------------------------------------------------ cp.async --
// Asynchronous global -> shared copies (LDGSTS) of 4/8/16 bytes; commit/wait by group.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ------------------------------------------------------- bulk copies (TMA) --
// One thread moves a contiguous global block into shared memory with cp.async.bulk (16-byte
// aligned addresses, size a multiple of 16); completion is counted on an mbarrier that every
// consumer waits on (one phase per barrier here: each is used once per CTA).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(m)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// issue (one thread): expect `bytes` on m, then copy
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(m))
               : "memory");
}
__device__ __forceinline__ void bulk_wait(uint64_t* m, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(m)), "r"(phase)
        : "memory");
}

// ------------------------------------------------------------ reductions --
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV doubles; result valid in thread 0. `scratch` holds 32*NV doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * 32 + warp] = v[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = lane < nwarps ? scratch[i * 32 + lane] : 0.0;
      v[i] = warp_sum(s);
    }
  }
  __syncthreads();
}

// atomic max for non-negative doubles (bit pattern order == value order)
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  if (!(v >= 0.0)) v = __longlong_as_double(0x7ff8000000000000ULL);  // NaN -> propagate as huge
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// Half-spectrum (rfft2 along W) Hermitian weight of column v: the number of
// full-spectrum points the stored value stands for in a real sum.
__device__ __forceinline__ int herm_weight(int v, int W) {
  return (v == 0 || (2 * v == W)) ? 1 : 2;
}

__host__ __device__ __forceinline__ int64_t packed_index(int i, int j) {  // j <= i
  return (int64_t)i * (i + 1) / 2 + j;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// the per-sample stopping test of one code-ADMM iteration (coding.py:105-118) by one CTA: k_decide,
// or the last CTA of the plane-resident stream kernel.  flags = (done[B], bad[B], all_done,
// iteration count, ...); acc = (B, 4) squared norms, zeroed for the next iteration
__device__ __forceinline__ void decide_block(int B, double tol, double* acc, int32_t* flags, int32_t* iters,
                                             int32_t* status) {
  int32_t* done = flags;
  int32_t* bad = flags + B;
  int32_t* all_done = flags + 2 * B;
  int32_t* itc = flags + 2 * B + 1;
  if (*all_done) return;
  __shared__ int it_s;
  __syncthreads();
  if (threadIdx.x == 0) it_s = ++(*itc);
  __syncthreads();
  const int it = it_s;
  int mine = 1;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (!done[b]) {
      iters[b] = it;
      if (bad[b]) {
        done[b] = 1;
        status[b] = 2;
      } else {
        const double num = sqrt(acc[4 * b]), den = sqrt(acc[4 * b + 1]);
        const double gap = sqrt(acc[4 * b + 2]), dual = sqrt(acc[4 * b + 3]);
        const double gap_scale = fmax(fmax(den, dual), 1e-12);
        if (num <= tol * fmax(den, 1e-12) && gap <= tol * gap_scale) {
          done[b] = 1;
          status[b] = 1;
        }
      }
      acc[4 * b] = acc[4 * b + 1] = acc[4 * b + 2] = acc[4 * b + 3] = 0.0;
    }
    mine &= done[b];
  }
  const int all = __syncthreads_and(mine);
  if (threadIdx.x == 0 && all) *all_done = 1;
}

}  // namespace ocsc
