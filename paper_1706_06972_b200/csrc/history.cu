// Frequency-domain history and the dictionary row solve (dictionary.py:30-142).
//
// The reference keeps, per frequency p, the averaged cross term and the exact
// inverse ((1/t) sum z z^H + rho P I)^-1, refreshed by an O(K^3) solve per
// sample (dictionary.py:73-114).  Here the state is the un-normalised sums
//     S_p = sum_b z_bp z_bp^H  (packed lower, K(K+1)/2),   c_p = sum_b conj(x_bp) z_bp
// updated by a rank-B accumulation per mini-batch; the inverse is rebuilt once per
// mini-batch by a per-frequency Cholesky (A = S + t rho P I = L L^H) and an explicit
// packed inverse, which the J dictionary rounds then apply as a Hermitian GEMV.
// Algebra: ((1/t)S + rho P I)^-1 = t (S + t rho P I)^-1, so the row solve
// d = (conj(c/t) + rho P (v - theta)) . inv_gram  becomes
// conj(d) = (S + t rho P I)^-1 (c + t rho P conj(v - theta)).
#include "common.cuh"
#include "transforms.cuh"

namespace ocsc {

// ---------------------------------------------------------- accumulation --
// One CTA per frequency.  Codes of a chunk of BC samples are staged as Zs[bb][k];
// each thread owns 4x4 tiles of the packed lower triangle.
template <typename Tin, typename Th>
__global__ void __launch_bounds__(256) k_hist_accum(int K, int nf, int B, int BC, const cx<Tin>* __restrict__ z,
                                                    int64_t z_sb, int64_t z_sk, int64_t z_sp,
                                                    const cx<Tin>* __restrict__ x, int64_t x_sb, int64_t x_sp,
                                                    cx<Th>* S, cx<Th>* c) {
  using C = cx<Th>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* Zs = reinterpret_cast<C*>(smem_raw);  // [BC][K]
  C* xs = Zs + (int64_t)BC * K;            // [BC]
  const int p = blockIdx.x;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  C* Sp = S + (int64_t)p * npk;
  const int nt = (K + 3) / 4;
  const int ntiles = nt * (nt + 1) / 2;
  for (int b0 = 0; b0 < B; b0 += BC) {
    const int bc = min(BC, B - b0);
    for (int e = threadIdx.x; e < bc * K; e += blockDim.x) {
      const int bb = e / K, k = e % K;
      Zs[bb * K + k] = ccast<Th>(z[(int64_t)(b0 + bb) * z_sb + (int64_t)k * z_sk + (int64_t)p * z_sp]);
    }
    for (int bb = threadIdx.x; bb < bc; bb += blockDim.x)
      xs[bb] = ccast<Th>(x[(int64_t)(b0 + bb) * x_sb + (int64_t)p * x_sp]);
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      C acc = mkc<C>(0, 0);
      for (int bb = 0; bb < bc; ++bb) cfmac(acc, xs[bb], Zs[bb * K + k]);
      C& dst = c[(int64_t)p * K + k];
      dst = cadd(dst, acc);
    }
    for (int tile = threadIdx.x; tile < ntiles; tile += blockDim.x) {
      int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
      while (I * (I + 1) / 2 > tile) --I;
      while ((I + 1) * (I + 2) / 2 <= tile) ++I;
      const int J = tile - I * (I + 1) / 2;
      C acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = mkc<C>(0, 0);
      for (int bb = 0; bb < bc; ++bb) {
        C zi[4], zj[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = 4 * I + r, j = 4 * J + r;
          zi[r] = i < K ? Zs[bb * K + i] : mkc<C>(0, 0);
          zj[r] = j < K ? Zs[bb * K + j] : mkc<C>(0, 0);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q) cfmac(acc[r][q], zj[q], zi[r]);  // z_i conj(z_j)
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = 4 * I + r;
        if (i >= K) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 4 * J + q;
          if (j > i) continue;
          C& dst = Sp[packed_index(i, j)];
          dst = cadd(dst, acc[r][q]);
        }
      }
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------- inversion --
// One CTA per frequency, two packed K x K buffers in shared memory:
// Cholesky in place, triangular inverse into the second, then A^-1 = L^-H L^-1
// back into the first.
template <typename Th>
__global__ void __launch_bounds__(256) k_hist_invert(int K, const cx<Th>* __restrict__ S, Th ridge, Th scale,
                                                     cx<Th>* inv, int32_t* info) {
  using C = cx<Th>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  C* A = reinterpret_cast<C*>(smem_raw);
  C* Li = A + npk;
  __shared__ Th inv_d;
  const int p = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const C* Sp = S + (int64_t)p * npk;
  for (int64_t e = threadIdx.x; e < npk; e += blockDim.x) A[e] = Sp[e];
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) A[packed_index(i, i)].x += ridge;
  __syncthreads();
  for (int j = 0; j < K; ++j) {
    if (threadIdx.x == 0) {
      Th d = A[packed_index(j, j)].x;
      if (!(d > (Th)0)) {
        atomicCAS(info, 0, p + 1);
        d = (Th)NAN;
      }
      d = sqrt(d);
      A[packed_index(j, j)] = mkc<C>(d, 0);
      inv_d = (Th)1 / d;
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < K; i += blockDim.x) A[packed_index(i, j)] = cscale(A[packed_index(i, j)], inv_d);
    __syncthreads();
    for (int i = j + 1 + warp; i < K; i += nwarps) {
      const C lij = A[packed_index(i, j)];
      C* rowi = A + packed_index(i, 0);
      for (int k = j + 1 + lane; k <= i; k += 32) {
        const C lkj = A[packed_index(k, j)];
        // A[i][k] -= L[i][j] conj(L[k][j])
        rowi[k] = csub(rowi[k], mkc<C>(lij.x * lkj.x + lij.y * lkj.y, lij.y * lkj.x - lij.x * lkj.y));
      }
    }
    __syncthreads();
  }
  // Li = L^-1 (lower), column c by thread c
  for (int col = threadIdx.x; col < K; col += blockDim.x) {
    Li[packed_index(col, col)] = mkc<C>((Th)1 / A[packed_index(col, col)].x, 0);
    for (int i = col + 1; i < K; ++i) {
      C acc = mkc<C>(0, 0);
      const C* rowi = A + packed_index(i, 0);
      for (int k = col; k < i; ++k) cfma(acc, rowi[k], Li[packed_index(k, col)]);
      Li[packed_index(i, col)] = cscale(acc, -(Th)1 / rowi[i].x);
    }
  }
  __syncthreads();
  // A^-1[i][j] = sum_{k >= i} conj(Li[k][i]) Li[k][j]   (i >= j)
  C* out = inv + (int64_t)p * npk;
  for (int i = warp; i < K; i += nwarps) {
    for (int j = lane; j <= i; j += 32) {
      C acc = mkc<C>(0, 0);
      for (int k = i; k < K; ++k) cfmac(acc, Li[packed_index(k, i)], Li[packed_index(k, j)]);
      out[packed_index(i, j)] = cscale(acc, scale);
    }
  }
}

template <typename T>
__global__ void k_packed_to_full(int K, int nf, const cx<T>* packed, T scale, cx<T>* full) {
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  const int64_t total = (int64_t)nf * K * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % K);
    const int64_t r = e / K;
    const int i = (int)(r % K);
    const int64_t p = r / K;
    cx<T> v = i >= j ? packed[p * npk + packed_index(i, j)] : cconj(packed[p * npk + packed_index(j, i)]);
    full[e] = cscale(v, scale);
  }
}

template <typename T>
__global__ void k_nonfinite(int64_t n, const T* a, int32_t* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(a[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ------------------------------------------------------------- row solve --
// One CTA per frequency; thread j forms row j of the packed Hermitian GEMV.
template <typename Tc, typename Th>
__global__ void __launch_bounds__(128) k_rowsolve(int K, int nf, const cx<Th>* __restrict__ inv,
                                                  const cx<Th>* __restrict__ c, Th ridge,
                                                  const cx<Tc>* __restrict__ Vh, const cx<Tc>* __restrict__ Th_,
                                                  int64_t sk, int64_t sp, cx<Tc>* Dh) {
  using C = cx<Th>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* rhs = reinterpret_cast<C*>(smem_raw);
  const int p = blockIdx.x;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const int64_t o = (int64_t)k * sk + (int64_t)p * sp;
    const C v = csub(ccast<Th>(Vh[o]), ccast<Th>(Th_[o]));
    const C ck = c[(int64_t)p * K + k];
    rhs[k] = mkc<C>(ck.x + ridge * v.x, ck.y - ridge * v.y);
  }
  __syncthreads();
  const C* Ap = inv + (int64_t)p * npk;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    C acc = mkc<C>(0, 0);
    const C* row = Ap + packed_index(j, 0);
    for (int k = 0; k <= j; ++k) cfma(acc, row[k], rhs[k]);
    for (int k = j + 1; k < K; ++k) cfmac(acc, Ap[packed_index(k, j)], rhs[k]);
    Dh[(int64_t)j * sk + (int64_t)p * sp] = mkc<cx<Tc>>((Tc)acc.x, (Tc)-acc.y);
  }
}

}  // namespace ocsc

using namespace ocsc;

static size_t csize(int dtype) { return dtype == OCSC_F64 ? 16 : 8; }

extern "C" int ocsc_history_accumulate(int dtype_in, int dtype_hist, int K, int nfreq, int B, const void* z,
                                       int64_t z_sb, int64_t z_sk, int64_t z_sp, const void* x, int64_t x_sb,
                                       int64_t x_sp, void* S, void* c, void* stream) {
  if (K <= 0 || nfreq < 0 || B < 0) return fail(OCSC_ESHAPE, "history_accumulate: bad extents");
  if (nfreq == 0 || B == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  const size_t cs = csize(dtype_hist);
  int BC = (int)((160 * 1024) / (cs * (K + 1)));
  if (BC > 32) BC = 32;
  if (BC < 1) return fail(OCSC_EARG, "history_accumulate: K too large for one CTA");
  const size_t smem = cs * ((size_t)BC * K + BC);
#define HA(TI, TH)                                                                                       \
  do {                                                                                                   \
    OCSC_CUDA(cudaFuncSetAttribute(k_hist_accum<TI, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_hist_accum<TI, TH><<<nfreq, 256, smem, s>>>(K, nfreq, B, BC, (const cx<TI>*)z, z_sb, z_sk, z_sp,   \
                                                   (const cx<TI>*)x, x_sb, x_sp, (cx<TH>*)S, (cx<TH>*)c); \
  } while (0)
  if (dtype_in == OCSC_F32 && dtype_hist == OCSC_F32) HA(float, float);
  else if (dtype_in == OCSC_F32 && dtype_hist == OCSC_F64) HA(float, double);
  else if (dtype_in == OCSC_F64 && dtype_hist == OCSC_F64) HA(double, double);
  else return fail(OCSC_EARG, "history_accumulate: unsupported dtype pair");
#undef HA
  OCSC_LAUNCHED("k_hist_accum");
  return OCSC_OK;
}

extern "C" int ocsc_history_invert(int dtype_hist, int K, int nfreq, const void* S, double ridge, double scale,
                                   void* inv, int32_t* info, void* stream) {
  if (K <= 0 || nfreq < 0) return fail(OCSC_ESHAPE, "history_invert: bad extents");
  cudaStream_t s = as_stream(stream);
  OCSC_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
  if (nfreq == 0) return OCSC_OK;
  const size_t smem = 2 * csize(dtype_hist) * (size_t)K * (K + 1) / 2;
  if (smem > 227 * 1024)
    return fail(OCSC_EARG, "history_invert: K=" + std::to_string(K) + " exceeds the shared-memory Cholesky (K<=120 f64, K<=170 f32)");
  if (dtype_hist == OCSC_F32) {
    OCSC_CUDA(cudaFuncSetAttribute(k_hist_invert<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist_invert<float><<<nfreq, 256, smem, s>>>(K, (const float2*)S, (float)ridge, (float)scale, (float2*)inv, info);
  } else if (dtype_hist == OCSC_F64) {
    OCSC_CUDA(cudaFuncSetAttribute(k_hist_invert<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist_invert<double><<<nfreq, 256, smem, s>>>(K, (const double2*)S, ridge, scale, (double2*)inv, info);
  } else {
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  }
  OCSC_LAUNCHED("k_hist_invert");
  return OCSC_OK;
}

extern "C" int ocsc_packed_to_full(int dtype, int K, int nfreq, const void* packed, double scale, void* full,
                                   void* stream) {
  int64_t n = (int64_t)nfreq * K * K;
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_packed_to_full<float><<<grid_for(n, 256), 256, 0, s>>>(K, nfreq, (const float2*)packed, (float)scale, (float2*)full);
  else if (dtype == OCSC_F64)
    k_packed_to_full<double><<<grid_for(n, 256), 256, 0, s>>>(K, nfreq, (const double2*)packed, scale, (double2*)full);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_packed_to_full");
  return OCSC_OK;
}

extern "C" int ocsc_nonfinite(int dtype, int64_t n_reals, const void* a, int32_t* flag, void* stream) {
  if (n_reals <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_nonfinite<float><<<grid_for(n_reals, 256), 256, 0, s>>>(n_reals, (const float*)a, flag);
  else if (dtype == OCSC_F64)
    k_nonfinite<double><<<grid_for(n_reals, 256), 256, 0, s>>>(n_reals, (const double*)a, flag);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_nonfinite");
  return OCSC_OK;
}

extern "C" int ocsc_dict_rowsolve(int dtype, int dtype_hist, int K, int nfreq, const void* inv, const void* c,
                                  double ridge, const void* Vh, const void* Th, int64_t sk, int64_t sp, void* Dh,
                                  void* stream) {
  if (K <= 0 || nfreq < 0) return fail(OCSC_ESHAPE, "dict_rowsolve: bad extents");
  if (nfreq == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  const size_t smem = csize(dtype_hist) * K;
#define RS(TC, TH)                                                                                       \
  k_rowsolve<TC, TH><<<nfreq, 128, smem, s>>>(K, nfreq, (const cx<TH>*)inv, (const cx<TH>*)c, (TH)ridge, \
                                              (const cx<TC>*)Vh, (const cx<TC>*)Th, sk, sp, (cx<TC>*)Dh)
  if (dtype == OCSC_F32 && dtype_hist == OCSC_F32) RS(float, float);
  else if (dtype == OCSC_F32 && dtype_hist == OCSC_F64) RS(float, double);
  else if (dtype == OCSC_F64 && dtype_hist == OCSC_F64) RS(double, double);
  else return fail(OCSC_EARG, "dict_rowsolve: unsupported dtype pair");
#undef RS
  OCSC_LAUNCHED("k_rowsolve");
  return OCSC_OK;
}
