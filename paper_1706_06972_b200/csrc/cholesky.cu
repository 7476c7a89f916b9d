// Large-K history factorisation and row solve (dictionary.py:101-111, 134-142) for
// K beyond the shared-memory inverse (BASELINE config 3: K = 256; config 4: K <= 512).
//
// Per frequency p, A_p = S_p + ridge I (K x K Hermitian positive definite) is factored
// A = L L^H by a blocked right-looking Cholesky, one CTA per frequency, 32 x 32 tiles:
//   for each tile column kb:  factor the diagonal tile in shared memory;
//                             panel  L[ib][kb] = A[ib][kb] L[kb][kb]^-H  (row-parallel TRSM);
//                             stage the whole panel in shared memory;
//                             trailing update A[ib][jb] -= L[ib][kb] L[jb][kb]^H (jb <= ib),
//                             one warp per 32x32 target tile (lane = column).
// L stays in global memory (full K x K per frequency, lower triangle).  The dictionary row
// solve then runs two blocked triangular solves per frequency and round:
//   conj(d) = L^-H L^-1 (c + ridge conj(v - theta)).
#include "common.cuh"
#include "transforms.cuh"

namespace ocsc {

constexpr int CT = 32;  // tile edge

template <typename C>
__device__ __forceinline__ C* tile_ptr(C* L, int K, int ib, int jb) {
  return L + (int64_t)ib * CT * K + (int64_t)jb * CT;
}

// A (packed lower, K(K+1)/2 per frequency) + ridge I -> full lower L = chol(A)
template <typename T>
__global__ void __launch_bounds__(256) k_chol_blocked(int K, const cx<T>* __restrict__ S, T ridge, cx<T>* Lall,
                                                      int32_t* info) {
  using C = cx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nb = K / CT;
  C* D = reinterpret_cast<C*>(smem_raw);          // diagonal tile [CT][CT+1]
  C* Pn = D + CT * (CT + 1);                      // panel tiles [nb][CT][CT+1]
  const int p = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  const C* Sp = S + (int64_t)p * npk;
  C* L = Lall + (int64_t)p * K * K;
  constexpr int LD = CT + 1;

  // expand the packed lower triangle (+ ridge) into the full-layout workspace
  for (int64_t e = tid; e < (int64_t)K * K; e += nt) {
    const int i = (int)(e / K), j = (int)(e % K);
    C v = mkc<C>(0, 0);
    if (j <= i) {
      v = Sp[packed_index(i, j)];
      if (i == j) v = mkc<C>(v.x + ridge, (T)0);
    }
    L[e] = v;
  }
  __syncthreads();

  for (int kb = 0; kb < nb; ++kb) {
    // ---- factor the diagonal tile in shared memory (unblocked, right-looking) ----
    C* Lkk = tile_ptr(L, K, kb, kb);
    for (int e = tid; e < CT * CT; e += nt) {
      const int i = e / CT, j = e % CT;
      D[i * LD + j] = Lkk[(int64_t)i * K + j];
    }
    __syncthreads();
    for (int j = 0; j < CT; ++j) {
      if (tid == 0) {
        T d = D[j * LD + j].x;
        if (!(d > (T)0)) {
          atomicCAS(info, 0, p + 1);
          d = (T)NAN;
        }
        D[j * LD + j] = mkc<C>(sqrt(d), (T)0);
      }
      __syncthreads();
      const T inv = (T)1 / D[j * LD + j].x;
      for (int i = j + 1 + tid; i < CT; i += nt) D[i * LD + j] = cscale(D[i * LD + j], inv);
      __syncthreads();
      for (int e = tid; e < CT * CT; e += nt) {
        const int i = e / CT, k = e % CT;
        if (k > j && k <= i) {
          const C a = D[i * LD + j], bb = D[k * LD + j];
          C& t = D[i * LD + k];
          t.x -= a.x * bb.x + a.y * bb.y;  // a conj(b)
          t.y -= a.y * bb.x - a.x * bb.y;
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < CT * CT; e += nt) {
      const int i = e / CT, j = e % CT;
      Lkk[(int64_t)i * K + j] = j <= i ? D[i * LD + j] : mkc<C>(0, 0);
    }
    // ---- panel: X = A[ib][kb] Lkk^-H, one thread per panel row, in place in shared memory ----
    const int prow = (nb - kb - 1) * CT;
    for (int rr = tid; rr < prow; rr += nt) {
      const int ib = kb + 1 + rr / CT, i = rr % CT;
      const C* arow = tile_ptr(L, K, ib, kb) + (int64_t)i * K;
      C* x = Pn + ((ib - kb - 1) * CT + i) * LD;
      for (int j = 0; j < CT; ++j) x[j] = arow[j];
    }
    __syncthreads();
    for (int rr = tid; rr < prow; rr += nt) {
      C* x = Pn + rr * LD;
      // x L^H = a  ->  x_j = (a_j - sum_{k<j} x_k conj(L_jk)) / L_jj
      for (int j = 0; j < CT; ++j) {
        C acc = x[j];
        for (int k = 0; k < j; ++k) {
          const C l = D[j * LD + k], xk = x[k];
          acc.x -= xk.x * l.x + xk.y * l.y;
          acc.y -= xk.y * l.x - xk.x * l.y;
        }
        x[j] = cscale(acc, (T)1 / D[j * LD + j].x);
      }
    }
    __syncthreads();
    for (int e = tid; e < prow * CT; e += nt) {  // write the panel back (coalesced)
      const int rr = e / CT, j = e % CT;
      const int ib = kb + 1 + rr / CT, i = rr % CT;
      tile_ptr(L, K, ib, kb)[(int64_t)i * K + j] = Pn[rr * LD + j];
    }
    __syncthreads();
    // ---- trailing update: A[ib][jb] -= P_ib P_jb^H for kb < jb <= ib ----
    // one warp per 32 x 32 target tile, lane = target column: per k, one own panel value
    // and 32 broadcast panel values feed 32 complex FMAs
    const int nrem = nb - kb - 1;
    const int ntile = nrem * (nrem + 1) / 2;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    for (int t = warp; t < ntile; t += nwarps) {
      int I = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while (I * (I + 1) / 2 > t) --I;
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      const int J = t - I * (I + 1) / 2;  // panel tile indices, J <= I
      const C* Pi = Pn + I * CT * LD;
      const C* Pj = Pn + J * CT * LD;
      C acc[CT];
#pragma unroll
      for (int i = 0; i < CT; ++i) acc[i] = mkc<C>(0, 0);
#pragma unroll 4
      for (int k = 0; k < CT; ++k) {
        const C bj = Pj[lane * LD + k];  // P_jb[lane][k]
#pragma unroll
        for (int i = 0; i < CT; ++i) cfmac(acc[i], bj, Pi[i * LD + k]);  // P_ib[i][k] conj(P_jb[lane][k])
      }
      C* tgt = tile_ptr(L, K, kb + 1 + I, kb + 1 + J) + lane;
#pragma unroll
      for (int i = 0; i < CT; ++i) {
        if (I != J || lane <= i) {
          C& v = tgt[(int64_t)i * K];
          v = csub(v, acc[i]);
        }
      }
    }
    __syncthreads();
  }
}

// conj(D_p) = L^-H L^-1 (c_p + ridge conj(V_p - Theta_p)), one CTA per frequency
template <typename Tc, typename Th>
__global__ void __launch_bounds__(256) k_rowsolve_chol(int K, const cx<Th>* __restrict__ Lall,
                                                       const cx<Th>* __restrict__ c, Th ridge,
                                                       const cx<Tc>* __restrict__ Vh, const cx<Tc>* __restrict__ Th_,
                                                       int64_t sk, int64_t sp, cx<Tc>* Dh) {
  using C = cx<Th>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* y = reinterpret_cast<C*>(smem_raw);  // [K]
  C* part = y + K;                        // [nt]
  const int p = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const C* L = Lall + (int64_t)p * K * K;
  for (int k = tid; k < K; k += nt) {
    const int64_t o = (int64_t)k * sk + (int64_t)p * sp;
    const C v = csub(ccast<Th>(Vh[o]), ccast<Th>(Th_[o]));
    const C ck = c[(int64_t)p * K + k];
    y[k] = mkc<C>(ck.x + ridge * v.x, ck.y - ridge * v.y);
  }
  __syncthreads();
  // forward: L y = b, row by row; each warp handles rows, lanes split the dot product
  for (int i = 0; i < K; ++i) {
    if (warp == 0) {
      C acc = mkc<C>(0, 0);
      const C* row = L + (int64_t)i * K;
      for (int k = lane; k < i; k += 32) cfma(acc, row[k], y[k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) y[i] = cscale(csub(y[i], acc), (Th)1 / row[i].x);
    }
    __syncwarp();
  }
  __syncthreads();
  // backward: L^H x = y, column-oriented: x_i = y_i / L_ii; y_k -= conj(L_ik) x_i for k < i
  for (int i = K - 1; i >= 0; --i) {
    const C* row = L + (int64_t)i * K;
    const C xi = cscale(y[i], (Th)1 / row[i].x);
    __syncthreads();
    for (int k = tid; k < i; k += nt) {
      const C l = row[k];
      C& t = y[k];
      t.x -= l.x * xi.x + l.y * xi.y;  // conj(l) x
      t.y -= l.x * xi.y - l.y * xi.x;
    }
    if (tid == 0) y[i] = xi;
    __syncthreads();
  }
  (void)part;
  (void)nw;
  for (int j = tid; j < K; j += nt)
    Dh[(int64_t)j * sk + (int64_t)p * sp] = mkc<cx<Tc>>((Tc)y[j].x, (Tc)-y[j].y);
}

}  // namespace ocsc

using namespace ocsc;

extern "C" size_t ocsc_history_factor_bytes(int dtype_hist, int K, int nfreq) {
  return (size_t)(dtype_hist == OCSC_F64 ? 16 : 8) * (size_t)K * K * nfreq;
}

extern "C" int ocsc_history_factor(int dtype_hist, int K, int nfreq, const void* S, double ridge, void* L,
                                   int32_t* info, void* stream) {
  if (K <= 0 || nfreq < 0) return fail(OCSC_ESHAPE, "history_factor: bad extents");
  if (K % CT) return fail(OCSC_EARG, "history_factor: K must be a multiple of 32");
  cudaStream_t s = as_stream(stream);
  OCSC_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
  if (nfreq == 0) return OCSC_OK;
  const int nb = K / CT;
  const size_t cs = dtype_hist == OCSC_F64 ? 16 : 8;
  const size_t smem = cs * (size_t)CT * (CT + 1) * (size_t)nb;  // diagonal + up to nb-1 panel tiles
  if (smem > 227 * 1024) return fail(OCSC_EARG, "history_factor: panel exceeds shared memory for this K/dtype");
  if (dtype_hist == OCSC_F32) {
    OCSC_CUDA(cudaFuncSetAttribute(k_chol_blocked<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_chol_blocked<float><<<nfreq, 256, smem, s>>>(K, (const float2*)S, (float)ridge, (float2*)L, info);
  } else if (dtype_hist == OCSC_F64) {
    OCSC_CUDA(cudaFuncSetAttribute(k_chol_blocked<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_chol_blocked<double><<<nfreq, 256, smem, s>>>(K, (const double2*)S, ridge, (double2*)L, info);
  } else {
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  }
  OCSC_LAUNCHED("k_chol_blocked");
  return OCSC_OK;
}

extern "C" int ocsc_dict_rowsolve_chol(int dtype, int dtype_hist, int K, int nfreq, const void* L, const void* c,
                                       double ridge, const void* Vh, const void* Th, int64_t sk, int64_t sp,
                                       void* Dh, void* stream) {
  if (K <= 0 || nfreq < 0) return fail(OCSC_ESHAPE, "dict_rowsolve_chol: bad extents");
  if (nfreq == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  const size_t smem = (dtype_hist == OCSC_F64 ? 16 : 8) * ((size_t)K + 256);
#define RC(TC, TH)                                                                                          \
  k_rowsolve_chol<TC, TH><<<nfreq, 256, smem, s>>>(K, (const cx<TH>*)L, (const cx<TH>*)c, (TH)ridge,        \
                                                   (const cx<TC>*)Vh, (const cx<TC>*)Th, sk, sp, (cx<TC>*)Dh)
  if (dtype == OCSC_F32 && dtype_hist == OCSC_F32) RC(float, float);
  else if (dtype == OCSC_F32 && dtype_hist == OCSC_F64) RC(float, double);
  else if (dtype == OCSC_F64 && dtype_hist == OCSC_F64) RC(double, double);
  else return fail(OCSC_EARG, "dict_rowsolve_chol: unsupported dtype pair");
#undef RC
  OCSC_LAUNCHED("k_rowsolve_chol");
  return OCSC_OK;
}
