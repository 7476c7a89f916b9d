// Frequency-domain history and the dictionary row solve (dictionary.py:30-142).
//
// The reference keeps, per frequency p, the averaged cross term and the exact
// inverse ((1/t) sum z z^H + rho P I)^-1, refreshed by an O(K^3) solve per
// sample (dictionary.py:73-114).  Here the state is the un-normalised sums
//     S_p = sum_b z_bp z_bp^H  (packed lower, K(K+1)/2),   c_p = sum_b conj(x_bp) z_bp
// updated by a rank-B accumulation per mini-batch; the inverse of A = S + t rho P I is
// rebuilt once per mini-batch per frequency (in-place Gauss-Jordan in shared memory) and
// stored packed; the J dictionary rounds then apply it as a Hermitian GEMV.
// Algebra: ((1/t)S + rho P I)^-1 = t (S + t rho P I)^-1, so the row solve
// d = (conj(c/t) + rho P (v - theta)) . inv_gram  becomes
// conj(d) = (S + t rho P I)^-1 (c + t rho P conj(v - theta)).
#include <cstdlib>

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
  // products of one chunk of <= BC samples are formed in the input precision (FP32 FMAs in
  // float32 mode: the chunk sum of <= 32 terms keeps ~1e-7 relative accuracy); the running
  // history sums themselves are kept in the history precision
  using Ci = cx<Tin>;
  using C = cx<Th>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ci* Zs = reinterpret_cast<Ci*>(smem_raw);  // [BC][K]
  Ci* xs = Zs + (int64_t)BC * K;             // [BC]
  const int p = blockIdx.x;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  C* Sp = S + (int64_t)p * npk;
  const int nt = (K + 3) / 4;
  const int ntiles = nt * (nt + 1) / 2;
  for (int b0 = 0; b0 < B; b0 += BC) {
    const int bc = min(BC, B - b0);
    for (int e = threadIdx.x; e < bc * K; e += blockDim.x) {
      const int bb = e / K, k = e % K;
      Zs[bb * K + k] = z[(int64_t)(b0 + bb) * z_sb + (int64_t)k * z_sk + (int64_t)p * z_sp];
    }
    for (int bb = threadIdx.x; bb < bc; bb += blockDim.x) xs[bb] = x[(int64_t)(b0 + bb) * x_sb + (int64_t)p * x_sp];
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      Ci acc = mkc<Ci>(0, 0);
      for (int bb = 0; bb < bc; ++bb) cmacc_sep(acc, xs[bb], Zs[bb * K + k]);
      C& dst = c[(int64_t)p * K + k];
      dst = cadd(dst, ccast<Th>(acc));
    }
    for (int tile = threadIdx.x; tile < ntiles; tile += blockDim.x) {
      int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
      while (I * (I + 1) / 2 > tile) --I;
      while ((I + 1) * (I + 2) / 2 <= tile) ++I;
      const int J = tile - I * (I + 1) / 2;
      Ci acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = mkc<Ci>(0, 0);
      for (int bb = 0; bb < bc; ++bb) {
        Ci zi[4], zj[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = 4 * I + r, j = 4 * J + r;
          zi[r] = i < K ? Zs[bb * K + i] : mkc<Ci>(0, 0);
          zj[r] = j < K ? Zs[bb * K + j] : mkc<Ci>(0, 0);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q) cmacc_sep(acc[r][q], zj[q], zi[r]);  // z_i conj(z_j)
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
          dst = cadd(dst, ccast<Th>(acc[r][q]));
        }
      }
    }
    __syncthreads();
  }
}

// Tiled accumulation for float32 code spectra (the trainer's float32 mode, BASELINE config 4):
// per frequency, S += Z Z^H is a K x K x B complex GEMM; one CTA computes a 64 x 64 block
// (I >= J) of the lower triangle, 16 x 16 threads x 4 x 4 complex in registers, samples staged
// through shared memory 32 at a time.  Each complex multiply-add is two FP32x2 FMAs
// (acc += zi * zj.x + (zi.y, -zi.x) * zj.y), the form that reaches the FP32 pipe's full rate.
// The diagonal-block CTAs also accumulate the cross term c for their 64 rows.  Chunk sums of
// <= 32 samples are added to a float64 history per chunk (as k_hist_accum), to a float32
// history once at the end.
constexpr int HT = 64, HCH = 32;

// tensor-core (3xTF32 tcgen05) accumulation, history_tc.cu; OCSC_HIST_TC=0 selects the FP32x2 kernel
int history_accumulate_tc(int dtype_hist, int K, int nfreq, int B, const void* z, int64_t z_sb, int64_t z_sk,
                          int64_t z_sp, const void* x, int64_t x_sb, int64_t x_sp, void* S, void* c, cudaStream_t s);
static bool use_tensor_cores() {
  static const bool on = [] {
    const char* e = getenv("OCSC_HIST_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename Th>
__global__ void __launch_bounds__(256) k_hist_accum_tiled(int K, int B, const float2* __restrict__ z, int64_t z_sb,
                                                          int64_t z_sk, int64_t z_sp, const float2* __restrict__ x,
                                                          int64_t x_sb, int64_t x_sp, cx<Th>* S, cx<Th>* c,
                                                          int pairs) {
  __shared__ __align__(16) float2 Zi[HCH][HT];
  __shared__ __align__(16) float2 Zj[HCH][HT];
  __shared__ float2 Xs[HCH];
  // all block pairs of one frequency are consecutive CTAs, so its codes are re-read from L2
  const int p = blockIdx.x / pairs, tp = blockIdx.x - (blockIdx.x / pairs) * pairs;
  int I = (int)((sqrtf(8.0f * tp + 1.0f) - 1.0f) * 0.5f);
  while (I * (I + 1) / 2 > tp) --I;
  while ((I + 1) * (I + 2) / 2 <= tp) ++I;
  const int J = tp - I * (I + 1) / 2;
  const bool diag = I == J;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  float2 acc[4][4];
  float2 cacc = make_float2(0.f, 0.f);
  auto zero = [&]() {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = make_float2(0.f, 0.f);
  };
  auto flush = [&]() {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = I * HT + ty * 4 + r;
      if (i >= K) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = J * HT + tx * 4 + q;
        if (j > i) continue;
        cx<Th>& dst = S[(int64_t)p * npk + packed_index(i, j)];
        dst = mkc<cx<Th>>(dst.x + (Th)acc[r][q].x, dst.y + (Th)acc[r][q].y);
      }
    }
    if (diag && tid < HT && I * HT + tid < K) {
      cx<Th>& dst = c[(int64_t)p * K + I * HT + tid];
      dst = mkc<cx<Th>>(dst.x + (Th)cacc.x, dst.y + (Th)cacc.y);
    }
  };
  zero();
  for (int b0 = 0; b0 < B; b0 += HCH) {
    const int bc = min(HCH, B - b0);
    for (int e = tid; e < HCH * HT; e += 256) {
      const int bb = e / HT, k = e % HT;
      const int ki = I * HT + k, kj = J * HT + k;
      const int64_t base = (int64_t)(b0 + bb) * z_sb + (int64_t)p * z_sp;
      Zi[bb][k] = (bb < bc && ki < K) ? z[base + (int64_t)ki * z_sk] : make_float2(0.f, 0.f);
      if (!diag) Zj[bb][k] = (bb < bc && kj < K) ? z[base + (int64_t)kj * z_sk] : make_float2(0.f, 0.f);
    }
    if (diag && tid < HCH) Xs[tid] = tid < bc ? x[(int64_t)(b0 + tid) * x_sb + (int64_t)p * x_sp] : make_float2(0.f, 0.f);
    __syncthreads();
    const float2(*ZJ)[HT] = diag ? Zi : Zj;
#pragma unroll 4
    for (int bb = 0; bb < bc; ++bb) {
      const float4* ri = reinterpret_cast<const float4*>(&Zi[bb][ty * 4]);
      const float4* rj = reinterpret_cast<const float4*>(&ZJ[bb][tx * 4]);
      const float4 i01 = ri[0], i23 = ri[1], j01 = rj[0], j23 = rj[1];
      const float2 zi[4] = {make_float2(i01.x, i01.y), make_float2(i01.z, i01.w), make_float2(i23.x, i23.y),
                            make_float2(i23.z, i23.w)};
      const float2 zj[4] = {make_float2(j01.x, j01.y), make_float2(j01.z, j01.w), make_float2(j23.x, j23.y),
                            make_float2(j23.z, j23.w)};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float2 zs = make_float2(zi[r].y, -zi[r].x);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[r][q] = vfma(zi[r], make_float2(zj[q].x, zj[q].x), acc[r][q]);
          acc[r][q] = vfma(zs, make_float2(zj[q].y, zj[q].y), acc[r][q]);
        }
      }
    }
    if (diag && tid < HT) {
      for (int bb = 0; bb < bc; ++bb) cfmac(cacc, Xs[bb], Zi[bb][tid]);  // conj(x) z
    }
    __syncthreads();
    if (sizeof(Th) == 8) {  // float64 history: add each chunk's float32 sums
      flush();
      zero();
      cacc = make_float2(0.f, 0.f);
    }
  }
  if (sizeof(Th) == 4) flush();
}

// -------------------------------------------------------------- inversion --
// One CTA per frequency: A = S + ridge I expanded to a full K x K Hermitian matrix in shared
// memory, inverted in place by Gauss-Jordan elimination (A is Hermitian positive definite,
// so no pivoting is needed: every pivot is a positive Schur-complement diagonal).  Each of
// the K steps is one fully parallel rank-1 update (three block barriers per step).
template <typename Th, typename Ti>
__global__ void __launch_bounds__(512) k_hist_invert(int K, const cx<Th>* __restrict__ S, Th ridge, Th scale,
                                                     cx<Ti>* inv, int32_t* info) {
  using C = cx<Th>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int LD = K + 1;  // padded row stride
  C* A = reinterpret_cast<C*>(smem_raw);
  C* rowk = A + (int64_t)K * LD;
  C* colk = rowk + K;
  __shared__ Th pinv_s;
  const int p = blockIdx.x;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  const C* Sp = S + (int64_t)p * npk;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int i = e / K, j = e % K;
    C v = i >= j ? Sp[packed_index(i, j)] : cconj(Sp[packed_index(j, i)]);
    if (i == j) v = mkc<C>(v.x + ridge, (Th)0);
    A[i * LD + j] = v;
  }
  __syncthreads();
  for (int k = 0; k < K; ++k) {
    if (threadIdx.x == 0) {
      const Th pv = A[k * LD + k].x;
      if (!(pv > (Th)0)) atomicCAS(info, 0, p + 1);
      pinv_s = (Th)1 / pv;
    }
    __syncthreads();
    const Th pinv = pinv_s;
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
      rowk[j] = cscale(A[k * LD + j], pinv);
      colk[j] = A[j * LD + k];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = threadIdx.x >> 5; i < K; i += nw) {
      C* Ai = A + i * LD;
      if (i == k) {
        for (int j = lane; j < K; j += 32) Ai[j] = j == k ? mkc<C>(pinv, (Th)0) : rowk[j];
      } else {
        const C ci = colk[i];
        for (int j = lane; j < K; j += 32) {
          if (j == k) {
            Ai[j] = cscale(ci, -pinv);
          } else {
            const C rj = rowk[j];
            C a = Ai[j];
            a.x -= ci.x * rj.x - ci.y * rj.y;
            a.y -= ci.x * rj.y + ci.y * rj.x;
            Ai[j] = a;
          }
        }
      }
    }
    __syncthreads();
  }
  cx<Ti>* out = inv + (int64_t)p * npk;
  for (int64_t e = threadIdx.x; e < npk; e += blockDim.x) {
    // packed (i, j), j <= i
    int i = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
    while ((int64_t)i * (i + 1) / 2 > e) --i;
    while ((int64_t)(i + 1) * (i + 2) / 2 <= e) ++i;
    const int j = (int)(e - (int64_t)i * (i + 1) / 2);
    out[e] = ccast<Ti>(cscale(A[i * LD + j], scale));
  }
}

// Register-blocked Gauss-Jordan for moderate K (the BASELINE K = 100): thread t owns the
// BI x BJ block of A at (bi*BI, bj*BJ) in registers for all K steps; per step only row k and
// column k travel through shared memory, so shared traffic is O(K) instead of O(K^2).
template <typename Th, typename Ti, int BI, int BJ>
__global__ void __launch_bounds__(512, 1) k_hist_invert_reg(int K, const cx<Th>* __restrict__ S, Th ridge, Th scale,
                                                            cx<Ti>* inv, int32_t* info, int nfreq, int* ctr) {
  using C = cx<Th>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // row k / column k / 1 / pivot, double-buffered by step parity: the owners of step k + 1
  // publish while the others may still read step k's copies, so one barrier per step suffices
  C* rowb = reinterpret_cast<C*>(smem_raw);  // [2][K]
  C* colb = rowb + 2 * K;                    // [2][K]
  __shared__ Th piv_b[2];
  // ctr == null: one frequency per CTA (p = blockIdx.x); otherwise a persistent grid that claims
  // frequencies from *ctr (a few CTAs can run beside another kernel and a later full grid finishes)
  __shared__ int pclaim;
  for (int it = 0;; ++it) {
    int p;
    if (ctr) {
      if (threadIdx.x == 0) pclaim = atomicAdd(ctr, 1);
      __syncthreads();
      p = pclaim;
      __syncthreads();
      if (p >= nfreq) break;
    } else {
      if (it > 0) break;
      p = blockIdx.x;
    }
    const int64_t npk = (int64_t)K * (K + 1) / 2;
    const C* Sp = S + (int64_t)p * npk;
    const int tjn = (K + BJ - 1) / BJ, tin = (K + BI - 1) / BI;
    const int t = threadIdx.x;
    const bool active = t < tin * tjn;
    const int i0 = active ? (t / tjn) * BI : K, j0 = active ? (t % tjn) * BJ : K;
    C a[BI][BJ];
  #pragma unroll
    for (int ii = 0; ii < BI; ++ii)
  #pragma unroll
      for (int jj = 0; jj < BJ; ++jj) {
        const int i = i0 + ii, j = j0 + jj;
        C v = mkc<C>(0, 0);
        if (i < K && j < K) {
          v = i >= j ? Sp[packed_index(i, j)] : cconj(Sp[packed_index(j, i)]);
          if (i == j) v = mkc<C>(v.x + ridge, (Th)0);
        }
        a[ii][jj] = v;
      }
    for (int k = 0; k < K; ++k) {
      C* rowk = rowb + (k & 1) * K;
      C* colk = colb + (k & 1) * K;
      const bool own_row = k >= i0 && k < i0 + BI, own_col = k >= j0 && k < j0 + BJ;
      // publish row k and column k (only their owners)
      if (own_row) {
  #pragma unroll
        for (int ii = 0; ii < BI; ++ii)
          if (i0 + ii == k)
  #pragma unroll
            for (int jj = 0; jj < BJ; ++jj) {
              if (j0 + jj < K) rowk[j0 + jj] = a[ii][jj];
              if (j0 + jj == k) {  // pivot owner: one reciprocal per step for the whole CTA
                const Th d = a[ii][jj].x;
                piv_b[k & 1] = (Th)1 / d;
                if (!(d > (Th)0)) atomicCAS(info, 0, p + 1);
              }
            }
      }
      if (own_col) {
  #pragma unroll
        for (int jj = 0; jj < BJ; ++jj)
          if (j0 + jj == k)
  #pragma unroll
            for (int ii = 0; ii < BI; ++ii)
              if (i0 + ii < K) colk[i0 + ii] = a[ii][jj];
      }
      __syncthreads();
      const Th pinv = piv_b[k & 1];
      // generic rank-1 update with row/column k masked out (ci = 0 on row k, rs = 0 on column k)
      C rs[BJ];
  #pragma unroll
      for (int jj = 0; jj < BJ; ++jj) {
        const int j = j0 + jj;
        rs[jj] = (j < K && j != k) ? cscale(rowk[j], pinv) : mkc<C>(0, 0);
      }
  #pragma unroll
      for (int ii = 0; ii < BI; ++ii) {
        const int i = i0 + ii;
        const C ci = (i < K && i != k) ? colk[i] : mkc<C>(0, 0);
  #pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
          C& v = a[ii][jj];
          v.x = fma(-ci.x, rs[jj].x, fma(ci.y, rs[jj].y, v.x));
          v.y = fma(-ci.x, rs[jj].y, fma(-ci.y, rs[jj].x, v.y));
        }
      }
      // row k -> scaled row, column k -> -scaled column, pivot -> 1/pivot (owners only)
      if (own_row) {
  #pragma unroll
        for (int ii = 0; ii < BI; ++ii)
          if (i0 + ii == k)
  #pragma unroll
            for (int jj = 0; jj < BJ; ++jj) a[ii][jj] = (j0 + jj == k) ? mkc<C>(pinv, (Th)0) : rs[jj];
      }
      if (own_col) {
  #pragma unroll
        for (int jj = 0; jj < BJ; ++jj)
          if (j0 + jj == k)
  #pragma unroll
            for (int ii = 0; ii < BI; ++ii)
              if (i0 + ii != k && i0 + ii < K) a[ii][jj] = cscale(colk[i0 + ii], -pinv);
      }
    }
    cx<Ti>* out = inv + (int64_t)p * npk;
  #pragma unroll
    for (int ii = 0; ii < BI; ++ii)
  #pragma unroll
      for (int jj = 0; jj < BJ; ++jj) {
        const int i = i0 + ii, j = j0 + jj;
        if (i < K && j <= i) out[packed_index(i, j)] = ccast<Ti>(cscale(a[ii][jj], scale));
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
template <typename Tc, typename Th, typename Ti>
__global__ void __launch_bounds__(128) k_rowsolve(int K, int nf, const cx<Ti>* __restrict__ inv,
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
  const cx<Ti>* Ap = inv + (int64_t)p * npk;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    C acc = mkc<C>(0, 0);
    const cx<Ti>* row = Ap + packed_index(j, 0);
    C acc2 = mkc<C>(0, 0);  // second chain: loads of both loops issue 8 ahead
#pragma unroll 8
    for (int k = 0; k <= j; ++k) cfma(acc, ccast<Th>(row[k]), rhs[k]);
#pragma unroll 8
    for (int k = j + 1; k < K; ++k) cfmac(acc2, ccast<Th>(Ap[packed_index(k, j)]), rhs[k]);
    acc = cadd(acc, acc2);
    Dh[(int64_t)j * sk + (int64_t)p * sp] = mkc<cx<Tc>>((Tc)acc.x, (Tc)-acc.y);
  }
}

}  // namespace ocsc

using namespace ocsc;

static size_t csize(int dtype) { return dtype == OCSC_F64 ? 16 : 8; }

// Low-rank refresh of a packed Hermitian inverse (Woodbury):
//   (A + U U^H)^-1 = A^-1 - W (I + U^H W)^-1 W^H,  W = A^-1 U,  U = the nb new code spectra (K x nb)
// One CTA per frequency; A^-1 (packed, f64) is staged in shared memory, the nb x nb capacitance
// matrix is inverted by one warp (nb is a mini-batch remainder, <= 16).  Lets the trainer
// invert S + (most of the batch) while the rest of the batch is still being coded.  Shared
// memory: A^-1, U in the codes' own precision, W, the capacitance and one row of X = W C^-1 per
// warp (formed where the output phase needs it): K = 100 with nb <= 11 stays under 113 KB, so two
// CTAs share an SM (config 1: nb = 9, config 2: nb = 10).
template <typename Tz, typename To>
__global__ void __launch_bounds__(512, 2) k_hist_woodbury(int K, int nb, const double2* __restrict__ inv_in,
                                                         const typename Cx<Tz>::type* __restrict__ z, int64_t zb,
                                                         int64_t zk, int64_t zp, typename Cx<To>::type* out,
                                                         int32_t* info, const typename Cx<Tz>::type* __restrict__ x,
                                                         int64_t xb, int64_t xp, double2* S, double2* cvec) {
  using C = double2;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int p = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  const int nbp = nb | 1;  // odd row pitch (complex): lanes along K hit distinct bank groups
  using CZ = typename Cx<Tz>::type;
  C* A = reinterpret_cast<C*>(smraw);  // packed A^-1
  C* Wm = A + npk;                     // [K][nbp]  W = A^-1 U
  C* Cm = Wm + K * nbp;                // [nb][nb] capacitance, inverted in place
  C* Xr = Cm + nb * nb;                // [16 warps][16] the output phase's row of X = W Cinv
  CZ* U = reinterpret_cast<CZ*>(Xr + 16 * 16);  // [K][nbp] the new codes, own precision
  auto up = [](CZ v) { return make_double2((double)v.x, (double)v.y); };
  const double2* Ap = inv_in + (int64_t)p * npk;
  for (int64_t e = tid; e < npk; e += nt) cp_async<16>(A + e, Ap + e);  // all in flight at once
  cp_async_commit();
  if (S)  // the final phase read-modify-writes this frequency's S: bring it into L2 meanwhile
    for (int64_t l = tid; l < (npk * 16 + 127) / 128; l += nt)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(S + (int64_t)p * npk) + l * 128));
  for (int e = tid; e < K * nb; e += nt) {
    const int k = e / nb, j = e - k * nb;
    U[k * nbp + j] = z[j * zb + k * zk + p * zp];
  }
  cp_async_wait<0>();
  __syncthreads();
  // W[t][j] = sum_{k<=t} A[t][k] U[k][j] + sum_{i>t} conj(A[i][t]) U[i][j]: the packed row of t,
  // then its packed column (K terms for every t, branch-free), two interleaved accumulators
  for (int e = tid; e < K * nb; e += nt) {
    const int t = e / nb, j = e - t * nb;
    C a0 = make_double2(0, 0), a1 = make_double2(0, 0);
    const C* row = A + packed_index(t, 0);
    int k = 0;
    for (; k + 1 <= t; k += 2) {
      cfma(a0, row[k], up(U[k * nbp + j]));
      cfma(a1, row[k + 1], up(U[(k + 1) * nbp + j]));
    }
    if (k <= t) cfma(a0, row[k], up(U[k * nbp + j]));
    int i = t + 1;
    int64_t q = packed_index(i, t);  // packed (i, t): advances by i + 1 per row
    for (; i + 1 < K; i += 2) {
      cfma(a0, cconj(A[q]), up(U[i * nbp + j]));
      q += i + 1;
      cfma(a1, cconj(A[q]), up(U[(i + 1) * nbp + j]));
      q += i + 2;
    }
    if (i < K) cfma(a0, cconj(A[q]), up(U[i * nbp + j]));
    Wm[t * nbp + j] = make_double2(a0.x + a1.x, a0.y + a1.y);
  }
  __syncthreads();
  {  // C = I + U^H W: one warp per entry, lanes split the K-sum, shuffle reduction
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int e = warp; e < nb * nb; e += nw) {
      const int a = e / nb, b = e - a * nb;
      double ax = 0, ay = 0;
      for (int k = lane; k < K; k += 32) {
        const C u = up(U[k * nbp + a]), w = Wm[k * nbp + b];
        ax += u.x * w.x + u.y * w.y;  // conj(u) w
        ay += u.x * w.y - u.y * w.x;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ax += __shfl_xor_sync(0xffffffffu, ax, o);
        ay += __shfl_xor_sync(0xffffffffu, ay, o);
      }
      if (lane == 0) Cm[e] = make_double2(ax + (a == b ? 1.0 : 0.0), ay);
    }
  }
  __syncthreads();
  if (tid < 32) {  // in-place Gauss-Jordan of the nb x nb HPD capacitance matrix, one warp
    constexpr int PER = 8;  // entries per lane (nb <= 16)
    for (int k = 0; k < nb; ++k) {
      const double d = Cm[k * nb + k].x;
      if (tid == 0 && !(d > 0)) atomicCAS(info, 0, p + 1);
      const double pinv = 1.0 / d;
      C nv[PER];
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int e = tid + 32 * r;
        if (e >= nb * nb) break;
        const int i = e / nb, j = e - i * nb;
        const C cij = Cm[e], cik = Cm[i * nb + k], ckj = Cm[k * nb + j];
        if (i == k && j == k) nv[r] = make_double2(pinv, 0);
        else if (i == k) nv[r] = cscale(ckj, pinv);
        else if (j == k) nv[r] = cscale(cik, -pinv);
        else nv[r] = make_double2(cij.x - pinv * (cik.x * ckj.x - cik.y * ckj.y),
                                  cij.y - pinv * (cik.x * ckj.y + cik.y * ckj.x));
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int e = tid + 32 * r;
        if (e >= nb * nb) break;
        Cm[e] = nv[r];
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (S) {  // fold the same samples into the history sums: c_p += sum_b conj(x_b) z_b
    for (int k = tid; k < K; k += nt) {
      C acc = cvec[(int64_t)p * K + k];
      for (int m = 0; m < nb; ++m) {
        const auto xv = x[m * xb + p * xp];
        const C u = up(U[k * nbp + m]);
        acc.x += (double)xv.x * u.x + (double)xv.y * u.y;
        acc.y += (double)xv.x * u.y - (double)xv.y * u.x;
      }
      cvec[(int64_t)p * K + k] = acc;
    }
  }
  double2* Sp = S ? S + (int64_t)p * npk : nullptr;
  typename Cx<To>::type* o = out + (int64_t)p * npk;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  C* xr = Xr + warp * 16;
  for (int i = warp; i < K; i += nw) {
    if (lane < nb) {  // row i of X = W Cinv
      C acc = make_double2(0, 0);
      for (int m = 0; m < nb; ++m) cfma(acc, Wm[i * nbp + m], Cm[m * nb + lane]);
      xr[lane] = acc;
    }
    __syncwarp();
    for (int j = lane; j <= i; j += 32) {  // out[i][j] = A^-1[i][j] - sum_m X[i][m] conj(W[j][m])
      C sv = Sp ? Sp[packed_index(i, j)] : make_double2(0, 0);  // (issued first: its latency overlaps)
      C acc = A[packed_index(i, j)];
      for (int m = 0; m < nb; ++m) {
        const C x = xr[m], w = Wm[j * nbp + m];
        acc.x -= x.x * w.x + x.y * w.y;
        acc.y -= x.y * w.x - x.x * w.y;
      }
      o[packed_index(i, j)] = ccast<To>(acc);
      if (Sp) {  // S_p[i][j] += sum_m U[i][m] conj(U[j][m])
        for (int m = 0; m < nb; ++m) {
          const C ui = up(U[i * nbp + m]), uj = up(U[j * nbp + m]);
          sv.x += ui.x * uj.x + ui.y * uj.y;
          sv.y += ui.y * uj.x - ui.x * uj.y;
        }
        Sp[packed_index(i, j)] = sv;
      }
    }
    __syncwarp();  // xr is rewritten for the next row
  }
}

static size_t woodbury_smem(int K, int nb, size_t zsize) {
  return sizeof(double2) * ((size_t)K * (K + 1) / 2 + (size_t)K * (nb | 1) + (size_t)nb * nb + 16 * 16) +
         zsize * (size_t)K * (nb | 1);
}
extern "C" size_t ocsc_history_woodbury_smem(int K, int nb) { return woodbury_smem(K, nb, 16); }

extern "C" int ocsc_history_woodbury(int dtype_z, int dtype_out, int K, int nfreq, int nb, const void* inv_in,
                                     const void* z, int64_t z_sb, int64_t z_sk, int64_t z_sp, void* out,
                                     int32_t* info, const void* x, int64_t x_sb, int64_t x_sp, void* S, void* c,
                                     void* stream) {
  if (K <= 0 || nfreq < 0 || nb < 0 || nb > 16) return fail(OCSC_ESHAPE, "history_woodbury: bad extents (nb <= 16)");
  if ((S != nullptr) != (c != nullptr) || (S && !x)) return fail(OCSC_EARG, "history_woodbury: S, c and x go together");
  cudaStream_t s = as_stream(stream);
  OCSC_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
  if (nfreq == 0) return OCSC_OK;
  const size_t sm = woodbury_smem(K, nb, dtype_z == OCSC_F32 ? 8 : 16);
  if (sm > 227 * 1024) return fail(OCSC_EARG, "history_woodbury: K too large for the shared-memory inverse");
#define OCSC_WB(TZ, TO)                                                                                        \
  do {                                                                                                         \
    OCSC_CUDA(cudaFuncSetAttribute(k_hist_woodbury<TZ, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                   (int)sm));                                                                  \
    k_hist_woodbury<TZ, TO><<<nfreq, 512, sm, s>>>(K, nb, (const double2*)inv_in,                               \
                                                   (const typename Cx<TZ>::type*)z, z_sb, z_sk, z_sp,           \
                                                   (typename Cx<TO>::type*)out, info,                          \
                                                   (const typename Cx<TZ>::type*)x, x_sb, x_sp, (double2*)S,    \
                                                   (double2*)c);                                               \
  } while (0)
  if (dtype_z == OCSC_F32 && dtype_out == OCSC_F32) OCSC_WB(float, float);
  else if (dtype_z == OCSC_F32 && dtype_out == OCSC_F64) OCSC_WB(float, double);
  else if (dtype_z == OCSC_F64 && dtype_out == OCSC_F64) OCSC_WB(double, double);
  else if (dtype_z == OCSC_F64 && dtype_out == OCSC_F32) OCSC_WB(double, float);
  else return fail(OCSC_EARG, "history_woodbury: dtype must be 4 or 8");
#undef OCSC_WB
  OCSC_LAUNCHED("k_hist_woodbury");
  return OCSC_OK;
}

extern "C" int ocsc_history_accumulate(int dtype_in, int dtype_hist, int K, int nfreq, int B, const void* z,
                                       int64_t z_sb, int64_t z_sk, int64_t z_sp, const void* x, int64_t x_sb,
                                       int64_t x_sp, void* S, void* c, void* stream) {
  if (K <= 0 || nfreq < 0 || B < 0) return fail(OCSC_ESHAPE, "history_accumulate: bad extents");
  if (nfreq == 0 || B == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype_in == OCSC_F32 && K >= 96 && use_tensor_cores())
    return history_accumulate_tc(dtype_hist, K, nfreq, B, z, z_sb, z_sk, z_sp, x, x_sb, x_sp, S, c, s);
  if (dtype_in == OCSC_F32 && K >= 48) {
    const int nb = (K + HT - 1) / HT, pairs = nb * (nb + 1) / 2;
    const int64_t grid = (int64_t)nfreq * pairs;
    if (grid > 0x7fffffff) return fail(OCSC_EARG, "history_accumulate: too many blocks");
    if (dtype_hist == OCSC_F32)
      k_hist_accum_tiled<float><<<(unsigned)grid, 256, 0, s>>>(K, B, (const float2*)z, z_sb, z_sk, z_sp,
                                                                (const float2*)x, x_sb, x_sp, (float2*)S, (float2*)c,
                                                                pairs);
    else if (dtype_hist == OCSC_F64)
      k_hist_accum_tiled<double><<<(unsigned)grid, 256, 0, s>>>(K, B, (const float2*)z, z_sb, z_sk, z_sp,
                                                                 (const float2*)x, x_sb, x_sp, (double2*)S,
                                                                 (double2*)c, pairs);
    else
      return fail(OCSC_EARG, "history_accumulate: unsupported dtype pair");
    OCSC_LAUNCHED("k_hist_accum_tiled");
    return OCSC_OK;
  }
  const size_t cs = csize(dtype_in);
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

template <typename Th, typename Ti>
static int launch_invert(int K, int nfreq, const void* S, double ridge, double scale, void* inv, int32_t* info,
                         cudaStream_t s) {
  if (K > 32 && K <= 100) {
    // register-blocked path: 4 x 5 blocks, ceil(K/4) * ceil(K/5) <= 500 threads
    const int threads = ((((K + 3) / 4) * ((K + 4) / 5)) + 31) / 32 * 32;
    const size_t sm = sizeof(cx<Th>) * 4 * (size_t)K;
    k_hist_invert_reg<Th, Ti, 4, 5><<<nfreq, threads, sm, s>>>(K, (const cx<Th>*)S, (Th)ridge, (Th)scale,
                                                              (cx<Ti>*)inv, info, nfreq, nullptr);
    OCSC_LAUNCHED("k_hist_invert_reg");
    return OCSC_OK;
  }
  const size_t smem = sizeof(cx<Th>) * ((size_t)K * (K + 1) + 2 * (size_t)K);
  if (smem > 227 * 1024)
    return fail(OCSC_EARG, "history_invert: K=" + std::to_string(K) +
                               " exceeds the shared-memory inverse (K<=118 complex128, K<=167 complex64)");
  OCSC_CUDA(cudaFuncSetAttribute(k_hist_invert<Th, Ti>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_hist_invert<Th, Ti><<<nfreq, 512, smem, s>>>(K, (const cx<Th>*)S, (Th)ridge, (Th)scale, (cx<Ti>*)inv, info);
  OCSC_LAUNCHED("k_hist_invert");
  return OCSC_OK;
}

extern "C" int ocsc_history_invert(int dtype_hist, int dtype_inv, int K, int nfreq, const void* S, double ridge,
                                   double scale, void* inv, int32_t* info, void* stream) {
  if (K <= 0 || nfreq < 0) return fail(OCSC_ESHAPE, "history_invert: bad extents");
  cudaStream_t s = as_stream(stream);
  OCSC_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
  if (nfreq == 0) return OCSC_OK;
  if (dtype_hist == OCSC_F64 && dtype_inv == OCSC_F64) return launch_invert<double, double>(K, nfreq, S, ridge, scale, inv, info, s);
  if (dtype_hist == OCSC_F64 && dtype_inv == OCSC_F32) return launch_invert<double, float>(K, nfreq, S, ridge, scale, inv, info, s);
  if (dtype_hist == OCSC_F32 && dtype_inv == OCSC_F32) return launch_invert<float, float>(K, nfreq, S, ridge, scale, inv, info, s);
  return fail(OCSC_EARG, "history_invert: unsupported dtype pair");
}

// Persistent variant of the register-blocked inverse (32 < K <= 100): `ctas` CTAs claim
// frequencies from the device counter *ctr (zeroed by the caller before the first launch) until
// none are left.  Two launches sharing the counter split the work: e.g. a few CTAs beside the
// streaming code kernel, then a full grid after it.  info is not reset here.
extern "C" int ocsc_history_invert_claim(int dtype_hist, int dtype_inv, int K, int nfreq, const void* S,
                                         double ridge, double scale, void* inv, int32_t* info, int32_t* ctr,
                                         int ctas, void* stream) {
  if (K <= 32 || K > 100 || nfreq < 0 || ctas <= 0) return fail(OCSC_ESHAPE, "history_invert_claim: 32 < K <= 100");
  cudaStream_t s = as_stream(stream);
  if (nfreq == 0) return OCSC_OK;
  const int threads = ((((K + 3) / 4) * ((K + 4) / 5)) + 31) / 32 * 32;
  const size_t sm = csize(dtype_hist) * 4 * (size_t)K;
#define OCSC_GJC(TH, TI)                                                                                        \
  k_hist_invert_reg<TH, TI, 4, 5><<<ctas, threads, sm, s>>>(K, (const cx<TH>*)S, (TH)ridge, (TH)scale,         \
                                                            (cx<TI>*)inv, info, nfreq, (int*)ctr)
  if (dtype_hist == OCSC_F64 && dtype_inv == OCSC_F64) OCSC_GJC(double, double);
  else if (dtype_hist == OCSC_F64 && dtype_inv == OCSC_F32) OCSC_GJC(double, float);
  else if (dtype_hist == OCSC_F32 && dtype_inv == OCSC_F32) OCSC_GJC(float, float);
  else return fail(OCSC_EARG, "history_invert_claim: unsupported dtype pair");
#undef OCSC_GJC
  OCSC_LAUNCHED("k_hist_invert_reg");
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

extern "C" int ocsc_dict_rowsolve(int dtype, int dtype_hist, int dtype_inv, int K, int nfreq, const void* inv,
                                  const void* c, double ridge, const void* Vh, const void* Th, int64_t sk, int64_t sp,
                                  void* Dh, void* stream) {
  if (K <= 0 || nfreq < 0) return fail(OCSC_ESHAPE, "dict_rowsolve: bad extents");
  if (nfreq == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  const size_t smem = csize(dtype_hist) * K;
#define RS(TC, TH, TI)                                                                                   \
  k_rowsolve<TC, TH, TI><<<nfreq, 128, smem, s>>>(K, nfreq, (const cx<TI>*)inv, (const cx<TH>*)c, (TH)ridge, \
                                                  (const cx<TC>*)Vh, (const cx<TC>*)Th, sk, sp, (cx<TC>*)Dh)
  if (dtype == OCSC_F32 && dtype_hist == OCSC_F32 && dtype_inv == OCSC_F32) RS(float, float, float);
  else if (dtype == OCSC_F32 && dtype_hist == OCSC_F64 && dtype_inv == OCSC_F64) RS(float, double, double);
  else if (dtype == OCSC_F32 && dtype_hist == OCSC_F64 && dtype_inv == OCSC_F32) RS(float, double, float);
  else if (dtype == OCSC_F64 && dtype_hist == OCSC_F64 && dtype_inv == OCSC_F64) RS(double, double, double);
  else return fail(OCSC_EARG, "dict_rowsolve: unsupported dtype combination");
#undef RS
  OCSC_LAUNCHED("k_rowsolve");
  return OCSC_OK;
}
