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
#include <cstdlib>

#include "common.cuh"
#include "fft_small.cuh"
#include "transforms.cuh"

namespace ocsc {

using sfft::static_for;
constexpr int CT = 32;  // tile edge

// optional phase stamps of CTA 0 (development aid): [0] start, [1] after the expansion, [2] after
// diag(0), then per step kb: [3+4kb] panel done, [4+4kb] trailing queue start, [5+4kb] next
// diagonal tile factored, [6+4kb] step done (clock64)
__device__ long long* g_chol_prof = nullptr;

template <typename C>
__device__ __forceinline__ C* tile_ptr(C* L, int K, int ib, int jb) {
  return L + (int64_t)ib * CT * K + (int64_t)jb * CT;
}

template <typename T>
__host__ __device__ constexpr int chol_panel_offset() {
  // L_kk [CT + 8][CT+1] complex (8 padding rows read by the diagonal factor's unrolled groups) +
  // 1/L_jj [CT] real, rounded up to 16 bytes
  return (int)(((sizeof(cx<T>) * (CT + 8) * (CT + 1) + sizeof(T) * (CT + 2)) + 15) / 16 * 16);
}

// two consecutive complex values from 16-byte aligned shared memory (one 16-byte load for float)
__device__ __forceinline__ void ld2(const float2* p, float2& a, float2& b) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  a = make_float2(v.x, v.y);
  b = make_float2(v.z, v.w);
}
__device__ __forceinline__ void ld2(const double2* p, double2& a, double2& b) {
  a = p[0];
  b = p[1];
}
// panel row position: inside each 32-row group, rows 4c + q (c = 0..7, q = 0..3) are stored as
// [q = 0,1 of c = 0..7][q = 2,3 of c = 0..7], so four consecutive rows are two aligned pairs and the
// same pair of eight consecutive c is 128 contiguous bytes (float)
__device__ __forceinline__ int ppos(int r) { return (r & ~31) | (((r >> 1) & 1) << 4) | (((r >> 2) & 7) << 1) | (r & 1); }

// acc += a * conj(b) on 2-wide FP32 (FFMA2) / FP64 pairs: acc += a * b.x + (a.y, -a.x) * b.y
template <typename C>
__device__ __forceinline__ void cmac_conj2(C& acc, C a, C as, decltype(C::x) bx, decltype(C::x) by) {
  acc = vfma(a, vsplat<C>(bx), acc);
  acc = vfma(as, vsplat<C>(by), acc);
}

// explicit shared-memory complex loads / stores (32-bit shared addresses: LDS / STS even where a
// generic pointer would lose its address space)
template <typename C>
__device__ __forceinline__ C lds_c(uint32_t a);
template <>
__device__ __forceinline__ float2 lds_c<float2>(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
template <>
__device__ __forceinline__ double2 lds_c<double2>(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_c(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void sts_c(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// predicated store (no branch around the volatile asm)
__device__ __forceinline__ void sts_c_if(bool c, uint32_t a, float2 v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.shared.v2.f32 [%0], {%1, %2};\n}" ::"r"(a),
               "f"(v.x), "f"(v.y), "r"((int)c)
               : "memory");
}
__device__ __forceinline__ void sts_c_if(bool c, uint32_t a, double2 v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(a),
               "d"(v.x), "d"(v.y), "r"((int)c)
               : "memory");
}

// Cholesky of one CT x CT diagonal tile by one warp (lane = row), in place in shared memory
// (sD: [CT + 8][CT + 1] complex, the last 8 rows padding), the lower triangle read from and written back to `tile` (global,
// row stride K); 1 / L_jj into dinv.  Right-looking, one column per step: every lane reads the
// pivot (broadcast), the rows below scale their entry of column j, then update their row of the
// trailing triangle from the column (broadcast reads).  Rolled loops keep the routine small: it
// runs once per tile column on the critical path, beside the trailing update of the other warps.
// (A register-resident, fully unrolled variant is faster alone -- 13.6 k against 21.4 k cycles per
// tile, scripts/diag_bench.cu -- but spills inside this kernel's 128-register budget.)
template <typename T>
__device__ __noinline__ void diag_tile(cx<T>* tile, int K, uint32_t sD, T* dinv, int lane, int32_t* info, int p) {
  using C = cx<T>;
  constexpr int LD = CT + 1;
  constexpr uint32_t SZ = sizeof(C);
  const C* row = tile + (int64_t)lane * K;
#pragma unroll 8
  for (int j = 0; j < CT; ++j) sts_c(sD + (uint32_t)(lane * LD + j) * SZ, j <= lane ? row[j] : mkc<C>(0, 0));
  __syncwarp();
#pragma unroll 1
  for (int j = 0; j < CT; ++j) {
    T d = lds_c<C>(sD + (uint32_t)(j * LD + j) * SZ).x;
    if (!(d > (T)0)) {
      if (lane == 0) atomicCAS(info, 0, p + 1);
      d = (T)NAN;
    }
    T ljj, inv;
    if constexpr (sizeof(T) == 4) {  // one MUFU rsqrt + a Newton step (< 1 ulp off IEEE)
      const T y = rsqrtf(d);
      inv = y * ((T)1.5 - (T)0.5 * d * y * y);
      ljj = d * inv;
    } else {
      ljj = sqrt(d);
      inv = (T)1 / ljj;
    }
    const uint32_t own = sD + (uint32_t)(lane * LD) * SZ;
    // (loads are unconditional and stores predicated: no branches around the shared-memory asm; a
    // row's entries past column 31 -- the pad column, the next row -- and the rows past 31 -- the
    // tile's 8 padding rows -- only feed values that are never stored)
    const C aij = lds_c<C>(own + j * SZ);
    const C lij = lane > j ? cscale(aij, inv) : mkc<C>(0, 0);
    sts_c_if(lane >= j, own + j * SZ, lane == j ? mkc<C>(ljj, (T)0) : lij);
    if (lane == 0) dinv[j] = inv;
    __syncwarp();
    // D[i][k] -= L[i][j] conj(L[k][j]),  j < k <= i: eight columns at a time, all sixteen loads
    // issued before the first store (the shared-memory asm keeps program order)
    // (t -= lij conj(lk) as two 2-wide FMAs: t + lij (-lk.x) + swap(lij) (-lk.y, lk.y); addresses are
    // a per-group base plus immediates)
#pragma unroll 1
    for (int k0 = j + 1; k0 < CT; k0 += 8) {
      const uint32_t colk = sD + (uint32_t)(k0 * LD + j) * SZ, rowk = own + k0 * SZ;
      C lk[8], t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) lk[u] = lds_c<C>(colk + u * LD * SZ);
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = lds_c<C>(rowk + u * SZ);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        t[u] = vfma(lij, vsplat<C>(-lk[u].x), t[u]);
        t[u] = vfma(vswap(lij), mkc<C>(-lk[u].y, lk[u].y), t[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) sts_c_if(k0 + u <= lane, rowk + u * SZ, t[u]);
    }
    __syncwarp();
  }
  C* out = tile + (int64_t)lane * K;
#pragma unroll 8
  for (int j = 0; j < CT; ++j) {
    const C v = lds_c<C>(sD + (uint32_t)(lane * LD + j) * SZ);
    if (j <= lane) out[j] = v;
  }
}

// A (packed lower, K(K+1)/2 per frequency) + ridge I -> full-layout lower L = chol(A).
// One CTA (256 threads) per frequency, right-looking over 32-wide tile columns:
//   diagonal tile: warp 0, lane = row, the row in registers, 32 shuffle steps (no CTA barrier);
//   panel:         thread per row, X = A L_kk^-H by substitution against L_kk in SMEM;
//                  the panel is also written transposed (k-major) into SMEM;
//   trailing:      A22 -= P P^H over the lower triangle as 64 x 64 block pairs, 16 x 16 threads
//                  x 4 x 4 complex, two 2-wide FMAs per complex multiply-add (HERK microkernel);
//                  target values are loaded before the products so their latency overlaps them.
// NT = 256 (8 warps; two CTAs per SM where shared memory allows) or 512 (16 warps, two 64 x 64
// block pairs of the trailing update at a time: K = 512, where one CTA fills the SM anyway)
template <typename T, int NT>
__global__ void __launch_bounds__(NT, (sizeof(T) == 8 || NT >= 512) ? 1 : (NT >= 256 ? 2 : 3)) k_chol_blocked(int K, int Kv, const cx<T>* __restrict__ S, T ridge,
                                                          cx<T>* Lall, int32_t* info) {
  // K: factored order (a multiple of 32); Kv <= K: the history's order (S packed with Kv). Rows
  // and columns Kv..K-1 are the decoupled padding ridge * I, so L = diag(chol(A), sqrt(ridge) I).
  using C = cx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int LD = CT + 1;
  C* D = reinterpret_cast<C*>(smem_raw);  // L_kk [CT][LD]
  T* dinv = reinterpret_cast<T*>(D + (CT + 8) * LD);  // 1 / L_jj [CT] (after the padded tile)
  C* PT = reinterpret_cast<C*>(smem_raw + chol_panel_offset<T>());  // panel, k-major: PT[k][r]
  const uint32_t sD = (uint32_t)__cvta_generic_to_shared(D);
  const int nb = K / CT;
  const int p = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t npk = (int64_t)Kv * (Kv + 1) / 2;
  const C* Sp = S + (int64_t)p * npk;
  C* L = Lall + (int64_t)p * K * K;
  const int PR = K - CT;  // panel row stride (k-major panel, rows pair-interleaved within 32-row groups)
  long long* prof = (blockIdx.x == 0 && threadIdx.x == 0) ? g_chol_prof : nullptr;
  if (prof) prof[0] = clock64();

  // expand the packed lower triangle (+ ridge) into the lower half of the full layout; each
  // lane issues up to 8 loads of its row before storing (the copy is latency-bound otherwise)
  for (int i = warp; i < K; i += NT / 32) {
    const C* src = Sp + packed_index(i, 0);
    C* dst = L + (int64_t)i * K;
    for (int j0 = lane; j0 <= i; j0 += 8 * 32) {
      C v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 32 * u;
        v[u] = j <= i && i < Kv ? src[j] : mkc<C>(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + 32 * u;
        if (j <= i) dst[j] = j == i ? mkc<C>(v[u].x + ridge, (T)0) : v[u];
      }
    }
  }
  __syncthreads();
  if (prof) prof[1] = clock64();

  // ---- diagonal tile kbx: warp 0, the tile in shared memory (D, lane = row), rolled loops:
  // one column per step (broadcast pivot, scale the column, rank-1 update of the rows below)
  auto diag = [&](int kbx) {
    diag_tile<T>(L + (int64_t)(kbx * CT) * K + kbx * CT, K, sD, dinv, lane, info, p);
  };
  // ---- one warp's 32 x 32 tile (ti, tj), ti >= tj, of the trailing update A22 -= P P^H: lane
  // (ry, cx) = (lane / 8, lane % 8) owns rows 8 ry.. 8 ry + 7 and columns 4 cx.. 4 cx + 3 (8 x 4
  // complex accumulators, two 2-wide FMAs per complex multiply-add); per k the eight lanes of a
  // quarter-warp read one broadcast 16-byte pair of the row operand and eight consecutive pairs
  // of the column operand (the pair-interleaved panel layout, ppos), so every shared load is one
  // wavefront; the targets are read-modified-written once, coalesced, after the k loop ----
  auto tile_upd = [&](int r0, int ti, int tj) {
    const int ry = lane >> 3, cx = lane & 7;
    const int j0 = tj * CT + 4 * cx;
    // the targets come from DRAM (the factors of the frequencies in flight exceed L2): ask for
    // them now, read them after the k loop
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const C* t = L + (int64_t)(r0 + ti * CT + 8 * ry + r) * K + r0 + j0;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(t));
    }
    C acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = mkc<C>(0, 0);
    const C* pi = PT + ti * CT + 4 * ry;
    const C* pj = PT + tj * CT + 2 * cx;
#pragma unroll 2
    for (int k = 0; k < CT; ++k) {
      C zi[8], zj[4];
      ld2(pi + k * PR, zi[0], zi[1]);            // rows 8 ry + 0, 1
      ld2(pi + k * PR + 16, zi[2], zi[3]);       //            2, 3
      ld2(pi + k * PR + 2, zi[4], zi[5]);        //            4, 5
      ld2(pi + k * PR + 18, zi[6], zi[7]);       //            6, 7
      ld2(pj + k * PR, zj[0], zj[1]);            // columns 4 cx + 0, 1
      ld2(pj + k * PR + 16, zj[2], zj[3]);       //                2, 3
      // acc += zi conj(zj) = zi * zj.x + swap(zi) * (zj.y, -zj.y): the swap is an operand swizzle of
      // the 2-wide FMA, so a complex multiply-add is two FFMA2 and the sign vector costs one op per zj
      C zn[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) zn[q] = mkc<C>(zj[q].y, -zj[q].y);
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[r][q] = vfma(zi[r], vsplat<C>(zj[q].x), acc[r][q]);
          acc[r][q] = vfma(vswap(zi[r]), zn[q], acc[r][q]);
        }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = ti * CT + 8 * ry + r;
      C* dst = L + (int64_t)(r0 + i) * K + r0 + j0;
      C t[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = j0 + q <= i ? dst[q] : mkc<C>(0, 0);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (j0 + q <= i) dst[q] = csub(t[q], acc[r][q]);
    }
  };
  __shared__ int ctr;

  if (warp == 0) diag(0);
  __syncthreads();
  if (prof) prof[2] = clock64();
  for (int kb = 0; kb < nb; ++kb) {
    const int r0 = (kb + 1) * CT;  // first trailing row
    const int R = K - r0;          // trailing rows
    if (R == 0) break;
    // ---- panel: x L_kk^H = a for every trailing row (thread per row) ----
    for (int rr = tid; rr < R; rr += NT) {
      C x[CT];
      C* row = L + (int64_t)(r0 + rr) * K + kb * CT;
#pragma unroll
      for (int j = 0; j < CT; ++j) x[j] = row[j];
      static_for<0, CT>([&](auto J) {
        constexpr int j = decltype(J)::value;
        // acc -= x_k conj(L_jk) = x_k (-l.x) + swap(x_k) (-l.y, l.y): two 2-wide FMAs (the swap and
        // the signs are FFMA2 operand modifiers); two partial sums keep the chains short
        C acc[2] = {x[j], mkc<C>(0, 0)};
        static_for<0, j>([&](auto Kk) {
          constexpr int k = decltype(Kk)::value;
          const C l = lds_c<C>(sD + (uint32_t)((j * LD + k) * sizeof(C)));
          acc[k & 1] = vfma(x[k], vsplat<C>(-l.x), acc[k & 1]);
          acc[k & 1] = vfma(vswap(x[k]), mkc<C>(-l.y, l.y), acc[k & 1]);
        });
        x[j] = cscale(vadd(acc[0], acc[1]), dinv[j]);
      });
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        row[j] = x[j];
        PT[j * PR + ppos(rr)] = x[j];
      }
    }
    if (tid == 0) ctr = 0;
    __syncthreads();
    if (prof && kb < 16) prof[3 + 4 * kb] = clock64();
    // ---- trailing update, one dynamic queue of 32 x 32 tiles: first the next tile column (tiles
    // (ti, 0): the next diagonal tile and panel -- the lookahead), then the rest (tiles (ti, tj),
    // 1 <= tj <= ti).  The warp that finishes tile (0, 0) factors the next diagonal tile at once
    // and then rejoins the queue; the end-of-step barrier orders everything for the next panel ----
    const int nbr = R / CT;
    const int nT = nbr * (nbr + 1) / 2;
    if (prof && kb < 16) prof[4 + 4 * kb] = clock64();
    for (;;) {
      int q = 0;
      if (lane == 0) q = atomicAdd(&ctr, 1);
      q = __shfl_sync(0xffffffffu, q, 0);
      if (q >= nT) break;
      if (q < nbr) {
        tile_upd(r0, q, 0);
        if (q == 0) {
          __syncwarp();
          diag(kb + 1);
          if (blockIdx.x == 0 && lane == 0 && g_chol_prof && kb < 16) g_chol_prof[5 + 4 * kb] = clock64();
        }
      } else {
        const int qb = q - nbr;
        int b = (int)((sqrtf(8.0f * qb + 1.0f) - 1.0f) * 0.5f);
        while (b * (b + 1) / 2 > qb) --b;
        while ((b + 1) * (b + 2) / 2 <= qb) ++b;
        tile_upd(r0, b + 1, qb - b * (b + 1) / 2 + 1);
      }
    }
    __syncthreads();
    if (prof && kb < 16) prof[6 + 4 * kb] = clock64();
  }
}

// Whole-matrix Cholesky in shared memory for K <= 64 (config 4's K = 64): unblocked
// right-looking, one column per step, thread per trailing column.  Small CTAs (two warps,
// <= 65 KB) so many frequencies are in flight per SM; no global traffic besides reading S
// and writing L once.
template <typename T>
__global__ void __launch_bounds__(128) k_chol_smem(int K, const cx<T>* __restrict__ S, T ridge, cx<T>* Lall,
                                                   int32_t* info) {
  using C = cx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* A = reinterpret_cast<C*>(smem_raw);  // [K][K+1], lower triangle used
  const int LD = K + 1;
  const int p = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int npk = K * (K + 1) / 2;
  const C* Sp = S + (int64_t)p * npk;
  for (int e = tid; e < npk; e += nt) {  // flat, coalesced, independent loads of the packed triangle
    int i = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    while (i * (i + 1) / 2 > e) --i;
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    const int j = e - i * (i + 1) / 2;
    C v = Sp[e];
    if (i == j) v = mkc<C>(v.x + ridge, (T)0);
    A[i * LD + j] = v;
  }
  __syncthreads();
  for (int j = 0; j < K; ++j) {
    T d = A[j * LD + j].x;
    if (!(d > (T)0)) {
      if (tid == 0) atomicCAS(info, 0, p + 1);
      d = (T)NAN;
    }
    const T ljj = sqrt(d), inv = (T)1 / ljj;
    for (int i = j + 1 + tid; i < K; i += nt) A[i * LD + j] = cscale(A[i * LD + j], inv);
    __syncthreads();
    if (tid == 0) A[j * LD + j] = mkc<C>(ljj, (T)0);
    // trailing triangle: thread -> column k, rows i >= k; A[i][j] is a broadcast read and row i's
    // columns are contiguous across threads; the i loop carries no dependence (unrolled)
    for (int k = j + 1 + tid; k < K; k += nt) {
      const C lk = A[k * LD + j];
#pragma unroll 4
      for (int i = k; i < K; ++i) {
        const C lij = A[i * LD + j];
        C& t = A[i * LD + k];
        t.x -= lij.x * lk.x + lij.y * lk.y;  // lij conj(lk)
        t.y -= lij.y * lk.x - lij.x * lk.y;
      }
    }
    __syncthreads();
  }
  C* L = Lall + (int64_t)p * K * K;
  for (int i = 0; i < K; ++i)
    for (int j = tid; j <= i; j += nt) L[(int64_t)i * K + j] = A[i * LD + j];
}

template <int K>
constexpr int chol_reg_threads() {
  return ((K / 4) * (K / 4 + 1) / 2 + 31) / 32 * 32;
}

// Register-resident BLOCKED right-looking Cholesky (K <= 128): thread t owns the 4 x 4 block
// (bi, bj), bi >= bj, for the whole factorisation; one step per 4-wide block column kb:
//   1. the owner of (kb, kb) factors its block in registers and publishes L_kk;      barrier
//   2. the owners of (bi, kb), bi > kb, solve X L_kk^H = A_{bi,kb} in registers and publish X
//      into a parity-double-buffered panel;                                          barrier
//   3. every trailing owner (bj > kb) applies A_{bi,bj} -= X_bi X_bj^H (64 complex FMAs).
// Two barriers per 4 columns and a rank-4 update per thread.
template <typename T, int K>
__global__ void __launch_bounds__(chol_reg_threads<K>()) k_chol_rb(const cx<T>* __restrict__ S, T ridge,
                                                                    cx<T>* Lall, int32_t* info) {
  using C = cx<T>;
  constexpr int NB = K / 4, NTH = NB * (NB + 1) / 2;
  __shared__ __align__(16) C Lkk[4][4];
  __shared__ T Ldinv[4];  // 1 / L_kk[c][c]
  __shared__ __align__(16) C P[2][4][4][NB];  // element-major: lanes (consecutive blocks) hit consecutive words
  const int p = blockIdx.x, t = threadIdx.x;
  const bool act = t < NTH;
  // column-major block order: the blocks of early (finished) block columns are contiguous, so
  // whole warps retire from the trailing updates instead of running partially masked
  int bi = 0, bj = 0;
  if (act) {
    int off = 0;
    while (off + (NB - bj) <= t) {
      off += NB - bj;
      ++bj;
    }
    bi = bj + (t - off);
  }
  const int i0 = bi * 4, k0 = bj * 4;
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  const C* Sp = S + (int64_t)p * npk;
  C a[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + r, k = k0 + c;
      C v = mkc<C>(0, 0);
      if (act && i >= k) {
        v = Sp[packed_index(i, k)];
        if (i == k) v = mkc<C>(v.x + ridge, (T)0);
      }
      a[r][c] = v;
    }
  bool bad = false;
  for (int kb = 0; kb < NB; ++kb) {
    // ---- 1. diagonal block ----
    if (act && bi == kb && bj == kb) {
      static_for<0, 4>([&](auto Jc) {
        constexpr int j = decltype(Jc)::value;
        T d = a[j][j].x;
        if (!(d > (T)0)) {
          bad = true;
          d = (T)NAN;
        }
        T ljj, inv;
        if constexpr (sizeof(T) == 4) {  // one MUFU rsqrt + a Newton step (< 1 ulp off IEEE)
          const T y = rsqrtf(d);
          inv = y * ((T)1.5 - (T)0.5 * d * y * y);
          ljj = d * inv;
        } else {
          ljj = sqrt(d);
          inv = (T)1 / ljj;
        }
        a[j][j] = mkc<C>(ljj, (T)0);
        Ldinv[j] = inv;
        static_for<j + 1, 4>([&](auto Rr) { a[decltype(Rr)::value][j] = cscale(a[decltype(Rr)::value][j], inv); });
        static_for<j + 1, 4>([&](auto Cc) {
          constexpr int c = decltype(Cc)::value;
          const C lc = a[c][j];
          static_for<c, 4>([&](auto Rr) {  // a[r][c] -= L[r][j] conj(L[c][j])
            constexpr int r = decltype(Rr)::value;
            a[r][c].x -= a[r][j].x * lc.x + a[r][j].y * lc.y;
            a[r][c].y -= a[r][j].y * lc.x - a[r][j].x * lc.y;
          });
        });
      });
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) Lkk[r][c] = a[r][c];
    }
    __syncthreads();
    C (*Pb)[4][NB] = P[kb & 1];
    // ---- 2. panel: X L_kk^H = A (columns in order) ----
    if (act && bj == kb && bi > kb) {
      static_for<0, 4>([&](auto Cc) {
        constexpr int c = decltype(Cc)::value;
        const T inv = Ldinv[c];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          C x = a[r][c];
          static_for<0, c>([&](auto Mm) {  // x -= X[r][m] conj(L_kk[c][m])
            constexpr int m = decltype(Mm)::value;
            const C l = Lkk[c][m];
            x.x -= a[r][m].x * l.x + a[r][m].y * l.y;
            x.y -= a[r][m].y * l.x - a[r][m].x * l.y;
          });
          a[r][c] = cscale(x, inv);
        }
      });
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) Pb[r][c][bi] = a[r][c];
    }
    __syncthreads();
    // ---- 3. trailing: A_{bi,bj} -= X_bi X_bj^H ----
    if (act && bj > kb) {
      C xi[4][4], xj[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          xi[r][m] = Pb[r][m][bi];
          xj[r][m] = Pb[r][m][bj];
        }
      // a -= xi conj(xj) as two 2-wide FMAs: a += xi * (-xj.x) + (-xi.y, xi.x) * xj.y
      // (diagonal blocks also update their upper part: never stored)
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const C xs = mkc<C>(-xi[r][m].y, xi[r][m].x);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            a[r][c] = vfma(xi[r][m], vsplat<C>(-xj[c][m].x), a[r][c]);
            a[r][c] = vfma(xs, vsplat<C>(xj[c][m].y), a[r][c]);
          }
        }
    }
  }
  if (bad) atomicCAS(info, 0, p + 1);
  if (!act) return;
  C* L = Lall + (int64_t)p * K * K;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (i0 + r >= k0 + c) L[(int64_t)(i0 + r) * K + k0 + c] = a[r][c];
}

// conj(D_p) = L^-H L^-1 (c_p + ridge conj(V_p - Theta_p)), one CTA (256 threads) per frequency,
// blocked by 32.  Forward: y_b -= L_b,<b y_<b as a tile GEMV (thread = row r, 4 columns of every
// tile to the left; all its tile loads issue back to back, 8 threads per row reduce by
// shuffles), then L_bb y_b = rhs_b by warp 0 from a shared-memory copy of the tile.  Backward:
// y_b -= L_>b,b^H x_>b as the transposed tile GEMV (column sums through shared memory), then
// L_bb^H x_b = y_b by warp 0.  Every element of L is read once per direction.
template <typename Tc, typename Th>
__global__ void __launch_bounds__(256) k_rowsolve_chol(int K, int Kv, const cx<Th>* __restrict__ Lall,
                                                       const cx<Th>* __restrict__ c, Th ridge,
                                                       const cx<Tc>* __restrict__ Vh, const cx<Tc>* __restrict__ Th_,
                                                       int64_t sk, int64_t sp, cx<Tc>* Dh) {
  using C = cx<Th>;
  constexpr int LD = CT + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* y = reinterpret_cast<C*>(smem_raw);  // [K]
  C* Ld = y + K;                          // [CT][LD] diagonal tile / column-sum staging
  const int p = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tr = tid >> 3, tq = (tid & 7) * 4;  // tile row, first of 4 tile columns
  const C* L = Lall + (int64_t)p * K * K;
  for (int k = tid; k < K; k += 256) {  // padding rows (k >= Kv) have a zero right-hand side
    if (k >= Kv) {
      y[k] = mkc<C>(0, 0);
      continue;
    }
    const int64_t o = (int64_t)k * sk + (int64_t)p * sp;
    const C v = csub(ccast<Th>(Vh[o]), ccast<Th>(Th_[o]));
    const C ck = c[(int64_t)p * Kv + k];
    y[k] = mkc<C>(ck.x + ridge * v.x, ck.y - ridge * v.y);
  }
  __syncthreads();
  const int nb = K / CT;
  // ---- forward: L y = rhs ----
  for (int b = 0; b < nb; ++b) {
    const int r0 = b * CT;
    const C* lrow = L + (int64_t)(r0 + tr) * K + tq;
    C acc = mkc<C>(0, 0);
#pragma unroll 4
    for (int m = 0; m < b; ++m) {
      const C* t = lrow + m * CT;
      const C* ym = y + m * CT + tq;
#pragma unroll
      for (int q = 0; q < 4; ++q) cfma(acc, t[q], ym[q]);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    const C* dt = lrow + r0;
#pragma unroll
    for (int q = 0; q < 4; ++q) Ld[tr * LD + tq + q] = dt[q];
    if ((tid & 7) == 0) y[r0 + tr] = csub(y[r0 + tr], acc);
    __syncthreads();
    if (warp == 0) {  // lane i: row i of the tile
      C yi = y[r0 + lane];
      static_for<0, CT>([&](auto J) {
        constexpr int j = decltype(J)::value;
        if (lane == j) yi = cscale(yi, (Th)1 / Ld[j * LD + j].x);
        const Th yx = __shfl_sync(0xffffffffu, yi.x, j), yy = __shfl_sync(0xffffffffu, yi.y, j);
        if (lane > j) {  // yi -= L[i][j] y_j
          const C l = Ld[lane * LD + j];
          yi.x -= l.x * yx - l.y * yy;
          yi.y -= l.x * yy + l.y * yx;
        }
      });
      y[r0 + lane] = yi;
    }
    __syncthreads();
  }
  // ---- backward: L^H x = y ----
  for (int b = nb - 1; b >= 0; --b) {
    const int c0 = b * CT;
    C acc[4] = {mkc<C>(0, 0), mkc<C>(0, 0), mkc<C>(0, 0), mkc<C>(0, 0)};
#pragma unroll 4
    for (int m = b + 1; m < nb; ++m) {  // acc[q] += conj(L[m*CT+tr][c0+tq+q]) x[m*CT+tr]
      const C* t = L + (int64_t)(m * CT + tr) * K + c0 + tq;
      const C xr = y[m * CT + tr];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const C l = t[q];
        acc[q].x += l.x * xr.x + l.y * xr.y;
        acc[q].y += l.x * xr.y - l.y * xr.x;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) Ld[tr * LD + tq + q] = acc[q];
    __syncthreads();
    if (warp == 0) {
      C s = mkc<C>(0, 0);
      for (int r = 0; r < CT; ++r) s = cadd(s, Ld[r * LD + lane]);
      y[c0 + lane] = csub(y[c0 + lane], s);
    }
    __syncthreads();
    {  // the diagonal tile, for the warp solve
      const C* dt = L + (int64_t)(c0 + tr) * K + c0 + tq;
#pragma unroll
      for (int q = 0; q < 4; ++q) Ld[tr * LD + tq + q] = dt[q];
    }
    __syncthreads();
    if (warp == 0) {  // lane k: x_k; L_bb^H x = y, rows from the bottom
      C xk = y[c0 + lane];
      static_for<0, CT>([&](auto Jr) {
        constexpr int i = CT - 1 - decltype(Jr)::value;
        if (lane == i) xk = cscale(xk, (Th)1 / Ld[i * LD + i].x);
        const Th xx = __shfl_sync(0xffffffffu, xk.x, i), xy = __shfl_sync(0xffffffffu, xk.y, i);
        if (lane < i) {  // x_k -= conj(L[i][k]) x_i
          const C l = Ld[i * LD + lane];
          xk.x -= l.x * xx + l.y * xy;
          xk.y -= l.x * xy - l.y * xx;
        }
      });
      y[c0 + lane] = xk;
    }
    __syncthreads();
  }
  for (int j = tid; j < Kv; j += 256)
    Dh[(int64_t)j * sk + (int64_t)p * sp] = mkc<cx<Tc>>((Tc)y[j].x, (Tc)-y[j].y);
}

}  // namespace ocsc

using namespace ocsc;

// the factor of a K that is not a multiple of 32 is stored padded to the next multiple
static int chol_order(int K) { return K % CT ? (K / CT + 1) * CT : K; }

extern "C" int ocsc_debug_chol_profile(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  OCSC_CUDA(cudaMemcpyToSymbol(g_chol_prof, &p, sizeof(p)));
  return OCSC_OK;
}

extern "C" size_t ocsc_history_factor_bytes(int dtype_hist, int K, int nfreq) {
  const size_t Kp = (size_t)chol_order(K);
  return (size_t)(dtype_hist == OCSC_F64 ? 16 : 8) * Kp * Kp * nfreq;
}

extern "C" int ocsc_history_factor(int dtype_hist, int K, int nfreq, const void* S, double ridge, void* L,
                                   int32_t* info, void* stream) {
  if (K <= 0 || nfreq < 0) return fail(OCSC_ESHAPE, "history_factor: bad extents");
  cudaStream_t s = as_stream(stream);
  const int Kv = K;
  K = chol_order(K);
  OCSC_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
  if (nfreq == 0) return OCSC_OK;
  const int nb = K / CT;
  const size_t cs = dtype_hist == OCSC_F64 ? 16 : 8;
  const size_t whole = cs * (size_t)K * (K + 1);
#define OCSC_CHOL_REG(KK)                                                                                    \
  if (K == KK) {                                                                                             \
    if (dtype_hist == OCSC_F32)                                                                              \
      k_chol_rb<float, KK><<<nfreq, chol_reg_threads<KK>(), 0, s>>>((const float2*)S, (float)ridge,          \
                                                                    (float2*)L, info);                      \
    else if (dtype_hist == OCSC_F64)                                                                         \
      k_chol_rb<double, KK><<<nfreq, chol_reg_threads<KK>(), 0, s>>>((const double2*)S, ridge,               \
                                                                     (double2*)L, info);                    \
    else                                                                                                     \
      return fail(OCSC_EARG, "dtype must be 4 or 8");                                                        \
    OCSC_LAUNCHED("k_chol_rb");                                                                              \
    return OCSC_OK;                                                                                          \
  }
  if (K == Kv && !getenv("OCSC_CHOL_NOREG")) {  // dev knob: the shared-memory / blocked kernels instead
    OCSC_CHOL_REG(32)
    OCSC_CHOL_REG(64)
    OCSC_CHOL_REG(96)
    OCSC_CHOL_REG(128)
  }
#undef OCSC_CHOL_REG
  if (K == Kv && K <= 64) {  // small K: the whole matrix in one CTA's shared memory, many CTAs per SM
    const int threads = 64;
    if (dtype_hist == OCSC_F32) {
      OCSC_CUDA(cudaFuncSetAttribute(k_chol_smem<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)whole));
      k_chol_smem<float><<<nfreq, threads, whole, s>>>(K, (const float2*)S, (float)ridge, (float2*)L, info);
    } else if (dtype_hist == OCSC_F64) {
      OCSC_CUDA(cudaFuncSetAttribute(k_chol_smem<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)whole));
      k_chol_smem<double><<<nfreq, threads, whole, s>>>(K, (const double2*)S, ridge, (double2*)L, info);
    } else {
      return fail(OCSC_EARG, "dtype must be 4 or 8");
    }
    OCSC_LAUNCHED("k_chol_smem");
    return OCSC_OK;
  }
  (void)nb;
  const size_t smem = (dtype_hist == OCSC_F64 ? (size_t)chol_panel_offset<double>() : (size_t)chol_panel_offset<float>()) +
                      cs * (size_t)CT * (K - CT);  // L_kk + 1/L_jj + panel
  if (smem > 227 * 1024) return fail(OCSC_EARG, "history_factor: panel exceeds shared memory for this K/dtype");
  size_t smem_req = smem;  // dev knob: request more shared memory (fewer CTAs per SM, a smaller L2 working set)
  if (const char* e = getenv("OCSC_CHOL_MINSMEM")) smem_req = std::max(smem, (size_t)atol(e));
  // float: 512 threads (one CTA per SM) from K = 384; up to K = 288, 128-thread CTAs, three per SM (measured
  // at K = 256: 19.0 ms with 128, 20.8 with 256, 30.3 with 512 threads); OCSC_CHOL_NT overrides
  int nt = dtype_hist == OCSC_F32 ? (K >= 384 ? 512 : (K <= 288 ? 128 : 256)) : 256;
  if (const char* e = getenv("OCSC_CHOL_NT")) nt = atoi(e);
  if (dtype_hist == OCSC_F32 && nt == 512) {
    OCSC_CUDA(cudaFuncSetAttribute(k_chol_blocked<float, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_req));
    k_chol_blocked<float, 512><<<nfreq, 512, smem_req, s>>>(K, Kv, (const float2*)S, (float)ridge, (float2*)L, info);
  } else if (dtype_hist == OCSC_F32 && nt == 256) {
    OCSC_CUDA(cudaFuncSetAttribute(k_chol_blocked<float, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_req));
    k_chol_blocked<float, 256><<<nfreq, 256, smem_req, s>>>(K, Kv, (const float2*)S, (float)ridge, (float2*)L, info);
  } else if (dtype_hist == OCSC_F32) {
    OCSC_CUDA(cudaFuncSetAttribute(k_chol_blocked<float, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_req));
    k_chol_blocked<float, 128><<<nfreq, 128, smem_req, s>>>(K, Kv, (const float2*)S, (float)ridge, (float2*)L, info);
  } else if (dtype_hist == OCSC_F64) {
    OCSC_CUDA(cudaFuncSetAttribute(k_chol_blocked<double, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_req));
    k_chol_blocked<double, 256><<<nfreq, 256, smem_req, s>>>(K, Kv, (const double2*)S, ridge, (double2*)L, info);
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
  const int Kv = K;
  K = chol_order(K);
  const size_t smem = (dtype_hist == OCSC_F64 ? 16 : 8) * ((size_t)K + CT * (CT + 1));
#define RC(TC, TH)                                                                                          \
  k_rowsolve_chol<TC, TH><<<nfreq, 256, smem, s>>>(K, Kv, (const cx<TH>*)L, (const cx<TH>*)c, (TH)ridge,        \
                                                   (const cx<TC>*)Vh, (const cx<TC>*)Th, sk, sp, (cx<TC>*)Dh)
  if (dtype == OCSC_F32 && dtype_hist == OCSC_F32) RC(float, float);
  else if (dtype == OCSC_F32 && dtype_hist == OCSC_F64) RC(float, double);
  else if (dtype == OCSC_F64 && dtype_hist == OCSC_F64) RC(double, double);
  else return fail(OCSC_EARG, "dict_rowsolve_chol: unsupported dtype pair");
#undef RC
  OCSC_LAUNCHED("k_rowsolve_chol");
  return OCSC_OK;
}
