// Streaming code ADMM for grids too large to keep a sample on chip (
// reference coding.py:67-119) -- BASELINE configs 2 (100 x 100) and 3 (266 x 266).
//
// Same iteration as the fused kernel (code_fused.cu), in the single-state form
//     U = S_kappa(w), Gamma = clip_kappa(w), t = U - Gamma,
//     g = (X - sum_k D_k F(t_k)) / den,  c_k = F^-1(conj(D_k) g),  w' = S_kappa(w) + c,
// but with the state w (B, K, H, W) streamed from HBM and the 2-D real FFTs written here
// as two line passes (rows along W, columns along H), each line a Good-Thomas prime-factor
// transform of two register FFTs (fft_small.cuh) through shared memory:
//
//   k_rows   (per R rows of one sample): inverse row FFT of the column-inverse output ->
//            c; w' = S(w) + c / P; the four stopping norms; t' = S(w') - clip(w'); forward
//            row FFT of t' -> back into the same spectrum rows.   HBM: spectrum r+w, w r+w.
//   k_cols_f (per L columns x K-group of one sample): forward column FFT of every plane,
//            times D_k, summed over the group in registers -> one partial per group.
//   k_gsum   g = (X - sum of partials) / den per frequency.
//   k_cols_i (per L columns x K-group): conj(D_k) g -> inverse column FFT -> spectrum.
//   k_decide the per-sample stopping test (code.cu), which freezes converged samples.
//   k_plane  (float 100 x 100, config 2): the whole iteration of a (sample, filter) plane on
//            chip, one CTA per (sample, filter group); its last CTA takes the stopping test.
//
// Per iteration and sample that is 6 passes over K*P reals (spectrum written and read twice,
// w read and written once) where the cuFFT path needs 10+ (and 5 kernels per 266-point
// 2-D transform); the row passes of consecutive iterations are fused.  The FFT arithmetic is
// FP32x2 straight-line code with compile-time twiddles.
#include <cufft.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "fft_small.cuh"
#include "transforms.cuh"

namespace ocsc {

__global__ void k_decide(int B, double tol, double* acc, int32_t* flags, int32_t* iters, int32_t* status);

namespace {

using sfft::fft;
using sfft::modinv;

// ------------------------------------------------------------------ geometry --
// NR = W/2 = RA * RB and H = CA * CB, coprime pairs (Good-Thomas).  R rows per row-CTA,
// L columns per column-CTA; thread counts cover the stage-2 tasks of one pass.
template <typename T, int H_, int W_> struct SGeo;

template <typename T> struct SGeo<T, 100, 100> {
  // float: two planes + state + partial (164 KB) fit one CTA -> k_plane; double -> row/column kernels
  static constexpr bool PLANE = sizeof(T) == 4;
  static constexpr int H = 100, W = 100, RA = 2, RB = 25, CA = 4, CB = 25;
  static constexpr int R = 64, NTR = 128;
  static constexpr int L = 17, NTC = 96;
};
template <typename T> struct SGeo<T, 266, 266> {
  static constexpr bool PLANE = false;
  static constexpr int H = 266, W = 266, RA = 7, RB = 19, CA = 14, CB = 19;
  static constexpr int R = 16, NTR = 128;
  static constexpr int L = 8, NTC = 160;  // stage 1: 19 x 8 = 152 tasks in one round
};

template <class G> struct Derived {
  static constexpr int NR = G::W / 2, WH = G::W / 2 + 1, NF = G::H * WH;
  static constexpr int PR = NR + 1;  // smem row pitch (complex)
  static_assert(G::RA * G::RB == NR && G::CA * G::CB == G::H, "factorisation");
  static_assert(G::L * G::CA <= G::NTC, "column stage-2 tasks must fit one pass");
  static_assert(G::R * G::RA <= G::NTR, "row stage-2 tasks must fit one pass (in-place stage 2)");
};

template <typename T>
__device__ __forceinline__ T shrink(T a, T kappa) {
  return a > kappa ? a - kappa : (a < -kappa ? a + kappa : (a == a ? (T)0 : a));
}
template <typename T>
__device__ __forceinline__ T clip(T a, T kappa) {
  return fmin(fmax(a, -kappa), kappa);  // a NaN w gives a finite clip; S(w) = w - clip(w) stays NaN
}

struct Flags {
  const int32_t* done;
  const int32_t* all_done;
};

// e = tid, tid + STEP, ... over rows of length L: (row, column) kept incrementally instead of a
// division per element; branch-free (ceil(STEP / L) conditional subtractions)
template <int L, int STEP>
struct RowWalk {
  int i, k;
  __device__ __forceinline__ RowWalk(int e0) : i(e0 / L), k(e0 - (e0 / L) * L) {}
  __device__ __forceinline__ void advance() {
    k += STEP;
#pragma unroll
    for (int r = 0; r < (STEP + L - 1) / L; ++r) {
      const int q = k >= L;
      k -= q * L;
      i += q;
    }
  }
};

// ---------------------------------------------------------------- line FFTs --
// Good-Thomas line transform of length N = A * B on a shared-memory line (stride 1):
// stage 1 (tasks n2 < B): A-point DFTs on positions (B n1 + A n2) mod N, in place;
// stage 2 (tasks k1 < A): B-point DFTs on (B k1 + A n2) mod N; output k = CRT(k1, k2).
template <int A, int B_>
struct Pfa {
  static constexpr int N = A * B_;
  static constexpr int tB = modinv(B_ % A, A), tA = modinv(A % B_, B_);
  __device__ static constexpr int in_pos(int n1, int n2) { return (B_ * n1 + A * n2) % N; }
  __device__ static constexpr int out_pos(int k1, int k2) { return (B_ * tB * k1 + A * tA * k2) % N; }
  // base + compile-time offset, both in [0, N): one conditional subtract instead of a modulo
  template <int OFF>
  __device__ static __forceinline__ int wrap(int base) {
    const int p = base + OFF % N;
    return p >= N ? p - N : p;
  }
};

template <typename C, int A, int B_, bool INV>
__device__ __forceinline__ void stage1(C* line, int stride, int n2) {
  using P = Pfa<A, B_>;
  const int base = (A * n2) % P::N;
  C v[A];
  sfft::static_for<0, A>([&](auto I) { v[I.value] = line[P::template wrap<B_ * I.value>(base) * stride]; });
  fft<C, A, INV>(v);
  sfft::static_for<0, A>([&](auto I) { line[P::template wrap<B_ * I.value>(base) * stride] = v[I.value]; });
}

template <typename C, int A, int B_, bool INV>
__device__ __forceinline__ void stage2_load(const C* line, int stride, int k1, C (&v)[B_]) {
  using P = Pfa<A, B_>;
  const int base = B_ * k1;  // < N
  sfft::static_for<0, B_>([&](auto I) { v[I.value] = line[P::template wrap<A * I.value>(base) * stride]; });
  fft<C, B_, INV>(v);
}

// natural-order row of stage-2 output k2 of task k1
template <int A, int B_>
struct OutRow {
  int base;
  __device__ __forceinline__ explicit OutRow(int k1) : base((B_ * Pfa<A, B_>::tB * k1) % Pfa<A, B_>::N) {}
  template <int K2>
  __device__ __forceinline__ int at() const { return Pfa<A, B_>::template wrap<A * Pfa<A, B_>::tA * K2>(base); }
};

// stage-1 task e of a row pass -> (row i, task n2): 16 consecutive n2 of one row per half-warp
// (positions step by RA: distinct bank pairs), the RB - 16 remaining tasks of every row after
// them with lanes over rows
template <int RB>
__device__ __forceinline__ void row_task1(int e, int nr, int& i, int& n2) {
  if constexpr (RB >= 16) {
    if (e < nr * 16) {
      i = e >> 4;
      n2 = e & 15;
    } else {
      const int j = e - nr * 16;
      n2 = 16 + j / nr;
      i = j - (n2 - 16) * nr;
    }
  } else {
    i = e / RB;
    n2 = e - i * RB;
  }
}

// stage-2 task t of a row pass -> (row i, task k1): each half-warp takes 8 rows x two consecutive
// k1 (positions of k1 + 1 are an odd number of bank pairs away from those of k1, the 8 rows an even
// number apart: 16 distinct bank pairs); an odd RA's last k1 runs with lanes over rows
template <int RA>
__device__ __forceinline__ void row_task2(int t, int nr, int& i, int& k1) {
  constexpr int P = RA / 2;
  const int npair = (nr & 7) == 0 ? (nr >> 3) * P * 16 : 0;
  if (t < npair) {
    const int h = t >> 4, l = t & 15, rbk = h / P, pi = h - rbk * P;
    i = 8 * rbk + (l & 7);
    k1 = 2 * pi + (l >> 3);
  } else if (npair > 0) {
    i = t - npair;
    k1 = RA - 1;
  } else {
    k1 = t / nr;
    i = t - k1 * nr;
  }
}

// stage 2 of the row transform in place: every task loads its B-line into registers, the CTA
// syncs, then the outputs land in natural order (tasks <= threads, one round); ends synced.
template <typename C, class G, bool INV>
__device__ __forceinline__ void row_stage2(C* SA, int nr, int tid) {
  constexpr int PR = Derived<G>::PR;
  const bool act = tid < nr * G::RA;
  int i, k1;
  row_task2<G::RA>(tid, nr, i, k1);
  C v[G::RB];
  if (act) stage2_load<C, G::RA, G::RB, INV>(SA + i * PR, 1, k1, v);
  __syncthreads();
  if (act) {
    const OutRow<G::RA, G::RB> o(k1);
    sfft::static_for<0, G::RB>([&](auto K2) { SA[i * PR + o.template at<K2.value>()] = v[K2.value]; });
  }
  __syncthreads();
}


// Rows with RA = 2 (W = 100): the Hermitian pre-/post-processing that maps a half spectrum to
// the packed NR-point complex transform pairs bin k with bin NR - k.  Stage-1 task n2 touches
// bins {2 n2, 2 n2 + RB} and task RB - n2 their partners, so one thread runs both tasks with the
// pre-processing fused in; every stage-2 task holds both bins of each pair in registers, so the
// post-processing is fused into its stores.
// (2-wide forms: s = x1 + conj(x2), d = x1 - conj(x2) are one FFMA2 each, the products with the
// twiddle t two more; same arithmetic as the scalar textbook split)
template <typename C>
__device__ __forceinline__ C herm_pre(C x1, C x2, C t) {  // Z[k] from X[k], X[NR-k]: s + i conj(t) d
  const C s = vfma(x2, mkc<C>(1, -1), x1), d = vfma(x2, mkc<C>(-1, 1), x1);
  return add_i(s, cmulc2(t, d));
}
template <typename C>
__device__ __forceinline__ C herm_post(C z1, C z2, C t) {  // X[k] from Z[k], Z[NR-k]: (s - i t d) / 2
  using T = decltype(C::x);
  const C s = vfma(z2, mkc<C>(1, -1), z1), d = vfma(z2, mkc<C>(-1, 1), z1);
  return vmul(sub_i(s, cmul2(t, d)), vsplat<C>((T)0.5));
}

// Hermitian pre-processing + inverse row stage 1, in place on rows of S; ends synced
template <typename C, class G>
__device__ __forceinline__ void row_stage1_inv_pre(C* S, const C* tws, int nr, int tid) {
  static_assert(G::RA == 2 && G::RB % 2 == 1, "pair fusion needs RA = 2");
  constexpr int NR = Derived<G>::NR, PR = Derived<G>::PR, RB = G::RB, TPR = RB / 2 + 1;
  for (int e = tid; e < nr * TPR; e += blockDim.x) {  // lanes -> rows: distinct bank pairs
    const int n2 = e / nr, i = e - n2 * nr;
    C* row = S + i * PR;
    if (n2 == 0) {  // bins 0 (partner: the X[NR] slot) and RB = NR / 2 (its own partner)
      const C a0 = row[0], b0 = row[NR], a1 = row[RB];
      const C z0 = herm_pre(a0, b0, tws[0]), z1 = herm_pre(a1, a1, tws[RB]);
      row[0] = vadd(z0, z1);
      row[RB] = vsub(z0, z1);
    } else {
      const int p0 = 2 * n2, p1 = 2 * n2 + RB, q0 = NR - p0, q1 = NR - p1;
      const C a0 = row[p0], a1 = row[p1], b0 = row[q0], b1 = row[q1];
      const C za0 = herm_pre(a0, b0, tws[p0]), za1 = herm_pre(a1, b1, tws[p1]);
      const C zb0 = herm_pre(b0, a0, tws[q0]), zb1 = herm_pre(b1, a1, tws[q1]);
      row[p0] = vadd(za0, za1);
      row[p1] = vsub(za0, za1);
      row[q0] = vadd(zb0, zb1);
      row[q1] = vsub(zb0, zb1);
    }
  }
  __syncthreads();
}


// ----------------------------------------------------------------- row pass --
template <typename T, class G>
struct RowArgs {
  int K, B;
  T kappa, invP;
  T* w;                 // (B, K, H, W) state
  cx<T>* spec;          // (B, K, H, WH): in = column-inverse output, out = forward row FFT of t'
  const cx<T>* tw;      // (WH,) e^{-2 pi i k / W}
  double* acc;          // (B, 4) stopping norms
  int32_t* bad;         // (B,) non-finite iterate seen (coding.py:105-106)
  Flags fl;
  int first;            // 1: w = 0 before this pass (cold start): c only, no previous state
};

template <typename T, class G>
__global__ void __launch_bounds__(G::NTR) k_rows(RowArgs<T, G> a) {
  using C = cx<T>;
  using D = Derived<G>;
  constexpr int R = G::R, NR = D::NR, WH = D::WH, PR = D::PR, W = G::W, H = G::H;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* SA = reinterpret_cast<C*>(smraw);
  __shared__ double scratch[4 * 32];
  __shared__ C tws[WH];  // e^{-2 pi i k / W}, k <= NR
  const int b = blockIdx.y;
  if (*a.fl.all_done || a.fl.done[b]) return;
  for (int k = threadIdx.x; k < WH; k += G::NTR) tws[k] = a.tw[k];
  const int64_t rows = (int64_t)a.K * H;
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int nr = (int)(rows - r0 < R ? rows - r0 : R);
  const int tid = threadIdx.x;
  C* spec = a.spec + ((int64_t)b * rows + r0) * WH;
  T* w = a.w + ((int64_t)b * rows + r0) * W;

  // 0. this block's state rows (contiguous) into WB, consumed by the update, and 1. its spectrum
  // rows into SA (the row pitch equals WH: one contiguous block).  float: two TMA bulk copies
  // issued by one thread (no per-thread copy instructions, no bank conflicts on the shared-memory
  // side); double: cp.async / plain copies
  C* WB = SA + R * PR;
  constexpr bool BULK = PR == WH && sizeof(C) == 8;
  __shared__ __align__(8) uint64_t mb_bulk[2];
  const uint32_t wbytes = (uint32_t)(nr * NR * sizeof(C)), sbytes = (uint32_t)(nr * WH * sizeof(C));
  const bool bulk = BULK && (wbytes % 16 == 0) && (sbytes % 16 == 0) && ((uintptr_t)w % 16 == 0) &&
                    ((uintptr_t)spec % 16 == 0);
  if (bulk) {
    if (tid == 0) {
      bulk_mbar_init(&mb_bulk[0]);
      bulk_mbar_init(&mb_bulk[1]);
      bulk_g2s(SA, spec, sbytes, &mb_bulk[0]);
      if (!a.first) bulk_g2s(WB, w, wbytes, &mb_bulk[1]);
    }
    __syncthreads();  // barriers initialised before anyone waits on them
    bulk_wait(&mb_bulk[0], 0);
  } else {
    if (!a.first) {
      const C* wsrc = reinterpret_cast<const C*>(w);
      if constexpr (sizeof(C) == 8) {  // 16-byte copies (two complex)
        const int n = nr * NR;
        for (int e = 2 * tid; e < n; e += 2 * G::NTR) {
          if (e + 1 < n) cp_async<16>(WB + e, wsrc + e);
          else cp_async<8>(WB + e, wsrc + e);
        }
      } else {
        for (int e = tid; e < nr * NR; e += G::NTR) cp_async<sizeof(C)>(WB + e, wsrc + e);
      }
      cp_async_commit();
    }
    if constexpr (PR == WH && sizeof(C) == 8) {
      const int n = nr * WH;
      for (int e = 2 * tid; e < n; e += 2 * G::NTR) {
        if (e + 1 < n) cp_async<16>(SA + e, spec + e);
        else cp_async<8>(SA + e, spec + e);
      }
      cp_async_commit();
      cp_async_wait<0>();
    } else {
      for (int e = tid; e < nr * WH; e += G::NTR) {
        const int i = e / WH, k = e - i * WH;
        SA[i * PR + k] = spec[(int64_t)i * WH + k];
      }
    }
  }
  __syncthreads();
  // 2. Hermitian pre-processing (pairs k, NR-k): Z = (X_k + X*_{NR-k}) + i e^{+i 2pi k/W}(X_k - X*_{NR-k}),
  // 3. inverse FFT_NR in place: stage 1, then stage 2 through registers (one round of tasks)
  if constexpr (G::RA % 2 == 1) {
    // odd RA (266: 7 x 19): the pre-processing pairs position p with NR - p, and the stage-1 task
    // n2 (positions p(n1, n2) = (RB n1 + RA n2) mod NR) with task RB - n2 (positions NR - p(-n1, n2)),
    // so one thread forms both tasks' inputs from the same 2 RA loads and runs both transforms
    // (task 0 is its own partner; its p = 0 pairs with the Nyquist bin X[NR])
    using P = Pfa<G::RA, G::RB>;
    constexpr int RA = G::RA, RB = G::RB, NT1 = RB / 2 + 1;
    for (int e = tid; e < nr * NT1; e += G::NTR) {
      const int n2 = e / nr, i = e - n2 * nr;  // lanes over rows
      C* row = SA + i * PR;
      const int base = (RA * n2) % NR;
      int pos[RA];
      C u[RA], v[RA];
      sfft::static_for<0, RA>([&](auto I) {
        pos[I.value] = P::template wrap<RB * I.value>(base);
        const C x = row[pos[I.value]], y = row[NR - pos[I.value]];
        u[I.value] = herm_pre(x, y, tws[pos[I.value]]);
        v[I.value] = herm_pre(y, x, tws[NR - pos[I.value]]);
      });
      fft<C, RA, true>(u);
      sfft::static_for<0, RA>([&](auto I) { row[pos[I.value]] = u[I.value]; });
      if (n2 != 0) {  // task RB - n2: its n1-th input sits at NR - p((RA - n1) % RA, n2)
        C w[RA];
        sfft::static_for<0, RA>([&](auto I) { w[I.value] = v[(RA - I.value) % RA]; });
        fft<C, RA, true>(w);
        sfft::static_for<0, RA>([&](auto I) { row[NR - pos[(RA - I.value) % RA]] = w[I.value]; });
      }
    }
    __syncthreads();
  } else {
    constexpr int NP = NR / 2 + 1;
    RowWalk<NP, G::NTR> rw(tid);
    for (int e = tid; e < nr * NP; e += G::NTR, rw.advance()) {
      const int i = rw.i, k = rw.k, k2 = NR - k;
      C* row = SA + i * PR;
      const C x1 = row[k], x2 = row[k2];
      const C z1 = herm_pre(x1, x2, tws[k]);   // (forward twiddles; the inverse uses the conjugate)
      const C z2 = herm_pre(x2, x1, tws[k2]);  // Z[NR-k] (k2 in (0, NR]; for k = 0 there is no Z[NR])
      row[k] = z1;
      if (k != 0 && k2 != k) row[k2] = z2;
    }
    __syncthreads();
    for (int e = tid; e < nr * G::RB; e += G::NTR) {
      int i, n2;
      row_task1<G::RB>(e, nr, i, n2);
      stage1<C, G::RA, G::RB, true>(SA + i * PR, 1, n2);
    }
    __syncthreads();
  }
  row_stage2<C, G, true>(SA, nr, tid);
  // 4. update: c = (Re z[n], Im z[n]) = (c[2n], c[2n+1]); w' = S(w) + c/P; norms; t' packed into SA
  // (x, y) pairs run as 2-wide arithmetic; Gamma = clip(w) by min/max, U = w - Gamma
  C sl[4] = {mkc<C>(0, 0), mkc<C>(0, 0), mkc<C>(0, 0), mkc<C>(0, 0)};  // per-thread partial norms
  bool nonfinite = false;
  if (!a.first) {
    if (bulk) {
      bulk_wait(&mb_bulk[1], 0);
    } else {
      cp_async_wait<0>();
      __syncthreads();
    }
  }
  const C ip2 = mkc<C>(a.invP, a.invP);
  RowWalk<NR, G::NTR> uw(tid);
  for (int e = tid; e < nr * NR; e += G::NTR, uw.advance()) {
    const int i = uw.i, n = uw.k;
    const C z = SA[i * PR + n];
    C* wp = reinterpret_cast<C*>(w) + e;  // state rows are contiguous pairs (W = 2 NR)
    const C wo = a.first ? mkc<C>(0, 0) : WB[e];
    const C go = mkc<C>(clip(wo.x, a.kappa), clip(wo.y, a.kappa));
    const C uo = vsub(wo, go);
    const C wn = vfma(z, ip2, uo);
    const C gn = mkc<C>(clip(wn.x, a.kappa), clip(wn.y, a.kappa));
    const C un = vsub(wn, gn);  // S(w') (NaN propagates through w')
    const C d0 = vsub(un, uo), d2 = vsub(gn, go);
    sl[0] = vfma(d0, d0, sl[0]);
    sl[1] = vfma(un, un, sl[1]);
    sl[2] = vfma(d2, d2, sl[2]);
    sl[3] = vfma(gn, gn, sl[3]);
    nonfinite |= !isfinite(wn.x) || !isfinite(wn.y);
    *wp = wn;
    SA[i * PR + n] = vsub(un, gn);
  }
  if (__syncthreads_or(nonfinite) && tid == 0) atomicOr(a.bad + b, 1);
  double s[4] = {(double)sl[0].x + sl[0].y, (double)sl[1].x + sl[1].y, (double)sl[2].x + sl[2].y,
                 (double)sl[3].x + sl[3].y};
  block_sum<4>(s, scratch);  // (contains __syncthreads)
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) atomicAdd(a.acc + 4 * b + j, s[j]);
  }
  // 5. forward FFT_NR of t' in place
  for (int e = tid; e < nr * G::RB; e += G::NTR) {
    int i, n2;
    row_task1<G::RB>(e, nr, i, n2);
    stage1<C, G::RA, G::RB, false>(SA + i * PR, 1, n2);
  }
  __syncthreads();
  row_stage2<C, G, false>(SA, nr, tid);
  // 6. post-processing X_k = (Z_k + Z*_{NR-k})/2 + e^{-i 2pi k/W} (Z_k - Z*_{NR-k})/(2i), k = 0..NR
  RowWalk<WH, G::NTR> pw(tid);
  C* sp = spec + tid;
  for (int e = tid; e < nr * WH; e += G::NTR, pw.advance(), sp += G::NTR) {  // (spec rows are contiguous)
    const int i = pw.i, k = pw.k;
    const C* row = SA + i * PR;
    const C z1 = row[k == NR ? 0 : k], z2 = row[k == 0 ? 0 : NR - k];
    *sp = herm_post(z1, z2, tws[k]);
  }
}

// -------------------------------------------------------------- column passes --
template <typename T, class G>
struct ColArgs {
  int K, B, groups, kper;
  const cx<T>* Wh;      // (K, H, WH)
  const cx<T>* xh;      // (B, H, WH)
  const T* den;         // (H, WH)
  cx<T>* spec;          // (B, K, H, WH)
  cx<T>* part;          // (B, groups, H, WH)
  cx<T>* g;             // (B, H, WH)
  Flags fl;
};

// async copy of one plane's L-column block (H rows, row stride WH) into a [H][L] tile
template <typename C, int H, int L, int NT>
__device__ __forceinline__ void fetch_block(C* dst, const C* src, int WH, int nc, int tid) {
  if constexpr (sizeof(C) == 8 && L % 2 == 0) {
    // complex64: 16-byte copies of column pairs (tiles and spectrum rows are 16-byte aligned;
    // an odd trailing column goes alone)
    constexpr int L2 = L / 2;
    for (int e = tid; e < H * L2; e += NT) {
      const int h = e / L2, c = 2 * (e - h * L2);
      if (c + 1 < nc) cp_async<16>(dst + h * L + c, src + (int64_t)h * WH + c);
      else if (c < nc) cp_async<8>(dst + h * L + c, src + (int64_t)h * WH + c);
    }
  } else {
    for (int e = tid; e < H * L; e += NT) {
      const int h = e / L, c = e - h * L;
      if (c < nc) cp_async<sizeof(C)>(dst + h * L + c, src + (int64_t)h * WH + c);
    }
  }
  cp_async_commit();
}

// forward column FFT of every plane of the group, times D_k, summed in registers.  The
// spectrum and D_k tiles of plane k+1 stream into the second buffer pair (cp.async)
// while plane k is transformed.
template <typename T, class G>
__global__ void __launch_bounds__(G::NTC) k_cols_f(ColArgs<T, G> a) {
  using C = cx<T>;
  using D = Derived<G>;
  constexpr int L = G::L, H = G::H, WH = D::WH, TILE = H * L;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* buf = reinterpret_cast<C*>(smraw);  // [2][Y, Dk][H][L]
  const int b = blockIdx.z, grp = blockIdx.y, c0 = blockIdx.x * L;
  if (*a.fl.all_done || a.fl.done[b]) return;
  const int nc = min(L, WH - c0);
  const int tid = threadIdx.x;
  const int k0 = grp * a.kper, k1e = min(a.K, k0 + a.kper);
  const int c2 = tid % L, q1 = tid / L;  // stage-2 task: column c2, k1 = q1
  const bool own = q1 < G::CA && c2 < nc;
  C acc[G::CB];
#pragma unroll
  for (int j = 0; j < G::CB; ++j) acc[j] = mkc<C>(0, 0);
  auto spec_of = [&](int k) { return a.spec + (((int64_t)b * a.K + k) * H) * WH + c0; };
  auto dict_of = [&](int k) { return a.Wh + (int64_t)k * H * WH + c0; };
  if (k0 < k1e) {
    fetch_block<C, H, L, G::NTC>(buf, spec_of(k0), WH, nc, tid);
    fetch_block<C, H, L, G::NTC>(buf + TILE, dict_of(k0), WH, nc, tid);
  }
  for (int k = k0; k < k1e; ++k) {
    C* Y = buf + ((k - k0) & 1) * 2 * TILE;
    const C* Dk = Y + TILE;
    cp_async_wait<0>();
    __syncthreads();
    if (k + 1 < k1e) {
      C* nxt = buf + ((k + 1 - k0) & 1) * 2 * TILE;
      fetch_block<C, H, L, G::NTC>(nxt, spec_of(k + 1), WH, nc, tid);
      fetch_block<C, H, L, G::NTC>(nxt + TILE, dict_of(k + 1), WH, nc, tid);
    }
    for (int e = tid; e < G::CB * L; e += G::NTC) {
      const int n2 = e / L, c = e - n2 * L;
      if (c < nc) stage1<C, G::CA, G::CB, false>(Y + c, L, n2);
    }
    __syncthreads();
    if (own) {
      C v[G::CB];
      stage2_load<C, G::CA, G::CB, false>(Y + c2, L, q1, v);
      const OutRow<G::CA, G::CB> o(q1);
      sfft::static_for<0, G::CB>([&](auto K2) { cfma(acc[K2.value], Dk[o.template at<K2.value>() * L + c2], v[K2.value]); });
    }
  }
  if (own) {
    C* dst = (a.groups == 1 ? a.g + (int64_t)b * H * WH : a.part + ((int64_t)b * a.groups + grp) * H * WH) + c0 + c2;
    if (a.groups == 1) {
      // g = (X - sum) / den directly
      const C* x = a.xh + (int64_t)b * H * WH + c0 + c2;
      const T* dn = a.den + c0 + c2;
#pragma unroll
      for (int k2 = 0; k2 < G::CB; ++k2) {
        const int row = Pfa<G::CA, G::CB>::out_pos(q1, k2);
        const T inv = (T)1 / dn[row * WH];
        const C xv = x[(int64_t)row * WH];
        dst[(int64_t)row * WH] = mkc<C>((xv.x - acc[k2].x) * inv, (xv.y - acc[k2].y) * inv);
      }
    } else {
#pragma unroll
      for (int k2 = 0; k2 < G::CB; ++k2) {
        const int row = Pfa<G::CA, G::CB>::out_pos(q1, k2);
        dst[(int64_t)row * WH] = acc[k2];
      }
    }
  }
}

// g = (X - sum_groups part) / den  (first iteration: no partials, T = 0)
template <typename T>
__global__ void k_gsum(int B, int nf, int groups, const cx<T>* __restrict__ xh, const T* __restrict__ den,
                       const cx<T>* __restrict__ part, cx<T>* __restrict__ g, Flags fl) {
  const int b = blockIdx.y;
  if (*fl.all_done || fl.done[b]) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nf) return;
  cx<T> s = mkc<cx<T>>(0, 0);
  if (part)
    for (int j = 0; j < groups; ++j) s = cadd(s, part[((int64_t)b * groups + j) * nf + p]);
  const T inv = (T)1 / den[p];
  const cx<T> x = xh[(int64_t)b * nf + p];
  g[(int64_t)b * nf + p] = mkc<cx<T>>((x.x - s.x) * inv, (x.y - s.y) * inv);
}

// conj(D_k) g -> inverse column FFT -> spectrum rows (for the row pass); the D_k tile of
// plane k+1 streams in (cp.async) while plane k is transformed in the other buffer.
template <typename T, class G>
__global__ void __launch_bounds__(G::NTC) k_cols_i(ColArgs<T, G> a) {
  using C = cx<T>;
  using D = Derived<G>;
  constexpr int L = G::L, H = G::H, WH = D::WH, TILE = H * L;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* Gs = reinterpret_cast<C*>(smraw);  // [H][L] g tile
  C* buf = Gs + TILE;                   // [2][H][L] D_k tiles, transformed in place
  const int b = blockIdx.z, grp = blockIdx.y, c0 = blockIdx.x * L;
  if (*a.fl.all_done || a.fl.done[b]) return;
  const int nc = min(L, WH - c0);
  const int tid = threadIdx.x;
  const int k0 = grp * a.kper, k1e = min(a.K, k0 + a.kper);
  auto dict_of = [&](int k) { return a.Wh + (int64_t)k * H * WH + c0; };
  fetch_block<C, H, L, G::NTC>(Gs, a.g + (int64_t)b * H * WH + c0, WH, nc, tid);
  if (k0 < k1e) fetch_block<C, H, L, G::NTC>(buf, dict_of(k0), WH, nc, tid);
  const int c2 = tid % L, q1 = tid / L;
  const bool own = q1 < G::CA && c2 < nc;
  for (int k = k0; k < k1e; ++k) {
    C* Y = buf + ((k - k0) & 1) * TILE;
    cp_async_wait<0>();
    __syncthreads();
    if (k + 1 < k1e) fetch_block<C, H, L, G::NTC>(buf + ((k + 1 - k0) & 1) * TILE, dict_of(k + 1), WH, nc, tid);
    for (int e = tid; e < G::CB * L; e += G::NTC) {
      const int n2 = e / L, c = e - n2 * L;
      if (c < nc) {
        // stage 1 with the input conj(D_k) g formed on the fly (positions of this task only)
        using P = Pfa<G::CA, G::CB>;
        const int base = (G::CA * n2) % P::N;
        C v[G::CA];
        sfft::static_for<0, G::CA>([&](auto I) {
          const int idx = P::template wrap<G::CB * I.value>(base) * L + c;
          v[I.value] = cmulc(Y[idx], Gs[idx]);
        });
        fft<C, G::CA, true>(v);
        sfft::static_for<0, G::CA>([&](auto I) { Y[P::template wrap<G::CB * I.value>(base) * L + c] = v[I.value]; });
      }
    }
    __syncthreads();
    if (own) {
      C v[G::CB];
      stage2_load<C, G::CA, G::CB, true>(Y + c2, L, q1, v);
      C* dst = a.spec + (((int64_t)b * a.K + k) * H) * WH + c0 + c2;
      const OutRow<G::CA, G::CB> o(q1);
      sfft::static_for<0, G::CB>([&](auto K2) { dst[(int64_t)o.template at<K2.value>() * WH] = v[K2.value]; });
    }
  }
}

// ------------------------------------------------------------ plane-resident --
// For grids whose half-spectrum plane fits one CTA's shared memory (100 x 100: 41 KB) the whole
// iteration of a (sample, filter) plane stays on chip: conj(D_k) g -> column IFFT -> row IFFT ->
// update of w (row-major, requested into registers at the plane's start) -> row FFT of t' ->
// column FFT -> times D_k, accumulated over the CTA's filter group into a shared-memory partial.
// HBM per plane and iteration: w read + write and the group partial (vs six passes over the
// spectrum for the row/column kernels).
template <typename T, class G>
struct PlaneArgs {
  int K, B, groups, kper;
  T kappa, invP;
  T* w;                 // (B, K, H, W) state
  const cx<T>* Wh;      // (K, H, WH)
  const cx<T>* g;       // (B, H, WH)
  cx<T>* part;          // (B, groups, H, WH)
  const cx<T>* tw;      // (WH,) e^{-2 pi i k / W}
  double* acc;          // (B, 4)
  int32_t* bad;
  Flags fl;
  int first;
  // the stopping test runs in the last CTA to finish (ticket counter; no k_decide launch)
  int32_t* flags;       // (2 B + 3): done, bad, all_done, iteration count, ticket
  int32_t* iters;
  int32_t* status;
  double tol;
};

__host__ __device__ constexpr int ceil_div_c(int a, int b) { return (a + b - 1) / b; }
constexpr int PLANE_NT = 512;  // one CTA per SM: plane + state + partial in shared memory

// The 25-point stage 2 of a Good-Thomas A x 25 line transform, split across threads as a 5 x 5
// Cooley-Tukey transform so that a plane pass has ~1000 small tasks instead of ~200 long ones
// (the 25-point register FFT kept only 6 warps busy).  With y[m] = line[(25 k1 + A m) mod N],
// m = 5 m1 + m2 and output bin k2 = a + 5 b:
//   Y[a + 5 b] = sum_m2 W5^{m2 b} W25^{m2 a} sum_m1 y[5 m1 + m2] W5^{m1 a}.
// Stage a (task k1, m2): the inner 5-point DFT over m1, times W25^{m2 a}, back into the slots of
// y[5 a + m2] (in place: each task owns its five slots).  Stage b (task k1, a): the outer 5-point
// DFT over the slots 5 a + m2 -> Y[a + 5 b], whose natural-order position is
// (25 tB k1 + A tA (a + 5 b)) mod N (the Good-Thomas output map of Pfa::out_pos).
template <int A>
struct S25 {
  using P = Pfa<A, 25>;
  static constexpr int N = P::N;
  template <typename C, bool INV>
  __device__ static __forceinline__ void stage_a(C* line, int stride, int k1, int m2, const C* tw25) {
    const int base = (25 * k1 + A * m2) % N;
    C v[5];
    sfft::static_for<0, 5>([&](auto I) { v[I.value] = line[P::template wrap<5 * A * I.value>(base) * stride]; });
    fft<C, 5, INV>(v);
    sfft::static_for<1, 5>([&](auto I) {
      const C t = tw25[m2 * I.value];  // e^{-2 pi i m2 a / 25}
      v[I.value] = INV ? cmulc2(t, v[I.value]) : cmul2(t, v[I.value]);
    });
    sfft::static_for<0, 5>([&](auto I) { line[P::template wrap<5 * A * I.value>(base) * stride] = v[I.value]; });
  }
  template <typename C, bool INV>
  __device__ static __forceinline__ void stage_b(const C* line, int stride, int k1, int a, C (&v)[5]) {
    const int base = (25 * k1 + 5 * A * a) % N;
    sfft::static_for<0, 5>([&](auto I) { v[I.value] = line[P::template wrap<A * I.value>(base) * stride]; });
    fft<C, 5, INV>(v);
  }
  // natural-order position of output Y[a + 5 b] of task (k1, a)
  struct Out {
    int base;
    __device__ __forceinline__ Out(int k1, int a) : base((25 * P::tB * k1 + A * P::tA * a) % N) {}
    template <int B5>
    __device__ __forceinline__ int at() const { return P::template wrap<5 * A * P::tA * B5>(base); }
  };
};

// debug: clock64 stamps of CTA (0, 0) over its first 4 planes (scripts/plane_prof.py)
__device__ long long* g_plane_prof = nullptr;
#define PLANE_STAMP(slot) \
  if (prof && k - k0 < 4) prof[(k - k0) * 16 + (slot)] = clock64();

template <typename T, class G>
__global__ void __launch_bounds__(PLANE_NT, 1) k_plane(PlaneArgs<T, G> a) {
  using C = cx<T>;
  using D = Derived<G>;
  constexpr int H = G::H, W = G::W, NR = D::NR, WH = D::WH, PR = D::PR, NF = D::NF, NT = PLANE_NT;
  constexpr int CA = G::CA, RA = G::RA;
  static_assert(G::CB == 25 && G::RB == 25, "k_plane splits the 25-point stage 2 as 5 x 5");
  static_assert(RA == 2, "the forward row pass fuses the Hermitian post-processing (RA = 2)");
  using SC = S25<CA>;
  using SR = S25<RA>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* SA = reinterpret_cast<C*>(smraw);  // [H][PR] plane
  C* SB = SA + H * PR;                  // [H][PR] second plane: stage-b passes run out of place
  C* PT = SB + H * PR;                  // [NF] the group's synthesis partial
  C* GS = PT + NF;                      // [NF] the sample's g, loaded once for all the group's planes
  __shared__ double scratch[4 * 32];
  __shared__ C tws[NR + 1];  // e^{-2 pi i k / W}, k <= NR
  __shared__ C tw25[17];     // e^{-2 pi i j / 25}, j <= 16 (= 4 * 4)
  const int b = blockIdx.y, grp = blockIdx.x;
  if (*a.fl.all_done) return;  // (every CTA sees the same flag: no ticket is taken this launch)
  const int tid = threadIdx.x;
  __shared__ int s_last;
  // this CTA's ticket; the last one runs the stopping test of the iteration
  auto ticket = [&]() {
    __syncthreads();
    if (tid == 0) {
      __threadfence();  // the norms' atomics above are visible before the ticket
      const int t = atomicAdd(a.flags + 2 * a.B + 2, 1);
      s_last = t == (int)(gridDim.x * gridDim.y) - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (tid == 0) a.flags[2 * a.B + 2] = 0;
      decide_block(a.B, a.tol, a.acc, a.flags, a.iters, a.status);
    }
  };
  if (a.fl.done[b]) {
    ticket();
    return;
  }
  const int k0 = grp * a.kper, k1 = min(a.K, k0 + a.kper);
  const C* gb = a.g + (int64_t)b * NF;
  for (int f = tid; f < NF; f += NT) {
    PT[f] = mkc<C>(0, 0);
    GS[f] = gb[f];
  }
  for (int i = tid; i <= NR; i += NT) tws[i] = a.tw[i];
  if (tid < 17) {
    double sn, cs;
    sincospi(-2.0 * tid / 25.0, &sn, &cs);
    tw25[tid] = mkc<C>((T)cs, (T)sn);
  }
  C sl[4] = {mkc<C>(0, 0), mkc<C>(0, 0), mkc<C>(0, 0), mkc<C>(0, 0)};
  bool nonfinite = false;
  const C ip2 = mkc<C>(a.invP, a.invP);
  long long* prof = (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) ? g_plane_prof : nullptr;
  static_assert(sizeof(C) == 8, "k_plane is the float path");
  // column tasks: lanes -> consecutive columns c (conflict-free, D/g loads coalesced);
  // row tasks: lanes -> consecutive rows i (row pitch PR = 51 complex: 16 distinct bank pairs)
  constexpr int NCA = 5 * CA * WH, NRA = 5 * RA * H;
  constexpr int NWV = (H * NR + NT - 1) / NT;  // state pairs per thread
  __syncthreads();
  for (int k = k0; k < k1; ++k) {
    PLANE_STAMP(0)
    C* wpl = reinterpret_cast<C*>(a.w + ((int64_t)b * a.K + k) * H * W);  // H x NR pairs
    const C* dk = a.Wh + (int64_t)k * NF;
    // this thread's state pairs e = tid + j NT of the update below, requested now into registers
    // (their latency hides under the inverse passes; no shared-memory staging of w)
    C wv[NWV];
#pragma unroll
    for (int j = 0; j < NWV; ++j) {
      const int e = tid + j * NT;
      wv[j] = (!a.first && e < H * NR) ? wpl[e] : mkc<C>(0, 0);
    }
    PLANE_STAMP(1)
    // (a) inverse input conj(D_k) g formed as column IFFT stage 1 loads it (g from shared memory,
    // loaded once per CTA; D_k from L2), (b) column IFFT (length H along u, WH columns)
    #pragma unroll
    for (int j_ = 0; j_ < ceil_div_c(G::CB * WH, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= G::CB * WH) break;
      const int n2 = e / WH, c = e - n2 * WH;
      using P = Pfa<CA, G::CB>;
      const int base = (CA * n2) % H;
      C v[CA];
      sfft::static_for<0, CA>([&](auto I) {
        const int u = P::template wrap<G::CB * I.value>(base);
        v[I.value] = cmulc2(dk[u * WH + c], GS[u * WH + c]);
      });
      fft<C, CA, true>(v);
      sfft::static_for<0, CA>([&](auto I) { SA[P::template wrap<G::CB * I.value>(base) * PR + c] = v[I.value]; });
    }
    __syncthreads();
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(NCA, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= NCA) break;
      const int c = e % WH, q = e / WH, q1 = q % CA, m2 = q / CA;
      SC::template stage_a<C, true>(SA + c, PR, q1, m2, tw25);
    }
    __syncthreads();
    PLANE_STAMP(2)
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(NCA, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= NCA) break;
      const int c = e % WH, q = e / WH, q1 = q % CA, a5 = q / CA;
      C v[5];
      SC::template stage_b<C, true>(SA + c, PR, q1, a5, v);
      const typename SC::Out o(q1, a5);
      sfft::static_for<0, 5>([&](auto B5) { SB[o.template at<B5.value>() * PR + c] = v[B5.value]; });
    }
    __syncthreads();
    PLANE_STAMP(3)
    // (c) Hermitian pre-processing of every row fused into (d) row IFFT stage 1
    row_stage1_inv_pre<C, G>(SB, tws, H, tid);
    PLANE_STAMP(4)
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(NRA, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= NRA) break;
      const int i = e % H, q = e / H, q1 = q % RA, m2 = q / RA;
      SR::template stage_a<C, true>(SB + i * PR, 1, q1, m2, tw25);
    }
    __syncthreads();
    PLANE_STAMP(5)
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(NRA, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= NRA) break;
      const int i = e % H, q = e / H, q1 = q % RA, a5 = q / RA;
      C v[5];
      SR::template stage_b<C, true>(SB + i * PR, 1, q1, a5, v);
      const typename SR::Out o(q1, a5);
      sfft::static_for<0, 5>([&](auto B5) { SA[i * PR + o.template at<B5.value>()] = v[B5.value]; });
    }
    __syncthreads();
    PLANE_STAMP(6)
    // (e) update w (pairs), norms, t' packed
    PLANE_STAMP(7)
#pragma unroll
    for (int j = 0; j < NWV; ++j) {
      const int e = tid + j * NT;
      if (e >= H * NR) break;
      const int i = e / NR, n = e - i * NR;
      const C z = SA[i * PR + n];
      const C wo = wv[j];
      const C go = mkc<C>(clip(wo.x, a.kappa), clip(wo.y, a.kappa));
      const C uo = vsub(wo, go);
      const C wn = vfma(z, ip2, uo);
      const C gn = mkc<C>(clip(wn.x, a.kappa), clip(wn.y, a.kappa));
      const C un = vsub(wn, gn);
      const C d0 = vsub(un, uo), d2 = vsub(gn, go);
      sl[0] = vfma(d0, d0, sl[0]);
      sl[1] = vfma(un, un, sl[1]);
      sl[2] = vfma(d2, d2, sl[2]);
      sl[3] = vfma(gn, gn, sl[3]);
      nonfinite |= !isfinite(wn.x) || !isfinite(wn.y);
      wpl[e] = wn;
      SA[i * PR + n] = vsub(un, gn);
    }
    __syncthreads();
    PLANE_STAMP(8)
    // (f) row FFT of t': stage 1 (2-point), then the split 25-point stage
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(H * G::RB, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= H * G::RB) break;
      const int i = e % H, n2 = e / H;
      stage1<C, RA, G::RB, false>(SA + i * PR, 1, n2);
    }
    __syncthreads();
    PLANE_STAMP(9)
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(NRA, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= NRA) break;
      const int i = e % H, q = e / H, q1 = q % RA, m2 = q / RA;
      SR::template stage_a<C, false>(SA + i * PR, 1, q1, m2, tw25);
    }
    __syncthreads();
    PLANE_STAMP(10)
    // (g) stage b with the Hermitian post-processing fused into its stores (SA -> SB = forward
    // half-spectrum rows): bin k2 pairs with bin 25 - k2 of the same k1, i.e. outer task a with
    // task 5 - a, so a thread runs task 0 alone or the pair (1, 4) / (2, 3)
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(3 * RA * H, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= 3 * RA * H) break;
      const int i = e % H, q = e / H, q1 = q % RA, s = q / RA;
      const C* src = SA + i * PR;
      C* row = SB + i * PR;
      C u[5];
      SR::template stage_b<C, false>(src, 1, q1, s, u);
      const typename SR::Out ou(q1, s);
      if (s == 0) {
        sfft::static_for<0, 5>([&](auto B5) {
          constexpr int bb = B5.value, bp = (5 - bb) % 5;
          const int kk = ou.template at<bb>();
          row[kk] = herm_post(u[bb], u[bp], tws[kk]);
        });
        if (q1 == 0) row[NR] = herm_post(u[0], u[0], tws[NR]);
      } else {
        C w[5];
        SR::template stage_b<C, false>(src, 1, q1, 5 - s, w);
        const typename SR::Out ow(q1, 5 - s);
        sfft::static_for<0, 5>([&](auto B5) {
          constexpr int bb = B5.value;
          const int ku = ou.template at<bb>(), kw = ow.template at<bb>();
          row[ku] = herm_post(u[bb], w[4 - bb], tws[ku]);
          row[kw] = herm_post(w[bb], u[4 - bb], tws[kw]);
        });
      }
    }
    __syncthreads();
    PLANE_STAMP(11)
    // (h) column FFT: stage 1 in place, stage a in place, stage b with (i) the synthesis partial
    // fused into its stores: PT[f] += D_k[f] T_k[f] (every f is one output of one task: no race)
    #pragma unroll
    for (int j_ = 0; j_ < ceil_div_c(G::CB * WH, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= G::CB * WH) break;
      const int n2 = e / WH, c = e - n2 * WH;
      stage1<C, CA, G::CB, false>(SB + c, PR, n2);
    }
    __syncthreads();
    PLANE_STAMP(12)
    #pragma unroll 1
    for (int j_ = 0; j_ < ceil_div_c(NCA, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= NCA) break;
      const int c = e % WH, q = e / WH, q1 = q % CA, m2 = q / CA;
      SC::template stage_a<C, false>(SB + c, PR, q1, m2, tw25);
    }
    __syncthreads();
    PLANE_STAMP(13)
    #pragma unroll
    for (int j_ = 0; j_ < ceil_div_c(NCA, NT); ++j_) {
      const int e = tid + j_ * NT;
      if (e >= NCA) break;
      const int c = e % WH, q = e / WH, q1 = q % CA, a5 = q / CA;
      C v[5];
      SC::template stage_b<C, false>(SB + c, PR, q1, a5, v);
      const typename SC::Out o(q1, a5);
      sfft::static_for<0, 5>([&](auto B5) {
        const int f = o.template at<B5.value>() * WH + c;
        PT[f] = vfma_c(dk[f], v[B5.value], PT[f]);
      });
    }
    __syncthreads();  // SA / SB are rewritten by the next plane
    PLANE_STAMP(14)
  }
  C* part = a.part + ((int64_t)b * a.groups + grp) * NF;
  for (int f = tid; f < NF; f += NT) part[f] = PT[f];
  if (__syncthreads_or(nonfinite) && tid == 0) atomicOr(a.bad + b, 1);
  double sn[4] = {(double)sl[0].x + sl[0].y, (double)sl[1].x + sl[1].y, (double)sl[2].x + sl[2].y,
                  (double)sl[3].x + sl[3].y};
  block_sum<4>(sn, scratch);
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) atomicAdd(a.acc + 4 * b + j, sn[j]);
  }
  ticket();
}

// final pass: u = S(w) in place
template <typename T>
__global__ void k_shrink_inplace(int64_t n, T kappa, T* __restrict__ u) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    u[i] = shrink(u[i], kappa);
}

// ------------------------------------------------------------------ host side --
struct StreamWork {
  void* part;
  void* g;
  double* acc;
  int32_t* flags;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int k_groups(int K, int B, int ncb) {
  // enough CTAs for ~4 waves of 148 SMs, at least 8 planes per CTA
  int g = ceil_div(4 * 148, (int64_t)B * ncb);
  g = std::max(1, std::min(g, K / 4));
  return g;
}

int plane_groups(int K, int B) {
  // one CTA per SM over the whole batch (at most one wave), at least one filter per CTA
  int g = std::max(1, 148 / std::max(B, 1));
  g = std::max(1, std::min(g, K));
  const int kper = ceil_div(K, g);
  return ceil_div(K, kper);
}

size_t stream_layout(int dtype, int H, int W, int K, int B, int groups, StreamWork* w, char* base) {
  const size_t s = dtype == OCSC_F64 ? 16 : 8;
  const size_t nf = (size_t)H * (W / 2 + 1);
  size_t off = 0;
  auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += align256(bytes); return p; };
  char* part = take((size_t)B * groups * nf * s);
  char* g = take((size_t)B * nf * s);
  char* acc = take((size_t)B * 4 * sizeof(double));
  char* flags = take((size_t)(2 * B + 3) * sizeof(int32_t));  // + the plane kernel's ticket
  if (w) {
    w->part = part; w->g = g; w->acc = (double*)acc; w->flags = (int32_t*)flags;
  }
  return off;
}

template <typename T>
const cx<T>* twiddles(int W) {  // per (device, W) table of e^{-2 pi i k / W}, k <= W/2
  static std::mutex mu;
  static std::map<std::pair<int, int>, void*> cache;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(dev, W);
  auto it = cache.find(key);
  if (it != cache.end()) return (const cx<T>*)it->second;
  const int n = W / 2 + 1;
  std::vector<cx<T>> h(n);
  for (int k = 0; k < n; ++k) {
    const double a = -2.0 * sfft::kPi * k / W;
    h[k] = mkc<cx<T>>((T)cos(a), (T)sin(a));
  }
  void* d = nullptr;
  if (cudaMalloc(&d, n * sizeof(cx<T>)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), n * sizeof(cx<T>), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  cache[key] = d;
  return (const cx<T>*)d;
}

int32_t* pinned_flag() {
  static int32_t* p = nullptr;
  if (!p && cudaHostAlloc((void**)&p, 8 * sizeof(int32_t), cudaHostAllocPortable) != cudaSuccess) p = nullptr;
  return p;
}

template <typename T, class G>
int run(int K, int B, const void* xh, const void* Wh, const void* den, double beta, double rho, int max_iters,
        double rel_tol, void* u, void* work, int32_t* iters, int32_t* status, int poll, cudaStream_t s) {
  using D = Derived<G>;
  constexpr int H = G::H, W = G::W, WH = D::WH, NF = D::NF;
  const int dtype = sizeof(T) == 4 ? OCSC_F32 : OCSC_F64;
  const int ncb = ceil_div(WH, G::L);
  const int groups = G::PLANE ? plane_groups(K, B) : k_groups(K, B, ncb);
  const int kper = ceil_div(K, groups);
  StreamWork sw;
  stream_layout(dtype, H, W, K, B, groups, &sw, (char*)work);
  // the spectrum lives in the caller's t buffer region: (B, K, H, WH) complex needs
  // B*K*H*(W+2) reals; the workspace passed in holds it after the small buffers
  cx<T>* spec = (cx<T>*)((char*)work + stream_layout(dtype, H, W, K, B, groups, nullptr, nullptr));
  const cx<T>* tw = twiddles<T>(W);
  if (!tw) return fail(OCSC_ECUDA, "code_stream: twiddle table allocation failed");
  OCSC_CUDA(cudaMemsetAsync(sw.acc, 0, sizeof(double) * 4 * B, s));
  OCSC_CUDA(cudaMemsetAsync(sw.flags, 0, sizeof(int32_t) * (2 * B + 3), s));
  OCSC_CUDA(cudaMemsetAsync(iters, 0, sizeof(int32_t) * B, s));
  OCSC_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * B, s));
  if (B == 0 || max_iters <= 0) {
    OCSC_CUDA(cudaMemsetAsync(u, 0, sizeof(T) * (size_t)B * K * H * W, s));
    return OCSC_OK;
  }
  Flags fl{sw.flags, sw.flags + 2 * B};

  RowArgs<T, G> ra{K, B, (T)(beta / rho), (T)(1.0 / ((double)H * W)), (T*)u, spec, tw, sw.acc, sw.flags + B, fl, 1};
  ColArgs<T, G> ca{K, B, groups, kper, (const cx<T>*)Wh, (const cx<T>*)xh, (const T*)den, spec,
                   (cx<T>*)sw.part, (cx<T>*)sw.g, fl};
  const size_t row_smem = (size_t)G::R * (D::PR + D::NR) * sizeof(cx<T>);
  const size_t colf_smem = 4 * (size_t)H * G::L * sizeof(cx<T>);
  const size_t coli_smem = 3 * (size_t)H * G::L * sizeof(cx<T>);
  OCSC_CUDA(cudaFuncSetAttribute(k_rows<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem));
  OCSC_CUDA(cudaFuncSetAttribute(k_cols_f<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)colf_smem));
  OCSC_CUDA(cudaFuncSetAttribute(k_cols_i<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coli_smem));
  const dim3 rgrid(ceil_div((int64_t)K * H, G::R), B);
  const dim3 cgrid(ncb, groups, B);
  const dim3 ggrid(ceil_div(NF, 256), B);

  int32_t* host = poll > 0 ? pinned_flag() : nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (host) {
    OCSC_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    OCSC_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  }
  PlaneArgs<T, G> pa{K, B, groups, kper, (T)(beta / rho), (T)(1.0 / ((double)H * W)), (T*)u, (const cx<T>*)Wh,
                     (const cx<T>*)sw.g, (cx<T>*)sw.part, tw, sw.acc, sw.flags + B, fl, 1, sw.flags, iters, status,
                     rel_tol};
  const size_t plane_smem = ((size_t)H * 2 * D::PR + 2 * NF) * sizeof(cx<T>);
  if constexpr (G::PLANE)
    OCSC_CUDA(cudaFuncSetAttribute(k_plane<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plane_smem));
  int rc = OCSC_OK, chunk = 0;
  bool stop = false;
  for (int it = 1; it <= max_iters && !stop; ++it) {
    if constexpr (G::PLANE) {
      // g from the previous iteration's group partials (none at the cold start: T = 0)
      k_gsum<T><<<ggrid, 256, 0, s>>>(B, NF, groups, (const cx<T>*)xh, (const T*)den,
                                      it > 1 ? (const cx<T>*)sw.part : nullptr, (cx<T>*)sw.g, fl);
      pa.first = it == 1;
      k_plane<T, G><<<dim3(groups, B), PLANE_NT, plane_smem, s>>>(pa);  // (its last CTA decides)
      count_launches(2);
    } else {
    if (it > 1) {
      k_cols_f<T, G><<<cgrid, G::NTC, colf_smem, s>>>(ca);  // groups == 1: writes g itself
      count_launches(1);
      if (groups > 1) {
        k_gsum<T><<<ggrid, 256, 0, s>>>(B, NF, groups, (const cx<T>*)xh, (const T*)den, (const cx<T>*)sw.part,
                                        (cx<T>*)sw.g, fl);
        count_launches(1);
      }
    } else {
      k_gsum<T><<<ggrid, 256, 0, s>>>(B, NF, groups, (const cx<T>*)xh, (const T*)den, nullptr, (cx<T>*)sw.g, fl);
      count_launches(1);
    }
    k_cols_i<T, G><<<cgrid, G::NTC, coli_smem, s>>>(ca);
    ra.first = it == 1;
    k_rows<T, G><<<rgrid, G::NTR, row_smem, s>>>(ra);
    k_decide<<<1, 256, 0, s>>>(B, rel_tol, sw.acc, sw.flags, iters, status);
    count_launches(3);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { rc = cuda_fail(e, "code_stream launch"); break; }
    if (host && it % poll == 0 && it < max_iters) {
      const int slot = chunk & 1;
      cudaMemcpyAsync(host + slot, sw.flags + 2 * B, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaEventRecord(ev[slot], s);
      if (chunk > 0) {
        cudaEventSynchronize(ev[slot ^ 1]);
        if (host[slot ^ 1]) stop = true;
      }
      ++chunk;
    }
  }
  if (host) {
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  }
  if (rc) return rc;
  const int64_t n = (int64_t)B * K * H * W;
  k_shrink_inplace<T><<<grid_for(n, 256), 256, 0, s>>>(n, (T)(beta / rho), (T*)u);
  OCSC_LAUNCHED("k_shrink_inplace");
  return OCSC_OK;
}

template <typename T>
int dispatch(int H, int W, bool query, int K, int B, const void* xh, const void* Wh, const void* den, double beta,
             double rho, int max_iters, double rel_tol, void* u, void* work, int32_t* iters, int32_t* status,
             int poll, cudaStream_t s) {
#define OCSC_STREAM_CASE(HH, WW)                                                                      \
  if (H == HH && W == WW) {                                                                           \
    if (query) return 1;                                                                              \
    return run<T, SGeo<T, HH, WW>>(K, B, xh, Wh, den, beta, rho, max_iters, rel_tol, u, work, iters, \
                                   status, poll, s);                                                  \
  }
  OCSC_STREAM_CASE(100, 100)
  OCSC_STREAM_CASE(266, 266)
#undef OCSC_STREAM_CASE
  return query ? 0 : fail(OCSC_ESHAPE, "code_stream: no streaming instantiation for this grid");
}

}  // namespace
}  // namespace ocsc

using namespace ocsc;

extern "C" int ocsc_code_stream_supported(int dtype, int H, int W) {
  if (dtype == OCSC_F32) return dispatch<float>(H, W, true, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
  if (dtype == OCSC_F64) return dispatch<double>(H, W, true, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
  return 0;
}

extern "C" int ocsc_code_stream_plane_ctas(int dtype, int H, int W, int K, int B) {
  // CTAs one iteration of the plane-resident kernel occupies (one per SM; 0: not that path)
  if (dtype != OCSC_F32 || H != 100 || W != 100 || K <= 0 || B <= 0) return 0;
  return plane_groups(K, B) * B;
}

extern "C" size_t ocsc_code_stream_workspace_bytes(int dtype, int H, int W, int K, int B) {
  const int WH = W / 2 + 1;
  const int L = H == 266 ? SGeo<float, 266, 266>::L : SGeo<float, 100, 100>::L;
  const int groups = std::max(k_groups(K, B, ceil_div(WH, L)), plane_groups(K, B));
  const size_t s = dtype == OCSC_F64 ? 16 : 8;
  return stream_layout(dtype, H, W, K, B, groups, nullptr, nullptr) + (size_t)B * K * H * WH * s;
}

extern "C" int ocsc_code_stream(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh,
                                const void* den, double beta, double rho, int max_iters, double rel_tol, void* u,
                                void* work, int32_t* iters, int32_t* status, int poll, void* stream) {
  if (H <= 0 || W <= 0 || K <= 0 || B < 0) return fail(OCSC_ESHAPE, "code_stream: bad extents");
  if (!(rho > 0)) return fail(OCSC_EARG, "code_stream: rho must be positive");
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    return dispatch<float>(H, W, false, K, B, xh, Wh, den, beta, rho, max_iters, rel_tol, u, work, iters, status,
                           poll, s);
  if (dtype == OCSC_F64)
    return dispatch<double>(H, W, false, K, B, xh, Wh, den, beta, rho, max_iters, rel_tol, u, work, iters, status,
                            poll, s);
  return fail(OCSC_EARG, "dtype must be 4 or 8");
}

extern "C" int ocsc_debug_plane_profile(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  OCSC_CUDA(cudaMemcpyToSymbol(ocsc::g_plane_prof, &p, sizeof(p)));
  return OCSC_OK;
}
