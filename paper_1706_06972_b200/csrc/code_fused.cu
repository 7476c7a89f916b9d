// Fused, on-chip code ADMM: one thread-block CLUSTER per sample runs every
// iteration of coding.py:67-119 without leaving the SMs.
//
// State.  With U = S_k(w) and Gamma = w - S_k(w) (= clip(w, -k, k)), one array
// w per (filter, pixel) carries the whole ADMM state (the reference's
// U' = S(U + c), Gamma' = (U + c) - U'), so an iteration is
//     t = S(w) - clip(w);  y = sum_k D_k F(t_k);  g = (X - y) / den;
//     c_k = F^-1(conj(D_k) g);  w' = S(w) + c_k.
// The CTA of cluster rank r owns filters [r K/CS, (r+1) K/CS) of its sample:
// their w planes and their half-spectrum workspace live in shared memory for
// the whole solve.  Each 2-D transform is done as register-resident 1-D FFTs
// (fft_small.cuh: compile-time length, compile-time twiddles): a thread
// transforms two real rows packed as one complex row, or one column.  The only
// cross-CTA traffic per iteration is the cluster reduction of the partial
// synthesis sum_k D_k T_k (one half spectrum per CTA) through distributed
// shared memory, plus the four stopping norms; D is read from L2.
//
// Per iteration and CTA:  [col FFT + D multiply] -> [sum over own filters] ->
// cluster.sync -> [decide previous iteration] -> [reduce-scatter y, g slice,
// broadcast g] -> cluster.sync -> [conj(D) g, col IFFT] -> [row IFFT, update w,
// norms, next t, row FFT].  After the last iteration the same machinery
// produces F(U) (needed by the history), the code U, and the objective.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <tuple>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "fft_small.cuh"

namespace cg = cooperative_groups;

namespace ocsc {

// optional phase timestamps (development aid): CTA 0, thread 0, iterations 8..15
__device__ long long* g_fused_prof = nullptr;
__device__ long long* g_fused_timeline = nullptr;  // [sample][2]: globaltimer at start / end (CTA rank 0)
__device__ long long* g_fused_iter = nullptr;      // [2][512]: globaltimer / clock64 at each iteration (CTA 0)
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define OCSC_STAMP(slot)                                                                       \
  do {                                                                                         \
    if (prof && pit >= 8 && pit < 16) prof[(pit - 8) * 8 + (slot)] = clock64();               \
  } while (0)

template <typename T>
struct FusedArgs {
  int K, B, max_iters;
  int b0;  // first sample of this launch (a mini-batch may be split over two cluster shapes)
  double tol, beta;
  T kappa;
  const cx<T>* xh;  // (B, nf)
  const cx<T>* Wh;  // (K, nf)
  const T* den;     // (nf)
  T* u_out;         // (B, K, H, W)
  T* t_out;         // optional (B, K, H, W): U - Gamma
  cx<T>* uh_out;    // (B, K, nf)
  double* obj;      // (B)
  double* resid;    // optional (B)
  int32_t* iters;   // (B)
  int32_t* status;  // (B)
  // persistent schedule (concurrent plans): cluster c of this launch codes samples
  // sched[(sched_c0 + c) * sched_w + i], i = 0.. until -1; null: cluster c codes sample b0 + c
  const int32_t* sched = nullptr;
  int sched_w = 0, sched_c0 = 0;
  // residency probe (plan calibration): no coding; every CTA spins probe_ns, role 0 records its end,
  // role 1 records when each cluster started
  unsigned long long* probe = nullptr;
  long long probe_ns = 0;
  int probe_role = 0;
};

// Grid N x N with N = 2M, M odd (42 = 2 * 21 for BASELINE config 1).
//  * a real row of N pixels is one M-point complex FFT of (even, odd) pixel pairs plus a
//    twiddled real pre/post-processing step: one thread per row, the update of w runs on
//    the row's values in registers between the inverse and the forward row transform;
//  * a column (N complex) is the Good-Thomas split N = 2 x M (no twiddles): lanes l and
//    l^16 each run the M-point FFT of one index parity and finish the 2-point stage with
//    one butterfly shuffle.
// Every transform goes through ONE call site of the M-point FFT (inverse = conj o FFT o conj),
// which keeps the kernel's instruction footprint inside the instruction caches.
template <int N>
struct Geo {
  static constexpr int M = N / 2;
  static constexpr int Wh = M + 1;
  // float row stride of w: even (float2 accesses) and odd in 8-byte units (N = 2 * odd), so a
  // warp of row tasks (one row per lane) hits distinct 8-byte bank pairs
  static constexpr int WP = N;
  static constexpr int NF = N * Wh;
  // complex row stride of the workspace: odd, >= Wh, and N*RS == Wh (mod 16) when possible,
  // so the row tasks (lane -> row) and the column half-warps (lane -> column, running across
  // plane boundaries) both hit 16 distinct 8-byte bank pairs
  static constexpr int pick_rs() {
    for (int r = Wh | 1; r < Wh + 17; r += 2)
      if (((N * r - Wh) % 16 + 16) % 16 == 0) return r;
    return Wh | 1;
  }
  static constexpr int RS = pick_rs();
  static constexpr int PS = N * RS + (((Wh - N * RS) % 16) + 16) % 16;  // == Wh (mod 16)
  static_assert(N % 2 == 0 && (N / 2) % 2 == 1, "fused grid must be N = 2 * odd");
};

// shared-memory carve-up (all offsets 16-byte aligned)
template <typename T, int N>
struct Smem {
  using G = Geo<N>;
  static __host__ __device__ size_t al(size_t x) { return (x + 15) & ~(size_t)15; }
  static __host__ __device__ size_t w_bytes(int nk) { return al(sizeof(T) * (size_t)nk * N * G::WP); }
  static __host__ __device__ size_t x_bytes(int nk) { return al(sizeof(cx<T>) * (size_t)nk * G::PS); }
  static __host__ __device__ size_t g_bytes() { return al(sizeof(cx<T>) * (size_t)N * G::RS); }
  static __host__ __device__ size_t p_bytes(int cs) {
    return al(sizeof(cx<T>) * (size_t)cs * ((G::NF + cs - 1) / cs));
  }
  // per-warp norm partials from every CTA of the cluster: [CS][32 warps][8] (arithmetic type)
  static __host__ __device__ size_t n_bytes(int cs) { return al(sizeof(T) * 2 * 8 * 32 * (size_t)cs); }
  // this CTA's slice of the sample spectrum and of den
  static __host__ __device__ size_t s_bytes(int cs) {
    const size_t sl = (G::NF + cs - 1) / cs;
    return al(sizeof(cx<T>) * sl) + al(sizeof(T) * sl);
  }
  static __host__ __device__ size_t total(int nk, int cs) {
    return w_bytes(nk) + x_bytes(nk) + g_bytes() + p_bytes(cs) + n_bytes(cs) + s_bytes(cs) + 6 * 32 * sizeof(double);
  }
  static __host__ __device__ int threads(int nk) {
    const int wc = (nk * G::Wh + 15) / 16, wr = (nk * N + 31) / 32;
    return 32 * (wc > wr ? wc : wr);
  }
};

// block-wide sum of NV doubles, result broadcast to every thread
template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * 32 + warp] = v[i];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = lane < nw ? scratch[i * 32 + lane] : 0.0;
      s = warp_sum(s);
      if (lane == 0) scratch[32 * NV + i] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = scratch[32 * NV + i];
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T clampk(T w, T k) {
  return fmin(fmax(w, -k), k);  // Gamma = clip(w); NaN maps to -k so U = w - Gamma stays NaN
}

// Real rows of N = 2M pixels as M-point complex FFTs of p[m] = x[2m] + i x[2m+1].  Both
// conversions below are written in 2-wide form (FFMA2 with swizzled operands, the +-1 factors
// exact) and carry a factor 2 against the textbook split, which the callers fold elsewhere.
//
// half spectrum row[0..M] of a real row  ->  z with FFT_M(z) = 2 M conj(p) (inverse through the
// forward FFT):  z_k = conj(Ze' + i Zo'),  Ze' = A + conj(B),  Zo' = (A - conj(B)) e^{+2 pi i k/N},
// A = row[k], B = row[M - k]  (the textbook Ze, Zo are half of these)
template <typename C, int N>
__device__ __forceinline__ void row_inverse_pre(const C* row, C (&z)[N / 2]) {
  using T = decltype(C::x);
  constexpr int M = N / 2;
  sfft::static_for<0, M>([&](auto Kk) {
    constexpr int k = decltype(Kk)::value;
    C A_ = row[k], B_ = row[M - k];
    if constexpr (k == 0) {  // DC and Nyquist are real for a real row
      A_.y = 0;
      B_.y = 0;
    }
    constexpr T c = (T)sfft::ce_cos(2.0 * sfft::kPi * k / N);
    constexpr T s = (T)sfft::ce_sin(2.0 * sfft::kPi * k / N);
    const C d = vfma(B_, mkc<C>(-1, 1), A_);                 // A - conj(B)
    const C ze = vfma(A_, mkc<C>(1, -1), B_);                // conj(A) + B = conj(Ze')
    // conj(Ze' + i Zo') = conj(Ze') - c swap(d) + s (-d.x, d.y)
    z[k] = vfma(d, mkc<C>(-s, s), vfma(vswap(d), vsplat<C>(-c), ze));
  });
}

// Z = FFT_M(p / 2)  ->  half spectrum row[0..M] of the real row:
// X_k = Ze + W^k Zo with Ze = Z_k + conj(Z_{M-k}), Zo = -i (Z_k - conj(Z_{M-k})), W = e^{-2 pi i/N}
template <typename C, int N>
__device__ __forceinline__ void row_forward_post(const C (&Z)[N / 2], C* row) {
  using T = decltype(C::x);
  constexpr int M = N / 2;
  sfft::static_for<0, M + 1>([&](auto Kk) {
    constexpr int k = decltype(Kk)::value;
    const C a = Z[k % M], bb = Z[(M - k) % M];
    constexpr T c = (T)sfft::ce_cos(2.0 * sfft::kPi * k / N);
    constexpr T s = (T)sfft::ce_sin(2.0 * sfft::kPi * k / N);
    const C ze = vfma(bb, mkc<C>(1, -1), a);   // a + conj(bb)
    const C dm = vfma(bb, mkc<C>(-1, 1), a);   // a - conj(bb)
    // W^k (-i) dm = (-s - i c) dm = -s dm + c (dm.y, -dm.x)
    row[k] = vfma(vswap(dm), mkc<C>(c, -c), vfma(dm, vsplat<C>(-s), ze));
  });
}

enum ColMode : int { COL_F = 0, COL_I = 1, COL_FE = 2 };

// ---- cluster exchange without cluster barriers: remote stores that complete a transaction count
// on the receiver's mbarrier (st.async ... mbarrier::complete_tx), local waits on that mbarrier.
// A receiver proceeds once its own data has landed; no GPU-scope fence or L1 invalidation (what
// barrier.cluster.arrive.release / wait.acquire compile to) sits in the iteration.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(a), "r"(rank));
  return out;
}
__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* m, uint32_t tx) {  // the phase's one arrival + tx bytes
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {  // plain arrival (release: prior stores visible)
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
      "r"(parity), "r"(0x989680u)  // suspend-time hint: the warp sleeps instead of spinning
      : "memory");
}
__device__ __forceinline__ void st_async(uint32_t dst, float2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "f"(v.x), "f"(v.y), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t dst, double2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "d"(v.x), "d"(v.y), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t dst, float v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(dst), "f"(v),
               "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t dst, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(dst), "d"(v),
               "r"(mbar)
               : "memory");
}

// DREG_: keep the lane's D column in registers for the whole solve (float only, 120 registers,
// at most 16 warps = 11 filters per CTA); otherwise reload D from L2 each iteration (96 registers,
// up to 17 warps = 12 filters per CTA, or 18 warps with 13)
template <typename T, int N, bool DREG_>
__global__ void __maxnreg__(DREG_ ? 120 : 96) k_code_fused(FusedArgs<T> a) {
  using C = cx<T>;
  using G = Geo<N>;
  using S = Smem<T, N>;
  constexpr int M = G::M, Wh = G::Wh, WP = G::WP, RS = G::RS, PS = G::PS, NF = G::NF;

  // a concurrent plan launches its second cluster shape programmatically after this grid: let it
  // start as soon as every cluster of this (persistent, fully resident) grid is running
  asm volatile("griddepcontrol.launch_dependents;");
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int r = (int)cl.block_rank();
  const int ci = (int)(blockIdx.x / CS);  // cluster index within this launch
  if (a.probe) {  // both roles hold their SMs for probe_ns, so a side cluster that started
    const long long t0 = global_ns();  // before the main grid's first exit was co-resident with it
    if (a.probe_role == 1 && threadIdx.x == 0 && r == 0) a.probe[1 + ci] = (unsigned long long)t0;
    while (global_ns() - t0 < a.probe_ns) {
    }
    if (a.probe_role == 0 && threadIdx.x == 0) atomicMin(a.probe, (unsigned long long)global_ns());
    return;
  }
  const int K = a.K;
  const int k0 = (int)((int64_t)r * K / CS), k1 = (int)((int64_t)(r + 1) * K / CS);
  const int nk = k1 - k0;
  const int nkmax = (K + CS - 1) / CS;

  extern __shared__ __align__(16) unsigned char smem[];
  size_t off = 0;
  T* wS = reinterpret_cast<T*>(smem + off);   off += S::w_bytes(nkmax);
  C* X = reinterpret_cast<C*>(smem + off);    off += S::x_bytes(nkmax);
  C* gS = reinterpret_cast<C*>(smem + off);   off += S::g_bytes();
  C* part = reinterpret_cast<C*>(smem + off); off += S::p_bytes(CS);
  T* nrm = reinterpret_cast<T*>(smem + off); off += S::n_bytes(CS);
  const int slice_ = (NF + CS - 1) / CS;
  C* xsl = reinterpret_cast<C*>(smem + off);  off += S::al(sizeof(C) * slice_);
  T* dsl = reinterpret_cast<T*>(smem + off);  off += S::al(sizeof(T) * slice_);
  double* scratch = reinterpret_cast<double*>(smem + off);

  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const T kappa = a.kappa;
  const T cscl = (T)(1.0 / ((double)N * N));  // c = (1/P) FFT_M(z): z carries 2x (row_inverse_pre)
  const C* Dg = a.Wh + (int64_t)k0 * NF;

  // column task of this lane: item (plane cj, column cv) shared by lanes l and l^16, index parity h
  const int citem = warp * 16 + (lane & 15);
  const int hpar = lane >> 4;
  const bool cvalid = citem < nk * Wh;
  const int cj = cvalid ? citem / Wh : 0, cv = cvalid ? citem % Wh : 0;
  C* colp = X + cj * PS + cv;
  const C* dcol = Dg + (int64_t)cj * NF + cv;
  // row task of this thread: plane rj, row rq
  const bool rvalid = tid < nk * N;
  const int rj = rvalid ? tid / N : 0, rq = rvalid ? tid % N : 0;
  C* xrow = X + rj * PS + rq * RS;
  T* wrow = wS + (rj * N + rq) * WP;

  for (int i = tid; i < slice_; i += nt) {
    const int f = r * slice_ + i;
    dsl[i] = f < NF ? (T)1 / a.den[f] : (T)0;
  }
  const int nwarps = nt >> 5;
  const int slice = (NF + CS - 1) / CS;
  // exchange state: mb_part completes when every CTA's partial synthesis for this CTA's slice
  // (and, from the second iteration on, every warp's stopping norms) has landed; mb_g when the
  // g slices of every owner have landed.  Cluster addresses of every CTA's buffers, per rank.
  __shared__ __align__(8) uint64_t mb_part, mb_g;
  __shared__ int s_stat;  // the stopping decision of this iteration (last warp)
  __shared__ uint32_t t_g[16], t_mbg[16], t_part[16], t_mbp[16], t_nrm[16];
  if (tid < CS) {
    t_g[tid] = mapa_u32(smem_u32(gS), tid);
    t_mbg[tid] = mapa_u32(smem_u32(&mb_g), tid);
    t_part[tid] = mapa_u32(smem_u32(part), tid);
    t_mbp[tid] = mapa_u32(smem_u32(&mb_part), tid);
    t_nrm[tid] = mapa_u32(smem_u32(nrm), tid);
  }
  const int my_slice = min(NF, (r + 1) * slice) - r * slice;
  const uint32_t part_bytes = (uint32_t)(CS * my_slice * sizeof(C));
  const uint32_t nrm_bytes = (uint32_t)(CS * nwarps * 5 * sizeof(T));
  if (tid == 0) {
    mbar_init(&mb_part, 1);
    mbar_init(&mb_g, 2);  // tid 0's expect_tx + the last warp's arrival after it publishes the decision
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t ph_part = 0, ph_g = 0;
  if (tid == 0) s_stat = 0;
  cl.sync();  // every CTA's barriers initialised before the first remote st.async

  // ---- column transform of item (cj, cv): Good-Thomas 2 x M across lanes l, l^16 ----------
  // lane parity h shifts every input/output row index by +-M (mod N): the shift's sign is a
  // compile-time function of the row, its magnitude a per-lane register, so no selects
  const int dpx = hpar ? M * RS : 0;  // +M rows in the workspace
  const int dpd = hpar ? M * Wh : 0;  // +M rows in D / F(U)
  const T sgn = hpar ? (T)-1 : (T)1;
  struct ColRegs {
    C v[M];
  };
  // D of this lane's column task: the lane of index parity h touches the rows of parity h both as
  // COL_I inputs (row 2n (+-M), n = 0..M-1) and as COL_F outputs (row (M+1) k2 mod N = 2n (+-M)),
  // so one array of M values covers both passes.  float: loaded once for the whole solve and kept
  // in registers (no per-iteration D traffic); double: reloaded from L2 before each COL_I pass.
  constexpr bool DREG = DREG_;
  static_assert(!DREG || sizeof(T) == 4, "register-resident D is the float path");
  auto load_dcol = [&](ColRegs& dz) {
    sfft::static_for<0, M>([&](auto Nn) {
      constexpr int n2 = decltype(Nn)::value;
      constexpr int u0 = 2 * n2;
      constexpr int sh = (u0 < M) ? 1 : -1;
      dz.v[n2] = dcol[u0 * Wh + sh * dpd];
    });
  };
  ColRegs dreg;  // (loaded at each sample's start: nothing of it stays live across samples)
  // COL_F / COL_FE: forward column transform of the row-transformed planes times D (COL_FE also
  // emits the raw transform, F(U) for the history); COL_I: inverse column transform of conj(D) g
  // (double: z holds D on entry)
  auto col_phase = [&](auto mode_c, C* emit, ColRegs& zr) {
    constexpr int mode = decltype(mode_c)::value;
    C (&z)[M] = zr.v;
    sfft::static_for<0, M>([&](auto Nn) {
      constexpr int n2 = decltype(Nn)::value;
      constexpr int u0 = 2 * n2;                  // row for h = 0
      constexpr int sh = (u0 < M) ? 1 : -1;       // row for h = 1 is u0 + sh*M
      const int ox = u0 * RS + sh * dpx;
      if constexpr (mode == COL_I) {
        const C g = gS[ox + cv];
        const C d = DREG ? dreg.v[n2] : z[n2];
        z[n2] = cmul2(d, mkc<C>(g.x, -g.y));  // conj(conj(D) g): inverse via forward FFT
      } else {
        z[n2] = colp[ox];
      }
    });
    sfft::fft<C, M, false>(z);
    sfft::static_for<0, M>([&](auto Kk) {
      constexpr int k2 = decltype(Kk)::value;
      constexpr int kA = ((M + 1) * k2) % N;      // output row for h = 0; h = 1 is kA + sh*M
      constexpr int sh = (kA < M) ? 1 : -1;
      const C p = mkc<C>(__shfl_xor_sync(0xffffffffu, z[k2].x, 16), __shfl_xor_sync(0xffffffffu, z[k2].y, 16));
      const C o = vfma(z[k2], vsplat<C>(sgn), p);  // h=0: z+p, h=1: p-z
      if (cvalid) {
        const int ox = kA * RS + sh * dpx;
        if constexpr (mode == COL_I) {
          colp[ox] = mkc<C>(o.x, -o.y);
        } else {
          if constexpr (mode == COL_FE) emit[(int64_t)cj * NF + kA * Wh + sh * dpd + cv] = o;
          if constexpr (DREG) colp[ox] = cmul2(dreg.v[kA / 2], o);  // kA is even (M + 1 is)
          else colp[ox] = o;
        }
      }
    });
  };
  // partial synthesis sum over own filters, pushed straight into the owner CTA's receive slot
  // (owner of frequency f = the CTA whose slice [f0, f1) contains it); part is CS x slice
  // thread -> frequencies f = tid + i nt (consecutive across lanes: coalesced D loads); the
  // workspace offset and the owner's receive slot are computed once
  constexpr int RP = 3;  // frequencies per thread: NF <= RP * threads for every launch shape
  int ro[RP], rown[RP];
  uint32_t rdst[RP];
  const C* rdg[RP];
  auto reduce_items = [&]() {  // (recomputed per sample, like D: short live ranges)
#pragma unroll
    for (int i = 0; i < RP; ++i) {
      const int f = tid + i * nt;
      ro[i] = -1;
      rdst[i] = 0;
      rown[i] = 0;
      rdg[i] = Dg;
      if (f < NF) {
        const int u = f / Wh, v = f - u * Wh, owner = f / slice;
        ro[i] = u * RS + v;
        rown[i] = owner;
        rdst[i] = t_part[owner] + (uint32_t)((r * slice + (f - owner * slice)) * sizeof(C));
        rdg[i] = Dg + f;
      }
    }
  };
  // partial synthesis sum_k D_k F(t_k) over own filters, pushed into the owner CTA's slot;
  // the nk (D, X) loads of a frequency are independent, so they issue back to back
  auto push_item = [&](int o, const C* dg, uint32_t dst, int owner) {
    C s = mkc<C>(0, 0), s2 = mkc<C>(0, 0);
    int j = 0;
    if constexpr (DREG) {  // X already holds D F(t): a plain sum over the CTA's planes
      for (; j + 3 < nk; j += 4) {
        s = vadd(s, vadd(X[j * PS + o], X[(j + 1) * PS + o]));
        s2 = vadd(s2, vadd(X[(j + 2) * PS + o], X[(j + 3) * PS + o]));
      }
      for (; j < nk; ++j) s = vadd(s, X[j * PS + o]);
    } else {
      for (; j + 1 < nk; j += 2) {
        s = vfma_c(dg[(int64_t)j * NF], X[j * PS + o], s);
        s2 = vfma_c(dg[(int64_t)(j + 1) * NF], X[(j + 1) * PS + o], s2);
      }
      if (j < nk) s = vfma_c(dg[(int64_t)j * NF], X[j * PS + o], s);
    }
    st_async(dst, vadd(s, s2), t_mbp[owner]);
  };
  // (the D loads of a frequency's planes are L2-bandwidth bound: ~100 KB per CTA per
  // iteration; issuing all of a thread's loads at once measured slower, profiles/README.md)
  auto reduce_push = [&]() {
#pragma unroll
    for (int i = 0; i < RP; ++i)
      if (ro[i] >= 0) push_item(ro[i], rdg[i], rdst[i], rown[i]);
    for (int f = tid + RP * nt; f < NF; f += nt) {  // small launch shapes only
      const int u = f / Wh, v = f - u * Wh, owner = f / slice;
      push_item(u * RS + v, Dg + f, t_part[owner] + (uint32_t)((r * slice + (f - owner * slice)) * sizeof(C)),
                owner);
    }
  };
  // y[f] for my slice from the CS received partials (local loads only)
  auto gather_y = [&](int f) {
    C y = mkc<C>(0, 0);
    const int fl = f - r * slice;
    for (int qq = 0; qq < CS; ++qq) y = cadd(y, part[qq * slice + fl]);
    return y;
  };

  // ---- the samples of this cluster: one (plain launch) or a schedule row (persistent launch) --
  // (the row position lives in shared memory and the sample is re-derived after the iterations,
  // so the outer loop adds no register live across them)
  __shared__ int s_sw;
  auto sample_at = [&](int sw) {
    if (a.sched) return sw < a.sched_w ? a.sched[(a.sched_c0 + ci) * a.sched_w + sw] : -1;
    return sw == 0 ? a.b0 + ci : -1;
  };
  if (tid == 0) s_sw = 0;
  __syncthreads();
  for (;;) {
  const int sw = s_sw;
  const int b = sample_at(sw);
  if (b < 0) break;
  // per-sample state: a fresh phase of both exchange barriers (a remote transaction may land
  // before the arm; the tx count just dips below zero), zero workspace, this sample's spectrum
  if (tid == 0) {
    mbar_arm(&mb_part, part_bytes);  // first phase of a sample: partials only
    mbar_arm(&mb_g, (uint32_t)(NF * sizeof(C)));
  }
  for (int i = tid; i < nk * N * WP; i += nt) wS[i] = (T)0;
  for (int i = tid; i < nk * PS; i += nt) X[i] = mkc<C>(0, 0);
  for (int i = tid; i < slice_; i += nt) {
    const int f = r * slice_ + i;
    xsl[i] = f < NF ? a.xh[(int64_t)b * NF + f] : mkc<C>(0, 0);
  }
  if constexpr (DREG) load_dcol(dreg);
  reduce_items();
  __syncthreads();
  int it = 0, stat = 0;
  const bool first = blockIdx.x == 0 && a.b0 == 0 && sw == 0 && a.sched_c0 == 0 && tid == 0;
  long long* prof = first ? g_fused_prof : nullptr;
  long long* tl = (r == 0 && tid == 0) ? g_fused_timeline : nullptr;
  if (tl) tl[2 * b] = global_ns();
  long long* itl = first ? g_fused_iter : nullptr;
  for (;;) {
    const int pit = it;
    if (itl && it < 512) {
      itl[it] = global_ns();
      itl[512 + it] = clock64();
    }
    // ---- A: forward column transforms, partial synthesis sum_k D_k F(t_k) ----------------
    OCSC_STAMP(0);
    {
      ColRegs zc;
      col_phase(std::integral_constant<int, COL_F>{}, nullptr, zc);
    }
    __syncthreads();
    OCSC_STAMP(1);
    reduce_push();
    OCSC_STAMP(3);
    // #1: this CTA's slice of every partial (and every warp's stopping norms) has landed
    mbar_wait(&mb_part, ph_part);
    ph_part ^= 1;
    OCSC_STAMP(2);
    const T* nr = nrm + (it & 1) * (8 * 32 * CS);  // the norms pushed by the last row phase
    if (warp == nwarps - 1 && it > 0) {
      // the last warp (no g work below) reduces the CS x nwarps partials in a fixed order
      // (lane-strided, then a fixed butterfly): the same decision in every CTA; the rest of the
      // CTA reads it after the g wait below (which orders it: this warp's own g stores follow)
      T n4[5] = {0, 0, 0, 0, 0};
      for (int qq = 0; qq < CS; ++qq) {
        if (lane < nwarps) {
          const T* src = nr + qq * 8 * 32 + lane;  // [qq][i][warp]: lanes read consecutive words
#pragma unroll
          for (int i = 0; i < 5; ++i) n4[i] += src[i * 32];
        }
      }
#pragma unroll
      for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n4[i] += __shfl_xor_sync(0xffffffffu, n4[i], o);
      // coding.py:113-118 on squared norms: num <= tol max(den, 1e-12) and
      // gap <= tol max(den, |dual|, 1e-12)
      const T tol2 = (T)(a.tol * a.tol), fl2 = (T)1e-24;
      int st_ = 0;
      if (n4[4] > (T)0) st_ = 2;
      else if (n4[0] <= tol2 * fmax(n4[1], fl2) && n4[2] <= tol2 * fmax(fmax(n4[1], n4[3]), fl2)) st_ = 1;
      if (lane == 0) {
        s_stat = st_;
        // arm the next partial phase: the output stage's (partials only) or the next
        // iteration's (partials + the norms of the row phase below)
        mbar_arm(&mb_part, st_ || it == a.max_iters ? part_bytes : part_bytes + nrm_bytes);
      }
    } else if (warp == nwarps - 1 && lane == 0) {
      mbar_arm(&mb_part, it == a.max_iters ? part_bytes : part_bytes + nrm_bytes);
    }
    if (warp == nwarps - 1 && lane == 0) mbar_arrive(&mb_g);  // s_stat is published with this phase
    // ---- y on my slice from the pushed partials, g = (X - y)/den, pushed to every rank -----
    {
      const int f0 = r * slice, f1 = min(NF, f0 + slice);
      for (int f = f0 + tid; f < f1; f += nt) {
        const C y = gather_y(f);
        const int fl = f - f0;
        const C g = cscale(csub(xsl[fl], y), dsl[fl]);
        const uint32_t o = (uint32_t)(((f / Wh) * RS + f % Wh) * sizeof(C));
        for (int qq = 0; qq < CS; ++qq) st_async(t_g[qq] + o, g, t_mbg[qq]);
      }
    }
    OCSC_STAMP(4);
    // double: D for the inverse column pass, loaded before the wait (its L2 latency hides there)
    ColRegs zi;
    if constexpr (!DREG) load_dcol(zi);
    // #2: every owner's g slice has landed in this CTA (g of a stopping iteration is pushed and
    // waited for too, so no remote store is in flight when the CTAs leave the loop)
    mbar_wait(&mb_g, ph_g);
    ph_g ^= 1;
    if (it > 0 && s_stat) {
      stat = s_stat;
      break;
    }
    if (it == a.max_iters) break;
    ++it;
    if (tid == 0) mbar_arm(&mb_g, (uint32_t)(NF * sizeof(C)));
    OCSC_STAMP(5);
    // ---- B: inverse column transforms of conj(D) g ---------------------------------------
    col_phase(std::integral_constant<int, COL_I>{}, nullptr, zi);
    __syncthreads();
    OCSC_STAMP(7);
    // ---- C: row IFFT -> c -> update w (registers) -> t -> row FFT --------------------------
    // (even, odd) pixel pairs run as 2-wide FP32x2 arithmetic
    C s0 = mkc<C>(0, 0), s1 = mkc<C>(0, 0), s2 = mkc<C>(0, 0), s3 = mkc<C>(0, 0);
    if (rvalid) {
      C z[M];
      row_inverse_pre<C, N>(xrow, z);
      sfft::fft<C, M, false>(z);
      const C cs2 = mkc<C>(cscl, -cscl);  // c = (Re, -Im) / P of the conjugated result
      C* w2 = reinterpret_cast<C*>(wrow);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const C wo = w2[m];
        const C go = mkc<C>(clampk(wo.x, kappa), clampk(wo.y, kappa));
        const C uo = vsub(wo, go);
        const C wn = vfma(z[m], cs2, uo);  // w' = S(w) + c
        const C gn = mkc<C>(clampk(wn.x, kappa), clampk(wn.y, kappa));
        const C un = vsub(wn, gn);
        const C d0 = vsub(un, uo), d2 = vsub(gn, go);  // a non-finite code poisons these sums
        s0 = vfma(d0, d0, s0);
        s1 = vfma(un, un, s1);
        s2 = vfma(d2, d2, s2);
        s3 = vfma(gn, gn, s3);
        w2[m] = wn;
        z[m] = vfma(wn, vsplat<C>((T)0.5), mkc<C>(-gn.x, -gn.y));  // t / 2 = (w' - 2 clip(w')) / 2 (row_forward_post)
      }
      sfft::fft<C, M, false>(z);
      row_forward_post<C, N>(z, xrow);
    }
    // a non-finite code value poisons this thread's partial sums; warp-reduce in float and
    // push each warp's five partials straight into every CTA of the cluster (no block barrier)
    {
      T q[5] = {s0.x + s0.y, s1.x + s1.y, s2.x + s2.y, s3.x + s3.y, (T)0};
      q[4] = (isfinite(q[0]) && isfinite(q[1]) && isfinite(q[2]) && isfinite(q[3])) ? (T)0 : (T)1;
#pragma unroll
      for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q[i] += __shfl_xor_sync(0xffffffffu, q[i], o);
      if (lane < CS) {  // into the buffer the next decision reads (parity of the incremented it)
        const uint32_t dst = t_nrm[lane] + (uint32_t)((((it & 1) * CS + r) * 8 * 32 + warp) * sizeof(T));
#pragma unroll
        for (int i = 0; i < 5; ++i) st_async(dst + (uint32_t)(i * 32 * sizeof(T)), q[i], t_mbp[lane]);
      }
    }
    OCSC_STAMP(6);
    __syncthreads();  // row outputs complete before the next column phase
  }

  // ---- outputs: U = S(w) (and t), F(U), objective -------------------------------------------
  if (itl) itl[505] = global_ns();
  {
  const int b = sample_at(s_sw);
  double l1 = 0.0;
  if (rvalid) {
    const int64_t rowoff = (((int64_t)b * K + k0 + rj) * N + rq) * N;
    T* uo = a.u_out + rowoff;
    T* to = a.t_out ? a.t_out + rowoff : nullptr;
    C z[M];
    const C* w2 = reinterpret_cast<const C*>(wrow);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const T va = w2[m].x, vb = w2[m].y;
      const T ga = clampk(va, kappa), gb = clampk(vb, kappa);
      const T ua = va - ga, ub = vb - gb;
      uo[2 * m] = ua;
      uo[2 * m + 1] = ub;
      if (to) {
        to[2 * m] = ua - ga;
        to[2 * m + 1] = ub - gb;
      }
      l1 += fabs((double)ua) + fabs((double)ub);
      z[m] = mkc<C>((T)0.5 * ua, (T)0.5 * ub);  // row_forward_post takes the half-scaled row
    }
    sfft::fft<C, M, false>(z);
    row_forward_post<C, N>(z, xrow);
  }
  __syncthreads();
  if (itl) itl[506] = global_ns();
  {
    ColRegs zc;
    col_phase(std::integral_constant<int, COL_FE>{}, a.uh_out + ((int64_t)b * K + k0) * NF, zc);
  }
  __syncthreads();
  if (itl) itl[507] = global_ns();
  reduce_push();
  mbar_wait(&mb_part, ph_part);
  ph_part ^= 1;
  if (itl) itl[508] = global_ns();
  double e = 0.0;
  {
    const int f0 = r * slice, f1 = min(NF, f0 + slice);
    for (int f = f0 + tid; f < f1; f += nt) {
      const C y = gather_y(f);
      const C res = csub(xsl[f - f0], y);
      e += herm_weight(f % Wh, N) * ((double)res.x * res.x + (double)res.y * res.y);
    }
  }
  double ev[2] = {e, l1};
  block_allsum<2>(ev, scratch);
  double* fin = scratch + 6 * 32 - 2 * 16;  // [16][2] slots at the end of the scratch area
  if (tid == 0) {
    double* dst = cl.map_shared_rank(fin, 0) + 2 * r;
    dst[0] = ev[0];
    dst[1] = ev[1];
  }
  cl.sync();
  if (itl) itl[509] = global_ns();
  if (r == 0 && tid == 0) {
    double energy = 0.0, l1s = 0.0;
    for (int qq = 0; qq < CS; ++qq) {
      energy += fin[2 * qq];
      l1s += fin[2 * qq + 1];
    }
    const double invPd = 1.0 / ((double)N * N);
    a.obj[b] = 0.5 * invPd * energy + a.beta * l1s;
    if (a.resid) a.resid[b] = invPd * energy;
    a.iters[b] = it;
    a.status[b] = stat;
    if (tl) tl[2 * b + 1] = global_ns();
  }
  }
  if (tid == 0) s_sw = s_sw + 1;  // (every thread read it before the barriers above)
  __syncthreads();
  }  // samples of this cluster
  // a programmatically launched grid completes only after the grid it overlaps (so stream order
  // holds for whatever follows it); a no-op for a plain launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------- dispatch --
struct FusedShape {
  int cs = 0, threads = 0, nk = 0, active = 0;
  bool dreg = false;
  size_t smem = 0;
};
// the kernel instantiation of a shape's variant (double has only the L2-D variant)
template <typename T, int N>
static auto kernel_of(bool dreg) -> void (*)(FusedArgs<T>) {
  if constexpr (sizeof(T) == 4) return dreg ? k_code_fused<T, N, true> : k_code_fused<T, N, false>;
  else return k_code_fused<T, N, false>;
}
// A plan is one of two kinds.
//  * sequential: `main` clusters in waves (one cluster per sample) for the first b_main samples,
//    then the rest on `tail`, a wider shape, instead of a mostly idle last wave;
//  * concurrent: `main` runs persistent (n_main resident clusters, each coding a row of a
//    static schedule), and `side`, a smaller shape that fits the SMs the main clusters leave
//    free (GPC packing: eleven 10-CTA clusters leave 38 of 148 SMs, which hold four 8-CTA
//    clusters), is launched programmatically behind it on the same stream and codes its own
//    schedule rows at the same time.
struct FusedPlan {
  FusedShape main, tail, side;
  int b_main = 0;                  // sequential: samples on the main waves
  int n_main = 0, n_side = 0;      // concurrent: clusters launched per shape
  int sched_w = 0;                 // concurrent: samples per schedule row
  int32_t* sched = nullptr;        // concurrent: device table [(main.active + n_side) x sched_w]
  int b_split = 0;                 // samples the plan finishes before its last main round starts
  double makespan = 0;             // modelled, in cost units
};

template <typename T, int N>
static int max_active_clusters(const FusedShape& sh, int B) {
  auto kern = kernel_of<T, N>(sh.dreg);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem);
  if (sh.cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B * sh.cs, 1, 1);
  cfg.blockDim = dim3(sh.threads, 1, 1);
  cfg.dynamicSmemBytes = sh.smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = sh.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// launch `nclu` clusters of shape sh; pdl: programmatic launch behind the previous grid on s
template <typename T, int N>
static cudaError_t launch_clusters(const FusedArgs<T>& a, const FusedShape& sh, int nclu, bool pdl, cudaStream_t s) {
  auto kern = kernel_of<T, N>(sh.dreg);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem);
  if (e != cudaSuccess) return e;
  if (sh.cs > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclu * sh.cs, 1, 1);
  cfg.blockDim = dim3(sh.threads, 1, 1);
  cfg.dynamicSmemBytes = sh.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = sh.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// How many clusters of `side` run while main.active clusters of `main` are resident: measured
// once per shape pair with the kernels themselves in probe mode (the main grid spins for a
// while, the side grid is launched programmatically behind it and stamps when each cluster
// starts).  Cached; 0 when the probe cannot run (e.g. inside a stream capture).
template <typename T, int N>
static int side_capacity(const FusedShape& main, const FusedShape& side) {
  static std::map<std::tuple<int, int, int, int, int, int, int, int>, int> cache;  // (caller holds the plan lock)
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, main.cs, (int)main.dreg, (int)main.smem, side.cs, (int)side.dreg,
                                   (int)side.smem, side.threads);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  cudaStream_t s = nullptr;
  unsigned long long* rec = nullptr;
  const int nrec = 1 + side.active;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
      cudaMalloc(&rec, sizeof(unsigned long long) * nrec) == cudaSuccess &&
      cudaMemsetAsync(rec, 0xff, sizeof(unsigned long long) * nrec, s) == cudaSuccess) {
    FusedArgs<T> pa{};
    pa.probe = rec;
    pa.probe_ns = 300000;  // 0.3 ms: every co-resident side cluster starts well inside it
    pa.probe_role = 0;
    bool ok = launch_clusters<T, N>(pa, main, main.active, false, s) == cudaSuccess;
    pa.probe_role = 1;
    ok = ok && launch_clusters<T, N>(pa, side, side.active, true, s) == cudaSuccess;
    std::vector<unsigned long long> h(nrec);
    ok = ok && cudaStreamSynchronize(s) == cudaSuccess &&
         cudaMemcpy(h.data(), rec, sizeof(unsigned long long) * nrec, cudaMemcpyDeviceToHost) == cudaSuccess;
    if (ok)
      for (int c = 0; c < side.active; ++c) n += h[1 + c] < h[0];
    if (ok && getenv("OCSC_FUSED_PROBE_DEBUG")) {
      unsigned long long t0 = h[0];
      for (int c = 0; c < side.active; ++c) t0 = std::min(t0, h[1 + c]);
      fprintf(stderr, "side_capacity main cs=%d x%d side cs=%d x%d: main end %+.1f us, side starts", main.cs,
              main.active, side.cs, side.active, (h[0] - t0) * 1e-3);
      for (int c = 0; c < side.active; ++c) fprintf(stderr, " %.1f", (h[1 + c] - t0) * 1e-3);
      fprintf(stderr, " -> %d\n", n);
    }
  }
  cudaGetLastError();
  if (rec) cudaFree(rec);
  if (s) cudaStreamDestroy(s);
  cache.emplace(key, n);
  return n;
}

// cost of one sample on a shape, in model units: filters per CTA plus a fixed per-iteration
// cluster overhead (fitted to scripts/cluster_sweep.py on a B200); register-resident D: 17.8 k
// cycles per iteration at 10 filters per CTA against 23.9 k at 12 filters with D reloaded from
// L2 (profiles/r2_phase_*.log)
static double shape_cost(const FusedShape& sh) { return ((double)sh.nk + 3.5) * (sh.dreg ? 0.856 : 1.0); }

// Static list schedule of B equal-cost samples over nm clusters of cost cm and ns of cost cs_:
// each sample goes to the cluster that would finish it first (main first on ties); samples are
// then numbered in order of modelled completion, so [0, b) are the first b to finish.
struct Schedule {
  std::vector<std::vector<int>> rows;  // per cluster (main rows first), sample indices
  double makespan = 0, last_main_start = 0;
  int used_side = 0, b_split = 0;
};
static Schedule list_schedule(int B, int nm, double cm, int ns, double cs_) {
  Schedule sc;
  const int nc = nm + ns;
  std::vector<double> fin(nc, 0.0);
  std::vector<std::tuple<double, int, int>> slots;  // (completion, cluster, position in row)
  std::vector<int> len(nc, 0);
  for (int s = 0; s < B; ++s) {
    int best = 0;
    double bt = 1e300;
    for (int c = 0; c < nc; ++c) {
      const double t = fin[c] + (c < nm ? cm : cs_);
      if (t < bt - 1e-9) {
        bt = t;
        best = c;
      }
    }
    fin[best] = bt;
    slots.emplace_back(bt, best, len[best]++);
  }
  std::sort(slots.begin(), slots.end());
  sc.rows.assign(nc, {});
  for (int c = 0; c < nc; ++c) sc.rows[c].assign(len[c], -1);
  for (int i = 0; i < B; ++i) sc.rows[std::get<1>(slots[i])][std::get<2>(slots[i])] = i;
  for (int c = 0; c < nc; ++c) {
    sc.makespan = std::max(sc.makespan, fin[c]);
    if (c < nm) sc.last_main_start = std::max(sc.last_main_start, fin[c] - cm);
    if (c >= nm && len[c]) ++sc.used_side;
  }
  for (int i = 0; i < B; ++i) sc.b_split += std::get<0>(slots[i]) <= sc.last_main_start + 1e-9;
  return sc;
}

// Choose the plan with the smallest modelled makespan: every (main, tail) pair of the
// sequential kind, and (main, side) pairs of the concurrent kind for the three main shapes with
// the highest throughput and every narrower side shape that co-resides with them.  BASELINE
// config 1 (K = 100, B = 50, float): eleven 10-CTA clusters (register-resident D) plus four
// 8-CTA clusters; 42 + 8 samples, four main rounds.
template <typename T, int N>
static FusedPlan plan_for(int K, int B, bool can_probe) {
  FusedPlan plan;
  int dev = 0, max_smem = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return plan;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  FusedShape shapes[32];
  int ns = 0;
  const char* force = getenv("OCSC_FUSED_CS");  // dev knob: a single cluster size, no tail/side
  const int fcs = force ? atoi(force) : 0;
  const char* fdr = getenv("OCSC_FUSED_DREG");  // dev knob: 0 / 1 forces the D variant
  const char* fside = getenv("OCSC_FUSED_SIDE");  // dev knob: 0 disables the concurrent kind
  for (int v = 0; v < (sizeof(T) == 4 ? 2 : 1); ++v) {
    const bool dreg = sizeof(T) == 4 && v == 0;
    if (fdr && atoi(fdr) != (int)dreg) continue;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kernel_of<T, N>(dreg)) != cudaSuccess) continue;
    for (int cs = 2; cs <= 16; ++cs) {
      if (cs > K) break;
      if (fcs && cs != fcs) continue;
      FusedShape sh;
      sh.cs = cs;
      sh.dreg = dreg;
      sh.nk = (K + cs - 1) / cs;
      sh.smem = Smem<T, N>::total(sh.nk, cs);
      sh.threads = Smem<T, N>::threads(sh.nk);
      if (sh.smem > (size_t)max_smem || sh.threads > fa.maxThreadsPerBlock) continue;
      sh.active = max_active_clusters<T, N>(sh, 1024);
      if (sh.active > 0) shapes[ns++] = sh;
    }
  }
  if (!ns) return plan;
  double best_t = 1e300;
  // sequential kind: full waves of the main shape, then the remainder either as one more main
  // wave or on the tail shape's waves
  for (int m = 0; m < ns; ++m) {
    const FusedShape& M = shapes[m];
    const int nfull = B / M.active, rem = B - nfull * M.active;
    double t = nfull * shape_cost(M);
    int tail = -1;
    if (rem > 0) {
      double tr = shape_cost(M);
      if (nfull > 0)
        for (int i = 0; i < ns; ++i) {
          const double ti = (double)((rem + shapes[i].active - 1) / shapes[i].active) * shape_cost(shapes[i]);
          if (ti < tr * 0.98) {
            tr = ti;
            tail = i;
          }
        }
      t += tr;
    }
    if (t < best_t * 0.999) {
      best_t = t;
      plan = FusedPlan{};
      plan.main = M;
      plan.tail = tail >= 0 ? shapes[tail] : FusedShape{};
      plan.b_main = tail >= 0 ? nfull * M.active : B;
      plan.b_split = tail >= 0 ? plan.b_main : B;
      plan.makespan = t;
    }
  }
  // concurrent kind
  if (!can_probe || fcs || (fside && atoi(fside) == 0) || B <= 1) return plan;
  int order[32];
  for (int i = 0; i < ns; ++i) order[i] = i;
  std::sort(order, order + ns, [&](int x, int y) {
    return shapes[x].active / shape_cost(shapes[x]) > shapes[y].active / shape_cost(shapes[y]);
  });
  Schedule best_sc;
  int best_m = -1, best_s = -1, best_nside = 0;
  for (int oi = 0; oi < std::min(ns, 3); ++oi) {
    const FusedShape& M = shapes[order[oi]];
    if (B <= M.active) continue;  // one round: nothing for a side shape to take
    for (int si = 0; si < ns; ++si) {
      const FusedShape& S = shapes[si];
      if (S.cs > M.cs) continue;
      const int cap = side_capacity<T, N>(M, S);
      if (cap <= 0) continue;
      Schedule sc = list_schedule(B, M.active, shape_cost(M), cap, shape_cost(S));
      if (sc.used_side == 0) continue;
      if (sc.makespan < best_t * 0.98) {
        best_t = sc.makespan;
        best_sc = sc;
        best_m = order[oi];
        best_s = si;
        best_nside = cap;
      }
    }
  }
  if (best_m < 0) return plan;
  FusedPlan cp;
  cp.main = shapes[best_m];
  cp.side = shapes[best_s];
  cp.n_main = std::min(cp.main.active, B);
  cp.n_side = best_sc.used_side;
  cp.makespan = best_sc.makespan;
  cp.b_split = best_sc.b_split;
  cp.b_main = B;
  int w = 0;
  for (const auto& row : best_sc.rows) w = std::max(w, (int)row.size());
  cp.sched_w = w;
  const int rows = cp.main.active + best_nside;
  std::vector<int32_t> h((size_t)rows * w, -1);
  for (int c = 0; c < rows; ++c)
    for (size_t i = 0; i < best_sc.rows[c].size(); ++i) h[(size_t)c * w + i] = best_sc.rows[c][i];
  if (cudaMalloc(&cp.sched, h.size() * sizeof(int32_t)) != cudaSuccess ||
      cudaMemcpy(cp.sched, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    if (cp.sched) cudaFree(cp.sched);
    return plan;  // (the table lives as long as the cached plan: the process)
  }
  return cp;
}

template <typename T, int N>
static const FusedPlan& cached_plan(int K, int B, cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, FusedPlan> cache;  // map nodes are stable
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  auto key = std::make_tuple(dev, K, B);
  auto it = cache.find(key);
  if (it == cache.end()) {
    // the side-shape probe launches and synchronises: not from inside a stream capture (such a
    // plan is not cached, so a later uncaptured call still gets the concurrent kind)
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (s) cudaStreamIsCapturing(s, &cst);
    cudaStreamCaptureStatus lst = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(cudaStreamLegacy, &lst);
    cudaGetLastError();
    const bool can_probe = cst == cudaStreamCaptureStatusNone && lst == cudaStreamCaptureStatusNone;
    if (!can_probe) {
      static thread_local FusedPlan tmp;
      tmp = plan_for<T, N>(K, B, false);
      return tmp;
    }
    it = cache.emplace(key, plan_for<T, N>(K, B, true)).first;
  }
  return it->second;
}

template <typename T, int N>
static int launch_shape(FusedArgs<T> a, const FusedShape& sh, int b0, int nb, cudaStream_t s) {
  if (nb <= 0) return OCSC_OK;
  a.b0 = b0;
  a.sched = nullptr;
  OCSC_CUDA((launch_clusters<T, N>(a, sh, nb, false, s)));
  OCSC_LAUNCHED("k_code_fused");
  return OCSC_OK;
}

template <typename T, int N>
static int launch_fused(const FusedArgs<T>& a, cudaStream_t s) {
  const FusedPlan& p = cached_plan<T, N>(a.K, a.B, s);
  if (!p.main.cs) return fail(OCSC_EARG, "fused code ADMM: no cluster shape fits this device");
  if (p.sched) {  // concurrent: persistent main grid, the side grid programmatically behind it
    FusedArgs<T> m = a;
    m.b0 = 0;
    m.sched = p.sched;
    m.sched_w = p.sched_w;
    m.sched_c0 = 0;
    OCSC_CUDA((launch_clusters<T, N>(m, p.main, p.n_main, false, s)));
    OCSC_LAUNCHED("k_code_fused");
    m.sched_c0 = p.main.active;
    OCSC_CUDA((launch_clusters<T, N>(m, p.side, p.n_side, true, s)));
    OCSC_LAUNCHED("k_code_fused");
    return OCSC_OK;
  }
  int rc = launch_shape<T, N>(a, p.main, 0, p.b_main, s);
  if (rc) return rc;
  return launch_shape<T, N>(a, p.tail, p.b_main, a.B - p.b_main, s);
}

template <typename T, int N>
static int query_fused(int K, int B, int* info, int* side) {
  const FusedPlan& p = cached_plan<T, N>(K, B, nullptr);
  if (info) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kernel_of<T, N>(p.main.dreg));
    info[0] = p.main.cs;
    info[1] = p.main.threads;
    info[2] = (int)p.main.smem;
    info[3] = fa.numRegs;
    info[4] = p.main.active;
    info[5] = p.b_split;
    FusedShape rest = p.tail;
    if (p.sched && p.b_split < B) {
      const FusedPlan& q = cached_plan<T, N>(K, B - p.b_split, nullptr);
      rest = q.main;
      rest.active = q.main.active;
    }
    info[6] = p.b_split < B ? rest.cs : 0;
    info[7] = p.b_split < B ? rest.active : 0;
  }
  if (side) {
    side[0] = p.sched ? p.side.cs : 0;
    side[1] = p.n_side;
    side[2] = (int)p.side.dreg;
    side[3] = p.n_main;
    side[4] = p.sched_w;
    side[5] = (int)p.main.dreg;
    side[6] = (int)(p.makespan * 1000.0);
    side[7] = p.sched ? 1 : 0;
  }
  return p.main.cs;
}

// the grids the fused kernel is instantiated for (BASELINE config 1 is 42 x 42)
#define OCSC_FUSED_SIZES(X) X(42) X(10) X(14) X(18) X(30)

template <typename T>
static int fused_dispatch(int H, int W, bool query, const FusedArgs<T>* a, int K, int B, cudaStream_t s,
                          int* info = nullptr, int* side = nullptr) {
#define OCSC_CASE(NN) \
  if (H == NN && W == NN) return query ? query_fused<T, NN>(K, B, info, side) : launch_fused<T, NN>(*a, s);
  OCSC_FUSED_SIZES(OCSC_CASE)
#undef OCSC_CASE
  return query ? 0 : fail(OCSC_EARG, "fused code ADMM: grid not instantiated");
}

}  // namespace ocsc

using namespace ocsc;

extern "C" int ocsc_debug_fused_profile(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  OCSC_CUDA(cudaMemcpyToSymbol(g_fused_prof, &p, sizeof(p)));
  return OCSC_OK;
}

extern "C" int ocsc_debug_fused_iterations(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  OCSC_CUDA(cudaMemcpyToSymbol(g_fused_iter, &p, sizeof(p)));
  return OCSC_OK;
}

extern "C" int ocsc_debug_fused_timeline(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  OCSC_CUDA(cudaMemcpyToSymbol(g_fused_timeline, &p, sizeof(p)));
  return OCSC_OK;
}

extern "C" int ocsc_code_fused_info(int dtype, int H, int W, int K, int B, int32_t* info) {
  for (int i = 0; i < 8; ++i) info[i] = 0;
  if (K <= 0 || B <= 0) return 0;
  if (dtype == OCSC_F32) return fused_dispatch<float>(H, W, true, nullptr, K, B, nullptr, info);
  if (dtype == OCSC_F64) return fused_dispatch<double>(H, W, true, nullptr, K, B, nullptr, info);
  return 0;
}

extern "C" int ocsc_code_fused_side_info(int dtype, int H, int W, int K, int B, int32_t* info) {
  for (int i = 0; i < 8; ++i) info[i] = 0;
  if (K <= 0 || B <= 0) return 0;
  if (dtype == OCSC_F32) return fused_dispatch<float>(H, W, true, nullptr, K, B, nullptr, nullptr, info);
  if (dtype == OCSC_F64) return fused_dispatch<double>(H, W, true, nullptr, K, B, nullptr, nullptr, info);
  return 0;
}

extern "C" int ocsc_code_fused_cluster(int dtype, int H, int W, int K, int B) {
  if (K <= 0 || B <= 0) return 0;
  if (dtype == OCSC_F32) return fused_dispatch<float>(H, W, true, nullptr, K, B, nullptr);
  if (dtype == OCSC_F64) return fused_dispatch<double>(H, W, true, nullptr, K, B, nullptr);
  return 0;
}

extern "C" int ocsc_code_fused(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh,
                               const void* den, double beta, double rho, int max_iters, double rel_tol, void* u,
                               void* t, void* uh, double* obj, double* resid, int32_t* iters, int32_t* status,
                               void* stream) {
  if (H <= 0 || W <= 0 || K <= 0 || B < 0) return fail(OCSC_ESHAPE, "code_fused: bad extents");
  if (!(rho > 0)) return fail(OCSC_EARG, "code_fused: rho must be positive");
  if (B == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32) {
    FusedArgs<float> a{K, B, max_iters, 0, rel_tol, beta, (float)(beta / rho), (const float2*)xh, (const float2*)Wh,
                       (const float*)den, (float*)u, (float*)t, (float2*)uh, obj, resid, iters, status};
    return fused_dispatch<float>(H, W, false, &a, K, B, s);
  }
  if (dtype == OCSC_F64) {
    FusedArgs<double> a{K, B, max_iters, 0, rel_tol, beta, beta / rho, (const double2*)xh, (const double2*)Wh,
                        (const double*)den, (double*)u, (double*)t, (double2*)uh, obj, resid, iters, status};
    return fused_dispatch<double>(H, W, false, &a, K, B, s);
  }
  return fail(OCSC_EARG, "dtype must be 4 or 8");
}
