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

#include "common.cuh"
#include "fft_small.cuh"

namespace cg = cooperative_groups;

namespace ocsc {

template <typename T>
struct FusedArgs {
  int K, B, max_iters;
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
};

template <int H, int W>
struct Geo {
  static constexpr int Wh = W / 2 + 1;
  static constexpr int WP = (W % 2 == 0) ? W + 1 : W;   // odd row stride of w (bank-conflict free)
  static constexpr int WhP = (Wh % 2 == 0) ? Wh + 1 : Wh;  // odd complex row stride of the workspace
  static constexpr int NF = H * Wh;
  static constexpr int H2 = H / 2;
  static_assert(H % 2 == 0, "fused path pairs rows: H must be even");
};

template <typename T>
__device__ __forceinline__ T soft(T a, T k) {
  return a > k ? a - k : (a < -k ? a + k : (a == a ? (T)0 : a));
}
template <typename T>
__device__ __forceinline__ T clipk(T a, T k) {
  return a > k ? k : (a < -k ? -k : a);
}

// shared-memory carve-up (all offsets 16-byte aligned)
template <typename T, int H, int W>
struct Smem {
  using G = Geo<H, W>;
  static __host__ __device__ size_t w_bytes(int nk) { return align16(sizeof(T) * (size_t)nk * H * G::WP); }
  static __host__ __device__ size_t x_bytes(int nk) { return align16(sizeof(cx<T>) * (size_t)nk * H * G::WhP); }
  static __host__ __device__ size_t g_bytes() { return align16(sizeof(cx<T>) * (size_t)H * G::WhP); }
  static __host__ __device__ size_t p_bytes() { return align16(sizeof(cx<T>) * (size_t)G::NF); }
  static __host__ __device__ size_t n_bytes(int cs) { return align16(sizeof(double) * 8 * (size_t)cs); }
  static __host__ __device__ size_t total(int nk, int cs) {
    return w_bytes(nk) + x_bytes(nk) + g_bytes() + p_bytes() + n_bytes(cs) + 6 * 32 * sizeof(double);  // + block_allsum scratch
  }
  static __host__ __device__ size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
};

// block-wide sum of NV doubles, result broadcast to every thread
template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * 32 + warp] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = 0.0;
    for (int q = 0; q < nw; ++q) s += scratch[i * 32 + q];
    v[i] = s;
  }
  __syncthreads();
}

template <typename T, int H, int W>
__global__ void __launch_bounds__(384, 1) k_code_fused(FusedArgs<T> a) {
  using C = cx<T>;
  using G = Geo<H, W>;
  using S = Smem<T, H, W>;
  constexpr int Wh = G::Wh, WP = G::WP, WhP = G::WhP, NF = G::NF, H2 = G::H2;

  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int r = (int)cl.block_rank();
  const int b = blockIdx.x / CS;
  const int K = a.K;
  const int k0 = (int)((int64_t)r * K / CS), k1 = (int)((int64_t)(r + 1) * K / CS);
  const int nk = k1 - k0;
  const int nkmax = (K + CS - 1) / CS;

  extern __shared__ __align__(16) unsigned char smem[];
  T* wS = reinterpret_cast<T*>(smem);
  C* Xf = reinterpret_cast<C*>(smem + S::w_bytes(nkmax));
  C* gS = reinterpret_cast<C*>(smem + S::w_bytes(nkmax) + S::x_bytes(nkmax));
  C* part = reinterpret_cast<C*>(smem + S::w_bytes(nkmax) + S::x_bytes(nkmax) + S::g_bytes());
  double* norms = reinterpret_cast<double*>(smem + S::w_bytes(nkmax) + S::x_bytes(nkmax) + S::g_bytes() +
                                            S::p_bytes());
  double* scratch = norms + 8 * CS;

  const int tid = threadIdx.x, nt = blockDim.x;
  const T kappa = a.kappa;
  const T invP = (T)(1.0 / ((double)H * W));
  const C* Dg = a.Wh + (int64_t)k0 * NF;
  const int nrow_tasks = nk * H2, ncol_tasks = nk * Wh;

  // cold start: w = 0, so t = 0 and its row transforms are 0
  for (int i = tid; i < nk * H * WP; i += nt) wS[i] = (T)0;
  for (int i = tid; i < nk * H * WhP; i += nt) Xf[i] = mkc<C>(0, 0);
  __syncthreads();

  // ---------------------------------------------------------------- pieces --
  // forward column FFT of the row-transformed plane j, column v; optionally emit it; Xf <- D * col
  auto col_forward = [&](int j, int v, C* emit) {
    C col[H];
#pragma unroll
    for (int u = 0; u < H; ++u) col[u] = Xf[(j * H + u) * WhP + v];
    sfft::fft<C, H, false>(col);
#pragma unroll
    for (int u = 0; u < H; ++u) {
      if (emit) emit[u * Wh + v] = col[u];
      Xf[(j * H + u) * WhP + v] = cmul(Dg[(int64_t)j * NF + u * Wh + v], col[u]);
    }
  };
  // sum over own filters -> part (the CTA's share of sum_k D_k T_k)
  auto reduce_part = [&]() {
    for (int f = tid; f < NF; f += nt) {
      const int u = f / Wh, v = f % Wh;
      C s = mkc<C>(0, 0);
      for (int j = 0; j < nk; ++j) s = cadd(s, Xf[(j * H + u) * WhP + v]);
      part[f] = s;
    }
  };
  // rows q and q+H/2 of plane j: value(w) of the stored w -> packed forward row FFT -> Xf rows
  auto row_forward_store = [&](int j, int q, auto value) {
    const T* wa = wS + (j * H + q) * WP;
    const T* wb = wS + (j * H + q + H2) * WP;
    C z[W];
#pragma unroll
    for (int n = 0; n < W; ++n) z[n] = mkc<C>(value(wa[n]), value(wb[n]));
    sfft::fft<C, W, false>(z);
    C* xa = Xf + (j * H + q) * WhP;
    C* xb = Xf + (j * H + q + H2) * WhP;
#pragma unroll
    for (int k = 0; k < Wh; ++k) {
      const C p = z[k], m = z[(W - k) % W];
      // A = (Z[k] + conj Z[-k]) / 2 ;  B = -i (Z[k] - conj Z[-k]) / 2
      xa[k] = mkc<C>((T)0.5 * (p.x + m.x), (T)0.5 * (p.y - m.y));
      xb[k] = mkc<C>((T)0.5 * (p.y + m.y), (T)0.5 * (m.x - p.x));
    }
  };
  auto t_of = [kappa](T wv) { const T uv = soft(wv, kappa); return uv - (wv - uv); };
  auto u_of = [kappa](T wv) { return soft(wv, kappa); };

  int it = 0, stat = 0;
  for (;;) {
    // ---- A: forward column transforms, multiply by D, partial synthesis -------------------
    for (int task = tid; task < ncol_tasks; task += nt) col_forward(task / Wh, task % Wh, nullptr);
    __syncthreads();
    reduce_part();
    cl.sync();  // #1: partials and the previous iteration's norms are visible cluster-wide
    bool stop = false;
    if (it > 0) {
      double n4[5] = {0, 0, 0, 0, 0};
      for (int q = 0; q < CS; ++q)
        for (int i = 0; i < 5; ++i) n4[i] += norms[8 * q + i];
      if (n4[4] > 0.0) {
        stat = 2;
        stop = true;
      } else {
        const double num = sqrt(n4[0]), den = sqrt(n4[1]), gap = sqrt(n4[2]), dual = sqrt(n4[3]);
        if (num <= a.tol * fmax(den, 1e-12) && gap <= a.tol * fmax(fmax(den, dual), 1e-12)) {
          stat = 1;
          stop = true;
        }
      }
    }
    if (!stop && it == a.max_iters) stop = true;
    if (stop) break;
    ++it;
    // ---- reduce-scatter y over the cluster, g = (X - y) / den on my slice, all-gather g ---
    {
      const int f0 = (int)((int64_t)r * NF / CS), f1 = (int)((int64_t)(r + 1) * NF / CS);
      for (int f = f0 + tid; f < f1; f += nt) {
        C y = mkc<C>(0, 0);
        for (int q = 0; q < CS; ++q) y = cadd(y, cl.map_shared_rank(part, q)[f]);
        const T inv = (T)1 / a.den[f];
        const C g = cscale(csub(a.xh[(int64_t)b * NF + f], y), inv);
        const int u = f / Wh, v = f % Wh;
        for (int q = 0; q < CS; ++q) cl.map_shared_rank(gS, q)[u * WhP + v] = g;
      }
    }
    cl.sync();  // #2: g complete in every CTA
    // ---- B: C_k = conj(D_k) g, inverse column transforms ----------------------------------
    for (int task = tid; task < ncol_tasks; task += nt) {
      const int j = task / Wh, v = task % Wh;
      C col[H];
#pragma unroll
      for (int u = 0; u < H; ++u) col[u] = cmulc(Dg[(int64_t)j * NF + u * Wh + v], gS[u * WhP + v]);
      sfft::fft<C, H, true>(col);
#pragma unroll
      for (int u = 0; u < H; ++u) Xf[(j * H + u) * WhP + v] = col[u];
    }
    __syncthreads();
    // ---- rows: inverse row FFT -> c, update w, norms, next t, forward row FFT -------------
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    bool bad = false;
    for (int task = tid; task < nrow_tasks; task += nt) {
      const int j = task / H2, q = task % H2;
      C z[W];
      {
        const C* xa = Xf + (j * H + q) * WhP;
        const C* xb = Xf + (j * H + q + H2) * WhP;
#pragma unroll
        for (int k = 0; k < Wh; ++k) {
          C A = xa[k], Bv = xb[k];
          if (k == 0 || 2 * k == W) {
            A.y = 0;
            Bv.y = 0;
          }
          z[k] = mkc<C>(A.x - Bv.y, A.y + Bv.x);            // A + iB
          if (k > 0 && 2 * k != W) z[W - k] = mkc<C>(A.x + Bv.y, Bv.x - A.y);  // conj A + i conj B
        }
      }
      sfft::fft<C, W, true>(z);
      T* wa = wS + (j * H + q) * WP;
      T* wb = wS + (j * H + q + H2) * WP;
#pragma unroll
      for (int n = 0; n < W; ++n) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          T* wp = half ? wb : wa;
          const T c = (half ? z[n].y : z[n].x) * invP;
          const T wo = wp[n];
          const T uo = soft(wo, kappa), go = wo - uo;
          const T wn = uo + c;
          const T un = soft(wn, kappa), gn = wn - un;
          bad |= !isfinite(un);
          const float d0 = (float)(un - uo), d2 = (float)(gn - go);
          s0 = fmaf(d0, d0, s0);
          s1 = fmaf((float)un, (float)un, s1);
          s2 = fmaf(d2, d2, s2);
          s3 = fmaf((float)gn, (float)gn, s3);
          wp[n] = wn;
        }
      }
      row_forward_store(j, q, t_of);
    }
    double nv[5] = {s0, s1, s2, s3, bad ? 1.0 : 0.0};
    block_allsum<5>(nv, scratch);
    if (tid < CS) {
      double* dst = cl.map_shared_rank(norms, tid) + 8 * r;
      for (int i = 0; i < 5; ++i) dst[i] = nv[i];
    }
    __syncthreads();
  }

  // ---- outputs: U = S(w) (and t), F(U), objective -----------------------------------------
  const int64_t plane0 = ((int64_t)b * K + k0) * H * W;
  double l1 = 0.0;
  for (int task = tid; task < nrow_tasks; task += nt) {
    const int j = task / H2, q = task % H2;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int row = q + half * H2;
      const T* wp = wS + (j * H + row) * WP;
      T* uo = a.u_out + plane0 + ((int64_t)j * H + row) * W;
      T* to = a.t_out ? a.t_out + plane0 + ((int64_t)j * H + row) * W : nullptr;
      for (int n = 0; n < W; ++n) {
        const T wv = wp[n];
        const T uv = soft(wv, kappa);
        l1 += fabs((double)uv);
        uo[n] = uv;
        if (to) to[n] = uv - (wv - uv);
      }
    }
    row_forward_store(j, q, u_of);
  }
  __syncthreads();
  C* uh = a.uh_out + ((int64_t)b * K + k0) * NF;
  for (int task = tid; task < ncol_tasks; task += nt) {
    const int j = task / Wh, v = task % Wh;
    col_forward(j, v, uh + (int64_t)j * NF);
  }
  __syncthreads();
  reduce_part();
  cl.sync();
  double e = 0.0;
  {
    const int f0 = (int)((int64_t)r * NF / CS), f1 = (int)((int64_t)(r + 1) * NF / CS);
    for (int f = f0 + tid; f < f1; f += nt) {
      C y = mkc<C>(0, 0);
      for (int q = 0; q < CS; ++q) y = cadd(y, cl.map_shared_rank(part, q)[f]);
      const C res = csub(a.xh[(int64_t)b * NF + f], y);
      e += herm_weight(f % Wh, W) * ((double)res.x * res.x + (double)res.y * res.y);
    }
  }
  double ev[2] = {e, l1};
  block_allsum<2>(ev, scratch);
  if (tid == 0) {
    double* dst = cl.map_shared_rank(norms, 0) + 8 * r;
    dst[5] = ev[0];
    dst[6] = ev[1];
  }
  cl.sync();
  if (r == 0 && tid == 0) {
    double energy = 0.0, l1s = 0.0;
    for (int q = 0; q < CS; ++q) {
      energy += norms[8 * q + 5];
      l1s += norms[8 * q + 6];
    }
    const double invPd = 1.0 / ((double)H * W);
    a.obj[b] = 0.5 * invPd * energy + a.beta * l1s;
    if (a.resid) a.resid[b] = invPd * energy;
    a.iters[b] = it;
    a.status[b] = stat;
  }
}

// ---------------------------------------------------------------- dispatch --
struct FusedPlan {
  int cs = 0, threads = 0;
  size_t smem = 0;
};

template <typename T, int H, int W>
static FusedPlan plan_for(int K, int B) {
  using G = Geo<H, W>;
  FusedPlan best;
  int dev = 0, max_smem = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double best_cost = 1e300;
  for (int cs : {2, 4, 8, 16}) {
    if (cs > K) break;
    const int nk = (K + cs - 1) / cs;
    const size_t smem = Smem<T, H, W>::total(nk, cs);
    if (smem > (size_t)max_smem) continue;
    int work = nk * (G::Wh > G::H2 ? G::Wh : G::H2);
    int threads = ((work + 31) / 32) * 32;
    if (threads > 384) threads = 384;
    if (threads < 64) threads = 64;
    // clusters resident at once (1 CTA per SM for these footprints), then waves over B samples
    int per_sm = (int)(228 * 1024 / (smem + 1024));
    if (per_sm < 1) per_sm = 1;
    const int resident = (sms * per_sm) / cs;
    if (resident < 1) continue;
    const int waves = (B + resident - 1) / resident;
    const double cost = (double)waves * nk * (1.0 + 0.05 * cs);  // mild penalty for cluster sync width
    if (cost < best_cost) {
      best_cost = cost;
      best.cs = cs;
      best.threads = threads;
      best.smem = smem;
    }
  }
  return best;
}

template <typename T, int H, int W>
static int launch_fused(const FusedArgs<T>& a, cudaStream_t s) {
  FusedPlan p = plan_for<T, H, W>(a.K, a.B);
  if (!p.cs) return fail(OCSC_EARG, "fused code ADMM: no cluster shape fits shared memory");
  auto kern = k_code_fused<T, H, W>;
  OCSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  if (p.cs > 8) OCSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.B * p.cs, 1, 1);
  cfg.blockDim = dim3(p.threads, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OCSC_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  OCSC_LAUNCHED("k_code_fused");
  return OCSC_OK;
}

template <typename T, int H, int W>
static int query_fused(int K, int B) {
  return plan_for<T, H, W>(K, B).cs;
}

// the grids the fused kernel is instantiated for (BASELINE config 1 is 42 x 42)
#define OCSC_FUSED_SIZES(X) X(42, 42) X(12, 12) X(10, 10) X(16, 16) X(24, 24) X(20, 20) X(8, 8) X(12, 9)

template <typename T>
static int fused_dispatch(int H, int W, bool query, const FusedArgs<T>* a, int K, int B, cudaStream_t s) {
#define OCSC_CASE(HH, WW) \
  if (H == HH && W == WW) return query ? query_fused<T, HH, WW>(K, B) : launch_fused<T, HH, WW>(*a, s);
  OCSC_FUSED_SIZES(OCSC_CASE)
#undef OCSC_CASE
  return query ? 0 : fail(OCSC_EARG, "fused code ADMM: grid not instantiated");
}

}  // namespace ocsc

using namespace ocsc;

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
    FusedArgs<float> a{K, B, max_iters, rel_tol, beta, (float)(beta / rho), (const float2*)xh, (const float2*)Wh,
                       (const float*)den, (float*)u, (float*)t, (float2*)uh, obj, resid, iters, status};
    return fused_dispatch<float>(H, W, false, &a, K, B, s);
  }
  if (dtype == OCSC_F64) {
    FusedArgs<double> a{K, B, max_iters, rel_tol, beta, beta / rho, (const double2*)xh, (const double2*)Wh,
                        (const double*)den, (double*)u, (double*)t, (double2*)uh, obj, resid, iters, status};
    return fused_dispatch<double>(H, W, false, &a, K, B, s);
  }
  return fail(OCSC_EARG, "dtype must be 4 or 8");
}
