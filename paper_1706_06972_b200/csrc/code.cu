// Sparse-code ADMM (coding.py:45-134) for a mini-batch of B samples on one device.
//
// The reference iteration (coding.py:99-118) is
//     T = F(U - G);  Z = T + conj(D) (X - sum_k D_k T_k) / den;  z = F^-1 Z
//     U' = S_k(z + G);  G' = G + z - U'
// By linearity z + G = U + c with c_k = F^-1(conj(D_k) g),  g = (X - sum_k D_k T_k)/den,
// and G' = (U + c) - S_k(U + c).  So one iteration is
//     R2C(t) -> [residual: g per frequency, C_k = conj(D_k) g] -> C2R -> [update]
// with t = U - G kept beside U.  The update kernel also produces the four norms of
// the two-part stopping test (coding.py:108-118) per sample; a one-block
// decision kernel freezes converged samples, so every sample stops at exactly the
// iteration the reference would, without a host sync.
#include <cufft.h>

#include <deque>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "transforms.cuh"

namespace ocsc {

struct CodeWork {
  void* spec;      // (B, K, nfreq) complex: T then C (in place)
  void* cbuf;      // (B, K, P) real: c (unscaled C2R output)
  void* zsp;       // (B, K, P) real: z of the last active iteration (optional)
  double* acc;     // (B, 4)
  int32_t* flags;  // done[B], bad[B], all_done, it
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t layout(int dtype, int H, int W, int K, int B, int want_z, CodeWork* w, char* base) {
  const size_t s = dtype == OCSC_F64 ? 8 : 4;
  const size_t nf = (size_t)H * (W / 2 + 1), P = (size_t)H * W;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += align256(bytes); return p; };
  char* spec = take((size_t)B * K * nf * 2 * s);
  char* cbuf = take((size_t)B * K * P * s);
  char* zsp = want_z ? take((size_t)B * K * P * s) : nullptr;
  char* acc = take((size_t)B * 4 * sizeof(double));
  char* flags = take((size_t)(2 * B + 2) * sizeof(int32_t));
  if (w) {
    w->spec = spec; w->cbuf = cbuf; w->zsp = zsp;
    w->acc = (double*)acc; w->flags = (int32_t*)flags;
  }
  return off;
}

template <typename T>
__device__ __forceinline__ T shrink(T a, T kappa) {
  // sign(a) * max(|a| - kappa, 0) with NaN propagated (coding.py:45-48)
  return a > kappa ? a - kappa : (a < -kappa ? a + kappa : (a == a ? (T)0 : a));
}

template <typename T>
__global__ void k_den(int K, int nf, const cx<T>* __restrict__ Wh, T rho, T* __restrict__ den) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nf) return;
  T s = rho;
  for (int k = 0; k < K; ++k) s += cabs2(Wh[(int64_t)k * nf + p]);
  den[p] = s;
}

// thread per (b, p): g = (X - sum_k D_k T_k) / den, then C_k = conj(D_k) g in place of T_k
template <typename T>
__global__ void __launch_bounds__(256) k_residual(int B, int K, int nf, const cx<T>* __restrict__ Wh,
                                                  const cx<T>* __restrict__ xh, const T* __restrict__ den,
                                                  cx<T>* spec, const int32_t* __restrict__ done,
                                                  const int32_t* __restrict__ all_done) {
  if (*all_done) return;
  const int b = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nf || done[b]) return;
  cx<T>* sp = spec + (int64_t)b * K * nf + p;
  cx<T> y = mkc<cx<T>>(0, 0);
  for (int k = 0; k < K; ++k) cfma(y, Wh[(int64_t)k * nf + p], sp[(int64_t)k * nf]);
  const T inv = (T)1 / den[p];
  cx<T> g = cscale(csub(xh[(int64_t)b * nf + p], y), inv);
  for (int k = 0; k < K; ++k) sp[(int64_t)k * nf] = cmulc(Wh[(int64_t)k * nf + p], g);
}

// elementwise update of one sample's (K, P) block; norms of coding.py:108-116
template <typename T, bool WANTZ>
__global__ void __launch_bounds__(256) k_update(int64_t n, T invP, T kappa, T* __restrict__ u,
                                                T* __restrict__ t, const T* __restrict__ c,
                                                T* __restrict__ zsp, const int32_t* __restrict__ done,
                                                int32_t* bad, const int32_t* __restrict__ all_done,
                                                double* acc) {
  __shared__ double scratch[4 * 32];
  if (*all_done) return;
  const int b = blockIdx.y;
  if (done[b]) return;
  const int64_t off = (int64_t)b * n;
  double s[4] = {0, 0, 0, 0};
  bool nonfinite = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T uo = u[off + i], to = t[off + i], cc = c[off + i] * invP;
    const T a = uo + cc;
    const T un = shrink(a, kappa);
    const T gn = a - un;
    const T go = uo - to;
    nonfinite |= !isfinite(un);
    const double d0 = (double)un - uo, d2 = (double)gn - go;
    s[0] += d0 * d0;
    s[1] += (double)un * un;
    s[2] += d2 * d2;
    s[3] += (double)gn * gn;
    u[off + i] = un;
    t[off + i] = un - gn;
    if (WANTZ) zsp[off + i] = to + cc;
  }
  if (__syncthreads_or(nonfinite) && threadIdx.x == 0) atomicOr(bad + b, 1);
  block_sum<4>(s, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) atomicAdd(acc + 4 * b + j, s[j]);
  }
}

// one block: per-sample stopping decision (coding.py:105-118)
__global__ void k_decide(int B, double tol, double* acc, int32_t* flags, int32_t* iters, int32_t* status) {
  decide_block(B, tol, acc, flags, iters, status);
}

// objective: spectral residual energy (Parseval, half-spectrum weights) per sample
template <typename T>
__global__ void __launch_bounds__(256) k_obj_spec(int H, int W, int K, int nf, const cx<T>* __restrict__ xh,
                                                  const cx<T>* __restrict__ Wh, const cx<T>* __restrict__ uh,
                                                  double scale, double* obj, double* resid) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const int Wh_ = W / 2 + 1;
  double e[1] = {0.0};
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nf; p += gridDim.x * blockDim.x) {
    cx<T> y = mkc<cx<T>>(0, 0);
    const cx<T>* ub = uh + (int64_t)b * K * nf + p;
    for (int k = 0; k < K; ++k) cfma(y, Wh[(int64_t)k * nf + p], ub[(int64_t)k * nf]);
    const cx<T> r = csub(xh[(int64_t)b * nf + p], y);
    e[0] += herm_weight(p % Wh_, W) * ((double)r.x * r.x + (double)r.y * r.y);
  }
  block_sum<1>(e, scratch);
  if (threadIdx.x == 0) {
    atomicAdd(obj + b, e[0] * scale);
    if (resid) atomicAdd(resid + b, e[0] * 2.0 * scale);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_obj_l1(int64_t n, const T* __restrict__ u, double beta, double* obj) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  double e[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    e[0] += fabs((double)u[(int64_t)b * n + i]);
  block_sum<1>(e, scratch);
  if (threadIdx.x == 0) atomicAdd(obj + b, e[0] * beta);
}

template <typename T>
__global__ void k_synth(int K, int nf, int B, const cx<T>* __restrict__ Wh, const cx<T>* __restrict__ zh, cx<T>* out) {
  const int b = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nf) return;
  cx<T> y = mkc<cx<T>>(0, 0);
  for (int k = 0; k < K; ++k) cfma(y, Wh[(int64_t)k * nf + p], zh[((int64_t)b * K + k) * nf + p]);
  out[(int64_t)b * nf + p] = y;
}

template <typename T>
__global__ void k_soft(int64_t n, const T* in, T kappa, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T x = in[i];
    // np.sign(x) * np.maximum(np.abs(x) - kappa, 0.0)
    T mag = fabs(x) - kappa;
    mag = mag > (T)0 ? mag : (mag == mag ? (T)0 : mag);
    T sg = x > (T)0 ? (T)1 : (x < (T)0 ? (T)-1 : (x == x ? (T)0 : x));
    out[i] = sg * mag;
  }
}

// coding.py:51-64 on reference rows, same operation order
template <typename T>
__global__ void k_solve_rows(int nrows, int K, const cx<T>* d, const cx<T>* x, const cx<T>* t, T rho, cx<T>* out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nrows) return;
  const cx<T>* dp = d + (int64_t)p * K;
  const cx<T>* tp = t + (int64_t)p * K;
  cx<T>* op = out + (int64_t)p * K;
  const cx<T> xp = x[p];
  cx<T> s = mkc<cx<T>>(0, 0);
  T den = 0;
  for (int k = 0; k < K; ++k) {
    cx<T> rhs = cadd(cmulc(dp[k], xp), cscale(tp[k], rho));
    s = cadd(s, cmul(dp[k], rhs));
    den += cabs2(dp[k]);
  }
  den += rho;
  const cx<T> q = cscale(s, (T)1 / den);
  for (int k = 0; k < K; ++k) {
    cx<T> rhs = cadd(cmulc(dp[k], xp), cscale(tp[k], rho));
    cx<T> v = csub(rhs, cmulc(dp[k], q));
    op[k] = cscale(v, (T)1 / rho);
  }
}

// pinned flags for the lagged convergence poll
static int32_t* pinned_flags() {
  static int32_t* p = nullptr;
  if (!p) {
    if (cudaHostAlloc((void**)&p, 64 * sizeof(int32_t), cudaHostAllocPortable) != cudaSuccess) p = nullptr;
  }
  return p;
}

// One ADMM iteration of the batch (R2C, residual, C2R, update, decide) enqueued on stream s.
template <typename T>
static int admm_iteration(int dtype, int H, int W, int K, int B, const CodeWork& w, const void* xh, const void* Wh,
                          const void* den, T invP, T kappa, double rel_tol, void* u, void* t, bool want_z,
                          int32_t* iters, int32_t* status, cudaStream_t s) {
  const int nf = H * (W / 2 + 1);
  const int64_t n = (int64_t)K * H * W;
  int32_t* flags = w.flags;
  const dim3 rgrid(ceil_div(nf, 256), B);
  int ux = ceil_div(n, 256 * 4);
  if (ux > 1024) ux = 1024;
  const dim3 ugrid(ux, B);
  int rc = exec_r2c(dtype, H, W, B * K, t, w.spec, s);
  if (rc) return rc;
  k_residual<T><<<rgrid, 256, 0, s>>>(B, K, nf, (const cx<T>*)Wh, (const cx<T>*)xh, (const T*)den,
                                       (cx<T>*)w.spec, flags, flags + 2 * B);
  rc = exec_c2r(dtype, H, W, B * K, w.spec, w.cbuf, s);
  if (rc) return rc;
  if (want_z)
    k_update<T, true><<<ugrid, 256, 0, s>>>(n, invP, kappa, (T*)u, (T*)t, (const T*)w.cbuf, (T*)w.zsp, flags,
                                             flags + B, flags + 2 * B, w.acc);
  else
    k_update<T, false><<<ugrid, 256, 0, s>>>(n, invP, kappa, (T*)u, (T*)t, (const T*)w.cbuf, nullptr, flags,
                                              flags + B, flags + 2 * B, w.acc);
  k_decide<<<1, 256, 0, s>>>(B, rel_tol, w.acc, flags, iters, status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OCSC_OK : cuda_fail(e, "code ADMM launch");
}

// Chunks of iterations as CUDA graphs: the cuFFT path of a small problem (the reference's B = 1
// OnlineTrainer.step, evaluation) is launch-bound at ~5 launches per iteration; one graph launch
// per poll interval replaces them.  Graphs are captured on a private stream (the caller's may be
// the legacy default stream, which cannot be captured), cached per argument set (the trainer's
// buffers are stable across calls), and replayed on the caller's stream.  OCSC_NO_GRAPH=1 keeps
// plain stream launches.
namespace {
using GraphKey = std::tuple<int, int, int, int, int, int, std::vector<const void*>, double, double, double, int>;
std::map<GraphKey, cudaGraphExec_t>& graph_cache() {
  static std::map<GraphKey, cudaGraphExec_t> m;
  return m;
}
std::deque<GraphKey>& graph_order() {  // insertion order: the cache keeps the newest kMaxGraphs
  static std::deque<GraphKey> q;
  return q;
}
std::map<GraphKey, int>& graph_seen() {  // capture on the second call with an argument set only
  static std::map<GraphKey, int> m;
  return m;
}
constexpr size_t kMaxGraphs = 64;
std::mutex& graph_mu() {
  static std::mutex m;
  return m;
}
cudaStream_t capture_stream(int dev) {
  static std::map<int, cudaStream_t> m;
  auto it = m.find(dev);
  if (it != m.end()) return it->second;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  m[dev] = st;
  return st;
}
}  // namespace

template <typename T>
static int code_admm_impl(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh, const void* den,
                          double beta, double rho, int max_iters, double rel_tol, void* u, void* t, void* zh,
                          void* work, int32_t* iters, int32_t* status, int poll, cudaStream_t s) {
  CodeWork w;
  layout(dtype, H, W, K, B, zh != nullptr, &w, (char*)work);
  int32_t* flags = w.flags;
  OCSC_CUDA(cudaMemsetAsync(w.acc, 0, sizeof(double) * 4 * B, s));
  OCSC_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * (2 * B + 2), s));
  OCSC_CUDA(cudaMemsetAsync(iters, 0, sizeof(int32_t) * B, s));
  OCSC_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * B, s));
  if (B == 0 || max_iters <= 0) return OCSC_OK;

  // make sure plans exist before the loop (plan creation allocates)
  cufftHandle ph;
  int rc = get_plan(0, dtype, H, W, B * K, &ph);
  if (rc) return rc;
  rc = get_plan(1, dtype, H, W, B * K, &ph);
  if (rc) return rc;

  const T invP = (T)(1.0 / ((double)H * W));
  const T kappa = (T)(beta / rho);
  const bool want_z = zh != nullptr;
  const int step = poll > 0 ? poll : 16;  // iterations per graph / per convergence poll
  static const bool no_graph = getenv("OCSC_NO_GRAPH") != nullptr;
  int dev = 0;
  OCSC_CUDA(cudaGetDevice(&dev));

  // the graph of n iterations for these arguments (captured on first use)
  auto chunk_graph = [&](int n, cudaGraphExec_t* out) -> int {
    GraphKey key{dev, dtype, H, W, K, B, {xh, Wh, den, u, t, zh, work, iters, status}, beta, rho, rel_tol, n};
    std::lock_guard<std::mutex> lk(graph_mu());
    auto it = graph_cache().find(key);
    if (it != graph_cache().end()) {
      *out = it->second;
      return OCSC_OK;
    }
    *out = nullptr;
    if (graph_seen()[key]++ == 0) return OCSC_OK;  // a one-off argument set runs as plain launches
    if (graph_seen().size() > 4 * kMaxGraphs) graph_seen().clear();
    cudaStream_t cap = capture_stream(dev);
    if (!cap) return fail(OCSC_ECUDA, "code_admm: capture stream");
    OCSC_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    int rc2 = OCSC_OK;
    for (int i = 0; i < n && rc2 == OCSC_OK; ++i)
      rc2 = admm_iteration<T>(dtype, H, W, K, B, w, xh, Wh, den, invP, kappa, rel_tol, u, t, want_z, iters, status,
                              cap);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap, &g);
    if (rc2) {
      if (g) cudaGraphDestroy(g);
      return rc2;
    }
    if (e != cudaSuccess) return cuda_fail(e, "code_admm: end capture");
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "code_admm: instantiate");
    graph_cache()[key] = ex;
    graph_order().push_back(key);
    if (graph_order().size() > kMaxGraphs) {
      auto old = graph_cache().find(graph_order().front());
      if (old != graph_cache().end()) {
        cudaGraphExecDestroy(old->second);
        graph_cache().erase(old);
      }
      graph_order().pop_front();
    }
    *out = ex;
    return OCSC_OK;
  };

  int32_t* host = poll > 0 ? pinned_flags() : nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (host) {
    OCSC_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    OCSC_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  }
  int chunk = 0;
  bool stop = false;
  for (int it = 0; it < max_iters && !stop && rc == OCSC_OK;) {
    const int n = std::min(step, max_iters - it);
    cudaGraphExec_t ex = nullptr;
    if (!no_graph) rc = chunk_graph(n, &ex);
    if (rc == OCSC_OK && ex) {
      cudaError_t e = cudaGraphLaunch(ex, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "code_admm: graph launch");
    } else {
      for (int i = 0; i < n && rc == OCSC_OK; ++i)
        rc = admm_iteration<T>(dtype, H, W, K, B, w, xh, Wh, den, invP, kappa, rel_tol, u, t, want_z, iters, status,
                               s);
    }
    count_launches(3 * n);
    it += n;
    if (host && it < max_iters && rc == OCSC_OK) {
      const int slot = chunk & 1;
      cudaMemcpyAsync(host + slot, flags + 2 * B, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaEventRecord(ev[slot], s);
      if (chunk > 0) {  // look one chunk behind: the device still has work queued
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
  if (zh) {
    rc = exec_r2c(dtype, H, W, B * K, w.zsp, zh, s);
    if (rc) return rc;
  }
  return OCSC_OK;
}

}  // namespace ocsc

using namespace ocsc;

extern "C" size_t ocsc_code_workspace_bytes(int dtype, int H, int W, int K, int B, int want_z) {
  return layout(dtype, H, W, K, B, want_z, nullptr, nullptr);
}

extern "C" int ocsc_code_admm(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh,
                              const void* den, double beta, double rho, int max_iters, double rel_tol, void* u,
                              void* t, void* zh, void* work, int32_t* iters, int32_t* status, int poll,
                              void* stream) {
  if (H <= 0 || W <= 0 || K <= 0 || B < 0) return fail(OCSC_ESHAPE, "code_admm: bad extents");
  if (!(rho > 0)) return fail(OCSC_EARG, "code_admm: rho must be positive");
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    return code_admm_impl<float>(dtype, H, W, K, B, xh, Wh, den, beta, rho, max_iters, rel_tol, u, t, zh, work,
                                 iters, status, poll, s);
  if (dtype == OCSC_F64)
    return code_admm_impl<double>(dtype, H, W, K, B, xh, Wh, den, beta, rho, max_iters, rel_tol, u, t, zh, work,
                                  iters, status, poll, s);
  return fail(OCSC_EARG, "dtype must be 4 or 8");
}

extern "C" int ocsc_code_den(int dtype, int K, int nfreq, const void* Wh, double rho, void* den, void* stream) {
  if (nfreq <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_den<float><<<ceil_div(nfreq, 256), 256, 0, s>>>(K, nfreq, (const float2*)Wh, (float)rho, (float*)den);
  else if (dtype == OCSC_F64)
    k_den<double><<<ceil_div(nfreq, 256), 256, 0, s>>>(K, nfreq, (const double2*)Wh, rho, (double*)den);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_den");
  return OCSC_OK;
}

extern "C" int ocsc_code_objective(int dtype, int H, int W, int K, int B, const void* xh, const void* Wh,
                                   const void* u, double beta, void* uh, double* obj, double* resid,
                                   void* stream) {
  if (H <= 0 || W <= 0 || K <= 0 || B < 0) return fail(OCSC_ESHAPE, "code_objective: bad extents");
  if (B == 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  OCSC_CUDA(cudaMemsetAsync(obj, 0, sizeof(double) * B, s));
  if (resid) OCSC_CUDA(cudaMemsetAsync(resid, 0, sizeof(double) * B, s));
  int rc = exec_r2c(dtype, H, W, B * K, u, uh, s);
  if (rc) return rc;
  const int nf = H * (W / 2 + 1);
  const int64_t n = (int64_t)K * H * W;
  const double scale = 0.5 / ((double)H * W);
  dim3 g1(ceil_div(nf, 256) > 64 ? 64 : ceil_div(nf, 256), B);
  int gx = ceil_div(n, 1024);
  dim3 g2(gx > 256 ? 256 : gx, B);
  if (dtype == OCSC_F32) {
    k_obj_spec<float><<<g1, 256, 0, s>>>(H, W, K, nf, (const float2*)xh, (const float2*)Wh, (const float2*)uh, scale, obj, resid);
    k_obj_l1<float><<<g2, 256, 0, s>>>(n, (const float*)u, beta, obj);
  } else if (dtype == OCSC_F64) {
    k_obj_spec<double><<<g1, 256, 0, s>>>(H, W, K, nf, (const double2*)xh, (const double2*)Wh, (const double2*)uh, scale, obj, resid);
    k_obj_l1<double><<<g2, 256, 0, s>>>(n, (const double*)u, beta, obj);
  } else {
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  }
  count_launches(1);  // two kernels above
  OCSC_LAUNCHED("k_obj");
  return OCSC_OK;
}

extern "C" int ocsc_soft_threshold(int dtype, int64_t n, const void* in, double kappa, void* out, void* stream) {
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_soft<float><<<grid_for(n, 256), 256, 0, s>>>(n, (const float*)in, (float)kappa, (float*)out);
  else if (dtype == OCSC_F64)
    k_soft<double><<<grid_for(n, 256), 256, 0, s>>>(n, (const double*)in, kappa, (double*)out);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_soft");
  return OCSC_OK;
}

extern "C" int ocsc_solve_code_rows(int dtype, int nrows, int K, const void* d, const void* x, const void* t,
                                    double rho, void* out, void* stream) {
  if (nrows <= 0 || K <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_solve_rows<float><<<ceil_div(nrows, 128), 128, 0, s>>>(nrows, K, (const float2*)d, (const float2*)x,
                                                             (const float2*)t, (float)rho, (float2*)out);
  else if (dtype == OCSC_F64)
    k_solve_rows<double><<<ceil_div(nrows, 128), 128, 0, s>>>(nrows, K, (const double2*)d, (const double2*)x,
                                                              (const double2*)t, rho, (double2*)out);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_solve_rows");
  return OCSC_OK;
}

extern "C" int ocsc_synthesize(int dtype, int K, int nfreq, int B, const void* Wh, const void* zh, void* out,
                               void* stream) {
  if (nfreq <= 0 || B <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  dim3 g(ceil_div(nfreq, 256), B);
  if (dtype == OCSC_F32)
    k_synth<float><<<g, 256, 0, s>>>(K, nfreq, B, (const float2*)Wh, (const float2*)zh, (float2*)out);
  else if (dtype == OCSC_F64)
    k_synth<double><<<g, 256, 0, s>>>(K, nfreq, B, (const double2*)Wh, (const double2*)zh, (double2*)out);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_synth");
  return OCSC_OK;
}
