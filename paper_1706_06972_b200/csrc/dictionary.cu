// Dictionary projection (dictionary.py:145-154, 199-207) as one fused kernel per filter.
//
// The reference projects with a full inverse FFT, crops the M0 x M1 support,
// scales into the unit ball, pads and runs a full forward FFT.  Only M = M0*M1
// spatial taps survive the crop, so both transforms are pruned separable DFTs on
// the half spectrum (H x Wh):
//   Y[m0][v]  = sum_u X[u][v] e^{+2 pi i u m0 / H}                 (M0*Wh outputs)
//   a[m0][m1] = (1/P) sum_v w_v Re(Y[m0][v] e^{+2 pi i v m1 / W})  (w_v = 1 at v = 0, W/2; else 2)
//   a        /= max(||a||, 1)
//   Q[m0][v]  = sum_m1 a[m0][m1] e^{-2 pi i v m1 / W}
//   V[u][v]   = sum_m0 Q[m0][v] e^{-2 pi i u m0 / H}
// and the dual step Theta += D - V is fused into the last stage.
#include "common.cuh"
#include "transforms.cuh"

namespace ocsc {

// PROJECT, CROP_ONLY, SUPPORT_RFFT act on the whole half plane.  The frequency-sharded
// trainer (sharded.py) owns rows [u0, u1) of it: CROP_PARTIAL sums the
// pruned inverse over those rows only (double partial support, all-reduced across ranks),
// SUPPORT_RFFT evaluates V on those rows only and, with D and Theta given, takes the dual
// step there.  Slice arrays are (K, u1-u0, Wh).
enum ProjMode { PROJECT = 0, CROP_ONLY = 1, SUPPORT_RFFT = 2, CROP_PARTIAL = 3 };

template <typename T>
__global__ void __launch_bounds__(256) k_project(int mode, int staged, int H, int W, int M0, int M1, int u0, int u1,
                                                 const cx<T>* __restrict__ Dh, cx<T>* Th, cx<T>* Vh, T* alpha,
                                                 double* apart) {
  using C = cx<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Wh = W / 2 + 1, nf = (u1 - u0) * Wh, M = M0 * M1;
  C* twH = reinterpret_cast<C*>(smem_raw);  // e^{+2 pi i n / H}
  C* twW = twH + H;                         // e^{+2 pi i n / W}
  C* Y = twW + W;                           // [M0][Wh], reused as Q
  T* al = reinterpret_cast<T*>(Y + (int64_t)M0 * Wh);
  C* Xs = reinterpret_cast<C*>(smem_raw) + H + W + (int64_t)M0 * Wh + (M + 1) / 2 + 1;  // [nf] D + Theta
  __shared__ double scratch[32];
  __shared__ double norm_s;
  const int k = blockIdx.x;
  const C* Dk = Dh ? Dh + (int64_t)k * nf : nullptr;
  C* Tk = Th ? Th + (int64_t)k * nf : nullptr;

  for (int n = threadIdx.x; n < H; n += blockDim.x) {
    double sn, cn;
    sincospi(2.0 * n / H, &sn, &cn);
    twH[n] = mkc<C>((T)cn, (T)sn);
  }
  for (int n = threadIdx.x; n < W; n += blockDim.x) {
    double sn, cn;
    sincospi(2.0 * n / W, &sn, &cn);
    twW[n] = mkc<C>((T)cn, (T)sn);
  }
  __syncthreads();

  if (mode != SUPPORT_RFFT) {
    // stage D + Theta (coalesced, every load of the plane in flight at once) when it fits
    if (staged) {
      for (int o = threadIdx.x; o < nf; o += blockDim.x) Xs[o] = Tk ? cadd(Dk[o], Tk[o]) : Dk[o];
      __syncthreads();
    }
    // pruned inverse along u
    for (int o = threadIdx.x; o < M0 * Wh; o += blockDim.x) {
      const int m0 = o / Wh, v = o % Wh;
      C acc = mkc<C>(0, 0);
      int idx = (int)(((int64_t)u0 * m0) % H);
      for (int u = u0; u < u1; ++u) {
        const int64_t q = (int64_t)(u - u0) * Wh + v;
        const C x = staged ? Xs[q] : (Tk ? cadd(Dk[q], Tk[q]) : Dk[q]);
        cfma(acc, x, twH[idx]);
        idx += m0;
        if (idx >= H) idx -= H;
      }
      Y[o] = acc;
    }
    __syncthreads();
    // pruned inverse along v onto the support (real part, Hermitian weights)
    const double invP = 1.0 / ((double)H * W);
    double ss[1] = {0.0};
    for (int o = threadIdx.x; o < M; o += blockDim.x) {
      const int m0 = o / M1, m1 = o % M1;
      double acc = 0.0;
      int idx = 0;
      for (int v = 0; v < Wh; ++v) {
        const C y = Y[m0 * Wh + v], w = twW[idx];
        acc += herm_weight(v, W) * ((double)y.x * w.x - (double)y.y * w.y);
        idx += m1;
        if (idx >= W) idx -= W;
      }
      if (mode == CROP_PARTIAL) {
        apart[(int64_t)k * M + o] = acc * invP;
        continue;
      }
      const T a = (T)(acc * invP);
      al[o] = a;
      ss[0] += (double)a * a;
    }
    if (mode == CROP_PARTIAL) return;
    if (mode == PROJECT) {
      block_sum<1>(ss, scratch);
      if (threadIdx.x == 0) norm_s = 1.0 / fmax(sqrt(ss[0]), 1.0);
      __syncthreads();
      const T sc = (T)norm_s;
      for (int o = threadIdx.x; o < M; o += blockDim.x) al[o] *= sc;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < M; o += blockDim.x) alpha[(int64_t)k * M + o] = al[o];
    if (mode == CROP_ONLY) return;
  } else {
    for (int o = threadIdx.x; o < M; o += blockDim.x) al[o] = alpha[(int64_t)k * M + o];
    __syncthreads();
  }
  // pruned forward along v: Q[m0][v] (reuses Y)
  for (int o = threadIdx.x; o < M0 * Wh; o += blockDim.x) {
    const int m0 = o / Wh, v = o % Wh;
    C acc = mkc<C>(0, 0);
    int idx = 0;
    for (int m1 = 0; m1 < M1; ++m1) {
      const C w = twW[idx];
      const T a = al[m0 * M1 + m1];
      acc.x += a * w.x;
      acc.y -= a * w.y;
      idx += v;
      if (idx >= W) idx -= W;
    }
    Y[o] = acc;
  }
  __syncthreads();
  // pruned forward along u over rows [u0, u1), fused dual step
  C* Vk = Vh + (int64_t)k * nf;
  for (int o = threadIdx.x; o < nf; o += blockDim.x) {
    const int u = o / Wh + u0, v = o % Wh;
    C acc = mkc<C>(0, 0);
    int idx = 0;
    for (int m0 = 0; m0 < M0; ++m0) {
      cfmac(acc, twH[idx], Y[m0 * Wh + v]);  // conj(tw) * Q
      idx += u;
      if (idx >= H) idx -= H;
    }
    Vk[o] = acc;
    if (Tk && Dk) Tk[o] = cadd(Tk[o], csub(Dk[o], acc));
  }
}

// alpha_k = (T) apart_k / max(||(T) apart_k||, 1): the projection's normalisation (dictionary.py:150-152)
// applied to the all-reduced partial supports of the sharded trainer
template <typename T>
__global__ void k_normalize_support(int M, const double* __restrict__ apart, T* __restrict__ alpha) {
  __shared__ double scratch[32];
  __shared__ double sc_s;
  const int k = blockIdx.x;
  double ss[1] = {0.0};
  for (int o = threadIdx.x; o < M; o += blockDim.x) {
    const T a = (T)apart[(int64_t)k * M + o];
    ss[0] += (double)a * a;
  }
  block_sum<1>(ss, scratch);
  if (threadIdx.x == 0) sc_s = 1.0 / fmax(sqrt(ss[0]), 1.0);
  __syncthreads();
  const T sc = (T)sc_s;
  for (int o = threadIdx.x; o < M; o += blockDim.x) alpha[(int64_t)k * M + o] = (T)apart[(int64_t)k * M + o] * sc;
}

// reference columns: padded (P, K) <- crop/normalise of spatial (P, K)
template <typename T>
__global__ void k_crop_normalize_cols(int H, int W, int M0, int M1, int K, const T* spatial, T* padded) {
  __shared__ double scratch[32];
  __shared__ double sc_s;
  const int k = blockIdx.x;
  const int M = M0 * M1;
  double ss[1] = {0.0};
  for (int o = threadIdx.x; o < M; o += blockDim.x) {
    const int m0 = o / M1, m1 = o % M1;
    const double a = spatial[((int64_t)m0 * W + m1) * K + k];
    ss[0] += a * a;
  }
  block_sum<1>(ss, scratch);
  if (threadIdx.x == 0) sc_s = 1.0 / fmax(sqrt(ss[0]), 1.0);
  __syncthreads();
  const int64_t P = (int64_t)H * W;
  for (int64_t q = threadIdx.x; q < P; q += blockDim.x) {
    const int u = (int)(q / W), v = (int)(q % W);
    padded[q * K + k] = (u < M0 && v < M1) ? (T)(spatial[q * K + k] * sc_s) : (T)0;
  }
}

template <typename T>
__global__ void k_norms2(int64_t n, const T* a, const T* b, double* out) {
  __shared__ double scratch[64];
  double s[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[i], y = b ? (double)b[i] : 0.0;
    s[0] += (x - y) * (x - y);
    s[1] += x * x;
  }
  block_sum<2>(s, scratch);
  if (threadIdx.x == 0) {
    atomicAdd(out, s[0]);
    atomicAdd(out + 1, s[1]);
  }
}

template <typename T>
static int launch_project(int mode, int H, int W, int M0, int M1, int K, int u0, int u1, const void* Dh, void* Th,
                          void* Vh, void* alpha, double* apart, cudaStream_t s) {
  const int Wh = W / 2 + 1;
  const int M = M0 * M1;
  const size_t base = sizeof(cx<T>) * ((size_t)H + W + (size_t)M0 * Wh + (M + 1) / 2 + 1);
  const size_t with_plane = base + sizeof(cx<T>) * (size_t)(u1 - u0) * Wh;  // + staged D + Theta
  const int staged = with_plane <= 100 * 1024;  // small grids (config 1: 7 KB); large ones read L2
  const size_t smem = staged ? with_plane : base;
  if (smem > 227 * 1024) return fail(OCSC_EARG, "dict_project: grid too large for the fused projection");
  OCSC_CUDA(cudaFuncSetAttribute(k_project<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_project<T><<<K, 256, smem, s>>>(mode, staged, H, W, M0, M1, u0, u1, (const cx<T>*)Dh, (cx<T>*)Th, (cx<T>*)Vh,
                                    (T*)alpha, apart);
  OCSC_LAUNCHED("k_project");
  return OCSC_OK;
}

static int project_dispatch(int dtype, int mode, int H, int W, int M0, int M1, int K, const void* Dh, void* Th,
                            void* Vh, void* alpha, void* stream, int u0 = 0, int u1 = -1, double* apart = nullptr) {
  if (u1 < 0) u1 = H;
  if (H <= 0 || W <= 0 || M0 <= 0 || M1 <= 0 || M0 > H || M1 > W || K < 0 || u0 < 0 || u1 > H || u0 > u1)
    return fail(OCSC_ESHAPE, "projection: bad extents");
  if (K == 0 || u0 == u1) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32) return launch_project<float>(mode, H, W, M0, M1, K, u0, u1, Dh, Th, Vh, alpha, apart, s);
  if (dtype == OCSC_F64) return launch_project<double>(mode, H, W, M0, M1, K, u0, u1, Dh, Th, Vh, alpha, apart, s);
  return fail(OCSC_EARG, "dtype must be 4 or 8");
}

}  // namespace ocsc

using namespace ocsc;

extern "C" int ocsc_dict_project(int dtype, int H, int W, int M0, int M1, int K, const void* Dh, void* Th,
                                 void* Vh, void* alpha, void* stream) {
  return project_dispatch(dtype, PROJECT, H, W, M0, M1, K, Dh, Th, Vh, alpha, stream);
}

extern "C" int ocsc_crop_irfft_rows(int dtype, int H, int W, int M0, int M1, int K, int u0, int u1,
                                    const void* Xh, const void* Th, double* apart, void* stream) {
  if (u0 == u1) {  // an empty slice contributes zero to the all-reduce
    if (K > 0 && apart) OCSC_CUDA(cudaMemsetAsync(apart, 0, sizeof(double) * K * M0 * M1, as_stream(stream)));
    return OCSC_OK;
  }
  return project_dispatch(dtype, CROP_PARTIAL, H, W, M0, M1, K, Xh, (void*)Th, nullptr, nullptr, stream, u0, u1,
                          apart);
}

extern "C" int ocsc_support_rfft_rows(int dtype, int H, int W, int M0, int M1, int K, int u0, int u1,
                                      const void* alpha, void* Vh, const void* Dh, void* Th, void* stream) {
  if ((Dh == nullptr) != (Th == nullptr)) return fail(OCSC_EARG, "support_rfft_rows: D and Theta go together");
  return project_dispatch(dtype, SUPPORT_RFFT, H, W, M0, M1, K, Dh, Th, Vh, (void*)alpha, stream, u0, u1);
}

extern "C" int ocsc_normalize_support(int dtype, int M, int K, const double* apart, void* alpha, void* stream) {
  if (K <= 0 || M <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_normalize_support<float><<<K, 256, 0, s>>>(M, apart, (float*)alpha);
  else if (dtype == OCSC_F64)
    k_normalize_support<double><<<K, 256, 0, s>>>(M, apart, (double*)alpha);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_normalize_support");
  return OCSC_OK;
}

extern "C" int ocsc_crop_irfft(int dtype, int H, int W, int M0, int M1, int K, const void* Xh, void* alpha,
                               void* stream) {
  return project_dispatch(dtype, CROP_ONLY, H, W, M0, M1, K, Xh, nullptr, nullptr, alpha, stream);
}

extern "C" int ocsc_support_rfft(int dtype, int H, int W, int M0, int M1, int K, const void* alpha, void* Vh,
                                 void* stream) {
  return project_dispatch(dtype, SUPPORT_RFFT, H, W, M0, M1, K, nullptr, nullptr, Vh, (void*)alpha, stream);
}

extern "C" int ocsc_crop_normalize_cols(int dtype, int H, int W, int M0, int M1, int K, const void* spatial,
                                        void* padded, void* stream) {
  if (K <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_crop_normalize_cols<float><<<K, 256, 0, s>>>(H, W, M0, M1, K, (const float*)spatial, (float*)padded);
  else if (dtype == OCSC_F64)
    k_crop_normalize_cols<double><<<K, 256, 0, s>>>(H, W, M0, M1, K, (const double*)spatial, (double*)padded);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_crop_normalize_cols");
  return OCSC_OK;
}

extern "C" int ocsc_norms2(int dtype, int64_t n, const void* a, const void* b, double* out, void* stream) {
  if (n <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  int g = grid_for(n, 256);
  if (g > 512) g = 512;
  if (dtype == OCSC_F32)
    k_norms2<float><<<g, 256, 0, s>>>(n, (const float*)a, (const float*)b, out);
  else if (dtype == OCSC_F64)
    k_norms2<double><<<g, 256, 0, s>>>(n, (const double*)a, (const double*)b, out);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_norms2");
  return OCSC_OK;
}

namespace ocsc {
// per filter: out[2k] += sum_p w_p |D_k[p] - V_k[p]|^2, out[2k+1] += sum_p w_p |D_k[p]|^2 over the
// half spectrum with Hermitian weights (= full-spectrum squared norms, dictionary.py:210-214)
template <typename T>
__global__ void k_dict_gaps(int H, int W, const cx<T>* __restrict__ Dh, const cx<T>* __restrict__ Vh, double* out) {
  __shared__ double scratch[64];
  const int k = blockIdx.x;
  const int Wh = W / 2 + 1, nf = H * Wh;
  double s[2] = {0.0, 0.0};
  for (int p = threadIdx.x; p < nf; p += blockDim.x) {
    const cx<T> d = Dh[(int64_t)k * nf + p], v = Vh[(int64_t)k * nf + p];
    const double w = herm_weight(p % Wh, W);
    const double ex = (double)d.x - v.x, ey = (double)d.y - v.y;
    s[0] += w * (ex * ex + ey * ey);
    s[1] += w * ((double)d.x * d.x + (double)d.y * d.y);
  }
  block_sum<2>(s, scratch);
  if (threadIdx.x == 0) {
    out[2 * k] = s[0];
    out[2 * k + 1] = s[1];
  }
}
}  // namespace ocsc

extern "C" int ocsc_dict_gaps(int dtype, int H, int W, int K, const void* Dh, const void* Vh, double* out,
                              void* stream) {
  if (K <= 0) return OCSC_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == OCSC_F32)
    k_dict_gaps<float><<<K, 256, 0, s>>>(H, W, (const float2*)Dh, (const float2*)Vh, out);
  else if (dtype == OCSC_F64)
    k_dict_gaps<double><<<K, 256, 0, s>>>(H, W, (const double2*)Dh, (const double2*)Vh, out);
  else
    return fail(OCSC_EARG, "dtype must be 4 or 8");
  OCSC_LAUNCHED("k_dict_gaps");
  return OCSC_OK;
}
