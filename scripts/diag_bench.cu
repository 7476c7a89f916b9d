// Microbenchmark of the blocked Cholesky's diagonal-tile factor (dev aid): one warp per SM
// factors a 32 x 32 HPD tile REPS times; clock64 per call.  Variants isolate the phases.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//   -I paper_1706_06972_b200/csrc scripts/diag_bench.cu paper_1706_06972_b200/csrc/errors.cu -o scripts/diag_bench
#include <cstdio>
#include <vector>
#include "../paper_1706_06972_b200/csrc/cholesky.cu"

using namespace ocsc;

// MODE 0: the product routine; 1: no trailing update; 2: no global load/store; 3: steps only
template <int MODE, int GRP = 8>
__device__ __noinline__ void diag_var(float2* tile, int K, uint32_t sD, float* dinv, int lane, int32_t* info) {
  using C = float2;
  using T = float;
  constexpr int LD = CT + 1;
  constexpr uint32_t SZ = sizeof(C);
  if (MODE == 0 || MODE == 1) {
    const C* row = tile + (int64_t)lane * K;
#pragma unroll 8
    for (int j = 0; j < CT; ++j) sts_c(sD + (uint32_t)(lane * LD + j) * SZ, j <= lane ? row[j] : mkc<C>(0, 0));
  }
  __syncwarp();
#pragma unroll 1
  for (int j = 0; j < CT; ++j) {
    T d = lds_c<C>(sD + (uint32_t)(j * LD + j) * SZ).x;
    if (!(d > (T)0)) d = (T)NAN;
    const T y = rsqrtf(d);
    const T inv = y * ((T)1.5 - (T)0.5 * d * y * y);
    const T ljj = d * inv;
    const uint32_t own = sD + (uint32_t)(lane * LD) * SZ;
    const C aij = lds_c<C>(own + j * SZ);
    const C lij = lane > j ? cscale(aij, inv) : mkc<C>(0, 0);
    sts_c_if(lane >= j, own + j * SZ, lane == j ? mkc<C>(ljj, (T)0) : lij);
    if (lane == 0) dinv[j] = inv;
    __syncwarp();
    if (MODE != 1 && MODE != 3) {
#pragma unroll 1
      for (int k0 = j + 1; k0 < CT; k0 += GRP) {
        C lk[GRP], t[GRP];
#pragma unroll
        for (int u = 0; u < GRP; ++u) lk[u] = lds_c<C>(sD + (uint32_t)(min(k0 + u, CT - 1) * LD + j) * SZ);
#pragma unroll
        for (int u = 0; u < GRP; ++u) t[u] = lds_c<C>(own + min(k0 + u, LD - 1) * SZ);
#pragma unroll
        for (int u = 0; u < GRP; ++u) {
          t[u].x -= lij.x * lk[u].x + lij.y * lk[u].y;
          t[u].y -= lij.y * lk[u].x - lij.x * lk[u].y;
        }
#pragma unroll
        for (int u = 0; u < GRP; ++u) sts_c_if(k0 + u <= lane, own + (k0 + u) * SZ, t[u]);
      }
      __syncwarp();
    }
  }
  if (MODE == 0 || MODE == 1) {
    C* out = tile + (int64_t)lane * K;
#pragma unroll 8
    for (int j = 0; j < CT; ++j) {
      const C v = lds_c<C>(sD + (uint32_t)(lane * LD + j) * SZ);
      if (j <= lane) out[j] = v;
    }
  }
}


// register-resident rows (lane = row, compile-time indices), raw column j broadcast through a
// parity-double-buffered shared column (one store per lane and step, broadcast loads)
__device__ __noinline__ void diag_reg(float2* tile, int K, uint32_t sD, uint32_t scol, float* dinv, int lane) {
  using C = float2;
  using T = float;
  constexpr int LD = CT + 1;
  constexpr uint32_t SZ = sizeof(C);
  C a[CT];
  const C* row = tile + (int64_t)lane * K;
#pragma unroll
  for (int j = 0; j < CT; ++j) a[j] = j <= lane ? row[j] : mkc<C>(0, 0);
  sfft::static_for<0, CT>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const uint32_t col = scol + (uint32_t)((j & 1) * CT) * SZ;
    sts_c(col + (uint32_t)lane * SZ, a[j]);
    __syncwarp();
    T d = lds_c<C>(col + (uint32_t)j * SZ).x;
    const T y = rsqrtf(d);
    const T inv = y * ((T)1.5 - (T)0.5 * d * y * y);
    const T ljj = d * inv;
    const C lij = cscale(a[j], inv);
    const C li2 = cscale(lij, inv);
    a[j] = lane == j ? mkc<C>(ljj, (T)0) : (lane > j ? lij : a[j]);
    if (lane == 0) dinv[j] = inv;
    sfft::static_for<j + 1, CT>([&](auto Kk) {
      constexpr int k = decltype(Kk)::value;
      const C rk = lds_c<C>(col + (uint32_t)k * SZ);
      const C nt = vfma(vswap(li2), mkc<C>(-rk.y, rk.y), vfma(li2, vsplat<C>(-rk.x), a[k]));
      a[k] = lane >= k ? nt : a[k];
    });
  });
  C* out = tile + (int64_t)lane * K;
#pragma unroll
  for (int j = 0; j < CT; ++j) {
    sts_c(sD + (uint32_t)(lane * LD + j) * SZ, a[j]);
    if (j <= lane) out[j] = a[j];
  }
}

template <int MODE, int GRP = 8>
__global__ void k_diag_bench(float2* tiles, int K, int reps, long long* cyc, int32_t* info) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* D = reinterpret_cast<float2*>(sm);
  float* dinv = reinterpret_cast<float*>(D + 40 * 33);
  const uint32_t sD = (uint32_t)__cvta_generic_to_shared(D);
  const int lane = threadIdx.x & 31;
  float2* tile = tiles + (size_t)blockIdx.x * K * K;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE == 9) diag_tile<float>(tile, K, sD, dinv, lane, info, 0);
    else if (MODE == 8) diag_reg(tile, K, sD, sD + 40 * 33 * 8 + 64 * 4, dinv, lane);
    else diag_var<MODE, GRP>(tile, K, sD, dinv, lane, info);
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

template <int MODE, int GRP = 8>
void run(float2* d, const std::vector<float2>& h, int K, long long* c, int32_t* info, const char* name) {
  const int nb = 148, reps = 4;
  std::vector<long long> hc(nb);
  for (int pass = 0; pass < 2; ++pass) {
    cudaMemcpy(d, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
    k_diag_bench<MODE, GRP><<<nb, 32, 40 * 33 * 8 + 64 * 4 + 64 * 8>>>(d, K, reps, c, info);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(hc.data(), c, nb * 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7lld cycles per call (%s)\n", name, hc[0], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int K = 32, nb = 148;
  std::vector<float2> h((size_t)nb * K * K);
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j)
        h[(size_t)b * K * K + i * K + j] =
            make_float2(i == j ? 64.f : 0.01f * ((i * 7 + j * 3) % 11), i == j ? 0.f : 0.001f * (i - j));
  float2* d; long long* c; int32_t* info;
  cudaMalloc(&d, h.size() * sizeof(float2)); cudaMalloc(&c, nb * 8); cudaMalloc(&info, 4);
  run<9>(d, h, K, c, info, "diag_tile (product)");
  run<8>(d, h, K, c, info, "register rows");
  run<0>(d, h, K, c, info, "copy: full");
  run<1>(d, h, K, c, info, "no trailing update");
  run<2>(d, h, K, c, info, "no global load/store");
  run<3>(d, h, K, c, info, "pivot steps only");
  run<0, 16>(d, h, K, c, info, "groups of 16");
  run<0, 4>(d, h, K, c, info, "groups of 4");
  return 0;
}
