// Probe of the tcgen05 TF32 path used by the tensor-core history accumulation (dev aid):
// C[128][N] = A[128][K] * B[N][K]^T with A, B K-major in shared memory (no swizzle,
// 8-row x 16-byte core matrices), accumulator in TMEM, read back with tcgen05.ld.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe scripts/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 128, KK = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// smem layout of a K-major operand tile (rows x KK tf32): k-unit u (4 tf32 = 16 B) of row r at
// u * (rows * 16) + r * 16  ->  core matrices (8 rows x 16 B) contiguous, SBO = 128 B between
// 8-row groups, LBO = rows * 16 B between k-units
__global__ void probe(const float* A, const float* B, float* C) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* As = reinterpret_cast<uint32_t*>(smem);
  uint32_t* Bs = As + M * KK;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * KK; e += blockDim.x) {
    const int r = e / KK, k = e % KK;
    As[(k / 4) * (M * 4) + r * 4 + (k % 4)] = tf32_rna(A[r * KK + k]);
  }
  for (int e = tid; e < N * KK; e += blockDim.x) {
    const int r = e / KK, k = e % KK;
    Bs[(k / 4) * (N * 4) + r * 4 + (k % 4)] = tf32_rna(B[r * KK + k]);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // instruction descriptor: F32 accumulate, TF32 A/B, K-major both, N>>3, M>>4
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs);
    for (int kk = 0; kk < KK / 8; ++kk) {  // one MMA per 8 tf32 of K = 2 k-units
      const uint64_t ad = make_desc(a0 + kk * 2 * (M * 16), M * 16, 128);
      const uint64_t bd = make_desc(b0 + kk * 2 * (N * 16), N * 16, 128);
      const uint32_t acc = kk > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads TMEM lanes 32w..32w+31 (= rows), 32 columns at a time
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + lane;
    for (int j = 0; j < 32; ++j) C[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
}

int main() {
  std::vector<float> A(M * KK), B(N * KK), C(M * N), R(M * N);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX - 0.5f;
  for (auto& x : B) x = (float)rand() / RAND_MAX - 0.5f;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < KK; ++k) s += (double)A[i * KK + k] * B[j * KK + k];
      R[i * N + j] = (float)s;
    }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, C.size() * 4);
  const int smem = (M + N) * KK * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dB, dC);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, ref = 0;
  for (int i = 0; i < M * N; ++i) {
    err = fmax(err, fabs(C[i] - R[i]));
    ref = fmax(ref, fabs(R[i]));
  }
  printf("max abs err %.3e (max |ref| %.3e) C[0]=%f R[0]=%f C[1]=%f R[1]=%f C[129]=%f R[129]=%f\n", err, ref, C[0], R[0],
         C[1], R[1], C[129], R[129]);
  return 0;
}
