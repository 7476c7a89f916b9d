// Dev aid: do a second kernel's clusters co-schedule on the SMs a resident first cluster kernel
// leaves free?  Kernel A: NA clusters of CA CTAs (one CTA per SM through its shared memory), each
// CTA spinning SPIN_US; kernel B, launched right after on another stream: NB clusters of CB CTAs.
// Prints, per B cluster size, how many B clusters started while A was still running.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/probe scripts/probe_cosched.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void spin(unsigned long long* rec, unsigned long long ns) {
  extern __shared__ char smem[];
  const unsigned long long t0 = gtime();
  if (threadIdx.x == 0) smem[0] = 1;
  while (gtime() - t0 < ns) {
  }
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    rec[3 * blockIdx.x] = t0;
    rec[3 * blockIdx.x + 1] = gtime();
    rec[3 * blockIdx.x + 2] = smid;
  }
}

static void launch(int nclu, int cs, int threads, int smem, unsigned long long* rec, unsigned long long ns,
                   cudaStream_t s) {
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(spin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclu * cs);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, spin, rec, ns);
  if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
}

static int max_active(int cs, int threads, int smem) {
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(spin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  cudaOccupancyMaxActiveClusters(&n, spin, &cfg);
  return n;
}

int main(int argc, char** argv) {
  const int CA = argc > 1 ? atoi(argv[1]) : 10;
  const int smemA = 186160, smemB = 226656;
  printf("max active clusters (1 CTA/SM):");
  for (int c = 1; c <= 16; ++c) printf(" c%d=%d", c, max_active(c, 256, smemB));
  printf("\n");
  const int NA = max_active(CA, 448, smemA);
  unsigned long long *ra, *rb;
  cudaMalloc(&ra, 3 * 8 * 2048);
  cudaMalloc(&rb, 3 * 8 * 2048);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  const unsigned long long ns = 3000000ull;
  for (int CB = 2; CB <= 10; ++CB) {
    const int NB = 40;
    for (int rep = 0; rep < 2; ++rep) {
      launch(NA, CA, 448, smemA, ra, ns, s1);
      launch(NB, CB, 256, smemB, rb, ns, s2);
      cudaDeviceSynchronize();
    }
    std::vector<unsigned long long> ha(3 * NA * CA), hb(3 * NB * CB);
    cudaMemcpy(ha.data(), ra, ha.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), rb, hb.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long a0 = ~0ull, a1 = 0;
    for (int i = 0; i < NA * CA; ++i) a0 = std::min(a0, ha[3 * i]), a1 = std::max(a1, ha[3 * i + 1]);
    int during = 0, sms = 0;
    for (int c = 0; c < NB; ++c) {
      unsigned long long st = ~0ull;
      for (int j = 0; j < CB; ++j) st = std::min(st, hb[3 * (c * CB + j)]);
      if (st < a1 - ns / 2) ++during, sms += CB;
    }
    printf("A: %d x %d-CTA clusters (%d SMs), B cluster %2d: %2d clusters (%3d SMs) co-resident with A; "
           "total %d SMs busy\n", NA, CA, NA * CA, CB, during, sms, NA * CA + sms);
  }
  return 0;
}
