// Dev aid: residency of a programmatically launched (PDL) cluster grid behind a spinning
// cluster grid.  Each CTA records start, end and SM id; prints the overlap picture.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/probe_pdl scripts/probe_pdl.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void spin(unsigned long long* rec, unsigned long long ns, int trigger) {
  if (trigger) asm volatile("griddepcontrol.launch_dependents;");
  const unsigned long long t0 = gtime();
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

static void launch(int nclu, int cs, int threads, int smem, unsigned long long* rec, unsigned long long ns, int trig,
                   bool pdl, cudaStream_t s) {
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(spin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclu * cs);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, spin, rec, ns, trig);
  if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
}

int main(int argc, char** argv) {
  const int CA = 10, NA = 11, CB = argc > 1 ? atoi(argv[1]) : 8, NB = argc > 2 ? atoi(argv[2]) : 15;
  const unsigned long long nsA = 300000, nsB = argc > 3 ? atoll(argv[3]) : 1000;
  unsigned long long *ra, *rb;
  cudaMalloc(&ra, 3 * 8 * 4096);
  cudaMalloc(&rb, 3 * 8 * 4096);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ra, 0, 3 * 8 * 4096);
    cudaMemset(rb, 0, 3 * 8 * 4096);
    cudaDeviceSynchronize();
    launch(NA, CA, 448, 186160, ra, nsA, 1, false, s);
    launch(NB, CB, 576, 226656, rb, nsB, 0, true, s);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> ha(3 * NA * CA), hb(3 * NB * CB);
    cudaMemcpy(ha.data(), ra, ha.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), rb, hb.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, a_start_max = 0, a_end_min = ~0ull;
    for (int i = 0; i < NA * CA; ++i) {
      t0 = std::min(t0, ha[3 * i]);
      a_start_max = std::max(a_start_max, ha[3 * i]);
      a_end_min = std::min(a_end_min, ha[3 * i + 1]);
    }
    for (int i = 0; i < NB * CB; ++i) t0 = std::min(t0, hb[3 * i]);
    printf("rep %d: A starts [%.1f, %.1f] us, A first end %.1f us; A SMs:", rep,
           (double)(std::min_element(ha.begin(), ha.end()) == ha.end() ? 0 : 0), (a_start_max - t0) * 1e-3,
           (a_end_min - t0) * 1e-3);
    std::vector<int> sm_used(160, 0);
    for (int i = 0; i < NA * CA; ++i) sm_used[ha[3 * i + 2]] |= 1;
    int na = 0;
    for (int i = 0; i < 160; ++i) na += sm_used[i] & 1;
    printf(" %d distinct\n", na);
    int during = 0;
    for (int c = 0; c < NB; ++c) {
      unsigned long long st = ~0ull;
      int shared_sm = 0;
      for (int j = 0; j < CB; ++j) {
        st = std::min(st, hb[3 * (c * CB + j)]);
        shared_sm += sm_used[hb[3 * (c * CB + j) + 2]] & 1;
      }
      const bool d = st < a_end_min;
      during += d;
      printf("  B cluster %2d start %8.1f us %s (SMs also used by A: %d)\n", c, (st - t0) * 1e-3, d ? "DURING A" : "", shared_sm);
    }
    printf("  -> %d B clusters started while A ran\n", during);
  }
  return 0;
}
