// FMA-chain microbenchmark (FP32 / FP64 peaks are not in MEASURED_PEAKS.json).
// Measures the sustained per-SM rate of register-operand FFMA, FFMA2 (FP32x2) and DFMA with
// many independent chains per thread and a full grid, timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak scripts/fma_peak.cu
//   ./fma_peak  ->  one JSON line: flops per clock per SM and TFLOP/s at the observed clock
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 16;        // independent chains per thread
constexpr int ITERS = 4096;   // loop trips (each: CH FMAs per chain set)

__global__ void k_ffma(float* out, const float* ab, int iters) {
  const float a = ab[0], b = ab[1];  // register operands (not constant-bank / immediate forms)
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
#pragma unroll 4
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);  // a, b in registers (kernel args)
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, const float* ab, int iters) {
  const float a = ab[0], b = ab[1];
  float2 x[CH];
  const float2 av = make_float2(a, a * 0.5f), bv = make_float2(b, b * 0.5f);
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
#pragma unroll 4
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(x[c], av, bv);
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c].x + x[c].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_dfma(double* out, const double* ab, int iters) {
  const double a = ab[0], b = ab[1];
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
#pragma unroll 4
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename F>
static double time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* fo;
  double* dout;
  cudaMalloc(&fo, 4096 * sizeof(float));
  cudaMalloc(&dout, 4096 * sizeof(double));
  float* fab;
  double* dab;
  const float hf[2] = {0.999f, 1e-3f};
  const double hd[2] = {0.999, 1e-3};
  cudaMalloc(&fab, sizeof(hf));
  cudaMalloc(&dab, sizeof(hd));
  cudaMemcpy(fab, hf, sizeof(hf), cudaMemcpyHostToDevice);
  cudaMemcpy(dab, hd, sizeof(hd), cudaMemcpyHostToDevice);
  const int threads = 256, blocks = sms * 8;
  const double nthr = (double)threads * blocks;
  const double t32 = time_ms([&] { k_ffma<<<blocks, threads>>>(fo, fab, ITERS); });
  const double t2 = time_ms([&] { k_ffma2<<<blocks, threads>>>(fo, fab, ITERS); });
  const double t64 = time_ms([&] { k_dfma<<<blocks, threads / 2>>>(dout, dab, ITERS / 4); });
  const cudaError_t e = cudaDeviceSynchronize();
  const double f32 = 2.0 * CH * ITERS * nthr / (t32 * 1e-3);            // flops/s
  const double f2 = 4.0 * CH * ITERS * nthr / (t2 * 1e-3);
  const double f64 = 2.0 * CH * (ITERS / 4) * (nthr / 2) / (t64 * 1e-3);
  printf("{\"status\": \"%s\", \"sms\": %d, \"attr_clock_mhz\": %.0f, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, "
         "\"dfma_tflops\": %.2f, \"ms\": [%.3f, %.3f, %.3f]}\n",
         cudaGetErrorString(e), sms, clk_khz / 1e3, f32 / 1e12, f2 / 1e12, f64 / 1e12, t32, t2, t64);
  return 0;
}
