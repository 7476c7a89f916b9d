// History accumulation on the 5th-generation tensor cores (dictionary.py:94-97, 117-127;
// SURVEY.md 8(a) a11/a12; BASELINE config 4): per frequency p,
//     S_p += Z_p Z_p^H,   c_p += Z_p conj(x_p)      (Z_p: K x B complex codes of the batch)
// as real GEMMs with the sample axis as the reduction dimension (Z = X + iY):
//     Re S = X X^T + Y Y^T,     Im S = Y X^T - X Y^T.
// The north_star allows tensor cores for this accumulation only with a split precision that
// keeps float32 accuracy: every operand is split into TF32 hi + lo parts and each product is
// hi*hi + hi*lo + lo*hi (3xTF32, ~2^-21 relative), accumulated in FP32 in TMEM.
//
// One CTA (128 threads) computes a 128 x 128 block pair (I >= J) of the lower triangle of one
// frequency: samples are staged 8 at a time into one of two shared-memory buffers as K-major
// TF32 tiles (no swizzle: 8-row x 16-byte core matrices), one thread issues the chunk's twelve
// tcgen05.mma.kind::tf32 (M = N = 128, K = 8) into two TMEM accumulators (Re: columns 0-127,
// Im: 128-255; the minus sign of X Y^T through the instruction descriptor's negate-A bit) and
// commits them to the buffer's mbarrier, so the next chunk stages while they run; at the end the
// four warps read their 32 TMEM lanes (= rows) with tcgen05.ld, transpose through shared memory
// and add to the packed lower triangle with row-coalesced updates (history precision).  The diagonal-block CTAs also
// accumulate c on CUDA cores while staging.  K is padded to 128 with zero rows, B to 8.
#include "common.cuh"

namespace ocsc {
namespace {

constexpr int TB = 128;      // block edge (MMA M = N)
constexpr int TKC = 8;       // samples staged per chunk (one MMA K-step); two chunk buffers
constexpr int TILE_WORDS = TB * TKC;  // one operand tile (tf32 words)
constexpr int BUF_WORDS = 8 * TILE_WORDS;  // the eight operand tiles of one chunk (32 KB)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); base offset 0; SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mbar), "r"(phase));
  }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
}

// operand tiles in shared memory: [XI hi, XI lo, YI hi, YI lo, XJ hi, XJ lo, YJ hi, YJ lo], each
// TB rows x TKC tf32, k-unit u (4 tf32 = 16 B) of row r at u * TB * 16 + r * 16 bytes
// (LBO = TB * 16 between k-units, SBO = 128 B between 8-row groups)
template <typename Th>
__global__ void __launch_bounds__(256) k_hist_accum_tc(int K, int B, const float2* __restrict__ z, int64_t z_sb,
                                                       int64_t z_sk, int64_t z_sp, const float2* __restrict__ x,
                                                       int64_t x_sb, int64_t x_sp, cx<Th>* S, cx<Th>* c, int pairs) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* T = reinterpret_cast<uint32_t*>(smem);  // two chunk buffers, then reused by the epilogue
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int p = blockIdx.x / pairs, tp = blockIdx.x - (blockIdx.x / pairs) * pairs;
  int I = (int)((sqrtf(8.0f * tp + 1.0f) - 1.0f) * 0.5f);
  while (I * (I + 1) / 2 > tp) --I;
  while ((I + 1) * (I + 2) / 2 <= tp) ++I;
  const int J = tp - I * (I + 1) / 2;
  const bool diag = I == J;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int trow = tid & (TB - 1), thalf = tid >> 7;  // staging: row trow, samples thalf*4 .. +3
  const int ri = I * TB + trow, rj = J * TB + trow;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[1])));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TB >> 3) << 17) | ((uint32_t)(TB >> 4) << 24);
  const uint32_t idesc_neg = idesc | (1u << 13);  // negate A

  // the epilogue read-modify-writes this block of S (DRAM-resident): ask L2 for its rows now, so
  // the staging and the MMAs run while they arrive (128-byte lines; a row of the block is
  // TB complex = 1 KB (float) / 2 KB (double) of the packed triangle)
  {
    const int64_t npk_ = (int64_t)K * (K + 1) / 2;
    constexpr int LINES = TB * (int)sizeof(cx<Th>) / 128;  // lines per block row
    for (int e = tid; e < TB * LINES; e += 256) {
      const int rr = e / LINES, ln = e - rr * LINES, row = I * TB + rr, col = J * TB + ln * (128 / (int)sizeof(cx<Th>));
      if (row < K && col <= row)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(S + (int64_t)p * npk_ + packed_index(row, col)));
    }
  }
  float2 cacc = make_float2(0.f, 0.f);
  uint32_t phase[2] = {0, 0};
  const int nchunk = (B + TKC - 1) / TKC;
  // raw code values of a chunk, loaded one chunk ahead (the loads of chunk ch + 1 are in flight
  // while chunk ch is converted, staged and issued)
  float2 rvi[TKC / 2], rvj[TKC / 2];
  auto load_raw = [&](int ch) {
#pragma unroll
    for (int s4 = 0; s4 < TKC / 2; ++s4) {
      const int b = ch * TKC + thalf * (TKC / 2) + s4;
      rvi[s4] = make_float2(0.f, 0.f);
      rvj[s4] = make_float2(0.f, 0.f);
      if (b < B) {
        const int64_t base = (int64_t)b * z_sb + (int64_t)p * z_sp;
        if (ri < K) rvi[s4] = z[base + (int64_t)ri * z_sk];
        if (!diag && rj < K) rvj[s4] = z[base + (int64_t)rj * z_sk];
      }
    }
  };
  load_raw(0);
  for (int ch = 0; ch < nchunk; ++ch) {
    const int buf = ch & 1;
    if (ch >= 2) {  // the MMAs of chunk ch-2 read this buffer: wait for their commit
      mbar_wait(su32(&mbar[buf]), phase[buf]);
      phase[buf] ^= 1;
    }
    uint32_t* Tb = T + buf * BUF_WORDS;
    const int b0 = ch * TKC;
    // ---- stage 8 samples (4 per thread): TF32 hi / lo split, K-major core-matrix layout ----
    // a thread's 4 samples of one row are one 16-byte k-unit of every tile: one vector store per
    // tile (a warp's 32 rows then fill 512 contiguous bytes, no bank conflicts)
    {
      uint32_t xh[4], xl[4], yh[4], yl[4], jxh[4], jxl[4], jyh[4], jyl[4];
#pragma unroll
      for (int s4 = 0; s4 < TKC / 2; ++s4) {
        const int b = b0 + thalf * (TKC / 2) + s4;
        const float2 vi = rvi[s4], vj = rvj[s4];
        if (diag && b < B && ri < K) {  // cross term c_i += conj(x_b) z_bi on CUDA cores
          const float2 xb = x[(int64_t)b * x_sb + (int64_t)p * x_sp];
          cacc.x += xb.x * vi.x + xb.y * vi.y;
          cacc.y += xb.x * vi.y - xb.y * vi.x;
        }
        xh[s4] = to_tf32(vi.x);
        xl[s4] = to_tf32(vi.x - __uint_as_float(xh[s4]));
        yh[s4] = to_tf32(vi.y);
        yl[s4] = to_tf32(vi.y - __uint_as_float(yh[s4]));
        jxh[s4] = to_tf32(vj.x);
        jxl[s4] = to_tf32(vj.x - __uint_as_float(jxh[s4]));
        jyh[s4] = to_tf32(vj.y);
        jyl[s4] = to_tf32(vj.y - __uint_as_float(jyh[s4]));
      }
      if (ch + 1 < nchunk) load_raw(ch + 1);
      const uint32_t off = thalf * (TB * 4) + trow * 4;  // word offset of the k-unit inside a tile
      auto st4 = [&](int tile, const uint32_t (&v)[4]) {
        *reinterpret_cast<uint4*>(Tb + tile * TILE_WORDS + off) = make_uint4(v[0], v[1], v[2], v[3]);
      };
      st4(0, xh);
      st4(1, xl);
      st4(2, yh);
      st4(3, yl);
      if (!diag) {
        st4(4, jxh);
        st4(5, jxl);
        st4(6, jyh);
        st4(7, jyl);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy writes -> visible to the MMA
    __syncthreads();
    if (tid == 0) {  // one thread issues; the MMAs run asynchronously while the next chunk stages
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t t0 = su32(Tb);
      const int j0 = diag ? 0 : 4;  // B-side tiles
      auto tile = [&](int t) { return umma_desc(t0 + (uint32_t)(t * TILE_WORDS * 4), TB * 16, 128); };
      const uint32_t re = tmem, im = tmem + TB;
      const uint64_t XIh = tile(0), XIl = tile(1), YIh = tile(2), YIl = tile(3);
      const uint64_t XJh = tile(j0 + 0), XJl = tile(j0 + 1), YJh = tile(j0 + 2), YJl = tile(j0 + 3);
      const uint32_t acc0 = ch > 0;
      // Re S += X_I X_J^T + Y_I Y_J^T
      mma_tf32(re, XIh, XJh, idesc, acc0);
      mma_tf32(re, XIh, XJl, idesc, 1);
      mma_tf32(re, XIl, XJh, idesc, 1);
      mma_tf32(re, YIh, YJh, idesc, 1);
      mma_tf32(re, YIh, YJl, idesc, 1);
      mma_tf32(re, YIl, YJh, idesc, 1);
      // Im S += Y_I X_J^T - X_I Y_J^T
      mma_tf32(im, YIh, XJh, idesc, acc0);
      mma_tf32(im, YIh, XJl, idesc, 1);
      mma_tf32(im, YIl, XJh, idesc, 1);
      mma_tf32(im, XIh, YJh, idesc_neg, 1);
      mma_tf32(im, XIh, YJl, idesc_neg, 1);
      mma_tf32(im, XIl, YJh, idesc_neg, 1);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(&mbar[buf])));
    }
  }
  // all MMAs done (tcgen05 ops complete in issue order: the last commit covers them all)
  {
    const int last = (nchunk - 1) & 1;
    mbar_wait(su32(&mbar[last]), phase[last]);
    if (nchunk >= 2) mbar_wait(su32(&mbar[last ^ 1]), phase[last ^ 1]);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");

  // ---- epilogue: TMEM -> shared memory -> coalesced row updates.  Warp w reads TMEM lanes
  // 32(w%4)..+31 (= rows), the real accumulator for w < 4, the imaginary one for w >= 4 ----
  float* E = reinterpret_cast<float*>(smem);  // [2][TB][33]: the Re plane, then the Im plane (odd row
                                              // stride: conflict-free column writes and row reads)
  const int64_t npk = (int64_t)K * (K + 1) / 2;
  const uint32_t lanebase = (uint32_t)((warp & 3) * 32) << 16;
  const int part = warp >> 2;  // 0: Re, 1: Im
#pragma unroll 1
  for (int c0 = 0; c0 < TB; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + lanebase + part * TB + c0, v);
    const int r = (warp & 3) * 32 + lane;
#pragma unroll
    for (int q = 0; q < 32; ++q) E[part * (TB * 33) + r * 33 + q] = __uint_as_float(v[q]);
    __syncthreads();
    const int col = J * TB + c0 + lane;
    // lanes = 32 consecutive columns of one row; NB of a warp's 16 rows have their loads in
    // flight before the first add (float: all 16)
    constexpr int NB = sizeof(Th) == 4 ? 16 : 8;  // rows in flight per warp (double: 8 keeps two CTAs per SM)
#pragma unroll 1
    for (int rb = 0; rb < TB / 8; rb += NB) {
      cx<Th> cur[NB];
      int64_t at[NB];
      bool ok[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int rr = warp + 8 * (rb + u), row = I * TB + rr;
        ok[u] = row < K && col <= row && col < K;
        at[u] = (int64_t)p * npk + packed_index(row, col);
        if (ok[u]) cur[u] = S[at[u]];
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int rr = warp + 8 * (rb + u);
        if (ok[u]) {
          const float vr = E[rr * 33 + lane], vi = E[TB * 33 + rr * 33 + lane];
          S[at[u]] = mkc<cx<Th>>(cur[u].x + (Th)vr, cur[u].y + (Th)vi);
        }
      }
    }
    __syncthreads();
  }
  // cross term: the two halves of every diagonal-block row
  float2* cs = reinterpret_cast<float2*>(smem);
  if (diag && thalf == 1) cs[trow] = cacc;
  __syncthreads();
  if (diag && thalf == 0 && ri < K) {
    cx<Th>& d = c[(int64_t)p * K + ri];
    const float2 o = cs[trow];
    d = mkc<cx<Th>>(d.x + (Th)(cacc.x + o.x), d.y + (Th)(cacc.y + o.y));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

}  // namespace

// float32 code spectra -> history (float32 or float64) on the tensor cores; returns 0 when launched
int history_accumulate_tc(int dtype_hist, int K, int nfreq, int B, const void* z, int64_t z_sb, int64_t z_sk,
                          int64_t z_sp, const void* x, int64_t x_sb, int64_t x_sp, void* S, void* c, cudaStream_t s) {
  const int nb = (K + TB - 1) / TB, pairs = nb * (nb + 1) / 2;
  const int64_t grid = (int64_t)nfreq * pairs;
  if (grid > 0x7fffffff) return fail(OCSC_EARG, "history_accumulate: too many blocks");
  // two chunk buffers of 8 operand tiles = 64 KB (the epilogue's 33 KB staging reuses them); at
  // most three CTAs fit an SM by shared memory, two by TMEM (2 x 256 columns): a third waits in alloc
  const size_t smem = 2 * BUF_WORDS * sizeof(uint32_t);
  if (dtype_hist == OCSC_F32) {
    OCSC_CUDA(cudaFuncSetAttribute(k_hist_accum_tc<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist_accum_tc<float><<<(unsigned)grid, 256, smem, s>>>(K, B, (const float2*)z, z_sb, z_sk, z_sp,
                                                              (const float2*)x, x_sb, x_sp, (float2*)S, (float2*)c,
                                                              pairs);
  } else if (dtype_hist == OCSC_F64) {
    OCSC_CUDA(cudaFuncSetAttribute(k_hist_accum_tc<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist_accum_tc<double><<<(unsigned)grid, 256, smem, s>>>(K, B, (const float2*)z, z_sb, z_sk, z_sp,
                                                               (const float2*)x, x_sb, x_sp, (double2*)S,
                                                               (double2*)c, pairs);
  } else {
    return fail(OCSC_EARG, "history_accumulate: unsupported dtype pair");
  }
  OCSC_LAUNCHED("k_hist_accum_tc");
  return OCSC_OK;
}

}  // namespace ocsc
