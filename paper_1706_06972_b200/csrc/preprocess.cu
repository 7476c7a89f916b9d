// Image preparation on the device (reference preprocessing.py:36-100):
// grayscale -> Gaussian local contrast normalisation -> seeded edge taper, in ONE kernel launch
// for a whole stack of images, with no host work per image.
//
// One CTA produces a T x T output tile of one image.  Everything the tile depends on is staged
// in shared memory once:
//   X      grayscale input over the tile's double halo (LCN halo around the taper halo),
//          gathered with scipy "reflect" indexing (d c b a | a b c d | d c b a);
//   MV,QV  vertical (axis 0) correlation of x and x*x (scipy correlate1d order, :53-55, :68-69);
//   NRM    (x - mean) / max(std, eps) on the taper's source region (:70-71);
//   BV     vertical pass of the taper blur, then the blended output tile (:80-89).
// The taper's source region is kept in TRUE image coordinates (it spans min..max of the
// reflected halo indices), and the blur reads it through reflect tables, so mirrored taps see
// the real normalised values for any kernel size, even or odd, and any image size.
//
// Per image the taper sigma is drawn on the device from numpy's default_rng(seed) stream
// (SeedSequence -> PCG64 -> uniform, the published algorithms numpy 2.x implements), so
// preprocess_batch matches `preprocess(image, PreprocessSpec(seed=seed0 + i))` (cli.py:116)
// without a host loop.  Gaussian weights are built per CTA in shared memory (:46-50).
//
// Arithmetic is float64 (the reference's).  The fast path (window 9, taper 11: the reference
// defaults) is register-blocked: each thread correlates a strip of RB outputs with the taps in
// registers, so shared-memory loads per output drop from S to (RB + S - 1) / RB.  Other sizes
// run the same kernel with runtime-length loops.  Roofline: FP64.

#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace ocsc {
namespace {

// ----------------------------------------------- numpy default_rng(seed).uniform(lo, hi) --
// SeedSequence (pool size 4, hashmix/mix constants) -> generate_state(4, uint64) -> PCG64
// (128-bit LCG, XSL-RR output) -> next_double = (next64 >> 11) * 2^-53.
typedef unsigned __int128 u128;

__host__ __device__ inline uint32_t ss_hash(uint32_t v, uint32_t& h, uint32_t mult) {
  v ^= h;
  h *= mult;
  v *= h;
  return v ^ (v >> 16);
}

__host__ __device__ inline double seeded_uniform(uint64_t seed, double lo, double hi) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  const uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const int nent = (seed >> 32) ? 2 : 1;
  uint32_t h = INIT_A, pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = ss_hash(i < nent ? ent[i] : 0u, h, MULT_A);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) {
        uint32_t r = MIX_L * pool[d] - MIX_R * ss_hash(pool[s], h, MULT_A);
        pool[d] = r ^ (r >> 16);
      }
  uint32_t hb = INIT_B, w[8];
  for (int i = 0; i < 8; ++i) w[i] = ss_hash(pool[i & 3], hb, MULT_B);
  uint64_t s64[4];
  for (int i = 0; i < 4; ++i) s64[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
  const u128 initstate = ((u128)s64[0] << 64) | s64[1];
  const u128 inc = ((((u128)s64[2] << 64) | s64[3]) << 1) | 1u;
  u128 st = inc;  // state = 0; step
  st += initstate;
  st = st * mult + inc;
  st = st * mult + inc;  // next64 advances, then outputs
  const uint64_t x = (uint64_t)(st >> 64) ^ (uint64_t)st;
  const unsigned r = (unsigned)(st >> 122);
  const uint64_t out = (x >> r) | (x << ((64u - r) & 63u));
  return lo + (hi - lo) * ((double)(out >> 11) * (1.0 / 9007199254740992.0));
}

// ----------------------------------------------------------------------------- geometry --
__host__ __device__ __forceinline__ int reflect_index(int i, int n) {
  // scipy.ndimage mode="reflect": period 2n, mirror about -0.5 and n-0.5
  if (i >= -n && i < 2 * n) return i < 0 ? -1 - i : (i >= n ? 2 * n - 1 - i : i);  // one mirror at most
  const int p = 2 * n;
  int m = i % p;
  if (m < 0) m += p;
  return m < n ? m : p - 1 - m;
}

struct Span {
  int lo, hi;  // [lo, hi) in image coordinates
};

// [min, max] of reflect(i) over i in [lo, hi)
__host__ __device__ inline Span reflected_span(int lo, int hi, int n) {
  if (lo >= 0 && hi <= n) return {lo, hi};
  int mn = n, mx = -1;
  for (int i = lo; i < hi; ++i) {
    const int r = reflect_index(i, n);
    mn = r < mn ? r : mn;
    mx = r > mx ? r : mx;
  }
  return {mn, mx + 1};
}

template <typename Tin>
__device__ __forceinline__ double load_gray(const Tin* img, int channels, int64_t idx) {
  if (channels == 1) return (double)img[idx];
  // luminance mix (preprocessing.py:13, :42): ((r*0.299) + g*0.587) + b*0.114, no contraction
  const Tin* px = img + 3 * idx;
  double v = __dmul_rn((double)px[0], 0.299);
  v = __dadd_rn(v, __dmul_rn((double)px[1], 0.587));
  return __dadd_rn(v, __dmul_rn((double)px[2], 0.114));
}

struct PrepArgs {
  int N, H, W, channels;
  int s1, c1;             // LCN window and its centre (window // 2, scipy origin 0)
  int s2, c2;             // taper kernel size and centre; also the ramp width (preprocessing.py:86)
  double sigma1, eps;     // LCN Gaussian width and std floor
  const double* sigma2;   // (N,) taper widths, or null: drawn from default_rng(seed0 + i)
  uint64_t seed0;
  double sig_lo, sig_hi;  // PreprocessSpec.taper_sigma_range
  int flags;              // bit 0: LCN, bit 1: taper
  const double* kg;       // Gaussian tables from k_prep_weights: LCN [s1], then taper [N][s2]
};

constexpr int T = 32;         // output tile edge
constexpr int NT = 256;       // threads per CTA
constexpr int MAXS = 64;      // largest kernel held in the shared weight table

__device__ void gaussian_table(double* k, int size, double sigma) {
  // preprocessing.py:46-50: exp(-0.5 ((x - (size-1)/2) / sigma)^2) / sum
  const double half = (size - 1) / 2.0;
  double sum = 0.0;
  for (int t = 0; t < size; ++t) {
    const double z = (t - half) / sigma;
    k[t] = exp(-0.5 * (z * z));
    sum += k[t];
  }
  for (int t = 0; t < size; ++t) k[t] /= sum;
}

// acc[o] = sum_t k[t] * v[o + t], o < RB, over a strip whose values come from `load(u)`, u < RB+S-1
template <int S, int RB, typename Load>
__device__ __forceinline__ void strip(const double (&k)[S], Load load, double (&acc)[RB]) {
#pragma unroll
  for (int o = 0; o < RB; ++o) acc[o] = 0.0;
#pragma unroll
  for (int u = 0; u < RB + S - 1; ++u) {
    const double v = load(u);
#pragma unroll
    for (int o = 0; o < RB; ++o)
      if (u - o >= 0 && u - o < S) acc[o] = fma(k[u - o], v, acc[o]);
  }
}

template <int S, int RB, typename Load>
__device__ __forceinline__ void strip2(const double (&k)[S], Load load, double (&a)[RB], double (&b)[RB]) {
#pragma unroll
  for (int o = 0; o < RB; ++o) a[o] = b[o] = 0.0;
#pragma unroll
  for (int u = 0; u < RB + S - 1; ++u) {
    const double v = load(u), v2 = v * v;
#pragma unroll
    for (int o = 0; o < RB; ++o)
      if (u - o >= 0 && u - o < S) {
        a[o] = fma(k[u - o], v, a[o]);
        b[o] = fma(k[u - o], v2, b[o]);
      }
  }
}

struct Region {
  int Rlo, Rh, Clo, Cw;  // this tile's taper source region (true coordinates)
  int Xh, Xw;            // this tile's grayscale halo tile
};

__device__ __forceinline__ Region region(const PrepArgs& a, int r0, int r1, int q0, int q1, bool lcn, bool taper) {
  Region g;
  const int h2lo = taper ? a.c2 : 0, h2hi = taper ? a.s2 - 1 - a.c2 : 0;
  const Span R = reflected_span(r0 - h2lo, r1 + h2hi, a.H);
  const Span C = reflected_span(q0 - h2lo, q1 + h2hi, a.W);
  g.Rlo = R.lo; g.Rh = R.hi - R.lo; g.Clo = C.lo; g.Cw = C.hi - C.lo;
  const int h1 = lcn ? a.s1 - 1 : 0;
  g.Xh = g.Rh + h1; g.Xw = g.Cw + h1;
  return g;
}

// Launch-uniform shared-memory plan (every tile fits the largest one; the odd pitches keep
// column-wise accesses bank-conflict free; SLACK rows/entries absorb the register strips'
// over-reads so the unrolled loops need no clamps).
constexpr int SLACK = 8;

struct Plan {
  int XP, NP, OP;                         // pitches (doubles)
  int oX, oMV, oQV, oNRM, oK1, oK2, nD;   // double offsets, total
  int oRX, oCX, oRT, oCT, nI;             // int offsets, total
};

__host__ __device__ inline Plan make_plan(int H, int W, int s1, int s2, int flags) {
  const bool lcn = flags & 1, taper = flags & 2;
  const int hl = taper ? s2 - 1 : 0, h1 = lcn ? s1 - 1 : 0;
  const int Rh = H < T + hl ? H : T + hl, Cw = W < T + hl ? W : T + hl;
  Plan p;
  p.XP = (Cw + h1) | 1;
  p.NP = Cw | 1;
  p.OP = T + 1;
  p.oX = 0;
  p.oMV = p.oX + (Rh + h1 + SLACK) * p.XP;
  p.oQV = p.oMV + Rh * p.XP;
  const int mvq_a = 2 * Rh * p.XP + SLACK, mvq_b = T * p.NP + T * p.OP;  // BV + output tile alias MV/QV
  p.oNRM = p.oMV + (mvq_a > mvq_b ? mvq_a : mvq_b);
  p.oK1 = p.oNRM + Rh * p.NP;
  p.oK2 = p.oK1 + MAXS;
  p.nD = p.oK2 + MAXS;
  p.oRX = 0;
  p.oCX = p.oRX + Rh + h1;
  p.oRT = p.oCX + Cw + h1;
  p.oCT = p.oRT + T + s2 + SLACK;
  p.nI = p.oCT + T + s2 + SLACK;
  return p;
}

inline size_t smem_bytes(const Plan& p) { return (size_t)p.nD * sizeof(double) + (size_t)p.nI * sizeof(int); }

// S1/S2 > 0: compile-time kernel sizes (register-blocked strips); 0: runtime sizes.
// Per-launch Gaussian tables (preprocessing.py:46-50): thread N builds the LCN kernel, thread
// i < N the taper kernel of image i (its width from taper_sigmas or default_rng(seed0 + i)).
__global__ void k_prep_weights(PrepArgs a, double* kg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool lcn = a.flags & 1, taper = a.flags & 2;
  if (i == a.N && lcn) {
    gaussian_table(kg, a.s1, a.sigma1);
  } else if (i < a.N && taper) {
    const double sg = a.sigma2 ? a.sigma2[i] : seeded_uniform(a.seed0 + (uint64_t)i, a.sig_lo, a.sig_hi);
    gaussian_table(kg + a.s1 + (int64_t)i * a.s2, a.s2, sg);
  }
}

template <typename Tin, typename Tout, int S1, int S2>
__global__ void __launch_bounds__(NT) k_preprocess(const Tin* __restrict__ in, Tout* __restrict__ out, PrepArgs a) {
  extern __shared__ double sm[];
  const int img = blockIdx.z;
  const int H = a.H, W = a.W;
  const int r0 = blockIdx.y * T, r1 = min(r0 + T, H);
  const int q0 = blockIdx.x * T, q1 = min(q0 + T, W);
  const int Th = r1 - r0, Tw = q1 - q0;
  const bool lcn = a.flags & 1, taper = a.flags & 2;
  const int s1 = S1 ? S1 : a.s1, s2 = S2 ? S2 : a.s2;
  const int c1 = s1 / 2, c2 = s2 / 2;
  const Region L = region(a, r0, r1, q0, q1, lcn, taper);
  const Plan P = make_plan(H, W, a.s1, a.s2, a.flags);
  const int h1lo = lcn ? c1 : 0;
  const int XP = P.XP, NP = P.NP, OP = P.OP;

  double* X = sm + P.oX;
  double* MV = sm + P.oMV;
  double* QV = sm + P.oQV;
  double* NRM = sm + P.oNRM;
  double* K1 = sm + P.oK1;
  double* K2 = sm + P.oK2;
  int* ism = reinterpret_cast<int*>(sm + P.nD);
  int* rowx = ism + P.oRX;
  int* colx = ism + P.oCX;
  int* rtb = ism + P.oRT;  // taper rows: reflect(r0 + u - c2) - Rlo, u < Th + s2 - 1 (0 beyond)
  int* ctb = ism + P.oCT;  // taper cols: reflect(q0 + u - c2) - Clo, u < Tw + s2 - 1 (0 beyond)
  double* BV = MV;           // Th x NP   (after NRM is complete)
  double* OT = MV + T * NP;  // Th x OP   blended output tile

  const int tid = threadIdx.x;
  // Gaussian tables (built once per launch by k_prep_weights, not per tile)
  if (lcn && tid < s1) K1[tid] = a.kg[tid];
  if (taper && tid >= 32 && tid < 32 + s2) K2[tid - 32] = a.kg[s1 + (int64_t)img * s2 + (tid - 32)];
  for (int u = tid; u < L.Xh; u += NT) rowx[u] = reflect_index(L.Rlo - h1lo + u, H);
  for (int u = tid; u < L.Xw; u += NT) colx[u] = reflect_index(L.Clo - h1lo + u, W);
  if (taper) {
    for (int u = tid; u < T + s2 + SLACK; u += NT) {
      rtb[u] = u < Th + s2 - 1 ? reflect_index(r0 + u - c2, H) - L.Rlo : 0;
      ctb[u] = u < Tw + s2 - 1 ? reflect_index(q0 + u - c2, W) - L.Clo : 0;
    }
  }
  __syncthreads();

  // ---- grayscale halo tile
  const Tin* src = in + (int64_t)img * H * W * a.channels;
  for (int i = tid / 32; i < L.Xh; i += NT / 32) {
    const int64_t rb = (int64_t)rowx[i] * W;
    for (int j = tid % 32; j < L.Xw; j += 32) X[i * XP + j] = load_gray(src, a.channels, rb + colx[j]);
  }
  __syncthreads();

  // ---- local contrast normalisation
  if (lcn) {
    if constexpr (S1 > 0) {
      constexpr int RB = 9, RC = 7;  // 5 x 50 and 6 x 42 strips: one pass of 256 threads each
      double k[S1];
#pragma unroll
      for (int t = 0; t < S1; ++t) k[t] = K1[t];
      const int nb = (L.Rh + RB - 1) / RB;
      for (int it = tid; it < nb * L.Xw; it += NT) {  // lanes along columns
        const int j = it % L.Xw, i0 = (it / L.Xw) * RB;
        double m[RB], q[RB];
        const double* col = X + i0 * XP + j;
        strip2<S1, RB>(k, [&](int u) { return col[u * XP]; }, m, q);
#pragma unroll
        for (int o = 0; o < RB; ++o)
          if (i0 + o < L.Rh) {
            MV[(i0 + o) * XP + j] = m[o];
            QV[(i0 + o) * XP + j] = q[o];
          }
      }
      __syncthreads();
      const int nc = (L.Cw + RC - 1) / RC;
      const double eps2 = a.eps * a.eps, inv_eps = 1.0 / a.eps;
      for (int it = tid; it < nc * L.Rh; it += NT) {  // lanes along rows (odd pitch)
        const int i = it % L.Rh, j0 = (it / L.Rh) * RC;
        double m[RC], q[RC];
        const double* mrow = MV + i * XP + j0;
        const double* qrow = QV + i * XP + j0;
        strip<S1, RC>(k, [&](int u) { return mrow[u]; }, m);
        strip<S1, RC>(k, [&](int u) { return qrow[u]; }, q);
#pragma unroll
        for (int o = 0; o < RC; ++o)
          if (j0 + o < L.Cw) {
            // (x - mean) / max(sqrt(var), eps): multiply by rsqrt(var) (1 ulp) above the floor
            const double var = fmax(q[o] - m[o] * m[o], 0.0);
            const double inv = var > eps2 ? rsqrt(var) : inv_eps;
            NRM[i * NP + j0 + o] = (X[(i + c1) * XP + j0 + o + c1] - m[o]) * inv;
          }
      }
    } else {
      for (int it = tid; it < L.Rh * L.Xw; it += NT) {
        const int i = it / L.Xw, j = it - i * L.Xw;
        double m = 0.0, q = 0.0;
        for (int t = 0; t < s1; ++t) {
          const double x = X[(i + t) * XP + j];
          m = fma(K1[t], x, m);
          q = fma(K1[t], x * x, q);
        }
        MV[i * XP + j] = m;
        QV[i * XP + j] = q;
      }
      __syncthreads();
      for (int it = tid; it < L.Rh * L.Cw; it += NT) {
        const int i = it / L.Cw, j = it - i * L.Cw;
        double m = 0.0, q = 0.0;
        for (int t = 0; t < s1; ++t) {
          m = fma(K1[t], MV[i * XP + j + t], m);
          q = fma(K1[t], QV[i * XP + j + t], q);
        }
        const double sd = sqrt(fmax(q - m * m, 0.0));
        NRM[i * NP + j] = (X[(i + c1) * XP + j + c1] - m) / fmax(sd, a.eps);
      }
    }
  } else {
    for (int it = tid; it < L.Rh * L.Cw; it += NT) {
      const int i = it / L.Cw, j = it - i * L.Cw;
      NRM[i * NP + j] = X[i * XP + j];
    }
  }
  __syncthreads();

  // ---- edge taper: blur (reflect tables), ramp blend; output tile staged for coalesced stores
  if (taper) {
    if constexpr (S2 > 0) {
      constexpr int RB = 6, RC = 4;  // 6 x 42 and 8 x 32 strips
      double k[S2];
#pragma unroll
      for (int t = 0; t < S2; ++t) k[t] = K2[t];
      const int nb = (Th + RB - 1) / RB;
      for (int it = tid; it < nb * L.Cw; it += NT) {  // lanes along columns
        const int j = it % L.Cw, i0 = (it / L.Cw) * RB;
        double b[RB];
        const int* rt = rtb + i0;
        strip<S2, RB>(k, [&](int u) { return NRM[rt[u] * NP + j]; }, b);
#pragma unroll
        for (int o = 0; o < RB; ++o)
          if (i0 + o < Th) BV[(i0 + o) * NP + j] = b[o];
      }
      __syncthreads();
      const int nc = (Tw + RC - 1) / RC;
      for (int it = tid; it < nc * Th; it += NT) {  // lanes along rows
        const int i = it % Th, j0 = (it / Th) * RC;
        double b[RC];
        const int* ct = ctb + j0;
        const double* brow = BV + i * NP;
        strip<S2, RC>(k, [&](int u) { return brow[ct[u]]; }, b);
        const double ir = r0 + i + 0.5;
        const double wr = fmin(fmin(ir, H - ir) / (double)S2, 1.0);
#pragma unroll
        for (int o = 0; o < RC; ++o)
          if (j0 + o < Tw) {
            const double jc = q0 + j0 + o + 0.5;
            const double w = wr * fmin(fmin(jc, W - jc) / (double)S2, 1.0);
            const double x = NRM[(r0 + i - L.Rlo) * NP + q0 + j0 + o - L.Clo];
            OT[i * OP + j0 + o] = w * x + (1.0 - w) * b[o];
          }
      }
    } else {
      for (int it = tid; it < Th * L.Cw; it += NT) {
        const int i = it / L.Cw, j = it - i * L.Cw;
        double b = 0.0;
        for (int t = 0; t < s2; ++t) b = fma(K2[t], NRM[rtb[i + t] * NP + j], b);
        BV[i * NP + j] = b;
      }
      __syncthreads();
      for (int it = tid; it < Th * Tw; it += NT) {
        const int i = it / Tw, j = it - i * Tw;
        double b = 0.0;
        for (int t = 0; t < s2; ++t) b = fma(K2[t], BV[i * NP + ctb[j + t]], b);
        const double ir = r0 + i + 0.5, jc = q0 + j + 0.5;
        const double w = fmin(fmin(ir, H - ir) / (double)s2, 1.0) * fmin(fmin(jc, W - jc) / (double)s2, 1.0);
        const double x = NRM[(r0 + i - L.Rlo) * NP + q0 + j - L.Clo];
        OT[i * OP + j] = w * x + (1.0 - w) * b;
      }
    }
  } else {
    for (int it = tid; it < Th * Tw; it += NT) {
      const int i = it / Tw, j = it - i * Tw;
      OT[i * OP + j] = NRM[(r0 + i - L.Rlo) * NP + q0 + j - L.Clo];
    }
  }
  __syncthreads();
  Tout* dst = out + (int64_t)img * H * W;
  for (int i = tid / 32; i < Th; i += NT / 32)
    for (int j = tid % 32; j < Tw; j += 32) dst[(int64_t)(r0 + i) * W + q0 + j] = (Tout)OT[i * OP + j];
}

template <typename Tin, typename Tout, int S1, int S2>
int launch_k(const void* in, void* out, PrepArgs a, size_t bytes, cudaStream_t st) {
  auto kern = k_preprocess<Tin, Tout, S1, S2>;
  OCSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  double* kg = nullptr;  // stream-ordered scratch for the Gaussian tables
  OCSC_CUDA(cudaMallocAsync((void**)&kg, sizeof(double) * ((size_t)a.s1 + (size_t)a.N * a.s2 + 1), st));
  k_prep_weights<<<(a.N + 1 + 127) / 128, 128, 0, st>>>(a, kg);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    a.kg = kg;
    dim3 grid((a.W + T - 1) / T, (a.H + T - 1) / T, a.N);
    kern<<<grid, NT, bytes, st>>>(static_cast<const Tin*>(in), static_cast<Tout*>(out), a);
    count_launches(1);
    e = cudaGetLastError();
  }
  const cudaError_t ef = cudaFreeAsync(kg, st);  // freed on every path (no leak on a launch error)
  if (e != cudaSuccess) return cuda_fail(e, "k_preprocess");
  if (ef != cudaSuccess) return cuda_fail(ef, "cudaFreeAsync");
  return OCSC_OK;
}

template <typename Tin, typename Tout>
int launch(const void* in, void* out, const PrepArgs& a, cudaStream_t st) {
  const size_t bytes = smem_bytes(make_plan(a.H, a.W, a.s1, a.s2, a.flags));
  if (a.s1 > MAXS || a.s2 > MAXS || bytes > 220 * 1024)
    return fail(OCSC_ESHAPE, "ocsc_preprocess: LCN window / taper size too large for a shared-memory tile");
  const bool fast1 = !(a.flags & 1) || a.s1 == 9, fast2 = !(a.flags & 2) || a.s2 == 11;
  if (fast1 && fast2) return launch_k<Tin, Tout, 9, 11>(in, out, a, bytes, st);
  return launch_k<Tin, Tout, 0, 0>(in, out, a, bytes, st);
}

template <typename Tin>
int dispatch_out(int dtype_out, const void* in, void* out, const PrepArgs& a, cudaStream_t st) {
  if (dtype_out == OCSC_F64) return launch<Tin, double>(in, out, a, st);
  if (dtype_out == OCSC_F32) return launch<Tin, float>(in, out, a, st);
  return fail(OCSC_EARG, "ocsc_preprocess: output dtype must be OCSC_F32 or OCSC_F64");
}

}  // namespace
}  // namespace ocsc

extern "C" int ocsc_taper_sigmas(int64_t seed0, int n, double lo, double hi, double* out) {
  if (seed0 < 0 || n < 0 || (n && !out)) return ocsc::fail(OCSC_EARG, "ocsc_taper_sigmas: seeds must be >= 0");
  for (int i = 0; i < n; ++i) out[i] = ocsc::seeded_uniform((uint64_t)seed0 + (uint64_t)i, lo, hi);
  return OCSC_OK;
}

extern "C" int ocsc_preprocess(int dtype_in, int dtype_out, int N, int H, int W, int channels, const void* in,
                               int flags, int lcn_window, double lcn_sigma, double lcn_epsilon, int taper_size,
                               const double* taper_sigmas, int64_t taper_seed0, double taper_sigma_lo,
                               double taper_sigma_hi, void* out, void* stream) {
  using namespace ocsc;
  if (N < 0 || H <= 0 || W <= 0 || (channels != 1 && channels != 3))
    return fail(OCSC_ESHAPE, "ocsc_preprocess: expected (N, H, W) or (N, H, W, 3) images");
  if ((flags & 1) && lcn_window <= 0) return fail(OCSC_ESHAPE, "ocsc_preprocess: LCN window must be positive");
  if ((flags & 2) && taper_size <= 0) return fail(OCSC_ESHAPE, "ocsc_preprocess: taper size must be positive");
  if ((flags & 2) && !taper_sigmas && taper_seed0 < 0) return fail(OCSC_EARG, "ocsc_preprocess: negative seed");
  if (N == 0) return OCSC_OK;
  if (!in || !out) return fail(OCSC_ESHAPE, "ocsc_preprocess: null image pointer");
  PrepArgs a{};
  a.N = N; a.H = H; a.W = W; a.channels = channels;
  a.s1 = lcn_window; a.c1 = lcn_window / 2;
  a.s2 = taper_size; a.c2 = taper_size / 2;
  a.sigma1 = lcn_sigma; a.eps = lcn_epsilon;
  a.sigma2 = taper_sigmas; a.seed0 = (uint64_t)taper_seed0;
  a.sig_lo = taper_sigma_lo; a.sig_hi = taper_sigma_hi;
  a.flags = flags & 3;
  cudaStream_t st = as_stream(stream);
  switch (dtype_in) {
    case OCSC_U8: return dispatch_out<uint8_t>(dtype_out, in, out, a, st);
    case OCSC_F32: return dispatch_out<float>(dtype_out, in, out, a, st);
    case OCSC_F64: return dispatch_out<double>(dtype_out, in, out, a, st);
    default: return fail(OCSC_EARG, "ocsc_preprocess: input dtype must be OCSC_U8, OCSC_F32 or OCSC_F64");
  }
}
