// Register-resident small FFTs with compile-time length and compile-time twiddles.
//
// fft<C, N, INV>(x) transforms x[0..N) held in registers (N known at compile
// time): mixed-radix decimation in time on the smallest prime factor, prime
// lengths by the symmetric direct DFT.  Every index and every twiddle is a
// compile-time constant, so after unrolling the transform is straight-line
// FFMA code with immediate operands -- no shared-memory twiddle loads.
// Forward uses e^{-2 pi i jk/N}, inverse e^{+2 pi i jk/N}, both unnormalised.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace ocsc {
namespace sfft {

constexpr double kPi = 3.14159265358979323846264338327950288;

__host__ __device__ constexpr double reduce_angle(double x) {
  // to [-pi, pi]
  const double two_pi = 2.0 * kPi;
  long long n = (long long)(x / two_pi + (x >= 0 ? 0.5 : -0.5));
  return x - (double)n * two_pi;
}

__host__ __device__ constexpr double ce_sin(double x) {
  x = reduce_angle(x);
  double term = x, sum = x;
  for (int n = 1; n < 30; ++n) {
    term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
    sum += term;
  }
  return sum;
}

__host__ __device__ constexpr double ce_cos(double x) {
  x = reduce_angle(x);
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < 30; ++n) {
    term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
    sum += term;
  }
  return sum;
}

__host__ __device__ constexpr int smallest_factor(int n) {
  for (int f = 2; f * f <= n; ++f)
    if (n % f == 0) return f;
  return n;
}

// p^e exactly dividing n for the smallest prime p | n
__host__ __device__ constexpr int prime_power_factor(int n) {
  const int p = smallest_factor(n);
  int q = p;
  while (n % (q * p) == 0) q *= p;
  return q;
}

__host__ __device__ constexpr int modinv(int a, int m) {
  a %= m;
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 1;  // m == 1
}

template <int Begin, int End, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (Begin < End) {
    f(std::integral_constant<int, Begin>{});
    static_for<Begin + 1, End>(f);
  }
}

// v * e^{(INV ? +1 : -1) 2 pi i E / N}
template <typename C, int N, int E, bool INV>
__device__ __forceinline__ C twiddle(C v) {
  using T = decltype(C::x);
  constexpr int e = E % N;
  if constexpr (e == 0) {
    return v;
  } else if constexpr (4 * e == N) {  // -i (fwd) / +i (inv)
    return INV ? mkc<C>(-v.y, v.x) : mkc<C>(v.y, -v.x);
  } else if constexpr (2 * e == N) {
    return mkc<C>(-v.x, -v.y);
  } else if constexpr (4 * e == 3 * N) {
    return INV ? mkc<C>(v.y, -v.x) : mkc<C>(-v.y, v.x);
  } else {
    constexpr T c = (T)ce_cos(2.0 * kPi * e / N);
    constexpr T s = (T)((INV ? 1.0 : -1.0) * ce_sin(2.0 * kPi * e / N));
    return vfma(vswap(v), mkc<C>(-s, s), vmul(v, vsplat<C>(c)));  // (v.x c - v.y s, v.y c + v.x s)
  }
}

// direct DFT of prime length R (R = 2 butterfly; odd R with the j <-> R-j pairing).
// Complex adds and real-by-complex products run as 2-wide FP32x2 instructions.
template <typename C, int R, bool INV>
__device__ __forceinline__ void dft_prime(C (&x)[R]) {
  using T = decltype(C::x);
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    const C a = x[0], b = x[1];
    x[0] = vadd(a, b);
    x[1] = vsub(a, b);
  } else {
    constexpr int Hh = (R - 1) / 2;
    C s[Hh], d[Hh];
    const C x0 = x[0];
    C sum = x0;
    static_for<1, Hh + 1>([&](auto J) {
      constexpr int j = decltype(J)::value;
      s[j - 1] = vadd(x[j], x[R - j]);
      d[j - 1] = vsub(x[j], x[R - j]);
      sum = vadd(sum, s[j - 1]);
    });
    static_for<1, Hh + 1>([&](auto Kk) {
      constexpr int k = decltype(Kk)::value;
      C a = x0, bsum = mkc<C>(0, 0);
      static_for<1, Hh + 1>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr T c = (T)ce_cos(2.0 * kPi * ((j * k) % R) / R);
        constexpr T sn = (T)ce_sin(2.0 * kPi * ((j * k) % R) / R);
        a = vfma(s[j - 1], vsplat<C>(c), a);
        if constexpr (j == 1) bsum = vmul(d[0], vsplat<C>(sn));
        else bsum = vfma(d[j - 1], vsplat<C>(sn), bsum);
      });
      // forward: X[k] = a - i*b, X[R-k] = a + i*b (b = sum d_j sin); inverse swaps
      if constexpr (!INV) {
        x[k] = sub_i(a, bsum);
        x[R - k] = add_i(a, bsum);
      } else {
        x[k] = add_i(a, bsum);
        x[R - k] = sub_i(a, bsum);
      }
    });
    x[0] = sum;
  }
}

template <typename C, int N, bool INV>
__device__ __forceinline__ void fft(C (&x)[N]);

// Cooley-Tukey decimation in time on the smallest prime (prime powers)
template <typename C, int N, bool INV>
__device__ __forceinline__ void fft_ct(C (&x)[N]) {
  constexpr int R = smallest_factor(N);
  constexpr int M = N / R;
  C sub[R][M];
  static_for<0, R>([&](auto Rr) {
    constexpr int r = decltype(Rr)::value;
    static_for<0, M>([&](auto Mm) {
      constexpr int m = decltype(Mm)::value;
      sub[r][m] = x[m * R + r];
    });
    fft<C, M, INV>(sub[r]);
  });
  static_for<0, M>([&](auto Kk) {
    constexpr int k = decltype(Kk)::value;
    C tmp[R];
    static_for<0, R>([&](auto Rr) {
      constexpr int r = decltype(Rr)::value;
      tmp[r] = twiddle<C, N, r * k, INV>(sub[r][k]);
    });
    dft_prime<C, R, INV>(tmp);
    static_for<0, R>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      x[k + M * q] = tmp[q];
    });
  });
}

// Good-Thomas prime-factor algorithm for N = N1 * N2 with gcd(N1, N2) = 1: no twiddles.
// input  n = (N2 n1 + N1 n2) mod N ;  output k = (N2 t2 k1 + N1 t1 k2) mod N,
// t2 = N2^-1 mod N1, t1 = N1^-1 mod N2.
template <typename C, int N, bool INV>
__device__ __forceinline__ void fft_pfa(C (&x)[N]) {
  constexpr int N1 = prime_power_factor(N);
  constexpr int N2 = N / N1;
  constexpr int t2 = modinv(N2 % N1, N1), t1 = modinv(N1 % N2, N2);
  C sub[N1][N2];
  static_for<0, N1>([&](auto A) {
    constexpr int n1 = decltype(A)::value;
    static_for<0, N2>([&](auto Bb) {
      constexpr int n2 = decltype(Bb)::value;
      sub[n1][n2] = x[(N2 * n1 + N1 * n2) % N];
    });
    fft<C, N2, INV>(sub[n1]);
  });
  static_for<0, N2>([&](auto Kk) {
    constexpr int k2 = decltype(Kk)::value;
    C tmp[N1];
    static_for<0, N1>([&](auto A) {
      constexpr int n1 = decltype(A)::value;
      tmp[n1] = sub[n1][k2];
    });
    fft<C, N1, INV>(tmp);
    static_for<0, N1>([&](auto A) {
      constexpr int k1 = decltype(A)::value;
      x[(N2 * t2 * k1 + N1 * t1 * k2) % N] = tmp[k1];
    });
  });
}

template <typename C, int N, bool INV>
__device__ __forceinline__ void fft(C (&x)[N]) {
  if constexpr (N == 1) {
    return;
  } else if constexpr (smallest_factor(N) == N) {
    dft_prime<C, N, INV>(x);
  } else if constexpr (prime_power_factor(N) == N) {
    fft_ct<C, N, INV>(x);
  } else {
    fft_pfa<C, N, INV>(x);
  }
}

}  // namespace sfft
}  // namespace ocsc
