// Register-resident FFT codelets with compile-time length and compile-time
// twiddles, for the pencil transforms of the spectral layer (the
// DFFT is a chain of local sequential FFTs over index sets).
//
// fft<L, DIR>(x): in place, natural order in and out, unnormalised,
//   X[k] = sum_s x[s] exp(DIR * 2 pi i k s / L),  DIR = -1 forward, +1 inverse.
// Mixed radix 4/2/3/5 decimation in time; other primes fall back to a direct
// DFT.  Every twiddle index is a compile-time constant once the loops are
// unrolled, so the twiddles become FFMA immediates and the trivial ones
// (1, -1, +-i) disappear.  Twiddles are computed in double by a constexpr
// routine (exact at multiples of pi/2) and rounded once to float.
//
// The same header compiles for the host (tests/csrc/test_fft_host.cu), so the
// codelets are unit-tested on the CPU against a brute-force DFT.
#pragma once

#include <cuda_runtime.h>

#ifdef __CUDACC__
#define FNO_HD __host__ __device__ __forceinline__
#else
#define FNO_HD inline
#endif

namespace fno {

// --------------------------------------------------------------------------
// constexpr cos/sin(2 pi j / n) in double
// --------------------------------------------------------------------------
constexpr double kPi = 3.14159265358979323846264338327950288;

constexpr double taylor_sin(double x) {
  double term = x, sum = x;
  for (int k = 1; k < 14; ++k) {
    term *= -x * x / double((2 * k) * (2 * k + 1));
    sum += term;
  }
  return sum;
}
constexpr double taylor_cos(double x) {
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 14; ++k) {
    term *= -x * x / double((2 * k - 1) * (2 * k));
    sum += term;
  }
  return sum;
}
// angle 2*pi*j/n reduced to a quarter turn q and a remainder in [-pi/4, pi/4]
constexpr double cos2pi(long long j, long long n) {
  long long r = ((j % n) + n) % n;
  long long q = (4 * r + n / 2) / n;            // nearest quarter turn 0..4
  long long num = 4 * r - q * n;                // remainder numerator, |num| <= n/2
  double a = 2.0 * kPi * double(num) / double(4 * n);
  double c = (num == 0) ? 1.0 : taylor_cos(a);
  double s = (num == 0) ? 0.0 : taylor_sin(a);
  switch (q & 3) {
    case 0: return c;
    case 1: return -s;
    case 2: return -c;
    default: return s;
  }
}
constexpr double sin2pi(long long j, long long n) {
  long long r = ((j % n) + n) % n;
  long long q = (4 * r + n / 2) / n;
  long long num = 4 * r - q * n;
  double a = 2.0 * kPi * double(num) / double(4 * n);
  double c = (num == 0) ? 1.0 : taylor_cos(a);
  double s = (num == 0) ? 0.0 : taylor_sin(a);
  switch (q & 3) {
    case 0: return s;
    case 1: return c;
    case 2: return -s;
    default: return -c;
  }
}

template <int N>
struct TwTable {
  float c[N > 0 ? N : 1];
  float s[N > 0 ? N : 1];
  constexpr TwTable() : c(), s() {
    for (int j = 0; j < N; ++j) {
      c[j] = float(cos2pi(j, N));
      s[j] = float(sin2pi(j, N));
    }
  }
};

#ifdef __CUDACC__
template <int N>
__device__ constexpr TwTable<N> kTwDev{};
#endif
template <int N>
constexpr TwTable<N> kTwHost{};

template <int N>
FNO_HD float tw_cos(int j) {
#ifdef __CUDA_ARCH__
  return kTwDev<N>.c[j];
#else
  return kTwHost<N>.c[j];
#endif
}
template <int N>
FNO_HD float tw_sin(int j) {
#ifdef __CUDA_ARCH__
  return kTwDev<N>.s[j];
#else
  return kTwHost<N>.s[j];
#endif
}

// --------------------------------------------------------------------------
// complex helpers
// --------------------------------------------------------------------------
FNO_HD float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
FNO_HD float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
FNO_HD float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
FNO_HD float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
FNO_HD float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// acc + a*b
FNO_HD float2 cfma(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a)*b
FNO_HD float2 cfma_conj_a(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
  return acc;
}

// a * exp(DIR * 2 pi i j / N), j a compile-time constant after unrolling
template <int N, int DIR>
FNO_HD float2 twiddle(float2 a, int j) {
  j %= N;
  if (j == 0) return a;
  if (2 * j == N) return make_float2(-a.x, -a.y);
  if (4 * j == N) return DIR > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);     // * (+-i)
  if (4 * j == 3 * N) return DIR > 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x); // * (-+i)
  const float c = tw_cos<N>(j);
  const float s = DIR > 0 ? tw_sin<N>(j) : -tw_sin<N>(j);
  return make_float2(fmaf(a.x, c, -a.y * s), fmaf(a.x, s, a.y * c));
}

constexpr int pick_radix(int n) {
  return (n % 4 == 0) ? 4 : (n % 2 == 0) ? 2 : (n % 3 == 0) ? 3 : (n % 5 == 0) ? 5 : n;
}

// small DFT of prime-ish length P (2, 3, 4, 5 specialised; others direct)
template <int P, int DIR>
FNO_HD void dft_small(float2 (&x)[P]) {
  if constexpr (P == 1) {
    return;
  } else if constexpr (P == 2) {
    float2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  } else if constexpr (P == 4) {
    float2 a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]);
    float2 b0 = cadd(x[1], x[3]), b1 = csub(x[1], x[3]);
    // b1 * (DIR i)
    float2 b1r = DIR > 0 ? make_float2(-b1.y, b1.x) : make_float2(b1.y, -b1.x);
    x[0] = cadd(a0, b0);
    x[2] = csub(a0, b0);
    x[1] = cadd(a1, b1r);
    x[3] = csub(a1, b1r);
  } else if constexpr (P == 3) {
    constexpr float c1 = -0.5f;
    const float s1 = (DIR > 0 ? 1.0f : -1.0f) * 0.866025403784438646763723170752936183f;
    float2 t = cadd(x[1], x[2]);
    float2 d = csub(x[1], x[2]);
    float2 m = make_float2(fmaf(c1, t.x, x[0].x), fmaf(c1, t.y, x[0].y));
    float2 r = make_float2(-s1 * d.y, s1 * d.x);  // i*s1*d
    x[0] = cadd(x[0], t);
    x[1] = cadd(m, r);
    x[2] = csub(m, r);
  } else {
    float2 y[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      float2 acc = x[0];
#pragma unroll
      for (int s = 1; s < P; ++s) acc = cadd(acc, twiddle<P, DIR>(x[s], (k * s) % P));
      y[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = y[k];
  }
}

template <int N, int DIR>
FNO_HD void fft(float2 (&x)[N]) {
  if constexpr (N == 1) {
    return;
  } else {
    constexpr int P = pick_radix(N);
    if constexpr (P == N) {
      dft_small<N, DIR>(x);
    } else {
      constexpr int M = N / P;
      float2 sub[P][M];
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int m = 0; m < M; ++m) sub[r][m] = x[P * m + r];
#pragma unroll
      for (int r = 0; r < P; ++r) fft<M, DIR>(sub[r]);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        float2 t[P];
#pragma unroll
        for (int r = 0; r < P; ++r) t[r] = twiddle<N, DIR>(sub[r][k], r * k);
        dft_small<P, DIR>(t);
#pragma unroll
        for (int l = 0; l < P; ++l) x[k + M * l] = t[l];
      }
    }
  }
}

}  // namespace fno
