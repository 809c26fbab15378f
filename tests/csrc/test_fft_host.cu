// Host-side unit test of the register FFT codelets (paper_2204_01205_b200/csrc/fft.cuh)
// against a brute-force double-precision DFT.  Built and run by tests/test_fft_codelets.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include "../../paper_2204_01205_b200/csrc/fft.cuh"

static unsigned long long g_state = 88172645463325252ull;
static double urand() { g_state ^= g_state << 13; g_state ^= g_state >> 7; g_state ^= g_state << 17; return (g_state >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0; }

template <int N, int DIR>
static double check() {
  double worst = 0;
  for (int trial = 0; trial < 20; ++trial) {
    float2 x[N]; double xr[N], xi[N];
    for (int s = 0; s < N; ++s) { x[s].x = (float)urand(); x[s].y = (float)urand(); xr[s] = x[s].x; xi[s] = x[s].y; }
    fno::fft<N, DIR>(x);
    double num = 0, den = 0;
    for (int k = 0; k < N; ++k) {
      double re = 0, im = 0;
      for (int s = 0; s < N; ++s) {
        double a = DIR * 2.0 * M_PI * (double)((long long)k * s % N) / N;
        re += xr[s] * cos(a) - xi[s] * sin(a);
        im += xr[s] * sin(a) + xi[s] * cos(a);
      }
      num += (x[k].x - re) * (x[k].x - re) + (x[k].y - im) * (x[k].y - im);
      den += re * re + im * im;
    }
    double rel = sqrt(num / den);
    if (rel > worst) worst = rel;
  }
  printf("N=%d DIR=%d rel_l2=%.3e\n", N, DIR, worst);
  return worst;
}

static double twiddle_table_error() {
  double worst = 0;
  const int ns[] = {2, 3, 4, 5, 6, 8, 12, 15, 16, 30, 32, 64};
  for (int n : ns)
    for (int j = 0; j < n; ++j) {
      double e = fabs(fno::cos2pi(j, n) - cos(2 * M_PI * j / n)) + fabs(fno::sin2pi(j, n) - sin(2 * M_PI * j / n));
      if (e > worst) worst = e;
    }
  printf("constexpr twiddle max abs error vs libm: %.3e\n", worst);
  return worst;
}

int main() {
  double w = 0;
  w = fmax(w, check<2, -1>()); w = fmax(w, check<3, -1>()); w = fmax(w, check<4, -1>());
  w = fmax(w, check<5, 1>()); w = fmax(w, check<6, -1>()); w = fmax(w, check<7, 1>());
  w = fmax(w, check<8, -1>()); w = fmax(w, check<8, 1>()); w = fmax(w, check<12, 1>());
  w = fmax(w, check<15, -1>()); w = fmax(w, check<16, -1>()); w = fmax(w, check<16, 1>());
  w = fmax(w, check<30, -1>()); w = fmax(w, check<30, 1>()); w = fmax(w, check<32, -1>());
  w = fmax(w, check<32, 1>()); w = fmax(w, check<64, -1>());
  double t = twiddle_table_error();
  int ok = (w < 2e-6) && (t < 1e-14);
  printf("%s worst=%.3e\n", ok ? "PASS" : "FAIL", w);
  return ok ? 0 : 1;
}
