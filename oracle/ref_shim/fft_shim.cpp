// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Stand-in for the reference's FFTW wrapper (proj/core/src/fft.cpp:105-126),
// which cannot be built here because FFTW3 is not installed
// (proj/core/CMakeLists.txt:2-3, unpinned `find_library(fftw3)`).
// Only the 1D real transforms used by the hot path are provided; they keep
// FFTW's published semantics (proj/core/include/radonkit/fft.hpp:8-14):
//   rfft : n reals -> n/2+1 complex bins, unnormalised forward transform
//   irfft: n/2+1 bins (Hermitian half spectrum) -> n reals, scaled by 1/n
// The 2D transforms (shearlets) use the same 1-D FFT
// along rows then columns.
//
// Algorithm (both precisions): iterative radix-2 decimation-in-time FFT of
// the real row embedded as complex, twiddles W_n^k = exp(-/+ 2 pi i k / n)
// evaluated in double as cos/sin((2 pi k) / n) and rounded to the working
// precision; arithmetic in the working precision (float for the filter,
// sino_filter.cpp:106-123; double for make_filter, :81).  In double this
// reproduces the golden bins of proj/tests/test_sino_filter.cpp:14-31 bit
// for bit (as numpy's pocketfft does).  Non power-of-two n (never produced by
// the reference, which pads to a power of two, sino_filter.cpp:69) falls back
// to a direct DFT.
#include <cmath>
#include <complex>
#include <stdexcept>
#include <vector>

#include "radonkit/fft.hpp"

namespace radonkit::fft {

namespace {

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// twiddle exp(sign * 2 pi i k / n)... with sign = +1 meaning the forward
// transform exp(-2 pi i k / n); the angle is reduced exactly in integers
template <class T>
std::complex<T> twiddle(long k, long n, int sign) {
  long r = ((k % n) + n) % n;
  double ang = 2.0 * M_PI * double(r) / double(n);
  return std::complex<T>(T(std::cos(ang)), T(-double(sign) * std::sin(ang)));
}

// twiddle table W_n^k, k < n/2, cached per thread (filter_sinogram calls
// rfft/irfft from parallel_for workers, sino_filter.cpp:109-121)
template <class T>
const std::vector<std::complex<T>>& twiddle_table(int n, int sign) {
  thread_local std::vector<std::complex<T>> tab[2];
  thread_local int tab_n[2] = {0, 0};
  int slot = sign > 0 ? 0 : 1;
  if (tab_n[slot] != n) {
    tab[slot].resize(size_t(n / 2));
    for (int k = 0; k < n / 2; ++k) tab[slot][size_t(k)] = twiddle<T>(k, n, sign);
    tab_n[slot] = n;
  }
  return tab[slot];
}

template <class T>
void fft_radix2(std::vector<std::complex<T>>& a, int sign) {
  int n = int(a.size());
  if (n < 2) return;
  const std::vector<std::complex<T>>& w = twiddle_table<T>(n, sign);
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[size_t(i)], a[size_t(j)]);
  }
  for (int len = 2; len <= n; len <<= 1) {
    int half = len / 2;
    int stride = n / len;
    for (int i = 0; i < n; i += len) {
      for (int k = 0; k < half; ++k) {
        std::complex<T> u = a[size_t(i + k)];
        std::complex<T> v = a[size_t(i + k + half)] * w[size_t(k * stride)];
        a[size_t(i + k)] = u + v;
        a[size_t(i + k + half)] = u - v;
      }
    }
  }
}

template <class T>
void dft_direct(std::vector<std::complex<T>>& a, int sign) {
  int n = int(a.size());
  std::vector<std::complex<T>> out(a.size());
  for (int k = 0; k < n; ++k) {
    std::complex<T> acc(0, 0);
    for (int j = 0; j < n; ++j) acc += a[size_t(j)] * twiddle<T>(long(j) * k, n, sign);
    out[size_t(k)] = acc;
  }
  a.swap(out);
}

template <class T>
void cfft(std::vector<std::complex<T>>& a, int sign) {
  if (is_pow2(int(a.size())))
    fft_radix2(a, sign);
  else
    dft_direct(a, sign);
}

}  // namespace

void rfft(int n, const float* in, std::complex<float>* out) {
  std::vector<std::complex<float>> a(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) a[size_t(i)] = {in[i], 0.0f};
  cfft(a, +1);
  for (int q = 0; q <= n / 2; ++q) out[q] = a[size_t(q)];
}

void irfft(int n, const std::complex<float>* in, float* out) {
  std::vector<std::complex<float>> a(static_cast<size_t>(n));
  for (int q = 0; q <= n / 2; ++q) a[size_t(q)] = in[q];
  for (int q = n / 2 + 1; q < n; ++q) a[size_t(q)] = std::conj(in[n - q]);
  // c2r ignores the imaginary parts of the DC and Nyquist bins
  a[0] = {a[0].real(), 0.0f};
  if (n % 2 == 0) a[size_t(n / 2)] = {a[size_t(n / 2)].real(), 0.0f};
  cfft(a, -1);
  float inv = 1.0f / float(n);
  for (int i = 0; i < n; ++i) out[i] = a[size_t(i)].real() * inv;
}

void rfft(int n, const double* in, std::complex<double>* out) {
  std::vector<std::complex<double>> a(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) a[size_t(i)] = {in[i], 0.0};
  cfft(a, +1);
  for (int q = 0; q <= n / 2; ++q) out[q] = a[size_t(q)];
}

void irfft(int n, const std::complex<double>* in, double* out) {
  std::vector<std::complex<double>> a(static_cast<size_t>(n));
  for (int q = 0; q <= n / 2; ++q) a[size_t(q)] = in[q];
  for (int q = n / 2 + 1; q < n; ++q) a[size_t(q)] = std::conj(in[n - q]);
  a[0] = {a[0].real(), 0.0};
  if (n % 2 == 0) a[size_t(n / 2)] = {a[size_t(n / 2)].real(), 0.0};
  cfft(a, -1);
  double inv = 1.0 / double(n);
  for (int i = 0; i < n; ++i) out[i] = a[size_t(i)].real() * inv;
}

// 2-D transforms (shearlet.cpp's rfft2 / irfft2): row transforms then column
// transforms with the same 1-D FFT, in the working precision; h x (w/2+1) half
// spectrum; the inverse keeps FFTW's c2r semantics (Hermitian completion of
// every row, 1/(h w) normalisation).
namespace {
template <class T>
void rfft2_t(int h, int w, const T* in, std::complex<T>* out) {
  const int wc = w / 2 + 1;
  std::vector<std::complex<T>> full(static_cast<size_t>(h) * static_cast<size_t>(w));
  std::vector<std::complex<T>> row(static_cast<size_t>(w));
  for (int i = 0; i < h; ++i) {
    for (int j = 0; j < w; ++j) row[size_t(j)] = {in[size_t(i) * w + j], T(0)};
    cfft(row, +1);
    for (int j = 0; j < w; ++j) full[size_t(i) * w + j] = row[size_t(j)];
  }
  std::vector<std::complex<T>> col(static_cast<size_t>(h));
  for (int j = 0; j < wc; ++j) {
    for (int i = 0; i < h; ++i) col[size_t(i)] = full[size_t(i) * w + j];
    cfft(col, +1);
    for (int i = 0; i < h; ++i) out[size_t(i) * wc + j] = col[size_t(i)];
  }
}

template <class T>
void irfft2_t(int h, int w, const std::complex<T>* in, T* out) {
  const int wc = w / 2 + 1;
  // inverse along columns on the half spectrum, then a c2r row transform
  std::vector<std::complex<T>> half(static_cast<size_t>(h) * static_cast<size_t>(wc));
  std::vector<std::complex<T>> col(static_cast<size_t>(h));
  for (int j = 0; j < wc; ++j) {
    for (int i = 0; i < h; ++i) col[size_t(i)] = in[size_t(i) * wc + j];
    cfft(col, -1);
    for (int i = 0; i < h; ++i) half[size_t(i) * wc + j] = col[size_t(i)];
  }
  std::vector<std::complex<T>> row(static_cast<size_t>(w));
  const T inv = T(1) / (T(h) * T(w));
  for (int i = 0; i < h; ++i) {
    for (int q = 0; q < wc; ++q) row[size_t(q)] = half[size_t(i) * wc + q];
    for (int q = wc; q < w; ++q) row[size_t(q)] = std::conj(half[size_t(i) * wc + (w - q)]);
    row[0] = {row[0].real(), T(0)};
    if (w % 2 == 0) row[size_t(w / 2)] = {row[size_t(w / 2)].real(), T(0)};
    cfft(row, -1);
    for (int j = 0; j < w; ++j) out[size_t(i) * w + j] = row[size_t(j)].real() * inv;
  }
}
}  // namespace

void rfft2(int h, int w, const float* in, std::complex<float>* out) { rfft2_t(h, w, in, out); }
void irfft2(int h, int w, const std::complex<float>* in, float* out) { irfft2_t(h, w, in, out); }
void rfft2(int h, int w, const double* in, std::complex<double>* out) { rfft2_t(h, w, in, out); }
void irfft2(int h, int w, const std::complex<double>* in, double* out) { irfft2_t(h, w, in, out); }

}  // namespace radonkit::fft
