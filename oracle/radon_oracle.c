/*
 * ORACLE TEST INFRASTRUCTURE — not product code.  Only tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load
 * this library, and only as the checker.
 *
 * Plain-C restatement of the reference's hot path (TorchRadon's CPU
 * restatement "radonkit", /root/reference/proj/core/src).  Every function
 * follows the cited reference lines operation by operation (same double
 * expressions, same evaluation order, same loop order), so with
 * -ffp-contract=off it reproduces the reference bit for bit; tests pin this
 * against oracle/_ref (the reference compiled in place) and against the
 * golden vectors of the reference's own test-suite (tests/golden/).
 *
 * Conventions (geometry.hpp:10-16): image B x s x s row-major, row 0 at the
 * top; pixel (i,j) centre (j - s/2 + .5, s/2 - i - .5); detector cell k at
 * u_k = (k - nd/2 + .5) * spacing; theta rotates counter-clockwise; at
 * theta = 0 parallel rays travel along +y.
 *
 * All projector entry points take the image / sinogram already widened to
 * double (the reference widens half -> float -> double exactly,
 * projector.cpp:207-224, 59) and return the double accumulators; narrowing
 * to the storage precision is done by the caller (tensor.cpp:111-124).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------- geometry */

/* geometry.cpp:67-73 */
void or_angles_linspace(double start, double stop, int64_t n, double* out) {
  double step = (stop - start) / (double)n;
  for (int64_t i = 0; i < n; ++i) out[i] = start + (double)i * step;
}

/* ---------------------------------------------------------------- projector */

/* projector.cpp:37-45 */
static inline int clip_slab(double o, double d, double lo, double hi, double* t0, double* t1) {
  if (d == 0.0) return o >= lo && o <= hi;
  double a = (lo - o) / d;
  double b = (hi - o) / d;
  if (a > b) {
    double tmp = a;
    a = b;
    b = tmp;
  }
  if (a > *t0) *t0 = a; /* std::max(t0, a) */
  if (b < *t1) *t1 = b; /* std::min(t1, b) */
  return 1;
}

/* projector.cpp:47-64 */
static inline double bilinear(const double* img, int64_t s, double x, double y) {
  double px = x + 0.5 * (double)s - 0.5;
  double py = 0.5 * (double)s - y - 0.5;
  double fj = floor(px);
  double fi = floor(py);
  int64_t j0 = (int64_t)fj;
  int64_t i0 = (int64_t)fi;
  double fx = px - fj;
  double fy = py - fi;
#define VAL(i, j) (((i) < 0 || (i) >= s || (j) < 0 || (j) >= s) ? 0.0 : img[(i) * s + (j)])
  double top = (1.0 - fx) * VAL(i0, j0) + fx * VAL(i0, j0 + 1);
  double bot = (1.0 - fx) * VAL(i0 + 1, j0) + fx * VAL(i0 + 1, j0 + 1);
#undef VAL
  return (1.0 - fy) * top + fy * bot;
}

/* projector.cpp:66-83 */
static double integrate_ray(const double* img, int64_t s, double ox, double oy, double dx, double dy, double tmin,
                            double tmax, double step) {
  double half = 0.5 * (double)s;
  double t0 = tmin, t1 = tmax;
  if (!clip_slab(ox, dx, -half, half, &t0, &t1)) return 0.0;
  if (!clip_slab(oy, dy, -half, half, &t0, &t1)) return 0.0;
  if (!(t1 > t0)) return 0.0;
  double len = t1 - t0;
  int64_t n = (int64_t)ceil(len / step);
  if (n < 1) n = 1;
  double h = len / (double)n;
  double acc = 0.0;
  for (int64_t m = 0; m < n; ++m) {
    double t = t0 + ((double)m + 0.5) * h;
    acc += bilinear(img, s, ox + t * dx, oy + t * dy);
  }
  return h * acc;
}

/* Number of samples the reference takes on one ray (projector.cpp:66-78);
 * returns 0 for a ray that misses the image. Used for the exact algorithmic
 * work count of the roofline. */
static int64_t ray_samples(int64_t s, double ox, double oy, double dx, double dy, double tmin, double tmax,
                           double step) {
  double half = 0.5 * (double)s;
  double t0 = tmin, t1 = tmax;
  if (!clip_slab(ox, dx, -half, half, &t0, &t1)) return 0;
  if (!clip_slab(oy, dy, -half, half, &t0, &t1)) return 0;
  if (!(t1 > t0)) return 0;
  int64_t n = (int64_t)ceil((t1 - t0) / step);
  return n < 1 ? 1 : n;
}

/* projector.cpp:95-113 */
void or_forward_parallel(int64_t s, int64_t na, const double* angles, int64_t nd, double spacing, double step,
                         int64_t nb, const double* img, double* out) {
  double inf = INFINITY;
#pragma omp parallel for schedule(static)
  for (int64_t ba = 0; ba < nb * na; ++ba) {
    int64_t b = ba / na, a = ba % na;
    const double* im = img + b * s * s;
    double c = cos(angles[a]), sn = sin(angles[a]); /* angle_trig, projector.cpp:89-93 */
    double* row = out + ba * nd;
    for (int64_t k = 0; k < nd; ++k) {
      double u = ((double)k - 0.5 * (double)nd + 0.5) * spacing;
      row[k] = integrate_ray(im, s, u * c, u * sn, -sn, c, -inf, inf, step);
    }
  }
}

/* projector.cpp:115-139 */
void or_forward_fanbeam(int64_t s, int64_t na, const double* angles, int64_t nd, double spacing, double source_distance,
                        double det_distance, double step, int64_t nb, const double* img, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t ba = 0; ba < nb * na; ++ba) {
    int64_t b = ba / na, a = ba % na;
    const double* im = img + b * s * s;
    double c = cos(angles[a]), sn = sin(angles[a]);
    double sx = source_distance * sn;
    double sy = -source_distance * c;
    double* row = out + ba * nd;
    for (int64_t k = 0; k < nd; ++k) {
      double u = ((double)k - 0.5 * (double)nd + 0.5) * spacing;
      double px = u * c - det_distance * sn;
      double py = u * sn + det_distance * c;
      double dx = px - sx, dy = py - sy;
      double len = sqrt(dx * dx + dy * dy);
      row[k] = integrate_ray(im, s, sx, sy, dx / len, dy / len, 0.0, len, step);
    }
  }
}

/* Exact forward sample count per image: sum over rays of max(1, ceil(len/step)). */
int64_t or_forward_samples(int kind, int64_t s, int64_t na, const double* angles, int64_t nd, double spacing,
                           double source_distance, double det_distance, double step) {
  int64_t total = 0;
  double inf = INFINITY;
#pragma omp parallel for reduction(+ : total) schedule(static)
  for (int64_t a = 0; a < na; ++a) {
    double c = cos(angles[a]), sn = sin(angles[a]);
    for (int64_t k = 0; k < nd; ++k) {
      double u = ((double)k - 0.5 * (double)nd + 0.5) * spacing;
      if (kind == 0) {
        total += ray_samples(s, u * c, u * sn, -sn, c, -inf, inf, step);
      } else {
        double sx = source_distance * sn, sy = -source_distance * c;
        double px = u * c - det_distance * sn, py = u * sn + det_distance * c;
        double dx = px - sx, dy = py - sy;
        double len = sqrt(dx * dx + dy * dy);
        total += ray_samples(s, sx, sy, dx / len, dy / len, 0.0, len, step);
      }
    }
  }
  return total;
}

/* projector.cpp:141-168 */
void or_backprojection_parallel(int64_t s, int64_t na, const double* angles, int64_t nd, double spacing, int64_t nb,
                                const double* sino, double* out) {
  double* trig = (double*)malloc(sizeof(double) * 2 * (size_t)na);
  for (int64_t a = 0; a < na; ++a) {
    trig[2 * a] = cos(angles[a]);
    trig[2 * a + 1] = sin(angles[a]);
  }
#pragma omp parallel for schedule(static)
  for (int64_t bi = 0; bi < nb * s; ++bi) {
    int64_t b = bi / s, i = bi % s;
    const double* sg = sino + b * na * nd;
    double y = 0.5 * (double)s - (double)i - 0.5;
    double* row = out + bi * s;
    for (int64_t j = 0; j < s; ++j) {
      double x = (double)j - 0.5 * (double)s + 0.5;
      double acc = 0.0;
      for (int64_t a = 0; a < na; ++a) {
        double u = x * trig[2 * a] + y * trig[2 * a + 1];
        double kf = u / spacing + 0.5 * (double)nd - 0.5;
        double fk = floor(kf);
        int64_t k0 = (int64_t)fk;
        double w = kf - fk;
        const double* srow = sg + a * nd;
        if (k0 >= 0 && k0 < nd) acc += (1.0 - w) * srow[k0];
        if (k0 + 1 >= 0 && k0 + 1 < nd) acc += w * srow[k0 + 1];
      }
      row[j] = acc;
    }
  }
  free(trig);
}

/* projector.cpp:170-203 */
void or_backprojection_fanbeam(int64_t s, int64_t na, const double* angles, int64_t nd, double spacing,
                               double source_distance, double det_distance, int64_t nb, const double* sino,
                               double* out) {
  double* trig = (double*)malloc(sizeof(double) * 2 * (size_t)na);
  for (int64_t a = 0; a < na; ++a) {
    trig[2 * a] = cos(angles[a]);
    trig[2 * a + 1] = sin(angles[a]);
  }
  double span = source_distance + det_distance;
#pragma omp parallel for schedule(static)
  for (int64_t bi = 0; bi < nb * s; ++bi) {
    int64_t b = bi / s, i = bi % s;
    const double* sg = sino + b * na * nd;
    double y = 0.5 * (double)s - (double)i - 0.5;
    double* row = out + bi * s;
    for (int64_t j = 0; j < s; ++j) {
      double x = (double)j - 0.5 * (double)s + 0.5;
      double acc = 0.0;
      for (int64_t a = 0; a < na; ++a) {
        double c = trig[2 * a], sn = trig[2 * a + 1];
        double qx = x * c + y * sn;
        double qy = -x * sn + y * c;
        double u = qx * span / (qy + source_distance);
        double kf = u / spacing + 0.5 * (double)nd - 0.5;
        double fk = floor(kf);
        int64_t k0 = (int64_t)fk;
        double w = kf - fk;
        const double* srow = sg + a * nd;
        if (k0 >= 0 && k0 < nd) acc += (1.0 - w) * srow[k0];
        if (k0 + 1 >= 0 && k0 + 1 < nd) acc += w * srow[k0 + 1];
      }
      row[j] = acc;
    }
  }
  free(trig);
}

/* ---------------------------------------------------------------- filter */

/* sino_filter.cpp:37-41 */
int64_t or_next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

/* sino_filter.cpp:43-60; kind 0 ram-lak, 1 shepp-logan, 2 cosine, 3 hamming, 4 hann */
static double window_gain(int kind, double nu) {
  switch (kind) {
    case 1: {
      if (nu == 0.0) return 1.0;
      double t = 0.5 * M_PI * nu;
      return sin(t) / t;
    }
    case 2: return cos(0.5 * M_PI * nu);
    case 3: return 0.54 + 0.46 * cos(M_PI * nu);
    case 4: return 0.5 + 0.5 * cos(M_PI * nu);
    default: return 1.0;
  }
}

/* Real part of the double rfft of the ramp kernel (fft.cpp:109-111).  FFTW
 * is a third-party dependency (unpinned, absent here); its published result
 * is the DFT sum_j x_j exp(-2 pi i j q / n).  Restated as the iterative
 * radix-2 decimation-in-time FFT with double twiddles cos/sin((2 pi k)/n),
 * which reproduces the golden bins of test_sino_filter.cpp:14-31 bit for bit
 * (numpy's pocketfft agrees on them too). */
typedef struct {
  double re, im;
} cf64;

static void fft_radix2_d(cf64* a, int64_t n) {
  for (int64_t i = 1, j = 0; i < n; ++i) {
    int64_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      cf64 t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
  for (int64_t len = 2; len <= n; len <<= 1) {
    int64_t half = len / 2, stride = n / len;
    for (int64_t i = 0; i < n; i += len) {
      for (int64_t k = 0; k < half; ++k) {
        double ang = 2.0 * M_PI * (double)(k * stride) / (double)n;
        cf64 w = {cos(ang), -sin(ang)};
        cf64 u = a[i + k], x = a[i + k + half];
        cf64 v = {x.re * w.re - x.im * w.im, x.re * w.im + x.im * w.re};
        a[i + k].re = u.re + v.re;
        a[i + k].im = u.im + v.im;
        a[i + k + half].re = u.re - v.re;
        a[i + k + half].im = u.im - v.im;
      }
    }
  }
}

static void rfft_real_d(int64_t n, const double* in, double* re_out) {
  cf64* a = (cf64*)malloc(sizeof(cf64) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    a[i].re = in[i];
    a[i].im = 0.0;
  }
  fft_radix2_d(a, n);
  for (int64_t q = 0; q <= n / 2; ++q) re_out[q] = a[q].re;
  free(a);
}

/* sino_filter.cpp:64-92: resp / resp_f receive padded/2+1 bins; returns padded size */
int64_t or_make_filter(int kind, int64_t det_count, double* resp, float* resp_f) {
  int64_t n = or_next_pow2(2 * det_count);
  if (n < 2) n = 2;
  double* kernel = (double*)calloc((size_t)n, sizeof(double));
  kernel[0] = 0.25;
  for (int64_t p = 1; p < n; ++p) {
    int64_t m = p < n - p ? p : n - p;
    if (m % 2 == 1) kernel[p] = -1.0 / ((double)m * (double)m * M_PI * M_PI);
  }
  double* re = (double*)malloc(sizeof(double) * (size_t)(n / 2 + 1));
  rfft_real_d(n, kernel, re);
  for (int64_t q = 0; q <= n / 2; ++q) {
    double nu = (double)q / (double)(n / 2);
    double v = 2.0 * re[q] * window_gain(kind, nu);
    if (resp) resp[q] = v;
    if (resp_f) resp_f[q] = (float)v;
  }
  free(re);
  free(kernel);
  return n;
}

typedef struct {
  float re, im;
} cf32;

static inline cf32 cmul(cf32 a, cf32 b) {
  cf32 r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}

/* Single-precision radix-2 FFT, the restatement of the float path of the
 * oracle's FFTW stand-in (oracle/ref_shim/fft_shim.cpp): twiddles
 * exp(-sign * 2 pi i k/n) evaluated in double and rounded, bit-reversal then
 * iterative butterflies. n must be a power of two (the reference always pads
 * to one, sino_filter.cpp:69). */
static void fft_f32(cf32* a, int64_t n, int sign, const cf32* tw) {
  for (int64_t i = 1, j = 0; i < n; ++i) {
    int64_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      cf32 t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
  for (int64_t len = 2; len <= n; len <<= 1) {
    int64_t half = len / 2, stride = n / len;
    for (int64_t i = 0; i < n; i += len) {
      for (int64_t k = 0; k < half; ++k) {
        cf32 u = a[i + k];
        cf32 v = cmul(a[i + k + half], tw[k * stride]);
        a[i + k].re = u.re + v.re;
        a[i + k].im = u.im + v.im;
        a[i + k + half].re = u.re - v.re;
        a[i + k + half].im = u.im - v.im;
      }
    }
  }
  (void)sign;
}

static void twiddles_f32(int64_t n, int sign, cf32* tw) {
  for (int64_t k = 0; k < n / 2; ++k) {
    double ang = 2.0 * M_PI * (double)k / (double)n;
    tw[k].re = (float)cos(ang);
    tw[k].im = (float)(-(double)sign * sin(ang));
  }
}

/* sino_filter.cpp:98-124 on float rows (the reference widens every storage
 * precision to float first, :106, and narrows the float result, :123).
 * rows = batch * n_angles. */
void or_filter_sinogram(int64_t rows, int64_t n_angles, int64_t det_count, int64_t padded, const float* resp_f,
                        const float* in, float* out) {
  int64_t n = padded;
  float scale = (float)(M_PI / (2.0 * (double)n_angles));
  cf32* twf = (cf32*)malloc(sizeof(cf32) * (size_t)(n / 2 + 1));
  cf32* twi = (cf32*)malloc(sizeof(cf32) * (size_t)(n / 2 + 1));
  twiddles_f32(n, +1, twf);
  twiddles_f32(n, -1, twi);
#pragma omp parallel
  {
    cf32* a = (cf32*)malloc(sizeof(cf32) * (size_t)n);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
      const float* src = in + r * det_count;
      /* zero-pad, rfft (fft.cpp:105-107) */
      for (int64_t i = 0; i < n; ++i) {
        a[i].re = i < det_count ? src[i] : 0.0f;
        a[i].im = 0.0f;
      }
      fft_f32(a, n, +1, twf);
      /* spec[q] *= response_f[q] on the half spectrum (sino_filter.cpp:117) */
      for (int64_t q = 0; q <= n / 2; ++q) {
        a[q].re = a[q].re * resp_f[q];
        a[q].im = a[q].im * resp_f[q];
      }
      /* irfft (fft.cpp:113-119): Hermitian fill, DC/Nyquist imaginary dropped, x 1/n */
      for (int64_t q = n / 2 + 1; q < n; ++q) {
        a[q].re = a[n - q].re;
        a[q].im = -a[n - q].im;
      }
      a[0].im = 0.0f;
      a[n / 2].im = 0.0f;
      fft_f32(a, n, -1, twi);
      float inv = 1.0f / (float)n;
      float* dst = out + r * det_count;
      for (int64_t k = 0; k < det_count; ++k) dst[k] = (a[k].re * inv) * scale;
    }
    free(a);
  }
  free(twf);
  free(twi);
}

/* ---------------------------------------------------------------- phantom */

typedef struct {
  double value, a, b, x0, y0, theta_deg;
} ellipse_t;

/* phantom.cpp:18-29 (Toft's modified Shepp-Logan) */
static const ellipse_t kSL[10] = {
    {1.0, 0.69, 0.92, 0.0, 0.0, 0.0},        {-0.8, 0.6624, 0.874, 0.0, -0.0184, 0.0},
    {-0.2, 0.11, 0.31, 0.22, 0.0, -18.0},    {-0.2, 0.16, 0.41, -0.22, 0.0, 18.0},
    {0.1, 0.21, 0.25, 0.0, 0.35, 0.0},       {0.1, 0.046, 0.046, 0.0, 0.1, 0.0},
    {0.1, 0.046, 0.046, 0.0, -0.1, 0.0},     {0.1, 0.046, 0.023, -0.08, -0.605, 0.0},
    {0.1, 0.023, 0.023, 0.0, -0.606, 0.0},   {0.1, 0.023, 0.046, 0.06, -0.605, 0.0},
};

/* phantom.cpp:33-51 */
static void rasterize(int64_t size, double* img) {
  memset(img, 0, sizeof(double) * (size_t)(size * size));
  for (int e = 0; e < 10; ++e) {
    const ellipse_t* E = &kSL[e];
    double th = E->theta_deg * M_PI / 180.0;
    double ct = cos(th), st = sin(th);
    double inv_a2 = 1.0 / (E->a * E->a), inv_b2 = 1.0 / (E->b * E->b);
    for (int64_t i = 0; i < size; ++i) {
      double y = (double)(size - 1 - 2 * i) / (double)size;
      for (int64_t j = 0; j < size; ++j) {
        double x = (double)(2 * j + 1 - size) / (double)size;
        double dx = x - E->x0, dy = y - E->y0;
        double u = dx * ct + dy * st;
        double v = -dx * st + dy * ct;
        if (u * u * inv_a2 + v * v * inv_b2 <= 1.0) img[i * size + j] += E->value;
      }
    }
  }
}

/* phantom.cpp:61-101: 1 x size x size in double (narrow with from_double_as) */
void or_shepp_logan(int64_t size, double* out) {
  const int64_t kBase = 400;
  double* base = (double*)malloc(sizeof(double) * (size_t)(kBase * kBase));
  rasterize(kBase, base);
  if (size == kBase) {
    memcpy(out, base, sizeof(double) * (size_t)(kBase * kBase));
    free(base);
    return;
  }
  int64_t* lo = (int64_t*)malloc(sizeof(int64_t) * (size_t)size);
  int64_t* hi = (int64_t*)malloc(sizeof(int64_t) * (size_t)size);
  double* frac = (double*)malloc(sizeof(double) * (size_t)size);
  for (int64_t i = 0; i < size; ++i) {
    double c = (double)((2 * i + 1) * kBase - size) / (double)(2 * size);
    double fl = floor(c);
    int64_t i0 = (int64_t)fl;
    double f = c - fl;
    if (i0 < 0) {
      i0 = 0;
      f = 0.0;
    }
    if (i0 >= kBase - 1) {
      i0 = kBase - 1;
      f = 0.0;
    }
    lo[i] = i0;
    hi[i] = i0 + 1 < kBase - 1 ? i0 + 1 : kBase - 1;
    frac[i] = f;
  }
  for (int64_t i = 0; i < size; ++i) {
    const double* r0 = base + lo[i] * kBase;
    const double* r1 = base + hi[i] * kBase;
    double fy = frac[i];
    for (int64_t j = 0; j < size; ++j) {
      double fx = frac[j];
      int64_t j0 = lo[j], j1 = hi[j];
      double top = (1.0 - fx) * r0[j0] + fx * r0[j1];
      double bot = (1.0 - fx) * r1[j0] + fx * r1[j1];
      out[i * size + j] = (1.0 - fy) * top + fy * bot;
    }
  }
  free(lo);
  free(hi);
  free(frac);
  free(base);
}

/* ---------------------------------------------------------------- rng */

/* std::mt19937 (the engine behind rng.hpp:13-38), restated. */
typedef struct {
  uint32_t mt[624];
  int idx;
} mt19937_t;

static void mt_seed(mt19937_t* g, uint32_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 624; ++i) g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
  g->idx = 624;
}

static uint32_t mt_next(mt19937_t* g) {
  if (g->idx >= 624) {
    for (int i = 0; i < 624; ++i) {
      uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
      g->mt[i] = g->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    }
    g->idx = 0;
  }
  uint32_t y = g->mt[g->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

/* rng.hpp:15-25: Rng(seed) then n draws of uniform() (pm1 = 0) or
 * uniform_pm1() (pm1 = 1), as float. */
void or_rng_uniform(uint64_t seed, int64_t n, int pm1, float* out) {
  mt19937_t g;
  mt_seed(&g, (uint32_t)(seed ^ (seed >> 32)));
  for (int64_t i = 0; i < n; ++i) {
    float u = (float)(mt_next(&g) >> 8) * 0x1.0p-24f;
    out[i] = pm1 ? 2.0f * u - 1.0f : u;
  }
}

/* ---------------------------------------------------------------- half */

/* half.hpp:12-37 */
float or_half_to_float(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1Fu;
  uint32_t mant = h & 0x3FFu;
  uint32_t bits;
  if (exp == 0) {
    if (mant == 0) {
      bits = sign;
    } else {
      int shift = 0;
      while (!(mant & 0x400u)) {
        mant <<= 1;
        ++shift;
      }
      mant &= 0x3FFu;
      bits = sign | (uint32_t)(113 - shift) << 23 | mant << 13;
    }
  } else if (exp == 31) {
    bits = sign | 0x7F800000u | mant << 13;
  } else {
    bits = sign | (exp + 112) << 23 | mant << 13;
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

/* half.hpp:39-62 */
uint16_t or_float_to_half(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  uint32_t fexp = (x >> 23) & 0xFFu;
  uint32_t mant = x & 0x7FFFFFu;
  if (fexp == 0xFF) {
    uint16_t payload = mant ? (uint16_t)(0x200u | (mant >> 13)) : 0;
    return (uint16_t)(sign | 0x7C00u | payload);
  }
  int exp = (int)fexp - 127 + 15;
  if (exp >= 31) return (uint16_t)(sign | 0x7C00u);
  if (exp <= 0) {
    if (exp < -10) return sign;
    mant |= 0x800000u;
    uint32_t shift = (uint32_t)(14 - exp);
    uint32_t q = mant >> shift;
    uint32_t rem = mant & ((1u << shift) - 1);
    uint32_t halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (q & 1))) ++q;
    return (uint16_t)(sign | q);
  }
  uint16_t h = (uint16_t)(sign | (uint32_t)exp << 10 | (mant >> 13));
  uint32_t rem = mant & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1))) ++h;
  return h;
}

void or_float_to_half_array(int64_t n, const float* in, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = or_float_to_half(in[i]);
}

void or_half_to_float_array(int64_t n, const uint16_t* in, float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = or_half_to_float(in[i]);
}
