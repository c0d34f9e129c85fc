// Alpha-shearlet frame as full-grid Fourier multipliers (host, fp64) — the
// restatement of the reference's make_plan (shearlet.cpp:18-198, §8f rank 3):
// cone-adapted real-valued windows (Meyer-type radial bands x directional
// bumps), exact evenness under frequency negation, joint Parseval
// normalisation.  The device applies them with the 2-D FFT kernels of
// shearlet.cu (upload_shearlet builds the device tables there).
#include <algorithm>
#include <cmath>

#include "rk_internal.hpp"

namespace rk {

namespace {

// Meyer auxiliary polynomial v(t) + v(1 - t) = 1 (shearlet.cpp:21-25)
double meyer_v(double t) {
  if (t <= 0.0) return 0.0;
  if (t >= 1.0) return 1.0;
  return t * t * t * t * (35.0 - 84.0 * t + (70.0 - 20.0 * t) * t * t);
}
double rise(double t) { return std::sin(0.5 * M_PI * meyer_v(t)); }
double fall(double t) { return std::cos(0.5 * M_PI * meyer_v(t)); }
// directional bump with g(t)^2 + g(t-1)^2 = 1 on [0, 1] (shearlet.cpp:32-36)
double bump(double t) {
  const double a = std::abs(t);
  if (a >= 1.0) return 0.0;
  return std::cos(0.5 * M_PI * meyer_v(a));
}
double lowpass(double r, double c0) {  // shearlet.cpp:38-42
  if (r <= c0) return 1.0;
  if (r >= 2.0 * c0) return 0.0;
  return fall(r / c0 - 1.0);
}
// radial band rising on [c, 2c], falling on [2c, 4c]; the top scale stays 1
// past its peak so the grid corners are covered (shearlet.cpp:44-53)
double band(double r, double c, bool top) {
  if (r <= c) return 0.0;
  if (r < 2.0 * c) return rise(r / c - 1.0);
  if (top) return 1.0;
  if (r < 4.0 * c) return fall(r / (2.0 * c) - 1.0);
  return 0.0;
}

}  // namespace

void build_shearlet(Shearlet& sp, int64_t height, int64_t width, const std::vector<double>& alphas,
                    const double* stored) {
  // shearlet.cpp:68-80
  if (height != width)
    throw ValidationError("shearlet plan requires a square grid, got " + std::to_string(height) + "x" +
                          std::to_string(width));
  if (height < 2) throw ValidationError("shearlet plan grid must be at least 2x2");
  if (alphas.empty() || alphas.size() > 8)
    throw ValidationError("shearlet plan needs between 1 and 8 scales, got " + std::to_string(alphas.size()));
  for (double a : alphas)
    if (!(a >= 0.0 && a <= 1.0)) throw ValidationError("shearlet alpha " + std::to_string(a) + " is outside [0, 1]");
  if (sp.device >= 0 && height > 8192)
    throw ValidationError("the device shearlet transform supports grids up to 8192, got " + std::to_string(height));
  const int64_t h = height, w = width, J = int64_t(alphas.size());
  sp.height = h;
  sp.width = w;
  sp.alphas = alphas;
  // shear counts K_j = ceil(2^(j (1 - alpha_j))), n_coeff = 1 + sum 2 (2 K_j + 1) (shearlet.cpp:55-66)
  std::vector<int64_t> K(static_cast<size_t>(J));
  for (int64_t j = 0; j < J; ++j) K[size_t(j)] = int64_t(std::ceil(std::exp2(double(j) * (1.0 - alphas[size_t(j)]))));
  sp.n_coeff = 1;
  for (int64_t kj : K) sp.n_coeff += 2 * (2 * kj + 1);
  sp.scales.assign(1, 0.0);
  for (int64_t j = 0; j < J; ++j)
    for (int64_t i = 0; i < 2 * (2 * K[size_t(j)] + 1); ++i) sp.scales.push_back(double(j + 1));

  const int64_t bins = h * w;
  std::vector<double>& mult = sp.multipliers;
  if (stored) {  // make_plan_cached's stored multipliers (shearlet.cpp:224-237)
    mult.assign(stored, stored + sp.n_coeff * bins);
    upload_shearlet(sp);
    return;
  }
  const double R = double(h) / 2.0;
  std::vector<double> c(static_cast<size_t>(J));
  for (int64_t j = 0; j < J; ++j) c[size_t(j)] = R * std::exp2(double(j - J));
  std::vector<double> fy(static_cast<size_t>(h)), fx(static_cast<size_t>(w));
  for (int64_t i = 0; i < h; ++i) fy[size_t(i)] = double(i < (h + 1) / 2 ? i : i - h);
  for (int64_t j = 0; j < w; ++j) fx[size_t(j)] = double(j < (w + 1) / 2 ? j : j - w);

  struct Window {
    int64_t scale;  // -1: low-pass
    bool horizontal;
    int64_t shear;
  };
  std::vector<Window> layout{{-1, false, 0}};
  for (int64_t j = 0; j < J; ++j) {
    for (int64_t l = -K[size_t(j)]; l <= K[size_t(j)]; ++l) layout.push_back({j, true, l});
    for (int64_t l = -K[size_t(j)]; l <= K[size_t(j)]; ++l) layout.push_back({j, false, l});
  }
  mult.assign(size_t(sp.n_coeff * bins), 0.0);
  for (int64_t k = 0; k < sp.n_coeff; ++k) {
    const Window& win = layout[size_t(k)];
    double* dst = mult.data() + k * bins;
    for (int64_t i = 0; i < h; ++i)
      for (int64_t j = 0; j < w; ++j) {
        const double r = std::hypot(fx[size_t(j)], fy[size_t(i)]);
        double v;
        if (win.scale < 0) {
          v = lowpass(r, c[0]);
        } else {
          const double radial = band(r, c[size_t(win.scale)], win.scale == J - 1);
          double ang = 0.0;
          if (radial != 0.0) {
            const double kr = double(K[size_t(win.scale)]);
            if (win.horizontal) {
              if (fx[size_t(j)] != 0.0) ang = bump(kr * (fy[size_t(i)] / fx[size_t(j)]) - double(win.shear));
            } else {
              if (fy[size_t(i)] != 0.0) ang = bump(kr * (fx[size_t(j)] / fy[size_t(i)]) - double(win.shear));
            }
          }
          v = radial * ang;
        }
        dst[i * w + j] = v;
      }
    // exact evenness under frequency negation (shearlet.cpp:160-171)
    for (int64_t i = 0; i < h; ++i) {
      const int64_t i2 = (h - i) % h;
      for (int64_t j = 0; j < w; ++j) {
        const int64_t j2 = (w - j) % w;
        if (i2 * w + j2 <= i * w + j) continue;
        const double m = 0.5 * (dst[i * w + j] + dst[i2 * w + j2]);
        dst[i * w + j] = m;
        dst[i2 * w + j2] = m;
      }
    }
  }
  // joint Parseval normalisation (shearlet.cpp:175-191)
  std::vector<double> ssum(static_cast<size_t>(bins), 0.0);
  for (int64_t k = 0; k < sp.n_coeff; ++k)
    for (int64_t b = 0; b < bins; ++b) ssum[size_t(b)] += mult[size_t(k * bins + b)] * mult[size_t(k * bins + b)];
  for (int64_t b = 0; b < bins; ++b) {
    if (!(ssum[size_t(b)] > 1e-8))
      throw NumericalError("shearlet construction left frequency bin " + std::to_string(b) + " uncovered");
    ssum[size_t(b)] = 1.0 / std::sqrt(ssum[size_t(b)]);
  }
  for (int64_t k = 0; k < sp.n_coeff; ++k)
    for (int64_t b = 0; b < bins; ++b) mult[size_t(k * bins + b)] *= ssum[size_t(b)];
  upload_shearlet(sp);
}

}  // namespace rk
