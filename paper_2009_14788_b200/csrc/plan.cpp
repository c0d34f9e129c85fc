// Host side of the B200 Radon projector: geometry resolution/validation, the
// fp64 per-ray and per-angle tables the kernels consume, and the ramp filter
// response.  Compiled with -ffp-contract=off so every fp64 expression below
// is evaluated exactly as written — the same expressions, in the same order,
// as the reference (cited per function), which keeps the discontinuous
// sample count n = max(1, ceil(len/step)) identical on every ray (SURVEY
// appendix A.2).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <complex>
#include <cstring>
#include <limits>
#include <mutex>

#include "rk_internal.hpp"

namespace rk {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void DeviceBuffer::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

void DeviceBuffer::reserve(size_t n) {
  if (n <= bytes) return;
  release();
  RK_CUDA(cudaMalloc(&ptr, n));
  bytes = n;
}

Plan::~Plan() {
  if (scratch_free) cudaEventDestroy(scratch_free);
}

Shearlet::~Shearlet() {
  if (scratch_free) cudaEventDestroy(scratch_free);
}

HostPipeline::~HostPipeline() {
  for (auto& s : streams)
    if (s) cudaStreamDestroy(s);
}

void HostPipeline::synchronize() {
  for (auto s : streams)
    if (s) cudaStreamSynchronize(s);
  cudaGetLastError();
}

size_t dtype_size(int dtype) {
  switch (dtype) {
    case RK_F16: return 2;
    case RK_F32: return 4;
    case RK_F64: return 8;
  }
  throw ValidationError("unknown dtype " + std::to_string(dtype) + " (expected RK_F16, RK_F32 or RK_F64)");
}

// ----------------------------------------------------------------- geometry
// geometry.cpp:12-19 (check_common), :22-33 (make_parallel), :35-55 (make_fanbeam)
rk_geometry resolve_geometry(const rk_geometry& in) {
  if (in.image_size < 1) throw ValidationError("image_size must be >= 1, got " + std::to_string(in.image_size));
  if (in.n_angles < 1 || in.angles == nullptr) throw ValidationError("angle list must not be empty");
  for (int64_t a = 0; a < in.n_angles; ++a)
    if (!std::isfinite(in.angles[a])) throw ValidationError("angles must be finite");
  rk_geometry g = in;
  g.has = RK_HAS_DET_COUNT | RK_HAS_DET_SPACING | RK_HAS_DET_DISTANCE;
  g.det_count = (in.has & RK_HAS_DET_COUNT) ? in.det_count : in.image_size;
  if (in.kind == RK_PARALLEL) {
    g.det_spacing = (in.has & RK_HAS_DET_SPACING) ? in.det_spacing : 1.0;
    if (g.det_count < 1) throw ValidationError("det_count must be >= 1, got " + std::to_string(g.det_count));
    if (!(g.det_spacing > 0.0)) throw ValidationError("det_spacing must be positive");
    g.source_distance = 0.0;
    g.det_distance = 0.0;
  } else if (in.kind == RK_FANBEAM) {
    double rmin = double(in.image_size) * std::sqrt(2.0) / 2.0;
    if (!(in.source_distance > rmin))
      throw ValidationError("source_distance " + std::to_string(in.source_distance) +
                            " must exceed image_size/sqrt(2) = " + std::to_string(rmin) +
                            " so the source stays outside the image");
    g.det_distance = (in.has & RK_HAS_DET_DISTANCE) ? in.det_distance : in.source_distance;
    if (!(g.det_distance > 0.0)) throw ValidationError("det_distance must be positive");
    if (g.det_count < 1) throw ValidationError("det_count must be >= 1, got " + std::to_string(g.det_count));
    double magnification = (g.source_distance + g.det_distance) / g.source_distance;
    g.det_spacing = (in.has & RK_HAS_DET_SPACING) ? in.det_spacing
                                                  : magnification * double(in.image_size) / double(g.det_count);
    if (!(g.det_spacing > 0.0)) throw ValidationError("det_spacing must be positive");
  } else {
    throw ValidationError("unknown geometry kind " + std::to_string(in.kind));
  }
  return g;
}

namespace {

// projector.cpp:37-45
inline bool clip_slab(double o, double d, double lo, double hi, double& t0, double& t1) {
  if (d == 0.0) return o >= lo && o <= hi;
  double a = (lo - o) / d;
  double b = (hi - o) / d;
  if (a > b) std::swap(a, b);
  t0 = std::max(t0, a);
  t1 = std::min(t1, b);
  return true;
}

// The clip / sample-count / spacing prologue of integrate_ray
// (projector.cpp:66-78), kept in fp64 for the planners.
RayD setup_ray(int64_t s, double ox, double oy, double dx, double dy, double tmin, double tmax, double step) {
  RayD r{ox, oy, dx, dy, 0.0, 0.0, 0.0, 0};
  double half = 0.5 * double(s);
  double t0 = tmin, t1 = tmax;
  bool hit = clip_slab(ox, dx, -half, half, t0, t1) && clip_slab(oy, dy, -half, half, t0, t1) && (t1 > t0);
  if (!hit) return r;
  double len = t1 - t0;
  r.n = std::max<int64_t>(1, int64_t(std::ceil(len / step)));
  r.h = len / double(r.n);
  r.t0 = t0;
  r.t1 = t1;
  return r;
}

// forward_parallel_t / forward_fanbeam_t ray setup (projector.cpp:95-139), fp64.
std::vector<RayD> compute_rays(const Plan& p, const std::vector<double2>& trig, int64_t* total_samples) {
  const rk_geometry& g = p.g;
  const int64_t s = p.s, na = p.na, nd = p.nd;
  const bool fan = g.kind == RK_FANBEAM;
  std::vector<RayD> rays(static_cast<size_t>(na * nd));
  const double inf = std::numeric_limits<double>::infinity();
  int64_t total = 0;
  for (int64_t a = 0; a < na; ++a) {
    double c = trig[size_t(a)].x, sn = trig[size_t(a)].y;
    double sx = g.source_distance * sn;  // projector.cpp:123-124
    double sy = -g.source_distance * c;
    for (int64_t k = 0; k < nd; ++k) {
      double u = (double(k) - 0.5 * double(nd) + 0.5) * g.det_spacing;
      RayD r;
      if (!fan) {
        // projector.cpp:107-109: origin u*(c, s), direction (-s, c), t unbounded
        r = setup_ray(s, u * c, u * sn, -sn, c, -inf, inf, g.step);
      } else {
        // projector.cpp:128-135: source -> detector cell, t in [0, len]
        double px = u * c - g.det_distance * sn;
        double py = u * sn + g.det_distance * c;
        double dx = px - sx, dy = py - sy;
        double len = std::sqrt(dx * dx + dy * dy);
        r = setup_ray(s, sx, sy, dx / len, dy / len, 0.0, len, g.step);
      }
      if (r.n > (int64_t(1) << 30)) throw ValidationError("projector step too small: ray sample count overflows");
      rays[size_t(a * nd + k)] = r;
      total += r.n;
    }
  }
  if (total_samples) *total_samples = total;
  return rays;
}

std::vector<double2> angle_trig(const Plan& p) {  // projector.cpp:89-93
  std::vector<double2> trig(static_cast<size_t>(p.na));
  for (int64_t a = 0; a < p.na; ++a)
    trig[size_t(a)] = make_double2(std::cos(p.angles[size_t(a)]), std::sin(p.angles[size_t(a)]));
  return trig;
}

}  // namespace

// The forward schedule (fwd_plan.cpp) and per-ray records, built and uploaded
// once, on the first forward projection through the plan.
void ensure_forward_schedule(Plan& p) {
  if (p.device < 0) return;  // host-only plans schedule eagerly and never launch
  std::call_once(p.fwd_once, [&] {
    std::vector<RayD> rays = compute_rays(p, angle_trig(p), nullptr);
    std::vector<float4> rg, ra;
    build_forward_plan(p, rays, rg, ra);
    rk::set_device(p.device);
    p.ray_geom.reserve(rg.size() * sizeof(float4));
    p.ray_aux.reserve(ra.size() * sizeof(float4));
    RK_CUDA(cudaMemcpy(p.ray_geom.ptr, rg.data(), rg.size() * sizeof(float4), cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(p.ray_aux.ptr, ra.data(), ra.size() * sizeof(float4), cudaMemcpyHostToDevice));
    p.fwd_boxes.reserve(p.fwd.boxes.size() * sizeof(int4));
    p.fwd_cta.reserve(p.fwd.cta.size() * sizeof(int4));
    RK_CUDA(cudaMemcpy(p.fwd_boxes.ptr, p.fwd.boxes.data(), p.fwd.boxes.size() * sizeof(int4),
                       cudaMemcpyHostToDevice));
    RK_CUDA(cudaMemcpy(p.fwd_cta.ptr, p.fwd.cta.data(), p.fwd.cta.size() * sizeof(int4), cudaMemcpyHostToDevice));
    p.fwd_warps.reserve(p.fwd.warps.size() * sizeof(int2));
    RK_CUDA(cudaMemcpy(p.fwd_warps.ptr, p.fwd.warps.data(), p.fwd.warps.size() * sizeof(int2),
                       cudaMemcpyHostToDevice));
  });
}

// Tile geometry of the backprojection kernel (kernels.cu): 32 x 32 pixels.
constexpr int kBpTile = 32;

void build_plan(Plan& p) {
  const rk_geometry& g = p.g;
  p.s = g.image_size;
  p.na = g.n_angles;
  p.nd = g.det_count;
  if (!(g.step > 0.0)) throw ValidationError("projector step must be positive");  // projector.cpp:31-33
  if (p.s > 32768) throw ValidationError("image_size " + std::to_string(p.s) + " exceeds the supported 32768");
  if (p.na * p.nd > (int64_t(1) << 31)) throw ValidationError("n_angles * det_count exceeds 2^31 rays");

  const int64_t s = p.s, na = p.na, nd = p.nd;
  const bool fan = g.kind == RK_FANBEAM;

  const std::vector<double2> trig = angle_trig(p);

  // ----- forward ray table (exact per-image work); the forward schedule is
  // built on the first forward call (ensure_forward_schedule): FBP-only and
  // backprojection-only users never pay for its planning
  int64_t total = 0;
  std::vector<RayD> rays = compute_rays(p, trig, &total);
  p.forward_samples = total;
  if (p.device < 0) {  // host-only plan (inspection): schedule now
    std::vector<float4> rg, ra;
    build_forward_plan(p, rays, rg, ra);
  }
  rays.clear();
  rays.shrink_to_fit();
  const double inf = std::numeric_limits<double>::infinity();

  // ----- backprojection staging window: the widest detector footprint of a
  // 32x32 pixel tile over all tiles and angles (+ one cell on each side for
  // the second tap and rounding).  kf as in projector.cpp:153-154 / 186-188.
  const double half = 0.5 * double(s);
  const double off = 0.5 * double(nd) - 0.5;
  const double span = g.source_distance + g.det_distance;
  int64_t tiles = (s + kBpTile - 1) / kBpTile;
  // per tile: the widest footprint over all angles (fan beam: tiles far from
  // the source need far fewer cells than the ones next to it)
  std::vector<int64_t> tile_need(size_t(tiles * tiles), 0);
  for (int64_t a = 0; a < na; ++a) {
    double c = trig[size_t(a)].x, sn = trig[size_t(a)].y;
    for (int64_t ty = 0; ty < tiles; ++ty) {
      for (int64_t tx = 0; tx < tiles; ++tx) {
        // in-image part of the tile (kernels.cu uses the same extent)
        double x0 = double(tx * kBpTile) - half + 0.5, x1 = x0 + double(std::min<int64_t>(kBpTile, s - tx * kBpTile) - 1);
        double y0 = half - double(ty * kBpTile) - 0.5, y1 = y0 - double(std::min<int64_t>(kBpTile, s - ty * kBpTile) - 1);
        double lo = inf, hi = -inf;
        for (double x : {x0, x1})
          for (double y : {y0, y1}) {
            double kf;
            if (!fan) {
              kf = (x * c + y * sn) / g.det_spacing + off;
            } else {
              double qx = x * c + y * sn, qy = -x * sn + y * c;
              kf = (qx * span / (qy + g.source_distance)) / g.det_spacing + off;
            }
            lo = std::min(lo, kf);
            hi = std::max(hi, kf);
          }
        // window [floor(lo) - 1, floor(hi) + 2] clipped to [-2, nd + 1]: beyond
        // that every tap is outside the detector (zero), and the kernel's
        // clamp lands on the two zero cells at the clipped end
        int64_t ws = std::max<int64_t>(int64_t(std::floor(lo)) - 1, -2);
        int64_t we = std::min<int64_t>(int64_t(std::floor(hi)) + 2, nd + 1);
        int64_t& tn = tile_need[size_t(ty * tiles + tx)];
        tn = std::max(tn, we - ws + 1);
      }
      // every tile row, also for parallel beam: the unclipped footprint width is translation
      // invariant, but the clip to [-2, nd + 1] is not — with a detector narrower than the
      // image the first tile row can be clipped where another row is not (r2 stress sweep)
    }
  }
  int64_t need = 0;
  for (int64_t t = 0; t < tiles * tiles; ++t) need = std::max(need, tile_need[size_t(t)]);
  // + floor effects across tiles (parallel) + a rounding margin (the kernel
  // derives each angle's window start in its own fp64 arithmetic)
  auto padded_window = [&](int64_t n) { return (n + (fan ? 1 : 2) + 3) / 4 * 4; };
  int64_t window = padded_window(need);
  if (window > 12 * 1024)
    throw ValidationError("backprojection window of " + std::to_string(window) +
                          " detector cells exceeds shared memory (det_count too large)");
  p.bp_window = int(window);
  std::vector<int> tile_window(size_t(tiles * tiles));
  for (int64_t t = 0; t < tiles * tiles; ++t)
    tile_window[size_t(t)] = int(fan ? padded_window(tile_need[size_t(t)]) : window);
  // fp32 (tile-relative) fan map unless the magnification span / (sp (D_so - R))
  // of the pixels nearest the source is large (kernels.cu, kBpFan32 / kBpFan64)
  if (fan) {
    const double rmax = half * std::sqrt(2.0);
    const double mag = span / (g.det_spacing * (g.source_distance - rmax));
    static const double max_mag = [] {
      const char* e = std::getenv("RK_BP_FAN32_MAXMAG");
      return e ? std::atof(e) : 3.5;
    }();
    p.bp_fan_fp64 = !(mag <= max_mag);
  }
  // angles per staging pass: keep the window slab near 32 KB (>= 1 angle, up to
  // 192 KB) for the widest tile; narrower tiles stage more angles per pass in
  // the same cells (kernels.cu: chunk = min(32, cells / tile window)).  The
  // NARROW kernel (128 threads, register-bound at seven CTAs per SM) gets a
  // 30 KB slab: with the 32 constant records and the 1 KB the runtime reserves
  // per CTA, seven then fit an SM's 228 KB (cfg3's fan windows left six at
  // 32 KB: fan backprojection 4.36 -> 4.32 ms); the 512-thread kernels (two
  // CTAs per SM) keep more angles per pass.
  auto slab_chunk = [&](int64_t bytes) { return std::max<int64_t>(1, std::min<int64_t>(32, bytes / (window * 16))); };
  static const int64_t narrow_slab = [] {
    const char* e = std::getenv("RK_BP_WINDOW_BYTES");
    return e ? std::max<int64_t>(1024, std::atoll(e)) : int64_t(30 * 1024);
  }();
  const int64_t chunk = slab_chunk(32 * 1024);
  p.bp_angle_chunk = int(chunk);
  p.bp_cells = int(chunk * window);
  p.bp_cells_narrow = int(slab_chunk(narrow_slab) * window);

  // ----- upload (device < 0: host-only plan, used for inspection on machines without a GPU)
  if (p.device < 0) return;
  rk::set_device(p.device);
  p.trig.reserve(trig.size() * sizeof(double2));
  RK_CUDA(cudaMemcpy(p.trig.ptr, trig.data(), trig.size() * sizeof(double2), cudaMemcpyHostToDevice));
  p.bp_tile_window.reserve(tile_window.size() * sizeof(int));
  RK_CUDA(cudaMemcpy(p.bp_tile_window.ptr, tile_window.data(), tile_window.size() * sizeof(int),
                     cudaMemcpyHostToDevice));
  RK_CUDA(cudaEventCreateWithFlags(&p.scratch_free, cudaEventDisableTiming));
}

// ----------------------------------------------------------------- filter
const char* filter_kind_name(int kind) {  // sino_filter.cpp:24-33
  switch (kind) {
    case RK_RAM_LAK: return "ram-lak";
    case RK_SHEPP_LOGAN: return "shepp-logan";
    case RK_COSINE: return "cosine";
    case RK_HAMMING: return "hamming";
    case RK_HANN: return "hann";
  }
  return "?";
}

int filter_kind_from_name(const std::string& name) {  // sino_filter.cpp:14-22
  for (int k = RK_RAM_LAK; k <= RK_HANN; ++k)
    if (name == filter_kind_name(k)) return k;
  throw ValidationError("unknown filter '" + name + "' (expected ram-lak, shepp-logan, cosine, hamming, or hann)");
}

namespace {

// sino_filter.cpp:43-60
double window_gain(int kind, double nu) {
  switch (kind) {
    case RK_SHEPP_LOGAN: {
      if (nu == 0.0) return 1.0;
      double t = 0.5 * M_PI * nu;
      return std::sin(t) / t;
    }
    case RK_COSINE: return std::cos(0.5 * M_PI * nu);
    case RK_HAMMING: return 0.54 + 0.46 * std::cos(M_PI * nu);
    case RK_HANN: return 0.5 + 0.5 * std::cos(M_PI * nu);
    default: return 1.0;
  }
}

// Real-input FFT in fp64 (the make_filter call of fft::rfft, sino_filter.cpp:81):
// iterative radix-2 decimation in time, twiddles cos/sin((2 pi k)/n).  n is
// always a power of two here (sino_filter.cpp:69).
void rfft_pow2(const std::vector<double>& x, std::vector<std::complex<double>>& out) {
  size_t n = x.size();
  std::vector<std::complex<double>> a(n);
  for (size_t i = 0; i < n; ++i) a[i] = {x[i], 0.0};
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    size_t h = len / 2, stride = n / len;
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < h; ++k) {
        double ang = 2.0 * M_PI * double(k * stride) / double(n);
        std::complex<double> w(std::cos(ang), -std::sin(ang));
        std::complex<double> u = a[i + k];
        std::complex<double> xv = a[i + k + h];
        std::complex<double> v(xv.real() * w.real() - xv.imag() * w.imag(), xv.real() * w.imag() + xv.imag() * w.real());
        a[i + k] = {u.real() + v.real(), u.imag() + v.imag()};
        a[i + k + h] = {u.real() - v.real(), u.imag() - v.imag()};
      }
  }
  out.assign(a.begin(), a.begin() + ptrdiff_t(n / 2 + 1));
}

}  // namespace

// sino_filter.cpp:64-92
void build_filter(Filter& f, int kind, int64_t det_count) {
  if (kind < RK_RAM_LAK || kind > RK_HANN) throw ValidationError("unknown filter kind " + std::to_string(kind));
  if (det_count < 2) throw ValidationError("det_count must be >= 2, got " + std::to_string(det_count));
  int64_t n = 1;
  while (n < 2 * det_count) n <<= 1;
  n = std::max<int64_t>(n, 2);
  if (n > 32768)
    throw ValidationError("det_count " + std::to_string(det_count) + " pads to " + std::to_string(n) +
                          " > 32768, beyond the two-CTA shared-memory FFT of the filter kernel");
  f.kind = kind;
  f.det_count = det_count;
  f.padded = n;
  std::vector<double> kernel(size_t(n), 0.0);
  kernel[0] = 0.25;
  for (int64_t p = 1; p < n; ++p) {
    int64_t m = std::min(p, n - p);
    if (m % 2 == 1) kernel[size_t(p)] = -1.0 / (double(m) * double(m) * M_PI * M_PI);
  }
  std::vector<std::complex<double>> bins;
  rfft_pow2(kernel, bins);
  f.response.resize(size_t(n / 2 + 1));
  f.response_f.resize(size_t(n / 2 + 1));
  for (int64_t q = 0; q <= n / 2; ++q) {
    double nu = double(q) / double(n / 2);
    double v = 2.0 * bins[size_t(q)].real() * window_gain(kind, nu);
    f.response[size_t(q)] = v;
    f.response_f[size_t(q)] = float(v);
  }
  // forward twiddles exp(-2 pi i k / n), k < n/2, evaluated in fp64 and rounded
  std::vector<float2> tw(static_cast<size_t>(std::max<int64_t>(n / 2, 1)));
  for (int64_t k = 0; k < n / 2; ++k) {
    double ang = 2.0 * M_PI * double(k) / double(n);
    tw[size_t(k)] = make_float2(float(std::cos(ang)), float(-std::sin(ang)));
  }
  // the same twiddles regrouped per radix-2 stage s (offset 2^s - 1, 2^s entries: W^(k n / 2^(s+1))),
  // so a stage's butterflies read consecutive entries (filter.cu) instead of a strided gather
  int logn = 0;
  while ((int64_t(1) << logn) < n) ++logn;
  std::vector<float2> tws(static_cast<size_t>(std::max<int64_t>(n - 1, 1)));
  for (int st = 0; st < logn; ++st)
    for (int64_t k = 0; k < (int64_t(1) << st); ++k)
      tws[size_t((int64_t(1) << st) - 1 + k)] = tw[size_t(k << (logn - 1 - st))];
  if (f.device < 0) return;  // host-only filter (response inspection without a GPU)
  rk::set_device(f.device);
  f.d_twiddle_stage.reserve(tws.size() * sizeof(float2));
  RK_CUDA(cudaMemcpy(f.d_twiddle_stage.ptr, tws.data(), tws.size() * sizeof(float2), cudaMemcpyHostToDevice));
  f.d_response.reserve(f.response_f.size() * sizeof(float));
  f.d_twiddle.reserve(tw.size() * sizeof(float2));
  RK_CUDA(cudaMemcpy(f.d_response.ptr, f.response_f.data(), f.response_f.size() * sizeof(float),
                     cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(f.d_twiddle.ptr, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice));
}

}  // namespace rk
