// radonkit_b200.hpp — header-only C++ drop-in layer over the C ABI
// (radon_b200.h), mirroring the reference's C++ operator API
// (/root/reference/proj/core/include/radonkit/{geometry,projector,
// sino_filter,linop,solvers}.hpp) for code that holds its data in host
// vectors or device buffers.
//
//   radonkit::make_parallel / make_fanbeam / angles_linspace  -> rkb::make_parallel / ...
//   radonkit::forward / backprojection (host Tensor in/out)   -> rkb::forward / rkb::backprojection
//   radonkit::make_filter / filter_sinogram / fbp             -> rkb::make_filter / ...
//   radonkit::projector_operator -> LinearOperator            -> rkb::projector_operator
//   radonkit::ValidationError / NumericalError                -> rkb::ValidationError / ...
//
// Host calls are synchronous and return freshly allocated results, exactly
// like the reference's Tensor-returning functions; the *_device calls take
// device pointers and a cudaStream_t and are asynchronous.  Plans (device
// geometry tables) are cached per geometry + step + device.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <variant>
#include <vector>

#include "radon_b200.h"

namespace rkb {

// ------------------------------------------------------------------ errors (errors.hpp:9-40)
struct ValidationError : std::invalid_argument {
  explicit ValidationError(const std::string& w) : std::invalid_argument(w) {}
};
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w, long it = -1) : std::runtime_error(w), iteration(it) {}
  long iteration;
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int status, long iteration = -1) {
  if (status == RK_OK) return;
  std::string msg = rk_last_error();
  if (status == RK_ERR_VALIDATION) throw ValidationError(msg);
  if (status == RK_ERR_NUMERICAL) throw NumericalError(msg, iteration);
  throw CudaError(msg);
}

// ------------------------------------------------------------------ precision
enum class Precision { Half = RK_F16, Single = RK_F32, Double = RK_F64 };
template <class T> struct precision_of;
template <> struct precision_of<uint16_t> { static constexpr Precision value = Precision::Half; };  // binary16 bits
template <> struct precision_of<float> { static constexpr Precision value = Precision::Single; };
template <> struct precision_of<double> { static constexpr Precision value = Precision::Double; };

// ------------------------------------------------------------------ geometry (geometry.hpp:18-56)
struct ParallelGeometry {
  int64_t image_size = 0;
  std::vector<double> angles;
  int64_t det_count = 0;
  double det_spacing = 1.0;
};

struct FanbeamGeometry {
  int64_t image_size = 0;
  std::vector<double> angles;
  double source_distance = 0.0;
  double det_distance = 0.0;
  int64_t det_count = 0;
  double det_spacing = 1.0;
  double magnification() const { return (source_distance + det_distance) / source_distance; }
};

using Geometry = std::variant<ParallelGeometry, FanbeamGeometry>;

struct ProjectorOptions {
  double step = 1.0;
};

inline rk_geometry to_c(const ParallelGeometry& g, double step) {
  rk_geometry c{};
  c.kind = RK_PARALLEL;
  c.has = RK_HAS_DET_COUNT | RK_HAS_DET_SPACING;
  c.image_size = g.image_size;
  c.n_angles = int64_t(g.angles.size());
  c.angles = g.angles.data();
  c.det_count = g.det_count;
  c.det_spacing = g.det_spacing;
  c.step = step;
  return c;
}

inline rk_geometry to_c(const FanbeamGeometry& g, double step) {
  rk_geometry c{};
  c.kind = RK_FANBEAM;
  c.has = RK_HAS_DET_COUNT | RK_HAS_DET_SPACING | RK_HAS_DET_DISTANCE;
  c.image_size = g.image_size;
  c.n_angles = int64_t(g.angles.size());
  c.angles = g.angles.data();
  c.det_count = g.det_count;
  c.det_spacing = g.det_spacing;
  c.source_distance = g.source_distance;
  c.det_distance = g.det_distance;
  c.step = step;
  return c;
}

inline ParallelGeometry make_parallel(int64_t image_size, std::vector<double> angles,
                                      std::optional<int64_t> det_count = std::nullopt,
                                      std::optional<double> det_spacing = std::nullopt) {
  rk_geometry in{};
  in.kind = RK_PARALLEL;
  in.image_size = image_size;
  in.n_angles = int64_t(angles.size());
  in.angles = angles.data();
  if (det_count) in.has |= RK_HAS_DET_COUNT, in.det_count = *det_count;
  if (det_spacing) in.has |= RK_HAS_DET_SPACING, in.det_spacing = *det_spacing;
  in.step = 1.0;
  rk_geometry out{};
  check(rk_geometry_resolve(&in, &out));
  return ParallelGeometry{out.image_size, std::move(angles), out.det_count, out.det_spacing};
}

inline FanbeamGeometry make_fanbeam(int64_t image_size, std::vector<double> angles, double source_distance,
                                    std::optional<double> det_distance = std::nullopt,
                                    std::optional<int64_t> det_count = std::nullopt,
                                    std::optional<double> det_spacing = std::nullopt) {
  rk_geometry in{};
  in.kind = RK_FANBEAM;
  in.image_size = image_size;
  in.n_angles = int64_t(angles.size());
  in.angles = angles.data();
  in.source_distance = source_distance;
  if (det_distance) in.has |= RK_HAS_DET_DISTANCE, in.det_distance = *det_distance;
  if (det_count) in.has |= RK_HAS_DET_COUNT, in.det_count = *det_count;
  if (det_spacing) in.has |= RK_HAS_DET_SPACING, in.det_spacing = *det_spacing;
  in.step = 1.0;
  rk_geometry out{};
  check(rk_geometry_resolve(&in, &out));
  return FanbeamGeometry{out.image_size, std::move(angles), out.source_distance, out.det_distance, out.det_count,
                         out.det_spacing};
}

inline std::vector<double> angles_linspace(double start, double stop, int64_t n) {
  std::vector<double> out(size_t(n > 0 ? n : 1));
  check(rk_angles_linspace(start, stop, n, out.data()));
  out.resize(size_t(n));
  return out;
}

inline int64_t geometry_image_size(const Geometry& g) {
  return std::visit([](const auto& x) { return x.image_size; }, g);
}
inline int64_t geometry_det_count(const Geometry& g) {
  return std::visit([](const auto& x) { return x.det_count; }, g);
}
inline int64_t geometry_n_angles(const Geometry& g) {
  return std::visit([](const auto& x) { return int64_t(x.angles.size()); }, g);
}

// ------------------------------------------------------------------ plans
class Plan {
 public:
  Plan(const Geometry& g, const ProjectorOptions& opts, int device) {
    rk_geometry c = std::visit([&](const auto& x) { return to_c(x, opts.step); }, g);
    rk_plan* p = nullptr;
    check(rk_plan_create(&c, device, &p));
    handle_.reset(p);
  }
  rk_plan* get() const { return handle_.get(); }
  rk_plan_info info() const {
    rk_plan_info i{};
    check(rk_plan_info_get(handle_.get(), &i));
    return i;
  }

 private:
  struct Del {
    void operator()(rk_plan* p) const { rk_plan_destroy(p); }
  };
  std::unique_ptr<rk_plan, Del> handle_;
};

inline std::shared_ptr<Plan> plan_for(const Geometry& g, const ProjectorOptions& opts = {}, int device = 0) {
  static std::mutex mu;
  static std::map<std::tuple<int, int64_t, std::vector<double>, int64_t, double, double, double, double, int>,
                  std::shared_ptr<Plan>>
      cache;
  auto key = std::visit(
      [&](const auto& x) {
        rk_geometry c = to_c(x, opts.step);
        return std::make_tuple(int(c.kind), c.image_size, x.angles, c.det_count, c.det_spacing, c.source_distance,
                               c.det_distance, c.step, device);
      },
      g);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto p = std::make_shared<Plan>(g, opts, device);
  cache.emplace(std::move(key), p);
  return p;
}

// ------------------------------------------------------------------ projector (projector.hpp:19-29)
// image: batch x s x s -> batch x n_angles x det_count, host memory, same element type out.
template <class T>
std::vector<T> forward(const Geometry& g, const std::vector<T>& image, int64_t batch, const ProjectorOptions& opts = {},
                       int device = 0) {
  const int64_t s = geometry_image_size(g);
  if (batch < 1 || int64_t(image.size()) != batch * s * s)
    throw ValidationError("image must hold batch x image_size x image_size elements");
  auto plan = plan_for(g, opts, device);
  std::vector<T> out(size_t(batch * geometry_n_angles(g) * geometry_det_count(g)));
  check(rk_forward_host(plan->get(), int(precision_of<T>::value), image.data(), batch, out.data()));
  return out;
}

template <class T>
std::vector<T> backprojection(const Geometry& g, const std::vector<T>& sino, int64_t batch,
                              const ProjectorOptions& opts = {}, int device = 0) {
  const int64_t s = geometry_image_size(g);
  if (batch < 1 || int64_t(sino.size()) != batch * geometry_n_angles(g) * geometry_det_count(g))
    throw ValidationError("sinogram must hold batch x n_angles x det_count elements");
  auto plan = plan_for(g, opts, device);
  std::vector<T> out(size_t(batch * s * s));
  check(rk_backproject_host(plan->get(), int(precision_of<T>::value), sino.data(), batch, out.data()));
  return out;
}

// device-pointer variants (asynchronous on `stream`)
inline void forward_device(const Geometry& g, Precision p, const void* d_image, int64_t batch, void* d_sino,
                           void* stream = nullptr, const ProjectorOptions& opts = {}, int device = 0) {
  check(rk_forward(plan_for(g, opts, device)->get(), int(p), d_image, batch, d_sino, stream));
}
inline void backprojection_device(const Geometry& g, Precision p, const void* d_sino, int64_t batch, void* d_image,
                                  void* stream = nullptr, const ProjectorOptions& opts = {}, int device = 0) {
  check(rk_backproject(plan_for(g, opts, device)->get(), int(p), d_sino, batch, d_image, stream));
}

// ------------------------------------------------------------------ filter (sino_filter.hpp:12-42)
enum class FilterKind { RamLak = RK_RAM_LAK, SheppLogan = RK_SHEPP_LOGAN, Cosine = RK_COSINE, Hamming = RK_HAMMING,
                        Hann = RK_HANN };

inline FilterKind filter_kind_from_name(const std::string& name) {
  int k = 0;
  check(rk_filter_kind_from_name(name.c_str(), &k));
  return FilterKind(k);
}
inline const char* filter_kind_name(FilterKind k) { return rk_filter_kind_name(int(k)); }

struct FilterSpec {
  FilterKind kind = FilterKind::RamLak;
  int64_t det_count = 0;
  int64_t padded_size = 0;
  std::vector<double> frequency_response;
  std::vector<float> frequency_response_f;
  std::shared_ptr<rk_filter> handle;  // device copy of the response
};

inline FilterSpec make_filter(FilterKind kind, int64_t det_count, int device = 0) {
  rk_filter* f = nullptr;
  check(rk_filter_create(int(kind), det_count, device, &f));
  FilterSpec spec;
  spec.handle.reset(f, [](rk_filter* x) { rk_filter_destroy(x); });
  spec.kind = kind;
  spec.det_count = det_count;
  check(rk_filter_response(f, &spec.padded_size, nullptr, nullptr));
  spec.frequency_response.resize(size_t(spec.padded_size / 2 + 1));
  spec.frequency_response_f.resize(size_t(spec.padded_size / 2 + 1));
  check(rk_filter_response(f, &spec.padded_size, spec.frequency_response.data(), spec.frequency_response_f.data()));
  return spec;
}
inline FilterSpec make_filter(const std::string& kind, int64_t det_count, int device = 0) {
  return make_filter(filter_kind_from_name(kind), det_count, device);
}

template <class T>
std::vector<T> filter_sinogram(const std::vector<T>& sino, int64_t batch, int64_t n_angles, const FilterSpec& f) {
  if (batch < 1 || int64_t(sino.size()) != batch * n_angles * f.det_count)
    throw ValidationError("sinogram must hold batch x n_angles x det_count elements");
  std::vector<T> out(sino.size());
  check(rk_filter_sinogram_host(f.handle.get(), int(precision_of<T>::value), sino.data(), batch, n_angles, out.data()));
  return out;
}

template <class T>
std::vector<T> fbp(const Geometry& g, const std::vector<T>& sino, int64_t batch, FilterKind kind = FilterKind::RamLak,
                   int device = 0) {
  auto plan = plan_for(g, {}, device);
  FilterSpec f = make_filter(kind, geometry_det_count(g), device);
  const int64_t s = geometry_image_size(g);
  if (batch < 1 || int64_t(sino.size()) != batch * geometry_n_angles(g) * geometry_det_count(g))
    throw ValidationError("sinogram must hold batch x n_angles x det_count elements");
  std::vector<T> out(size_t(batch * s * s));
  check(rk_fbp_host(plan->get(), f.handle.get(), int(precision_of<T>::value), sino.data(), batch, out.data()));
  return out;
}

// ------------------------------------------------------------------ linear operator (linop.hpp:14-21)
// Host single-precision vectors; shapes per batch element; batch inferred from the size.
struct LinearOperator {
  std::vector<int64_t> domain_shape;
  std::vector<int64_t> range_shape;
  std::function<std::vector<float>(const std::vector<float>&)> apply;
  std::function<std::vector<float>(const std::vector<float>&)> adjoint;
};

inline LinearOperator projector_operator(const Geometry& g, const ProjectorOptions& opts = {}, int device = 0) {
  const int64_t s = geometry_image_size(g), na = geometry_n_angles(g), nd = geometry_det_count(g);
  LinearOperator op;
  op.domain_shape = {s, s};
  op.range_shape = {na, nd};
  op.apply = [g, opts, device, s](const std::vector<float>& x) {
    return forward(g, x, int64_t(x.size()) / (s * s), opts, device);
  };
  op.adjoint = [g, opts, device, na, nd](const std::vector<float>& y) {
    return backprojection(g, y, int64_t(y.size()) / (na * nd), opts, device);
  };
  return op;
}

}  // namespace rkb
