// ORACLE TEST INFRASTRUCTURE — not product code.
//
// A flat extern "C" face over the UNMODIFIED reference sources
// (/root/reference/proj/core/src/*.cpp, compiled in place by oracle/Makefile
// into oracle/_ref/libradonkit_ref.so) so the Python tests and bench.py's
// reference arm can call the reference's own forward / backprojection /
// filter / fbp / solver code through ctypes.  Nothing here re-implements the
// algorithm; every entry point forwards to the reference function named in
// its comment.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <optional>
#include <string>
#include <vector>

#include "radonkit/admm.hpp"
#include "radonkit/errors.hpp"
#include "radonkit/geometry.hpp"
#include "radonkit/linop.hpp"
#include "radonkit/phantom.hpp"
#include "radonkit/projector.hpp"
#include "radonkit/rng.hpp"
#include "radonkit/shearlet.hpp"
#include "radonkit/sino_filter.hpp"
#include "radonkit/solvers.hpp"
#include "radonkit/tensor.hpp"
#include "radonkit/threading.hpp"

using namespace radonkit;

namespace {

thread_local std::string g_err;

// kind: 0 parallel, 1 fan-beam. Optional fields use sentinels: det_count
// < -1e17 -> nullopt; NaN doubles -> nullopt.
struct RefGeom {
  int32_t kind;
  int32_t pad;
  int64_t image_size;
  int64_t n_angles;
  const double* angles;
  int64_t det_count;
  double det_spacing;
  double source_distance;
  double det_distance;
  double step;
};

constexpr int64_t kNoDet = std::numeric_limits<int64_t>::min();

Geometry build(const RefGeom* g) {
  std::vector<double> angles(g->angles, g->angles + g->n_angles);
  std::optional<int64_t> det = g->det_count == kNoDet ? std::nullopt : std::optional<int64_t>(g->det_count);
  std::optional<double> sp = std::isnan(g->det_spacing) ? std::nullopt : std::optional<double>(g->det_spacing);
  if (g->kind == 0) return make_parallel(g->image_size, std::move(angles), det, sp);  // geometry.cpp:22-33
  std::optional<double> dd = std::isnan(g->det_distance) ? std::nullopt : std::optional<double>(g->det_distance);
  return make_fanbeam(g->image_size, std::move(angles), g->source_distance, dd, det, sp);  // geometry.cpp:35-55
}

Precision prec_of(int p) {
  if (p == 0) return Precision::Half;
  if (p == 1) return Precision::Single;
  return Precision::Double;
}

size_t esize(Precision p) { return p == Precision::Half ? 2 : p == Precision::Single ? 4 : 8; }

Tensor make_tensor(Shape shape, Precision p, const void* data) {
  int64_t n = shape_numel(shape);
  if (p == Precision::Half) {
    std::vector<uint16_t> v(static_cast<size_t>(n));
    std::memcpy(v.data(), data, size_t(n) * 2);
    return Tensor::from_half_bits(std::move(shape), std::move(v));
  }
  if (p == Precision::Single) {
    std::vector<float> v(static_cast<size_t>(n));
    std::memcpy(v.data(), data, size_t(n) * 4);
    return Tensor::from_vec(std::move(shape), std::move(v));
  }
  std::vector<double> v(static_cast<size_t>(n));
  std::memcpy(v.data(), data, size_t(n) * 8);
  return Tensor::from_vec(std::move(shape), std::move(v));
}

void store(const Tensor& t, void* out) {
  size_t n = size_t(t.size());
  switch (t.precision()) {
    case Precision::Half: std::memcpy(out, t.half_bits().data(), n * 2); break;
    case Precision::Single: std::memcpy(out, t.float_data().data(), n * 4); break;
    case Precision::Double: std::memcpy(out, t.double_data().data(), n * 8); break;
  }
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_num_threads(int n) {
  return guard([&] { set_num_threads(n); });  // threading.cpp:24-27
}

int ref_num_threads() { return num_threads(); }

// Resolved geometry after the make_* defaults: det_count, det_spacing, det_distance.
int ref_resolve_geometry(const RefGeom* g, int64_t* det_count, double* det_spacing, double* det_distance) {
  return guard([&] {
    Geometry geo = build(g);
    if (auto* p = std::get_if<ParallelGeometry>(&geo)) {
      *det_count = p->det_count;
      *det_spacing = p->det_spacing;
      *det_distance = 0.0;
    } else {
      auto& f = std::get<FanbeamGeometry>(geo);
      *det_count = f.det_count;
      *det_spacing = f.det_spacing;
      *det_distance = f.det_distance;
    }
  });
}

int ref_angles_linspace(double start, double stop, int64_t n, double* out) {
  return guard([&] {
    std::vector<double> a = angles_linspace(start, stop, n);  // geometry.cpp:67-73
    std::memcpy(out, a.data(), a.size() * 8);
  });
}

// projector.cpp:248 (forward over the Geometry variant)
int ref_forward(const RefGeom* g, int prec, int64_t batch, const void* image, void* sino) {
  return guard([&] {
    Geometry geo = build(g);
    int64_t s = geometry_image_size(geo);
    Tensor img = make_tensor({batch, s, s}, prec_of(prec), image);
    store(forward(geo, img, ProjectorOptions{g->step}), sino);
  });
}

// projector.cpp:272 (backprojection over the Geometry variant)
int ref_backprojection(const RefGeom* g, int prec, int64_t batch, const void* sino, void* image) {
  return guard([&] {
    Geometry geo = build(g);
    Tensor sg = make_tensor({batch, geometry_n_angles(geo), geometry_det_count(geo)}, prec_of(prec), sino);
    store(backprojection(geo, sg, ProjectorOptions{g->step}), image);
  });
}

// sino_filter.cpp:64-92; resp_d/resp_f receive padded/2+1 bins
int ref_make_filter(int kind, int64_t det_count, int64_t* padded, double* resp_d, float* resp_f) {
  return guard([&] {
    FilterSpec f = make_filter(FilterKind(kind), det_count);
    *padded = f.padded_size;
    if (resp_d) std::memcpy(resp_d, f.frequency_response.data(), f.frequency_response.size() * 8);
    if (resp_f) std::memcpy(resp_f, f.frequency_response_f.data(), f.frequency_response_f.size() * 4);
  });
}

int ref_filter_kind_from_name(const char* name, int* kind) {
  return guard([&] { *kind = int(filter_kind_from_name(name)); });  // sino_filter.cpp:14-22
}

// sino_filter.cpp:98-124
int ref_filter_sinogram(int kind, int prec, int64_t batch, int64_t n_angles, int64_t det_count, const void* in,
                        void* out) {
  return guard([&] {
    FilterSpec f = make_filter(FilterKind(kind), det_count);
    Tensor sg = make_tensor({batch, n_angles, det_count}, prec_of(prec), in);
    store(filter_sinogram(sg, f), out);
  });
}

// sino_filter.cpp:134-136
int ref_fbp(const RefGeom* g, int kind, int prec, int64_t batch, const void* sino, void* image) {
  return guard([&] {
    Geometry geo = build(g);
    Tensor sg = make_tensor({batch, geometry_n_angles(geo), geometry_det_count(geo)}, prec_of(prec), sino);
    store(fbp(geo, sg, FilterKind(kind)), image);
  });
}

// phantom.cpp:61-101
int ref_shepp_logan(int64_t size, int prec, void* out) {
  return guard([&] { store(shepp_logan(size, prec_of(prec)), out); });
}

// rng.hpp:13-38: n draws of uniform() or uniform_pm1() as float
int ref_rng_uniform(uint64_t seed, int64_t n, int pm1, float* out) {
  return guard([&] {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = pm1 ? r.uniform_pm1() : r.uniform();
  });
}

// linop.cpp:65-80 on projector_operator (linop.cpp:33-41)
int ref_adjoint_check(const RefGeom* g, int trials, uint64_t seed, double* defect) {
  return guard([&] {
    Geometry geo = build(g);
    *defect = adjoint_check(projector_operator(geo, ProjectorOptions{g->step}), trials, seed);
  });
}

// solvers.cpp:111-128
int ref_estimate_alpha(const RefGeom* g, int iterations, uint64_t seed, double* alpha) {
  return guard([&] {
    Geometry geo = build(g);
    *alpha = estimate_alpha(projector_operator(geo, ProjectorOptions{g->step}), iterations, seed);
  });
}

// solvers.cpp:130-145 (y, guess and out share the precision `prec`)
int ref_landweber(const RefGeom* g, int prec, int64_t batch, const void* y, const void* guess, double alpha,
                  int iterations, void* out) {
  return guard([&] {
    Geometry geo = build(g);
    int64_t s = geometry_image_size(geo);
    Tensor yt = make_tensor({batch, geometry_n_angles(geo), geometry_det_count(geo)}, prec_of(prec), y);
    Tensor x0 = make_tensor({batch, s, s}, prec_of(prec), guess);
    store(landweber(projector_operator(geo, ProjectorOptions{g->step}), yt, x0, alpha, iterations), out);
  });
}

// solvers.cpp:162-166
int ref_cgne(const RefGeom* g, int prec, int64_t batch, const void* y, const void* guess, int max_iter,
             double tolerance, void* out) {
  return guard([&] {
    Geometry geo = build(g);
    int64_t s = geometry_image_size(geo);
    Tensor yt = make_tensor({batch, geometry_n_angles(geo), geometry_det_count(geo)}, prec_of(prec), y);
    Tensor x0 = make_tensor({batch, s, s}, prec_of(prec), guess);
    store(cgne(projector_operator(geo, ProjectorOptions{g->step}), x0, yt, max_iter, tolerance), out);
  });
}

// half.hpp:12-71
// shearlet.cpp:103-198 (make_plan): n_coeff, scale labels, fp64 multipliers
int ref_shearlet_plan(int64_t h, int64_t w, const double* alphas, int n_scales, int64_t* n_coeff, double* scales,
                      double* multipliers) {
  return guard([&] {
    ShearletPlan p = make_plan(h, w, std::vector<double>(alphas, alphas + n_scales));
    *n_coeff = p.n_coeff;
    if (scales) std::memcpy(scales, p.scales.data(), p.scales.size() * 8);
    if (multipliers) std::memcpy(multipliers, p.multipliers.data(), p.multipliers.size() * 8);
  });
}

// shearlet.cpp:296-311 (forward: B x h x w -> B x n_coeff x h x w)
int ref_shearlet_forward(int64_t h, int64_t w, const double* alphas, int n_scales, int prec, int64_t batch,
                         const void* image, void* coeff) {
  return guard([&] {
    ShearletPlan p = make_plan(h, w, std::vector<double>(alphas, alphas + n_scales));
    store(forward(p, make_tensor({batch, h, w}, prec_of(prec), image)), coeff);
  });
}

// shearlet.cpp:313-330 (backward: B x n_coeff x h x w -> B x h x w)
int ref_shearlet_backward(int64_t h, int64_t w, const double* alphas, int n_scales, int prec, int64_t batch,
                          const void* coeff, void* image) {
  return guard([&] {
    ShearletPlan p = make_plan(h, w, std::vector<double>(alphas, alphas + n_scales));
    store(backward(p, make_tensor({batch, p.n_coeff, h, w}, prec_of(prec), coeff)), image);
  });
}

// admm.cpp:111-163 (default weights 3^scale / 400 when weights == NULL)
int ref_admm(const RefGeom* g, const double* alphas, int n_scales, int prec, int64_t batch, const void* sino,
             double p0, double p1, const double* weights, int64_t outer, int64_t inner, void* image) {
  return guard([&] {
    Geometry geo = build(g);
    const int64_t s = geometry_image_size(geo);
    ShearletPlan plan = make_plan(s, s, std::vector<double>(alphas, alphas + n_scales));
    AdmmParams prm;
    prm.p0 = p0;
    prm.p1 = p1;
    prm.outer_iterations = outer;
    prm.inner_cg_iterations = inner;
    if (weights) prm.weights = Tensor::from_vec({1, plan.n_coeff, 1, 1}, std::vector<double>(weights, weights + plan.n_coeff));
    Tensor y = make_tensor({batch, geometry_n_angles(geo), geometry_det_count(geo)}, prec_of(prec), sino);
    store(admm_reconstruct(projector_operator(geo, ProjectorOptions{g->step}), plan, y, prm), image);
  });
}

uint16_t ref_float_to_half(float f) { return float_to_half(f); }
float ref_half_to_float(uint16_t h) { return half_to_float(h); }

}  // extern "C"
