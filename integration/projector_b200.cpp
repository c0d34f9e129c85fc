// projector_b200.cpp — the reference's projector translation unit, re-bodied
// on the B200 C ABI.  Drop-in for radonkit's proj/core/src/projector.cpp: it
// implements exactly the functions radonkit/projector.hpp declares
// (projector.hpp:19-35), with the reference's validation and messages
// (projector.cpp:15-33), its precision contract (output in the input's
// storage precision, projector.cpp:207-224) and its Tensor-in / fresh-Tensor-
// out ownership, but every forward / backprojection runs the sm_100a kernels
// through rk_forward_host / rk_backproject_host (include/radon_b200.h).
//
// Everything above this file — LinearOperator (linop.cpp:33-41), the solvers
// (solvers.cpp), fbp (sino_filter_b200.cpp), ADMM, the CLI — is the
// reference's own unmodified code; integration/Makefile links it.
//
// Plans (device geometry tables + the forward schedule) are cached per
// (geometry, step) for the process, like the Python mirror's get_plan; the
// forward schedule itself also persists across processes in the plan cache
// ($RK_PLAN_CACHE, csrc/plan_cache.cpp).
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <variant>
#include <vector>

#include "radon_b200.h"
#include "radonkit/errors.hpp"
#include "radonkit/projector.hpp"
#include "rk_binding.hpp"

namespace radonkit {

namespace b200 {

int dtype_of(const Tensor& t) {
  switch (t.precision()) {
    case Precision::Half: return RK_F16;
    case Precision::Single: return RK_F32;
    default: return RK_F64;
  }
}

const void* data_of(const Tensor& t) {
  switch (t.precision()) {
    case Precision::Half: return t.half_bits().data();
    case Precision::Single: return t.float_data().data();
    default: return t.double_data().data();
  }
}

void* data_of(Tensor& t) {
  switch (t.precision()) {
    case Precision::Half: return t.half_bits().data();
    case Precision::Single: return t.float_data().data();
    default: return t.double_data().data();
  }
}

void check(int status) {
  if (status == RK_OK) return;
  const std::string msg = rk_last_error();
  if (status == RK_ERR_VALIDATION) throw ValidationError(msg);
  if (status == RK_ERR_NUMERICAL) throw NumericalError(msg);
  throw std::runtime_error("radon_b200: " + msg);
}

int device() {
  const char* e = std::getenv("RK_DEVICE");
  return e ? std::atoi(e) : 0;
}

namespace {

struct PlanKey {
  int kind;
  int64_t s, nd;
  double spacing, src, dd, step;
  std::vector<double> angles;
  bool operator<(const PlanKey& o) const {
    return std::tie(kind, s, nd, spacing, src, dd, step, angles) <
           std::tie(o.kind, o.s, o.nd, o.spacing, o.src, o.dd, o.step, o.angles);
  }
};

struct PlanHandle {
  rk_plan* p = nullptr;
  ~PlanHandle() {
    if (p) rk_plan_destroy(p);
  }
};

std::mutex g_mu;
std::map<PlanKey, std::shared_ptr<PlanHandle>>& plans() {
  static auto* m = new std::map<PlanKey, std::shared_ptr<PlanHandle>>();  // outlives static teardown
  return *m;
}

rk_plan* plan_for(rk_geometry c) {
  PlanKey key{int(c.kind), c.image_size, c.det_count, c.det_spacing, c.source_distance,
              c.det_distance, c.step, std::vector<double>(c.angles, c.angles + c.n_angles)};
  std::lock_guard<std::mutex> lock(g_mu);
  auto& m = plans();
  auto it = m.find(key);
  if (it != m.end()) return it->second->p;
  auto h = std::make_shared<PlanHandle>();
  check(rk_plan_create(&c, device(), &h->p));
  m.emplace(std::move(key), h);
  return h->p;
}

}  // namespace

rk_plan* plan_for(const ParallelGeometry& g, double step) {
  rk_geometry c{};
  c.kind = RK_PARALLEL;
  c.has = RK_HAS_DET_COUNT | RK_HAS_DET_SPACING;  // the struct already carries the make_parallel defaults
  c.image_size = g.image_size;
  c.n_angles = int64_t(g.angles.size());
  c.angles = g.angles.data();
  c.det_count = g.det_count;
  c.det_spacing = g.det_spacing;
  c.step = step;
  return plan_for(c);
}

rk_plan* plan_for(const FanbeamGeometry& g, double step) {
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
  return plan_for(c);
}

}  // namespace b200

namespace {

// projector.cpp:15-33: the reference's shape and option checks, same messages.
void check_image(const Tensor& image, int64_t size) {
  if (image.ndim() != 3)
    throw ValidationError("image must be 3-dimensional (batch, h, w), got " + shape_str(image.shape()));
  if (image.dim(1) != size || image.dim(2) != size)
    throw ValidationError("image shape " + shape_str(image.shape()) + " does not match geometry image_size " +
                          std::to_string(size));
}

void check_sino(const Tensor& sino, int64_t n_angles, int64_t det_count) {
  if (sino.ndim() != 3)
    throw ValidationError("sinogram must be 3-dimensional (batch, angles, det), got " + shape_str(sino.shape()));
  if (sino.dim(1) != n_angles || sino.dim(2) != det_count)
    throw ValidationError("sinogram shape " + shape_str(sino.shape()) + " does not match geometry (" +
                          std::to_string(n_angles) + " angles, " + std::to_string(det_count) + " cells)");
}

void check_opts(const ProjectorOptions& opts) {
  if (!(opts.step > 0.0)) throw ValidationError("projector step must be positive");
}

template <class G>
Tensor forward_b200(const G& g, const Tensor& image, const ProjectorOptions& opts) {
  check_image(image, g.image_size);
  check_opts(opts);
  Tensor out = Tensor::zeros({image.batch(), int64_t(g.angles.size()), g.det_count}, image.precision());
  if (image.batch() == 0) return out;
  b200::check(rk_forward_host(b200::plan_for(g, opts.step), b200::dtype_of(image), b200::data_of(image),
                              image.batch(), b200::data_of(out)));
  return out;
}

template <class G>
Tensor backprojection_b200(const G& g, const Tensor& sino, const ProjectorOptions& opts) {
  check_sino(sino, int64_t(g.angles.size()), g.det_count);
  check_opts(opts);
  Tensor out = Tensor::zeros({sino.batch(), g.image_size, g.image_size}, sino.precision());
  if (sino.batch() == 0) return out;
  b200::check(rk_backproject_host(b200::plan_for(g, opts.step), b200::dtype_of(sino), b200::data_of(sino),
                                  sino.batch(), b200::data_of(out)));
  return out;
}

}  // namespace

Tensor forward(const ParallelGeometry& g, const Tensor& image, const ProjectorOptions& opts) {
  return forward_b200(g, image, opts);
}
Tensor forward(const FanbeamGeometry& g, const Tensor& image, const ProjectorOptions& opts) {
  return forward_b200(g, image, opts);
}
Tensor forward(const Geometry& g, const Tensor& image, const ProjectorOptions& opts) {
  return std::visit([&](const auto& gg) { return forward(gg, image, opts); }, g);
}

Tensor backprojection(const ParallelGeometry& g, const Tensor& sino, const ProjectorOptions& opts) {
  return backprojection_b200(g, sino, opts);
}
Tensor backprojection(const FanbeamGeometry& g, const Tensor& sino, const ProjectorOptions& opts) {
  return backprojection_b200(g, sino, opts);
}
Tensor backprojection(const Geometry& g, const Tensor& sino, const ProjectorOptions& opts) {
  return std::visit([&](const auto& gg) { return backprojection(gg, sino, opts); }, g);
}

// projector.hpp:31-35: column c = forward of the c-th unit image, in double.
// All s^2 unit images go through one batched forward (one launch) instead of
// the reference's column-by-column loop; batched == per-element bit for bit.
Tensor materialize_matrix(const Geometry& g, const ProjectorOptions& opts) {
  const int64_t s = geometry_image_size(g);
  if (s > 64)
    throw ValidationError("materialize_matrix refuses image_size " + std::to_string(s) +
                          " (> 64); the dense matrix would be too large");
  check_opts(opts);
  const int64_t rows = geometry_n_angles(g) * geometry_det_count(g), cols = s * s;
  Tensor units = Tensor::zeros({cols, s, s}, Precision::Double);
  for (int64_t c = 0; c < cols; ++c) units.double_data()[size_t(c * cols + c)] = 1.0;
  const Tensor fw = forward(g, units, opts);  // cols x n_angles x det_count
  std::vector<double> mat(size_t(rows) * size_t(cols));
  const std::vector<double>& v = fw.double_data();
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r) mat[size_t(r * cols + c)] = v[size_t(c * rows + r)];
  return Tensor::from_vec({rows, cols}, std::move(mat));
}

}  // namespace radonkit
