// sino_filter_b200.cpp — the reference's filter_sinogram and fbp
// (sino_filter.cpp:98-136) re-bodied on the B200 C ABI.
//
// make_filter / filter_kind_from_name / the window functions stay the
// reference's own code (sino_filter.cpp, linked unmodified; integration/
// Makefile weakens only the four symbols defined here, so these strong
// definitions replace them at link time).  The device filter is built from
// the same response (rk_filter_create reproduces make_filter's bins bit for
// bit; checked below against the FilterSpec the caller passes).
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <variant>
#include <vector>

#include "radon_b200.h"
#include "radonkit/errors.hpp"
#include "radonkit/projector.hpp"
#include "radonkit/sino_filter.hpp"
#include "rk_binding.hpp"

namespace radonkit {

namespace {

struct FilterHandle {
  rk_filter* f = nullptr;
  ~FilterHandle() {
    if (f) rk_filter_destroy(f);
  }
};

std::mutex g_mu;

// Device filter for (kind, det_count); its float response must equal the
// caller's FilterSpec (a hand-edited spec cannot silently be replaced).
rk_filter* filter_for(const FilterSpec& spec) {
  static auto* cache = new std::map<std::pair<int, int64_t>, std::shared_ptr<FilterHandle>>();
  const auto key = std::make_pair(int(spec.kind), spec.det_count);
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = cache->find(key);
  if (it == cache->end()) {
    auto h = std::make_shared<FilterHandle>();
    b200::check(rk_filter_create(int(spec.kind), spec.det_count, b200::device(), &h->f));
    it = cache->emplace(key, h).first;
  }
  int64_t padded = 0;
  b200::check(rk_filter_response(it->second->f, &padded, nullptr, nullptr));
  std::vector<float> resp(size_t(padded / 2 + 1));
  b200::check(rk_filter_response(it->second->f, nullptr, nullptr, resp.data()));
  if (padded != spec.padded_size || resp.size() != spec.frequency_response_f.size() ||
      std::memcmp(resp.data(), spec.frequency_response_f.data(), resp.size() * sizeof(float)) != 0)
    throw ValidationError("filter response differs from make_filter(" + std::string(filter_kind_name(spec.kind)) +
                          ", " + std::to_string(spec.det_count) + "); custom responses are not supported by the GPU path");
  return it->second->f;
}

template <class G>
Tensor fbp_b200(const G& g, const Tensor& sino, FilterKind kind) {
  // fbp = backprojection(filter_sinogram(sino, make_filter(kind, det_count))) (sino_filter.cpp:126-136);
  // the same validation order: filter_sinogram's checks, then backprojection's.
  const FilterSpec spec = make_filter(kind, g.det_count);
  if (sino.ndim() != 3)
    throw ValidationError("sinogram must be 3-dimensional (batch, angles, det), got " + shape_str(sino.shape()));
  if (sino.dim(2) != spec.det_count)
    throw ValidationError("sinogram det_count " + std::to_string(sino.dim(2)) + " does not match filter " +
                          std::to_string(spec.det_count));
  if (sino.dim(1) != int64_t(g.angles.size()) || sino.batch() == 0)
    return backprojection(g, filter_sinogram(sino, spec));  // the reference's error (or empty result)
  Tensor out = Tensor::zeros({sino.batch(), g.image_size, g.image_size}, sino.precision());
  b200::check(rk_fbp_host(b200::plan_for(g, 1.0), filter_for(spec), b200::dtype_of(sino), b200::data_of(sino),
                          sino.batch(), b200::data_of(out)));
  return out;
}

}  // namespace

Tensor filter_sinogram(const Tensor& sino, const FilterSpec& filter) {
  if (sino.ndim() != 3)
    throw ValidationError("sinogram must be 3-dimensional (batch, angles, det), got " + shape_str(sino.shape()));
  if (sino.dim(2) != filter.det_count)
    throw ValidationError("sinogram det_count " + std::to_string(sino.dim(2)) + " does not match filter " +
                          std::to_string(filter.det_count));
  Tensor out = Tensor::zeros(sino.shape(), sino.precision());
  if (sino.batch() == 0 || sino.dim(1) == 0) return out;
  b200::check(rk_filter_sinogram_host(filter_for(filter), b200::dtype_of(sino), b200::data_of(sino), sino.batch(),
                                      sino.dim(1), b200::data_of(out)));
  return out;
}

Tensor fbp(const ParallelGeometry& g, const Tensor& sino, FilterKind kind) { return fbp_b200(g, sino, kind); }
Tensor fbp(const FanbeamGeometry& g, const Tensor& sino, FilterKind kind) { return fbp_b200(g, sino, kind); }
Tensor fbp(const Geometry& g, const Tensor& sino, FilterKind kind) {
  return std::visit([&](const auto& gg) { return fbp(gg, sino, kind); }, g);
}

}  // namespace radonkit
