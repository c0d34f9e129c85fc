// Host-side planners under AddressSanitizer + UndefinedBehaviorSanitizer
// (sanitizers on the C++ layer): geometry resolution, the fp64
// ray tables, the forward schedule (with its self-check), backprojection
// windows, ramp filters and alpha-shearlet plans, all host-only (device -1).
// Built and run by tests/test_host_sanitize_cpu.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "rk_internal.hpp"

namespace rk {
void upload_shearlet(Shearlet&) {}  // device-side table upload (shearlet.cu): not part of this host test
void set_device(int device) { RK_CUDA(cudaSetDevice(device)); }  // capi.cpp's scope-restoring switch; host-only plans never call it
}  // namespace rk

static void plan(int kind, int64_t s, const std::vector<double>& ang, int64_t nd, double sp, double src, double dd,
                 double step) {
  rk::Plan p;
  p.device = -1;
  p.angles = ang;
  rk_geometry in{};
  in.kind = kind;
  in.image_size = s;
  in.n_angles = int64_t(ang.size());
  in.angles = p.angles.data();
  in.has = 0;
  if (nd > 0) in.has |= RK_HAS_DET_COUNT, in.det_count = nd;
  if (sp > 0) in.has |= RK_HAS_DET_SPACING, in.det_spacing = sp;
  if (dd > 0) in.has |= RK_HAS_DET_DISTANCE, in.det_distance = dd;
  in.source_distance = src;
  in.step = step;
  p.g = rk::resolve_geometry(in);
  p.g.angles = p.angles.data();
  rk::build_plan(p);
}

int main() {
  std::mt19937 rng(11);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  auto lin = [](int n, double stop) {
    std::vector<double> a(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) a[size_t(i)] = stop * double(i) / double(n);
    return a;
  };
  plan(RK_PARALLEL, 256, lin(256, M_PI), 0, 0, 0, 0, 1.0);
  plan(RK_FANBEAM, 256, lin(200, 2 * M_PI), 0, 0, 256.0, 0, 1.0);
  plan(RK_FANBEAM, 96, lin(64, 2 * M_PI), 0, 0, 70.0, 300.0, 1.0);
  for (int i = 0; i < 24; ++i) {
    const int64_t s = std::vector<int64_t>{1, 3, 17, 40, 64, 97, 131}[size_t(i % 7)];
    std::vector<double> ang(size_t(1 + int(U(rng) * 50)));
    for (double& a : ang) a = -7.0 + 14.0 * U(rng);
    const int64_t nd = 1 + int64_t(U(rng) * double(3 * s + 7));
    const double sp = 0.3 + 2.2 * U(rng), step = i % 3 == 0 ? 0.5 : 1.0;
    if (i % 2)
      plan(RK_FANBEAM, s, ang, nd, sp, double(s) * (0.75 + 3.25 * U(rng)), double(s) * (0.5 + 2.5 * U(rng)), step);
    else
      plan(RK_PARALLEL, s, ang, nd, sp, 0, 0, step);
  }
  for (int kind = RK_RAM_LAK; kind <= RK_HANN; ++kind)
    for (int64_t nd : {2, 8, 725, 1449}) {
      rk::Filter f;
      f.device = -1;
      rk::build_filter(f, kind, nd);
    }
  for (int64_t n : {32, 64, 128}) {
    rk::Shearlet sh;
    sh.device = -1;
    rk::build_shearlet(sh, n, n, std::vector<double>(3, 0.5));
  }
  std::printf("host planners clean\n");
  return 0;
}
