// C++ consumer of the drop-in layer (include/radonkit_b200.hpp): restates a
// few of proj/tests/test_projector.cpp / test_sino_filter.cpp assertions
// through the C++ API and prints one line per check (exit code = failures).
// Built and run by tests/test_cpp_wrapper.py (compile on CPU, run on the GPU).
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "radonkit_b200.hpp"

static int failures = 0;
static void report(const char* name, bool ok, double v) {
  std::printf("%s %s %.3e\n", ok ? "PASS" : "FAIL", name, v);
  if (!ok) ++failures;
}

int main(int argc, char** argv) {
  const bool validate_only = argc > 1 && std::string(argv[1]) == "--validate-only";
  // geometry defaults and validation (test_geometry.cpp:10-73) — no GPU needed
  auto gf = rkb::make_fanbeam(512, rkb::angles_linspace(0.0, 2.0 * M_PI, 512), 512.0);
  report("fan-default-spacing", gf.det_spacing == 2.0 && gf.det_distance == 512.0 && gf.det_count == 512,
         gf.det_spacing);
  bool threw = false;
  try {
    rkb::make_fanbeam(512, {0.0}, 300.0);
  } catch (const rkb::ValidationError&) {
    threw = true;
  }
  report("fan-source-inside-rejected", threw, 0.0);
  auto spec = rkb::make_filter("ram-lak", 8, validate_only ? -1 : 0);
  report("filter-padded", spec.padded_size == 16, double(spec.padded_size));
  report("filter-dc", spec.frequency_response[0] > 0.0 && spec.frequency_response[0] < 0.05,
         spec.frequency_response[0]);
  if (validate_only) return failures;

  // axis-aligned closed forms (test_projector.cpp:137-163)
  const int64_t s = 16;
  auto g = rkb::make_parallel(s, {0.0});
  std::vector<float> img(size_t(s * s));
  for (int64_t i = 0; i < s * s; ++i) img[size_t(i)] = float((i * 37) % 11) / 11.0f;
  auto f = rkb::forward(rkb::Geometry(g), img, 1);
  double err = 0.0;
  for (int64_t k = 0; k < s; ++k) {
    double col = 0.0;
    for (int64_t i = 0; i < s; ++i) col += img[size_t(i * s + k)];
    err = std::max(err, std::abs(col - f[size_t(k)]));
  }
  report("forward-theta0-column-sums", err < 1e-5, err);
  std::vector<float> delta(size_t(s), 0.0f);
  delta[5] = 1.0f;
  auto bp = rkb::backprojection(rkb::Geometry(g), delta, 1);
  bool col_ok = true;
  for (int64_t i = 0; i < s; ++i)
    for (int64_t j = 0; j < s; ++j) col_ok &= bp[size_t(i * s + j)] == (j == 5 ? 1.0f : 0.0f);
  report("backprojection-delta-column", col_ok, 0.0);

  // linear operator + FBP round trip on a disc
  auto gp = rkb::make_parallel(64, rkb::angles_linspace(0.0, M_PI, 90), 95);
  std::vector<float> disc(64 * 64);
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) {
      double x = j - 31.5, y = 31.5 - i;
      disc[size_t(i * 64 + j)] = (x * x + y * y < 20.0 * 20.0) ? 1.0f : 0.0f;
    }
  auto op = rkb::projector_operator(gp);
  auto sino = op.apply(disc);
  auto rec = rkb::fbp(rkb::Geometry(gp), sino, 1, rkb::FilterKind::RamLak);
  double se = 0.0;
  for (size_t i = 0; i < rec.size(); ++i) se += (rec[i] - disc[i]) * (rec[i] - disc[i]);
  report("fbp-disc-mse", se / double(rec.size()) < 0.02, se / double(rec.size()));
  // half storage round trip keeps the precision (projector.cpp:207-224)
  std::vector<uint16_t> h(size_t(64 * 64), 0x3c00);  // 1.0
  auto hs = rkb::forward(rkb::Geometry(gp), h, 1);
  report("half-storage-forward", hs.size() == size_t(90 * 95), double(hs.size()));
  return failures;
}
