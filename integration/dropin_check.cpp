// dropin_check — a reference user's program, unchanged: it calls only the
// reference's public API (radonkit/*.hpp), here linked against the reference's
// own tensor / geometry / phantom / linop / solvers / sino_filter / npy code
// with projector_b200.cpp + sino_filter_b200.cpp in place of projector.cpp's
// and sino_filter.cpp's projector bodies (integration/Makefile).  So every
// forward / backprojection / filter below — including the ones inside
// adjoint_check (linop.cpp:65-80), estimate_alpha, landweber and cgne
// (solvers.cpp:47-166) — runs on the B200.
//
//   dropin_check <outdir>
// writes the inputs and results as .npy (the reference's own writer) and one
// JSON line of scalars; tests/test_dropin_reference_gpu.py recomputes all of
// it with the unmodified reference (oracle/_ref) and compares.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <string>

#include "radonkit/geometry.hpp"
#include "radonkit/linop.hpp"
#include "radonkit/npy.hpp"
#include "radonkit/phantom.hpp"
#include "radonkit/projector.hpp"
#include "radonkit/rng.hpp"
#include "radonkit/sino_filter.hpp"
#include "radonkit/solvers.hpp"
#include "radonkit/tensor.hpp"

using namespace radonkit;

namespace {

// bench.py's batch, elements 0..1: phantom x 1/128 and Rng(1) uniform
Tensor bench_pair(int64_t s) {
  Tensor ph = shepp_logan(s);
  Tensor u = Rng(1).uniform_tensor({1, s, s});
  std::vector<float> v(size_t(2 * s * s));
  for (int64_t i = 0; i < s * s; ++i) {
    v[size_t(i)] = ph.float_data()[size_t(i)] * float(1.0 / 128.0);
    v[size_t(s * s + i)] = u.float_data()[size_t(i)];
  }
  return Tensor::from_vec({2, s, s}, std::move(v));
}

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: dropin_check <outdir>\n");
    return 1;
  }
  const std::string out = argv[1];
  auto save = [&](const char* name, const Tensor& t) { write_array(out + "/" + name + ".npy", t); };
  try {
    // config 2 / 3 geometries: forward, backprojection, half storage
    const Tensor x = bench_pair(512);
    save("x512", x);
    const ParallelGeometry gp = make_parallel(512, angles_linspace(0.0, M_PI, 512));
    const FanbeamGeometry gf = make_fanbeam(512, angles_linspace(0.0, 2.0 * M_PI, 512), 512.0);
    const double t0 = now();
    const Tensor yp = forward(Geometry(gp), x);
    const Tensor bp = backprojection(Geometry(gp), yp);
    const double t1 = now();
    save("fwd_par", yp);
    save("bp_par", bp);
    const Tensor yf = forward(Geometry(gf), x);
    save("fwd_fan", yf);
    save("bp_fan", backprojection(Geometry(gf), yf));
    const Tensor xh = convert(x, Precision::Half);
    save("x512_half", xh);
    save("fwd_par_half", forward(gp, xh));
    // FBP (sino_filter.cpp:126-136) and filter_sinogram on config 1's geometry
    const ParallelGeometry g1 = make_parallel(256, angles_linspace(0.0, M_PI, 256));
    const Tensor s1 = forward(g1, shepp_logan(256));
    save("sino256", s1);
    save("fbp256", fbp(Geometry(g1), s1));
    save("filt256_hann", filter_sinogram(s1, make_filter(FilterKind::Hann, 256)));
    // the LinearOperator consumers (linop.cpp, solvers.cpp) over the GPU projector
    const ParallelGeometry g5 = make_parallel(512, angles_linspace(0.0, M_PI, 256));
    const LinearOperator op = projector_operator(Geometry(g5));
    const double defect5 = adjoint_check(op, 1, 0);
    const double defect_fan = adjoint_check(projector_operator(Geometry(gf)), 1, 0);
    const double alpha = 0.95 * estimate_alpha(op, 20, 0);
    Tensor x5 = shepp_logan(512);
    const Tensor y5 = forward(g5, x5);
    const Tensor z = Tensor::zeros({1, 512, 512});
    save("y5", y5);
    save("landweber10", landweber(op, y5, z, alpha, 10));
    save("cgne10", cgne(op, z, y5, 10));
    // the dense matrix (projector.hpp:31-35) at a small size
    save("matrix16", materialize_matrix(Geometry(make_parallel(16, angles_linspace(0.0, M_PI, 12)))));
    std::printf("{\"adjoint_defect_cfg5\": %.17g, \"adjoint_defect_fan512\": %.17g, \"alpha\": %.17g, "
                "\"cfg2_pair_fwd_bp_s\": %.6f}\n",
                defect5, defect_fan, alpha, t1 - t0);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "dropin_check: %s\n", e.what());
    return 2;
  }
  return 0;
}
