// Forward-projection schedule (host, fp64).
//
// The forward kernel (kernels.cu) gives each CTA a block of A consecutive
// angles x W consecutive detector cells (one warp per angle, one lane per
// ray) and marches all of its rays together, chunk by chunk, along the ray
// parameter t (reference: t_m = t0 + (m + 0.5) h, projector.cpp:75-81).
// Before each chunk the CTA stages into shared memory the axis-aligned box of
// packed image texels (4 images per 16-byte texel) that the chunk's samples
// can touch; every bilinear tap (projector.cpp:47-64) is then a 128-bit
// shared-memory load.  This file computes, per CTA:
//   * the box of every chunk, from the exact fp64 ray segments, with one
//     unit of slack in t and one texel of slack around the taps (the kernel
//     assigns samples to chunks in fp32);
//   * the shared-memory orientation and row pitch: the 8 lanes of a quarter
//     warp read 8 neighbouring rays at one sample step, i.e. 8 texels along
//     a digital line; the planner simulates the bank slots of those
//     addresses for both orientations (the transposed copy of the packed
//     image serves the "mostly vertical" lanes) and every pitch residue mod 8
//     and keeps the cheapest.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>

#include "rk_internal.hpp"

namespace rk {

namespace {

struct Pt {
  double px, py;  // padded pixel coordinates (column, row) of a world point
};

inline Pt to_pixel(double x, double y, double half) { return {x + half + 0.5, half - y + 0.5}; }

// Bank-conflict cost of one orientation / pitch: sum over quarter warps and
// taps of the number of distinct 16-byte cells that share a slot (1 = free).
// swap: 0 none, 1 odd lanes load the bottom row first, 2 odd lanes load the
// right column first (kernel: which tap each lane issues in each of its four
// 128-bit loads; spreads the quarter warp over more bank slots).
double conflict_cost(const std::vector<Pt>& lanes_at_step, int lanes_per_warp, bool transposed, int pitch, int swap) {
  double cost = 0.0;
  const int nw = int(lanes_at_step.size()) / lanes_per_warp;
  for (int w = 0; w < nw; ++w) {
    for (int q = 0; q < lanes_per_warp; q += 8) {
      int64_t bi[8], bj[8];
      int lane_of[8];
      int used = 0;
      for (int l = 0; l < 8 && q + l < lanes_per_warp; ++l) {
        const Pt& pt = lanes_at_step[size_t(w * lanes_per_warp + q + l)];
        if (std::isnan(pt.px)) continue;
        const double cx = transposed ? pt.py : pt.px, cy = transposed ? pt.px : pt.py;
        bj[used] = int64_t(std::floor(cx));
        bi[used] = int64_t(std::floor(cy));
        lane_of[used] = q + l;
        ++used;
      }
      for (int tap = 0; tap < 4; ++tap) {
        int64_t addr[8];
        int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int worst = used ? 1 : 0;
        for (int u = 0; u < used; ++u) {
          const bool odd = (lane_of[u] & 1) != 0;
          const int dy = (swap == 1 && odd) ? 1 - (tap >> 1) : (tap >> 1);
          const int dx = (swap == 2 && odd) ? 1 - (tap & 1) : (tap & 1);
          addr[u] = (bi[u] + dy) * pitch + bj[u] + dx;
          bool dup = false;
          for (int v = 0; v < u && !dup; ++v) dup = addr[v] == addr[u];
          if (!dup) worst = std::max(worst, ++cnt[int(((addr[u] % 8) + 8) % 8)]);
        }
        cost += worst;
      }
    }
  }
  return cost;
}

}  // namespace

void build_forward_plan(Plan& p, const std::vector<RayD>& rays, std::vector<float4>& ray_geom,
                        std::vector<float4>& ray_aux) {
  const int64_t s = p.s, na = p.na, nd = p.nd;
  const bool fan = p.g.kind == RK_FANBEAM;
  const double half = 0.5 * double(s);
  const int64_t P2 = s + 2;  // padded image width

  // ---- per-ray float records
  ray_geom.resize(rays.size());
  ray_aux.resize(rays.size());
  for (size_t r = 0; r < rays.size(); ++r) {
    const RayD& R = rays[r];
    if (R.n == 0) {
      ray_geom[r] = make_float4(0.f, 0.f, 0.f, 0.f);
      int zero = 0;
      float zf;
      std::memcpy(&zf, &zero, 4);
      ray_aux[r] = make_float4(0.f, zf, 0.f, 0.f);
      continue;
    }
    // px(m) = x(t_m) + s/2 - 0.5 (+1 border) = px0 + (m + 0.5) hx, t_m = t0 + (m + 0.5) h
    const double ex = R.ox + R.t0 * R.dx, ey = R.oy + R.t0 * R.dy;
    ray_geom[r] = make_float4(float(ex + half + 0.5), float(half - ey + 0.5), float(R.h * R.dx), float(-(R.h * R.dy)));
    int ni = int(R.n);
    float nf;
    std::memcpy(&nf, &ni, 4);
    ray_aux[r] = make_float4(float(R.h), nf, float(R.t0), float(1.0 / R.h));
  }

  // ---- CTA angle sets: angles sorted by direction (mod 2 pi: theta and theta + pi
  // march the same lines in opposite t), A_eff consecutive ones per CTA (the
  // reference accepts arbitrary angle lists, geometry.cpp:12-18)
  ForwardSchedule& F = p.fwd;
  F.A = 8;
  F.W = 32;
  std::vector<int> order(static_cast<size_t>(na));
  for (int64_t a = 0; a < na; ++a) order[size_t(a)] = int(a);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    const double tx = std::fmod(std::fmod(p.angles[size_t(x)], 2.0 * M_PI) + 2.0 * M_PI, 2.0 * M_PI);
    const double ty = std::fmod(std::fmod(p.angles[size_t(y)], 2.0 * M_PI) + 2.0 * M_PI, 2.0 * M_PI);
    return tx < ty;
  });
  const double R = half * std::sqrt(2.0);  // every image point lies within R of the centre
  const double t_lo = (fan ? p.g.source_distance : 0.0) - R - 1.0;
  const double t_hi = (fan ? p.g.source_distance : 0.0) + R + 1.0;
  F.ctas_k = int((nd + F.W - 1) / F.W);
  const int64_t box_budget = 6 * 1024;  // float4 cells (96 KB)

  for (int a_eff : {8, 4, 2, 1}) {
  F.ctas_a = int((na + a_eff - 1) / a_eff);
  const int ctas = F.ctas_a * F.ctas_k;
  F.slots.assign(size_t(F.ctas_a) * F.A, -1);
  for (int64_t i = 0; i < na; ++i) F.slots[size_t((i / a_eff) * F.A + (i % a_eff))] = order[size_t(i)];
  for (double tlen : {32.0, 24.0, 16.0, 12.0, 8.0, 6.0, 4.0}) {
    F.tlen = float(tlen);
    F.tbase = float(t_lo);
    F.chunks = int(std::ceil((t_hi - t_lo) / tlen));
    F.boxes.assign(size_t(ctas) * F.chunks, make_int4(0, 0, 0, 0));
    F.cta.assign(size_t(ctas), make_int2(0, 0));
    F.max_box = 0;
    F.any_transposed = false;
    auto plan_rows = [&](int ca_lo, int ca_hi, int64_t& max_box_out) {
    std::vector<Pt> sim;
    for (int ca = ca_lo; ca < ca_hi; ++ca) {
      for (int ck = 0; ck < F.ctas_k; ++ck) {
        const int cta = ca * F.ctas_k + ck;
        int64_t maxcols[2] = {0, 0};
        std::vector<int4> bx(size_t(F.chunks));  // normal orientation {row0, col0, rows, cols}
        for (int c = 0; c < F.chunks; ++c) {
          const double ta = double(F.tbase) + double(c) * tlen - 1.0;
          const double tb = double(F.tbase) + double(c + 1) * tlen + 1.0;
          double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
          for (int ai = 0; ai < F.A; ++ai) {
            const int a = F.slots[size_t(ca) * F.A + ai];
            if (a < 0) continue;
            for (int ki = 0; ki < F.W; ++ki) {
              const int64_t k = int64_t(ck) * F.W + ki;
              if (k >= nd) break;
              const RayD& ry = rays[size_t(a * nd + k)];
              if (ry.n == 0) continue;
              const double u0 = std::max(ta, ry.t0), u1 = std::min(tb, ry.t1);
              if (!(u1 >= u0)) continue;
              for (double t : {u0, u1}) {
                Pt q = to_pixel(ry.ox + t * ry.dx, ry.oy + t * ry.dy, half);
                xmin = std::min(xmin, q.px);
                xmax = std::max(xmax, q.px);
                ymin = std::min(ymin, q.py);
                ymax = std::max(ymax, q.py);
              }
            }
          }
          if (xmin > xmax) continue;  // no samples of this CTA in the chunk
          int64_t c0 = std::max<int64_t>(0, int64_t(std::floor(xmin)) - 1);
          int64_t c1 = std::min<int64_t>(P2 - 1, int64_t(std::floor(xmax)) + 2);
          int64_t r0 = std::max<int64_t>(0, int64_t(std::floor(ymin)) - 1);
          int64_t r1 = std::min<int64_t>(P2 - 1, int64_t(std::floor(ymax)) + 2);
          bx[size_t(c)] = make_int4(int(r0), int(c0), int(r1 - r0 + 1), int(c1 - c0 + 1));
          maxcols[0] = std::max(maxcols[0], c1 - c0 + 1);
          maxcols[1] = std::max(maxcols[1], r1 - r0 + 1);
        }
        // ---- orientation + pitch by simulated bank conflicts at a few aligned sample steps
        sim.clear();
        const int steps = 4;
        for (int st = 0; st < steps; ++st) {
          const double tt = t_lo + (t_hi - t_lo) * (0.2 + 0.6 * double(st) / double(steps - 1));
          for (int ai = 0; ai < F.A; ++ai) {
            const int a = F.slots[size_t(ca) * F.A + ai];
            for (int ki = 0; ki < F.W; ++ki) {
              const int64_t k = int64_t(ck) * F.W + ki;
              Pt q{NAN, NAN};
              if (a >= 0 && k < nd) {
                const RayD& ry = rays[size_t(a * nd + k)];
                if (ry.n > 0 && tt >= ry.t0 && tt <= ry.t1) {
                  // the sample the lane reaches when the chunk-aligned march is at tt
                  double m = std::floor((tt - ry.t0) / ry.h);
                  double t = ry.t0 + (m + 0.5) * ry.h;
                  q = to_pixel(ry.ox + t * ry.dx, ry.oy + t * ry.dy, half);
                }
              }
              sim.push_back(q);
            }
          }
        }
        double best = 1e300;
        int best_pitch = int(maxcols[0]), best_tr = 0, best_swap = 0;
        for (int tr = 0; tr < 2; ++tr) {
          if (maxcols[tr] == 0) continue;
          for (int swap = 0; swap < 3; ++swap) {
            for (int d = 0; d < 8; ++d) {
              const int pitch = int(maxcols[tr]) + d;
              const double cst =
                  conflict_cost(sim, F.W, tr == 1, pitch, swap) * (1.0 + 1e-4 * d + 1e-3 * tr + 1e-5 * swap);
              if (cst < best) {
                best = cst;
                best_pitch = pitch;
                best_tr = tr;
                best_swap = swap;
              }
            }
          }
        }
        // cfg.y: bit 0 transposed image, bits 1-2 per-lane tap order
        F.cta[size_t(cta)] = make_int2(best_pitch, best_tr | (best_swap << 1));
        for (int c = 0; c < F.chunks; ++c) {
          int4 b = bx[size_t(c)];
          if (b.z == 0) continue;
          if (best_tr) b = make_int4(b.y, b.x, b.w, b.z);  // box in transposed-image coordinates
          F.boxes[size_t(cta) * F.chunks + c] = b;
          max_box_out = std::max<int64_t>(max_box_out, int64_t(b.z) * best_pitch);
        }
      }
    }
    };
    const int nthreads = std::max(1, std::min<int>(int(std::thread::hardware_concurrency()), F.ctas_a));
    std::vector<int64_t> mb(size_t(nthreads), 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t) {
      const int lo = int(int64_t(F.ctas_a) * t / nthreads), hi = int(int64_t(F.ctas_a) * (t + 1) / nthreads);
      pool.emplace_back(plan_rows, lo, hi, std::ref(mb[size_t(t)]));
    }
    for (auto& th : pool) th.join();
    for (int64_t v : mb) F.max_box = std::max(F.max_box, v);
    for (const int2& c : F.cta) F.any_transposed |= (c.y & 1) == 1;
    if (F.max_box <= box_budget) {
      if (std::getenv("RK_DEBUG_PLAN")) {
        int64_t boxes = 0, cells = 0, ntr = 0;
        for (const int4& b : F.boxes)
          if (b.z) ++boxes, cells += int64_t(b.z) * b.w;
        for (const int2& c : F.cta) ntr += c.y & 1;
        std::fprintf(stderr,
                     "[rk] forward schedule: %d angles/CTA, tlen %.0f, %d chunks, %d CTAs (%lld transposed), "
                     "%lld boxes, mean box %.0f texels, max box %lld cells (%.1f KB), staged texels per image "
                     "%.2fM\n",
                     a_eff, double(F.tlen), F.chunks, ctas, (long long)ntr, (long long)boxes,
                     boxes ? double(cells) / double(boxes) : 0.0, (long long)F.max_box,
                     double(F.max_box) * 16.0 / 1024.0, double(cells) / 1e6);
      }
      return;
    }
  }
  }
  throw ValidationError("forward schedule: no chunk length keeps the staged image box within shared memory");
}

}  // namespace rk
