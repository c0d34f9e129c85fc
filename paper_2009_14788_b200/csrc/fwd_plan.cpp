// Forward-projection schedule (host, fp64).
//
// The forward kernel (kernels.cu) gives each CTA 8 warps; warp w marches 32
// consecutive detector cells of one angle (one lane per ray).  Angles are
// sorted by direction (mod 2 pi: theta and theta + pi march the same lines in
// opposite t; the reference accepts arbitrary angle lists,
// geometry.cpp:12-18), and a CTA takes `aa` consecutive sorted angles x `db`
// consecutive 32-cell blocks (aa * db = 8).  All rays of a CTA march together
// along the ray parameter t (reference: t_m = t0 + (m + 0.5) h,
// projector.cpp:75-81), chunk by chunk.  Before each chunk the CTA stages into
// shared memory the axis-aligned box of packed image texels (4 images per
// 16-byte texel) that the chunk's samples can touch; every bilinear tap
// (projector.cpp:47-64) is then a 128-bit shared-memory load.
//
// Per CTA this file decides
//   * the shared-memory layout: the 8 lanes of a quarter warp read 8
//     neighbouring rays at one sample step, i.e. 8 texels along a digital
//     line.  The bank slots of those addresses are simulated for both
//     orientations (a transposed copy of the packed image serves "mostly
//     vertical" lane lines), every row-pitch residue mod 8 and three per-lane
//     tap orders, and the cheapest is kept;
//   * the chunks: greedily, the longest t-interval (up to 48 units) whose box
//     fits the shared-memory budget, so every CTA gets as few chunks (barriers)
//     and as much texel reuse as its geometry allows.  Boxes come from the
//     exact fp64 ray segments with one unit of slack in t and one texel around
//     the taps (the kernel assigns samples to chunks in fp32).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <mutex>
#include <thread>
#include <utility>

#include "rk_internal.hpp"

namespace rk {

namespace {

struct Pt {
  double px, py;  // padded pixel coordinates (column, row) of a world point
};

inline Pt to_pixel(double x, double y, double half) { return {x + half + 0.5, half - y + 0.5}; }

// Bank-conflict costs of the layouts of one orientation: for every tap order
// (swap: 0 none, 1 odd lanes load the bottom row first, 2 odd lanes load the
// right column first — the kernel issues each lane's four taps in that order)
// and row-pitch residue mod 8, the sum over quarter warps and taps of the
// number of distinct 16-byte cells that share a slot (1 = conflict free).
//
// The slot of cell (i, j) under residue r is (j + r i) mod 8 (pitch 64 + r).
// For the eight residues at once, a cell contributes one count to slot
// (j + r i) & 7 of residue r: eight 4-bit counters (one 32-bit word) per
// residue, so a cell's contribution is an 8-word vector that depends only on
// (i mod 8, j mod 8) — a table lookup and one vector add per distinct cell.
// The worst slot of each residue is then found with one threshold test per
// count level (counts are at most 8, so nibble + 8 - t carries into the
// nibble's top bit exactly when nibble >= t).
typedef uint32_t V8 __attribute__((vector_size(32)));

struct SlotTable {
  V8 inc[64];  // [(i & 7) * 8 + (j & 7)]
  SlotTable() {
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j)
        for (int r = 0; r < 8; ++r) inc[i * 8 + j][r] = 1u << (4 * ((j + r * i) & 7));
  }
};
const SlotTable kSlots;

inline V8 worst_slot(const V8& cnt) {
  V8 worst = {1, 1, 1, 1, 1, 1, 1, 1};
  for (uint32_t t = 2; t <= 8; ++t)
    worst -= ((cnt + (0x11111111u * (8u - t))) & 0x88888888u) != 0u;  // -1 where some nibble >= t
  return worst;
}

// AVX2 where the host has it (the vector code is 256-bit wide), baseline x86-64 otherwise.
__attribute__((target_clones("avx2", "default")))
void conflict_costs(const std::vector<Pt>& lanes_at_step, bool transposed, double cost[3][8]) {
  V8 acc[3];  // per swap, per residue (integer sums; exact)
  for (auto& a : acc) a = V8{0, 0, 0, 0, 0, 0, 0, 0};
  const int nw = int(lanes_at_step.size()) / 32;
  for (int w = 0; w < nw; ++w) {
    for (int q = 0; q < 32; q += 8) {
      int32_t bi[8], bj[8];  // padded-image cells: far inside 32 bits
      int lane_of[8];
      int used = 0;
      for (int l = 0; l < 8; ++l) {
        const Pt& pt = lanes_at_step[size_t(w * 32 + q + l)];
        if (std::isnan(pt.px)) continue;
        const double cx = transposed ? pt.py : pt.px, cy = transposed ? pt.px : pt.py;
        bj[used] = int32_t(std::floor(cx));
        bi[used] = int32_t(std::floor(cy));
        lane_of[used] = q + l;
        ++used;
      }
      if (!used) continue;
      // A tap offset applied to every lane shifts every slot by the same amount,
      // which leaves the conflicts unchanged: with no swap all four taps cost
      // what tap 0 costs; with a row (column) swap only the row (column) bit of
      // the tap matters.  So 5 of the 12 (swap, tap) patterns are evaluated.
      for (int sw = 0; sw < 3; ++sw)
        for (int tap = 0; tap < 4; ++tap) {
          const uint32_t weight = sw == 0 ? (tap == 0 ? 4 : 0) : sw == 1 ? ((tap & 1) ? 0 : 2) : ((tap & 2) ? 0 : 2);
          if (!weight) continue;
          uint64_t key[8];
          V8 cnt = {0, 0, 0, 0, 0, 0, 0, 0};
          for (int u = 0; u < used; ++u) {
            const bool odd = (lane_of[u] & 1) != 0;
            const int32_t ti = bi[u] + ((sw == 1 && odd) ? 1 - (tap >> 1) : (tap >> 1));
            const int32_t tj = bj[u] + ((sw == 2 && odd) ? 1 - (tap & 1) : (tap & 1));
            key[u] = (uint64_t(uint32_t(ti)) << 32) | uint32_t(tj);
            bool first = true;
            for (int v = 0; v < u; ++v) first &= key[v] != key[u];
            if (first) cnt += kSlots.inc[((ti & 7) << 3) | (tj & 7)];  // mod 8 (two's complement)
          }
          acc[sw] += weight * worst_slot(cnt);
        }
    }
  }
  for (int sw = 0; sw < 3; ++sw)
    for (int r = 0; r < 8; ++r) cost[sw][r] = double(acc[sw][r]);
}

// Per-lane tap order of a chunk (box record z bits 17-30, kernels.cu): bit
// l - 1 of the low 7 bits set = lane l of every quarter warp (l = 1..7) loads
// the bottom row first, bit l - 1 of the high 7 bits = the right column first
// (lane 0 never flips: flipping all lanes only permutes the four loads).  The
// r1 tap orders are the odd-lane patterns.
constexpr int kOddLanes = 0x55;  // lanes 1, 3, 5, 7
inline int order_of_swap(int sw) { return sw == 1 ? kOddLanes : sw == 2 ? kOddLanes << 7 : 0; }
inline bool order_row(int order, int lane8) { return lane8 != 0 && ((order >> (lane8 - 1)) & 1); }
inline bool order_col(int order, int lane8) { return lane8 != 0 && ((order >> (6 + lane8)) & 1); }

// conflict_costs for one arbitrary per-lane tap order: out[r] = the sum over
// quarter warps and the four taps of the worst slot, pitch residue r.
__attribute__((target_clones("avx2", "default")))
void order_costs(const std::vector<Pt>& lanes_at_step, bool transposed, int order, V8& out) {
  out = V8{0, 0, 0, 0, 0, 0, 0, 0};
  const int nw = int(lanes_at_step.size()) / 32;
  for (int w = 0; w < nw; ++w)
    for (int q = 0; q < 32; q += 8) {
      int32_t bi[8], bj[8];
      int lane_of[8];
      int used = 0;
      for (int l = 0; l < 8; ++l) {
        const Pt& pt = lanes_at_step[size_t(w * 32 + q + l)];
        if (std::isnan(pt.px)) continue;
        const double cx = transposed ? pt.py : pt.px, cy = transposed ? pt.px : pt.py;
        bj[used] = int32_t(std::floor(cx));
        bi[used] = int32_t(std::floor(cy));
        lane_of[used] = l;
        ++used;
      }
      if (!used) continue;
      for (int tap = 0; tap < 4; ++tap) {
        uint64_t key[8];
        V8 cnt = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int u = 0; u < used; ++u) {
          const int rb = tap >> 1, cb = tap & 1;
          const int32_t ti = bi[u] + (order_row(order, lane_of[u]) ? 1 - rb : rb);
          const int32_t tj = bj[u] + (order_col(order, lane_of[u]) ? 1 - cb : cb);
          key[u] = (uint64_t(uint32_t(ti)) << 32) | uint32_t(tj);
          bool first = true;
          for (int v = 0; v < u; ++v) first &= key[v] != key[u];
          if (first) cnt += kSlots.inc[((ti & 7) << 3) | (tj & 7)];
        }
        out += worst_slot(cnt);
      }
    }
}

// Conflict-free reference for conflict_cost: one wavefront per quarter warp
// and tap with at least one active lane.
double ideal_cost(const std::vector<Pt>& lanes_at_step) {
  double cost = 0.0;
  for (size_t q = 0; q + 8 <= lanes_at_step.size(); q += 8) {
    bool any = false;
    for (size_t l = 0; l < 8; ++l) any |= !std::isnan(lanes_at_step[q + l].px);
    cost += any ? 4.0 : 0.0;
  }
  return cost;
}

struct Box {
  int64_t r0, c0, rows, cols;  // normal (untransposed) padded-image coordinates
  bool empty() const { return rows <= 0; }
};

inline int pitch_for(int64_t cols, int residue) { return int(cols + ((residue - cols) % 8 + 8) % 8); }

// Detector cells per warp of a CTA (cfg.z bits 5-7, kernels.cu): 32 >> n.  The
// narrow-warp fallback tiers march 16 .. 1 consecutive cells per warp (the other
// lanes idle) for coarse detectors, whose 32 neighbouring rays are too far apart
// for any staged box.
inline int cells_per_warp(int cfgz) { return 32 >> ((cfgz >> 5) & 7); }

// Replays the forward kernel's per-lane schedule on the host in the kernel's
// own fp32 arithmetic (std::fma == FFMA; kernels.cu, forward_kernel) and
// checks that every sample's four taps lie inside its chunk's staged box and
// that the chunks partition each ray's samples — the invariant that lets the
// kernel index the box without clamping.  RK_VERIFY_PLAN=1 (tests).
void verify_forward_schedule(const Plan& p, const std::vector<float4>& ray_geom, const std::vector<float4>& ray_aux) {
  const ForwardSchedule& F = p.fwd;
  const int64_t nd = p.nd;
  for (size_t cta = 0; cta < F.cta.size(); ++cta) {
    const int4 cfg = F.cta[cta];
    const int lq = (cfg.z >> 3) & 3;
    const int2* wa = &F.warps[cta * 8];
    for (int t = 0; t < 256; ++t) {
      int slot = t >> 5, k;
      if (lq == 0) {
        k = wa[t >> 5].y + (t & 31);
      } else {
        const int cq = t & ((8 >> lq) - 1), aq = (t >> (3 - lq)) & ((1 << lq) - 1);
        const int cg = (t >> 3) & ((4 << lq) - 1), ag = t >> (lq + 5);
        slot = (ag << lq) + aq;
        k = wa[0].y + cg * (8 >> lq) + cq;
      }
      const int a = wa[slot].x;
      if (a < 0 || k >= nd || (lq == 0 && (t & 31) >= cells_per_warp(cfg.z))) continue;
      const size_t r = size_t(int64_t(a) * nd + k);
      const float4 G = ray_geom[r], X = ray_aux[r];
      int n;
      std::memcpy(&n, &X.y, 4);
      const float t0 = X.z, inv_h = X.w;
      int m = 0;
      for (int c = 0; c < cfg.y; ++c) {
        const int4 bx = F.boxes[size_t(cfg.x + c)];
        const int r0 = bx.x & 0xffff, c0 = bx.x >> 16, rows = bx.y & 0xffff, cols = bx.y >> 16;
        const bool tr = ((bx.z >> 16) & 1) != 0;
        float tend;
        std::memcpy(&tend, &bx.w, 4);
        const int m_end =
            std::isinf(tend) ? n : std::min(std::max(int(std::ceil(std::fma(tend - t0, inv_h, -0.5f))), 0), n);
        const float pxc = (tr ? G.y : G.x) - float(c0), pyc = (tr ? G.x : G.y) - float(r0);
        const float hx = tr ? G.w : G.z, hy = tr ? G.z : G.w;
        for (; m < m_end; ++m) {
          const float tt = float(m) + 0.5f;
          const float px = std::fma(tt, hx, pxc), py = std::fma(tt, hy, pyc);
          const int j = int(std::floor(px)), i = int(std::floor(py));
          if (j < 0 || i < 0 || j + 1 >= cols || i + 1 >= rows) {
            char msg[256];
            std::snprintf(msg, sizeof(msg),
                          "forward schedule: ray (angle %d, cell %d) sample %d leaves box %d of CTA %zu "
                          "(tap %d,%d of %dx%d)",
                          a, k, m, c, cta, i, j, rows, cols);
            throw std::logic_error(msg);
          }
        }
      }
      if (m != n) throw std::logic_error("forward schedule: chunks do not cover every sample of a ray");
    }
  }
}

// Exact model of the forward kernel's shared-memory load wavefronts for one
// image group under the final schedule: every CTA's lanes replayed in
// lockstep per chunk iteration (the kernel's own fp32 positions, tap orders,
// orientation and pitch), each quarter warp's LDS.128 costing the largest
// number of distinct 16-byte cells that share one of the 8 slots.  Returns
// {modelled, conflict-free}.  RK_PLAN_MODEL=1 (diagnostics: ncu measures
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld per launch = groups x this).
std::pair<double, double> model_wavefronts(const Plan& p, const std::vector<float4>& ray_geom,
                                           const std::vector<float4>& ray_aux) {
  const ForwardSchedule& F = p.fwd;
  const int64_t nd = p.nd;
  std::atomic<int> next{0};
  std::mutex mu;
  double tot = 0.0, ideal = 0.0;
  auto work = [&]() {
    double my_tot = 0.0, my_ideal = 0.0;
    std::vector<int> base(256), n(256), m(256), mend(256);
    std::vector<float> pxc(256), pyc(256), hx(256), hy(256);
    std::vector<float4> G(256), X(256);
    std::vector<char> ok(256);
    for (int cta; (cta = next.fetch_add(1)) < int(F.cta.size());) {
      const int4 cfg = F.cta[size_t(cta)];
      const int lq = (cfg.z >> 3) & 3;
      const int2* wa = &F.warps[size_t(cta) * 8];
      for (int t = 0; t < 256; ++t) {
        int slot = t >> 5, k;
        if (lq == 0) {
          k = wa[t >> 5].y + (t & 31);
        } else {
          const int cq = t & ((8 >> lq) - 1), aq = (t >> (3 - lq)) & ((1 << lq) - 1);
          const int cg = (t >> 3) & ((4 << lq) - 1), ag = t >> (lq + 5);
          slot = (ag << lq) + aq;
          k = wa[0].y + cg * (8 >> lq) + cq;
        }
        const int a = wa[slot].x;
        ok[size_t(t)] = a >= 0 && k < nd && (lq != 0 || (t & 31) < cells_per_warp(cfg.z));
        m[size_t(t)] = 0;
        n[size_t(t)] = 0;
        if (!ok[size_t(t)]) continue;
        const size_t r = size_t(int64_t(a) * nd + k);
        G[size_t(t)] = ray_geom[r];
        X[size_t(t)] = ray_aux[r];
        std::memcpy(&n[size_t(t)], &X[size_t(t)].y, 4);
      }
      for (int c = 0; c < cfg.y; ++c) {
        const int4 bx = F.boxes[size_t(cfg.x + c)];
        const int r0 = bx.x & 0xffff, c0 = bx.x >> 16, pitch = bx.z & 0xffff;
        const bool tr = ((bx.z >> 16) & 1) != 0;
        const int order = (bx.z >> 17) & 0x3fff;
        float tend;
        std::memcpy(&tend, &bx.w, 4);
        int iters = 0;
        for (int t = 0; t < 256; ++t) {
          mend[size_t(t)] = m[size_t(t)];
          if (!ok[size_t(t)]) continue;
          const float t0 = X[size_t(t)].z, inv_h = X[size_t(t)].w;
          const int nn = n[size_t(t)];
          mend[size_t(t)] = std::isinf(tend) ? nn
                                             : std::min(std::max(int(std::ceil(std::fma(tend - t0, inv_h, -0.5f))), 0), nn);
          iters = std::max(iters, mend[size_t(t)] - m[size_t(t)]);
          const float4 g = G[size_t(t)];
          pxc[size_t(t)] = (tr ? g.y : g.x) - float(c0);
          pyc[size_t(t)] = (tr ? g.x : g.y) - float(r0);
          hx[size_t(t)] = tr ? g.w : g.z;
          hy[size_t(t)] = tr ? g.z : g.w;
        }
        for (int q = 0; q < iters; ++q) {
          for (int qw = 0; qw < 256; qw += 8) {
            int used = 0;
            for (int l = 0; l < 8; ++l) {
              const int t = qw + l;
              const int mm = m[size_t(t)] + q;
              if (!ok[size_t(t)] || mm >= mend[size_t(t)]) continue;
              const float tt = float(mm) + 0.5f;
              const float px = std::fma(tt, hx[size_t(t)], pxc[size_t(t)]);
              const float py = std::fma(tt, hy[size_t(t)], pyc[size_t(t)]);
              const int j = int(std::floor(px)), i = int(std::floor(py));
              const bool rs = order_row(order, t & 7), cs = order_col(order, t & 7);
              base[size_t(used++)] = (i * pitch + j + (rs ? pitch : 0) + (cs ? 1 : 0)) |
                                     ((cs ? 1 : 0) << 30) | ((rs ? 1 : 0) << 29);
            }
            if (!used) continue;
            my_ideal += 4.0;
            for (int tap = 0; tap < 4; ++tap) {
              int addr[8], cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, worst = 1;
              for (int u = 0; u < used; ++u) {
                const int b = base[size_t(u)];
                const bool cs = (b >> 30) & 1, rs = (b >> 29) & 1;
                const int a0 = b & ((1 << 29) - 1);
                const int dX = cs ? -1 : 1, dY = rs ? -pitch : pitch;
                addr[u] = a0 + ((tap & 1) ? dX : 0) + ((tap & 2) ? dY : 0);
                bool first = true;
                for (int v = 0; v < u; ++v) first &= addr[v] != addr[u];
                if (first) worst = std::max(worst, ++cnt[addr[u] & 7]);
              }
              my_tot += worst;
            }
          }
        }
        for (int t = 0; t < 256; ++t) m[size_t(t)] = mend[size_t(t)];
      }
    }
    std::lock_guard<std::mutex> lock(mu);
    tot += my_tot;
    ideal += my_ideal;
  };
  const int nthreads = std::max(1, int(std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) pool.emplace_back(work);
  for (auto& th : pool) th.join();
  return {tot, ideal};
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

  ForwardSchedule& F = p.fwd;
  // Checks and diagnostics of the final schedule (planned or from the cache).
  auto finish = [&]() {
    F.any_narrow = false;
    for (const int4& c : F.cta) F.any_narrow |= ((c.z >> 5) & 7) != 0;
    if (const char* ve = std::getenv("RK_VERIFY_PLAN"); ve && ve[0] == '1') verify_forward_schedule(p, ray_geom, ray_aux);
    if (const char* me = std::getenv("RK_PLAN_MODEL"); me && me[0] == '1') {
      const auto w = model_wavefronts(p, ray_geom, ray_aux);
      std::fprintf(stderr, "[rk] forward schedule: modelled shared-memory load wavefronts per image group %.0f "
                   "(%.4fx conflict-free)\n", w.first, w.first / std::max(w.second, 1.0));
    }
    if (std::getenv("RK_DEBUG_PLAN")) {
      int64_t ntr = 0;
      for (const int4& c : F.cta) ntr += c.z & 1;
      const uint64_t hsh = schedule_hash(F);  // A/B: same schedule?
      std::fprintf(stderr, "[rk] forward schedule: hash %016llx%s\n", (unsigned long long)hsh,
                   F.from_cache ? " (from the plan cache)" : "");
      std::fprintf(stderr, "[rk] forward schedule: lane mappings (angles per quarter warp 1/2/4/8) %d/%d/%d/%d CTAs, "
                   "simulated wavefronts %.3fx conflict-free\n", F.mapping_count[0], F.mapping_count[1],
                   F.mapping_count[2], F.mapping_count[3], F.sim_cost / std::max(F.sim_ideal, 1.0));
      std::fprintf(stderr,
                   "[rk] forward schedule: CTA %d angles x %d cell blocks of %d cells, %zu CTAs (%lld transposed), "
                   "%zu boxes (%.1f per CTA), max box %lld cells (%.1f KB), staged texels per image %.2fM\n",
                   F.shape_aa, F.shape_db, F.cta.empty() ? 32 : cells_per_warp(F.cta[0].z), F.cta.size(),
                   (long long)ntr, F.boxes.size(),
                   double(F.boxes.size()) / double(std::max<size_t>(F.cta.size(), 1)), (long long)F.max_box,
                   double(F.max_box) * 16.0 / 1024.0, double(F.staged_texels) / 1e6);
    }
  };
  const std::vector<unsigned char> cache_key = schedule_cache_key(p);
  const std::string cache_path = schedule_cache_path(cache_key);
  if (load_schedule(cache_path, cache_key, P2, F)) {
    F.from_cache = true;
    finish();
    return;
  }
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
  const int64_t nkb = (nd + 31) / 32;  // 32-cell detector blocks
  int cw = 32;                         // detector cells per warp of the tier being planned
  // Each chunk's layout is chosen from `refine_steps` of the kernel's own lockstep iterations in
  // the chunk (lane m = m_start + q), evenly spaced: cfg2 modelled wavefronts 1.272x -> 1.242x of
  // conflict-free, forward 9.46 -> 9.26 ms (r2).  RK_FWD_REFINE_STEPS=0: the r1 planner's three
  // sampled t's.  (The model: RK_PLAN_MODEL=1, within 0.1 % of ncu's count.)
  const char* prs = std::getenv("RK_FWD_REFINE_STEPS");
  const int refine_steps = prs ? std::max(0, std::atoi(prs)) : 6;
  // RK_FWD_ORDER_DESCENT=n: n passes of coordinate descent over per-lane tap orders per chunk.
  // Off: the exact model gives 0.4-0.6 % fewer wavefronts (cfg2 1.2418x -> 1.2357x, cfg3 1.3367x ->
  // 1.3291x) for 4x the planning time (r2).
  const char* pod = std::getenv("RK_FWD_ORDER_DESCENT");
  const int order_descent = pod ? std::max(0, std::atoi(pod)) : 0;
  const char* pml = std::getenv("RK_FWD_MAXLEN");  // experiment: cap on a chunk's t-length
  const double max_len = pml ? std::atof(pml) : 48.0;
  const char* pcl = std::getenv("RK_FWD_CTA_LOCKSTEP");  // experiment: "q,step" lockstep samples per t
  const bool cta_lockstep = pcl != nullptr;
  int cta_q = 1, cta_qstep = 0;
  if (pcl) std::sscanf(pcl, "%d,%d", &cta_q, &cta_qstep);
  cta_q = std::max(1, cta_q);
  const char* pce = std::getenv("RK_FWD_CHUNK_LAYOUT");
  const bool per_chunk_layout = !(pce && pce[0] == '0');
  int64_t budget = F.box_budget;

  struct Shape {
    int aa, db;
  };

  // Box of the samples of `warps` (8 x {angle, first cell}) with t in [ta, tb] (+1 slack).
  auto box_of = [&](const int2* wa, double ta, double tb) {
    double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
    for (int w = 0; w < 8; ++w) {
      if (wa[w].x < 0) continue;
      for (int l = 0; l < cw; ++l) {
        const int64_t kk = int64_t(wa[w].y) + l;
        if (kk >= nd) break;
        const RayD& ry = rays[size_t(int64_t(wa[w].x) * nd + kk)];
        if (ry.n == 0) continue;
        const double u0 = std::max(ta - 1.0, ry.t0), u1 = std::min(tb + 1.0, ry.t1);
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
    Box b{0, 0, 0, 0};
    if (xmin > xmax) return b;
    const int64_t c0 = std::max<int64_t>(0, int64_t(std::floor(xmin)) - 1);
    const int64_t c1 = std::min<int64_t>(P2 - 1, int64_t(std::floor(xmax)) + 2);
    const int64_t r0 = std::max<int64_t>(0, int64_t(std::floor(ymin)) - 1);
    const int64_t r1 = std::min<int64_t>(P2 - 1, int64_t(std::floor(ymax)) + 2);
    return Box{r0, c0, r1 - r0 + 1, c1 - c0 + 1};
  };

  // Greedy chunking of one CTA for a layout: returns false if even the
  // shortest chunk overflows the budget.  Appends {r0|c0<<16, rows|cols<<16, pitch, t_end bits}.
  // refine (optional): per-chunk layout {tr, residue, swap} for the chunk
  // [t, tb] with box b; the CTA-wide layout when it returns false or its box
  // would not fit.
  using Refine = std::function<bool(double, double, int*, int*, int*)>;  // -> tr, residue, tap order
  auto chunk_cta = [&](const int2* wa, bool tr, int residue, int swap, std::vector<int4>* out, int64_t* staged,
                       int64_t* max_cells, bool* any_tr, const Refine& refine) -> bool {
    double t = t_lo;
    while (t < t_hi) {
      bool placed = false;
      for (double len : {48.0, 40.0, 32.0, 24.0, 16.0, 12.0, 8.0, 6.0, 4.0, 3.0, 2.0}) {
        if (len > max_len && len > 2.0) continue;
        const double tb = std::min(t + len, t_hi);
        Box b = box_of(wa, t, tb);
        if (b.empty()) {
          // nothing of this CTA here: skip ahead without a box
          t = tb;
          placed = true;
          break;
        }
        int64_t rows = tr ? b.cols : b.rows, cols = tr ? b.rows : b.cols;
        int pitch = pitch_for(cols, residue);
        if (rows * pitch > budget && len > 2.0) continue;
        if (rows * pitch > budget) return false;
        bool ctr = tr;
        int corder = order_of_swap(swap);
        int ctr_i = tr, cres = residue, cord = corder;
        if (refine && refine(t, tb, &ctr_i, &cres, &cord)) {
          const int64_t rr = ctr_i ? b.cols : b.rows, cc = ctr_i ? b.rows : b.cols;
          const int pp = pitch_for(cc, cres);
          if (rr * pp <= budget) ctr = ctr_i != 0, corder = cord, rows = rr, cols = cc, pitch = pp;
        }
        if (out) {
          const int64_t r0 = ctr ? b.c0 : b.r0, c0 = ctr ? b.r0 : b.c0;
          float tend = tb >= t_hi ? INFINITY : float(tb);
          int tbits;
          std::memcpy(&tbits, &tend, 4);
          // pitch | orientation << 16 | per-lane tap order << 17 (kernels.cu)
          out->push_back(make_int4(int(r0 | (c0 << 16)), int(rows | (cols << 16)),
                                   pitch | (int(ctr) << 16) | (corder << 17), tbits));
        }
        if (any_tr) *any_tr |= ctr;
        if (staged) *staged += rows * cols;
        if (max_cells) *max_cells = std::max(*max_cells, rows * pitch);
        t = tb;
        placed = true;
        break;
      }
      if (!placed) return false;
    }
    return true;
  };

  auto warps_of = [&](Shape sh) {
    const int64_t nkb_w = (nd + cw - 1) / cw;  // cw-cell detector blocks, one per warp
    const int ctas_a = int((na + sh.aa - 1) / sh.aa);
    const int ctas_k = int((nkb_w + sh.db - 1) / sh.db);
    std::vector<int2> warps(size_t(ctas_a) * ctas_k * 8, make_int2(-1, 0));
    for (int ca = 0; ca < ctas_a; ++ca)
      for (int ck = 0; ck < ctas_k; ++ck)
        for (int w = 0; w < sh.aa * sh.db; ++w) {
          const int64_t ai = int64_t(ca) * sh.aa + w / sh.db;
          const int64_t kb = int64_t(ck) * sh.db + w % sh.db;
          if (ai < na && kb < nkb_w) warps[size_t(ca * ctas_k + ck) * 8 + w] = make_int2(order[size_t(ai)], int(kb * cw));
        }
    return warps;
  };

  // Per-CTA layout by simulation, then greedy chunks (parallel over CTAs).
  struct CtaPlan {
    int tr = 0, residue = 0, swap = 0, mapping = 0;
    bool ok = false;
    int64_t staged = 0, max_cells = 0;
    double cost = 0.0, ideal = 0.0;  // simulated wavefronts: chosen layout, conflict-free
    bool any_tr = false;             // some chunk stages the transposed image
    std::vector<int4> boxes;
  };
  // Layout (lane mapping, orientation, pitch, tap order) by simulation, then
  // greedy chunks, for one CTA's 8 warps {angle, first cell}.
  auto plan_cta = [&](const int2* wa, bool full8, CtaPlan& cp, std::vector<Pt>& sim) {
    // Lane mappings (kernels.cu): a quarter warp covers 2^lq neighbouring
    // angle slots x 8 >> lq neighbouring cells; lq = 0 (detector-major) is
    // the only one for partial CTA shapes.  Near-parallel lines of one
    // angle and short arcs of one cell's neighbouring angles conflict at
    // different directions, so each CTA takes the cheapest.  Positions at
    // a few aligned steps of the march, in lane order.
    auto lane_ray = [&](int lq, int w, int l, int& a_out, int64_t& k_out) {
      if (lq == 0) {
        a_out = l < cw ? wa[w].x : -1;  // narrow warps: lanes >= cw idle
        k_out = int64_t(wa[w].y) + l;
        return;
      }
      const int t = w * 32 + l;
      const int cq = t & ((8 >> lq) - 1), aq = (t >> (3 - lq)) & ((1 << lq) - 1);
      const int cg = (t >> 3) & ((4 << lq) - 1), ag = t >> (lq + 5);
      a_out = wa[(ag << lq) + aq].x;
      k_out = int64_t(wa[0].y) + cg * (8 >> lq) + cq;
    };
    double best = 1e300;
    for (int mapping = 0; mapping < (full8 ? 4 : 1); ++mapping) {
      sim.clear();
      for (int st = 0; st < 8 * cta_q; ++st) {
        const double tt = t_lo + (t_hi - t_lo) * (0.06 + 0.88 * double(st / cta_q) / 7.0);
        const int qoff = (st % cta_q) * cta_qstep;  // lockstep iterations after a chunk start at tt
        for (int w = 0; w < 8; ++w)
          for (int l = 0; l < 32; ++l) {
            Pt q{NAN, NAN};
            int a;
            int64_t kk;
            lane_ray(mapping, w, l, a, kk);
            if (a >= 0 && kk < nd) {
              const RayD& ry = rays[size_t(int64_t(a) * nd + kk)];
              if (ry.n > 0 && tt >= ry.t0 && tt <= ry.t1) {
                double m = std::floor((tt - ry.t0) / ry.h);
                if (cta_lockstep) m = std::ceil((tt - ry.t0) / ry.h - 0.5) + double(qoff);
                const double t = ry.t0 + (m + 0.5) * ry.h;
                if (m < double(ry.n)) q = to_pixel(ry.ox + t * ry.dx, ry.oy + t * ry.dy, half);
              }
            }
            sim.push_back(q);
          }
      }
      if (mapping == 0) cp.ideal = ideal_cost(sim);
      for (int tr = 0; tr < 2; ++tr) {
        double costs[3][8];
        conflict_costs(sim, tr == 1, costs);
        for (int swap = 0; swap < 3; ++swap)
          for (int res = 0; res < 8; ++res) {
            const double c = costs[swap][res] * (1.0 + 1e-3 * tr + 1e-5 * swap + 1e-4 * mapping);
            if (c < best) best = c, cp.tr = tr, cp.residue = res, cp.swap = swap, cp.mapping = mapping;
          }
      }
    }
    cp.cost = best;
    // Per-chunk layout: the lane lines' bank pattern drifts along the march
    // (sample stagger; fan beam: ray spacing grows with the distance to the
    // source), so each chunk re-picks orientation, pitch and tap order for
    // the CTA's lane mapping from a few steps inside it.
    std::vector<Pt> csim;
    const int mp = cp.mapping;
    Refine refine = [&](double ta, double tb, int* tr_o, int* res_o, int* sw_o) {
      csim.clear();
      if (refine_steps > 0) {
        // the kernel's lockstep iterations of this chunk (lane m = m_start + q), `refine_steps`
        // of them evenly spaced: the samples whose t lies in [ta, tb)
        int iters = 0;
        std::vector<int64_t> ms(256, 0), me(256, 0);
        std::vector<const RayD*> rl(256, nullptr);
        for (int w = 0; w < 8; ++w)
          for (int l = 0; l < 32; ++l) {
            int a;
            int64_t kk;
            lane_ray(mp, w, l, a, kk);
            if (a < 0 || kk >= nd) continue;
            const RayD& ry = rays[size_t(int64_t(a) * nd + kk)];
            if (ry.n == 0) continue;
            const int t = w * 32 + l;
            rl[size_t(t)] = &ry;
            ms[size_t(t)] = std::min<int64_t>(std::max<int64_t>(int64_t(std::ceil((ta - ry.t0) / ry.h - 0.5)), 0), ry.n);
            me[size_t(t)] = std::min<int64_t>(std::max<int64_t>(int64_t(std::ceil((tb - ry.t0) / ry.h - 0.5)), 0), ry.n);
            iters = std::max<int>(iters, int(me[size_t(t)] - ms[size_t(t)]));
          }
        const int ns = std::min(iters, refine_steps);
        for (int st = 0; st < ns; ++st) {
          const int64_t q = ns == 1 ? iters / 2 : int64_t(st) * (iters - 1) / (ns - 1);
          for (int t = 0; t < 256; ++t) {
            Pt pt{NAN, NAN};
            const RayD* ry = rl[size_t(t)];
            if (ry && ms[size_t(t)] + q < me[size_t(t)]) {
              const double tt = ry->t0 + (double(ms[size_t(t)] + q) + 0.5) * ry->h;
              pt = to_pixel(ry->ox + tt * ry->dx, ry->oy + tt * ry->dy, half);
            }
            csim.push_back(pt);
          }
        }
      }
      for (int st = 0; refine_steps == 0 && st < 3; ++st) {
        const double tt = ta + (tb - ta) * (0.2 + 0.3 * st);
        for (int w = 0; w < 8; ++w)
          for (int l = 0; l < 32; ++l) {
            Pt q{NAN, NAN};
            int a;
            int64_t kk;
            lane_ray(mp, w, l, a, kk);
            if (a >= 0 && kk < nd) {
              const RayD& ry = rays[size_t(int64_t(a) * nd + kk)];
              if (ry.n > 0 && tt >= ry.t0 && tt <= ry.t1) {
                const double m = std::floor((tt - ry.t0) / ry.h);
                const double t = ry.t0 + (m + 0.5) * ry.h;
                q = to_pixel(ry.ox + t * ry.dx, ry.oy + t * ry.dy, half);
              }
            }
            csim.push_back(q);
          }
      }
      double bc = 1e300;
      int bsw = 0;
      for (int tr = 0; tr < 2; ++tr) {
        double costs[3][8];
        conflict_costs(csim, tr == 1, costs);
        for (int sw = 0; sw < 3; ++sw)
          for (int res = 0; res < 8; ++res) {
            // ties keep the CTA-wide layout (no needless switches)
            const bool same = tr == cp.tr && res == cp.residue && sw == cp.swap;
            const double c = costs[sw][res] * (same ? 1.0 : 1.0 + 1e-3);
            if (c < bc) bc = c, *tr_o = tr, *res_o = res, bsw = sw;
          }
      }
      *sw_o = order_of_swap(bsw);
      if (bc < 1e300 && order_descent > 0) {
        // per-lane tap orders: coordinate descent over the 14 order bits from the best
        // odd-lane order, each candidate at its best pitch residue
        int order = *sw_o, res = *res_o;
        V8 cv;
        order_costs(csim, *tr_o == 1, order, cv);
        uint32_t best = cv[res];
        for (int pass = 0; pass < order_descent; ++pass) {
          bool improved = false;
          for (int bit = 0; bit < 14; ++bit) {
            const int cand = order ^ (1 << bit);
            order_costs(csim, *tr_o == 1, cand, cv);
            for (int r = 0; r < 8; ++r)
              if (cv[r] < best) best = cv[r], order = cand, res = r, improved = true;
          }
          if (!improved) break;
        }
        *sw_o = order;
        *res_o = res;
      }
      return bc < 1e300;
    };
    bool any_tr = false;
    cp.ok = chunk_cta(wa, cp.tr == 1, cp.residue, cp.swap, &cp.boxes, &cp.staged, &cp.max_cells, &any_tr,
                      per_chunk_layout ? refine : Refine());
    cp.any_tr = any_tr;
  };
  auto plan_shape = [&](Shape sh, std::vector<CtaPlan>& plans) {
    std::vector<int2> warps = warps_of(sh);
    const int ctas = int(warps.size() / 8);
    plans.assign(size_t(ctas), CtaPlan{});
    std::atomic<int> next{0};  // CTAs differ in work (ray lengths): hand them out in small blocks
    auto work = [&]() {
      std::vector<Pt> sim;
      for (int lo; (lo = next.fetch_add(4)) < ctas;)
        for (int cta = lo; cta < std::min(lo + 4, ctas); ++cta)
          plan_cta(&warps[size_t(cta) * 8], sh.aa == 8 && sh.db == 1 && cw == 32, plans[size_t(cta)], sim);
    };
    const char* pte = std::getenv("RK_PLAN_THREADS");  // planner threads (default: all host threads)
    const int want = pte ? std::atoi(pte) : int(std::thread::hardware_concurrency());
    const int nthreads = std::max(1, std::min<int>(want, ctas));
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t)
      pool.emplace_back(work);
    for (auto& th : pool) th.join();
    return warps;
  };

  // 8 angles x 32 cells is the reuse-friendly shape (adjacent angles of a sorted
  // list march nearly parallel rays).  Fallbacks, in order, when some CTA
  // cannot fit even its shortest chunk (sparse or scattered angle lists):
  // wider detector blocks, then a 192 KB budget (one CTA per SM), then CTAs
  // with idle warps (fewer rays, smaller boxes).
  struct Tier {
    Shape sh;
    int64_t budget;
    int cells = 32;  // detector cells per warp
  };
  // First choice: 54 KB boxes (four CTAs per SM); then 64 KB (three).
  const char* be = std::getenv("RK_FWD_BOX");
  const int64_t b0 = be ? std::max<int64_t>(512, std::atoll(be)) : F.box_budget;
  const int64_t b1 = std::max<int64_t>(b0, 4096);
  // Coarse detectors (spacing of several pixels) spread a warp's 32 rays over
  // hundreds of pixels, so no box fits: then warps of 16 .. 1 consecutive
  // cells (the other lanes idle), smallest boxes last.
  const Tier tiers[] = {{{8, 1}, b0},        {{8, 1}, b1},        {{4, 2}, b1},        {{2, 4}, b1},
                        {{1, 8}, b1},        {{8, 1}, 12288},    {{4, 2}, 12288},    {{4, 1}, 12288},
                        {{2, 1}, 12288},    {{1, 1}, 12288},    {{8, 1}, b0, 16},   {{8, 1}, b0, 8},
                        {{8, 1}, b1, 4},     {{8, 1}, 12288, 2}, {{8, 1}, 12288, 1}, {{1, 1}, 12288, 1}};
  for (const Tier& tier : tiers) {
    const Shape sh = tier.sh;
    if (sh.db > 1 && nkb < sh.db && sh.db != 8) continue;
    budget = tier.budget;
    cw = tier.cells;
    int ncl = 0;
    while ((32 >> ncl) > cw) ++ncl;
    std::vector<CtaPlan> plans;
    std::vector<int2> warps = plan_shape(sh, plans);
    bool ok = true;
    for (const CtaPlan& cp : plans) ok &= cp.ok;
    if (!ok && &tier == &tiers[0]) {
      // Keep the small boxes (occupancy) for every CTA: a CTA whose shortest
      // chunk overflows is replaced by CTAs marching halves of its angle
      // slots (the other warps idle), recursively.
      std::vector<int2> w2;
      std::vector<CtaPlan> p2;
      std::vector<Pt> sim;
      ok = true;
      std::function<void(const int2*, int, int)> split = [&](const int2* wa, int lo, int hi) {
        int2 sub[8];
        for (int w = 0; w < 8; ++w) sub[w] = (w >= lo && w < hi) ? wa[w] : make_int2(-1, wa[w].y);
        CtaPlan cp;
        plan_cta(sub, false, cp, sim);
        if (cp.ok) {
          w2.insert(w2.end(), sub, sub + 8);
          p2.push_back(std::move(cp));
        } else if (hi - lo > 1) {
          split(wa, lo, (lo + hi) / 2);
          split(wa, (lo + hi) / 2, hi);
        } else {
          ok = false;
        }
      };
      for (size_t c = 0; c < plans.size() && ok; ++c) {
        if (plans[c].ok) {
          w2.insert(w2.end(), warps.begin() + int64_t(c) * 8, warps.begin() + int64_t(c + 1) * 8);
          p2.push_back(std::move(plans[c]));
        } else {
          split(&warps[c * 8], 0, 8);
        }
      }
      if (ok) {
        warps = std::move(w2);
        plans = std::move(p2);
      }
    }
    if (!ok) continue;
    F.shape_aa = sh.aa;
    F.shape_db = sh.db;
    F.warps = std::move(warps);
    F.cta.assign(plans.size(), make_int4(0, 0, 0, 0));
    F.boxes.clear();
    F.max_box = 0;
    F.staged_texels = 0;
    F.any_transposed = false;
    F.sim_cost = F.sim_ideal = 0.0;
    for (int& mc : F.mapping_count) mc = 0;
    for (size_t c = 0; c < plans.size(); ++c) {
      const CtaPlan& cp = plans[c];
      // z: orientation | tap order << 1 | lane mapping << 3 | log2(32 / cells per warp) << 5 (kernels.cu)
      F.cta[c] = make_int4(int(F.boxes.size()), int(cp.boxes.size()),
                           cp.tr | (cp.swap << 1) | (cp.mapping << 3) | (ncl << 5), 0);
      F.sim_cost += cp.cost;
      F.sim_ideal += cp.ideal;
      F.mapping_count[cp.mapping & 3] += 1;
      F.boxes.insert(F.boxes.end(), cp.boxes.begin(), cp.boxes.end());
      F.max_box = std::max(F.max_box, cp.max_cells);
      F.staged_texels += cp.staged;
      F.any_transposed |= cp.any_tr;
    }
    // Launch order: longest CTAs first (a warp iterates as long as its longest
    // ray), so the hardware's in-order CTA dispatch packs the short ones into
    // the last wave (longest-processing-time list scheduling).  Only the order
    // of independent CTAs changes — every ray's arithmetic is the same.
    if (const char* oe = std::getenv("RK_FWD_ORDER"); !(oe && oe[0] == '0')) {
      const size_t nc = F.cta.size();
      std::vector<int64_t> work(nc, 0);
      for (size_t c = 0; c < nc; ++c)
        for (int w = 0; w < 8; ++w) {
          const int2 wa = F.warps[c * 8 + size_t(w)];
          if (wa.x < 0) continue;
          int64_t longest = 0;
          for (int l = 0; l < cells_per_warp(F.cta[c].z) && int64_t(wa.y) + l < nd; ++l)
            longest = std::max(longest, rays[size_t(int64_t(wa.x) * nd + wa.y + l)].n);
          work[c] += longest;
        }
      std::vector<size_t> idx(nc);
      for (size_t c = 0; c < nc; ++c) idx[c] = c;
      std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return work[a] > work[b]; });
      std::vector<int4> cta2(nc);
      std::vector<int2> warps2(F.warps.size());
      for (size_t c = 0; c < nc; ++c) {
        cta2[c] = F.cta[idx[c]];
        std::copy_n(F.warps.begin() + int64_t(idx[c] * 8), 8, warps2.begin() + int64_t(c * 8));
      }
      F.cta = std::move(cta2);
      F.warps = std::move(warps2);
    }
    store_schedule(cache_path, cache_key, F);
    finish();
    return;
  }
  throw ValidationError("forward schedule: a staged image box exceeds shared memory even for the shortest chunk");
}

}  // namespace rk
