// On-disk cache of forward schedules (fwd_plan.cpp), keyed by the geometry.
//
// Planning a forward schedule costs 0.1-1 s of host time per geometry (the
// bank-conflict simulation); the reference's forward (projector.cpp:228-236)
// has no such step, so a one-shot projection would pay it every process.
// Like the reference's shearlet plan cache (make_plan_cached,
// shearlet.cpp:202-251) the result is stored once per geometry and reused:
//   $RK_PLAN_CACHE (a directory; "0" or "off" disables), else
//   $XDG_CACHE_HOME/radon_b200, else $HOME/.cache/radon_b200.
// The file holds the full key (planner version, geometry with every angle's
// bits, the planner's environment knobs), so a hash collision or a stale
// planner can never hand back the wrong schedule; any read problem falls back
// to planning.  Writes go to a temporary file renamed into place (atomic for
// concurrent processes).
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rk_internal.hpp"

namespace rk {

namespace {

// Bump whenever fwd_plan.cpp's decisions change (the key then misses).
constexpr uint32_t kPlannerVersion = 5;  // 5: narrow-warp CTAs (cfg.z bits 5-7)
constexpr char kMagic[4] = {'R', 'K', 'F', 'S'};

void put(std::vector<unsigned char>& b, const void* d, size_t n) {
  const auto* c = static_cast<const unsigned char*>(d);
  b.insert(b.end(), c, c + n);
}
template <class T>
void put_v(std::vector<unsigned char>& b, const T& v) {
  put(b, &v, sizeof(T));
}
void put_env(std::vector<unsigned char>& b, const char* name) {
  const char* v = std::getenv(name);
  const std::string s = std::string(name) + "=" + (v ? v : "");
  put_v(b, uint32_t(s.size()));
  put(b, s.data(), s.size());
}

std::string cache_dir() {
  if (const char* d = std::getenv("RK_PLAN_CACHE")) {
    if (!std::strcmp(d, "0") || !std::strcmp(d, "off") || !*d) return "";
    return d;
  }
  if (const char* x = std::getenv("XDG_CACHE_HOME"); x && *x) return std::string(x) + "/radon_b200";
  if (const char* h = std::getenv("HOME"); h && *h) return std::string(h) + "/.cache/radon_b200";
  return "";
}

bool make_dirs(const std::string& path) {
  std::string cur;
  for (size_t i = 0; i <= path.size(); ++i) {
    if (i == path.size() || path[i] == '/') {
      if (!cur.empty() && mkdir(cur.c_str(), 0755) != 0 && errno != EEXIST) return false;
    }
    if (i < path.size()) cur.push_back(path[i]);
  }
  return true;
}

uint64_t fnv1a(const std::vector<unsigned char>& b) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : b) h = (h ^ c) * 1099511628211ull;
  return h;
}

template <class T>
bool read_vec(FILE* f, std::vector<T>& v) {
  uint64_t n = 0;
  if (std::fread(&n, sizeof n, 1, f) != 1 || n > (uint64_t(1) << 32)) return false;
  v.resize(size_t(n));
  return n == 0 || std::fread(v.data(), sizeof(T), size_t(n), f) == size_t(n);
}
template <class T>
bool write_vec(FILE* f, const std::vector<T>& v) {
  const uint64_t n = v.size();
  return std::fwrite(&n, sizeof n, 1, f) == 1 && (n == 0 || std::fwrite(v.data(), sizeof(T), v.size(), f) == v.size());
}

}  // namespace

uint64_t schedule_hash(const ForwardSchedule& F) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* d, size_t n) {
    for (size_t b = 0; b < n; ++b) h = (h ^ static_cast<const unsigned char*>(d)[b]) * 1099511628211ull;
  };
  mix(F.boxes.data(), F.boxes.size() * sizeof(int4));
  mix(F.cta.data(), F.cta.size() * sizeof(int4));
  mix(F.warps.data(), F.warps.size() * sizeof(int2));
  return h;
}

std::vector<unsigned char> schedule_cache_key(const Plan& p) {
  std::vector<unsigned char> k;
  put_v(k, kPlannerVersion);
  put_v(k, int32_t(p.g.kind));
  put_v(k, p.s);
  put_v(k, p.na);
  put_v(k, p.nd);
  put_v(k, p.g.det_spacing);
  put_v(k, p.g.source_distance);
  put_v(k, p.g.det_distance);
  put_v(k, p.g.step);
  put(k, p.angles.data(), p.angles.size() * sizeof(double));
  put_v(k, p.fwd.box_budget);
  for (const char* e : {"RK_FWD_CHUNK_LAYOUT", "RK_FWD_BOX", "RK_FWD_ORDER", "RK_FWD_REFINE_STEPS", "RK_FWD_MAXLEN",
                        "RK_FWD_CTA_LOCKSTEP", "RK_FWD_ORDER_DESCENT"})
    put_env(k, e);
  return k;
}

std::string schedule_cache_path(const std::vector<unsigned char>& key) {
  const std::string dir = cache_dir();
  if (dir.empty()) return "";
  char name[64];
  std::snprintf(name, sizeof name, "/fwd_%016llx.rkfs", (unsigned long long)fnv1a(key));
  return dir + name;
}

bool load_schedule(const std::string& path, const std::vector<unsigned char>& key, int64_t padded, ForwardSchedule& F) {
  if (path.empty()) return false;
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  bool ok = false;
  do {
    char magic[4];
    uint32_t version = 0;
    std::vector<unsigned char> k;
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kMagic, 4) != 0) break;
    if (std::fread(&version, sizeof version, 1, f) != 1 || version != kPlannerVersion) break;
    if (!read_vec(f, k) || k != key) break;
    ForwardSchedule G;
    G.box_budget = F.box_budget;
    int32_t any_tr = 0;
    if (std::fread(&G.shape_aa, sizeof G.shape_aa, 1, f) != 1 || std::fread(&G.shape_db, sizeof G.shape_db, 1, f) != 1 ||
        std::fread(&G.max_box, sizeof G.max_box, 1, f) != 1 ||
        std::fread(&G.staged_texels, sizeof G.staged_texels, 1, f) != 1 || std::fread(&any_tr, sizeof any_tr, 1, f) != 1 ||
        std::fread(&G.sim_cost, sizeof G.sim_cost, 1, f) != 1 || std::fread(&G.sim_ideal, sizeof G.sim_ideal, 1, f) != 1 ||
        std::fread(G.mapping_count, sizeof G.mapping_count, 1, f) != 1)
      break;
    G.any_transposed = any_tr != 0;
    if (!read_vec(f, G.boxes) || !read_vec(f, G.cta) || !read_vec(f, G.warps)) break;
    if (G.cta.size() * 8 != G.warps.size()) break;
    // a damaged file must not reach the kernel: every CTA's box range lies in
    // the box table, every box inside the padded image and its staging budget
    bool sane = G.max_box > 0 && G.max_box <= 12288;
    for (const int4& c : G.cta) sane &= c.x >= 0 && c.y >= 0 && size_t(c.x) + size_t(c.y) <= G.boxes.size();
    for (const int4& b : G.boxes) {
      const int64_t r0 = b.x & 0xffff, c0 = b.x >> 16, rows = b.y & 0xffff, cols = b.y >> 16, pitch = b.z & 0xffff;
      sane &= r0 + rows <= padded && c0 + cols <= padded && cols <= pitch && rows * pitch <= G.max_box;
    }
    if (!sane) break;
    F = std::move(G);
    ok = true;
  } while (false);
  std::fclose(f);
  return ok;
}

void store_schedule(const std::string& path, const std::vector<unsigned char>& key, const ForwardSchedule& F) {
  if (path.empty()) return;
  const std::string dir = path.substr(0, path.rfind('/'));
  if (!make_dirs(dir)) return;
  // one temporary file per writer (threads of one process may plan the same
  // geometry at once): the rename then publishes only complete files
  static std::atomic<unsigned> serial{0};
  const std::string tmp = path + ".tmp." + std::to_string(long(getpid())) + "." + std::to_string(serial.fetch_add(1));
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;
  const int32_t any_tr = F.any_transposed ? 1 : 0;
  bool ok = std::fwrite(kMagic, 1, 4, f) == 4 && std::fwrite(&kPlannerVersion, sizeof kPlannerVersion, 1, f) == 1 &&
            write_vec(f, key) && std::fwrite(&F.shape_aa, sizeof F.shape_aa, 1, f) == 1 &&
            std::fwrite(&F.shape_db, sizeof F.shape_db, 1, f) == 1 && std::fwrite(&F.max_box, sizeof F.max_box, 1, f) == 1 &&
            std::fwrite(&F.staged_texels, sizeof F.staged_texels, 1, f) == 1 &&
            std::fwrite(&any_tr, sizeof any_tr, 1, f) == 1 && std::fwrite(&F.sim_cost, sizeof F.sim_cost, 1, f) == 1 &&
            std::fwrite(&F.sim_ideal, sizeof F.sim_ideal, 1, f) == 1 &&
            std::fwrite(F.mapping_count, sizeof F.mapping_count, 1, f) == 1 && write_vec(f, F.boxes) &&
            write_vec(f, F.cta) && write_vec(f, F.warps);
  ok &= std::fclose(f) == 0;
  if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) std::remove(tmp.c_str());
}

}  // namespace rk
