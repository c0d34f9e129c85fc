// Internal declarations shared by the host plan code, the C ABI and the
// CUDA kernels of the B200 Radon projector.  Not part of the public ABI
// (include/radon_b200.h is).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "radon_b200.h"

namespace rk {

// ----------------------------------------------------------------- errors
// Mirrors the reference's exception taxonomy (errors.hpp:9-40); the C ABI
// maps them onto rk_status codes.
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

void cuda_check(cudaError_t e, const char* what);
#define RK_CUDA(call) ::rk::cuda_check((call), #call)

// Makes `device` current for the rest of the enclosing C-ABI call.  The first
// switch inside a call remembers the caller's device, and the call restores it
// on return (capi.cpp DeviceScope), so a call on a cuda:1 plan never moves the
// calling thread's current device — torch shares that context state.
void set_device(int device);

// ----------------------------------------------------------------- device buffers
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { release(); }
  void release();
  // grows (never shrinks); contents are not preserved
  void reserve(size_t n);
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

// ----------------------------------------------------------------- layouts
// Packed ("image-interleaved") layouts used inside the library.  Four batch
// elements share one 16-byte texel so that one 128-bit shared-memory load
// delivers a tap for four images: the index/weight arithmetic of a ray
// sample or pixel/angle pair is paid once per four images.
//   image : [G][s+2][s+2] float4, one zero texel of border on every side
//           (the reference's zero padding, projector.cpp:57-60)
//   sino  : [G][n_angles][det_count] float4
// with G = ceil(batch / 4); missing images of the last group are zero.
constexpr int kPack = 4;

inline int64_t groups_of(int64_t batch) { return (batch + kPack - 1) / kPack; }

// fp16 storage (user-facing projector / FBP calls, batch > 1): eight images
// per 16-byte texel, stored as half — exact, because the values are halves
// already — so each shared-memory tap load serves twice the images; the
// arithmetic stays fp32 and per image identical to the float4 layout.
constexpr int kPackH8 = 8;
inline int64_t groups_of_h8(int64_t batch) { return (batch + kPackH8 - 1) / kPackH8; }
bool use_h8(int dtype, int64_t batch);

// ----------------------------------------------------------------- forward schedule
// fp64 ray after the reference's clip prologue (projector.cpp:66-78)
struct RayD {
  double ox, oy, dx, dy;  // origin and unit direction (world coordinates)
  double t0, t1, h;       // clipped parameter range and sample spacing
  int64_t n;              // samples (0: the ray misses the image)
};

struct ForwardSchedule {
  int64_t box_budget = 3456;       // float4 cells per staged box (54 KB: four CTAs per SM)
  int shape_aa = 8, shape_db = 1;  // angles x 32-cell detector blocks per CTA
  int64_t max_box = 0;             // largest rows * pitch over all boxes (float4 cells)
  int64_t staged_texels = 0;       // per image group, all CTAs and chunks
  bool any_transposed = false;
  bool any_narrow = false;         // some CTA runs narrow warps (cfg.z bits 5-7 nonzero)
  double sim_cost = 0.0, sim_ideal = 0.0;  // planner's simulated shared-memory wavefronts (chosen, conflict-free)
  bool from_cache = false;                 // loaded from the on-disk schedule cache (plan_cache.cpp)
  int mapping_count[4] = {0, 0, 0, 0};      // CTAs per lane mapping (log2 angles per quarter warp)
  // per chunk {row0 | col0 << 16, rows | cols << 16, pitch, t_end (float bits; inf = last)},
  // in staged-image coordinates, CTA after CTA
  std::vector<int4> boxes;
  std::vector<int4> cta;    // per CTA {first box, box count, bit0 transposed | bits1-2 lane tap order | bits3-4 lane mapping, 0}
  std::vector<int2> warps;  // per CTA x 8 warps {angle (-1: idle), first detector cell}
};

// ----------------------------------------------------------------- host pipelines
// Scratch of the reference-shaped host-buffer calls (rk_*_host): chunks of the
// batch stream through kSlots non-blocking streams, each with its own device
// buffers, so one chunk's copy-in, another's kernels and a third's copy-out
// overlap.  Grown on demand, kept for the owner's lifetime (no per-call
// allocation once warm).
struct HostPipeline {
  static constexpr int kSlots = 3;
  cudaStream_t streams[kSlots] = {nullptr, nullptr, nullptr};
  DeviceBuffer in[kSlots], out[kSlots], pk[kSlots], pkt[kSlots];
  HostPipeline() = default;
  HostPipeline(const HostPipeline&) = delete;
  HostPipeline& operator=(const HostPipeline&) = delete;
  ~HostPipeline();
  void synchronize();  // waits for every slot's stream (errors ignored and cleared)
};

// ----------------------------------------------------------------- plan
struct Plan;
void build_forward_plan(Plan& p, const std::vector<RayD>& rays, std::vector<float4>& ray_geom,
                        std::vector<float4>& ray_aux);

// On-disk schedule cache (plan_cache.cpp): key = planner version + geometry
// + planner knobs; path "" when the cache is disabled.
std::vector<unsigned char> schedule_cache_key(const Plan& p);
std::string schedule_cache_path(const std::vector<unsigned char>& key);
bool load_schedule(const std::string& path, const std::vector<unsigned char>& key, int64_t padded, ForwardSchedule& F);
uint64_t schedule_hash(const ForwardSchedule& F);  // FNV-1a over boxes, CTA records, warps
void store_schedule(const std::string& path, const std::vector<unsigned char>& key, const ForwardSchedule& F);

// Builds and uploads the plan's forward schedule once (plan.cpp); every
// forward launch path calls it first.
void ensure_forward_schedule(Plan& p);

struct Plan {
  int device = 0;
  rk_geometry g{};              // resolved; g.angles -> angles.data()
  std::vector<double> angles;
  int64_t s = 0, na = 0, nd = 0;
  int64_t forward_samples = 0;  // exact algorithmic work per image

  // forward: one record per ray (a * nd + k), built in fp64 on the host
  DeviceBuffer ray_geom;   // float4 {px0, py0, hx, hy} in padded pixel coordinates
  DeviceBuffer ray_aux;    // float4 {h, n (int bits), t0, 1/h}
  // forward schedule (fwd_plan.cpp): CTA = A angles x W detectors; the rays
  // are marched chunk by chunk along t, each chunk's image footprint (box) is
  // staged in shared memory
  ForwardSchedule fwd;      // built on the first forward call (ensure_forward_schedule)
  std::once_flag fwd_once;
  DeviceBuffer fwd_boxes;  // int4 per chunk (see ForwardSchedule::boxes)
  DeviceBuffer fwd_cta;    // int4 per CTA
  DeviceBuffer fwd_warps;  // int2 {angle, first detector} per (cta, warp); angle -1 = idle
  // backprojection: per-angle trig in fp64
  DeviceBuffer trig;       // double2 {cos, sin}
  int bp_window = 0;       // staged detector cells per (tile, angle), widest tile
  int bp_angle_chunk = 0;  // angles staged per pass, widest tile
  int bp_cells = 0;        // staged cells per pass (shared memory), all tiles
  int bp_cells_narrow = 0; // the same for the NARROW kernel (seven CTAs per SM)
  DeviceBuffer bp_tile_window;  // int per 32x32 tile: its staged cells per angle
  bool bp_fan_fp64 = false;  // fan beam with the source close to the image: fp64 pixel map

  // scratch (serialised by `mu`; `scratch_free` orders reuse across streams)
  std::mutex mu;
  DeviceBuffer packed_image, packed_image_t, packed_sino;
  cudaEvent_t scratch_free = nullptr;
  HostPipeline pipe;  // host-buffer (*_host) calls
  // solver scratch
  DeviceBuffer solver_a, solver_b, solver_c, solver_d, solver_scalars;

  ~Plan();
};

struct Filter {
  int device = 0;
  int kind = 0;
  int64_t det_count = 0;
  int64_t padded = 0;
  std::vector<double> response;   // padded/2+1 bins (double)
  std::vector<float> response_f;  // same, float (sino_filter.cpp:89)
  DeviceBuffer d_response;        // float, padded/2+1
  DeviceBuffer d_twiddle;         // float2, padded/2 (forward twiddles)
  DeviceBuffer d_twiddle_stage;   // float2, padded - 1: the same values per radix-2 stage (filter.cu)
  HostPipeline pipe;              // rk_filter_sinogram_host
  std::mutex mu;
};

// Alpha-shearlet frame (shearlet_plan.cpp / shearlet.cu; reference shearlet.cpp)
struct Shearlet {
  int device = 0;
  int64_t height = 0, width = 0, n_coeff = 0;
  std::vector<double> alphas, scales;
  std::vector<double> multipliers;  // n_coeff x h x w (fp64, natural layout)
  // device tables (shearlet.cu): coefficient pairs {M_2j, M_2j+1} per bin in
  // bit-reversed row and column order (the order the DIF passes leave spectra
  // in), and the n/2 forward twiddles; fp32 built with the plan, fp64 on first use
  DeviceBuffer d_mult2, d_twiddle;
  DeviceBuffer d_mult2_64, d_twiddle64;
  // grids that are not a power of two (shearlet_generic.cu): natural-order
  // pairs and the n-entry DFT table
  DeviceBuffer g_mult2, g_twiddle, g_mult2_64, g_twiddle64;
  DeviceBuffer work_a, work_b;      // spectra scratch
  std::mutex mu;
  // work_a / work_b reuse across streams: every enqueue waits on and records
  // this event (capi.cpp ShearletLease; created on first device use)
  cudaEvent_t scratch_free = nullptr;
  Shearlet() = default;
  Shearlet(const Shearlet&) = delete;
  Shearlet& operator=(const Shearlet&) = delete;
  ~Shearlet();
};
// stored != nullptr: n_coeff x h x w multipliers from a plan cache, used verbatim
void build_shearlet(Shearlet& sp, int64_t height, int64_t width, const std::vector<double>& alphas,
                    const double* stored = nullptr);
void upload_shearlet(Shearlet& sp);
void shearlet_forward(Shearlet& sp, int dtype, const void* image, int64_t batch, void* coeff, cudaStream_t st);
void shearlet_backward(Shearlet& sp, int dtype, const void* coeff, int64_t batch, void* image, cudaStream_t st);
// ADMM fusions (fp32, user layouts): z1 = shrink(SH(f) + u1, thresh_k), u1 += SH(f) - z1
// (non-finite u1 -> atomicMin(flag, iteration)); image = SH'(z1 - u1)
void shearlet_admm_shrink(Shearlet& sp, const float* f, int64_t batch, float* z1, float* u1, const float* thresh,
                          int* flag, const int* iteration, cudaStream_t st);
void shearlet_admm_synth(Shearlet& sp, const float* z1, const float* u1, int64_t batch, float* image,
                         cudaStream_t st);
// grids that are not a power of two (shearlet_generic.cu): the same transforms
// by DFT-matrix contractions; GenericAdmm non-null = the ADMM shrink store
inline bool shearlet_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
struct GenericAdmm {
  float* z1 = nullptr;
  float* u1 = nullptr;
  const float* thresh = nullptr;
  int* flag = nullptr;
  const int* iteration = nullptr;
};
template <class C>
void build_generic_tables(const Shearlet& sp, std::vector<C>& mult2, std::vector<C>& tw);
void upload_shearlet_generic(Shearlet& sp);
void shearlet_forward_generic(Shearlet& sp, int dtype, const void* image, int64_t batch, void* coeff,
                              const GenericAdmm& admm, cudaStream_t st);
void shearlet_backward_generic(Shearlet& sp, int dtype, const void* coeff, const void* sub, int64_t batch,
                               void* image, cudaStream_t st);

// CG system coefficients: (c0 A'A + c1 I) (solver.cu cg_packed)
struct CgSystem {
  float c0, c1;
};

// l1-shearlet ADMM state (admm.cu; reference admm.cpp:111-163).  Radon-side
// vectors in the packed image layout, shearlet-side split/dual variables in the
// coefficient layout [B][K][n][n]; fp32 throughout (the reference's float path).
struct Admm {
  Plan* plan = nullptr;
  Shearlet* sh = nullptr;
  int dtype = 1;
  int64_t batch = 0;
  CgSystem sys{0.f, 0.f};
  float p0f = 0.f, p1f = 0.f;
  int inner = 0;
  int64_t iterations_done = 0;
  int failed = -1;  // first outer iteration whose state turned non-finite
  DeviceBuffer packed;   // F, BP, Z2, U2, CGY, 4 CG work planes
  DeviceBuffer sino;     // packed sinogram scratch
  DeviceBuffer user;     // fU, shU  ([B][n][n] fp32)
  DeviceBuffer coeff;    // z1, u1   ([B][K][n][n] fp32)
  DeviceBuffer small;    // thresholds, flags, CG scalars
  float4* F = nullptr;
  float4* BP = nullptr;
  float4* Z2 = nullptr;
  float4* U2 = nullptr;
  float4* CGY = nullptr;
  float4* work = nullptr;
  float* fU = nullptr;
  float* shU = nullptr;
  float* z1 = nullptr;
  float* u1 = nullptr;
  float* thresh = nullptr;
  int* flags = nullptr;  // [0] divergence iteration, [1] CG non-positive curvature
  int* iter_dev = nullptr;  // the current outer iteration, advanced on the device (graph replays)
  void* cg_scalars = nullptr;
  // One outer iteration captured as a CUDA graph and replayed (admm_iterate):
  // a batch-1 iteration is ~460 short launches.  Valid while the shearlet
  // plan's scratch keeps its addresses (graph_key); replayed on graph_stream,
  // ordered after / before the caller's stream by events.
  cudaGraphExec_t graph = nullptr;
  cudaStream_t graph_stream = nullptr;
  cudaEvent_t graph_in = nullptr, graph_out = nullptr;
  const void* graph_key[2] = {nullptr, nullptr};
  Admm() = default;
  Admm(const Admm&) = delete;
  Admm& operator=(const Admm&) = delete;
  ~Admm();
};
// bp = A'y, zero state; thresholds[k] = w_k p0 / p1 in fp64, used as float (admm.cpp:129-140)
void admm_init(Admm& a, const void* d_sino, const std::vector<double>& thresholds, cudaStream_t st);
// n outer iterations (admm.cpp:146-160); returns the first failed iteration or -1
int64_t admm_iterate(Admm& a, int64_t n, cudaStream_t st);
// which: 0 f, 1 z1, 2 u1, 3 z2, 4 u2 -> dst in the storage dtype
void admm_read(Admm& a, int which, int dtype, void* dst, cudaStream_t st);

// ----------------------------------------------------------------- host helpers (plan.cpp)
rk_geometry resolve_geometry(const rk_geometry& in);
void build_plan(Plan& p);
void build_filter(Filter& f, int kind, int64_t det_count);
const char* filter_kind_name(int kind);
int filter_kind_from_name(const std::string& name);

// ----------------------------------------------------------------- launchers (kernels.cu / filter.cu)
// All launchers enqueue on `stream` and never synchronise.
void launch_pack_images(int dtype, const void* src, int64_t batch, int64_t s, float4* dst, cudaStream_t st);
void launch_pack_images_h8(const void* src, int64_t batch, int64_t s, float4* dst, cudaStream_t st);
void launch_pack_sino_h8(const void* src, int64_t batch, int64_t na, int64_t nd, float4* dst, cudaStream_t st);
void launch_pack_sino(int dtype, const void* src, int64_t batch, int64_t na, int64_t nd, float4* dst,
                      cudaStream_t st);
// Kernel epilogues.  kOutUser: user layout in the storage dtype (the default
// reference-shaped result); kOutPacked: packed float4 layout (values narrowed
// through the dtype first); forward kOutResidual: packed (A x - y); backprojection
// kOutAxpy: packed x <- (-alpha) * (A' r) + x with a non-finite flag.
// kOutSystem: packed out = c0 * (A' s) + c1 * src (the ADMM CG system, admm.cpp:142).
enum { kOutUser = 0, kOutPacked = 1, kOutResidual = 2, kOutAxpy = 3, kOutSystem = 4 };
struct FwdEpilogue {
  int mode = kOutUser;
  float4* packed = nullptr;       // [G][na][nd]
  const float4* resid = nullptr;  // y for kOutResidual, same layout
};
struct BpEpilogue {
  int mode = kOutUser;
  float4* packed = nullptr;  // [G][s+2][s+2] (interior written)
  float neg_alpha = 0.f;     // kOutAxpy
  int* flag = nullptr;       // kOutAxpy: atomicMin(iteration) on a non-finite iterate
  int iteration = 0;
  const float4* src = nullptr;  // kOutSystem
  float c0 = 0.f, c1 = 0.f;
};

// packed image -> its transpose ([G][s+2][s+2], rows <-> columns)
void launch_transpose_images(const float4* src, int64_t groups, int64_t s, float4* dst, cudaStream_t st);
// packed_image_t is only read when the schedule has transposed CTAs
void launch_forward(const Plan& p, const float4* packed_image, const float4* packed_image_t, int64_t batch,
                    int dtype, void* sino, cudaStream_t st, FwdEpilogue epi = FwdEpilogue{});
void launch_backproject(const Plan& p, const float4* packed_sino, int64_t batch, int dtype, void* image,
                        cudaStream_t st, BpEpilogue epi = BpEpilogue{});
// filter: rows of det_count in `dtype`; writes either the user layout
// (`out`, dtype) or, when `packed_out` is set, the packed sino layout.
void launch_filter(const Filter& f, int dtype, const void* in, int64_t batch, int64_t n_angles, void* out,
                   float4* packed_out, cudaStream_t st);

size_t dtype_size(int dtype);

// ----------------------------------------------------------------- solvers (solver.cu)
void unpack_images(int dtype, const float4* src, int64_t batch, int64_t s, void* dst, cudaStream_t st);
// return the first failing iteration (DivergenceError / NotPositiveDefiniteError) or -1
int run_landweber(Plan& p, int dtype, const void* d_y, const void* d_guess, int64_t batch, double alpha,
                  int iterations, void* d_x, cudaStream_t st);
// CG over packed images (solver.cu; solvers.cpp:47-107) on A'A x = b (sys null) or
// (c0 A'A + c1 I) x = b; x updated in place; work = 4 packed image planes.
size_t cg_scalar_bytes(int64_t batch);
void cg_packed(Plan& p, int64_t batch, const float4* b, float4* x, int max_iter, double tol, const CgSystem* sys,
               float4* work, float4* sino, void* scalars, int* npd, cudaStream_t st);
int run_cgne(Plan& p, int dtype, const void* d_y, const void* d_guess, int64_t batch, int max_iter, double tol,
             void* d_x, cudaStream_t st);
double run_estimate_alpha(Plan& p, int iterations, uint64_t seed, cudaStream_t st);

// ----------------------------------------------------------------- instrumentation (profiling.cu)
constexpr int kKernelKinds = RK_KERNEL_KINDS;
// Counts the launch; when profiling is enabled also records start/stop events
// on `st` around the scope (construct right before the <<<>>> launch).
class KernelTimer {
 public:
  KernelTimer(int kind, cudaStream_t st);
  ~KernelTimer();
  KernelTimer(const KernelTimer&) = delete;
  KernelTimer& operator=(const KernelTimer&) = delete;

 private:
  int kind_;
  cudaStream_t st_;
  cudaEvent_t start_ = nullptr, stop_ = nullptr;
  bool active_ = false;
};
// Raises a kernel's dynamic shared-memory cap to at least `bytes` (> 48 KB
// needs the opt-in).  The cap is a process-wide attribute of the function,
// so it only ever grows: a call needing less never lowers it under a
// concurrent launch that needs more (calls from several host threads).
void allow_dynamic_smem(const void* func, size_t bytes);
void profiling_enable(bool on);
bool profiling_enabled();
void profiling_read(rk_kernel_stats* out, bool reset);
double probe_smem_bandwidth(int device);

}  // namespace rk

struct rk_plan {
  rk::Plan p;
};
struct rk_filter {
  rk::Filter f;
};
struct rk_shearlet {
  rk::Shearlet s;
};
