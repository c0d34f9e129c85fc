// extern "C" boundary of the B200 Radon projector (include/radon_b200.h).
// Each entry point validates like the reference function it replaces
// (cited), enqueues the CUDA work and maps exceptions onto rk_status codes.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include <nvtx3/nvToolsExt.h>

#include "rk_internal.hpp"

namespace {

thread_local std::string g_last_error;

// Device-restoring scope of one C-ABI call (see rk::set_device).  Nested entry
// points (rk_admm -> rk_admm_create ...) share the outermost scope.
thread_local int g_scope_depth = 0;
thread_local int g_saved_device = -1;

struct DeviceScope {
  DeviceScope() {
    if (g_scope_depth++ == 0) g_saved_device = -1;
  }
  ~DeviceScope() {
    if (--g_scope_depth == 0 && g_saved_device >= 0) {
      int cur = -1;
      if (cudaGetDevice(&cur) == cudaSuccess && cur != g_saved_device) cudaSetDevice(g_saved_device);
      cudaGetLastError();  // a failed restore must not surface as the next launch's error
      g_saved_device = -1;
    }
  }
};

// NVTX range per C-ABI call (header-only NVTX v3: a no-op unless a profiler
// such as Nsight Systems injects itself), named after the entry point.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
int guarded_named(const char* name, F&& f) {
  NvtxRange range(name);
  DeviceScope device_scope;
  try {
    f();
    return RK_OK;
  } catch (const rk::ValidationError& e) {
    g_last_error = e.what();
    return RK_ERR_VALIDATION;
  } catch (const rk::NumericalError& e) {
    g_last_error = e.what();
    return RK_ERR_NUMERICAL;
  } catch (const rk::CudaError& e) {
    g_last_error = e.what();
    return RK_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RK_ERR_CUDA;
  }
}

void require(bool ok, const std::string& msg) {
  if (!ok) throw rk::ValidationError(msg);
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// The plan's scratch is shared by every call on the plan: serialise host
// enqueue with the mutex and order device reuse across streams with an event.
struct ScratchLease {
  rk::Plan& p;
  cudaStream_t st;
  std::lock_guard<std::mutex> lock;
  ScratchLease(rk::Plan& plan, cudaStream_t stream) : p(plan), st(stream), lock(plan.mu) {
    rk::set_device(p.device);
    RK_CUDA(cudaStreamWaitEvent(st, p.scratch_free, 0));
  }
  ~ScratchLease() { cudaEventRecord(p.scratch_free, st); }
};

// The same for a shearlet plan's spectra scratch (work_a / work_b), which the
// analysis / synthesis calls and every ADMM state built on the plan share.
struct ShearletLease {
  rk::Shearlet& s;
  cudaStream_t st;
  std::lock_guard<std::mutex> lock;
  ShearletLease(rk::Shearlet& sh, cudaStream_t stream) : s(sh), st(stream), lock(sh.mu) {
    rk::set_device(s.device);
    if (!s.scratch_free) RK_CUDA(cudaEventCreateWithFlags(&s.scratch_free, cudaEventDisableTiming));
    RK_CUDA(cudaStreamWaitEvent(st, s.scratch_free, 0));
  }
  ~ShearletLease() { cudaEventRecord(s.scratch_free, st); }
};

size_t packed_image_bytes(const rk::Plan& p, int64_t batch) {
  return size_t(rk::groups_of(batch)) * size_t(p.s + 2) * size_t(p.s + 2) * sizeof(float4);
}
size_t packed_sino_bytes(const rk::Plan& p, int64_t batch) {
  return size_t(rk::groups_of(batch)) * size_t(p.na) * size_t(p.nd) * sizeof(float4);
}

void check_plan(const rk_plan* plan) { require(plan != nullptr, "plan is null"); }

void check_device_plan(const rk_plan* plan) {
  check_plan(plan);
  require(plan->p.device >= 0, "plan was created host-only (device -1); it cannot run kernels");
}

void check_device_filter(const rk_filter* f) {
  require(f != nullptr, "filter is null");
  require(f->f.device >= 0, "filter was created host-only (device -1); it cannot run kernels");
}

// Device-pointer bodies, reused by the host-buffer pipelines with their own scratch.
// One launch covers at most 65535 packed groups (the kernels' grid.y / grid.z);
// larger batches run as consecutive sub-batches (results are per image, so
// bit-identical to one launch).
constexpr int64_t kMaxLaunchBatch = int64_t(65535) * rk::kPack;

template <class F>
void for_sub_batches(int64_t batch, F&& f) {
  for (int64_t b0 = 0; b0 < batch; b0 += kMaxLaunchBatch) f(b0, std::min(kMaxLaunchBatch, batch - b0));
}
const void* advance(const void* ptr, int64_t items, size_t item_bytes) {
  return static_cast<const char*>(ptr) + size_t(items) * item_bytes;
}
void* advance(void* ptr, int64_t items, size_t item_bytes) {
  return static_cast<char*>(ptr) + size_t(items) * item_bytes;
}

void forward_launch(rk::Plan& p, int dtype, const void* d_image, int64_t batch, void* d_sino, rk::DeviceBuffer& pk,
                  rk::DeviceBuffer& pkt, cudaStream_t st) {
  rk::ensure_forward_schedule(p);
  pk.reserve(packed_image_bytes(p, batch));
  const bool h8 = rk::use_h8(dtype, batch);
  if (h8)
    rk::launch_pack_images_h8(d_image, batch, p.s, pk.as<float4>(), st);
  else
    rk::launch_pack_images(dtype, d_image, batch, p.s, pk.as<float4>(), st);
  if (p.fwd.any_transposed) {
    pkt.reserve(packed_image_bytes(p, batch));
    rk::launch_transpose_images(pk.as<float4>(), h8 ? rk::groups_of_h8(batch) : rk::groups_of(batch), p.s,
                                pkt.as<float4>(), st);
  }
  rk::launch_forward(p, pk.as<float4>(), pkt.as<float4>(), batch, dtype, d_sino, st);
}

void backproject_launch(rk::Plan& p, int dtype, const void* d_sino, int64_t batch, void* d_image,
                        rk::DeviceBuffer& pk, cudaStream_t st) {
  pk.reserve(packed_sino_bytes(p, batch));
  if (rk::use_h8(dtype, batch))
    rk::launch_pack_sino_h8(d_sino, batch, p.na, p.nd, pk.as<float4>(), st);
  else
    rk::launch_pack_sino(dtype, d_sino, batch, p.na, p.nd, pk.as<float4>(), st);
  rk::launch_backproject(p, pk.as<float4>(), batch, dtype, d_image, st);
}

void fbp_launch(rk::Plan& p, rk::Filter& f, int dtype, const void* d_sino, int64_t batch, void* d_image,
                rk::DeviceBuffer& pk, cudaStream_t st) {
  pk.reserve(packed_sino_bytes(p, batch));
  // the filter writes straight into the packed layout the backprojector reads
  rk::launch_filter(f, dtype, d_sino, batch, p.na, nullptr, pk.as<float4>(), st);
  rk::launch_backproject(p, pk.as<float4>(), batch, dtype, d_image, st);
}

void forward_into(rk::Plan& p, int dtype, const void* d_image, int64_t batch, void* d_sino, rk::DeviceBuffer& pk,
                  rk::DeviceBuffer& pkt, cudaStream_t st) {
  const size_t es = rk::dtype_size(dtype), img = size_t(p.s * p.s) * es, sino = size_t(p.na * p.nd) * es;
  for_sub_batches(batch, [&](int64_t b0, int64_t nb) {
    forward_launch(p, dtype, advance(d_image, b0, img), nb, advance(d_sino, b0, sino), pk, pkt, st);
  });
}

void backproject_into(rk::Plan& p, int dtype, const void* d_sino, int64_t batch, void* d_image,
                      rk::DeviceBuffer& pk, cudaStream_t st) {
  const size_t es = rk::dtype_size(dtype), img = size_t(p.s * p.s) * es, sino = size_t(p.na * p.nd) * es;
  for_sub_batches(batch, [&](int64_t b0, int64_t nb) {
    backproject_launch(p, dtype, advance(d_sino, b0, sino), nb, advance(d_image, b0, img), pk, st);
  });
}

void fbp_into(rk::Plan& p, rk::Filter& f, int dtype, const void* d_sino, int64_t batch, void* d_image,
              rk::DeviceBuffer& pk, cudaStream_t st) {
  const size_t es = rk::dtype_size(dtype), img = size_t(p.s * p.s) * es, sino = size_t(p.na * p.nd) * es;
  for_sub_batches(batch, [&](int64_t b0, int64_t nb) {
    fbp_launch(p, f, dtype, advance(d_sino, b0, sino), nb, advance(d_image, b0, img), pk, st);
  });
}

void filter_into(rk::Filter& f, int dtype, const void* d_in, int64_t batch, int64_t n_angles, void* d_out,
                 cudaStream_t st) {
  const size_t sino = size_t(n_angles * f.det_count) * rk::dtype_size(dtype);
  for_sub_batches(batch, [&](int64_t b0, int64_t nb) {
    rk::launch_filter(f, dtype, advance(d_in, b0, sino), nb, n_angles, advance(d_out, b0, sino), nullptr, st);
  });
}

// the solvers and ADMM keep whole-batch packed state: one launch per operator
void check_launch_batch(int64_t batch) {
  if (batch > kMaxLaunchBatch)
    throw rk::ValidationError("batch of " + std::to_string(batch) + " exceeds the solver limit of " +
                              std::to_string(kMaxLaunchBatch) + " images per call; split the batch");
}

void check_dtype(int dtype) { (void)rk::dtype_size(dtype); }

// ------------------------------------------------------------------ host pipelines
// Reference-shaped calls (host Tensor in, host Tensor out): the batch is cut
// into chunks of whole packed groups, and chunk i+1's host->device copy, chunk
// i's kernels and chunk i-1's device->host copy overlap on three streams (each
// stream runs copy-in, kernels, copy-out of its chunk in order, so two streams
// would cap the throughput at one chunk per half of that sum).
bool is_pinned(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

// Runs under the owner's lock; `wait_first` (the plan's scratch event) is
// synchronised first, so device-pointer calls still using scratch finish.
template <class Body>
void run_host_pipeline(rk::HostPipeline& pipe, int device, std::mutex& mu, int64_t batch, size_t in_item,
                       size_t out_item, const void* h_in, void* h_out, cudaEvent_t wait_first, Body body) {
  std::lock_guard<std::mutex> lock(mu);
  rk::set_device(device);
  for (auto& s : pipe.streams)
    if (!s) RK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // host calls are synchronous: wait for any device-pointer call still using scratch
  if (wait_first) RK_CUDA(cudaEventSynchronize(wait_first));
  // ~8 chunks (RK_PIPE_CHUNKS), each a whole number of packed groups and >= 4 MB of input
  static const int64_t n_chunks = [] {
    const char* e = std::getenv("RK_PIPE_CHUNKS");
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(8);
  }();
  static const bool use_ramp = [] {
    const char* e = std::getenv("RK_PIPE_RAMP");
    return !(e && e[0] == '0');
  }();
  int64_t chunk = std::max<int64_t>(rk::kPack, (batch + n_chunks - 1) / n_chunks);
  chunk = (chunk + rk::kPack - 1) / rk::kPack * rk::kPack;
  int64_t min_items = std::max<int64_t>(1, int64_t((4u << 20) / std::max<size_t>(in_item, 1)));
  min_items = (min_items + rk::kPack - 1) / rk::kPack * rk::kPack;
  chunk = std::min(batch, std::max(chunk, min_items));
  const bool pinned_in = is_pinned(h_in), pinned_out = is_pinned(h_out);
  constexpr int kSlots = rk::HostPipeline::kSlots;
  for (int i = 0; i < kSlots; ++i) {
    pipe.in[i].reserve(size_t(chunk) * in_item);
    pipe.out[i].reserve(size_t(chunk) * out_item);
  }
  // chunk sizes: ramp up from one packed group and back down at the end, so
  // the copy-in before the first kernel and the copy-out after the last one
  // (the parts no kernel overlaps) are short
  static const int64_t ramp_start = [] {  // RK_PIPE_RAMP_START: first / last chunk (images)
    const char* e = std::getenv("RK_PIPE_RAMP_START");
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(rk::kPack);
  }();
  std::vector<int64_t> sizes, ramp;
  for (int64_t c = ramp_start; c < chunk; c *= 2) ramp.push_back(c);
  int64_t ramp_total = 0;
  for (int64_t c : ramp) ramp_total += 2 * c;
  if (use_ramp && !ramp.empty() && batch >= ramp_total + chunk) {
    sizes = ramp;
    for (int64_t rem = batch - ramp_total; rem > 0; rem -= std::min(chunk, rem)) sizes.push_back(std::min(chunk, rem));
    sizes.insert(sizes.end(), ramp.rbegin(), ramp.rend());
  } else {
    for (int64_t rem = batch; rem > 0; rem -= std::min(chunk, rem)) sizes.push_back(std::min(chunk, rem));
  }
  int slot = 0;
  int64_t b0 = 0;
  for (const int64_t nb : sizes) {
    cudaStream_t st = pipe.streams[slot];
    const char* src = static_cast<const char*>(h_in) + size_t(b0) * in_item;
    char* dst = static_cast<char*>(h_out) + size_t(b0) * out_item;
    RK_CUDA(cudaMemcpyAsync(pipe.in[slot].ptr, src, size_t(nb) * in_item, cudaMemcpyHostToDevice, st));
    body(pipe.in[slot].ptr, nb, pipe.out[slot].ptr, slot, st);
    RK_CUDA(cudaMemcpyAsync(dst, pipe.out[slot].ptr, size_t(nb) * out_item, cudaMemcpyDeviceToHost, st));
    if (!pinned_in || !pinned_out) RK_CUDA(cudaStreamSynchronize(st));
    b0 += nb;
    slot = (slot + 1) % kSlots;
  }
  for (auto s : pipe.streams) RK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void rk::set_device(int device) {
  if (g_scope_depth > 0 && g_saved_device < 0) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess)
      g_saved_device = cur;
    else
      cudaGetLastError();
  }
  RK_CUDA(cudaSetDevice(device));
}

namespace {
// Waits for a plan's own device work (its scratch-reuse event and copy
// streams) before teardown, instead of draining the whole device; errors are
// deliberately ignored here and cleared so they cannot surface later.
void quiesce_plan(rk::Plan& p) {
  if (p.device < 0) return;
  if (cudaSetDevice(p.device) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (p.scratch_free) cudaEventSynchronize(p.scratch_free);
  p.pipe.synchronize();
}
}  // namespace

struct rk_admm_state {
  rk::Admm a;
};

namespace {
// Finished ADMM states kept for the next call with the same plan, shearlet plan,
// batch, dtype, penalties and inner iterations: their device buffers and the
// captured outer-iteration graph are reused (admm_init re-zeroes the state), so a
// repeated admm_reconstruct does not pay cudaMalloc / cudaFree / graph capture —
// which made single calls vary by up to +50 % (destroy alone 2 .. 560 ms,
// tools/admm_phase_probe.py).  Heap-allocated and never destroyed: the CUDA
// context may be gone at static destruction.
std::mutex g_admm_idle_mu;
std::vector<rk_admm_state*>* g_admm_idle = new std::vector<rk_admm_state*>();
constexpr size_t kAdmmIdleMax = 2;

rk_admm_state* admm_take_idle(const rk::Plan* p, const rk::Shearlet* sh, int dtype, int64_t batch, float p0f,
                              float p1f, int inner) {
  std::lock_guard<std::mutex> lock(g_admm_idle_mu);
  for (auto it = g_admm_idle->begin(); it != g_admm_idle->end(); ++it) {
    const rk::Admm& a = (*it)->a;
    if (a.plan == p && a.sh == sh && a.dtype == dtype && a.batch == batch && a.p0f == p0f && a.p1f == p1f &&
        a.inner == inner) {
      rk_admm_state* h = *it;
      g_admm_idle->erase(it);
      return h;
    }
  }
  return nullptr;
}

void admm_release(rk_admm_state* h) {  // the state's work is complete (its caller synchronised)
  rk_admm_state* evicted = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_admm_idle_mu);
    g_admm_idle->push_back(h);
    if (g_admm_idle->size() > kAdmmIdleMax) {
      evicted = g_admm_idle->front();
      g_admm_idle->erase(g_admm_idle->begin());
    }
  }
  delete evicted;
}

// before a plan or shearlet plan goes away: drop the idle states that point at it
void admm_purge(const rk::Plan* p, const rk::Shearlet* sh) {
  std::vector<rk_admm_state*> drop;
  {
    std::lock_guard<std::mutex> lock(g_admm_idle_mu);
    for (auto it = g_admm_idle->begin(); it != g_admm_idle->end();) {
      if ((p && (*it)->a.plan == p) || (sh && (*it)->a.sh == sh)) {
        drop.push_back(*it);
        it = g_admm_idle->erase(it);
      } else {
        ++it;
      }
    }
  }
  for (auto* h : drop) delete h;
}
}  // namespace

extern "C" {

const char* rk_last_error(void) { return g_last_error.c_str(); }

const char* rk_version(void) { return "radon_b200 0.1 (sm_100a)"; }

int rk_geometry_resolve(const rk_geometry* in, rk_geometry* out) {
  return guarded_named(__func__, [&] {
    require(in != nullptr && out != nullptr, "geometry pointer is null");
    *out = rk::resolve_geometry(*in);
  });
}

int rk_angles_linspace(double start, double stop, int64_t n, double* out) {
  return guarded_named(__func__, [&] {  // geometry.cpp:67-73
    if (n < 1) throw rk::ValidationError("angle count must be >= 1, got " + std::to_string(n));
    require(out != nullptr, "output pointer is null");
    double step = (stop - start) / double(n);
    for (int64_t i = 0; i < n; ++i) out[i] = start + double(i) * step;
  });
}

int rk_plan_create(const rk_geometry* geometry, int device, rk_plan** plan) {
  return guarded_named(__func__, [&] {
    require(geometry != nullptr && plan != nullptr, "geometry / plan pointer is null");
    *plan = nullptr;
    auto hp = std::make_unique<rk_plan>();
    rk::Plan& p = hp->p;
    p.device = device;
    p.angles.assign(geometry->angles, geometry->angles + std::max<int64_t>(geometry->n_angles, 0));
    rk_geometry in = *geometry;
    in.angles = p.angles.data();
    p.g = rk::resolve_geometry(in);
    p.g.angles = p.angles.data();
    if (device >= 0) {
      int count = 0;
      RK_CUDA(cudaGetDeviceCount(&count));
      require(device < count, "device " + std::to_string(device) + " out of range");
    }
    rk::build_plan(p);
    *plan = hp.release();
  });
}

int rk_plan_destroy(rk_plan* plan) {
  return guarded_named(__func__, [&] {
    if (!plan) return;
    admm_purge(&plan->p, nullptr);  // idle ADMM states built on this plan
    {
      std::lock_guard<std::mutex> lock(plan->p.mu);  // no call is enqueueing on it
      quiesce_plan(plan->p);
    }
    delete plan;  // frees on the plan's device (current after quiesce_plan)
    cudaGetLastError();
  });
}

int rk_plan_info_get(const rk_plan* plan, rk_plan_info* info) {
  return guarded_named(__func__, [&] {
    check_plan(plan);
    require(info != nullptr, "info pointer is null");
    const rk::Plan& p = plan->p;
    info->geometry = p.g;
    info->forward_samples = p.forward_samples;
    info->backproject_samples = p.s * p.s * p.na;
    info->device = p.device;
    const bool built = !p.fwd.cta.empty();
    info->flags = (built ? RK_PLAN_SCHEDULED : 0) | (built && p.fwd.from_cache ? RK_PLAN_SCHEDULE_CACHED : 0);
  });
}

int rk_plan_prepare(rk_plan* plan, uint64_t* hash) {
  return guarded_named(__func__, [&] {
    check_plan(plan);
    rk::Plan& p = plan->p;
    {
      std::lock_guard<std::mutex> lock(p.mu);
      rk::ensure_forward_schedule(p);  // host-only plans scheduled at creation
    }
    if (hash) *hash = rk::schedule_hash(p.fwd);
  });
}

// projector.cpp:228-236 (forward: shape + options checked, output keeps the precision)
int rk_forward(rk_plan* plan, int dtype, const void* d_image, int64_t batch, void* d_sino, void* stream) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(d_image != nullptr && d_sino != nullptr, "image / sinogram pointer is null");
    rk::Plan& p = plan->p;
    ScratchLease lease(p, as_stream(stream));
    forward_into(p, dtype, d_image, batch, d_sino, p.packed_image, p.packed_image_t, as_stream(stream));
  });
}

// projector.cpp:252-260
int rk_backproject(rk_plan* plan, int dtype, const void* d_sino, int64_t batch, void* d_image, void* stream) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(d_image != nullptr && d_sino != nullptr, "image / sinogram pointer is null");
    rk::Plan& p = plan->p;
    ScratchLease lease(p, as_stream(stream));
    backproject_into(p, dtype, d_sino, batch, d_image, p.packed_sino, as_stream(stream));
  });
}

int rk_filter_kind_from_name(const char* name, int* kind) {
  return guarded_named(__func__, [&] {
    require(name != nullptr && kind != nullptr, "name / kind pointer is null");
    *kind = rk::filter_kind_from_name(name);
  });
}

const char* rk_filter_kind_name(int kind) { return rk::filter_kind_name(kind); }

int rk_filter_create(int kind, int64_t det_count, int device, rk_filter** filter) {
  return guarded_named(__func__, [&] {
    require(filter != nullptr, "filter pointer is null");
    *filter = nullptr;
    auto hf = std::make_unique<rk_filter>();
    hf->f.device = device;
    if (device >= 0) {
      int count = 0;
      RK_CUDA(cudaGetDeviceCount(&count));
      require(device < count, "device " + std::to_string(device) + " out of range");
    }
    rk::build_filter(hf->f, kind, det_count);
    *filter = hf.release();
  });
}

int rk_filter_destroy(rk_filter* filter) {
  return guarded_named(__func__, [&] {
    if (!filter) return;
    if (filter->f.device >= 0) {
      // the filter's tables may still be read by kernels enqueued on any stream
      if (cudaSetDevice(filter->f.device) == cudaSuccess) cudaDeviceSynchronize();
      cudaGetLastError();
    }
    delete filter;
    cudaGetLastError();
  });
}

int rk_filter_response(const rk_filter* filter, int64_t* padded_size, double* response, float* response_f) {
  return guarded_named(__func__, [&] {
    require(filter != nullptr, "filter is null");
    const rk::Filter& f = filter->f;
    if (padded_size) *padded_size = f.padded;
    if (response) std::memcpy(response, f.response.data(), f.response.size() * sizeof(double));
    if (response_f) std::memcpy(response_f, f.response_f.data(), f.response_f.size() * sizeof(float));
  });
}

// sino_filter.cpp:98-104 (3-D shape, det_count must match the filter)
int rk_filter_sinogram(rk_filter* filter, int dtype, const void* d_in, int64_t batch, int64_t n_angles,
                       void* d_out, void* stream) {
  return guarded_named(__func__, [&] {
    check_device_filter(filter);
    check_dtype(dtype);
    require(batch >= 1 && n_angles >= 1, "sinogram must have batch >= 1 and n_angles >= 1");
    require(d_in != nullptr && d_out != nullptr, "sinogram pointer is null");
    rk::Filter& f = filter->f;
    std::lock_guard<std::mutex> lock(f.mu);
    rk::set_device(f.device);
    filter_into(f, dtype, d_in, batch, n_angles, d_out, as_stream(stream));
  });
}

// sino_filter.cpp:126-136
int rk_fbp(rk_plan* plan, rk_filter* filter, int dtype, const void* d_sino, int64_t batch, void* d_image,
           void* stream) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_device_filter(filter);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(d_sino != nullptr && d_image != nullptr, "sinogram / image pointer is null");
    rk::Plan& p = plan->p;
    require(filter->f.det_count == p.nd, "sinogram det_count " + std::to_string(p.nd) +
                                             " does not match filter " + std::to_string(filter->f.det_count));
    require(filter->f.device == p.device, "filter and plan live on different devices");
    ScratchLease lease(p, as_stream(stream));
    fbp_into(p, filter->f, dtype, d_sino, batch, d_image, p.packed_sino, as_stream(stream));
  });
}

int rk_forward_host(rk_plan* plan, int dtype, const void* h_image, int64_t batch, void* h_sino) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(h_image != nullptr && h_sino != nullptr, "image / sinogram pointer is null");
    rk::Plan& p = plan->p;
    const size_t es = rk::dtype_size(dtype);
    run_host_pipeline(p.pipe, p.device, p.mu, batch, size_t(p.s * p.s) * es, size_t(p.na * p.nd) * es, h_image,
                      h_sino, p.scratch_free,
                      [&](const void* din, int64_t nb, void* dout, int slot, cudaStream_t st) {
                        forward_into(p, dtype, din, nb, dout, p.pipe.pk[slot], p.pipe.pkt[slot], st);
                      });
  });
}

int rk_backproject_host(rk_plan* plan, int dtype, const void* h_sino, int64_t batch, void* h_image) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(h_image != nullptr && h_sino != nullptr, "image / sinogram pointer is null");
    rk::Plan& p = plan->p;
    const size_t es = rk::dtype_size(dtype);
    run_host_pipeline(p.pipe, p.device, p.mu, batch, size_t(p.na * p.nd) * es, size_t(p.s * p.s) * es, h_sino,
                      h_image, p.scratch_free,
                      [&](const void* din, int64_t nb, void* dout, int slot, cudaStream_t st) {
                        backproject_into(p, dtype, din, nb, dout, p.pipe.pk[slot], st);
                      });
  });
}

int rk_filter_sinogram_host(rk_filter* filter, int dtype, const void* h_in, int64_t batch, int64_t n_angles,
                            void* h_out) {
  return guarded_named(__func__, [&] {
    check_device_filter(filter);
    check_dtype(dtype);
    require(batch >= 1 && n_angles >= 1, "sinogram must have batch >= 1 and n_angles >= 1");
    require(h_in != nullptr && h_out != nullptr, "sinogram pointer is null");
    rk::Filter& f = filter->f;
    const size_t item = size_t(n_angles * f.det_count) * rk::dtype_size(dtype);  // one sinogram
    run_host_pipeline(f.pipe, f.device, f.mu, batch, item, item, h_in, h_out, nullptr,
                      [&](const void* din, int64_t nb, void* dout, int, cudaStream_t st) {
                        filter_into(f, dtype, din, nb, n_angles, dout, st);
                      });
  });
}

int rk_fbp_host(rk_plan* plan, rk_filter* filter, int dtype, const void* h_sino, int64_t batch, void* h_image) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_device_filter(filter);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(h_image != nullptr && h_sino != nullptr, "image / sinogram pointer is null");
    rk::Plan& p = plan->p;
    require(filter->f.det_count == p.nd, "sinogram det_count " + std::to_string(p.nd) +
                                             " does not match filter " + std::to_string(filter->f.det_count));
    require(filter->f.device == p.device, "filter and plan live on different devices");
    const size_t es = rk::dtype_size(dtype);
    run_host_pipeline(p.pipe, p.device, p.mu, batch, size_t(p.na * p.nd) * es, size_t(p.s * p.s) * es, h_sino,
                      h_image, p.scratch_free,
                      [&](const void* din, int64_t nb, void* dout, int slot, cudaStream_t st) {
                        fbp_into(p, filter->f, dtype, din, nb, dout, p.pipe.pk[slot], st);
                      });
  });
}

// solvers.cpp:111-128
int rk_estimate_alpha(rk_plan* plan, int iterations, uint64_t seed, double* alpha) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    require(alpha != nullptr, "alpha pointer is null");
    rk::Plan& p = plan->p;
    cudaStream_t st = nullptr;
    ScratchLease lease(p, st);
    *alpha = rk::run_estimate_alpha(p, iterations, seed, st);
  });
}

// solvers.cpp:130-145
int rk_landweber(rk_plan* plan, int dtype, const void* d_y, const void* d_guess, int64_t batch, double alpha,
                 int iterations, void* d_x, int* failed_iteration, void* stream) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(d_y != nullptr && d_guess != nullptr && d_x != nullptr, "landweber pointer is null");
    check_launch_batch(batch);
    rk::Plan& p = plan->p;
    int failed = -1;
    {
      ScratchLease lease(p, as_stream(stream));
      failed = rk::run_landweber(p, dtype, d_y, d_guess, batch, alpha, iterations, d_x, as_stream(stream));
    }
    if (failed_iteration) *failed_iteration = failed;
    if (failed >= 0)
      throw rk::NumericalError("landweber produced a non-finite iterate at iteration " + std::to_string(failed),
                               failed);
  });
}

// solvers.cpp:162-166 (cg_impl :47-107)
int rk_cgne(rk_plan* plan, int dtype, const void* d_y, const void* d_guess, int64_t batch, int max_iter,
            double tolerance, void* d_x, int* failed_iteration, void* stream) {
  return guarded_named(__func__, [&] {
    check_device_plan(plan);
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(d_y != nullptr && d_guess != nullptr && d_x != nullptr, "cgne pointer is null");
    check_launch_batch(batch);
    rk::Plan& p = plan->p;
    int failed = -1;
    {
      ScratchLease lease(p, as_stream(stream));
      failed = rk::run_cgne(p, dtype, d_y, d_guess, batch, max_iter, tolerance, d_x, as_stream(stream));
    }
    if (failed_iteration) *failed_iteration = failed;
    if (failed >= 0)
      throw rk::NumericalError("cg: curvature p'Ap is not positive at iteration " + std::to_string(failed), failed);
  });
}

int rk_shearlet_create(int64_t height, int64_t width, const double* alphas, int n_scales, int device,
                       rk_shearlet** plan) {
  return guarded_named(__func__, [&] {
    require(plan != nullptr, "plan pointer is null");
    require(alphas != nullptr || n_scales == 0, "alphas pointer is null");
    *plan = nullptr;
    auto hs = std::make_unique<rk_shearlet>();
    hs->s.device = device;
    if (device >= 0) {
      int count = 0;
      RK_CUDA(cudaGetDeviceCount(&count));
      require(device < count, "device " + std::to_string(device) + " out of range");
    }
    rk::build_shearlet(hs->s, height, width, std::vector<double>(alphas, alphas + std::max(n_scales, 0)));
    *plan = hs.release();
  });
}

int rk_shearlet_create_stored(int64_t height, int64_t width, const double* alphas, int n_scales,
                              const double* multipliers, int device, rk_shearlet** plan) {
  return guarded_named(__func__, [&] {
    require(plan != nullptr, "plan pointer is null");
    require(alphas != nullptr || n_scales == 0, "alphas pointer is null");
    require(multipliers != nullptr, "multipliers pointer is null");
    *plan = nullptr;
    auto hs = std::make_unique<rk_shearlet>();
    hs->s.device = device;
    if (device >= 0) {
      int count = 0;
      RK_CUDA(cudaGetDeviceCount(&count));
      require(device < count, "device " + std::to_string(device) + " out of range");
    }
    rk::build_shearlet(hs->s, height, width, std::vector<double>(alphas, alphas + std::max(n_scales, 0)),
                       multipliers);
    *plan = hs.release();
  });
}

int rk_shearlet_destroy(rk_shearlet* plan) {
  return guarded_named(__func__, [&] {
    if (!plan) return;
    admm_purge(nullptr, &plan->s);  // idle ADMM states built on this shearlet plan
    if (plan->s.device >= 0) {
      if (cudaSetDevice(plan->s.device) == cudaSuccess) cudaDeviceSynchronize();
      cudaGetLastError();
    }
    delete plan;
    cudaGetLastError();
  });
}

int rk_shearlet_info(const rk_shearlet* plan, int64_t* n_coeff, double* scales, double* multipliers) {
  return guarded_named(__func__, [&] {
    require(plan != nullptr, "plan is null");
    const rk::Shearlet& s = plan->s;
    if (n_coeff) *n_coeff = s.n_coeff;
    if (scales) std::memcpy(scales, s.scales.data(), s.scales.size() * sizeof(double));
    if (multipliers) std::memcpy(multipliers, s.multipliers.data(), s.multipliers.size() * sizeof(double));
  });
}

// shearlet.cpp:296-311
int rk_shearlet_forward(rk_shearlet* plan, int dtype, const void* d_image, int64_t batch, void* d_coeff,
                        void* stream) {
  return guarded_named(__func__, [&] {
    require(plan != nullptr && plan->s.device >= 0, "shearlet plan is null or host-only");
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(d_image != nullptr && d_coeff != nullptr, "image / coefficient pointer is null");
    ShearletLease lease(plan->s, as_stream(stream));
    rk::shearlet_forward(plan->s, dtype, d_image, batch, d_coeff, as_stream(stream));
  });
}

// shearlet.cpp:313-330
int rk_shearlet_backward(rk_shearlet* plan, int dtype, const void* d_coeff, int64_t batch, void* d_image,
                         void* stream) {
  return guarded_named(__func__, [&] {
    require(plan != nullptr && plan->s.device >= 0, "shearlet plan is null or host-only");
    check_dtype(dtype);
    require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
    require(d_image != nullptr && d_coeff != nullptr, "image / coefficient pointer is null");
    ShearletLease lease(plan->s, as_stream(stream));
    rk::shearlet_backward(plan->s, dtype, d_coeff, batch, d_image, as_stream(stream));
  });
}

// ---------------------------------------------------------------- ADMM (admm.cpp:111-163)
namespace {
void check_admm_args(rk_plan* plan, rk_shearlet* sh, int dtype, int64_t batch, double p0, double p1) {
  check_device_plan(plan);
  require(sh != nullptr && sh->s.device >= 0, "shearlet plan is null or host-only");
  require(sh->s.device == plan->p.device, "shearlet plan and projector plan live on different devices");
  check_dtype(dtype);
  require(batch >= 1, "batch must be >= 1, got " + std::to_string(batch));
  if (!(p0 > 0.0) || !(p1 > 0.0))
    throw rk::ValidationError("admm penalties must be positive, got p0 = " + std::to_string(p0) +
                              ", p1 = " + std::to_string(p1));
  if (sh->s.height != plan->p.s || sh->s.width != plan->p.s)
    throw rk::ValidationError("operator domain (" + std::to_string(plan->p.s) + ", " + std::to_string(plan->p.s) +
                              ") does not match plan grid " + std::to_string(sh->s.height) + "x" +
                              std::to_string(sh->s.width));
}

// default_weights (admm.cpp:11-15) or the caller's; thresh = scale(w, p0 / p1) (admm.cpp:135)
std::vector<double> admm_thresholds(const rk::Shearlet& s, const double* weights, double p0, double p1) {
  std::vector<double> t(static_cast<size_t>(s.n_coeff));
  for (int64_t k = 0; k < s.n_coeff; ++k) {
    const double w = weights ? weights[k] : std::pow(3.0, s.scales[size_t(k)]) / 400.0;
    t[size_t(k)] = w * (p0 / p1);
    if (!(t[size_t(k)] >= 0.0))
      throw rk::ValidationError("shrink threshold must be nonnegative, got " + std::to_string(t[size_t(k)]) +
                                " at index " + std::to_string(k));
  }
  return t;
}
}  // namespace


int rk_admm_create(rk_plan* plan, rk_shearlet* shearlet, int dtype, const void* d_sino, int64_t batch, double p0,
                   double p1, const double* weights, int inner_cg_iterations, void* stream, rk_admm_state** out) {
  return guarded_named(__func__, [&] {
    require(out != nullptr, "admm pointer is null");
    *out = nullptr;
    check_admm_args(plan, shearlet, dtype, batch, p0, p1);
    check_launch_batch(batch);
    require(d_sino != nullptr, "sinogram pointer is null");
    if (inner_cg_iterations < 1) throw rk::ValidationError("admm inner_cg_iterations must be at least 1");
    std::unique_ptr<rk_admm_state> h(
        admm_take_idle(&plan->p, &shearlet->s, dtype, batch, float(p0), float(p1), inner_cg_iterations));
    if (!h) h = std::make_unique<rk_admm_state>();
    rk::Admm& a = h->a;
    a.plan = &plan->p;
    a.sh = &shearlet->s;
    a.dtype = dtype;
    a.batch = batch;
    a.p0f = float(p0);
    a.p1f = float(p1);
    a.sys = rk::CgSystem{float(p0), float(1.0 + p1)};
    a.inner = inner_cg_iterations;
    const std::vector<double> th = admm_thresholds(shearlet->s, weights, p0, p1);
    ScratchLease lease(plan->p, as_stream(stream));
    ShearletLease sh_lease(shearlet->s, as_stream(stream));
    rk::admm_init(a, d_sino, th, as_stream(stream));
    *out = h.release();
  });
}

int rk_admm_iterate(rk_admm_state* admm, int64_t n, int64_t* failed_iteration, void* stream) {
  return guarded_named(__func__, [&] {
    require(admm != nullptr, "admm is null");
    if (n < 0) throw rk::ValidationError("admm outer_iterations must be nonnegative");
    rk::Admm& a = admm->a;
    int64_t failed = a.failed;
    if (failed < 0 && n > 0) {
      ScratchLease lease(*a.plan, as_stream(stream));
      ShearletLease sh_lease(*a.sh, as_stream(stream));
      failed = rk::admm_iterate(a, n, as_stream(stream));
    }
    if (failed_iteration) *failed_iteration = failed;
    if (failed >= 0)
      throw rk::NumericalError("admm state became non-finite at iteration " + std::to_string(failed), int(failed));
  });
}

int rk_admm_read(rk_admm_state* admm, int which, int dtype, void* d_dst, void* stream) {
  return guarded_named(__func__, [&] {
    require(admm != nullptr, "admm is null");
    require(d_dst != nullptr, "destination pointer is null");
    check_dtype(dtype);
    rk::Admm& a = admm->a;
    rk::set_device(a.plan->device);
    RK_CUDA(cudaStreamWaitEvent(as_stream(stream), a.plan->scratch_free, 0));
    rk::admm_read(a, which, dtype, d_dst, as_stream(stream));
  });
}

int rk_admm_destroy(rk_admm_state* admm) {
  return guarded_named(__func__, [&] {
    if (!admm) return;
    // every stream that may still touch the state (a trailing rk_admm_read on the caller's)
    if (cudaSetDevice(admm->a.plan->device) == cudaSuccess) cudaDeviceSynchronize();
    cudaGetLastError();
    if (admm->a.failed < 0)
      admm_release(admm);  // healthy: kept for the next compatible call
    else
      delete admm;
    cudaGetLastError();
  });
}

int rk_admm(rk_plan* plan, rk_shearlet* shearlet, int dtype, const void* d_sino, int64_t batch, double p0, double p1,
            const double* weights, int64_t outer_iterations, int inner_cg_iterations, void* d_image,
            int64_t* failed_iteration, void* stream) {
  rk_admm_state* h = nullptr;
  int st = rk_admm_create(plan, shearlet, dtype, d_sino, batch, p0, p1, weights, inner_cg_iterations, stream, &h);
  if (st != RK_OK) return st;
  if (failed_iteration) *failed_iteration = -1;
  st = rk_admm_iterate(h, outer_iterations, failed_iteration, stream);
  if (st == RK_OK) st = rk_admm_read(h, 0, dtype, d_image, stream);
  if (st == RK_OK) {
    st = rk_admm_destroy(h);
  } else {
    const std::string err = rk_last_error();
    rk_admm_destroy(h);
    g_last_error = err;  // keep the first failure's message
  }
  return st;
}

int rk_profiling_enable(int enable) {
  return guarded_named(__func__, [&] { rk::profiling_enable(enable != 0); });
}

int rk_profiling_read(rk_kernel_stats* stats, int reset) {
  return guarded_named(__func__, [&] {
    require(stats != nullptr, "stats pointer is null");
    rk::profiling_read(stats, reset != 0);
  });
}

int rk_probe_smem_bandwidth(int device, double* gbs) {
  return guarded_named(__func__, [&] {
    require(gbs != nullptr, "output pointer is null");
    *gbs = rk::probe_smem_bandwidth(device);
  });
}

}  // extern "C"
