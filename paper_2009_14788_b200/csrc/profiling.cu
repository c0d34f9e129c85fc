// Instrumentation (no reference equivalent): counts every kernel the library
// launches and, when enabled, brackets each launch with CUDA events on its
// stream so bench.py can report per-kernel device time (roofline
// denominators) without a profiler.  Also a shared-memory bandwidth probe —
// the L1TEX/SMEM roofline peak the projector kernels are bound by.
#include <atomic>
#include <map>
#include <mutex>
#include <vector>

#include "rk_internal.hpp"

namespace rk {

namespace {

struct Record {
  int kind;
  int device;
  cudaEvent_t start, stop;
};

std::atomic<int64_t> g_launches[kKernelKinds];
std::atomic<bool> g_timing{false};
std::mutex g_mu;
std::vector<Record> g_records;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  RK_CUDA(cudaEventCreate(&e));
  return e;
}

}  // namespace

KernelTimer::KernelTimer(int kind, cudaStream_t st) : kind_(kind), st_(st) {
  g_launches[kind].fetch_add(1);
  if (!g_timing.load()) return;
  std::lock_guard<std::mutex> lock(g_mu);
  start_ = take_event();
  stop_ = take_event();
  RK_CUDA(cudaEventRecord(start_, st_));
  active_ = true;
}

KernelTimer::~KernelTimer() {
  if (!active_) return;
  std::lock_guard<std::mutex> lock(g_mu);
  cudaEventRecord(stop_, st_);
  int dev = 0;
  cudaGetDevice(&dev);
  g_records.push_back({kind_, dev, start_, stop_});
}

void profiling_enable(bool on) { g_timing.store(on); }
bool profiling_enabled() { return g_timing.load(); }

void allow_dynamic_smem(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> caps;
  int dev = 0;
  RK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cap = caps[{func, dev}];
  if (bytes <= cap) return;
  RK_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  cap = bytes;
}

void profiling_read(rk_kernel_stats* out, bool reset) {
  std::lock_guard<std::mutex> lock(g_mu);
  std::memset(out, 0, sizeof(*out));
  for (int k = 0; k < kKernelKinds; ++k) out->launches[k] = g_launches[k].load();
  for (const Record& r : g_records) {
    RK_CUDA(cudaEventSynchronize(r.stop));
    float ms = 0.f;
    RK_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
    out->ms[r.kind] += double(ms);
    out->timed[r.kind] += 1;
  }
  if (reset) {
    for (const Record& r : g_records) {
      g_pool.push_back(r.start);
      g_pool.push_back(r.stop);
    }
    g_records.clear();
    for (int k = 0; k < kKernelKinds; ++k) g_launches[k].store(0);
  }
}

// ----------------------------------------------------------------- SMEM probe
// Every warp streams conflict-free 128-bit shared-memory loads (each quarter
// warp touches 8 distinct 16-byte slots of one 128-byte row): the
// LDS.128 data rate per SM is the denominator of the projector rooflines.
namespace {
constexpr int kProbeThreads = 1024;
constexpr int kProbeIters = 4096;

__global__ void __launch_bounds__(kProbeThreads) smem_probe_kernel(float* out, int iters) {
  __shared__ float4 buf[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(float(i), 1.f, 2.f, 3.f);
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int idx = threadIdx.x & 2047;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 v = buf[(idx + u * 256) & 2047];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    idx = (idx + 32) & 2047;
  }
  if (acc.x + acc.y + acc.z + acc.w == -1.f) out[0] = acc.x;  // keep the loads alive
}
}  // namespace

double probe_smem_bandwidth(int device) {
  rk::set_device(device);
  int sms = 0;
  RK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  float* out = nullptr;
  RK_CUDA(cudaMalloc(&out, sizeof(float)));
  const int blocks = sms * 2;
  smem_probe_kernel<<<blocks, kProbeThreads>>>(out, 64);  // warm up clocks
  cudaEvent_t a, b;
  RK_CUDA(cudaEventCreate(&a));
  RK_CUDA(cudaEventCreate(&b));
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    RK_CUDA(cudaEventRecord(a));
    smem_probe_kernel<<<blocks, kProbeThreads>>>(out, kProbeIters);
    RK_CUDA(cudaEventRecord(b));
    RK_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    RK_CUDA(cudaEventElapsedTime(&ms, a, b));
    const double bytes = double(blocks) * kProbeThreads * double(kProbeIters) * 8.0 * 16.0;
    best = std::max(best, bytes / (double(ms) * 1e-3) / 1e9);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  RK_CUDA(cudaGetLastError());
  return best;  // GB/s
}

}  // namespace rk
