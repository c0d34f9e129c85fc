// l1-shearlet ADMM on the device (§8f rank 4; reference admm.cpp:111-163,
// paper §4.3): argmin_{f >= 0} ||SH(f)||_{1,w} + 0.5 ||A f - y||^2 with a
// shearlet split (z1, u1) and a positivity split (z2, u2).  One outer
// iteration, all on one stream with no host synchronisation:
//
//   shU  = SH'(z1 - u1)                     synthesis reads the difference (shearlet.cu)
//   cg_y = p0 bp + (p1 shU + (z2 - u2))     assemble_kernel (packed layout)
//   f    = CG(p0 A'A + (1 + p1) I, f, cg_y) cg_packed (solver.cu), the system
//                                           term fused into the backprojection epilogue
//   z1, u1 <- shrink(SH(f) + u1, t_k), u1 + (SH(f) - z1)
//                                           fused into the analysis's last row pass
//   z2, u2 <- max(f + u2, 0), u2 + (f - z2) positivity_kernel
//
// with the reference's fp32 operation order (tensor.cpp:319-354) and its
// non-finite check (admm.cpp:157-159) folded into the update kernels as an
// atomicMin(iteration) flag read once per call.
#include <cuda_fp16.h>

#include <climits>
#include <cstdlib>
#include <cmath>

#include "rk_internal.hpp"

namespace rk {

namespace {

inline unsigned grid_for(int64_t n, int threads, unsigned cap = 8192) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap)));
}

__device__ __forceinline__ float lane(const float4& v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }

// cg_y = axpy(p0, bp, axpy(p1, shU, sub(z2, u2))) over packed images; zero border (admm.cpp:147)
__global__ void assemble_kernel(const float4* __restrict__ bp, const float* __restrict__ sh,
                                const float4* __restrict__ z2, const float4* __restrict__ u2, int64_t batch, int s,
                                int64_t total, float p0, float p1, float4* __restrict__ out) {
  const int P = s + 2;
  const int64_t plane = int64_t(P) * P, n = int64_t(s) * s;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = idx / plane, rem = idx - g * plane;
    const int pi = int(rem / P), pj = int(rem - int64_t(pi) * P);
    if (pi < 1 || pi > s || pj < 1 || pj > s) {
      out[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    const float4 b = bp[idx], z = z2[idx], u = u2[idx];
    float r[4];
#pragma unroll
    for (int q = 0; q < kPack; ++q) {
      const int64_t e = g * kPack + q;
      const float shv = e < batch ? sh[e * n + int64_t(pi - 1) * s + (pj - 1)] : 0.f;
      const float inner = __fadd_rn(__fmul_rn(p1, shv), __fsub_rn(lane(z, q), lane(u, q)));
      r[q] = __fadd_rn(__fmul_rn(p0, lane(b, q)), inner);
    }
    out[idx] = make_float4(r[0], r[1], r[2], r[3]);
  }
}

// z2 = clamp_min(f + u2, 0); u2 = u2 + (f - z2); all_finite(f), all_finite(u2) (admm.cpp:152-159)
__global__ void positivity_kernel(const float4* __restrict__ f, float4* __restrict__ z2, float4* __restrict__ u2,
                                  int64_t batch, int64_t plane, int64_t total, int* flag, const int* iteration) {
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = idx / plane;
    const float4 fv = f[idx], uv = u2[idx];
    float z[4], u[4];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < kPack; ++q) {
      const float fq = lane(fv, q), uq = lane(uv, q);
      const float sq = __fadd_rn(fq, uq);
      z[q] = sq < 0.f ? 0.f : sq;
      u[q] = __fadd_rn(uq, __fsub_rn(fq, z[q]));
      if (g * kPack + q < batch && (!isfinite(fq) || !isfinite(u[q]))) bad = true;
    }
    z2[idx] = make_float4(z[0], z[1], z[2], z[3]);
    u2[idx] = make_float4(u[0], u[1], u[2], u[3]);
    if (bad) atomicMin(flag, *iteration);
  }
}

// the end of an outer iteration: advance the device iteration counter
__global__ void next_iteration_kernel(int* iteration) { ++*iteration; }

template <class T>
__global__ void convert_kernel(const float* __restrict__ in, int64_t n, T* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = T(in[i]);
}
template <>
__global__ void convert_kernel<__half>(const float* __restrict__ in, int64_t n, __half* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = __float2half_rn(in[i]);
}

}  // namespace

void admm_init(Admm& a, const void* d_sino, const std::vector<double>& thresholds, cudaStream_t st) {
  Plan& p = *a.plan;
  const int64_t G = groups_of(a.batch), P = p.s + 2, img_plane = P * P;
  const int64_t K = a.sh->n_coeff, npx = p.s * p.s;
  const size_t ib = size_t(G * img_plane) * sizeof(float4);
  a.packed.reserve(9 * ib);
  a.sino.reserve(size_t(G * p.na * p.nd) * sizeof(float4));
  a.user.reserve(2 * size_t(a.batch * npx) * sizeof(float));
  a.coeff.reserve(2 * size_t(a.batch * K * npx) * sizeof(float));
  const size_t thresh_bytes = (size_t(K) * sizeof(float) + 255) / 256 * 256;  // then flags[2], iteration
  a.small.reserve(thresh_bytes + 256 + cg_scalar_bytes(a.batch));
  char* pk = a.packed.as<char>();
  a.F = reinterpret_cast<float4*>(pk);
  a.BP = reinterpret_cast<float4*>(pk + ib);
  a.Z2 = reinterpret_cast<float4*>(pk + 2 * ib);
  a.U2 = reinterpret_cast<float4*>(pk + 3 * ib);
  a.CGY = reinterpret_cast<float4*>(pk + 4 * ib);
  a.work = reinterpret_cast<float4*>(pk + 5 * ib);
  a.fU = a.user.as<float>();
  a.shU = a.fU + a.batch * npx;
  a.z1 = a.coeff.as<float>();
  a.u1 = a.z1 + a.batch * K * npx;
  a.thresh = a.small.as<float>();
  a.flags = reinterpret_cast<int*>(a.small.as<char>() + thresh_bytes);
  a.iter_dev = a.flags + 2;
  a.cg_scalars = a.small.as<char>() + thresh_bytes + 256;
  // thresh = scale(w, p0 / p1) in fp64 (computed by the caller), read as float by shrink (admm.cpp:135, :53-82)
  std::vector<float> th(static_cast<size_t>(K));
  for (int64_t k = 0; k < K; ++k) th[size_t(k)] = float(thresholds[size_t(k)]);
  RK_CUDA(cudaMemcpyAsync(a.thresh, th.data(), th.size() * sizeof(float), cudaMemcpyHostToDevice, st));
  const int none[2] = {INT_MAX, INT_MAX};
  RK_CUDA(cudaMemcpyAsync(a.flags, none, sizeof(none), cudaMemcpyHostToDevice, st));
  // zero state (admm.cpp:138-143): f, z2, u2 packed; z1, u1 coefficients
  RK_CUDA(cudaMemsetAsync(pk, 0, 9 * ib, st));
  RK_CUDA(cudaMemsetAsync(a.coeff.ptr, 0, 2 * size_t(a.batch * K * npx) * sizeof(float), st));
  // bp = A'(y) with y in the compute precision (half storage converted to single, admm.cpp:131-136)
  launch_pack_sino(a.dtype, d_sino, a.batch, p.na, p.nd, a.sino.as<float4>(), st);
  BpEpilogue be;
  be.mode = kOutPacked;
  be.packed = a.BP;
  launch_backproject(p, a.sino.as<float4>(), a.batch, RK_F32, nullptr, st, be);
  a.iterations_done = 0;
  a.failed = -1;
}

Admm::~Admm() {
  if (graph) cudaGraphExecDestroy(graph);
  if (graph_in) cudaEventDestroy(graph_in);
  if (graph_out) cudaEventDestroy(graph_out);
  if (graph_stream) cudaStreamDestroy(graph_stream);
}

namespace {

// One outer iteration (admm.cpp:146-160), all on `st`.
void outer_iteration(Admm& a, cudaStream_t st) {
  Plan& p = *a.plan;
  Shearlet& sh = *a.sh;
  const int64_t G = groups_of(a.batch), P = p.s + 2, img_plane = P * P, total = G * img_plane;
  shearlet_admm_synth(sh, a.z1, a.u1, a.batch, a.shU, st);
  {
    KernelTimer t(RK_KERNEL_SOLVER, st);
    assemble_kernel<<<grid_for(total, 256), 256, 0, st>>>(a.BP, a.shU, a.Z2, a.U2, a.batch, int(p.s), total, a.p0f,
                                                          a.p1f, a.CGY);
    RK_CUDA(cudaGetLastError());
  }
  cg_packed(p, a.batch, a.CGY, a.F, a.inner, 0.0, &a.sys, a.work, a.sino.as<float4>(), a.cg_scalars, a.flags + 1, st);
  unpack_images(RK_F32, a.F, a.batch, p.s, a.fU, st);
  shearlet_admm_shrink(sh, a.fU, a.batch, a.z1, a.u1, a.thresh, a.flags, a.iter_dev, st);
  {
    KernelTimer t(RK_KERNEL_SOLVER, st);
    positivity_kernel<<<grid_for(total, 256), 256, 0, st>>>(a.F, a.Z2, a.U2, a.batch, img_plane, total, a.flags,
                                                            a.iter_dev);
    next_iteration_kernel<<<1, 1, 0, st>>>(a.iter_dev);
    RK_CUDA(cudaGetLastError());
  }
}

bool graph_current(const Admm& a) {
  return a.graph && a.graph_key[0] == a.sh->work_a.ptr && a.graph_key[1] == a.sh->work_b.ptr;
}

// Captures outer_iteration on the ADMM's own stream (the caller's may be the
// legacy default stream, which cannot be captured).  Every buffer the
// iteration touches must already have its size: the caller runs one eager
// iteration first.
void capture(Admm& a) {
  if (a.graph) {
    cudaGraphExecDestroy(a.graph);
    a.graph = nullptr;
  }
  if (!a.graph_stream) {
    RK_CUDA(cudaStreamCreateWithFlags(&a.graph_stream, cudaStreamNonBlocking));
    RK_CUDA(cudaEventCreateWithFlags(&a.graph_in, cudaEventDisableTiming));
    RK_CUDA(cudaEventCreateWithFlags(&a.graph_out, cudaEventDisableTiming));
  }
  cudaGraph_t g = nullptr;
  RK_CUDA(cudaStreamBeginCapture(a.graph_stream, cudaStreamCaptureModeThreadLocal));
  try {
    outer_iteration(a, a.graph_stream);
  } catch (...) {
    cudaStreamEndCapture(a.graph_stream, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    throw;
  }
  RK_CUDA(cudaStreamEndCapture(a.graph_stream, &g));
  const cudaError_t e = cudaGraphInstantiate(&a.graph, g, 0);
  cudaGraphDestroy(g);
  RK_CUDA(e);
  a.graph_key[0] = a.sh->work_a.ptr;
  a.graph_key[1] = a.sh->work_b.ptr;
}

}  // namespace

int64_t admm_iterate(Admm& a, int64_t n, cudaStream_t st) {
  // the device counter starts at the number of iterations done (flags name the outer iteration)
  const int start = int(a.iterations_done);
  RK_CUDA(cudaMemcpyAsync(a.iter_dev, &start, sizeof(int), cudaMemcpyHostToDevice, st));
  // Graph replay unless the per-kernel event timing is on (its records are per launch) or
  // RK_ADMM_GRAPH=0; identical kernels and arguments either way, so identical results.
  const char* ge = std::getenv("RK_ADMM_GRAPH");
  const bool use_graph = !profiling_enabled() && !(ge && ge[0] == '0');
  int64_t i = 0;
  if (use_graph && n > 0) {
    if (!graph_current(a)) {
      outer_iteration(a, st);  // sizes every scratch buffer before the capture
      ++i;
      capture(a);  // also when n == 1: the observer's one-iteration calls replay it next time
    }
    if (i < n) {
      RK_CUDA(cudaEventRecord(a.graph_in, st));
      RK_CUDA(cudaStreamWaitEvent(a.graph_stream, a.graph_in, 0));
      for (; i < n; ++i) RK_CUDA(cudaGraphLaunch(a.graph, a.graph_stream));
      RK_CUDA(cudaEventRecord(a.graph_out, a.graph_stream));
      RK_CUDA(cudaStreamWaitEvent(st, a.graph_out, 0));
    }
  }
  for (; i < n; ++i) outer_iteration(a, st);
  a.iterations_done += n;
  int h[2] = {INT_MAX, INT_MAX};
  RK_CUDA(cudaMemcpyAsync(h, a.flags, sizeof(h), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaStreamSynchronize(st));
  if (h[1] != INT_MAX)  // NotPositiveDefiniteError from the inner cg (solvers.cpp:69-75)
    throw NumericalError("cg: curvature p'Ap is not positive at iteration " + std::to_string(h[1]), h[1]);
  if (h[0] != INT_MAX && a.failed < 0) a.failed = h[0];
  return a.failed;
}

void admm_read(Admm& a, int which, int dtype, void* dst, cudaStream_t st) {
  const int64_t s = a.plan->s, npx = s * s, K = a.sh->n_coeff;
  if (which == 0 || which == 3 || which == 4) {
    const float4* src = which == 0 ? a.F : which == 3 ? a.Z2 : a.U2;
    unpack_images(dtype, src, a.batch, s, dst, st);
    return;
  }
  if (which != 1 && which != 2) throw ValidationError("admm state index must be 0..4, got " + std::to_string(which));
  const float* src = which == 1 ? a.z1 : a.u1;
  const int64_t n = a.batch * K * npx;
  KernelTimer t(RK_KERNEL_SOLVER, st);
  switch (dtype) {
    case RK_F16: convert_kernel<__half><<<grid_for(n, 256), 256, 0, st>>>(src, n, static_cast<__half*>(dst)); break;
    case RK_F32:
      RK_CUDA(cudaMemcpyAsync(dst, src, size_t(n) * sizeof(float), cudaMemcpyDeviceToDevice, st));
      break;
    case RK_F64: convert_kernel<double><<<grid_for(n, 256), 256, 0, st>>>(src, n, static_cast<double*>(dst)); break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
  RK_CUDA(cudaGetLastError());
}

}  // namespace rk
