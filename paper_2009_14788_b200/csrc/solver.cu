// Iterative reconstruction on the device (config 5): Landweber, CGNE and the
// power-iteration step size of the reference's solvers (solvers.cpp:47-166).
//
// All iterates live in the packed layouts of kernels.cu (four images per
// float4 texel, image border kept at zero), so every forward / backprojection
// of an iteration reads its operand directly, and the vector work is fused
// into the projector epilogues where the reference composes tensor ops:
//   Landweber   forward epilogue  r = A x - y        (solvers.cpp:136)
//               backproj epilogue x = (-alpha) A'r + x, non-finite flag (:139-142)
//   CG          per-element fp64 dot products with a fixed reduction tree,
//               fp32 vector updates, per-element freeze flags (:47-107)
// Per-element scalars stay on the device; the host only launches, so an
// iteration never waits on the GPU.  Every reduction has a fixed order that
// depends neither on the batch size nor on the grid, so batched runs equal
// per-element runs bit for bit (the reference's batch invariance, solvers.hpp:24-27).
#include <cuda_fp16.h>

#include <climits>
#include <cmath>
#include <random>

#include "rk_internal.hpp"

namespace rk {

namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 64;  // partial sums per packed group (fixed: reduction order is batch-independent)

template <class T>
__device__ __forceinline__ T cast_from(float v);
template <>
__device__ __forceinline__ float cast_from<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half cast_from<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ double cast_from<double>(float v) { return double(v); }

__device__ __forceinline__ void block_reduce_store(double4 v, double4* partial_out) {
  __shared__ double4 red[kRedThreads];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      double4 a = red[threadIdx.x], b = red[threadIdx.x + w];
      red[threadIdx.x] = make_double4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *partial_out = red[0];
}

// per packed group g and image q: sum_i a[i].q * b[i].q in fp64 (tensor.cpp:378-389)
__global__ void __launch_bounds__(kRedThreads) dot_partial_kernel(const float4* __restrict__ a,
                                                                  const float4* __restrict__ b, int64_t plane,
                                                                  double4* __restrict__ partial) {
  const int64_t g = blockIdx.y;
  const float4* pa = a + g * plane;
  const float4* pb = b + g * plane;
  double4 acc = make_double4(0, 0, 0, 0);
  for (int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; i < plane; i += int64_t(kRedBlocks) * kRedThreads) {
    const float4 x = pa[i], y = pb[i];
    acc.x += double(x.x) * double(y.x);
    acc.y += double(x.y) * double(y.y);
    acc.z += double(x.z) * double(y.z);
    acc.w += double(x.w) * double(y.w);
  }
  block_reduce_store(acc, partial + g * kRedBlocks + blockIdx.x);
}

// out[4g + q] = sum over the group's partials, in order
__global__ void dot_final_kernel(const double4* __restrict__ partial, int64_t groups, double* __restrict__ out) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  double4 s = make_double4(0, 0, 0, 0);
  for (int k = 0; k < kRedBlocks; ++k) {
    const double4 v = partial[g * kRedBlocks + k];
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  out[4 * g + 0] = s.x;
  out[4 * g + 1] = s.y;
  out[4 * g + 2] = s.z;
  out[4 * g + 3] = s.w;
}

// packed image -> user layout [B][s][s] in the storage dtype (convert(x, guess.precision()))
template <class T>
__global__ void unpack_images_kernel(const float4* __restrict__ src, int64_t batch, int s, T* __restrict__ dst) {
  const int P = s + 2;
  const int64_t g = blockIdx.y;
  const int64_t n = int64_t(s) * s;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < n; idx += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(idx / s), j = int(idx % s);
    const float4 v = src[g * int64_t(P) * P + int64_t(i + 1) * P + (j + 1)];
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < kPack; ++q) {
      const int64_t b = g * kPack + q;
      if (b < batch) dst[b * n + idx] = cast_from<T>(vv[q]);
    }
  }
}

// c = a - b (elementwise, packed)
__global__ void sub_kernel(const float4* __restrict__ a, const float4* __restrict__ b, int64_t n,
                           float4* __restrict__ c) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 x = a[i], y = b[i];
    c[i] = make_float4(x.x - y.x, x.y - y.y, x.z - y.z, x.w - y.w);
  }
}

// x = float(double(z) * inv)   (estimate_alpha's rescale, solvers.cpp:125)
__global__ void scale_kernel(const float4* __restrict__ z, int64_t n, double inv, float4* __restrict__ x) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = z[i];
    x[i] = make_float4(float(double(v.x) * inv), float(double(v.y) * inv), float(double(v.z) * inv),
                       float(double(v.w) * inv));
  }
}

// CG state per batch element e
struct CgScalars {
  double* rs;      // r'r of the current residual
  double* normb;   // ||b||
  double* pap;     // p'Ap
  double* rsn;     // r'r after the update
  float* alpha;    // T(rs / pap)
  float* beta;     // T(rsn / rs)
  int* done;       // frozen (tolerance reached)
  int* act;        // updated this iteration
  int* pupd;       // p refreshed this iteration
  int* npd;        // first iteration with non-positive curvature (INT_MAX = none)
};

__global__ void cg_init_kernel(CgScalars c, int64_t batch, double tol) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= batch) return;
  c.normb[e] = sqrt(c.normb[e]);  // normb held b'b
  c.done[e] = sqrt(c.rs[e]) <= tol * c.normb[e] ? 1 : 0;  // solvers.cpp:58-63
}

// solvers.cpp:66-79
__global__ void cg_alpha_kernel(CgScalars c, int64_t groups, int64_t batch, int iteration) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= groups * kPack) return;
  int act = 0;
  float alpha = 0.f;
  if (e < batch && !c.done[e]) {
    if (c.pap[e] <= 0.0) atomicMin(c.npd, iteration);  // NotPositiveDefiniteError (solvers.cpp:69-75)
    alpha = float(c.rs[e] / c.pap[e]);
    act = 1;
  }
  c.alpha[e] = alpha;
  c.act[e] = act;
}

// x += alpha p; r -= alpha ap (active elements only), and partial r'r (solvers.cpp:80-92)
__global__ void __launch_bounds__(kRedThreads) cg_update_kernel(float4* __restrict__ x, float4* __restrict__ r,
                                                                const float4* __restrict__ p,
                                                                const float4* __restrict__ ap, int64_t plane,
                                                                CgScalars c, double4* __restrict__ partial) {
  const int64_t g = blockIdx.y;
  const float a0 = c.alpha[4 * g], a1 = c.alpha[4 * g + 1], a2 = c.alpha[4 * g + 2], a3 = c.alpha[4 * g + 3];
  const bool m0 = c.act[4 * g], m1 = c.act[4 * g + 1], m2 = c.act[4 * g + 2], m3 = c.act[4 * g + 3];
  double4 acc = make_double4(0, 0, 0, 0);
  for (int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; i < plane; i += int64_t(kRedBlocks) * kRedThreads) {
    const int64_t k = g * plane + i;
    float4 xv = x[k], rv = r[k];
    const float4 pv = p[k], av = ap[k];
    if (m0) xv.x = __fadd_rn(xv.x, __fmul_rn(a0, pv.x)), rv.x = __fsub_rn(rv.x, __fmul_rn(a0, av.x));
    if (m1) xv.y = __fadd_rn(xv.y, __fmul_rn(a1, pv.y)), rv.y = __fsub_rn(rv.y, __fmul_rn(a1, av.y));
    if (m2) xv.z = __fadd_rn(xv.z, __fmul_rn(a2, pv.z)), rv.z = __fsub_rn(rv.z, __fmul_rn(a2, av.z));
    if (m3) xv.w = __fadd_rn(xv.w, __fmul_rn(a3, pv.w)), rv.w = __fsub_rn(rv.w, __fmul_rn(a3, av.w));
    x[k] = xv;
    r[k] = rv;
    acc.x += double(rv.x) * double(rv.x);
    acc.y += double(rv.y) * double(rv.y);
    acc.z += double(rv.z) * double(rv.z);
    acc.w += double(rv.w) * double(rv.w);
  }
  block_reduce_store(acc, partial + g * kRedBlocks + blockIdx.x);
}

// freeze / beta (solvers.cpp:93-104)
__global__ void cg_beta_kernel(CgScalars c, int64_t groups, double tol) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= groups * kPack) return;
  int pupd = 0;
  float beta = 0.f;
  if (c.act[e]) {
    const double rsn = c.rsn[e];
    if (sqrt(rsn) <= tol * c.normb[e]) {
      c.done[e] = 1;
    } else {
      beta = float(rsn / c.rs[e]);
      pupd = 1;
    }
    c.rs[e] = rsn;
  }
  c.beta[e] = beta;
  c.pupd[e] = pupd;
}

// p = r + beta p for refreshed elements (solvers.cpp:102)
__global__ void cg_p_kernel(float4* __restrict__ p, const float4* __restrict__ r, int64_t plane, CgScalars c) {
  const int64_t g = blockIdx.y;
  const float b0 = c.beta[4 * g], b1 = c.beta[4 * g + 1], b2 = c.beta[4 * g + 2], b3 = c.beta[4 * g + 3];
  const bool m0 = c.pupd[4 * g], m1 = c.pupd[4 * g + 1], m2 = c.pupd[4 * g + 2], m3 = c.pupd[4 * g + 3];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < plane; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = g * plane + i;
    float4 pv = p[k];
    const float4 rv = r[k];
    if (m0) pv.x = __fadd_rn(rv.x, __fmul_rn(b0, pv.x));
    if (m1) pv.y = __fadd_rn(rv.y, __fmul_rn(b1, pv.y));
    if (m2) pv.z = __fadd_rn(rv.z, __fmul_rn(b2, pv.z));
    if (m3) pv.w = __fadd_rn(rv.w, __fmul_rn(b3, pv.w));
    p[k] = pv;
  }
}

inline unsigned grid_for(int64_t n, int threads, unsigned cap = 8192) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap)));
}

// ------------------------------------------------------------------ host helpers
void dot(const float4* a, const float4* b, int64_t groups, int64_t plane, double4* partial, double* out,
         cudaStream_t st) {
  {
    KernelTimer t(RK_KERNEL_SOLVER, st);
    dot_partial_kernel<<<dim3(kRedBlocks, unsigned(groups)), kRedThreads, 0, st>>>(a, b, plane, partial);
  }
  KernelTimer t(RK_KERNEL_SOLVER, st);
  dot_final_kernel<<<grid_for(groups, 128), 128, 0, st>>>(partial, groups, out);
}

// forward of a packed image (+ its transpose when the schedule needs one)
void apply_forward(Plan& p, const float4* x, float4* xt, int64_t batch, FwdEpilogue epi, cudaStream_t st) {
  ensure_forward_schedule(p);
  if (p.fwd.any_transposed) launch_transpose_images(x, groups_of(batch), p.s, xt, st);
  launch_forward(p, x, xt, batch, RK_F32, nullptr, st, epi);
}

}  // namespace

void unpack_images(int dtype, const float4* src, int64_t batch, int64_t s, void* dst, cudaStream_t st) {
  dim3 grid(grid_for(s * s, 256, 4096), unsigned(groups_of(batch)));
  KernelTimer t(RK_KERNEL_PACK, st);
  switch (dtype) {
    case RK_F16: unpack_images_kernel<__half><<<grid, 256, 0, st>>>(src, batch, int(s), static_cast<__half*>(dst)); break;
    case RK_F32: unpack_images_kernel<float><<<grid, 256, 0, st>>>(src, batch, int(s), static_cast<float*>(dst)); break;
    case RK_F64: unpack_images_kernel<double><<<grid, 256, 0, st>>>(src, batch, int(s), static_cast<double*>(dst)); break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
  RK_CUDA(cudaGetLastError());
}

// solvers.cpp:130-145
int run_landweber(Plan& p, int dtype, const void* d_y, const void* d_guess, int64_t batch, double alpha,
                  int iterations, void* d_x, cudaStream_t st) {
  if (iterations < 0) throw ValidationError("landweber iteration count must be >= 0");
  const int64_t G = groups_of(batch), P = p.s + 2;
  const int64_t img_plane = P * P, sino_plane = p.na * p.nd;
  p.solver_a.reserve(size_t(G * img_plane) * sizeof(float4));   // x
  p.solver_b.reserve(size_t(G * img_plane) * sizeof(float4));   // x transposed
  p.solver_c.reserve(size_t(G * sino_plane) * sizeof(float4));  // y
  p.solver_d.reserve(size_t(G * sino_plane) * sizeof(float4));  // residual
  p.solver_scalars.reserve(sizeof(int) * 16);
  float4* X = p.solver_a.as<float4>();
  float4* XT = p.solver_b.as<float4>();
  float4* Y = p.solver_c.as<float4>();
  float4* Rs = p.solver_d.as<float4>();
  int* flag = p.solver_scalars.as<int>();
  const int none = INT_MAX;
  RK_CUDA(cudaMemcpyAsync(flag, &none, sizeof(int), cudaMemcpyHostToDevice, st));
  launch_pack_images(dtype, d_guess, batch, p.s, X, st);  // convert(guess, compute precision)
  launch_pack_sino(dtype, d_y, batch, p.na, p.nd, Y, st);
  const float neg_alpha = float(-alpha);  // axpy(-alpha, ...) narrows alpha to float (tensor.cpp:338-343)
  for (int it = 0; it < iterations; ++it) {
    FwdEpilogue fe;
    fe.mode = kOutResidual;
    fe.packed = Rs;
    fe.resid = Y;
    apply_forward(p, X, XT, batch, fe, st);
    BpEpilogue be;
    be.mode = kOutAxpy;
    be.packed = X;
    be.neg_alpha = neg_alpha;
    be.flag = flag;
    be.iteration = it;
    launch_backproject(p, Rs, batch, RK_F32, nullptr, st, be);
  }
  unpack_images(dtype, X, batch, p.s, d_x, st);
  int h_flag = none;
  RK_CUDA(cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaStreamSynchronize(st));
  return h_flag == none ? -1 : h_flag;
}

size_t cg_scalar_bytes(int64_t batch) {
  const size_t ne = size_t(groups_of(batch) * kPack);
  return size_t(groups_of(batch)) * kRedBlocks * sizeof(double4) + ne * (4 * sizeof(double) + 2 * sizeof(float) + 4 * sizeof(int)) + 64;
}

// system apply over packed images: out = A'(A in)  (sys == nullptr, solvers.cpp:164)
// or out = c0 A'(A in) + c1 in  (admm.cpp:142: axpy(p0, A'A x, scale(x, 1 + p1)))
static void apply_system(Plan& p, const float4* in, float4* out, int64_t batch, const CgSystem* sys, float4* xt,
                         float4* sino, cudaStream_t st) {
  FwdEpilogue fe;
  fe.mode = kOutPacked;
  fe.packed = sino;
  apply_forward(p, in, xt, batch, fe, st);
  BpEpilogue be;
  be.mode = sys ? kOutSystem : kOutPacked;
  be.packed = out;
  if (sys) {
    be.src = in;
    be.c0 = sys->c0;
    be.c1 = sys->c1;
  }
  launch_backproject(p, sino, batch, RK_F32, nullptr, st, be);
}

// solvers.cpp:47-107: CG from x (updated in place) on the packed system; the
// image borders of b and x are zero.  work: 4 packed image planes (r, p, ap,
// transposed scratch); npd receives atomicMin(first non-positive-curvature iteration).
void cg_packed(Plan& p, int64_t batch, const float4* Bv, float4* X, int max_iter, double tol, const CgSystem* sys,
               float4* work, float4* S, void* scalars, int* npd, cudaStream_t st) {
  const int64_t G = groups_of(batch), P = p.s + 2, img_plane = P * P;
  const size_t ne = size_t(G * kPack);
  float4* R = work;
  float4* Pv = work + G * img_plane;
  float4* AP = work + 2 * G * img_plane;
  float4* T = work + 3 * G * img_plane;
  char* sc = static_cast<char*>(scalars);
  double4* partial = reinterpret_cast<double4*>(sc);
  sc += size_t(G) * kRedBlocks * sizeof(double4);
  CgScalars c;
  c.rs = reinterpret_cast<double*>(sc);
  c.normb = c.rs + ne;
  c.pap = c.normb + ne;
  c.rsn = c.pap + ne;
  c.alpha = reinterpret_cast<float*>(c.rsn + ne);
  c.beta = c.alpha + ne;
  c.done = reinterpret_cast<int*>(c.beta + ne);
  c.act = c.done + ne;
  c.pupd = c.act + ne;
  c.npd = npd;
  // the backprojection writes interiors only: keep ap's border zero
  RK_CUDA(cudaMemsetAsync(AP, 0, size_t(G * img_plane) * sizeof(float4), st));
  // r = b - apply(x); p = r (solvers.cpp:51-52)
  apply_system(p, X, AP, batch, sys, T, S, st);
  {
    KernelTimer t(RK_KERNEL_SOLVER, st);
    sub_kernel<<<grid_for(G * img_plane, 256), 256, 0, st>>>(Bv, AP, G * img_plane, R);
  }
  RK_CUDA(cudaMemcpyAsync(Pv, R, size_t(G * img_plane) * sizeof(float4), cudaMemcpyDeviceToDevice, st));
  dot(R, R, G, img_plane, partial, c.rs, st);
  dot(Bv, Bv, G, img_plane, partial, c.normb, st);
  {
    KernelTimer t(RK_KERNEL_SOLVER, st);
    cg_init_kernel<<<grid_for(batch, 128), 128, 0, st>>>(c, batch, tol);
  }
  if (ne > size_t(batch))
    RK_CUDA(cudaMemsetAsync(c.done + batch, 0xff, sizeof(int) * (ne - size_t(batch)), st));  // padding: frozen
  for (int it = 0; it < max_iter; ++it) {
    apply_system(p, Pv, AP, batch, sys, T, S, st);
    dot(Pv, AP, G, img_plane, partial, c.pap, st);
    {
      KernelTimer t(RK_KERNEL_SOLVER, st);
      cg_alpha_kernel<<<grid_for(G * kPack, 128), 128, 0, st>>>(c, G, batch, it);
    }
    {
      KernelTimer t(RK_KERNEL_SOLVER, st);
      cg_update_kernel<<<dim3(kRedBlocks, unsigned(G)), kRedThreads, 0, st>>>(X, R, Pv, AP, img_plane, c, partial);
    }
    {
      KernelTimer t(RK_KERNEL_SOLVER, st);
      dot_final_kernel<<<grid_for(G, 128), 128, 0, st>>>(partial, G, c.rsn);
    }
    {
      KernelTimer t(RK_KERNEL_SOLVER, st);
      cg_beta_kernel<<<grid_for(G * kPack, 128), 128, 0, st>>>(c, G, tol);
    }
    {
      KernelTimer t(RK_KERNEL_SOLVER, st);
      cg_p_kernel<<<dim3(grid_for(img_plane, 256, 512), unsigned(G)), 256, 0, st>>>(Pv, R, img_plane, c);
    }
  }
}

// solvers.cpp:47-107 + 162-166 (CG on A'A x = A'y)
int run_cgne(Plan& p, int dtype, const void* d_y, const void* d_guess, int64_t batch, int max_iter, double tol,
             void* d_x, cudaStream_t st) {
  if (max_iter < 0) throw ValidationError("cg max_iter must be >= 0");
  if (tol < 0.0) throw ValidationError("cg tolerance must be >= 0");
  const int64_t G = groups_of(batch), P = p.s + 2;
  const int64_t img_plane = P * P, sino_plane = p.na * p.nd;
  const size_t ib = size_t(G * img_plane) * sizeof(float4), sb = size_t(G * sino_plane) * sizeof(float4);
  // x, b, 4 CG work planes | sinogram scratch
  p.solver_a.reserve(6 * ib);
  p.solver_c.reserve(sb);
  p.solver_scalars.reserve(cg_scalar_bytes(batch) + 64);
  char* base = p.solver_a.as<char>();
  float4* X = reinterpret_cast<float4*>(base);
  float4* Bv = reinterpret_cast<float4*>(base + ib);
  float4* work = reinterpret_cast<float4*>(base + 2 * ib);
  float4* S = p.solver_c.as<float4>();
  int* npd = p.solver_scalars.as<int>();
  void* scalars = p.solver_scalars.as<char>() + 64;
  const int none = INT_MAX;
  RK_CUDA(cudaMemcpyAsync(npd, &none, sizeof(int), cudaMemcpyHostToDevice, st));

  // b = A'y, narrowed to the storage precision like op.adjoint(y) (solvers.cpp:163)
  launch_pack_sino(dtype, d_y, batch, p.na, p.nd, S, st);
  BpEpilogue pk;
  pk.mode = kOutPacked;
  pk.packed = Bv;
  RK_CUDA(cudaMemsetAsync(Bv, 0, ib, st));
  launch_backproject(p, S, batch, dtype, nullptr, st, pk);
  // x = guess
  launch_pack_images(dtype, d_guess, batch, p.s, X, st);
  cg_packed(p, batch, Bv, X, max_iter, tol, nullptr, work, S, scalars, npd, st);
  unpack_images(dtype, X, batch, p.s, d_x, st);
  int h_npd = none;
  RK_CUDA(cudaMemcpyAsync(&h_npd, npd, sizeof(int), cudaMemcpyDeviceToHost, st));
  RK_CUDA(cudaStreamSynchronize(st));
  return h_npd == none ? -1 : h_npd;
}

// solvers.cpp:111-128 (batch 1; fp32 apply, fp64 norms and rescale)
double run_estimate_alpha(Plan& p, int iterations, uint64_t seed, cudaStream_t st) {
  if (iterations < 1) throw ValidationError("estimate_alpha needs at least one iteration");
  const int64_t s = p.s, P = s + 2, img_plane = P * P, sino_plane = p.na * p.nd;
  // x = Rng(seed).uniform_tensor({1, s, s}, Double) (rng.hpp:13-31)
  std::mt19937 eng(uint32_t(seed ^ (seed >> 32)));
  std::vector<double> x0(size_t(s * s));
  double nx2 = 0.0;
  for (auto& v : x0) {
    v = double(float(eng() >> 8) * 0x1.0p-24f);
    nx2 += v * v;
  }
  const double nx = std::sqrt(nx2);
  if (nx == 0.0) throw NumericalError("estimate_alpha: start vector is zero");
  for (auto& v : x0) v = v * (1.0 / nx);
  const size_t ib = size_t(img_plane) * sizeof(float4);
  p.solver_a.reserve(3 * ib + s * s * sizeof(double));
  p.solver_c.reserve(size_t(sino_plane) * sizeof(float4));
  p.solver_scalars.reserve(kRedBlocks * sizeof(double4) + 4 * sizeof(double));
  char* base = p.solver_a.as<char>();
  float4* X = reinterpret_cast<float4*>(base);
  float4* T = reinterpret_cast<float4*>(base + ib);
  float4* Z = reinterpret_cast<float4*>(base + 2 * ib);
  double* staging = reinterpret_cast<double*>(base + 3 * ib);
  float4* S = p.solver_c.as<float4>();
  double4* partial = p.solver_scalars.as<double4>();
  double* nz_d = reinterpret_cast<double*>(partial + kRedBlocks);
  RK_CUDA(cudaMemcpyAsync(staging, x0.data(), x0.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  launch_pack_images(RK_F64, staging, 1, s, X, st);
  RK_CUDA(cudaMemsetAsync(Z, 0, ib, st));
  FwdEpilogue fe;
  fe.mode = kOutPacked;
  fe.packed = S;
  BpEpilogue be;
  be.mode = kOutPacked;
  be.packed = Z;
  double sigma2 = 0.0;
  for (int it = 0; it < iterations; ++it) {
    apply_forward(p, X, T, 1, fe, st);
    launch_backproject(p, S, 1, RK_F32, nullptr, st, be);
    dot(Z, Z, 1, img_plane, partial, nz_d, st);
    double nz2 = 0.0;
    RK_CUDA(cudaMemcpyAsync(&nz2, nz_d, sizeof(double), cudaMemcpyDeviceToHost, st));
    RK_CUDA(cudaStreamSynchronize(st));
    const double nz = std::sqrt(nz2);
    if (!(nz > 0.0) || !std::isfinite(nz))
      throw NumericalError("estimate_alpha: power iteration collapsed at iteration " + std::to_string(it));
    sigma2 = nz;
    KernelTimer t(RK_KERNEL_SOLVER, st);
    scale_kernel<<<grid_for(img_plane, 256), 256, 0, st>>>(Z, img_plane, 1.0 / nz, X);
  }
  RK_CUDA(cudaStreamSynchronize(st));
  return 2.0 / sigma2;
}

}  // namespace rk
