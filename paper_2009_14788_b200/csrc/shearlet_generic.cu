// Alpha-shearlet analysis / synthesis on grids that are not a power of two
// (§8f rank 3; reference shearlet.cpp:253-294 accepts any square grid >= 2,
// its FFTW plans any size).  shearlet.cu's radix-2 shared-memory FFTs cover
// power-of-two grids; here a 2-D DFT is two complex contractions with the
// n x n DFT matrix W[j][k] = exp(-2 pi i j k / n), generated on the fly from
// an n-entry table ((j k) mod n):
//   rows:    O[p][r][k] = sum_j A[p][r][j] W[j][k]
//   columns: O[p][k][c] = sum_i W[k][i] A[p][i][c]
// as 32 x 32 output tiles (a CTA stages 32 x 32 tiles of A and W in shared
// memory, each thread owns four outputs).  O(n^3) per plane instead of
// O(n^2 log n) — a completeness path (e.g. 1000^2: ~12 ms per image and
// transform), fp32 for fp32 / fp16 storage and fp64 for fp64 storage, as the
// reference splits precision (shearlet.cpp:303-310).
//
// Transform structure as in shearlet.cu (natural order here): analysis
// X = DFT2(x); coefficient pair q: Re/Im(IDFT2(X (M_2q + i M_2q+1))) / n^2 =
// c_2q, c_2q+1 (the multipliers are real and even).  Synthesis: Z_q =
// DFT2(c_2q + i c_2q+1), S = sum_q Z_q (M_2q - i M_2q+1) in ascending q (a
// batch-independent order), image = Re(IDFT2(S)) / n^2.  The ADMM fusions
// (shrink + dual update in the analysis store, synthesis of z1 - u1) are
// the same epilogues as shearlet.cu's.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "rk_internal.hpp"

namespace rk {

namespace {

template <class R>
struct Cg;
template <>
struct Cg<float> {
  using T = float2;
};
template <>
struct Cg<double> {
  using T = double2;
};

template <class R, class T>
__device__ __forceinline__ R ldr(const T* p) {
  return R(*p);
}
template <>
__device__ __forceinline__ float ldr<float, __half>(const __half* p) {
  return __half2float(*p);
}
template <class T, class R>
__device__ __forceinline__ T str(R v) {
  return T(v);
}
template <>
__device__ __forceinline__ __half str<__half, float>(float v) {
  return __float2half_rn(v);
}

constexpr int kT = 32;      // output tile edge
constexpr int kRows = 8;    // thread rows per CTA (kT x kRows threads, kT / kRows outputs each)

// One 2-D DFT half-pass over `planes` n x n complex planes (LEFT: columns,
// W on the left; else rows, W on the right).  CONJ: inverse (conjugate W).
template <class R, bool LEFT, bool CONJ>
__global__ void __launch_bounds__(kT * kRows) dft_pass_kernel(const typename Cg<R>::T* __restrict__ in,
                                                             typename Cg<R>::T* __restrict__ out, int n,
                                                             const typename Cg<R>::T* __restrict__ tw, R scale) {
  using C = typename Cg<R>::T;
  __shared__ C sa[kT][kT + 1];  // LEFT: A[i][c]; else A[r][j]
  __shared__ C sw[kT][kT + 1];  // LEFT: W[k][i]; else W[j][k]
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t plane = int64_t(n) * n;
  const C* a = in + blockIdx.z * plane;
  // output tile: LEFT rows k0.., cols c0..; else rows r0.., cols k0..
  const int o_row0 = blockIdx.y * kT, o_col0 = blockIdx.x * kT;
  C acc[kT / kRows];
#pragma unroll
  for (int i = 0; i < kT / kRows; ++i) acc[i] = C{R(0), R(0)};
  for (int s0 = 0; s0 < n; s0 += kT) {  // contraction index j (rows) / i (columns)
#pragma unroll
    for (int i = 0; i < kT / kRows; ++i) {
      const int rr = ty + kRows * i;
      // A tile (coalesced along tx)
      int ar, ac;
      if (LEFT) {
        ar = s0 + rr;
        ac = o_col0 + tx;
      } else {
        ar = o_row0 + rr;
        ac = s0 + tx;
      }
      sa[rr][tx] = (ar < n && ac < n) ? a[int64_t(ar) * n + ac] : C{R(0), R(0)};
      // W tile: W[x][y] = tw[(x y) mod n], symmetric
      int wx, wy;
      if (LEFT) {
        wx = o_row0 + rr;  // k
        wy = s0 + tx;      // i
      } else {
        wx = s0 + rr;      // j
        wy = o_col0 + tx;  // k
      }
      C w = C{R(0), R(0)};
      if (wx < n && wy < n) {
        w = __ldg(tw + int((int64_t(wx) * wy) % n));
        if (CONJ) w.y = -w.y;
      }
      sw[rr][tx] = w;
    }
    __syncthreads();
    const int lim = min(kT, n - s0);
    for (int t = 0; t < lim; ++t) {
      if (LEFT) {
        const C av = sa[t][tx];  // A[i = s0 + t][c]
#pragma unroll
        for (int i = 0; i < kT / kRows; ++i) {
          const C w = sw[ty + kRows * i][t];  // W[k][i]
          acc[i].x = fma(w.x, av.x, fma(-w.y, av.y, acc[i].x));
          acc[i].y = fma(w.x, av.y, fma(w.y, av.x, acc[i].y));
        }
      } else {
        const C w = sw[t][tx];  // W[j = s0 + t][k]
#pragma unroll
        for (int i = 0; i < kT / kRows; ++i) {
          const C av = sa[ty + kRows * i][t];  // A[r][j]
          acc[i].x = fma(av.x, w.x, fma(-av.y, w.y, acc[i].x));
          acc[i].y = fma(av.x, w.y, fma(av.y, w.x, acc[i].y));
        }
      }
    }
    __syncthreads();
  }
  C* o = out + blockIdx.z * plane;
#pragma unroll
  for (int i = 0; i < kT / kRows; ++i) {
    const int r = o_row0 + ty + kRows * i, c = o_col0 + tx;
    if (r < n && c < n) o[int64_t(r) * n + c] = C{acc[i].x * scale, acc[i].y * scale};
  }
}

template <class R>
struct Gen {
  using C = typename Cg<R>::T;
  int n;
  const C* tw;
  const C* mult2;  // {M_2q, M_2q+1} per bin, natural order
};

// 2-D DFT of `planes` planes: src -> (rows) tmp -> (columns) dst; tmp must differ
// from both (a pass reads whole planes), src may equal dst.
template <class R, bool INV>
void dft2(const Gen<R>& g, const typename Cg<R>::T* src, typename Cg<R>::T* tmp, typename Cg<R>::T* dst,
          int64_t planes, R scale, cudaStream_t st) {
  const int tiles = (g.n + kT - 1) / kT;
  for (int64_t p0 = 0; p0 < planes; p0 += 65535) {
    const int64_t np = std::min<int64_t>(65535, planes - p0);
    const int64_t off = p0 * int64_t(g.n) * g.n;
    const dim3 grid{unsigned(tiles), unsigned(tiles), unsigned(np)}, block{unsigned(kT), unsigned(kRows), 1u};
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    dft_pass_kernel<R, false, INV><<<grid, block, 0, st>>>(src + off, tmp + off, g.n, g.tw, R(1));
    dft_pass_kernel<R, true, INV><<<grid, block, 0, st>>>(tmp + off, dst + off, g.n, g.tw, scale);
  }
  RK_CUDA(cudaGetLastError());
}

// images [B][n][n] (real) -> complex planes
template <class T, class R>
__global__ void to_cx_kernel(const T* __restrict__ x, int64_t count, typename Cg<R>::T* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x)
    out[e] = {ldr<R>(x + e), R(0)};
}

// synthesis input: plane (b, qq) = (c[b][2q] - sub) + i (c[b][2q+1] - sub), q = q0 + qq
template <class T, class R>
__global__ void pack_pairs_kernel(const T* __restrict__ c, const T* __restrict__ sub, int64_t n2, int64_t B,
                                  int64_t q0, int64_t nq, int64_t K, typename Cg<R>::T* __restrict__ out) {
  const int64_t total = B * nq * n2;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bin = e % n2, item = e / n2, qq = item % nq, b = item / nq, k = 2 * (q0 + qq);
    const int64_t i0 = (b * K + k) * n2 + bin;
    R re = ldr<R>(c + i0), im = R(0);
    if (sub) re = re - ldr<R>(sub + i0);
    if (k + 1 < K) {
      im = ldr<R>(c + i0 + n2);
      if (sub) im = im - ldr<R>(sub + i0 + n2);
    }
    out[e] = {re, im};
  }
}

// analysis: plane (b, qq) = X[b] (M_2q + i M_2q+1)
template <class R>
__global__ void mul_pairs_kernel(const typename Cg<R>::T* __restrict__ X, const typename Cg<R>::T* __restrict__ m2,
                                 int64_t n2, int64_t B, int64_t q0, int64_t nq, typename Cg<R>::T* __restrict__ out) {
  const int64_t total = B * nq * n2;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bin = e % n2, item = e / n2, qq = item % nq, b = item / nq;
    const auto x = X[b * n2 + bin];
    const auto m = m2[(q0 + qq) * n2 + bin];
    out[e] = {x.x * m.x - x.y * m.y, x.x * m.y + x.y * m.x};
  }
}

// synthesis: S[b] (+)= sum_qq Z[b][qq] (M_2q - i M_2q+1), ascending qq
template <class R>
__global__ void acc_pairs_kernel(const typename Cg<R>::T* __restrict__ Z, const typename Cg<R>::T* __restrict__ m2,
                                 int64_t n2, int64_t B, int64_t q0, int64_t nq, bool first,
                                 typename Cg<R>::T* __restrict__ S) {
  const int64_t total = B * n2;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bin = e % n2, b = e / n2;
    auto s = first ? typename Cg<R>::T{R(0), R(0)} : S[e];
    for (int64_t qq = 0; qq < nq; ++qq) {
      const auto z = Z[(b * nq + qq) * n2 + bin];
      const auto m = m2[(q0 + qq) * n2 + bin];
      s.x += z.x * m.x + z.y * m.y;
      s.y += z.y * m.x - z.x * m.y;
    }
    S[e] = s;
  }
}

// analysis store: coeff[b][2q] = Re, coeff[b][2q+1] = Im (ADMM: the shrink / dual update instead)
template <class T, class R>
__global__ void store_pairs_kernel(const typename Cg<R>::T* __restrict__ Z, int64_t n2, int64_t B, int64_t q0,
                                   int64_t nq, int64_t K, T* __restrict__ coeff, float* __restrict__ z1,
                                   float* __restrict__ u1, const float* __restrict__ thresh, int* flag,
                                   const int* iteration) {
  const int64_t total = B * nq * n2;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bin = e % n2, item = e / n2, qq = item % nq, b = item / nq, k = 2 * (q0 + qq);
    const auto z = Z[e];
    for (int h = 0; h < 2 && k + h < K; ++h) {
      const R v = h ? z.y : z.x;
      const int64_t gi = (b * K + k + h) * n2 + bin;
      if (z1) {  // admm.cpp:150-153 (fp32), as shearlet.cu's admm_update
        const float c = float(v), u = u1[gi];
        float mabs = __fsub_rn(fabsf(__fadd_rn(c, u)), thresh[k + h]);
        if (mabs < 0.f) mabs = 0.f;
        const float a = __fadd_rn(c, u);
        const float zz = a < 0.f ? -mabs : (a > 0.f ? mabs : 0.f);
        const float un = __fadd_rn(u, __fsub_rn(c, zz));
        z1[gi] = zz;
        u1[gi] = un;
        if (!isfinite(un)) atomicMin(flag, *iteration);
      } else {
        coeff[gi] = str<T>(v);
      }
    }
  }
}

template <class T, class R>
__global__ void store_real_kernel(const typename Cg<R>::T* __restrict__ Z, int64_t count, T* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x)
    out[e] = str<T>(Z[e].x);
}

unsigned grid_for(int64_t count) { return unsigned(std::min<int64_t>((count + 255) / 256, 148 * 16)); }

template <class R>
Gen<R> gen_tables(Shearlet& sp);
template <>
Gen<float> gen_tables<float>(Shearlet& sp) {
  return {int(sp.height), sp.g_twiddle.as<float2>(), sp.g_mult2.as<float2>()};
}
template <>
Gen<double> gen_tables<double>(Shearlet& sp) {
  if (!sp.g_mult2_64.ptr) {
    std::vector<double2> m2, tw;
    build_generic_tables(sp, m2, tw);
    sp.g_twiddle64.reserve(tw.size() * sizeof(double2));
    RK_CUDA(cudaMemcpy(sp.g_twiddle64.ptr, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
    sp.g_mult2_64.reserve(m2.size() * sizeof(double2));
    RK_CUDA(cudaMemcpy(sp.g_mult2_64.ptr, m2.data(), m2.size() * sizeof(double2), cudaMemcpyHostToDevice));
  }
  return {int(sp.height), sp.g_twiddle64.as<double2>(), sp.g_mult2_64.as<double2>()};
}

// pairs per chunk so that the chunk's two scratch plane sets stay <= 1 GB
int64_t pair_chunk(int64_t B, int64_t P, int64_t plane_bytes) {
  return std::max<int64_t>(1, std::min<int64_t>(P, (int64_t(1) << 29) / std::max<int64_t>(B * plane_bytes, 1)));
}

template <class T, class R>
void forward_generic_impl(Shearlet& sp, const T* image, int64_t B, T* coeff, const GenericAdmm& admm, cudaStream_t st) {
  using C = typename Cg<R>::T;
  const Gen<R> g = gen_tables<R>(sp);
  const int64_t n = sp.height, n2 = n * n, K = sp.n_coeff, P = (K + 1) / 2;
  const int64_t nq = pair_chunk(B, P, n2 * int64_t(sizeof(C)));
  sp.work_a.reserve(size_t(2 * B * n2) * sizeof(C));
  sp.work_b.reserve(size_t(2 * B * nq * n2) * sizeof(C));
  C* X = sp.work_a.as<C>();
  C* T1 = X + B * n2;
  C* W1 = sp.work_b.as<C>();
  C* W2 = W1 + B * nq * n2;
  {
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    to_cx_kernel<T, R><<<grid_for(B * n2), 256, 0, st>>>(image, B * n2, X);
  }
  dft2<R, false>(g, X, T1, X, B, R(1), st);  // X = DFT2(x) (rows into T1, columns back into X)
  const R scale = R(1) / R(n2);
  for (int64_t q0 = 0; q0 < P; q0 += nq) {
    const int64_t cq = std::min(nq, P - q0);
    {
      KernelTimer t(RK_KERNEL_SHEARLET, st);
      mul_pairs_kernel<R><<<grid_for(B * cq * n2), 256, 0, st>>>(X, g.mult2, n2, B, q0, cq, W1);
    }
    dft2<R, true>(g, W1, W2, W1, B * cq, scale, st);
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    store_pairs_kernel<T, R><<<grid_for(B * cq * n2), 256, 0, st>>>(W1, n2, B, q0, cq, K, coeff, admm.z1, admm.u1,
                                                                     admm.thresh, admm.flag, admm.iteration);
  }
  RK_CUDA(cudaGetLastError());
}

template <class T, class R>
void backward_generic_impl(Shearlet& sp, const T* coeff, const T* sub, int64_t B, T* image, cudaStream_t st) {
  using C = typename Cg<R>::T;
  const Gen<R> g = gen_tables<R>(sp);
  const int64_t n = sp.height, n2 = n * n, K = sp.n_coeff, P = (K + 1) / 2;
  const int64_t nq = pair_chunk(B, P, n2 * int64_t(sizeof(C)));
  sp.work_a.reserve(size_t(2 * B * n2) * sizeof(C));
  sp.work_b.reserve(size_t(2 * B * nq * n2) * sizeof(C));
  C* S = sp.work_a.as<C>();
  C* T1 = S + B * n2;
  C* W1 = sp.work_b.as<C>();
  C* W2 = W1 + B * nq * n2;
  for (int64_t q0 = 0; q0 < P; q0 += nq) {
    const int64_t cq = std::min(nq, P - q0);
    {
      KernelTimer t(RK_KERNEL_SHEARLET, st);
      pack_pairs_kernel<T, R><<<grid_for(B * cq * n2), 256, 0, st>>>(coeff, sub, n2, B, q0, cq, K, W1);
    }
    dft2<R, false>(g, W1, W2, W1, B * cq, R(1), st);
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    acc_pairs_kernel<R><<<grid_for(B * n2), 256, 0, st>>>(W1, g.mult2, n2, B, q0, cq, q0 == 0, S);
  }
  dft2<R, true>(g, S, T1, S, B, R(1) / R(n2), st);
  {
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    store_real_kernel<T, R><<<grid_for(B * n2), 256, 0, st>>>(S, B * n2, image);
  }
  RK_CUDA(cudaGetLastError());
}

}  // namespace

// {M_2q, M_2q+1} per bin in natural order (zero for a missing odd partner) and
// the n-entry DFT table exp(-2 pi i m / n), both from the fp64 plan
template <class C>
void build_generic_tables(const Shearlet& sp, std::vector<C>& mult2, std::vector<C>& tw) {
  const int64_t n = sp.height, bins = n * n, K = sp.n_coeff, P = (K + 1) / 2;
  using R = decltype(C{}.x);
  mult2.assign(size_t(P * bins), C{R(0), R(0)});
  for (int64_t k = 0; k < K; ++k) {
    const double* m = sp.multipliers.data() + k * bins;
    C* d = mult2.data() + (k / 2) * bins;
    for (int64_t b = 0; b < bins; ++b) {
      if (k % 2 == 0)
        d[b].x = R(m[b]);
      else
        d[b].y = R(m[b]);
    }
  }
  tw.resize(size_t(n));
  for (int64_t m = 0; m < n; ++m) {
    const double ang = 2.0 * M_PI * double(m) / double(n);
    tw[size_t(m)] = C{R(std::cos(ang)), R(-std::sin(ang))};
  }
}
template void build_generic_tables<float2>(const Shearlet&, std::vector<float2>&, std::vector<float2>&);
template void build_generic_tables<double2>(const Shearlet&, std::vector<double2>&, std::vector<double2>&);

void upload_shearlet_generic(Shearlet& sp) {
  std::vector<float2> m2, tw;
  build_generic_tables(sp, m2, tw);
  rk::set_device(sp.device);
  sp.g_mult2.reserve(m2.size() * sizeof(float2));
  sp.g_twiddle.reserve(tw.size() * sizeof(float2));
  RK_CUDA(cudaMemcpy(sp.g_mult2.ptr, m2.data(), m2.size() * sizeof(float2), cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(sp.g_twiddle.ptr, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice));
}

void shearlet_forward_generic(Shearlet& sp, int dtype, const void* image, int64_t batch, void* coeff,
                              const GenericAdmm& admm, cudaStream_t st) {
  switch (dtype) {
    case RK_F16:
      forward_generic_impl<__half, float>(sp, static_cast<const __half*>(image), batch, static_cast<__half*>(coeff),
                                          admm, st);
      break;
    case RK_F32:
      forward_generic_impl<float, float>(sp, static_cast<const float*>(image), batch, static_cast<float*>(coeff),
                                         admm, st);
      break;
    case RK_F64:
      forward_generic_impl<double, double>(sp, static_cast<const double*>(image), batch, static_cast<double*>(coeff),
                                           admm, st);
      break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
}

void shearlet_backward_generic(Shearlet& sp, int dtype, const void* coeff, const void* sub, int64_t batch,
                               void* image, cudaStream_t st) {
  switch (dtype) {
    case RK_F16:
      backward_generic_impl<__half, float>(sp, static_cast<const __half*>(coeff), static_cast<const __half*>(sub),
                                           batch, static_cast<__half*>(image), st);
      break;
    case RK_F32:
      backward_generic_impl<float, float>(sp, static_cast<const float*>(coeff), static_cast<const float*>(sub), batch,
                                          static_cast<float*>(image), st);
      break;
    case RK_F64:
      backward_generic_impl<double, double>(sp, static_cast<const double*>(coeff), static_cast<const double*>(sub),
                                            batch, static_cast<double*>(image), st);
      break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
}

}  // namespace rk
