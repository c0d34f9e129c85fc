// Ramp-filter kernel (sm_100a): per detector row, zero-pad to P, FFT,
// multiply by the real frequency response, inverse FFT, crop and scale by
// pi / (2 n_angles) — sino_filter.cpp:98-124 (filtration always fp32,
// :106-123).
//
// One CTA filters the four rows (b = 4g..4g+3, angle a) that share one
// packed float4 sinogram cell, as two complex shared-memory radix-2 FFTs:
// the response is real and even, so for z = x + i y,
// IFFT(FFT(z) H) = x*h + i (y*h) filters two real rows at once (SURVEY
// 7.3-6).  The inverse transform reuses the forward twiddles through
// IFFT(X) = conj(FFT(conj(X))) / P.
#include <cuda_fp16.h>

#include "rk_internal.hpp"

namespace rk {

namespace {

template <class T>
__device__ __forceinline__ float ld_f32(const T* p);
template <>
__device__ __forceinline__ float ld_f32<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld_f32<__half>(const __half* p) { return __half2float(*p); }
template <>
__device__ __forceinline__ float ld_f32<double>(const double* p) { return float(__ldg(p)); }

template <class T>
__device__ __forceinline__ T st_cast(float v);
template <>
__device__ __forceinline__ float st_cast<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half st_cast<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ double st_cast<double>(float v) { return double(v); }

constexpr int kFilterThreads = 256;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// In-place radix-2 DIT over bit-reversed input, two independent signals.
__device__ void fft2_inplace(float2* za, float2* zb, int P, const float2* __restrict__ tw) {
  for (int len = 2; len <= P; len <<= 1) {
    const int half = len >> 1, stride = P / len;
    for (int bidx = threadIdx.x; bidx < P / 2; bidx += blockDim.x) {
      const int grp = bidx / half, k = bidx - grp * half;
      const int i = grp * len + k;
      const float2 w = __ldg(tw + k * stride);
      const float2 ua = za[i], va = cmul(za[i + half], w);
      za[i] = make_float2(ua.x + va.x, ua.y + va.y);
      za[i + half] = make_float2(ua.x - va.x, ua.y - va.y);
      const float2 ub = zb[i], vb = cmul(zb[i + half], w);
      zb[i] = make_float2(ub.x + vb.x, ub.y + vb.y);
      zb[i + half] = make_float2(ub.x - vb.x, ub.y - vb.y);
    }
    __syncthreads();
  }
}

template <class TIn, class TOut, bool PACKED>
__global__ void __launch_bounds__(kFilterThreads) filter_kernel(const TIn* __restrict__ in, int64_t batch, int na,
                                                                int nd, int P, int logP,
                                                                const float* __restrict__ resp,
                                                                const float2* __restrict__ tw, float scale,
                                                                TOut* __restrict__ out, float4* __restrict__ packed) {
  extern __shared__ float2 fsm[];
  float2* za = fsm;      // rows q=0 (re) and q=1 (im)
  float2* zb = fsm + P;  // rows q=2 (re) and q=3 (im)
  const int a = blockIdx.x;
  const int64_t g = blockIdx.y;
  const int shift = 32 - logP;
  // ---- load (zero pad) into bit-reversed positions
  const TIn* rows[4];
  bool valid[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t b = g * kPack + q;
    valid[q] = b < batch;
    rows[q] = in + (valid[q] ? (b * na + a) * int64_t(nd) : 0);
  }
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (k < nd) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (valid[q]) v[q] = ld_f32(rows[q] + k);
    }
    const int rk = int(__brev(unsigned(k)) >> shift);
    za[rk] = make_float2(v[0], v[1]);
    zb[rk] = make_float2(v[2], v[3]);
  }
  __syncthreads();
  fft2_inplace(za, zb, P, tw);
  // ---- multiply by the real, even response and conjugate (inverse via forward FFT)
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const float h = __ldg(resp + (q <= P / 2 ? q : P - q));
    const float2 x = za[q], y = zb[q];
    za[q] = make_float2(x.x * h, -(x.y * h));
    zb[q] = make_float2(y.x * h, -(y.y * h));
  }
  __syncthreads();
  // ---- bit-reversal permutation in place
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const int rk = int(__brev(unsigned(k)) >> shift);
    if (k < rk) {
      float2 t = za[k];
      za[k] = za[rk];
      za[rk] = t;
      t = zb[k];
      zb[k] = zb[rk];
      zb[rk] = t;
    }
  }
  __syncthreads();
  fft2_inplace(za, zb, P, tw);
  // ---- crop, x 1/P (irfft normalisation, fft.cpp:117-118), x pi/(2 na)
  const float inv = 1.0f / float(P);
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    const float2 x = za[k], y = zb[k];
    const float v[4] = {(x.x * inv) * scale, (-x.y * inv) * scale, (y.x * inv) * scale, (-y.y * inv) * scale};
    if (PACKED) {
      // fbp = backprojection(filter_sinogram(sino)) narrows the filtered rows
      // to the storage precision first (sino_filter.cpp:123, 126-128)
      packed[(g * na + a) * int64_t(nd) + k] =
          make_float4(float(st_cast<TOut>(v[0])), float(st_cast<TOut>(v[1])), float(st_cast<TOut>(v[2])),
                      float(st_cast<TOut>(v[3])));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (valid[q]) out[((g * kPack + q) * na + a) * int64_t(nd) + k] = st_cast<TOut>(v[q]);
    }
  }
}

template <class F>
void dispatch(int dtype, F&& f) {
  switch (dtype) {
    case RK_F16: f(__half{}); break;
    case RK_F32: f(float{}); break;
    case RK_F64: f(double{}); break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
}

}  // namespace

void launch_filter(const Filter& f, int dtype, const void* in, int64_t batch, int64_t n_angles, void* out,
                   float4* packed_out, cudaStream_t st) {
  const int P = int(f.padded);
  int logP = 0;
  while ((1 << logP) < P) ++logP;
  const size_t smem = size_t(2) * P * sizeof(float2);
  const float scale = float(M_PI / (2.0 * double(n_angles)));  // sino_filter.cpp:108
  dim3 grid(unsigned(n_angles), unsigned(groups_of(batch)));
  dispatch(dtype, [&](auto tag) {
    using T = decltype(tag);
    auto kern = packed_out ? filter_kernel<T, T, true> : filter_kernel<T, T, false>;
    if (smem > 48 * 1024) RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    KernelTimer timer(RK_KERNEL_FILTER, st);
    kern<<<grid, kFilterThreads, smem, st>>>(static_cast<const T*>(in), batch, int(n_angles), int(f.det_count), P,
                                             logP, f.d_response.as<float>(), f.d_twiddle.as<float2>(), scale,
                                             static_cast<T*>(out), packed_out);
  });
  RK_CUDA(cudaGetLastError());
}

}  // namespace rk
