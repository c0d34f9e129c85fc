// Ramp-filter kernel (sm_100a): per detector row, zero-pad to P, FFT,
// multiply by the real frequency response, inverse FFT, crop and scale by
// pi / (2 n_angles) — sino_filter.cpp:98-124 (filtration always fp32,
// :106-123).
//
// One CTA filters the four rows (b = 4g..4g+3, angle a) that share one
// packed float4 sinogram cell, as two complex shared-memory FFTs: the
// response is real and even, so for z = x + i y, IFFT(FFT(z) H) = x*h + i (y*h)
// filters two real rows at once.  The forward transform is
// decimation-in-frequency (natural in, bit-reversed out), the response is
// applied in bit-reversed order, and the inverse is decimation-in-time with
// conjugate twiddles (bit-reversed in, natural out): no permutation pass.
#include <cuda_fp16.h>

#include <type_traits>

#include "fft_smem.cuh"
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

// PACKED 0: user layout; 1: packed float4 cells (four images); 2: half of a
// packed half8 cell (fp16 storage, use_h8): this CTA's four rows are images
// 4g .. 4g+3, i.e. the low or high 8 bytes of group g / 2's cells.
template <class TIn, class TOut, int PACKED>
__global__ void __launch_bounds__(kFilterThreads) filter_kernel(const TIn* __restrict__ in, int64_t batch, int na,
                                                                int nd, int P, int logP,
                                                                const float* __restrict__ resp,
                                                                const float2* __restrict__ tw, float scale,
                                                                TOut* __restrict__ out, float4* __restrict__ packed) {
  extern __shared__ float2 fsm[];
  float2* za = fsm;      // rows q=0 (re) and q=1 (im), swizzled slots (swz)
  float2* zb = fsm + P;  // rows q=2 (re) and q=3 (im)
  const int a = blockIdx.x;
  const int64_t g = blockIdx.y;
  const int shift = 32 - logP;
  // ---- load (zero pad), natural order
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
    za[fft_swz(k)] = make_float2(v[0], v[1]);
    zb[fft_swz(k)] = make_float2(v[2], v[3]);
  }
  __syncthreads();
  fft_dif_seq(fsm, 2, P, logP, tw);
  // ---- multiply by the real, even response; slot q holds frequency brev(q)
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int f = int(__brev(unsigned(q)) >> shift);
    const float h = __ldg(resp + (f <= P / 2 ? f : P - f));
    const int sq = fft_swz(q);
    const float2 x = za[sq], y = zb[sq];
    za[sq] = make_float2(x.x * h, x.y * h);
    zb[sq] = make_float2(y.x * h, y.y * h);
  }
  __syncthreads();
  ifft_dit_seq(fsm, 2, P, logP, tw);
  // ---- crop, x 1/P (irfft normalisation, fft.cpp:117-118), x pi/(2 na)
  const float inv = 1.0f / float(P);
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    const float2 x = za[fft_swz(k)], y = zb[fft_swz(k)];
    const float v[4] = {(x.x * inv) * scale, (x.y * inv) * scale, (y.x * inv) * scale, (y.y * inv) * scale};
    if (PACKED == 2) {
      // four halves: exactly the values the float4 path narrows through fp16
      const __half h0 = __float2half_rn(v[0]), h1 = __float2half_rn(v[1]), h2 = __float2half_rn(v[2]),
                   h3 = __float2half_rn(v[3]);
      const uint2 bits = make_uint2(unsigned(__half_as_ushort(h0)) | (unsigned(__half_as_ushort(h1)) << 16),
                                    unsigned(__half_as_ushort(h2)) | (unsigned(__half_as_ushort(h3)) << 16));
      reinterpret_cast<uint2*>(packed)[(((g >> 1) * na + a) * int64_t(nd) + k) * 2 + (g & 1)] = bits;
    } else if (PACKED == 1) {
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
    auto kern = packed_out ? filter_kernel<T, T, 1> : filter_kernel<T, T, 0>;
    if constexpr (std::is_same<T, __half>::value)
      if (packed_out && use_h8(dtype, batch)) kern = filter_kernel<T, T, 2>;
    allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    KernelTimer timer(RK_KERNEL_FILTER, st);
    kern<<<grid, kFilterThreads, smem, st>>>(static_cast<const T*>(in), batch, int(n_angles), int(f.det_count), P,
                                             logP, f.d_response.as<float>(), f.d_twiddle.as<float2>(), scale,
                                             static_cast<T*>(out), packed_out);
  });
  RK_CUDA(cudaGetLastError());
}

}  // namespace rk
