// Micro-benchmark: cost of the fp16-storage (half8) tap arithmetic on sm_100a.
// Each iteration mimics one forward sample of the half8 path: four 128-bit
// shared loads (eight halves each), conversion to fp32 and the weighted sums
// of eight images.  Variants:
//   0  cvt.f32.f16 of all 32 halves + 32 scalar FFMA        (r2 kernel)
//   1  cvt of all 32 + 16 FFMA2 on the converted pairs
//   2  odd halves by integer ops with 2^112-scaled weights, even by cvt; 32 FFMA
//   3  as 2 with 16 FFMA2
//   4  no conversion (taps reinterpreted as floats): 32 FFMA      (pipe floor)
//   5  no conversion: 16 FFMA2
//   6  split-weight mixed FMA: w = w_hi + w_lo (halves), 2 x fma.rn.f32.f16 per tap and image
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pipe_rates pipe_rates.cu
// Run:   ./pipe_rates   (prints ns per warp-iteration per SMSP for each variant)
#include <cuda_fp16.h>
#include <cstdio>

__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  float2 aa = make_float2(a, a);
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&aa), rb = *reinterpret_cast<unsigned long long*>(&b),
                     rc = *reinterpret_cast<unsigned long long*>(&c), rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}
__device__ __forceinline__ float cvt_lo(unsigned w) {
  float f;
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; cvt.f32.f16 %0, l;}" : "=f"(f) : "r"(w));
  return f;
}
__device__ __forceinline__ float cvt_hi(unsigned w) {
  float f;
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; cvt.f32.f16 %0, h;}" : "=f"(f) : "r"(w));
  return f;
}
// upper half of w as (value * 2^-112) in fp32 bits: sign to bit 31, the 15
// magnitude bits to 27..13 (exact for normal and subnormal halves)
__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float hi_scaled(unsigned w) {
  return __int_as_float(int(unsigned(int(w) >> 3)) & int(0x8FFFE000u));
}

template <int V>
__global__ void __launch_bounds__(256, 4) kern(int iters, float* out) {
  __shared__ uint4 cells[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x)
    cells[i] = make_uint4(0x3c003c00u + i, 0x3c013c02u + i, 0x3c033c04u + i, 0x3c053c06u + i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.f;
  float2 a2[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) a2[q] = make_float2(0.f, 0.f);
  float px = 0.37f * lane;
  for (int it = 0; it < iters; ++it) {
    px = fmaf(0.731f, 1.f, px);
    const float fj = floorf(px);
    const float fx = px - fj;
    const int j = int(fj) & 255;
    const float gx = 1.f - fx;
    const float w1 = gx * 0.25f, w2 = fx * 0.25f, w3 = gx * 0.75f, w4 = fx * 0.75f;
    const uint4* q8 = cells + j;
    const uint4 u1 = q8[0], u2 = q8[1], u3 = q8[32], u4 = q8[33];
    const unsigned U1[4] = {u1.x, u1.y, u1.z, u1.w}, U2[4] = {u2.x, u2.y, u2.z, u2.w};
    const unsigned U3[4] = {u3.x, u3.y, u3.z, u3.w}, U4[4] = {u4.x, u4.y, u4.z, u4.w};
    if constexpr (V == 0 || V == 1) {
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
        const float2 f1 = make_float2(cvt_lo(U1[wd]), cvt_hi(U1[wd])), f2 = make_float2(cvt_lo(U2[wd]), cvt_hi(U2[wd]));
        const float2 f3 = make_float2(cvt_lo(U3[wd]), cvt_hi(U3[wd])), f4 = make_float2(cvt_lo(U4[wd]), cvt_hi(U4[wd]));
        if constexpr (V == 0) {
          acc[2 * wd] = fmaf(w1, f1.x, fmaf(w2, f2.x, fmaf(w3, f3.x, fmaf(w4, f4.x, acc[2 * wd]))));
          acc[2 * wd + 1] = fmaf(w1, f1.y, fmaf(w2, f2.y, fmaf(w3, f3.y, fmaf(w4, f4.y, acc[2 * wd + 1]))));
        } else {
          a2[wd] = ffma2(w1, f1, ffma2(w2, f2, ffma2(w3, f3, ffma2(w4, f4, a2[wd]))));
        }
      }
    } else if constexpr (V == 2 || V == 3) {
      const float S = 5.192296858534828e33f;  // 2^112
      const float v1 = w1 * S, v2 = w2 * S, v3 = w3 * S, v4 = w4 * S;
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
        if constexpr (V == 2) {
          acc[2 * wd] = fmaf(w1, cvt_lo(U1[wd]), fmaf(w2, cvt_lo(U2[wd]), fmaf(w3, cvt_lo(U3[wd]), fmaf(w4, cvt_lo(U4[wd]), acc[2 * wd]))));
          acc[2 * wd + 1] = fmaf(v1, hi_scaled(U1[wd]), fmaf(v2, hi_scaled(U2[wd]), fmaf(v3, hi_scaled(U3[wd]), fmaf(v4, hi_scaled(U4[wd]), acc[2 * wd + 1]))));
        } else {
          // pairs (lo exact, hi scaled) need a per-lane weight pair: FFMA2 with a float2 weight
          float2 r = a2[wd];
          const float2 W1 = make_float2(w1, v1), W2 = make_float2(w2, v2), W3 = make_float2(w3, v3), W4 = make_float2(w4, v4);
          auto f2v = [](float2 a, float2 b, float2 c) {
            unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b),
                               rc = *reinterpret_cast<unsigned long long*>(&c), rd;
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
            return *reinterpret_cast<float2*>(&rd);
          };
          r = f2v(W4, make_float2(cvt_lo(U4[wd]), hi_scaled(U4[wd])), r);
          r = f2v(W3, make_float2(cvt_lo(U3[wd]), hi_scaled(U3[wd])), r);
          r = f2v(W2, make_float2(cvt_lo(U2[wd]), hi_scaled(U2[wd])), r);
          r = f2v(W1, make_float2(cvt_lo(U1[wd]), hi_scaled(U1[wd])), r);
          a2[wd] = r;
        }
      }
    } else if constexpr (V == 6) {
      const float W[4] = {w1, w2, w3, w4};
      unsigned short wh[4], wl[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const __half h = __float2half_rn(W[t]);
        wh[t] = __half_as_ushort(h);
        wl[t] = __half_as_ushort(__float2half_rn(W[t] - __half2float(h)));
      }
      const unsigned* UU[4] = {U1, U2, U3, U4};
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float a = acc[2 * wd + hh];
#pragma unroll
          for (int t = 3; t >= 0; --t) {
            const unsigned short v = (unsigned short)(hh ? (UU[t][wd] >> 16) : (UU[t][wd] & 0xffffu));
            a = fhfma(v, wl[t], a);
            a = fhfma(v, wh[t], a);
          }
          acc[2 * wd + hh] = a;
        }
      }
    } else {
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
        const float2 f1 = make_float2(__uint_as_float(U1[wd]), __uint_as_float(U1[wd] ^ 0x1000u));
        const float2 f2 = make_float2(__uint_as_float(U2[wd]), __uint_as_float(U2[wd] ^ 0x1000u));
        const float2 f3 = make_float2(__uint_as_float(U3[wd]), __uint_as_float(U3[wd] ^ 0x1000u));
        const float2 f4 = make_float2(__uint_as_float(U4[wd]), __uint_as_float(U4[wd] ^ 0x1000u));
        if constexpr (V == 4) {
          acc[2 * wd] = fmaf(w1, f1.x, fmaf(w2, f2.x, fmaf(w3, f3.x, fmaf(w4, f4.x, acc[2 * wd]))));
          acc[2 * wd + 1] = fmaf(w1, f1.y, fmaf(w2, f2.y, fmaf(w3, f3.y, fmaf(w4, f4.y, acc[2 * wd + 1]))));
        } else {
          a2[wd] = ffma2(w1, f1, ffma2(w2, f2, ffma2(w3, f3, ffma2(w4, f4, a2[wd]))));
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += acc[q];
#pragma unroll
  for (int q = 0; q < 4; ++q) s += a2[q].x + a2[q].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run(const char* name, float* out) {
  const int iters = 4096, blocks = 148 * 4 * 8;
  kern<V><<<blocks, 256>>>(iters, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<V><<<blocks, 256>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  // warp-iterations per SMSP
  const double wi = double(blocks) * 8 * iters / (148.0 * 4);
  printf("V%d %-40s %.3f ms  %.2f ns / warp-iter / SMSP  (%.1f cycles at 1.965 GHz)\n", V, name, ms, ms * 1e6 / wi,
         ms * 1e6 / wi * 1.965);
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 4 * 8 * 256 * sizeof(float));
  run<0>("cvt x32 + FFMA x32 (r2 kernel)", out);
  run<1>("cvt x32 + FFMA2 x16", out);
  run<2>("cvt x16 + int-hi x16 + FFMA x32", out);
  run<3>("cvt x16 + int-hi x16 + FFMA2 x16", out);
  run<4>("no cvt, FFMA x32", out);
  run<5>("no cvt, FFMA2 x16", out);
  run<6>("split-weight FHFMA x64", out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
