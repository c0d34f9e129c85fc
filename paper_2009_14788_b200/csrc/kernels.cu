// CUDA kernels (sm_100a) of the B200 Radon projector: layout packing, the
// ray-driven forward projector and the pixel-driven backprojector.
//
// Reference semantics: projector.cpp:47-203 (bilinear, integrate_ray,
// forward_{parallel,fanbeam}_t, backprojection_{parallel,fanbeam}_t).
// Arithmetic is fp32 (north star), accumulation order per output element is
// fixed and independent of batch size and grid shape, so batched results
// equal per-element results bit for bit (acceptance.cpp:340-389).
#include <cuda_fp16.h>

#include "rk_internal.hpp"

namespace rk {

namespace {

template <class T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f32<double>(double v) { return float(v); }

template <class T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ double from_f32<double>(float v) { return double(v); }

template <class F>
void dispatch_dtype(int dtype, F&& f) {
  switch (dtype) {
    case RK_F16: f(__half{}); break;
    case RK_F32: f(float{}); break;
    case RK_F64: f(double{}); break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
}

inline unsigned blocks_for(int64_t n, int threads) { return unsigned((n + threads - 1) / threads); }

// ------------------------------------------------------------------ packing
// image [B][s][s] (T) -> [G][s+2][s+2] float4 with a zero border.
template <class T>
__global__ void pack_images_kernel(const T* __restrict__ src, int64_t batch, int s, float4* __restrict__ dst) {
  const int P = s + 2;
  const int64_t plane = int64_t(P) * P;
  const int64_t g = blockIdx.y;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < plane;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int pi = int(idx / P), pj = int(idx % P);
    float v[kPack] = {0.f, 0.f, 0.f, 0.f};
    if (pi >= 1 && pi <= s && pj >= 1 && pj <= s) {
      int64_t off = int64_t(pi - 1) * s + (pj - 1);
#pragma unroll
      for (int q = 0; q < kPack; ++q) {
        int64_t b = g * kPack + q;
        if (b < batch) v[q] = to_f32(src[b * int64_t(s) * s + off]);
      }
    }
    dst[g * plane + idx] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// sino [B][na*nd] (T) -> [G][na*nd] float4
template <class T>
__global__ void pack_sino_kernel(const T* __restrict__ src, int64_t batch, int64_t plane, float4* __restrict__ dst) {
  const int64_t g = blockIdx.y;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < plane;
       idx += int64_t(gridDim.x) * blockDim.x) {
    float v[kPack] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < kPack; ++q) {
      int64_t b = g * kPack + q;
      if (b < batch) v[q] = to_f32(src[b * plane + idx]);
    }
    dst[g * plane + idx] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// ------------------------------------------------------------------ forward
// One thread per (ray, image group): ray march with software bilinear
// interpolation (projector.cpp:47-83).  The clipped entry point, step and
// sample count come from the fp64 ray table; sample m sits at
// (px0, py0) + (m + 0.5) * (hx, hy) in padded pixel coordinates, exactly
// the reference's t_m = t0 + (m + 0.5) h.  Taps of four images are read as
// one float4 each; the 4-tap weights are shared by the four images.
template <class TOut>
__global__ void __launch_bounds__(256) forward_kernel(const float4* __restrict__ img, int s,
                                                      const float4* __restrict__ ray_geom,
                                                      const float2* __restrict__ ray_len, int64_t n_rays,
                                                      int64_t batch, TOut* __restrict__ sino) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const int P = s + 2;
  const int64_t g = blockIdx.y;
  const float4* im = img + g * int64_t(P) * P;
  const float4 R = __ldg(ray_geom + r);
  const float2 L = __ldg(ray_len + r);
  const int n = __float_as_int(L.y);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  for (int m = 0; m < n; ++m) {
    const float t = float(m) + 0.5f;
    const float px = fmaf(t, R.z, R.x);
    const float py = fmaf(t, R.w, R.y);
    const float fj = floorf(px), fi = floorf(py);
    const float fx = px - fj, fy = py - fi;
    const int j0 = min(max(int(fj), 0), P - 2);
    const int i0 = min(max(int(fi), 0), P - 2);
    const float4* p = im + i0 * P + j0;
    const float4 v00 = __ldg(p), v01 = __ldg(p + 1), v10 = __ldg(p + P), v11 = __ldg(p + P + 1);
    const float gx = 1.f - fx, gy = 1.f - fy;
    const float w00 = gx * gy, w01 = fx * gy, w10 = gx * fy, w11 = fx * fy;
    a0 = fmaf(w00, v00.x, fmaf(w01, v01.x, fmaf(w10, v10.x, fmaf(w11, v11.x, a0))));
    a1 = fmaf(w00, v00.y, fmaf(w01, v01.y, fmaf(w10, v10.y, fmaf(w11, v11.y, a1))));
    a2 = fmaf(w00, v00.z, fmaf(w01, v01.z, fmaf(w10, v10.z, fmaf(w11, v11.z, a2))));
    a3 = fmaf(w00, v00.w, fmaf(w01, v01.w, fmaf(w10, v10.w, fmaf(w11, v11.w, a3))));
  }
  const float h = L.x;
  const float acc[kPack] = {a0 * h, a1 * h, a2 * h, a3 * h};
#pragma unroll
  for (int q = 0; q < kPack; ++q) {
    const int64_t b = g * kPack + q;
    if (b < batch) sino[b * n_rays + r] = from_f32<TOut>(acc[q]);
  }
}

// ------------------------------------------------------------------ backprojection
// One CTA per (32x32 pixel tile, image group); 256 threads, each owning 4
// pixels of one column (rows ty, ty+8, ty+16, ty+24) for 4 images.
// Angles are processed in chunks: for every angle of the chunk the
// detector window that the tile's footprint can touch is staged into shared
// memory (zero outside [0, det_count), which is the reference's skipped-tap
// rule, projector.cpp:159-162), then every pixel accumulates its two-tap
// lerp for each angle in ascending angle order (projector.cpp:152-163).
struct AngleConst {
  float a, b, c, d;  // parallel: base, cx, cy, -; fan: qx00, den00, offw, -
  float e, f, g, h;  // fan: cos, sin, -, -
};

constexpr int kTile = 32;
constexpr int kRowsPerThread = 4;
constexpr int kBpThreads = kTile * (kTile / kRowsPerThread);  // 256

template <bool FAN, class TOut>
__global__ void __launch_bounds__(kBpThreads) backproject_kernel(
    const float4* __restrict__ sino, int s, int na, int nd, double spacing, double source_distance,
    double det_distance, const double2* __restrict__ trig, int window, int chunk, int64_t batch,
    TOut* __restrict__ out) {
  extern __shared__ float4 smem[];
  float4* win = smem;                                                      // chunk * window cells
  AngleConst* cst = reinterpret_cast<AngleConst*>(smem + size_t(chunk) * window);  // chunk records
  int* ws_s = reinterpret_cast<int*>(cst + chunk);                          // chunk window starts

  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kTile + tx;
  const int j0 = blockIdx.x * kTile, i0 = blockIdx.y * kTile;
  const int64_t g = blockIdx.z;
  const double half = 0.5 * double(s);
  const double off = 0.5 * double(nd) - 0.5;
  const double span = source_distance + det_distance;
  // centre of the tile's first pixel (projector.cpp:150,154)
  const double x0 = double(j0) - half + 0.5;
  const double y0 = half - double(i0) - 0.5;
  const float4* sg = sino + g * int64_t(na) * nd;

  float4 acc[kRowsPerThread];
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);

  for (int a0 = 0; a0 < na; a0 += chunk) {
    const int nac = min(chunk, na - a0);
    // ---- per-angle constants, fp64 (one thread per angle)
    if (tid < nac) {
      const double2 cs = trig[a0 + tid];
      const double c = cs.x, sn = cs.y;
      const double x1 = x0 + double(kTile - 1), y1 = y0 - double(kTile - 1);
      double lo;
      AngleConst k;
      if (!FAN) {
        const double k00 = (x0 * c + y0 * sn) / spacing + off;
        const double k10 = (x1 * c + y0 * sn) / spacing + off;
        const double k01 = (x0 * c + y1 * sn) / spacing + off;
        const double k11 = (x1 * c + y1 * sn) / spacing + off;
        lo = fmin(fmin(k00, k10), fmin(k01, k11));
        const int ws = int(floor(lo)) - 1;
        k.a = float(k00 - double(ws));
        k.b = float(c / spacing);
        k.c = float(-sn / spacing);
        k.d = 0.f;
        k.e = k.f = k.g = k.h = 0.f;
        ws_s[tid] = ws;
      } else {
        auto kfan = [&](double x, double y) {
          const double qx = x * c + y * sn, qy = -x * sn + y * c;
          return (qx * span / (qy + source_distance)) / spacing + off;
        };
        lo = fmin(fmin(kfan(x0, y0), kfan(x1, y0)), fmin(kfan(x0, y1), kfan(x1, y1)));
        const int ws = int(floor(lo)) - 1;
        const double qx00 = x0 * c + y0 * sn;
        const double den00 = -x0 * sn + y0 * c + source_distance;
        k.a = float(qx00);
        k.b = float(den00);
        k.c = float(off - double(ws));
        k.d = 0.f;
        k.e = float(c);
        k.f = float(sn);
        k.g = k.h = 0.f;
        ws_s[tid] = ws;
      }
      cst[tid] = k;
    }
    __syncthreads();
    // ---- stage the detector windows (coalesced 16-byte cells)
    for (int e = tid; e < nac * window; e += kBpThreads) {
      const int q = e / window, cidx = e - q * window;
      const int k = ws_s[q] + cidx;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k >= 0 && k < nd) v = __ldg(sg + int64_t(a0 + q) * nd + k);
      win[e] = v;
    }
    __syncthreads();
    // ---- accumulate
    const float fspan = float(span / spacing);
    for (int q = 0; q < nac; ++q) {
      const AngleConst k = cst[q];
      const float4* w = win + q * window;
#pragma unroll
      for (int r = 0; r < kRowsPerThread; ++r) {
        const float lx = float(tx), ly = float(ty + r * (kTile / kRowsPerThread));
        float kf;
        if (!FAN) {
          kf = fmaf(lx, k.b, fmaf(ly, k.c, k.a));
        } else {
          const float qx = fmaf(lx, k.e, fmaf(-ly, k.f, k.a));
          const float den = fmaf(-lx, k.f, fmaf(-ly, k.e, k.b));
          kf = fmaf(qx * fspan, __frcp_rn(den), k.c);
        }
        const float fk = floorf(kf);
        const float wt = kf - fk;
        const int c0 = min(max(int(fk), 0), window - 2);
        const float4 s0 = w[c0], s1 = w[c0 + 1];
        const float wl = 1.f - wt;
        acc[r].x = fmaf(wt, s1.x, fmaf(wl, s0.x, acc[r].x));
        acc[r].y = fmaf(wt, s1.y, fmaf(wl, s0.y, acc[r].y));
        acc[r].z = fmaf(wt, s1.z, fmaf(wl, s0.z, acc[r].z));
        acc[r].w = fmaf(wt, s1.w, fmaf(wl, s0.w, acc[r].w));
      }
    }
    __syncthreads();
  }
  // ---- store
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) {
    const int i = i0 + ty + r * (kTile / kRowsPerThread), j = j0 + tx;
    if (i >= s || j >= s) continue;
    const float v[kPack] = {acc[r].x, acc[r].y, acc[r].z, acc[r].w};
#pragma unroll
    for (int q = 0; q < kPack; ++q) {
      const int64_t b = g * kPack + q;
      if (b < batch) out[(b * s + i) * int64_t(s) + j] = from_f32<TOut>(v[q]);
    }
  }
}

}  // namespace

void launch_pack_images(int dtype, const void* src, int64_t batch, int64_t s, float4* dst, cudaStream_t st) {
  const int64_t plane = (s + 2) * (s + 2);
  dim3 grid(std::min<unsigned>(blocks_for(plane, 256), 4096u), unsigned(groups_of(batch)));
  dispatch_dtype(dtype, [&](auto tag) {
    using T = decltype(tag);
    KernelTimer timer(RK_KERNEL_PACK, st);
    pack_images_kernel<T><<<grid, 256, 0, st>>>(static_cast<const T*>(src), batch, int(s), dst);
  });
  RK_CUDA(cudaGetLastError());
}

void launch_pack_sino(int dtype, const void* src, int64_t batch, int64_t na, int64_t nd, float4* dst,
                      cudaStream_t st) {
  const int64_t plane = na * nd;
  dim3 grid(std::min<unsigned>(blocks_for(plane, 256), 4096u), unsigned(groups_of(batch)));
  dispatch_dtype(dtype, [&](auto tag) {
    using T = decltype(tag);
    KernelTimer timer(RK_KERNEL_PACK, st);
    pack_sino_kernel<T><<<grid, 256, 0, st>>>(static_cast<const T*>(src), batch, plane, dst);
  });
  RK_CUDA(cudaGetLastError());
}

void launch_forward(const Plan& p, const float4* packed_image, int64_t batch, int dtype, void* sino,
                    cudaStream_t st) {
  const int64_t n_rays = p.na * p.nd;
  dim3 grid(blocks_for(n_rays, 256), unsigned(groups_of(batch)));
  dispatch_dtype(dtype, [&](auto tag) {
    using T = decltype(tag);
    KernelTimer timer(RK_KERNEL_FORWARD, st);
    forward_kernel<T><<<grid, 256, 0, st>>>(packed_image, int(p.s), p.ray_geom.as<float4>(),
                                            p.ray_len.as<float2>(), n_rays, batch, static_cast<T*>(sino));
  });
  RK_CUDA(cudaGetLastError());
}

void launch_backproject(const Plan& p, const float4* packed_sino, int64_t batch, int dtype, void* image,
                        cudaStream_t st) {
  const int tiles = int((p.s + kTile - 1) / kTile);
  dim3 grid(tiles, tiles, unsigned(groups_of(batch)));
  dim3 block(kTile, kTile / kRowsPerThread);
  const size_t smem = size_t(p.bp_angle_chunk) * p.bp_window * sizeof(float4) +
                      size_t(p.bp_angle_chunk) * (sizeof(AngleConst) + sizeof(int));
  const bool fan = p.g.kind == RK_FANBEAM;
  dispatch_dtype(dtype, [&](auto tag) {
    using T = decltype(tag);
    auto kern = fan ? backproject_kernel<true, T> : backproject_kernel<false, T>;
    if (smem > 48 * 1024) RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    KernelTimer timer(RK_KERNEL_BACKPROJECT, st);
    kern<<<grid, block, smem, st>>>(packed_sino, int(p.s), int(p.na), int(p.nd), p.g.det_spacing,
                                    p.g.source_distance, p.g.det_distance, p.trig.as<double2>(), p.bp_window,
                                    p.bp_angle_chunk, batch, static_cast<T*>(image));
  });
  RK_CUDA(cudaGetLastError());
}

}  // namespace rk
