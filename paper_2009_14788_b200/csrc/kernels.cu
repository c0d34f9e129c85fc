// CUDA kernels (sm_100a) of the B200 Radon projector: layout packing, the
// ray-driven forward projector and the pixel-driven backprojector.
//
// Reference semantics: projector.cpp:47-203 (bilinear, integrate_ray,
// forward_{parallel,fanbeam}_t, backprojection_{parallel,fanbeam}_t).
// Arithmetic is fp32 (north star), accumulation order per output element is
// fixed and independent of batch size and grid shape, so batched results
// equal per-element results bit for bit (acceptance.cpp:340-389).
#include <cuda_fp16.h>

#include <cstdlib>
#include <type_traits>

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

// ---- fp16 storage: eight images per 16-byte texel (kPackH8)
__device__ __forceinline__ unsigned h2_bits(__half lo, __half hi) {
  return unsigned(__half_as_ushort(lo)) | (unsigned(__half_as_ushort(hi)) << 16);
}
// word w of a half8 texel -> images 2w, 2w+1 as floats (exact)
__device__ __forceinline__ float2 h8_pair(unsigned w) {
  return __half22float2(*reinterpret_cast<const __half2*>(&w));
}
__device__ __forceinline__ unsigned h8_word(const uint4& u, int i) {
  return i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w;
}

// image [B][s][s] half -> [G8][s+2][s+2] half8 texels with a zero border
__global__ void pack_images_h8_kernel(const __half* __restrict__ src, int64_t batch, int s, uint4* __restrict__ dst) {
  const int P = s + 2;
  const int64_t plane = int64_t(P) * P;
  const int64_t g = blockIdx.y;
  const __half z = __float2half_rn(0.f);
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < plane;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int pi = int(idx / P), pj = int(idx % P);
    __half v[kPackH8];
#pragma unroll
    for (int q = 0; q < kPackH8; ++q) v[q] = z;
    if (pi >= 1 && pi <= s && pj >= 1 && pj <= s) {
      const int64_t off = int64_t(pi - 1) * s + (pj - 1);
#pragma unroll
      for (int q = 0; q < kPackH8; ++q) {
        const int64_t b = g * kPackH8 + q;
        if (b < batch) v[q] = src[b * int64_t(s) * s + off];
      }
    }
    dst[g * plane + idx] = make_uint4(h2_bits(v[0], v[1]), h2_bits(v[2], v[3]), h2_bits(v[4], v[5]), h2_bits(v[6], v[7]));
  }
}

// sino [B][na*nd] half -> [G8][na*nd] half8 texels
__global__ void pack_sino_h8_kernel(const __half* __restrict__ src, int64_t batch, int64_t plane, uint4* __restrict__ dst) {
  const int64_t g = blockIdx.y;
  const __half z = __float2half_rn(0.f);
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < plane;
       idx += int64_t(gridDim.x) * blockDim.x) {
    __half v[kPackH8];
#pragma unroll
    for (int q = 0; q < kPackH8; ++q) {
      const int64_t b = g * kPackH8 + q;
      v[q] = b < batch ? src[b * plane + idx] : z;
    }
    dst[g * plane + idx] = make_uint4(h2_bits(v[0], v[1]), h2_bits(v[2], v[3]), h2_bits(v[4], v[5]), h2_bits(v[6], v[7]));
  }
}

// ------------------------------------------------------------------ forward
// packed image -> transposed packed image, 32x32-texel tiles through shared
// memory (coalesced both ways).
__global__ void transpose_images_kernel(const float4* __restrict__ src, int P, float4* __restrict__ dst) {
  __shared__ float4 tile[32][33];
  const int64_t plane = int64_t(P) * P;
  const float4* s = src + blockIdx.z * plane;
  float4* d = dst + blockIdx.z * plane;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = by + r, j = bx + threadIdx.x;
    if (i < P && j < P) tile[r][threadIdx.x] = s[int64_t(i) * P + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = bx + r, j = by + threadIdx.x;  // dst row = src column
    if (i < P && j < P) d[int64_t(i) * P + j] = tile[threadIdx.x][r];
  }
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// one row of the staged box: `bytes` (multiple of 16) from global to shared
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// cp.async (LDGSTS) helpers
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Blackwell packed FP32 FMA (FFMA2): two independent fmaf's in one instruction,
// each rounded exactly as fmaf — so pairs of images share one issue slot and
// the results are bit-identical to the scalar chain.  The broadcast weight
// becomes FFMA2's scalar operand.
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  float2 aa = make_float2(a, a);
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&aa), rb = *reinterpret_cast<unsigned long long*>(&b),
                     rc = *reinterpret_cast<unsigned long long*>(&c), rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}
__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }

constexpr int kFwdThreads = 256;  // A = 8 angles (warps) x W = 32 detectors (lanes)

// Ray-driven forward projection (projector.cpp:66-139), one CTA per block of
// 8 angles x 32 detector cells and per packed group of four images.  All rays
// of the CTA march together chunk by chunk along t; before each chunk the
// box of padded-image texels its samples can touch (fwd_plan.cpp) is copied
// to shared memory by TMA bulk copies (one per box row, completing on an
// mbarrier), then each lane runs its own samples of the
// chunk: sample m at (px0, py0) + (m + 0.5) (hx, hy) — the reference's
// t_m = t0 + (m + 0.5) h — bilinear taps as four 128-bit shared loads (one
// tap of four images each), weights shared by the four images.  Samples are
// visited in ascending m, so each output is a fixed-order fp32 sum.
// Chunk membership: m < ceil((T_{c+1} - t0) / h - 0.5), evaluated in fp32;
// the boxes carry one unit of slack in t and a texel around the taps, so no
// sample leaves its box (proved per plan by RK_VERIFY_PLAN, fwd_plan.cpp) and
// the tap indices need no clamping.  Chunks whose lane lines run mostly along
// image columns stage the transposed packed image with x and y swapped
// (bilinear is symmetric).
//
// LANE (batch 1): only lane 0 of the packed group carries an image, so the box
// is staged as scalars (lane 0 of each texel, 4-byte cp.async into two
// alternating boxes) and every tap is a 32-bit shared load: a quarter of the
// shared-memory traffic and FMAs of the packed loop, with the same operations
// on lane 0 in the same order, so its results equal the packed kernel's bit
// for bit.
// H8 (fp16 storage, batch > 1): half8 texels, eight images per lane, each tap
// load converted to fp32 pairs; per image the same operations and order.
// NW: the schedule holds narrow-warp CTAs (ForwardSchedule::any_narrow); the
// lane check is compiled in only then (it costs the half8 loop ~3 %).
// CM: grid (groups, CTAs) instead of (CTAs, groups) — CTA-major launch order for few groups
// (launch_forward); a template flag because any change to the half8 loop's code costs it ~1 %.
template <class TOut, bool LANE, bool H8, bool NW, bool CM>
__global__ void __launch_bounds__(kFwdThreads, 4) forward_kernel(
    const float4* __restrict__ img, const float4* __restrict__ img_t, int s, const float4* __restrict__ ray_geom,
    const float4* __restrict__ ray_aux, const int4* __restrict__ boxes, const int4* __restrict__ cta_cfg,
    const int2* __restrict__ warps, int na, int nd, int64_t batch, TOut* __restrict__ sino, FwdEpilogue epi,
    int lane_box) {
  extern __shared__ float4 box_s[];
  __shared__ unsigned long long box_bar;  // TMA completion of the current chunk's box
  // grid (CTAs, groups), or (groups, CTAs) for few groups: the launch order then follows the
  // planner's longest-first CTA order across all groups, not group after group (launch_forward)
  const int cta = CM ? blockIdx.y : blockIdx.x;
  const int64_t g = CM ? blockIdx.x : blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 cfg = __ldg(cta_cfg + cta);  // {first box, boxes, flags}
  // lane -> ray, chosen by the planner against bank conflicts (angles are
  // sorted by direction).  A quarter warp (8 lanes, one shared-memory
  // wavefront per 128-bit load) covers 2^lq neighbouring angles x 8 >> lq
  // neighbouring cells: lq = 0 detector-major (warp = angle slot, lane = cell;
  // any CTA shape), lq = 3 angle-major (one cell's 8 angles); 1, 2 mixed.
  const int lq = (cfg.z >> 3) & 3;
  int slot = warp, k;
  if (lq == 0) {
    // narrow-warp CTAs (coarse detectors, fwd_plan.cpp, cfg.z bits 5-7): lanes >= 32 >> n idle
    k = __ldg(warps + cta * (kFwdThreads / 32) + warp).y + lane;
    if (NW && (lane >> (5 - ((cfg.z >> 5) & 7))) != 0) k = nd;
  } else {
    const int t = threadIdx.x;
    const int cq = t & ((8 >> lq) - 1), aq = (t >> (3 - lq)) & ((1 << lq) - 1);
    const int cg = (t >> 3) & ((4 << lq) - 1), ag = t >> (lq + 5);
    slot = (ag << lq) + aq;
    k = __ldg(warps + cta * (kFwdThreads / 32)).y + cg * (8 >> lq) + cq;
  }
  const int a = __ldg(warps + cta * (kFwdThreads / 32) + slot).x;
  const bool valid = a >= 0 && k < nd;
  const int64_t r = int64_t(a) * nd + k;
  // Per-chunk layout chosen by the planner against bank conflicts (box record
  // z = pitch | orientation << 16 | per-lane tap order << 17): chunks of
  // transposed orientation stage the transposed packed image with x and y
  // swapped, and lanes flagged by the tap order issue the bottom row first or
  // the right column first.  Loads L1..L4 = (rowA,colA) (rowA,colB) (rowB,colA)
  // (rowB,colB); the weights follow the same order, so no value is moved
  // between registers.
  float4 G = make_float4(0.f, 0.f, 0.f, 0.f), X = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) {
    G = __ldg(ray_geom + r);
    X = __ldg(ray_aux + r);
  }
  const int n = __float_as_int(X.y);
  const float t0 = X.z, inv_h = X.w;
  const int P = s + 2;
  const int64_t goff = g * int64_t(P) * P;
  const int4* bxs = boxes + cfg.x;

  if (threadIdx.x == 0) {
    mbar_init(&box_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  float2 a01 = make_float2(0.f, 0.f), a23 = a01;  // images 0-1, 2-3 (LANE: a01.x)
  float2 a8[H8 ? kPackH8 / 2 : 1];                 // H8: image pairs
#pragma unroll
  for (int q = 0; q < (H8 ? kPackH8 / 2 : 1); ++q) a8[q] = make_float2(0.f, 0.f);
  int m = 0;
  // LANE: lane 0 of the box's texels by 4-byte cp.async (warp w takes rows w,
  // w + 8, ...) into two alternating scalar boxes, the next chunk's copies in
  // flight while the current chunk is marched
  const int box_cells = lane_box;  // LANE: the second box's offset (max box cells of the plan)
  auto stage_lane = [&](int cc_, float* dst) {
    const int4 b = __ldg(bxs + cc_);
    const int br0 = b.x & 0xffff, bc0 = b.x >> 16, brows = b.y & 0xffff, bcols = b.y >> 16, bpitch = b.z & 0xffff;
    const float4* bsrc = (((b.z >> 16) & 1) ? img_t : img) + goff;
    for (int rr = warp; rr < brows; rr += kFwdThreads / 32) {
      const float4* row = bsrc + int64_t(br0 + rr) * P + bc0;
      for (int cc = lane; cc < bcols; cc += 32) cp_async4(dst + rr * bpitch + cc, row + cc);
    }
    cp_async_commit();
  };
  if constexpr (LANE) {
    if (cfg.y > 0) stage_lane(0, reinterpret_cast<float*>(box_s));
  }
  for (int c = 0; c < cfg.y; ++c) {
    const int4 bx = __ldg(bxs + c);  // CTA-uniform
    const int r0 = bx.x & 0xffff, c0 = bx.x >> 16, rows = bx.y & 0xffff, cols = bx.y >> 16, pitch = bx.z & 0xffff;
    const bool tr = ((bx.z >> 16) & 1) != 0;
    // per-lane tap order (fwd_plan.cpp order_row / order_col): lane l of each quarter
    // warp loads the bottom row first / the right column first
    const int order = (bx.z >> 17) & 0x3fff, l8 = threadIdx.x & 7;
    const bool rs = l8 != 0 && ((order >> (l8 - 1)) & 1), cs = l8 != 0 && ((order >> (l8 + 6)) & 1);
    const int dX = cs ? -1 : 1;
    const float px0 = tr ? G.y : G.x, py0 = tr ? G.x : G.y;
    const float hx = tr ? G.w : G.z, hy = tr ? G.z : G.w;
    const float4* src = (tr ? img_t : img) + goff;
    const float tend = __int_as_float(bx.w);
    // samples of this chunk: t_m < t_end  <=>  m < ceil((t_end - t0) / h - 0.5)
    const int m_end =
        isinf(tend) ? n : min(max(int(ceilf(fmaf(tend - t0, inv_h, -0.5f))), 0), n);
    __syncthreads();  // previous chunk's samples are done with the box
    const float* box1 = reinterpret_cast<const float*>(box_s) + (c & 1) * box_cells;
    if constexpr (LANE) {
      if (c + 1 < cfg.y) {
        stage_lane(c + 1, reinterpret_cast<float*>(box_s) + ((c + 1) & 1) * box_cells);
        cp_async_wait_1();
      } else {
        cp_async_wait_all();
      }
      __syncthreads();
    } else {
      // stage the box: one TMA bulk copy per row (warp 0), completion on the mbarrier
      if (warp == 0) {
        if (lane == 0) mbar_arrive_expect_tx(&box_bar, unsigned(rows * cols) * 16u);
        __syncwarp();
        for (int rr = lane; rr < rows; rr += 32)
          tma_bulk_g2s(box_s + rr * pitch, src + int64_t(r0 + rr) * P + c0, unsigned(cols) * 16u, &box_bar);
      }
      mbar_wait(&box_bar, unsigned(c & 1));
    }
    const float ox = float(c0), oy = float(r0);
    const int dA = (rs ? pitch : 0) + (cs ? 1 : 0);
    const int dY = rs ? -pitch : pitch;
    // chunk-relative entry point: the box origin is an integer, so the shift
    // is exact and the per-sample position one FMA
    const float pxc = px0 - ox, pyc = py0 - oy;
    for (; m < m_end; ++m) {
      const float t = float(m) + 0.5f;
      const float px = fmaf(t, hx, pxc);
      const float py = fmaf(t, hy, pyc);
      const float fj = floorf(px), fi = floorf(py);
      const float fx = px - fj, fy = py - fi;
      const int j = int(fj), i = int(fi);  // inside the box by construction (fwd_plan.cpp slack)
      const float gx = 1.f - fx, gy = 1.f - fy;
      const float ya = rs ? fy : gy, yb = rs ? gy : fy;
      const float xa = cs ? fx : gx, xb = cs ? gx : fx;
      const float w1 = xa * ya, w2 = xb * ya, w3 = xa * yb, w4 = xb * yb;
      if constexpr (LANE) {
        const float* q = box1 + (i * pitch + j + dA);
        const float v1 = q[0], v2 = q[dX], v3 = q[dY], v4 = q[dY + dX];
        a01.x = fmaf(w1, v1, fmaf(w2, v2, fmaf(w3, v3, fmaf(w4, v4, a01.x))));
        continue;
      } else if constexpr (H8) {
        const uint4* q8 = reinterpret_cast<const uint4*>(box_s) + (i * pitch + j + dA);
        const uint4 u1 = q8[0], u2 = q8[dX], u3 = q8[dY], u4 = q8[dY + dX];
#pragma unroll
        for (int wd = 0; wd < 4; ++wd) {
          const float2 f1 = h8_pair(h8_word(u1, wd)), f2 = h8_pair(h8_word(u2, wd));
          const float2 f3 = h8_pair(h8_word(u3, wd)), f4 = h8_pair(h8_word(u4, wd));
          // scalar FMAs: FFMA2 on converted pairs (no register moves) measured equal for the forward
          // and 11 % slower for the backprojection (r2 A/B, tools/ab_bench.sh): the conversions and
          // FMAs share the FP32 pipe, which FFMA2 occupies for two slots
          a8[wd].x = fmaf(w1, f1.x, fmaf(w2, f2.x, fmaf(w3, f3.x, fmaf(w4, f4.x, a8[wd].x))));
          a8[wd].y = fmaf(w1, f1.y, fmaf(w2, f2.y, fmaf(w3, f3.y, fmaf(w4, f4.y, a8[wd].y))));
        }
      } else {
      const float4* q = box_s + (i * pitch + j + dA);
      const float4 v1 = q[0], v2 = q[dX], v3 = q[dY], v4 = q[dY + dX];
      a01 = ffma2(w1, lo2(v1), ffma2(w2, lo2(v2), ffma2(w3, lo2(v3), ffma2(w4, lo2(v4), a01))));
      a23 = ffma2(w1, hi2(v1), ffma2(w2, hi2(v2), ffma2(w3, hi2(v3), ffma2(w4, hi2(v4), a23))));
      }
    }
  }
  if (!valid) return;
  const float h = X.x;
  if constexpr (H8) {  // user layout only (fp16 storage)
    const int64_t n_rays8 = int64_t(na) * nd;
#pragma unroll
    for (int q = 0; q < kPackH8; ++q) {
      const int64_t b = g * kPackH8 + q;
      if (b < batch) sino[b * n_rays8 + r] = from_f32<TOut>((q & 1 ? a8[q >> 1].y : a8[q >> 1].x) * h);
    }
    return;
  }
  const float acc[kPack] = {a01.x * h, a01.y * h, a23.x * h, a23.y * h};
  const int64_t n_rays = int64_t(na) * nd;
  if (epi.mode == kOutUser) {
#pragma unroll
    for (int q = 0; q < kPack; ++q) {
      const int64_t b = g * kPack + q;
      if (b < batch) sino[b * n_rays + r] = from_f32<TOut>(acc[q]);
    }
  } else {
    // packed sinogram for the solvers; kOutResidual subtracts y (solvers.cpp:136: A x - y)
    float4 v = make_float4(acc[0], acc[1], acc[2], acc[3]);
    if (epi.mode == kOutResidual) {
      const float4 y = __ldg(epi.resid + g * n_rays + r);
      v = make_float4(v.x - y.x, v.y - y.y, v.z - y.z, v.w - y.w);
    }
    epi.packed[g * n_rays + r] = v;
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
// Per-angle constants of one tile.  Parallel beam: kf - ws is affine in the
// pixel offsets, fp32 suffices (no magnification).  Fan beam: the pixel ->
// detector map u = qx * span / (qy + D_so) magnifies position errors by
// span / (sp (qy + D_so)).  kBpFan32 evaluates it relative to the tile corner,
//   kf - ws = base + (dq K - u00 dd) / (den00 + dd),   dq, dd = O(tile) offsets,
// which keeps fp32 accurate for moderate magnification; kBpFan64 (source close
// to the image, plan.cpp picks it) runs the per-pixel map in fp64.  With
// dq = lx c - ly s and dd = -lx s - ly c both numerator and denominator are
// affine in the tile offsets (lx, ly): num = A lx + B ly, den = den00 + C lx +
// D ly (A, B from fp64), and every lx term is shared by a thread's pixels.
// kBpParHP (parallel beam, wide windows: fine detector spacing): kf reaches
// the window width (hundreds to thousands of cells), where one fp32 ulp is a
// visible weight error, so kf is carried as an exact "hi" part (multiples of
// 2^-10 below 2^14: every partial sum is exact in fp32) plus a small "lo"
// correction; floor and fraction come from hi, lo is added to the fraction.
enum { kBpParallel = 0, kBpFan32 = 1, kBpFan64 = 2, kBpParHP = 3 };
struct ParConst {
  float base, cx, cy, pad;
};
struct ParHPConst {
  float base_hi, cx_hi, cy_hi, base_lo, cx_lo, cy_lo, pad0, pad1;
};
struct Fan32Const {
  float base, a, b, den00, c, d, pad0, pad1;
};
struct FanConst {
  double qx00, den00, c, s, offw, pad;
};
template <int KIND>
struct BpConst {
  using type = ParConst;
};
template <>
struct BpConst<kBpFan32> {
  using type = Fan32Const;
};
template <>
struct BpConst<kBpFan64> {
  using type = FanConst;
};
template <>
struct BpConst<kBpParHP> {
  using type = ParHPConst;
};

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

constexpr int kTile = 32;
constexpr int kBpHPWindow = 128;  // staged cells above which kf leaves the fp32-exact range (kBpParHP / kBpFan64)
constexpr int kMaxBpChunk = 32;  // angles per staging pass (one constants record per thread of the first warp)
// LANE stages 4-byte cells, so the same shared memory holds four times the angles: fewer
// passes and barriers per tile (the batch-1 kernel's largest stall, ncu r2h)
constexpr int kMaxBpChunkLane = 128;
// H8 (two CTAs per SM of 512 threads): a window slab up to four times the plan's, as many
// as two CTAs per SM still fit (launch_backproject), up to 128 angles per pass
constexpr int kMaxBpChunkH8 = 128;
constexpr int kRowsPerThread = 4;
constexpr int kBpThreads = kTile * (kTile / kRowsPerThread);  // 256

// LANE (batch 1): only lane 0 of the packed group carries a sinogram; the
// windows are staged as scalars (lane 0 of each cell) and the CTA has 512
// threads x 2 pixels, so the 32x32 tiles of one image fill the GPU.  Per
// pixel the operations on lane 0 and their order are the packed kernel's
// (same tile-relative constants), so the results are bit-identical.
// H8 (fp16 storage, batch > 1): half8 cells, eight images per pixel, 512
// threads x 2 pixels (the accumulators of eight images), each tap load
// converted to fp32 pairs; per image the same operations and order.
// WIDE (small batches, float4 cells): 512 threads x 2 pixels per tile, so the
// few tiles of one or two image groups still fill the SMs with warps; per pixel
// the operations and their order are the 256-thread kernel's (bit-identical).
// NARROW (float4 cells, parallel / fan fp32 map): 128 threads x 8 pixels per
// tile, seven CTAs per SM: the per-angle constants are read once per eight
// pixels instead of four, and 1,036 resident CTAs hold a four-group batch's
// 1,024 tiles in one wave; per pixel the same operations (bit-identical).
template <int KIND, class TOut, bool LANE, bool H8 = false, bool WIDE = false, bool NARROW = false>
__global__ void __launch_bounds__(NARROW ? 128 : (LANE || H8 || WIDE) ? 512 : kBpThreads,
                                  NARROW ? 7 : (LANE || H8 || WIDE) ? 2 : (KIND == kBpFan64 ? 3 : 4))
    backproject_kernel(
    const float4* __restrict__ sino, int s, int na, int nd, double spacing, double source_distance,
    double det_distance, const double2* __restrict__ trig, const int* __restrict__ tile_window, int cells,
    int64_t batch, TOut* __restrict__ out, BpEpilogue epi) {
  using Const = typename BpConst<KIND>::type;
  using Cell = typename std::conditional<LANE, float, float4>::type;
  constexpr int RPT = NARROW ? 8 : (LANE || H8 || WIDE) ? 2 : kRowsPerThread;  // pixels (rows) per thread
  constexpr int NT = kTile * kTile / RPT;         // threads
  static_assert(kTile % RPT == 0, "pixels per thread must divide the tile height");
  extern __shared__ float4 smem_raw[];
  Cell* smem = reinterpret_cast<Cell*>(smem_raw);
  // this tile's staged cells per angle, and as many angles per pass as fit
  const int window = __ldg(tile_window + blockIdx.y * gridDim.x + blockIdx.x);
  // middle cell: the fp32 kinds measure kf from it (fp32 / fp64 storage; the fp16-storage
  // kernels keep the window-start origin — their tolerance is 1e-3 and they are issue-bound)
  constexpr bool kCentred = (KIND == kBpParallel || KIND == kBpFan32) && !std::is_same<TOut, __half>::value;
  const int wc = kCentred ? window >> 1 : 0;
  // cells: staged window cells per pass (LANE: 4-byte cells, launch_backproject)
  constexpr int kCap = LANE ? kMaxBpChunkLane : (H8 || WIDE) ? kMaxBpChunkH8 : kMaxBpChunk;
  const int chunk = min(kCap, cells / window);
  Cell* win = smem;                                                    // chunk * window <= cells
  Const* cst = reinterpret_cast<Const*>(smem_raw + (LANE ? (cells + 3) / 4 : cells));  // kCap records
  int* ws_s = reinterpret_cast<int*>(cst + kCap);                      // kCap window starts

  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kTile + tx;
  const int j0 = blockIdx.x * kTile, i0 = blockIdx.y * kTile;
  // Tile-relative (row, column) of the thread's r-th pixel.  Parallel beam: a
  // warp is one row of 32 pixels (adjacent pixels read adjacent detector
  // cells, conflict free).  Fan beam: magnification up to span / (sp (D_so -
  // R)) spreads a row of 8 pixels over more than 8 cells, so a quarter warp
  // takes a 4 x 2 block (a warp an 8 x 4 block; block w * RPT + r of the
  // tile's 32), which keeps its cells within one bank period.
  auto pixel_of = [&](int t, int r, int& pr, int& pc) {
    if constexpr (KIND == kBpParallel || KIND == kBpParHP) {
      pr = (t >> 5) + r * (kTile / RPT);
      pc = t & 31;
    } else {
      const int l = t & 31, qq = l >> 3, e = l & 7, blk = (t >> 5) * RPT + r;
      pc = 8 * (blk & 3) + 4 * (qq & 1) + (e & 3);
      pr = 4 * (blk >> 2) + 2 * (qq >> 1) + (e >> 2);
    }
  };
  const int64_t g = blockIdx.z;
  const double half = 0.5 * double(s);
  const double off = 0.5 * double(nd) - 0.5;
  const double span = source_distance + det_distance;
  // centre of the tile's first pixel (projector.cpp:150,154)
  const double x0 = double(j0) - half + 0.5;
  const double y0 = half - double(i0) - 0.5;
  const float4* sg = sino + g * int64_t(na) * nd;

  float4 acc[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  float acc8[H8 ? RPT : 1][H8 ? kPackH8 : 1];
#pragma unroll
  for (int r = 0; r < (H8 ? RPT : 1); ++r)
#pragma unroll
    for (int q = 0; q < (H8 ? kPackH8 : 1); ++q) acc8[r][q] = 0.f;

  // Packed cells (float4 / half8) are staged by TMA bulk copies: one per angle
  // (the in-detector part of its window, a contiguous run of 16-byte cells),
  // issued by the thread that derived the window, completing on an mbarrier
  // that threads 0 .. kCap-1 arrive on each pass; the out-of-detector cells are
  // zero-filled by the CTA.  This keeps the staging off the LSU (r1 loaded
  // the cells through L1 into registers and stored them).  LANE (lane 0 of
  // each cell) still stages through registers.
  __shared__ unsigned long long win_bar;
  if constexpr (!LANE) {
    if (tid == 0) {
      mbar_init(&win_bar, min(kCap, NT));  // one arrival per thread tid < kCap each pass
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  unsigned win_phase = 0;
  for (int a0 = 0; a0 < na; a0 += chunk) {
    const int nac = min(chunk, na - a0);
    // ---- per-angle constants, fp64 (one thread per angle)
    if (tid < nac) {
      const double2 cs = trig[a0 + tid];
      const double c = cs.x, sn = cs.y;
      // last in-image pixel of the tile: the footprint extremes sit at the
      // corners only where qy + D_so keeps its sign, i.e. inside the image
      const double x1 = x0 + double(min(kTile, s - j0) - 1), y1 = y0 - double(min(kTile, s - i0) - 1);
      double lo;
      Const k;
      if constexpr (KIND == kBpParallel || KIND == kBpParHP) {
        const double k00 = (x0 * c + y0 * sn) / spacing + off;
        const double k10 = (x1 * c + y0 * sn) / spacing + off;
        const double k01 = (x0 * c + y1 * sn) / spacing + off;
        const double k11 = (x1 * c + y1 * sn) / spacing + off;
        lo = fmin(fmin(k00, k10), fmin(k01, k11));
        const int ws = max(int(floor(lo)) - 1, -2);  // clipped like the host window (plan.cpp)
        if constexpr (KIND == kBpParallel) {
          k.base = float(k00 - double(ws) - double(wc));  // relative to the window's middle cell
          k.cx = float(c / spacing);
          k.cy = float(-sn / spacing);
          k.pad = 0.f;
        } else {
          constexpr double q = 1.0 / 1024.0;  // hi parts: multiples of 2^-10
          const double base = k00 - double(ws), cx = c / spacing, cy = -sn / spacing;
          const double bh = rint(base / q) * q, xh = rint(cx / q) * q, yh = rint(cy / q) * q;
          k.base_hi = float(bh);
          k.cx_hi = float(xh);
          k.cy_hi = float(yh);
          k.base_lo = float(base - bh);
          k.cx_lo = float(cx - xh);
          k.cy_lo = float(cy - yh);
          k.pad0 = k.pad1 = 0.f;
        }
        ws_s[tid] = ws;
      } else {
        auto kfan = [&](double x, double y) {
          const double qx = x * c + y * sn, qy = -x * sn + y * c;
          return (qx * span / (qy + source_distance)) / spacing + off;
        };
        const double k00 = kfan(x0, y0);
        lo = fmin(fmin(k00, kfan(x1, y0)), fmin(kfan(x0, y1), kfan(x1, y1)));
        const int ws = max(int(floor(lo)) - 1, -2);  // clipped like the host window (plan.cpp)
        const double qx00 = x0 * c + y0 * sn;
        const double den00 = -x0 * sn + y0 * c + source_distance;
        if constexpr (KIND == kBpFan32) {
          const double K = span / spacing, u00 = qx00 * K / den00;
          k.base = float(k00 - double(ws) - double(wc));  // relative to the window's middle cell
          k.a = float(c * K + u00 * sn);
          k.b = float(u00 * c - sn * K);
          k.den00 = float(den00);
          k.c = float(-sn);
          k.d = float(-c);
          k.pad0 = k.pad1 = 0.f;
        } else {
          k.qx00 = qx00;
          k.den00 = den00;
          k.c = c;
          k.s = sn;
          k.offw = off - double(ws);
          k.pad = 0.0;
        }
        ws_s[tid] = ws;
      }
      cst[tid] = k;
      if constexpr (!LANE) {
        // this angle's in-detector cells [k0, k1) of the window [ws, ws + window)
        const int ws = ws_s[tid];
        const int k0 = max(ws, 0), k1 = min(ws + window, nd);
        const unsigned bytes = k1 > k0 ? unsigned(k1 - k0) * 16u : 0u;
        // the previous pass read (generic proxy) what this copy overwrites (async proxy)
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_expect_tx(&win_bar, bytes);
        if (bytes)
          tma_bulk_g2s(win + tid * window + (k0 - ws), sg + int64_t(a0 + tid) * nd + k0, bytes, &win_bar);
      }
    } else if (!LANE && tid < kCap) {
      mbar_arrive(&win_bar);
    }
    __syncthreads();
    // ---- stage the detector windows (16-byte cells; zero outside [0, det_count))
    for (int e = tid; e < nac * window; e += NT) {
      const int q = e / window, cidx = e - q * window;
      const int k = ws_s[q] + cidx;
      if constexpr (LANE) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k >= 0 && k < nd) v = __ldg(sg + int64_t(a0 + q) * nd + k);
        win[e] = v.x;
      } else {
        if (k < 0 || k >= nd) win[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if constexpr (!LANE) {
      mbar_wait(&win_bar, win_phase);
      win_phase ^= 1u;
    }
    __syncthreads();
    // ---- accumulate
    const double kmag = span / spacing;
    for (int q = 0; q < nac; ++q) {
      const Const k = cst[q];
      // fp32 kinds: kf relative to the middle cell wc of the window (half the magnitude, half the
      // fp32 rounding of kf); the pointer carries the offset back
      const Cell* w = win + q * window + wc;
      // parallel: the column term is shared by the thread's pixels (one column);
      // fan (fp32 map): the row terms (a thread's pixels share one row)
      float col0 = 0.f, nrow = 0.f, drow = 0.f;
      if constexpr (KIND == kBpParallel) col0 = fmaf(float(tx), k.cx, k.base);
      if constexpr (KIND == kBpParHP) {
        col0 = fmaf(float(tx), k.cx_hi, k.base_hi);  // exact
        nrow = fmaf(float(tx), k.cx_lo, k.base_lo);  // the small correction
      }
      if constexpr (KIND == kBpFan32) {
        int pr0, pc0;
        pixel_of(tid, 0, pr0, pc0);
        nrow = k.b * float(pr0);
        drow = fmaf(k.d, float(pr0), k.den00);
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        int pr, pc;
        pixel_of(tid, r, pr, pc);
        const float lx = float(pc), ly = float(pr);
        if constexpr (KIND == kBpFan32 && RPT > 4) {
          if (r > 0 && r % 4 == 0) {  // NARROW: pixels r = 4.. sit on the next row
            nrow = k.b * ly;
            drow = fmaf(k.d, ly, k.den00);
          }
        }
        float fk, wt;
        if constexpr (KIND == kBpParallel) {
          const float kf = fmaf(ly, k.cy, col0);
          fk = floorf(kf);
          wt = kf - fk;
        } else if constexpr (KIND == kBpParHP) {
          const float hi = fmaf(ly, k.cy_hi, col0);  // exact (multiples of 2^-10 below 2^14)
          const float lo = fmaf(ly, k.cy_lo, nrow);
          fk = floorf(hi);
          wt = (hi - fk) + lo;  // hi - fk exact
          if (wt >= 1.f) {
            fk += 1.f;
            wt -= 1.f;
          } else if (wt < 0.f) {
            fk -= 1.f;
            wt += 1.f;
          }
        } else if constexpr (KIND == kBpFan32) {
          const float num = fmaf(k.a, lx, nrow);  // (qx - qx00) K - u00 (den - den00)
          const float den = fmaf(k.c, lx, drow);  // qy + D_so
          float r = rcp_approx(den);
          r = fmaf(r, fmaf(-den, r, 1.f), r);  // one Newton step: the reciprocal to ~0.5 ulp
          const float kf = fmaf(num, r, k.base);
          fk = floorf(kf);
          wt = kf - fk;
        } else {
          const double dlx = double(lx), dly = double(ly);
          const double qx = fma(dlx, k.c, fma(-dly, k.s, k.qx00));
          const double den = fma(-dlx, k.s, fma(-dly, k.c, k.den00));
          double r = double(rcp_approx(float(den)));
          r = fma(r, fma(-den, r, 1.0), r);  // one Newton step: ~1e-14 relative
          const double kd = fma(qx * kmag, r, k.offw);
          const double fd = floor(kd);  // floor and fraction in fp64: kf can be thousands of cells
          fk = float(fd);
          wt = float(kd - fd);
        }
        const int c0 = min(max(int(fk), -wc), window - 2 - wc);
        const float wl = 1.f - wt;
        if constexpr (LANE) {
          const float s0 = w[c0], s1 = w[c0 + 1];
          acc[r].x = fmaf(wt, s1, fmaf(wl, s0, acc[r].x));
        } else if constexpr (H8) {
          const float4 s0f = w[c0], s1f = w[c0 + 1];
          const uint4 s0 = *reinterpret_cast<const uint4*>(&s0f), s1 = *reinterpret_cast<const uint4*>(&s1f);
#pragma unroll
          for (int wd = 0; wd < 4; ++wd) {
            const float2 f0 = h8_pair(h8_word(s0, wd)), f1 = h8_pair(h8_word(s1, wd));
            acc8[r][2 * wd] = fmaf(wt, f1.x, fmaf(wl, f0.x, acc8[r][2 * wd]));
            acc8[r][2 * wd + 1] = fmaf(wt, f1.y, fmaf(wl, f0.y, acc8[r][2 * wd + 1]));
          }
        } else {
          const float4 s0 = w[c0], s1 = w[c0 + 1];
          const float2 lo = ffma2(wt, lo2(s1), ffma2(wl, lo2(s0), lo2(acc[r])));
          const float2 hi = ffma2(wt, hi2(s1), ffma2(wl, hi2(s0), hi2(acc[r])));
          acc[r] = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
      }
    }
    __syncthreads();
  }
  // ---- store
  const int P = s + 2;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    int pr, pc;
    pixel_of(tid, r, pr, pc);
    const int i = i0 + pr, j = j0 + pc;
    if (i >= s || j >= s) continue;
    if constexpr (H8) {  // user layout only (fp16 storage)
#pragma unroll
      for (int q = 0; q < kPackH8; ++q) {
        const int64_t b = g * kPackH8 + q;
        if (b < batch) out[(b * s + i) * int64_t(s) + j] = from_f32<TOut>(acc8[r][q]);
      }
      continue;
    }
    if (epi.mode == kOutUser) {
      const float v[kPack] = {acc[r].x, acc[r].y, acc[r].z, acc[r].w};
#pragma unroll
      for (int q = 0; q < kPack; ++q) {
        const int64_t b = g * kPack + q;
        if (b < batch) out[(b * s + i) * int64_t(s) + j] = from_f32<TOut>(v[q]);
      }
      continue;
    }
    float4* dst = epi.packed + g * int64_t(P) * P + int64_t(i + 1) * P + (j + 1);
    if (epi.mode == kOutPacked) {
      // narrowed through the storage precision like a user-visible result
      *dst = make_float4(float(from_f32<TOut>(acc[r].x)), float(from_f32<TOut>(acc[r].y)),
                         float(from_f32<TOut>(acc[r].z)), float(from_f32<TOut>(acc[r].w)));
    } else if (epi.mode == kOutSystem) {
      // axpy(p0, A'A x, scale(x, 1 + p1)) in fp32 (admm.cpp:142, tensor.cpp:334-347)
      const float4 x = __ldg(epi.src + (dst - epi.packed));
      const float c0 = epi.c0, c1 = epi.c1;
      *dst = make_float4(__fadd_rn(__fmul_rn(c0, acc[r].x), __fmul_rn(c1, x.x)),
                         __fadd_rn(__fmul_rn(c0, acc[r].y), __fmul_rn(c1, x.y)),
                         __fadd_rn(__fmul_rn(c0, acc[r].z), __fmul_rn(c1, x.z)),
                         __fadd_rn(__fmul_rn(c0, acc[r].w), __fmul_rn(c1, x.w)));
    } else {
      // Landweber update x <- (-alpha) * grad + x in fp32 (solvers.cpp:139, tensor.cpp:338-343)
      const float4 x = *dst;
      const float na_ = epi.neg_alpha;
      const float4 v = make_float4(__fadd_rn(__fmul_rn(na_, acc[r].x), x.x), __fadd_rn(__fmul_rn(na_, acc[r].y), x.y),
                                   __fadd_rn(__fmul_rn(na_, acc[r].z), x.z), __fadd_rn(__fmul_rn(na_, acc[r].w), x.w));
      *dst = v;
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < kPack; ++q)
        if (g * kPack + q < batch && !isfinite(vv[q])) atomicMin(epi.flag, epi.iteration);  // all_finite, :140-142
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

void launch_pack_images_h8(const void* src, int64_t batch, int64_t s, float4* dst, cudaStream_t st) {
  const int64_t plane = (s + 2) * (s + 2);
  dim3 grid(std::min<unsigned>(blocks_for(plane, 256), 4096u), unsigned(groups_of_h8(batch)));
  KernelTimer timer(RK_KERNEL_PACK, st);
  pack_images_h8_kernel<<<grid, 256, 0, st>>>(static_cast<const __half*>(src), batch, int(s),
                                              reinterpret_cast<uint4*>(dst));
  RK_CUDA(cudaGetLastError());
}

void launch_pack_sino_h8(const void* src, int64_t batch, int64_t na, int64_t nd, float4* dst, cudaStream_t st) {
  const int64_t plane = na * nd;
  dim3 grid(std::min<unsigned>(blocks_for(plane, 256), 4096u), unsigned(groups_of_h8(batch)));
  KernelTimer timer(RK_KERNEL_PACK, st);
  pack_sino_h8_kernel<<<grid, 256, 0, st>>>(static_cast<const __half*>(src), batch, plane,
                                            reinterpret_cast<uint4*>(dst));
  RK_CUDA(cudaGetLastError());
}

// RK_H8=0 keeps fp16 storage on the float4 layout (A/B).
bool use_h8(int dtype, int64_t batch) {
  static const bool on = [] {
    const char* e = std::getenv("RK_H8");
    return !(e && e[0] == '0');
  }();
  return on && dtype == RK_F16 && batch > 1;
}

void launch_transpose_images(const float4* src, int64_t groups, int64_t s, float4* dst, cudaStream_t st) {
  const int P = int(s + 2);
  dim3 grid(unsigned((P + 31) / 32), unsigned((P + 31) / 32), unsigned(groups));
  KernelTimer timer(RK_KERNEL_PACK, st);
  transpose_images_kernel<<<grid, dim3(32, 8), 0, st>>>(src, P, dst);
  RK_CUDA(cudaGetLastError());
}

// Batch 1: the single-lane kernels (RK_SINGLE_LANE=0 forces the packed ones, for A/B).
static bool single_lane(int64_t batch) {
  static const bool on = [] {
    const char* e = std::getenv("RK_SINGLE_LANE");
    return !(e && e[0] == '0');
  }();
  return on && batch == 1;
}

// float4 backprojection as 128 threads x 8 pixels per tile (RK_BP_NARROW=0: 256 x 4)
static bool narrow_bp() {
  static const bool on = [] {
    const char* e = std::getenv("RK_BP_NARROW");
    return !(e && e[0] == '0');
  }();
  return on;
}

// backprojection of at most kWideGroups packed groups: the 512-thread variant
static bool wide_bp(int64_t groups) {
  static const int limit = [] {
    const char* e = std::getenv("RK_BP_WIDE_GROUPS");
    return e ? std::atoi(e) : 1;
  }();
  return groups <= limit;
}

void launch_forward(const Plan& p, const float4* packed_image, const float4* packed_image_t, int64_t batch,
                    int dtype, void* sino, cudaStream_t st, FwdEpilogue epi) {
  const ForwardSchedule& F = p.fwd;
  const bool h8 = epi.mode == kOutUser && use_h8(dtype, batch);
  const int64_t groups = h8 ? groups_of_h8(batch) : groups_of(batch);
  // few groups (small batches, e.g. a rank's shard): CTA-major launch order, so the longest
  // CTAs of every group start first and the last wave holds the shortest; with many groups
  // group-major order keeps one group's image in L2 while its CTAs run
  static const int64_t cta_major_groups = [] {
    const char* e = std::getenv("RK_FWD_CTA_MAJOR_GROUPS");
    return e ? int64_t(std::atoll(e)) : int64_t(8);
  }();
  const bool cta_major = !single_lane(batch) && groups <= cta_major_groups && F.cta.size() <= 65535;
  const dim3 grid = cta_major ? dim3(unsigned(groups), unsigned(F.cta.size()))
                              : dim3(unsigned(F.cta.size()), unsigned(groups));
  dispatch_dtype(dtype, [&](auto tag) {
    using T = decltype(tag);
    const bool lane = single_lane(batch);
    const bool nw = F.any_narrow;
    // the variant for (single lane, half8): narrow-lane check and launch order from the schedule
    auto pick = [&](auto lane_tag, auto h8_tag) {
      constexpr bool L = decltype(lane_tag)::value, H = decltype(h8_tag)::value;
      if constexpr (L) {
        return nw ? forward_kernel<T, L, H, true, false> : forward_kernel<T, L, H, false, false>;
      } else {
        return nw ? (cta_major ? forward_kernel<T, L, H, true, true> : forward_kernel<T, L, H, true, false>)
                  : (cta_major ? forward_kernel<T, L, H, false, true> : forward_kernel<T, L, H, false, false>);
      }
    };
    auto kern = lane ? pick(std::true_type{}, std::false_type{}) : pick(std::false_type{}, std::false_type{});
    if constexpr (std::is_same<T, __half>::value)
      if (h8) kern = pick(std::false_type{}, std::true_type{});
    const size_t smem = size_t(F.max_box) * (lane ? 2 * sizeof(float) : sizeof(float4));
    allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    KernelTimer timer(RK_KERNEL_FORWARD, st);
    kern<<<grid, kFwdThreads, smem, st>>>(packed_image, packed_image_t, int(p.s), p.ray_geom.as<float4>(),
                                         p.ray_aux.as<float4>(), p.fwd_boxes.as<int4>(), p.fwd_cta.as<int4>(),
                                         p.fwd_warps.as<int2>(), int(p.na), int(p.nd), batch,
                                         static_cast<T*>(sino), epi, int(F.max_box));
  });
  RK_CUDA(cudaGetLastError());
}

void launch_backproject(const Plan& p, const float4* packed_sino, int64_t batch, int dtype, void* image,
                        cudaStream_t st, BpEpilogue epi) {
  const int tiles = int((p.s + kTile - 1) / kTile);
  const bool h8 = epi.mode == kOutUser && use_h8(dtype, batch);
  dim3 grid(tiles, tiles, unsigned(h8 ? groups_of_h8(batch) : groups_of(batch)));
  const bool lane = single_lane(batch);
  const bool wide = !lane && !h8 && wide_bp(groups_of(batch));
  // wide windows (fine detectors): kf spans hundreds of cells, so parallel beam carries it in
  // two parts and fan beam uses the fp64 map (r2 extreme-geometry sweep, tools/stress_extreme.py)
  const bool fan = p.g.kind == RK_FANBEAM;
  const int kind = !fan ? (p.bp_window > kBpHPWindow ? kBpParHP : kBpParallel)
                        : (p.bp_fan_fp64 || p.bp_window > 2 * kBpHPWindow ? kBpFan64 : kBpFan32);
  const bool narrow = !lane && !h8 && !wide && kind != kBpFan64 && narrow_bp();
  dim3 block(kTile, kTile / (narrow ? 8 : (lane || h8 || wide) ? 2 : kRowsPerThread));
  const size_t rec = kind == kBpParallel ? sizeof(ParConst)
                     : kind == kBpParHP  ? sizeof(ParHPConst)
                     : kind == kBpFan32  ? sizeof(Fan32Const)
                                         : sizeof(FanConst);
  const int cells = narrow ? p.bp_cells_narrow : p.bp_cells;
  // LANE: the same bytes as 4-byte cells, up to kMaxBpChunkLane angles per pass (RK_BP_LANE_WIDE=0: as
  // many angles as the float4 kernels)
  static const bool lane_wide = [] {
    const char* e = std::getenv("RK_BP_LANE_WIDE");
    return !(e && e[0] == '0');
  }();
  static const bool wide_slab = [] {
    const char* e = std::getenv("RK_BP_WIDE_SLAB");
    return !(e && e[0] == '0');
  }();
  const int cap = lane ? kMaxBpChunkLane : (h8 || wide) ? kMaxBpChunkH8 : kMaxBpChunk;
  // H8 / WIDE (512 threads, two CTAs per SM): the widest slab (4x, 2x the plan's) with which
  // two CTAs still fit an SM's 228 KB (1 KB runtime reserve each): cfg2 windows take 4x
  // (128 angles per pass), cfg3's 2x
  int slab_factor = 1;
  if ((h8 || wide) && wide_slab)
    for (int f : {4, 2})
      if (2 * (size_t(f) * cells * sizeof(float4) + size_t(cap) * (rec + sizeof(int)) + 1024 + 64) <= 233472) {
        slab_factor = f;
        break;
      }
  const int cells_arg = lane && lane_wide ? 4 * cells : (h8 || wide) ? slab_factor * cells : cells;
  const size_t smem = size_t(lane ? cells : cells_arg) * sizeof(float4) + size_t(cap) * (rec + sizeof(int));
  dispatch_dtype(dtype, [&](auto tag) {
    using T = decltype(tag);
    // the kernel variant for one kind: single-lane (batch 1), half8, WIDE (one group), NARROW or 256 x 4
    auto pick = [&](auto kind_tag) {
      constexpr int K = decltype(kind_tag)::value;
      auto kern = lane ? backproject_kernel<K, T, true> : backproject_kernel<K, T, false>;
      if constexpr (K != kBpFan64)
        if (narrow) kern = backproject_kernel<K, T, false, false, false, true>;
      if (wide) kern = backproject_kernel<K, T, false, false, true>;
      if constexpr (std::is_same<T, __half>::value)
        if (h8) kern = backproject_kernel<K, T, false, true>;
      return kern;
    };
    auto kern = kind == kBpParallel ? pick(std::integral_constant<int, kBpParallel>{})
                : kind == kBpParHP  ? pick(std::integral_constant<int, kBpParHP>{})
                : kind == kBpFan32  ? pick(std::integral_constant<int, kBpFan32>{})
                                    : pick(std::integral_constant<int, kBpFan64>{});
    allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    KernelTimer timer(RK_KERNEL_BACKPROJECT, st);
    kern<<<grid, block, smem, st>>>(packed_sino, int(p.s), int(p.na), int(p.nd), p.g.det_spacing,
                                    p.g.source_distance, p.g.det_distance, p.trig.as<double2>(),
                                    p.bp_tile_window.as<int>(), cells_arg, batch, static_cast<T*>(image), epi);
  });
  RK_CUDA(cudaGetLastError());
}

}  // namespace rk
