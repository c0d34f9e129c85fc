// Micro-benchmark: are the L1TEX LSU (shared-memory) and TEX data pipes additive?
// Each warp streams conflict-free LDS.128 from shared memory and/or float4
// texture fetches (tex1Dfetch, L1-resident working set).  If the two pipes
// share one data path, LDS+TEX bytes/clk stay at the LDS-only rate.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lsu_tex lsu_tex.cu
#include <cstdio>

template <int NLDS, int NTEX>
__global__ void __launch_bounds__(256, 4) kern(cudaTextureObject_t tex, int iters, float* out) {
  __shared__ float4 cells[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) cells[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int a = (threadIdx.x * 8 + lane) & 2047;
  int t = (blockIdx.x * 256 + threadIdx.x) & 4095;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NLDS; ++k) {
      const float4 v = cells[(a + 32 * k) & 2047];
      acc.x += v.x;
      acc.y += v.w;
    }
#pragma unroll
    for (int k = 0; k < NTEX; ++k) {
      const float4 v = tex1Dfetch<float4>(tex, (t + 32 * k) & 4095);
      acc.z += v.x;
      acc.w += v.y;
    }
    a = (a + 64 + int(acc.x == -1.f)) & 2047;
    t = (t + 64 + int(acc.z == -1.f)) & 4095;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <int NLDS, int NTEX>
void run(cudaTextureObject_t tex, float* out) {
  const int iters = 2000, blocks = 148 * 4 * 4;
  kern<NLDS, NTEX><<<blocks, 256, 0>>>(tex, iters, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<NLDS, NTEX><<<blocks, 256, 0>>>(tex, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = double(blocks) * 256 * iters * (NLDS + NTEX) * 16.0;
  const double per_clk_sm = bytes / (ms * 1e-3) / 148.0 / 1.965e9;
  printf("LDS.128 x%d + TEX float4 x%d: %.3f ms, %.1f B/clk/SM (LDS part %.1f, TEX part %.1f)\n", NLDS, NTEX, ms,
         per_clk_sm, per_clk_sm * NLDS / (NLDS + NTEX), per_clk_sm * NTEX / (NLDS + NTEX));
}

int main() {
  float4* buf;
  cudaMalloc(&buf, 4096 * sizeof(float4));
  cudaMemset(buf, 0, 4096 * sizeof(float4));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = buf;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = 4096 * sizeof(float4);
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  float* out;
  cudaMalloc(&out, 148 * 16 * 256 * sizeof(float));
  run<4, 0>(tex, out);
  run<0, 4>(tex, out);
  run<4, 2>(tex, out);
  run<4, 4>(tex, out);
  run<2, 2>(tex, out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
