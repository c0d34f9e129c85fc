// Micro-benchmark of the shared-memory bank model for 128-bit loads (LDS.128)
// on sm_100a: each lane of every warp loads float4 texels at a pattern of
// 16-byte cell indices; ncu's l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld
// per executed load tells how the hardware groups lanes into wavefronts.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o smem_model smem_model.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void probe(const int* __restrict__ pattern, int iters, float* out) {
  __shared__ float4 cells[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) cells[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  int a = pattern[threadIdx.x & 31];
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const float4 v = cells[a];
    acc += v.x + v.w;
    a = (a + int(v.y == -1.f)) & 1023;  // data dependence, never taken
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  std::vector<int> p(32);
  for (int l = 0; l < 32; ++l) {
    const int q = l / 8, i = l % 8, h = l / 16;
    switch (which) {
      case 0: p[l] = l; break;                                  // consecutive: 4 wavefronts
      case 1: p[l] = l < 8 ? 8 * l : 64 + l; break;             // quarter 0 all in slot 0
      case 2: p[l] = (i / 2) + 8 * (i & 1) + 4 * (q & 1) + 16 * h; break;  // 2-way within quarters, disjoint slot halves per quarter pair
      case 3: p[l] = 5; break;                                  // broadcast
      case 4: p[l] = i; break;                                  // every quarter reads the same 8 cells
      case 5: p[l] = (l * 37) % 29 * 3; break;                  // scattered
      case 6: p[l] = q == 0 ? i : (q == 1 ? 8 + i : 16 + i); break;  // quarters 0,1,2.. distinct rows, same slots
      case 7: p[l] = (i < 4 ? i : 8 + i) + 32 * q; break;       // within quarter: slots 0-3 row A, 4-7 row B (no conflict)
      case 8: p[l] = (i < 4 ? i : 8 + (i - 4)) + 32 * q; break; // within quarter: slots 0-3 twice, different rows (2-way)
      case 9: p[l] = (l & 1) ? 8 + (l / 2 % 8) : (l / 2 % 8); break;  // even/odd lanes different rows, same slots
      case 10: p[l] = l / 2; break;                             // 16 consecutive cells, lane pairs share
      case 11: p[l] = l / 4; break;                             // 8 consecutive cells, lane quads share
      case 12: p[l] = (l * 3) / 4; break;                       // 24 cells, slope 3/4 (backprojection row)
      case 13: p[l] = (l * 5) / 8; break;                       // 20 cells, slope 5/8
      case 14: p[l] = 2 * q + (i & 1); break;                   // quarters: 2 cells, lanes alternate
      case 15: p[l] = 8 * q + (i & 3); break;                   // quarters: 4 cells, same slots across quarters
      case 16: p[l] = 4 * q + (i & 3); break;                   // quarters: 4 cells, slots disjoint within a half
      case 17: p[l] = 2 * q + (i & 3); break;                   // quarters: 4 cells, overlapping with the neighbour quarter
      case 18: p[l] = 3 * q + (i % 3); break;                   // quarters: 3 cells
      case 19: p[l] = 8 * q + (i < 5 ? i : i - 5); break;       // quarters: 5 cells
      case 20: p[l] = q == 0 ? i : q == 1 ? 8 + (i & 1) : q == 2 ? 10 + (i & 1) : 16 + i; break;  // merge q1+q2?
      case 21: p[l] = 12 * q + (i & 3); break;                  // quarters: 4 cells, q1 slots 4-7 (cells 12-15)
      case 22: p[l] = 4 * h + (l & 3); break;                   // halves: 4 cells each (all lanes of a half)
      case 24: { const int qd = l >> 2, e = l & 3, b = (qd & 1) + 4 * ((qd >> 1) & 1) + 8 * (qd >> 2); p[l] = b + 2 * ((e == 1 || e == 2) ? 1 : 0); } break;  // quads {b, b+2}, halves conflict-free
      case 25: p[l] = (l >> 2) * 2 + ((l & 1) ? 16 : 0); break;  // quads {c, c+16}: same slot inside a quad
      case 26: { const int qd = l >> 2; p[l] = ((qd & 1) ? 8 : 0) + 2 * (qd >> 1) + (l & 1); } break;  // quads 2 cells; quads 0,1 same slots, different cells
      case 27: { const int qd = (l >> 2) & 3; p[l] = 2 * qd + (l & 1); } break;  // both halves read cells 0-7, quads 2 cells
      case 28: { const int qd = l >> 2; p[l] = 2 * qd + ((l & 3) == 3 ? 1 : 0); } break;  // quads {c,c,c,c+1}, 16 cells over the warp
      case 23: p[l] = (i & 3) + 4 * ((q + 1) & 1) + 16 * h; break;  // q0 slots 4-7, q1 slots 0-3
    }
  }
  int* d_p;
  float* d_out;
  cudaMalloc(&d_p, 32 * sizeof(int));
  cudaMalloc(&d_out, 148 * 256 * sizeof(float));
  cudaMemcpy(d_p, p.data(), 32 * sizeof(int), cudaMemcpyHostToDevice);
  probe<<<148, 256>>>(d_p, 1000, d_out);
  cudaDeviceSynchronize();
  printf("pattern %d:", which);
  for (int l = 0; l < 32; ++l) printf(" %d", p[l]);
  printf("\n");
  return 0;
}
